for L in default pf; do
  if [ $L = default ]; then unset QTN_LIB; else export QTN_LIB=$PWD/paper_2210_15874_b200/lib/libqtn_b200_$L.so; fi
  for d in c64 c128; do
    python scripts/ab_time.py $d
    python scripts/one_step.py $d --dominant | tail -1
  done
done
