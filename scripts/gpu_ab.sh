# A/B: default library vs the variant builds named in $VARIANTS, and environment settings named in
# $ENVS (comma-separated "NAME=V" sets, "-" = none) — scripts/ab_time.py, L2 flushed
for i in 1 2 3; do for v in default $VARIANTS; do for en in ${ENVS:--}; do for d in c128 c64; do
  lib=""; [ $v != default ] && lib="QTN_LIB=$PWD/paper_2210_15874_b200/lib/libqtn_b200_$v.so"
  envs=""; [ "$en" != "-" ] && envs=$(echo $en | tr ',' ' ')
  echo -n "[$en] "; env $lib $envs timeout 120 python scripts/ab_time.py $d
done; done; done; done > gpurun_out/ab.txt 2>&1
sort gpurun_out/ab.txt
