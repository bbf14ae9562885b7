# fresh ncu --set full captures of the dominant cfg-2 node (K6 pair) at both element types
for d in ${DTYPES:-c128 c64}; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/k6_dom_$d -f python scripts/one_step.py $d --dominant > gpurun_out/k6_ncu_$d.log 2>&1
  echo "$d ncu rc=$?"
done
