set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_c128.json 2> gpurun_out/bench_c128.err
timeout 600 python bench.py --dtype c64 > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/nodes_c128.csv python scripts/one_step.py c128 > gpurun_out/one_step_c128.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/nodes_c64.csv python scripts/one_step.py c64 > gpurun_out/one_step_c64.log 2>&1
tail -3 gpurun_out/gputest.log; cat gpurun_out/bench_c128.json | head -c 1500
