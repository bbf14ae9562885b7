# refresh of the secondary evidence: per-item timelines and the full-graph (45-cone) bench lines
timeout 200 python scripts/bucket_timeline.py complex128 > gpurun_out/timeline_c128.txt 2>&1
timeout 200 python scripts/bucket_timeline.py complex64 > gpurun_out/timeline_c64.txt 2>&1
timeout 900 python bench.py --workload graph --dtype c64 > gpurun_out/bench_graph_c64.json 2> gpurun_out/bench_graph_c64.err
timeout 900 python bench.py --workload graph --dtype c128 > gpurun_out/bench_graph_c128.json 2> gpurun_out/bench_graph_c128.err
timeout 600 python bench.py --workload bucket --dtype c64 > gpurun_out/bench_bucket_c64.json 2> gpurun_out/bench_bucket_c64.err
head -2 gpurun_out/timeline_c128.txt; tail -c 300 gpurun_out/bench_graph_c64.json
