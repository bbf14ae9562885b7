# the driver's N>1 launch shape on the one GPU this pool gives: torchrun with one rank (NCCL
# communicator, barrier, max-over-ranks all-reduce on the device) for both arms
set -x
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/torchrun_c128.json 2> gpurun_out/torchrun_c128.err; echo "rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 0 > gpurun_out/torchrun_ref.json 2> gpurun_out/torchrun_ref.err; echo "rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --workload graph --gpus 1 > gpurun_out/torchrun_graph.json 2> gpurun_out/torchrun_graph.err; echo "rc=$?"
tail -c 400 gpurun_out/torchrun_c128.json; tail -5 gpurun_out/torchrun_c128.err
