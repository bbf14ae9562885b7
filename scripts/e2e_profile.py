import sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
import bench
import paper_2210_15874_b200 as Q
g, params, lc, order = bench.build_workload()
tn = lc.network
be = Q.Backend.b200(dtype="complex64", profile=False)
for _ in range(20):
    Q.contract_network(tn, order, be)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    Q.contract_network(tn, order, be)
t1 = time.perf_counter()
print("e2e us", (t1 - t0) / n * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    Q.contract_network(tn, order, be)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
