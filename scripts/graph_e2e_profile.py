import sys, time, cProfile, pstats
sys.path.insert(0, "/root/repo")
import torch
import paper_2210_15874_b200 as Q
g = Q.random_regular_graph(30, 3, seed=0)
be = Q.Backend.b200(dtype="complex64", profile=False)
for k in range(3):
    Q.qaoa_energy(g, Q.QaoaParams.seeded(4, 100 + k), be, cone="tight", balance_ranks=8)
torch.cuda.synchronize()
t = time.perf_counter()
for k in range(10):
    Q.qaoa_energy(g, Q.QaoaParams.seeded(4, 200 + k), be, cone="tight", balance_ranks=8)
print("per call ms", (time.perf_counter() - t) / 10 * 1e3)
pr = cProfile.Profile(); pr.enable()
for k in range(10):
    Q.qaoa_energy(g, Q.QaoaParams.seeded(4, 300 + k), be, cone="tight", balance_ranks=8)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
