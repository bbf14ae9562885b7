"""K2 stage items of the cfg-2 lightcone program with their live spans
(globaltimer stamps), sorted by start, and the consumers of each stage's
items: python scripts/k2_timeline.py [complex128|complex64]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "complex128"
g, params, lc, order = bench.build_workload()
tn = lc.network
t = E.plan_template([x.indices for x in tn.tensors], order, dtype, wave_aware=True)
prog = E.Program([E.Instance(t)], dtype)
ex = E.Executor(prog, timing=True)
raw = np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])
ex.stage_inputs([raw])
for _ in range(5):
    ex.launch()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush.zero_()
ex.launch()
torch.cuda.synchronize()
t0, t1 = ex.fetch_timing()
B = prog.buckets
node_of = prog.node_of_item()
out_of = {int(B[g_]["out_off"]): g_ for g_ in range(prog.n_buckets) if B[g_]["w"] >= 0}
consumer = {}
for g_ in range(prog.n_buckets):
    b = B[g_]
    for m in prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]:
        p_ = out_of.get(int(m["off"]))
        if p_ is not None:
            consumer[p_] = g_
origin = t0.min()
rows = []
for gid in range(prog.n_buckets):
    if int(prog.nodes[node_of[gid]]["kind"]) != 0:
        continue
    b = B[gid]
    c = consumer.get(gid, -1)
    rows.append(((t0[gid] - origin) / 1e3, (t1[gid] - origin) / 1e3, gid, int(b["w"]), int(b["k"]), int(b["n_tiles"]),
                 int(b["n_mem"]), node_of[gid], c, node_of.get(c, -1)))
rows.sort()
print("start_us end_us dur gid w k tiles nmem node consumer consumer_node")
for r in rows:
    print(f"{r[0]:7.1f} {r[1]:7.1f} {r[1]-r[0]:5.1f} {r[2]:4d} {r[3]:3d} {r[4]} {r[5]:4d} {r[6]} {r[7]:3d} {r[8]:4d} {r[9]:3d}")
