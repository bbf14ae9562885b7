"""Per-bucket device timeline of the cfg-2 lightcone program (globaltimer
stamps recorded by the program kernel): where the 0.x ms go."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "complex64"
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
esz = E.ELEM_BYTES[dtype]
B = prog.buckets
origin = t0.min()
rows = []
for gid in range(prog.n_buckets):
    b = B[gid]
    if b["w"] < 0:
        continue
    mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
    by = (1 << int(b["w"])) + sum(1 << (bin(int(m["smask"])).count("1") + bin(int(m["mask"])).count("1")) for m in mem)
    rows.append((t0[gid] - origin, t1[gid] - origin, int(b["w"]), int(b["tile_bits"]), int(b["n_tiles"]),
                 int(b["n_mem"]), by * esz, int(b["k"])))
rows.sort()
tot = t1.max() - origin
print(f"total {tot/1e3:.1f} us, buckets {len(rows)}")
small = [r for r in rows if r[2] < 12]
print(f"small (w<12): {len(small)} buckets, span {max(r[1] for r in small)/1e3:.1f} us")
print(f"algorithmic {prog.algorithmic_bytes()/1e9:.3f} GB, executed {prog.executed_bytes()/1e9:.3f} GB, {prog.describe()}")
print(" start_us   end_us   dur_us  w  k  L  tiles nmem   MB    GB/s")
for r in rows:
    if r[2] >= 12 or r[7] > 1:
        d = r[1] - r[0]
        print(f"{r[0]/1e3:8.1f} {r[1]/1e3:8.1f} {d/1e3:8.1f} {r[2]:2d} {r[7]:2d} {r[3]:2d} {r[4]:6d} {r[5]:3d} {r[6]/1e6:7.1f} {r[6]/max(d,1):7.0f}")

# ---- critical path: walk back from the last-finishing item through the
# producer that finished last ----
gid_rows = {}
for gid in range(prog.n_buckets):
    gid_rows[gid] = (t0[gid] - origin, t1[gid] - origin)
node_of = {}
for ni, nd in enumerate(prog.nodes):
    for gg in range(int(nd["first"]), int(nd["first"]) + int(nd["count"])):
        node_of[gg] = (ni, int(nd["kind"]), int(nd["variant"]))
# producers per item (global ids) from the member offsets
out_of = {}
for gid in range(prog.n_buckets):
    b = B[gid]
    if b["w"] >= 0:
        out_of[int(b["out_off"])] = gid
def producers(gid):
    b = B[gid]
    mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
    return [out_of[int(m["off"])] for m in mem if int(m["off"]) in out_of]
cur = max(gid_rows, key=lambda g: gid_rows[g][1])
path = []
while cur is not None:
    path.append(cur)
    ps = producers(cur)
    cur = max(ps, key=lambda g: gid_rows[g][1]) if ps else None
fam = ex.node_kernels(io=False)   # the kernel family the graph actually runs per node
print("critical path (first -> last): start end dur | w k L tiles nmem | node kernel variant")
for gid in reversed(path):
    b = B[gid]
    s_, e_ = gid_rows[gid]
    ni, kind, var = node_of[gid]
    print(f"  {s_/1e3:7.1f} {e_/1e3:7.1f} {(e_-s_)/1e3:6.1f} | {int(b['w']):3d} {int(b['k'])} {int(b['tile_bits']):2d} "
          f"{int(b['n_tiles']):5d} {int(b['n_mem'])} | node {ni:3d} {fam[ni]} {var:#x}")
