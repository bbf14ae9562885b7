"""Kernel family chosen for every large item of a program, with the item's
shape (width, summed bits, member coverage): where the bytes go per family.
python scripts/route_report.py [graph|lightcone] [c64|c128]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "graph"
dtype = "complex128" if "c128" in sys.argv[2:] else "complex64"
if which == "graph":
    args = bench.parse(["--workload", "graph"])
    _, _, _, _, plan, prep, _ = bench.graph_setup(args, 0, 1, 0, dtype)
    exs = [ex for ex, _ in prep.batches]
else:
    g, params, lc, order = bench.build_workload()
    exs = [bench._Lightcone(lc, order, dtype, 0).ex]
per = collections.Counter()
rows = []
for ex in exs:
    prog = ex.prog
    fam = ex.node_kernels()
    node_of = prog.node_of_item()
    for gid in range(prog.n_buckets):
        b = prog.buckets[gid]
        f = fam[node_of[gid]]
        if f == "K2":
            continue
        w = int(b["w"])
        mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
        cover = sorted((bin(int(m["mask"]) & ((1 << w) - 1)).count("1") for m in mem), reverse=True)
        by = prog.item_bytes(gid)
        per[f] += by
        rows.append((by, f, w, int(b["k"]), cover))
print({k: f"{v / 1e9:.2f} GB" for k, v in per.items()})
for r in sorted(rows, reverse=True)[:30]:
    print(f"{r[0] / 1e6:8.1f} MB {r[1]} w{r[2]} k{r[3]} cover {r[4]}")
