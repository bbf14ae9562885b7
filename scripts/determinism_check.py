"""Bitwise repeatability of program results (cfg-4 N=200 p=5 tight cones
sliced to 32, first --cones cones): every batch program launched 3 times;
prints units whose values differ between launches, and the values for a
cross-build comparison (QTN_K6=0 vs default)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import distributed as D  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cones", type=int, default=40)
ap.add_argument("--dtype", default="complex64")
ap.add_argument("--out", default="")
ap.add_argument("--poison", action="store_true", help="fill each arena with NaN before staging the inputs")
a = ap.parse_args()
g = Q.random_regular_graph(200, 3, seed=0)
c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(5, 0))
be = Q.Backend.b200(dtype=a.dtype, profile=False)
cones = [Q.extract_lightcone(c, e, cone="tight") for e in g.edges[: a.cones]]
plan = D.plan_units(cones, be, slice_target=32, mem_cap=1 << 40, n_workers=8)
free, _ = torch.cuda.mem_get_info()
vals, bad = {}, 0
for batch in D._batches(list(range(len(plan.units))), plan, be, int(0.5 * free)):
    insts = [E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch]
    ex = E.Executor(E.Program(insts, be.dtype), device=0, timing=False)
    if a.poison:
        ex.buf.fill_(float("nan"))
    ex.stage_inputs([plan.raws[plan.units[u].cone] for u in batch])
    runs = []
    for _ in range(3):
        ex.launch()
        runs.append(np.array(ex.fetch_results()).copy())
    for r in runs[1:]:
        d = np.nonzero(r != runs[0])[0]
        if len(d):
            bad += len(d)
            print("NONDETERMINISTIC units", [batch[k] for k in d[:8]], "kinds", ex.kernel_mix(), flush=True)
    for k, u in enumerate(batch):
        vals[u] = complex(runs[0][k])
        if not np.isfinite(runs[0][k]):
            print("NaN unit", u, "width", plan.templates[plan.units[u].cone].max_width, "kinds", ex.kernel_mix(), flush=True)
    del ex
    torch.cuda.empty_cache()
print(json.dumps({"units": len(vals), "nondeterministic": bad}))
if a.out:
    json.dump({str(u): [v.real, v.imag] for u, v in vals.items()}, open(a.out, "w"))
