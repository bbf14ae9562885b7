"""Full-energy runs of the heavy BASELINE configs on one GPU (or under
torchrun, sharded): cfg3 = N=30 p=3, REFERENCE cones sliced to width 30;
cfg4 = N=200 p=5, tight cones sliced to width 32.  Prints plan statistics,
device time, energy and (cfg3) the deviation from the golden energy."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import distributed as D  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", choices=["cfg3", "cfg3tight", "cfg4"])
ap.add_argument("--dtype", default="complex64")
ap.add_argument("--max-cones", type=int, default=0)
ap.add_argument("--repeat", type=int, default=2)
ap.add_argument("--api", action="store_true",
                help="time the public call qaoa_energy(...) end to end (planning, streamed batches, readback)")
a = ap.parse_args()
if a.config.startswith("cfg3"):
    n, p, cone, target, golden = 30, 3, ("reference" if a.config == "cfg3" else "tight"), 30, 26.219826685935914
else:
    n, p, cone, target, golden = 200, 5, "tight", 32, None
g = Q.random_regular_graph(n, 3, seed=0)
params = Q.QaoaParams.seeded(p, 0)
be = Q.Backend.b200(dtype=a.dtype, profile=False)
if a.api:
    for r in range(a.repeat):
        torch.cuda.synchronize()
        t = time.perf_counter()
        e = Q.qaoa_energy(g, params, be, mem_cap=1 << 40, n_workers=8, cone=cone, slice_target=target)
        wall = time.perf_counter() - t
        rec = {"config": a.config, "api": "qaoa_energy", "repeat": r, "wall_s": wall, "energy": e,
               "lightcones_per_s": g.n_edges / wall if hasattr(g, "n_edges") else len(g.edges) / wall}
        if golden is not None:
            rec["rel_err_vs_golden"] = abs(e - golden) / golden
        print(json.dumps(rec), flush=True)
    sys.exit(0)
t0 = time.perf_counter()
c = Q.qaoa_maxcut_circuit(g, params)
edges = g.edges[: a.max_cones] if a.max_cones else g.edges
cones = [Q.extract_lightcone(c, e, cone=cone) for e in edges]
plan = D.plan_units(cones, be, slice_target=target, mem_cap=1 << 40, n_workers=8)
t_plan = time.perf_counter() - t0
alg = sum(E.algorithmic_bytes(plan.templates[u.cone], a.dtype) for u in plan.units)
exe = sum(E.executed_bytes(plan.templates[u.cone], a.dtype) for u in plan.units)
widths = [t.max_width for t in plan.templates]
print(json.dumps({"config": a.config, "cones": len(cones), "units": len(plan.units), "max_width_after_slicing": max(widths),
                  "algorithmic_GB": alg / 1e9, "executed_GB": exe / 1e9, "host_plan_s": t_plan}), flush=True)
# batches sized to the free HBM; executed one after another (each batch's
# executor is freed before the next), device time = sum of graph launches
free, _ = torch.cuda.mem_get_info()
batches = list(D._batches(list(range(len(plan.units))), plan, be, int(0.7 * free)))
print(json.dumps({"batches": len(batches)}), flush=True)
for r in range(a.repeat):
    dt, t_host = 0.0, time.perf_counter()
    vals = {}
    for batch in batches:
        insts = [E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch]
        ex = E.Executor(E.Program(insts, be.dtype), device=0, timing=False)
        ex.stage_inputs([plan.raws[plan.units[u].cone] for u in batch])
        ex.graph   # build + instantiate the CUDA graph outside the timed region
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ex.launch()
        e1.record()
        res = ex.fetch_results()
        dt += e0.elapsed_time(e1) / 1e3
        for k, u in enumerate(batch):
            vals[u] = complex(res[k])
        del ex
        torch.cuda.empty_cache()
    zz = [0j] * len(cones)
    for u, unit in enumerate(plan.units):
        zz[unit.cone] += vals[u]
    energy = sum(0.5 * (1 - z.real) for z in zz)
    rec = {"repeat": r, "device_s": dt, "wall_s_incl_plan_build": time.perf_counter() - t_host, "energy": energy,
           "alg_GBps": alg / dt / 1e9, "exec_GBps": exe / dt / 1e9, "lightcones_per_s": len(cones) / dt}
    if golden is not None and not a.max_cones:
        rec["rel_err_vs_golden"] = abs(energy - golden) / golden
    print(json.dumps(rec), flush=True)
