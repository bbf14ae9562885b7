"""Sweep the per-unit latency charge of the LPT cost model (distributed.UNIT_LATENCY_BYTES)
on the 45-cone N=30 p=4 energy: one-GPU step time and the per-rank shares timed alone
(bench.rank_shares) at 4 and 8 ranks.  Usage: python scripts/lpt_latency_sweep.py [c64|c128]"""
import json
import os
import sys
import types

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2210_15874_b200 import distributed as D

dt = sys.argv[1] if len(sys.argv) > 1 else "c128"
dtype = "complex64" if dt == "c64" else "complex128"
args = types.SimpleNamespace(simplify=False, steps=10, no_shares=True)
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for lat in (0, 250_000_000, 500_000_000, 1_000_000_000, 2_000_000_000, 4_000_000_000):
    D.UNIT_LATENCY_BYTES = lat
    g, params, be, cones, plan, prep, t_plan = bench.graph_setup(args, 0, 1, 0, dtype)
    del prep
    sh = bench.rank_shares(plan, be, 0, stream, flush, ns=(1, 4, 8))
    print(json.dumps({"dtype": dt, "unit_latency_bytes": lat, "units": len(plan.units),
                      "ms": {n: v["makespan_ms"] for n, v in sh.items()},
                      "ranks8_ms": [r["ms"] for r in sh["8"]["ranks"]]}), flush=True)
