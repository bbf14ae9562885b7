"""One step of the 45-cone N=30 p=4 energy program (bench --workload graph's
batches), for ncu launch lists: python scripts/graph_step.py [c64|c128]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import distributed as D  # noqa: E402

dtype = "complex128" if "c128" in sys.argv[1:] else "complex64"
args = bench.parse(["--workload", "graph"])
g, params, be, cones, plan, prep, t_plan = bench.graph_setup(args, 0, 1, 0, dtype)
s = torch.cuda.current_stream()
D.launch_prepared(prep, s)
torch.cuda.synchronize()
vals = D.collect_prepared(prep, s)
energy = 0.0
zz = [0j] * len(cones)
for u, unit in enumerate(plan.units):
    zz[unit.cone] += vals[u]
print(f"batches={len(prep.batches)} nodes={sum(ex.prog.n_nodes for ex, _ in prep.batches)} "
      f"energy={sum(0.5 * (1 - z.real) for z in zz):.12f} "
      f"executed_GB={sum(ex.prog.executed_bytes() for ex, _ in prep.batches) / 1e9:.3f} "
      f"algorithmic_GB={sum(ex.prog.algorithmic_bytes() for ex, _ in prep.batches) / 1e9:.3f}")
