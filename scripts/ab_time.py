"""A/B timing of the cfg-2 lightcone program (kernels-only graph, L2
flushed, CUDA events): `python scripts/ab_time.py [c64|c128] [--no-hi]`.
Set QTN_LIB to time a variant build of the library."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

dtype = "complex128" if "c128" in sys.argv else "complex64"
g, params, lc, order = bench.build_workload()
tn = lc.network
t = E.plan_template([x.indices for x in tn.tensors], order, dtype, wave_aware=True)
prog = E.Program([E.Instance(t)], dtype)
if "--no-hi-buf" in sys.argv:
    prog.device_elems -= prog.hi_elems
    prog.hi_elems = 0
ex = E.Executor(prog, timing=False)
if "--no-hi" in sys.argv:
    ex.c.inputs_hi = None
    ex.c.n_in_elems = 0
raw = np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])
ex.stage_inputs([raw])
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    ex.launch(s)
ts = []
for _ in range(200):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    ex.launch(s)
    b.record(s)
    b.synchronize()
    ts.append(a.elapsed_time(b))
v = ex.fetch_results()[0]
print(f"{os.path.basename(os.environ.get('QTN_LIB', 'default'))} {dtype} {' '.join(sys.argv[1:])}: "
      f"median {np.median(ts) * 1e3:.1f} us  min {min(ts) * 1e3:.1f} us  zz {v.real:.12e} "
      f"rel {abs(v.real + 0.0017371891851279) / 0.0017371891851279:.2e}")
