"""Device time of single-contraction (wave-aware) programs over many cones of
the N=30 p=4 graph: checks that a planner constant tuned on cfg-2's cone
(edge (0,15)) generalises.  Env QTN_HOP_SINGLE_C64_S / _C128_S are read at
import, so run one process per value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "complex64"
g = Q.random_regular_graph(30, 3, seed=0)
c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(4, 0))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tot, n = 0.0, 0
rows = []
for e in g.edges:
    lc = Q.extract_lightcone(c, e, cone="tight")
    tn = lc.network
    order = Q.greedy_order(tn)
    w = Q.dry_run(tn, order).contraction_width
    if w < 20:
        continue
    t = E.plan_template([x.indices for x in tn.tensors], order, dtype, wave_aware=True)
    ex = E.Executor(E.Program([E.Instance(t)], dtype))
    ex.stage_inputs([np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])])
    s = torch.cuda.current_stream()
    for _ in range(3):
        ex.launch(s)
    ms = 0.0
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        ex.launch(s)
        b.record(s)
        b.synchronize()
        ms += a.elapsed_time(b)
    rows.append((e, w, ms / 20))
    tot += ms / 20
    n += 1
    del ex
print(f"{dtype} cones(w>=20)={n} total_ms={tot:.4f} " + " ".join(f"{e[0]}-{e[1]}:{w}:{t:.3f}" for e, w, t in rows))
