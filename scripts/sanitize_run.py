"""One small run of every code path for compute-sanitizer: cfg-1 cones, the
cfg-2 lightcone (c64 + c128), a few standalone buckets."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2210_15874_b200 as Q  # noqa: E402

g, params, lc, order = bench.build_workload()
for dt in ("complex64", "complex128"):
    v, _ = Q.contract_network(lc.network, order, Q.Backend.b200(dtype=dt, profile=False))
    print(dt, v)
g1 = Q.random_regular_graph(10, 3, 0)
print("cfg1", Q.qaoa_energy(g1, Q.QaoaParams.seeded(1, 0), Q.Backend.b200()))
rng = np.random.default_rng(1)
for w in (3, 9, 14):
    a = Q.Tensor(tuple(range(w + 1)), rng.standard_normal((2,) * (w + 1)) + 0j)
    b = Q.Tensor((0, 1, 2), rng.standard_normal((2, 2, 2)) + 0j)
    out, _ = Q.contract_bucket(Q.Bucket(0, [a, b]), Q.Backend.b200(dtype="complex64"))
    print("bucket", w, out.rank)
