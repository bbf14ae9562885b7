"""Where the end-to-end cfg-2 call spends its time beyond the device program:
contract_network loop vs Executor.run vs bare graph launches (+ sync)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import _native as N  # noqa: E402
from paper_2210_15874_b200 import ordering as O  # noqa: E402

g, params, lc, order = bench.build_workload()
tn = lc.network
be = Q.Backend.b200(dtype=sys.argv[1] if len(sys.argv) > 1 else "complex64", profile=False)
for _ in range(20):
    Q.contract_network(tn, order, be)
torch.cuda.synchronize()
struct, raw, plans = O.NETWORK_INPUTS.get(tn)
ex = [v for k, v in plans.items() if k[0] == "exec"][0][0]
lib = N.load()
s = torch.cuda.current_stream()
n = 300


def timeit(name, fn):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{name:48s} {(time.perf_counter() - t0) / n * 1e6:8.1f} us")


timeit("contract_network (public call)", lambda: Q.contract_network(tn, order, be))
nets = [bench.build_workload(seed=1 + k)[2].network for k in range(8)]
cyc = [0]


def new_angles():
    cyc[0] += 1
    return Q.contract_network(nets[cyc[0] % 8], order, be)


timeit("contract_network, new angles every call", new_angles)
timeit("Executor.run (stage + io graph + sync)", lambda: ex.run([raw]))
raws = [n_.packed()[2] for n_ in nets]
timeit("Executor.run, new inputs every call", lambda: ex.run([raws[(cyc.__setitem__(0, cyc[0] + 1) or cyc[0]) % 8]]))
gio = ex._io_graph([raw])[0].g
timeit("io graph (device gather) launch + stream sync", lambda: (N.check(lib.qtn_graph_launch(gio, ctypes.c_void_p(s.cuda_stream))),
                                                 s.synchronize()))
gk = ex.graph
timeit("kernel graph launch + stream sync", lambda: (N.check(lib.qtn_graph_launch(gk, ctypes.c_void_p(s.cuda_stream))),
                                                     s.synchronize()))
timeit("kernel graph launch, no sync (throughput)",
       lambda: N.check(lib.qtn_graph_launch(gk, ctypes.c_void_p(s.cuda_stream))))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(n):
    N.check(lib.qtn_graph_launch(gk, ctypes.c_void_p(s.cuda_stream)))
e1.record(s)
e1.synchronize()
print(f"{'kernel graph, device time per launch (events)':48s} {e0.elapsed_time(e1) / n * 1e3:8.1f} us")
