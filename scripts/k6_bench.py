"""K6 pair nodes of the cfg-2 lightcone program timed alone (node graph, L2
flushed before every launch, CUDA events) and the whole program step:
`python scripts/k6_bench.py [c64|c128]`.  Set QTN_LIB for a variant build."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402


def timed(fn, flush, reps=30):
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts))


for dtype in [d for d in ("complex128", "complex64") if not sys.argv[1:] or d[7:] in "".join(sys.argv[1:])]:
    g, params, lc, order = bench.build_workload()
    lcp = bench._Lightcone(lc, order, dtype, 0)
    ex, prog = lcp.ex, lcp.prog
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ex.launch(s)
    torch.cuda.synchronize()
    zz = complex(*ex.results[:2].cpu().numpy()).real
    step = timed(lambda: ex.launch(s), flush)
    fams = ex.node_kernels()
    out = [f"{dtype}: step {step:.1f} us zz {zz:.15e} mix {ex.kernel_mix()}"]
    for ni, nd in enumerate(prog.nodes):
        if nd["kind"] != 1:
            continue
        gr, fam = ex.node_graph(ni)
        us = timed(lambda: ex.launch_graph(gr, s), flush)
        ws = [int(prog.buckets[g_]["w"]) for g_ in range(nd["first"], nd["first"] + nd["count"])]
        if us > 5 or nd["count"] == 2:
            out.append(f"   node {ni:2d} {fam} items {list(range(nd['first'], nd['first'] + nd['count']))} w {ws}: {us:.1f} us")
    print("\n".join(out), flush=True)
