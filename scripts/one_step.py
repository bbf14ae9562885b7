"""Exactly one launch of the cfg-2 lightcone program (for ncu launch lists),
or — with `--dominant` / `--item G` — the program once outside the profiled
range, then its dominant node / the node of item G alone inside
cudaProfilerStart/Stop (for `ncu --profile-from-start off --set full`).

    python scripts/one_step.py [c128|c64] [--dominant | --item G]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dtype = "complex64" if "c64" in sys.argv[1:] else "complex128"
g, params, lc, order = bench.build_workload()
lcp = bench._Lightcone(lc, order, dtype, 0)
s = torch.cuda.current_stream()
if "--dominant" in sys.argv or "--item" in sys.argv:
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    dom = bench.dominant_kernel(lcp, s, flush, reps=3)
    if "--item" in sys.argv:
        g_ = int(sys.argv[sys.argv.index("--item") + 1])
        b_ = lcp.prog.buckets[g_]
        dom.update(item=g_, w=int(b_["w"]), k=int(b_["k"]), bytes=lcp.prog.item_bytes(g_), key="-", us=0.0)
    node = lcp.prog.node_of_item()[dom["item"]]
    gr, fam = lcp.ex.node_graph(node)
    lcp.ex.launch(s)
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    lcp.ex.launch_graph(gr, s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"dominant item {dom['item']} node {node} {fam} w={dom['w']} k={dom['k']} bytes={dom['bytes']} "
          f"key={dom['key']} alone={dom['us']:.1f} us")
else:
    lcp.ex.launch(s)
    torch.cuda.synchronize()
    print(f"nodes={lcp.prog.n_nodes} kernels={sum(lcp.ex.kernel_mix(io=False).values())} zz={complex(*lcp.ex.results[:2].cpu().numpy()).real:.15e}")
