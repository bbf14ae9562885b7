"""Isolated per-item timing: every device item of the cfg-2 lightcone program
run alone (dependencies dropped, arena filled with random data), CUDA events
over repeated launches.  Separates kernel efficiency from schedule overlap."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_15874_b200 import _native as N  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "complex64"
minw = int(sys.argv[2]) if len(sys.argv) > 2 else 12
only = int(sys.argv[3]) if len(sys.argv) > 3 else -1   # run one item (for ncu)
g, params, lc, order = bench.build_workload()
tn = lc.network
t = E.plan_template([x.indices for x in tn.tensors], order, dtype, wave_aware=True)
prog = E.Program([E.Instance(t)], dtype)
ex = E.Executor(prog, timing=False)
ex.arena.copy_(torch.randn(prog.arena_elems, dtype=ex.tdt, device="cuda") * 0.5)
esz = E.ELEM_BYTES[dtype]
lib = N.load()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tot = 0.0
print(" gid   w  k  L  tiles nmem stmask        MB     us    GB/s  variant")
for gid in range(prog.n_buckets):
    b = prog.buckets[gid].copy()
    if b["w"] < minw or (only >= 0 and gid != only):
        continue
    mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]].copy()
    by = ((1 << int(b["w"])) + sum(1 << (bin(int(m["smask"])).count("1") + bin(int(m["mask"])).count("1")) for m in mem)) * esz
    b["mem_begin"] = 0
    b["n_dep"] = 0
    b["dep_begin"] = 0
    b["tick_begin"] = 0
    blob = np.zeros(4096, np.uint8)
    blob[0:N.BUCKET_DT.itemsize] = np.frombuffer(b.tobytes(), np.uint8)
    blob[64:64 + mem.nbytes] = np.frombuffer(mem.tobytes(), np.uint8)
    tab = torch.from_numpy(blob).cuda()
    base = tab.data_ptr()
    c = N.ProgramC()
    c.dtype = E.DTYPE_CODE[dtype]
    c.n_buckets = 1
    c.n_nodes = 1
    c.buckets = base
    c.members = base + 64
    c.deps = base + 64
    c.tick_begin = base + 1024   # int32 0
    c.ctrl = base + 2048
    c.arena = ex.arena.data_ptr()
    c.results = ex.results.data_ptr()
    c.timing = None
    s = torch.cuda.current_stream()
    node = np.zeros(1, N.NODE_DT)
    small = int(b["w"]) >= 0 and (1 << int(b["tile_bits"])) < E.VEC[dtype] * E.NT
    var = [int(nd["variant"]) for nd in prog.nodes if nd["kind"] == N.QTN_NODE_LARGE and nd["first"] == gid]
    if small or not var:
        continue
    node[0] = (N.QTN_NODE_LARGE, 0, 1, 0, var[0], 0, 0, prog.smem_bytes)
    npt = node.ctypes.data_as(ctypes.c_void_p)
    for _ in range(3):
        N.check(lib.qtn_node_launch(ctypes.byref(c), npt, 0, ctypes.c_void_p(s.cuda_stream)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        flush.zero_()
        e0.record(s)
        N.check(lib.qtn_node_launch(ctypes.byref(c), npt, 0, ctypes.c_void_p(s.cuda_stream)))
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    tot += us
    print(f"{gid:4d} {int(b['w']):3d} {int(b['k']):2d} {int(b['tile_bits']):2d} {int(b['n_tiles']):6d} {int(b['n_mem']):4d} "
          f"{int(b['stmask']):012b} {by/1e6:8.1f} {us:7.1f} {by/us/1e3:7.0f}  {var[0]:#x}")
print(f"sum of isolated items (w >= {minw}): {tot:.1f} us")
