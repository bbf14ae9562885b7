"""cfg-5 synthetic bucket microbench sweep (BASELINE.json configs[4]): K3
(fused permutation-aware bucket kernel) achieved HBM GB/s vs result width,
class and member count.  Device-resident inputs, CUDA events around each
launch, L2 flushed between launches.

usage: python scripts/bucket_sweep.py [dtype] [wmin] [wmax] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import _native as N  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402
from paper_2210_15874_b200 import workloads as W  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "complex64"
wmin = int(sys.argv[2]) if len(sys.argv) > 2 else 8
wmax = int(sys.argv[3]) if len(sys.argv) > 3 else 28
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
cases = [(c[0], int(c[1:])) for c in sys.argv[5].split(",")] if len(sys.argv) > 5 else [("A", 3), ("A", 6), ("B", 2)]
tag = os.environ.get("SWEEP_TAG", "")
esz = E.ELEM_BYTES[dtype]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
rows = []
for w in range(wmin, wmax + 1, 2):
    for cls, k in cases:
        mem = W.synthetic_bucket_device(w, k, cls, 0, dtype)
        b = Q.Bucket(W.BUCKET, [Q.DeviceTensor(i, t) for i, t in mem])
        res = tuple(range(1, w + 1))
        st = Q.tensor_core.bucket_strides(b, res)
        out = torch.empty(1 << w, dtype=mem[0][1].dtype, device="cuda")
        d = N.bucket_desc(E.DTYPE_CODE[dtype], w, out.data_ptr(), [(t.data_ptr(), x) for (_, t), x in zip(mem, st)])
        plan = N.bucket_plan(d)
        nbytes = W.bucket_bytes(mem, w, esz)
        N.bucket_launch(d, s.cuda_stream)
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            N.bucket_launch(d, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        t = sorted(ts)[len(ts) // 2]
        row = {"tag": tag, "w": w, "cls": cls, "k": k, "ranks": [len(i) for i, _ in mem], "bytes": nbytes,
               "us": t * 1e6, "GBps": nbytes / t / 1e9, "tile_bits": plan[0], "smem": plan[2]}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del mem, b, out
        torch.cuda.empty_cache()
