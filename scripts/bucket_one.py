"""Run one cfg-5 bucket through K3 `reps` times (for ncu captures).
usage: python scripts/bucket_one.py w cls k [dtype] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2210_15874_b200 as Q  # noqa: E402
from paper_2210_15874_b200 import _native as N  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402
from paper_2210_15874_b200 import workloads as W  # noqa: E402

w, cls, k = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
dtype = sys.argv[4] if len(sys.argv) > 4 else "complex64"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
mem = W.synthetic_bucket_device(w, k, cls, 0, dtype)
b = Q.Bucket(W.BUCKET, [Q.DeviceTensor(i, t) for i, t in mem])
st = Q.tensor_core.bucket_strides(b, tuple(range(1, w + 1)))
out = torch.empty(1 << w, dtype=mem[0][1].dtype, device="cuda")
d = N.bucket_desc(E.DTYPE_CODE[dtype], w, out.data_ptr(), [(t.data_ptr(), x) for (_, t), x in zip(mem, st)])
print("plan", N.bucket_plan(d), "bytes", W.bucket_bytes(mem, w, E.ELEM_BYTES[dtype]))
for _ in range(reps):
    N.bucket_launch(d, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
