"""The reference-side bindings INTEGRATION.md §2 shows a maintainer adding
to `qtnsim` (kept here verbatim so tests exercise them; test infrastructure)."""
import numpy as np
import torch

from paper_2210_15874_b200 import _native as N
from paper_2210_15874_b200 import engine as E

_cache = {}


def contract_network_b200(tn, order, dtype="complex128", device=0):
    key = (tuple(t.indices for t in tn.tensors), tuple(order), dtype)
    ex = _cache.get(key)
    if ex is None:                                       # plan once per structure
        tmpl = E.plan_template([t.indices for t in tn.tensors], order, dtype)
        ex = _cache[key] = E.Executor(E.Program([E.Instance(tmpl)], dtype), device=device)
    raw = np.concatenate([t.data.ravel() for t in tn.tensors])
    return complex(ex.run([raw])[0])                     # get-result scalar


def contract_bucket_b200(b, dtype=N.QTN_C128):
    res = sorted(set().union(*[set(t.indices) for t in b.tensors]) - {b.bucket_index})
    bit = {a: len(res) - 1 - j for j, a in enumerate(res)}
    bit[b.bucket_index] = len(res)
    dev = [torch.from_numpy(np.ascontiguousarray(t.data).ravel().copy()).cuda() for t in b.tensors]
    out = torch.empty(1 << len(res), dtype=torch.complex128, device="cuda")
    members = [(d.data_ptr(), {bit[a]: 1 << (t.rank - 1 - ax) for ax, a in enumerate(t.indices)})
               for t, d in zip(b.tensors, dev)]
    desc = N.bucket_desc(dtype, len(res), out.data_ptr(), members)
    N.bucket_launch(desc, torch.cuda.current_stream().cuda_stream)
    return tuple(res), out.cpu().numpy().reshape((2,) * len(res))
