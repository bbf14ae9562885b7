"""K5 (csrc/bucket_stream.cu): streaming buckets — one member carries every
result bit — through the C ABI (qtn_bucket_stream), against a complex128
torch einsum of the same members (the reference's fast_kernel semantics,
src/tensor_core.py:148-164: product of the members, summed over the bucket
indices).  Members in the canonical layout (16-byte pair loads at
complex64) and in random axis orders (strided descriptors: scalar loads);
k = 1..3 summed indices, 1..4 loaded members, members without result bits."""
import numpy as np
import pytest

from paper_2210_15874_b200 import _native as N
from test_k4_expand import LETTERS


def _case(w, k, n_part, n_uniform, seed, permute):
    """Iteration bits 0..w-1 (result), w..w+k-1 (summed).  B: every result
    bit and the summed bits; `n_part` members with a random ~60 % of the
    result bits and random summed bits; `n_uniform` members with summed bits
    only."""
    rng = np.random.default_rng(seed)
    summ = list(range(w, w + k))
    mems = [list(range(w)) + summ]
    for _ in range(n_part):
        bits = [b for b in range(w) if rng.random() < 0.6] or [0]
        mems.append(bits + [s for s in summ if rng.random() < 0.6])
    for _ in range(n_uniform):
        mems.append([s for s in summ if rng.random() < 0.7] or [summ[0]])
    if permute:
        return [list(int(x) for x in rng.permutation(m)) for m in mems]
    # canonical: slowest axis first = highest bit first (summed bits slowest)
    return [sorted(m, reverse=True) for m in mems]


def _run(w, k, mems, dtype, seed):
    import torch
    cdt = torch.complex64 if dtype == "complex64" else torch.complex128
    rdt = torch.float32 if dtype == "complex64" else torch.float64
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    data = []
    for ids in mems:
        n = 1 << len(ids)
        x = torch.randn(2 * n, generator=gen, device="cuda", dtype=rdt) * (1.0 / np.sqrt(2.0))
        data.append(torch.view_as_complex(x.view(n, 2)).view(cdt))
    members = [(t.data_ptr(), {b: 1 << (len(ids) - 1 - ax) for ax, b in enumerate(ids)}) for ids, t in zip(mems, data)]
    out = torch.full((1 << w,), float("nan"), dtype=cdt, device="cuda")
    code = N.QTN_C64 if dtype == "complex64" else N.QTN_C128
    d = N.bucket_desc(code, w, out.data_ptr(), members, k=k)
    N.bucket_stream_launch(d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    ops = [t.to(torch.complex128).view((2,) * len(ids)) for ids, t in zip(mems, data)]
    subs = ",".join("".join(LETTERS[b] for b in ids) for ids in mems)
    ref = torch.einsum(subs + "->" + "".join(LETTERS[b] for b in reversed(range(w))), *ops).reshape(-1)
    return out.to(torch.complex128), ref


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("permute", [False, True])
@pytest.mark.parametrize("w,k,n_part,n_uniform", [(9, 1, 0, 0), (10, 1, 1, 1), (13, 2, 1, 2), (16, 2, 2, 0),
                                                  (18, 3, 3, 1), (20, 1, 0, 2), (21, 3, 1, 3), (22, 2, 2, 2)])
def test_k5_vs_einsum(dtype, permute, w, k, n_part, n_uniform):
    mems = _case(w, k, n_part, n_uniform, seed=w * 100 + k * 10 + n_part, permute=permute)
    out, ref = _run(w, k, mems, dtype, seed=w + k + n_part)
    tol = 1e-5 if dtype == "complex64" else 1e-12
    assert not out.isnan().any()
    err = (out - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err


@pytest.mark.gpu
def test_k5_rejects_non_streaming():
    """No member carries every result bit; too many loaded members."""
    import torch
    x = torch.zeros(1 << 17, dtype=torch.complex64, device="cuda")
    out = torch.zeros(1 << 16, dtype=torch.complex64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    a = {b: 1 << i for i, b in enumerate(list(range(15)) + [16])}
    d = N.bucket_desc(N.QTN_C64, 16, out.data_ptr(), [(x.data_ptr(), a), (x.data_ptr(), {15: 1, 16: 2})], k=1)
    with pytest.raises(N.NativeError, match="every result bit"):
        N.bucket_stream_launch(d, s)
    full = {b: 1 << b for b in range(17)}
    part = {b: 1 << i for i, b in enumerate([0, 16])}
    d = N.bucket_desc(N.QTN_C64, 16, out.data_ptr(), [(x.data_ptr(), full)] + [(x.data_ptr(), part)] * 4, k=1)
    with pytest.raises(N.NativeError, match="carry result bits"):
        N.bucket_stream_launch(d, s)
    torch.cuda.synchronize()
