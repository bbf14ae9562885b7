"""K4 (csrc/bucket_expand.cu): expansion buckets — one dominant member that
lacks 1..4 result bits, the others small — through the C ABI
(qtn_bucket_expand), against a complex128 torch einsum of the same members
(the reference's fast_kernel semantics, src/tensor_core.py:148-164: product of
the members, summed over the bucket indices).  Members arrive in random axis
orders (strided descriptors); k = 1..3 summed indices (merged chains)."""
import numpy as np
import pytest

from paper_2210_15874_b200 import _native as N

LETTERS = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"


def _case(w, k, ne, n_small, seed, in_tile_extra=1, big_lacks_s=False):
    """Iteration bits 0..w-1 (result), w..w+k-1 (summed).  Dominant member:
    every result bit but the expansion bits E (chosen among bits 1..w-1) and
    the summed bits; small members: E split among them, plus a few other
    result bits (in_tile_extra of them among bits 0..7) and random summed
    bits."""
    rng = np.random.default_rng(seed)
    E = sorted(int(x) for x in rng.choice(np.arange(1, w), size=ne, replace=False))
    summ = list(range(w, w + k))
    big = [b for b in range(w) if b not in E] + (summ[1:] if big_lacks_s else summ)
    smalls = [[] for _ in range(n_small)]
    for e in E:
        smalls[int(rng.integers(n_small))].append(e)
    low = [b for b in range(8) if b not in E]
    high = [b for b in range(12, w) if b not in E]
    for j in range(n_small):
        for b in rng.choice(low, size=min(in_tile_extra, len(low)), replace=False):
            if int(b) not in smalls[j]:
                smalls[j].append(int(b))
        if high:
            b = int(rng.choice(high))
            if b not in smalls[j]:
                smalls[j].append(b)
        smalls[j] += [s for s in summ if rng.random() < 0.6]
    if big_lacks_s and summ[0] not in smalls[0]:
        smalls[0].append(summ[0])
    mems = [big] + smalls
    return [list(int(x) for x in rng.permutation(m)) for m in mems]


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
    # member axis ax (C order: last axis fastest) carries iteration bit ids[ax]
    members = [(t.data_ptr(), {b: 1 << (len(ids) - 1 - ax) for ax, b in enumerate(ids)}) for ids, t in zip(mems, data)]
    out = torch.full((1 << w,), float("nan"), dtype=cdt, device="cuda")
    code = N.QTN_C64 if dtype == "complex64" else N.QTN_C128
    d = N.bucket_desc(code, w, out.data_ptr(), members, k=k)
    N.bucket_expand_launch(d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    # einsum: letter per iteration bit; output axes = result bits w-1 .. 0 (bit 0 fastest)
    ops = [t.to(torch.complex128).view((2,) * len(ids)) for ids, t in zip(mems, data)]
    subs = ",".join("".join(LETTERS[b] for b in ids) for ids in mems)
    ref = torch.einsum(subs + "->" + "".join(LETTERS[b] for b in reversed(range(w))), *ops).reshape(-1)
    return out.to(torch.complex128), ref


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("w,k,ne,n_small", [(12, 1, 1, 1), (13, 2, 2, 2), (16, 2, 4, 3), (18, 3, 3, 2), (16, 1, 4, 4),
                                            (20, 2, 1, 3), (14, 3, 2, 5), (22, 2, 4, 2), (20, 1, 5, 2), (20, 2, 6, 3),
                                            (21, 1, 7, 2), (22, 1, 8, 2)])
def test_k4_vs_einsum(dtype, w, k, ne, n_small):
    mems = _case(w, k, ne, n_small, seed=w * 100 + k * 10 + ne)
    out, ref = _run(w, k, mems, dtype, seed=w + k + ne)
    tol = 1e-5 if dtype == "complex64" else 1e-12
    assert not out.isnan().any()
    err = (out - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_k4_dominant_member_without_a_summed_index(dtype):
    """The dominant member need not carry every summed index (merged chains)."""
    mems = _case(16, 2, 3, 2, seed=5, big_lacks_s=True)
    out, ref = _run(16, 2, mems, dtype, seed=5)
    tol = 1e-5 if dtype == "complex64" else 1e-12
    assert (out - ref).abs().max().item() <= tol * max(1.0, ref.abs().max().item())


@pytest.mark.gpu
def test_k4_rejects_non_expansions():
    """More than 4 expansion bits, too few dominant bits, min_e not met."""
    import torch
    x = torch.zeros(1 << 17, dtype=torch.complex64, device="cuda")
    out = torch.zeros(1 << 16, dtype=torch.complex64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    # dominant member lacks 9 result bits (K4 takes at most 8)
    x = torch.zeros(1 << 20, dtype=torch.complex64, device="cuda")
    out = torch.zeros(1 << 18, dtype=torch.complex64, device="cuda")
    big = {b: 1 << i for i, b in enumerate([0, 1, 2, 3, 4, 5, 6, 7, 8] + [18])}
    small = {b: 1 << i for i, b in enumerate([9, 10, 11, 12, 13, 14, 15, 16, 17, 18])}
    d = N.bucket_desc(N.QTN_C64, 18, out.data_ptr(), [(x.data_ptr(), big), (x.data_ptr(), small)], k=1)
    with pytest.raises(N.NativeError, match="expansion bits"):
        N.bucket_expand_launch(d, s)
    out = torch.zeros(1 << 16, dtype=torch.complex64, device="cuda")
    # no expansion bit but min_e = 1
    full = {b: 1 << b for b in range(17)}
    d = N.bucket_desc(N.QTN_C64, 16, out.data_ptr(), [(x.data_ptr(), full)], k=1)
    with pytest.raises(N.NativeError, match="expansion bits"):
        N.bucket_expand_launch(d, s, min_e=1)
    N.bucket_expand_launch(d, s, min_e=0)   # allowed: plain streaming bucket
    torch.cuda.synchronize()
