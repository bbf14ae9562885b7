"""K6 (csrc/bucket_expand.cu): an expansion bucket fused with the only bucket
that reads it — the consumer's member is the producer's whole result, its
summed indices the producer's slowest result axes — through the C ABI
(qtn_bucket_expand_fused), against complex128 torch einsums of the two
buckets one after the other (the reference's contract_bucket twice,
src/tensor_core.py:148-188: the producer's result re-bucketed and contracted
by the consumer, src/ordering.py:175-187).  The producer's output buffer must
stay untouched: K6 never materialises it."""
import numpy as np
import pytest

from paper_2210_15874_b200 import _native as N
from test_k4_expand import LETTERS, _case


def _rand(n, gen, rdt, cdt):
    import torch
    x = torch.randn(2 * n, generator=gen, device="cuda", dtype=rdt) * (1.0 / np.sqrt(2.0))
    return torch.view_as_complex(x.view(n, 2)).view(cdt)


def _run_pair(wc, kc, kp, ne, n_small, n_gather, n_uniform, dtype, seed):
    import torch
    cdt = torch.complex64 if dtype == "complex64" else torch.complex128
    rdt = torch.float32 if dtype == "complex64" else torch.float64
    code = N.QTN_C64 if dtype == "complex64" else N.QTN_C128
    wp = wc + kc
    rng = np.random.default_rng(seed)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    # producer: iteration bits 0..wp-1 result, wp..wp+kp-1 summed
    pm = _case(wp, kp, ne, n_small, seed)
    pdata = [_rand(1 << len(ids), gen, rdt, cdt) for ids in pm]
    pmem = [(t.data_ptr(), {b: 1 << (len(ids) - 1 - ax) for ax, b in enumerate(ids)}) for ids, t in zip(pm, pdata)]
    pout = torch.full((1 << wp,), float("nan"), dtype=cdt, device="cuda")
    dp = N.bucket_desc(code, wp, pout.data_ptr(), pmem, k=kp)
    # consumer: bits 0..wc-1 result, wc..wc+kc-1 summed; member 0 = the
    # producer's result (consumer bit b = producer bit b); gathered members
    # over random result bits (+ summed bits), uniform members on summed bits
    cm = []
    for _ in range(n_gather):
        ids = sorted(int(x) for x in rng.choice(wc, size=min(wc - 2, int(rng.integers(2, 12))), replace=False))
        ids += [wc + q for q in range(kc) if rng.random() < 0.6]
        cm.append([int(x) for x in rng.permutation(ids)])
    for _ in range(n_uniform):
        cm.append([wc + q for q in range(kc) if rng.random() < 0.7] or [wc])
    cdata = [_rand(1 << len(ids), gen, rdt, cdt) for ids in cm]
    cmem = [(pout.data_ptr(), {b: 1 << b for b in range(wp)})]
    cmem += [(t.data_ptr(), {b: 1 << (len(ids) - 1 - ax) for ax, b in enumerate(ids)}) for ids, t in zip(cm, cdata)]
    cout = torch.full((1 << wc,), float("nan"), dtype=cdt, device="cuda")
    dc = N.bucket_desc(code, wc, cout.data_ptr(), cmem, k=kc)
    N.bucket_expand_fused_launch(dp, dc, 0, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert pout.isnan().all(), "K6 wrote the producer's result"
    # reference: producer einsum, then consumer einsum (complex128)
    ops = [t.to(torch.complex128).view((2,) * len(ids)) for ids, t in zip(pm, pdata)]
    subs = ",".join("".join(LETTERS[b] for b in ids) for ids in pm)
    x = torch.einsum(subs + "->" + "".join(LETTERS[b] for b in reversed(range(wp))), *ops)
    ops = [x] + [t.to(torch.complex128).view((2,) * len(ids)) for ids, t in zip(cm, cdata)]
    subs = ",".join(["".join(LETTERS[b] for b in reversed(range(wp)))] +
                    ["".join(LETTERS[b] for b in ids) for ids in cm])
    ref = torch.einsum(subs + "->" + "".join(LETTERS[b] for b in reversed(range(wc))), *ops).reshape(-1)
    return cout.to(torch.complex128), ref


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
@pytest.mark.parametrize("wc,kc,kp,ne,n_small,n_gather,n_uniform", [
    (12, 1, 1, 1, 1, 0, 0), (14, 2, 2, 2, 2, 1, 2), (16, 2, 2, 4, 3, 1, 1), (15, 1, 3, 3, 2, 1, 0),
    (18, 2, 1, 4, 2, 1, 1), (20, 2, 2, 4, 2, 1, 2), (19, 3, 1, 2, 2, 1, 1), (20, 1, 2, 6, 3, 1, 1),
    (13, 3, 2, 0, 1, 0, 3)])
def test_k6_vs_two_einsums(dtype, wc, kc, kp, ne, n_small, n_gather, n_uniform):
    if (1 << kc) * (1 << kp) > 16:
        pytest.skip("K6 holds at most 16 B values per thread")
    out, ref = _run_pair(wc, kc, kp, ne, n_small, n_gather, n_uniform, dtype, seed=wc * 100 + kc * 10 + kp)
    assert not out.isnan().any()
    tol = 1e-5 if dtype == "complex64" else 1e-12
    err = (out - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err


@pytest.mark.gpu
def test_k6_rejects_other_shapes():
    """The consumer member must be the producer's whole result in order; at
    most 2^kc * 2^kp = 16 B registers per thread; at most one consumer member
    carries result bits."""
    import torch
    s = torch.cuda.current_stream().cuda_stream
    x = torch.zeros(1 << 16, dtype=torch.complex128, device="cuda")
    pout = torch.zeros(1 << 14, dtype=torch.complex128, device="cuda")
    cout = torch.zeros(1 << 12, dtype=torch.complex128, device="cuda")
    dp = N.bucket_desc(N.QTN_C128, 14, pout.data_ptr(), [(x.data_ptr(), {b: 1 << b for b in range(16)})], k=2)
    perm = {b: 1 << b for b in range(14)}
    perm[0], perm[1] = 2, 1   # axes 0 and 1 swapped: not the canonical result
    dc = N.bucket_desc(N.QTN_C128, 12, cout.data_ptr(), [(pout.data_ptr(), perm)], k=2)
    with pytest.raises(N.NativeError, match="whole producer result"):
        N.bucket_expand_fused_launch(dp, dc, 0, s)
    x = torch.zeros(1 << 17, dtype=torch.complex128, device="cuda")
    dp3 = N.bucket_desc(N.QTN_C128, 14, pout.data_ptr(), [(x.data_ptr(), {b: 1 << b for b in range(17)})], k=3)
    dc = N.bucket_desc(N.QTN_C128, 12, cout.data_ptr(), [(pout.data_ptr(), {b: 1 << b for b in range(14)})], k=2)
    with pytest.raises(N.NativeError, match="registers"):
        N.bucket_expand_fused_launch(dp3, dc, 0, s)
    x = torch.zeros(1 << 16, dtype=torch.complex128, device="cuda")
    g = {b: 1 << i for i, b in enumerate(range(4))}
    dp = N.bucket_desc(N.QTN_C128, 14, pout.data_ptr(), [(x.data_ptr(), {b: 1 << b for b in range(16)})], k=2)
    dc = N.bucket_desc(N.QTN_C128, 12, cout.data_ptr(), [(pout.data_ptr(), {b: 1 << b for b in range(14)}),
                                                          (x.data_ptr(), g), (x.data_ptr(), g)], k=2)
    with pytest.raises(N.NativeError, match="more than one consumer member"):
        N.bucket_expand_fused_launch(dp, dc, 0, s)
    torch.cuda.synchronize()
