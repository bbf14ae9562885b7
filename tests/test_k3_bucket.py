"""K3 — the fused permutation-aware bucket kernel (csrc/bucket_strided.cu)
behind contract_bucket (src/tensor_core.py:167-188), on the cfg-5 synthetic
buckets.  CPU tests cover the host planner through the C ABI
(qtn_bucket_plan needs no device); GPU tests compare with the oracle
(numpy restatement of fast_kernel, src/tensor_core.py:148-164) at complex128
(1e-12 abs per element) / complex64 (1e-5 relative to the result scale), and
at large widths with a torch complex128 einsum of the same bucket."""
import numpy as np
import pytest

from oracle import qtn_oracle as O

import paper_2210_15874_b200 as Q
from paper_2210_15874_b200 import _native as N
from paper_2210_15874_b200 import workloads as W

C128 = Q.Backend.b200(dtype="complex128")
C64 = Q.Backend.b200(dtype="complex64")


def _desc(mem, dtype_code=N.QTN_C64, base=1 << 20):
    b = Q.Bucket(W.BUCKET, [Q.Tensor(i, np.zeros((2,) * len(i))) for i, _ in mem])
    res = tuple(sorted(set().union(*[set(i) for i, _ in mem]) - {W.BUCKET}))
    st = Q.tensor_core.bucket_strides(b, res)
    ptrs = [base * (k + 1) for k in range(len(mem))]   # fake, 16-byte aligned
    return N.bucket_desc(dtype_code, len(res), base * 64, list(zip(ptrs, st))), res


# ---------------------------------------------------------------- CPU ----
def test_structure_classes():
    for w in (0, 1, 5, 12):
        for k in (1, 3, 6):
            mem = W.bucket_structure(w, k, "A", 7)
            assert sorted(mem[0]) == list(range(w + 1)) and len(mem) == k
            assert all(W.BUCKET in m for m in mem)
        mb = W.bucket_structure(w, 2, "B", 7)
        assert len(mb) == 2 and set(mb[0]) | set(mb[1]) == set(range(w + 1))
    assert W.bucket_structure(10, 3, "A", 1) == W.bucket_structure(10, 3, "A", 1)


@pytest.mark.parametrize("cls,w,k", [("A", 8, 3), ("A", 20, 6), ("A", 30, 3), ("B", 16, 2), ("B", 30, 2), ("B", 26, 2),
                                     ("A", 0, 2), ("A", 3, 4)])
@pytest.mark.parametrize("code", [N.QTN_C64, N.QTN_C128])
def test_plan_fits(cls, w, k, code):
    mem = W.bucket_structure(w, k, cls, 3)
    d, res = _desc([(m, None) for m in mem], code)
    nt, stage, smem, tiles, nb, nf, nu, inv = N.bucket_plan(d)
    assert nt <= min(w, 11 if code == N.QTN_C64 else 10) and tiles == 1 << (w - nt)
    assert smem <= 227 * 1024 and stage >= 2
    if w >= 5:
        assert nt >= 5          # the output's 5 lowest bits are always tile bits
    assert (1 <= nb <= 4 or nb == -1) and (nb + nf == k or nb == -1) and nu <= 5
    if cls == "A" and w >= 20 and k > 1:
        assert nb >= 1 and nf >= 1       # small members folded into the product table
        assert inv == 1                  # ... and the table is loaded once per tile
    if cls == "B" and w >= 16:
        assert nb == 2 and nf == 0       # large members are all staged
    if cls == "B" and w >= 24:
        assert inv == 1                  # one of them is read once per tile


def test_plan_errors():
    mem = W.bucket_structure(6, 3, "A", 0)
    d, _ = _desc([(m, None) for m in mem])
    d.mem[1].strides[d.w] = 0           # member without the bucket index
    with pytest.raises(N.NativeError) as e:
        N.bucket_plan(d)
    assert e.value.code == N.QTN_E_INVALID
    d, _ = _desc([(m, None) for m in W.bucket_structure(32, 2, "B", 0)])
    with pytest.raises(N.NativeError) as e:
        N.bucket_plan(d)
    assert e.value.code == N.QTN_E_UNSUPPORTED
    d, _ = _desc([(m, None) for m in mem])
    d.n_mem = 0
    with pytest.raises(N.NativeError):
        N.bucket_plan(d)


# ---------------------------------------------------------------- GPU ----
CASES = [("A", w, k, s) for w in (0, 1, 2, 5, 8, 11, 14) for k in (1, 3, 6) for s in (0, 1)] + \
        [("B", w, 2, s) for w in (1, 4, 8, 12, 15) for s in (0, 1, 2)]


@pytest.mark.gpu
@pytest.mark.parametrize("cls,w,k,seed", CASES)
def test_k3_vs_oracle(cls, w, k, seed):
    mem = W.synthetic_bucket(w, k, cls, seed)
    ridx, ref = O.bucket_fast(W.BUCKET, mem)
    b = Q.Bucket(W.BUCKET, [Q.Tensor(i, d) for i, d in mem])
    out, st = Q.contract_bucket(b, C128)
    assert out.indices == ridx and st.width == len(ridx)
    np.testing.assert_allclose(out.data, ref, rtol=1e-12, atol=1e-12)
    out64, _ = Q.contract_bucket(b, C64)
    scale = max(1.0, float(np.abs(ref).max()))
    np.testing.assert_allclose(out64.data, ref, rtol=1e-5, atol=1e-5 * scale)


@pytest.mark.gpu
def test_k3_brute_force_small():
    for seed in range(4):
        mem = W.synthetic_bucket(4, 4, "A", seed)
        _, ref = O.bucket_brute(W.BUCKET, mem)
        out, _ = Q.contract_bucket(Q.Bucket(W.BUCKET, [Q.Tensor(i, d) for i, d in mem]), C128)
        np.testing.assert_allclose(out.data, ref, atol=1e-12)


def _einsum_ref(mem_dev, w):
    """torch complex128 einsum of the same bucket (checker for large widths)."""
    import torch
    letters = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"
    ops, subs = [], []
    for idx, t in mem_dev:
        ops.append(t.to(torch.complex128).view((2,) * len(idx)))
        subs.append("".join(letters[i] for i in idx))
    return torch.einsum(",".join(subs) + "->" + "".join(letters[i] for i in range(1, w + 1)), *ops).reshape(-1)


@pytest.mark.gpu
@pytest.mark.parametrize("cls,w,k", [("A", 20, 3), ("A", 22, 6), ("B", 22, 2), ("A", 24, 4)])
def test_k3_large_vs_einsum(cls, w, k):
    import torch
    for dtype, tol in (("complex64", 1e-5), ("complex128", 1e-12)):
        mem = W.synthetic_bucket_device(w, k, cls, 11, dtype)
        b = Q.Bucket(W.BUCKET, [Q.DeviceTensor(i, t) for i, t in mem])
        out, st = Q.contract_bucket(b, Q.Backend.b200(dtype=dtype))
        ref = _einsum_ref(mem, w)
        err = (out.storage.to(torch.complex128) - ref).abs().max().item()
        assert err <= tol * max(1.0, ref.abs().max().item()), (dtype, err)


@pytest.mark.gpu
def test_k3_strided_device_members_and_mixed_dtypes():
    # device members in c128 feeding a c64 contraction are converted first
    mem = W.synthetic_bucket(9, 3, "A", 4)
    ridx, ref = O.bucket_fast(W.BUCKET, mem)
    b = Q.Bucket(W.BUCKET, [Q.DeviceTensor.from_host(Q.Tensor(i, d)) for i, d in mem])
    out, _ = Q.contract_bucket(b, C64)
    assert isinstance(out, Q.DeviceTensor) and out.dtype == "complex64"
    np.testing.assert_allclose(out.data, ref, rtol=1e-5, atol=1e-5 * max(1.0, np.abs(ref).max()))


def _multisum_case(w, k, nmem, seed, dtype, big_ranks=True):
    """Members over result ids 1..w and summed ids w+1..w+k, random axis
    orders; every summed index carried by at least one member."""
    import torch
    rng = np.random.default_rng(seed)
    res = list(range(1, w + 1))
    summ = list(range(w + 1, w + k + 1))
    mem = []
    for i in range(nmem):
        if i == 0 and big_ranks:
            ids = res + summ
        else:
            pick = [x for x in res if rng.random() < (0.6 if big_ranks else 0.2)]
            sp = [x for x in summ if rng.random() < 0.7]
            ids = pick + sp
        mem.append(list(int(x) for x in rng.permutation(ids)))
    for x in summ + res:                 # every index somewhere (result = union - summed)
        if not any(x in m for m in mem):
            mem[int(rng.integers(nmem))].append(x)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    cdt = torch.complex64 if dtype == "complex64" else torch.complex128
    rdt = torch.float32 if dtype == "complex64" else torch.float64
    data = []
    for ids in mem:
        n = 1 << len(ids)
        x = torch.randn(2 * n, generator=gen, device="cuda", dtype=rdt) * (1.0 / np.sqrt(2.0))
        data.append(torch.view_as_complex(x.view(n, 2)).view(cdt))
    return res, summ, mem, data


@pytest.mark.gpu
@pytest.mark.parametrize("w,k,nmem,big", [(10, 2, 3, True), (16, 2, 4, True), (20, 3, 4, True), (14, 3, 2, False),
                                          (22, 2, 5, True), (9, 3, 6, False), (0, 2, 2, False), (5, 3, 3, True)])
@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_k3_multisum_vs_einsum(w, k, nmem, big, dtype):
    """K3 with k summed indices (the program path's merged-chain items)."""
    import torch
    from paper_2210_15874_b200 import engine as E
    res, summ, mem, data = _multisum_case(w, k, nmem, 7 + w + k, dtype, big)
    bit = {a: w - 1 - j for j, a in enumerate(res)}
    for q, a in enumerate(summ):
        bit[a] = w + q
    members = [(t.data_ptr(), {bit[a]: 1 << (len(ids) - 1 - ax) for ax, a in enumerate(ids)})
               for ids, t in zip(mem, data)]
    out = torch.empty(max(1, 1 << w), dtype=data[0].dtype, device="cuda")
    d = N.bucket_desc(E.DTYPE_CODE[dtype], w, out.data_ptr(), members, k=k)
    N.bucket_launch(d, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    letters = "abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ"
    ops = [t.to(torch.complex128).view((2,) * len(ids)) for ids, t in zip(mem, data)]
    subs = ",".join("".join(letters[a] for a in ids) for ids in mem)
    ref = torch.einsum(subs + "->" + "".join(letters[a] for a in res), *ops).reshape(-1)
    tol = 1e-5 if dtype == "complex64" else 1e-12
    err = (out[: 1 << w].to(torch.complex128) - ref).abs().max().item()
    assert err <= tol * max(1.0, ref.abs().max().item()), err
