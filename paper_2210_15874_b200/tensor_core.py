"""Tensors, buckets, backend policy and the process-bucket call on B200.

Mirrors the reference's L0 (src/tensor_core.py): `Tensor`, `Bucket`,
`BucketStats`, `Backend`, `memory_estimate`, `permute`, `contract_bucket`.
The CPU kernels (`reference_kernel`, `fast_kernel`) are replaced by the
sm_100a program kernel; there is no CPU fallback — a missing library or
device raises `NativeUnavailable`.

Host tensors (`Tensor`) are exactly the reference's: immutable complex128
numpy arrays of shape (2,)*rank, C order, last listed index fastest.
`DeviceTensor` is the same contract with the data resident in HBM (torch
storage); `.data` copies it back lazily.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import engine as E

B200 = "b200"
DEFAULT_MIXED_THRESHOLD = 11   # src/tensor_core.py:17 (small/large split)
KINDS = (B200,)


@dataclass(frozen=True)
class Backend:
    """Kernel policy.  `kind` is always "b200".

    threshold: buckets with result width <= threshold (w + k <= threshold + 1
      for a merged item summing k indices) run in the batched small-bucket
      schedule (K2 persistent stages, "b200-small"), wider ones in the fused
      large-bucket kernels (K1, "b200-large") — the B200 analogue of the
      reference's Mixed routing (src/tensor_core.py:176-184); both run inside
      the same CUDA graph.  `tune-threshold` (tuning.py) picks it on the B200.
    dtype: "complex64" or "complex128" (the reference is complex128 only).
    device: CUDA device ordinal.
    profile: record per-bucket device time (BucketStats.elapsed_ns).
    """

    kind: str = B200
    threshold: int | None = None
    dtype: str = "complex128"
    device: int = 0
    profile: bool = True

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown backend kind: {self.kind!r}")
        if self.threshold is not None and self.threshold < 0:
            raise ValueError("mixed threshold must be >= 0")
        object.__setattr__(self, "dtype", E.norm_dtype(self.dtype))

    @classmethod
    def b200(cls, dtype="complex128", threshold=None, device=0, profile=True):
        return cls(B200, threshold, dtype, device, profile)

    # drop-in aliases for code written against the reference's constructors
    @classmethod
    def fast(cls) -> "Backend":
        return cls(B200)

    @classmethod
    def reference(cls) -> "Backend":
        return cls(B200)

    @classmethod
    def mixed(cls, threshold: int = DEFAULT_MIXED_THRESHOLD) -> "Backend":
        return cls(B200, threshold)

    def route(self, width: int) -> str:
        thr = DEFAULT_MIXED_THRESHOLD if self.threshold is None else self.threshold
        return "b200-large" if width > thr else "b200-small"

    @property
    def elem_bytes(self) -> int:
        return E.ELEM_BYTES[self.dtype]


class Tensor:
    """Immutable dense host tensor over binary indices (src/tensor_core.py:46-74)."""

    __slots__ = ("indices", "data")

    def __init__(self, indices, data):
        indices = tuple(int(i) for i in indices)
        if len(set(indices)) != len(indices):
            raise ValueError("duplicate index id in tensor")
        data = np.asarray(data, dtype=np.complex128)
        if data.shape != (2,) * len(indices):
            data = data.reshape((2,) * len(indices))
        data.setflags(write=False)
        object.__setattr__(self, "indices", indices)
        object.__setattr__(self, "data", data)

    def __setattr__(self, *a):
        raise AttributeError("Tensor is immutable")

    @classmethod
    def _trusted(cls, indices: tuple, data: np.ndarray) -> "Tensor":
        """Internal constructor for the network builders: `indices` is a
        tuple of distinct ints and `data` a read-only complex128 array of
        shape (2,)*rank (shared gate arrays are safe: Tensors are immutable)."""
        t = object.__new__(cls)
        object.__setattr__(t, "indices", indices)
        object.__setattr__(t, "data", data)
        return t

    @property
    def rank(self) -> int:
        return len(self.indices)

    def __repr__(self):
        return f"Tensor(indices={self.indices}, rank={self.rank})"


class DeviceTensor:
    """Tensor resident in HBM: a flat torch complex tensor of 2^rank elements,
    C order over `indices`.  `.data` returns a host numpy copy (complex128,
    shape (2,)*rank) so code written against `Tensor` keeps working."""

    __slots__ = ("indices", "storage", "_host")

    def __init__(self, indices, storage):
        indices = tuple(int(i) for i in indices)
        if len(set(indices)) != len(indices):
            raise ValueError("duplicate index id in tensor")
        if storage.numel() != 1 << len(indices):
            raise ValueError("storage size does not match rank")
        object.__setattr__(self, "indices", indices)
        object.__setattr__(self, "storage", storage)
        object.__setattr__(self, "_host", None)

    def __setattr__(self, *a):
        raise AttributeError("DeviceTensor is immutable")

    @property
    def rank(self) -> int:
        return len(self.indices)

    @property
    def dtype(self) -> str:
        return E.norm_dtype(self.storage.dtype)

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            import torch
            # widen on the device (one D2H copy, no host conversion pass)
            h = self.storage.detach().to(torch.complex128).cpu().numpy().reshape((2,) * self.rank)
            h.setflags(write=False)
            object.__setattr__(self, "_host", h)
        return self._host

    def to_host(self) -> Tensor:
        return Tensor(self.indices, self.data)

    @classmethod
    def from_host(cls, t, dtype="complex128", device=0):
        import torch
        dt = torch.complex64 if E.norm_dtype(dtype) == "complex64" else torch.complex128
        arr = np.array(np.asarray(t.data).ravel(), dtype=np.complex128)  # writable copy
        return cls(t.indices, torch.from_numpy(arr).to(device=f"cuda:{device}", dtype=dt))

    def __repr__(self):
        return f"DeviceTensor(indices={self.indices}, rank={self.rank}, dtype={self.dtype})"


@dataclass(frozen=True)
class Bucket:
    """All tensors sharing `bucket_index` (src/tensor_core.py:77-90)."""

    bucket_index: int
    tensors: tuple

    def __post_init__(self):
        object.__setattr__(self, "tensors", tuple(self.tensors))
        for t in self.tensors:
            if self.bucket_index not in t.indices:
                raise ValueError(f"tensor {t!r} does not contain bucket index {self.bucket_index}")


@dataclass(frozen=True)
class BucketStats:
    """width = result rank (src/tensor_core.py:93-97); elapsed_ns = the
    bucket's device time, 0 when profiling is off — the reference times every
    bucket's kernel (185-187); here a device item may be a merged chain of
    buckets, so its measured span (first tile start -> last tile end,
    %globaltimer) is split over its buckets in proportion to their
    algorithmic elements (the sum over an item's buckets is the item's time);
    backend_used = the route, "b200-small" (batched K2 stage) or
    "b200-large" (fused kernels) — the analogue of the reference's Mixed
    reference/fast split; kernel = the kernel family that ran it (K1..K5)."""

    width: int
    elapsed_ns: int
    backend_used: str
    kernel: str = ""


def memory_estimate(width: int, dtype: str = "complex128") -> int:
    """Bytes of one rank-`width` tensor (src/tensor_core.py:100-104; dtype-aware)."""
    if width < 0:
        raise ValueError("width must be >= 0")
    return E.ELEM_BYTES[E.norm_dtype(dtype)] * (1 << width)


def permute(t, new_order):
    """Reorder tensor indices keeping element values (src/tensor_core.py:107-114).
    Host tensors are permuted with numpy; device tensors with qtn_permute."""
    new_order = tuple(int(i) for i in new_order)
    if sorted(new_order) != sorted(t.indices) or len(new_order) != t.rank:
        raise ValueError("new_order is not a permutation of the tensor's indices")
    if isinstance(t, DeviceTensor):
        return _device_permute(t, new_order, t.dtype)
    src = {idx: ax for ax, idx in enumerate(t.indices)}
    return Tensor(new_order, np.transpose(t.data, tuple(src[i] for i in new_order)))


def _result_indices(b: Bucket) -> tuple:
    u = set()
    for t in b.tensors:
        u.update(t.indices)
    u.discard(b.bucket_index)
    return tuple(sorted(u))


def _device_permute(t: DeviceTensor, new_order, dtype) -> DeviceTensor:
    """Device copy of `t` with axes `new_order` and element type `dtype`."""
    import torch
    dtype = E.norm_dtype(dtype)
    if tuple(new_order) == t.indices and t.dtype == dtype:
        return t
    r = t.rank
    srcpos = {idx: ax for ax, idx in enumerate(t.indices)}
    # dst bit j (j = 0 fastest) is axis new_order[r-1-j]
    strides = [1 << (r - 1 - srcpos[new_order[r - 1 - j]]) for j in range(r)]
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    out = torch.empty(1 << r, dtype=tdt, device=t.storage.device)
    stream = torch.cuda.current_stream(t.storage.device).cuda_stream
    N.permute(E.DTYPE_CODE[t.dtype], t.storage.data_ptr(), 0, E.DTYPE_CODE[dtype], out.data_ptr(),
              r, strides, stream)
    return DeviceTensor(new_order, out)


def _upload(arr, dev):
    """Host ndarray -> flat device tensor (read-only arrays are copied by the
    H2D transfer itself; torch only warns that it cannot write to them)."""
    import torch
    import warnings
    a = np.ascontiguousarray(arr).reshape(-1)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(a).to(dev)


def bucket_strides(b: Bucket, res):
    """Iteration strides of every member of `b` for K3 (include/qtn_b200.h,
    qtn_bucket_desc_t): bit j < w is result axis j counted from the LAST
    sorted index (src/tensor_core.py:117-122), bit w the bucket index; a
    member in C order over its own indices has stride 2^(rank-1-axis)."""
    w = len(res)
    bit = {a: w - 1 - j for j, a in enumerate(res)}
    bit[b.bucket_index] = w
    out = []
    for t in b.tensors:
        r = len(t.indices)
        out.append({bit[a]: 1 << (r - 1 - ax) for ax, a in enumerate(t.indices)})
    return out


def contract_bucket(b: Bucket, backend: Backend = None):
    """Process-bucket: sum `bucket_index` out of the product of the members
    (src/tensor_core.py:167-188), on the B200, in ONE fused kernel (K3,
    csrc/bucket_strided.cu) that reads every member in its own axis order —
    no member is transposed first (the reference's fast_kernel transposes and
    broadcasts each member, src/tensor_core.py:148-164).

    Returns (result, BucketStats).  The result's indices are the sorted union
    minus the bucket index (src/tensor_core.py:117-122).  Host members give a
    host `Tensor`; if any member is a `DeviceTensor` the result stays on the
    device as a `DeviceTensor` (members in another dtype are converted on
    the device first).  BucketStats.elapsed_ns is the kernel's device time
    (CUDA events), like the reference's kernel-only timing (185-187)."""
    import torch
    backend = backend or Backend()
    if not b.tensors:
        raise ValueError("empty bucket")
    N.require_device()
    res = _result_indices(b)
    w = len(res)
    if len(b.tensors) > N.MAX_MEMBERS:
        raise ValueError(f"bucket has {len(b.tensors)} members; at most {N.MAX_MEMBERS} supported")
    dtype = backend.dtype
    dev = torch.device("cuda", backend.device)
    tdt = torch.complex64 if dtype == "complex64" else torch.complex128
    any_dev = any(isinstance(t, DeviceTensor) for t in b.tensors)
    strides = bucket_strides(b, res)
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        members = []
        for t in b.tensors:
            if isinstance(t, DeviceTensor):
                st = t.storage if t.storage.device == dev else t.storage.to(dev)
                if st.dtype != tdt or not st.is_contiguous():
                    st = st.to(tdt).contiguous()
            else:   # host member: uploaded as is (complex128), narrowed on the device
                st = _upload(t.data, dev)
                if st.dtype != tdt:
                    st = st.to(tdt)
            members.append(st)
        out = torch.empty(1 << w, dtype=tdt, device=dev)
        desc = N.bucket_desc(E.DTYPE_CODE[dtype], w, out.data_ptr(),
                             [(m.data_ptr(), s) for m, s in zip(members, strides)])
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        N.bucket_launch(desc, stream.cuda_stream)
        ev1.record(stream)
        ev1.synchronize()
        elapsed = int(ev0.elapsed_time(ev1) * 1e6)
    result = DeviceTensor(res, out)
    if not any_dev:
        result = result.to_host()
    # one fused K3 launch whatever the width (no small-bucket route here)
    return result, BucketStats(width=w, elapsed_ns=elapsed if backend.profile else 0,
                               backend_used="b200-large", kernel="K3")


# BASELINE.json vocabulary: "process-bucket"
process_bucket = contract_bucket
