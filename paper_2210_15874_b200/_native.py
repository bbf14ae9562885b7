"""ctypes binding of libqtn_b200.so (include/qtn_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` /
`make -C paper_2210_15874_b200` into `paper_2210_15874_b200/lib/`.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises `NativeUnavailable`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.environ.get("QTN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                     "libqtn_b200.so")

QTN_OK = 0
QTN_E_INVALID = -1
QTN_E_CUDA = -2
QTN_E_UNSUPPORTED = -3
QTN_E_NODEVICE = -4
QTN_C64 = 0
QTN_C128 = 1
QTN_FINALIZE = -1
MAX_MEMBERS = 8
MAX_WIDTH = 40
MAX_SUMMED = 6
ABI_VERSION = 10
QTN_NODE_SMALL = 0
QTN_NODE_LARGE = 1
QTN_VARIANT_GENERIC = -1
# graph node kernel families (qtn_graph_node_kinds codes 0..4)
KERNEL_FAMILIES = ("K1", "K2", "K3", "K4", "K5", "K6")

# every symbol include/qtn_b200.h declares
EXPORTS = (
    "qtn_abi_version",
    "qtn_last_error",
    "qtn_device_count",
    "qtn_program_reset",
    "qtn_node_launch",
    "qtn_graph_create",
    "qtn_graph_create_io",
    "qtn_graph_create_host",
    "qtn_graph_kinds",
    "qtn_bucket_expand",
    "qtn_bucket_stream",
    "qtn_bucket_expand_fused",
    "qtn_bucket_expand_fused_plan",
    "qtn_route_config",
    "qtn_graph_node_kinds",
    "qtn_graph_launch",
    "qtn_graph_destroy",
    "qtn_permute",
    "qtn_greedy_order",
    "qtn_dry_run",
    "qtn_suggest_slicing",
    "qtn_bucket",
    "qtn_bucket_plan",
    "qtn_plan_build",
    "qtn_plan_scalars",
    "qtn_plan_array_len",
    "qtn_plan_array",
    "qtn_plan_destroy",
)
PLAN_ARRAYS = ("w", "k", "L", "level", "out_off", "mem_ptr", "mem_kind", "mem_ref", "mem_mask", "mem_smask",
               "smem_elems", "stmask", "mem_cls", "variant", "ref_w", "ref_item", "ref_last", "ref_elems",
               "bucket_index", "fin_kind", "fin_ref", "in_off", "gdst", "gsrc", "gfix")

BUCKET_DT = np.dtype([
    ("out_off", "<u8"), ("w", "<i4"), ("tile_bits", "<i4"), ("k", "<i4"), ("mem_begin", "<i4"),
    ("n_mem", "<i4"), ("dep_begin", "<i4"), ("n_dep", "<i4"), ("tick_begin", "<i4"),
    ("n_tiles", "<i4"), ("slot", "<i4"), ("smem_elems", "<i4"), ("stmask", "<u4"), ("reserved0", "<i4"),
    ("reserved1", "<i4"),
])
MEMBER_DT = np.dtype([("off", "<u8"), ("mask", "<u8"), ("smask", "<u4"), ("cls", "<u4")])
NODE_DT = np.dtype([("kind", "<i4"), ("first", "<i4"), ("count", "<i4"), ("n_tickets", "<i4"),
                    ("variant", "<i4"), ("dep_begin", "<i4"), ("n_dep", "<i4"), ("smem_bytes", "<i4")])
DEP_DT = np.dtype([("bucket", "<i4"), ("need", "<i4")])
assert BUCKET_DT.itemsize == 64 and MEMBER_DT.itemsize == 24 and DEP_DT.itemsize == 8
assert NODE_DT.itemsize == 32


class NativeUnavailable(RuntimeError):
    """The CUDA library or device is missing: the B200 path cannot run."""


class NativeError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"qtn_b200 error {code}: {msg}")


class ProgramC(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32), ("n_buckets", ctypes.c_int32), ("n_tickets", ctypes.c_int32),
        ("smem_bytes", ctypes.c_int32), ("grid", ctypes.c_int32), ("n_nodes", ctypes.c_int32),
        ("buckets", ctypes.c_void_p), ("members", ctypes.c_void_p), ("deps", ctypes.c_void_p),
        ("tick_begin", ctypes.c_void_p), ("ctrl", ctypes.c_void_p), ("arena", ctypes.c_void_p),
        ("results", ctypes.c_void_p), ("timing", ctypes.c_void_p), ("arena_elems", ctypes.c_int64),
        ("inputs_hi", ctypes.c_void_p), ("n_in_elems", ctypes.c_int64),
    ]


class BMemberC(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("strides", ctypes.c_int64 * (MAX_WIDTH + 1))]


class BucketDescC(ctypes.Structure):
    """qtn_bucket_desc_t: one standalone bucket, members in any axis order."""
    _fields_ = [("dtype", ctypes.c_int32), ("w", ctypes.c_int32), ("n_mem", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("out", ctypes.c_void_p), ("mem", BMemberC * MAX_MEMBERS)]


class GraphIOC(ctypes.Structure):
    """qtn_graph_io_t: input upload / result download nodes of a program graph."""
    _fields_ = [("h2d_src", ctypes.c_void_p), ("h2d_dst", ctypes.c_void_p), ("h2d_bytes", ctypes.c_int64),
                ("d2h_src", ctypes.c_void_p), ("d2h_dst", ctypes.c_void_p), ("d2h_bytes", ctypes.c_int64),
                ("gather_raw", ctypes.c_void_p), ("gather_src", ctypes.c_void_p), ("gather_dst", ctypes.c_void_p),
                ("n_gather", ctypes.c_int64)]


class PlanParamsC(ctypes.Structure):
    """qtn_plan_params_t: the engine's cost-model constants."""
    _fields_ = [("elem_bytes", ctypes.c_int32), ("tile_bits", ctypes.c_int32), ("small_tile_bits", ctypes.c_int32),
                ("min_tile_bits", ctypes.c_int32), ("kmax", ctypes.c_int32), ("max_members", ctypes.c_int32),
                ("vec", ctypes.c_int32), ("nt", ctypes.c_int32), ("small_iter_bits", ctypes.c_int32),
                ("merge", ctypes.c_int32), ("resident_blocks", ctypes.c_int32), ("smem_budget", ctypes.c_int64),
                ("hop_s", ctypes.c_double), ("hop_k2_s", ctypes.c_double), ("bw_bps", ctypes.c_double),
                ("block_terms_ps", ctypes.c_double), ("small_load_s", ctypes.c_double),
                ("cheap_member_w", ctypes.c_double), ("kmax_large", ctypes.c_int32),
                ("wave_slots", ctypes.c_int32), ("wave_ov_elems", ctypes.c_int32)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the library (no device needed) and declare the signatures."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    lib.qtn_abi_version.restype = ctypes.c_int
    lib.qtn_abi_version.argtypes = []
    lib.qtn_last_error.restype = ctypes.c_char_p
    lib.qtn_last_error.argtypes = []
    lib.qtn_device_count.restype = ctypes.c_int
    lib.qtn_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.qtn_program_reset.restype = ctypes.c_int
    lib.qtn_program_reset.argtypes = [ctypes.POINTER(ProgramC), vp]
    lib.qtn_node_launch.restype = ctypes.c_int
    lib.qtn_node_launch.argtypes = [ctypes.POINTER(ProgramC), vp, i32, vp]
    lib.qtn_graph_create.restype = ctypes.c_int
    lib.qtn_graph_create.argtypes = [ctypes.POINTER(ProgramC), vp, i32, vp, ctypes.POINTER(ctypes.c_void_p)]
    lib.qtn_graph_node_kinds.restype = ctypes.c_int
    lib.qtn_graph_node_kinds.argtypes = [vp, vp, i32]
    lib.qtn_bucket_expand.restype = ctypes.c_int
    lib.qtn_bucket_expand.argtypes = [ctypes.POINTER(BucketDescC), i32, vp]
    lib.qtn_bucket_expand_fused.restype = ctypes.c_int
    lib.qtn_bucket_expand_fused.argtypes = [ctypes.POINTER(BucketDescC), ctypes.POINTER(BucketDescC), i32, vp]
    lib.qtn_bucket_expand_fused_plan.restype = ctypes.c_int
    lib.qtn_bucket_expand_fused_plan.argtypes = [ctypes.POINTER(BucketDescC), ctypes.POINTER(BucketDescC), i32, vp]
    lib.qtn_bucket_stream.restype = ctypes.c_int
    lib.qtn_bucket_stream.argtypes = [ctypes.POINTER(BucketDescC), vp]
    lib.qtn_route_config.restype = ctypes.c_char_p
    lib.qtn_route_config.argtypes = []
    lib.qtn_graph_kinds.restype = ctypes.c_int
    lib.qtn_graph_kinds.argtypes = [vp, vp]
    lib.qtn_graph_create_host.restype = ctypes.c_int
    lib.qtn_graph_create_host.argtypes = [ctypes.POINTER(ProgramC), vp, vp, ctypes.c_int64, vp, i32, vp,
                                          ctypes.POINTER(GraphIOC), ctypes.POINTER(ctypes.c_void_p)]
    lib.qtn_graph_create_io.restype = ctypes.c_int
    lib.qtn_graph_create_io.argtypes = [ctypes.POINTER(ProgramC), vp, i32, vp, ctypes.POINTER(GraphIOC),
                                        ctypes.POINTER(ctypes.c_void_p)]
    lib.qtn_graph_launch.restype = ctypes.c_int
    lib.qtn_graph_launch.argtypes = [ctypes.c_void_p, vp]
    lib.qtn_graph_destroy.restype = ctypes.c_int
    lib.qtn_graph_destroy.argtypes = [ctypes.c_void_p]
    lib.qtn_dry_run.restype = ctypes.c_int
    lib.qtn_dry_run.argtypes = [i32, vp, vp, i32, vp, i32, vp, vp, vp, ctypes.POINTER(i32)]
    lib.qtn_suggest_slicing.restype = ctypes.c_int
    lib.qtn_suggest_slicing.argtypes = [i32, vp, vp, i32, vp, i32, i32, vp, ctypes.POINTER(i32)]
    lib.qtn_greedy_order.restype = ctypes.c_int
    lib.qtn_greedy_order.argtypes = [i32, vp, vp, i32, vp, i32, vp, ctypes.POINTER(i32)]
    lib.qtn_permute.restype = ctypes.c_int
    lib.qtn_permute.argtypes = [i32, vp, i64, i32, vp, i32, ctypes.POINTER(i64), vp]
    lib.qtn_bucket.restype = ctypes.c_int
    lib.qtn_bucket.argtypes = [ctypes.POINTER(BucketDescC), vp]
    lib.qtn_bucket_plan.restype = ctypes.c_int
    lib.qtn_bucket_plan.argtypes = [ctypes.POINTER(BucketDescC), ctypes.POINTER(i32)]
    lib.qtn_plan_build.restype = ctypes.c_int
    lib.qtn_plan_build.argtypes = [i32, vp, vp, i32, vp, i32, vp, ctypes.POINTER(PlanParamsC),
                                   ctypes.POINTER(ctypes.c_void_p)]
    lib.qtn_plan_scalars.restype = ctypes.c_int
    lib.qtn_plan_scalars.argtypes = [vp, vp]
    lib.qtn_plan_array_len.restype = ctypes.c_int
    lib.qtn_plan_array_len.argtypes = [vp, i32, ctypes.POINTER(i64)]
    lib.qtn_plan_array.restype = ctypes.c_int
    lib.qtn_plan_array.argtypes = [vp, i32, vp]
    lib.qtn_plan_destroy.restype = ctypes.c_int
    lib.qtn_plan_destroy.argtypes = [vp]
    if lib.qtn_abi_version() != ABI_VERSION:
        raise NativeUnavailable(f"ABI mismatch: library {lib.qtn_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(rc: int):
    if rc != QTN_OK:
        raise NativeError(rc, _lib.qtn_last_error().decode(errors="replace"))


def require_device():
    """Fail loudly (no CPU fallback) when no CUDA device is usable."""
    lib = load()
    import torch
    n = ctypes.c_int(0)
    lib.qtn_device_count(ctypes.byref(n))
    if n.value < 1 or not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the B200 backend has no CPU fallback")
    return lib


def greedy_order(index_lists, open_indices=(), heuristic=0):
    """Host-side greedy elimination order (qtn_greedy_order); no device needed."""
    lib = load()
    ptr, idx = _csr(index_lists)
    opn = np.asarray(list(open_indices), dtype=np.int64)
    n_distinct = len(np.unique(idx)) if len(idx) else 0
    out = np.zeros(max(1, n_distinct), np.int64)
    n_out = ctypes.c_int32(0)
    check(lib.qtn_greedy_order(len(index_lists), ptr.ctypes.data_as(ctypes.c_void_p),
                               idx.ctypes.data_as(ctypes.c_void_p) if len(idx) else None, len(opn),
                               opn.ctypes.data_as(ctypes.c_void_p) if len(opn) else None, heuristic,
                               out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n_out)))
    return out[: n_out.value].tolist()


def _csr(index_lists):
    ptr = np.zeros(len(index_lists) + 1, np.int32)
    lens = [len(ids) for ids in index_lists]
    if lens:
        ptr[1:] = np.cumsum(lens)
    flat = np.fromiter((i for ids in index_lists for i in ids), dtype=np.int64, count=int(ptr[-1]))
    return ptr, flat


def _vp(a):
    return a.ctypes.data_as(ctypes.c_void_p) if len(a) else None


def dry_run(index_lists, order, fixed=()):
    """Host dry run (qtn_dry_run): (widths, active order); no device needed."""
    lib = load()
    ptr, flat = _csr(index_lists)
    o = np.asarray(list(order), dtype=np.int64)
    fx = np.asarray(list(fixed), dtype=np.int64)
    widths = np.zeros(max(1, len(o)), np.int32)
    active = np.zeros(max(1, len(o)), np.int64)
    n = ctypes.c_int32(0)
    check(lib.qtn_dry_run(len(index_lists), ptr.ctypes.data_as(ctypes.c_void_p), _vp(flat), len(o), _vp(o), len(fx),
                          _vp(fx), widths.ctypes.data_as(ctypes.c_void_p), active.ctypes.data_as(ctypes.c_void_p),
                          ctypes.byref(n)))
    return widths[: n.value].tolist(), active[: n.value].tolist()


def suggest_slicing(index_lists, order, target_width):
    """Host greedy slicing (qtn_suggest_slicing); no device needed."""
    lib = load()
    ptr, flat = _csr(index_lists)
    o = np.asarray(list(order), dtype=np.int64)
    out = np.zeros(max(1, len(o)), np.int64)
    n = ctypes.c_int32(0)
    check(lib.qtn_suggest_slicing(len(index_lists), ptr.ctypes.data_as(ctypes.c_void_p), _vp(flat), len(o), _vp(o),
                                  int(target_width), len(out), out.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
    return out[: n.value].tolist()


def permute(src_dtype, src_ptr, src_offset, dst_dtype, dst_ptr, rank, strides, stream):
    lib = require_device()
    arr = (ctypes.c_int64 * max(1, rank))(*[int(s) for s in strides])
    check(lib.qtn_permute(src_dtype, ctypes.c_void_p(src_ptr), int(src_offset), dst_dtype,
                          ctypes.c_void_p(dst_ptr), int(rank), arr, ctypes.c_void_p(stream)))


def bucket_desc(dtype_code, w, out_ptr, members, k=1):
    """members: [(device_ptr, {iteration_bit: element_stride})]; bits w .. w+k-1
    are the summed indices (k = 1: one reference bucket)."""
    d = BucketDescC()
    d.dtype = dtype_code
    d.w = w
    d.reserved = k
    d.n_mem = len(members)
    d.out = out_ptr
    for i, (ptr, strides) in enumerate(members):
        d.mem[i].data = ptr
        for b, st in strides.items():
            d.mem[i].strides[b] = int(st)
    return d


def bucket_plan(desc):
    """(tile bits, staged elements per tile, smem bytes, tiles, staged members
    (-1: v1 kernel), folded members, product-table bits, invariant operand) — no device needed."""
    lib = load()
    info = (ctypes.c_int32 * 8)()
    check(lib.qtn_bucket_plan(ctypes.byref(desc), info))
    return tuple(info)


def bucket_launch(desc, stream):
    lib = require_device()
    check(lib.qtn_bucket(ctypes.byref(desc), ctypes.c_void_p(stream)))


def bucket_expand_launch(desc, stream, min_e=0):
    """K4 on one expansion bucket (QTN_E_UNSUPPORTED -> NativeError when the
    descriptor is not an expansion of one dominant member)."""
    lib = require_device()
    check(lib.qtn_bucket_expand(ctypes.byref(desc), int(min_e), ctypes.c_void_p(stream)))


def bucket_expand_fused_launch(producer, consumer, member, stream):
    """K6 on a producer bucket fused with the consumer that reads its whole
    result as member `member` (QTN_E_UNSUPPORTED -> NativeError when the pair
    does not have K6's shape); the producer's output is not written."""
    lib = require_device()
    check(lib.qtn_bucket_expand_fused(ctypes.byref(producer), ctypes.byref(consumer), int(member),
                                      ctypes.c_void_p(stream)))


def bucket_expand_fused_plan(producer, consumer, member):
    """K6 plan only (no device): (producer k, consumer k, expansion bits,
    product-table bits, gathered members, uniform members, q bits no gathered
    member carries, tile-id bits)."""
    lib = load()
    info = (ctypes.c_int32 * 8)()
    check(lib.qtn_bucket_expand_fused_plan(ctypes.byref(producer), ctypes.byref(consumer), int(member), info))
    return tuple(info)


def bucket_stream_launch(desc, stream):
    """K5 on one streaming bucket (QTN_E_UNSUPPORTED -> NativeError when no
    member carries every result bit)."""
    lib = require_device()
    check(lib.qtn_bucket_stream(ctypes.byref(desc), ctypes.c_void_p(stream)))


def route_config() -> dict:
    """The routing / tuning knobs in effect (qtn_route_config)."""
    txt = load().qtn_route_config().decode()
    return {k: int(v) for k, v in (kv.split("=") for kv in txt.split())}


def plan_build(index_lists, order, fixed, params):
    """Run the native planner; returns (scalars, {name: int64 array})."""
    lib = load()
    ptr, idx = _csr(index_lists)
    od = np.asarray(order, dtype=np.int64)
    fx = np.asarray(fixed, dtype=np.int64)
    h = ctypes.c_void_p()
    rc = lib.qtn_plan_build(len(index_lists), ptr.ctypes.data_as(ctypes.c_void_p),
                            idx.ctypes.data_as(ctypes.c_void_p) if len(idx) else None, len(od),
                            od.ctypes.data_as(ctypes.c_void_p) if len(od) else None, len(fx),
                            fx.ctypes.data_as(ctypes.c_void_p) if len(fx) else None, ctypes.byref(params),
                            ctypes.byref(h))
    if rc == QTN_E_INVALID:
        raise ValueError(lib.qtn_last_error().decode(errors="replace"))
    check(rc)
    try:
        sc = np.zeros(4, np.int64)
        check(lib.qtn_plan_scalars(h, sc.ctypes.data_as(ctypes.c_void_p)))
        out = {}
        n = ctypes.c_int64(0)
        for i, name in enumerate(PLAN_ARRAYS):
            check(lib.qtn_plan_array_len(h, i, ctypes.byref(n)))
            a = np.empty(n.value, np.int64)
            check(lib.qtn_plan_array(h, i, a.ctypes.data_as(ctypes.c_void_p) if n.value else None))
            out[name] = a
        return sc, out
    finally:
        lib.qtn_plan_destroy(h)
