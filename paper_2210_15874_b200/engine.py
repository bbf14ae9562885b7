"""Planner and executor of device programs (the B200 "bucket lists").

The reference contracts a network bucket by bucket from Python
(`contract_network`, src/ordering.py:148-189): tensors go to the bucket of
their earliest index in the order, each bucket's product is summed over its
index (`contract_bucket` -> `fast_kernel`, src/tensor_core.py:148-188) and
the result is re-bucketed at its earliest remaining index; rank-0 values are
multiplied into the scalar.

Here the same symbolic replay (the dry run, src/ordering.py:97-145) is done
once on the host and frozen into a *program*: a table of buckets with member
descriptors, completion dependencies and arena offsets.  The whole program is
then executed by ONE launch of the persistent sm_100a kernel
(`program_kernel`, csrc/qtn_b200.cu).  Layout in HBM:

  arena = [ input region | intermediate region ]   (one torch allocation)

Every tensor is stored in the *canonical* layout: axes sorted by elimination
position, the earliest-eliminated axis slowest.  A member of bucket x then
has x as its slowest axis and its remaining axes in the order of the
bucket's result axes, so its element offset is  b * 2^popc(mask) + pext(r, mask).

Many instances (lightcones, slices) can share one program; each instance
ends with a finaliser item that writes its scalar to a result slot.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

ELEM_BYTES = {"complex64": 8, "complex128": 16}
DTYPE_CODE = {"complex64": N.QTN_C64, "complex128": N.QTN_C128}
# tile bits: 2^L results per tile (4096 c64 / 2048 c128 = 32 KiB of output)
TILE_BITS = {"complex64": 12, "complex128": 11}
SMEM_BUDGET = 48 * 1024
NT = 256


def norm_dtype(dtype) -> str:
    s = str(dtype).replace("torch.", "").replace("np.", "").replace("numpy.", "")
    aliases = {"c64": "complex64", "c128": "complex128", "complex64": "complex64",
               "complex128": "complex128", "<class 'complex64'>": "complex64",
               "<class 'complex128'>": "complex128"}
    if s not in aliases:
        raise ValueError(f"unsupported dtype {dtype!r} (complex64 or complex128)")
    return aliases[s]


def _align(n, a):
    return (n + a - 1) // a * a


def _tensor_align(size):
    # every rank>=1 tensor starts on a multiple of min(size, 32) elements so
    # streamed members can use 16-byte vector loads
    return max(1, min(size, 32))


@dataclass
class Template:
    """Symbolic plan of one network structure + order (+ sliced indices).

    Offsets are relative to the instance's input / intermediate bases."""
    n_in_elems: int
    n_inter_elems: int
    # per bucket (elimination order of non-empty buckets)
    w: np.ndarray            # result width
    L: np.ndarray            # tile bits
    level: np.ndarray
    out_off: np.ndarray      # relative to intermediate base
    mem_ptr: np.ndarray      # CSR into mem_* arrays
    mem_kind: np.ndarray     # 0 = input tensor, 1 = bucket result
    mem_ref: np.ndarray      # input tensor id or bucket id
    mem_mask: np.ndarray     # uint64 result-axis coverage
    smem_elems: np.ndarray
    step: np.ndarray         # position in the active order (for stats)
    bucket_index: np.ndarray # eliminated index id
    # finaliser (rank-0 values in reference multiplication order)
    fin_kind: np.ndarray
    fin_ref: np.ndarray
    # inputs
    in_off: np.ndarray       # per input tensor: relative arena offset (-1 never)
    gdst: np.ndarray         # canonical element -> relative input offset
    gsrc: np.ndarray         # ... -> element of the raw concatenated source data
    gfix: dict               # fixed index id -> per-element source offset weight
    n_raw: int               # elements of the raw concatenation
    max_width: int


def plan_template(index_sets, order, dtype, fixed=()):
    """Replay contract_network's bucket assignment (src/ordering.py:165-187)
    over index sets only and freeze it into a Template.

    index_sets: per input tensor, its indices in its own storage order
    (before slicing).  `fixed` indices are sliced out (src/ordering.py:233-248)."""
    dtype = norm_dtype(dtype)
    fixed = set(int(f) for f in fixed)
    act = [int(i) for i in order if int(i) not in fixed]
    pos = {x: k for k, x in enumerate(act)}
    lmax = TILE_BITS[dtype]
    esz = ELEM_BYTES[dtype]

    # ---- inputs: canonical layout and gather maps ----
    n_raw = 0
    in_off = np.full(len(index_sets), -1, dtype=np.int64)
    cur = 0
    gd, gs = [], []
    gfix = {f: [] for f in fixed}
    sets = []
    raw_base = []
    for t, idx in enumerate(index_sets):
        idx = tuple(int(i) for i in idx)
        r0 = len(idx)
        raw_base.append(n_raw)
        kept = [i for i in idx if i not in fixed]
        for i in kept:
            if i not in pos:
                raise ValueError(f"order is missing indices: {sorted(set(kept) - set(pos))}")
        canon = sorted(kept, key=pos.__getitem__)
        r = len(canon)
        size = 1 << r
        cur = _align(cur, _tensor_align(size))
        in_off[t] = cur
        k = np.arange(size, dtype=np.int64)
        src = np.full(size, n_raw, dtype=np.int64)
        for p, a in enumerate(canon):
            bit = (k >> (r - 1 - p)) & 1
            src += bit << (r0 - 1 - idx.index(a))
        gd.append(cur + k)
        gs.append(src)
        for f in fixed:
            wgt = (1 << (r0 - 1 - idx.index(f))) if f in idx else 0
            gfix[f].append(np.full(size, wgt, dtype=np.int64))
        cur += size
        n_raw += 1 << r0
        sets.append(frozenset(kept))
    n_in = _align(cur, 32)
    gdst = np.concatenate(gd) if gd else np.zeros(0, np.int64)
    gsrc = np.concatenate(gs) if gs else np.zeros(0, np.int64)
    gfix = {f: (np.concatenate(v) if v else np.zeros(0, np.int64)) for f, v in gfix.items()}

    # ---- bucket replay ----
    buckets = {x: [] for x in act}
    fin = []  # (kind, ref) in multiplication order
    for t, s in enumerate(sets):
        if not s:
            fin.append((0, t))
        else:
            buckets[min(s, key=pos.__getitem__)].append((0, t, s))
    W, Ls, lev, outo, mptr, mkind, mref, mmask, smem, steps, bidx = ([] for _ in range(11))
    mptr.append(0)
    inter = 0
    maxw = 0
    for step, x in enumerate(act):
        mem = buckets.pop(x)
        if not mem:
            continue
        b = len(W)
        union = set()
        for _, _, s in mem:
            union |= s
        union.discard(x)
        R = sorted(union, key=pos.__getitem__)
        w = len(R)
        if w > N.MAX_WIDTH:
            raise ValueError(f"bucket width {w} exceeds {N.MAX_WIDTH}")
        maxw = max(maxw, w)
        bit = {a: w - 1 - j for j, a in enumerate(R)}
        masks = []
        lv = 0
        for kind, ref, s in mem:
            m = 0
            for a in s:
                if a != x:
                    m |= 1 << bit[a]
            masks.append(m)
            if kind == 1:
                lv = max(lv, lev[ref] + 1)
        # tile bits: largest L <= lmax whose staged runs fit the smem budget
        L = min(w, lmax)
        while True:
            low = (1 << L) - 1
            st = sum(2 << bin(m & low).count("1") for m in masks if (m & low) != low)
            if st * esz <= SMEM_BUDGET or L == 0:
                break
            L -= 1
        if len(mem) > N.MAX_MEMBERS:
            raise ValueError(f"bucket with {len(mem)} members exceeds {N.MAX_MEMBERS}")
        size = 1 << w
        inter = _align(inter, _tensor_align(size))
        W.append(w); Ls.append(L); lev.append(lv); outo.append(inter); smem.append(st)
        steps.append(step); bidx.append(x)
        inter += size
        for (kind, ref, s), m in zip(mem, masks):
            mkind.append(kind); mref.append(ref); mmask.append(m)
        mptr.append(len(mkind))
        if w == 0:
            fin.append((1, b))
        else:
            buckets[R[0]].append((1, b, frozenset(R)))
    return Template(
        n_in_elems=n_in, n_inter_elems=_align(inter, 32),
        w=np.array(W, np.int64), L=np.array(Ls, np.int64), level=np.array(lev, np.int64),
        out_off=np.array(outo, np.int64), mem_ptr=np.array(mptr, np.int64),
        mem_kind=np.array(mkind, np.int64), mem_ref=np.array(mref, np.int64),
        mem_mask=np.array(mmask, np.uint64), smem_elems=np.array(smem, np.int64),
        step=np.array(steps, np.int64), bucket_index=np.array(bidx, np.int64),
        fin_kind=np.array([k for k, _ in fin], np.int64), fin_ref=np.array([r for _, r in fin], np.int64),
        in_off=in_off, gdst=gdst, gsrc=gsrc, gfix=gfix, n_raw=n_raw, max_width=maxw,
    )


def algorithmic_bytes(t: Template, dtype) -> int:
    """per bucket (sum_members 2^rank_i + 2^w) * sizeof(elem)."""
    esz = ELEM_BYTES[norm_dtype(dtype)]
    tot = 0
    for b in range(len(t.w)):
        tot += 1 << int(t.w[b])
        for k in range(t.mem_ptr[b], t.mem_ptr[b + 1]):
            tot += 1 << (1 + bin(int(t.mem_mask[k])).count("1"))
    return tot * esz


@dataclass
class Instance:
    template: Template
    assignment: dict = field(default_factory=dict)   # fixed index -> 0/1


class Program:
    """Several instances laid out in one arena and one ticket space."""

    def __init__(self, instances, dtype):
        self.dtype = norm_dtype(dtype)
        self.instances = list(instances)
        esz = ELEM_BYTES[self.dtype]
        n_in = 0
        in_base = []
        for inst in self.instances:
            in_base.append(n_in)
            n_in += inst.template.n_in_elems
        n_in = _align(n_in, 32)
        inter = n_in
        inter_base = []
        for inst in self.instances:
            inter_base.append(inter)
            inter += inst.template.n_inter_elems
        self.n_input_elems = n_in
        self.arena_elems = max(_align(inter, 32), 32)
        self.in_base = in_base
        self.inter_base = inter_base

        # global ticket order: (level, instance, step) — a topological order
        keys = []
        for i, inst in enumerate(self.instances):
            t = inst.template
            for b in range(len(t.w)):
                keys.append((int(t.level[b]), i, b))
            top = int(t.level.max()) + 1 if len(t.level) else 0
            keys.append((top, i, -1))  # finaliser
        keys.sort(key=lambda k: (k[0], k[1], k[2] if k[2] >= 0 else 1 << 40))
        gid = {(i, b): g for g, (_, i, b) in enumerate(keys)}
        nb = len(keys)
        B = np.zeros(nb, N.BUCKET_DT)
        members, deps = [], []
        tick = 0
        smem_max = 0
        self.bucket_gid = []   # per instance: global id per local bucket
        self.fin_gid = []
        for i, inst in enumerate(self.instances):
            t = inst.template
            self.bucket_gid.append(np.array([gid[(i, b)] for b in range(len(t.w))], np.int64))
            self.fin_gid.append(gid[(i, -1)])
        ntiles = np.zeros(nb, np.int64)
        for g, (_, i, b) in enumerate(keys):
            t = self.instances[i].template
            if b >= 0:
                ntiles[g] = 1 << int(t.w[b] - t.L[b])
            else:
                ntiles[g] = 1
        for g, (_, i, b) in enumerate(keys):
            t = self.instances[i].template
            ib, xb = in_base[i], inter_base[i]
            rec = B[g]
            rec["tick_begin"] = tick
            rec["n_tiles"] = ntiles[g]
            rec["mem_begin"] = len(members)
            rec["dep_begin"] = len(deps)
            if b >= 0:
                rec["w"] = t.w[b]
                rec["tile_bits"] = t.L[b]
                rec["out_off"] = xb + t.out_off[b]
                rec["slot"] = -1
                rec["smem_elems"] = t.smem_elems[b]
                smem_max = max(smem_max, int(t.smem_elems[b]) * esz)
                for k in range(t.mem_ptr[b], t.mem_ptr[b + 1]):
                    kind, ref = int(t.mem_kind[k]), int(t.mem_ref[k])
                    if kind == 0:
                        off = ib + int(t.in_off[ref])
                    else:
                        pg = gid[(i, ref)]
                        off = xb + int(t.out_off[ref])
                        deps.append((pg, ntiles[pg]))
                    members.append((off, int(t.mem_mask[k])))
                rec["n_mem"] = t.mem_ptr[b + 1] - t.mem_ptr[b]
            else:
                rec["w"] = N.QTN_FINALIZE
                rec["tile_bits"] = 0
                rec["out_off"] = 0
                rec["slot"] = i
                rec["smem_elems"] = 0
                for kind, ref in zip(t.fin_kind, t.fin_ref):
                    if kind == 0:
                        off = ib + int(t.in_off[ref])
                    else:
                        pg = gid[(i, int(ref))]
                        off = xb + int(t.out_off[ref])
                        deps.append((pg, ntiles[pg]))
                    members.append((off, 0))
                rec["n_mem"] = len(t.fin_kind)
            rec["n_dep"] = len(deps) - rec["dep_begin"]
            tick += int(ntiles[g])
        if tick >= 2 ** 31 - 1 - 100000:
            raise ValueError("program too large for one launch (ticket space)")
        self.n_buckets = nb
        self.n_tickets = tick
        self.smem_bytes = _align(smem_max, 16)
        self.buckets = B
        self.members = np.array(members, dtype=N.MEMBER_DT) if members else np.zeros(0, N.MEMBER_DT)
        self.deps = np.array(deps, dtype=N.DEP_DT) if deps else np.zeros(0, N.DEP_DT)
        self.tick_begin = np.ascontiguousarray(B["tick_begin"]).astype(np.int32)
        # input image gather (per instance, slice assignment applied)
        dst, src, srcinst = [], [], []
        for i, inst in enumerate(self.instances):
            t = inst.template
            s = t.gsrc.copy()
            for f, bitv in inst.assignment.items():
                if int(bitv):
                    s += t.gfix[int(f)]
            dst.append(in_base[i] + t.gdst)
            src.append(s)
        self.img_dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
        self.img_src_parts = src

    def table_bytes(self) -> bytes:
        return b"".join([self.buckets.tobytes(), self.members.tobytes(), self.deps.tobytes(),
                         self.tick_begin.tobytes()])

    def algorithmic_bytes(self) -> int:
        return sum(algorithmic_bytes(inst.template, self.dtype) for inst in self.instances)


class Executor:
    """Device-resident copy of a Program: tables, control block, arena and
    result slots, all owned by torch; launches go through the C ABI."""

    def __init__(self, prog: Program, device=0, timing=False):
        import torch
        self.torch = torch
        N.require_device()
        self.prog = prog
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        dev = self.device
        tdt = torch.complex64 if prog.dtype == "complex64" else torch.complex128
        self.tdt = tdt
        with torch.cuda.device(dev):
            # one table buffer: buckets | members | deps | tick_begin | ctrl
            parts = [prog.buckets.tobytes(), prog.members.tobytes(), prog.deps.tobytes(),
                     prog.tick_begin.tobytes()]
            offs, cur = [], 0
            for p in parts:
                offs.append(cur)
                cur = _align(cur + len(p), 16)
            ctrl_off = cur
            total = ctrl_off + 4 * (2 + prog.n_buckets)
            host = np.zeros(_align(total, 16), np.uint8)
            for o, p in zip(offs, parts):
                host[o:o + len(p)] = np.frombuffer(p, np.uint8)
            self.tables = torch.from_numpy(host).to(dev)
            base = self.tables.data_ptr()
            self.arena = torch.empty(prog.arena_elems, dtype=tdt, device=dev)
            self.results = torch.zeros(2 * max(1, len(prog.instances)), dtype=torch.float64, device=dev)
            self.results_host = torch.zeros_like(self.results, device="cpu").pin_memory()
            self.timing = None
            if timing:
                self.timing = torch.zeros(2 * max(1, prog.n_buckets), dtype=torch.int64, device=dev)
                self.timing_init = torch.zeros_like(self.timing)
                self.timing_init[0::2] = np.iinfo(np.int64).max
            self.img_pinned = torch.zeros(max(1, prog.n_input_elems), dtype=tdt).pin_memory()
            self.c = N.ProgramC()
            c = self.c
            c.dtype = DTYPE_CODE[prog.dtype]
            c.n_buckets = prog.n_buckets
            c.n_tickets = prog.n_tickets
            c.smem_bytes = prog.smem_bytes
            c.grid = N.program_grid(c.dtype, prog.smem_bytes)
            c.flags = 0
            c.buckets = base + offs[0]
            c.members = base + offs[1]
            c.deps = base + offs[2]
            c.tick_begin = base + offs[3]
            c.ctrl = base + ctrl_off
            c.arena = self.arena.data_ptr()
            c.results = self.results.data_ptr()
            c.timing = self.timing.data_ptr() if timing else None
        self.grid = c.grid

    # -- input image -------------------------------------------------------
    def stage_inputs(self, raw_parts):
        """raw_parts: per instance, the raw concatenation of its input tensors
        (complex128, each tensor C-order in its own index order)."""
        img = np.zeros(self.prog.n_input_elems, dtype=np.complex128)
        srcs = [raw[s] for raw, s in zip(raw_parts, self.prog.img_src_parts)]
        if srcs:
            img[self.prog.img_dst] = np.concatenate(srcs)
        view = self.img_pinned.numpy()
        view[: len(img)] = img
        n = self.prog.n_input_elems
        if n:
            self.arena[:n].copy_(self.img_pinned[:n], non_blocking=True)

    def launch(self, stream=None):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.timing is not None:
            self.timing.copy_(self.timing_init, non_blocking=True)
        lib = N.load()
        N.check(lib.qtn_program_launch(ctypes.byref(self.c), ctypes.c_void_p(s.cuda_stream)))

    def reset(self, stream=None):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.load().qtn_program_reset(ctypes.byref(self.c), ctypes.c_void_p(s.cuda_stream)))

    def fetch_results(self, stream=None):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.results_host.copy_(self.results, non_blocking=True)
        s.synchronize()
        r = self.results_host.numpy()
        return r[0::2] + 1j * r[1::2]

    def fetch_timing(self):
        t = self.timing.cpu().numpy()
        return t[0::2], t[1::2]

    def run(self, raw_parts, stream=None):
        self.stage_inputs(raw_parts)
        self.launch(stream)
        return self.fetch_results(stream)
