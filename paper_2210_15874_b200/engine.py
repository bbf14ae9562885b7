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
position, the earliest-eliminated axis slowest.  A device item sums k >= 1
indices (a chain of reference buckets merged by the cost model below); its
summed indices are eliminated before all of its result indices, so each
member's element offset is  (pext(s, smask) << popc(mask)) + pext(r, mask).

Many instances (lightcones, slices) can share one program; each instance
ends with a finaliser item that writes its scalar to a result slot.
"""
from __future__ import annotations

import bisect
import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

ELEM_BYTES = {"complex64": 8, "complex128": 16}
DTYPE_CODE = {"complex64": N.QTN_C64, "complex128": N.QTN_C128}
# tile bits: 2^L results per tile (4096 c64 / 2048 c128 = 32 KiB of output)
TILE_BITS = {"complex64": 12, "complex128": 11}
SMEM_BUDGET = 48 * 1024
# intermediate-memory reuse (liveness + WAR dependencies): only for programs
# whose no-reuse footprint exceeds this, and only for blocks >= REUSE_MIN_ELEMS
REUSE_ABOVE_BYTES = int(float(os.environ.get("QTN_REUSE_ABOVE_GB", "16")) * (1 << 30))
REUSE_MIN_ELEMS = 1 << 20
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


KMAX = N.MAX_SUMMED
# summed indices of a merged large item: 3 at both dtypes (complex64 with
# the K4 expansion kernel: cfg-2 0.2487 -> 0.2480 ms, 45-cone graph 9.03 ->
# 8.80 ms, cfg-3 0.267 -> 0.262 s, cfg-4 8.63 -> 8.04 s against 2)
_KL = os.environ.get("QTN_KMAX_LARGE")
KMAX_LARGE = {"complex64": int(_KL) if _KL else 3, "complex128": int(_KL) if _KL else 3}
SMALL_PROD_ELEMS = 1024   # smem products per round of a small tile (csrc)
K2_HI_SLOT = 64           # staged unrounded input member per K2 item (csrc)
VEC = {"complex64": 2, "complex128": 1}
# merge cost model (seconds).  Effective constants, tuned end to end on the
# B200 (sweep over hop cost and term rate, profiles/r01_configs.md): a K1
# dependency hop (~3 us measured + the lost overlap of a serial node) is
# charged 8 us, a hop inside a K2 stage 0.8 us; streaming ~5.5 TB/s; one
# block evaluates ~5e9 member-terms/s (complex64); a small-tile round is
# L2-latency bound (~0.65 us per dependent member load, r01 K2 timeline).
# Tuned values: cfg-2 0.327 -> 0.318 ms, 45-cone graph 10.4 -> 9.5 ms, cfg-3
# 0.286 -> 0.267 s.  Re-swept with K4 and 3-index large merges: multi-
# instance plans charge 12 us (45-cone graph 8.80 -> 8.52 ms; cfg-3 / cfg-4
# unchanged within 0.6 %).  QTN_* environment overrides are for A/B sweeps.
HOP_S = float(os.environ.get("QTN_HOP_S", 12.0e-6))       # K1 graph node (multi-instance programs)
HOP_K2_S = float(os.environ.get("QTN_HOP_K2_S", 0.8e-6))   # item inside a K2 stage
# K1 hop in wave-aware plans (one contraction per graph, nothing to overlap a
# hop with), measured end to end: c64 3 us — cfg-2 0.2484 (5 us) -> 0.2366 ms;
# over the 40 widest N=30 p=4 tight cones the sum is flat (3 us 12.51 ms,
# 5 us 12.49 ms, 8 us 12.61 ms; scripts/hop_check.py); c128 keeps 8 us (5 us
# was 1.4 % slower on cfg-2)
HOP_SINGLE_S = {"complex64": float(os.environ.get("QTN_HOP_SINGLE_C64_S", 3.0e-6)),
                "complex128": float(os.environ.get("QTN_HOP_SINGLE_C128_S", 8.0e-6))}
BW_BPS = float(os.environ.get("QTN_BW_BPS", 5.5e12))
_TERMS_SCALE = float(os.environ.get("QTN_TERMS_SCALE", 1.0))
CHEAP_MEMBER_W = float(os.environ.get("QTN_CHEAP_W", 1.0))   # per-result weight of uniform/invariant members
BLOCK_TERMS_PS = {"complex64": 5.0e9 * _TERMS_SCALE, "complex128": 2.4e9 * _TERMS_SCALE}
RESIDENT_BLOCKS = {"complex64": 296, "complex128": 296}
# Wave-aware tile size: resident K1 blocks (3 per SM at both dtypes) and the
# per-tile fixed cost in result-element equivalents; 0 slots = off.
WAVE_SLOTS = {d: int(os.environ.get("QTN_WAVE_SLOTS", 444)) for d in ("complex64", "complex128")}
WAVE_OV_ELEMS = int(os.environ.get("QTN_WAVE_OV", 2048))
SMALL_LOAD_S = 0.65e-6
MIN_TILE_BITS = {"complex64": 9, "complex128": 8}   # vector path needs VEC*NT results
# items with w + k <= this run in K2 (default per dtype, measured on cfg-2:
# complex64 flat over 12..16, complex128 best at 16: 0.473 -> 0.452 ms)
_SIB = os.environ.get("QTN_SMALL_ITER")
SMALL_ITER_BITS = {"complex64": int(_SIB) if _SIB else 12, "complex128": int(_SIB) if _SIB else 16}
# single-contraction (wave-aware) complex64 plans: one bit lower (cfg-2 0.2366
# -> 0.2337 ms; flat over the 40 widest N=30 p=4 cones, 12.513 vs 12.506 ms)
SMALL_ITER_BITS_SINGLE = {"complex64": int(_SIB) if _SIB else 11, "complex128": SMALL_ITER_BITS["complex128"]}
SMALL_TILE_BITS = {"complex64": 8, "complex128": 7}  # K2 tiles: below one vector step
# QTN_MERGE=0 disables chain merging (A/B measurements)
MERGE_DEFAULT = os.environ.get("QTN_MERGE", "1") != "0"
# producer / consumer pair nodes (K6 in the graph builder; the library knob
# QTN_K6 sets the narrowest producer it fuses, 0 = two kernels per pair)
FUSE_PAIRS = True


@dataclass
class Template:
    """Symbolic plan of one network structure + order (+ sliced indices).

    Two levels: the reference buckets of the replay (one per non-empty
    index in the order, for stats and algorithmic bytes) and the device
    items — chains of reference buckets merged by the cost model, each
    summing k indices.  Offsets are relative to the instance's input /
    intermediate bases."""
    n_in_elems: int
    n_inter_elems: int
    # device items (a topological order)
    w: np.ndarray            # result width
    k: np.ndarray            # summed indices
    L: np.ndarray            # tile bits
    level: np.ndarray
    out_off: np.ndarray      # relative to intermediate base
    mem_ptr: np.ndarray      # CSR into mem_* arrays
    mem_kind: np.ndarray     # 0 = input tensor, 1 = item result
    mem_ref: np.ndarray      # input tensor id or item id
    mem_mask: np.ndarray     # uint64 result-axis coverage
    mem_smask: np.ndarray    # summed-axis coverage
    smem_elems: np.ndarray
    stmask: np.ndarray       # per-thread sequential tile bits (vector path)
    mem_cls: np.ndarray      # member class (CLS_*) for the large-item kernels
    variant: np.ndarray      # kernel variant per item (VARIANT_SMALL = K2 stage)
    # reference buckets (elimination order of non-empty buckets)
    ref_w: np.ndarray
    ref_item: np.ndarray     # item that computes it
    ref_last: np.ndarray     # 1 if it is its item's final bucket
    ref_elems: np.ndarray    # algorithmic elements (sum of member sizes + output)
    bucket_index: np.ndarray
    # finaliser (rank-0 values in reference multiplication order)
    fin_kind: np.ndarray
    fin_ref: np.ndarray
    # inputs
    in_off: np.ndarray       # per input tensor: relative arena offset
    gdst: np.ndarray         # canonical element -> relative input offset
    gsrc: np.ndarray         # ... -> element of the raw concatenated source data
    gfix: dict               # fixed index id -> per-element source offset weight
    n_raw: int
    max_width: int

    @property
    def n_items(self):
        return len(self.w)


def _popc(x):
    return bin(x).count("1")


def _tile_bits(w, masks, smasks, dtype, slots=0):
    """Largest L <= TILE_BITS whose staged runs fit the smem budget; with
    `slots` (resident K1 blocks, wave-aware plans) up to 2 bits smaller when
    that fills the persistent grid's last wave better."""
    esz = ELEM_BYTES[dtype]
    L = min(w, TILE_BITS[dtype])
    while True:
        low = (1 << L) - 1
        st = sum(((1 << _popc(sm)) << _popc(m & low)) + 1 for m, sm in zip(masks, smasks) if (m & low) != low)
        st += 1 << KMAX   # U[s] (tile-uniform product)
        if st * esz <= SMEM_BUDGET or L == 0:
            break
        L -= 1
    if slots > 0:
        # wave-aware: a smaller tile when the last wave of the persistent grid
        # would run mostly empty (up to 2 bits smaller, ties keep the larger)
        best, best_t = L, None
        for l in range(L, max(min(w, MIN_TILE_BITS[dtype]), L - 2) - 1, -1):
            t = -(-(1 << (w - l)) // slots) * ((1 << l) + WAVE_OV_ELEMS)
            if best_t is None or t < best_t:
                best, best_t = l, t
        if best != L:
            L = best
            low = (1 << L) - 1
            st = sum(((1 << _popc(sm)) << _popc(m & low)) + 1 for m, sm in zip(masks, smasks) if (m & low) != low)
            st += 1 << KMAX
    return L, st


def _step_mask(L, masks, dtype):
    """Tile bits each thread walks sequentially (vector path): among the bits
    above lane + warp-minimum positions choose the subset that leaves the most
    partially-covering (staged) members invariant, so they are multiplied
    once per tile (csrc vec_tile_hoist)."""
    lb = 1 if VEC[dtype] == 2 else 0
    n_st = L - lb - 8
    if n_st <= 0:
        return 0
    full = (1 << L) - 1
    staged = [m & full for m in masks if (m & full) != full]
    best, best_key = 0, None
    from itertools import combinations
    for bits in combinations(range(lb + 5, L), n_st):
        sm = sum(1 << b for b in bits)
        inv = sum(1 for m in staged if (m & sm) == 0)
        key = (inv, sm)           # ties: prefer the higher bits
        if best_key is None or key > best_key:
            best, best_key = sm, key
    return best


CLS_STREAMED, CLS_UNIFORM, CLS_INVARIANT, CLS_VARYING = 0, 1, 2, 3
VARIANT_SMALL = -2
VARIANT_GENERIC = N.QTN_VARIANT_GENERIC


def member_classes(w, k, L, stm, masks):
    """Per-member class for the large-item kernels (csrc large_kernel)."""
    full = (1 << L) - 1
    out = []
    for m in masks:
        lo = m & full
        if lo == full:
            out.append(CLS_STREAMED)
        elif lo == 0:
            out.append(CLS_UNIFORM)
        elif k <= 3 and (lo & stm) == 0:
            out.append(CLS_INVARIANT)
        else:
            out.append(CLS_VARYING)
    return out


def kernel_variant(w, k, L, cls, dtype, masks=()):
    """K2 small stage for tiles below one vector step; otherwise the K1
    specialisation (2^k, varying members, streamed) or the generic kernel."""
    if (1 << L) < VEC[dtype] * NT:
        return VARIANT_SMALL
    nv = sum(1 for c in cls if c == CLS_VARYING)
    nst = sum(1 for c in cls if c == CLS_STREAMED)
    if k <= 3 and nv <= 4 and nst <= 1:
        # varying members carrying result bit 0 (c64: 16-byte v-pair gathers)
        nb0 = sum(1 for c, m in zip(cls, masks) if c == CLS_VARYING and m & 1) if VEC[dtype] == 2 else 0
        return k | (nv << 4) | (nst << 8) | (nb0 << 12)
    return VARIANT_GENERIC


def _item_cost(w, k, L, sizes, dtype, hop=None, nm_eff=None):
    """Estimated device time of one item: dependency hop + max(streaming,
    per-tile term evaluation x waves of tiles).  nm_eff: members weighted by
    their per-result cost (large items: uniform / invariant members count
    CHEAP_MEMBER_W, see _cost_of)."""
    hop = HOP_S if hop is None else hop
    nm = max(1, len(sizes)) if nm_eff is None else nm_eff
    byt = ELEM_BYTES[dtype] * ((1 << w) + sum(sizes))
    tiles = 1 << (w - L)
    waves = -(-tiles // RESIDENT_BLOCKS[dtype])
    nelem = 1 << L
    if nelem >= VEC[dtype] * NT:
        per_tile = (nelem << k) * nm / BLOCK_TERMS_PS[dtype]
    else:
        # K2: each thread handles 2 (element, assignment) units per round; all
        # member loads of a round are in flight together (one L2 round trip)
        rounds = -(-(nelem << k) // (2 * NT))
        per_tile = 1e-6 + rounds * SMALL_LOAD_S
    return hop + max(byt / BW_BPS, waves * per_tile)


def _cost_of(it, dtype, small_iter_bits=None, slots=0):
    sib = SMALL_ITER_BITS[dtype] if small_iter_bits is None else small_iter_bits
    masks, smasks = _masks(it["members"], it["X"], it["R"])
    w, k = len(it["R"]), len(it["X"])
    if w + k <= sib:
        L = min(w, SMALL_TILE_BITS[dtype])
        return _item_cost(w, k, L, [1 << len(s2) for _, _, s2 in it["members"]], dtype, hop=HOP_K2_S)
    L, _ = _tile_bits(w, masks, smasks, dtype, slots)
    nm_eff = None
    if CHEAP_MEMBER_W != 1.0 and (1 << L) >= VEC[dtype] * NT:
        stm = _step_mask(L, masks, dtype)
        cls = member_classes(w, k, L, stm, masks)
        n_cheap = sum(1 for c in cls if c in (CLS_UNIFORM, CLS_INVARIANT))
        nm_eff = max(1.0, (len(cls) - n_cheap) + CHEAP_MEMBER_W * n_cheap)
    return _item_cost(len(it["R"]), len(it["X"]), L, [1 << len(s2) for _, _, s2 in it["members"]], dtype,
                      hop=HOP_SINGLE_S[dtype] if slots else HOP_S, nm_eff=nm_eff)


def small_iter_bits_for(threshold, dtype="complex64", single=False):
    """Backend.threshold (result width at or below which a bucket runs in the
    batched small-bucket schedule, the analogue of the reference's Mixed
    threshold, src/tensor_core.py:176-184) -> iteration bits (w + k) of the
    K2 routing rule; None -> the measured per-dtype default (`single`: for a
    program that runs one contraction alone, see SMALL_ITER_BITS_SINGLE)."""
    if threshold is None:
        return (SMALL_ITER_BITS_SINGLE if single else SMALL_ITER_BITS)[norm_dtype(dtype)]
    return int(threshold) + 1


def _plan_params(dtype, merge, sib, wave_aware=False):
    return N.PlanParamsC(
        elem_bytes=ELEM_BYTES[dtype], tile_bits=TILE_BITS[dtype], small_tile_bits=SMALL_TILE_BITS[dtype],
        min_tile_bits=MIN_TILE_BITS[dtype], kmax=KMAX, max_members=N.MAX_MEMBERS, vec=VEC[dtype], nt=NT,
        small_iter_bits=sib, merge=1 if merge else 0, resident_blocks=RESIDENT_BLOCKS[dtype],
        smem_budget=SMEM_BUDGET, hop_s=HOP_SINGLE_S[dtype] if wave_aware else HOP_S, hop_k2_s=HOP_K2_S,
        bw_bps=BW_BPS,
        block_terms_ps=BLOCK_TERMS_PS[dtype], small_load_s=SMALL_LOAD_S, cheap_member_w=CHEAP_MEMBER_W,
        kmax_large=KMAX_LARGE[dtype], wave_slots=WAVE_SLOTS[dtype] if wave_aware else 0,
        wave_ov_elems=WAVE_OV_ELEMS)


def plan_template(index_sets, order, dtype, fixed=(), merge=None, small_iter_bits=None, wave_aware=False):
    """The symbolic plan of one network structure + order (+ sliced
    indices), computed by the native planner (csrc/plan_template.cpp,
    qtn_plan_build) — the C++ restatement of plan_template_py below, which
    stays as its checker (tests compare the two array by array).

    wave_aware: the program will run this network alone (one contraction per
    graph launch), so large items pick tile sizes that fill the last wave of
    the persistent grid; programs of many instances overlap items instead and
    keep the largest tiles."""
    dtype = norm_dtype(dtype)
    merge = MERGE_DEFAULT if merge is None else merge
    sib = small_iter_bits_for(None, dtype, wave_aware) if small_iter_bits is None else int(small_iter_bits)
    fixed = list(dict.fromkeys(int(f) for f in fixed))
    sc, a = N.plan_build(index_sets, order, fixed, _plan_params(dtype, merge, sib, wave_aware))
    ncanon = len(a["gdst"])
    gfix = {f: a["gfix"][j * ncanon:(j + 1) * ncanon] for j, f in enumerate(fixed)}
    return Template(
        n_in_elems=int(sc[0]), n_inter_elems=int(sc[1]),
        w=a["w"], k=a["k"], L=a["L"], level=a["level"], out_off=a["out_off"], mem_ptr=a["mem_ptr"],
        mem_kind=a["mem_kind"], mem_ref=a["mem_ref"], mem_mask=a["mem_mask"].view(np.uint64),
        mem_smask=a["mem_smask"].view(np.uint64), smem_elems=a["smem_elems"], stmask=a["stmask"],
        mem_cls=a["mem_cls"], variant=a["variant"],
        ref_w=a["ref_w"], ref_item=a["ref_item"], ref_last=a["ref_last"], ref_elems=a["ref_elems"],
        bucket_index=a["bucket_index"], fin_kind=a["fin_kind"], fin_ref=a["fin_ref"],
        in_off=a["in_off"], gdst=a["gdst"], gsrc=a["gsrc"], gfix=gfix, n_raw=int(sc[2]),
        max_width=int(sc[3]),
    )


def plan_template_py(index_sets, order, dtype, fixed=(), merge=None, small_iter_bits=None, wave_aware=False):
    """Replay contract_network's bucket assignment (src/ordering.py:165-187)
    over index sets only and freeze it into a Template.

    index_sets: per input tensor, its indices in its own storage order
    (before slicing).  `fixed` indices are sliced out (src/ordering.py:233-248).
    merge: fold chains of buckets into k-sum items when the cost model says
    the saved hop latency / HBM round trip outweighs the extra multiplies.
    small_iter_bits: items with w + k <= this run in a K2 small stage
    (default SMALL_ITER_BITS = Backend threshold 11 + 1)."""
    dtype = norm_dtype(dtype)
    sib = small_iter_bits_for(None, dtype, wave_aware) if small_iter_bits is None else int(small_iter_bits)
    merge = MERGE_DEFAULT if merge is None else merge
    slots = WAVE_SLOTS[dtype] if wave_aware else 0
    fixed = set(int(f) for f in fixed)
    act = [int(i) for i in order if int(i) not in fixed]
    pos = {x: k for k, x in enumerate(act)}

    # ---- inputs: canonical layout and gather maps ----
    # (plain-Python index arithmetic: gate tensors have rank <= 4, where numpy
    # per-tensor calls would dominate; permutation tables are memoised)
    n_raw = 0
    in_off = np.full(len(index_sets), -1, dtype=np.int64)
    cur = 0
    gd, gs = [], []
    gfix = {f: [] for f in fixed}
    sets = []
    perm_cache = {}
    for t, idx in enumerate(index_sets):
        idx = tuple(int(i) for i in idx)
        r0 = len(idx)
        kept = [i for i in idx if i not in fixed] if fixed else list(idx)
        for i in kept:
            if i not in pos:
                raise ValueError(f"order is missing indices: {sorted(set(kept) - set(pos))}")
        canon = sorted(kept, key=pos.__getitem__)
        r = len(canon)
        size = 1 << r
        cur = _align(cur, _tensor_align(size))
        in_off[t] = cur
        weights = tuple(1 << (r0 - 1 - idx.index(a)) for a in canon)
        key = (r, weights)
        tab = perm_cache.get(key)
        if tab is None:
            tab = [sum(w for p_, w in enumerate(weights) if (k >> (r - 1 - p_)) & 1) for k in range(size)]
            perm_cache[key] = tab
        gd.extend(range(cur, cur + size))
        gs.extend(n_raw + x for x in tab)
        for f in fixed:
            wgt = (1 << (r0 - 1 - idx.index(f))) if f in idx else 0
            gfix[f].extend([wgt] * size)
        cur += size
        n_raw += 1 << r0
        sets.append(frozenset(kept))
    n_in = _align(cur, 32)
    gdst = np.asarray(gd, dtype=np.int64)
    gsrc = np.asarray(gs, dtype=np.int64)
    gfix = {f: np.asarray(v, dtype=np.int64) for f, v in gfix.items()}

    # ---- reference bucket replay ----
    pending = {x: [] for x in act}
    fin = []      # (kind, ref): kind 0 input tensor, kind 1 reference bucket
    for t, st in enumerate(sets):
        if not st:
            fin.append((0, t))
        else:
            pending[min(st, key=pos.__getitem__)].append((0, t, st))
    refs = []     # (x, members, R)
    for x in act:
        mem = pending.pop(x)
        if not mem:
            continue
        union = set()
        for _, _, st in mem:
            union |= st
        union.discard(x)
        R = sorted(union, key=pos.__getitem__)
        if len(R) > N.MAX_WIDTH:
            raise ValueError(f"bucket width {len(R)} exceeds {N.MAX_WIDTH}")
        b = len(refs)
        refs.append((x, mem, R))
        if R:
            pending[R[0]].append((1, b, frozenset(R)))
        else:
            fin.append((1, b))

    # ---- merge chains into items ----
    items = []           # dict(X, R, members[(kind, ref(item|input), set)], refs)
    item_of = []
    for b, (x, mem, R) in enumerate(refs):
        it = {"X": [x], "R": R, "refs": [b],
              "members": [(k_, (item_of[r_] if k_ == 1 else r_), st) for k_, r_, st in mem]}
        it["cost"] = _cost_of(it, dtype, sib, slots)
        changed = merge
        while changed:
            changed = False
            for mi, (k_, r_, st) in enumerate(it["members"]):
                if k_ != 1 or items[r_] is None:
                    continue
                p_ = items[r_]
                X2 = sorted(set(it["X"]) | set(p_["X"]), key=pos.__getitem__)
                mem2 = it["members"][:mi] + p_["members"] + it["members"][mi + 1:]
                if len(X2) > KMAX or len(mem2) > N.MAX_MEMBERS:
                    continue
                w = len(R)
                cand = {"X": X2, "R": R, "members": mem2}
                if w + len(X2) > sib:
                    masks, smasks = _masks(mem2, X2, R)
                    L, _ = _tile_bits(w, masks, smasks, dtype, slots)
                    if L < min(w, MIN_TILE_BITS[dtype]):
                        continue
                if w + len(X2) > sib and len(X2) > KMAX_LARGE[dtype]:
                    continue   # k > 3 would need the generic K1 kernel (no specialisation)
                c2 = _cost_of(cand, dtype, sib, slots)
                if c2 >= it["cost"] + p_["cost"]:
                    continue
                it["X"], it["members"], it["cost"] = X2, mem2, c2
                it["refs"] = p_["refs"] + it["refs"]
                items[r_] = None
                changed = True
                break
        item_of.append(len(items))
        items.append(it)
    # compact (drop absorbed items) and renumber
    live = [i for i, it in enumerate(items) if it is not None]
    renum = {old: new for new, old in enumerate(live)}
    W, K, Ls, lev, outo, mptr, mkind, mref, mmask, msmask, smem, stm, mcls, var = ([] for _ in range(14))
    mptr.append(0)
    inter = 0
    ref_item = np.zeros(len(refs), np.int64)
    ref_last = np.zeros(len(refs), np.int64)
    for new, old in enumerate(live):
        it = items[old]
        R, X = it["R"], it["X"]
        w, k = len(R), len(X)
        masks, smasks = _masks(it["members"], X, R)
        if w + k <= sib:
            # small iteration space: K2 stage, scalar-path tiles (latency-bound
            # work; a K2 dependency hop costs ~1.5 us against ~7 us for a K1 node)
            L, st = min(w, SMALL_TILE_BITS[dtype]), 0
        else:
            L, st = _tile_bits(w, masks, smasks, dtype, slots)
        lv = 0
        for (k_, r_, _), m, sm in zip(it["members"], masks, smasks):
            if k_ == 1:
                r_ = renum[r_]
                lv = max(lv, lev[r_] + 1)
            mkind.append(k_)
            mref.append(r_)
            mmask.append(m)
            msmask.append(sm)
        mptr.append(len(mkind))
        size = 1 << w
        inter = _align(inter, _tensor_align(size))
        W.append(w); K.append(k); Ls.append(L); lev.append(lv); outo.append(inter); smem.append(st)
        sm_ = _step_mask(L, masks, dtype) if (1 << L) >= VEC[dtype] * NT else 0
        stm.append(sm_)
        cls_ = member_classes(w, k, L, sm_, masks)
        mcls.extend(cls_)
        var.append(kernel_variant(w, k, L, cls_, dtype, masks))
        inter += size
        for r_ in it["refs"]:
            ref_item[r_] = new
        ref_last[it["refs"][-1]] = 1
    ref_w = np.array([len(R) for _, _, R in refs], np.int64)
    ref_elems = np.array([(1 << len(R)) + sum(1 << len(st) for _, _, st in mem) for _, mem, R in refs], np.int64)
    fin_kind = np.array([k_ for k_, _ in fin], np.int64)
    fin_ref = np.array([(ref_item[r_] if k_ == 1 else r_) for k_, r_ in fin], np.int64)
    return Template(
        n_in_elems=n_in, n_inter_elems=_align(inter, 32),
        w=np.array(W, np.int64), k=np.array(K, np.int64), L=np.array(Ls, np.int64),
        level=np.array(lev, np.int64), out_off=np.array(outo, np.int64), mem_ptr=np.array(mptr, np.int64),
        mem_kind=np.array(mkind, np.int64), mem_ref=np.array(mref, np.int64),
        mem_mask=np.array(mmask, np.uint64), mem_smask=np.array(msmask, np.uint64),
        smem_elems=np.array(smem, np.int64), stmask=np.array(stm, np.int64),
        mem_cls=np.array(mcls, np.int64), variant=np.array(var, np.int64),
        ref_w=ref_w, ref_item=ref_item, ref_last=ref_last, ref_elems=ref_elems,
        bucket_index=np.array([x for x, _, _ in refs], np.int64),
        fin_kind=fin_kind, fin_ref=fin_ref,
        in_off=in_off, gdst=gdst, gsrc=gsrc, gfix=gfix, n_raw=n_raw,
        max_width=int(ref_w.max()) if len(ref_w) else 0,
    )


def _masks(members, X, R):
    """Result / summed coverage masks: bit j <-> R[w-1-j] / X[k-1-j]."""
    w, k = len(R), len(X)
    rbit = {a: w - 1 - j for j, a in enumerate(R)}
    sbit = {a: k - 1 - j for j, a in enumerate(X)}
    masks, smasks = [], []
    for _, _, st in members:
        m = sm = 0
        for a in st:
            if a in rbit:
                m |= 1 << rbit[a]
            else:
                sm |= 1 << sbit[a]   # KeyError = a planner bug (index outside X and R)
        masks.append(m)
        smasks.append(sm)
    return masks, smasks


def algorithmic_bytes(t: Template, dtype) -> int:
    """per reference bucket (sum_members 2^rank_i + 2^w) * sizeof(elem)."""
    return int(t.ref_elems.sum()) * ELEM_BYTES[norm_dtype(dtype)]


def executed_bytes(t: Template, dtype) -> int:
    """Bytes the device items must move: every item reads each member once
    and writes its result once (merged chains skip the intermediates)."""
    tot = 0
    for i in range(t.n_items):
        tot += 1 << int(t.w[i])
        for j in range(t.mem_ptr[i], t.mem_ptr[i + 1]):
            tot += 1 << (_popc(int(t.mem_mask[j])) + _popc(int(t.mem_smask[j])))
    return tot * ELEM_BYTES[norm_dtype(dtype)]


def _blk_start(blk):
    return blk[0]


class _Pool:
    """Best-fit arena allocator over element offsets with free-block
    coalescing.  A freed block remembers the items that last READ it; an
    allocation that reuses any of its memory inherits them as write-after-read
    dependencies."""

    def __init__(self, base):
        self.top = base
        self.free = []          # [start, size, readers(set)] sorted by start, coalesced

    def alloc(self, size, align):
        size = _align(size, align)
        best = None
        for bi, (st, sz, _) in enumerate(self.free):
            a = _align(st, align)
            if a + size <= st + sz and (best is None or sz < self.free[best][1]):
                best = bi
        if best is not None:
            st, sz, rd = self.free.pop(best)
            a = _align(st, align)
            if a > st:
                self._insert(st, a - st, set(rd))
            if a + size < st + sz:
                self._insert(a + size, st + sz - a - size, set(rd))
            return a, set(rd)
        if self.free and self.free[-1][0] + self.free[-1][1] == self.top:
            st, sz, rd = self.free.pop()      # extend the top free block
            a = _align(st, align)
            if a > st:
                self._insert(st, a - st, set(rd))
            self.top = a + size
            return a, set(rd)
        a = _align(self.top, align)
        self.top = a + size
        return a, set()

    def release(self, start, size, reader):
        self._insert(start, size, {reader})

    def _insert(self, st, sz, rd):
        # the list is sorted and coalesced (no two blocks touch): only the
        # neighbours of the new block can merge with it
        free = self.free
        i = bisect.bisect_left(free, st, key=_blk_start)
        if i > 0 and free[i - 1][0] + free[i - 1][1] == st:
            prev = free[i - 1]
            prev[1] += sz
            prev[2] = prev[2] | rd
            if i < len(free) and prev[0] + prev[1] == free[i][0]:
                nxt = free.pop(i)
                prev[1] += nxt[1]
                prev[2] = prev[2] | nxt[2]
        elif i < len(free) and st + sz == free[i][0]:
            nxt = free[i]
            nxt[0] = st
            nxt[1] += sz
            nxt[2] = rd | nxt[2]
        else:
            free.insert(i, [st, sz, rd])


def template_peak_elems(t: Template) -> int:
    """Peak intermediate elements of one instance under the liveness-based
    reuse of Program (same allocator, items in level order)."""
    order = sorted(range(t.n_items), key=lambda b: (int(t.level[b]), b))
    pool = _Pool(0)
    off = {}
    for b in order:
        size = 1 << int(t.w[b])
        off[b], _ = pool.alloc(size, _tensor_align(size))
        for j in range(t.mem_ptr[b], t.mem_ptr[b + 1]):
            if t.mem_kind[j] == 1:
                r = int(t.mem_ref[j])
                pool.release(off[r], 1 << int(t.w[r]), b)
    return pool.top


@dataclass
class Instance:
    template: Template
    assignment: dict = field(default_factory=dict)   # fixed index -> 0/1


def _template_lists(t: Template) -> dict:
    """Python-list copies of a template's item/member tables (cached on it)."""
    tl = getattr(t, "_lists", None)
    if tl is None:
        tl = {name: getattr(t, name).tolist() for name in
              ("w", "k", "L", "level", "smem_elems", "stmask", "variant", "mem_ptr", "mem_kind", "mem_ref",
               "mem_mask", "mem_smask", "mem_cls", "in_off", "fin_kind", "fin_ref")}
        t._lists = tl
    return tl


class Program:
    """Several instances laid out in one arena, their items grouped into the
    nodes of one CUDA graph.

    Items of all instances are ordered by (level, instance, item) — a
    topological order.  Large items (K1 variants) are one node each; small
    items (VARIANT_SMALL: tiles below one vector step) and finalisers are
    batched into persistent K2 stages.  A small item joins the open stage
    unless it depends on a large node created after the stage was opened
    (that would be a cycle); dependencies inside a stage are per-item
    completion counters, across nodes they are graph edges."""

    def __init__(self, instances, dtype, reuse_above=None):
        self.dtype = norm_dtype(dtype)
        self.instances = list(instances)
        esz = ELEM_BYTES[self.dtype]
        n_in = 0
        in_base = []
        for inst in self.instances:
            in_base.append(n_in)
            n_in += inst.template.n_in_elems
        n_in = _align(n_in, 32)
        self.n_input_elems = n_in
        self.in_base = in_base

        # ---- global item order (topological) ----
        tls = [_template_lists(inst.template) for inst in self.instances]
        keys = []
        for i, tl in enumerate(tls):
            lev = tl["level"]
            keys.extend((lev[b], i, b) for b in range(len(lev)))
            keys.append(((max(lev) + 1) if lev else 0, i, -1))  # finaliser
        keys.sort(key=lambda q: (q[0], q[1], q[2] if q[2] >= 0 else 1 << 40))

        # ---- producers of every item (global ids) ----
        order_gid = {(i, b): g for g, (_, i, b) in enumerate(keys)}
        prods = []
        for (_, i, b) in keys:
            tl = tls[i]
            if b >= 0:
                mk, mr = tl["mem_kind"], tl["mem_ref"]
                ps = [order_gid[(i, mr[j])] for j in range(tl["mem_ptr"][b], tl["mem_ptr"][b + 1]) if mk[j] == 1]
            else:
                ps = [order_gid[(i, r)] for kd, r in zip(tl["fin_kind"], tl["fin_ref"]) if kd == 1]
            prods.append(ps)

        # ---- intermediates: liveness-based reuse in item order ----
        # An item's output is allocated before its inputs are released; a
        # block freed by its reader R and reused by writer W makes W depend on
        # R (write-after-read), folded into the graph / stage dependencies.
        # Reuse costs concurrency (WAR edges), so it is used only when the
        # program would not fit otherwise, and only for large blocks.
        no_reuse = sum(inst.template.n_inter_elems for inst in self.instances) * esz
        self.reuse = (REUSE_ABOVE_BYTES if reuse_above is None else reuse_above) < no_reuse
        pool = _Pool(n_in)
        small_pool = _Pool(0)   # never reused; placed after the reusable pool
        out_elem, war = {}, [set() for _ in keys]
        wid, in_small = {}, set()
        for g, (_, i, b) in enumerate(keys):
            if b >= 0:
                size = 1 << tls[i]["w"][b]
                wid[g] = size
                if self.reuse and size >= REUSE_MIN_ELEMS:
                    off, readers = pool.alloc(size, _tensor_align(size))
                    war[g] = readers - {g}
                else:
                    off, _ = small_pool.alloc(size, _tensor_align(size))
                    in_small.add(g)
                out_elem[g] = off
            for p_ in prods[g]:
                if p_ not in in_small:
                    pool.release(out_elem[p_], wid[p_], g)
        small_base = _align(pool.top, 32)
        for g in in_small:
            out_elem[g] += small_base
        self.arena_elems = max(_align(small_base + small_pool.top, 32), 32)
        # complex64: the input region also as complex128 in front of the arena
        # (qtn_program_t.inputs_hi; K2 stages read the gates unrounded) —
        # counted in arena elements: 2 complex64 slots per complex128 value
        self.hi_elems = 2 * n_in if self.dtype == "complex64" else 0
        self.device_elems = self.hi_elems + self.arena_elems
        deps_all = [sorted(set(prods[g]) | war[g]) for g in range(len(keys))]

        # ---- nodes: large items alone, small items in stages ----
        def is_small(q):
            _, i, b = q
            return b < 0 or tls[i]["variant"][b] == VARIANT_SMALL

        # producer / consumer pairs (one node, K6 in the graph builder)
        self.fused = self._pairs(keys, tls, order_gid, prods, deps_all, war, is_small) if FUSE_PAIRS else {}
        fused_c = {c: p_ for p_, c in self.fused.items()}
        node_of = [-1] * len(keys)
        nodes = []           # dict(kind, items, deps:set)
        open_stage = -1
        for g, q in enumerate(keys):
            if g in self.fused:
                continue          # placed with its consumer
            if g in fused_c:
                p_ = fused_c[g]
                ext = {node_of[x] for x in set(deps_all[p_]) | set(deps_all[g]) if x not in (p_, g)}
                nodes.append({"kind": N.QTN_NODE_LARGE, "items": [p_, g], "deps": ext})
                node_of[p_] = node_of[g] = len(nodes) - 1
                continue
            ext = {node_of[p] for p in deps_all[g]}
            if is_small(q):
                # join the open stage unless a producer is a node created after it
                if open_stage >= 0 and all(n <= open_stage for n in ext):
                    nd = open_stage
                else:
                    nodes.append({"kind": N.QTN_NODE_SMALL, "items": [], "deps": set()})
                    open_stage = len(nodes) - 1
                    nd = open_stage
                nodes[nd]["items"].append(g)
                nodes[nd]["deps"] |= {n for n in ext if n != nd}
                node_of[g] = nd
            else:
                nodes.append({"kind": N.QTN_NODE_LARGE, "items": [g], "deps": set(ext)})
                node_of[g] = len(nodes) - 1

        # ---- final item numbering: node by node (stage items contiguous) ----
        new_of = {}
        for nd in nodes:
            for g in nd["items"]:
                new_of[g] = len(new_of)
        item_keys = [None] * len(keys)
        for g, q in enumerate(keys):
            item_keys[new_of[g]] = (q, g)

        nb = len(keys)
        # tables built from plain Python lists (numpy scalar field writes cost
        # ~1 us each; cfg-4 batches have thousands of items)
        recs = [None] * nb
        members, deps = [], []
        smem_max = 0
        self.bucket_gid = [np.zeros(inst.template.n_items, np.int64) for inst in self.instances]
        self.fin_gid = [0] * len(self.instances)
        ntiles = [0] * nb
        for gid, ((_, i, b), g) in enumerate(item_keys):
            tl = tls[i]
            ntiles[gid] = (1 << (tl["w"][b] - tl["L"][b])) if b >= 0 else 1
            if b >= 0:
                self.bucket_gid[i][b] = gid
            else:
                self.fin_gid[i] = gid
        node_list = []
        node_deps = []
        small_kind = N.QTN_NODE_SMALL
        for ni, nd in enumerate(nodes):
            gids = [new_of[g] for g in nd["items"]]
            first, count = min(gids), len(gids)
            assert gids == list(range(first, first + count))
            tick = 0
            is_stage = nd["kind"] == small_kind
            # K2 stage: double-precision products + staged unrounded input members
            node_smem = SMALL_PROD_ELEMS * 16 + N.MAX_MEMBERS * K2_HI_SLOT * 16 if is_stage else 0
            variant = 0
            pair_variant = 0   # LARGE pair: the producer's K1 variant (qtn_node_t.n_tickets)
            for gid in gids:
                (_, i, b), g = item_keys[gid]
                tl = tls[i]
                ib = in_base[i]
                mem_begin, dep_begin = len(members), len(deps)
                if b >= 0:
                    in_off, mk, mr = tl["in_off"], tl["mem_kind"], tl["mem_ref"]
                    mm, msm, mc = tl["mem_mask"], tl["mem_smask"], tl["mem_cls"]
                    j0, j1 = tl["mem_ptr"][b], tl["mem_ptr"][b + 1]
                    for j in range(j0, j1):
                        ref = mr[j]
                        off = ib + in_off[ref] if mk[j] == 0 else out_elem[order_gid[(i, ref)]]
                        members.append((off, mm[j], msm[j], mc[j]))
                    if not is_stage:
                        if gid == first and count == 2:
                            pair_variant = tl["variant"][b]
                            smem_max = max(smem_max, _align(tl["smem_elems"][b] * esz, 16))
                        variant = tl["variant"][b]
                        node_smem = _align(tl["smem_elems"][b] * esz, 16)
                    w_, k_, L_, out_, slot_, nmem_ = tl["w"][b], tl["k"][b], tl["L"][b], out_elem[g], -1, j1 - j0
                    smem_, stm_ = tl["smem_elems"][b], tl["stmask"][b]
                else:
                    in_off = tl["in_off"]
                    for kd, ref in zip(tl["fin_kind"], tl["fin_ref"]):
                        off = ib + in_off[ref] if kd == 0 else out_elem[order_gid[(i, ref)]]
                        members.append((off, 0, 0, 0))
                    w_, k_, L_, out_, slot_, nmem_ = N.QTN_FINALIZE, 0, 0, 0, i, len(tl["fin_kind"])
                    smem_, stm_ = 0, 0
                # completion dependencies inside this stage (RAW + WAR; a
                # pair node's consumer follows its producer in stream order)
                for dg in (deps_all[g] if is_stage else ()):
                    if node_of[dg] == ni:
                        pg = new_of[dg]
                        deps.append((pg, ntiles[pg]))
                # BUCKET_DT field order
                recs[gid] = (out_, w_, L_, k_, mem_begin, nmem_, dep_begin, len(deps) - dep_begin,
                             tick if is_stage else 0, ntiles[gid], slot_, smem_, stm_, 0, 0)
                tick += ntiles[gid]
            smem_max = max(smem_max, node_smem)
            dl = sorted(nd["deps"])
            node_list.append((nd["kind"], first, count, tick if is_stage else pair_variant,
                              variant, len(node_deps), len(dl), node_smem))
            node_deps.extend(dl)
        B = np.array(recs, dtype=N.BUCKET_DT) if nb else np.zeros(0, N.BUCKET_DT)
        if max(int(n[3]) for n in node_list) >= 2 ** 31 - 1:
            raise ValueError("program stage too large (ticket space)")
        self.n_buckets = nb
        self.nodes = np.array(node_list, dtype=N.NODE_DT)
        self.node_deps = np.array(node_deps if node_deps else [0], dtype=np.int32)
        self.n_nodes = len(node_list)
        self.smem_bytes = smem_max
        self.buckets = B
        self.members = np.array(members, dtype=N.MEMBER_DT) if members else np.zeros(1, N.MEMBER_DT)
        self.deps = np.array(deps, dtype=N.DEP_DT) if deps else np.zeros(1, N.DEP_DT)
        self.tick_begin = np.ascontiguousarray(B["tick_begin"]).astype(np.int32)
        # input image gather (per instance, slice assignment applied)
        dst, src = [], []
        for i, inst in enumerate(self.instances):
            t = inst.template
            s_ = t.gsrc.copy()
            for f, bitv in inst.assignment.items():
                if int(bitv):
                    s_ += t.gfix[int(f)]
            dst.append(in_base[i] + t.gdst)
            src.append(s_)
        self.img_dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
        self.img_src_parts = src

    @staticmethod
    def _pairs(keys, tls, order_gid, prods, deps_all, war, is_small):
        """Producer -> consumer pairs for K6 (csrc/bucket_expand.cu): the
        consumer C is a large item reading the producer P's whole result as a
        member that carries every result and summed index of C (P.w = C.w +
        C.k, C.k <= 3), P is a large item with k <= 3 read by C alone, and no
        other item waits for P (no write-after-read edge on P's inputs), and
        C's result does not reuse memory P reads (K6 reads P's members while
        it writes C's result: a reused block would be overwritten in flight).  The
        pair becomes one node; the graph builder runs it as one K6 kernel when
        P is a K4 expansion with C's summed bits set aside (else as two
        kernels).  A producer is never itself a consumer of another pair."""
        dependents = {}
        for g, ds in enumerate(deps_all):
            for d in ds:
                dependents.setdefault(d, set()).add(g)
        readers = {}
        for g, ps in enumerate(prods):
            for p_ in ps:
                readers[p_] = readers.get(p_, 0) + 1
        pairs, used = {}, set()
        for g, (_, i, b) in enumerate(keys):
            if b < 0 or is_small(keys[g]) or g in used:
                continue
            tl = tls[i]
            w, k = tl["w"][b], tl["k"][b]
            if not 1 <= k <= 3:
                continue
            for j in range(tl["mem_ptr"][b], tl["mem_ptr"][b + 1]):
                if tl["mem_kind"][j] != 1:
                    continue
                if tl["mem_mask"][j] != (1 << w) - 1 or tl["mem_smask"][j] != (1 << k) - 1:
                    continue
                pb = tl["mem_ref"][j]
                p_ = order_gid[(i, pb)]
                if p_ in used or is_small(keys[p_]) or not 1 <= tl["k"][pb] <= 3 or tl["w"][pb] != w + k:
                    continue
                if readers.get(p_, 0) != 1 or dependents.get(p_, set()) != {g} or p_ in war[g]:
                    continue
                pairs[p_] = g
                used |= {p_, g}
                break
        return pairs

    def algorithmic_bytes(self) -> int:
        return sum(algorithmic_bytes(inst.template, self.dtype) for inst in self.instances)

    def executed_bytes(self) -> int:
        return sum(executed_bytes(inst.template, self.dtype) for inst in self.instances)

    def item_bytes(self, gid) -> int:
        """Compulsory bytes of device item `gid`: each member read once, the
        result written once (the item's roofline numerator)."""
        b = self.buckets[gid]
        if int(b["w"]) < 0:
            return 0
        mem = self.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
        n = (1 << int(b["w"])) + sum(1 << (_popc(int(m["mask"])) + _popc(int(m["smask"]))) for m in mem)
        return n * ELEM_BYTES[self.dtype]

    def node_of_item(self):
        """gid -> graph node index."""
        out = {}
        for ni, nd in enumerate(self.nodes):
            for g in range(int(nd["first"]), int(nd["first"]) + int(nd["count"])):
                out[g] = ni
        return out

    def describe(self):
        kinds = self.nodes["kind"]
        return {"items": int(self.n_buckets), "nodes": int(self.n_nodes),
                "small_stages": int((kinds == N.QTN_NODE_SMALL).sum()),
                "large_items": int((kinds == N.QTN_NODE_LARGE).sum())}


class _OwnedGraph:
    """A qtn_graph_t destroyed with its Python owner."""

    def __init__(self, g):
        self.g = g

    def __del__(self):
        if self.g is not None and self.g.value:
            try:
                N.load().qtn_graph_destroy(self.g)
            except Exception:
                pass


class Executor:
    """Device-resident copy of a Program: tables, control block, arena and
    result slots owned by torch; the node graph is built once through the C
    ABI (qtn_graph_create_host, from the host copies of the tables: no device
    synchronisation, so an executor can be built while earlier work runs) and
    every run is one cudaGraphLaunch.

    arena: optional caller-owned element buffer (dtype of the program, at
    least prog.device_elems) shared by executors that run one after another on
    one stream — stream order keeps a later upload behind earlier kernels.

    Device buffer layout: [complex128 input image (complex64 programs only) |
    arena = input region + intermediates]; the pinned host image has the same
    [hi | lo] layout, so every upload is one copy."""

    def __init__(self, prog: Program, device=0, timing=False, arena=None):
        import torch
        self.torch = torch
        N.require_device()
        self.prog = prog
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        dev = self.device
        tdt = torch.complex64 if prog.dtype == "complex64" else torch.complex128
        self.tdt = tdt
        lib = N.load()
        with torch.cuda.device(dev):
            parts = [prog.buckets.tobytes(), prog.members.tobytes(), prog.deps.tobytes(),
                     prog.tick_begin.tobytes()]
            offs, cur = [], 0
            for p_ in parts:
                offs.append(cur)
                cur = _align(cur + len(p_), 16)
            ctrl_off = cur
            total = ctrl_off + 4 * (2 * prog.n_nodes + prog.n_buckets)
            host = np.zeros(_align(total, 16), np.uint8)
            for o, p_ in zip(offs, parts):
                host[o:o + len(p_)] = np.frombuffer(p_, np.uint8)
            # pinned + non_blocking: a pageable copy would wait for the stream
            self.tables = torch.from_numpy(host).pin_memory().to(dev, non_blocking=True)
            base = self.tables.data_ptr()
            if arena is not None:
                if arena.dtype != tdt or arena.device != dev or arena.numel() < prog.device_elems:
                    raise ValueError(f"arena: need {prog.device_elems} {tdt} elements on {dev}, got "
                                     f"{arena.numel()} {arena.dtype} on {arena.device}")
                self.buf = arena
            else:
                self.buf = torch.empty(prog.device_elems, dtype=tdt, device=dev)
            self.arena = self.buf[prog.hi_elems:]
            self.results = torch.zeros(2 * max(1, len(prog.instances)), dtype=torch.float64, device=dev)
            self.results_host = torch.zeros_like(self.results, device="cpu").pin_memory()
            self.timing = None
            if timing:
                self.timing = torch.zeros(2 * max(1, prog.n_buckets), dtype=torch.int64, device=dev)
                self.timing_init = torch.zeros_like(self.timing)
                self.timing_init[0::2] = np.iinfo(np.int64).max
            esz = ELEM_BYTES[prog.dtype]
            n_in = prog.n_input_elems
            self.img_bytes = n_in * esz + (n_in * 16 if prog.hi_elems else 0)
            self.img_pinned = torch.zeros(max(16, self.img_bytes), dtype=torch.uint8).pin_memory()
            v = self.img_pinned.numpy()
            if prog.hi_elems:
                self._img_hi = v[:16 * n_in].view(np.complex128)
                self._img_lo = v[16 * n_in: 16 * n_in + esz * n_in].view(np.complex64)
            else:
                self._img_hi = None
                self._img_lo = v[:esz * n_in].view(np.complex64 if prog.dtype == "complex64" else np.complex128)
            c = N.ProgramC()
            c.dtype = DTYPE_CODE[prog.dtype]
            c.n_buckets = prog.n_buckets
            c.n_tickets = 0
            c.smem_bytes = prog.smem_bytes
            c.grid = 0
            c.n_nodes = prog.n_nodes
            c.buckets = base + offs[0]
            c.members = base + offs[1]
            c.deps = base + offs[2]
            c.tick_begin = base + offs[3]
            c.ctrl = base + ctrl_off
            c.arena = self.arena.data_ptr()
            c.results = self.results.data_ptr()
            c.timing = self.timing.data_ptr() if timing else None
            c.arena_elems = prog.arena_elems
            c.inputs_hi = self.buf.data_ptr() if prog.hi_elems else None
            c.n_in_elems = n_in   # input region (K2 stages stage small input members from it)
            self.c = c
            self.done = torch.cuda.Event()
        self._graph = None
        self._io_graphs = {}  # raw-part pattern -> end-to-end graph + its pinned raw buffer
        self._staged = None
        self._res_np = self.results_host.numpy()

    def _create_graph(self, io, prog_c=None):
        nodes = np.ascontiguousarray(self.prog.nodes)
        deps = np.ascontiguousarray(self.prog.node_deps)
        items = np.ascontiguousarray(self.prog.buckets)
        mems = np.ascontiguousarray(self.prog.members)
        g = ctypes.c_void_p()
        with self.torch.cuda.device(self.device):
            N.check(N.load().qtn_graph_create_host(
                ctypes.byref(prog_c if prog_c is not None else self.c), items.ctypes.data_as(ctypes.c_void_p),
                mems.ctypes.data_as(ctypes.c_void_p),
                len(mems), nodes.ctypes.data_as(ctypes.c_void_p), self.prog.n_nodes,
                deps.ctypes.data_as(ctypes.c_void_p), ctypes.byref(io) if io is not None else None, ctypes.byref(g)))
        return g

    def kernel_mix(self, io=False):
        """{'K1', ..., 'K6'}: kernels per family in the program graph."""
        g = self.graph
        c = (ctypes.c_int32 * 6)()
        N.check(N.load().qtn_graph_kinds(g, c))
        return dict(zip(N.KERNEL_FAMILIES, (int(x) for x in c)))

    def node_kernels(self, io=False):
        """Per graph node, the kernel family that runs it ('K1'..'K6')."""
        g = self.graph
        n = int(self.prog.n_nodes)
        c = (ctypes.c_int32 * max(n, 1))()
        N.check(N.load().qtn_graph_node_kinds(g, c, n))
        return [N.KERNEL_FAMILIES[c[i]] for i in range(n)]

    def node_bytes(self, ni) -> int:
        """Compulsory bytes of graph node `ni` as it runs: each member read
        once, each result written once — a K6 pair moves neither its
        producer's result nor the consumer's read of it."""
        prog = self.prog
        nd = prog.nodes[ni]
        first, count = int(nd["first"]), int(nd["count"])
        tot = sum(prog.item_bytes(g) for g in range(first, first + count))
        if count == 2 and int(nd["kind"]) == N.QTN_NODE_LARGE and self.node_kernels()[ni] == "K6":
            tot -= 2 * (1 << int(prog.buckets[first]["w"])) * ELEM_BYTES[prog.dtype]
        return tot

    def executed_bytes(self) -> int:
        """Bytes the program's kernels must move (engine.executed_bytes of the
        templates, less the producer results K6 pairs keep on chip)."""
        tot = self.prog.executed_bytes()
        fam = self.node_kernels()
        for ni, nd in enumerate(self.prog.nodes):
            if int(nd["count"]) == 2 and int(nd["kind"]) == N.QTN_NODE_LARGE and fam[ni] == "K6":
                tot -= 2 * (1 << int(self.prog.buckets[int(nd["first"])]["w"])) * ELEM_BYTES[self.prog.dtype]
        return tot

    def node_graph(self, ni):
        """A graph of node `ni` alone (no dependencies; the same kernel and
        launch configuration the program graph runs it with): times one
        kernel in isolation, its inputs left in the arena by an earlier run."""
        nd = np.array(self.prog.nodes[ni: ni + 1]).copy()
        nd["dep_begin"] = 0
        nd["n_dep"] = 0
        if int(nd["kind"][0]) == N.QTN_NODE_SMALL:
            raise ValueError("node_graph: K2 stages depend on their control words; time large nodes only")
        deps = np.zeros(1, np.int32)
        items = np.ascontiguousarray(self.prog.buckets)
        mems = np.ascontiguousarray(self.prog.members)
        g = ctypes.c_void_p()
        with self.torch.cuda.device(self.device):
            N.check(N.load().qtn_graph_create_host(
                ctypes.byref(self.c), items.ctypes.data_as(ctypes.c_void_p), mems.ctypes.data_as(ctypes.c_void_p),
                len(mems), nd.ctypes.data_as(ctypes.c_void_p), 1, deps.ctypes.data_as(ctypes.c_void_p), None,
                ctypes.byref(g)))
        kinds = (ctypes.c_int32 * 1)()
        N.check(N.load().qtn_graph_node_kinds(g, kinds, 1))
        return _OwnedGraph(g), N.KERNEL_FAMILIES[kinds[0]]

    def launch_graph(self, g, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        N.check(N.load().qtn_graph_launch(g.g, ctypes.c_void_p(s.cuda_stream)))

    @property
    def graph(self):
        """The program graph (kernels only), built on first use."""
        if self._graph is None:
            self._graph = self._create_graph(None)
        return self._graph

    def __del__(self):
        for name in ("_graph",):
            g = getattr(self, name, None)
            if g is not None and g.value:
                try:
                    N.load().qtn_graph_destroy(g)
                except Exception:
                    pass

    # -- input image -------------------------------------------------------
    def stage_inputs(self, raw_parts):
        """raw_parts: per instance, the raw concatenation of its input tensors
        (complex128, each tensor C-order in its own index order).  Gathered
        into canonical layout (and narrowed) straight into the pinned staging
        buffer, then one H2D copy; alignment padding is never read."""
        self._staged = None
        self._gather(raw_parts)
        if self.img_bytes:
            self.buf.view(self.torch.uint8)[:self.img_bytes].copy_(self.img_pinned[:self.img_bytes],
                                                                   non_blocking=True)

    def _gather(self, raw_parts):
        """Canonical-layout gather of the raw inputs into the pinned image
        (complex128 image first when the program keeps one, then the arena's
        input region in the program's element type)."""
        parts = self.prog.img_src_parts
        if len(parts) == 1:
            vals = raw_parts[0][parts[0]]
        elif parts:
            vals = np.concatenate([raw[s] for raw, s in zip(raw_parts, parts)])
        else:
            return
        if self._img_hi is not None:
            self._img_hi[self.prog.img_dst] = vals
        self._img_lo[self.prog.img_dst] = vals

    def launch(self, stream=None):
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if self.timing is not None:
            self.timing.copy_(self.timing_init, non_blocking=True)
        N.check(N.load().qtn_graph_launch(self.graph, ctypes.c_void_p(s.cuda_stream)))

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

    def _io_graph(self, raw_parts):
        """The end-to-end program graph for this pattern of raw input parts
        (built on first use, cached per pattern): a first kernel node gathers
        the raw input tensors — complex128, concatenated into a pinned,
        device-mapped host buffer, one slot per distinct part — into the
        canonical input image (narrowing for complex64, the unrounded copy
        into inputs_hi); then the kernels; the finalisers write the result
        slots straight into pinned host memory.  run() is then one host copy of
        the raw parts, one graph launch and one stream synchronisation."""
        torch = self.torch
        slot_of, slots = {}, []
        mapping = []
        for i, part in enumerate(raw_parts):
            k = id(part)
            if k not in slot_of:
                slot_of[k] = len(slots)
                slots.append(int(part.size))
            mapping.append(slot_of[k])
        key = (tuple(mapping), tuple(slots))
        hit = self._io_graphs.get(key)
        if hit is None:
            base = np.concatenate([[0], np.cumsum(slots)]).astype(np.int64)
            src = np.concatenate([base[m] + p_ for m, p_ in zip(mapping, self.prog.img_src_parts)]) \
                if len(mapping) else np.zeros(0, np.int64)
            dst = np.ascontiguousarray(self.prog.img_dst, dtype=np.int64)
            raw_host = torch.zeros(max(1, int(base[-1])), dtype=torch.complex128).pin_memory()
            idx = torch.from_numpy(np.concatenate([src, dst])).to(self.device)
            # the finalisers write the result slots straight into the pinned
            # (device-mapped) host buffer: no download node after the last kernel
            c_io = N.ProgramC.from_buffer_copy(self.c)
            c_io.results = self.results_host.data_ptr()
            n = len(dst)
            io = N.GraphIOC(h2d_src=None, h2d_dst=None, h2d_bytes=0, d2h_src=None, d2h_dst=None, d2h_bytes=0,
                            gather_raw=raw_host.data_ptr(), gather_src=idx.data_ptr(),
                            gather_dst=idx.data_ptr() + 8 * n, n_gather=n)
            g = _OwnedGraph(self._create_graph(io, c_io))
            hit = self._io_graphs[key] = (g, raw_host, raw_host.numpy(), base, idx, c_io, [None] * len(slots))
        return hit

    def run(self, raw_parts, stream=None):
        """Copy the raw inputs into the pinned buffer, then one graph launch
        (device gather, kernels, results into pinned host memory) and one
        synchronisation."""
        self.submit(raw_parts, stream)
        return self.collect()

    def submit(self, raw_parts, stream=None):
        """run() without the wait: copy the raw parts into the pinned buffer,
        launch the end-to-end graph and record `done`; collect() waits.  The
        buffer must not be restaged before collect()."""
        torch = self.torch
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        g, raw_host, view, base, _, _, staged = self._io_graph(raw_parts)
        done_slots = set()
        for i, part in enumerate(raw_parts):
            k = id(part)
            if k in done_slots:
                continue
            done_slots.add(k)
            sl = self._io_graphs_slot(raw_parts, i)
            # the buffer already holds a read-only (immutable Tensors') part
            if staged[sl] is part and not part.flags.writeable:
                continue
            np.copyto(view[base[sl]: base[sl] + part.size], part.reshape(-1), casting="no")
            staged[sl] = part
        if self.timing is not None:
            self.timing.copy_(self.timing_init, non_blocking=True)
        N.check(N.load().qtn_graph_launch(g.g, ctypes.c_void_p(s.cuda_stream)))
        self.done.record(s)

    @staticmethod
    def _io_graphs_slot(raw_parts, i):
        seen = {}
        for j, part in enumerate(raw_parts[: i + 1]):
            seen.setdefault(id(part), len(seen))
        return seen[id(raw_parts[i])]

    def collect(self):
        """Wait for the last submit() and return its per-instance values."""
        self.done.synchronize()
        r = self._res_np
        if len(r) == 2:
            return [complex(r[0], r[1])]
        return r[0::2] + 1j * r[1::2]
