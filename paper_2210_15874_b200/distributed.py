"""Work units, sharding and the energy all-reduce.

The reference parallelises the energy over lightcones with a thread pool
(src/tn_build.py:176-186) and sums (1 - <ZZ>)/2 in sorted-edge order
(src/tn_build.py:199).  Here:

  * every cone is planned on the host; a cone wider than the slice target is
    expanded into 2^s slice units (suggest_slicing, src/ordering.py:192-230);
  * units are costed by algorithmic bytes and assigned to
    ranks with LPT (largest first, to the least-loaded rank, ties to the
    lowest rank) — deterministic, no data-path communication;
  * each rank runs its units as batched device programs (one persistent
    launch per batch) and writes each unit's complex value into its slot of
    a zero-filled float64 vector;
  * one all-reduce (NCCL over NVLink on GPUs, gloo on CPU) sums the slot
    vector.  Every slot has exactly one non-zero contributor, so the sum is
    exact and the per-cone totals (summed on the host in slice order) are
    bitwise identical for any number of ranks.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import engine as E
from .tensor_core import Backend, memory_estimate


PLAN_THREADS = max(1, min(16, os.cpu_count() or 1))
# LPT cost of a (cone, slice) unit: the bytes its device items must move
# (members once + results once; merged chains write no intermediates) plus a
# fixed charge for its latency-bound chains (~80 us at HBM rate).  Round 1
# used SURVEY 8(d) algorithmic bytes, which overweight merged items.
# Measured on the 45-cone N=30 p=4 energy (c64, bench rank_shares): 1 GPU
# 6.94 -> 6.82 ms, predicted 8-rank makespan 1.32 -> 1.25 ms.
UNIT_LATENCY_BYTES = 500_000_000


def unit_cost(tmpl, dtype):
    return E.executed_bytes(tmpl, dtype) + UNIT_LATENCY_BYTES


@dataclass
class Unit:
    cone: int
    assignment: dict
    cost: int


@dataclass
class UnitPlan:
    cones: list
    templates: list
    raws: list
    units: list
    widths: list = field(default_factory=list)


def plan_units(cones, backend: Backend, heuristic="minfill", mem_cap=4 << 30, slice_target=None, n_workers=1,
               balance_ranks=None, balance_factor=2.0):
    """Order every cone, slice the wide ones, build templates and units.

    balance_ranks: additionally slice the heaviest cones (one more index at a
    time, suggest_slicing with a narrower target) until no unit costs more
    than total / (balance_ranks * balance_factor) — so LPT can spread an
    over-wide lightcone's index slices across that many GPUs.  The plan
    depends only on balance_ranks, not on the actual world size, so energies
    stay bitwise identical for any number of ranks."""
    from .ordering import MemoryCapError, greedy_order, suggest_slicing

    def one(lc):
        tn = lc.network
        order = greedy_order(tn, heuristic)
        ix = [t.indices for t in tn.tensors]
        sib = E.small_iter_bits_for(backend.threshold, backend.dtype)
        tmpl = E.plan_template(ix, order, backend.dtype, small_iter_bits=sib)
        sliced = []
        if slice_target is not None and tmpl.max_width > slice_target:   # width = the dry run's
            sliced = suggest_slicing(tn, order, slice_target)
            tmpl = E.plan_template(ix, order, backend.dtype, fixed=sliced, small_iter_bits=sib)
        if memory_estimate(tmpl.max_width, backend.dtype) > mem_cap:
            raise MemoryCapError(tmpl.max_width, memory_estimate(tmpl.max_width, backend.dtype), mem_cap)
        raw = tn.packed()[2]      # the builders' packed host image (TensorNetwork.packed)
        return tmpl, sliced, raw

    # the native planner calls (greedy_order, qtn_plan_build) release the GIL:
    # plan the cones on host threads (at least PLAN_THREADS; the result does
    # not depend on the thread count)
    n_workers = max(int(n_workers or 1), PLAN_THREADS)
    if n_workers > 1 and len(cones) > 1:
        with ThreadPoolExecutor(max_workers=n_workers) as pool:
            res = list(pool.map(one, cones))
    else:
        res = [one(lc) for lc in cones]
    if balance_ranks and balance_ranks > 1:
        res = _balance(cones, res, backend, heuristic, mem_cap, balance_ranks, balance_factor)
    units = []
    templates, raws = [], []
    for ci, (tmpl, sliced, raw) in enumerate(res):
        templates.append(tmpl)
        raws.append(raw)
        cost = unit_cost(tmpl, backend.dtype)
        for bits in np.ndindex(*(2,) * len(sliced)):
            units.append(Unit(ci, dict(zip(sliced, (int(b) for b in bits))), cost))
    return UnitPlan(list(cones), templates, raws, units)


def _balance(cones, res, backend, heuristic, mem_cap, n_ranks, factor, max_rounds=64, max_extra_bits=6):
    """Slice the most expensive cone one index further until every unit is at
    most total / (n_ranks * factor) (algorithmic bytes per slice)."""
    from .ordering import greedy_order, suggest_slicing
    res = list(res)
    orders = {}
    base = [len(s_) for _, s_, _ in res]
    stuck = set()
    sib = E.small_iter_bits_for(backend.threshold, backend.dtype)
    for _ in range(max_rounds):
        per = [unit_cost(t, backend.dtype) for t, _, _ in res]
        total = sum(c << len(s_) for c, (_, s_, _) in zip(per, res))
        target = total / (n_ranks * factor)
        cand = [i for i in range(len(res)) if i not in stuck and per[i] > target]
        if not cand:
            break
        ci = max(cand, key=lambda i: (per[i], -i))
        tmpl, sliced, raw = res[ci]
        if len(sliced) - base[ci] >= max_extra_bits or tmpl.max_width <= 1:
            stuck.add(ci)
            continue
        tn = cones[ci].network
        order = orders.get(ci) or greedy_order(tn, heuristic)
        orders[ci] = order
        new = suggest_slicing(tn, order, tmpl.max_width - 1)
        if len(new) <= len(sliced) or not set(sliced) <= set(new):
            stuck.add(ci)
            continue
        t2 = E.plan_template([t.indices for t in tn.tensors], order, backend.dtype, fixed=new, small_iter_bits=sib)
        res[ci] = (t2, new, raw)
    return res


def lpt_assign(costs, n_ranks):
    """Largest-processing-time-first assignment; returns rank per unit."""
    owner = [0] * len(costs)
    load = [0] * n_ranks
    for u in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(n_ranks), key=lambda k: (load[k], k))
        owner[u] = r
        load[r] += costs[u]
    return owner


def _batches(units, plan, backend, budget_bytes):
    """Greedy batching of units into programs under an HBM budget."""
    esz = backend.elem_bytes
    cur, cur_b = [], 0
    for ui in units:
        t = plan.templates[plan.units[ui].cone]
        if not hasattr(t, "_peak"):
            t._peak = E.template_peak_elems(t)
        b = (t.n_in_elems + t._peak) * esz + 4096
        if cur and cur_b + b > budget_bytes:
            yield cur
            cur, cur_b = [], 0
        cur.append(ui)
        cur_b += b
    if cur:
        yield cur


@dataclass
class Prepared:
    """Executors for one rank's units, built once (plans, graphs, HBM) and
    re-run many times (bench loop / parameter sweeps over the same structure)."""
    batches: list          # [(Executor, [unit ids])]
    raws: list


def prepare_local(plan: UnitPlan, mine, backend: Backend, device: int, budget_bytes=None) -> Prepared:
    import torch
    if budget_bytes is None:
        free, _ = torch.cuda.mem_get_info(device)
        budget_bytes = int(0.6 * free)
    be = Backend(backend.kind, backend.threshold, backend.dtype, device, backend.profile)
    out = []
    for batch in _batches(mine, plan, be, budget_bytes):
        insts = [E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch]
        ex = E.Executor(E.Program(insts, be.dtype), device=device, timing=be.profile)
        ex.stage_inputs([plan.raws[plan.units[u].cone] for u in batch])
        out.append((ex, batch))
    return Prepared(out, plan.raws)


def launch_prepared(prep: Prepared, stream=None):
    """Launch every batch (inputs already resident)."""
    for ex, _ in prep.batches:
        ex.launch(stream)


def collect_prepared(prep: Prepared, stream=None) -> dict:
    vals = {}
    for ex, batch in prep.batches:
        res = ex.fetch_results(stream)
        for k, u in enumerate(batch):
            vals[u] = complex(res[k])
    return vals


def run_local(plan: UnitPlan, mine, backend: Backend, device: int, budget_bytes=None, cache=None):
    """Execute units `mine` on one device; returns {unit: complex}, {cone: stats}.
    `cache` (a dict owned by the caller) keeps the batches' executors — plans,
    CUDA graphs, HBM — for the next call on the same structure, which then only
    re-stages the inputs."""
    import torch
    be = Backend(backend.kind, backend.threshold, backend.dtype, device, backend.profile)
    key = ("batches", tuple(mine), device, be.dtype, be.profile)
    skey = ("streamed", tuple(mine), device, be.dtype, be.profile)
    if cache is not None and skey in cache:
        return _run_streamed(plan, None, be, device, cache[skey])
    if cache is not None and key in cache:
        built = cache[key]
    else:
        if budget_bytes is None:
            free, _ = torch.cuda.mem_get_info(device)
            budget_bytes = int(0.6 * free)
        batches = list(_batches(mine, plan, be, budget_bytes))
        if len(batches) > 1:
            # does not fit at once: stream the batches through one arena; only
            # the host programs are kept for the next call on this structure
            progs = []
            out = _run_streamed(plan, batches, be, device, progs)
            if cache is not None:
                cache[skey] = progs
            return out
        built = []
        for batch in batches:
            insts = [E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch]
            built.append((E.Executor(E.Program(insts, be.dtype), device=device, timing=be.profile), batch))
        if cache is not None:
            cache[key] = built
    vals, stats = {}, {}
    for ex, batch in built:
        prog = ex.prog
        res = ex.run([plan.raws[plan.units[u].cone] for u in batch])
        if be.profile:
            t0, t1 = ex.fetch_timing()
        from .ordering import _item_families, ref_stats
        for k, u in enumerate(batch):
            vals[u] = complex(res[k])
            ci = plan.units[u].cone
            tm = plan.templates[ci]
            el = np.maximum(t1[prog.bucket_gid[k]] - t0[prog.bucket_gid[k]], 0) if be.profile else None
            stats.setdefault(ci, []).extend(ref_stats(tm, be, el, _item_families(ex, k)) if be.profile
                                            else _plain_stats(tm, be))
    return vals, stats


def _plain_stats(tmpl, be):
    """BucketStats without timings depend on the plan only (immutable): built
    once per template (ordering._stats does the same for contract_network)."""
    from .ordering import _stats
    return _stats(tmpl, None, be)


def _run_streamed(plan, batches, be, device, progs):
    """Batches that do not fit in HBM together, run one after another through
    one shared arena: batch k+1's Program (host planning, the expensive part)
    and Executor (graph build from host tables, pinned uploads) are prepared
    while batch k runs, then queued behind it on the same stream; batch k's
    results are read after k+1 was submitted.  The arena grows (after a wait)
    when a batch needs more.  `progs`: [(Program, batch)] — filled when
    `batches` is given, replayed (no host planning) when `batches` is None."""
    import torch
    from .ordering import _item_families, ref_stats
    tdt = torch.complex64 if be.dtype == "complex64" else torch.complex128
    vals, stats = {}, {}
    arena, prev = None, None

    def finish(ex, batch):
        res = ex.collect()
        if be.profile:
            t0, t1 = ex.fetch_timing()
        for k, u in enumerate(batch):
            vals[u] = complex(res[k])
            ci = plan.units[u].cone
            el = (np.maximum(t1[ex.prog.bucket_gid[k]] - t0[ex.prog.bucket_gid[k]], 0) if be.profile else None)
            tm = plan.templates[ci]
            stats.setdefault(ci, []).extend(ref_stats(tm, be, el, _item_families(ex, k)) if be.profile
                                            else _plain_stats(tm, be))

    ex = None
    work = progs if batches is None else batches
    if batches is None and progs:   # replay: the largest arena up front (no mid-stream waits)
        arena = torch.empty(max(pr.device_elems for pr, _ in progs), dtype=tdt, device=torch.device("cuda", device))
    for item in work:
        if batches is None:
            prog, batch = item
        else:
            batch = item
            insts = [E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch]
            prog = E.Program(insts, be.dtype)
            progs.append((prog, batch))
        if arena is None or arena.numel() < prog.device_elems:
            if prev is not None:
                finish(*prev)
                prev = None
            ex = None      # the last executor holds the old arena too
            arena = None   # freed before the larger one is allocated
            arena = torch.empty(prog.device_elems, dtype=tdt, device=torch.device("cuda", device))
        ex = E.Executor(prog, device=device, timing=be.profile, arena=arena)
        ex.submit([plan.raws[plan.units[u].cone] for u in batch])
        if prev is not None:
            finish(*prev)
        prev = (ex, batch)
    if prev is not None:
        finish(*prev)
    return vals, stats


def _combine(plan, slot_vec):
    n_cones = len(plan.cones)
    values = [0j] * n_cones
    for u, unit in enumerate(plan.units):   # units are in (cone, ndindex) order
        values[unit.cone] += complex(slot_vec[2 * u], slot_vec[2 * u + 1])
    return values


def run_units(plan: UnitPlan, backend: Backend, group=None, n_gpus=None, cache=None):
    """Run all units; returns (per-cone complex values, per-cone stats).
    `cache`: see run_local (one dict per structure, shared by the ranks'
    devices)."""
    import torch
    import torch.distributed as dist
    costs = [u.cost for u in plan.units]
    n_units = len(plan.units)
    if group is not None or (dist.is_available() and dist.is_initialized()):
        rank = dist.get_rank(group)
        world = dist.get_world_size(group)
        owner = lpt_assign(costs, world)
        mine = [u for u in range(n_units) if owner[u] == rank]
        dev = torch.cuda.current_device() if torch.cuda.is_available() else backend.device
        vals, stats = run_local(plan, mine, backend, dev, cache=cache) if mine else ({}, {})
        slots = np.zeros(2 * n_units, np.float64)
        for u, v in vals.items():
            slots[2 * u], slots[2 * u + 1] = v.real, v.imag
        on_gpu = dist.get_backend(group) == "nccl"
        t = torch.from_numpy(slots).to("cuda" if on_gpu else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        slots = t.cpu().numpy()
        st = [stats.get(ci, []) for ci in range(len(plan.cones))]
        return _combine(plan, slots), st
    ng = n_gpus or 1
    owner = lpt_assign(costs, ng)
    results = [None] * ng
    stats = {}
    if ng > 1:
        # one host thread per GPU; each device's unit values go into its own
        # zero slot vector, summed across the devices by ONE NCCL all-reduce
        # (single process, one communicator per device: ncclCommInitAll)
        dev_slots = [None] * ng

        def work(r):
            mine = [u for u in range(n_units) if owner[u] == r]
            with torch.cuda.device(r):
                results[r] = run_local(plan, mine, backend, r, cache=cache) if mine else ({}, {})
                sl = np.zeros(2 * n_units, np.float64)
                for u, v in results[r][0].items():
                    sl[2 * u], sl[2 * u + 1] = v.real, v.imag
                dev_slots[r] = torch.from_numpy(sl).to(f"cuda:{r}")

        with ThreadPoolExecutor(max_workers=ng) as pool:
            list(pool.map(work, range(ng)))
        slots = slot_allreduce_devices(dev_slots)
    else:
        results[0] = run_local(plan, list(range(n_units)), backend, backend.device, cache=cache)
        slots = np.zeros(2 * n_units, np.float64)
        for u, v in results[0][0].items():
            slots[2 * u], slots[2 * u + 1] = v.real, v.imag
    for _, st in results:
        for ci, s in st.items():
            stats.setdefault(ci, []).extend(s)
    return _combine(plan, slots), [stats.get(ci, []) for ci in range(len(plan.cones))]


def slot_allreduce_devices(dev_slots):
    """Sum per-device slot vectors (float64, one per GPU of this process) with
    a single-process NCCL all-reduce (torch.cuda.nccl: one communicator per
    device); every slot has one non-zero contributor, so the sum is exact.
    Returns the summed vector on the host."""
    import torch
    import torch.cuda.nccl as nccl
    if not nccl.is_available(dev_slots):
        raise RuntimeError("NCCL unavailable for the slot all-reduce")
    nccl.all_reduce(dev_slots)
    torch.cuda.synchronize(dev_slots[0].device)
    return dev_slots[0].cpu().numpy()
