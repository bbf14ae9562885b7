"""Small/large routing threshold tuned on the B200 (reference: src/tuning.py,
`qtnsim tune-threshold`, src/cli.py:285-307).

The reference times its two CPU kernels (pure-Python `reference_kernel`,
NumPy `fast_kernel`) on every bucket of real lightcones and picks the Mixed
width threshold that minimises the projected total (src/tuning.py:30-129).
On the B200 the two routes are the batched small-bucket schedule (K2
persistent stages — the "reference" column) and the fused large-bucket
kernels (K1 — the "fast" column); `Backend.threshold` decides which route a
bucket takes (engine.small_iter_bits_for).  Two measurements:

  * profile_kernels: per-bucket device times (globaltimer stamps of the
    program kernels) with every bucket routed to K2 (up to
    `max_ref_width`), then to K1, merging disabled so items are reference
    buckets -> KernelTimings, the crossover CSV and the projected best
    threshold (same selection rule as the reference, choose_threshold);
  * sweep_thresholds: the whole lightcone program (merging on, as in
    production) timed with CUDA events for each candidate threshold —
    buckets overlap inside one CUDA graph, so this is the number that
    decides; `measured_best` is its argmin.

Timings need a CUDA device (no CPU fallback); the selection logic is host
code and is tested on synthetic timings.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import engine as E
from .tensor_core import Backend


@dataclass
class KernelTimings:
    """Per-width device timings from real bucket contractions
    (src/tuning.py:11-31).  ref_ns: K2 small-batched route; fast_ns: K1
    fused route (missing where that route cannot run the bucket)."""

    ref_ns: dict
    fast_ns: dict
    counts: dict

    def mean(self, table, width):
        xs = table.get(width)
        return sum(xs) / len(xs) if xs else None

    def rows(self):
        return [(w, self.mean(self.ref_ns, w), self.mean(self.fast_ns, w)) for w in sorted(self.counts)]


def _item_times(tn, order, backend, threshold, dtype):
    """(per reference bucket widths, per reference bucket ns, per bucket 'ran in K2')."""
    import torch
    tmpl = E.plan_template([t.indices for t in tn.tensors], order, dtype, merge=False,
                           small_iter_bits=E.small_iter_bits_for(threshold, dtype))
    prog = E.Program([E.Instance(tmpl)], dtype)
    ex = E.Executor(prog, device=backend.device, timing=True)
    raw = np.concatenate([np.asarray(t.data, np.complex128).ravel() for t in tn.tensors])
    ex.stage_inputs([raw])
    for _ in range(3):
        ex.launch()
    torch.cuda.synchronize(backend.device)
    t0, t1 = ex.fetch_timing()
    gids = prog.bucket_gid[0]
    el = np.maximum(t1[gids] - t0[gids], 0)
    small = tmpl.variant == E.VARIANT_SMALL
    # merge=False: item i is reference bucket i (elimination order)
    return tmpl.ref_w, el[tmpl.ref_item], small[tmpl.ref_item]


def profile_kernels(tn, order, max_reference_width: int = 18, backend: Backend = None) -> KernelTimings:
    """Time every bucket of one contraction through both routes
    (src/tuning.py:34-69).  The K2 route is used up to max_reference_width."""
    backend = backend or Backend.b200()
    timings = KernelTimings({}, {}, {})
    w_s, ns_s, small_s = _item_times(tn, order, backend, max_reference_width, backend.dtype)
    w_f, ns_f, small_f = _item_times(tn, order, backend, -1, backend.dtype)
    for w, ns, sm in zip(w_s, ns_s, small_s):
        w = int(w)
        timings.counts[w] = timings.counts.get(w, 0) + 1
        if sm:
            timings.ref_ns.setdefault(w, []).append(int(ns))
    for w, ns, sm in zip(w_f, ns_f, small_f):
        if not sm:   # too narrow for a K1 tile: that route does not exist there
            timings.fast_ns.setdefault(int(w), []).append(int(ns))
    return timings


def merge_timings(parts) -> KernelTimings:
    out = KernelTimings({}, {}, {})
    for t in parts:
        for w, xs in t.ref_ns.items():
            out.ref_ns.setdefault(w, []).extend(xs)
        for w, xs in t.fast_ns.items():
            out.fast_ns.setdefault(w, []).extend(xs)
        for w, c in t.counts.items():
            out.counts[w] = out.counts.get(w, 0) + c
    return out


def projected_total(timings: KernelTimings, threshold: int) -> float:
    """Total if widths > threshold take the K1 route and the rest K2
    (src/tuning.py:86-104); a route with no sample for a width it would
    have to take makes the projection infinite."""
    total = 0.0
    for w, count in timings.counts.items():
        mean = timings.mean(timings.fast_ns, w) if w > threshold else timings.mean(timings.ref_ns, w)
        if mean is None:
            return float("inf")
        total += mean * count
    return total


@dataclass
class ThresholdReport:
    best_threshold: int
    crossover: int | None
    mixed_total_ns: float
    all_reference_total_ns: float
    all_fast_total_ns: float
    measured: dict = field(default_factory=dict)   # threshold -> device ns per contraction
    measured_best: int | None = None


def choose_threshold(timings: KernelTimings) -> ThresholdReport:
    """Same selection rule as src/tuning.py:107-129."""
    widths = sorted(timings.counts)
    candidates = sorted({-1, 0, *widths})
    totals = {thr: projected_total(timings, thr) for thr in candidates}
    best = min(candidates, key=lambda thr: (totals[thr], thr))
    crossover = None
    for w in widths:
        ref = timings.mean(timings.ref_ns, w)
        fast = timings.mean(timings.fast_ns, w)
        if ref is not None and fast is not None and fast < ref:
            crossover = w
            break
    if crossover is None and any(timings.mean(timings.ref_ns, w) is None for w in widths):
        crossover = min(w for w in widths if timings.mean(timings.ref_ns, w) is None)
    return ThresholdReport(
        best_threshold=best,
        crossover=crossover,
        mixed_total_ns=totals[best],
        all_reference_total_ns=projected_total(timings, max(widths)) if widths else 0.0,
        all_fast_total_ns=projected_total(timings, -1),
    )


def sweep_thresholds(cones, orders, thresholds, backend: Backend = None, reps: int = 20) -> dict:
    """Device ns per contraction of all `cones` (summed) for each threshold:
    the production plan (merging on) in one CUDA graph per cone, CUDA
    events around `reps` launches after warm-up."""
    import torch
    backend = backend or Backend.b200()
    out = {}
    for thr in thresholds:
        tot = 0.0
        for lc, order in zip(cones, orders):
            tn = lc.network
            tmpl = E.plan_template([t.indices for t in tn.tensors], order, backend.dtype,
                                   small_iter_bits=E.small_iter_bits_for(thr, backend.dtype))
            ex = E.Executor(E.Program([E.Instance(tmpl)], backend.dtype), device=backend.device, timing=False)
            ex.stage_inputs([np.concatenate([np.asarray(t.data, np.complex128).ravel() for t in tn.tensors])])
            s = torch.cuda.current_stream(backend.device)
            for _ in range(3):
                ex.launch(s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                ex.launch(s)
            e1.record(s)
            e1.synchronize()
            tot += e0.elapsed_time(e1) * 1e6 / reps
            del ex
        out[int(thr)] = tot
    return out


def write_crossover_csv(path, timings: KernelTimings):
    """width,mean_ns_reference,mean_ns_fast (src/tuning.py:132-139); the
    columns are the K2 (small-batched) and K1 (fused) routes."""
    with open(path, "w") as f:
        f.write("width,mean_ns_reference,mean_ns_fast\n")
        for w, ref, fast in timings.rows():
            ref_s = "" if ref is None else f"{ref:.1f}"
            fast_s = "" if fast is None else f"{fast:.1f}"
            f.write(f"{w},{ref_s},{fast_s}\n")
