"""Benchmark of the north-star path: one N=30, p=4 QAOA MaxCut edge lightcone
(BASELINE.json configs[1]; SURVEY 8(d) cfg 2: tight cone of edge (0,15),
width 25, 270 buckets) contracted by bucket elimination on the B200.

  python bench.py [--gpus N --steps K --warmup W --dtype c128|c64]
  python bench.py --impl reference ...   (the reference algorithm on host cores)

A step = one full contraction of the lightcone per rank (weak scaling: every
rank contracts its own copy; at N > 1 the per-rank <ZZ> slots are summed by
one NCCL all-reduce inside the step).  The headline dtype is complex128, the
reference's own arithmetic (src/tensor_core.py:59); complex64 is reported
beside it.  `value` = lightcones/s from CUDA events on the launching stream
(L2 flushed before every step, max over ranks); `e2e` = the public call
`contract_network(tn, order, backend)` with HOST tensors, a different set of
angles every step (new gate tensors: gather, upload, kernels, result read),
wall clock, max over ranks.  `strong` = the full-graph energy (45 lightcones
of the same graph, LPT over the ranks, slot all-reduce) at this N.

`--gpus N` without torchrun re-executes itself under torch.distributed.run
(one rank per GPU, 127.0.0.1 rendezvous).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lightcones/s (N=30,p=4 single-lightcone contraction)"
UNIT = "lightcones/s"
PAPER_BEST_S = 2.1       # NumPy+CuPy mixed, V100
N_QUBITS, DEGREE, P_LAYERS, SEED = 30, 3, 4, 0
EDGE = (0, 15)
GRAPH_MEM_CAP = 64 << 30   # HBM-sized widest-bucket cap (the reference's 4 GiB default is a CPU cap)
GRAPH_BALANCE = 8          # slice over-wide cones so 8 GPUs can share them (same plan at every N)
WORKLOAD = ("cfg2: 3-regular N=30 (seed 0), p=4 (seeded angles), tight lightcone of edge (0,15): "
            "564 tensors, 270 buckets, widths 0-25")
# identical in both arms (the driver compares them)
CONFIG = {"workload": WORKLOAD, "graph": "random_regular_graph(30, 3, seed=0)", "p": P_LAYERS,
          "angles": "QaoaParams.seeded(4, 0)", "edge": list(EDGE), "cone": "tight", "order": "greedy_order minfill"}
L2_NOTE = "flushed (256 MiB write) before every timed step"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--dtype", default="c128", choices=["c64", "c128"], help="headline dtype")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=2, help="oracle contractions for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong", action="store_true", help="skip the full-graph strong-scaling figure")
    ap.add_argument("--no-shares", action="store_true",
                    help="skip the per-rank share timings (predicted strong scaling on one GPU)")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--sustain-s", type=float, default=1.0, help="clock-sampled sustained loop after the timed region")
    ap.add_argument("--simplify", action="store_true",
                    help="graph workload: simplify each lightcone network before ordering (tn_build.simplify_network)")
    ap.add_argument("--workload", default="lightcone", choices=["lightcone", "graph", "bucket", "selftest"],
                    help="lightcone: cfg-2 single lightcone per rank (weak) + full-graph strong figure; graph: "
                         "all 45 N=30 p=4 tight lightcones sharded over ranks by LPT + slot all-reduce (strong); "
                         "bucket: cfg-5 synthetic bucket microbench through K3; selftest: the multi-rank harness "
                         "alone (spawn, rendezvous, max-over-ranks, slot all-reduce) on CPU/gloo")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# multi-rank harness
# ---------------------------------------------------------------------------
def _free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n, argv):
    """Re-execute this script as n ranks under torch.distributed.run (one
    process per GPU, 127.0.0.1 rendezvous); returns the launcher's exit code.
    Rank 0's JSON line is the launcher's stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator lines show the N ranks ...
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # ... on stderr, not in the JSON stdout
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def dist_setup():
    """(rank, world, local_rank); process group over NCCL when CUDA is
    present, gloo otherwise (the CPU harness test)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return rank, world, local


def _dev():
    import torch
    return "cuda" if torch.cuda.is_available() else "cpu"


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def finish(world):
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """NVML clocks + clock-event (throttle) reasons, polled every `period` s by
    a background thread while the timed region runs (NVML calls release the
    GIL; the timed loop only enqueues work, so the device queue stays fed)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, local, period=0.0005):
        self.period = period
        self.samples = []
        self.max_mhz = None
        self.h = None
        self.err = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            uuid = str(torch.cuda.get_device_properties(local).uuid)
            self.h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception as e:   # no NVML: the line says so
            self.err = f"{type(e).__name__}: {e}"

    def __enter__(self):
        self.stop = threading.Event()
        if self.h is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def _run(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.h is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    **({"error": self.err} if self.err else {})}
        reasons = set()
        for _, rs in self.samples:
            for bit, name in self.REASONS.items():
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def peak_fp(dtype):
    """Measured FMA peak of the element type's arithmetic (tools/fp_peak.cu,
    profiles/r02_fp_peak.json): TFLOP/s and its source."""
    p = os.path.join(ROOT, "profiles", "r02_fp_peak.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["fp64_fma_tflops" if dtype == "complex128" else "fp32_fma_tflops"]), \
            "measured (tools/fp_peak.cu, profiles/r02_fp_peak.json)"
    except Exception:
        return None, None


def node_flops(prog, node):
    """Algorithmic floating-point work of one graph node: every complex
    multiply-add 8 flops.  An item: 2^(w+k) (result, assignment) products of
    its n_mem members (n_mem - 1 complex multiplies + the add).  A K6 pair:
    the producer's X values (2^(w_P + k_P) multiply-adds with its dominant
    member) and the consumer's 2^(w_C + k_C) multiply-adds of X by its other
    members' product."""
    nd = prog.nodes[node]
    first, count = int(nd["first"]), int(nd["count"])
    b = prog.buckets
    if count == 2:
        p_, c_ = b[first], b[first + 1]
        return 8 * ((1 << (int(p_["w"]) + int(p_["k"]))) + (1 << (int(c_["w"]) + int(c_["k"]))))
    it = b[first]
    return 8 * (1 << (int(it["w"]) + int(it["k"]))) * max(1, int(it["n_mem"]) - 1)


def arith_block(dom, dtype):
    """The dominant node's arithmetic against the measured FMA peak of its
    element type (a K6 pair is not HBM-bound: it moves 151 MB but does
    0.6 GFLOP of complex128 work at cfg-2)."""
    pk, src = peak_fp(dtype)
    tf = dom["flops"] / (dom["us"] * 1e-6) / 1e12
    return {"flops": dom["flops"], "achieved_tflops": tf, "peak_tflops": pk, "frac": (tf / pk) if pk else None,
            "peak_source": src, "note": "flops = 8 per complex multiply-add (bench.node_flops)"}


def ncu_traffic(key):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/traffic.json, keyed by
    dtype:kernel:item signature); None when that kernel was not captured."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            rec = json.load(f).get(key)
        return rec
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def _host_threads():
    """All host cores, capped by host memory (a cfg-2 contraction peaks at
    ~3 x 2^25 x 16 B = 1.6 GB in the reference's fast_kernel)."""
    n = os.cpu_count() or 1
    try:
        import psutil
        n = max(1, min(n, int(psutil.virtual_memory().available // (2 << 30))))
    except Exception:
        pass
    return n


def run_reference(args):
    """The reference algorithm on the host cores: the oracle port of the
    reference NumPy path (src/ordering.py:148-189 + src/tensor_core.py:148-164,
    complex128), network and order built by the oracle too (no product code
    is imported in this arm).  Every step = one bounded sample: `threads`
    concurrent contractions of the cfg-2 lightcone."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from concurrent.futures import ThreadPoolExecutor
    from oracle import qtn_oracle as O
    edges = O.random_regular_graph(N_QUBITS, DEGREE, SEED)
    gammas, betas = O.seeded_angles(P_LAYERS, SEED)
    ts = O.lightcone_tensors(N_QUBITS, edges, gammas, betas, EDGE, cone="tight")
    order = O.greedy_order(ts)
    threads = _host_threads()

    def one(_):
        v, _ = O.contract_network(ts, order)
        return v

    pool = ThreadPoolExecutor(max_workers=threads)
    t0 = time.perf_counter()
    list(pool.map(one, range(threads)))       # warm-up step (capped at 1)
    est = time.perf_counter() - t0
    steps = max(1, min(args.steps, int(args.ref_budget_s // max(est, 1e-3))))
    t0 = time.perf_counter()
    vals = []
    for _ in range(steps):
        vals = list(pool.map(one, range(threads)))
    dt = time.perf_counter() - t0
    pool.shutdown()
    value = threads * steps / dt
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "steps_requested": args.steps, "warmup": 1, "ms_per_step": 1e3 * dt / steps,
        "s_per_lightcone": dt * 1.0 / (steps * threads), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded graph/angles)", "config": CONFIG,
        "impl": "reference",
        "details": {"impl": "oracle port of the reference NumPy path (Backend.fast()); network + order from the oracle",
                    "threads": threads, "host_cpus": os.cpu_count(), "zz": vals[0].real},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps} steps x {threads} concurrent full contractions of the cfg-2 lightcone "
                                   f"(numpy complex128, one thread each; {os.cpu_count()} host CPUs)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm: cfg-2 lightcone
# ---------------------------------------------------------------------------
def build_workload(seed=SEED):
    import paper_2210_15874_b200 as Q
    g = Q.random_regular_graph(N_QUBITS, DEGREE, seed=SEED)
    params = Q.QaoaParams.seeded(P_LAYERS, seed)
    c = Q.qaoa_maxcut_circuit(g, params)
    lc = Q.extract_lightcone(c, EDGE, cone="tight")
    order = Q.greedy_order(lc.network)
    return g, params, lc, order


def cpu_oracle_time(lc, order, n):
    """The reference algorithm (oracle port of src/ordering.py:148-189 +
    src/tensor_core.py:148-164, numpy complex128) on one host core."""
    from oracle import qtn_oracle as O
    ts = [(t.indices, t.data) for t in lc.network.tensors]
    t0 = time.perf_counter()
    val = None
    for _ in range(n):
        val, _ = O.contract_network(ts, order)
    dt = (time.perf_counter() - t0) / n
    return dt, val


class _Lightcone:
    """Device program of the cfg-2 lightcone at one dtype (the plan
    contract_network makes), inputs resident in HBM."""

    def __init__(self, lc, order, dtype, local):
        from paper_2210_15874_b200 import engine as E
        self.E = E
        tn = lc.network
        self.dtype = dtype
        self.tmpl = E.plan_template([t.indices for t in tn.tensors], order, dtype, wave_aware=True)
        self.prog = E.Program([E.Instance(self.tmpl)], dtype)
        self.ex = E.Executor(self.prog, device=local, timing=False)
        self.raw = np.concatenate([np.asarray(t.data).ravel() for t in tn.tensors])
        self.ex.stage_inputs([self.raw])


def time_device(lcp, stream, flush, steps, world, rank, slots):
    import torch
    ex = lcp.ex

    def step():
        ex.launch(stream)
        if world > 1:
            slots.zero_()
            slots[2 * rank: 2 * rank + 2].copy_(ex.results[:2])
            torch.distributed.all_reduce(slots)

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(world)
    torch.cuda.synchronize()
    for i in range(steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    return sum(a.elapsed_time(b) for a, b in evs) / 1e3


def time_e2e(nets, order, be, steps, world):
    """The public call from host tensors, a different network (angles) every
    step: gather into the pinned image, one graph launch (upload node,
    kernels, result into pinned host memory), one synchronisation."""
    import torch
    import paper_2210_15874_b200 as Q
    for tn in nets[:3]:
        Q.contract_network(tn, order, be)
    torch.cuda.synchronize()
    barrier(world)
    vals = []
    t0 = time.perf_counter()
    for i in range(steps):
        v, _ = Q.contract_network(nets[i % len(nets)], order, be)
        vals.append(v)
    t = time.perf_counter() - t0
    return t, vals


def dominant_kernel(lcp, stream, flush, reps=50):
    """The device item with the longest live span (globaltimer stamps of the
    program kernels, L2 flushed), then that node ALONE timed with CUDA events
    on the launching stream over `reps` launches: compulsory bytes / mean
    launch duration, and its share of the step."""
    import torch
    E = lcp.E
    prog = lcp.prog
    ext = E.Executor(prog, device=lcp.ex.device, timing=True)
    ext.stage_inputs([lcp.raw])
    for _ in range(3):
        ext.launch(stream)
    acc = np.zeros(prog.n_buckets)
    for _ in range(20):
        flush.zero_()
        ext.launch(stream)
        torch.cuda.synchronize()
        t0_, t1_ = ext.fetch_timing()
        acc += np.maximum(t1_ - t0_, 0)
    acc /= 20
    node_of = prog.node_of_item()
    large = [g for g in range(prog.n_buckets) if int(prog.nodes[node_of[g]]["kind"]) == 1]
    top = sorted(large, key=lambda g: -acc[g])[:3]
    fam = ext.node_kernels(io=False)
    items = [{"item": int(g), "w": int(prog.buckets[g]["w"]), "k": int(prog.buckets[g]["k"]),
              "kernel": fam[node_of[g]], "live_us": round(float(acc[g]) / 1e3, 1),
              "node_bytes_MB": round(lcp.ex.node_bytes(node_of[g]) / 1e6, 1)} for g in top]
    del ext
    g = top[0]
    gr, fam0 = lcp.ex.node_graph(node_of[g])
    lcp.ex.launch(stream)                 # the node's inputs in the arena
    for _ in range(3):
        lcp.ex.launch_graph(gr, stream)
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        lcp.ex.launch_graph(gr, stream)
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    dur = sum(a.elapsed_time(b) for a, b in ts) / reps / 1e3
    b = prog.buckets[g]
    nd = prog.nodes[node_of[g]]
    key = f"{lcp.dtype}:{fam0}:w{int(b['w'])}k{int(b['k'])}"
    return {"item": int(g), "kernel": fam0, "key": key, "w": int(b["w"]), "k": int(b["k"]),
            "items": list(range(int(nd["first"]), int(nd["first"]) + int(nd["count"]))),
            "flops": node_flops(prog, node_of[g]),
            "bytes": lcp.ex.node_bytes(node_of[g]), "us": dur * 1e6, "top_items_live": items}


def sustained_clocks(lcp, stream, flush, seconds, local):
    """The step repeated for >= `seconds` under the clock sampler."""
    import torch
    n = 0
    with ClockSampler(local, period=0.005) as clk:
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            for _ in range(50):
                flush.zero_()
                lcp.ex.launch(stream)
            torch.cuda.synchronize()
            n += 50
    s = clk.summary()
    s["loop_s"] = round(time.perf_counter() - t0, 3)
    s["steps"] = n
    return s


def run_ours(args):
    import torch
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import _native as N

    rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    hd = "complex128" if args.dtype == "c128" else "complex64"
    sd = "complex64" if hd == "complex128" else "complex128"
    g, params, lc, order = build_workload()
    tn = lc.network
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    slots = torch.zeros(2 * world, dtype=torch.float64, device="cuda")

    progs = {d: _Lightcone(lc, order, d, local) for d in (hd, sd)}
    for lcp in progs.values():
        for _ in range(max(3, args.warmup)):
            lcp.ex.launch(stream)
    torch.cuda.synchronize()
    val = {d: complex(*progs[d].ex.results[:2].cpu().numpy()) for d in progs}

    # ---- headline: device time, K steps, clocks sampled during the region ----
    with ClockSampler(local) as clk:
        t_dev = time_device(progs[hd], stream, flush, args.steps, world, rank, slots)
    clocks = clk.summary()
    t_dev = max_over_ranks(t_dev, world)
    t_side = max_over_ranks(time_device(progs[sd], stream, flush, args.steps, world, rank, slots), world)

    # ---- e2e through the public API, new angles every step ----
    nets = [build_workload(seed=SEED + 1 + k)[2].network for k in range(8)]
    e2e = {}
    for d in (hd, sd):
        be = Q.Backend.b200(dtype=d, device=local, profile=False)
        t, vals = time_e2e(nets, order, be, args.steps, world)
        e2e[d] = (max_over_ranks(t, world), vals)

    # ---- dominant kernel alone + sustained clocks ----
    dom = dominant_kernel(progs[hd], stream, flush)
    sustained = sustained_clocks(progs[hd], stream, flush, args.sustain_s, local)

    strong = None
    if not args.no_strong:
        strong = graph_figure(args, rank, world, local, "complex64", stream, flush)

    if rank != 0:
        finish(world)
        return 0
    peak, peak_src = peak_hbm()
    prog = progs[hd].prog
    ms = 1e3 * t_dev / args.steps
    alg, exe = prog.algorithmic_bytes(), progs[hd].ex.executed_bytes()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        dt, v_cpu = cpu_oracle_time(lc, order, args.cpu_sample)
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"{args.cpu_sample} full contractions of the cfg-2 lightcone, oracle port of the reference "
                         f"NumPy path (complex128, one core); <ZZ> = {v_cpu.real:.15f}"}
    ref_zz = val["complex128"].real
    rel64 = abs(val["complex64"].real - ref_zz) / abs(ref_zz)
    esz = {"complex64": 8, "complex128": 16}
    h2d = {d: progs[d].ex.img_bytes for d in progs}
    value = world * args.steps / t_dev
    achieved = dom["bytes"] / dom["us"] / 1e3
    traffic = ncu_traffic(dom["key"])
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms, "s_per_lightcone": t_dev / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": value * PAPER_BEST_S,
        "dtype": args.dtype, "data": "synthetic (seeded graph/angles)", "config": CONFIG,
        "details": {
            "parallelism": f"{world} rank(s), one cfg-2 lightcone per rank per step" +
                           (", per-rank <ZZ> slots all-reduced (NCCL) inside the step" if world > 1 else ""),
            "l2": L2_NOTE, "zz": val[hd].real, "program": prog.describe(),
            "kernel_mix": progs[hd].ex.kernel_mix(io=False),
            "route_config": N.route_config(),
            "algorithmic_bytes_per_step": alg, "executed_bytes_per_step": exe,
            "vs_baseline_ref": "value x 2.1 s: speed-up over the paper's best single-lightcone time "
                               "(NumPy+CuPy mixed on V100, PAPER.md:64)",
            "side_dtype": {"dtype": sd, "ms_per_step": 1e3 * t_side / args.steps,
                           "value": world * args.steps / t_side, "zz": val[sd].real,
                           "e2e_value": world * args.steps / e2e[sd][0]},
            "c64_rel_err_vs_c128": rel64,
        },
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": (traffic or {}).get("dram_bytes"), "peak_source": peak_src,
            "kernel": f"{dom['kernel']} on item(s) {dom['items']} (w={dom['w']}, k={dom['k']}), node timed alone with "
                      f"CUDA events ({dom['us']:.1f} us per launch); achieved = compulsory bytes (members once + "
                      f"result once{'; a K6 pair neither writes nor reads its producer result' if dom['kernel'] == 'K6' else ''}"
                      f" = {dom['bytes']}) / launch duration",
            "dominant_share_of_step": dom["us"] / 1e3 / ms,
            "arith": arith_block(dom, hd),
            "traffic_source": (traffic or {}).get("source"),
            "step": {"executed_GBps": exe / (ms / 1e3) / 1e9, "frac_executed": exe / (ms / 1e3) / 1e9 / peak,
                     "frac_vs_unfused": alg / (ms / 1e3) / 1e9 / peak,
                     "note": "whole step at ms_per_step: executed = bytes the fused items must move; unfused = "
                             "SURVEY 8(d) algorithmic bytes (every reference bucket's members + result, incl. "
                             "intermediates the merged items never write)"},
            "top_items_live": dom["top_items_live"],
        },
        "cpu_baseline": cpu,
        "e2e": {"value": world * args.steps / e2e[hd][0], "unit": UNIT, "h2d_bytes_per_step": h2d[hd],
                "d2h_bytes_per_step": 16, "s_per_lightcone": e2e[hd][0] / args.steps,
                "call": "paper_2210_15874_b200.contract_network(tn_k, order, Backend.b200(...)) from host Tensors, "
                        "tn_k = the lightcone at QaoaParams.seeded(4, 1 + k % 8): new gate tensors every step",
                "h2d_note": f"input image per step ({'complex128 + complex64 copies' if hd == 'complex64' else 'complex128'})"},
        "gpu_launches": args.steps * sum(progs[hd].ex.kernel_mix(io=False).values()),
        "gpu_launches_note": f"{sum(progs[hd].ex.kernel_mix(io=False).values())} kernels per step "
                             f"({prog.n_nodes} graph nodes), issued as one CUDA graph launch",
        "clocks": clocks,
        "clocks_sustained": sustained,
        "strong": strong,
    }
    print(json.dumps(line), flush=True)
    finish(world)
    return 0


# ---------------------------------------------------------------------------
# full graph (strong scaling)
# ---------------------------------------------------------------------------
def graph_setup(args, rank, world, local, dtype):
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import distributed as D
    g = Q.random_regular_graph(N_QUBITS, DEGREE, seed=SEED)
    params = Q.QaoaParams.seeded(P_LAYERS, SEED)
    be = Q.Backend.b200(dtype=dtype, device=local, profile=False)
    t0 = time.perf_counter()
    c = Q.qaoa_maxcut_circuit(g, params)
    cones = [Q.extract_lightcone(c, e, cone="tight", simplify=args.simplify) for e in g.edges]
    plan = D.plan_units(cones, be, mem_cap=GRAPH_MEM_CAP, balance_ranks=GRAPH_BALANCE)
    t_plan = time.perf_counter() - t0
    owner = D.lpt_assign([u.cost for u in plan.units], world)
    mine = [u for u in range(len(plan.units)) if owner[u] == rank]
    prep = D.prepare_local(plan, mine, be, local)
    return g, params, be, cones, plan, prep, t_plan


def graph_figure(args, rank, world, local, dtype, stream, flush):
    """Full-graph energy (45 tight cones, LPT over the ranks, slot all-reduce)
    device throughput at this N — the strong-scaling figure."""
    import torch
    import torch.distributed as dist
    from paper_2210_15874_b200 import distributed as D
    g, params, be, cones, plan, prep, t_plan = graph_setup(args, rank, world, local, dtype)
    n_units = len(plan.units)
    slots = torch.zeros(2 * n_units, dtype=torch.float64, device="cuda")
    idx = [torch.tensor([2 * u + q for u in batch for q in (0, 1)], device="cuda") for _, batch in prep.batches]

    def step():
        D.launch_prepared(prep, stream)
        slots.zero_()
        for (ex, batch), ix in zip(prep.batches, idx):
            slots.index_copy_(0, ix, ex.results[: 2 * len(batch)])
        if world > 1:
            dist.all_reduce(slots)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    barrier(world)
    steps = max(3, min(args.steps, 20))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    t = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs) / 1e3, world)
    v = slots.cpu().numpy()
    zz = [0j] * len(cones)
    for u, unit in enumerate(plan.units):
        zz[unit.cone] += complex(v[2 * u], v[2 * u + 1])
    energy = sum(0.5 * (1 - z.real) for z in zz)
    shares = None
    if world == 1 and not args.no_shares:
        shares = rank_shares(plan, be, local, stream, flush)
    return {"metric": "lightcones/s (N=30,p=4 full-graph energy, 45 tight lightcones)",
            "value": len(cones) * steps / t, "ms_per_energy": 1e3 * t / steps, "n_gpus": world, "dtype": dtype,
            "rank_shares": shares,
            "scaling": "strong", "units": n_units, "energy": energy, "steps": steps,
            "lpt_makespan_share": round(_lpt_share([u.cost for u in plan.units], world), 4),
            "host_plan_s": round(t_plan, 3)}


def rank_shares(plan, be, local, stream, flush, ns=(2, 4, 8), reps=5):
    """Predicted strong scaling from this one GPU: for N ranks, each rank's
    LPT share of the units is built as its own program and timed ALONE
    (CUDA events, L2 flushed); the N-rank makespan is the slowest share (the
    ranks never wait on one another until the final all-reduce of a few KB).
    A prediction, not a multi-GPU measurement."""
    import torch
    from paper_2210_15874_b200 import distributed as D
    costs = [u.cost for u in plan.units]
    out = {}
    for n in ns:
        owner = D.lpt_assign(costs, n)
        worst = 0.0
        per_rank = []
        for r in range(n):
            mine = [u for u in range(len(plan.units)) if owner[u] == r]
            if not mine:
                continue
            prep = D.prepare_local(plan, mine, be, local)
            for _ in range(2):
                D.launch_prepared(prep, stream)
            ts = []
            for _ in range(reps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                D.launch_prepared(prep, stream)
                b.record(stream)
                ts.append((a, b))
            torch.cuda.synchronize()
            t_r = sum(a.elapsed_time(b) for a, b in ts) / reps
            per_rank.append({"units": len(mine), "ms": round(t_r, 4),
                             "cost_share": round(sum(costs[u] for u in mine) / max(sum(costs), 1e-30), 4)})
            worst = max(worst, t_r)
            del prep
        out[str(n)] = {"makespan_ms": round(worst, 4), "ranks": per_rank}
    return out


def run_graph(args):
    """Full MaxCut energy of the N=30, p=4 graph: 45 tight lightcones as
    (cone, slice) units, LPT-sharded over ranks, each rank's units batched
    into device programs, per-step slot-vector all-reduce (NCCL at N > 1)."""
    import torch
    import torch.distributed as dist
    import paper_2210_15874_b200 as Q

    rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    dtype = "complex64" if args.dtype == "c64" else "complex128"
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    with ClockSampler(local) as clk:
        fig = graph_figure(args, rank, world, local, dtype, stream, flush)
    g = Q.random_regular_graph(N_QUBITS, DEGREE, seed=SEED)
    params = Q.QaoaParams.seeded(P_LAYERS, SEED)
    be = Q.Backend.b200(dtype=dtype, device=local, profile=False)
    barrier(world)
    grp = dist.group.WORLD if world > 1 else None
    t0 = time.perf_counter()
    e_api = Q.qaoa_energy(g, params, be, cone="tight", group=grp, simplify=args.simplify, mem_cap=GRAPH_MEM_CAP,
                          balance_ranks=GRAPH_BALANCE)
    torch.cuda.synchronize()
    t_cold = max_over_ranks(time.perf_counter() - t0, world)
    n_sweep = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for k in range(n_sweep):
        Q.qaoa_energy(g, Q.QaoaParams.seeded(P_LAYERS, 100 + k), be, cone="tight", group=grp,
                      simplify=args.simplify, mem_cap=GRAPH_MEM_CAP, balance_ranks=GRAPH_BALANCE)
    torch.cuda.synchronize()
    t_api = max_over_ranks((time.perf_counter() - t0) / n_sweep, world)
    if rank != 0:
        finish(world)
        return 0
    peak, peak_src = peak_hbm()
    line = {
        "metric": fig["metric"], "value": fig["value"], "unit": UNIT, "n_gpus": world, "steps": fig["steps"],
        "warmup": 3, "ms_per_step": fig["ms_per_energy"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (seeded graph/angles)",
        "config": {"workload": "graph: all 45 tight lightcones of the cfg-2 graph, over-wide cones sliced for 8-way "
                               "balance, LPT over ranks, slot all-reduce", "l2": L2_NOTE},
        "details": fig,
        "roofline": None,
        "cpu_baseline": None,
        "e2e": {"value": 45 / t_api, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                "call": f"qaoa_energy(g, QaoaParams.seeded(4, 100+k), backend, cone='tight'): angle sweep of "
                        f"{n_sweep} calls", "cold_call_s": t_cold, "energy": e_api},
        "gpu_launches": None,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    finish(world)
    return 0


# ---------------------------------------------------------------------------
# cfg-5 bucket microbench (K3)
# ---------------------------------------------------------------------------
BUCKET_CASES = [(w, cls, k) for w in (24, 26, 28) for cls, k in (("A", 3), ("A", 6), ("B", 2))]


def run_bucket(args):
    """cfg 5 (BASELINE.json configs[4]): synthetic buckets of random complex
    tensors over binary indices in random axis permutations, one bucket index
    contracted by K3 (csrc/bucket_strided.cu).  A step = one launch per case
    of BUCKET_CASES; value = compulsory bytes of all cases / device time
    (every member read once, result written once; inputs > L2 and L2
    flushed between launches)."""
    import torch
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import _native as N
    from paper_2210_15874_b200 import engine as E
    from paper_2210_15874_b200 import workloads as W

    rank, world, local = dist_setup()
    torch.cuda.set_device(local)
    dtype = "complex64" if args.dtype == "c64" else "complex128"
    esz = E.ELEM_BYTES[dtype]
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cases = []
    for w, cls, k in BUCKET_CASES:
        mem = W.synthetic_bucket_device(w, k, cls, 0, dtype, device=local)
        b = Q.Bucket(W.BUCKET, [Q.DeviceTensor(i, t) for i, t in mem])
        st = Q.tensor_core.bucket_strides(b, tuple(range(1, w + 1)))
        out = torch.empty(1 << w, dtype=mem[0][1].dtype, device="cuda")
        d = N.bucket_desc(E.DTYPE_CODE[dtype], w, out.data_ptr(), [(t.data_ptr(), x) for (_, t), x in zip(mem, st)])
        cases.append({"w": w, "cls": cls, "k": k, "desc": d, "keep": (mem, out), "bytes": W.bucket_bytes(mem, w, esz),
                      "plan": N.bucket_plan(d), "t": 0.0})
    for _ in range(max(3, args.warmup)):
        for c in cases:
            N.bucket_launch(c["desc"], stream.cuda_stream)
    torch.cuda.synchronize()
    barrier(world)
    evs = []
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            for c in cases:
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                N.bucket_launch(c["desc"], stream.cuda_stream)
                e1.record(stream)
                evs.append((c, e0, e1))
        torch.cuda.synchronize()
    for c, e0, e1 in evs:
        c["t"] += e0.elapsed_time(e1) / 1e3
    t_dev = max_over_ranks(sum(c["t"] for c in cases), world)
    tot_bytes = sum(c["bytes"] for c in cases) * args.steps
    we, ke = 22, 3
    host = [Q.Tensor(i, d) for i, d in W.synthetic_bucket(we, ke, "A", 0)]
    be = Q.Backend.b200(dtype=dtype, device=local, profile=False)
    bh = Q.Bucket(W.BUCKET, host)
    Q.contract_bucket(bh, be)
    n_e2e = max(2, min(args.steps, 5))
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        Q.contract_bucket(bh, be)
    t_e2e = max_over_ranks((time.perf_counter() - t0) / n_e2e, world)
    e2e_bytes = (sum(1 << len(t.indices) for t in host) + (1 << we)) * esz
    if rank != 0:
        finish(world)
        return 0
    peak, peak_src = peak_hbm()
    value = world * tot_bytes / t_dev / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import qtn_oracle as O   # CPU baseline only
        mem = W.synthetic_bucket(20, 3, "A", 0)
        t0 = time.perf_counter()
        O.bucket_fast(W.BUCKET, mem)
        dt = time.perf_counter() - t0
        cpu = {"value": W.bucket_bytes(mem, 20, 16) / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
               "sample": "one w=20 class-A k=3 bucket through the oracle port of fast_kernel (numpy complex128)"}
    sweep = [{"w": c["w"], "class": c["cls"], "k": c["k"], "GBps": round(c["bytes"] * args.steps / c["t"] / 1e9, 1),
              "frac": round(c["bytes"] * args.steps / c["t"] / 1e9 / peak, 3), "tile_bits": c["plan"][0],
              "staged": c["plan"][4], "folded": c["plan"][5], "invariant": c["plan"][7]} for c in cases]
    line = {
        "metric": "GB/s (cfg-5 synthetic bucket contraction, K3)", "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": 1e3 * t_dev / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (seeded standard complex normal entries, random index permutations)",
        "config": {"workload": "cfg5: buckets w in {24,26,28} x {class A k=3, class A k=6, class B k=2}, one bucket "
                               "index contracted, members in random axis order",
                   "l2": "inputs > L2 and flushed (256 MiB write) before every launch", "sweep": sweep},
        "roofline": {"bound": "hbm", "achieved": value, "peak": peak, "unit": "GB/s", "frac": value / peak,
                     "traffic": None, "peak_source": peak_src, "kernel": "k3v2_kernel (csrc/bucket_strided.cu)"},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_bytes / t_e2e / 1e9, "unit": "GB/s", "h2d_bytes_per_step": e2e_bytes - (1 << we) * esz,
                "d2h_bytes_per_step": (1 << we) * esz, "call": f"contract_bucket(Bucket of host Tensors), w={we} class A k={ke}"},
        "gpu_launches": args.steps * len(cases),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    finish(world)
    return 0


def run_selftest(args):
    """The multi-rank harness without a GPU (gloo): rendezvous, barrier,
    max-over-ranks and the slot-vector all-reduce exactly as the GPU
    workloads use them, on a deterministic per-rank value."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_setup()
    t = max_over_ranks(0.001 * (rank + 1), world)
    slots = torch.zeros(2 * world, dtype=torch.float64)
    slots[2 * rank: 2 * rank + 2] = torch.tensor([rank + 1.0, -(rank + 1.0)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(slots)
    barrier(world)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_ranks": world, "max_over_ranks": t,
                          "slots": slots.tolist(), "backend": dist.get_backend() if world > 1 else None}), flush=True)
    finish(world)
    return 0


def _lpt_share(costs, n):
    """Largest rank load / total under the LPT assignment (algorithmic bytes):
    the predicted strong-scaling limit at n ranks is 1 / this."""
    from paper_2210_15874_b200 import distributed as D
    own = D.lpt_assign(costs, n)
    load = [0] * n
    for c, r in zip(costs, own):
        load[r] += c
    return max(load) / max(1, sum(costs))


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, argv)
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "selftest":
        return run_selftest(args)
    if args.workload == "graph":
        return run_graph(args)
    if args.workload == "bucket":
        return run_bucket(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
