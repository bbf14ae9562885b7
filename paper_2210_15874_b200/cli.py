"""Command-line entry point for the path's subcommands (reference:
src/cli.py — `amplitude` 95-111, `qaoa-energy` 126-183, `tune-threshold`
285-307; exit codes 0 success, 2 usage/config error, 3 resource cap).

Same flags and output formats as the reference; the backend flags map onto
the B200 backend (`--backend reference|fast|mixed` are accepted as aliases,
`--threshold` is the K2/K1 routing width), plus the B200 options
`--dtype complex64|complex128`, `--device`, and for qaoa-energy `--cone
reference|tight`, `--slice-target T`, `--gpus N`.

    python -m paper_2210_15874_b200 qaoa-energy --graph g.txt --p 4 --dtype complex64 --cone tight
"""
from __future__ import annotations

import argparse
import sys

from .circuits import DEFAULT_BETA, DEFAULT_GAMMA, QaoaParams, qaoa_maxcut_circuit, read_circuit, read_graph
from .ordering import DEFAULT_MEM_CAP, MemoryCapError, contract_network, dry_run, greedy_order
from .tensor_core import Backend
from .tn_build import amplitude_network, extract_lightcone, qaoa_energy_detailed

EXIT_OK = 0
EXIT_USAGE = 2
EXIT_RESOURCE = 3


class UsageError(Exception):
    pass


def _parse_angles(text, p, default):
    if text is None:
        return (default,) * p
    vals = tuple(float(x) for x in text.split(","))
    if len(vals) == 1 and p > 1:
        vals = vals * p
    if len(vals) != p:
        raise UsageError(f"expected {p} comma-separated angles, got {len(vals)}")
    return vals


def _backend_from_args(args) -> Backend:
    # every reference kind runs on the B200; the threshold is the K2/K1 split
    return Backend.b200(dtype=args.dtype, threshold=args.threshold, device=args.device,
                        profile=bool(getattr(args, "stats_out", None) or getattr(args, "profile", None)))


def _add_backend_flags(p):
    p.add_argument("--backend", choices=["b200", "reference", "fast", "mixed"], default="b200")
    p.add_argument("--threshold", type=int, default=None,
                   help="K2/K1 routing width (result rank); default: the measured per-dtype value")
    p.add_argument("--heuristic", choices=["minfill", "mindegree"], default="minfill")
    p.add_argument("--mem-cap", type=int, default=DEFAULT_MEM_CAP, help="contraction memory cap in bytes")
    p.add_argument("--dtype", choices=["complex64", "complex128"], default="complex128")
    p.add_argument("--device", type=int, default=0)


def _load_qaoa(args):
    graph = read_graph(args.graph)
    params = QaoaParams(p=args.p, gammas=_parse_angles(args.gammas, args.p, DEFAULT_GAMMA),
                        betas=_parse_angles(args.betas, args.p, DEFAULT_BETA))
    return graph, params


def cmd_amplitude(args) -> int:
    circuit = read_circuit(args.circuit)
    bitstring = [int(ch) for ch in args.bitstring]
    tn = amplitude_network(circuit, bitstring)
    order = greedy_order(tn, args.heuristic)
    value, stats = contract_network(tn, order, _backend_from_args(args), args.mem_cap)
    print(f"{round(value.real, 8)} {round(value.imag, 8)}")
    if args.stats_out:   # same pairing as src/cli.py:104-108
        with open(args.stats_out, "w") as f:
            f.write("step,bucket_index,width,elapsed_ns,backend\n")
            for step, (idx, st) in enumerate(zip(order, stats)):
                f.write(f"{step},{idx},{st.width},{st.elapsed_ns},{st.backend_used}\n")
    return EXIT_OK


def _aggregate_profile(per_cone_stats):
    agg = {}
    for cone_id, stats in per_cone_stats:
        for step, st in enumerate(stats):
            key = (cone_id, st.width, st.backend_used)
            if key not in agg:
                agg[key] = [step, 0, 0]
            agg[key][1] += 1
            agg[key][2] += st.elapsed_ns
    return agg


def cmd_qaoa_energy(args) -> int:
    graph, params = _load_qaoa(args)
    if args.dry_run:
        circuit = qaoa_maxcut_circuit(graph, params)
        all_widths, rows = [], []
        for cone_id, edge in enumerate(graph.edges):
            lc = extract_lightcone(circuit, edge, cone=args.cone)
            order = greedy_order(lc.network, args.heuristic)
            profile = dry_run(lc.network, order)
            all_widths.extend(profile.per_bucket_widths)
            print(f"lightcone {edge}: contraction width {profile.contraction_width}")
            for step, (idx, w) in enumerate(zip(profile.bucket_indices, profile.per_bucket_widths)):
                rows.append((cone_id, step, idx, w))
        small = sum(1 for w in all_widths if w < 5)
        print(f"buckets: {len(all_widths)}, width<5: {100.0 * small / max(1, len(all_widths)):.1f}%")
        if args.profile:
            with open(args.profile, "w") as f:
                f.write("lightcone,step,bucket_index,width\n")
                for row in rows:
                    f.write(",".join(str(x) for x in row) + "\n")
        return EXIT_OK
    detail = qaoa_energy_detailed(graph, params, _backend_from_args(args), args.heuristic, args.mem_cap,
                                  args.threads, cone=args.cone, slice_target=args.slice_target,
                                  n_gpus=args.gpus)
    energy = sum(0.5 * (1.0 - zz) for _, zz, _ in detail)
    print(round(energy, 10))
    if args.profile:
        agg = _aggregate_profile([(cone_id, stats) for cone_id, (_, _, stats) in enumerate(detail)])
        with open(args.profile, "w") as f:
            f.write("lightcone,step,width,count,total_time_ns,mean_time_ns,backend\n")
            for (cone_id, width, bk), (step, count, total) in sorted(agg.items()):
                f.write(f"{cone_id},{step},{width},{count},{total},{total // count},{bk}\n")
    return EXIT_OK


def cmd_tune_threshold(args) -> int:
    from . import tuning
    graph, params = _load_qaoa(args)
    circuit = qaoa_maxcut_circuit(graph, params)
    edges = graph.edges[: args.edges] if args.edges else graph.edges
    be = Backend.b200(dtype=args.dtype, device=args.device)
    cones, orders, parts = [], [], []
    for edge in edges:
        lc = extract_lightcone(circuit, edge, cone=args.cone)
        order = greedy_order(lc.network, args.heuristic)
        cones.append(lc)
        orders.append(order)
        parts.append(tuning.profile_kernels(lc.network, order, args.max_ref_width, be))
    timings = tuning.merge_timings(parts)
    report = tuning.choose_threshold(timings)
    cand = sorted({t for t in range(max(0, report.best_threshold - 3), report.best_threshold + 4)} | {11})
    report.measured = tuning.sweep_thresholds(cones, orders, cand, be)
    report.measured_best = min(report.measured, key=lambda t: (report.measured[t], t))
    if args.out:
        tuning.write_crossover_csv(args.out, timings)
    print(f"crossover_width {report.crossover}")
    print(f"best_threshold {report.best_threshold}")
    print(f"mixed_total_ns {report.mixed_total_ns:.0f}")
    print(f"all_reference_total_ns {report.all_reference_total_ns:.0f}")
    print(f"all_fast_total_ns {report.all_fast_total_ns:.0f}")
    print(f"measured_best_threshold {report.measured_best}")
    for t in sorted(report.measured):
        print(f"measured_total_ns[{t}] {report.measured[t]:.0f}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="qtnsim-b200")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("amplitude", help="contract an amplitude network")
    p.add_argument("--circuit", required=True)
    p.add_argument("--bitstring", required=True)
    p.add_argument("--stats-out")
    _add_backend_flags(p)
    p.set_defaults(func=cmd_amplitude)

    p = sub.add_parser("qaoa-energy", help="MaxCut energy via lightcone contraction")
    p.add_argument("--graph", required=True)
    p.add_argument("--p", type=int, default=1)
    p.add_argument("--gammas")
    p.add_argument("--betas")
    p.add_argument("--dry-run", action="store_true", help="report contraction widths only, no numeric work")
    p.add_argument("--profile", help="per-bucket CSV output path")
    p.add_argument("--plot", action="store_true", help="accepted for compatibility (no plotting here)")
    p.add_argument("--threads", type=int, default=1, help="host threads for ordering / planning")
    p.add_argument("--cone", choices=["reference", "tight"], default="reference")
    p.add_argument("--slice-target", type=int, default=None)
    p.add_argument("--gpus", type=int, default=None, help="GPUs (ranks) to shard lightcones over")
    _add_backend_flags(p)
    p.set_defaults(func=cmd_qaoa_energy)

    p = sub.add_parser("tune-threshold", help="time the K2/K1 routes and pick a width threshold")
    p.add_argument("--graph", required=True)
    p.add_argument("--p", type=int, default=1)
    p.add_argument("--gammas")
    p.add_argument("--betas")
    p.add_argument("--edges", type=int, help="only sample the first N lightcones")
    p.add_argument("--max-ref-width", type=int, default=18)
    p.add_argument("--heuristic", choices=["minfill", "mindegree"], default="minfill")
    p.add_argument("--cone", choices=["reference", "tight"], default="reference")
    p.add_argument("--dtype", choices=["complex64", "complex128"], default="complex64")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--out", help="crossover CSV path")
    p.add_argument("--plot", action="store_true", help="accepted for compatibility (no plotting here)")
    p.set_defaults(func=cmd_tune_threshold)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return EXIT_USAGE if e.code not in (0, None) else 0
    try:
        return args.func(args)
    except MemoryCapError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_RESOURCE
    except (UsageError, ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE


def entry():
    raise SystemExit(main())


if __name__ == "__main__":
    entry()
