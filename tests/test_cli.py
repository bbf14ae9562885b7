"""CLI (reference: src/cli.py; tests/test_cli.py): same subcommands, flags,
output formats and exit codes (0 ok, 2 usage, 3 resource cap) on the B200
backend.  CPU tests cover parsing, dry runs, error paths and the threshold
selection rule; GPU tests run the contractions."""
import numpy as np
import pytest

from paper_2210_15874_b200 import tuning
from paper_2210_15874_b200.cli import main

BELL_CIRCUIT = "H 0\nCX 0 1\n"
TRIANGLE_GRAPH = "# triangle\nnodes 3\n0 1\n0 2\n1 2\n"


@pytest.fixture
def bell(tmp_path):
    path = tmp_path / "bell.txt"
    path.write_text(BELL_CIRCUIT)
    return path


@pytest.fixture
def triangle(tmp_path):
    path = tmp_path / "triangle.txt"
    path.write_text(TRIANGLE_GRAPH)
    return path


def run(capsys, *argv):
    code = main(list(argv))
    out = capsys.readouterr()
    return code, out.out, out.err


# ---------------------------------------------------------------- CPU ----
def test_usage_error_unknown_flag():
    assert main(["amplitude", "--bogus"]) == 2


def test_amplitude_bad_bitstring_exits_2(capsys, bell):
    code, _, err = run(capsys, "amplitude", "--circuit", str(bell), "--bitstring", "0")
    assert code == 2 and "bitstring length mismatch" in err


def test_amplitude_missing_file_exits_2(capsys, tmp_path):
    assert run(capsys, "amplitude", "--circuit", str(tmp_path / "nope.txt"), "--bitstring", "0")[0] == 2


def test_amplitude_memory_cap_exits_3(capsys, tmp_path):
    # the cap is checked on the plan, before any device work
    path = tmp_path / "wide.txt"
    n = 8
    lines = [f"H {q}" for q in range(n)] + [f"CX {q} {(q + 1) % n}" for q in range(n)] * 2
    path.write_text("\n".join(lines) + "\n")
    code, _, err = run(capsys, "amplitude", "--circuit", str(path), "--bitstring", "0" * n, "--mem-cap", "16")
    assert code == 3 and "memory cap" in err


def test_qaoa_dry_run_profile(capsys, triangle, tmp_path):
    profile = tmp_path / "widths.csv"
    code, out, _ = run(capsys, "qaoa-energy", "--graph", str(triangle), "--dry-run", "--profile", str(profile))
    assert code == 0 and "contraction width" in out and "width<5" in out
    lines = profile.read_text().strip().splitlines()
    assert lines[0] == "lightcone,step,bucket_index,width" and len(lines) > 1


def test_qaoa_dry_run_tight_cone(capsys, tmp_path):
    g = tmp_path / "g.txt"
    from paper_2210_15874_b200 import random_regular_graph
    gr = random_regular_graph(16, 3, seed=0)
    g.write_text(f"nodes {gr.n_nodes}\n" + "".join(f"{u} {v}\n" for u, v in gr.edges))
    code, out_ref, _ = run(capsys, "qaoa-energy", "--graph", str(g), "--p", "2", "--dry-run")
    code2, out_tight, _ = run(capsys, "qaoa-energy", "--graph", str(g), "--p", "2", "--dry-run", "--cone", "tight")
    assert code == code2 == 0
    wr = [int(x.split()[-1]) for x in out_ref.splitlines() if "contraction width" in x]
    wt = [int(x.split()[-1]) for x in out_tight.splitlines() if "contraction width" in x]
    assert len(wr) == len(wt) == len(gr.edges) and max(wt) <= max(wr)


def test_bad_angles_exit_2(capsys, triangle):
    code, _, err = run(capsys, "qaoa-energy", "--graph", str(triangle), "--p", "2", "--gammas", "0.1,0.2,0.3",
                       "--dry-run")
    assert code == 2 and "angles" in err


def test_choose_threshold_rule():
    # K2 beats K1 below width 5, K1 wins from 5 on; K1 cannot run widths < 3
    t = tuning.KernelTimings({}, {}, {})
    for w in range(0, 10):
        t.counts[w] = 10
        t.ref_ns[w] = [100.0 * (w + 1)]
        if w >= 3:
            t.fast_ns[w] = [600.0 - 10 * w]
    rep = tuning.choose_threshold(t)
    assert rep.crossover == 5
    assert rep.best_threshold == 4
    assert rep.all_fast_total_ns == float("inf")
    assert rep.mixed_total_ns == pytest.approx(sum(10 * 100.0 * (w + 1) for w in range(5))
                                               + sum(10 * (600.0 - 10 * w) for w in range(5, 10)))


def test_crossover_csv(tmp_path):
    t = tuning.KernelTimings({2: [10, 20]}, {5: [7]}, {2: 2, 5: 1})
    p = tmp_path / "x.csv"
    tuning.write_crossover_csv(p, t)
    assert p.read_text().splitlines() == ["width,mean_ns_reference,mean_ns_fast", "2,15.0,", "5,,7.0"]


# ---------------------------------------------------------------- GPU ----
@pytest.mark.gpu
def test_amplitude_bell(capsys, bell):
    code, out, _ = run(capsys, "amplitude", "--circuit", str(bell), "--bitstring", "00")
    assert code == 0 and out.strip() == "0.70710678 0.0"


@pytest.mark.gpu
def test_amplitude_stats_csv(capsys, bell, tmp_path):
    stats = tmp_path / "stats.csv"
    code, _, _ = run(capsys, "amplitude", "--circuit", str(bell), "--bitstring", "11", "--stats-out", str(stats))
    assert code == 0
    lines = stats.read_text().strip().splitlines()
    assert lines[0] == "step,bucket_index,width,elapsed_ns,backend" and len(lines) > 1
    for line in lines[1:]:
        step, idx, width, ns, backend = line.split(",")
        assert backend in ("b200-small", "b200-large")


@pytest.mark.gpu
def test_qaoa_energy_triangle_zero_angles(capsys, triangle):
    code, out, _ = run(capsys, "qaoa-energy", "--graph", str(triangle), "--p", "1", "--gammas", "0", "--betas", "0")
    assert code == 0 and float(out.strip()) == pytest.approx(1.5, abs=1e-10)


@pytest.mark.gpu
def test_qaoa_energy_matches_library_and_dtypes(capsys, triangle):
    import paper_2210_15874_b200 as Q
    args = ("qaoa-energy", "--graph", str(triangle), "--p", "2", "--gammas", "0.5,0.3", "--betas", "0.2,0.4")
    code, out, _ = run(capsys, *args)
    g = Q.Graph(3, ((0, 1), (0, 2), (1, 2)))
    expected = Q.qaoa_energy(g, Q.QaoaParams(2, [0.5, 0.3], [0.2, 0.4]), Q.Backend.b200())
    assert code == 0 and float(out.strip()) == pytest.approx(expected, abs=1e-10)
    code, out64, _ = run(capsys, *args, "--dtype", "complex64", "--cone", "tight")
    assert code == 0 and float(out64.strip()) == pytest.approx(expected, rel=1e-5)


@pytest.mark.gpu
def test_qaoa_profile_aggregated(capsys, triangle, tmp_path):
    profile = tmp_path / "profile.csv"
    code, _, _ = run(capsys, "qaoa-energy", "--graph", str(triangle), "--profile", str(profile))
    assert code == 0
    lines = profile.read_text().strip().splitlines()
    assert lines[0] == "lightcone,step,width,count,total_time_ns,mean_time_ns,backend" and len(lines) > 1


@pytest.mark.gpu
def test_tune_threshold(capsys, tmp_path):
    g = tmp_path / "g.txt"
    from paper_2210_15874_b200 import random_regular_graph
    gr = random_regular_graph(16, 3, seed=0)
    g.write_text(f"nodes {gr.n_nodes}\n" + "".join(f"{u} {v}\n" for u, v in gr.edges))
    out_csv = tmp_path / "x.csv"
    code, out, _ = run(capsys, "tune-threshold", "--graph", str(g), "--p", "2", "--edges", "2", "--cone", "tight",
                       "--out", str(out_csv))
    assert code == 0
    keys = {line.split()[0] for line in out.splitlines()}
    assert {"crossover_width", "best_threshold", "measured_best_threshold"} <= keys
    assert out_csv.read_text().splitlines()[0] == "width,mean_ns_reference,mean_ns_fast"
