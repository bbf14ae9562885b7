"""Race test of the K2 completion-counter protocol under schedule perturbation
(VERDICT r1 "missing" 7; compute-sanitizer is closed on this pool).

A child process runs the cfg-2 lightcone programs with QTN_K2_JITTER set:
every K2 block stalls a pseudo-random 0-4 us before each tile, so producers
finish in an order unrelated to their tickets and to the undisturbed run.
Before EVERY launch the whole device buffer is filled with NaN (the inputs
are re-staged by run()), so a consumer that read a member before its
producer's release-add was visible would read poison (or a value of the
previous launch's different interleaving) and the bits would change.  The
stage grid is varied (all resident blocks, 3, 7) and each configuration is
launched repeatedly (the last-block counter reset between launches).  The
child's bits must equal the unperturbed parent's bit for bit.

The reference has only thread-count determinism tests for this
(tests/test_acceptance.py:272-313)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

GRIDS = (0, 3, 7)
REPS = 5


def _cfg2():
    from conftest import load_json
    return load_json("qaoa.json")["cfg2"]


def _run_all():
    from conftest import load_json
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import engine as E
    g = load_json("qaoa.json")["cfg2"]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"]))
    c = Q.qaoa_maxcut_circuit(graph, Q.QaoaParams(g["p"], g["gammas"], g["betas"]))
    out = {}
    for dtype in ("complex64", "complex128"):
        insts, raws = [], []
        for rec in g["cones"]:
            lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
            insts.append(E.Instance(E.plan_template([x.indices for x in lc.network.tensors], rec["order"], dtype)))
            raws.append(np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors]))
        prog = E.Program(insts, dtype)
        for grid in GRIDS:
            ex = E.Executor(prog)
            ex.c.grid = grid
            runs = []
            for _ in range(REPS):
                ex.buf.fill_(float("nan"))
                v = np.asarray(ex.run(raws), dtype=np.complex128)
                runs.append([[x.real.hex(), x.imag.hex()] for x in v])
            out[f"{dtype}/{grid}"] = runs
    from paper_2210_15874_b200 import _native as N
    return out, {k: str(v) for k, v in N.route_config().items()}


@pytest.mark.gpu
def test_k2_bits_under_schedule_jitter():
    ref, knobs = _run_all()
    assert knobs["k2_jitter"] == "0"
    for key, runs in ref.items():
        assert all(r == runs[0] for r in runs)
        # the unperturbed bits are right (golden <ZZ> from the reference)
        tol = 1e-5 if key.startswith("complex64") else 1e-10
        for (re_, _), rec in zip(runs[0], _cfg2()["cones"]):
            assert abs(float.fromhex(re_) - rec["zz"][0]) <= tol * abs(rec["zz"][0]), key
    for seed in (1, 977):
        env = dict(os.environ, QTN_K2_JITTER=str(seed))
        p = subprocess.run([sys.executable, os.path.abspath(__file__), "--child"], env=env,
                           capture_output=True, text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        got, kn = json.loads(p.stdout.strip().splitlines()[-1])
        assert kn["k2_jitter"] == str(seed)
        for key, runs in ref.items():
            for r in got[key]:
                assert r == runs[0], (seed, key, r, runs[0])


if __name__ == "__main__" and "--child" in sys.argv:
    print(json.dumps(_run_all()))
