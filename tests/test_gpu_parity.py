"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Tolerances (BASELINE.json north_star):
complex128 <= 1e-10 (relative on scalars; 1e-12 abs on bucket elements),
complex64 <= 1e-5."""
import numpy as np
import pytest

from conftest import load_golden_buckets, load_json
from oracle import qtn_oracle as O

import paper_2210_15874_b200 as Q

pytestmark = pytest.mark.gpu
C128 = Q.Backend.b200(dtype="complex128")
C64 = Q.Backend.b200(dtype="complex64")


def _cfg(name):
    g = load_json("qaoa.json")[name]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"])) if "edges" in g else None
    params = Q.QaoaParams(g["p"], g["gammas"], g["betas"])
    return g, graph, params


@pytest.mark.parametrize("case", range(len(load_golden_buckets())))
def test_bucket_golden_c128(case):
    bidx, mem, ridx, rdata = load_golden_buckets()[case]
    b = Q.Bucket(bidx, [Q.Tensor(i, d) for i, d in mem])
    out, st = Q.contract_bucket(b, C128)
    assert out.indices == ridx and st.width == len(ridx)
    np.testing.assert_allclose(out.data, rdata, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("case", range(len(load_golden_buckets())))
def test_bucket_golden_c64(case):
    bidx, mem, ridx, rdata = load_golden_buckets()[case]
    b = Q.Bucket(bidx, [Q.Tensor(i, d) for i, d in mem])
    out, _ = Q.contract_bucket(b, C64)
    scale = max(1.0, float(np.abs(rdata).max()))
    np.testing.assert_allclose(out.data, rdata, rtol=1e-5, atol=1e-5 * scale)


def test_bucket_device_tensors_stay_on_device():
    rng = np.random.default_rng(5)
    a = Q.Tensor((3, 1, 0), rng.standard_normal((2, 2, 2)) + 1j * rng.standard_normal((2, 2, 2)))
    b = Q.Tensor((0, 2), rng.standard_normal((2, 2)) + 0j)
    da = Q.DeviceTensor.from_host(a)
    out, _ = Q.contract_bucket(Q.Bucket(0, [da, b]), C128)
    assert isinstance(out, Q.DeviceTensor) and out.indices == (1, 2, 3)
    ridx, ref = O.bucket_fast(0, [(a.indices, a.data), (b.indices, b.data)])
    np.testing.assert_allclose(out.data, ref, atol=1e-12)


def test_bucket_errors():
    with pytest.raises(ValueError, match="empty bucket"):
        Q.contract_bucket(Q.Bucket(0, []), C128)


@pytest.mark.parametrize("k", range(12))
def test_networks_golden(k):
    rec = load_json("networks.json")[k]
    c = Q.Circuit(rec["n"], [Q.Gate(a, tuple(b), x) for a, b, x in rec["gates"]])
    tn = Q.amplitude_network(c, rec["bits"])
    order = rec["order_minfill"]
    for be, tol in ((C128, 1e-10), (C64, 1e-5)):
        v, stats = Q.contract_network(tn, order, be)
        assert abs(v - complex(*rec["value"])) <= tol
        assert [s.width for s in stats] == [w for w in rec["widths_minfill"]]
        sv = Q.contract_sliced(tn, order, rec["sliced"], be)
        assert abs(sv - complex(*rec["sliced_value"])) <= tol


def test_cfg1_energy_c128_c64():
    g, graph, params = _cfg("cfg1")
    e128 = Q.qaoa_energy(graph, params, C128)
    assert abs(e128 - g["energy"]) <= 1e-10 * abs(g["energy"])
    e64 = Q.qaoa_energy(graph, params, C64)
    assert abs(e64 - g["energy"]) <= 1e-5 * abs(g["energy"])
    det = Q.qaoa_energy_detailed(graph, params, C128)
    for (edge, zz, stats), rec in zip(det, g["cones"]):
        assert list(edge) == rec["edge"]
        assert abs(zz - rec["zz"][0]) <= 1e-10
        assert [s.width for s in stats] == rec["widths"]


@pytest.mark.parametrize("ci", [0, 1])
def test_cfg2_lightcone(ci):
    g, graph, params = _cfg("cfg2")
    rec = g["cones"][ci]
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
    order = Q.greedy_order(lc.network)
    assert order == rec["order"]
    v128, st = Q.contract_network(lc.network, order, C128)
    assert abs(v128.real - rec["zz"][0]) <= 1e-10
    assert [s.width for s in st] == rec["widths"]
    v64, _ = Q.contract_network(lc.network, order, C64)
    # north star: complex64 relative error <= 1e-5 on the lightcone value
    # (the gates enter K2 unrounded, qtn_program_t.inputs_hi)
    assert abs(v64.real - rec["zz"][0]) <= 1e-5 * abs(rec["zz"][0])
    # repeated launches of the cached program (self-resetting control block)
    for _ in range(3):
        again, _ = Q.contract_network(lc.network, order, C64)
        assert again == v64


def test_cfg2_sliced_equals_unsliced():
    g, graph, params = _cfg("cfg2")
    rec = g["cones"][1]
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
    order = rec["order"]
    sl = Q.suggest_slicing(lc.network, order, 21)
    assert Q.dry_run(lc.network, order, fixed=sl).contraction_width <= 21
    v = Q.contract_sliced(lc.network, order, sl, C128)
    assert abs(v.real - rec["zz"][0]) <= 1e-10


def test_cfg3_energy_tight_c64():
    g, graph, params = _cfg("cfg3")
    e = Q.qaoa_energy(graph, params, C64, cone="tight")
    assert abs(e - g["energy"]) <= 1e-5 * abs(g["energy"])
    det = Q.qaoa_energy_detailed(graph, params, C128, cone="tight")
    for (edge, zz, _), rec in zip(det, g["cones_tight"]):
        assert abs(zz - rec["zz"][0]) <= 1e-10


def test_cfg4_sample_cones():
    g = load_json("qaoa.json")["cfg4"]
    graph = Q.random_regular_graph(200, 3, seed=0)
    params = Q.QaoaParams(5, g["gammas"], g["betas"])
    c = Q.qaoa_maxcut_circuit(graph, params)
    for rec in g["cones"]:
        lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
        order = Q.greedy_order(lc.network)
        v, st = Q.contract_network(lc.network, order, C64)
        assert abs(v.real - rec["zz"][0]) <= 1e-5
        assert [s.width for s in st] == rec["widths"]


def test_memory_cap_and_open_network():
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, (0, 15), cone="tight")
    order = Q.greedy_order(lc.network)
    with pytest.raises(Q.MemoryCapError, match="memory cap exceeded"):
        Q.contract_network(lc.network, order, C64, mem_cap=1 << 20)
    tn = Q.TensorNetwork([Q.Tensor((0,), [1, 2])], open_indices=(0,))
    with pytest.raises(ValueError, match="closed"):
        Q.contract_network(tn, [], C64)


def test_rank0_and_scalar_inputs():
    tn = Q.TensorNetwork([Q.Tensor((), 2.0 + 1j), Q.Tensor((0,), [1, 2]), Q.Tensor((0,), [3, 4j])])
    v, st = Q.contract_network(tn, [0], C128)
    assert abs(v - (2 + 1j) * (3 + 8j)) < 1e-12
    assert [s.width for s in st] == [0]


def test_forced_memory_reuse_on_device(monkeypatch):
    """Liveness reuse with WAR dependencies forced on every block: graph edges
    and in-stage counters must order writers after readers on the device."""
    from paper_2210_15874_b200 import engine as E
    monkeypatch.setattr(E, "REUSE_MIN_ELEMS", 1)
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    for dtype, tol in (("complex64", 1e-5), ("complex128", 1e-10)):
        insts, raws, want = [], [], []
        for rec in g["cones"]:
            lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
            t = E.plan_template([x.indices for x in lc.network.tensors], rec["order"], dtype)
            insts.append(E.Instance(t))
            raws.append(np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors]))
            want.append(rec["zz"][0])
        prog = E.Program(insts, dtype, reuse_above=0)
        assert prog.reuse
        ex = E.Executor(prog)
        for _ in range(2):
            vals = ex.run(raws)
            for v, w in zip(vals, want):
                assert abs(v.real - w) <= tol


def test_energy_sweep_reuses_plans():
    """qaoa_energy over an angle sweep: the second structure-identical call
    reuses plans and device programs (only inputs re-staged) and still
    matches the oracle for its own angles."""
    import time
    from paper_2210_15874_b200 import tn_build as T
    g = Q.random_regular_graph(12, 3, seed=4)
    vals = []
    for seed in range(3):
        params = Q.QaoaParams.seeded(2, seed)
        e = Q.qaoa_energy(g, params, C128, cone="tight")
        c = Q.qaoa_maxcut_circuit(g, params)
        ref = 0.0
        for edge in g.edges:
            lc = Q.extract_lightcone(c, edge, cone="tight")
            v, _ = O.contract_network([(t.indices, t.data) for t in lc.network.tensors], Q.greedy_order(lc.network))
            ref += 0.5 * (1 - v.real)
        assert abs(e - ref) <= 1e-10 * abs(ref)
        vals.append(e)
    assert len(set(vals)) == 3
    assert any(len(cache) > 0 for _, cache in T._ENERGY_PLANS.values())


_K3_ROUTE_CHECK = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np
from conftest import load_json
import paper_2210_15874_b200 as Q
errs = []
for rec in load_json("networks.json"):
    c = Q.Circuit(rec["n"], [Q.Gate(a, tuple(b), x) for a, b, x in rec["gates"]])
    tn = Q.amplitude_network(c, rec["bits"])
    for dt, tol in (("complex64", 1e-5), ("complex128", 1e-10)):
        v, _ = Q.contract_network(tn, rec["order_minfill"], Q.Backend.b200(dtype=dt))
        errs.append(abs(v - complex(*rec["value"])) / tol)
g = Q.random_regular_graph(30, 3, seed=0)
lc = Q.extract_lightcone(Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(4, 0)), (0, 15), cone="tight")
for dt, tol in (("complex64", 1e-5), ("complex128", 1e-10)):
    v, _ = Q.contract_network(lc.network, Q.greedy_order(lc.network), Q.Backend.b200(dtype=dt))
    errs.append(abs(v.real - (-0.0017371891851279)) / tol)
print(max(errs))
"""


@pytest.mark.parametrize("route", ["1", "2"])
def test_program_items_through_k3(route):
    """Program graphs with large items routed to K3 (QTN_K3_ROUTE, read once
    per process): golden networks and the cfg-2 cone at both dtypes."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _K3_ROUTE_CHECK.format(root=root, tests=os.path.join(root, "tests"))
    env = dict(os.environ, QTN_K3_ROUTE=route)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1.0


def test_streamed_batches_shared_arena():
    """Units that do not fit in one program's HBM budget run as streamed
    batches through one shared, growing arena (batch k+1 prepared and queued
    while k runs): same values as one batch, golden <ZZ> per cone."""
    from paper_2210_15874_b200 import distributed as D
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    recs = g["cones"]
    cones = [Q.extract_lightcone(c, tuple(r["edge"]), cone="tight") for r in recs]
    for be, tol in ((C64, 1e-5), (C128, 1e-10)):
        plan = D.plan_units(cones, be, slice_target=20, mem_cap=1 << 40)
        mine = list(range(len(plan.units)))
        one, _ = D.run_local(plan, mine, be, 0, budget_bytes=1 << 40)
        # ascending unit sizes: every few batches need a bigger arena
        mine_sorted = sorted(mine, key=lambda u: plan.units[u].cost)
        cache = {}
        streamed, _ = D.run_local(plan, mine_sorted, be, 0, budget_bytes=1, cache=cache)
        assert set(streamed) == set(one)
        for u in mine:
            assert abs(streamed[u] - one[u]) <= tol * 1e-2
        # the next call on the same structure replays the kept host programs
        assert any(k[0] == "streamed" for k in cache)
        again, _ = D.run_local(plan, mine_sorted, be, 0, budget_bytes=1, cache=cache)
        assert again == streamed
        zz = [0j] * len(cones)
        for u, unit in enumerate(plan.units):
            zz[unit.cone] += streamed[u]
        for z, r in zip(zz, recs):
            assert abs(z.real - r["zz"][0]) <= tol


_K4_CHECK = _K3_ROUTE_CHECK.replace("print(max(errs))", r"""
from paper_2210_15874_b200 import engine as E
mix = {{}}
for dt in ("complex64", "complex128"):
    t = E.plan_template([x.indices for x in lc.network.tensors], Q.greedy_order(lc.network), dt, wave_aware=True)
    ex = E.Executor(E.Program([E.Instance(t)], dt))
    mix[dt] = ex.kernel_mix()
    raw = np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors])
    v = ex.run([raw])[0]
    errs.append(abs(v.real - (-0.0017371891851279)) / (1e-5 if dt == "complex64" else 1e-10))
print(mix["complex64"]["K4"], mix["complex128"]["K4"])
print(max(errs))""")


@pytest.mark.parametrize("min_e", ["1", "3", "0"])
def test_program_items_through_k4(min_e):
    """Expansion items routed to K4 (QTN_K4 = fewest expansion bits, 0 =
    off): golden networks and the cfg-2 cone at both dtypes, and the cfg-2
    program really contains K4 nodes unless K4 is off."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = _K4_CHECK.format(root=root, tests=os.path.join(root, "tests"))
    env = dict(os.environ, QTN_K4=min_e)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    assert float(lines[-1]) <= 1.0
    n64, n128 = (int(x) for x in lines[-2].split())
    if min_e == "0":
        assert n64 == 0 and n128 == 0
    else:
        assert n64 > 0 and n128 > 0


def test_k6_pairs_with_memory_reuse_repeatable():
    """Programs with K6 pairs and liveness reuse of the large blocks (cfg-4
    cones sliced to 26, one batch, 75 pairs): NaN-poisoned arena (no
    uninitialised read), bitwise-identical repeat launches (no race between a
    pair's reads and its result writes), values equal to the no-reuse
    program."""
    from paper_2210_15874_b200 import distributed as D
    from paper_2210_15874_b200 import engine as E
    g = Q.random_regular_graph(200, 3, seed=0)
    c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(5, 0))
    cones = [Q.extract_lightcone(c, e, cone="tight") for e in g.edges[:12]]
    plan = D.plan_units(cones, C64, slice_target=26, mem_cap=1 << 40, n_workers=4)
    insts = [E.Instance(plan.templates[u.cone], u.assignment) for u in plan.units]
    raws = [plan.raws[u.cone] for u in plan.units]
    base = E.Executor(E.Program(insts, "complex64", reuse_above=1 << 62)).run(raws)
    prog = E.Program(insts, "complex64", reuse_above=0)
    assert prog.reuse and len(prog.fused) > 10
    ex = E.Executor(prog)
    ex.buf.fill_(float("nan"))
    first = np.array(ex.run(raws))
    assert np.isfinite(first).all()
    for _ in range(2):
        assert (np.array(ex.run(raws)) == first).all()
    np.testing.assert_allclose(first, np.array(base), rtol=1e-6, atol=1e-9)
