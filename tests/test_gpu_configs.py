"""BASELINE configs on the device beyond cfg-1/cfg-2:

* cfg-3 REFERENCE cones (N=30 p=3, widths to 34) sliced to T=30 — (0,11)
  and the two heaviest, (16,25) and (2,25) — at complex64 against the
  golden per-cone <ZZ> (tight-cone golden values equal reference-cone ones
  within 3e-15);
* cfg-4 (N=200 p=5) widest tight cones (width 36-37) sliced: two slicings
  at complex128 agree to 1e-10, complex64 at T=32 to 1e-5;
* simplify_network on the device at complex128;
* the INTEGRATION.md §2 bindings."""
import numpy as np
import pytest

from conftest import load_golden_buckets, load_json

import paper_2210_15874_b200 as Q

pytestmark = pytest.mark.gpu
C128 = Q.Backend.b200(dtype="complex128")
C64 = Q.Backend.b200(dtype="complex64")
BIG_CAP = 160 << 30


def _cfg(name):
    g = load_json("qaoa.json")[name]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"])) if "edges" in g else None
    params = Q.QaoaParams(g["p"], g["gammas"], g["betas"])
    return g, graph, params


@pytest.mark.parametrize("edge", [(0, 11), (16, 25), (2, 25)])
def test_cfg3_reference_cone_sliced_c64(edge):
    g, graph, params = _cfg("cfg3")
    want = {tuple(r["edge"]): r["zz"][0] for r in g["cones_tight"]}[edge]
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, edge)                   # the reference cone
    order = Q.greedy_order(lc.network)
    sl = Q.suggest_slicing(lc.network, order, 30)
    assert Q.dry_run(lc.network, order, fixed=sl).contraction_width <= 30
    if edge != (0, 11):
        assert Q.dry_run(lc.network, order).contraction_width > 30 and sl
    v = Q.contract_sliced(lc.network, order, sl, C64, mem_cap=BIG_CAP)
    assert abs(v.real - want) <= 1e-5 * abs(want), (v, want)


@pytest.mark.parametrize("edge", [(152, 183), (147, 156), (160, 162)])
def test_cfg4_wide_cone_two_slicings(edge):
    d = load_json("qaoa.json")["cfg4"]
    graph = Q.random_regular_graph(200, 3, seed=0)
    c = Q.qaoa_maxcut_circuit(graph, Q.QaoaParams(5, d["gammas"], d["betas"]))
    lc = Q.extract_lightcone(c, edge, cone="tight")
    order = Q.greedy_order(lc.network)
    assert Q.dry_run(lc.network, order).contraction_width >= 36
    vals = {}
    for t, be in ((30, C128), (28, C128), (32, C64)):
        sl = Q.suggest_slicing(lc.network, order, t)
        assert Q.dry_run(lc.network, order, fixed=sl).contraction_width <= t
        vals[(t, be.dtype)] = Q.contract_sliced(lc.network, order, sl, be, mem_cap=BIG_CAP)
    a, b = vals[(30, "complex128")], vals[(28, "complex128")]
    assert abs(a - b) <= 1e-10 * abs(a)
    assert abs(vals[(32, "complex64")].real - a.real) <= 1e-5 * abs(a.real)
    assert abs(a.imag) < 1e-8


def test_simplified_networks_c128():
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    for rec in g["cones"]:
        lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight", simplify=True)
        assert len(lc.network.tensors) < rec["n_tensors"]
        v, _ = Q.contract_network(lc.network, Q.greedy_order(lc.network), C128)
        assert abs(v.real - rec["zz"][0]) <= 1e-10 * abs(rec["zz"][0])
    g1, graph1, params1 = _cfg("cfg1")
    e = Q.qaoa_energy(graph1, params1, C128, simplify=True)
    assert abs(e - g1["energy"]) <= 1e-10 * abs(g1["energy"])


def test_integration_stubs():
    import integration_stubs as S
    g, graph, params = _cfg("cfg2")
    rec = g["cones"][0]
    lc = Q.extract_lightcone(Q.qaoa_maxcut_circuit(graph, params), tuple(rec["edge"]), cone="tight")
    v = S.contract_network_b200(lc.network, rec["order"])
    assert abs(v.real - rec["zz"][0]) <= 1e-10 * abs(rec["zz"][0])
    for bidx, mem, ridx, rdata in load_golden_buckets()[:8]:
        res, out = S.contract_bucket_b200(Q.Bucket(bidx, [Q.Tensor(i, d) for i, d in mem]))
        assert res == ridx
        np.testing.assert_allclose(out, rdata, rtol=1e-12, atol=1e-12)
