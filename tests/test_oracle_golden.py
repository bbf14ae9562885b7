"""Pin the CPU oracle (oracle/qtn_oracle.py) against golden vectors produced
by the real reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import load_golden_buckets, load_json
from oracle import qtn_oracle as O


def _gates(rec):
    return [(k, tuple(q), a) for k, q, a in rec["gates"]]


@pytest.mark.parametrize("case", range(len(load_golden_buckets())))
def test_bucket_fast_matches_reference(case):
    bidx, mem, ridx, rdata = load_golden_buckets()[case]
    got_idx, got = O.bucket_fast(bidx, mem)
    assert got_idx == ridx
    np.testing.assert_allclose(got, rdata, rtol=0, atol=1e-12)
    if len(ridx) <= 8:
        bidx2, b = O.bucket_brute(bidx, mem)
        np.testing.assert_allclose(b, rdata, atol=1e-10)


def test_known_answers():
    # src tests: marginal 7-1j (tests/test_tensor_core.py:21-27), identity (30-35)
    _, v = O.bucket_fast(0, [((0,), np.array([3 + 1j, 4 - 2j]))])
    assert v.reshape(()) == pytest.approx(7 - 1j)
    idx, v = O.bucket_fast(0, [((0,), np.array([1.0, 2.0])), ((0, 1), np.eye(2))])
    assert idx == (1,)
    np.testing.assert_allclose(v, [1, 2])
    with pytest.raises(ValueError, match="empty bucket"):
        O.bucket_fast(0, [])


@pytest.mark.parametrize("k", range(12))
def test_networks_orders_widths_values(k):
    rec = load_json("networks.json")[k]
    ts = O.amplitude_tensors(rec["n"], _gates(rec), rec["bits"])
    for h in ("minfill", "mindegree"):
        order = O.greedy_order(ts, h)
        assert order == rec[f"order_{h}"]
        widths, _ = O.dry_run([i for i, _ in ts], order)
        assert widths == rec[f"widths_{h}"]
    val, _ = O.contract_network(ts, rec["order_minfill"])
    assert abs(val - complex(*rec["value"])) < 1e-12
    sv = O.contract_sliced(ts, rec["order_minfill"], rec["sliced"])
    assert abs(sv - complex(*rec["sliced_value"])) < 1e-12
    if "suggest" in rec:
        assert O.suggest_slicing([i for i, _ in ts], rec["order_minfill"], rec["slice_target"]) == rec["suggest"]


def test_cfg1_energy_and_orders():
    g = load_json("qaoa.json")["cfg1"]
    edges = [tuple(e) for e in g["edges"]]
    assert edges == O.random_regular_graph(10, 3, 0)
    gm, bt = O.seeded_angles(1)
    assert gm == g["gammas"] and bt == g["betas"]
    tot = 0.0
    for rec in g["cones"]:
        ts = O.lightcone_tensors(10, edges, gm, bt, tuple(rec["edge"]), "reference")
        order = O.greedy_order(ts)
        assert order == rec["order"]
        v, widths = O.contract_network(ts, order)
        assert widths == rec["widths"]
        assert abs(v.real - rec["zz"][0]) < 1e-12
        tot += 0.5 * (1 - v.real)
    assert tot == pytest.approx(6.544118993880201, abs=1e-12)
    assert abs(tot - O.statevector_energy(10, edges, gm, bt)) < 1e-10


def test_cfg2_tight_cone_structure():
    g = load_json("qaoa.json")["cfg2"]
    edges = [tuple(e) for e in g["edges"]]
    assert edges == O.random_regular_graph(30, 3, 0)
    gm, bt = O.seeded_angles(4)
    for rec in g["cones"]:
        ts = O.lightcone_tensors(30, edges, gm, bt, tuple(rec["edge"]), "tight")
        assert len(ts) == rec["n_tensors"]
        order = O.greedy_order(ts)
        assert order == rec["order"]
        widths, _ = O.dry_run([i for i, _ in ts], order)
        assert widths == rec["widths"]


def test_cfg2_w22_value():
    """Full numpy contraction of the width-22 cone (~1 s)."""
    g = load_json("qaoa.json")["cfg2"]
    edges = [tuple(e) for e in g["edges"]]
    gm, bt = O.seeded_angles(4)
    rec = g["cones"][0]
    ts = O.lightcone_tensors(30, edges, gm, bt, tuple(rec["edge"]), "tight")
    v, _ = O.contract_network(ts, rec["order"])
    assert abs(v.real - rec["zz"][0]) < 1e-12


def test_cfg3_slicing_choice():
    g = load_json("qaoa.json")["cfg3"]
    edges = [tuple(e) for e in g["edges"]]
    gm, bt = O.seeded_angles(3)
    rc = g["ref_cone"]
    ts = O.lightcone_tensors(30, edges, gm, bt, tuple(rc["edge"]), "reference")
    order = O.greedy_order(ts)
    assert order == rc["order"]
    sets = [i for i, _ in ts]
    assert O.dry_run(sets, order)[0] == rc["widths"]
    assert O.suggest_slicing(sets, order, 30) == rc["suggest_30"]
    assert O.suggest_slicing(sets, order, 24) == rc["suggest_24"]
