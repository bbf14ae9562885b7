"""Reference-API behaviour on CPU (no device):

* the reference's A/B seam: `contract_network` looks `contract_bucket` up by
  module-global name (src/ordering.py:10,181); replacing
  `ordering.contract_bucket` runs the bucket-by-bucket driver on the
  replacement (here the oracle port of fast_kernel — test infrastructure);
* `slice_network` (src/ordering.py:233-248) against the oracle's np.take;
* the imaginary-residue ValueError of `_contract_zz` (src/tn_build.py:13,
  159-162);
* per-bucket stats: a merged item's time split over its buckets."""
import numpy as np
import pytest

from conftest import load_json
from oracle import qtn_oracle as O

import paper_2210_15874_b200 as Q
from paper_2210_15874_b200 import distributed as D
from paper_2210_15874_b200 import engine as E
from paper_2210_15874_b200 import ordering


def _oracle_bucket(b, backend):
    """A process-bucket kernel (the oracle port of fast_kernel) in the
    reference's contract_bucket signature."""
    res, data = O.bucket_fast(b.bucket_index, [(t.indices, t.data) for t in b.tensors])
    return Q.Tensor(res, data), Q.BucketStats(width=len(res), elapsed_ns=0, backend_used="oracle")


def _net(rec):
    c = Q.Circuit(rec["n"], [Q.Gate(a, tuple(b), x) for a, b, x in rec["gates"]])
    return Q.amplitude_network(c, rec["bits"])


@pytest.mark.parametrize("k", range(4))
def test_contract_bucket_seam(monkeypatch, k):
    rec = load_json("networks.json")[k]
    tn = _net(rec)
    monkeypatch.setattr(ordering, "contract_bucket", _oracle_bucket)
    v, stats = Q.contract_network(tn, rec["order_minfill"], Q.Backend.b200())
    assert abs(v - complex(*rec["value"])) < 1e-12
    assert [s.width for s in stats] == rec["widths_minfill"]
    assert {s.backend_used for s in stats} == {"oracle"}
    with pytest.raises(Q.MemoryCapError):
        Q.contract_network(tn, rec["order_minfill"], Q.Backend.b200(), mem_cap=1)


def test_contract_bucket_seam_qaoa_cone(monkeypatch):
    g = load_json("qaoa.json")["cfg1"]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"]))
    c = Q.qaoa_maxcut_circuit(graph, Q.QaoaParams(g["p"], g["gammas"], g["betas"]))
    monkeypatch.setattr(ordering, "contract_bucket", _oracle_bucket)
    for rec in g["cones"][:5]:
        lc = Q.extract_lightcone(c, tuple(rec["edge"]))
        v, stats = Q.contract_network(lc.network, rec["order"], Q.Backend.b200())
        assert abs(v.real - rec["zz"][0]) < 1e-12
        assert [s.width for s in stats] == rec["widths"]


@pytest.mark.parametrize("k", range(6))
def test_slice_network_matches_oracle(k):
    rec = load_json("networks.json")[k]
    tn = _net(rec)
    sl = rec["sliced"]
    ts = [(t.indices, t.data) for t in tn.tensors]
    total = 0j
    for bits in np.ndindex(*(2,) * len(sl)):
        a = dict(zip(sl, (int(x) for x in bits)))
        sub = Q.slice_network(tn, a)
        ref = O.slice_tensors(ts, a)
        assert [t.indices for t in sub.tensors] == [tuple(i) for i, _ in ref]
        for t, (_, d) in zip(sub.tensors, ref):
            np.testing.assert_array_equal(np.asarray(t.data), np.asarray(d))
        order = [i for i in rec["order_minfill"] if i not in a]
        v, _ = O.contract_network([(t.indices, t.data) for t in sub.tensors], order)
        total += v
    assert abs(total - complex(*rec["sliced_value"])) < 1e-12


def test_imaginary_residue_raises(monkeypatch):
    """A lightcone value with |Im| above IMAG_RESIDUE_TOL (1e-8) is an error,
    as in the reference's _contract_zz."""
    g = Q.random_regular_graph(6, 3, seed=1)
    params = Q.QaoaParams.seeded(1, 0)

    def fake_run(plan, backend, group=None, n_gpus=None, cache=None):
        return [0.25 + 3e-6j] + [0.25 + 0j] * (len(plan.cones) - 1), [[] for _ in plan.cones]

    monkeypatch.setattr(D, "run_units", fake_run)
    with pytest.raises(ValueError, match="imaginary residue"):
        Q.qaoa_energy(g, params, Q.Backend.b200(dtype="complex128"))
    # below the bar: accepted, the real part is used
    monkeypatch.setattr(D, "run_units", lambda plan, *a, **k: ([0.25 + 1e-10j] * len(plan.cones),
                                                                [[] for _ in plan.cones]))
    e = Q.qaoa_energy(g, Q.QaoaParams.seeded(1, 1), Q.Backend.b200(dtype="complex128"))
    assert abs(e - 0.5 * 0.75 * len(g.edges)) < 1e-12


def test_stats_split_merged_items():
    """ref_stats: every bucket of a merged item gets a share of the item's
    measured time in proportion to its algorithmic elements; per item the
    shares sum to the item's time exactly."""
    g = load_json("qaoa.json")["cfg2"]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"]))
    c = Q.qaoa_maxcut_circuit(graph, Q.QaoaParams(g["p"], g["gammas"], g["betas"]))
    rec = g["cones"][0]
    lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
    t = E.plan_template([x.indices for x in lc.network.tensors], rec["order"], "complex64")
    assert (t.k > 1).any()                      # merged chains exist
    rng = np.random.default_rng(3)
    el = rng.integers(1000, 100000, t.n_items)
    st = ordering.ref_stats(t, Q.Backend.b200(), el, ["K1"] * t.n_items)
    assert [s.width for s in st] == rec["widths"]
    per = np.zeros(t.n_items, np.int64)
    np.add.at(per, t.ref_item, [s.elapsed_ns for s in st])
    assert (per == el).all()
    assert all(s.elapsed_ns > 0 for s in st)
    assert {s.kernel for s in st} == {"K1"}
