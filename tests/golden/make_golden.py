"""Generate golden vectors by running the REAL reference (qtnsim) in the build
container.  The reference lives at /root/reference (read-only, never on the
GPU box), so its outputs are frozen here as small fixtures:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (all under tests/golden/):
  buckets.npz      random buckets (incl. edge cases) + reference fast_kernel
                   results  (src/tensor_core.py:148-164)
  networks.json    min-fill / min-degree orders, dry-run widths, scalar values
                   of small random amplitude networks (src/ordering.py)
  qaoa.json        per-edge <ZZ>, orders and width profiles for the BASELINE
                   configs (cfg 1 ref cones, cfg 2 tight cone, cfg 3 tight
                   cones, cfg 4 sampled narrow tight cones), slicing choices.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from qtnsim.circuits import Circuit, Gate, Graph, QaoaParams, qaoa_maxcut_circuit, random_regular_graph  # noqa: E402
from qtnsim.ordering import contract_network, contract_sliced, dry_run, greedy_order, suggest_slicing  # noqa: E402
from qtnsim.tensor_core import Backend, Bucket, Tensor, fast_kernel  # noqa: E402
from qtnsim.tn_build import amplitude_network, extract_lightcone, zz_sandwich_network  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FAST = Backend.fast()


def seeded_params(p, seed=0):
    rng = np.random.default_rng(seed)
    g = rng.uniform(0, np.pi, p)
    b = rng.uniform(0, np.pi, p)
    return QaoaParams(p, [float(x) for x in g], [float(x) for x in b])


def tight_circuit(g: Graph, params: QaoaParams, edge):
    """SURVEY App. B tight cone, emitted as a circuit for the reference's own
    zz_sandwich_network(prune=True)."""
    sup = set(edge)
    layers = []
    for k in reversed(range(params.p)):
        rx = [Gate("RX", (q,), 2 * params.betas[k]) for q in sorted(sup)]
        ek = [e for e in g.edges if e[0] in sup or e[1] in sup]
        zz = [Gate("ZZ", e, 2 * params.gammas[k]) for e in ek]
        for e in ek:
            sup.update(e)
        layers.append(zz + rx)
    gates = [Gate("H", (q,)) for q in sorted(sup)]
    for lay in reversed(layers):
        gates += lay
    return Circuit(g.n_nodes, gates)


def rand_t(rng, idx):
    shp = (2,) * len(idx)
    return Tensor(idx, rng.standard_normal(shp) + 1j * rng.standard_normal(shp))


def random_circuit(rng, n, m):
    """tests/conftest.py:56-69 gate pool (re-stated; same distribution)."""
    gates = []
    for _ in range(m):
        if n >= 2 and rng.random() < 0.4:
            kind = ["ZZ", "CX"][rng.integers(2)]
            q = rng.choice(n, size=2, replace=False)
            ang = float(rng.uniform(0, 2 * np.pi)) if kind == "ZZ" else None
            gates.append(Gate(kind, tuple(int(x) for x in q), ang))
        else:
            kind = ["H", "X", "Y", "Z", "RX", "RZ"][rng.integers(6)]
            q = int(rng.integers(n))
            ang = float(rng.uniform(0, 2 * np.pi)) if kind in ("RX", "RZ") else None
            gates.append(Gate(kind, (q,), ang))
    return Circuit(n, gates)


def gate_list(c: Circuit):
    return [[g.kind, list(g.qubits), g.angle] for g in c.gates]


def make_buckets():
    rng = np.random.default_rng(20221028)
    cases = []
    # edge cases the reference tests hold (tests/test_tensor_core.py:21-65)
    cases.append((0, [Tensor((0,), [3.0 + 1j, 4.0 - 2j])]))                      # rank-0 result
    cases.append((0, [Tensor((0,), [1.0, 2.0]), Tensor((0, 1), np.eye(2))]))     # identity
    cases.append((5, [rand_t(rng, i) for i in [(5, 1, 2), (5, 3), (5, 2, 4)]]))  # 3 members
    cases.append((0, [rand_t(rng, tuple(range(9))), rand_t(rng, (0,) + tuple(range(9, 17)))]))  # w=16
    cases.append((3, [rand_t(rng, (3,))] * 1 + [rand_t(rng, (3,))]))             # two vectors -> scalar
    # random class A / class B buckets with random permutations (cfg 5 shapes)
    for w in (1, 2, 3, 5, 8, 10, 12):
        for k in (1, 3, 6):
            ids = list(rng.permutation(np.arange(1, 40))[:w])
            big = [0] + ids
            big = [int(x) for x in rng.permutation(big)]
            mem = [rand_t(rng, tuple(big))]
            for _ in range(k - 1):
                r = int(rng.integers(0, min(4, w) + 1))
                sub = [0] + [int(x) for x in rng.choice(ids, size=r, replace=False)]
                mem.append(rand_t(rng, tuple(int(x) for x in rng.permutation(sub))))
            cases.append((0, mem))
    for w in (4, 9, 14):  # class B: two members covering the result together
        ids = [int(x) for x in rng.permutation(np.arange(1, 40))[:w]]
        a = set(rng.choice(ids, size=int(0.6 * w) + 1, replace=False).tolist())
        b = (set(ids) - a) | set(rng.choice(ids, size=int(0.3 * w), replace=False).tolist())
        m1 = rand_t(rng, tuple(int(x) for x in rng.permutation([0] + sorted(a))))
        m2 = rand_t(rng, tuple(int(x) for x in rng.permutation([0] + sorted(b))))
        cases.append((0, [m1, m2]))
    out = {"n": len(cases)}
    for ci, (bidx, mem) in enumerate(cases):
        res = fast_kernel(Bucket(bidx, mem))
        out[f"c{ci}_bidx"] = np.array(bidx)
        out[f"c{ci}_nmem"] = np.array(len(mem))
        for mi, t in enumerate(mem):
            out[f"c{ci}_m{mi}_idx"] = np.array(t.indices, dtype=np.int64)
            out[f"c{ci}_m{mi}_data"] = t.data.ravel().copy()
        out[f"c{ci}_res_idx"] = np.array(res.indices, dtype=np.int64)
        out[f"c{ci}_res_data"] = res.data.ravel().copy()
    np.savez_compressed(os.path.join(HERE, "buckets.npz"), **out)
    print("buckets:", len(cases))


def make_networks():
    rng = np.random.default_rng(777)
    nets = []
    for trial in range(12):
        n = int(rng.integers(3, 8))
        c = random_circuit(rng, n, int(rng.integers(10, 30)))
        bits = [int(b) for b in rng.integers(0, 2, size=n)]
        tn = amplitude_network(c, bits)
        rec = {"n": n, "gates": gate_list(c), "bits": bits}
        for h in ("minfill", "mindegree"):
            order = greedy_order(tn, h)
            rec[f"order_{h}"] = [int(x) for x in order]
            rec[f"widths_{h}"] = [int(x) for x in dry_run(tn, order).per_bucket_widths]
        val, _ = contract_network(tn, rec["order_minfill"], FAST)
        rec["value"] = [val.real, val.imag]
        allidx = sorted(tn.all_indices())
        k = int(rng.integers(1, 4))
        sl = [int(allidx[i]) for i in rng.choice(len(allidx), size=k, replace=False)]
        rec["sliced"] = sl
        sv = contract_sliced(tn, rec["order_minfill"], sl, FAST)
        rec["sliced_value"] = [sv.real, sv.imag]
        base = dry_run(tn, rec["order_minfill"]).contraction_width
        if base >= 2:
            rec["slice_target"] = base - 1
            rec["suggest"] = [int(x) for x in suggest_slicing(tn, rec["order_minfill"], base - 1)]
        nets.append(rec)
    with open(os.path.join(HERE, "networks.json"), "w") as f:
        json.dump(nets, f)
    print("networks:", len(nets))


def cone_record(c, edge, tight=False, g=None, params=None, contract=True, slice_target=None):
    if tight:
        tn = zz_sandwich_network(tight_circuit(g, params, edge), edge, prune=True)
    else:
        tn = extract_lightcone(c, edge).network
    t0 = time.time()
    order = greedy_order(tn)
    t_order = time.time() - t0
    prof = dry_run(tn, order)
    rec = {"edge": list(edge), "n_tensors": len(tn.tensors), "order": [int(x) for x in order],
           "widths": [int(x) for x in prof.per_bucket_widths], "order_s": t_order}
    if slice_target is not None:
        rec["slice_target"] = slice_target
        rec["suggest"] = [int(x) for x in suggest_slicing(tn, order, slice_target)]
    if contract:
        t0 = time.time()
        val, _ = contract_network(tn, order, FAST, mem_cap=1 << 40)
        rec["zz"] = [val.real, val.imag]
        rec["contract_s"] = time.time() - t0
    return rec


def make_qaoa():
    out = {}
    # cfg 1: N=10 p=1, reference cones, all 15 edges
    g = random_regular_graph(10, 3, seed=0)
    pr = seeded_params(1)
    c = qaoa_maxcut_circuit(g, pr)
    recs = [cone_record(c, e) for e in g.edges]
    out["cfg1"] = {"n": 10, "p": 1, "edges": [list(e) for e in g.edges], "gammas": list(pr.gammas),
                   "betas": list(pr.betas), "cones": recs,
                   "energy": sum(0.5 * (1 - r["zz"][0]) for r in recs)}
    print("cfg1 energy", out["cfg1"]["energy"])
    # cfg 2: N=30 p=4, tight cones (0,15) [w=25] and (0,11) [w=22]
    g = random_regular_graph(30, 3, seed=0)
    pr = seeded_params(4)
    c = qaoa_maxcut_circuit(g, pr)
    out["cfg2"] = {"n": 30, "p": 4, "edges": [list(e) for e in g.edges], "gammas": list(pr.gammas),
                   "betas": list(pr.betas),
                   "cones": [cone_record(c, e, tight=True, g=g, params=pr) for e in [(0, 11), (0, 15)]]}
    # widths (no contraction) of every tight cone + ref-cone widths for two edges
    out["cfg2"]["tight_widths"] = {f"{e[0]},{e[1]}": max(cone_record(c, e, True, g, pr, contract=False)["widths"])
                                   for e in g.edges}
    print("cfg2", [r["zz"] for r in out["cfg2"]["cones"]])
    # cfg 3: N=30 p=3, all 45 edges via tight cones (== reference cones within 3e-15)
    pr = seeded_params(3)
    c = qaoa_maxcut_circuit(g, pr)
    recs = [cone_record(c, e, tight=True, g=g, params=pr) for e in g.edges]
    for r in recs:
        r.pop("order")
    out["cfg3"] = {"n": 30, "p": 3, "edges": [list(e) for e in g.edges], "gammas": list(pr.gammas),
                   "betas": list(pr.betas), "cones_tight": recs,
                   "energy": sum(0.5 * (1 - r["zz"][0]) for r in recs)}
    # a reference cone of cfg 3 sliced: slicing choice + sliced value (small target)
    e = (0, 11)
    tn = extract_lightcone(c, e).network
    order = greedy_order(tn)
    prof = dry_run(tn, order)
    out["cfg3"]["ref_cone"] = {"edge": list(e), "order": [int(x) for x in order],
                               "widths": [int(x) for x in prof.per_bucket_widths],
                               "suggest_30": [int(x) for x in suggest_slicing(tn, order, 30)],
                               "suggest_24": [int(x) for x in suggest_slicing(tn, order, 24)]}
    print("cfg3 energy", out["cfg3"]["energy"])
    # cfg 4: N=200 p=5 tight cones: three narrow ones contracted, widths for a sample
    g = random_regular_graph(200, 3, seed=0)
    pr = seeded_params(5)
    c = qaoa_maxcut_circuit(g, pr)
    sample = []
    for e in g.edges[:40]:
        r = cone_record(c, e, True, g, pr, contract=False)
        sample.append((max(r["widths"]), tuple(e)))
    sample.sort()
    picks = [e for _, e in sample[:3]]
    out["cfg4"] = {"n": 200, "p": 5, "gammas": list(pr.gammas), "betas": list(pr.betas),
                   "n_edges": len(g.edges), "edges_head": [list(e) for e in g.edges[:40]],
                   "sample_widths": [[w, list(e)] for w, e in sample],
                   "cones": [cone_record(c, e, True, g, pr) for e in picks]}
    for r in out["cfg4"]["cones"]:
        r.pop("order")
    print("cfg4", [(r["edge"], max(r["widths"]), r["zz"]) for r in out["cfg4"]["cones"]])
    with open(os.path.join(HERE, "qaoa.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    make_buckets()
    make_networks()
    make_qaoa()
