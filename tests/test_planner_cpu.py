"""Host planner parity (CPU): orders, dry runs and slicing choices equal the
reference's golden outputs; device programs emulated in numpy equal the
oracle's values."""
import os

import numpy as np
import pytest

from conftest import load_golden_buckets, load_json
from emulator import run_program
from oracle import qtn_oracle as O

import paper_2210_15874_b200 as Q
from paper_2210_15874_b200 import engine as E


def _gates(rec):
    return [Q.Gate(k, tuple(q), a) for k, q, a in rec["gates"]]


def _cfg(name):
    g = load_json("qaoa.json")[name]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"]))
    params = Q.QaoaParams(g["p"], g["gammas"], g["betas"])
    return g, graph, params


def _emulate(tn, order, dtype="complex128", fixed=(), assignment=None):
    t = E.plan_template([x.indices for x in tn.tensors], order, dtype, fixed)
    prog = E.Program([E.Instance(t, assignment or {})], dtype)
    raw = np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])
    return run_program(prog, [raw])[0], t, prog


@pytest.mark.parametrize("k", range(12))
def test_network_orders_and_values(k):
    rec = load_json("networks.json")[k]
    c = Q.Circuit(rec["n"], _gates(rec))
    tn = Q.amplitude_network(c, rec["bits"])
    for h in ("minfill", "mindegree"):
        order = Q.greedy_order(tn, h)
        assert order == rec[f"order_{h}"]
        assert list(Q.dry_run(tn, order).per_bucket_widths) == rec[f"widths_{h}"]
    v, t, _ = _emulate(tn, rec["order_minfill"])
    assert abs(v - complex(*rec["value"])) < 1e-12
    assert list(t.ref_w) == rec["widths_minfill"]
    if "suggest" in rec:
        assert Q.suggest_slicing(tn, rec["order_minfill"], rec["slice_target"]) == rec["suggest"]
    # sliced: sum of emulated slices
    sl = rec["sliced"]
    t = E.plan_template([x.indices for x in tn.tensors], rec["order_minfill"], "complex128", sl)
    insts = [E.Instance(t, dict(zip(sl, bits))) for bits in np.ndindex(*(2,) * len(sl))]
    prog = E.Program(insts, "complex128")
    raw = np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])
    vals = run_program(prog, [raw] * len(insts))
    assert abs(vals.sum() - complex(*rec["sliced_value"])) < 1e-12


def test_cfg1_emulated_energy():
    g, graph, params = _cfg("cfg1")
    c = Q.qaoa_maxcut_circuit(graph, params)
    tot = 0.0
    for rec in g["cones"]:
        lc = Q.extract_lightcone(c, tuple(rec["edge"]))
        order = Q.greedy_order(lc.network)
        assert order == rec["order"]
        v, _, _ = _emulate(lc.network, order)
        assert abs(v.real - rec["zz"][0]) < 1e-12
        tot += 0.5 * (1 - v.real)
    assert tot == pytest.approx(g["energy"], abs=1e-12)


def test_cfg1_batched_program_and_c64():
    g, graph, params = _cfg("cfg1")
    c = Q.qaoa_maxcut_circuit(graph, params)
    insts, raws = [], []
    for rec in g["cones"]:
        tn = Q.extract_lightcone(c, tuple(rec["edge"])).network
        insts.append(E.Instance(E.plan_template([x.indices for x in tn.tensors], rec["order"], "complex64")))
        raws.append(np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors]))
    prog = E.Program(insts, "complex64")
    vals = run_program(prog, raws)
    for v, rec in zip(vals, g["cones"]):
        assert abs(v.real - rec["zz"][0]) < 1e-5


def test_cfg2_tight_cone_structure_and_plan():
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    for rec in g["cones"]:
        lc = Q.extract_lightcone(c, tuple(rec["edge"]), cone="tight")
        assert len(lc.network.tensors) == rec["n_tensors"]
        order = Q.greedy_order(lc.network)
        assert order == rec["order"]
        assert list(Q.dry_run(lc.network, order).per_bucket_widths) == rec["widths"]
        t = E.plan_template([x.indices for x in lc.network.tensors], order, "complex64")
        assert t.max_width == max(rec["widths"])
        prog = E.Program([E.Instance(t)], "complex64")
        # every dependency points to a lower ticket; smem fits the budget
        tb = prog.buckets["tick_begin"]
        for b in prog.buckets:
            for d in prog.deps[b["dep_begin"]: b["dep_begin"] + b["n_dep"]]:
                assert tb[d["bucket"]] < b["tick_begin"]
        for nd in prog.nodes:
            if nd["kind"] == 1:
                assert nd["smem_bytes"] <= E.SMEM_BUDGET      # large-item staging
            else:
                assert nd["smem_bytes"] <= 227 * 1024          # K2 stage (+ CTA groups)


def test_tight_cone_matches_reference_cone_small():
    """Tight and reference cones give the same <ZZ>."""
    g, graph, params = _cfg("cfg1")
    c = Q.qaoa_maxcut_circuit(graph, params)
    for e in graph.edges[:6]:
        a = Q.extract_lightcone(c, e)
        b = Q.extract_lightcone(c, e, cone="tight")
        va, _, _ = _emulate(a.network, Q.greedy_order(a.network))
        vb, _, _ = _emulate(b.network, Q.greedy_order(b.network))
        assert abs(va - vb) < 1e-13


def test_random_graph_matches_oracle_and_statevector():
    graph = Q.random_regular_graph(8, 3, seed=3)
    params = Q.QaoaParams(2, [0.5, 0.2], [0.3, 0.6])
    c = Q.qaoa_maxcut_circuit(graph, params)
    e_tot = 0.0
    for e in graph.edges:
        lc = Q.extract_lightcone(c, e)
        v, _, _ = _emulate(lc.network, Q.greedy_order(lc.network))
        e_tot += 0.5 * (1 - v.real)
    sv = O.statevector_energy(8, list(graph.edges), list(params.gammas), list(params.betas))
    assert abs(e_tot - sv) < 1e-10


def test_graph_and_params_generators():
    assert list(Q.random_regular_graph(30, 3, 0).edges) == O.random_regular_graph(30, 3, 0)
    p = Q.QaoaParams.seeded(4, 0)
    gm, bt = O.seeded_angles(4, 0)
    assert list(p.gammas) == gm and list(p.betas) == bt


def test_errors_mirror_reference(rng):
    tn = Q.TensorNetwork([Q.Tensor((0, 1), np.ones((2, 2))), Q.Tensor((1,), [1, 2])])
    with pytest.raises(ValueError, match="missing"):
        Q.dry_run(tn, [0])
    with pytest.raises(ValueError):
        Q.greedy_order(tn, "bogus")
    with pytest.raises(ValueError):
        Q.Tensor((0, 0), np.zeros((2, 2)))
    with pytest.raises(ValueError):
        Q.Bucket(3, [Q.Tensor((0,), [1, 2])])
    assert Q.memory_estimate(27) == 2147483648
    assert Q.memory_estimate(27, "complex64") == 1073741824
    with pytest.raises(ValueError):
        Q.memory_estimate(-1)


def test_plan_masks_follow_canonical_layout():
    """Every member of a bucket carries the bucket index as its slowest axis
    and a mask whose bits are a subset of the result axes."""
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, (0, 15), cone="tight")
    order = Q.greedy_order(lc.network)
    t = E.plan_template([x.indices for x in lc.network.tensors], order, "complex64")
    for b in range(len(t.w)):
        full = (1 << int(t.w[b])) - 1
        for k in range(t.mem_ptr[b], t.mem_ptr[b + 1]):
            assert int(t.mem_mask[k]) & ~full == 0
            assert int(t.mem_smask[k]) >> int(t.k[b]) == 0
    # algorithmic bytes of the cfg-2 cone (1.468 GB c64)
    gb = E.algorithmic_bytes(t, "complex64") / 1e9
    assert gb == pytest.approx(1.468, abs=0.01)


def test_kernel_variants_match_member_layout():
    """The K1 specialisation encoded by the planner must agree with the member
    classes the kernel derives (a mismatch would make the kernel gather wrong
    values; the kernel also traps on it)."""
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    for dtype in ("complex64", "complex128"):
        for edge in [(0, 15), (0, 11)]:
            lc = Q.extract_lightcone(c, edge, cone="tight")
            t = E.plan_template([x.indices for x in lc.network.tensors], Q.greedy_order(lc.network), dtype)
            for i in range(t.n_items):
                v = int(t.variant[i])
                if v < 0:
                    continue
                cls = [int(t.mem_cls[j]) for j in range(t.mem_ptr[i], t.mem_ptr[i + 1])]
                masks = [int(t.mem_mask[j]) for j in range(t.mem_ptr[i], t.mem_ptr[i + 1])]
                assert v & 15 == int(t.k[i])
                assert (v >> 4) & 15 == sum(1 for x in cls if x == E.CLS_VARYING)
                assert (v >> 8) & 1 == sum(1 for x in cls if x == E.CLS_STREAMED)
                nb0 = sum(1 for x, m in zip(cls, masks) if x == E.CLS_VARYING and m & 1)
                assert (v >> 12) & 15 == (nb0 if dtype == "complex64" else 0)


@pytest.mark.parametrize("k", range(6))
def test_memory_reuse_programs_emulate_correctly(k, monkeypatch):
    """Forced liveness reuse (every block, WAR dependencies) keeps the
    results: the emulator executes nodes in order and asserts every
    dependency precedes its dependent."""
    monkeypatch.setattr(E, "REUSE_MIN_ELEMS", 1)
    rec = load_json("networks.json")[k]
    c = Q.Circuit(rec["n"], _gates(rec))
    tn = Q.amplitude_network(c, rec["bits"])
    t = E.plan_template([x.indices for x in tn.tensors], rec["order_minfill"], "complex128")
    prog = E.Program([E.Instance(t), E.Instance(t)], "complex128", reuse_above=0)
    assert prog.reuse
    raw = np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors])
    vals = run_program(prog, [raw, raw])
    for v in vals:
        assert abs(v - complex(*rec["value"])) < 1e-12
    no = E.Program([E.Instance(t), E.Instance(t)], "complex128", reuse_above=1 << 62)
    assert prog.arena_elems <= no.arena_elems


def test_memory_reuse_cfg1_batched(monkeypatch):
    monkeypatch.setattr(E, "REUSE_MIN_ELEMS", 1)
    g, graph, params = _cfg("cfg1")
    c = Q.qaoa_maxcut_circuit(graph, params)
    insts, raws = [], []
    for rec in g["cones"]:
        tn = Q.extract_lightcone(c, tuple(rec["edge"])).network
        insts.append(E.Instance(E.plan_template([x.indices for x in tn.tensors], rec["order"], "complex128")))
        raws.append(np.concatenate([np.asarray(x.data).ravel() for x in tn.tensors]))
    prog = E.Program(insts, "complex128", reuse_above=0)
    vals = run_program(prog, raws)
    for v, rec in zip(vals, g["cones"]):
        assert abs(v.real - rec["zz"][0]) < 1e-12


@pytest.mark.parametrize("seed", range(8))
def test_native_greedy_order_matches_python(seed):
    """csrc/planner.cpp (qtn_greedy_order) == the Python restatement, both
    heuristics, with and without open indices."""
    from paper_2210_15874_b200 import ordering as OR
    rng = np.random.default_rng(seed)
    c = Q.Circuit(7, [Q.Gate(k, tuple(q), a) for k, q, a in
                      [("H", (int(rng.integers(7)),), None) if rng.random() < 0.3 else
                       ("ZZ", tuple(int(x) for x in rng.choice(7, 2, replace=False)), 0.3) if rng.random() < 0.5 else
                       ("CX", tuple(int(x) for x in rng.choice(7, 2, replace=False)), None) for _ in range(40)]])
    tn = Q.amplitude_network(c, [0] * 7)
    for h in ("minfill", "mindegree"):
        assert Q.greedy_order(tn, h) == OR.greedy_order_py(tn, h)
    ids = sorted(tn.all_indices())
    opened = Q.TensorNetwork(tn.tensors, open_indices=tuple(ids[:: 7]))
    for h in ("minfill", "mindegree"):
        assert Q.greedy_order(opened, h) == OR.greedy_order_py(opened, h)


def test_simplify_network_preserves_value():
    """simplify_network: same value through the oracle,
    fewer tensors, RX triplets folded."""
    from paper_2210_15874_b200 import tn_build as T
    from oracle import qtn_oracle as O
    g = Q.random_regular_graph(12, 3, seed=1)
    c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(2, 3))
    for e in g.edges[:4]:
        for cone in ("reference", "tight"):
            lc = Q.extract_lightcone(c, e, cone=cone)
            s = T.simplify_network(lc.network)
            assert len(s.tensors) < len(lc.network.tensors)
            v1, _ = O.contract_network([(t.indices, t.data) for t in lc.network.tensors], Q.greedy_order(lc.network))
            v2, _ = O.contract_network([(t.indices, t.data) for t in s.tensors], Q.greedy_order(s))
            assert abs(v1 - v2) < 1e-13
    # amplitude networks (non-QAOA gates): value preserved
    rng = np.random.default_rng(0)
    gates = []
    for _ in range(30):
        a, b = (int(x) for x in rng.choice(5, 2, replace=False))
        kind = ["H", "RX", "RZ", "ZZ", "CX"][int(rng.integers(5))]
        ang = float(rng.uniform(0, 3)) if kind in ("RX", "RZ", "ZZ") else None
        gates.append(Q.Gate(kind, (a, b) if kind in ("ZZ", "CX") else (a,), ang))
    circ = Q.Circuit(5, gates)
    tn = Q.amplitude_network(circ, [0, 1, 1, 0, 1])
    s = T.simplify_network(tn)
    v1, _ = O.contract_network([(t.indices, t.data) for t in tn.tensors], Q.greedy_order(tn))
    v2, _ = O.contract_network([(t.indices, t.data) for t in s.tensors], Q.greedy_order(s))
    assert abs(v1 - v2) < 1e-12 and len(s.tensors) < len(tn.tensors)


def _same_template(a, b):
    import dataclasses
    for f in dataclasses.fields(a):
        x, y = getattr(a, f.name), getattr(b, f.name)
        if isinstance(x, np.ndarray):
            assert x.shape == y.shape and np.array_equal(x, y), f.name
        elif isinstance(x, dict):
            assert x.keys() == y.keys() and all(np.array_equal(x[k], y[k]) for k in x), f.name
        else:
            assert x == y, f.name


def test_native_planner_matches_python_planner():
    """csrc/plan_template.cpp (qtn_plan_build) restates engine.plan_template_py:
    identical templates on QAOA cones (both cone modes, both dtypes, merging
    on/off, several K2 thresholds, wave-aware tiles on/off), sliced networks
    and random circuits."""
    cases = []
    g = Q.random_regular_graph(16, 3, seed=2)
    c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(3, 1))
    for e in g.edges[:6]:
        for cone in ("reference", "tight"):
            lc = Q.extract_lightcone(c, e, cone=cone)
            cases.append((lc.network, Q.greedy_order(lc.network), ()))
    for rec in load_json("networks.json"):
        circ = Q.Circuit(rec["n"], [Q.Gate(a, tuple(b), x) for a, b, x in rec["gates"]])
        tn = Q.amplitude_network(circ, rec["bits"])
        cases.append((tn, rec["order_minfill"], tuple(rec["sliced"])))
        cases.append((tn, rec["order_minfill"], ()))
    for tn, order, fixed in cases:
        ix = [t.indices for t in tn.tensors]
        for dtype in ("complex64", "complex128"):
            for merge, sib, wave in ((True, 12, False), (False, 12, False), (True, 8, False), (True, 16, False),
                                     (True, 12, True), (True, 8, True)):
                a = E.plan_template_py(ix, order, dtype, fixed, merge=merge, small_iter_bits=sib, wave_aware=wave)
                b = E.plan_template(ix, order, dtype, fixed, merge=merge, small_iter_bits=sib, wave_aware=wave)
                _same_template(a, b)


def test_native_planner_errors():
    tn = Q.amplitude_network(Q.Circuit(2, [Q.Gate("H", (0,)), Q.Gate("CX", (0, 1))]), [0, 0])
    order = Q.greedy_order(tn)
    with pytest.raises(ValueError, match="order is missing indices"):
        E.plan_template([t.indices for t in tn.tensors], order[:-1], "complex64")


def test_pool_incremental_coalescing_matches_full_merge():
    """_Pool keeps its free list sorted and coalesced incrementally; the
    allocations (offsets, inherited readers, top) equal those of a pool that
    re-sorts and re-merges the whole list on every insert."""
    import random
    from paper_2210_15874_b200 import engine as E

    class Naive(E._Pool):
        def _insert(self, st, sz, rd):
            self.free.append([st, sz, rd])
            self.free.sort(key=lambda blk: blk[0])
            merged = []
            for blk in self.free:
                if merged and merged[-1][0] + merged[-1][1] == blk[0]:
                    merged[-1][1] += blk[1]
                    merged[-1][2] = merged[-1][2] | blk[2]
                else:
                    merged.append(blk)
            self.free = merged

    for seed in range(20):
        rng = random.Random(seed)
        a, b = E._Pool(7), Naive(7)
        live = []
        for step in range(400):
            if live and rng.random() < 0.45:
                off, size = live.pop(rng.randrange(len(live)))
                a.release(off, size, step)
                b.release(off, size, step)
            else:
                size = 1 << rng.randrange(0, 12)
                align = E._tensor_align(size)
                ra, rb = a.alloc(size, align), b.alloc(size, align)
                assert ra == rb
                live.append((ra[0], size))
            assert a.top == b.top and a.free == b.free


def test_wave_aware_tiles(monkeypatch):
    """Wave-aware plans shrink a large item's tile (by <= 2 bits, never below
    the vector minimum) only when that fills the persistent grid's last wave
    better: w=21 (512 tiles of 2^12 on 444 slots) -> 2^11 at a per-tile cost
    of 1024 results; w=24 keeps 2^12."""
    monkeypatch.setattr(E, "WAVE_OV_ELEMS", 1024)
    slots = E.WAVE_SLOTS["complex64"]
    full = [(1 << 24) - 1]
    assert E._tile_bits(24, full, [3], "complex64", slots)[0] == 12
    assert E._tile_bits(21, [(1 << 21) - 1], [3], "complex64", slots)[0] == 11
    assert E._tile_bits(21, [(1 << 21) - 1], [3], "complex64", 0)[0] == 12
    for w in range(9, 30):
        L0 = E._tile_bits(w, [(1 << w) - 1], [1], "complex64", 0)[0]
        L1 = E._tile_bits(w, [(1 << w) - 1], [1], "complex64", slots)[0]
        assert L0 - 2 <= L1 <= L0 and L1 >= min(w, E.MIN_TILE_BITS["complex64"])


@pytest.mark.parametrize("cone,p", [("tight", 1), ("tight", 3), ("reference", 2)])
def test_energy_angle_recipe_restages_exact_inputs(monkeypatch, cone, p):
    """qaoa_energy angle sweeps: after the first call, the cones' inputs are
    restaged from the angle recipe (no circuit / network rebuild); they equal
    the inputs of freshly built lightcones element for element."""
    from paper_2210_15874_b200 import distributed as D
    from paper_2210_15874_b200 import tn_build as T
    seen = {}

    def fake_run_units(plan, backend, group=None, n_gpus=None, cache=None):
        seen["raws"] = plan.raws
        return [0j] * len(plan.cones), [[] for _ in plan.cones]

    monkeypatch.setattr(D, "run_units", fake_run_units)
    T._ENERGY_RECIPES.clear()
    g = Q.random_regular_graph(14, 3, seed=3)
    be = Q.Backend.b200(dtype="complex64")
    Q.qaoa_energy(g, Q.QaoaParams.seeded(p, 0), be, cone=cone)
    assert len(T._ENERGY_RECIPES) == 1
    for seed in (1, 2):
        params = Q.QaoaParams.seeded(p, seed)
        Q.qaoa_energy(g, params, be, cone=cone)
        c = Q.qaoa_maxcut_circuit(g, params)
        for e, got in zip(g.edges, seen["raws"]):
            ref = np.concatenate([np.asarray(t.data, np.complex128).ravel()
                                  for t in Q.extract_lightcone(c, e, cone=cone).network.tensors])
            assert np.array_equal(got, ref)
    # simplified networks merge gates: no recipe
    T._ENERGY_RECIPES.clear()
    Q.qaoa_energy(g, Q.QaoaParams.seeded(p, 0), be, cone=cone, simplify=True)
    assert len(T._ENERGY_RECIPES) == 0


@pytest.mark.parametrize("ci", [0, 1])
def test_c64_precision_model_cfg2(ci):
    """The complex64 precision model (emulator docstring: K2 in double from
    unrounded gates, large items in complex64) meets the north star's 1e-5
    RELATIVE bar on both cfg-2 cones (narrowing every gate before the
    contraction — the round-1 path — gave 1.1e-5 on (0, 15): the gates'
    rounding is coherent across their many copies)."""
    g, graph, params = _cfg("cfg2")
    rec = g["cones"][ci]
    lc = Q.extract_lightcone(Q.qaoa_maxcut_circuit(graph, params), tuple(rec["edge"]), cone="tight")
    t = E.plan_template([x.indices for x in lc.network.tensors], rec["order"], "complex64", wave_aware=True)
    prog = E.Program([E.Instance(t)], "complex64")
    raw = np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors])
    want = rec["zz"][0]
    v = run_program(prog, [raw])[0]
    assert abs(v.real - want) <= 1e-5 * abs(want)


def test_native_dry_run_and_slicing_match_python():
    """qtn_dry_run / qtn_suggest_slicing (csrc/planner.cpp) against their
    Python restatements (ordering.dry_run_py / suggest_slicing_py) on golden
    amplitude networks, the cfg-3 reference cone and random networks."""
    from paper_2210_15874_b200 import ordering as OR
    nets = []
    for rec in load_json("networks.json"):
        tn = Q.amplitude_network(Q.Circuit(rec["n"], _gates(rec)), rec["bits"])
        nets.append((tn, rec["order_minfill"], [rec.get("slice_target", 3), 2]))
    g, graph, params = _cfg("cfg3")
    lc = Q.extract_lightcone(Q.qaoa_maxcut_circuit(graph, params), tuple(g["ref_cone"]["edge"]))
    nets.append((lc.network, g["ref_cone"]["order"], [20, 14]))
    rng = np.random.default_rng(7)
    for _ in range(20):
        n_idx = int(rng.integers(6, 30))
        ts = [Q.Tensor(tuple(int(x) for x in rng.choice(n_idx, size=int(rng.integers(1, 5)), replace=False)),
                       np.ones((2,) * 1)) if False else None for _ in range(0)]
        ts = []
        for _ in range(int(rng.integers(5, 25))):
            r = int(rng.integers(1, 5))
            ids = tuple(int(x) for x in rng.choice(n_idx, size=r, replace=False))
            ts.append(Q.Tensor(ids, np.ones((2,) * r)))
        tn = Q.TensorNetwork(ts)
        order = [int(x) for x in rng.permutation(sorted(tn.all_indices()))]
        nets.append((tn, order, [2, 3, 4]))
    for tn, order, targets in nets:
        assert Q.dry_run(tn, order) == OR.dry_run_py(tn, order)
        for t in targets:
            sl = Q.suggest_slicing(tn, order, t)
            assert sl == OR.suggest_slicing_py(tn, order, t)
            assert Q.dry_run(tn, order, fixed=sl) == OR.dry_run_py(tn, order, fixed=sl)
    with pytest.raises(ValueError, match="missing"):
        Q.dry_run(nets[0][0], nets[0][1][:-1])
    with pytest.raises(ValueError, match="target_width"):
        Q.suggest_slicing(nets[0][0], nets[0][1], 0)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_producer_consumer_pairs_cfg2(dtype):
    """K6 pairs (engine.Program._pairs): the cfg-2 lightcone's widest
    intermediate (w = 24, read whole by the w = 22 k = 2 item) becomes one pair
    node; every pair's producer is read by its consumer only, as a member that
    carries every consumer index in canonical order; the program still
    evaluates to the oracle's value (emulator runs the pair's items in order)."""
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, (0, 15), cone="tight")
    order = Q.greedy_order(lc.network)
    t = E.plan_template([x.indices for x in lc.network.tensors], order, dtype, wave_aware=True)
    prog = E.Program([E.Instance(t)], dtype)
    B, M = prog.buckets, prog.members
    pairs = [nd for nd in prog.nodes if nd["kind"] == 1 and nd["count"] == 2]
    assert len(pairs) == len(prog.fused) >= 1
    widths = sorted((int(B[nd["first"]]["w"]), int(B[nd["first"] + 1]["w"])) for nd in pairs)
    assert (24, 22) in widths
    for nd in pairs:
        p_, c_ = B[nd["first"]], B[nd["first"] + 1]
        assert p_["w"] == c_["w"] + c_["k"]
        readers = [g for g in range(prog.n_buckets) for m in M[B[g]["mem_begin"]: B[g]["mem_begin"] + B[g]["n_mem"]]
                   if m["off"] == p_["out_off"]]
        assert readers == [nd["first"] + 1]
        m = [m for m in M[c_["mem_begin"]: c_["mem_begin"] + c_["n_mem"]] if m["off"] == p_["out_off"]][0]
        assert m["mask"] == (1 << int(c_["w"])) - 1 and m["smask"] == (1 << int(c_["k"])) - 1
    if dtype == "complex128":   # (the emulator takes ~30 s on this program)
        ts = [(x.indices, x.data) for x in lc.network.tensors]
        ref, _ = O.contract_network(ts, order)
        val = run_program(prog, [np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors])])[0]
        assert abs(val - ref) <= 1e-12 * abs(ref)


def test_pairs_with_memory_reuse(monkeypatch):
    """With liveness reuse a consumer's result may take a block its producer
    read; such a pair cannot run as one K6 kernel (the emulator asserts no
    pair result overlaps a member), and the values stay exact."""
    monkeypatch.setattr(E, "REUSE_MIN_ELEMS", 1)
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, (0, 11), cone="tight")
    order = Q.greedy_order(lc.network)
    t = E.plan_template([x.indices for x in lc.network.tensors], order, "complex128", wave_aware=True)
    prog = E.Program([E.Instance(t), E.Instance(t)], "complex128", reuse_above=0)
    assert prog.reuse
    raw = np.concatenate([np.asarray(x.data).ravel() for x in lc.network.tensors])
    ref, _ = O.contract_network([(x.indices, x.data) for x in lc.network.tensors], order)
    for v in run_program(prog, [raw, raw]):
        assert abs(v - ref) <= 1e-12 * abs(ref)


def test_cfg4_pairs_never_overwrite_their_inputs():
    """cfg-4 (N=200 p=5 tight cones sliced to 32) batched under a 125 GB
    budget: liveness reuse is on and thousands of producer/consumer pairs
    form; no pair's consumer result may take a block its producer reads
    (K6 writes one while reading the other — the race that made cfg-4
    energies run-dependent before the planner excluded such pairs)."""
    from emulator import pair_overlaps
    from paper_2210_15874_b200 import distributed as D
    g = Q.random_regular_graph(200, 3, seed=0)
    c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(5, 0))
    be = Q.Backend.b200(dtype="complex64")
    cones = [Q.extract_lightcone(c, e, cone="tight") for e in g.edges]
    plan = D.plan_units(cones, be, slice_target=32, mem_cap=1 << 40, n_workers=8)
    n_pairs = 0
    for batch in D._batches(list(range(len(plan.units))), plan, be, 125 << 30):
        prog = E.Program([E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in batch],
                         "complex64")
        for nd in prog.nodes:
            if nd["kind"] == 1 and nd["count"] == 2:
                n_pairs += 1
                assert not pair_overlaps(prog, nd)
    assert n_pairs > 1000


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_k6_plan_of_cfg2_pair(dtype):
    """The K6 planner (qtn_bucket_expand_fused_plan, host only) on the cfg-2
    w = 24 -> w = 22 pair: producer k = 2, the consumer's 2 summed bits set
    aside, 4 expansion bits, one gathered consumer member, two uniform ones."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from k6_survey import pair_plans
    g, graph, params = _cfg("cfg2")
    c = Q.qaoa_maxcut_circuit(graph, params)
    lc = Q.extract_lightcone(c, (0, 15), cone="tight")
    order = Q.greedy_order(lc.network)
    t = E.plan_template([x.indices for x in lc.network.tensors], order, dtype, wave_aware=True)
    plans = {(wp, wc): info for wp, wc, info in pair_plans(E.Program([E.Instance(t)], dtype))}
    info = plans[(24, 22)]
    assert not isinstance(info, str), info
    k, nq, ne, nf, ng, nu, nqn, nh = info
    assert (k, nq, ne, ng, nu) == (2, 2, 4, 1, 2)
    assert nf + k <= (12 if dtype == "complex64" else 11)
