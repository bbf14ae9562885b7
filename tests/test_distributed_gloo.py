"""N > 1 path on CPU: LPT sharding of (cone, slice) units and the slot-vector
all-reduce, world_size 2 over gloo.  Each rank executes its units with the
numpy program interpreter (tests/emulator.py) in place of the device run, so
the host logic (plan_units, lpt_assign, run_units, _combine) is exactly the
product's.  Checks: energies equal the single-rank result bit for bit and the
golden reference energy."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, load_json


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulated_run_local(plan, mine, backend, device, budget_bytes=None, cache=None):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from emulator import run_program
    from paper_2210_15874_b200 import engine as E
    vals, stats = {}, {}
    for u in mine:
        unit = plan.units[u]
        prog = E.Program([E.Instance(plan.templates[unit.cone], unit.assignment)], backend.dtype)
        vals[u] = complex(run_program(prog, [plan.raws[unit.cone]])[0])
    return vals, stats


def _energy(world, rank, port, out, slice_target, balance=None):
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import distributed as D
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    D.run_local = _emulated_run_local
    g = load_json("qaoa.json")["cfg1"]
    graph = Q.Graph(g["n"], tuple(tuple(e) for e in g["edges"]))
    params = Q.QaoaParams(g["p"], g["gammas"], g["betas"])
    be = Q.Backend.b200(dtype="complex128")
    c = Q.qaoa_maxcut_circuit(graph, params)
    cones = [Q.extract_lightcone(c, e) for e in graph.edges]
    plan = D.plan_units(cones, be, slice_target=slice_target, balance_ranks=balance)
    vals, _ = D.run_units(plan, be)
    e = sum(0.5 * (1.0 - v.real) for v in vals)
    owner = D.lpt_assign([u.cost for u in plan.units], max(world, 1))
    out[rank] = (e, len(plan.units), owner)
    if world > 1:
        dist.destroy_process_group()


def _worker(rank, world, port, out, slice_target, balance):
    _energy(world, rank, port, out, slice_target, balance)


@pytest.mark.parametrize("slice_target,balance", [(None, None), (2, None), (None, 16)])
def test_gloo_world2_matches_single_rank(slice_target, balance):
    """Energies are bitwise identical for 1 and 2 ranks, also with slicing
    and with balance slicing (the plan depends on balance_ranks only)."""
    single = {}
    _energy(1, 0, 0, single, slice_target, balance)
    e1, n_units, _ = single[0]
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out, slice_target, balance), nprocs=2, join=True)
    g = load_json("qaoa.json")["cfg1"]
    for r in (0, 1):
        e, n, owner = out[r]
        assert n == n_units
        assert e == e1                         # bitwise: one contributor per slot
        assert set(owner) == {0, 1}            # both ranks got work
    assert abs(e1 - g["energy"]) < 1e-10
    if slice_target is not None or balance is not None:
        assert n_units > len(g["cones"])       # some cones were sliced


def test_lpt_assignment_balanced_and_deterministic():
    from paper_2210_15874_b200 import distributed as D
    rng = np.random.default_rng(0)
    costs = [int(x) for x in rng.integers(1, 1000, size=45)]
    for n in (1, 2, 4, 8):
        own = D.lpt_assign(costs, n)
        assert own == D.lpt_assign(costs, n)
        loads = [sum(c for c, o in zip(costs, own) if o == r) for r in range(n)]
        assert max(loads) - min(loads) <= max(costs)


def test_balance_slicing_spreads_the_heaviest_cone():
    """plan_units(balance_ranks=8) on N=30 p=4 tight cones: no unit above
    total / 16 (the widest cone holds ~16 % of the unit cost unsliced:
    executed bytes + a per-unit latency charge, distributed.unit_cost), LPT
    makespan at 8 ranks within 15 % of ideal, total cost inflated < 25 %
    (the extra slices' latency charges)."""
    import paper_2210_15874_b200 as Q
    from paper_2210_15874_b200 import distributed as D
    g = Q.random_regular_graph(30, 3, seed=0)
    c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(4, 0))
    cones = [Q.extract_lightcone(c, e, cone="tight") for e in g.edges]
    be = Q.Backend.b200(dtype="complex64")
    p0 = D.plan_units(cones, be, mem_cap=1 << 40)
    p8 = D.plan_units(cones, be, mem_cap=1 << 40, balance_ranks=8)
    c0 = [u.cost for u in p0.units]
    c8 = [u.cost for u in p8.units]
    assert max(c0) > 0.12 * sum(c0)
    assert max(c8) <= sum(c8) / 16
    assert sum(c8) < 1.25 * sum(c0)
    own = D.lpt_assign(c8, 8)
    load = [sum(c for c, o in zip(c8, own) if o == r) for r in range(8)]
    assert max(load) <= 1.15 * sum(c8) / 8


@pytest.mark.gpu
def test_single_process_nccl_slot_allreduce():
    """The single-process multi-GPU reduction (qaoa_energy(n_gpus=N)): one
    NCCL all-reduce over per-device slot vectors; on a 1-GPU box the
    communicator has one member — the code path and exactness still hold."""
    import torch
    from paper_2210_15874_b200 import distributed as D
    n = torch.cuda.device_count()
    vecs = []
    for r in range(n):
        v = torch.zeros(8, dtype=torch.float64, device=f"cuda:{r}")
        v[2 * (r % 4)] = 1.0 + r
        vecs.append(v)
    out = D.slot_allreduce_devices(vecs)
    want = np.zeros(8)
    for r in range(n):
        want[2 * (r % 4)] += 1.0 + r
    assert np.array_equal(out, want)
