"""CPU oracle for the bucket-elimination hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2210_15874_b200/`) may import this module; only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / --impl reference
legs use it, and only as the checker or as the timed CPU baseline.

This is a compact numpy restatement of the reference's algorithm for the
path (reference = /root/reference/pkg/src/qtnsim, cited as `src/<file>:<line>`).
It is pinned against the reference itself: `tests/golden/make_golden.py`
imports the real reference in the build container and writes golden vectors
(bucket outputs, orders, widths, lightcone <ZZ> values, energies) that
`tests/test_oracle_golden.py` checks this module against.

Layout convention (same as the reference, src/tensor_core.py:3-5): a tensor
is (indices, data) with data complex128 of shape (2,)*rank, C order, the
last listed index fastest.
"""
from __future__ import annotations

import heapq
import itertools

import numpy as np

# ---------------------------------------------------------------------------
# gates / circuits / graphs            (src/circuits.py)
# ---------------------------------------------------------------------------
_SQ2 = np.sqrt(2.0)
_H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / _SQ2
_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
_Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
_Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
_CX = np.eye(4, dtype=np.complex128)[[0, 1, 3, 2]]
DIAG_KINDS = ("Z", "RZ", "ZZ")          # src/circuits.py:12


def gate_diag(kind, angle):
    """Diagonal of Z / RZ / ZZ (src/circuits.py:88-97)."""
    if kind == "Z":
        return np.array([1, -1], dtype=np.complex128)
    if kind == "RZ":
        return np.exp(np.array([-0.5j, 0.5j]) * angle)
    if kind == "ZZ":
        h = 0.5 * angle
        return np.exp(np.array([-1j, 1j, 1j, -1j]) * h)
    raise ValueError(kind)


def gate_matrix(kind, angle):
    """Unitary of a non-diagonal gate (src/circuits.py:68-86)."""
    if kind == "H":
        return _H.copy()
    if kind == "X":
        return _X.copy()
    if kind == "Y":
        return _Y.copy()
    if kind == "CX":
        return _CX.copy()
    if kind == "RX":
        c, s = np.cos(angle / 2), np.sin(angle / 2)
        return np.array([[c, -1j * s], [-1j * s, c]], dtype=np.complex128)
    if kind in DIAG_KINDS:
        return np.diag(gate_diag(kind, angle))
    raise ValueError(kind)


def random_regular_graph(n, d, seed):
    """Pairing model with rejection, numpy default_rng(seed) (src/circuits.py:167-191).

    Returns the sorted edge list."""
    rng = np.random.default_rng(seed)
    stubs = np.repeat(np.arange(n), d)
    for _ in range(100000):
        perm = rng.permutation(stubs)
        pairs = perm.reshape(-1, 2)
        es = set()
        ok = True
        for u, v in pairs:
            u, v = int(u), int(v)
            e = (min(u, v), max(u, v))
            if u == v or e in es:
                ok = False
                break
            es.add(e)
        if ok:
            return sorted(es)
    raise RuntimeError("pairing model failed")


def qaoa_gates(n, edges, gammas, betas):
    """H layer then p x [ZZ(2g) per sorted edge, RX(2b) per qubit] (src/circuits.py:156-164)."""
    gates = [("H", (q,), None) for q in range(n)]
    for g, b in zip(gammas, betas):
        gates += [("ZZ", (u, v), 2.0 * g) for (u, v) in sorted(edges)]
        gates += [("RX", (q,), 2.0 * b) for q in range(n)]
    return gates


def seeded_angles(p, seed=0):
    """rng = default_rng(seed); gammas then betas uniform [0, pi)."""
    rng = np.random.default_rng(seed)
    gammas = rng.uniform(0, np.pi, p)
    betas = rng.uniform(0, np.pi, p)
    return [float(x) for x in gammas], [float(x) for x in betas]


# ---------------------------------------------------------------------------
# network construction                  (src/tn_build.py)
# ---------------------------------------------------------------------------
class _Wires:
    """Live wire id per qubit + fresh-id counter (src/tn_build.py:34-52)."""

    def __init__(self, qubits):
        self.n = 0
        self.cur = {}
        for q in qubits:
            self.cur[q] = self.new()

    def new(self):
        self.n += 1
        return self.n - 1


def _emit(tensors, wires, gate, adjoint=False):
    """Gate -> tensor (src/tn_build.py:55-80): RX = H RZ H; diagonal gates keep
    wire ids; others get fresh output ids (outs then ins)."""
    kind, qs, ang = gate
    if kind == "RX":
        _emit(tensors, wires, ("H", qs, None))
        _emit(tensors, wires, ("RZ", qs, ang), adjoint)
        _emit(tensors, wires, ("H", qs, None))
        return
    if kind in DIAG_KINDS:
        d = gate_diag(kind, ang)
        if adjoint:
            d = d.conj()
        tensors.append((tuple(wires.cur[q] for q in qs), d.reshape((2,) * len(qs))))
        return
    u = gate_matrix(kind, ang)
    if adjoint:
        u = u.conj().T
    outs, ins = [], []
    for q in qs:
        ins.append(wires.cur[q])
        wires.cur[q] = wires.new()
        outs.append(wires.cur[q])
    tensors.append((tuple(outs) + tuple(ins), u.reshape((2,) * (2 * len(qs)))))


_KET0 = np.array([1.0, 0.0], dtype=np.complex128)


def amplitude_tensors(n, gates, bits):
    """<bits| C |0..0> network (src/tn_build.py:83-96)."""
    w = _Wires(range(n))
    ts = [((w.cur[q],), _KET0) for q in range(n)]
    for g in gates:
        _emit(ts, w, g)
    for q, b in enumerate(bits):
        pr = np.zeros(2, dtype=np.complex128)
        pr[int(b)] = 1.0
        ts.append(((w.cur[q],), pr))
    return ts


def reference_cone(gates, edge):
    """Backward support scan (src/tn_build.py:106-118)."""
    sup = set(edge)
    keep = []
    for g in reversed(gates):
        if sup.intersection(g[1]):
            keep.append(g)
            sup.update(g[1])
    keep.reverse()
    return keep, sup


def tight_cone(edges, gammas, betas, edge):
    """Commutation-aware QAOA cone: per layer (backward) keep RX
    on the current support, then ZZ on edges touching the support as it stood
    at the start of the layer; H on the final support.  Forward gate order."""
    sup = set(edge)
    layers = []
    for k in reversed(range(len(gammas))):
        rx = [("RX", (q,), 2.0 * betas[k]) for q in sorted(sup)]
        ek = [e for e in sorted(edges) if e[0] in sup or e[1] in sup]
        zz = [("ZZ", e, 2.0 * gammas[k]) for e in ek]
        for e in ek:
            sup.update(e)
        layers.append(zz + rx)
    gates = [("H", (q,), None) for q in sorted(sup)]
    for lay in reversed(layers):
        gates += lay
    return gates, sup


def zz_sandwich(gates, edge, qubits):
    """<0| C^dag Z_u Z_v C |0> over the given (already pruned) gates
    (src/tn_build.py:121-142)."""
    u, v = edge
    qs = sorted(set(qubits) | {u, v})
    w = _Wires(qs)
    ts = [((w.cur[q],), _KET0) for q in qs]
    for g in gates:
        _emit(ts, w, g)
    z = np.array([1.0, -1.0], dtype=np.complex128)
    ts.append(((w.cur[u],), z))
    ts.append(((w.cur[v],), z))
    for g in reversed(gates):
        _emit(ts, w, g, adjoint=True)
    for q in qs:
        ts.append(((w.cur[q],), _KET0))
    return ts


def lightcone_tensors(n, edges, gammas, betas, edge, cone="reference"):
    """extract_lightcone (src/tn_build.py:145-151) + the tight mode (App. B)."""
    if cone == "reference":
        gates, sup = reference_cone(qaoa_gates(n, edges, gammas, betas), edge)
    elif cone == "tight":
        gates, sup = tight_cone(edges, gammas, betas, edge)
    else:
        raise ValueError(cone)
    return zz_sandwich(gates, edge, sup)


# ---------------------------------------------------------------------------
# ordering / dry run / slicing          (src/ordering.py)
# ---------------------------------------------------------------------------
def greedy_order(tensors, heuristic="minfill", open_indices=()):
    """Min-fill / min-degree greedy elimination with a (score, id) heap and lazy
    invalidation (src/ordering.py:26-94)."""
    nb = {}
    for idx, _ in tensors:
        for a in idx:
            nb.setdefault(a, set()).update(b for b in idx if b != a)
    opn = set(open_indices)
    live = set(nb) - opn
    fill = heuristic == "minfill"

    def score(v):
        if not fill:
            return len(nb[v])
        ns = list(nb[v])
        return sum(1 for i in range(len(ns)) for j in range(i + 1, len(ns))
                   if ns[j] not in nb[ns[i]])

    cur = {v: score(v) for v in live}
    heap = [(s, v) for v, s in cur.items()]
    heapq.heapify(heap)
    out = []
    while live:
        s, v = heapq.heappop(heap)
        if v not in live or cur[v] != s:
            continue
        out.append(v)
        live.discard(v)
        ns = [x for x in nb[v] if x in live or x in opn]
        for x in nb[v]:
            nb[x].discard(v)
        del nb[v]
        for i in range(len(ns)):
            for j in range(i + 1, len(ns)):
                nb[ns[i]].add(ns[j])
                nb[ns[j]].add(ns[i])
        touched = set(ns)
        if fill:
            for x in ns:
                touched |= nb[x]
        for x in touched:
            if x in live:
                s2 = score(x)
                if s2 != cur[x]:
                    cur[x] = s2
                    heapq.heappush(heap, (s2, x))
    return out


def dry_run(index_sets, order, fixed=()):
    """Symbolic replay of the bucket assignment (src/ordering.py:97-145).
    Returns (widths, active_order)."""
    fixed = set(fixed)
    act = [i for i in order if i not in fixed]
    pos = {x: k for k, x in enumerate(act)}
    bk = {x: [] for x in act}
    for s in index_sets:
        s = frozenset(s) - fixed
        cl = [i for i in s if i in pos]
        if cl:
            bk[min(cl, key=pos.__getitem__)].append(s)
    widths = []
    for x in act:
        u = set().union(*bk[x]) - {x} if bk[x] else set()
        widths.append(len(u))
        cl = [i for i in u if i in pos]
        if cl:
            bk[min(cl, key=pos.__getitem__)].append(frozenset(u))
    return widths, act


def suggest_slicing(index_sets, order, target):
    """Greedy: smallest id of the widest bucket's union (src/ordering.py:192-230)."""
    sl = []
    while True:
        widths, act = dry_run(index_sets, order, sl)
        if max(widths, default=0) <= target:
            return sl
        step = int(np.argmax(widths))
        fixed = set(sl)
        pos = {x: k for k, x in enumerate(act)}
        bk = {x: [] for x in act}
        for s in index_sets:
            s = frozenset(s) - fixed
            cl = [i for i in s if i in pos]
            if cl:
                bk[min(cl, key=pos.__getitem__)].append(s)
        union = None
        for k, x in enumerate(act):
            u = set().union(*bk[x]) if bk[x] else set()
            if k == step:
                union = u
                break
            u.discard(x)
            cl = [i for i in u if i in pos]
            if cl:
                bk[min(cl, key=pos.__getitem__)].append(frozenset(u))
        cand = sorted(i for i in union if i not in fixed) or [act[step]]
        sl.append(cand[0])


# ---------------------------------------------------------------------------
# kernels and elimination               (src/tensor_core.py, src/ordering.py)
# ---------------------------------------------------------------------------
def bucket_fast(bidx, members):
    """Broadcast product over [bucket, sorted result] axes, then sum axis 0
    (src/tensor_core.py:148-164).  members: list of (indices, data)."""
    if not members:
        raise ValueError("empty bucket")
    res = sorted(set().union(*[set(i) for i, _ in members]) - {bidx})
    ax = {bidx: 0}
    ax.update({x: k + 1 for k, x in enumerate(res)})
    nd = len(res) + 1
    buf = np.ones((2,) * nd, dtype=np.complex128)
    for idx, d in members:
        perm = sorted(range(len(idx)), key=lambda a: ax[idx[a]])
        shp = [1] * nd
        for a in idx:
            shp[ax[a]] = 2
        buf *= np.transpose(np.asarray(d, dtype=np.complex128), perm).reshape(shp)
    return tuple(res), buf.sum(axis=0)


def bucket_brute(bidx, members):
    """Enumerate every joint assignment (tests/conftest.py:10-29 style)."""
    res = sorted(set().union(*[set(i) for i, _ in members]) - {bidx})
    out = np.zeros((2,) * len(res), dtype=np.complex128)
    for a in itertools.product((0, 1), repeat=len(res)):
        env = dict(zip(res, a))
        tot = 0j
        for b in (0, 1):
            env[bidx] = b
            pr = 1 + 0j
            for idx, d in members:
                pr *= complex(d[tuple(env[i] for i in idx)])
            tot += pr
        out[a] = tot
    return tuple(res), out


def contract_network(tensors, order, kernel=bucket_fast):
    """Bucket elimination (src/ordering.py:148-189): tensors go to the bucket of
    their earliest index; each result is re-bucketed at its earliest remaining
    index; rank-0 values multiply into the scalar.  Returns (scalar, widths)."""
    pos = {x: k for k, x in enumerate(order)}
    bk = {x: [] for x in order}
    scal = 1 + 0j
    for idx, d in tensors:
        if len(idx) == 0:
            scal *= complex(np.asarray(d).reshape(()))
        else:
            bk[min(idx, key=pos.__getitem__)].append((tuple(idx), np.asarray(d)))
    widths = []
    for x in order:
        mem = bk.pop(x)
        if not mem:
            continue
        ridx, rd = kernel(x, mem)
        widths.append(len(ridx))
        if not ridx:
            scal *= complex(rd.reshape(()))
        else:
            bk[min(ridx, key=pos.__getitem__)].append((ridx, rd))
    return scal, widths


def slice_tensors(tensors, assignment):
    """np.take the fixed indices out (src/ordering.py:233-248)."""
    out = []
    for idx, d in tensors:
        idx = list(idx)
        d = np.asarray(d)
        for x in [i for i in idx if i in assignment]:
            a = idx.index(x)
            d = np.take(d, assignment[x], axis=a)
            idx.pop(a)
        out.append((tuple(idx), d))
    return out


def contract_sliced(tensors, order, sliced):
    """Sum over all assignments in np.ndindex order (src/ordering.py:251-267)."""
    sub = [i for i in order if i not in sliced]
    tot = 0j
    for bits in itertools.product((0, 1), repeat=len(sliced)):
        v, _ = contract_network(slice_tensors(tensors, dict(zip(sliced, bits))), sub)
        tot += v
    return tot


def lightcone_zz(n, edges, gammas, betas, edge, cone="reference", slice_target=None):
    """_contract_zz (src/tn_build.py:154-163): min-fill order, contract, real part."""
    ts = lightcone_tensors(n, edges, gammas, betas, edge, cone)
    order = greedy_order(ts)
    if slice_target is not None:
        sl = suggest_slicing([i for i, _ in ts], order, slice_target)
        if sl:
            return contract_sliced(ts, order, sl).real
    v, _ = contract_network(ts, order)
    return v.real


def qaoa_energy(n, edges, gammas, betas, cone="reference"):
    """sum over sorted edges of (1 - <ZZ>)/2 (src/tn_build.py:189-199)."""
    return sum(0.5 * (1.0 - lightcone_zz(n, edges, gammas, betas, e, cone))
               for e in sorted(edges))


def statevector_energy(n, edges, gammas, betas):
    """Dense statevector MaxCut energy for small n (independent check,
    mirrors the role of src/oracle.py:57-73)."""
    psi = np.zeros(2 ** n, dtype=np.complex128)
    psi[0] = 1
    psi = psi.reshape((2,) * n)
    for kind, qs, ang in qaoa_gates(n, edges, gammas, betas):
        if kind in DIAG_KINDS:
            d = gate_diag(kind, ang).reshape((2,) * len(qs))
            shp = [1] * n
            for q in qs:
                shp[q] = 2
            perm = np.argsort(qs)
            psi = psi * np.transpose(d, perm).reshape(shp)
        else:
            u = gate_matrix(kind, ang)
            psi = np.moveaxis(np.tensordot(u, psi, axes=([1], [qs[0]])), 0, qs[0])
    prob = np.abs(psi) ** 2
    e = 0.0
    for u, v in edges:
        zz = np.fromfunction(lambda *a: (1 - 2 * a[u]) * (1 - 2 * a[v]), (2,) * n)
        e += 0.5 * (1 - float((prob * zz).sum()))
    return e
