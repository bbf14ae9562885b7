"""K6 plans of every producer/consumer pair of a workload's programs (host
only): python scripts/k6_survey.py [lightcone|graph|cfg4] [c64|c128]"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2210_15874_b200 import _native as N  # noqa: E402
from paper_2210_15874_b200 import engine as E  # noqa: E402


def item_desc(prog, gid, base=1 << 20):
    """Host descriptor of item gid in canonical layout (fake arena base)."""
    esz = E.ELEM_BYTES[prog.dtype]
    b = prog.buckets[gid]
    w, k = int(b["w"]), int(b["k"])
    mems = []
    for m in prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]:
        mask, smask = int(m["mask"]), int(m["smask"])
        st, r = {}, 0
        for bit in range(w):
            if (mask >> bit) & 1:
                st[bit] = 1 << r
                r += 1
        q = 0
        for j in range(k):
            if (smask >> j) & 1:
                st[w + j] = 1 << (r + q)
                q += 1
        mems.append((base + int(m["off"]) * esz, st))
    code = N.QTN_C64 if prog.dtype == "complex64" else N.QTN_C128
    return N.bucket_desc(code, w, base + int(b["out_off"]) * esz, mems, k=k), [int(mm["off"]) for mm in
                                                                                 prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]]


def pair_plans(prog):
    out = []
    for nd in prog.nodes:
        if nd["kind"] != 1 or nd["count"] != 2:
            continue
        p_, c_ = int(nd["first"]), int(nd["first"]) + 1
        dp, _ = item_desc(prog, p_)
        dc, offs = item_desc(prog, c_)
        ipc = offs.index(int(prog.buckets[p_]["out_off"]))
        try:
            info = N.bucket_expand_fused_plan(dp, dc, ipc)
        except N.NativeError as e:
            info = str(e)
        out.append((int(prog.buckets[p_]["w"]), int(prog.buckets[c_]["w"]), info))
    return out


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "lightcone"
    dtype = "complex128" if "c128" in sys.argv[2:] else "complex64"
    if which == "graph":
        import paper_2210_15874_b200 as Q
        from paper_2210_15874_b200 import distributed as D
        g = Q.random_regular_graph(30, 3, seed=0)
        c = Q.qaoa_maxcut_circuit(g, Q.QaoaParams.seeded(4, 0))
        cones = [Q.extract_lightcone(c, e, cone="tight") for e in g.edges]
        be = Q.Backend.b200(dtype=dtype)
        plan = D.plan_units(cones, be, mem_cap=bench.GRAPH_MEM_CAP, balance_ranks=bench.GRAPH_BALANCE)
        batches = list(D._batches(range(len(plan.units)), plan, be, 40 << 30))
        progs = [E.Program([E.Instance(plan.templates[plan.units[u].cone], plan.units[u].assignment) for u in b],
                           dtype) for b in batches]
    else:
        g, params, lc, order = bench.build_workload()
        t = E.plan_template([x.indices for x in lc.network.tensors], order, dtype, wave_aware=True)
        progs = [E.Program([E.Instance(t)], dtype)]
    cnt = collections.Counter()
    for prog in progs:
        for wp, wc, info in pair_plans(prog):
            key = info if isinstance(info, str) else "k=%d nq=%d ne=%d nf=%d ng=%d nu=%d nqn=%d" % info[:7]
            cnt[(wp, wc, key)] += 1
    for (wp, wc, key), n in sorted(cnt.items()):
        print(f"{n:4d} x  P w{wp} -> C w{wc}: {key}")
