"""Numpy interpreter of a device Program (test infrastructure).

Executes the planner's tables with the exact semantics the CUDA program
kernel implements (csrc/qtn_b200.cu): buckets in ticket order, member offset
off + (pext(s, smask) << popc(mask)) + pext(r, mask), out = sum_s prod_i,
finaliser = product of rank-0 values.  Lets the planner be checked on CPU.

Precision model of complex64 programs (qtn_program_t.inputs_hi): K2 stage
items (small nodes) and finalisers compute in double, reading input members
of rank <= 6 unrounded; large items compute in complex64 from the narrowed
arena; every stored intermediate is complex64."""
import numpy as np

from paper_2210_15874_b200 import _native as N


def pext_vec(r, mask):
    out = np.zeros_like(r)
    k = 0
    for j in range(64):
        if (mask >> j) & 1:
            out |= ((r >> j) & 1) << k
            k += 1
    return out


def pair_overlaps(prog, nd):
    """A K6 pair node reads both items' members while it writes the
    consumer's result: True when that result overlaps any of them."""
    B = prog.buckets
    bc = B[int(nd["first"]) + 1]
    lo, hi = int(bc["out_off"]), int(bc["out_off"]) + (1 << int(bc["w"]))
    for g in (int(nd["first"]), int(nd["first"]) + 1):
        for m in prog.members[B[g]["mem_begin"]: B[g]["mem_begin"] + B[g]["n_mem"]]:
            n = 1 << (bin(int(m["mask"])).count("1") + bin(int(m["smask"])).count("1"))
            if not (int(m["off"]) + n <= lo or int(m["off"]) >= hi):
                return True
    return False


def run_program(prog, raw_parts):
    A = np.zeros(prog.arena_elems, np.complex128)
    srcs = [raw[s] for raw, s in zip(raw_parts, prog.img_src_parts)]
    if srcs:
        A[prog.img_dst] = np.concatenate(srcs)
    n_hi = prog.n_input_elems if prog.dtype == "complex64" else 0
    hi = A[:n_hi].copy()
    if prog.dtype == "complex64":
        A = A.astype(np.complex64)
    res = np.zeros(len(prog.instances), np.complex128)
    B = prog.buckets
    done = set()
    node_done = set()
    for ni, nd in enumerate(prog.nodes):
        for d in prog.node_deps[nd["dep_begin"]: nd["dep_begin"] + nd["n_dep"]]:
            assert int(d) in node_done and int(d) < ni, "graph dependency not earlier"
        items = range(int(nd["first"]), int(nd["first"]) + int(nd["count"]))
        small = nd["kind"] == N.QTN_NODE_SMALL
        if not small and int(nd["count"]) == 2:
            assert not pair_overlaps(prog, nd), "pair result overlaps a member"
        if small:
            items = sorted(items, key=lambda g: int(B[g]["tick_begin"]))
        for g in items:
            b = B[g]
            for d in prog.deps[b["dep_begin"]: b["dep_begin"] + b["n_dep"]]:
                assert int(d["bucket"]) in done, "dependency not satisfied in ticket order"
            mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
            if b["w"] == N.QTN_FINALIZE:
                v = 1 + 0j
                for m in mem:
                    o = int(m["off"])
                    v *= complex(hi[o] if o < n_hi else A[o])
                res[int(b["slot"])] = v
            else:
                w, k = int(b["w"]), int(b["k"])
                r = np.arange(1 << w, dtype=np.int64)
                acc = None
                for s in range(1 << k):
                    p = None
                    for m in mem:
                        mask, smask = int(m["mask"]), int(m["smask"])
                        pc = bin(mask).count("1")
                        o = int(m["off"]) + (int(pext_vec(np.array([s]), smask)[0]) << pc) + pext_vec(r, mask)
                        if small and n_hi:
                            staged = int(m["off"]) < n_hi and pc + bin(smask).count("1") <= 6
                            x = hi[o] if staged else A[o].astype(np.complex128)
                        else:
                            x = A[o]
                        p = x.copy() if p is None else p * x
                    acc = p if acc is None else acc + p
                o = int(b["out_off"])
                A[o: o + (1 << w)] = acc.astype(A.dtype)
            done.add(int(g))
        node_done.add(ni)
    return res
