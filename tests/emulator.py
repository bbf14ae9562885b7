"""Numpy interpreter of a device Program (test infrastructure).

Executes the planner's tables with the exact semantics the CUDA program
kernel implements (csrc/qtn_b200.cu): buckets in ticket order, member offset
off + b * 2^popc(mask) + pext(r, mask), out = prod_i(b=0) + prod_i(b=1),
finaliser = product of rank-0 values.  Lets the planner be checked on CPU."""
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


def run_program(prog, raw_parts):
    A = np.zeros(prog.arena_elems, np.complex128)
    srcs = [raw[s] for raw, s in zip(raw_parts, prog.img_src_parts)]
    if srcs:
        A[prog.img_dst] = np.concatenate(srcs)
    if prog.dtype == "complex64":
        A = A.astype(np.complex64)
    res = np.zeros(len(prog.instances), np.complex128)
    B = prog.buckets
    order = np.argsort(B["tick_begin"], kind="stable")
    done = set()
    for g in order:
        b = B[g]
        for d in prog.deps[b["dep_begin"]: b["dep_begin"] + b["n_dep"]]:
            assert int(d["bucket"]) in done, "dependency not satisfied in ticket order"
        mem = prog.members[b["mem_begin"]: b["mem_begin"] + b["n_mem"]]
        if b["w"] == N.QTN_FINALIZE:
            v = 1 + 0j
            for m in mem:
                v *= complex(A[int(m["off"])])
            res[int(b["slot"])] = v
        else:
            w = int(b["w"])
            r = np.arange(1 << w, dtype=np.int64)
            p = [None, None]
            for m in mem:
                mask = int(m["mask"])
                pc = bin(mask).count("1")
                idx = int(m["off"]) + pext_vec(r, mask)
                for bb in (0, 1):
                    x = A[idx + (bb << pc)]
                    p[bb] = x.copy() if p[bb] is None else p[bb] * x
            o = int(b["out_off"])
            A[o: o + (1 << w)] = p[0] + p[1]
        done.add(int(g))
    return res
