"""Seeded synthetic inputs of the BASELINE configs (no dataset is involved).

cfg 5 — the synthetic bucket microbench (BASELINE.json configs[4], SURVEY
§8(d)): bucket index 0, result indices 1..w, members over binary indices in
random axis permutations, entries i.i.d. standard complex normal
(std_normal + 1j*std_normal)/sqrt(2), from np.random.default_rng(seed).

  class "A": member 0 carries all w+1 indices in a random permutation;
             members 1..k-1 carry the bucket index + 1-4 random result
             indices, permuted (a reduce bucket: read 2^(w+1), write 2^w).
  class "B": two members, each the bucket index + a random ~60% of the
             result indices, together covering all of them (an expansion
             bucket: the result is wider than either member).

The same index structure drives the oracle (complex128 numpy data, small w)
and the device microbench (`device=True`: data generated on the GPU from a
seeded torch generator, so w up to 30 never touches host memory).
"""
from __future__ import annotations

import numpy as np

BUCKET = 0


def bucket_structure(w: int, k: int, cls: str, seed: int):
    """Index tuples of the members of one cfg-5 bucket (deterministic in seed)."""
    rng = np.random.default_rng(seed)
    res = list(range(1, w + 1))
    if cls == "A":
        if k < 1:
            raise ValueError("class A needs k >= 1")
        mem = [tuple(int(x) for x in rng.permutation([BUCKET] + res))]
        for _ in range(k - 1):
            n = int(rng.integers(1, 5)) if w else 0
            ids = [int(x) for x in rng.choice(res, size=min(n, w), replace=False)] if w else []
            mem.append(tuple(int(x) for x in rng.permutation([BUCKET] + ids)))
        return mem
    if cls == "B":
        if w == 0:
            return [(BUCKET,), (BUCKET,)]
        pick = rng.random((2, w)) < 0.6
        for j in range(w):           # every result index in at least one member
            if not pick[:, j].any():
                pick[int(rng.integers(0, 2)), j] = True
        mem = []
        for m in range(2):
            ids = [res[j] for j in range(w) if pick[m, j]]
            mem.append(tuple(int(x) for x in rng.permutation([BUCKET] + ids)))
        return mem
    raise ValueError(f"unknown bucket class {cls!r}")


def synthetic_bucket(w: int, k: int = 3, cls: str = "A", seed: int = 0):
    """[(indices, complex128 data of shape (2,)*rank)] of a cfg-5 bucket."""
    mem = bucket_structure(w, k, cls, seed)
    rng = np.random.default_rng(seed + 1)
    out = []
    for idx in mem:
        shp = (2,) * len(idx)
        d = (rng.standard_normal(shp) + 1j * rng.standard_normal(shp)) / np.sqrt(2.0)
        out.append((idx, d))
    return out


def synthetic_bucket_device(w: int, k: int = 3, cls: str = "A", seed: int = 0, dtype="complex64",
                            device=0):
    """Same structure with the data generated on the GPU: [(indices, flat torch tensor)]."""
    import torch
    mem = bucket_structure(w, k, cls, seed)
    gen = torch.Generator(device=f"cuda:{device}")
    gen.manual_seed(seed + 1)
    rdt = torch.float32 if dtype in ("complex64", "c64") else torch.float64
    cdt = torch.complex64 if rdt == torch.float32 else torch.complex128
    out = []
    for idx in mem:
        n = 1 << len(idx)
        x = torch.randn(2 * n, generator=gen, device=f"cuda:{device}", dtype=rdt)
        x.mul_(1.0 / np.sqrt(2.0))
        out.append((idx, torch.view_as_complex(x.view(n, 2)).view(cdt)))
    return out


def bucket_bytes(members, w: int, elem_bytes: int) -> int:
    """Algorithmic bytes of one bucket: every member read once
    and the result written once."""
    return (sum(1 << len(idx) for idx, _ in members) + (1 << w)) * elem_bytes
