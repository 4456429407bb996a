"""Test-side restatement of §8 N2's host planning (exact splitting), kept as an independent
numpy cross-check of libbsort's C++ planning (bsort_dist_exact_boundaries / _send_counts, which
the product path calls).  Not imported by the package."""
from __future__ import annotations

from typing import Callable

import numpy as np


def exact_boundaries(hg: np.ndarray, nranks: int, width: int, refine: Callable):
    """§8 N2 (host part): the transformed key K_r of global rank T_r = floor(r N / P) for every
    boundary r = 1..P-1, and quota_r = T_r - #{keys < K_r} (how many keys equal to K_r precede
    the boundary).  ``hg`` is the global top-16-bit histogram; ``refine(prefixes, bits)`` returns
    the GLOBAL uint64[m, 65536] histogram of the next 16 bits below each ``bits``-bit prefix.

    Each boundary descends the radix tree 16 bits at a time (the MSD digit order of P:427-433)
    until its rank falls on a bin start (quota 0: K_r = the prefix followed by zeros, which need
    not be a key) or the prefix is the whole key.  Returns (values: strictly increasing distinct
    K's as np.uint64, idx: index of K_r in values, quota: np.int64, levels)."""
    N = int(hg.astype(np.int64).sum())
    R = nranks - 1
    T = [(r * N) // nranks for r in range(1, nranks)]
    pv, below, bits = [0] * R, [0] * R, [16] * R
    cum = np.cumsum(hg.astype(np.int64))
    for i in range(R):
        b = int(np.searchsorted(cum, T[i], side="right"))  # bin holding the key of rank T_i
        pv[i] = b
        below[i] = int(cum[b - 1]) if b > 0 else 0
    levels, level_bits = 0, 16
    open_ = [i for i in range(R) if T[i] > below[i]]
    while open_ and level_bits < width:
        prefixes = sorted({pv[i] for i in open_})
        H = np.asarray(refine(np.array(prefixes, dtype=np.uint64), level_bits)).astype(np.int64)
        levels += 1
        row = {p: j for j, p in enumerate(prefixes)}
        for i in open_:
            c = np.cumsum(H[row[pv[i]]])
            sb = int(np.searchsorted(c, T[i] - below[i], side="right"))
            below[i] += int(c[sb - 1]) if sb > 0 else 0
            pv[i] = (pv[i] << 16) | sb
            bits[i] += 16
        level_bits += 16
        open_ = [i for i in open_ if T[i] > below[i]]
    K = [pv[i] << (width - bits[i]) for i in range(R)]
    values = sorted(set(K))
    vi = {v: j for j, v in enumerate(values)}
    idx = np.array([vi[k] for k in K], dtype=np.int64)
    quota = np.array([T[i] - below[i] for i in range(R)], dtype=np.int64)
    return np.array(values, dtype=np.uint64), idx, quota, levels


def exact_send_counts(class_counts_all: np.ndarray, me: int, idx: np.ndarray,
                      quota: np.ndarray) -> np.ndarray:
    """Per-destination send counts of rank ``me`` over its class-ordered keys (§8 N2).

    ``class_counts_all[q]`` = rank q's 2m+1 class counts.  Boundary r cuts my buffer after all
    classes below K_r (classes 0..2j) plus my share of the keys equal to K_r: the equal keys are
    assigned to the left in rank order, quota_r of them in total, so my share is
    clip(quota_r - (equal keys on ranks < me), 0, my equal keys).  Summed over ranks every
    boundary lands exactly on global rank T_r."""
    c = class_counts_all.astype(np.int64)
    mine = c[me]
    start = np.concatenate([[0], np.cumsum(mine)])
    eq_before = c[:me, 1::2].sum(axis=0) if me > 0 else np.zeros(c.shape[1] // 2, dtype=np.int64)
    splits = [0]
    for r in range(len(idx)):
        j = int(idx[r])
        share = min(max(int(quota[r]) - int(eq_before[j]), 0), int(mine[2 * j + 1]))
        splits.append(int(start[2 * j + 1]) + share)
    splits.append(int(mine.sum()))
    return np.diff(np.array(splits, dtype=np.int64)).astype(np.uint64)
