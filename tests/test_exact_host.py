"""Host logic of exact splitting (§8 N2) against brute force on small multisets.

``exact_boundaries`` must find, for every boundary r, the key of global rank floor(rN/P) (or a
value with exactly floor(rN/P) keys below it and quota 0), and ``exact_send_counts`` must cut
every rank's class-ordered keys so that the concatenated shards are the sorted multiset split
at exactly those ranks.  The histograms fed in are computed here by brute force over explicit
unsigned keys, so no kernel and no oracle arithmetic is involved: the check is sorting itself.
"""
import numpy as np
import pytest

from paper_2603_08929_b200.dist import exact_boundaries, exact_send_counts


def _hist(keys, width, bits, prefix=None, pbits=0):
    ks = [k for k in keys if prefix is None or (k >> (width - pbits)) == prefix]
    h = np.zeros(65536, dtype=np.uint64)
    for k in ks:
        h[(k >> (width - bits)) & 0xFFFF] += 1
    return h


def _run(ranks_keys, width):
    P = len(ranks_keys)
    allk = [k for ks in ranks_keys for k in ks]
    hg = _hist(allk, width, 16)
    calls = []

    def refine(prefixes, bits):
        calls.append(bits)
        return np.stack([_hist(allk, width, bits + 16, int(p), bits) for p in prefixes])

    values, idx, quota, levels = exact_boundaries(hg, P, width, refine)
    vals = [int(v) for v in values]
    assert vals == sorted(set(vals))
    N = len(allk)
    srt = sorted(allk)
    for r in range(1, P):
        T = r * N // P
        K = vals[idx[r - 1]]
        below = sum(1 for k in allk if k < K)
        assert below + quota[r - 1] == T
        assert quota[r - 1] == 0 or srt[T] == K  # a positive quota only on a real key
    C = np.stack([np.array([sum(1 for k in ks if k == vals[c // 2]) if c % 2 else
                            sum(1 for k in ks if (c == 0 or k > vals[c // 2 - 1]) and
                                (c // 2 == len(vals) or k < vals[c // 2]))
                            for c in range(2 * len(vals) + 1)]) for ks in ranks_keys])
    assert (C.sum(axis=1) == [len(ks) for ks in ranks_keys]).all()
    shards = [[] for _ in range(P)]
    for me, ks in enumerate(ranks_keys):
        sc = exact_send_counts(C, me, idx, quota).astype(np.int64)
        assert sc.sum() == len(ks)
        ordered = sorted(ks, key=lambda k: (2 * sum(v < k for v in vals) + (k in vals)))
        pos = 0
        for d in range(P):
            shards[d] += ordered[pos:pos + sc[d]]
            pos += sc[d]
    assert [len(s) for s in shards] == [(d + 1) * N // P - d * N // P for d in range(P)]
    assert [k for s in shards for k in sorted(s)] == srt
    return levels


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_random_mixes(width, P):
    rng = np.random.default_rng(width * 10 + P)
    for trial in range(4):
        kinds = trial % 4
        out = []
        for r in range(P):
            n = int(rng.integers(0, 60))
            if kinds == 0:    # uniform
                ks = [int(x) for x in rng.integers(0, 1 << 62, n)] if width == 64 else \
                    [int(x) for x in rng.integers(0, 1 << 32, n)]
            elif kinds == 1:  # few distinct values
                ks = [int(x) << (width - 20) for x in rng.integers(0, 3, n)]
            elif kinds == 2:  # share the top 48 bits (64-bit) / 16 bits (32-bit)
                base = 0xABCD << (width - 16)
                ks = [base | int(x) for x in rng.integers(0, 50, n)]
            else:             # all equal
                ks = [12345] * n
            out.append(ks)
        if sum(len(k) for k in out) == 0:
            out[0] = [1]
        _run(out, width)


def test_deep_refinement_64():
    """Keys equal in their top 48 bits: boundaries need all three refinement levels."""
    base = 0x0123456789AB << 16
    ranks = [[base | 5, base | 9, base | 1], [base | 2, base | 7, base | 3, base | 4]]
    assert _run(ranks, 64) == 3


def test_bin_start_resolves_without_refinement():
    """A boundary rank that falls on a bin start needs no refinement (quota 0)."""
    ranks = [[0 << 16] * 3, [1 << 16] * 3]
    assert _run(ranks, 32) == 0
