"""Host logic of exact splitting (§8 N2) against brute force on small multisets.

``exact_boundaries`` must find, for every boundary r, the key of global rank floor(rN/P) (or a
value with exactly floor(rN/P) keys below it and quota 0), and ``exact_send_counts`` must cut
every rank's class-ordered keys so that the concatenated shards are the sorted multiset split
at exactly those ranks.  The histograms fed in are computed here by brute force over explicit
unsigned keys, so no kernel and no oracle arithmetic is involved: the check is sorting itself.
"""
import numpy as np
import pytest

from _exact_ref import exact_boundaries, exact_send_counts


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


# ---- the C++ planning in libbsort (bsort_dist_exact_boundaries / _send_counts), used by the
# native bsort_sort_dist_ex(BSORT_DIST_EXACT): same answers as above, on the same brute force

def _native(ranks_keys, width):
    import ctypes
    import paper_2603_08929_b200 as B
    from paper_2603_08929_b200 import _lib
    P = len(ranks_keys)
    allk = [k for ks in ranks_keys for k in ks]
    hg = np.ascontiguousarray(_hist(allk, width, 16))
    calls = []

    @_lib.REFINE_FN
    def refine(ctx, prefixes, m, bits, out):
        pre = [int(prefixes[j]) for j in range(m)]
        calls.append((bits, pre))
        h = np.stack([_hist(allk, width, bits + 16, p, bits) for p in pre]).reshape(-1)
        ctypes.memmove(out, h.ctypes.data, h.nbytes)
        return 0

    R = max(P - 1, 1)
    values = (ctypes.c_uint64 * R)()
    idx = (ctypes.c_int * R)()
    quota = (ctypes.c_uint64 * R)()
    m = ctypes.c_int(0)
    levels = ctypes.c_int(0)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    st = B.lib.bsort_dist_exact_boundaries(hg.ctypes.data_as(u64p), P, width, refine, None, values,
                                           ctypes.byref(m), idx, quota, ctypes.byref(levels))
    assert st == 0
    return (np.array(values[:m.value], dtype=np.uint64), np.array(idx[:P - 1], dtype=np.int64),
            np.array(quota[:P - 1], dtype=np.int64), levels.value)


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_native_planning_matches(width, P):
    import ctypes
    import paper_2603_08929_b200 as B
    rng = np.random.default_rng(width + 7 * P)
    for kind in range(4):
        ranks = []
        for r in range(P):
            n = int(rng.integers(1, 50))
            if kind == 0:
                ks = [int(x) for x in rng.integers(0, 1 << 62, n)] if width == 64 else \
                    [int(x) for x in rng.integers(0, 1 << 32, n)]
            elif kind == 1:
                ks = [int(x) << (width - 20) for x in rng.integers(0, 3, n)]
            elif kind == 2:
                ks = [(0xABCD << (width - 16)) | int(x) for x in rng.integers(0, 50, n)]
            else:
                ks = [12345] * n
            ranks.append(ks)
        allk = [k for ks in ranks for k in ks]
        hg = _hist(allk, width, 16)

        def refine(prefixes, bits):
            return np.stack([_hist(allk, width, bits + 16, int(p), bits) for p in prefixes])

        v_py, i_py, q_py, l_py = exact_boundaries(hg, P, width, refine)
        v_c, i_c, q_c, l_c = _native(ranks, width)
        assert np.array_equal(v_py, v_c) and np.array_equal(i_py, i_c) and np.array_equal(q_py, q_c)
        assert l_py == l_c
        vals = [int(v) for v in v_c]
        C = np.stack([np.array([sum(1 for k in ks if k == vals[c // 2]) if c % 2 else
                                sum(1 for k in ks if (c == 0 or k > vals[c // 2 - 1]) and
                                    (c // 2 == len(vals) or k < vals[c // 2]))
                                for c in range(2 * len(vals) + 1)]) for ks in ranks]).astype(np.uint64)
        Cc = np.ascontiguousarray(C)
        idx_c = (ctypes.c_int * (P - 1))(*[int(x) for x in i_c])
        quo_c = (ctypes.c_uint64 * (P - 1))(*[int(x) for x in q_c])
        u64p = ctypes.POINTER(ctypes.c_uint64)
        for me in range(P):
            out = (ctypes.c_uint64 * P)()
            st = B.lib.bsort_dist_exact_send_counts(Cc.ctypes.data_as(u64p), P, len(vals), me, idx_c, quo_c, out)
            assert st == 0
            assert list(out) == [int(x) for x in exact_send_counts(C, me, i_py, q_py)]


def test_native_planning_rejects_bad_args():
    import ctypes
    import paper_2603_08929_b200 as B
    from paper_2603_08929_b200 import _lib
    hg = np.zeros(65536, dtype=np.uint64)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    v = (ctypes.c_uint64 * 4)()
    i = (ctypes.c_int * 4)()
    q = (ctypes.c_uint64 * 4)()
    m = ctypes.c_int(0)
    cb = _lib.REFINE_FN(lambda *a: 0)
    # no keys at all with 2 ranks: there is no key of rank T_1
    assert B.lib.bsort_dist_exact_boundaries(hg.ctypes.data_as(u64p), 2, 32, cb, None, v, ctypes.byref(m), i, q,
                                             None) == 1
    hg[5] = 10
    assert B.lib.bsort_dist_exact_boundaries(hg.ctypes.data_as(u64p), 2, 16, cb, None, v, ctypes.byref(m), i, q,
                                             None) == 1  # key_bits must be 32 or 64
    assert B.lib.bsort_dist_exact_boundaries(hg.ctypes.data_as(u64p), 2, 32, _lib.REFINE_FN(), None, v,
                                             ctypes.byref(m), i, q, None) == 1  # NULL callback
