"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test pins the oracle to something other than itself: the paper's worked examples
(tests/golden/, cited), textbook orders computed by numpy / exact rationals, exhaustive
brute force against the plain definition, and the complexity bounds of Theorems 4-5.
None of these tests touches the GPU.
"""
import itertools
import random
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import parse_golden


def _scheme(vals):
    kind = vals[0]
    if kind == "U":
        return oracle.U(int(vals[1]))
    if kind == "I":
        return oracle.I(int(vals[1]))
    return oracle.F(int(vals[1]), int(vals[2]), int(vals[3]))


def _words(vals, scheme):
    mask = (1 << scheme.width) - 1
    return [int(v, 0) & mask for v in vals]


@pytest.mark.parametrize("fixture", ["fig1_unsigned.txt", "fig2_signed.txt", "fig4_float.txt"])
def test_paper_figures(fixture):
    """Figs. 1, 2, 4: final rows and the first partition index k."""
    g = parse_golden(fixture)
    s = _scheme(g["scheme"])
    asc = bool(int(g["asc"][0]))
    inp = _words(g["input"], s)
    exp = _words(g["output"], s)
    assert list(oracle.bsort(inp, s, asc)) == exp
    assert list(oracle.sort_by_key(inp, s, asc)) == exp
    # The first pass (Algorithm 1) on the MSB: plain for unsigned, with not-asc for
    # the signed / float sign pass.
    first_asc = asc if s.kind == oracle.UNSIGNED else (not asc)
    k, after = oracle.single_pass(inp, int(g["first_pass_mask"][0]), 0, len(inp), first_asc)
    assert k == int(g["first_pass_k"][0])
    assert sorted(after) == sorted(inp)  # multiset preserved


def test_fig4_literal_algorithm4_is_wrong():
    """Reading Q1: Algorithm 4 as printed (asc to both halves) misorders Fig. 4."""
    g = parse_golden("fig4_float.txt")
    s = _scheme(g["scheme"])
    inp = _words(g["input"], s)
    exp = _words(g["output"], s)
    lit = list(oracle.bsort_float_literal(inp, s, True))
    assert lit != exp
    assert lit == [0b110001, 0b111100, 0b001101, 0b001111]  # -2.5 before -inf


def test_mixed_sign_failure_proof():
    """Section III proof: naive binary quicksort puts -1 after 0; bsortSigned not."""
    g = parse_golden("mixed_sign.txt")
    s = _scheme(g["scheme"])
    inp = _words(g["input"], s)
    assert list(oracle.bsort(inp, s, True)) == _words(g["output"], s)
    naive = list(oracle.bsort(inp, oracle.U(s.width), True))  # Algorithm 2 on raw bits
    assert naive == _words(g["naive_unsigned_output"], s)
    for w in (2, 4, 16, 32, 64):
        m = (1 << w) - 1
        assert list(oracle.bsort([(-1) & m, 0], oracle.I(w), True)) == [(-1) & m, 0]


# --------------------------------------------------------------------------- library orders

INT_DTYPES = [np.uint8, np.int8, np.uint16, np.int16, np.uint32, np.int32, np.uint64, np.int64]


@pytest.mark.parametrize("dtype", INT_DTYPES)
@pytest.mark.parametrize("n", [0, 1, 2, 7, 1000, 4099])
def test_integers_match_numpy_sort(dtype, n):
    """Integers: bsort order is numeric order (the problem statement) == np.sort."""
    rng = np.random.default_rng(n * 31 + np.dtype(dtype).itemsize)
    info = np.iinfo(dtype)
    a = rng.integers(info.min, info.max, size=n, dtype=dtype, endpoint=True)
    if n > 100:
        a[:50] = a[50]  # duplicates
    np.testing.assert_array_equal(oracle.sort_native(a), np.sort(a))
    np.testing.assert_array_equal(oracle.sort_native(a, descending=True), np.sort(a)[::-1])


def _float_bits_equal_numeric(out, ref):
    """out (bsort) vs ref (np.sort): equal values; among equal zeros -0 precedes +0."""
    assert np.array_equal(out, ref)  # numeric equality (-0 == +0)
    z = np.flatnonzero(out == 0)
    sb = np.signbit(out[z])
    # all -0 (signbit True) come before all +0 inside the zero run ("-0 < +0")
    assert not np.any(sb[1:] & ~sb[:-1])


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_floats_match_numpy_sort(dtype):
    rng = np.random.default_rng(7)
    a = np.concatenate([
        rng.standard_normal(3000), rng.uniform(-1e6, 1e6, 3000),
        np.array([0.0, -0.0, np.inf, -np.inf, 5e-324, -5e-324, 1e-40, -1e-40] * 5),
    ]).astype(dtype)
    rng.shuffle(a)
    out = oracle.sort_native(a)
    _float_bits_equal_numeric(out, np.sort(a))
    outd = oracle.sort_native(a, descending=True)
    assert np.array_equal(outd, out[::-1])
    # descending is exactly the bit-reverse of ascending (Q9)
    assert outd.tobytes() == out[::-1].tobytes()


def _toy_value(word, e, t):
    """Exact value of a Float(1+e+t) word with IEEE-754 conventions (bias 2^(e-1)-1, implicit
    leading 1 for normals, subnormals at exponent 0, all-ones exponent = inf/NaN)."""
    sign = (word >> (e + t)) & 1
    ex = (word >> t) & ((1 << e) - 1)
    man = word & ((1 << t) - 1)
    bias = (1 << (e - 1)) - 1
    if ex == (1 << e) - 1:
        return ("nan", sign, man) if man else ("inf", sign, None)
    if ex == 0:
        v = Fraction(man, 1 << t) * Fraction(2) ** (1 - bias)
    else:
        v = (1 + Fraction(man, 1 << t)) * Fraction(2) ** (ex - bias)
    return ("num", sign, -v if sign else v)


def _toy_rank(word, e, t):
    """Ascending rank key from the paper's statements on special values:
    -NaN first (larger payload first), -inf, finite numeric order with -0 before +0, +inf,
    +NaN last (larger payload last).  Written from values, not bits."""
    kind, sign, v = _toy_value(word, e, t)
    if kind == "nan":
        return (0, -v) if sign else (4, v)
    if kind == "inf":
        return (1, 0) if sign else (3, 0)
    return (2, v, 0 if sign else 1)


@pytest.mark.parametrize("e,t", [(3, 2), (4, 3), (2, 1), (5, 2)])
def test_toy_float_exhaustive_numeric_order(e, t):
    """Exhaustive: every pattern of Float(1+e+t), shuffled, sorts into exact numeric order."""
    w = 1 + e + t
    words = list(range(1 << w))
    random.Random(w).shuffle(words)
    s = oracle.F(w, e, t)
    exp = sorted(words, key=lambda x: _toy_rank(x, e, t))
    assert list(oracle.bsort(words, s, True)) == exp
    assert list(oracle.bsort(words, s, False)) == exp[::-1]


def _f32(x):
    return struct.unpack("<I", struct.pack("<f", x))[0]


def _f32_nan(sign, payload):
    return (sign << 31) | (0xFF << 23) | payload


def test_special_values_f32():
    """+inf after all non-NaN, -inf before, NaN at the extremities ordered by
    payload, -0 < +0; subnormals in numeric order (Q11)."""
    vals = [1.0, -1.0, 0.0, -0.0, float("inf"), float("-inf"), 1e-45, -1e-45, 3.5, -2.5]
    words = [_f32(v) for v in vals] + [_f32_nan(0, 1), _f32_nan(0, 0x400000), _f32_nan(1, 1),
                                       _f32_nan(1, 0x7FFFFF)]
    s = oracle.F(32, 8, 23)
    out = list(oracle.bsort(words, s, True))
    exp = [_f32_nan(1, 0x7FFFFF), _f32_nan(1, 1), _f32(float("-inf")), _f32(-2.5), _f32(-1.0),
           _f32(-1e-45), _f32(-0.0), _f32(0.0), _f32(1e-45), _f32(1.0), _f32(3.5),
           _f32(float("inf")), _f32_nan(0, 1), _f32_nan(0, 0x400000)]
    assert out == exp
    assert list(oracle.bsort(words, s, False)) == exp[::-1]


def test_theorem2_counterexamples_sort_correctly():
    """Theorem 2: [-2.0, 0.0, 0.5] and [0.75, 2.0] under the sign->exponent->
    mantissa hierarchy come out numerically ascending (the wrong hierarchies would give
    [0.0, 0.5, -2.0] / [0.5, 0.0, -2.0] / [2.0, 0.75])."""
    for arr in ([-2.0, 0.0, 0.5], [0.5, 0.0, -2.0], [0.75, 2.0], [2.0, 0.75]):
        for dt in (np.float32, np.float64):
            a = np.array(arr, dtype=dt)
            assert list(oracle.sort_native(a)) == sorted(arr)


# ------------------------------------------------------------------------------- brute force

@pytest.mark.parametrize("scheme,max_len", [
    (oracle.U(3), 6), (oracle.I(3), 6), (oracle.F(3, 1, 1), 6),
    (oracle.U(4), 5), (oracle.I(4), 5), (oracle.F(4, 2, 1), 5),
])
def test_bruteforce_r1_equals_r2(scheme, max_len):
    """Every array of length <= max_len over all 2^w patterns, both directions: R1 == R2."""
    bad, cases = oracle.bruteforce(scheme, max_len)
    base = 1 << scheme.width
    assert cases == 2 * sum(base ** k for k in range(max_len + 1))
    assert bad == 0


def test_r2_key_is_pinned_by_brute_force_on_values():
    """R2's key order equals the value order for tiny schemes (brute force over all words)."""
    for w in (3, 4, 5):
        words = list(range(1 << w))
        # signed: value order of two's complement
        sval = lambda x: x - (1 << w) if x >> (w - 1) else x  # noqa: E731
        assert list(oracle.sort_by_key(words, oracle.I(w), True)) == sorted(words, key=sval)
        assert list(oracle.sort_by_key(words, oracle.U(w), True)) == sorted(words)
    e, t = 2, 2
    words = list(range(1 << 5))
    assert list(oracle.sort_by_key(words, oracle.F(5, e, t), True)) == \
        sorted(words, key=lambda x: _toy_rank(x, e, t))


# ---------------------------------------------------------------------------- invariants

@pytest.mark.parametrize("scheme", [oracle.U(8), oracle.I(16), oracle.F(32, 8, 23),
                                    oracle.U(64), oracle.F(64, 11, 52), oracle.I(7)])
def test_theorem4_theorem5_counters(scheme):
    """Theorem 4: each level inspects <= n elements, total <= w*n.
    Theorem 5: recursion depth <= w."""
    rng = np.random.default_rng(scheme.width)
    n = 5000
    m = (1 << scheme.width) - 1
    words = rng.integers(0, 2**63, size=n, dtype=np.uint64) & np.uint64(m)
    words[:500] = words[0]
    for asc in (True, False):
        out, st = oracle.bsort(words, scheme, asc, with_stats=True)
        assert st["max_depth"] <= scheme.width
        assert all(c <= n for c in st["inspections_per_level"])
        assert st["inspections"] <= scheme.width * n
        assert np.array_equal(out, oracle.sort_by_key(words, scheme, asc))


def test_single_pass_partition_invariant():
    """Algorithm 1's output contract: asc puts mask-clear words in [ps,k), set in [k,pe)."""
    rng = random.Random(3)
    for _ in range(200):
        n = rng.randint(0, 40)
        a = [rng.randrange(256) for _ in range(n)]
        ps = rng.randint(0, n)
        pe = rng.randint(ps, n)
        m = 1 << rng.randrange(8)
        for asc in (True, False):
            k, b = oracle.single_pass(a, m, ps, pe, asc)
            b = list(b)
            assert ps <= k <= pe
            assert b[:ps] == a[:ps] and b[pe:] == a[pe:]
            assert sorted(b[ps:pe]) == sorted(a[ps:pe])
            want_clear_first = asc
            for i in range(ps, pe):
                in_first = i < k
                bit_clear = (b[i] & m) == 0
                assert in_first == (bit_clear == want_clear_first)


def test_descending_is_reverse_and_idempotent():
    rng = np.random.default_rng(11)
    for dt in (np.int32, np.float32, np.uint64, np.float64, np.int8):
        a = rng.integers(0, 2**63, size=3001, dtype=np.uint64).astype(
            {1: np.uint8, 4: np.uint32, 8: np.uint64}[np.dtype(dt).itemsize]).view(dt)
        up = oracle.sort_native(a)
        assert oracle.sort_native(up).tobytes() == up.tobytes()
        assert oracle.sort_native(a, True).tobytes() == up[::-1].tobytes()


def test_oracle_rejects_bad_input():
    with pytest.raises(ValueError):
        oracle.bsort([8], oracle.U(3))  # word wider than the scheme
    with pytest.raises(ValueError):
        oracle.bsort([1], oracle.F(6, 3, 3))  # w != e + t + 1


def test_all_permutations_small():
    """Every permutation of a small multiset sorts to the same output (order-independence)."""
    base = [3, 0, 7, 3, 5, 1]
    exp = sorted(base)
    for perm in itertools.permutations(base):
        assert list(oracle.bsort(list(perm), oracle.U(3), True)) == exp


def test_float16_matches_numpy_sort():
    """binary16 (Float(16,5,10)): bsort order is numeric order with -0 before +0 (np.sort on f16)."""
    rng = np.random.default_rng(16)
    a = np.concatenate([rng.standard_normal(3000) * 100, rng.uniform(-6e4, 6e4, 3000),
                        np.array([0.0, -0.0, np.inf, -np.inf, 6e-8, -6e-8, 65504, -65504] * 5)]).astype(np.float16)
    rng.shuffle(a)
    out = oracle.sort_native(a)
    _float_bits_equal_numeric(out, np.sort(a))
    assert oracle.sort_native(a, descending=True).tobytes() == out[::-1].tobytes()


def test_bfloat16_matches_float32_order():
    """bfloat16 words are the top halves of f32 words: sorting them as Float(16,8,7) must give the
    same order as sorting the widened f32 values (the exact numeric order of the bf16 values)."""
    rng = np.random.default_rng(17)
    f = np.concatenate([rng.standard_normal(2000) * 1e3, np.array([0.0, -0.0, np.inf, -np.inf] * 4)])
    w = (f.astype(np.float32).view(np.uint32) >> 16).astype(np.uint64)  # bf16 bit patterns
    w = np.concatenate([w, np.array([0x7FC1, 0xFFC1, 0x0001, 0x8001], np.uint64)])  # NaNs, subnormals
    rng.shuffle(w)
    got = oracle.bsort(w, oracle.BF16, True)
    widened = (got.astype(np.uint32) << 16).view(np.float32)
    ref = oracle.sort_native((w.astype(np.uint32) << 16).view(np.float32))
    assert np.array_equal(widened.view(np.uint32), ref.view(np.uint32))


def test_fullsize_order_key_matches_oracle_total_order():
    """tests/test_gpu_fullsize.py checks 2^30-key outputs with a torch restatement of the order
    (order_key); pin it to the oracle's own total-order key on every f32 pattern class: +-0,
    +-subnormals, +-normals of every exponent, +-inf, NaNs of both signs with assorted payloads,
    plus random bit patterns -- sorting by either key must give the same sequence."""
    import torch
    from test_gpu_fullsize import order_key
    rng = np.random.default_rng(20260)
    cls = [np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x00000001, 0x80000001,
                     0x007FFFFF, 0x807FFFFF, 0x7F800001, 0xFF800001, 0x7FC00000, 0xFFC00000,
                     0x7FFFFFFF, 0xFFFFFFFF, 0x00800000, 0x80800000], dtype=np.uint32)]
    for e in range(256):  # every exponent, both signs, a few mantissas
        m = rng.integers(0, 1 << 23, 4, dtype=np.uint32)
        for s in (0, 1):
            cls.append((np.uint32(s << 31) | np.uint32(e << 23) | m).astype(np.uint32))
    cls.append(rng.integers(0, 1 << 32, 1 << 20, dtype=np.uint64).astype(np.uint32))
    x = np.unique(np.concatenate(cls))
    rng.shuffle(x)
    k_test = order_key(torch.from_numpy(x.view(np.float32))).numpy()
    k_orc = oracle.total_order_keys(x.astype(np.uint64), oracle.NATIVE_SCHEMES[np.dtype(np.float32)])
    a = x[np.argsort(k_test, kind="stable")]
    b = x[np.argsort(k_orc, kind="stable")]
    assert np.array_equal(a, b)
    for dt, bits in ((np.float64, 64),):
        y = rng.integers(0, 1 << 63, 1 << 18, dtype=np.uint64) | (rng.integers(0, 2, 1 << 18, dtype=np.uint64) << 63)
        y = np.unique(np.concatenate([y, np.array([0, 1 << 63, 0x7FF0000000000000, 0xFFF0000000000000,
                                                   0x7FF8000000000000, 0xFFF8000000000000], dtype=np.uint64)]))
        kt = order_key(torch.from_numpy(y.view(np.int64)).view(torch.float64)).numpy()
        ko = oracle.total_order_keys(y, oracle.NATIVE_SCHEMES[np.dtype(dt)])
        assert np.array_equal(y[np.argsort(kt, kind="stable")], y[np.argsort(ko, kind="stable")])
