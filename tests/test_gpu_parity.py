"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit for bit.

Every case generates a seeded input on the device, copies it to the host for the oracle
(R1, oracle/), sorts on the GPU with paper_2603_08929_b200 (ctypes -> libbsort.so), copies
back and compares raw bytes.  Sizes span several tiles with ragged tails; edge cases cover
n in {0, 1, 2}, misaligned pointers, all-equal input (every digit trivial), odd numbers of
executed LSD passes, NaN payloads of both signs, +-0, +-inf and subnormals.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

ALL = [torch.uint8, torch.int8, torch.uint16, torch.int16, torch.uint32, torch.int32,
       torch.float32, torch.uint64, torch.int64, torch.float64]
NP = {torch.uint8: np.uint8, torch.int8: np.int8, torch.uint16: np.uint16, torch.int16: np.int16,
      torch.uint32: np.uint32, torch.int32: np.int32, torch.float32: np.float32,
      torch.uint64: np.uint64, torch.int64: np.int64, torch.float64: np.float64}
TILE = {1: 0, 2: 0, 4: 512 * 16, 8: 384 * 12}


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2603_08929_b200 as b
    return b


SIGNED = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}


def sview(t: torch.Tensor) -> torch.Tensor:
    """Same bits with a dtype every torch op supports (uint16/32/64 have few kernels)."""
    return t.view(SIGNED.get(t.dtype, t.dtype))


def host(t: torch.Tensor) -> np.ndarray:
    return sview(t).cpu().numpy().view(NP[t.dtype])


def gen(dtype, n, seed):
    if dtype.is_floating_point:
        return W.special_mix(dtype, n, seed, "cuda")
    return W.uniform_int(dtype, n, seed, "cuda")


def check_equal(B, t, descending, what=""):
    ref = oracle.sort_native(host(t), descending=descending)
    B.sort_(t, descending=descending)
    torch.cuda.synchronize()
    got = host(t)
    if got.tobytes() != ref.tobytes():
        bad = np.flatnonzero(got.view(np.uint8) != ref.view(np.uint8))
        raise AssertionError(f"{what}: mismatch at byte {bad[:5]} of {got.nbytes}")


def sizes_for(dtype):
    es = torch.empty(0, dtype=dtype).element_size()
    base = [0, 1, 2, 3, 31, 1000, 4099, 65537]
    if TILE[es]:
        T = TILE[es]
        base += [T - 1, T, T + 1, 3 * T + 17]
    return base


@pytest.mark.parametrize("dtype", ALL, ids=lambda d: str(d).split(".")[-1])
@pytest.mark.parametrize("descending", [False, True], ids=["asc", "desc"])
def test_random_sizes(B, dtype, descending):
    for n in sizes_for(dtype):
        check_equal(B, gen(dtype, n, 1000 + n), descending, f"{dtype} n={n}")


@pytest.mark.parametrize("dtype", ALL, ids=lambda d: str(d).split(".")[-1])
def test_medium_size(B, dtype):
    n = (1 << 20) + 12345
    for desc in (False, True):
        check_equal(B, gen(dtype, n, 77), desc, f"{dtype} n={n}")


@pytest.mark.parametrize("dtype", ALL, ids=lambda d: str(d).split(".")[-1])
def test_misaligned_pointer(B, dtype):
    base = gen(dtype, 50001, 5)
    for off in (1, 3):
        view = base[off:off + 40000]
        assert view.data_ptr() % 16 != 0 or off == 0
        ref = oracle.sort_native(host(view), descending=False)
        before = host(base).copy()
        B.sort_(view)
        torch.cuda.synchronize()
        assert host(view).tobytes() == ref.tobytes()
        after = host(base)
        assert after[:off].tobytes() == before[:off].tobytes()  # neighbours untouched
        assert after[off + 40000:].tobytes() == before[off + 40000:].tobytes()


@pytest.mark.parametrize("dtype", ALL, ids=lambda d: str(d).split(".")[-1])
def test_all_equal_and_few_distinct(B, dtype):
    n = 3 * 8192 + 5
    x = sview(gen(dtype, 1, 9)).repeat(n).view(dtype)
    check_equal(B, x.clone(), False, "all equal")
    check_equal(B, x.clone(), True, "all equal desc")
    idx = W.bits(n, 3, "cuda")
    table = sview(gen(dtype, 16, 10))
    y = table[((idx >> 60) & 15)].view(dtype)
    check_equal(B, y, False, "16 distinct")


@pytest.mark.parametrize("dtype,bits", [(torch.uint32, 24), (torch.uint32, 8), (torch.int64, 40),
                                        (torch.uint64, 56), (torch.uint64, 8)])
def test_trivial_digits_odd_pass_count(B, dtype, bits):
    """Keys confined to the low `bits` bits: the top digits are trivial and skipped on the
    device; an odd number of executed passes ends in the scratch buffer (final copy)."""
    n = 100003
    r = W.bits(n, 21, "cuda") & ((1 << bits) - 1)
    x = r.to(torch.int64).view(torch.uint64) if dtype == torch.uint64 else r.to(
        torch.int64 if dtype == torch.int64 else torch.int32)
    if dtype == torch.uint32:
        x = r.to(torch.int32).view(torch.uint32)
    for desc in (False, True):
        check_equal(B, x.clone(), desc, f"{dtype} {bits} bits")


@pytest.mark.parametrize("layout", ["sorted", "reverse", "equal", "distinct16"])
def test_cfg4_layouts_scaled(B, layout):
    x = W.make("cfg4", "cuda", n=(1 << 21) + 7, layout=layout)
    check_equal(B, x, False, layout)


def test_cfg1_full(B):
    """BASELINE.json cfg1 at full size: oracle parity on all 2^20 keys."""
    check_equal(B, W.make("cfg1", "cuda"), False, "cfg1")


def test_cfg3_scaled(B):
    x = W.make("cfg3", "cuda", n=(1 << 22) + 3)
    check_equal(B, x.clone(), False, "cfg3")
    check_equal(B, x.clone(), True, "cfg3 desc")


@pytest.mark.parametrize("dtype", [torch.uint8, torch.int8, torch.int16, torch.uint16])
def test_cfg2_scaled(B, dtype):
    x = W.make("cfg2", "cuda", n=(1 << 22) + 9, dtype=dtype)
    for desc in (False, True):
        check_equal(B, x.clone(), desc, f"cfg2 {dtype}")


def test_cfg5_scaled_local(B):
    for dt in (torch.int64, torch.float64):
        x = W.make("cfg5", "cuda", n=(1 << 21) + 1, dtype=dt)
        check_equal(B, x, False, f"cfg5 local {dt}")


def test_sort_host_roundtrip(B):
    x = gen(torch.float32, 300001, 8).cpu().pin_memory()
    ref = oracle.sort_native(x.numpy(), descending=True)
    B.sort_host(x, descending=True)
    assert x.numpy().tobytes() == ref.tobytes()


def test_sort_host_to_two_streams(B):
    """bsort_sort_host_to: pinned input never written; two sorts in flight on two streams (the
    bench's pipelined e2e), joint-histogram size (2^24 + 5) and a small one, both directions."""
    for n, dt in (((1 << 24) + 5, torch.float32), (70001, torch.int64)):
        x = gen(dt, n, 12).cpu().pin_memory()
        keep = x.clone()
        for desc in (False, True):
            ref = oracle.sort_native(x.numpy(), descending=desc)
            streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            sorters = [B.Sorter(dt, n, "cuda") for _ in range(2)]
            devs = [torch.empty(n, dtype=dt, device="cuda") for _ in range(2)]
            outs = [torch.empty(n, dtype=dt, pin_memory=True) for _ in range(2)]
            for i in range(4):
                sorters[i % 2].sort_host_to(x, outs[i % 2], devs[i % 2], desc, stream=streams[i % 2])
            torch.cuda.synchronize()
            for o in outs:
                assert o.numpy().tobytes() == ref.tobytes(), (n, dt, desc)
            assert x.numpy().tobytes() == keep.numpy().tobytes()  # the input was only read (NaNs: bytes)


def test_errors_raise(B):
    t = torch.zeros(10, dtype=torch.complex64, device="cuda")
    with pytest.raises(TypeError):
        B.sort_(t)
    with pytest.raises(TypeError):
        B.sort_(torch.zeros(10))  # CPU tensor: no fallback
    with pytest.raises(ValueError):
        B.sort_(torch.zeros(10, 2, device="cuda").t())


def test_launch_counter_moves(B):
    x = gen(torch.int32, (1 << 22) + 1, 1)
    c0 = B.launch_count()
    B.sort_(x)
    torch.cuda.synchronize()
    # hist (with the plan fused) + 4 passes + copy-back; memsets are not counted
    assert B.launch_count() - c0 == 6


@pytest.mark.parametrize("dtype", [torch.int16, torch.uint16])
def test_count16_drain_path(B, dtype):
    """16-bit histogram: a bin receiving more than 0x8000 keys inside one CTA drains to the
    global overflow counter (all-equal and 3-valued inputs large enough to drain several times)."""
    n = (1 << 23) + 5
    x = sview(gen(dtype, 1, 31)).repeat(n).view(dtype)
    check_equal(B, x.clone(), False, "all equal")
    check_equal(B, x.clone(), True, "all equal desc")
    table = sview(gen(dtype, 3, 32))
    y = table[(W.bits(n, 33, "cuda") >> 62) % 3].view(dtype)
    check_equal(B, y, True, "3 distinct")


@pytest.mark.parametrize("dtype", [torch.float32, torch.int32, torch.uint64, torch.float64])
def test_joint_pass1_paths(B, dtype):
    """n >= 2^24 switches the histogram to the joint (digit 0, digit 1) form.  Pass 1 then runs
    look-back-free when every nonzero digit-0 bucket is at least one tile long (random keys), and
    falls back to the look-back pass when one bucket is tiny (second case)."""
    n = (1 << 24) + 12345
    x = gen(dtype, n, 123)
    check_equal(B, x.clone(), dtype == torch.float32, "joint-eligible")
    es = x.element_size()
    ib = {4: torch.int32, 8: torch.int64}[es]
    b = x.view(ib).clone()
    low = b & 0xFF
    b = torch.where(low == 0x42, b + 1, b)       # empty digit-0 bucket 0x42 ...
    b[:100] = (b[:100] & ~0xFF) | 0x42           # ... except for 100 keys
    check_equal(B, b.view(dtype), False, "joint-ineligible")


@pytest.mark.parametrize("dtype", [torch.float64, torch.int64, torch.float32])
def test_large_descending_misaligned_and_trivial(B, dtype):
    """n >= 2^24 (joint histogram, J01/RUN2 passes) combined with: descending order, a caller
    pointer that is not 16-byte aligned (per-warp loads instead of TMA, ragged head and tail in
    the histogram), and keys confined to the low 24 bits (trivial high digits are skipped)."""
    n = (1 << 24) + 777
    base = gen(dtype, n + 3, 321)
    view = base[1:n + 1]  # element-aligned, not 16-byte aligned
    assert view.data_ptr() % 16 != 0
    check_equal(B, view, True, "misaligned desc")
    ib = {4: torch.int32, 8: torch.int64}[view.element_size()]
    low = (W.bits(n, 654, "cuda") & 0xFFFFFF).to(ib)
    check_equal(B, low.view(dtype), dtype == torch.int64, "low 24 bits")


@pytest.mark.parametrize("dtype", [torch.float16, torch.bfloat16])
@pytest.mark.parametrize("descending", [False, True], ids=["asc", "desc"])
def test_half_floats(B, dtype, descending):
    """f16 / bf16 (N4 widening): every bit pattern incl. NaNs of both signs, +-0, +-inf and
    subnormals, against the oracle's Float(16,5,10) / Float(16,8,7) schemes."""
    scheme = oracle.F(16, 5, 10) if dtype == torch.float16 else oracle.BF16
    for n in (0, 1, 2, 31, 1000, 65537, (1 << 20) + 13, 65536 * 3):
        bits16 = W.uniform_int(torch.int16, n, 500 + n, "cuda")
        if n == 65536 * 3:  # every pattern three times
            bits16 = (torch.arange(n, device="cuda", dtype=torch.int64) % 65536).to(torch.int32).to(torch.int16)
        x = bits16.view(dtype).clone()
        words = x.view(torch.int16).cpu().numpy().view(np.uint16).astype(np.uint64)
        ref = oracle.bsort(words, scheme, asc=not descending).astype(np.uint16)
        B.sort_(x, descending=descending)
        torch.cuda.synchronize()
        got = x.view(torch.int16).cpu().numpy().view(np.uint16)
        assert got.tobytes() == ref.tobytes(), f"{dtype} n={n}"


def check_pairs(B, x, descending, what=""):
    """Key-value sort (§8 N3) with values 0..n-1 (argsort): keys bit-exact vs the oracle; the
    values a permutation; every value points at an input key with the same bits as the output
    key beside it (equal keys may carry their values in any order)."""
    n = x.numel()
    ref = oracle.sort_native(host(x), descending=descending)
    keys, idx = B.argsort(x, descending)
    torch.cuda.synchronize()
    assert host(keys).tobytes() == ref.tobytes(), f"{what}: keys"
    ii = idx.to(torch.int64)
    assert bool((torch.sort(ii).values == torch.arange(n, device=ii.device)).all()), f"{what}: not a permutation"
    ib = {4: torch.int32, 8: torch.int64}[x.element_size()]
    assert torch.equal(x.view(ib)[ii], keys.view(ib)), f"{what}: value does not follow its key"


@pytest.mark.parametrize("dtype", [torch.float32, torch.int32, torch.uint32, torch.float64, torch.int64,
                                   torch.uint64], ids=lambda d: str(d).split(".")[-1])
def test_key_value_sort(B, dtype):
    for n in (0, 1, 2, 1000, 8191, 8193, 65537, (1 << 20) + 7):
        check_pairs(B, gen(dtype, n, 900 + n), n % 2 == 1, f"{dtype} n={n}")
    x = sview(gen(dtype, 1, 5)).repeat(50_000).view(dtype)   # all equal: any permutation is fine
    check_pairs(B, x, False, "all equal")


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_key_value_large_and_misaligned(B, dtype):
    """n >= 2^24 (joint histogram, J01 pass 1) and a keys pointer that is not 16-byte aligned."""
    n = (1 << 24) + 99
    check_pairs(B, gen(dtype, n, 77), False, "large")
    base = gen(dtype, 300_003, 78)
    check_pairs(B, base[1:300_001], True, "misaligned")


def test_key_value_rejects_small_keys(B):
    from paper_2603_08929_b200 import BsortError
    k = torch.zeros(100, dtype=torch.int16, device="cuda")
    v = torch.zeros(100, dtype=torch.int32, device="cuda")
    with pytest.raises(BsortError):
        B.sort_pairs_(k, v)


@pytest.mark.parametrize("dtype,n", [(torch.int32, 1 << 20), (torch.float64, 300_007), (torch.uint8, 100_000),
                                     (torch.float32, (1 << 24) + 5)])
def test_cuda_graph_capture_and_replay(B, dtype, n):
    """The whole path is stream-ordered with no host sync: it captures into a CUDA graph, and
    each replay sorts the buffer's current contents (device-side plan: trivial digits, J01
    eligibility and the final copy are decided at replay time, not at capture)."""
    buf = gen(dtype, n, 77)
    s = B.Sorter(dtype, n, "cuda")
    g = s.graph(buf, descending=False)
    for seed in (78, 79):
        x = gen(dtype, n, seed)
        if seed == 79 and buf.element_size() >= 4:  # different trivial digits than at capture
            ib = {4: torch.int32, 8: torch.int64}[buf.element_size()]
            x = (x.view(ib) & 0xFFFF).view(dtype)
        ref = oracle.sort_native(host(x))
        buf.copy_(x)
        g.replay()
        torch.cuda.synchronize()
        assert host(buf).tobytes() == ref.tobytes(), f"replay {seed}"


@pytest.mark.parametrize("dtype", [torch.uint32, torch.float32, torch.int64, torch.float64],
                         ids=lambda d: str(d).split(".")[-1])
@pytest.mark.parametrize("descending", [False, True], ids=["asc", "desc"])
def test_warp_specialised_sizes(B, dtype, descending):
    """n >= 2^22 routes the look-back passes (and 64-bit pass 0) through k_onesweep_pass_ws:
    ragged last tiles of its 10240 / 7168-key tiles, trivial high digits, and the key-value form."""
    for n in ((1 << 22) + 1, (1 << 22) + 10239, 3 * (1 << 22) + 7167):
        check_equal(B, gen(dtype, n, n % 1000), descending, f"ws n={n}")
    es = torch.empty(0, dtype=dtype).element_size()
    ib = {4: torch.int32, 8: torch.int64}[es]
    low = (W.bits((1 << 22) + 5, 31, "cuda") & 0xFFFFF).to(ib).view(dtype)  # top digits trivial
    check_equal(B, low, descending, "ws trivial digits")
    keys = gen(dtype, (1 << 22) + 333, 32)
    ref = oracle.sort_native(host(keys), descending=descending)
    vals = torch.arange(keys.numel(), dtype=torch.int32, device="cuda")
    orig = host(keys).copy()
    B.sort_pairs_(keys, vals, descending)
    torch.cuda.synchronize()
    assert host(keys).tobytes() == ref.tobytes()
    v = vals.cpu().numpy()
    assert np.array_equal(np.sort(v), np.arange(v.size))
    assert orig[v].tobytes() == ref.tobytes()  # every value followed its key


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint64, torch.float64],
                         ids=lambda d: str(d).split(".")[-1])
def test_presorted_fast_path(B, dtype):
    """The histogram sweep detects input already in the requested order (no pass runs) or in the
    opposite order (reversed in place): sorted, reversed, sorted-but-one-swap (must NOT take the
    fast path), duplicates, key-value payloads, small and >= 2^24 sizes."""
    for n in (3, 5000, 100_003, (1 << 24) + 77):
        x = gen(dtype, n, 900 + n % 97)
        srt_np = oracle.sort_native(host(x))
        asc = torch.from_numpy(srt_np.view({4: np.int32, 8: np.int64}[srt_np.itemsize]).copy()).to("cuda").view(dtype)
        for desc in (False, True):
            check_equal(B, asc.clone(), desc, f"sorted asc input, desc={desc}")
        swapped = asc.clone()
        if n > 3:
            iv = {4: torch.int32, 8: torch.int64}[asc.element_size()]
            swapped.view(iv)[n - 2:n] = asc.view(iv)[n - 2:n].flip(0)
            check_equal(B, swapped, False, "one swap at the end")
    # duplicates in reverse order
    base = gen(dtype, 64, 5)
    srt = oracle.sort_native(host(base), descending=True)
    rev = np.repeat(srt, 70_001)
    t = torch.from_numpy(rev.view({4: np.int32, 8: np.int64}[rev.itemsize])).to("cuda").view(dtype)
    check_equal(B, t, False, "reversed with duplicates")
    # key-value: reversed keys -> values reversed with them
    keys = torch.from_numpy(srt.view({4: np.int32, 8: np.int64}[srt.itemsize]).copy()).to("cuda").view(dtype)
    vals = torch.arange(keys.numel(), dtype=torch.int32, device="cuda")
    B.sort_pairs_(keys, vals)
    torch.cuda.synchronize()
    assert host(keys).tobytes() == oracle.sort_native(srt).tobytes()
    assert np.array_equal(vals.cpu().numpy(), np.arange(keys.numel())[::-1])


# ---- BASELINE.json's own signature: bsort_sort(dtype, dev_ptr, n, direction, stream), which
# allocates its workspace itself (stream-ordered cudaMallocAsync / cudaFreeAsync)

@pytest.mark.parametrize("dtype", ALL)
@pytest.mark.parametrize("desc", [False, True])
def test_bsort_sort_bj_signature(B, dtype, desc):
    import ctypes
    n = (1 << 22) + 13 if torch.empty(0, dtype=dtype).element_size() >= 4 else (1 << 20) + 13
    t = gen(dtype, n, 901 + ALL.index(dtype))
    ref = oracle.sort_native(host(t), descending=desc)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    st = B.lib.bsort_sort(B.dtype_code(dtype), ctypes.c_void_p(t.data_ptr()), n, int(desc), stream)
    assert st == 0, B.lib.bsort_status_string(st)
    torch.cuda.synchronize()
    assert host(t).tobytes() == ref.tobytes()


def test_second_device_after_first(B):
    """Launch set-up is per device: a sort on cuda:1 after one on cuda:0 works."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    for d in (0, 1):
        x = gen(torch.float32, (1 << 22) + 5, 77 + d).to(f"cuda:{d}")
        ref = oracle.sort_native(host(x), descending=False)
        B.sort_(x)
        torch.cuda.synchronize(d)
        assert host(x).tobytes() == ref.tobytes()


# ---- presorted fast path: the histogram sweep's adjacent-pair check must catch a
# single out-of-order pair wherever it sits -- inside a 16-byte vector, across vectors (taken
# from the next lane by a shuffle), across lane 31 / warps (read from memory) and across the
# grid-stride boundary -- for inputs in the requested order and in the opposite order.

@pytest.mark.parametrize("dtype", [torch.int32, torch.int64])
@pytest.mark.parametrize("n", [(1 << 22) + 7, (1 << 24) + 11])
@pytest.mark.parametrize("desc", [False, True])
def test_presorted_one_swap_interior(B, dtype, n, desc):
    import paper_2603_08929_b200 as b
    per_vec = 16 // torch.empty(0, dtype=dtype).element_size()
    base, _ = torch.sort(W.uniform_int(dtype, n, 4242, "cuda"))
    want = base.flip(0) if desc else base
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    spots = {"in-vector": 4 * per_vec + 1, "vector-boundary": 5 * per_vec - 1,
             "lane31": 32 * per_vec - 1, "warp": 3 * 32 * per_vec - 1,
             "grid-stride": sms * 1024 * per_vec - 1}
    for name, p in spots.items():
        for src in (want, want.flip(0)):  # requested order / opposite order, one swap each
            x = src.clone()
            x[p], x[p + 1] = src[p + 1].item(), src[p].item()
            if bool((x == src).all()):
                continue  # equal neighbours: nothing swapped
            b.sort_(x, descending=desc)
            torch.cuda.synchronize()
            assert bool((x == want).all()), f"{name} at {p} (n={n}, desc={desc})"


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint32], ids=lambda d: str(d).split(".")[-1])
def test_few_runs_passes(B, dtype):
    """Few distinct keys at joint-histogram sizes: the plan routes LSD passes 2-3 of 32-bit keys to
    the run-ranking look-back kernel (PassPlan::fewruns) instead of the lane-ordered k_pass2.
    Cases: 16 distinct values (every tile meets <= 2 runs), 300 distinct values of which 10 are
    rare (tiles around a rare value meet > 2 runs: per-tile fallback to the stable ranking), and
    a misaligned pointer (no TMA: k_pass2 alone)."""
    n = (1 << 24) + 4099
    idx = W.bits(n, 41, "cuda")
    table = sview(gen(dtype, 300, 42))
    y = table[((idx >> 60) & 15)].view(dtype)
    check_equal(B, y.clone(), False, "16 distinct asc")
    check_equal(B, y.clone(), True, "16 distinct desc")
    k = ((idx >> 33) & 0x7FFFFFFF) % 290
    pos = torch.arange(n, device="cuda")
    rare = pos % 100003 == 5
    k = torch.where(rare, 290 + (pos // 100003) % 10, k)
    z = table[k].view(dtype)
    check_equal(B, z.clone(), False, "290 common + 10 rare")
    check_equal(B, z.clone(), True, "290 common + 10 rare desc")
    buf = torch.empty(n + 1, dtype=dtype, device="cuda")
    buf[1:] = y
    check_equal(B, buf[1:], False, "16 distinct misaligned")


@pytest.mark.parametrize("dtype", [torch.uint32, torch.int32, torch.float32], ids=lambda d: str(d).split(".")[-1])
def test_chunked_lookback_passes(B, dtype):
    """LSD pass 2 of 32-bit keys at joint-histogram sizes runs as LB_NC = 4 look-back chains
    (chunks = top two bits of digit 1; chunk map from the histogram sweep's coarse joint,
    round-robin dispatch by segment table).  Edge cases: every key in one chunk (others empty),
    a trivial digit 1 (pass 1 skipped: pass 2's chunks follow digit 1 anyway), chunks of very
    different sizes (tile counts 1 vs ~1,600: segments of slope 4 then 1), both directions,
    ragged n."""
    n = (1 << 24) + 12345
    r = W.bits(n, 51, "cuda")
    lo = r & 0xFFFFFFFF

    def as_dtype(v):
        v = v & 0xFFFFFFFF
        v = torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32)
        return v.view(dtype)

    if dtype == torch.float32:
        lo = lo & ~(0xFF << 23) | (0x7E << 23)  # finite, both signs (exponent fixed, sign random)
    one = (lo & ~(3 << 14)) | (3 << 22)         # pass 2: all in chunk 0
    triv = (lo & ~(0xFF << 8)) | (0x5A << 8)    # digit 1 trivial
    skew = torch.where((r >> 40) % 100 == 0, lo, lo & ~(3 << 14))  # chunk 0 ~99%, others ~0.3%
    for v, what in ((lo, "random"), (one, "single chunks"), (triv, "trivial digit 1"), (skew, "skewed chunks")):
        x = as_dtype(v)
        check_equal(B, x.clone(), False, what)
        check_equal(B, x.clone(), True, what + " desc")


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32], ids=lambda d: str(d).split(".")[-1])
def test_blocks_of_equal_keys_joint_sizes(B, dtype):
    """Long runs of equal keys in non-sorted order at joint-histogram sizes: warps whose 128 keys
    share a joint bin add once (the u16 bins then cross 0x8000 by a 128-key step: drain path),
    the rest add per key; runs of 4096 keys of three values, plus a ragged tail."""
    n = (1 << 24) + 5
    i = torch.arange(n, device="cuda")
    vals = torch.tensor([0x40490FDB, -7, 0x12345], dtype=torch.int64, device="cuda")
    v = vals[((i // 4096) * 7919) % 3]
    x = torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32).view(dtype)
    check_equal(B, x.clone(), False, "blocks of equal keys")
    check_equal(B, x.clone(), True, "blocks of equal keys desc")


@pytest.mark.parametrize("env", [{"BSORT_P2": "0"}, {"BSORT_P2": "0", "BSORT_WS": "0"}, {"BSORT_WS": "0"}])
def test_round1_fallback_kernels_at_joint_sizes(env):
    """The kernels that run where k_pass2 cannot (BSORT_P2=0: what a device that fails the
    lane-order self-test gets) and where the warp-specialised kernel cannot (BSORT_WS=0, or a caller
    pointer that is not 16-byte aligned) -- k_onesweep_pass with 8,192-key look-back tiles -- on a
    32-bit joint-histogram sort, whose three look-back regions are sized for larger tiles
    (lsd_impl.cuh: they then serve as one region).  The switches are read once per process."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch, oracle, workloads as W, paper_2603_08929_b200 as B
n = (1 << 24) + 777
for dt, off in ((torch.float32, 1), (torch.float32, 0), (torch.int32, 3)):
    base = W.special_mix(dt, n + 4, 77, "cuda") if dt.is_floating_point else W.uniform_int(dt, n + 4, 77, "cuda")
    for desc in (False, True):
        x = base.clone()[off:off + n]
        assert (x.data_ptr() %% 16 != 0) == (off != 0)
        ref = oracle.sort_native(x.cpu().numpy(), descending=desc)
        B.sort_(x, descending=desc); torch.cuda.synchronize()
        assert x.cpu().numpy().tobytes() == ref.tobytes(), (dt, off, desc)
print("ok")
""" % repo
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=900, cwd=repo)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-500:], r.stderr[-2000:])
