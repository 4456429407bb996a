"""GPU parity of the in-place mode / hybrid: ``sort_inplace_`` (256-way in-place
MSD partitions by the top digits, then the LSD path on bucket groups of <= chunk keys) must give
the oracle's sort bit for bit.  Small chunks force several partition levels, including on
skewed inputs (all equal, few distinct, keys sharing their top 16/24 bits), ragged sizes that
leave a partial last slot, misaligned pointers and both directions."""
import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

NP = {torch.uint8: np.uint8, torch.int8: np.int8, torch.uint16: np.uint16, torch.int16: np.int16,
      torch.uint32: np.uint32, torch.int32: np.int32, torch.float32: np.float32,
      torch.uint64: np.uint64, torch.int64: np.int64, torch.float64: np.float64}
SIGNED = {torch.uint16: torch.int16, torch.uint32: torch.int32, torch.uint64: torch.int64}
WIDE = [torch.uint32, torch.int32, torch.float32, torch.uint64, torch.int64, torch.float64]


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2603_08929_b200 as b
    return b


def host(t):
    return t.view(SIGNED.get(t.dtype, t.dtype)).cpu().numpy().view(NP[t.dtype])


def gen(dtype, n, seed):
    if dtype.is_floating_point:
        return W.special_mix(dtype, n, seed, "cuda")
    return W.uniform_int(dtype, n, seed, "cuda")


def check(B, t, descending, chunk, what=""):
    ref = oracle.sort_native(host(t), descending=descending)
    B.sort_inplace_(t, descending=descending, chunk=chunk)
    torch.cuda.synchronize()
    got = host(t)
    if got.tobytes() != ref.tobytes():
        bad = np.flatnonzero(got.view(np.uint8) != ref.view(np.uint8))
        raise AssertionError(f"{what}: mismatch at byte {bad[:5]} of {got.nbytes}")


@pytest.mark.parametrize("dtype", WIDE, ids=lambda d: str(d).split(".")[-1])
@pytest.mark.parametrize("descending", [False, True], ids=["asc", "desc"])
def test_random_sizes_small_chunks(B, dtype, descending):
    for n, chunk in ((0, 16), (1, 16), (1000, 2000), (4097, 1000), (100_003, 1000), (300_001, 50_000),
                     (1_000_037, 4096)):
        check(B, gen(dtype, n, 7 + n), descending, chunk, f"n={n} chunk={chunk}")


@pytest.mark.parametrize("dtype", WIDE, ids=lambda d: str(d).split(".")[-1])
def test_skewed_recursion(B, dtype):
    n = 200_003
    es = torch.empty(0, dtype=dtype).element_size()
    idt = torch.int64 if es == 8 else torch.int32
    sv = SIGNED.get(dtype, dtype) if not dtype.is_floating_point else idt
    # all equal: every level is a single bucket, recursion runs through all digits
    x = gen(dtype, 1, 3).view(sv).repeat(n).view(dtype)
    check(B, x, False, 5000, "all equal")
    # 16 distinct values
    table = gen(dtype, 16, 4).view(sv)
    y = table[(W.bits(n, 5, "cuda") >> 60) & 15].view(dtype)
    check(B, y, True, 5000, "16 distinct")
    # keys sharing their top 16 bits with many duplicates: deep recursion, heavy buckets
    low = (W.bits(n, 6, "cuda") & 0xFFF).to(torch.int64)
    base = 0x3A5C << (es * 8 - 16)
    z = (low + base).to(idt)
    z[::3] = z[0]
    check(B, z.view(dtype), False, 3000, "shared prefix")


@pytest.mark.parametrize("dtype", [torch.float32, torch.int64])
def test_misaligned_and_ragged(B, dtype):
    base = gen(dtype, 250_000, 11)
    before = host(base).copy()
    off = 3
    part = base[off:off + 199_999]
    check(B, part, False, 10_000, "misaligned")
    after = host(base)
    assert after[:off].tobytes() == before[:off].tobytes()
    assert after[off + 199_999:].tobytes() == before[off + 199_999:].tobytes()


@pytest.mark.parametrize("dtype", [torch.uint8, torch.int16])
def test_small_words_pass_through(B, dtype):
    check(B, gen(dtype, 100_001, 12), True, 1000, "counting path")


def test_cfg3_scaled_default_chunk(B):
    x = W.make("cfg3", "cuda", n=(1 << 23) + 5)
    check(B, x.clone(), False, 0, "cfg3 default chunk")
    check(B, x.clone(), True, 1 << 18, "cfg3 desc")


def test_workspace_is_small(B):
    n = 1 << 26
    full = B.workspace_bytes(torch.float32, n)
    small = B.inplace_workspace_bytes(torch.float32, n)
    assert small < full / 4, (small, full)
    assert B.inplace_workspace_bytes(torch.float32, n, 1 << 20) < n * 4 * 0.1
