"""GPU parity of the small-n paths against the CPU oracle, bit for bit: csrc/small.cuh (the
whole LSD sort in shared memory by one CTA in one launch, keys-only n <= 20480 32-bit / 10240
64-bit keys) and csrc/small_grid.cuh (one cooperative launch, one CTA per SM with grid barriers,
up to SMs x 20480 / 10240 keys): sizes around warp segments, chunk and grid boundaries and both
sides of each bound, passes skipped for constant digits (odd and even numbers of moving
passes), both directions, the multi-launch path above the bounds (its look-back zeroing folded
into the pass kernels below 2^22 keys) and at the same sizes (BSORT_SMALL=0 / BSORT_GRID=0 /
BSORT_SMALL_MAX, in subprocesses: the switches are read once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NP = {torch.uint32: np.uint32, torch.int32: np.int32, torch.float32: np.float32,
      torch.uint64: np.uint64, torch.int64: np.int64, torch.float64: np.float64, torch.uint8: np.uint8}
SIGNED = {torch.uint32: torch.int32, torch.uint64: torch.int64}


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


def check(B, t, desc, what):
    ref = oracle.sort_native(host(t), descending=desc)
    B.sort_(t, descending=desc)
    torch.cuda.synchronize()
    got = host(t)
    if got.tobytes() != ref.tobytes():
        bad = np.flatnonzero(got != ref) if got.dtype.kind != "f" else np.flatnonzero(
            got.view(np.uint8) != ref.view(np.uint8))
        raise AssertionError(f"{what}: {len(bad)} mismatches, first at {bad[:4]} of n={got.size}")


def bound(dtype):
    return 20480 if torch.empty(0, dtype=dtype).element_size() == 4 else 10240


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint64, torch.float64],
                         ids=lambda d: str(d).split(".")[-1])
@pytest.mark.parametrize("desc", [False, True], ids=["asc", "desc"])
def test_small_sizes(B, dtype, desc):
    big = bound(dtype)
    gmax = torch.cuda.get_device_properties(0).multi_processor_count * big  # k_grid_sort capacity
    for n in [2, 3, 15, 16, 17, 31, 32, 33, 511, 512, 513, 4097, big // 2 + 3, big - 1, big, big + 1,
              2 * 8192 + 5, 3 * big + 7, 300_007, (1 << 20) + 3, gmax - 1, gmax, gmax + 1,
              (1 << 22) - 1, (1 << 22) + 1]:
        check(B, gen(dtype, n, 1000 + n), desc, f"n={n}")


@pytest.mark.parametrize("dtype,keep", [(torch.uint32, 0x000000FF), (torch.uint32, 0x00FF00FF),
                                        (torch.uint32, 0x00FFFFFF), (torch.int32, 0x7F00FF00),
                                        (torch.uint64, 0x00FF0000FF0000FF), (torch.int64, 0x0FFFFFFFFFFFFF00)])
@pytest.mark.parametrize("n", [5000, 1 << 20])
def test_small_skipped_passes(B, dtype, keep, n):
    """Constant digits: their passes are skipped; 1, 2, 3 (odd: copy-back) and 7 moving passes."""
    x = W.uniform_int(dtype, n, 77, "cuda")
    sd = SIGNED.get(dtype, dtype)
    x = (x.view(sd) & torch.tensor(keep, dtype=torch.int64).to(sd).item()).view(dtype)
    for desc in (False, True):
        check(B, x.clone(), desc, f"keep={keep:#x} desc={desc}")


def test_small_all_equal_and_two_values(B):
    for n in (9, 10_000, 100_000, 1 << 22):
        x = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        check(B, x.clone(), False, f"equal n={n}")
        x[::3] = 12
        check(B, x.clone(), True, f"two values n={n}")


def test_multilaunch_path_at_small_sizes():
    """BSORT_SMALL=0 BSORT_GRID=0: the multi-launch one-sweep path the small kernels replace, same sizes."""
    code = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch, oracle, workloads as W, paper_2603_08929_b200 as B
for dt, n in ((torch.int32, 1000), (torch.int32, 1 << 20), (torch.float64, 70001), (torch.float32, 8193)):
    x = W.special_mix(dt, n, 5, "cuda") if dt.is_floating_point else W.uniform_int(dt, n, 5, "cuda")
    h = x.cpu().numpy()
    for desc in (False, True):
        ref = oracle.sort_native(h, descending=desc)
        y = x.clone(); B.sort_(y, descending=desc); torch.cuda.synchronize()
        assert y.cpu().numpy().tobytes() == ref.tobytes(), (dt, n, desc)
print("ok")
""" % REPO
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, BSORT_SMALL="0", BSORT_GRID="0"), capture_output=True,
                       text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


def _subprocess_sorts(env, cases, expect_launches=None):
    code = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch, oracle, workloads as W, paper_2603_08929_b200 as B
U = {torch.uint32: (torch.int32, np.uint32), torch.uint64: (torch.int64, np.uint64)}
for dt, n in %r:
    x = W.special_mix(dt, n, 9, "cuda") if dt.is_floating_point else W.uniform_int(dt, n, 9, "cuda")
    sd, nd = U.get(dt, (dt, None))
    h = x.view(sd).cpu().numpy()
    h = h.view(nd) if nd else h
    for desc in (False, True):
        ref = oracle.sort_native(h, descending=desc)
        y = x.clone(); c0 = B.launch_count(); B.sort_(y, descending=desc); torch.cuda.synchronize()
        if %r is not None:
            assert B.launch_count() - c0 == %r, (dt, n, B.launch_count() - c0)
        assert y.view(sd).cpu().numpy().tobytes() == ref.tobytes(), (dt, n, desc)
print("ok")
""" % (REPO, cases, expect_launches, expect_launches)
    code = code.replace("torch.torch.", "torch.")
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600, cwd=REPO)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


CASES_SMALL = "[(torch.int32, 20480), (torch.float32, 20479), (torch.uint32, 16385), (torch.int32, 1001), " \
              "(torch.float32, 4097), (torch.float64, 1 << 18), (torch.int64, (1 << 18) + 7)]"


def test_grid_kernel_at_small_sizes():
    """BSORT_SMALL_MAX=1000: sizes the single-CTA kernel would take run k_grid_sort with 1-5 CTAs
    (chunks of >= 4096 keys), one launch each; 64-bit keys from k_grid_sort's 2^18 lower bound."""
    _subprocess_sorts({"BSORT_SMALL_MAX": "1000"}, eval(CASES_SMALL), expect_launches=1)


def test_multilaunch_at_grid_sizes():
    """BSORT_GRID=0: the multi-launch path at the sizes k_grid_sort takes by default."""
    _subprocess_sorts({"BSORT_GRID": "0"}, [(torch.int32, 300_007), (torch.float64, 70_001),
                                             (torch.uint32, (1 << 20) + 3), (torch.int64, 1 << 20)])


def test_small_launch_count(B):
    """One launch per small sort (the path's point): libbsort's own launch counter."""
    x = W.uniform_int(torch.int32, 10_000, 3, "cuda")
    B.sort_(x)
    torch.cuda.synchronize()
    c0 = B.launch_count()
    B.sort_(x)
    torch.cuda.synchronize()
    assert B.launch_count() - c0 == 1


def test_selftest_lane_order(B):
    """bsort_selftest: the shared-atomic lane order the stable rankings rely on holds here (if it
    did not, the library would route around those kernels and this documents that it does not
    need to on this part)."""
    assert B.selftest() == 0


@pytest.mark.parametrize("dtype,n", [(torch.int32, 1 << 20), (torch.float64, 300_007), (torch.uint8, 100_000),
                                     (torch.float32, (1 << 22) + 3)])
def test_graph_replay_same_buffers(B, dtype, n):
    """Repeated sorts of the same buffers (same Sorter workspace): call 1 runs plain launches,
    call 2 captures the launch sequence into a CUDA graph, later calls replay it (graphs.cu).
    New data every call, both directions: the replayed graph re-reads keys and re-plans."""
    s = B.Sorter(dtype, n, "cuda")
    w = torch.empty(n, dtype=dtype, device="cuda")
    for i in range(6):
        desc = bool(i % 2)
        src = gen(dtype, n, 4000 + i) if dtype != torch.uint8 else W.uniform_int(dtype, n, 4000 + i, "cuda")
        if i == 4:
            src = torch.sort(src)[0]  # presorted input through the replayed graph (plan skips passes)
        w.copy_(src)
        ref = oracle.sort_native(host(w) if dtype in NP else w.cpu().numpy(), descending=desc)
        c0 = B.launch_count()
        s(w, desc)
        torch.cuda.synchronize()
        assert B.launch_count() > c0
        got = host(w) if dtype in NP else w.cpu().numpy()
        assert got.tobytes() == ref.tobytes(), (i, desc)


def test_graph_replay_disabled_matches():
    """BSORT_GRAPH=0 (plain launches every call) gives the same bytes as the replayed graphs."""
    code = r"""
import sys; sys.path.insert(0, %r)
import torch, oracle, workloads as W, paper_2603_08929_b200 as B
n = 1 << 20
s = B.Sorter(torch.int32, n, "cuda")
w = torch.empty(n, dtype=torch.int32, device="cuda")
for i in range(4):
    w.copy_(W.uniform_int(torch.int32, n, 77 + i, "cuda"))
    ref = oracle.sort_native(w.cpu().numpy())
    s(w); torch.cuda.synchronize()
    assert w.cpu().numpy().tobytes() == ref.tobytes(), i
print("ok")
""" % REPO
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, BSORT_GRAPH="0"), capture_output=True,
                       text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint32], ids=lambda d: str(d).split(".")[-1])
@pytest.mark.parametrize("desc", [False, True], ids=["asc", "desc"])
def test_grid_msd_fast_path_and_fallback(B, dtype, desc):
    """k_grid_sort's MSD-first path (32-bit keys): one grid pass on the top digit, then every
    bucket sorted in one CTA's shared memory.  Cases: uniform keys (256 buckets of ~4K keys), a
    top byte confined to 48 values (buckets of ~21K, some above one CTA's capacity: the LSD
    fallback), 40 values over 700K keys (buckets of ~17K, below capacity: uneven bucket loads),
    a constant top byte (the MSD pass moves nothing; one bucket of all keys: fallback), and a
    5% heavy top byte (one bucket of ~52K keys: fallback)."""
    n = (1 << 20) + 3
    r = W.bits(n, 61, "cuda")
    lo = r & 0xFFFFFF

    def mk(top, m=n):
        v = ((top[:m] << 24) | lo[:m]) & 0xFFFFFFFF
        v = torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32)
        return v.view(dtype)

    tb = (r >> 40) & 255
    cases = [(mk(tb), "uniform"), (mk(0x30 + (r >> 40) % 48), "48 top values"),
             (mk(0x41 + (r >> 40) % 40, 700_001), "40 top values, 700K keys"),
             (mk(torch.full_like(tb, 0x3C)), "constant top byte"),
             (mk(torch.where((r >> 50) % 20 == 0, torch.full_like(tb, 0x3D), tb)), "5% heavy top byte")]
    for x, what in cases:
        check(B, x.clone(), desc, what)


def test_grid_lsd_only_at_grid_sizes():
    """BSORT_GRID_MSD=0: k_grid_sort's plain LSD passes (the MSD path's fallback) at grid sizes."""
    _subprocess_sorts({"BSORT_GRID_MSD": "0"}, [(torch.int32, 300_007), (torch.float32, (1 << 20) + 3),
                                                 (torch.uint32, 50_001)], expect_launches=1)


def test_grid_counter_barrier():
    """BSORT_GRID_CG=0: k_grid_sort's grid barriers on the workspace counter (memset before the
    launch) instead of cooperative groups' grid.sync(); MSD and LSD grid sizes, 64-bit keys."""
    _subprocess_sorts({"BSORT_GRID_CG": "0"}, [(torch.int32, (1 << 20) + 5), (torch.float32, 300_007),
                                               (torch.int64, (1 << 18) + 7)])


def test_grid_msd_single_bucket_in_place():
    """BSORT_SMALL_MAX=1000: a 20,000-key grid sort whose top digit is constant -- the MSD pass
    moves nothing and its one bucket (all keys, still in the caller's buffer) fits one CTA."""
    code = r"""
import sys; sys.path.insert(0, %r)
import numpy as np, torch, oracle, workloads as W, paper_2603_08929_b200 as B
x = (W.uniform_int(torch.int32, 20000, 3, "cuda") & 0x00FFFFFF) | 0x15000000
for desc in (False, True):
    ref = oracle.sort_native(x.cpu().numpy(), descending=desc)
    y = x.clone(); B.sort_(y, descending=desc); torch.cuda.synchronize()
    assert y.cpu().numpy().tobytes() == ref.tobytes(), desc
print("ok")
""" % REPO
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, BSORT_SMALL_MAX="1000"),
                       capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
