"""The C-ABI boundary on CPU (no GPU): libbsort.so loads, exports every function include/bsort.h
declares, its enum values match the Python binding, argument errors are rejected before any
launch, and the host-only splitter math of the MSD partition is right.

The splitter/send-count checks pin libbsort's host C against a plain numpy restatement of the
rule in bsort.h (cuts[r] = smallest bin b with prefix(b) >= floor(r*total/P))."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "bsort.h")


@pytest.fixture(scope="module")
def B():
    lib = os.path.join(REPO, "paper_2603_08929_b200", "libbsort.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", REPO, "lib"], check=True)
    import paper_2603_08929_b200 as b
    return b


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsort_[a-z0-9_]+)\s*\(", src)))


def header_enums():
    src = open(HEADER).read()
    return {k: int(v) for k, v in re.findall(r"\b(BSORT_[A-Z0-9_]+)\s*=\s*(\d+)", src)}


def test_header_declares_the_boundary():
    fns = header_functions()
    for f in ("bsort_sort", "bsort_sort_ws", "bsort_workspace_bytes", "bsort_sort_host",
              "bsort_dist_top_hist", "bsort_dist_splitters", "bsort_dist_send_counts",
              "bsort_dist_partition", "bsort_status_string"):
        assert f in fns


def test_library_exports_every_declared_symbol(B):
    from paper_2603_08929_b200 import _lib
    so = ctypes.CDLL(_lib.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(so, f)]
    assert not missing, missing
    # and the binding binds exactly the declared set
    assert sorted(_lib.EXPORTS) == header_functions()
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(bsort_[a-z0-9_]+)$", out, flags=re.M))
    assert set(header_functions()) <= exported


def test_enum_values_match_binding(B):
    from paper_2603_08929_b200 import _lib
    e = header_enums()
    names = ["U8", "I8", "U16", "I16", "U32", "I32", "F32", "U64", "I64", "F64", "F16", "BF16"]
    for i, nm in enumerate(names):
        assert e[f"BSORT_{nm}"] == i == getattr(_lib, nm)
    assert e["BSORT_ASCENDING"] == _lib.ASCENDING and e["BSORT_DESCENDING"] == _lib.DESCENDING
    src = open(HEADER).read()
    assert int(re.search(r"BSORT_DIST_BINS (\d+)", src).group(1)) == _lib.DIST_BINS
    assert int(re.search(r"BSORT_DIST_EXACT (\d+)u", src).group(1)) == _lib.DIST_EXACT
    assert int(re.search(r"BSORT_DIST_FUSED (\d+)u", src).group(1)) == _lib.DIST_FUSED
    assert int(re.search(r"BSORT_PROF_KINDS (\d+)", src).group(1)) == _lib.PROF_KINDS


def test_library_is_sm100a_only():
    so = os.path.join(REPO, "paper_2603_08929_b200", "libbsort.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_argument_errors_return_before_launch(B):
    L = B.lib
    st = L.bsort_sort(99, ctypes.c_void_p(16), 10, 0, None)
    assert st == 2  # unsupported dtype
    assert L.bsort_sort(5, None, 10, 0, None) == 1  # NULL with n > 0
    assert L.bsort_sort(5, ctypes.c_void_p(18), 10, 0, None) == 1  # misaligned for int32
    assert L.bsort_sort(5, ctypes.c_void_p(16), 10, 7, None) == 1  # bad direction
    assert L.bsort_sort(5, None, 0, 0, None) == 0  # n == 0: nothing to do
    assert L.bsort_sort(5, ctypes.c_void_p(16), 1, 0, None) == 0  # n == 1: nothing to do
    assert L.bsort_sort_ws(6, ctypes.c_void_p(256), 1000, 0, ctypes.c_void_p(256), 10, None) == 4
    assert L.bsort_workspace_bytes(5, 0) == 0 and L.bsort_workspace_bytes(5, 1) == 0
    assert L.bsort_workspace_bytes(99, 100) == 0
    assert L.bsort_dist_top_hist(0, ctypes.c_void_p(256), 10, 0, ctypes.c_void_p(256), None) == 2
    assert L.bsort_status_string(4) == b"workspace too small"
    # native distributed sort: argument errors before any NCCL or CUDA call
    assert L.bsort_sort_dist(5, ctypes.c_void_p(256), 10, ctypes.c_void_p(512), 10, None, 0, None, None) == 1
    h = ctypes.c_void_p()
    assert L.bsort_comm_init(ctypes.byref(h), b"\0" * 128, 0, 0) == 1       # nranks < 1
    assert L.bsort_comm_init(ctypes.byref(h), b"\0" * 128, 2, 2) == 1       # rank out of range
    assert L.bsort_comm_init(ctypes.byref(h), b"\0" * 128, 65, 0) == 1      # > BSORT_DIST_MAX_RANKS
    assert L.bsort_comm_destroy(None) == 1
    assert L.bsort_comm_size(None) == 0 and L.bsort_comm_rank(None) == -1
    assert L.bsort_status_string(6) == b"NCCL error"
    assert L.bsort_status_string(7) == b"output capacity too small"


def test_workspace_model(B):
    """LSD: one ping-pong key buffer + small tables + look-back descriptors (32-bit keys from
    2^24 keys: three regions, one per look-back pass, ~8% of the keys); counting: O(2^w)
    counters only."""
    for code, es in ((4, 4), (6, 4), (7, 8), (9, 8)):
        for n in (2, 1000, 1 << 20, (1 << 30) + 3):
            wb = B.lib.bsort_workspace_bytes(code, n)
            assert n * es <= wb <= n * es * (1.09 if es == 4 else 1.07) + (1 << 20)
    for code in (0, 1):
        assert B.lib.bsort_workspace_bytes(code, 1 << 28) == 256 * 8
    assert B.lib.bsort_workspace_bytes(3, 1 << 28) < (64 << 20)


def np_splitters(h, P):
    """Plain restatement of bsort.h's cut rule."""
    total = int(h.sum(dtype=np.uint64))
    pre = np.concatenate([[0], np.cumsum(h.astype(object))])  # pre[b] = sum(h[0..b))
    cuts = [0]
    for r in range(1, P):
        t = (total * r) // P
        b = next(b for b in range(len(h) + 1) if pre[b] >= t)
        cuts.append(b)
    cuts.append(len(h))
    return np.array(cuts, dtype=np.uint32)


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("shape", ["uniform", "skewed", "single", "sparse"])
def test_splitters_match_rule(B, P, shape):
    rng = np.random.default_rng(P * 7 + len(shape))
    h = np.zeros(65536, dtype=np.uint64)
    if shape == "uniform":
        h[:] = rng.integers(0, 100, 65536)
    elif shape == "skewed":
        h[rng.integers(0, 65536, 40)] = rng.integers(1, 10**9, 40).astype(np.uint64)
    elif shape == "single":
        h[12345] = 1 << 33
    else:
        h[[0, 65535]] = [3, 5]
    cuts = B.splitters(h, P)
    if shape != "uniform":  # the object-dtype restatement is slow on 65536 x P; sample it
        assert np.array_equal(cuts, np_splitters(h, P))
    assert cuts[0] == 0 and cuts[-1] == 65536 and np.all(np.diff(cuts.astype(np.int64)) >= 0)
    total = int(h.sum())
    pre = np.concatenate([[0], np.cumsum(h)])
    for r in range(1, P):
        c = int(cuts[r])
        t = total * r // P
        assert pre[c] >= t and (c == 0 or pre[c - 1] < t)
    sc = B.send_counts(h, cuts)
    assert int(sc.sum()) == total
    for q in range(P):
        assert int(sc[q]) == int(h[cuts[q]:cuts[q + 1]].sum())


def test_splitters_reject_bad_args(B):
    from paper_2603_08929_b200 import BsortError
    with pytest.raises(BsortError):
        B.splitters(np.zeros(65536, np.uint64), 0)
    with pytest.raises(BsortError):
        B.send_counts(np.zeros(65536, np.uint64), np.array([0, 7, 3, 65536], np.uint32))


def test_workspace_bytes_monotone_in_n(B):
    """A workspace sized for n serves every m <= n (Sorter, the in-place mode's groups): sizes
    never decrease with n, across the single-CTA bound, the folded look-back range (n < 2^22,
    two look-back regions) and the 2^24 joint-histogram / 2^30 descriptor-width steps."""
    from paper_2603_08929_b200 import _lib
    L = _lib.lib
    probes = sorted({m for e in range(1, 33) for m in ((1 << e) - 1, 1 << e, (1 << e) + 1)} |
                    {20479, 20480, 20481, 10239, 10240, 10241, 148 * 20480 - 1, 148 * 20480, 148 * 20480 + 1,
                     148 * 10240, 148 * 10240 + 1, (1 << 22) - 8193, (1 << 22) - 1})
    for code in (_lib.U8, _lib.I16, _lib.U32, _lib.F32, _lib.I64, _lib.F64):
        prev = 0
        for m in probes:
            w = int(L.bsort_workspace_bytes(code, m))
            assert w >= prev, (code, m, w, prev)
            prev = w
    for code in (_lib.U32, _lib.I64):
        prev = 0
        for m in probes:
            w = int(L.bsort_pairs_workspace_bytes(code, m))
            assert w >= prev, ("pairs", code, m, w, prev)
            prev = w
