"""Full-size parity against the oracle, memcmp of raw bytes, at BASELINE.json's stated sizes.

cfg3 (2^30 f32 keys), cfg4's 16-distinct layout (2^30 i32 keys; the sorted / reverse / all-equal
layouts have known answers, test_gpu_fullsize.py) and cfg2's int16 keys (2^28, both directions)
are sorted on the GPU in bench.py's launch configuration (Sorter) and compared byte for byte
with R1 (oracle/: Algorithms 1-5, single-threaded C) on a host copy of the same input -- the
order of P:609-617 checked exactly, not through invariants.  cfg1 at its full size is in
test_gpu_parity.py.  One more case goes past 2^30 keys (64-bit look-back descriptors and counts),
descending.  The oracle sorts run in host threads (ctypes releases the GIL), all started
when this module starts, so they overlap each other and the GPU work: about the time of the
slowest one (cfg3, a few minutes on one host core)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

NP = {torch.int16: np.int16, torch.int32: np.int32, torch.float32: np.float32}
SIGNED = {torch.int16: torch.int16, torch.int32: torch.int32, torch.float32: torch.int32}

CASES = {
    "cfg3": (lambda: W.make("cfg3", "cuda"), False),
    "cfg4_distinct16": (lambda: W.make("cfg4", "cuda", layout="distinct16"), False),
    "cfg2_i16_asc": (lambda: W.make("cfg2", "cuda", dtype=torch.int16), False),
    "cfg2_i16_desc": (lambda: W.make("cfg2", "cuda", dtype=torch.int16), True),
    # beyond 2^30 keys: the 64-bit look-back descriptors and counts of the LSD path, descending
    "cfg3_2^30+2^20+3_desc": (lambda: W.make("cfg3", "cuda", n=(1 << 30) + (1 << 20) + 3), True),
}


def host(t: torch.Tensor) -> np.ndarray:
    return t.view(SIGNED[t.dtype]).cpu().numpy().view(NP[t.dtype])


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2603_08929_b200 as b
    return b


@pytest.fixture(scope="module")
def oracle_runs(B):
    pool = ThreadPoolExecutor(max_workers=len(CASES))
    futs = {}
    for name, (make, desc) in CASES.items():
        x = make()
        futs[name] = pool.submit(oracle.sort_native, host(x), desc)
        del x
    yield futs
    pool.shutdown(wait=True)


@pytest.mark.parametrize("name", list(CASES))
def test_fullsize_memcmp_vs_oracle(B, oracle_runs, name):
    make, desc = CASES[name]
    x = make()
    s = B.Sorter(x.dtype, x.numel(), x.device)
    s(x, desc)
    torch.cuda.synchronize()
    got = host(x)
    ref = oracle_runs[name].result()
    assert got.size == ref.size
    if got.tobytes() != ref.tobytes():
        bad = np.flatnonzero(got != ref)
        raise AssertionError(f"{name}: {bad.size} mismatching keys, first at {bad[:5]}")
