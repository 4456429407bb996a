"""GPU parity of the MSD building blocks on one B200.

* ``top_hist`` (k_dist_tophist) against the oracle's total-order key, bit for bit.
* ``partition`` (unstable k_onesweep_pass over destination ranks): every bucket holds exactly
  the keys whose top-16-bit bin the splitters assign to it (multiset equality).
* P simulated ranks on one GPU: every device step of ``sort_dist`` runs in libbsort on rank
  slices; only the two collectives are stood in for by in-process tensor ops (there is one GPU
  in this pool, and ranks whose kernels wait on each other must not share a GPU).  The
  concatenated shards must equal the oracle's sort of all keys.
* ``sort_dist`` end to end over a real one-rank NCCL process group, with the NCCL keys
  all-to-all and with the fused partition + exchange of §8 N1 (symmetric memory).
* N1 on one GPU: every virtual rank's ``partition_remote`` writes straight into P owners'
  receive buffers at the offsets the fused path computes (no overrun, exact shards).
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle
import workloads as W

pytestmark = pytest.mark.gpu

NP = {torch.int32: np.int32, torch.float32: np.float32, torch.int64: np.int64,
      torch.float64: np.float64, torch.uint32: np.uint32, torch.uint64: np.uint64}
UINT = {4: np.uint32, 8: np.uint64}
SIGNED = {torch.uint32: torch.int32, torch.uint64: torch.int64}


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2603_08929_b200 as b
    return b


def host(t):
    return t.view(SIGNED.get(t.dtype, t.dtype)).cpu().numpy().view(NP[t.dtype])


def top16_oracle(arr: np.ndarray, descending: bool) -> np.ndarray:
    s = oracle.NATIVE_SCHEMES[arr.dtype]
    k = oracle.total_order_keys(arr.view(UINT[arr.itemsize]).astype(np.uint64), s)
    if descending:
        k = ~k & np.uint64((1 << s.width) - 1 if s.width < 64 else 0xFFFFFFFFFFFFFFFF)
    return (k >> np.uint64(s.width - 16)).astype(np.int64)


def gen(dtype, n, seed):
    if dtype.is_floating_point:
        return W.special_mix(dtype, n, seed, "cuda")
    return W.uniform_int(dtype, n, seed, "cuda")


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint64, torch.float64])
@pytest.mark.parametrize("descending", [False, True])
def test_top_hist(B, dtype, descending):
    for n in (1, 1000, 300_007):
        x = gen(dtype, n, 40 + n)
        h = B.top_hist(x, descending).view(torch.int64).cpu().numpy()
        ref = np.bincount(top16_oracle(host(x), descending), minlength=65536)
        assert np.array_equal(h, ref)


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.int64])
def test_top_hist_skewed(B, dtype):
    """Bins past 0x8000 keys per CTA (the u16 halves drain into the global counts), misaligned
    start, and a few-value input (32-way same-bin atomics)."""
    n = (1 << 22) + 5
    x = torch.full((n,), 3, dtype=dtype, device="cuda")
    x[::7] = 5
    x[1::13] = -2 if dtype.is_signed else 9
    for t in (x, x[1:]):
        h = B.top_hist(t, False).view(torch.int64).cpu().numpy()
        ref = np.bincount(top16_oracle(host(t), False), minlength=65536)
        assert np.array_equal(h, ref)
    y = gen(dtype, (1 << 24) + 3, 99)  # several grid-stride rounds
    h = B.top_hist(y, True).view(torch.int64).cpu().numpy()
    assert np.array_equal(h, np.bincount(top16_oracle(host(y), True), minlength=65536))


@pytest.mark.parametrize("dtype", [torch.int32, torch.float64])
@pytest.mark.parametrize("P", [2, 3, 8])
def test_partition_buckets(B, dtype, P):
    n = 200_003
    x = gen(dtype, n, 7 * P)
    desc = P == 3
    h = B.top_hist(x, desc).view(torch.int64).cpu().numpy().view(np.uint64)
    cuts = B.splitters(h, P)
    sc = B.send_counts(h, cuts)
    out = B.partition(x, cuts, sc, desc)
    torch.cuda.synchronize()
    xs, os_ = host(x), host(out)
    dest = np.searchsorted(cuts.astype(np.int64), top16_oracle(xs, desc), side="right") - 1
    starts = np.concatenate([[0], np.cumsum(sc.astype(np.int64))])
    for q in range(P):
        got = np.sort(os_[starts[q]:starts[q + 1]].view(UINT[xs.itemsize]))
        exp = np.sort(xs[dest == q].view(UINT[xs.itemsize]))
        assert np.array_equal(got, exp), f"bucket {q}"


def simulated_sort_dist(B, parts, descending):
    """sort_dist's data path on one GPU: libbsort kernels per rank slice, collectives as
    in-process tensor ops (all_reduce = sum, all_to_all = slicing + cat)."""
    P = len(parts)
    hl = [B.top_hist(p, descending) for p in parts]
    hg = torch.stack([h.view(torch.int64) for h in hl]).sum(0)  # all_reduce(sum)
    hg_np = hg.cpu().numpy().view(np.uint64)
    cuts = B.splitters(hg_np, P)
    sends = [B.send_counts(h.view(torch.int64).cpu().numpy().view(np.uint64), cuts) for h in hl]
    buckets = [B.partition(p, cuts, sc, descending) for p, sc in zip(parts, sends)]
    offs = [np.concatenate([[0], np.cumsum(sc.astype(np.int64))]) for sc in sends]
    shards = []
    for q in range(P):  # all_to_all: rank q receives bucket q of every rank, in rank order
        recv = torch.cat([buckets[r][int(offs[r][q]):int(offs[r][q + 1])] for r in range(P)])
        B.sort_(recv, descending)
        shards.append(recv)
    return shards


@pytest.mark.parametrize("dtype,P,desc", [(torch.int64, 2, False), (torch.float64, 4, False),
                                          (torch.float32, 8, True), (torch.int32, 3, False)])
def test_simulated_ranks_match_oracle(B, dtype, P, desc):
    n_per = 100_000
    parts = []
    for r in range(P):
        if dtype == torch.float64:
            parts.append(W.make("cfg5", "cuda", n=n_per * P, dtype=torch.float64, rank=r, world=P))
        elif dtype == torch.int64:
            parts.append(W.make("cfg5", "cuda", n=n_per * P, dtype=torch.int64, rank=r, world=P))
        else:
            parts.append(gen(dtype, n_per + 13 * r, 90 + r))
    allkeys = np.concatenate([host(p) for p in parts])
    shards = simulated_sort_dist(B, parts, desc)
    torch.cuda.synchronize()
    got = np.concatenate([host(s) for s in shards])
    assert got.tobytes() == oracle.sort_native(allkeys, descending=desc).tobytes()
    if dtype in (torch.int64, torch.float64):  # bit-uniform keys split evenly (SV-7)
        sizes = [s.numel() for s in shards]
        assert max(sizes) <= 1.05 * (n_per * P / P)


def test_simulated_ranks_all_equal(B):
    parts = [torch.full((50_000,), 7, dtype=torch.int32, device="cuda") for _ in range(4)]
    shards = simulated_sort_dist(B, parts, False)
    sizes = [s.numel() for s in shards]
    assert sorted(sizes) == [0, 0, 0, 200_000]  # bin-granular split (reading Q16)
    assert bool((torch.cat(shards) == 7).all())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_sort_dist_nccl_one_rank(B):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        x = W.make("cfg5", "cuda", n=300_001, dtype=torch.float64)
        ref = oracle.sort_native(host(x))
        out = B.sort_dist(x)
        torch.cuda.synchronize()
        assert host(out).tobytes() == ref.tobytes()
    finally:
        dist.destroy_process_group()


def simulated_fused(B, parts, descending):
    """§8 N1 on one GPU: each virtual rank's partition_remote writes its keys straight into the
    P owners' receive buffers (here ordinary allocations on the same GPU; on a multi-GPU box the
    same addresses are peer-mapped symmetric memory).  Offsets as _fused_exchange computes them."""
    P = len(parts)
    hl = [B.top_hist(p, descending) for p in parts]
    hg_np = torch.stack([h.view(torch.int64) for h in hl]).sum(0).cpu().numpy().view(np.uint64)
    cuts = B.splitters(hg_np, P)
    send = np.stack([B.send_counts(h.view(torch.int64).cpu().numpy().view(np.uint64), cuts)
                     for h in hl]).astype(np.int64)          # send[r][q]
    recv_tot = send.sum(0)
    bufs = [torch.full((int(recv_tot[q]) + 5,), -1, dtype=torch.int64 if parts[0].element_size() == 8
                       else torch.int32, device="cuda").view(parts[0].dtype) for q in range(P)]
    es = parts[0].element_size()
    for r in range(P):
        start = send[:r].sum(0)                               # r's first slot in each owner
        dst = [bufs[q].data_ptr() + int(start[q]) * es for q in range(P)]
        B.partition_remote(parts[r], cuts, send[r].astype(np.uint64), dst, descending)
    torch.cuda.synchronize()
    shards = []
    for q in range(P):
        tail = bufs[q][int(recv_tot[q]):]
        assert bool((tail.view(torch.int64 if es == 8 else torch.int32) == -1).all())  # no overrun
        shard = bufs[q][:int(recv_tot[q])].clone()
        B.sort_(shard, descending)
        shards.append(shard)
    return shards


@pytest.mark.parametrize("dtype,P,desc", [(torch.float64, 4, False), (torch.int32, 3, True),
                                          (torch.float32, 8, False), (torch.uint64, 2, True)])
def test_fused_partition_exchange_simulated(B, dtype, P, desc):
    parts = [gen(dtype, 70_000 + 17 * r, 200 + r) for r in range(P)]
    allkeys = np.concatenate([host(p) for p in parts])
    shards = simulated_fused(B, parts, desc)
    got = np.concatenate([host(s) for s in shards])
    assert got.tobytes() == oracle.sort_native(allkeys, descending=desc).tobytes()


def test_sort_dist_fused_nccl_one_rank(B):
    """sort_dist(fused=True): symmetric-memory receive buffer, partition_remote, local sort."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        for seed in (1, 2):  # second call reuses the cached symmetric buffer
            x = W.make("cfg5", "cuda", n=200_001 + seed, dtype=torch.float64)
            ref = oracle.sort_native(host(x))
            out = B.sort_dist(x, fused=True)
            torch.cuda.synchronize()
            assert host(out).tobytes() == ref.tobytes()
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ §8 N2 exact splitting

def enc_oracle(arr: np.ndarray, descending: bool) -> np.ndarray:
    """The oracle's total-order key, direction folded in (np.uint64)."""
    s = oracle.NATIVE_SCHEMES[arr.dtype]
    k = oracle.total_order_keys(arr.view(UINT[arr.itemsize]).astype(np.uint64), s)
    if descending:
        k = ~k & np.uint64((1 << s.width) - 1 if s.width < 64 else 0xFFFFFFFFFFFFFFFF)
    return k


def classes_oracle(k: np.ndarray, values: np.ndarray) -> np.ndarray:
    lo = np.searchsorted(values, k, side="left")
    hi = np.searchsorted(values, k, side="right")
    return 2 * lo + (hi - lo)


def clustered(dtype, n, seed):
    """Keys sharing their top bits (so boundaries need refinement) with heavy duplicates."""
    g = torch.Generator().manual_seed(seed)
    w = torch.empty(0, dtype=dtype).element_size() * 8
    idt = torch.int64 if w == 64 else torch.int32
    low = torch.randint(0, 1 << 10, (n,), generator=g, dtype=torch.int64)
    base = (0x1234 << (w - 20)) if w == 32 else (0x123456789 << 28)
    x = (low + base).to(idt)
    x[::3] = base + 77  # one heavily repeated key
    return x.view(dtype).cuda()


@pytest.mark.parametrize("dtype", [torch.int32, torch.float32, torch.uint64, torch.float64])
@pytest.mark.parametrize("descending", [False, True])
def test_refine_and_class_hist(B, dtype, descending):
    n = 250_011
    x = gen(dtype, n, 61) if dtype.is_floating_point else clustered(dtype, n, 61)
    k = enc_oracle(host(x), descending)
    w = x.element_size() * 8
    # refine below the two most populated 16-bit prefixes
    top = (k >> np.uint64(w - 16)).astype(np.int64)
    pre = np.sort(np.argsort(np.bincount(top, minlength=65536))[-2:]).astype(np.uint64)
    for bits in range(16, w, 16):
        if bits > 16:
            pre = np.unique(k >> np.uint64(w - bits))[:3]
        h = B.refine_hist(x, pre, bits, descending).view(torch.int64).cpu().numpy()
        for j, p in enumerate(pre):
            sel = k[(k >> np.uint64(w - bits)) == p]
            ref = np.bincount(((sel >> np.uint64(w - bits - 16)) & np.uint64(0xFFFF)).astype(np.int64),
                              minlength=65536)
            assert np.array_equal(h[j], ref), (bits, j)
    vals = np.unique(k[:: n // 5])[:6]
    vals = np.sort(np.concatenate([vals, vals[:1] + np.uint64(1)]))
    vals = np.unique(vals)
    c = B.class_hist(x, vals, descending).view(torch.int64).cpu().numpy()
    assert np.array_equal(c, np.bincount(classes_oracle(k, vals), minlength=2 * len(vals) + 1))
    out = B.partition_classes(x, vals, c.astype(np.uint64), descending)
    torch.cuda.synchronize()
    ko = enc_oracle(host(out), descending)
    cls = classes_oracle(ko, vals)
    assert (np.diff(cls) >= 0).all()  # grouped by class, increasing
    assert np.array_equal(np.sort(ko), np.sort(k))


def simulated_exact(B, parts, descending):
    """sort_dist(exact=True) on one GPU: kernels per virtual rank, collectives as tensor ops."""
    from paper_2603_08929_b200 import exact_boundaries, exact_send_counts  # libbsort planning
    P = len(parts)
    w = parts[0].element_size() * 8
    hg = sum(B.top_hist(p, descending).view(torch.int64).cpu().numpy() for p in parts).view(np.uint64)

    def refine(prefixes, bits):
        return sum(B.refine_hist(p, prefixes, bits, descending).view(torch.int64).cpu().numpy()
                   for p in parts).view(np.uint64)

    values, idx, quota, levels = exact_boundaries(hg, P, w, refine)
    C = np.stack([B.class_hist(p, values, descending).view(torch.int64).cpu().numpy() for p in parts])
    sends = [exact_send_counts(C, r, idx, quota).astype(np.int64) for r in range(P)]
    buckets = [B.partition_classes(p, values, C[r].astype(np.uint64), descending) for r, p in enumerate(parts)]
    offs = [np.concatenate([[0], np.cumsum(sc)]) for sc in sends]
    shards = []
    for q in range(P):
        recv = torch.cat([buckets[r][int(offs[r][q]):int(offs[r][q + 1])] for r in range(P)])
        B.sort_(recv, descending)
        shards.append(recv)
    return shards, levels


@pytest.mark.parametrize("dtype,P,desc,kind", [
    (torch.int32, 4, False, "equal"), (torch.float64, 3, True, "clustered"),
    (torch.uint64, 8, False, "clustered"), (torch.float32, 5, False, "random"),
    (torch.int64, 2, True, "random")])
def test_simulated_exact_split(B, dtype, P, desc, kind):
    parts = []
    for r in range(P):
        n = 60_000 + 101 * r
        if kind == "equal":
            parts.append(torch.full((n,), 7, dtype=dtype, device="cuda"))
        elif kind == "clustered":
            parts.append(clustered(dtype, n, 300 + r) if not dtype.is_floating_point else
                         clustered(torch.int64 if dtype == torch.float64 else torch.int32, n, 300 + r).view(dtype))
        else:
            parts.append(gen(dtype, n, 300 + r))
    allkeys = np.concatenate([host(p) for p in parts])
    shards, levels = simulated_exact(B, parts, desc)
    torch.cuda.synchronize()
    N = len(allkeys)
    assert [s.numel() for s in shards] == [(q + 1) * N // P - q * N // P for q in range(P)]
    got = np.concatenate([host(s) for s in shards])
    assert got.tobytes() == oracle.sort_native(allkeys, descending=desc).tobytes()
    if kind == "clustered":
        assert levels >= 1


def test_sort_dist_exact_nccl_one_rank(B):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        x = W.make("cfg5", "cuda", n=100_003, dtype=torch.float64)
        ref = oracle.sort_native(host(x))
        out = B.sort_dist(x, exact=True)
        torch.cuda.synchronize()
        assert host(out).tobytes() == ref.tobytes()
    finally:
        dist.destroy_process_group()


# ------------------------------------------------- §8 b native bsort_sort_dist over NCCL

@pytest.mark.parametrize("dtype,desc", [(torch.float64, False), (torch.int32, True),
                                        (torch.uint64, False), (torch.float32, True)])
def test_sort_dist_native_local_comm(B, dtype, desc):
    """bsort_comm_init (one rank, no torch.distributed) + bsort_sort_dist: the whole MSD path in
    libbsort (histogram, NCCL all-reduce / all-gather / send-recv, partition, local sort)."""
    comm = B.Comm.local()
    try:
        for n in (0, 1, 5000, 300_007):
            x = gen(dtype, n, 500 + n)
            before = x.clone()
            out = B.sort_dist_native(x, comm, desc, exact=(n % 2 == 1))  # both entry modes
            torch.cuda.synchronize()
            assert host(out).tobytes() == oracle.sort_native(host(before), descending=desc).tobytes()
            assert host(x).tobytes() == host(before).tobytes()  # dev_in left intact (bitwise)
    finally:
        comm.close()


def test_sort_dist_native_capacity(B):
    import ctypes
    comm = B.Comm.local()
    try:
        x = gen(torch.int64, 10_000, 77)
        out = torch.empty(100, dtype=torch.int64, device="cuda")
        n_out = ctypes.c_uint64(0)
        st = B.lib.bsort_sort_dist(8, ctypes.c_void_p(x.data_ptr()), x.numel(), ctypes.c_void_p(out.data_ptr()),
                                   100, ctypes.byref(n_out), 0, comm._h, None)
        torch.cuda.synchronize()
        assert st == 7 and n_out.value == 10_000
        got = B.sort_dist_native(x, comm, capacity=100)  # retried with the exact size
        torch.cuda.synchronize()
        assert host(got).tobytes() == oracle.sort_native(host(x)).tobytes()
        assert B.lib.bsort_sort_dist(3, ctypes.c_void_p(x.data_ptr()), 10, ctypes.c_void_p(out.data_ptr()),
                                     100, None, 0, comm._h, None) == 2  # i16: unsupported here
        assert B.lib.bsort_sort_dist_ex(8, ctypes.c_void_p(x.data_ptr()), 10, ctypes.c_void_p(out.data_ptr()),
                                        100, None, 0, 4, comm._h, None) == 1  # unknown flag
        assert B.lib.bsort_sort_dist_ex(8, ctypes.c_void_p(x.data_ptr()), 10, ctypes.c_void_p(out.data_ptr()),
                                        100, None, 0, 3, comm._h, None) == 1  # EXACT | FUSED
    finally:
        comm.close()


@pytest.mark.parametrize("dtype,desc", [(torch.float64, False), (torch.int32, True), (torch.uint32, False),
                                        (torch.int64, True)])
def test_sort_dist_native_fused_local_comm(B, dtype, desc):
    """bsort_sort_dist_ex(BSORT_DIST_FUSED) over a one-rank communicator: the partition writes
    into the communicator's receive buffer (the rank's own entry of the peer table), two
    device-side barriers on the signal pads, local sort, copy to dev_out.  Sizes grow across
    calls (the receive buffer is re-allocated) and shrink again (reused)."""
    comm = B.Comm.local()
    try:
        for n in (0, 1, 5000, 300_007, (1 << 20) + 3, 70_001):
            x = gen(dtype, n, 900 + n)
            before = x.clone()
            out = B.sort_dist_native(x, comm, desc, fused=True)
            torch.cuda.synchronize()
            assert host(out).tobytes() == oracle.sort_native(host(before), descending=desc).tobytes(), n
            assert host(x).tobytes() == host(before).tobytes()
    finally:
        comm.close()


def test_sort_dist_native_torch_group(B):
    """Comm over a torch.distributed group (unique id broadcast by the group)."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        comm = B.Comm()
        x = W.make("cfg5", "cuda", n=200_001, dtype=torch.float64)
        out = B.sort_dist_native(x, comm)
        torch.cuda.synchronize()
        assert host(out).tobytes() == oracle.sort_native(host(x)).tobytes()
        comm.close()
    finally:
        dist.destroy_process_group()
