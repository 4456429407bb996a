"""Multi-process MSD path on CPU: paper_2603_08929_b200.sort_dist's orchestration (histogram
all-reduce, host splitters from libbsort, counts all-to-all, keys all-to-all-v, local sort)
over a world-size-2/3 gloo group.  The three device steps are substituted by CPU stand-ins
written in this test from the oracle's total-order key (DESIGN.md
§Multi-GPU), so the host logic is checked without a GPU.  The concatenated shards must equal
the oracle's sort of all ranks' keys, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

NPD = {torch.int32: np.int32, torch.float32: np.float32, torch.int64: np.int64,
       torch.float64: np.float64, torch.uint32: np.uint32}
UINT = {4: np.uint32, 8: np.uint64}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _enc(arr: np.ndarray, descending: bool) -> np.ndarray:
    """The oracle's total-order key with the direction folded in (np.uint64)."""
    scheme = oracle.NATIVE_SCHEMES[arr.dtype]
    w = scheme.width
    k = oracle.total_order_keys(arr.view(UINT[arr.itemsize]).astype(np.uint64), scheme)
    if descending:
        k = ~k & np.uint64((1 << w) - 1 if w < 64 else 0xFFFFFFFFFFFFFFFF)
    return k


def _enc_top16(arr: np.ndarray, descending: bool) -> np.ndarray:
    w = arr.itemsize * 8
    return (_enc(arr, descending) >> np.uint64(w - 16)).astype(np.int64)


def _classes(t, values, desc):
    k = _enc(t.numpy(), desc)
    v = np.asarray(values, dtype=np.uint64)
    lo = np.searchsorted(v, k, side="left")   # number of values < key
    hi = np.searchsorted(v, k, side="right")
    return 2 * lo + (hi - lo)                 # 2j+1 if key == values[j], else 2 * #{values < key}


def cpu_ops():
    import paper_2603_08929_b200 as B
    from paper_2603_08929_b200.dist import DistOps

    def top_hist(t, desc):
        b = _enc_top16(t.numpy(), desc)
        return torch.from_numpy(np.bincount(b, minlength=65536).astype(np.int64)).view(torch.uint64)

    def partition(t, cuts, counts, desc):
        b = _enc_top16(t.numpy(), desc)
        dest = np.searchsorted(cuts.astype(np.int64), b, side="right") - 1
        order = np.argsort(dest, kind="stable")
        assert np.array_equal(np.bincount(dest, minlength=len(counts)), counts.astype(np.int64))
        return torch.from_numpy(np.ascontiguousarray(t.numpy()[order]))

    def local_sort(t, desc):
        t.copy_(torch.from_numpy(oracle.sort_native(t.numpy(), descending=desc)))
        return t

    def refine_hist(t, prefixes, bits, desc):
        w = t.element_size() * 8
        k = _enc(t.numpy(), desc)
        h = np.zeros((len(prefixes), 65536), dtype=np.int64)
        for j, p in enumerate(prefixes):
            sel = k[(k >> np.uint64(w - bits)) == np.uint64(p)]
            h[j] = np.bincount(((sel >> np.uint64(w - bits - 16)) & np.uint64(0xFFFF)).astype(np.int64),
                               minlength=65536)
        return torch.from_numpy(h).view(torch.uint64)

    def class_hist(t, values, desc):
        c = np.bincount(_classes(t, values, desc), minlength=2 * len(values) + 1)
        return torch.from_numpy(c.astype(np.int64)).view(torch.uint64)

    def partition_classes(t, values, counts, desc):
        cls = _classes(t, values, desc)
        assert np.array_equal(np.bincount(cls, minlength=len(counts)), counts.astype(np.int64))
        return torch.from_numpy(np.ascontiguousarray(t.numpy()[np.argsort(cls, kind="stable")]))

    return DistOps(top_hist=top_hist, splitters=B.splitters, send_counts=B.send_counts,
                   partition=partition, local_sort=local_sort, refine_hist=refine_hist,
                   class_hist=class_hist, partition_classes=partition_classes)


def _make_local(dtype, n, rank, seed, skew):
    rng = np.random.default_rng(seed + 1000 * rank)
    nd = NPD[dtype]
    if skew == "equal":
        a = np.full(n, 7, dtype=nd)
    elif skew == "few":   # heavy duplicates, a handful of distinct keys spanning several bins
        vals = np.array([-5, 0, 3, 3 + (1 << 20), 1 << 24], dtype=np.int64).astype(nd)
        a = vals[rng.integers(0, len(vals), size=n)]
    elif skew == "close":  # distinct keys sharing their top 16 (and for 64-bit, 32) bits
        base = 1 << (np.dtype(nd).itemsize * 8 - 2)
        a = (base + rng.integers(0, 1 << 12, size=n)).astype(nd)
    elif np.dtype(nd).kind == "f":
        a = np.concatenate([rng.standard_normal(n // 2), rng.uniform(-1e6, 1e6, n - n // 2)]).astype(nd)
        a[::97] = -0.0
        a[::101] = np.inf
    else:
        info = np.iinfo(nd)
        a = rng.integers(info.min, info.max, size=n, dtype=nd, endpoint=True)
    return a


def _worker(rank, world, port, dtype, n_per, desc, skew, q, exact=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_08929_b200.dist import sort_dist
        n = n_per + 37 * rank  # uneven shards
        a = _make_local(dtype, n, rank, 5, skew)
        out, st = sort_dist(torch.from_numpy(a.copy()), descending=desc, ops=cpu_ops(),
                            return_stats=True, exact=exact)
        q.put((rank, a, out.numpy().copy(), None if st.cuts is None else st.cuts.copy(),
               st.send_counts.copy(), st.recv_counts.copy(), st.levels))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dtype,desc,skew", [
    (2, torch.int32, False, "random"),
    (2, torch.float32, True, "random"),
    (3, torch.float64, False, "random"),
    (2, torch.int64, True, "random"),
    (2, torch.int32, False, "equal"),
])
def test_sort_dist_gloo(world, dtype, desc, skew):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, 20000, desc, skew, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    inputs = np.concatenate([r[1] for r in res])
    shards = [r[2] for r in res]
    ref = oracle.sort_native(inputs, descending=desc)
    assert np.concatenate(shards).tobytes() == ref.tobytes()
    cuts = res[0][3]
    for r in res:
        assert np.array_equal(r[3], cuts)  # every rank computed the same splitters
    send = np.stack([r[4] for r in res])
    recv = np.stack([r[5] for r in res])
    assert np.array_equal(send.T, recv)  # recv[r][q] == send[q][r]
    assert [len(s) for s in shards] == list(recv.sum(axis=1))
    if skew == "equal":
        assert sum(1 for s in shards if len(s)) == 1  # bin-granular split (reading Q16)


@pytest.mark.parametrize("world,dtype,desc,skew", [
    (2, torch.int32, False, "equal"),
    (3, torch.int64, True, "few"),
    (3, torch.float32, False, "random"),
    (2, torch.int64, False, "close"),
    (3, torch.int32, True, "close"),
])
def test_sort_dist_exact_gloo(world, dtype, desc, skew):
    """§8 N2: every shard holds exactly floor((r+1)N/P) - floor(rN/P) keys, whatever the skew."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_per = 6000
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, n_per, desc, skew, q, True))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    inputs = np.concatenate([r[1] for r in res])
    shards = [r[2] for r in res]
    assert np.concatenate(shards).tobytes() == oracle.sort_native(inputs, descending=desc).tobytes()
    N = len(inputs)
    assert [len(s) for s in shards] == [(r + 1) * N // world - r * N // world for r in range(world)]
    if skew == "close":
        assert res[0][6] >= 1  # the boundaries needed at least one refinement histogram
