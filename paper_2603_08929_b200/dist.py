"""Multi-GPU bsort (§8 rows a7-a11): MSD range partition + one all-to-all + local LSD sort.

Per rank (one process per GPU, torch.distributed over NCCL):

  a7  ``top_hist``      histogram of the top 16 bits of the transformed key (libbsort kernel)
      all_reduce(sum)   global histogram (NCCL, 512 KiB)
  a8  ``splitters``     cuts from the global histogram; ``send_counts`` per destination
      (host C in libbsort; the one host sync of the path is the D2H of the two histograms)
      all_to_all        per-destination counts
  a9  ``partition``     P-way partition by destination (libbsort one-sweep pass kernel, unstable:
                        order inside a bucket is irrelevant, every rank sorts what it receives)
  a10 all_to_all_v      keys to their owners (NCCL over NVLink / NVSwitch)
  a11 ``sort_``         local one-sweep LSD sort of the received keys

The top bits of the transformed key are its most significant bits in the paper's order
(sign -> exponent -> mantissa; direction folded in), so rank r's keys all precede
rank r+1's and the concatenation over ranks is the global order.  Shard sizes are
bin-granular (reading Q16).

``fused=True`` (or env BSORT_FUSED_A2A=1) replaces a9 + a10 by the fused partition + exchange
of §8 N1: every rank's receive buffer is torch symmetric memory, each rank learns where its
keys start in every owner's buffer (one more tiny all-to-all), and ``partition_remote`` writes
each key straight into the owner's buffer over NVLink (st.global to peer-mapped addresses) --
no local bucketed copy, no NCCL keys all-to-all.  A barrier after the kernels precedes the
local sort.

``ops`` lets the host-side orchestration run without a GPU (CPU/gloo tests substitute the
three device steps); the product default is the CUDA path and nothing else.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


@dataclass
class DistOps:
    top_hist: Callable        # (tensor, descending) -> uint64[65536] tensor on the tensor's device
    splitters: Callable       # (np.uint64[65536], nranks) -> np.uint32[nranks+1]
    send_counts: Callable     # (np.uint64[65536], cuts) -> np.uint64[nranks]
    partition: Callable       # (tensor, cuts, counts, descending) -> tensor (bucketed)
    local_sort: Callable      # (tensor, descending) -> tensor sorted in place
    # exact splitting (§8 N2)
    refine_hist: Optional[Callable] = None        # (tensor, prefixes, prefix_bits, desc) -> u64[m, 65536]
    class_hist: Optional[Callable] = None         # (tensor, values, desc) -> u64[2m+1]
    partition_classes: Optional[Callable] = None  # (tensor, values, class_counts, desc) -> tensor


def cuda_ops() -> DistOps:
    from . import (class_hist, partition, partition_classes, refine_hist, send_counts, sort_,
                   splitters, top_hist)
    return DistOps(top_hist=top_hist, splitters=splitters, send_counts=send_counts,
                   partition=partition, local_sort=sort_, refine_hist=refine_hist,
                   class_hist=class_hist, partition_classes=partition_classes)


@dataclass
class DistStats:
    cuts: Optional[np.ndarray]
    send_counts: np.ndarray
    recv_counts: np.ndarray
    values: Optional[np.ndarray] = None   # exact mode: the distinct split keys (transformed)
    quota: Optional[np.ndarray] = None    # exact mode: per boundary, equal keys sent left
    levels: int = 0                       # exact mode: refinement histograms taken


_SYMM = {}  # (group name, dtype, device) -> (buffer, handle): receive buffers of the fused path


def _symm_buffer(cap: int, dtype: torch.dtype, device, group):
    """Symmetric-memory receive buffer of at least ``cap`` keys, shared across calls (grown
    collectively when a call needs more; every rank passes the same all-reduced ``cap``)."""
    import torch.distributed._symmetric_memory as symm_mem
    pg = group if group is not None else dist.group.WORLD
    key = (pg.group_name, dtype, str(device))
    hit = _SYMM.get(key)
    if hit is None or hit[0].numel() < cap:
        buf = symm_mem.empty(max(cap, 1), dtype=dtype, device=device)
        handle = symm_mem.rendezvous(buf, pg)
        hit = (buf, handle)
        _SYMM[key] = hit
    return hit


def fused_default() -> bool:
    return os.environ.get("BSORT_FUSED_A2A", "0") == "1"


def sort_dist(t: torch.Tensor, group=None, descending: bool = False,
              ops: Optional[DistOps] = None, return_stats: bool = False,
              a2a_events: Optional[list] = None, fused: Optional[bool] = None,
              exact: bool = False):
    """Globally sort the keys held by all ranks of ``group``; returns this rank's shard.

    ``t`` (1-D, contiguous) may be clobbered.  The concatenation of the returned shards over
    ranks 0..P-1 is the sorted sequence of all keys, in the requested direction.
    ``a2a_events``: if a list is given (CUDA tensors only), a pair of timing events recorded
    around the keys all-to-all on the current stream is appended to it.
    ``fused``: partition straight into the owners' symmetric-memory buffers (§8 N1); the
    returned shard is then a view of the group's receive buffer, valid until the next fused
    ``sort_dist`` call on the same group, dtype and device.
    ``exact``: exact splitting (§8 N2) -- rank r receives exactly floor((r+1)N/P) - floor(rN/P)
    keys whatever the key distribution (one refinement histogram per 16 further key bits a
    boundary needs, plus a class histogram); default is the bin-granular split (reading Q16)."""
    if exact:
        return _sort_dist_exact(t, group, descending, ops or cuda_ops(), return_stats, a2a_events)
    if fused is None:
        fused = fused_default() and ops is None and t.is_cuda
    ops = ops or cuda_ops()
    P = dist.get_world_size(group)
    hl = ops.top_hist(t, descending)
    hg = hl.clone()
    dist.all_reduce(hg.view(torch.int64), op=dist.ReduceOp.SUM, group=group)
    hl_np = hl.view(torch.int64).cpu().numpy().view(np.uint64)
    hg_np = hg.view(torch.int64).cpu().numpy().view(np.uint64)
    cuts = ops.splitters(hg_np, P)
    sc = ops.send_counts(hl_np, cuts)
    send = torch.from_numpy(sc.astype(np.int64)).to(t.device)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    rc = recv.cpu().numpy().astype(np.int64)
    if fused:
        out = _fused_exchange(t, cuts, sc, rc, descending, group, a2a_events)
        ops.local_sort(out, descending)
        if return_stats:
            return out, DistStats(cuts=cuts, send_counts=sc, recv_counts=rc.astype(np.uint64))
        return out
    bucketed = ops.partition(t, cuts, sc, descending)
    es = t.element_size()
    out = torch.empty(int(rc.sum()), dtype=t.dtype, device=t.device)
    ev = None
    if a2a_events is not None and t.is_cuda:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    dist.all_to_all_single(out.view(torch.uint8), bucketed.view(torch.uint8),
                           output_split_sizes=[int(c) * es for c in rc],
                           input_split_sizes=[int(c) * es for c in sc], group=group)
    if ev is not None:
        ev[1].record()
        a2a_events.append((ev, int(sc.sum() - sc[dist.get_rank(group)]) * es))
    ops.local_sort(out, descending)
    if return_stats:
        return out, DistStats(cuts=cuts, send_counts=sc, recv_counts=rc.astype(np.uint64))
    return out


def _fused_exchange(t, cuts, sc, rc, descending, group, a2a_events=None):
    """§8 N1: partition every key straight into its owner's receive buffer (peer memory)."""
    from . import partition_remote
    P = dist.get_world_size(group)
    es = t.element_size()
    n_out = int(rc.sum())
    # Owner q stores its sources in rank order: source r's keys start at sum_{r' < r} rc_q[r'].
    starts = torch.from_numpy(np.concatenate([[0], np.cumsum(rc)[:-1]]).astype(np.int64)).to(t.device)
    mine = torch.empty_like(starts)
    dist.all_to_all_single(mine, starts, group=group)  # mine[q]: my first slot in q's buffer
    cap = torch.tensor([n_out], dtype=torch.int64, device=t.device)
    dist.all_reduce(cap, op=dist.ReduceOp.MAX, group=group)
    buf, handle = _symm_buffer(int(cap.item()), t.dtype, t.device, group)
    ptrs = handle.buffer_ptrs
    mine_h = mine.cpu().numpy()
    dst = np.array([int(ptrs[q]) + int(mine_h[q]) * es for q in range(P)], dtype=np.uint64)
    ev = None
    if a2a_events is not None:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    dist.barrier(group=group)  # every owner finished reading its buffer from the previous call
    partition_remote(t, cuts, sc, dst, descending)
    torch.cuda.current_stream(t.device).synchronize()
    dist.barrier(group=group)  # every rank's writes into my buffer have landed
    if ev is not None:
        ev[1].record()
        me = dist.get_rank(group)
        a2a_events.append((ev, int(sc.sum() - sc[me]) * es))
    return buf[:n_out]


def _u64_allreduce(x: torch.Tensor, group) -> np.ndarray:
    y = x.contiguous().view(torch.int64).clone()
    dist.all_reduce(y, op=dist.ReduceOp.SUM, group=group)
    return y.cpu().numpy().view(np.uint64)


def _keys_all_to_all(t, bucketed, sc, group, a2a_events):
    rc_t = torch.empty(len(sc), dtype=torch.int64, device=t.device)
    dist.all_to_all_single(rc_t, torch.from_numpy(sc.astype(np.int64)).to(t.device), group=group)
    rc = rc_t.cpu().numpy().astype(np.int64)
    es = t.element_size()
    out = torch.empty(int(rc.sum()), dtype=t.dtype, device=t.device)
    ev = None
    if a2a_events is not None and t.is_cuda:
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record()
    dist.all_to_all_single(out.view(torch.uint8), bucketed.view(torch.uint8),
                           output_split_sizes=[int(c) * es for c in rc],
                           input_split_sizes=[int(c) * es for c in sc], group=group)
    if ev is not None:
        ev[1].record()
        a2a_events.append((ev, int(sc.sum() - sc[dist.get_rank(group)]) * es))
    return out, rc


def _sort_dist_exact(t, group, descending, ops, return_stats, a2a_events):
    """§8 N2: exact splitters by histogram refinement, class partition, one keys all-to-all."""
    if ops.refine_hist is None or ops.class_hist is None or ops.partition_classes is None:
        raise ValueError("exact splitting needs refine_hist, class_hist and partition_classes ops")
    P = dist.get_world_size(group)
    me = dist.get_rank(group)
    width = t.element_size() * 8
    hg = _u64_allreduce(ops.top_hist(t, descending), group)
    N = int(hg.astype(np.int64).sum())

    def done(out, sc, rc, values=None, quota=None, levels=0):
        ops.local_sort(out, descending)
        if return_stats:
            return out, DistStats(cuts=None, send_counts=sc, recv_counts=rc.astype(np.uint64),
                                  values=values, quota=quota, levels=levels)
        return out

    if P == 1 or N == 0:
        sc = np.zeros(P, dtype=np.uint64)
        sc[me] = t.numel()
        return done(t, sc, sc.astype(np.int64))

    def refine(prefixes, bits):
        return _u64_allreduce(ops.refine_hist(t, prefixes, bits, descending), group).reshape(len(prefixes), -1)

    from . import exact_boundaries, exact_send_counts  # libbsort's C++ planning (marshalling only)
    values, idx, quota, levels = exact_boundaries(hg, P, width, refine)
    cc = ops.class_hist(t, values, descending)
    cc_all = [torch.empty_like(cc.view(torch.int64)) for _ in range(P)]
    dist.all_gather(cc_all, cc.view(torch.int64).contiguous(), group=group)
    C = np.stack([c.cpu().numpy() for c in cc_all]).astype(np.int64)
    sc = exact_send_counts(C, me, idx, quota)
    bucketed = ops.partition_classes(t, values, C[me].astype(np.uint64), descending)
    out, rc = _keys_all_to_all(t, bucketed, sc, group, a2a_events)
    return done(out, sc, rc, values, quota, levels)
