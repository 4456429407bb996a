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

``ops`` lets the host-side orchestration run without a GPU (CPU/gloo tests substitute the
three device steps); the product default is the CUDA path and nothing else.
"""
from __future__ import annotations

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


def cuda_ops() -> DistOps:
    from . import partition, send_counts, sort_, splitters, top_hist
    return DistOps(top_hist=top_hist, splitters=splitters, send_counts=send_counts,
                   partition=partition, local_sort=sort_)


@dataclass
class DistStats:
    cuts: np.ndarray
    send_counts: np.ndarray
    recv_counts: np.ndarray


def sort_dist(t: torch.Tensor, group=None, descending: bool = False,
              ops: Optional[DistOps] = None, return_stats: bool = False,
              a2a_events: Optional[list] = None):
    """Globally sort the keys held by all ranks of ``group``; returns this rank's shard.

    ``t`` (1-D, contiguous) may be clobbered.  The concatenation of the returned shards over
    ranks 0..P-1 is the sorted sequence of all keys, in the requested direction.
    ``a2a_events``: if a list is given (CUDA tensors only), a pair of timing events recorded
    around the keys all-to-all on the current stream is appended to it."""
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
