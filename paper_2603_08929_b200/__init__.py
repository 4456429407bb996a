"""bsort on B200: the hot path of arxiv 2603.08929 as sm_100a CUDA behind a C ABI.

Thin Python layer over ``include/bsort.h`` (see ``_lib.py``).  PyTorch supplies device memory
(the caching allocator owns every workspace), the current CUDA stream and, for the multi-GPU
path, the process group.  All sorting work runs in ``libbsort.so``.

Public API
----------
``sort_(t, descending=False)``        in-place sort of a contiguous CUDA tensor
``sort(t, descending=False)``         sorted copy
``Sorter(dtype, n, device)``          reusable workspace for repeated sorts (bench / serving)
``sort_dist(t, group=None, ...)``     globally sorted shards over a process group (MSD + a2a)
``profile()``                         per-kernel CUDA-event timing context manager
"""
from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import BsortError, check, lib

__all__ = ["sort_", "sort", "sort_inplace_", "inplace_workspace_bytes", "sort_pairs_", "argsort", "Sorter", "sort_host", "sort_dist", "dtype_code", "workspace_bytes",
           "top_hist", "splitters", "send_counts", "partition", "partition_remote", "refine_hist",
           "class_hist", "partition_classes", "exact_boundaries", "exact_send_counts", "Comm",
           "sort_dist_native", "profile",
           "launch_count", "selftest",
           "BsortError", "version"]

_TORCH_CODES = {
    torch.uint8: _lib.U8, torch.int8: _lib.I8, torch.uint16: _lib.U16, torch.int16: _lib.I16,
    torch.uint32: _lib.U32, torch.int32: _lib.I32, torch.float32: _lib.F32,
    torch.uint64: _lib.U64, torch.int64: _lib.I64, torch.float64: _lib.F64,
    torch.float16: _lib.F16, torch.bfloat16: _lib.BF16,
}


def version() -> str:
    return lib.bsort_version().decode()


def launch_count() -> int:
    """Kernels launched by libbsort.so since it was loaded."""
    return int(lib.bsort_launch_count())


def selftest(device=None) -> int:
    """bsort_selftest on ``device`` (default: current): 0 when the hardware behaviour the fast
    kernels rely on holds there (shared-atomic lane order), else the bitmask of failed checks."""
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        return int(lib.bsort_selftest())


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return _TORCH_CODES[dtype]
    except KeyError:
        raise TypeError(f"bsort: unsupported dtype {dtype}") from None


def workspace_bytes(dtype: torch.dtype, n: int) -> int:
    return int(lib.bsort_workspace_bytes(dtype_code(dtype), n))


_SAME_DEVICE = contextlib.nullcontext()


def _on(device):
    """Context that makes ``device`` current for libbsort's launches and allocations: a no-op
    when it already is (torch.cuda.device's switch costs microseconds per call, which small
    sorts notice)."""
    idx = device.index
    if idx is None or idx == torch._C._cuda_getDevice():
        return _SAME_DEVICE
    return torch.cuda.device(idx)


def _stream_ptr(device) -> ctypes.c_void_p:
    """The current torch stream of ``device`` as a raw cudaStream_t."""
    idx = device.index if device.index is not None else torch._C._cuda_getDevice()
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(idx))


def _check_tensor(t: torch.Tensor):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("bsort: expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("bsort: tensor must be contiguous")


def _workspace(nbytes: int, device) -> torch.Tensor:
    # 256-byte alignment is guaranteed by the caching allocator (512-byte blocks).
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, device=device)


def sort_(t: torch.Tensor, descending: bool = False) -> torch.Tensor:
    """Sort ``t`` in place in the paper's order (bit-exact; -0 < +0, NaNs at the ends)."""
    _check_tensor(t)
    code = dtype_code(t.dtype)
    n = t.numel()
    if n <= 1:
        return t
    wsb = int(lib.bsort_workspace_bytes(code, n))
    ws = _workspace(wsb, t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_sort_ws(code, ctypes.c_void_p(t.data_ptr()), n, int(bool(descending)),
                                ctypes.c_void_p(ws.data_ptr()), wsb, _stream_ptr(t.device)),
              "bsort_sort_ws")
    return t


def sort(t: torch.Tensor, descending: bool = False) -> torch.Tensor:
    return sort_(t.clone(), descending)


def inplace_workspace_bytes(dtype: torch.dtype, n: int, chunk: int = 0) -> int:
    return int(lib.bsort_inplace_workspace_bytes(dtype_code(dtype), n, chunk))


def sort_inplace_(t: torch.Tensor, descending: bool = False, chunk: int = 0) -> torch.Tensor:
    """§8 N4 in-place mode: same result as ``sort_`` with O(n/128 + chunk) scratch instead of n
    keys (256-way in-place MSD partitions, then the LSD path on bucket groups of <= chunk keys;
    chunk=0: max(2^22, n/32)).  Synchronises the host once per partition."""
    _check_tensor(t)
    code = dtype_code(t.dtype)
    n = t.numel()
    if n <= 1:
        return t
    wsb = int(lib.bsort_inplace_workspace_bytes(code, n, chunk))
    ws = _workspace(wsb, t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_sort_inplace_ws(code, ctypes.c_void_p(t.data_ptr()), n, int(bool(descending)), chunk,
                                        ctypes.c_void_p(ws.data_ptr()), wsb, _stream_ptr(t.device)),
              "bsort_sort_inplace_ws")
    return t


def sort_pairs_(keys: torch.Tensor, values: torch.Tensor, descending: bool = False):
    """Key-value sort in place (§8 N3): 32/64-bit keys, int32/uint32 values moved with them.
    Not stable: the values of equal keys come out in unspecified order."""
    _check_tensor(keys)
    _check_tensor(values)
    if values.dtype not in (torch.int32, torch.uint32) or values.numel() != keys.numel():
        raise ValueError("sort_pairs_: values must be int32/uint32 with one value per key")
    code = dtype_code(keys.dtype)
    n = keys.numel()
    if n <= 1:
        return keys, values
    wsb = int(lib.bsort_pairs_workspace_bytes(code, n))
    ws = _workspace(wsb, keys.device)
    with _on(keys.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_sort_pairs_ws(code, ctypes.c_void_p(keys.data_ptr()), ctypes.c_void_p(values.data_ptr()),
                                      n, int(bool(descending)), ctypes.c_void_p(ws.data_ptr()), wsb,
                                      _stream_ptr(keys.device)), "bsort_sort_pairs_ws")
    return keys, values


def argsort(t: torch.Tensor, descending: bool = False):
    """(sorted keys, int32 indices into t) -- the paper's order, like torch.sort(stable=False)."""
    keys = t.clone()
    idx = torch.arange(t.numel(), dtype=torch.int32, device=t.device)
    return sort_pairs_(keys, idx, descending)


class Sorter:
    """Holds a workspace for repeated sorts of up to ``n`` keys of one dtype."""

    def __init__(self, dtype: torch.dtype, n: int, device="cuda"):
        self.dtype = dtype
        self.code = dtype_code(dtype)
        self.n = int(n)
        self.device = torch.device(device)
        self.ws_bytes = int(lib.bsort_workspace_bytes(self.code, self.n))
        self.ws = _workspace(self.ws_bytes, self.device)

    def __call__(self, t: torch.Tensor, descending: bool = False) -> torch.Tensor:
        _check_tensor(t)
        if t.dtype != self.dtype or t.numel() > self.n:
            raise ValueError("Sorter: dtype mismatch or tensor larger than the workspace")
        with _on(t.device):  # launches and allocations on the tensor's GPU
            check(lib.bsort_sort_ws(self.code, ctypes.c_void_p(t.data_ptr()), t.numel(),
                                    int(bool(descending)), ctypes.c_void_p(self.ws.data_ptr()),
                                    self.ws_bytes, _stream_ptr(t.device)), "bsort_sort_ws")
        return t

    def graph(self, t: torch.Tensor, descending: bool = False) -> "torch.cuda.CUDAGraph":
        """Capture the sort of ``t`` (fixed address and size) into a CUDA graph: every launch of
        the path (memsets, histogram, plan, passes, final copy) is a graph node, so a replay
        costs one launch.  ``g.replay()`` re-sorts whatever ``t`` holds at that time."""
        self(t, descending)  # warm-up outside capture (one-time function attributes)
        torch.cuda.synchronize(t.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self(t, descending)
        return g

    def sort_host(self, host: torch.Tensor, dev_buf: torch.Tensor, descending: bool = False):
        """Enqueue H2D(host -> dev_buf), sort, D2H(dev_buf -> host) on the current stream."""
        if host.is_cuda or not host.is_contiguous() or host.dtype != self.dtype:
            raise ValueError("sort_host: need a contiguous host tensor of the Sorter dtype")
        _check_tensor(dev_buf)
        if dev_buf.numel() < host.numel() or host.numel() > self.n:
            raise ValueError("sort_host: device buffer / workspace too small")
        with _on(dev_buf.device):  # launches and allocations on the tensor's GPU
            check(lib.bsort_sort_host(self.code, ctypes.c_void_p(host.data_ptr()), host.numel(),
                                      int(bool(descending)), ctypes.c_void_p(dev_buf.data_ptr()),
                                      ctypes.c_void_p(self.ws.data_ptr()), self.ws_bytes,
                                      _stream_ptr(dev_buf.device)), "bsort_sort_host")
        return host

    def sort_host_to(self, host_in: torch.Tensor, host_out: torch.Tensor, dev_buf: torch.Tensor,
                     descending: bool = False, stream=None):
        """Enqueue H2D(host_in -> dev_buf), sort, D2H(dev_buf -> host_out) on `stream` (default:
        the current stream of dev_buf's device).  host_in is only read, so sorts on different
        streams (each with its own Sorter, dev_buf and host_out) can overlap."""
        for h in (host_in, host_out):
            if h.is_cuda or not h.is_contiguous() or h.dtype != self.dtype:
                raise ValueError("sort_host_to: need contiguous host tensors of the Sorter dtype")
        if host_out.numel() != host_in.numel():
            raise ValueError("sort_host_to: host_in and host_out differ in size")
        _check_tensor(dev_buf)
        if dev_buf.numel() < host_in.numel() or host_in.numel() > self.n:
            raise ValueError("sort_host_to: device buffer / workspace too small")
        sp = ctypes.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(dev_buf.device)
        with _on(dev_buf.device):
            check(lib.bsort_sort_host_to(self.code, ctypes.c_void_p(host_in.data_ptr()),
                                         ctypes.c_void_p(host_out.data_ptr()), host_in.numel(),
                                         int(bool(descending)), ctypes.c_void_p(dev_buf.data_ptr()),
                                         ctypes.c_void_p(self.ws.data_ptr()), self.ws_bytes, sp),
                  "bsort_sort_host_to")
        return host_out


def sort_host(host: torch.Tensor, descending: bool = False, device="cuda") -> torch.Tensor:
    """Sort a (preferably pinned) host tensor through the GPU; returns after completion."""
    s = Sorter(host.dtype, host.numel(), device)
    buf = torch.empty(max(host.numel(), 1), dtype=host.dtype, device=device)
    s.sort_host(host, buf, descending)
    torch.cuda.current_stream(torch.device(device)).synchronize()
    return host


# ---------------------------------------------------------------- MSD building blocks

def top_hist(t: torch.Tensor, descending: bool = False) -> torch.Tensor:
    """uint64[65536] device histogram of the top 16 bits of the transformed keys."""
    _check_tensor(t)
    h = torch.empty(_lib.DIST_BINS, dtype=torch.uint64, device=t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_top_hist(dtype_code(t.dtype), ctypes.c_void_p(t.data_ptr()), t.numel(),
                                      int(bool(descending)), ctypes.c_void_p(h.data_ptr()),
                                      _stream_ptr(t.device)), "bsort_dist_top_hist")
    return h


def _u64p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def splitters(global_hist: np.ndarray, nranks: int) -> np.ndarray:
    """Host: cuts[0..nranks] (uint32) from the global histogram (see bsort.h)."""
    h = np.ascontiguousarray(global_hist, dtype=np.uint64)
    if h.size != _lib.DIST_BINS:
        raise ValueError("histogram must have 65536 bins")
    cuts = np.zeros(nranks + 1, dtype=np.uint32)
    check(lib.bsort_dist_splitters(_u64p(h), nranks, _u32p(cuts)), "bsort_dist_splitters")
    return cuts


def send_counts(local_hist: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(local_hist, dtype=np.uint64)
    c = np.ascontiguousarray(cuts, dtype=np.uint32)
    out = np.zeros(c.size - 1, dtype=np.uint64)
    check(lib.bsort_dist_send_counts(_u64p(h), _u32p(c), c.size - 1, _u64p(out)),
          "bsort_dist_send_counts")
    return out


def partition(t: torch.Tensor, cuts: np.ndarray, counts: np.ndarray,
              descending: bool = False) -> torch.Tensor:
    """Stable partition of ``t`` by destination rank (buckets in rank order)."""
    _check_tensor(t)
    code = dtype_code(t.dtype)
    c = np.ascontiguousarray(cuts, dtype=np.uint32)
    sc = np.ascontiguousarray(counts, dtype=np.uint64)
    nranks = c.size - 1
    out = torch.empty_like(t)
    wsb = int(lib.bsort_dist_partition_workspace_bytes(code, t.numel(), nranks))
    ws = _workspace(wsb, t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_partition(code, ctypes.c_void_p(t.data_ptr()), t.numel(),
                                       int(bool(descending)), _u32p(c), _u64p(sc), nranks,
                                       ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                       wsb, _stream_ptr(t.device)), "bsort_dist_partition")
    return out


def partition_remote(t: torch.Tensor, cuts: np.ndarray, counts: np.ndarray, dst_addrs,
                     descending: bool = False) -> None:
    """Fused partition + exchange (§8 N1): every key of destination q is written straight to
    the device byte range starting at dst_addrs[q] (e.g. a peer rank's symmetric-memory receive
    buffer at this rank's offset); exactly counts[q] keys land there."""
    _check_tensor(t)
    code = dtype_code(t.dtype)
    c = np.ascontiguousarray(cuts, dtype=np.uint32)
    sc = np.ascontiguousarray(counts, dtype=np.uint64)
    da = np.ascontiguousarray(np.asarray(dst_addrs, dtype=np.uint64))
    nranks = c.size - 1
    wsb = int(lib.bsort_dist_partition_workspace_bytes(code, t.numel(), nranks))
    ws = _workspace(wsb, t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_partition_remote(code, ctypes.c_void_p(t.data_ptr()), t.numel(),
                                              int(bool(descending)), _u32p(c), _u64p(sc), nranks,
                                              _u64p(da), ctypes.c_void_p(ws.data_ptr()), wsb,
                                              _stream_ptr(t.device)), "bsort_dist_partition_remote")


def refine_hist(t: torch.Tensor, prefixes, prefix_bits: int, descending: bool = False) -> torch.Tensor:
    """§8 N2: uint64[m, 65536] histogram of the next 16 transformed-key bits of the keys whose
    top ``prefix_bits`` bits equal prefixes[j] (strictly increasing)."""
    _check_tensor(t)
    pre = np.ascontiguousarray(np.asarray(prefixes, dtype=np.uint64))
    h = torch.empty(pre.size * _lib.DIST_BINS, dtype=torch.uint64, device=t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_refine_hist(dtype_code(t.dtype), ctypes.c_void_p(t.data_ptr()), t.numel(),
                                         int(bool(descending)), _u64p(pre), pre.size, int(prefix_bits),
                                         ctypes.c_void_p(h.data_ptr()), _stream_ptr(t.device)), "bsort_dist_refine_hist")
    return h.view(pre.size, _lib.DIST_BINS)


def class_hist(t: torch.Tensor, values, descending: bool = False) -> torch.Tensor:
    """§8 N2: uint64[2m+1] counts of the key classes against the split keys ``values``."""
    _check_tensor(t)
    v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    c = torch.empty(2 * v.size + 1, dtype=torch.uint64, device=t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_class_hist(dtype_code(t.dtype), ctypes.c_void_p(t.data_ptr()), t.numel(),
                                        int(bool(descending)), _u64p(v), v.size, ctypes.c_void_p(c.data_ptr()),
                                        _stream_ptr(t.device)), "bsort_dist_class_hist")
    return c


def partition_classes(t: torch.Tensor, values, class_counts, descending: bool = False) -> torch.Tensor:
    """§8 N2: keys grouped by class (increasing), class c starting at sum(class_counts[:c])."""
    _check_tensor(t)
    v = np.ascontiguousarray(np.asarray(values, dtype=np.uint64))
    cc = np.ascontiguousarray(np.asarray(class_counts, dtype=np.uint64))
    out = torch.empty_like(t)
    if t.numel() == 0:
        return out
    wsb = int(lib.bsort_dist_class_partition_workspace_bytes())
    ws = _workspace(wsb, t.device)
    with _on(t.device):  # launches and allocations on the tensor's GPU
        check(lib.bsort_dist_partition_classes(dtype_code(t.dtype), ctypes.c_void_p(t.data_ptr()), t.numel(),
                                               int(bool(descending)), _u64p(v), v.size, _u64p(cc),
                                               ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()), wsb,
                                               _stream_ptr(t.device)), "bsort_dist_partition_classes")
    return out


class Comm:
    """A library-owned NCCL communicator (bsort_comm_t) for the native distributed sort.

    Collective: every rank of ``group`` (torch.distributed) constructs it with its own device
    current; rank 0's ncclUniqueId is broadcast over ``group``.  ``Comm.local()`` makes a
    one-rank communicator without torch.distributed."""

    def __init__(self, group=None, _rank: int = None, _world: int = None):
        if _world is None:
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
            uid = [None]
            if rank == 0:
                buf = ctypes.create_string_buffer(128)
                check(lib.bsort_get_unique_id(buf), "bsort_get_unique_id")
                uid[0] = buf.raw
            dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            raw = uid[0]
        else:
            rank, world = _rank, _world
            buf = ctypes.create_string_buffer(128)
            check(lib.bsort_get_unique_id(buf), "bsort_get_unique_id")
            raw = buf.raw
        self._h = ctypes.c_void_p()
        check(lib.bsort_comm_init(ctypes.byref(self._h), raw, world, rank), "bsort_comm_init")
        self.rank, self.size = rank, world

    @classmethod
    def local(cls) -> "Comm":
        return cls(_rank=0, _world=1)

    def close(self):
        if self._h:
            check(lib.bsort_comm_destroy(self._h), "bsort_comm_destroy")
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sort_dist_native(t: torch.Tensor, comm: Comm, descending: bool = False,
                     capacity: int = None, exact: bool = False, fused: bool = False) -> torch.Tensor:
    """§8 b ``bsort_sort_dist``: the whole MSD path in one libbsort call over ``comm`` (NCCL).
    Returns this rank's shard (sorted); ``t`` is left intact.  Collective over comm's ranks.
    If some rank's shard exceeds ``capacity`` (default 2 x n_local + 65,536) every rank gets
    BSORT_ERROR_CAPACITY and the call is retried once, collectively, with the exact sizes.
    ``exact``: exact splitting (§8 N2) inside libbsort (bsort_sort_dist_ex, BSORT_DIST_EXACT).
    ``fused``: the partition stores keys straight into the owners' receive buffers over CUDA IPC
    peer mappings (§8 N1, BSORT_DIST_FUSED; ranks on one node); not with ``exact``."""
    _check_tensor(t)
    n = t.numel()
    cap = capacity if capacity is not None else 2 * n + (1 << 16)
    for attempt in range(2):
        out = torch.empty(cap, dtype=t.dtype, device=t.device)
        n_out = ctypes.c_uint64(0)
        with _on(t.device):  # launches and allocations on the tensor's GPU
            st = lib.bsort_sort_dist_ex(dtype_code(t.dtype), ctypes.c_void_p(t.data_ptr()), n,
                                        ctypes.c_void_p(out.data_ptr()), cap, ctypes.byref(n_out),
                                        int(bool(descending)),
                                        (_lib.DIST_EXACT if exact else 0) | (_lib.DIST_FUSED if fused else 0), comm._h,
                                        _stream_ptr(t.device))
        if st == _lib.ERROR_CAPACITY and attempt == 0:
            cap = int(n_out.value)
            continue
        check(st, "bsort_sort_dist_ex")
        return out[:int(n_out.value)]
    raise AssertionError("unreachable")


def exact_boundaries(hg: np.ndarray, nranks: int, key_bits: int, refine):
    """§8 N2 host planning, libbsort's bsort_dist_exact_boundaries (marshalling only): for the
    GLOBAL top-16-bit histogram ``hg`` of keys of ``key_bits`` (32/64) bits, the transformed key
    K_r of global rank floor(r N / nranks) and its quota for every boundary r.  ``refine(prefixes,
    bits)`` returns the GLOBAL uint64[m, 65536] next-16-bit histograms below the prefixes.
    Returns (values np.uint64[m], idx np.int64[nranks-1], quota np.int64[nranks-1], levels)."""
    hg = np.ascontiguousarray(np.asarray(hg, dtype=np.uint64))
    err = []

    @_lib.REFINE_FN
    def _cb(ctx, prefixes, m, bits, out):
        try:
            pre = np.array([int(prefixes[j]) for j in range(m)], dtype=np.uint64)
            h = np.ascontiguousarray(np.asarray(refine(pre, int(bits)), dtype=np.uint64).reshape(-1))
            if h.size != m * _lib.DIST_BINS:
                raise ValueError("refine returned a wrong-sized histogram")
            ctypes.memmove(out, h.ctypes.data, h.nbytes)
            return 0
        except Exception as e:  # reported after the C call returns
            err.append(e)
            return 1

    R = max(nranks - 1, 1)
    values = (ctypes.c_uint64 * R)()
    idx = (ctypes.c_int * R)()
    quota = (ctypes.c_uint64 * R)()
    m = ctypes.c_int(0)
    levels = ctypes.c_int(0)
    st = lib.bsort_dist_exact_boundaries(_u64p(hg), nranks, key_bits, _cb, None, values, ctypes.byref(m), idx,
                                         quota, ctypes.byref(levels))
    if err:
        raise err[0]
    check(st, "bsort_dist_exact_boundaries")
    return (np.array(values[:m.value], dtype=np.uint64), np.array(idx[:nranks - 1], dtype=np.int64),
            np.array(quota[:nranks - 1], dtype=np.int64), int(levels.value))


def exact_send_counts(class_counts_all: np.ndarray, me: int, idx: np.ndarray, quota: np.ndarray) -> np.ndarray:
    """§8 N2: this rank's per-destination send counts over its class-ordered keys, libbsort's
    bsort_dist_exact_send_counts (marshalling only).  ``class_counts_all[q]`` = rank q's 2m+1
    class counts."""
    C = np.ascontiguousarray(np.asarray(class_counts_all, dtype=np.uint64))
    P, ncls = C.shape
    m = (ncls - 1) // 2
    idx_c = (ctypes.c_int * max(P - 1, 1))(*[int(x) for x in idx])
    quo_c = (ctypes.c_uint64 * max(P - 1, 1))(*[int(x) for x in quota])
    out = np.zeros(P, dtype=np.uint64)
    check(lib.bsort_dist_exact_send_counts(_u64p(C), P, m, int(me), idx_c, quo_c, _u64p(out)),
          "bsort_dist_exact_send_counts")
    return out


from .dist import sort_dist  # noqa: E402  (needs the helpers above)


# --------------------------------------------------------------------------- profiling

@contextlib.contextmanager
def profile():
    """Record CUDA events around every libbsort kernel; yields a dict filled on exit with
    {kind: {"ms": total_ms, "launches": count}} (events synchronised at exit)."""
    result: dict = {}
    lib.bsort_profile_enable(1)
    try:
        yield result
    finally:
        ms = (ctypes.c_double * _lib.PROF_KINDS)()
        cnt = (ctypes.c_uint64 * _lib.PROF_KINDS)()
        lib.bsort_profile_read(ms, cnt)
        lib.bsort_profile_enable(0)
        for k in range(_lib.PROF_KINDS):
            if cnt[k]:
                result[lib.bsort_profile_kind_name(k).decode()] = {"ms": ms[k], "launches": int(cnt[k])}
