"""ctypes binding of include/bsort.h (argument marshalling only).

Every step of the sort runs in ``libbsort.so`` (sm_100a CUDA).  There is no fallback: if the
library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BSORT_LIB: an alternative build of the same library (experiments); default the in-tree one
LIB_PATH = os.environ.get("BSORT_LIB") or os.path.join(_HERE, "libbsort.so")

# bsort_dtype_t
U8, I8, U16, I16, U32, I32, F32, U64, I64, F64, F16, BF16 = range(12)
DTYPE_NAMES = ["u8", "i8", "u16", "i16", "u32", "i32", "f32", "u64", "i64", "f64", "f16", "bf16"]
DTYPE_BYTES = [1, 1, 2, 2, 4, 4, 4, 8, 8, 8, 2, 2]
ASCENDING, DESCENDING = 0, 1
DIST_BINS = 65536
DIST_MAX_RANKS = 64
PROF_KINDS = 13

SUCCESS = 0
ERROR_NCCL = 6
ERROR_CAPACITY = 7

EXPORTS = [
    "bsort_workspace_bytes", "bsort_sort", "bsort_sort_ws", "bsort_sort_host", "bsort_sort_host_to",
    "bsort_pairs_workspace_bytes", "bsort_sort_pairs_ws", "bsort_sort_pairs",
    "bsort_inplace_workspace_bytes", "bsort_sort_inplace_ws",
    "bsort_dist_top_hist", "bsort_dist_splitters", "bsort_dist_send_counts",
    "bsort_dist_partition_workspace_bytes", "bsort_dist_partition", "bsort_dist_partition_remote",
    "bsort_dist_refine_hist", "bsort_dist_class_hist", "bsort_dist_class_partition_workspace_bytes",
    "bsort_dist_partition_classes",
    "bsort_get_unique_id", "bsort_comm_init", "bsort_comm_destroy", "bsort_comm_size", "bsort_comm_rank",
    "bsort_sort_dist", "bsort_sort_dist_ex", "bsort_last_nccl_error",
    "bsort_dist_exact_boundaries", "bsort_dist_exact_send_counts",
    "bsort_status_string", "bsort_last_cuda_error", "bsort_version", "bsort_launch_count",
    "bsort_selftest", "bsort_profile_enable", "bsort_profile_read", "bsort_profile_kind_name",
]


# bsort_refine_fn: int (*)(void* ctx, const uint64_t* prefixes, int m, int prefix_bits, uint64_t* hist)
REFINE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_int,
                             ctypes.c_int, ctypes.POINTER(ctypes.c_uint64))
DIST_EXACT = 1
DIST_FUSED = 2


class BsortError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib.bsort_status_string(status).decode()
        extra = ""
        if status == 5:
            extra = f" (cudaError {lib.bsort_last_cuda_error()})"
        elif status == 6:
            extra = f" (ncclResult {lib.bsort_last_nccl_error()})"
        super().__init__(f"{where}: {msg}{extra}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"bsort CUDA library not built: {LIB_PATH} missing (run `make lib` or "
            "`python -c 'import __graft_entry__ as g; g.build()'`)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, sz, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_size_t, ctypes.c_int
    u64p = ctypes.POINTER(ctypes.c_uint64)
    u32p = ctypes.POINTER(ctypes.c_uint32)
    i32p = ctypes.POINTER(ctypes.c_int)
    sig = {
        "bsort_workspace_bytes": (sz, [i32, u64]),
        "bsort_sort": (i32, [i32, vp, u64, i32, vp]),
        "bsort_sort_ws": (i32, [i32, vp, u64, i32, vp, sz, vp]),
        "bsort_sort_host": (i32, [i32, vp, u64, i32, vp, vp, sz, vp]),
        "bsort_sort_host_to": (i32, [i32, vp, vp, u64, i32, vp, vp, sz, vp]),
        "bsort_pairs_workspace_bytes": (sz, [i32, u64]),
        "bsort_sort_pairs_ws": (i32, [i32, vp, vp, u64, i32, vp, sz, vp]),
        "bsort_sort_pairs": (i32, [i32, vp, vp, u64, i32, vp]),
        "bsort_inplace_workspace_bytes": (sz, [i32, u64, u64]),
        "bsort_sort_inplace_ws": (i32, [i32, vp, u64, i32, u64, vp, sz, vp]),
        "bsort_dist_top_hist": (i32, [i32, vp, u64, i32, vp, vp]),
        "bsort_dist_splitters": (i32, [u64p, i32, u32p]),
        "bsort_dist_send_counts": (i32, [u64p, u32p, i32, u64p]),
        "bsort_dist_partition_workspace_bytes": (sz, [i32, u64, i32]),
        "bsort_dist_partition": (i32, [i32, vp, u64, i32, u32p, u64p, i32, vp, vp, sz, vp]),
        "bsort_dist_partition_remote": (i32, [i32, vp, u64, i32, u32p, u64p, i32, u64p, vp, sz, vp]),
        "bsort_dist_refine_hist": (i32, [i32, vp, u64, i32, u64p, i32, i32, vp, vp]),
        "bsort_dist_class_hist": (i32, [i32, vp, u64, i32, u64p, i32, vp, vp]),
        "bsort_dist_class_partition_workspace_bytes": (sz, []),
        "bsort_dist_partition_classes": (i32, [i32, vp, u64, i32, u64p, i32, u64p, vp, vp, sz, vp]),
        "bsort_get_unique_id": (i32, [ctypes.c_char_p]),
        "bsort_comm_init": (i32, [ctypes.POINTER(vp), ctypes.c_char_p, i32, i32]),
        "bsort_comm_destroy": (i32, [vp]),
        "bsort_comm_size": (i32, [vp]),
        "bsort_comm_rank": (i32, [vp]),
        "bsort_sort_dist": (i32, [i32, vp, u64, vp, u64, u64p, i32, vp, vp]),
        "bsort_sort_dist_ex": (i32, [i32, vp, u64, vp, u64, u64p, i32, ctypes.c_uint, vp, vp]),
        "bsort_dist_exact_boundaries": (i32, [u64p, i32, i32, REFINE_FN, vp, u64p, i32p, i32p, u64p, i32p]),
        "bsort_dist_exact_send_counts": (i32, [u64p, i32, i32, i32, i32p, u64p, u64p]),
        "bsort_last_nccl_error": (i32, []),
        "bsort_status_string": (ctypes.c_char_p, [i32]),
        "bsort_last_cuda_error": (i32, []),
        "bsort_version": (ctypes.c_char_p, []),
        "bsort_launch_count": (u64, []),
        "bsort_selftest": (i32, []),
        "bsort_profile_enable": (None, [i32]),
        "bsort_profile_read": (i32, [ctypes.POINTER(ctypes.c_double), u64p]),
        "bsort_profile_kind_name": (ctypes.c_char_p, [i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def check(status: int, where: str):
    if status != SUCCESS:
        raise BsortError(status, where)
