"""CPU oracle for bsort (arxiv 2603.08929) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2603_08929_b200``) never imports it; the two share no code.

This is a thin ctypes binding over ``oracle/bsort_oracle.c`` (plain single-threaded C written
from the paper, see that file for the per-function citations):

* ``bsort``          R1 — Algorithms 1-5 with the
                     readings Q1/Q2 listed in DESIGN.md.
* ``sort_by_key``    R2 — the plain definition: comparison sort by the total-order key
                     (SPEC S:82-90), reversed for descending.
* ``single_pass``    Algorithm 1 alone, for the figure pins (k values).
* ``sort_native``    R1 on a numpy array of one of the ten native dtypes (bit patterns).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

UNSIGNED, SIGNED, FLOAT = 0, 1, 2


class _Scheme(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("width", ctypes.c_int),
                ("exp_bits", ctypes.c_int), ("mant_bits", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("inspections_per_level", ctypes.c_uint64 * 64),
                ("inspections", ctypes.c_uint64), ("swaps", ctypes.c_uint64),
                ("partition_calls", ctypes.c_uint64), ("max_depth", ctypes.c_int)]


@dataclass(frozen=True)
class Scheme:
    """WordScheme: Unsigned(w), Signed(w) or Float(w, e, t), w = e + t + 1."""
    kind: int
    width: int
    exp_bits: int = 0
    mant_bits: int = 0

    def c(self) -> _Scheme:
        return _Scheme(self.kind, self.width, self.exp_bits, self.mant_bits)


def U(w):  # noqa: N802 - scheme constructors read like the paper's notation
    return Scheme(UNSIGNED, w)


def I(w):  # noqa: N802,E743
    return Scheme(SIGNED, w)


def F(w, e, t):  # noqa: N802
    return Scheme(FLOAT, w, e, t)


# Table II word sizes plus the unsigned variants BASELINE.json adds.
NATIVE_SCHEMES = {
    np.dtype(np.uint8): U(8), np.dtype(np.int8): I(8),
    np.dtype(np.uint16): U(16), np.dtype(np.int16): I(16),
    np.dtype(np.uint32): U(32), np.dtype(np.int32): I(32),
    np.dtype(np.float32): F(32, 8, 23),
    np.dtype(np.uint64): U(64), np.dtype(np.int64): I(64),
    np.dtype(np.float64): F(64, 11, 52),
    np.dtype(np.float16): F(16, 5, 10),   # IEEE binary16
}
BF16 = F(16, 8, 7)  # bfloat16 (numpy has no dtype for it: sort its uint16 bit patterns)
_UINT_OF_SIZE = {1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}

_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"oracle library missing: {_LIB_PATH} (run `make oracle`)")
    lib = ctypes.CDLL(_LIB_PATH)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    sp = ctypes.POINTER(_Scheme)
    stp = ctypes.POINTER(_Stats)
    lib.bo_single_pass.restype = ctypes.c_uint64
    lib.bo_single_pass.argtypes = [u64p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_int, stp, ctypes.c_int]
    for name in ("bo_bsort", "bo_bsort_float_literal"):
        f = getattr(lib, name)
        f.restype = ctypes.c_int
        f.argtypes = [u64p, ctypes.c_uint64, sp, ctypes.c_int, stp]
    lib.bo_sort_by_key.restype = ctypes.c_int
    lib.bo_sort_by_key.argtypes = [u64p, ctypes.c_uint64, sp, ctypes.c_int]
    lib.bo_total_order_keys.restype = None
    lib.bo_total_order_keys.argtypes = [u64p, u64p, ctypes.c_uint64, sp]
    lib.bo_bruteforce.restype = ctypes.c_int64
    lib.bo_bruteforce.argtypes = [sp, ctypes.c_int, u64p]
    _lib = lib
    return lib


def _u64(words) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(words, dtype=np.uint64)).copy()
    return a


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def single_pass(words, m: int, ps: int, pe: int, asc: bool):
    """Algorithm 1 on a copy; returns (k, array)."""
    a = _u64(words)
    k = _load().bo_single_pass(_ptr(a), m, ps, pe, int(asc), None, 1)
    return int(k), a


def bsort(words, scheme: Scheme, asc: bool = True, with_stats: bool = False):
    """R1 on a copy of ``words`` (raw w-bit patterns zero-extended to uint64)."""
    a = _u64(words)
    st = _Stats()
    rc = _load().bo_bsort(_ptr(a), a.size, ctypes.byref(scheme.c()), int(asc), ctypes.byref(st))
    if rc != 0:
        raise ValueError("oracle rejected the scheme or a word wider than the scheme")
    if with_stats:
        return a, {"inspections_per_level": list(st.inspections_per_level),
                   "inspections": st.inspections, "swaps": st.swaps,
                   "partition_calls": st.partition_calls, "max_depth": st.max_depth}
    return a


def bsort_float_literal(words, scheme: Scheme, asc: bool = True):
    """Algorithm 4 as printed (no Q1 fix) — only for the Q1 pin."""
    a = _u64(words)
    rc = _load().bo_bsort_float_literal(_ptr(a), a.size, ctypes.byref(scheme.c()), int(asc), None)
    if rc != 0:
        raise ValueError("bad scheme")
    return a


def sort_by_key(words, scheme: Scheme, asc: bool = True):
    """R2 on a copy."""
    a = _u64(words)
    if _load().bo_sort_by_key(_ptr(a), a.size, ctypes.byref(scheme.c()), int(asc)) != 0:
        raise ValueError("bad scheme")
    return a


def total_order_keys(words, scheme: Scheme) -> np.ndarray:
    a = _u64(words)
    out = np.empty_like(a)
    _load().bo_total_order_keys(_ptr(a), _ptr(out), a.size, ctypes.byref(scheme.c()))
    return out


def bruteforce(scheme: Scheme, max_len: int):
    """(mismatches, cases) of R1 vs R2 over every array of length <= max_len."""
    cases = ctypes.c_uint64(0)
    bad = _load().bo_bruteforce(ctypes.byref(scheme.c()), max_len, ctypes.byref(cases))
    return int(bad), int(cases.value)


def sort_native(arr: np.ndarray, descending: bool = False) -> np.ndarray:
    """R1 on a 1-D numpy array of a native dtype, returned with the same dtype (bit-exact)."""
    arr = np.ascontiguousarray(arr)
    scheme = NATIVE_SCHEMES[arr.dtype]
    ut = _UINT_OF_SIZE[arr.dtype.itemsize]
    words = arr.view(ut).astype(np.uint64)
    out = bsort(words, scheme, asc=not descending)
    return out.astype(ut).view(arr.dtype)
