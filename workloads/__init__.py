"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

Holds none of the method's arithmetic (no key transform, no ordering): only a counter-based
splitmix64 generator and the BASELINE.json config recipes built on it
(DESIGN.md §"Input recipe").  Integer-only bit generation is identical on CPU and GPU
(torch int64 ops with wrap-around); the float recipes (uniform / Box-Muller) use float32 ops
whose last-bit rounding may differ between devices, so parity tests always give the oracle
a host copy of the exact device input, never a regenerated one.
"""
from __future__ import annotations

import math

import torch

GOLDEN = 0x9E3779B97F4A7C15
_C1 = 0xBF58476D1CE4E5B9
_C2 = 0x94D049BB133111EB
CHUNK = 1 << 26


def _s64(c: int) -> int:
    c &= (1 << 64) - 1
    return c - (1 << 64) if c >= (1 << 63) else c


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def mix64(z: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (two's-complement wrap-around)."""
    z = (z ^ _lsr(z, 30)) * _s64(_C1)
    z = (z ^ _lsr(z, 27)) * _s64(_C2)
    return z ^ _lsr(z, 31)


def mix64_int(z: int) -> int:
    """Pure-Python big-int reference of mix64 (for the generator's own pin)."""
    m = (1 << 64) - 1
    z &= m
    z = ((z ^ (z >> 30)) * _C1) & m
    z = ((z ^ (z >> 27)) * _C2) & m
    return z ^ (z >> 31)


def bits(n: int, seed: int, device="cpu", offset: int = 0) -> torch.Tensor:
    """int64[n]: bits_i = mix64(seed + (offset + i + 1) * GOLDEN)."""
    out = torch.empty(n, dtype=torch.int64, device=device)
    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        i = torch.arange(offset + s + 1, offset + e + 1, dtype=torch.int64, device=device)
        out[s:e] = mix64(i * _s64(GOLDEN) + _s64(seed))
    return out


def _to_i32(x: torch.Tensor) -> torch.Tensor:
    """int64 holding a 32-bit pattern in [0, 2^32) -> int32 with the same bits."""
    return (x - ((x >> 31) & 1) * (1 << 32)).to(torch.int32)


def _low(x: torch.Tensor, nbits: int) -> torch.Tensor:
    m = x & ((1 << nbits) - 1)
    return m - ((m >> (nbits - 1)) & 1) * (1 << nbits)  # signed value with those bits


def uniform_int(dtype: torch.dtype, n: int, seed: int, device="cpu", offset: int = 0) -> torch.Tensor:
    """Uniform over all bit patterns of an integer dtype (BASELINE.json cfg1, cfg2, cfg5 i64)."""
    out = torch.empty(n, dtype=dtype, device=device)
    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        b = bits(e - s, seed, device, offset + s)
        if dtype in (torch.int64, torch.uint64):
            out[s:e] = b.view(dtype)
        elif dtype in (torch.int32, torch.uint32):
            out[s:e] = _to_i32(_lsr(b, 32)).view(dtype)
        elif dtype in (torch.int16, torch.uint16):
            out[s:e] = _low(b, 16).to(torch.int16).view(dtype)
        elif dtype in (torch.int8, torch.uint8):
            out[s:e] = _low(b, 8).to(torch.int8).view(dtype)
        else:
            raise TypeError(dtype)
    return out


def uniform_float_bits(dtype: torch.dtype, n: int, seed: int, device="cpu", offset: int = 0,
                       allow_nan: bool = False) -> torch.Tensor:
    """Uniform over the finite bit patterns of f32/f64 (BASELINE.json cfg5 f64, reading Q13):
    an all-ones exponent (inf/NaN) is remapped by clearing the exponent's top bit."""
    out = torch.empty(n, dtype=dtype, device=device)
    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        b = bits(e - s, seed, device, offset + s)
        if dtype == torch.float64:
            if not allow_nan:
                ex = _lsr(b, 52) & 0x7FF
                b = torch.where(ex == 0x7FF, b & ~(1 << 62), b)
            out[s:e] = b.view(torch.float64)
        else:
            w = _lsr(b, 32)
            if not allow_nan:
                ex = (w >> 23) & 0xFF
                w = torch.where(ex == 0xFF, w & ~(1 << 30), w)
            out[s:e] = _to_i32(w).view(torch.float32)
    return out


def mixed_f32(n: int, seed: int, device="cpu", offset: int = 0) -> torch.Tensor:
    """BASELINE.json cfg3: per element, by a hash class out of 10000: 50 -> +0.0, 50 -> -0.0,
    5 -> +inf, 5 -> -inf (1% +-0, 0.1% +-inf, reading Q14 "replace"); the rest split evenly
    between U[-1e6, 1e6] and N(0,1) (Box-Muller).  No NaN."""
    out = torch.empty(n, dtype=torch.float32, device=device)
    two24 = float(2 ** -24)
    for s in range(0, n, CHUNK):
        e = min(n, s + CHUNK)
        h = bits(e - s, seed, device, offset + s)
        g = bits(e - s, seed ^ 0x5DEECE66D, device, offset + s)
        cls = _lsr(h, 24) % 10000
        u24 = (_lsr(h, 40) & 0xFFFFFF).to(torch.float32) * two24
        uni = u24 * 2e6
        uni = uni - 1e6
        u1 = ((_lsr(g, 40) & 0xFFFFFF) + 1).to(torch.float32) * two24  # (0, 1]
        u2 = (g & 0xFFFFFF).to(torch.float32) * two24
        nrm = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * math.pi) * u2)
        v = torch.where((cls & 1) == 1, uni, nrm)
        v = torch.where(cls < 50, torch.zeros_like(v), v)
        v = torch.where((cls >= 50) & (cls < 100), torch.full_like(v, -0.0), v)
        v = torch.where((cls >= 100) & (cls < 105), torch.full_like(v, float("inf")), v)
        v = torch.where((cls >= 105) & (cls < 110), torch.full_like(v, float("-inf")), v)
        out[s:e] = v
    return out


def special_mix(dtype: torch.dtype, n: int, seed: int, device="cpu") -> torch.Tensor:
    """Parity stress for floats: uniform bit patterns INCLUDING NaNs of both signs and all
    payloads, plus sprinkled +-0, +-inf, subnormals (SPEC S:106 defines NaN placement)."""
    t = uniform_float_bits(dtype, n, seed, device, allow_nan=True)
    if n == 0:
        return t
    ib = torch.int64 if dtype == torch.float64 else torch.int32
    sel = bits(n, seed + 7, device)
    k = _lsr(sel, 56)  # 0..255
    specials = torch.tensor([0.0, -0.0, float("inf"), float("-inf")], dtype=dtype, device=device)
    t = torch.where(k < 4, specials[(k % 4).clamp(0, 3)], t)
    sub = (sel & 0xFFFF).to(ib)
    sub_v = sub.view(dtype) if dtype == torch.float32 else sub.view(dtype)
    t = torch.where((k >= 4) & (k < 8), sub_v, t)  # positive subnormals
    t = torch.where((k >= 8) & (k < 12), -sub_v, t)  # negative subnormals
    return t


def adversarial_i32(layout: str, n: int, seed: int, device="cpu") -> torch.Tensor:
    """BASELINE.json cfg4 layouts: 'sorted', 'reverse', 'equal', 'distinct16'."""
    if layout == "sorted":
        return torch.sort(uniform_int(torch.int32, n, seed, device)).values
    if layout == "reverse":
        return torch.sort(uniform_int(torch.int32, n, seed, device), descending=True).values
    if layout == "equal":
        v = _to_i32(torch.tensor([mix64_int(seed) >> 32], dtype=torch.int64))
        return torch.full((n,), int(v.item()), dtype=torch.int32, device=device)
    if layout == "distinct16":
        table = torch.tensor([mix64_int(seed + 1000 + j) >> 32 for j in range(16)], dtype=torch.int64)
        table = _to_i32(table).to(device)
        idx = _lsr(bits(n, seed, device), 60)
        return table[idx]
    raise ValueError(layout)


# BASELINE.json configs (sizes and seeds; DESIGN.md §"Input recipe").
SEEDS = {"cfg1": 0xC0FFEE01, "cfg2": 0xC0FFEE02, "cfg3": 0xC0FFEE03, "cfg4": 0xC0FFEE04,
         "cfg5": 0xC0FFEE05}
SIZES = {"cfg1": 1 << 20, "cfg2": 1 << 28, "cfg3": 1 << 30, "cfg4": 1 << 30, "cfg5": 1 << 33}


def make(cfg: str, device="cpu", n: int | None = None, dtype: torch.dtype | None = None,
         layout: str | None = None, rank: int = 0, world: int = 1) -> torch.Tensor:
    """Input of a BASELINE.json config (optionally rescaled to n).  cfg5: rank's slice of the
    global index range [r*N/P, (r+1)*N/P)."""
    seed = SEEDS[cfg]
    n = SIZES[cfg] if n is None else n
    if cfg == "cfg1":
        return uniform_int(torch.int32, n, seed, device)
    if cfg == "cfg2":
        return uniform_int(dtype or torch.uint8, n, seed, device)
    if cfg == "cfg3":
        return mixed_f32(n, seed, device)
    if cfg == "cfg4":
        return adversarial_i32(layout or "sorted", n, seed, device)
    if cfg == "cfg5":
        lo, hi = rank * n // world, (rank + 1) * n // world
        if (dtype or torch.int64) == torch.float64:
            return uniform_float_bits(torch.float64, hi - lo, seed, device, offset=lo)
        return uniform_int(torch.int64, hi - lo, seed, device, offset=lo)
    raise ValueError(cfg)
