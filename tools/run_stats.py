"""Fraction of LSD tiles with <= 2 distinct low-digit values (RUN2 fast path) per pass, for a
BASELINE config, computed with torch (the array after pass p is sorted by the low 8p bits)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
cfg = sys.argv[1]; layout = sys.argv[2] if len(sys.argv) > 2 else None
x = W.make(cfg, "cuda", layout=layout)
b = x.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
if x.dtype == torch.float32:
    neg = (b >> 31) == 1
    enc = torch.where(neg, (~b) & 0xFFFFFFFF, b | 0x80000000)
else:
    enc = b ^ 0x80000000
TILE = 8192
for p in (1, 2, 3):
    low = enc & ((1 << (8 * p)) - 1)
    s = torch.sort(low).values
    n = s.numel() // TILE * TILE
    t = s[:n].view(-1, TILE)
    k = 1 + (t[:, 1:] != t[:, :-1]).sum(1)
    print(f"{cfg} {layout} pass {p}: tiles {t.shape[0]}, K<=2 fraction {(k <= 2).float().mean().item():.4f}, "
          f"mean K {k.float().mean().item():.2f}, distinct low values {torch.unique(s).numel()}")
