"""Run a few sorts of one BASELINE.json config (for ncu / compute-sanitizer captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg3")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--dtype", default="")
ap.add_argument("--layout", default="")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--desc", action="store_true")
a = ap.parse_args()
dt = getattr(torch, a.dtype) if a.dtype else None
x = W.make(a.cfg, "cuda", n=a.n or None, dtype=dt, layout=a.layout or None)
s = B.Sorter(x.dtype, x.numel(), "cuda")
w = torch.empty_like(x)
for _ in range(a.reps):
    w.copy_(x)
    s(w, a.desc)
torch.cuda.synchronize()
print("ok", x.dtype, x.numel(), B.launch_count(), "selftest", B.selftest())
