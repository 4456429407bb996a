"""Per-kernel-kind time of one sort (libbsort's event profiler), averaged over reps, plus the
plain CUDA-event time of the same sort without the profiler.  Usage:
  python tools/breakdown.py --cfg cfg1 [--n N] [--dtype float32] [--inplace] [--reps 20]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg1")
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--dtype", default="")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--inplace", action="store_true")
ap.add_argument("--chunk", type=int, default=0)
ap.add_argument("--layout", default="")
a = ap.parse_args()
dt = getattr(torch, a.dtype) if a.dtype else None
x = W.make(a.cfg, "cuda", n=a.n or None, dtype=dt, layout=a.layout or None)
w = torch.empty_like(x)
s = B.Sorter(x.dtype, x.numel(), "cuda")
run = (lambda: B.sort_inplace_(w, chunk=a.chunk)) if a.inplace else (lambda: s(w))
for _ in range(3):
    w.copy_(x)
    run()
torch.cuda.synchronize()
ev = []
for _ in range(a.reps):
    w.copy_(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    ev.append((e0, e1))
torch.cuda.synchronize()
ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)
with B.profile() as prof:
    for _ in range(a.reps):
        w.copy_(x)
        run()
    torch.cuda.synchronize()
print(json.dumps({"cfg": a.cfg, "layout": a.layout, "n": x.numel(), "dtype": str(x.dtype), "inplace": a.inplace,
                  "median_ms": ms[len(ms) // 2], "min_ms": ms[0],
                  "per_sort": {k: {"ms": v["ms"] / a.reps, "launches": v["launches"] / a.reps}
                               for k, v in prof.items()}}))
