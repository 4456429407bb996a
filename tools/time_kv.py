"""Median CUDA-event time of the key-value sort (argsort payload) of cfg3 keys, for A/B runs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

dt = getattr(torch, sys.argv[1]) if len(sys.argv) > 1 else torch.float32
x = W.make("cfg3", "cuda") if dt == torch.float32 else W.make("cfg5", "cuda", n=1 << 30, dtype=dt)
k, v = torch.empty_like(x), torch.empty(x.numel(), dtype=torch.int32, device="cuda")
iota = torch.arange(x.numel(), dtype=torch.int32, device="cuda")
ts = []
for i in range(6):
    k.copy_(x)
    v.copy_(iota)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    B.sort_pairs_(k, v)
    b.record()
    torch.cuda.synchronize()
    if i:
        ts.append(a.elapsed_time(b))
print(json.dumps({"dtype": str(dt), "ws": os.environ.get("BSORT_WS", "1"), "median_ms": sorted(ts)[len(ts) // 2]}))
