"""Sort throughput vs n (CUDA events, median of reps, input restored between runs) for the
headline key types, one JSON line per (dtype, n).  python tools/sweep_n.py > sweep.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

CASES = [("cfg3", torch.float32), ("cfg1", torch.int32), ("cfg5", torch.int64), ("cfg5", torch.float64)]
# argv: [max_lg [step]] -- e.g. `sweep_n.py 24 1` for every power of two up to 2^24
MAX_LG = int(sys.argv[1]) if len(sys.argv) > 1 else 30
STEP = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for cfg, dt in CASES:
    for lg in range(16, MAX_LG + 1, STEP):
        n = 1 << lg
        x = W.make(cfg, "cuda", n=n, dtype=dt if cfg == "cfg5" else None)
        if x.dtype != dt:
            x = x.to(dt) if not dt.is_floating_point else x
        s = B.Sorter(x.dtype, n, "cuda")
        w = torch.empty_like(x)
        reps = 20 if lg <= 24 else 5
        ts = []
        for i in range(reps + 2):
            w.copy_(x)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s(w)
            b.record()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        ms = sorted(ts)[len(ts) // 2]
        print(json.dumps({"cfg": cfg, "dtype": str(x.dtype), "n": n, "median_ms": ms,
                          "gkeys_per_s": n / (ms / 1e3) / 1e9}), flush=True)
        del x, w, s
        torch.cuda.empty_cache()
