"""Time bsort_dist_top_hist (a7) on 2^30 cfg3 f32 keys and 2^30 cfg5 i64 keys: CUDA events,
algorithmic bytes = one read of the keys."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
for name, x in (("cfg3_f32_2^30", W.make("cfg3", "cuda")),
                ("cfg5_i64_2^30", W.make("cfg5", "cuda", n=1 << 30, dtype=torch.int64))):
    for _ in range(3):
        B.top_hist(x)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record()
    for _ in range(reps):
        B.top_hist(x)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    gbs = x.numel() * x.element_size() / (ms / 1e3) / 1e9
    print(json.dumps({"what": f"top_hist {name}", "ms": ms, "GBps": gbs, "frac_of_hbm": gbs / peak}))
    del x
