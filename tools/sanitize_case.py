"""One small sort per kernel family, for compute-sanitizer runs (memcheck /
racecheck / synccheck on small n).  argv: case names (default: all).  Each case sorts seeded
synthetic keys both directions and checks the bytes against the CPU oracle (test
infrastructure).  Paths are selected by size and by the library's A/B environment switches,
which the caller sets per case (see CASES)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

# name -> (dtype, n, env the CALLER must set for that path)
CASES = {
    "small_cta": (torch.int32, 3000, {}),                          # k_small_sort (one CTA)
    "grid_msd": (torch.float32, 300_007, {}),                      # k_grid_sort, MSD first
    "grid_lsd_i64": (torch.int64, (1 << 18) + 7, {}),              # k_grid_sort, LSD passes
    "multilaunch": (torch.float32, 200_003, {"BSORT_SMALL": "0", "BSORT_GRID": "0"}),  # hist+plan+k_onesweep_pass
    "count_u8": (torch.uint8, (1 << 20) + 3, {}),                  # k_count_hist8 / fill8
    "count_i16": (torch.int16, (1 << 20) + 5, {}),                 # k_count_hist16 / scan16 / fill16
    "pass2_ws": (torch.float32, (1 << 22) + 9, {}),                # k_pass2 (unchunked) + k_onesweep_pass_ws
    "joint_chunked": (torch.float32, (1 << 24) + 3, {}),           # order check, joint hist, J01, chunked k_pass2
    "ws64": (torch.float64, (1 << 22) + 1, {}),                    # 64-bit warp-specialised passes
}
_U = {torch.uint32: (torch.int32, np.uint32), torch.uint64: (torch.int64, np.uint64)}


def run(name):
    dt, n, _ = CASES[name]
    x = W.special_mix(dt, n, 5, "cuda") if dt.is_floating_point else W.uniform_int(dt, n, 5, "cuda")
    sd, nd = _U.get(dt, (dt, None))
    h = x.view(sd).cpu().numpy()
    h = h.view(nd) if nd else h
    for desc in (False, True):
        y = x.clone()
        B.sort_(y, descending=desc)
        torch.cuda.synchronize()
        ref = oracle.sort_native(h, descending=desc)
        assert y.view(sd).cpu().numpy().tobytes() == ref.tobytes(), (name, desc)
    print("ok", name)


if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        run(c)
