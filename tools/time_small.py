"""Small-n latency breakdown: host cost of one Sorter call (ctypes + libbsort enqueue), device
time per sort with CUDA events around single calls and around CUDA-graph replays (device only)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

lgs = [int(a) for a in sys.argv[1:]] or [16, 18, 20, 22]
for dt in (torch.int32, torch.int64):
    for lg in lgs:
        n = 1 << lg
        x = W.uniform_int(dt, n, 11, "cuda")
        w = x.clone()
        s = B.Sorter(dt, n, "cuda")
        for _ in range(3):
            s(w)
        torch.cuda.synchronize()
        reps = 200
        t0 = time.perf_counter()
        for _ in range(reps):
            s(w)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        host_us = (t1 - t0) / reps * 1e6
        # the C-ABI call alone (arguments prepared once): libbsort's own host cost
        import ctypes
        args = (s.code, ctypes.c_void_p(w.data_ptr()), n, 0, ctypes.c_void_p(s.ws.data_ptr()), s.ws_bytes,
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        t0 = time.perf_counter()
        for _ in range(reps):
            B.lib.bsort_sort_ws(*args)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        abi_us = (t1 - t0) / reps * 1e6
        ev = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s(w)
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        single = sorted(a.elapsed_time(b) for a, b in ev)[10] * 1e3
        g = s.graph(w)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        graph_us = a.elapsed_time(b) / 50 * 1e3
        print(json.dumps({"dtype": str(dt), "n": n, "host_us_per_call": round(host_us, 1), "abi_host_us_per_call": round(abi_us, 1),
                          "event_us_single_call": round(single, 1), "graph_replay_us": round(graph_us, 1)}),
              flush=True)
