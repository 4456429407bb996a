"""Small-n latency on RANDOM input every call (the input is restored from a pristine copy before
each sort, outside the timed events -- a sort of already-sorted keys would take the presorted
fast path): host µs per call (Python and bare C-ABI, enqueue only), CUDA-event µs per call, and
µs per replay of a user-captured CUDA graph (device only).  argv: log2 sizes."""
import ctypes
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_08929_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

lgs = [int(a) for a in sys.argv[1:]] or [10, 14, 16, 18, 20, 22]
for dt in (torch.int32, torch.int64):
    for lg in lgs:
        n = 1 << lg
        x = W.uniform_int(dt, n, 11, "cuda")
        w = x.clone()
        s = B.Sorter(dt, n, "cuda")
        for _ in range(3):
            w.copy_(x)
            s(w)
        torch.cuda.synchronize()
        # host enqueue cost (random input restored between calls; the restore is not timed)
        reps, host, abi = 100, 0.0, 0.0
        args = (s.code, ctypes.c_void_p(w.data_ptr()), n, 0, ctypes.c_void_p(s.ws.data_ptr()), s.ws_bytes,
                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(reps):
            w.copy_(x)
            t0 = time.perf_counter()
            s(w)
            host += time.perf_counter() - t0
            w.copy_(x)
            t0 = time.perf_counter()
            B.lib.bsort_sort_ws(*args)
            abi += time.perf_counter() - t0
        torch.cuda.synchronize()
        ev = []
        for _ in range(21):
            w.copy_(x)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            s(w)
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        single = statistics.median(a.elapsed_time(b) for a, b in ev[1:]) * 1e3
        g = s.graph(w)
        gev = []
        for _ in range(21):
            w.copy_(x)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            gev.append((a, b))
        torch.cuda.synchronize()
        graph_us = statistics.median(a.elapsed_time(b) for a, b in gev[1:]) * 1e3
        print(json.dumps({"dtype": str(dt), "n": n, "host_us_per_call": round(host / reps * 1e6, 1),
                          "abi_host_us_per_call": round(abi / reps * 1e6, 1),
                          "event_us_single_call": round(single, 1), "graph_replay_us": round(graph_us, 1)}),
              flush=True)
