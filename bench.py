#!/usr/bin/env python
"""bsort on B200 — benchmark (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--quick]

N=1 (default): one step = one full sort of BASELINE.json cfg3 (2^30 f32 keys, mixed
distribution, ascending) already resident in HBM.  N>1 (torchrun, one rank per GPU, NCCL):
one step = one bsort_sort_dist call (C-ABI) on BASELINE.json cfg5 -- 2^33 int64 keys in total,
2^33/N per rank (strong scaling; float64 and 2^30 keys per rank weak scaling measured too):
MSD histogram + all-reduce + partition + grouped send/recv + local sort.  --force-dist runs
that path on one GPU (weak shape).  Rank 0 prints ONE JSON line.

Timing: CUDA events on the sorting stream around each step (device time); the N=1 input is
restored by a device copy between steps, outside the events.  Inputs are >= 4 GiB per buffer,
far larger than the 126 MB L2, so no flush is needed.  The per-kernel roofline comes from
libbsort's own CUDA events recorded around every kernel during the same timed steps.
--impl reference times the CPU oracle (the reference arm for this tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = "keys/sec sorted (i32/f32/u8/f64) at 1/2/4/8 B200; % of HBM/NVLink roofline"
UNIT = "keys/s"
N_CFG3 = 1 << 30


def load_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(kernel: str):
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_cores_used():
    return 1  # the oracle is single-threaded C


def host_cpu():
    """The box's host CPU (model, nproc) for the cpu_baseline record."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def oracle_time(sample_np: np.ndarray, descending=False):
    import oracle
    t0 = time.perf_counter()
    oracle.sort_native(sample_np, descending=descending)
    return time.perf_counter() - t0


# ------------------------------------------------------------------------------ workloads

def cfg3_input(n, device, rank=0):
    import workloads as W
    if rank == 0:
        return W.mixed_f32(n, W.SEEDS["cfg3"], device)
    return W.mixed_f32(n, W.SEEDS["cfg3"], device, offset=rank * n)


def time_steps(fn, restore, steps, stream):
    """Per-step device time (ms) of fn() with restore() between steps, outside the events."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        restore()
        ev[i][0].record(stream)
        fn()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def e2e_single(args, B, pristine, work, sorter, stream, n):
    """End-to-end keys/s through the C-ABI with pinned HOST buffers: every step copies its input
    H2D from pinned memory, sorts, and reads the sorted keys back D2H, all inside the events.

    * serial (one sort at a time, bsort_sort_host in place; the host buffer is restored from a
      pristine copy between steps, outside the events): the latency of one end-to-end sort;
    * pipelined (the headline `value`): bsort_sort_host_to on two streams, each with its own
      device buffer, workspace and pinned output buffer, all reading the same pinned input
      (never written, so no restore is needed and every step sorts unsorted keys); one sort's
      D2H overlaps the next one's H2D and sort, so PCIe carries both directions at once.  Per
      step = the whole timed span / steps."""
    host_pristine = pristine.cpu().pin_memory()
    host = torch.empty(n, dtype=pristine.dtype, pin_memory=True)
    e2e_steps = max(1, min(args.steps, 3))
    times_e = []
    for i in range(e2e_steps + 1):
        host.copy_(host_pristine)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sorter.sort_host(host, work)
        b.record(stream)
        torch.cuda.synchronize()
        if i > 0:  # first one is a warm-up
            times_e.append(a.elapsed_time(b))
    serial_ms = sum(times_e) / len(times_e)
    del host
    # pipelined over two streams
    dev = work.device
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    sorters = [sorter, B.Sorter(pristine.dtype, n, dev)]
    devs = [work, torch.empty_like(work)]
    outs = [torch.empty(n, dtype=pristine.dtype, pin_memory=True) for _ in range(2)]
    torch.cuda.synchronize()

    def pipelined(k):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        done = [torch.cuda.Event(), torch.cuda.Event()]
        a.record(streams[0])
        streams[1].wait_event(a)
        for i in range(k):
            sorters[i % 2].sort_host_to(host_pristine, outs[i % 2], devs[i % 2], stream=streams[i % 2])
        done[1].record(streams[1])
        streams[0].wait_event(done[1])
        b.record(streams[0])
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    pipelined(2)  # warm-up (second sorter's first call)
    k = max(4, 2 * e2e_steps)
    pipe_ms = pipelined(k) / k
    ok = bool(torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32)))  # same keys sorted (bits)
    del outs, devs, sorters
    return {"value": n / (pipe_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": n * 4,
            "d2h_bytes_per_step": n * 4, "ms_per_step": pipe_ms, "steps": k, "streams": 2,
            "outputs_agree": ok,
            "serial": {"value": n / (serial_ms / 1e3), "ms_per_step": serial_ms, "steps": e2e_steps},
            "note": "bsort_sort_host_to on 2 streams (pinned host input -> H2D -> sort -> D2H into "
                    "pinned host output per step, steps overlapped), CUDA events around all k steps; "
                    "serial = bsort_sort_host one sort at a time"}


def bench_single(args, B):
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    n = args.n or N_CFG3
    pristine = cfg3_input(n, dev)
    work = torch.empty_like(pristine)
    sorter = B.Sorter(torch.float32, n, dev)
    restore = lambda: work.copy_(pristine)  # noqa: E731
    run = lambda: sorter(work)  # noqa: E731
    for _ in range(args.warmup):
        restore()
        run()
    torch.cuda.synchronize()
    hbm_peak, peak_src = load_peaks()
    launches0 = B.launch_count()
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        times = time_steps(run, restore, args.steps, stream)  # headline: no per-launch events
        torch.cuda.synchronize()
    launches = B.launch_count() - launches0
    ms = sum(times) / len(times)
    value = n / (ms / 1e3)
    # a separate profiled run (libbsort records CUDA events around each launch) for the
    # per-kernel shares and the pass roofline
    prof_steps = max(3, min(args.steps, 10))
    with B.profile() as prof:
        ptimes = time_steps(run, restore, prof_steps, stream)
    torch.cuda.synchronize()

    # roofline of the dominant kernel (onesweep pass): algorithmic bytes = read + write of
    # every key once per pass: 2 * n * 4 B per launch.
    # One sort runs 4 LSD passes (8-bit digits of 32-bit keys; none of cfg3's digits is trivial)
    # plus, at n >= 2^24, one extra pass-1 launch that exits at once (libbsort launches both
    # pass-1 variants and the device plan picks one).  The per-pass time is therefore the total
    # pass time / 4 (the idle launch's ~4 us is included: conservative).
    pk = prof.get("onesweep_pass", {"ms": float("nan"), "launches": 1})
    passes = 4 * len(ptimes)
    pass_ms = pk["ms"] / passes
    pass_bytes = 2 * n * 4
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9
    # whole-sort fraction against the fixed 36 B/key model
    sort_gbs = 36 * n / (ms / 1e3) / 1e9
    kernel_share = {k: round(v["ms"] / sum(ptimes), 4) for k, v in prof.items()}

    # end to end: C-ABI with host buffers (H2D + sort + D2H inside the events)
    e2e = None
    if not args.quick or args.e2e:
        e2e = e2e_single(args, B, pristine, work, sorter, stream, n)

    # CPU baseline: the oracle on a bounded sample of the same workload
    cpu = None
    if not args.no_cpu:
        sample_n = args.cpu_sample
        sample = pristine[:sample_n].cpu().numpy()
        secs = oracle_time(sample)
        cpu = {"value": sample_n / secs, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
               "host": host_cpu(),
               "sample": f"first {sample_n} keys of the cfg3 input (same distribution), "
                         f"single-threaded C R1 (Algorithms 1-5), {secs:.2f} s"}

    extra = {}
    if not args.quick:
        extra = bench_extra(B, dev, stream, args)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cfg3: n=2^30 f32 keys, half U[-1e6,1e6] + half N(0,1), 1% +-0.0, "
                               "0.1% +-inf, no NaN, ascending, 1 GPU (BASELINE.json configs[2])",
                   "n": n, "key": "f32", "direction": "ascending", "path": "one-sweep LSD, 4 x 8-bit passes",
                   "l2": "inputs 4 GiB >> 126 MB L2 (no flush); input restored by D2D copy between "
                         "steps outside the timed events", "parallelism": "single GPU"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": load_traffic("onesweep_pass"),
                     "kernel": "LSD scatter pass (k_onesweep_pass for passes 0-1; k_pass2 chunked look-back for passes 2-3)",
                     "algorithmic_bytes_per_launch": pass_bytes,
                     "avg_launch_ms": pass_ms, "working_launches_per_step": 4,
                     "launches_per_step": pk["launches"] / len(ptimes), "peak_source": peak_src,
                     "whole_sort_36B_per_key_GBps": sort_gbs, "whole_sort_frac": sort_gbs / hbm_peak,
                     "kernel_share_of_step": kernel_share},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "step_ms": [round(t, 4) for t in times],
    }
    if extra:
        line["configs"] = extra
    return line


def bench_extra(B, dev, stream, args):
    """Secondary BASELINE.json configs (context; parity is in tests/)."""
    import workloads as W
    out = {}

    def measure(name, x, desc, path_bytes_per_key, reps=5):
        work = torch.empty_like(x)
        s = B.Sorter(x.dtype, x.numel(), dev)
        restore = lambda: work.copy_(x)  # noqa: E731
        run = lambda: s(work, desc)  # noqa: E731
        restore(); run(); torch.cuda.synchronize()  # noqa: E702
        t = time_steps(run, restore, reps, stream)
        ms = statistics.median(t)
        n = x.numel()
        hb, _ = load_peaks()
        gbs = path_bytes_per_key * n / (ms / 1e3) / 1e9
        out[name] = {"keys_per_s": n / (ms / 1e3), "ms": ms, "model_GBps": gbs,
                     "model_bytes_per_key": path_bytes_per_key, "frac_of_hbm": gbs / hb}
        del work, s

    measure("cfg1_i32_2^20_asc", W.make("cfg1", dev), False, 36)
    # cfg1 is launch/latency-bound: the same sort replayed as one CUDA graph
    x = W.make("cfg1", dev)
    work = x.clone()
    s = B.Sorter(x.dtype, x.numel(), dev)
    g = s.graph(work)
    restore = lambda: work.copy_(x)  # noqa: E731
    restore(); g.replay(); torch.cuda.synchronize()  # noqa: E702
    t = time_steps(g.replay, restore, 20, stream)
    ms = statistics.median(t)
    out["cfg1_i32_2^20_asc_cuda_graph"] = {"keys_per_s": x.numel() / (ms / 1e3), "ms": ms,
                                           "note": "Sorter.graph(): the whole path as one graph replay"}
    del x, work, s, g
    for dt, nm in ((torch.uint8, "u8"), (torch.int8, "i8"), (torch.int16, "i16")):
        x = W.make("cfg2", dev, dtype=dt)
        bpk = 2 * x.element_size()
        measure(f"cfg2_{nm}_2^28_asc", x, False, bpk)
        measure(f"cfg2_{nm}_2^28_desc", x, True, bpk)
        del x
    for layout in ("sorted", "reverse", "equal", "distinct16"):
        x = W.make("cfg4", dev, layout=layout)
        measure(f"cfg4_i32_2^30_{layout}", x, False, 36)
        del x
    for dt, nm in ((torch.int64, "i64"), (torch.float64, "f64")):
        x = W.make("cfg5", dev, n=1 << 30, dtype=dt)
        measure(f"cfg5_local_{nm}_2^30_1gpu", x, False, 136, reps=3)
        del x
    # §8 N3: key-value sort (argsort payload: u32 values 0..n-1) of the cfg3 keys
    x = W.make("cfg3", dev)
    kw, vw = torch.empty_like(x), torch.empty(x.numel(), dtype=torch.int32, device=dev)
    iota = torch.arange(x.numel(), dtype=torch.int32, device=dev)
    restore = lambda: (kw.copy_(x), vw.copy_(iota))  # noqa: E731
    run = lambda: B.sort_pairs_(kw, vw)  # noqa: E731
    restore(); run(); torch.cuda.synchronize()  # noqa: E702
    t = time_steps(run, restore, 3, stream)
    ms = statistics.median(t)
    hb, _ = load_peaks()
    bpk = 4 + 4 * 2 * (4 + 4)  # histogram read + 4 passes of read+write of key and value
    out["cfg3_f32_kv_argsort_2^30"] = {"keys_per_s": x.numel() / (ms / 1e3), "ms": ms,
                                       "model_GBps": bpk * x.numel() / (ms / 1e3) / 1e9,
                                       "model_bytes_per_key": bpk,
                                       "frac_of_hbm": bpk * x.numel() / (ms / 1e3) / 1e9 / hb}
    del kw, vw, iota
    # §8 N4: in-place mode (default chunk) on the cfg3 keys: time and scratch vs bsort_sort's
    work = torch.empty_like(x)
    restore = lambda: work.copy_(x)  # noqa: E731
    run = lambda: B.sort_inplace_(work)  # noqa: E731
    restore(); run(); torch.cuda.synchronize()  # noqa: E702
    t = time_steps(run, restore, 3, stream)
    ms = statistics.median(t)
    out["cfg3_f32_inplace_2^30"] = {"keys_per_s": x.numel() / (ms / 1e3), "ms": ms,
                                    "scratch_bytes": B.inplace_workspace_bytes(x.dtype, x.numel()),
                                    "scratch_bytes_sort": B.workspace_bytes(x.dtype, x.numel()),
                                    "note": "host-synchronising per partition; default chunk max(2^22, n/32)"}
    del x, work
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------------ multi-GPU (N>1)

def nvlink_peak():
    """Measured NVLink reference of this pool (B200_PROFILING.md): peer copy per direction."""
    return 770.0, "B200_PROFILING.md measured peer copy 770 GB/s per direction (900 nominal)"


def a2a_microbench(dev, bytes_per_pair=1 << 28, reps=5):
    """NCCL all-to-all of `bytes_per_pair` per rank pair on this box; returns the
    per-rank egress GB/s (max-over-ranks time), or None at world size 1."""
    import torch.distributed as dist
    world = dist.get_world_size()
    if world < 2:
        return None
    send = torch.empty(bytes_per_pair * world, dtype=torch.uint8, device=dev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dist.all_to_all_single(recv, send)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del send, recv
    return bytes_per_pair * (world - 1) / (t.item() / 1e3) / 1e9


_JSON_FD = None  # multi-GPU runs: the real stdout (fd 1 is pointed at stderr meanwhile)


def emit(text: str):
    """Write the result line to the real stdout (NCCL prints its version banner on fd 1 at the
    first communicator, whatever NCCL_DEBUG says; the contract is ONE JSON line on stdout)."""
    if _JSON_FD is None:
        print(text, flush=True)
    else:
        os.write(_JSON_FD, (text + "\n").encode())


CFG5_TOTAL = 1 << 33   # BASELINE.json cfg5: 2^33 keys in total (strong scaling over 2/4/8 GPUs)
CFG5_WEAK = 1 << 30    # weak-scaling companion: 2^30 keys per rank


def multi_shapes(world: int, force_weak: bool = False):
    """The N > 1 measurements: [(name, mode, dtype, n_per_rank)], the headline first.
    At world size 1 (--force-dist) the 2^33-key strong shape does not fit one GPU (64 GiB of keys
    + a shard + the workspace), so the headline is the weak shape."""
    shapes = []
    if world > 1 and not force_weak:
        shapes += [("strong_i64", "strong", "i64", CFG5_TOTAL // world),
                   ("strong_f64", "strong", "f64", CFG5_TOTAL // world)]
    shapes += [("weak_i64", "weak", "i64", CFG5_WEAK), ("weak_f64", "weak", "f64", CFG5_WEAK)]
    return shapes


def multi_line(world, steps, warmup, head, results, e2e, a2a_ref, launches, clocks, exact=False):
    """The N > 1 JSON line (pure: tested on CPU by tests/test_bench_contract.py).
    head = the headline (name, mode, dtype, n_per_rank); results[name] = {"ms", "a2a_ms",
    "a2a_bytes", "pass_ms", "pass_bytes", "n_out"} (max-over-ranks ms); e2e = {"ms", "h2d", "d2h"}
    or {"error": ...}; a2a_ref = NCCL all_to_all_single per-rank egress GB/s at 1 GiB per pair."""
    name, mode, dt, n_loc = head
    r = results[name]
    total = n_loc * world
    hbm_peak, peak_src = load_peaks()
    achieved = r["pass_bytes"] / (r["pass_ms"] / 1e3) / 1e9 if r.get("pass_ms") else None
    a2a_gbs = r["a2a_bytes"] / (r["a2a_ms"] / 1e3) / 1e9 if r.get("a2a_ms") else None
    others = {}
    for k, v in results.items():
        nl = v["n_per_rank"]
        others[k] = {"keys_per_s": nl * world / (v["ms"] / 1e3), "ms": v["ms"], "n_per_rank": nl,
                     "dtype": v["dtype"], "mode": v["mode"], "a2a_ms": v.get("a2a_ms"),
                     "a2a_GBps_egress_rank0": (v["a2a_bytes"] / (v["a2a_ms"] / 1e3) / 1e9
                                               if v.get("a2a_ms") else None)}
        if v.get("note"):
            others[k]["note"] = v["note"]
    e2e_rec = None
    if e2e is not None:
        if "error" in e2e:
            e2e_rec = {"value": None, "unit": UNIT, "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
                       "error": e2e["error"]}
        else:
            e2e_rec = {"value": total / (e2e["ms"] / 1e3), "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                       "d2h_bytes_per_step": e2e["d2h"], "ms_per_step": e2e["ms"],
                       "note": "per rank: pinned host keys -> H2D -> bsort_sort_dist (C-ABI) -> D2H of the "
                               "shard; CUDA events, max over ranks; bytes are rank 0's"}
    return {
        "metric": METRIC, "value": total / (r["ms"] / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": r["ms"], "higher_is_better": True,
        "scaling": mode, "vs_baseline": None, "dtype": dt, "data": "synthetic",
        "config": {"workload": f"cfg5: {total} {dt} keys uniform over all "
                               f"{'bit patterns' if dt == 'i64' else 'finite bit patterns'}, "
                               f"{n_loc} per rank x {world} ranks, globally sorted shards",
                   "n_per_rank": n_loc, "n_total": total, "key": dt, "direction": "ascending",
                   "path": "bsort_sort_dist (C-ABI): a7 top-16-bit histogram + NCCL all-reduce + splitters "
                           "+ counts all-gather + a9 partition + grouped NCCL send/recv + local one-sweep LSD",
                   "parallelism": f"msd-a2a x{world}" + (" exact-split" if exact else ""),
                   "l2": f"inputs {n_loc * 8} B per rank >> 126 MB L2 (no flush); the input is const "
                         "(bsort_sort_dist reads dev_in, writes dev_out)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": (achieved / hbm_peak) if achieved else None, "traffic": None,
                     "kernel": "local LSD scatter pass of 64-bit keys (8 passes per step)",
                     "algorithmic_bytes_per_launch": r.get("pass_bytes"), "avg_launch_ms": r.get("pass_ms"),
                     "peak_source": peak_src,
                     "a2a": {"ms_per_step": r.get("a2a_ms"), "bytes_per_step_rank0": r.get("a2a_bytes"),
                             "GBps_egress_rank0": a2a_gbs, "nccl_all_to_all_1GiB_pair_GBps": a2a_ref,
                             "frac_of_nccl_a2a": (a2a_gbs / a2a_ref) if (a2a_gbs and a2a_ref) else None,
                             "note": "exchange = grouped ncclSend/ncclRecv inside bsort_sort_dist, timed by "
                                     "libbsort's dist_a2a profile events (a separate profiled run)"}},
        "cpu_baseline": None,
        "e2e": e2e_rec,
        "gpu_launches": launches,
        "clocks": clocks,
        "configs": others,
    }


def bench_multi(args, B):
    """N > 1 (torchrun, one rank per GPU) or --force-dist: BASELINE.json cfg5 through the C-ABI
    bsort_sort_dist (B.Comm + B.sort_dist_native).  Headline: 2^33 int64 keys in total (strong
    scaling); float64 and the 2^30-per-rank weak shape are measured too (under "configs").
    A step = one bsort_sort_dist call (input const, shard written to a separate buffer)."""
    import torch.distributed as dist
    import workloads as W
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    comm = B.Comm()
    shapes = multi_shapes(world)
    if args.n:
        shapes = [("weak_i64", "weak", "i64", args.n)]
    if args.quick:
        shapes = shapes[:1]
    head = shapes[0]
    tdt = {"i64": torch.int64, "f64": torch.float64}

    def maxr(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    results, e2e, launches, clocks = {}, None, None, None
    for name, mode, dt, n_loc in shapes:
        x = W.make("cfg5", dev, n=n_loc * world, dtype=tdt[dt], rank=rank, world=world)
        cap = n_loc + n_loc // 16 + (1 << 16)
        run = lambda: B.sort_dist_native(x, comm, capacity=cap, exact=args.exact)  # noqa: E731
        for _ in range(args.warmup):
            out = run()
            del out
        torch.cuda.synchronize()
        dist.barrier()
        l0 = B.launch_count()
        sampler = ClockSampler(local) if name == head[0] else None
        if sampler:
            sampler.__enter__()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for i in range(args.steps):
            ev[i][0].record(stream)
            out = run()
            ev[i][1].record(stream)
            del out
        torch.cuda.synchronize()
        if sampler:
            sampler.__exit__(None, None, None)
            clocks = sampler.summary()
            launches = B.launch_count() - l0
        dist.barrier()
        ms = maxr(sum(a.elapsed_time(b) for a, b in ev) / args.steps)
        # a separate profiled run: the exchange (dist_a2a events) and the local LSD passes
        with B.profile() as prof:
            out = run()
        n_out = out.numel()
        del out
        pk = prof.get("onesweep_pass", {"ms": 0.0})
        a2 = prof.get("dist_a2a", {"ms": 0.0})
        res = {"ms": ms, "mode": mode, "dtype": dt, "n_per_rank": n_loc,
               "a2a_ms": maxr(a2["ms"]), "a2a_bytes": None, "n_out": n_out,
               "pass_ms": maxr(pk["ms"] / 8) if pk["ms"] else None, "pass_bytes": 2 * n_out * 8}
        # rank 0's egress bytes (keys to the other ranks): n_loc minus what it keeps
        res["a2a_bytes"] = _egress_bytes(B, x, comm, world, rank) if world > 1 else 0
        results[name] = res
        if name == head[0] and not args.quick:
            # §8 N1: the same step with the fused partition + exchange over CUDA IPC peer memory
            runf = lambda: B.sort_dist_native(x, comm, capacity=cap, fused=True)  # noqa: E731
            for _ in range(args.warmup):
                del_ = runf()
                del del_
            torch.cuda.synchronize()
            dist.barrier()
            evf = []
            for _ in range(max(1, min(args.steps, 5))):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                o = runf()
                b.record(stream)
                evf.append((a, b))
                del o
            torch.cuda.synchronize()
            msf = maxr(sum(a.elapsed_time(b) for a, b in evf) / len(evf))
            results[name + "_fused"] = dict(res, ms=msf, a2a_ms=None, pass_ms=None,
                                            note="BSORT_DIST_FUSED: partition straight into the owners' "
                                                 "receive buffers (CUDA IPC), device-side barriers")
        if name == head[0] and not (args.quick and not args.e2e):
            e2e = _e2e_dist(B, x, comm, cap, args, dev, stream, maxr)
        del x
        torch.cuda.empty_cache()
    a2a_ref = a2a_microbench(dev, bytes_per_pair=1 << 30) if world > 1 else None
    comm.close()
    if rank == 0:
        emit(json.dumps(multi_line(world, args.steps, args.warmup, head, results, e2e, a2a_ref, launches,
                                   clocks, exact=args.exact)))


def _egress_bytes(B, x, comm, world, rank):
    """Bytes this rank sends to other ranks in one bsort_sort_dist of x (bin-granular split):
    from the same top-16-bit histograms libbsort computes (B.top_hist + all-reduce)."""
    import torch.distributed as dist
    hl = B.top_hist(x)
    hg = hl.clone()
    dist.all_reduce(hg.view(torch.int64), op=dist.ReduceOp.SUM)
    cuts = B.splitters(hg.view(torch.int64).cpu().numpy().view(np.uint64), world)
    sc = B.send_counts(hl.view(torch.int64).cpu().numpy().view(np.uint64), cuts)
    return int((int(sc.sum()) - int(sc[rank])) * x.element_size())


def _e2e_dist(B, x, comm, cap, args, dev, stream, maxr):
    """End to end through the public API: pinned host keys -> H2D -> bsort_sort_dist -> D2H."""
    try:
        host = x.cpu().pin_memory()
        host_out = torch.empty(cap, dtype=x.dtype).pin_memory()
    except RuntimeError as e:
        return {"error": f"pinned host buffers: {str(e).splitlines()[0]}"}
    work = torch.empty_like(x)
    times, out_bytes = [], 0
    for i in range(3):
        import torch.distributed as dist
        dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        work.copy_(host, non_blocking=True)
        shard = B.sort_dist_native(work, comm, capacity=cap, exact=args.exact)
        res = host_out[:shard.numel()]
        res.copy_(shard, non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        out_bytes = res.numel() * res.element_size()
        del shard
        if i:
            times.append(a.elapsed_time(b))
    ms = maxr(max(times))
    del host, host_out, work
    return {"ms": ms, "h2d": x.numel() * x.element_size(), "d2h": out_bytes}


# ------------------------------------------------------------------------ reference arm

def bench_reference(args):
    """The CPU oracle timed on the box's host cores, on a bounded sample of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import workloads as W
    sample_n = args.ref_sample
    x = W.mixed_f32(sample_n, W.SEEDS["cfg3"], "cpu").numpy()
    for _ in range(args.warmup):
        oracle_time(x)
    secs = [oracle_time(x) for _ in range(args.steps)]
    s = sum(secs) / len(secs)
    value = sample_n / s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "cfg3: f32 keys, half U[-1e6,1e6] + half N(0,1), 1% +-0.0, 0.1% +-inf, "
                               "ascending (bounded sample of the same distribution)",
                   "n": sample_n, "parallelism": "single CPU thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "host": host_cpu(),
                         "sample": f"{sample_n} keys of the cfg3 distribution (CPU-generated, same recipe)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=0, help="override keys (per rank)")
    ap.add_argument("--quick", action="store_true", help="skip secondary configs and e2e")
    ap.add_argument("--e2e", action="store_true", help="with --quick: still measure e2e")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 25)
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    ap.add_argument("--exact", action="store_true",
                    help="N > 1: exact splitting (SURVEY §8 N2) instead of bin-granular cuts")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU code path even at world size 1 (testing)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    if args.impl == "reference":
        bench_reference(args)
        return

    import paper_2603_08929_b200 as B
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.force_dist:
        global _JSON_FD
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)
        import torch.distributed as dist
        if "RANK" not in os.environ:  # --force-dist outside torchrun: a one-rank group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(port))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        try:
            bench_multi(args, B)
        finally:
            dist.destroy_process_group()
        return
    print(json.dumps(bench_single(args, B)), flush=True)


if __name__ == "__main__":
    main()
