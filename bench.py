#!/usr/bin/env python3
"""bench.py — sorted GB/s of 100-byte records on B200 (BASELINE.json metric), one JSON line on rank 0.

A "step" is one pass of the whole hot path (K-a .. K-e: SURVEY.md §8a rows a1-a6) over one batch of
synthetic records already resident in HBM: one ley_sort call through the C ABI. Default workload:
BASELINE.json configs[3] (C4: 6e8 uniform records = 60 GB, seed 3), the largest configuration that fits
one GPU, with configs[1] (C2: 1e8 records = 10 GB, seed 1) measured in the same run into the line's
`secondary` key. Inputs are >= 10 GB, far larger than the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--config c1..c7] [--secondary c2|none] [--impl ours|reference]

Keys beyond the base contract: `roofline` (dominant kernel, algorithmic bytes / CUDA-event time against
MEASURED_PEAKS.json hbm_gbs), `step_roofline` (the whole step: 200 B/record / HBM peak),
`cpu_baseline` (the oracle timed on this host on a bounded sample), `e2e` (same metric through the C
ABI with pinned host buffers: H2D + sort + D2H inside the timed region), `clocks`, `gpu_launches`.
Multi-GPU (N > 1, torchrun): the config's records are split into rank slices and sorted by the key-range
path (ley_sort_dist: splitters, fused partition + exchange over NVLink, local sort; "scaling": "strong").
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(n=1_000_000, seed=0, dist="uniform", name="C1 1e6 x 100 B uniform (BASELINE.json configs[0])"),
    "c2": dict(n=100_000_000, seed=1, dist="uniform", name="C2 1e8 x 100 B uniform, 10 GB (BASELINE.json configs[1])"),
    "c3": dict(n=200_000_000, seed=2, dist="skewed",
               name="C3 2e8 x 100 B Zipf(1.2) byte0, 8-valued byte1, 2% dup keys, 20 GB (BASELINE.json configs[2])"),
    "c4": dict(n=600_000_000, seed=3, dist="uniform", name="C4 6e8 x 100 B uniform, 60 GB (BASELINE.json configs[3])"),
    # external path: pinned host in/out; scaled from 6e8/4 GB to 2e8/(4/3) GB (same 15:1 data-to-budget
    # ratio) so in + out + run scratch (3 x 20 GB pinned) fits the GPU box's 196 GB host RAM
    "c5": dict(n=200_000_000, seed=4, dist="uniform", budget=(4 << 30) // 3,
               name="C5 external (scaled): 2e8 x 100 B uniform in pinned host memory, device budget 1.33 GB "
                    "(BASELINE.json configs[4] ratio 60 GB : 4 GB)"),
    # SURVEY §8f NEXT 4 workload variants (the paper's third data set: 20 GB, uniform, ASCII)
    "c6": dict(n=200_000_000, seed=5, dist="ascii",
               name="C6 ASCII 2e8 x 100 B printable records + CR LF, 20 GB, device-resident (P:126 20 GB set)"),
    "c7": dict(n=200_000_000, seed=5, dist="ascii", budget=30_000_000_000,
               name="C7 partial in-memory: ASCII 2e8 x 100 B in pinned host memory, device budget 30 GB "
                    "(P:126 / Table 2: 20 GB of data, 30 GB of memory)"),
}
METRIC = "sorted GB/s of 100-byte records"
# algorithmic bytes per record of each stage: what the step must move
STAGE_ALG_BYTES = {"K-a tile sort": 10 + 12, "K-c split": 12 + 12, "K-de sort+gather": 12 + 100 + 100}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML, every 5 ms; B200_PROFILING.md)."""

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    _BITS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}
    _nv = None

    def _init(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nv = (pynvml, h, pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nv = None

    def _sample_once(self):
        if self._nv is None:
            return
        try:
            pynvml, h, mx = self._nv
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            util = pynvml.nvmlDeviceGetUtilizationRates(h).gpu
            self.samples.append((sm, mx, {k for k, b in self._BITS.items() if reasons & b}, util))
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample_once()
            self._stop.wait(self.period)

    def __enter__(self):
        self._init()  # NVML handle ready before the timed region starts
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples:  # a timed region shorter than the first sample: one sample as it ends
            self._sample_once()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        loaded = [x for x in self.samples if x[3] > 0] or self.samples
        return {"sm_mhz": statistics.median(x[0] for x in loaded), "sm_max_mhz": max(x[1] for x in loaded),
                "reasons": sorted(set().union(*[x[2] for x in loaded])), "samples": len(loaded)}


def _oracle_step(recs, threads, key_bytes):
    """One oracle sort; (extract, sort, gather) seconds for the paper's 10-byte keys, else None."""
    import oracle

    if key_bytes == 10:
        return oracle.sort_timed(recs, threads=threads)[1]
    oracle.sort(recs, threads=threads, want_perm=False, key_bytes=key_bytes)
    return None


def host_link_gbs(nbytes: int = 1 << 30, reps: int = 3):
    """Pinned-memory copy-engine bandwidth of this GPU's host link (GB/s): H2D alone, D2H alone, and each
    direction while both run (two streams) — the denominators of the host-path rooflines."""
    import torch

    h = [torch.empty(nbytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
    d = [torch.empty(nbytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(reps):
            e0.record()
            fn()
            torch.cuda.synchronize()  # (both side streams joined)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return nbytes / (best / 1e3) / 1e9

    def h2d():
        with torch.cuda.stream(s1):
            d[0].copy_(h[0], non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h[1].copy_(d[1], non_blocking=True)

    def both():
        h2d()
        d2h()

    out = {"h2d": round(timed(h2d), 1), "d2h": round(timed(d2h), 1), "bidir_each": round(timed(both), 1)}
    del h, d
    torch.cuda.empty_cache()
    return out


def cpu_baseline(cfg, sample_n: int, key_bytes: int = 10):
    """The oracle as it stands (oracle/), timed on this host's cores on a bounded sample."""
    import gen

    recs = gen.records(sample_n, cfg["seed"], cfg["dist"])
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    st = _oracle_step(recs, threads, key_bytes)
    dt = time.perf_counter() - t0
    stages = (f"extract {st[0]:.2f} s, sort {st[1]:.2f} s, gather {st[2]:.2f} s (__gnu_parallel::sort, OpenMP)"
              if st else f"record-comparison sort on {key_bytes}-byte keys (__gnu_parallel::sort, OpenMP)")
    return {"value": round(sample_n * 100 / dt / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"first {sample_n:,} records of {cfg['name'].split(' (')[0]} (same generator/seed); {stages}",
            "seconds": round(dt, 3)}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gen

    sample_n = args.cpu_sample
    recs = gen.records(sample_n, cfg["seed"], cfg["dist"])
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        _oracle_step(recs[: min(sample_n, 1_000_000) * 100], threads, args.key_bytes)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        _oracle_step(recs, threads, args.key_bytes)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    v = sample_n * 100 / t / 1e9
    line = {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "n_records": cfg["n"], "sample_records": sample_n,
                       "key_bytes": args.key_bytes},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                             "sample": f"first {sample_n:,} records of the workload per step"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure(args, cfg_name, world, rank, local, comm, with_cpu=True):
    """One config on this rank's GPU: the device-timed step (value, stages, roofline), e2e through the C ABI
    with pinned host buffers, clocks, launches; the CPU baseline on rank 0. Returns the JSON fields."""
    import torch
    import torch.distributed as dist

    import gen
    import paper_1909_08006_b200 as ley

    cfg = CONFIGS[cfg_name]
    stream = torch.cuda.current_stream()
    n_total = cfg["n"]
    external = "budget" in cfg
    if comm is not None:
        # strong scaling: the config's records split into contiguous rank slices
        lo, hi = rank * n_total // world, (rank + 1) * n_total // world
        n = hi - lo
    else:
        lo, n = 0, n_total
    cap = n_total // world + 2 if comm is not None else n
    if external:
        x = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
        out = torch.empty(cap * 100, dtype=torch.uint8).pin_memory()
        stage = torch.empty(min(n, 50_000_000) * 100, dtype=torch.uint8, device="cuda")
        for at in range(0, n, 50_000_000):
            m = min(50_000_000, n - at)
            gen.records_cuda(stage.data_ptr(), m, cfg["seed"], cfg["dist"], i0=lo + at, stream=stream.cuda_stream)
            x[at * 100:(at + m) * 100].copy_(stage[: m * 100])
        del stage
        torch.cuda.empty_cache()
    else:
        x = torch.empty(max(n, 1) * 100, dtype=torch.uint8, device="cuda")
        gen.records_cuda(x.data_ptr(), n, cfg["seed"], cfg["dist"], i0=lo, stream=stream.cuda_stream)
        out = torch.empty(max(cap, 1) * 100, dtype=torch.uint8, device="cuda")
    budget = cfg.get("budget", 0)

    def step():
        if comm is not None:
            ley.ley_sort_dist(comm, x, n, out, cap, key_bytes=args.key_bytes, device_budget_bytes=budget, stream=stream)
        else:
            ley.ley_sort(x, out, n, key_bytes=args.key_bytes, device_budget_bytes=budget, stream=stream)

    def barrier():
        if world > 1:
            dist.barrier()

    ley.ley_set_option("async", 0 if comm is not None or external else 1)  # (as in the value pass below)
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    ley.ley_set_option("async", 0)

    # ---------------------------------------------------------------- timed region (device events)
    # (1) the step as a user runs it (no per-stage events: level 1 replays its cached CUDA graph) -> value;
    # (2) the same K steps again with per-stage CUDA events (the library's "profile" option, which launches
    #     level 1 directly) -> stages_ms and the dominant kernel's roofline, from its own timed region.
    # Inputs below 1e7 records (C1: 100 MB) fit the 126 MB L2: every timed step then gets its own event
    # pair, with a 256 MB write between steps (outside the timed intervals) flushing the L2.
    # (then a 256 MB read: the write leaves the L2 full of dirty lines, whose write-back would otherwise
    # land inside the next timed step; after the read the L2 is cold and clean)
    flush_buf = (torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
                 if n_total < 10**7 and comm is None and not external else None)
    flush_rd = torch.ones(64 << 20, dtype=torch.int32, device="cuda") if flush_buf is not None else None

    def timed_steps(profile):
        ley.ley_set_option("profile", profile)
        # the value pass uses the stream-ordered API (option async: a device sort without recursion returns
        # once enqueued, so back-to-back steps keep the GPU busy); every step's work is inside the timed
        # region, which ends with an event after the last step and a synchronize
        ley.ley_set_option("async", 0 if profile or comm is not None or external else 1)
        stage_ms: dict[str, list[float]] = {}
        launches = 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        per_step = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                    for _ in range(args.steps)] if flush_buf is not None else None
        barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            e0.record(stream)
            for i in range(args.steps):
                if per_step is not None:
                    with torch.cuda.stream(stream):
                        flush_buf.fill_(i & 0xFF)
                        flush_rd.sum(dtype=torch.int64)
                    per_step[i][0].record(stream)
                step()
                if per_step is not None:
                    per_step[i][1].record(stream)
                if profile:  # (the stage read-back is host work: kept out of the value pass)
                    st, nl = ley.ley_stage_times()
                    launches += nl
                    for name, ms_ in st:
                        stage_ms.setdefault(name, []).append(ms_)
            e1.record(stream)
            torch.cuda.synchronize()
        if not profile:  # every step sorts the same input: the last call's launch count times the steps
            launches = ley.ley_stage_times()[1] * args.steps
        barrier()
        ley.ley_set_option("profile", 0)
        ley.ley_set_option("async", 0)
        if per_step is not None:
            ts = [a.elapsed_time(b) for a, b in per_step]
            if os.environ.get("LEY_BENCH_STEPS"):
                print("per-step ms:", " ".join(f"{t:.4f}" for t in ts), file=sys.stderr)
            ms_ = sum(ts) / args.steps
        else:
            ms_ = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms_], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_ = float(t.item())
        return ms_, stage_ms, launches, clk

    ms, _, launches, clk = timed_steps(0)
    prof_ms, stage_ms, _, prof_clk = timed_steps(1)
    value = n_total * 100 / (ms / 1e3) / 1e9

    peak, peak_src = _peaks()
    avg = {k: statistics.mean(v) for k, v in stage_ms.items()}
    roofline = None
    kern = [k for k in avg if k in STAGE_ALG_BYTES]
    if kern and not external:  # (host paths: the host link is the bound, host_roofline below)
        dominant = max(kern, key=lambda k: avg[k])
        alg = STAGE_ALG_BYTES[dominant] * n
        achieved = alg / (avg[dominant] / 1e3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp) and world == 1:
            with open(tp) as f:
                ent = json.load(f).get(cfg_name, {}).get(dominant)
            if ent:  # DRAM bytes of the stage's launches in one call (ncu; tools/ncu_traffic.py)
                traffic = ent.get("bytes_per_launch")
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": dominant,
                    "alg_bytes_per_record": STAGE_ALG_BYTES[dominant], "peak_source": peak_src}
    step_roof_ms = 200 * n / (peak * 1e9) * 1e3
    host_roofline = None
    if external and rank == 0:
        # host-link roofline (SURVEY §8d HOST_alg): the external path crosses the link twice in each direction
        # (200 B/record per direction, the directions overlap); the resident path once each way, serially
        link = host_link_gbs()
        plan = ley.ley_plan_query(n, budget)
        if plan["host_path"] == 2:
            t_roof = 100 * n / (link["h2d"] * 1e9) + 100 * n / (link["d2h"] * 1e9)
            model = "resident path: 100 B/record H2D then 100 B/record D2H (serial: the sort needs all input)"
        else:
            t_roof = 200 * n / (link["bidir_each"] * 1e9)
            model = "external path: 200 B/record per direction, both directions at once"
        host_roofline = {"bound": "host-link", "t_roof_ms": round(t_roof * 1e3, 1),
                         "frac": round(t_roof * 1e3 / ms, 4), "link_gbs": link, "model": model,
                         "note": "measured pinned copy-engine bandwidth of this box (host_link_gbs)"}
    step_roofline = {"alg_bytes_per_record": 200, "t_roof_ms": round(step_roof_ms, 3),
                     "frac": round(step_roof_ms / ms, 4), "peak": peak, "unit": "GB/s",
                     "note": "HBM term only" + (" (external: host-link bound, see DESIGN.md)" if external else "")}

    # ---------------------------------------------------------------- e2e through the C ABI, host buffers
    e2e = None
    if external:
        e2e = {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": n * 100 * 2,
               "d2h_bytes_per_step": n * 100 * 2, "ms_per_step": round(ms, 3), "note": "the timed step is host-to-host"}
    elif not args.no_e2e and comm is not None:
        # each rank: its pinned host slice -> HBM, the distributed sort (ley_sort_dist), its sorted range
        # back to pinned host memory; max over ranks of the event-timed steps
        hin = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
        hin.copy_(x[: n * 100])
        hout = torch.empty(cap * 100, dtype=torch.uint8).pin_memory()

        def e2e_step():
            x[: n * 100].copy_(hin, non_blocking=True)
            n_out, _ = ley.ley_sort_dist(comm, x, n, out, cap, key_bytes=args.key_bytes, device_budget_bytes=budget,
                                         stream=stream)
            hout[: n_out * 100].copy_(out[: n_out * 100], non_blocking=True)
            return n_out

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        outs = 0
        for _ in range(args.e2e_steps // 4 or 1):
            outs = e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1) / (args.e2e_steps // 4 or 1)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": round(n_total * 100 / (ems / 1e3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": n * 100,
               "d2h_bytes_per_step": outs * 100, "ms_per_step": round(ems, 3), "steps": args.e2e_steps // 4 or 1,
               "api": "per rank: pinned slice H2D + ley_sort_dist + D2H of its range (bytes are this rank's)"}
        del hin, hout
    elif not args.no_e2e and world == 1:
        hin = torch.empty(n * 100, dtype=torch.uint8).pin_memory()
        hin.copy_(x[: n * 100])
        hout = torch.empty_like(hin).pin_memory()
        del x, out  # room for the library's staging of in + out
        torch.cuda.empty_cache()
        ley.ley_release_cache(-1)
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def timed(call, steps, finish=None):
            f0.record(stream)
            for _ in range(steps):
                call(hin, hout, n, key_bytes=args.key_bytes, stream=stream)
            if finish:  # the streaming call returns before its output lands: wait for every copy first
                finish()
            f1.record(stream)
            torch.cuda.synchronize()
            return f0.elapsed_time(f1) / steps

        # (1) the SURVEY §8(b) call itself, one blocking ley_sort per step: H2D of the step's input, the sort,
        #     D2H of its output, all inside the timed region
        ley.ley_sort(hin, hout, n, key_bytes=args.key_bytes, stream=stream)  # warm: the staging buffers
        bsteps = max(2, args.e2e_steps // 3) if n <= 200_000_000 else 2
        bms = timed(ley.ley_sort, bsteps)
        e2e = {"value": round(n * 100 / (bms / 1e3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": n * 100,
               "d2h_bytes_per_step": n * 100, "ms_per_step": round(bms, 3), "steps": bsteps,
               "api": "ley_sort (pinned host in/out, blocking: H2D + sort + D2H per step)"}
        # (2) the streaming call, when two device slots of in + out fit: H2D of step k+1 overlaps the D2H of
        #     step k (ley_sort_submit); the region ends after ley_sort_drain(), i.e. once the last output landed
        if 4 * n * 100 < torch.cuda.get_device_properties(0).total_memory * 0.8:
            ley.ley_release_cache(-1)
            ley.ley_sort_submit(hin, hout, n, key_bytes=args.key_bytes, stream=stream)  # warm: the two slots
            ley.ley_sort_drain()
            ems = timed(ley.ley_sort_submit, args.e2e_steps, finish=ley.ley_sort_drain)
            e2e["streaming"] = {"api": "ley_sort_submit / ley_sort_drain (consecutive calls overlap H2D and D2H)",
                                "value": round(n * 100 / (ems / 1e3) / 1e9, 3), "ms_per_step": round(ems, 3),
                                "steps": args.e2e_steps}
        del hin, hout
        ley.ley_release_cache(-1)

    cpu = None
    if with_cpu and not args.no_cpu and rank == 0:
        cpu = cpu_baseline(cfg, min(args.cpu_sample or cfg["n"], cfg["n"], 100_000_000), args.key_bytes)

    return {
        "value": round(value, 3), "ms_per_step": round(ms, 4), "n_gpus": world,
        "config": {"workload": cfg["name"] + ("" if args.key_bytes == 10 else f", {args.key_bytes}-byte keys (P:164)"),
                   "n_records": n_total, "record_bytes": 100, "key_bytes": args.key_bytes,
                   "seed": cfg["seed"], "distribution": cfg["dist"],
                   "device_budget_bytes": budget,
                   "l2": "inputs (>= 10 GB) larger than the 126 MB L2; no flush needed" if n_total >= 10**7
                   else "input fits the L2: a 256 MB write, then a 256 MB read, between timed steps flushes it "
                        "(per-step event pairs, the flush outside them)",
                   "api": "ley_sort on device buffers, stream-ordered (option async)" if comm is None and not external
                   else "ley_sort_dist" if comm is not None else "ley_sort on pinned host buffers",
                   "parallelism": (f"key-range dist x{world} (NCCL, " +
                                   ("all-to-all-v" if args.alltoall else "fused partition+exchange") +
                                   (", exchange at G=1" if args.exchange else "") + ")")
                   if comm is not None else "1 GPU"},
        "roofline": roofline, "step_roofline": step_roofline, "host_roofline": host_roofline,
        "stages_ms": {k: round(v, 4) for k, v in avg.items()},
        "stage_pass": {"ms_per_step": round(prof_ms, 4), "steps": args.steps, "clocks": prof_clk.summary(),
                       "note": "stages_ms and roofline come from this second timed pass of the same steps with "
                               "per-stage CUDA events (level 1 launched directly instead of its CUDA graph)"},
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": launches,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS),
                    help="default c4: BASELINE configs[3], the largest config that fits one GPU")
    ap.add_argument("--secondary", default="c2",
                    help="single GPU, default run: also measure this config into the line's `secondary` key "
                         "('none' to skip)")
    ap.add_argument("--cpu-sample", type=int, default=0, help="oracle sample records (0 = min(n, 1e8))")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true", help="use the NCCL key-range path even at one GPU (checks it)")
    ap.add_argument("--exchange", action="store_true",
                    help="with --dist at one GPU: also run the splitter/partition/exchange phases (dist_exchange_g1)")
    ap.add_argument("--key-bytes", type=int, default=10,
                    help="key = record bytes [0, k), 1..100 (P:164 flexible key sizes; default the paper's 10)")
    ap.add_argument("--alltoall", action="store_true", help="dist: K-p into a send buffer + NCCL all-to-all-v "
                                                            "instead of the fused exchange (dist_fused=0)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if not args.cpu_sample:
        args.cpu_sample = min(cfg["n"], 100_000_000)
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    import paper_1909_08006_b200 as ley

    if args.exchange:
        ley.ley_set_option("dist_exchange_g1", 1)
    if args.alltoall:
        ley.ley_set_option("dist_fused", 0)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = None
    if world > 1 or args.dist:
        obj = [ley.ley_comm_get_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        comm = ley.ley_comm_init(world, rank, obj[0], local)

    res = measure(args, args.config, world, rank, local, comm)
    secondary = None
    if (world == 1 and comm is None and args.secondary not in ("", "none") and args.secondary != args.config
            and args.secondary in CONFIGS):
        torch.cuda.empty_cache()
        ley.ley_release_cache(-1)
        sec = measure(args, args.secondary, world, rank, local, comm, with_cpu=False)
        secondary = {k: sec[k] for k in ("value", "ms_per_step", "config", "roofline", "step_roofline", "stages_ms",
                                         "stage_pass", "e2e", "clocks", "gpu_launches")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": res["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded counter-based generator, SURVEY App. A)",
            "config": res["config"],
            "roofline": res["roofline"], "step_roofline": res["step_roofline"], "host_roofline": res["host_roofline"],
            "stages_ms": res["stages_ms"], "stage_pass": res["stage_pass"],
            "cpu_baseline": res["cpu_baseline"], "e2e": res["e2e"], "clocks": res["clocks"],
            "gpu_launches": res["gpu_launches"] + (secondary["gpu_launches"] if secondary else 0),
        }
        if secondary:
            line["secondary"] = secondary
        print(json.dumps(line), flush=True)
    if comm is not None:
        ley.ley_comm_destroy(comm)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
