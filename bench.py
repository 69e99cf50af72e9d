#!/usr/bin/env python3
"""Benchmark: Mpoints/s of the 20M-point 2D convex hull on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One JSON line on rank 0. A "step" is one full_pipeline over the 20M-point
uniform-square input (seed 1), the configuration BASELINE.json's metric is
quoted on (configs[1]). Keys:
  value      device-resident throughput: inputs already in HBM, K steps timed
             with CUDA events on the pipeline's stream (max over ranks)
  e2e        same metric through the C-ABI host entry (gscan_hull_f64) with
             pinned host buffers: H2D of xs/ys + pipeline + D2H of the index
             list inside the timed region
  roofline   the filter pass as the pipeline runs it: on the default sparse
             path k_sp_hist (round-1 quad test + angle-bucket histogram),
             algorithmic bytes 16 B/point read + 2 B/point bucket code written;
             on the full-sort path k_filter_keys (16 B/point + 16 B/survivor);
             over its event-timed duration, against MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the unmodified reference (oracle/_ref) on this host, one full
             run of the same workload, timed by its own StageStats
N > 1 runs the sharded pipeline (paper_1508_05931_b200/distributed.py) on the
same 20M points split across ranks (strong scaling).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Mpoints/s for 20M-pt 2D hull at 1/2/4/8 B200; filter-pass HBM GB/s vs peak"
CONFIGS = {
    "C1": ("square", 1_000_000, "C1: 1M points uniform in unit square, seed 1"),
    "C2": ("square", 20_000_000, "C2: 20M points uniform in unit square, seed 1"),
    "C3": ("disk", 20_000_000, "C3: 20M points uniform in unit disk, seed 1"),
    "C4": ("circle", 20_000_000, "C4: 20M points on the unit circle, seed 1"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every ~2 ms from a thread (nvidia-smi -lms cannot resolve a
    sub-second region); falls back to nvidia-smi when NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason* bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index: int):
        self.index = index
        self.sm: list[float] = []
        self.reasons: set[str] = set()
        self.sm_max = None
        self._run = False
        self._thr = None
        self._nvml = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nvml = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.sm_max = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None
        self._run = True
        self._thr = threading.Thread(target=self._loop, daemon=True)
        self._thr.start()

    def _sample(self):
        nv = self._nvml
        if nv is not None:
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)))
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            for name, bit in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
            return
        out = subprocess.run(
            ["nvidia-smi", f"--id={self.index}",
             "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits"],
            capture_output=True, text=True, timeout=5).stdout.strip().split(",")
        if len(out) >= 6:
            self.sm.append(float(out[0]))
            self.sm_max = float(out[1])
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"], out[2:6]):
                if v.strip().lower().startswith("active"):
                    self.reasons.add(name)

    def _loop(self):
        while self._run:
            try:
                self._sample()
            except Exception:
                pass
            time.sleep(0.002 if self._nvml is not None else 0.05)

    def stop(self) -> dict:
        self._run = False
        if self._thr:
            self._thr.join(timeout=5)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.sm_max, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.sm_max,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def hull_hash(idx: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(idx, dtype=np.uint64).tobytes()).hexdigest()[:16]


def golden_for(name: str):
    p = ROOT / "tests" / "golden" / "configs.json"
    if not p.exists():
        return None
    g = json.loads(p.read_text())
    return g.get(name)


def cpu_baseline(xs, ys, n) -> dict:
    """The reference itself (oracle/_ref) on this host: one full run."""
    import oracle

    if oracle.ref_available():
        _, st = oracle.full_pipeline(xs, ys, impl="ref")
        kind, cores = "reference", 2  # hull2d uses <= 2 threads (parallel.hpp:18-28)
    else:
        _, st = oracle.full_pipeline(xs, ys)
        kind, cores = "port", 1
    t = st["t_total_ms"]
    return {"value": round(n / (t * 1e-3) / 1e6, 3), "unit": "Mpoints/s", "cores": cores,
            "kind": kind, "t_total_ms": round(t, 1),
            "sample": f"1 full run of the same {n}-point input, timed by StageStats.t_total_ms"}


def run_reference(args, cfgname):
    """--impl reference: the reference's own CPU path (oracle/_ref) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_1508_05931_b200 import generate

    kind, n, label = CONFIGS[cfgname]
    xs, ys = generate(kind, n, 1)
    impl = "ref" if oracle.ref_available() else "port"
    times = []
    for s in range(args.warmup + args.steps):
        _, st = oracle.full_pipeline(xs, ys, impl=impl)
        if s >= args.warmup:
            times.append(st["t_total_ms"])
    t = float(np.sum(times)) / 1e3
    value = n * args.steps / t / 1e6
    line = {"metric": METRIC, "value": round(value, 4), "unit": "Mpoints/s", "impl": "reference",
            "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t * 1e3 / args.steps, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "n_points": n},
            "cpu_baseline": {"value": round(value, 4), "unit": "Mpoints/s",
                             "cores": 2 if impl == "ref" else 1,
                             "kind": "reference" if impl == "ref" else "port",
                             "sample": f"{args.steps} timed full runs after {args.warmup} warm-up"},
            "e2e": {"value": round(value, 4), "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch
    import torch.distributed as dist

    from paper_1508_05931_b200 import Engine, PipelineConfig, generate
    from paper_1508_05931_b200.distributed import sharded_hull

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    kind, n, label = CONFIGS[args.config]
    xs, ys = generate(kind, n, 1)  # identical bits on every rank (seeded)
    lo = n * rank // world
    hi = n * (rank + 1) // world
    eng = Engine(local)
    eng.reserve(n if world == 1 or rank == 0 else hi - lo)
    stream = torch.cuda.current_stream()
    eng._lib.gscan_set_stream(eng.handle, stream.cuda_stream)
    d_xs = torch.from_numpy(xs[lo:hi].copy()).cuda()
    d_ys = torch.from_numpy(ys[lo:hi].copy()).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    cfg = PipelineConfig()

    def step():
        if world == 1:
            k, st = eng.hull_device(d_xs.data_ptr(), d_ys.data_ptr(), n, out.data_ptr(), n, cfg)
            return k, st
        hull, st = sharded_hull(eng, d_xs, d_ys, lo, cfg)
        return (len(hull) if hull is not None else 0), st

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sampler = ClockSampler(local)
    # ---- correctness of the benchmarked output (golden hash from the reference) ----
    k, st = step()
    parity = None
    if rank == 0:
        if world == 1:
            got = out[:k].cpu().numpy().astype(np.uint64)
        else:
            got, _ = None, None
        g = golden_for(args.config)
        if g is not None and world == 1:
            parity = (hull_hash(got) == g["hull_sha256_16"] and st.n_after_round1 == g["n_after_round1"]
                      and st.n_after_round2 == g["n_after_round2"])
    for _ in range(max(args.warmup - 1, 0)):
        step()
    barrier()

    # ---- device-resident timed region (clocks sampled from warm-up through it) ----
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    sampler.start()
    barrier()
    e0.record(stream)
    launches = 0
    for _ in range(args.steps):
        step()
        launches += eng.launch_count()
    e1.record(stream)
    barrier()
    clocks = sampler.stop()
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    ms_per_step = t_ms / args.steps
    value = n / (ms_per_step * 1e-3) / 1e6

    # ---- filter-pass roofline (event-timed kernel durations, profiled pass) ----
    eng.set_profiling(True)
    kt = {}
    reps = 3
    for _ in range(reps):
        step()
        for name, ms in eng.kernel_times():
            kt.setdefault(name, []).append(ms)
    eng.set_profiling(False)
    kernels = {k2: round(float(np.mean(v)) * (len(v) / reps), 4) for k2, v in kt.items()}
    peak, peak_src = peaks()
    fkern = "k_sp_hist" if "k_sp_hist" in kt else "k_filter_keys"
    filt = kt.get(fkern, [])
    t_filter = float(np.mean(filt)) if filt else None
    n_local = hi - lo
    n1 = st.n_after_round1 if st is not None else None
    roofline = None
    if t_filter:
        if fkern == "k_sp_hist":  # 16 B/pt read (xs, ys) + 2 B/pt bucket code written
            alg_bytes = 18 * n_local
        else:
            alg_bytes = 16 * n_local + 16 * (n1 if (world == 1 and n1) else int(0.664 * n_local))
        achieved = alg_bytes / (t_filter * 1e-3) / 1e9
        traffic = None
        tp = ROOT / "profiles" / "ncu_filter_traffic.json"
        if tp.exists():
            try:
                traffic = json.loads(tp.read_text()).get(f"{fkern}:{args.config}")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/)",
                    "kernel": fkern, "kernel_ms": round(t_filter, 4),
                    "algorithmic_bytes": alg_bytes, "peak_source": peak_src}

    # ---- e2e through the C-ABI host entry, pinned host buffers ----
    e2e = None
    if world == 1:
        hx = torch.from_numpy(xs).pin_memory()
        hy = torch.from_numpy(ys).pin_memory()
        hout = torch.empty(n, dtype=torch.int64).pin_memory()
        kk = 0
        for _ in range(2):
            kk, _ = eng.hull_ptr(hx.data_ptr(), hy.data_ptr(), n, hout.data_ptr(), n, cfg)
        torch.cuda.synchronize()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            kk, _ = eng.hull_ptr(hx.data_ptr(), hy.data_ptr(), n, hout.data_ptr(), n, cfg)
        f1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = f0.elapsed_time(f1) / args.steps
        e2e = {"value": round(n / (e2e_ms * 1e-3) / 1e6, 3), "unit": "Mpoints/s",
               "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 4 * int(kk),
               "ms_per_step": round(e2e_ms, 3), "path": "gscan_hull_f64 (pinned host buffers)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(xs, ys, n)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpoints/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": label, "n_points": n, "seed": 1,
                   "l2": "inputs (320 MB) larger than the 126 MB L2; no flush needed",
                   "parallelism": f"sharded x{world}" if world > 1 else "single device",
                   "pipeline_config": "chunk_count=1024, both rounds, chunked"},
        "parity_vs_golden": parity,
        "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": launches, "kernels_ms": kernels, "sparse_path": eng.sparse_info()[0] == 1,
        "stats": {k2: getattr(st, k2) for k2 in ("n_after_round1", "n_after_round2", "hull_size")}
        if st is not None else None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
