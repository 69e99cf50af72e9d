#!/usr/bin/env python3
"""Benchmark: Mpoints/s of the 20M-point 2D convex hull on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C1..C5] [--impl ours|reference]

One JSON line on rank 0. A "step" is one full_pipeline over the configured
input (default C2: the 20M-point uniform square, seed 1, the configuration
BASELINE.json's metric is quoted on, configs[1]). --gpus N > 1 re-launches
this script under torch.distributed.run (one rank per GPU, 127.0.0.1) unless
it already runs under it. Keys:
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
  cpu_baseline  the unmodified reference (oracle/_ref) on this host: median of
             up to 5 full runs of the same workload (bounded to ~20 s), timed
             by its own StageStats; host nproc and CPU model stated
N > 1 runs the sharded pipeline (paper_1508_05931_b200/distributed.py): C1-C4
split the same points across ranks (strong scaling), C5 (1B points) is the
sharded config of BASELINE.json (each rank generates and owns its contiguous
shard of the same 1B-point sequence).
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
    "C5": ("square", 1_000_000_000, "C5: 1B points uniform in unit square, seed 1"),
}
KIND_CODE = {"square": 0, "disk": 1, "circle": 2, "collinear": 3}  # datagen.hpp / gscan.h
SEED = 1
PIPELINE_CONFIG = "chunk_count=1024, both rounds, chunked"


def config_dict(cfgname: str, world: int) -> dict:
    """The `config` object both arms print (identical, so the driver can pair them)."""
    kind, n, label = CONFIGS[cfgname]
    return {"workload": label, "n_points": n, "seed": SEED,
            "l2": f"inputs ({16 * n / 1e6:.0f} MB) larger than the 126 MB L2; no flush needed"
            if 16 * n > 126e6 else "inputs fit in L2 (C1: 16 MB); no flush (the reference's own size)",
            "parallelism": f"sharded x{world}" if world > 1 else "single device",
            "pipeline_config": PIPELINE_CONFIG}


def host_info() -> dict:
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def bind_near_gpu(index: int) -> int | None:
    """Pin this process to the CPUs NVML reports as nearest GPU `index`, so the
    pinned host buffers of the e2e leg are first-touched on the GPU's NUMA node
    and, on multi-socket hosts, its H2D copies do not cross the inter-socket
    link. Returns the CPU count, or None when NVML is unavailable."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(index)
        ncpu = os.cpu_count() or 1
        mask = nv.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        return len(cpus)
    except Exception:  # noqa: BLE001
        return None


def relaunch_distributed(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve())] + sys.argv[1:]
    log("+", " ".join(cmd))
    return subprocess.call(cmd)


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
    """The reference itself (oracle/_ref) on this host: median of up to 5 full
    runs (stops early once ~20 s of CPU work is spent), like cli::bench_one's
    median of repeats (cli.hpp:176-207)."""
    import oracle

    impl = "ref" if oracle.ref_available() else "port"
    times = []
    t_start = time.time()
    while len(times) < 5 and (not times or time.time() - t_start < 20.0):
        _, st = oracle.full_pipeline(xs, ys, impl=impl)
        times.append(st["t_total_ms"])
    t = float(np.median(times))
    # the reference's own baseline hull (cli.hpp:183-186: oracle::monotone_chain), one run
    t0 = time.perf_counter()
    oracle.monotone_chain(xs, ys, impl=impl)
    t_mc = (time.perf_counter() - t0) * 1e3
    return {"value": round(n / (t * 1e-3) / 1e6, 3), "unit": "Mpoints/s",
            "cores": 2 if impl == "ref" else 1,  # hull2d uses <= 2 threads (parallel.hpp:18-28)
            "kind": "reference" if impl == "ref" else "port", "t_total_ms": round(t, 1),
            "runs_ms": [round(v, 1) for v in times], **host_info(),
            "monotone_chain_ms": round(t_mc, 1),
            "sample": f"median of {len(times)} full runs of the same {n}-point input, "
                      "timed by StageStats.t_total_ms; monotone_chain_ms: one wall-clock run of "
                      "the reference's oracle::monotone_chain on it"}


def run_reference(args, cfgname):
    """--impl reference: the reference's own CPU path (oracle/_ref, the
    unmodified hull2d headers) on host cores. The input comes from the
    reference's own generator (datagen.hpp via oracle/_ref), so this arm loads
    nothing from the product package. Rank 0 only (other ranks exit 0)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import oracle

    kind, n, label = CONFIGS[cfgname]
    impl = "ref" if oracle.ref_available() else "port"
    cfg = config_dict(cfgname, world)
    if n > 200_000_000:
        # 1B points: ~35 s of single-threaded generation and ~64-100 GB RSS in
        # the reference; each step is a bounded sample instead.
        n_s = 100_000_000
        sample = f"{n_s}-point prefix of the same sequence per step (1B exceeds a bounded CPU run)"
    else:
        n_s = n
        sample = f"full {n}-point runs"
    xs, ys = (oracle.ref_generate(KIND_CODE[kind], n_s, SEED) if impl == "ref"
              else _port_generate(kind, n_s))
    times = []
    for s in range(args.warmup + args.steps):
        _, st = oracle.full_pipeline(xs, ys, impl=impl)
        if s >= args.warmup:
            times.append(st["t_total_ms"])
    t = float(np.sum(times)) / 1e3
    value = n_s * args.steps / t / 1e6
    line = {"metric": METRIC, "value": round(value, 4), "unit": "Mpoints/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t * 1e3 / args.steps, 2), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": {"value": round(value, 4), "unit": "Mpoints/s",
                             "cores": 2 if impl == "ref" else 1,
                             "kind": "reference" if impl == "ref" else "port", **host_info(),
                             "sample": f"{args.steps} timed {sample} after {args.warmup} warm-up"},
            "e2e": {"value": round(value, 4), "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _port_generate(kind, n):
    raise RuntimeError("oracle/_ref not built: the reference arm needs the reference's generator")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rc = relaunch_distributed(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        return run_reference(args, args.config)

    import torch
    import torch.distributed as dist

    from paper_1508_05931_b200 import Engine, PipelineConfig
    from paper_1508_05931_b200.distributed import sharded_hull

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    near_cpus = bind_near_gpu(local)
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    kind, n, label = CONFIGS[args.config]
    lo = n * rank // world
    hi = n * (rank + 1) // world
    eng = Engine(local)
    eng.reserve(n if world == 1 or rank == 0 else hi - lo)
    stream = torch.cuda.current_stream()
    eng._lib.gscan_set_stream(eng.handle, stream.cuda_stream)
    # every rank materialises only its own shard [lo, hi) of the seeded sequence
    d_xs, d_ys, gen_how = make_shard(eng, kind, n, lo, hi, torch)
    out = torch.empty(n if world == 1 else 1, dtype=torch.int32, device="cuda")
    cfg = PipelineConfig()

    last = {}

    def step():
        if world == 1:
            k, st = eng.hull_device(d_xs.data_ptr(), d_ys.data_ptr(), n, out.data_ptr(), n, cfg)
            return k, st
        hull, st = sharded_hull(eng, d_xs, d_ys, lo, cfg)
        last["hull"] = hull
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
            got = last["hull"]
        g = golden_for(args.config)
        if g is not None and got is not None:
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
        if world > 1:
            launches += eng.launch_count()
    e1.record(stream)
    if world == 1:  # every replay of the call's graph launches the same kernels
        launches = eng.launch_count() * args.steps
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
    # the filter pass of the path that served the call: F2 on the sparse path;
    # k_filter_keys when the sparse path declined (its k_sp_hist then exits at once)
    fkern = "k_sp_hist" if eng.sparse_info()[0] == 1 and "k_sp_hist" in kt else "k_filter_keys"
    filt = kt.get(fkern, [])
    t_filter = float(np.mean(filt)) if filt else None
    n_local = hi - lo
    n1 = st.n_after_round1 if st is not None else None
    roofline = None
    if t_filter:
        if fkern == "k_sp_hist":  # 16 B/pt read (xs, ys)
            alg_bytes = 16 * n_local
        else:
            # 16 B/pt read + (survivor index, key, rank) = 16 B/survivor written
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
                    "algorithmic_bytes": alg_bytes, "peak_source": peak_src,
                    # the whole device-resident hull against one 16 B/pt read
                    "whole_call_frac": round(16 * n / (ms_per_step * 1e-3) / 1e9 / peak, 4)}

    # ---- sort throughput (keys/s, north star): the sort kernels of the path that served ----
    sort = None
    if world == 1:
        if eng.sparse_info()[0] == 1:  # gathered buckets + walk candidates, placed and sorted exactly
            names = ("k_sp_place_g", "k_sp_sort_gathered", "k_sp_sort_gathered_big",
                     "k_sp_sort_gathered_huge", "k_sp_rank_c", "k_sp_place_c", "k_sp_place_cand",
                     "k_sp_sort_cand_big", "k_sp_place_gathered")
            nkeys = int(eng.sparse_info()[2])  # the walk array: anchor + gathered + candidates
            what = "gathered points + walk candidates (sparse path)"
        else:  # every annotated survivor: bucket offsets, scatter, per-bucket sorts
            names = ("k_scan_u32", "k_scatter", "k_bucket_sort_block", "k_bucket_sort_cta")
            nkeys = int(n1) if n1 else 0
            what = "round-1 survivors (full sort: bucket scatter + per-bucket sorts)"
        t_sort = sum(kernels.get(k2, 0.0) for k2 in names)
        if t_sort > 0 and nkeys:
            sort = {"keys": nkeys, "ms": round(t_sort, 4),
                    "gkeys_per_s": round(nkeys / (t_sort * 1e-3) / 1e9, 3), "what": what}

    # ---- e2e: host buffers in, hull indices out, copies inside the timed region ----
    e2e = None
    n_local = hi - lo
    need = 16 * n_local * 2 + 8 * n
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = need * 4
    if need * 1.5 > avail:
        e2e = {"value": None, "unit": "Mpoints/s", "h2d_bytes_per_step": 16 * n_local,
               "d2h_bytes_per_step": None,
               "skipped": f"pinned host copy of the shard ({need / 1e9:.1f} GB) exceeds host RAM"}
    else:
        hx = torch.empty(n_local, dtype=torch.float64).pin_memory()
        hy = torch.empty(n_local, dtype=torch.float64).pin_memory()
        hx.copy_(d_xs)
        hy.copy_(d_ys)
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        if world == 1:
            # the reference-facing C-ABI host entry gscan_hull_f64 (include/gscan.h)
            hout = torch.empty(n, dtype=torch.int64).pin_memory()
            kk = 0
            for _ in range(2):
                kk, _ = eng.hull_ptr(hx.data_ptr(), hy.data_ptr(), n, hout.data_ptr(), n, cfg)
            torch.cuda.synchronize()
            f0.record(stream)
            for _ in range(args.steps):
                kk, _ = eng.hull_ptr(hx.data_ptr(), hy.data_ptr(), n, hout.data_ptr(), n, cfg)
            f1.record(stream)
            torch.cuda.synchronize()
            d2h = 8 * int(kk)
            path = "gscan_hull_f64 (pinned host buffers)"
        else:
            # each rank copies its shard in, sharded_hull returns the index list on rank 0
            kk = 0

            def e2e_step():
                d_xs.copy_(hx, non_blocking=True)
                d_ys.copy_(hy, non_blocking=True)
                hull, _ = sharded_hull(eng, d_xs, d_ys, lo, cfg)
                return len(hull) if hull is not None else 0

            for _ in range(2):
                e2e_step()
            barrier()
            f0.record(stream)
            for _ in range(args.steps):
                kk = e2e_step()
            f1.record(stream)
            barrier()
            d2h = 8 * int(kk)
            path = "distributed.sharded_hull (pinned host shard per rank)"
        e2e_ms = f0.elapsed_time(f1) / args.steps
        if world > 1:
            tt = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": round(n / (e2e_ms * 1e-3) / 1e6, 3), "unit": "Mpoints/s",
               "h2d_bytes_per_step": 16 * n_local, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(e2e_ms, 3), "path": path,
               "cpu_affinity": f"{near_cpus} CPUs nearest the GPU (NVML)" if near_cpus else "unbound"}
        del hx, hy

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        n_cpu = min(n, 20_000_000)
        hx = d_xs[:n_cpu].cpu().numpy()
        hy = d_ys[:n_cpu].cpu().numpy()
        cpu = cpu_baseline(hx, hy, n_cpu)
        if n_cpu < n:
            cpu["sample"] += f" (the first {n_cpu} points of the {n}-point sequence: bounded sample)"
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpoints/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic ({gen_how})",
        "config": config_dict(args.config, world),
        "parity_vs_golden": parity,
        "e2e": e2e, "roofline": roofline, "sort": sort, "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": launches, "kernels_ms": kernels, "sparse_path": eng.sparse_info()[0] == 1,
        "stats": {k2: getattr(st, k2) for k2 in ("n_after_round1", "n_after_round2", "hull_size")}
        if st is not None else None,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def make_shard(eng, kind, n, lo, hi, torch):
    """Device-resident SoA shard [lo, hi) of gen_<kind>(n, seed 1)
    (datagen.hpp:32-71): the on-device mt19937_64 generator for squares
    (bit-identical to the host sequence), else the host generator."""
    if kind == "square" and hasattr(eng, "generate_square_device"):
        d_xs = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        d_ys = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        eng.generate_square_device(SEED, lo, hi, d_xs.data_ptr(), d_ys.data_ptr())
        torch.cuda.synchronize()
        return d_xs, d_ys, "gen_square on the device (mt19937_64, bit-identical to datagen.hpp)"
    if n > 200_000_000:
        raise SystemExit(f"{kind} with {n} points needs the on-device generator")
    from paper_1508_05931_b200 import generate

    xs, ys = generate(kind, n, SEED)  # identical bits on every rank (seeded)
    d_xs = torch.from_numpy(xs[lo:hi].copy()).cuda()
    d_ys = torch.from_numpy(ys[lo:hi].copy()).cuda()
    return d_xs, d_ys, f"gen_{kind} on the host (datagen.hpp sequence)"


if __name__ == "__main__":
    main()
