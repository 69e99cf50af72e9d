"""Randomised parity stress on the device path: python tools/stress.py [cases] [seed] [--sharded]

Random families (uniform square/disk/circle, Gaussian, integer lattices with
duplicates, clustered blobs, thin annuli, points on a few lines), random sizes
(65K-1.5M, so both the sparse path and its declines run) and random pipeline
configs. Every case is compared bit for bit with the CPU oracle (indices and
stage counts). --sharded: the same cases as 2-4 simulated ranks with random
shard boundaries (the sharded sparse path, and the distributed sample sort
when it declines). Prints one line per failure and a summary."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
only = int(sys.argv[sys.argv.index("--only") + 1]) if "--only" in sys.argv else None
start = int(sys.argv[sys.argv.index("--from") + 1]) if "--from" in sys.argv else 0
oracle.port()
eng = Engine(0)


def make(kind, n):
    if kind in ("square", "disk", "circle"):
        return generate(kind, n, int(rng.integers(1, 1 << 30)))
    if kind == "gauss":
        return rng.standard_normal(n) * 1e3 + 5e5, rng.standard_normal(n)
    if kind == "lattice":  # many exact duplicates
        k = int(rng.integers(50, 3000))
        return rng.integers(0, k, n).astype(np.float64), rng.integers(0, k, n).astype(np.float64)
    if kind == "blobs":
        c = rng.uniform(-1, 1, (8, 2))
        w = rng.integers(0, 8, n)
        return c[w, 0] + rng.standard_normal(n) * 1e-3, c[w, 1] + rng.standard_normal(n) * 1e-3
    if kind == "annulus":
        t = rng.uniform(0, 2 * np.pi, n)
        r = 1 + rng.uniform(0, 1e-6, n)
        return r * np.cos(t), r * np.sin(t)
    # lines: points on 3 segments (collinear runs)
    s = rng.integers(0, 3, n)
    t = rng.uniform(0, 1, n)
    a = np.array([[0, 0], [1, 0], [0.5, 1]])
    b = np.roll(a, -1, axis=0)
    return a[s, 0] + t * (b[s, 0] - a[s, 0]), a[s, 1] + t * (b[s, 1] - a[s, 1])


kinds = ["square", "disk", "circle", "gauss", "lattice", "blobs", "annulus", "lines"]
SHARD_ENGINES = [Engine(0) for _ in range(4)] if "--sharded" in sys.argv else []
bad, sparse = 0, 0
for c in range(cases):
    kind = kinds[int(rng.integers(len(kinds)))]
    n = int(rng.integers(65_536, 1_500_000))
    cfg = dict(chunk_count=int(rng.choice([1, 7, 100, 1024, 5000])))
    if rng.random() < 0.15:
        cfg["chunked"] = False
    if rng.random() < 0.1:
        cfg["enable_round2"] = False
    xs, ys = make(kind, n)
    xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
    dev_entry = rng.random() < 0.5
    if (only is not None and c != only) or c < start:
        continue
    if "-v" in sys.argv:
        print(f"case {c}: {kind} n={n} cfg={cfg} device={dev_entry}", flush=True)
    if "--sharded" in sys.argv:  # R simulated ranks, random shard boundaries
        from paper_1508_05931_b200.distributed import simulate_sample_sort, simulate_sharded
        R = int(rng.integers(2, 5))
        cuts = np.sort(rng.choice(np.arange(1, n), R - 1, replace=False)).tolist()
        bounds = [0] + cuts + [n]
        engs = SHARD_ENGINES[:R]
        dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        res = simulate_sharded(engs, dx, dy, PipelineConfig(**cfg), bounds=bounds) \
            if (cfg.get("chunked", True) and cfg.get("enable_round2", True)) else None
        if res is None:  # declined (or a non-default config): the exact fallback
            res = simulate_sample_sort(engs, dx, dy, PipelineConfig(**cfg), bounds=bounds)
        else:
            sparse += 1
        got, st = res
        want, sw = oracle.full_pipeline(xs, ys, **cfg)
        ok = (np.array_equal(got, want) and st.n_after_round1 == sw["n_after_round1"]
              and st.n_after_round2 == sw["n_after_round2"] and st.hull_size == sw["hull_size"])
        if not ok:
            bad += 1
            print(f"FAIL case {c}: {kind} n={n} R={R} bounds={bounds} cfg={cfg}", flush=True)
        continue
    if dev_entry:  # the device entry (graph path) or the host entry (ingest)
        dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        k, st = eng.hull_device(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr(), n, PipelineConfig(**cfg))
        got = out[:k].cpu().numpy().astype(np.uint64)
    else:
        got, st = eng.hull_indices(xs, ys, PipelineConfig(**cfg))
    sparse += eng.sparse_info()[0] == 1
    want, sw = oracle.full_pipeline(xs, ys, **cfg)
    ok = (np.array_equal(got, want) and st.n_after_round1 == sw["n_after_round1"]
          and st.n_after_round2 == sw["n_after_round2"] and st.hull_size == sw["hull_size"])
    if not ok:
        bad += 1
        print(f"FAIL case {c}: {kind} n={n} cfg={cfg} got {len(got)} want {len(want)}", flush=True)
print(f"stress: {cases - bad}/{cases} bit-exact ({sparse} served by the sparse path)", flush=True)
sys.exit(1 if bad else 0)
