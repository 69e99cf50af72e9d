"""Device time per call for the BASELINE configs C1-C4 (seed 1), median of
5 warm calls, with the path taken. Usage: python tools/config_times.py"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402


def main():
    eng = Engine(0)
    for name, kind, n in (("C1", "square", 1_000_000), ("C2", "square", 20_000_000),
                          ("C3", "disk", 20_000_000), ("C4", "circle", 20_000_000)):
        xs, ys = generate(kind, n, 1)
        import torch
        dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        ts = []
        for _ in range(6):
            torch.cuda.synchronize()
            t = time.perf_counter()
            k, st = eng.hull_device(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t)
        used, fail, walked = eng.sparse_info()
        path, gf = eng.graham_info()
        print(f"{name} {kind:6s} n={n:>9d} hull={k:>9d} wall_ms={np.median(ts[1:]) * 1e3:8.3f} "
              f"dev_ms={st.t_total_ms:8.3f} sparse={used} fail={fail:#x} walked={walked} graham_path={path} "
              f"n1={st.n_after_round1} n2={st.n_after_round2} Mpts/s={n / np.median(ts[1:]) / 1e6:9.1f}",
              flush=True)


if __name__ == "__main__":
    main()
