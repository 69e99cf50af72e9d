#!/usr/bin/env python3
"""Per-kernel device times of the hull pipeline on the BASELINE configs.

Dev tool (runs on the GPU box): prints one line per kernel (mean ms over the
repeats) and the stage totals, and checks the hull against the CPU oracle
port once per config.
"""
import argparse
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402

CONFIGS = {
    "C1": ("square", 1_000_000),
    "C2": ("square", 20_000_000),
    "C3": ("disk", 20_000_000),
    "C4": ("circle", 20_000_000),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    import torch

    eng = Engine(0)
    for name in args.configs.split(","):
        kind, n = CONFIGS[name]
        t = time.time()
        xs, ys = generate(kind, n, 1)
        tg = time.time() - t
        dx = torch.from_numpy(xs).cuda()
        dy = torch.from_numpy(ys).cuda()
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        eng.reserve(n)
        for _ in range(2):
            eng.hull_device(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr(), n)
        eng.set_profiling(True)
        acc = defaultdict(float)
        tot = []
        for _ in range(args.reps):
            k, st = eng.hull_device(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr(), n)
            for kn, ms in eng.kernel_times():
                acc[kn] += ms / args.reps
            tot.append(st.t_total_ms)
        eng.set_profiling(False)
        walls = []
        for _ in range(args.reps):
            k, st = eng.hull_device(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr(), n)
            walls.append(st.t_total_ms)
        print(f"== {name} {kind} n={n} gen={tg:.2f}s r1={st.n_after_round1} r2={st.n_after_round2} "
              f"hull={st.hull_size} total_ms(median)={np.median(walls):.3f} "
              f"[r1 {st.t_round1_ms:.3f} ann {st.t_annotate_ms:.3f} sort {st.t_sort_ms:.3f} "
              f"r2 {st.t_round2_ms:.3f} fin {st.t_finalize_ms:.3f}] launches={eng.launch_count()}")
        for kn, ms in sorted(acc.items(), key=lambda kv: -kv[1]):
            print(f"   {kn:24s} {ms:9.4f} ms")
        if args.check:
            import oracle

            want, sw = oracle.full_pipeline(xs, ys)
            got = out[:k].cpu().numpy().astype(np.uint64)
            print("   parity:", "OK" if np.array_equal(got, want) else "MISMATCH",
                  sw["n_after_round2"], sw["hull_size"])
        del dx, dy, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
