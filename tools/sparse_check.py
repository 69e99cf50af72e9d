"""GPU dev check: sparse round-2 path vs the full-sort path (both native) on
the BASELINE configs and extra seeds/shapes; prints fail bits, walked sizes
and per-call device times. Usage: python tools/sparse_check.py [n]"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402
from paper_1508_05931_b200 import _native as N  # noqa: E402


def run(eng, xs, ys, debug):
    eng.set_debug(debug)
    t = time.perf_counter()
    idx, st = eng.hull_indices(xs, ys, PipelineConfig())
    return idx, st, time.perf_counter() - t


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
    eng = Engine(0)
    cases = [("square", n, 1), ("disk", n, 1), ("circle", n, 1), ("square", 1_000_000, 1)]
    cases += [("square", n // 4, s) for s in (2, 3, 4, 5)] + [("disk", n // 4, 7)]
    bad = 0
    for kind, m, seed in cases:
        xs, ys = generate(kind, m, seed)
        want, sw, tw = run(eng, xs, ys, N.DEBUG_FULL_SORT)
        got, sg, tg = run(eng, xs, ys, 0)
        used, fail, walked = eng.sparse_info()
        same = np.array_equal(want, got) and all(
            getattr(sw, k) == getattr(sg, k) for k in ("n_after_round1", "n_after_round2", "hull_size"))
        bad += not same
        print(f"{kind:7s} n={m:>9d} seed={seed} same={same} used={used} fail={fail:#x} walked={walked} "
              f"n1={sg.n_after_round1} n2={sg.n_after_round2}/{sw.n_after_round2} hull={sg.hull_size} "
              f"dev_ms full={sw.t_total_ms:.3f} sparse={sg.t_total_ms:.3f} "
              f"[r1 {sg.t_round1_ms:.3f} ann {sg.t_annotate_ms:.3f} sort {sg.t_sort_ms:.3f} "
              f"r2 {sg.t_round2_ms:.3f} fin {sg.t_finalize_ms:.3f}]", flush=True)
    # duplicates: the sparse path must decline and the answer must still match
    xs, ys = generate("square", n // 4, 9)
    edge = np.flatnonzero(ys < 0.01)  # round-1 survivors near the bottom edge
    xs[edge[1::50]] = xs[edge[0::50][: len(edge[1::50])]]
    ys[edge[1::50]] = ys[edge[0::50][: len(edge[1::50])]]
    want, sw, _ = run(eng, xs, ys, N.DEBUG_FULL_SORT)
    got, sg, _ = run(eng, xs, ys, 0)
    used, fail, walked = eng.sparse_info()
    print(f"dups: same={np.array_equal(want, got)} used={used} fail={fail:#x}")
    # dropped candidates: verification must reject, result still exact
    xs, ys = generate("square", n // 4, 3)
    want, sw, _ = run(eng, xs, ys, N.DEBUG_FULL_SORT)
    got, sg, _ = run(eng, xs, ys, N.DEBUG_SPARSE_DROP)
    used, fail, walked = eng.sparse_info()
    print(f"drop: same={np.array_equal(want, got)} used={used} fail={fail:#x}")
    got, sg, _ = run(eng, xs, ys, N.DEBUG_SPARSE_VERIFY)
    used, fail, walked = eng.sparse_info()
    print(f"forced verify: same={np.array_equal(want, got)} used={used} fail={fail:#x}")
    eng.set_debug(0)
    eng.set_profiling(True)
    xs, ys = generate("square", n, 1)
    for _ in range(3):
        eng.hull_indices(xs, ys, PipelineConfig())
    for name, ms in eng.kernel_times():
        print(f"  {name:28s} {ms * 1e3:9.1f} us")
    tot = sum(ms for _, ms in eng.kernel_times())
    print(f"  sum of kernel times {tot * 1e3:.1f} us")
    for flag, nm in ((N.DEBUG_FORCE_SEQUENTIAL, "graham sequential-candidate"),
                     (N.DEBUG_FORCE_PREFIX, "graham prefix")):
        eng.set_debug(flag)
        eng.hull_indices(xs, ys, PipelineConfig())
        ks = [(a, b) for a, b in eng.kernel_times() if "graham" in a or a == "k_gather_chains"]
        print(f"  {nm}: " + ", ".join(f"{a} {b * 1e3:.1f}" for a, b in ks)
              + f" | total {sum(b for _, b in ks) * 1e3:.1f} us")
    eng.set_debug(0)
    print("BAD" if bad else "ALL SAME")


if __name__ == "__main__":
    main()
