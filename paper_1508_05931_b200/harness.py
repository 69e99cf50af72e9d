"""Bench / verify harness with the reference CLI's outputs.

``bench`` mirrors ``cli::cmd_bench`` / ``bench_one`` (cli.hpp:176-238): one CSV
row per dataset with the reference's exact header (``kCsvHeader``,
cli.hpp:37-39), per-column medians over ``repeats`` runs, the '#'-prefixed
summary line (cli.hpp:69-81), plus GPU columns appended after the reference's
(which path served the call, and the wall time of the host-buffer call that
includes the H2D copy). ``baseline_ms`` is the monotone chain's wall time as
in the reference, computed here only when asked (it is a CPU O(n log n) run).

``verify`` mirrors ``cli::cmd_verify`` / ``check_case`` (cli.hpp:243-378) over
the GPU stage outputs: every point the GPU round 1 discards and every point
the GPU round-2 walk discards must be strictly inside the monotone-chain hull,
and the pipeline's hull must have the oracle's vertex set; the default matrix
is the reference's (square, disk, circle, collinear x seeds, tiny sizes, an
all-duplicate set) under chunk counts {1, 7, 1024} and the sequential walk.
``inject_fault`` flips one kept hull vertex to "discarded" and must fail.

The monotone chain and the hull tests here are a self-contained restatement of
``oracle::monotone_chain`` / ``strictly_inside_hull`` / ``same_vertex_set``
(oracle.hpp:40-142), in plain IEEE double arithmetic without FMA.

    python -m paper_1508_05931_b200.harness bench --dataset square --n 20000000 --seed 1
    python -m paper_1508_05931_b200.harness verify --seeds 50 --n 2000
"""
from __future__ import annotations

import argparse
import statistics
import sys
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .hull2d import Engine, PipelineConfig, generate

CSV_HEADER = ("dataset,n,seed,chunks,n_after_r1,n_after_r2,hull_size,t_r1_ms,t_annotate_ms,t_sort_ms,"
              "t_r2_ms,t_finalize_ms,t_total_ms,baseline_ms,speedup,remaining_r1_pct,remaining_r2_pct")
GPU_COLUMNS = "device,path,t_wall_ms"


# ---------------------------------------------------------------------------
# oracle hull (oracle.hpp:40-142)
def _orient(ax, ay, bx, by, cx, cy):
    """sign of (b - a) x (c - a) (geom.hpp:16-31), unfused double arithmetic."""
    return (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)


def monotone_chain(xs: np.ndarray, ys: np.ndarray) -> np.ndarray:
    """Andrew's monotone chain over the distinct points -> (k, 2) CCW vertices,
    collinear points dropped (oracle.hpp:40-79)."""
    if len(xs) == 0:
        raise ValueError("monotone_chain: no points")
    pts = np.unique(np.stack([np.asarray(xs, np.float64), np.asarray(ys, np.float64)], 1), axis=0)
    pts = [(float(x), float(y)) for x, y in pts]  # lexicographic (x, y)
    if len(pts) == 1:
        return np.array(pts)
    ring: list[tuple[float, float]] = []
    for p in pts:  # lower chain, left to right
        while len(ring) >= 2 and not _orient(*ring[-2], *ring[-1], *p) > 0:
            ring.pop()
        ring.append(p)
    lower = len(ring)
    for p in reversed(pts[:-1]):  # upper chain, right to left
        while len(ring) > lower and not _orient(*ring[-2], *ring[-1], *p) > 0:
            ring.pop()
        ring.append(p)
    ring.pop()  # the first point closes the ring
    return np.array(ring)


def strictly_inside(hull: np.ndarray, px: np.ndarray, py: np.ndarray) -> np.ndarray:
    """Per point: strictly Left of every CCW hull edge (oracle.hpp:126-133)."""
    px = np.asarray(px, np.float64)
    py = np.asarray(py, np.float64)
    if len(hull) < 3:
        return np.zeros(px.shape, bool)
    inside = np.ones(px.shape, bool)
    for i in range(len(hull)):
        ax, ay = hull[i]
        bx, by = hull[(i + 1) % len(hull)]
        e1 = (bx - ax) * (py - ay)
        e2 = (by - ay) * (px - ax)
        inside &= (e1 - e2) > 0
    return inside


def same_vertex_set(a: np.ndarray, b: np.ndarray) -> bool:
    sa = sorted(map(tuple, np.asarray(a).reshape(-1, 2).tolist()))
    sb = sorted(map(tuple, np.asarray(b).reshape(-1, 2).tolist()))
    return sa == sb


# ---------------------------------------------------------------------------
# verify
@dataclass
class Violation:
    label: str
    seed: int
    chunk_count: int
    chunked: bool
    reason: str
    point: tuple[float, float]

    def __str__(self) -> str:
        seq = "" if self.chunked else " (sequential)"
        return (f"verify: FAIL dataset={self.label} seed={self.seed} chunks={self.chunk_count}{seq} "
                f"point=({self.point[0]!r}, {self.point[1]!r}): {self.reason}")


def check_case(eng: Engine, label: str, seed: int, xs: np.ndarray, ys: np.ndarray,
               oracle_hull: np.ndarray, cfg: PipelineConfig, inject_fault: bool = False):
    """cli::check_case (cli.hpp:261-313) with every stage run on the GPU."""
    import torch

    def fail(reason, p):
        return Violation(label, seed, cfg.chunk_count, cfg.chunked, reason, (float(p[0]), float(p[1])))

    px, py = np.asarray(xs, np.float64), np.asarray(ys, np.float64)
    if cfg.enable_round1 and len(px) >= 1:
        dx, dy = torch.from_numpy(px).cuda(), torch.from_numpy(py).cuda()
        out = torch.empty(max(len(px), 1), dtype=torch.int32, device="cuda")
        k = eng.stage_round1(dx.data_ptr(), dy.data_ptr(), len(px), out.data_ptr())
        keep = np.zeros(len(px), bool)
        keep[out[:k].cpu().numpy()] = True
        bad = ~keep & ~strictly_inside(oracle_hull, px, py)
        if bad.any():
            i = int(np.flatnonzero(bad)[0])
            return fail("round-1 discarded a non-interior point", (px[i], py[i]))
        px, py = px[keep], py[keep]
    m = 0
    if cfg.enable_round2 and len(px) >= 1:
        dx, dy = torch.from_numpy(px).cuda(), torch.from_numpy(py).cuda()
        buf = torch.empty(len(px), dtype=torch.int32, device="cuda")
        m = eng.stage_sorted(dx.data_ptr(), dy.data_ptr(), len(px), buf.data_ptr())
    if m >= 2:  # the annotated (deduplicated) buffer, as cli.hpp:285
        flags = torch.empty(len(px), dtype=torch.uint8, device="cuda")
        eng.stage_discard(dx.data_ptr(), dy.data_ptr(), len(px), cfg.chunk_count, cfg.chunked,
                          flags.data_ptr())
        order = buf[:m].cpu().numpy()
        fl = flags[:m].cpu().numpy().astype(bool)
        if inject_fault:
            hv = set(map(tuple, oracle_hull.tolist()))
            for j in range(1, m):
                if (px[order[j]], py[order[j]]) in hv:
                    fl[j] = False
                    break
        gone = order[~fl]
        bad = ~strictly_inside(oracle_hull, px[gone], py[gone])
        if bad.any():
            i = int(gone[np.flatnonzero(bad)[0]])
            return fail("round-2 discarded a non-interior point", (px[i], py[i]))
    idx, _ = eng.hull_indices(np.asarray(xs, np.float64), np.asarray(ys, np.float64), cfg)
    got = np.stack([np.asarray(xs)[idx.astype(np.int64)], np.asarray(ys)[idx.astype(np.int64)]], 1)
    if not same_vertex_set(got, oracle_hull):
        gs = set(map(tuple, got.tolist()))
        off = next((v for v in map(tuple, oracle_hull.tolist()) if v not in gs), (0.0, 0.0))
        return fail("hull vertex set differs from oracle", off)
    return None


def default_matrix(seeds: int, n: int):
    """cli::default_matrix (cli.hpp:327-342)."""
    cases = []
    for s in range(seeds):
        for kind, m in (("square", n), ("disk", n), ("circle", max(n, 3)), ("collinear", n)):
            cases.append((kind, s, *generate(kind, m, s)))
    for tiny in (1, 2, 3):
        cases.append((f"square-n{tiny}", 7, *generate("square", tiny, 7)))
        cases.append((f"collinear-n{tiny}", 7, *generate("collinear", tiny, 7)))
    cases.append(("duplicate", 0, np.full(5, 0.25), np.full(5, 0.5)))
    return cases


def verify(seeds: int = 50, n: int = 2000, chunk_counts=(1, 7, 1024), include_sequential=True,
           inject_fault: bool = False, out=sys.stdout, eng: Engine | None = None) -> int:
    """cli::cmd_verify (cli.hpp:344-378): 0 on PASS, 1 on the first violation."""
    eng = eng or Engine(0)
    cases = default_matrix(seeds, n)
    configs = [PipelineConfig(chunk_count=k, chunked=True) for k in chunk_counts]
    if include_sequential:
        configs.append(PipelineConfig(chunked=False))
    for ci, (label, seed, xs, ys) in enumerate(cases):
        hull = monotone_chain(xs, ys)
        for gi, cfg in enumerate(configs):
            v = check_case(eng, label, seed, xs, ys, hull, cfg, inject_fault and ci == 0 and gi == 0)
            if v is not None:
                print(v, file=out)
                return 1
    print(f"verify: PASS ({len(cases)} datasets x {len(configs)} configs)", file=out)
    return 0


# ---------------------------------------------------------------------------
# bench
def bench_one(eng: Engine, kind: str, n: int, seed: int, cfg: PipelineConfig, repeats: int = 5,
              baseline: bool = False) -> dict:
    """cli::bench_one (cli.hpp:176-207): medians per column; GPU columns added."""
    xs, ys = generate(kind, n, seed)
    cols = {f: [] for f in ("t_round1_ms", "t_annotate_ms", "t_sort_ms", "t_round2_ms",
                            "t_finalize_ms", "t_total_ms")}
    walls, base = [], []
    st = None
    for _ in range(repeats):
        if baseline:
            t = time.perf_counter()
            monotone_chain(xs, ys)
            base.append((time.perf_counter() - t) * 1e3)
        t = time.perf_counter()
        idx, st = eng.hull_indices(xs, ys, cfg)
        walls.append((time.perf_counter() - t) * 1e3)
        for f in cols:
            cols[f].append(getattr(st, f))
    row = {"dataset": kind, "n": st.n_input, "seed": seed, "chunks": cfg.chunk_count,
           "n_after_r1": st.n_after_round1, "n_after_r2": st.n_after_round2,
           "hull_size": st.hull_size}
    for f, short in (("t_round1_ms", "t_r1_ms"), ("t_annotate_ms", "t_annotate_ms"),
                     ("t_sort_ms", "t_sort_ms"), ("t_round2_ms", "t_r2_ms"),
                     ("t_finalize_ms", "t_finalize_ms"), ("t_total_ms", "t_total_ms")):
        row[short] = statistics.median(cols[f])
    row["baseline_ms"] = statistics.median(base) if base else None
    row["speedup"] = row["baseline_ms"] / row["t_total_ms"] if base else None
    row["remaining_r1_pct"] = 100.0 * st.n_after_round1 / st.n_input
    row["remaining_r2_pct"] = 100.0 * st.n_after_round2 / st.n_input
    import torch

    row["device"] = torch.cuda.get_device_name(0).replace(",", " ")
    row["path"] = "sparse" if eng.sparse_info()[0] else "full-sort"
    row["t_wall_ms"] = statistics.median(walls)
    return row


def csv_row(r: dict) -> str:
    """cli::csv_row (cli.hpp:51-66) + the GPU columns."""
    f6 = lambda v: f"{v:.6f}"  # noqa: E731
    parts = [r["dataset"], str(r["n"]), str(r["seed"]), str(r["chunks"]), str(r["n_after_r1"]),
             str(r["n_after_r2"]), str(r["hull_size"]), f6(r["t_r1_ms"]), f6(r["t_annotate_ms"]),
             f6(r["t_sort_ms"]), f6(r["t_r2_ms"]), f6(r["t_finalize_ms"]), f6(r["t_total_ms"]),
             "" if r["baseline_ms"] is None else f6(r["baseline_ms"]),
             "" if r["speedup"] is None else f6(r["speedup"]), f6(r["remaining_r1_pct"]),
             f6(r["remaining_r2_pct"]), r["device"], r["path"], f6(r["t_wall_ms"])]
    return ",".join(parts)


def summary_line(r: dict) -> str:
    """cli::summary_line (cli.hpp:69-81)."""
    s = (f"# dataset={r['dataset']} n={r['n']} seed={r['seed']} chunks={r['chunks']} "
         f"n_after_r1={r['n_after_r1']} n_after_r2={r['n_after_r2']} hull_size={r['hull_size']} "
         f"t_total_ms={r['t_total_ms']:.3f} remaining_r1_pct={r['remaining_r1_pct']:.3f} "
         f"remaining_r2_pct={r['remaining_r2_pct']:.3f}")
    if r["baseline_ms"] is not None:
        s += f" baseline_ms={r['baseline_ms']:.3f} speedup={r['speedup']:.3f}"
    return s + f" path={r['path']} t_wall_ms={r['t_wall_ms']:.3f}"


def bench(specs, cfg: PipelineConfig, repeats: int = 5, csv_path: str | None = None,
          baseline: bool = False, out=sys.stdout, eng: Engine | None = None) -> int:
    """cli::cmd_bench (cli.hpp:209-238): header once (append mode keeps it), a
    row per dataset; the summary goes to `out` when the CSV goes to a file."""
    if repeats < 1:
        raise ValueError("bench: repeats must be >= 1")
    eng = eng or Engine(0)
    f = None
    header = True
    if csv_path:
        p = Path(csv_path)
        header = not p.exists() or p.stat().st_size == 0
        f = p.open("a")
    csv = f or out
    if header:
        print(CSV_HEADER + "," + GPU_COLUMNS, file=csv)
    for kind, n, seed in specs:
        r = bench_one(eng, kind, n, seed, cfg, repeats, baseline)
        print(csv_row(r), file=csv, flush=True)
        if f:
            print(summary_line(r), file=out)
    if f:
        f.close()
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1508_05931_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--dataset", action="append", default=None,
                   help="kind[:n[:seed]] (square, disk, circle, collinear); repeatable")
    b.add_argument("--n", type=int, default=1_000_000)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--chunks", type=int, default=1024)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--csv", default=None)
    b.add_argument("--baseline", action="store_true", help="also time the CPU monotone chain")
    v = sub.add_parser("verify")
    v.add_argument("--seeds", type=int, default=50)
    v.add_argument("--n", type=int, default=2000)
    v.add_argument("--chunks", type=int, nargs="*", default=[1, 7, 1024])
    v.add_argument("--no-sequential", action="store_true")
    v.add_argument("--inject-fault", action="store_true")
    a = ap.parse_args(argv)
    if a.cmd == "bench":
        specs = []
        for d in a.dataset or ["square"]:
            parts = d.split(":")
            specs.append((parts[0], int(parts[1]) if len(parts) > 1 else a.n,
                          int(parts[2]) if len(parts) > 2 else a.seed))
        return bench(specs, PipelineConfig(chunk_count=a.chunks), a.repeats, a.csv, a.baseline)
    return verify(a.seeds, a.n, tuple(a.chunks), not a.no_sequential, a.inject_fault)


if __name__ == "__main__":
    sys.exit(main())
