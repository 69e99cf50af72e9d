#!/usr/bin/env python3
"""Generate the golden fixtures from the UNMODIFIED reference.

Runs in the CPU container (needs oracle/_ref/libhull2d_ref.so, built by
`make -C oracle` from /root/reference/proj/include). Inputs come from the
reference's own generators (datagen.hpp) through the same C-ABI, and the
script checks that our harness generator (gscan_generate) is bit-identical.

Outputs (committed):
  configs.json  BASELINE configs C1-C4 (seed 1): input hashes, stage counts,
                hull index list (or its hash for the 20M-vertex circle)
  corpus.json   known-answer corpus: small seeded inputs x pipeline configs,
                full hull index lists and stage counts
  stages.json   stage-level goldens: extremes, sorted buffer, discard flags
  extra.json    C2-C4 at seeds 2-5 (SURVEY.md 8(d) secondary seeds) and the
                uniform square at 100M and 200M points (seed 1), the sizes
                where the sparse path's buckets outgrow shared memory
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1508_05931_b200 import generate, generate_grid  # noqa: E402

HERE = Path(__file__).resolve().parent
KINDS = {"square": 0, "disk": 1, "circle": 2, "collinear": 3}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def gen(kind, n, seed):
    if kind == "grid":
        return generate_grid(n, seed)
    xs, ys = oracle.ref_generate(KINDS[kind], n, seed)
    mx, my = generate(kind, n, seed)
    assert np.array_equal(xs.view(np.uint64), mx.view(np.uint64)), (kind, n, seed)
    assert np.array_equal(ys.view(np.uint64), my.view(np.uint64)), (kind, n, seed)
    return xs, ys


def run(xs, ys, **cfg):
    idx, st = oracle.full_pipeline(xs, ys, impl="ref", **cfg)
    return idx, {k: int(st[k]) for k in ("n_input", "n_after_round1", "n_after_round2", "hull_size")}


def configs():
    out = {}
    for name, kind, n in (("C1", "square", 1_000_000), ("C2", "square", 20_000_000),
                          ("C3", "disk", 20_000_000), ("C4", "circle", 20_000_000)):
        xs, ys = gen(kind, n, 1)
        idx, st = run(xs, ys)
        rec = {"kind": kind, "n": n, "seed": 1, "xs_sha256_16": sha(xs), "ys_sha256_16": sha(ys),
               **st, "hull_sha256_16": sha(idx.astype(np.uint64))}
        if idx.size <= 5000:
            rec["hull"] = [int(v) for v in idx]
        out[name] = rec
        print(name, st, flush=True)
    (HERE / "configs.json").write_text(json.dumps(out, indent=1) + "\n")


CFGS = [dict(), dict(chunk_count=1), dict(chunk_count=2), dict(chunk_count=7),
        dict(chunk_count=64), dict(enable_round1=False), dict(enable_round2=False),
        dict(enable_round1=False, enable_round2=False), dict(chunked=False)]


def corpus():
    cases = []
    for kind in ("square", "disk", "circle", "collinear", "grid"):
        for n in (1, 2, 3, 10, 100, 1000, 10000):
            for seed in (0, 1, 2):
                xs, ys = gen(kind, n, seed)
                for ci, cfg in enumerate(CFGS):
                    if n >= 10000 and ci not in (0, 1, 5, 8):
                        continue
                    idx, st = run(xs, ys, **cfg)
                    cases.append({"kind": kind, "n": n, "seed": seed, "cfg": cfg,
                                  "xs_sha256_16": sha(xs), **st,
                                  "hull": [int(v) for v in idx]})
    # the reference's own hand-written known answers (test_pipeline.cpp:19-28, 92-107)
    hand = [
        [[0, 0], [1, 0], [1, 1], [0, 1]],
        [[0, 0], [1, 0], [2, 0]],
        [[2, 3]],
        [[2, 3], [0, 1]],
        [[0, 0], [1, 0], [2, 0], [1, 0]],
        [[1, 1]] * 6,
        [[0, 0], [3, 1], [1, 4]],
        [[0.0, 0.0], [-0.0, 0.0], [1, 1], [-0.0, -0.0]],
        [[0, 0], [4, 1], [2, 1], [0, 5]],
    ]
    for pts in hand:
        p = np.array(pts, dtype=np.float64)
        for cfg in (dict(), dict(chunk_count=1), dict(chunked=False), dict(enable_round1=False)):
            idx, st = run(p[:, 0], p[:, 1], **cfg)
            cases.append({"kind": "hand", "points": [[float(a), float(b)] for a, b in pts],
                          "cfg": cfg, **st, "hull": [int(v) for v in idx]})
    (HERE / "corpus.json").write_text(json.dumps(cases) + "\n")
    print("corpus cases:", len(cases))


def stages():
    out = []
    for kind, n, seed in (("square", 5000, 3), ("disk", 5000, 4), ("circle", 3000, 5),
                          ("grid", 3000, 6), ("square", 200000, 7)):
        xs, ys = gen(kind, n, seed)
        q = np.zeros(4, np.uint64)
        oracle.ref().ref_find_extremes(oracle._d(xs), oracle._d(ys), n, oracle._u(q))
        flags = np.empty(n, np.uint8)
        oracle.ref().ref_classify(oracle._d(xs), oracle._d(ys), n, flags.ctypes.data_as(oracle._U8P))
        sidx, ang, d2 = oracle.ref_sorted_buffer(xs, ys)
        rec = {"kind": kind, "n": n, "seed": seed, "quad": [int(v) for v in q],
               "anchor": int(oracle.select_anchor(xs, ys)),
               "r1_survivors_sha256_16": sha(np.nonzero(flags)[0].astype(np.uint64)),
               "n_r1": int(flags.sum()),
               "sorted_len": int(sidx.size), "sorted_sha256_16": sha(sidx.astype(np.uint64)),
               "angles_sha256_16": sha(ang)}
        for chunks, chunked in ((1024, True), (7, True), (1, True), (1024, False)):
            f, l = oracle.ref_discard_flags(xs, ys, chunks, chunked)
            rec[f"discard_{chunks}_{int(chunked)}"] = {"longest": int(l),
                                                       "flags_sha256_16": sha(f[: sidx.size]),
                                                       "kept": int(f[: sidx.size].sum())}
        out.append(rec)
    (HERE / "stages.json").write_text(json.dumps(out, indent=1) + "\n")
    print("stage cases:", len(out))


def extra():
    out = {}
    cases = [(f"{c}s{sd}", kind, 20_000_000, sd) for sd in (2, 3, 4, 5)
             for c, kind in (("C2", "square"), ("C3", "disk"), ("C4", "circle"))]
    cases += [("S100M", "square", 100_000_000, 1), ("S200M", "square", 200_000_000, 1)]
    for name, kind, n, sd in cases:
        if n > 50_000_000:  # the reference's generator alone (RSS); ours is checked on the GPU
            xs, ys = oracle.ref_generate(KINDS[kind], n, sd)
        else:
            xs, ys = gen(kind, n, sd)
        idx, st = run(xs, ys)
        rec = {"kind": kind, "n": n, "seed": sd, "xs_sha256_16": sha(xs), "ys_sha256_16": sha(ys),
               **st, "hull_sha256_16": sha(idx.astype(np.uint64))}
        if idx.size <= 5000:
            rec["hull"] = [int(v) for v in idx]
        out[name] = rec
        print(name, st, flush=True)
        del xs, ys
    (HERE / "extra.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    what = sys.argv[1:] or ["configs", "corpus", "stages"]
    for w in what:
        globals()[w]()
