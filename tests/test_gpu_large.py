"""GPU: the sparse path at the sizes and seeds the round-1 tests did not reach.

* C2-C4 at the secondary seeds 2-5 against goldens from the
  unmodified reference (tests/golden/extra.json, make_golden.py extra);
* the uniform square at 100M and 200M points (seed 1) -- where the gathered
  buckets outgrow shared memory and the global-scratch sorters and the
  sub-partitioned duplicate check take over -- against the reference's
  goldens, on the sparse path;
* 1B points (BASELINE C5) on one device in large mode, cross-checked against
  the 8-rank sharded path on the same points and for convexity/containment.
Inputs come from the on-device generator (bit-identical to the reference's
gen_square, tests/test_gpu_datagen.py) or the host generators."""
import hashlib
import json
import os
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
EXTRA = Path(__file__).resolve().parent / "golden" / "extra.json"


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def gold():
    return json.loads(EXTRA.read_text())


def _inputs(eng, kind, n, seed):
    if kind == "square":
        xs = torch.empty(n, dtype=torch.float64, device="cuda")
        ys = torch.empty(n, dtype=torch.float64, device="cuda")
        eng.generate_square_device(seed, 0, n, xs.data_ptr(), ys.data_ptr())
        return xs, ys
    from paper_1508_05931_b200 import generate
    hx, hy = generate(kind, n, seed)
    return torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()


def _hull(eng, xs, ys):
    from paper_1508_05931_b200 import PipelineConfig
    n = xs.numel()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
    return out[:k].cpu().numpy().astype(np.uint64), st


def _compare(g, idx, st):
    assert st.n_after_round1 == g["n_after_round1"]
    assert st.n_after_round2 == g["n_after_round2"]
    assert st.hull_size == g["hull_size"]
    assert _sha(idx) == g["hull_sha256_16"]


@pytest.mark.parametrize("name", [f"{c}s{s}" for s in (2, 3, 4, 5) for c in ("C2", "C3", "C4")])
def test_secondary_seeds_match_reference(gold, name):
    from paper_1508_05931_b200 import Engine
    g = gold[name]
    eng = Engine(0)
    xs, ys = _inputs(eng, g["kind"], g["n"], g["seed"])
    assert _sha(xs.cpu().numpy()) == g["xs_sha256_16"]
    idx, st = _hull(eng, xs, ys)
    _compare(g, idx, st)


@pytest.mark.parametrize("name", ["S100M", "S200M"])
def test_large_square_sparse_matches_reference(gold, name):
    from paper_1508_05931_b200 import Engine
    g = gold[name]
    eng = Engine(0)
    xs, ys = _inputs(eng, "square", g["n"], g["seed"])
    idx, st = _hull(eng, xs, ys)
    assert eng.sparse_info()[0] == 1, f"declined: {eng.sparse_info()}"
    _compare(g, idx, st)
    del xs, ys, eng
    torch.cuda.empty_cache()


def test_large_mode_matches_normal_mode_100M(gold):
    """Large mode (walk-sized buffers, no full-sort fallback) forced at 100M
    gives the reference's hull."""
    from paper_1508_05931_b200 import Engine
    g = gold["S100M"]
    old = os.environ.get("GSCAN_LARGE_MIN")
    os.environ["GSCAN_LARGE_MIN"] = "50000000"
    try:
        eng = Engine(0)
        xs, ys = _inputs(eng, "square", g["n"], g["seed"])
        idx, st = _hull(eng, xs, ys)
    finally:
        if old is None:
            os.environ.pop("GSCAN_LARGE_MIN")
        else:
            os.environ["GSCAN_LARGE_MIN"] = old
    _compare(g, idx, st)
    del xs, ys, eng
    torch.cuda.empty_cache()


def test_c5_one_device_and_eight_simulated_ranks():
    """C5: 1B points on one device (large mode, sparse path) and as 8
    simulated ranks (LocalComm, large-mode handles) give the same hull, which
    is convex and contains every point."""
    from paper_1508_05931_b200 import Engine, PipelineConfig
    from paper_1508_05931_b200.distributed import simulate_sharded
    n = 1_000_000_000
    eng = Engine(0)
    xs, ys = _inputs(eng, "square", n, 1)
    idx, st = _hull(eng, xs, ys)
    assert eng.sparse_info()[0] == 1
    assert st.n_after_round1 > 0.2 * n and st.hull_size >= 4
    del eng
    torch.cuda.empty_cache()
    old = os.environ.get("GSCAN_LARGE_MIN")
    os.environ["GSCAN_LARGE_MIN"] = "50000000"
    try:
        engines = [Engine(0) for _ in range(8)]
        engines[0].reserve(n)  # rank 0 receives the gathered points of all ranks
        res = simulate_sharded(engines, xs, ys, PipelineConfig())
    finally:
        if old is None:
            os.environ.pop("GSCAN_LARGE_MIN")
        else:
            os.environ["GSCAN_LARGE_MIN"] = old
    assert res is not None, "the 8-rank sharded path declined on C5"
    got, sst = res
    assert np.array_equal(got, idx)
    assert (sst.n_after_round1, sst.n_after_round2, sst.hull_size) == (
        st.n_after_round1, st.n_after_round2, st.hull_size)
    del engines
    torch.cuda.empty_cache()
    # convex (CCW, strict left turns) and containing every point
    ii = torch.from_numpy(idx.astype(np.int64)).cuda()
    hx, hy = xs[ii], ys[ii]
    k = hx.numel()
    ax, ay = hx, hy
    bx, by = torch.roll(hx, -1), torch.roll(hy, -1)
    cx, cy = torch.roll(hx, -2), torch.roll(hy, -2)
    turn = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    assert bool((turn > 0).all())
    for e in range(k):
        ex, ey = bx[e] - ax[e], by[e] - ay[e]
        for lo in range(0, n, 250_000_000):
            c = ex * (ys[lo:lo + 250_000_000] - ay[e]) - ey * (xs[lo:lo + 250_000_000] - ax[e])
            assert float(c.min()) >= -1e-12, e
