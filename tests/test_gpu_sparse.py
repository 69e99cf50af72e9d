"""GPU: the sparse round-2 path (paper_1508_05931_b200/csrc/sparse.cuh), the
default for n >= 65536 with the reference's default toggles.

Every case is bit-exact against the CPU oracle (the reference algorithm,
pipeline.hpp:72-123) and, where the path declines, the decline is the
expected one: the fast path never guesses, it either proves its result or
reruns the full sort. Also covers the Graham tree strategy it feeds.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAIL_TIE, FAIL_DUP, FAIL_VERIFY, FAIL_MANY = 1, 8, 16, 256


def _run(engine, oracle_mod, xs, ys, debug=0, **cfg):
    from paper_1508_05931_b200 import PipelineConfig

    engine.set_debug(debug)
    try:
        got, st = engine.hull_indices(xs, ys, PipelineConfig(**cfg))
        info = engine.sparse_info()
    finally:
        engine.set_debug(0)
    want, sw = oracle_mod.full_pipeline(xs, ys, **cfg)
    assert np.array_equal(got, want), (cfg, got[:12], want[:12])
    for k in ("n_after_round1", "n_after_round2", "hull_size"):
        assert getattr(st, k) == sw[k], k
    return info


def _gen(kind, n, seed):
    from paper_1508_05931_b200 import generate

    rng = np.random.default_rng(seed)
    if kind in ("square", "disk", "circle", "collinear"):
        return generate(kind, n, seed)
    if kind == "wedge":  # every point inside a 1e-3 rad wedge: one crowded angle range
        r = np.sqrt(rng.random(n))
        t = 1.0 + 1e-3 * rng.random(n)
        return r * np.cos(t), r * np.sin(t)
    if kind == "gauss":
        return rng.standard_normal(n), rng.standard_normal(n)
    if kind == "shifted":  # far from the origin, tiny extent: relative rounding matters
        return 1e6 + 1e-3 * rng.random(n), -3e5 + 1e-3 * rng.random(n)
    if kind == "grid":  # tie-heavy integer lattice with duplicates
        return rng.integers(0, 300, n).astype(float), rng.integers(0, 300, n).astype(float)
    if kind == "annulus":
        r = 1.0 - 1e-4 * rng.random(n)
        t = 2 * np.pi * rng.random(n)
        return r * np.cos(t), r * np.sin(t)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["square", "disk", "gauss", "shifted", "wedge"])
@pytest.mark.parametrize("n,seed", [(70_000, 1), (300_000, 2), (1_000_000, 3)])
def test_sparse_matches_oracle(engine, oracle_mod, kind, n, seed):
    xs, ys = _gen(kind, n, seed)
    used, fail, walked = _run(engine, oracle_mod, xs, ys)
    if kind in ("square", "disk", "gauss") and n >= 300_000:
        # the fast path is the one being checked on these inputs
        assert used == 1 and fail == 0, hex(fail)
        assert 0 < walked < n


@pytest.mark.parametrize("kind", ["circle", "annulus", "collinear", "grid"])
def test_sparse_degenerate_inputs(engine, oracle_mod, kind):
    """Convex position, near-circles, collinear sets and lattices: exact
    whichever way the call resolves (fast path or declined to the sort)."""
    xs, ys = _gen(kind, 200_000, 5)
    used, fail, _ = _run(engine, oracle_mod, xs, ys)
    if kind == "circle":  # every point is a walk candidate: the full sort is faster
        assert used == 0 and fail & FAIL_MANY, hex(fail)


@pytest.mark.parametrize("chunks", [1, 7, 100, 5000])
def test_sparse_chunk_counts(engine, oracle_mod, chunks):
    """discard_chunked with other slice counts (discard.hpp:90-124)."""
    xs, ys = _gen("square", 300_000, 9)
    used, fail, _ = _run(engine, oracle_mod, xs, ys, chunk_count=chunks)
    assert used == 1, hex(fail)


def test_sparse_duplicates_decline(engine, oracle_mod):
    """annotate's dedup (angular.hpp:118-133) changes ranks: survivors with
    duplicates must make the fast path decline (exact result either way)."""
    xs, ys = _gen("square", 400_000, 4)
    edge = np.flatnonzero(ys < 0.01)
    xs[edge[1::40]] = xs[edge[0::40][: len(edge[1::40])]]
    ys[edge[1::40]] = ys[edge[0::40][: len(edge[1::40])]]
    used, fail, _ = _run(engine, oracle_mod, xs, ys)
    assert used == 0 and fail & FAIL_DUP, hex(fail)


@pytest.mark.parametrize("plant", [False, True])
def test_sparse_duplicate_check_in_rounds(engine, oracle_mod, plant):
    """36M points: ~18M round-1 survivors, so the duplicate-check partitions
    (with their sector padding) exceed one hash-set round (k_sp_dups checks
    them over sub-ranges of the hash). Clean input: the fast path serves.
    One duplicate pair among the survivors, at opposite ends of the input (so
    in different hash lists): it is found and the path declines."""
    xs, ys = _gen("square", 36_000_000, 5)
    if plant:
        edge = np.flatnonzero(ys < 0.001)
        xs[edge[-1]], ys[edge[-1]] = xs[edge[0]], ys[edge[0]]
    used, fail, _ = _run(engine, oracle_mod, xs, ys)
    if plant:
        assert used == 0 and fail & FAIL_DUP, hex(fail)
    else:
        assert used == 1 and fail == 0, hex(fail)


def test_sparse_duplicate_of_interior_point_is_harmless(engine, oracle_mod):
    """Duplicates of points strictly inside the round-1 quadrilateral never
    reach the buffer (classify_quad, prefilter.hpp:47-63): the fast path stays on."""
    import torch

    xs, ys = _gen("square", 400_000, 6)
    n = len(xs)
    dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    k = engine.stage_round1(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr())
    surv = np.zeros(n, bool)
    surv[out[:k].cpu().numpy()] = True
    inner = np.flatnonzero(~surv)
    xs[inner[1::2]] = xs[inner[0::2][: len(inner[1::2])]]
    ys[inner[1::2]] = ys[inner[0::2][: len(inner[1::2])]]
    used, fail, _ = _run(engine, oracle_mod, xs, ys)
    assert used == 1, hex(fail)


def test_sparse_tie_for_farthest_point_declines(engine, oracle_mod):
    """split_regions takes the FIRST maximal dist2 in sorted order
    (angular.hpp:197-204); a tie needs the exact order, so the path declines.
    An explicit anchor and two dyadic points make the tie exact in floating
    point, while round 1 still discards most of the square."""
    xs, ys = _gen("square", 300_000, 7)
    # anchor (0.5, -0.5); (-0.25, 1) and (1.25, 1): dx = -+0.75, dy = 1.5 ->
    # dist2 = 2.8125 for both, beyond every corner of the unit square (<= 2.5);
    # (0.5, 1.1) is the top extreme (dist2 2.56), so the quadrilateral is a
    # proper kite and round 1 keeps only ~12% of the square
    xs = np.append(xs, [0.5, -0.25, 1.25, 0.5])
    ys = np.append(ys, [-0.5, 1.0, 1.0, 1.1])
    used, fail, _ = _run(engine, oracle_mod, xs, ys)
    assert used == 0 and fail & FAIL_TIE, hex(fail)


def test_sparse_dropped_candidates_are_rejected(engine, oracle_mod):
    """Walking no candidates must be caught by the verification pass."""
    from paper_1508_05931_b200 import _native as N

    xs, ys = _gen("square", 300_000, 8)
    used, fail, _ = _run(engine, oracle_mod, xs, ys, debug=N.DEBUG_SPARSE_DROP)
    assert used == 0 and fail & FAIL_VERIFY, hex(fail)


def test_sparse_forced_verification_agrees(engine, oracle_mod):
    """The verification pass accepts what the error-bound certificate proved."""
    from paper_1508_05931_b200 import _native as N

    xs, ys = _gen("disk", 500_000, 3)
    used, fail, _ = _run(engine, oracle_mod, xs, ys, debug=N.DEBUG_SPARSE_VERIFY)
    assert used == 1 and fail == 0, hex(fail)


def test_full_sort_path_still_exact(engine, oracle_mod):
    from paper_1508_05931_b200 import _native as N

    xs, ys = _gen("square", 300_000, 11)
    used, _, _ = _run(engine, oracle_mod, xs, ys, debug=N.DEBUG_FULL_SORT)
    assert used == 0


@pytest.mark.parametrize("kind", ["square", "disk"])
def test_graham_tree_strategy(engine, oracle_mod, kind):
    """Round-2 output of squares and disks is pop-heavy: the tree strategy
    runs and its certificate holds (a disk's levels stop shrinking at its
    many hull vertices: the warp top scan takes the stalled level); a
    falsified candidate falls back exactly."""
    from paper_1508_05931_b200 import _native as N

    xs, ys = _gen(kind, 1_000_000, 2)
    _run(engine, oracle_mod, xs, ys)
    path, fails = engine.graham_info()
    assert fails == 0 and path == 8, (path, fails)
    _run(engine, oracle_mod, xs, ys, debug=N.DEBUG_CORRUPT_CANDIDATE)
    path, fails = engine.graham_info()
    assert (path & 4) and fails > 0, (path, fails)


def test_repeated_calls_reuse_the_graph(engine, oracle_mod):
    """The captured graph is replayed for the same input and recaptured when
    the input or the config changes; results stay exact."""
    xs, ys = _gen("square", 250_000, 12)
    for _ in range(3):
        _run(engine, oracle_mod, xs, ys)
    xs2, ys2 = _gen("disk", 250_000, 13)
    _run(engine, oracle_mod, xs2, ys2)
    _run(engine, oracle_mod, xs, ys, chunk_count=33)
    _run(engine, oracle_mod, xs, ys)


def test_decline_after_a_larger_call(engine, oracle_mod):
    """A call that declines before F2 (a circle: the sample says near-convex)
    right after a larger sparse call on the same handle: the P_l partials
    still hold the earlier call's indices, beyond this input, and must not be
    read (tools/stress.py found the out-of-bounds read under memcheck)."""
    from paper_1508_05931_b200 import PipelineConfig, generate

    for kind, n in (("square", 1_500_000), ("circle", 120_000), ("disk", 900_000), ("circle", 70_000)):
        xs, ys = generate(kind, n, 3)
        got, st = engine.hull_indices(xs, ys, PipelineConfig())
        want, sw = oracle_mod.full_pipeline(xs, ys)
        assert np.array_equal(got, want), kind
        assert (st.n_after_round1, st.n_after_round2) == (sw["n_after_round1"], sw["n_after_round2"])
