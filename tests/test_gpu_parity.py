"""GPU parity: the sm_100a pipeline against the CPU oracle on identical inputs.

Bit-exact index lists and stage counts (integer/index work: no tolerance).
Reference tests mirrored: test_pipeline.cpp, test_discard.cpp,
test_angular.cpp, test_prefilter.cpp, acceptance.cpp criteria 1/4/5.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = ("square", "disk", "circle", "collinear")


def _gen(kind, n, seed):
    from paper_1508_05931_b200 import generate, generate_grid

    if kind == "grid":
        return generate_grid(n, seed)
    return generate(kind, n, seed)


def _check(engine, oracle_mod, xs, ys, **cfg):
    from paper_1508_05931_b200 import PipelineConfig

    got, st = engine.hull_indices(xs, ys, PipelineConfig(**cfg))
    want, sw = oracle_mod.full_pipeline(xs, ys, **cfg)
    assert np.array_equal(got, want), (cfg, got[:16], want[:16])
    assert st.n_input == sw["n_input"]
    assert st.n_after_round1 == sw["n_after_round1"], cfg
    assert st.n_after_round2 == sw["n_after_round2"], cfg
    assert st.hull_size == sw["hull_size"]


def test_device_atan2_matches_host_libm(engine, oracle_mod):
    import torch

    rng = np.random.default_rng(7)
    n = 1 << 20
    y = np.concatenate([rng.random(n // 2), rng.standard_normal(n // 4) * 1e-3,
                        np.ldexp(rng.random(n // 4), rng.integers(-80, 20, n // 4))])
    x = np.concatenate([rng.standard_normal(n // 2), rng.standard_normal(n // 4),
                        np.ldexp(rng.standard_normal(n // 4), rng.integers(-80, 20, n // 4))])
    want = oracle_mod.atan2_array(y, x)  # host glibc atan2 (numpy's arctan2 is not libm's)
    dy = torch.from_numpy(y).cuda()
    dx = torch.from_numpy(x).cuda()
    out = torch.empty_like(dy)
    engine.device_atan2(dy.data_ptr(), dx.data_ptr(), out.data_ptr(), n)
    got = out.cpu().numpy()
    host = np.array([oracle_mod.atan2(float(a), float(b)) for a, b in zip(y[:2000], x[:2000])])
    assert np.array_equal(want[:2000].view(np.uint64), host.view(np.uint64))
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("kind", KINDS + ("grid",))
@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 100, 1000, 4097, 30000])
def test_full_pipeline_matches_oracle(engine, oracle_mod, kind, n):
    for seed in range(3):
        xs, ys = _gen(kind, n, seed)
        _check(engine, oracle_mod, xs, ys)


@pytest.mark.parametrize("cfg", [dict(chunk_count=1), dict(chunk_count=2), dict(chunk_count=3),
                                 dict(chunk_count=7), dict(chunk_count=64),
                                 dict(enable_round1=False), dict(enable_round2=False),
                                 dict(enable_round1=False, enable_round2=False),
                                 dict(chunked=False)])
@pytest.mark.parametrize("kind", KINDS + ("grid",))
def test_config_toggles_match_oracle(engine, oracle_mod, kind, cfg):
    for n, seed in ((10, 1), (100, 2), (1000, 3), (20000, 4)):
        xs, ys = _gen(kind, n, seed)
        _check(engine, oracle_mod, xs, ys, **cfg)


def test_known_answers(engine):
    """test_pipeline.cpp:19-28, 92-107 degenerate conventions."""
    from paper_1508_05931_b200 import EmptyInput, PipelineConfig, ZeroChunks

    def h(pts, **cfg):
        return engine.full_pipeline(np.array(pts, dtype=np.float64), PipelineConfig(**cfg))

    assert h([[0, 0], [1, 0], [1, 1], [0, 1]]).hull.vertices.tolist() == [[0, 0], [1, 0], [1, 1], [0, 1]]
    assert h([[0, 0], [1, 0], [2, 0]]).hull.vertices.tolist() == [[0, 0], [2, 0]]
    assert h([[2, 3]]).hull.vertices.tolist() == [[2, 3]]
    assert h([[2, 3], [0, 1]]).hull.vertices.tolist() == [[0, 1], [2, 3]]
    assert h([[0, 0], [1, 0], [2, 0], [1, 0]]).hull.vertices.tolist() == [[0, 0], [2, 0]]
    dup = h([[1, 1]] * 6)
    assert dup.hull.vertices.tolist() == [[1, 1]]
    assert dup.stats.n_after_round2 == 1
    with pytest.raises(EmptyInput):
        h(np.zeros((0, 2)))
    with pytest.raises(ZeroChunks):
        h([[0, 0]], chunk_count=0)
    tri = [[0, 0], [3, 1], [1, 4]]
    for cfg in (dict(), dict(chunk_count=1), dict(enable_round1=False),
                dict(enable_round2=False), dict(chunked=False)):
        r = h(tri, **cfg)
        assert r.hull.size() == 3 and r.stats.n_after_round1 == 3 and r.stats.n_after_round2 == 3


def test_circle_keeps_everything(engine, oracle_mod):
    """test_pipeline.cpp:73-81 / acceptance criterion 5."""
    from paper_1508_05931_b200 import generate

    xs, ys = generate("circle", 1000, 1)
    r = engine.full_pipeline(np.stack([xs, ys], 1))
    assert r.stats.n_after_round1 == 1000
    assert r.stats.n_after_round2 == 1000
    assert r.hull.size() == 1000


@pytest.mark.parametrize("kind", KINDS + ("grid",))
@pytest.mark.parametrize("flags", ["junction", "sequential", "prefix", "corrupt", "fallback"])
def test_graham_paths_are_exact(engine, oracle_mod, kind, flags):
    """Every Graham strategy (and the certificate's rejection of a falsified
    candidate) yields the sequential scan's exact output (pipeline.hpp:57-67)."""
    from paper_1508_05931_b200 import _native as N

    f = {"junction": N.DEBUG_FORCE_JUNCTION, "sequential": N.DEBUG_FORCE_SEQUENTIAL,
         "prefix": N.DEBUG_FORCE_PREFIX, "corrupt": N.DEBUG_CORRUPT_CANDIDATE,
         "fallback": N.DEBUG_FORCE_FALLBACK}[flags]
    try:
        engine.set_debug(f)
        for n, seed in ((300, 1), (5000, 2), (40000, 3)):
            xs, ys = _gen(kind, n, seed)
            for cfg in (dict(), dict(enable_round2=False), dict(enable_round1=False, enable_round2=False)):
                _check(engine, oracle_mod, xs, ys, **cfg)
                path, fails = engine.graham_info()
                if flags == "corrupt" and path != 0:
                    assert fails > 0 and (path & 4), (path, fails)
    finally:
        engine.set_debug(0)
