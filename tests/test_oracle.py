"""CPU: pin the oracle (plain-C port) to the reference's golden vectors and
to the known answers the reference's own tests hold."""
import hashlib
import json
import math
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _gen(kind, n, seed):
    from paper_1508_05931_b200 import generate, generate_grid

    return generate_grid(n, seed) if kind == "grid" else generate(kind, n, seed)


# ---- known answers: test_geom.cpp ----
def test_orient_turns(oracle_mod):
    o = oracle_mod.orient
    assert o((0, 0), (1, 0), (0, 1)) == 1
    assert o((0, 0), (1, 0), (2, 0)) == 0
    assert o((0, 0), (0, 1), (1, 1)) == -1


def test_orient_antisymmetric_and_translation_invariant(oracle_mod):
    rng = np.random.default_rng(42)
    for _ in range(2000):
        a, b, c = (tuple(map(float, rng.integers(-50, 51, 2))) for _ in range(3))
        assert oracle_mod.orient(a, b, c) == -oracle_mod.orient(a, c, b)
        d = tuple(map(float, rng.integers(-300, 301, 2)))
        sh = lambda p: (p[0] + d[0], p[1] + d[1])  # noqa: E731
        assert oracle_mod.orient(a, b, c) == oracle_mod.orient(sh(a), sh(b), sh(c))


def test_polar_key_known_values(oracle_mod):
    assert oracle_mod.atan2(1.0, 1.0) == math.pi / 4
    assert oracle_mod.atan2(0.0, -1.0) == math.pi
    assert oracle_mod.atan2(3.0, 0.0) == math.pi / 2


# ---- known answers: test_prefilter.cpp ----
def test_find_extremes_ties(oracle_mod):
    pts = np.array([[0, 0], [2, 1], [1, 3], [-1, 1]], float)
    assert oracle_mod.find_extremes(pts[:, 0], pts[:, 1]) == [3, 0, 1, 2]
    assert oracle_mod.find_extremes([5.0], [5.0]) == [0, 0, 0, 0]
    assert oracle_mod.find_extremes([1.0] * 3, [1.0] * 3) == [0, 0, 0, 0]


def test_classify_diamond(oracle_mod):
    pts = np.array([[-1, 0], [0, -1], [1, 0], [0, 1], [0, 0], [0.5, 0.5], [2, 0]], float)
    f = oracle_mod.classify_quad(pts[:, 0], pts[:, 1], [0, 1, 2, 3])
    assert f.tolist() == [1, 1, 1, 1, 0, 1, 1]
    col = np.array([[0, 0], [1, 0], [2, 0], [3, 0]], float)
    q = oracle_mod.find_extremes(col[:, 0], col[:, 1])
    assert oracle_mod.classify_quad(col[:, 0], col[:, 1], q).sum() == 4
    tri = np.array([[0, 0], [1, 0], [0, 1], [0.2, 0.2]], float)
    q = oracle_mod.find_extremes(tri[:, 0], tri[:, 1])
    assert oracle_mod.classify_quad(tri[:, 0], tri[:, 1], q).sum() == 4


# ---- known answers: test_angular.cpp ----
def test_select_anchor(oracle_mod):
    assert oracle_mod.select_anchor([1.0, 0.0, 3.0], [2.0, 0.0, 0.0]) == 1
    assert oracle_mod.select_anchor([5.0], [5.0]) == 0
    assert oracle_mod.select_anchor([0.0, 0.0], [1.0, 1.0]) == 0


# ---- known answers: test_discard.cpp / test_pipeline.cpp via the trace ----
def test_walk_example(oracle_mod):
    """test_discard.cpp:30-48: {(0,0),(4,1),(2,1),(0,5)} -> flags [1,1,0,1]."""
    pts = np.array([[0, 0], [4, 1], [2, 1], [0, 5]], float)
    _, st, tr = oracle_mod.full_pipeline(pts[:, 0], pts[:, 1], chunked=False,
                                         enable_round1=False, trace=True)
    assert tr["sorted_idx"].tolist() == [0, 1, 2, 3]
    assert tr["longest"] == 3
    assert tr["r2_flags"].tolist() == [1, 1, 0, 1]
    _, _, tr1 = oracle_mod.full_pipeline(pts[:, 0], pts[:, 1], chunk_count=1,
                                         enable_round1=False, trace=True)
    assert tr1["r2_flags"].tolist() == [1, 1, 0, 1]
    for c in (2, 100):
        _, _, trc = oracle_mod.full_pipeline(pts[:, 0], pts[:, 1], chunk_count=c,
                                             enable_round1=False, trace=True)
        assert trc["r2_flags"].tolist() == [1, 1, 1, 1]


def test_degenerate_conventions(oracle_mod):
    def h(pts, **cfg):
        p = np.array(pts, float)
        return oracle_mod.full_pipeline(p[:, 0], p[:, 1], **cfg)

    assert h([[0, 0], [1, 0], [1, 1], [0, 1]])[0].tolist() == [0, 1, 2, 3]
    assert h([[0, 0], [1, 0], [2, 0]])[0].tolist() == [0, 2]
    assert h([[2, 3]])[0].tolist() == [0]
    assert h([[2, 3], [0, 1]])[0].tolist() == [1, 0]
    idx, st = h([[1, 1]] * 6)
    assert idx.tolist() == [0] and st["n_after_round2"] == 1
    with pytest.raises(RuntimeError):
        oracle_mod.full_pipeline(np.zeros(0), np.zeros(0))
    with pytest.raises(RuntimeError):
        oracle_mod.full_pipeline([0.0], [0.0], chunk_count=0)


def test_circle_keeps_all(oracle_mod):
    xs, ys = _gen("circle", 1000, 1)
    idx, st = oracle_mod.full_pipeline(xs, ys)
    assert st["n_after_round1"] == 1000 and st["n_after_round2"] == 1000 and idx.size == 1000


def test_pipeline_equals_monotone_chain_vertex_set(oracle_mod):
    """acceptance criterion 1 on a small corpus: same vertex set as the oracle hull."""
    for kind in ("square", "disk", "circle", "grid"):
        for seed in range(10):
            xs, ys = _gen(kind, 300, seed)
            idx, _ = oracle_mod.full_pipeline(xs, ys)
            mc = oracle_mod.monotone_chain(xs, ys)
            a = sorted(zip(xs[idx], ys[idx]))
            b = sorted(zip(xs[mc], ys[mc]))
            assert a == b, (kind, seed)


# ---- golden vectors generated from the reference itself ----
def test_corpus_golden(oracle_mod):
    cases = json.loads((GOLDEN / "corpus.json").read_text())
    assert len(cases) > 800
    for c in cases:
        if c["kind"] == "hand":
            p = np.array(c["points"], float)
            xs, ys = p[:, 0], p[:, 1]
        else:
            xs, ys = _gen(c["kind"], c["n"], c["seed"])
            assert sha(xs) == c["xs_sha256_16"]
        idx, st = oracle_mod.full_pipeline(xs, ys, **c["cfg"])
        assert idx.tolist() == c["hull"], c
        for k in ("n_after_round1", "n_after_round2", "hull_size"):
            assert st[k] == c[k], (k, c["kind"], c.get("n"), c["cfg"])


def test_stage_golden(oracle_mod):
    for c in json.loads((GOLDEN / "stages.json").read_text()):
        xs, ys = _gen(c["kind"], c["n"], c["seed"])
        assert oracle_mod.find_extremes(xs, ys) == c["quad"]
        assert oracle_mod.select_anchor(xs, ys) == c["anchor"]
        f = oracle_mod.classify_quad(xs, ys, c["quad"])
        assert sha(np.nonzero(f)[0].astype(np.uint64)) == c["r1_survivors_sha256_16"]
        _, st, tr = oracle_mod.full_pipeline(xs, ys, enable_round1=False, trace=True)
        assert tr["sorted_idx"].size == c["sorted_len"]
        assert sha(tr["sorted_idx"].astype(np.uint64)) == c["sorted_sha256_16"]
        for chunks, chunked in ((1024, True), (7, True), (1, True), (1024, False)):
            _, _, t2 = oracle_mod.full_pipeline(xs, ys, enable_round1=False, chunk_count=chunks,
                                                chunked=chunked, trace=True)
            g = c[f"discard_{chunks}_{int(chunked)}"]
            assert t2["longest"] == g["longest"]
            assert sha(t2["r2_flags"]) == g["flags_sha256_16"]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_golden(oracle_mod, name):
    g = json.loads((GOLDEN / "configs.json").read_text())[name]
    xs, ys = _gen(g["kind"], g["n"], g["seed"])
    assert sha(xs) == g["xs_sha256_16"] and sha(ys) == g["ys_sha256_16"]
    idx, st = oracle_mod.full_pipeline(xs, ys)
    assert sha(idx.astype(np.uint64)) == g["hull_sha256_16"]
    for k in ("n_after_round1", "n_after_round2", "hull_size"):
        assert st[k] == g[k]


def test_port_equals_reference_build(oracle_mod):
    """When the reference is compiled here (oracle/_ref), the port matches it."""
    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    for kind in ("square", "disk", "circle", "collinear", "grid"):
        for n, seed in ((50, 1), (2000, 2), (30000, 3)):
            xs, ys = _gen(kind, n, seed)
            for cfg in (dict(), dict(chunk_count=3), dict(chunked=False)):
                a, sa = oracle_mod.full_pipeline(xs, ys, **cfg)
                b, sb = oracle_mod.full_pipeline(xs, ys, impl="ref", **cfg)
                assert a.tolist() == b.tolist()
                assert sa["n_after_round2"] == sb["n_after_round2"]
