"""The reference's acceptance corpus, run through the device path
(acceptance.cpp:62-170, `run_corpus_criteria`): 200 seeds x {square, disk,
circle} x n in {10, 100, 1000, 10000}, chunk counts {1, 7, 1024}.

Criteria 1/3 there compare the pipeline's hull with the monotone-chain oracle
and flag unsafe discards; here every case is compared with the oracle's full
pipeline instead, which is stronger: the same hull indices in the same order
and the same stage counts (n_after_round1, n_after_round2, hull_size).
Criterion 4 (chunking): chunk count 1 gives the sequential discard's buffer,
and a chunk count equal to the buffer size keeps every survivor.

The corpus stays below the sparse path's size; `test_sparse_corpus` runs the
same comparison over 100 seeds at 70K-300K points, where the default path is
the sparse round 2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FAMILIES = ("square", "disk", "circle")
SIZES = (10, 100, 1000, 10000)
CHUNKS = (1, 7, 1024)


def _dataset(kind, n, seed):
    from paper_1508_05931_b200 import generate

    return generate(kind, max(n, 3) if kind == "circle" else n, seed)  # make_dataset


def _run(engine, oracle_mod, xs, ys, **cfg):
    from paper_1508_05931_b200 import PipelineConfig

    got, st = engine.hull_indices(xs, ys, PipelineConfig(**cfg))
    want, sw = oracle_mod.full_pipeline(xs, ys, **cfg)
    ok = (np.array_equal(got, want) and st.n_after_round1 == sw["n_after_round1"]
          and st.n_after_round2 == sw["n_after_round2"] and st.hull_size == sw["hull_size"])
    return ok, st, sw


@pytest.mark.parametrize("kind", FAMILIES)
def test_acceptance_corpus(engine, oracle_mod, kind):
    bad = []
    cases = 0
    for seed in range(200):
        for n in SIZES:
            xs, ys = _dataset(kind, n, seed)
            for chunks in CHUNKS:
                ok, st, _ = _run(engine, oracle_mod, xs, ys, chunk_count=chunks)
                cases += 1
                if not ok:
                    bad.append((seed, n, chunks))
            # criterion 4: chunk count 1 == the sequential discard
            ok1, st1, _ = _run(engine, oracle_mod, xs, ys, chunk_count=1)
            oks, sts, _ = _run(engine, oracle_mod, xs, ys, chunked=False)
            cases += 2
            if not (ok1 and oks and st1.n_after_round2 == sts.n_after_round2):
                bad.append((seed, n, "sequential"))
            # ... and one chunk per buffer element keeps every survivor
            _, _, tr = oracle_mod.full_pipeline(xs, ys, trace=True)
            m = len(tr["sorted_idx"])
            if m >= 2:
                okw, stw, _ = _run(engine, oracle_mod, xs, ys, chunk_count=m)
                cases += 1
                if not (okw and stw.n_after_round2 == m):
                    bad.append((seed, n, "wide"))
    assert not bad, f"{len(bad)}/{cases} cases differ; first {bad[:5]}"


@pytest.mark.parametrize("kind", ("square", "disk"))
def test_sparse_corpus(engine, oracle_mod, kind):
    """100 seeds at sparse-path sizes, chunk counts {7, 1024}: bit-exact, and
    the sparse path serves (sparse_info()[0] == 1) on every case."""
    bad, served = [], 0
    for seed in range(100):
        n = (70_000, 150_000, 300_000)[seed % 3]
        xs, ys = _dataset(kind, n, 1000 + seed)
        for chunks in (7, 1024):
            ok, _, _ = _run(engine, oracle_mod, xs, ys, chunk_count=chunks)
            served += engine.sparse_info()[0] == 1
            if not ok:
                bad.append((seed, n, chunks))
    assert not bad, bad[:5]
    assert served == 200, served
