"""GPU vs the golden vectors generated from the unmodified reference
(tests/golden/make_golden.py): BASELINE configs C1-C4 at full size, the
906-case known-answer corpus, and stage-level dumps."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def _gen(kind, n, seed):
    from paper_1508_05931_b200 import generate, generate_grid

    return generate_grid(n, seed) if kind == "grid" else generate(kind, n, seed)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_baseline_configs_bit_exact(engine, name):
    from paper_1508_05931_b200 import PipelineConfig

    g = json.loads((GOLDEN / "configs.json").read_text())[name]
    xs, ys = _gen(g["kind"], g["n"], g["seed"])
    assert sha(xs) == g["xs_sha256_16"] and sha(ys) == g["ys_sha256_16"], "input generator drift"
    idx, st = engine.hull_indices(xs, ys, PipelineConfig())
    assert st.n_after_round1 == g["n_after_round1"]
    assert st.n_after_round2 == g["n_after_round2"]
    assert st.hull_size == g["hull_size"]
    assert sha(idx.astype(np.uint64)) == g["hull_sha256_16"]
    if "hull" in g:
        assert idx.tolist() == g["hull"]


def test_corpus_bit_exact(engine):
    from paper_1508_05931_b200 import PipelineConfig

    cases = json.loads((GOLDEN / "corpus.json").read_text())
    for c in cases:
        if c["kind"] == "hand":
            p = np.array(c["points"], float)
            xs, ys = p[:, 0].copy(), p[:, 1].copy()
        else:
            xs, ys = _gen(c["kind"], c["n"], c["seed"])
        idx, st = engine.hull_indices(xs, ys, PipelineConfig(**c["cfg"]))
        assert idx.tolist() == c["hull"], (c["kind"], c.get("n"), c.get("seed"), c["cfg"])
        assert st.n_after_round1 == c["n_after_round1"]
        assert st.n_after_round2 == c["n_after_round2"]


def test_stages_bit_exact(engine):
    import torch

    for c in json.loads((GOLDEN / "stages.json").read_text()):
        xs, ys = _gen(c["kind"], c["n"], c["seed"])
        n = c["n"]
        dx = torch.from_numpy(xs).cuda()
        dy = torch.from_numpy(ys).cuda()
        ext = engine.stage_extremes(dx.data_ptr(), dy.data_ptr(), n)
        assert ext[:4] == c["quad"] and ext[4] == c["anchor"]
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        k = engine.stage_round1(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr())
        assert k == c["n_r1"]
        assert sha(out[:k].cpu().numpy().astype(np.uint64)) == c["r1_survivors_sha256_16"]
        m = engine.stage_sorted(dx.data_ptr(), dy.data_ptr(), n, out.data_ptr())
        assert m == c["sorted_len"]
        assert sha(out[:m].cpu().numpy().astype(np.uint64)) == c["sorted_sha256_16"]
        flags = torch.empty(n, dtype=torch.uint8, device="cuda")
        for chunks, chunked in ((1024, True), (7, True), (1, True), (1024, False)):
            l, mm = engine.stage_discard(dx.data_ptr(), dy.data_ptr(), n, chunks, chunked,
                                         flags.data_ptr())
            g = c[f"discard_{chunks}_{int(chunked)}"]
            assert l == g["longest"]
            assert sha(flags[:mm].cpu().numpy()) == g["flags_sha256_16"]
