"""On-device gen_square (csrc/mtgen.cuh) against the
host generator, which restates datagen.hpp:32-41 with the same libstdc++
engine and distribution (its bits are pinned to the reference's by the
golden input hashes in tests/golden/configs.json)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "configs.json"


@pytest.fixture(scope="module")
def eng():
    from paper_1508_05931_b200 import Engine
    return Engine(0)


def dev_gen(eng, seed, lo, hi):
    import torch
    xs = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    ys = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
    eng.generate_square_device(seed, lo, hi, xs.data_ptr(), ys.data_ptr())
    return xs.cpu().numpy(), ys.cpu().numpy()


@pytest.mark.parametrize("seed", [1, 7, 2**63 + 5])
def test_prefix_bit_exact(eng, seed):
    from paper_1508_05931_b200 import generate
    n = 3_000_001
    hx, hy = generate("square", n, seed)
    dx, dy = dev_gen(eng, seed, 0, n)
    assert np.array_equal(hx.view(np.uint64), dx.view(np.uint64))
    assert np.array_equal(hy.view(np.uint64), dy.view(np.uint64))


@pytest.mark.parametrize("lo,hi", [(2_500_017, 3_000_000), (524_287, 524_289), (0, 1),
                                   (1_048_575, 1_048_577), (40_000_003, 40_100_000)])
def test_shards_bit_exact(eng, lo, hi):
    from paper_1508_05931_b200 import generate
    hx, hy = generate("square", hi, 1)
    dx, dy = dev_gen(eng, 1, lo, hi)
    assert np.array_equal(hx[lo:hi].view(np.uint64), dx.view(np.uint64))
    assert np.array_equal(hy[lo:hi].view(np.uint64), dy.view(np.uint64))


def test_c2_input_matches_golden_hash(eng):
    g = json.loads(GOLD.read_text())["C2"]
    dx, dy = dev_gen(eng, 1, 0, g["n"])
    assert hashlib.sha256(dx.tobytes()).hexdigest()[:16] == g["xs_sha256_16"]
    assert hashlib.sha256(dy.tobytes()).hexdigest()[:16] == g["ys_sha256_16"]
