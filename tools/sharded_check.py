"""The sharded sparse path as 3 simulated ranks (LocalComm) on a 600K disk,
once with the certificate and once with the distributed F6 forced, checked
against the one-device hull: python tools/sharded_check.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402
from paper_1508_05931_b200 import _native as N  # noqa: E402
from paper_1508_05931_b200.distributed import simulate_sharded  # noqa: E402

xs, ys = generate("disk", 600_000, 7)
one = Engine(0)
want, _ = one.hull_indices(xs, ys, PipelineConfig())
engines = [Engine(0) for _ in range(3)]
dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
for flags in (0, N.DEBUG_SPARSE_VERIFY):
    engines[0].set_debug(flags)
    res = simulate_sharded(engines, dx, dy, PipelineConfig())
    assert res is not None and np.array_equal(res[0], want), flags
print("sharded ok")
