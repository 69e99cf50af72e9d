"""Debug the sharded sparse path on one GPU (LocalComm). Usage: python tools/dist_debug.py [R] [n]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402
from paper_1508_05931_b200 import distributed as D  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 600_000
xs, ys = generate("square", n, 2)
eng1 = Engine(0)
want, st = eng1.hull_indices(xs, ys, PipelineConfig())
print("single:", st, eng1.sparse_info())
engines = [Engine(0) for _ in range(R)]
dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
orig = D._ck
res = D.simulate_sharded(engines, dx, dy)
print("sharded:", None if res is None else (np.array_equal(res[0], want), res[1]), "|", D.last_decline)
