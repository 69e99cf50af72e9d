"""Time the on-device gen_square (mtgen.cuh) for n points: python tools/gen_time.py [n]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000_000
eng = Engine(0)
xs = torch.empty(n, dtype=torch.float64, device="cuda")
ys = torch.empty(n, dtype=torch.float64, device="cuda")
for rep in range(2):
    t = time.perf_counter()
    eng.generate_square_device(1, 0, n, xs.data_ptr(), ys.data_ptr())
    print(f"n={n} gen {time.perf_counter() - t:.3f} s", flush=True)
print("last point", xs[-1].item(), ys[-1].item())
