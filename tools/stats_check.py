"""Stage stats of a few graph-replayed C2 calls (device stamps): python tools/stats_check.py"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1508_05931_b200 import Engine, PipelineConfig
eng = Engine(0)
n = 20_000_000
xs = torch.empty(n, dtype=torch.float64, device="cuda"); ys = torch.empty_like(xs)
eng.generate_square_device(1, 0, n, xs.data_ptr(), ys.data_ptr())
out = torch.empty(n, dtype=torch.int32, device="cuda")
for i in range(4):
    k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
print("STATS", k, st)
print("OUT", out[:5].tolist())
