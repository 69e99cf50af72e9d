"""Sparse vs full-sort path at large n (both native): python tools/big_ab.py n [seed] [kind]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402
from paper_1508_05931_b200 import _native as N  # noqa: E402

n = int(float(sys.argv[1]))
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kind = sys.argv[3] if len(sys.argv) > 3 else "square"
eng = Engine(0)
if kind == "square":
    xs = torch.empty(n, dtype=torch.float64, device="cuda")
    ys = torch.empty(n, dtype=torch.float64, device="cuda")
    eng.generate_square_device(seed, 0, n, xs.data_ptr(), ys.data_ptr())
else:
    hx, hy = generate(kind, n, seed)
    xs, ys = torch.from_numpy(hx).cuda(), torch.from_numpy(hy).cuda()
out = torch.empty(n, dtype=torch.int32, device="cuda")
res = {}
for name, dbg in (("full", N.DEBUG_FULL_SORT), ("sparse", 0)):
    eng.set_debug(dbg)
    k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
    res[name] = (out[:k].cpu().numpy().copy(), st, eng.sparse_info())
    print(name, "n1", st.n_after_round1, "n2", st.n_after_round2, "hull", st.hull_size,
          "sparse_info", eng.sparse_info(), "dev_ms", round(st.t_total_ms, 3), flush=True)
same = np.array_equal(res["full"][0], res["sparse"][0]) and all(
    getattr(res["full"][1], f) == getattr(res["sparse"][1], f) for f in ("n_after_round1", "n_after_round2", "hull_size"))
print("SAME" if same else "DIFFERENT", flush=True)
