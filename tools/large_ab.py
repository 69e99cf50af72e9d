"""Large mode (reserve's walk-sized buffers, no full-sort fallback) against a
normal handle's full sort on the same device-generated square:
python tools/large_ab.py n [seed]"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig  # noqa: E402
from paper_1508_05931_b200 import _native as N  # noqa: E402

n = int(float(sys.argv[1]))
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
xs = torch.empty(n, dtype=torch.float64, device="cuda")
ys = torch.empty(n, dtype=torch.float64, device="cuda")
out = torch.empty(n, dtype=torch.int32, device="cuda")
res = {}
for name in ("full", "large"):
    if name == "large":
        os.environ["GSCAN_LARGE_MIN"] = str(n // 2)
    eng = Engine(0)
    eng.generate_square_device(seed, 0, n, xs.data_ptr(), ys.data_ptr())
    if name == "full":
        eng.set_debug(N.DEBUG_FULL_SORT)
    k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
    free, total = torch.cuda.mem_get_info()
    res[name] = (out[:k].cpu().numpy().copy(), st)
    print(name, "n1", st.n_after_round1, "n2", st.n_after_round2, "hull", st.hull_size,
          "sparse", eng.sparse_info(), "dev_ms", round(st.t_total_ms, 3),
          "used_GB", round((total - free) / 1e9, 1), flush=True)
    del eng
    torch.cuda.empty_cache()
same = np.array_equal(res["full"][0], res["large"][0]) and all(
    getattr(res["full"][1], f) == getattr(res["large"][1], f)
    for f in ("n_after_round1", "n_after_round2", "hull_size"))
print("SAME" if same else "DIFFERENT", flush=True)
