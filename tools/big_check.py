"""Large-n sparse-path check: python tools/big_check.py n [n ...]
Generates gen_square(n, 1) on the device, runs the hull, prints the path,
fail bits, counts, device memory and wall time per call."""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig  # noqa: E402

for arg in sys.argv[1:]:
    n = int(float(arg))
    eng = Engine(0)
    xs = torch.empty(n, dtype=torch.float64, device="cuda")
    ys = torch.empty(n, dtype=torch.float64, device="cuda")
    eng.generate_square_device(1, 0, n, xs.data_ptr(), ys.data_ptr())
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    try:
        t0 = time.perf_counter()
        eng.reserve(n)
        t1 = time.perf_counter()
        for rep in range(3):
            t = time.perf_counter()
            k, st = eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        free, total = torch.cuda.mem_get_info()
        if os.environ.get("BIG_PROF"):
            eng.set_profiling(True)
            eng.hull_device(xs.data_ptr(), ys.data_ptr(), n, out.data_ptr(), n, PipelineConfig())
            kt = {}
            for name, ms in eng.kernel_times():
                kt[name] = kt.get(name, 0.0) + ms
            eng.set_profiling(False)
            print("  kernels (ms):", ", ".join(f"{k}={v:.2f}" for k, v in sorted(kt.items(), key=lambda a: -a[1])[:16]))
        print(f"n={n} reserve {t1 - t0:.2f}s call {dt * 1e3:.2f} ms dev_ms {st.t_total_ms:.2f} "
              f"sparse={eng.sparse_info()} n1={st.n_after_round1} n2={st.n_after_round2} "
              f"hull={st.hull_size} used={(total - free) / 1e9:.1f} GB "
              f"head={out[:4].tolist()}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"n={n} FAILED: {e}", flush=True)
    del eng, xs, ys, out
    torch.cuda.empty_cache()
