"""Per-kernel device times (profiled, non-graph) for one config.
Usage: python tools/kernel_breakdown.py kind n [debug_flag_name]"""
from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402
from paper_1508_05931_b200 import _native as N  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "circle"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
eng = Engine(0)
if len(sys.argv) > 3:
    eng.set_debug(getattr(N, sys.argv[3]))
xs, ys = generate(kind, n, 1)
eng.hull_indices(xs, ys, PipelineConfig())
eng.set_profiling(True)
idx, st = eng.hull_indices(xs, ys, PipelineConfig())
agg = {}
for name, ms in eng.kernel_times():
    agg[name] = agg.get(name, 0.0) + ms
tot = sum(agg.values())
for name, ms in sorted(agg.items(), key=lambda kv: -kv[1]):
    if ms > 0.005:
        print(f"  {name:28s} {ms * 1e3:9.1f} us  {100 * ms / tot:5.1f}%")
print(f"  sum {tot * 1e3:.1f} us; stats total {st.t_total_ms:.3f} ms; path {eng.sparse_info()} graham {eng.graham_info()}")
