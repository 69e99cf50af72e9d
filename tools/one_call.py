"""One C2-sized hull call (for ncu captures): python tools/one_call.py [kind] [n] [calls]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1508_05931_b200 import Engine, PipelineConfig, generate  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "square"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 1
xs, ys = generate(kind, n, 1)
eng = Engine(0)
for _ in range(calls):
    idx, st = eng.hull_indices(xs, ys, PipelineConfig())
print(kind, n, st.n_after_round1, st.n_after_round2, st.hull_size, eng.sparse_info(), flush=True)
