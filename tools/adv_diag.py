import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import test_gpu_adversarial as t
from paper_1508_05931_b200 import Engine, PipelineConfig
eng = Engine(0)
for f in t.FAMILIES:
    for n in (100_003, 1_000_000):
        xs, ys = t.make(f, n, 1)
        idx, st = eng.hull_indices(xs, ys, PipelineConfig())
        print(f, n, eng.sparse_info(), st.n_after_round1, st.n_after_round2, st.hull_size, flush=True)
