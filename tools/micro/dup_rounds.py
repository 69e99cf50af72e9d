"""Duplicate check in rounds (partitions over kSpDupRound entries): a 30M
square (round-1 survivors ~20M, partitions ~9.7K) with and without a planted
duplicate among the survivors."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import oracle
from paper_1508_05931_b200 import Engine, PipelineConfig, generate

eng = Engine(0)
n = 36_000_000
xs, ys = generate("square", n, 5)
got, st = eng.hull_indices(xs, ys, PipelineConfig())
print("clean", eng.sparse_info(), st.n_after_round1)
edge = np.flatnonzero(ys < 0.001)
a, b = edge[0], edge[-1]
xs[b], ys[b] = xs[a], ys[a]
got, st = eng.hull_indices(xs, ys, PipelineConfig())
print("dup", eng.sparse_info())
want, sw = oracle.full_pipeline(xs, ys)
print("dup exact", np.array_equal(got, want), st.n_after_round1 == sw["n_after_round1"])
