"""GPU: the sharded sparse path (paper_1508_05931_b200/distributed.py,
SURVEY.md 8e), run as R simulated ranks on one device (LocalComm): every
rank's phases run on its own handle and shard, the collectives are done in
process. Bit-exact against the CPU oracle on the concatenated input, and the
declines (duplicates across ranks, near-convex input) return None so the
caller takes the survivor gather."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engines():
    from paper_1508_05931_b200 import Engine

    return [Engine(0) for _ in range(4)]


def _check(engines, oracle_mod, xs, ys, R, **cfg):
    from paper_1508_05931_b200 import PipelineConfig
    from paper_1508_05931_b200.distributed import simulate_sharded

    dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    res = simulate_sharded(engines[:R], dx, dy, PipelineConfig(**cfg))
    if res is None:
        return None
    got, st = res
    want, sw = oracle_mod.full_pipeline(xs, ys, **cfg)
    assert np.array_equal(got, want), (R, got[:10], want[:10])
    for k in ("n_after_round1", "n_after_round2", "hull_size"):
        assert getattr(st, k) == sw[k], k
    assert st.n_input == len(xs)
    return st


@pytest.mark.parametrize("kind", ["square", "disk", "gauss"])
@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_sparse_matches_oracle(engines, oracle_mod, kind, R):
    from paper_1508_05931_b200 import generate

    n = 600_000
    if kind == "gauss":
        rng = np.random.default_rng(R)
        xs, ys = rng.standard_normal(n), rng.standard_normal(n)
    else:
        xs, ys = generate(kind, n, R)
    st = _check(engines, oracle_mod, xs, ys, R)
    from paper_1508_05931_b200 import distributed as D

    assert st is not None, f"the sharded sparse path declined: {D.last_decline}"


@pytest.mark.parametrize("chunks", [7, 100])
def test_sharded_sparse_chunk_counts(engines, oracle_mod, chunks):
    from paper_1508_05931_b200 import generate

    xs, ys = generate("square", 400_000, 11)
    assert _check(engines, oracle_mod, xs, ys, 2, chunk_count=chunks) is not None


def test_sharded_duplicate_across_ranks_declines(engines, oracle_mod):
    """A duplicate whose two copies live on different ranks must be found by
    the partition exchange: the path declines (the survivor gather is exact)."""
    from paper_1508_05931_b200 import generate

    xs, ys = generate("square", 400_000, 12)
    edge = np.flatnonzero(ys < 0.01)  # round-1 survivors near the bottom edge
    a, b = edge[0], edge[-1]          # first half / second half of the input
    assert a < 200_000 <= b
    xs[b], ys[b] = xs[a], ys[a]
    assert _check(engines, oracle_mod, xs, ys, 2) is None


def test_sharded_near_circle_declines(engines, oracle_mod):
    from paper_1508_05931_b200 import generate

    xs, ys = generate("circle", 300_000, 3)
    assert _check(engines, oracle_mod, xs, ys, 3) is None


NCCL_SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_1508_05931_b200 import Engine, PipelineConfig, generate
from paper_1508_05931_b200 import distributed as D
torch.cuda.set_device(0)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%s" % sys.argv[2], rank=0, world_size=1)
xs, ys = generate("square", 500_000, 21)
eng = Engine(0)
dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
got, st = D.sharded_hull(eng, dx, dy, 0, PipelineConfig())
assert D.last_decline == "", D.last_decline
want, sw = oracle.full_pipeline(xs, ys)
assert np.array_equal(got, want)
assert st.n_after_round2 == sw["n_after_round2"] and st.hull_size == sw["hull_size"]
dist.destroy_process_group()
print("ok")
"""


def test_sharded_hull_over_nccl(tmp_path):
    """sharded_hull through TorchComm on a 1-rank NCCL group: every collective
    of the multi-GPU run (all_gather_object, all_reduce, all_gather_into_tensor,
    broadcast, all_to_all_single) on CUDA tensors, and the sparse path serves."""
    import socket
    import subprocess
    import sys
    from pathlib import Path

    script = tmp_path / "n.py"
    script.write_text(NCCL_SCRIPT)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = Path(__file__).resolve().parents[1]
    p = subprocess.run([sys.executable, str(script), str(root), str(port)], capture_output=True,
                       text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "ok" in p.stdout


def test_sharded_uneven_shards_tiny_ranks(engines, oracle_mod):
    """Shards smaller than chunk_count next to a large one (the
    slice grids must follow the GLOBAL slice count, not rank 0's shard)."""
    from paper_1508_05931_b200 import PipelineConfig, generate
    from paper_1508_05931_b200.distributed import simulate_sharded

    xs, ys = generate("square", 400_000, 11)
    n = len(xs)
    for bounds in ([0, 100, n - 50, n], [0, 3, 7, n], [0, n - 900, n - 10, n]):
        dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        res = simulate_sharded(engines[:3], dx, dy, PipelineConfig(), bounds=bounds)
        if res is None:
            continue  # a decline is exact (the caller takes the survivor gather)
        got, st = res
        want, sw = oracle_mod.full_pipeline(xs, ys)
        assert np.array_equal(got, want), bounds
        assert st.n_after_round2 == sw["n_after_round2"], bounds


GLOO2_SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_1508_05931_b200 import Engine, PipelineConfig, generate
from paper_1508_05931_b200 import distributed as D
rank = int(sys.argv[3])
torch.cuda.set_device(0)
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % sys.argv[2], rank=rank,
                        world_size=2)
kind, n = sys.argv[4], int(sys.argv[5])
xs, ys = generate(kind, n, 23)
lo, hi = n * rank // 2, n * (rank + 1) // 2
eng = Engine(0)
if rank == 0:
    eng.reserve(n)
dx, dy = torch.from_numpy(xs[lo:hi].copy()).cuda(), torch.from_numpy(ys[lo:hi].copy()).cuda()
got, st = D.sharded_hull(eng, dx, dy, lo, PipelineConfig())
if rank == 0:
    want, sw = oracle.full_pipeline(xs, ys)
    assert np.array_equal(got, want), (got[:8], want[:8])
    assert st.n_after_round2 == sw["n_after_round2"] and st.hull_size == sw["hull_size"]
    print("ok", "sparse" if D.last_decline == "" else "declined: " + D.last_decline)
else:
    assert got is None
dist.destroy_process_group()
"""


@pytest.mark.parametrize("kind,n", [("square", 600_000), ("disk", 400_000), ("circle", 100_000)])
def test_sharded_hull_two_processes_gloo(tmp_path, kind, n):
    """The full sharded_hull with TorchComm across two real processes (world
    size 2, gloo staging device tensors through the host, both ranks on
    cuda:0): every exchange of the multi-GPU path, and the survivor-gather
    fallback for the circle (near-convex: the sparse path declines)."""
    import socket
    import subprocess
    import sys
    from pathlib import Path

    script = tmp_path / "g2.py"
    script.write_text(GLOO2_SCRIPT)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    root = Path(__file__).resolve().parents[1]
    procs = [subprocess.Popen([sys.executable, str(script), str(root), str(port), str(r), kind, str(n)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    assert outs[0][0].startswith("ok")
    if kind != "circle":
        assert "sparse" in outs[0][0], outs[0][0]


def test_sharded_distributed_verification(engines, oracle_mod):
    """Rank 0's certificate forced off (GSCAN_DEBUG_SPARSE_VERIFY): every rank
    runs F6 on its own shard against rank 0's broadcast round-2 output
    (distributed F6), and the sharded path still serves, bit-exact."""
    from paper_1508_05931_b200 import _native as N
    from paper_1508_05931_b200 import distributed as D
    from paper_1508_05931_b200 import generate

    xs, ys = generate("disk", 500_000, 21)
    engines[0].set_debug(N.DEBUG_SPARSE_VERIFY)
    try:
        st = _check(engines, oracle_mod, xs, ys, 3)
    finally:
        engines[0].set_debug(0)
    assert st is not None, f"declined: {D.last_decline}"


def test_sharded_host_waits(engines, oracle_mod, monkeypatch):
    """The device-side data plane: one call reads device data back on the
    host at most four times (three verdict points and the output)."""
    from paper_1508_05931_b200 import distributed as D
    from paper_1508_05931_b200 import generate

    xs, ys = generate("square", 400_000, 5)
    calls = []
    real_cpu = torch.Tensor.cpu

    def counting_cpu(self, *a, **k):
        if self.is_cuda:
            calls.append(tuple(self.shape))
        return real_cpu(self, *a, **k)

    monkeypatch.setattr(torch.Tensor, "cpu", counting_cpu)
    st = _check(engines, oracle_mod, xs, ys, 4)
    monkeypatch.undo()
    assert st is not None, D.last_decline
    assert len(calls) <= 4, calls


@pytest.mark.parametrize("kind", ["circle", "square", "disk", "dups"])
@pytest.mark.parametrize("R", [2, 3, 4])
def test_sample_sort_matches_oracle(engines, oracle_mod, kind, R):
    """The distributed sample sort (the sharded path's exact fallback for
    near-convex inputs): round-1 survivors routed by exact key
    ranges, sorted and deduplicated per rank, round 2 and Graham on rank 0 --
    bit-exact against the oracle, duplicates across ranks included."""
    from paper_1508_05931_b200 import PipelineConfig, generate
    from paper_1508_05931_b200.distributed import simulate_sample_sort

    n = 200_000
    if kind == "dups":  # every point twice, the copies in other shards
        xs, ys = generate("disk", n // 2, R)
        xs, ys = np.concatenate([xs, xs[::-1]]), np.concatenate([ys, ys[::-1]])
    else:
        xs, ys = generate(kind, n, R)
    for cfg in (dict(), dict(chunk_count=7), dict(enable_round2=False), dict(chunked=False)):
        dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
        got, st = simulate_sample_sort(engines[:R], dx, dy, PipelineConfig(**cfg))
        want, sw = oracle_mod.full_pipeline(xs, ys, **cfg)
        assert np.array_equal(got, want), (kind, R, cfg, got[:8], want[:8])
        for k in ("n_after_round1", "n_after_round2", "hull_size"):
            assert getattr(st, k) == sw[k], (k, cfg)


def test_sample_sort_uneven_shards(engines, oracle_mod):
    """Shards of 1, 5 and the rest points, and a shard that receives no key range."""
    from paper_1508_05931_b200 import PipelineConfig, generate
    from paper_1508_05931_b200.distributed import simulate_sample_sort

    xs, ys = generate("circle", 50_000, 4)
    dx, dy = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    got, st = simulate_sample_sort(engines[:3], dx, dy, PipelineConfig(), bounds=[0, 1, 6, 50_000])
    want, sw = oracle_mod.full_pipeline(xs, ys)
    assert np.array_equal(got, want)
    assert st.n_after_round2 == sw["n_after_round2"]
