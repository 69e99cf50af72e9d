"""CPU: host logic and the C-ABI boundary (no compute calls without a GPU)."""
import os
import re
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    from paper_1508_05931_b200 import _native

    lib = _native.load()
    hdr = (ROOT / "include" / "gscan.h").read_text()
    names = set(re.findall(r"\b(gscan_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) > 20
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.SIGNATURES) == names


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          str(ROOT / "paper_1508_05931_b200/_lib/libgscan.so")],
                         capture_output=True, text=True)
    assert "sm_100a" in out.stdout


PROBE = r"""
#include "device_common.cuh"
using namespace gscan;
// each predicate alone in a kernel, its operands from memory so nothing folds
extern "C" __global__ void probe_cross(const double* p, double* o) {
  o[0] = cross_rn(p[0], p[1], p[2], p[3], p[4], p[5]);
}
extern "C" __global__ void probe_cross_edge(const double* p, double* o) {
  o[0] = cross_edge(p[0], p[1], p[2], p[3], p[4], p[5]);
}
extern "C" __global__ void probe_dist2(const double* p, double* o) { o[0] = dist2_rn(p[0], p[1]); }
"""


def test_no_fma_in_predicates(tmp_path):
    """geom.hpp:19-21 cross() and dist2 (geom.hpp:42) are unfused double
    arithmetic (the reference binary has no FMA): the device predicates,
    compiled with the library's flags, contain DMUL/DADD and no DFMA. (Fused
    ops elsewhere in the library -- the glibc atan2 restatement's intentional
    __fma_rn, the Newton steps of screened reciprocals -- are not predicates.)"""
    from paper_1508_05931_b200 import build as B
    src = tmp_path / "probe.cu"
    src.write_text(PROBE)
    obj = tmp_path / "probe.cubin"
    subprocess.run([B.NVCC, *[f for f in B.NVCC_FLAGS if f not in ("-Xcompiler", "-fPIC")],
                    f"-I{B.CSRC}", "-cubin", str(src), "-o", str(obj)], check=True)
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(obj)],
                          capture_output=True, text=True, check=True).stdout
    funcs = sass.split("Function : ")[1:]
    assert len(funcs) == 3
    for f in funcs:
        name = f.split()[0]
        assert "DMUL" in f, name
        assert "DFMA" not in f, f"{name} contains a fused multiply-add"


def test_datagen_bit_identical_to_reference(oracle_mod):
    from paper_1508_05931_b200 import generate

    if not oracle_mod.ref_available():
        pytest.skip("oracle/_ref not built")
    for kind, k in (("square", 0), ("disk", 1), ("circle", 2), ("collinear", 3)):
        for n, seed in ((1, 0), (1000, 1), (100000, 5)):
            a = generate(kind, n, seed)
            b = oracle_mod.ref_generate(k, n, seed)
            assert np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64))
            assert np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))


def test_glibc_atan2_restatement_bit_exact(tmp_path):
    """csrc/glibc_atan2.h (the device routine, compiled for the host) == host libm."""
    src = tmp_path / "t.c"
    src.write_text(textwrap.dedent("""
        #include <math.h>
        #include <stdio.h>
        #include <string.h>
        #include "glibc_atan2.h"
        static unsigned long long s = 88172645463325252ull;
        static unsigned long long r(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
        int main(void) {
          long bad = 0;
          for (long i = 0; i < 4000000; ++i) {
            double y, x;
            unsigned long long a = r(), b = r();
            switch (i % 4) {
              case 0: y = (double)(a >> 11) * 0x1p-53; x = (double)(b >> 11) * 0x1p-52 - 1.0; break;
              case 1: y = ldexp((double)(a >> 11) * 0x1p-53, (int)(b % 200) - 100);
                      x = ldexp((double)(b >> 11) * 0x1p-53, (int)(a % 200) - 100) * ((a & 1) ? -1 : 1); break;
              case 2: memcpy(&y, &a, 8); memcpy(&x, &b, 8);
                      if (!isfinite(y) || !isfinite(x)) { y = 1.0; x = -2.0; } break;
              default: y = (double)(a % 2001) - 1000.0; x = (double)(b % 2001) - 1000.0; break;
            }
            double u = atan2(y, x), v = glibc_atan2(y, x);
            if (memcmp(&u, &v, 8)) { if (bad < 5) printf("%a %a %a %a\\n", y, x, u, v); ++bad; }
          }
          printf("bad=%ld\\n", bad);
          return bad != 0;
        }
    """))
    exe = tmp_path / "t"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", f"-I{ROOT}/paper_1508_05931_b200/csrc",
                    str(src), "-o", str(exe), "-lm"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout


def test_pipeline_config_and_errors():
    from paper_1508_05931_b200 import PipelineConfig, hull2d

    c = PipelineConfig()
    assert (c.chunk_count, c.enable_round1, c.enable_round2, c.chunked) == (1024, True, True, True)
    g = c._c()
    assert g.chunk_count == 1024 and g.enable_round1 == 1 and g.reserved == 0
    with pytest.raises(ValueError):
        PipelineConfig(chunk_count=-1)._c()
    xs, ys = hull2d._as_soa(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert xs.tolist() == [1.0, 3.0] and ys.tolist() == [2.0, 4.0]
    with pytest.raises(hull2d.LengthMismatch):
        hull2d._as_soa([1.0, 2.0], [1.0])
    assert issubclass(hull2d.EmptyInput, hull2d.Error)
    assert issubclass(hull2d.ZeroChunks, hull2d.Error)


def test_engine_fails_loudly_without_gpu():
    """No CPU fallback: without a device the product raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1508_05931_b200 import Engine, NativeUnavailable

    with pytest.raises(NativeUnavailable):
        Engine(0)


def test_combine_extremes_tie_rules():
    from paper_1508_05931_b200.distributed import _combine

    # rank 0 holds the tie at lower global index, rank 1 later
    r0 = np.array([[0, 1, 2, 3, 1], [0.0, 5.0, 9.0, 5.0, 5.0], [5.0, 0.0, 5.0, 9.0, 0.0]])
    r1 = np.array([[10, 11, 12, 13, 14], [0.0, 4.0, 9.0, 6.0, 4.0], [1.0, 0.0, 1.0, 9.0, 0.0]])
    g = _combine(np.stack([r0, r1]))
    assert g[0].tolist() == [0, 1, 2, 3, 14]


GLOO_SCRIPT = r"""
import os, sys
sys.path.insert(0, sys.argv[1])
import numpy as np, torch, torch.distributed as dist
import oracle
from paper_1508_05931_b200 import generate
from paper_1508_05931_b200.distributed import _combine
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % sys.argv[2],
                        rank=int(sys.argv[3]), world_size=2)
r = dist.get_rank()
for kind, n, seed in (("square", 10001, 3), ("disk", 5000, 4), ("grid", 999, 5)):
    if kind == "grid":
        from paper_1508_05931_b200 import generate_grid
        xs, ys = generate_grid(n, seed)
    else:
        xs, ys = generate(kind, n, seed)
    lo, hi = n * r // 2, n * (r + 1) // 2
    q = oracle.find_extremes(xs[lo:hi], ys[lo:hi])
    a = oracle.select_anchor(xs[lo:hi], ys[lo:hi])
    ids = [lo + v for v in q + [a]]
    mine = torch.tensor([[float(i) for i in ids], [xs[i] for i in ids], [ys[i] for i in ids]],
                        dtype=torch.float64)
    allr = [torch.empty_like(mine) for _ in range(2)]
    dist.all_gather(allr, mine)
    g = _combine(torch.stack(allr).numpy())
    want = oracle.find_extremes(xs, ys) + [oracle.select_anchor(xs, ys)]
    assert [int(v) for v in g[0]] == want, (kind, g[0], want)
dist.barrier()
dist.destroy_process_group()
print("ok", r)
"""


def test_sharded_extremes_exchange_gloo(tmp_path):
    """The N>1 extremes exchange (distributed.py step 1) on CPU with gloo, world_size 2."""
    script = tmp_path / "g.py"
    script.write_text(GLOO_SCRIPT)
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [subprocess.Popen([sys.executable, str(script), str(ROOT), str(port), str(r)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
        assert "ok" in o


COMM_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import torch, torch.distributed as dist
from paper_1508_05931_b200.distributed import LocalComm, TorchComm
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % sys.argv[2],
                        rank=int(sys.argv[3]), world_size=2)
r = dist.get_rank()
tc, lc = TorchComm(), LocalComm(2)
# what every rank holds, as LocalComm sees all of them at once
vals = [torch.tensor([1, -5, 7 + k, 2 ** 31 - 1 - k], dtype=torch.int32) for k in range(2)]
for op in ("sum", "max", "min"):
    want = lc.allreduce(vals, op)[0]
    got = tc.allreduce([vals[r]], op)[0]
    assert got.dtype == torch.int32 and torch.equal(got, want), (op, got, want)
    # in place (the device-side data plane's form)
    loc = [v.clone() for v in vals]
    lc.allreduce_(loc, op)
    mine = vals[r].clone()
    tc.allreduce_([mine], op)
    assert torch.equal(mine, loc[r]) and torch.equal(loc[0], loc[1]), (op, mine, loc)
# fixed records: all-gather into a rank-major block
rows = [torch.arange(4, dtype=torch.int64) + 100 * k for k in range(2)]
outs = [torch.zeros(8, dtype=torch.int64) for _ in range(2)]
lc.allgather_(rows, outs)
mine = torch.zeros(8, dtype=torch.int64)
tc.allgather_([rows[r]], [mine])
assert torch.equal(mine, outs[r]) and torch.equal(mine, torch.cat(rows)), mine
var = [torch.arange(3 + 5 * k, dtype=torch.float64) * (k + 1) for k in range(2)]
for sizes in (None, [3, 8]):
    got = tc.gather_root([var[r]], sizes=sizes)
    if r == 0:
        assert all(torch.equal(a, b) for a, b in zip(got, lc.gather_root(var)))
    else:
        assert got is None
b = tc.bcast_root(var[0] if r == 0 else None, [torch.empty_like(var[0])])[0]
assert torch.equal(b, var[0])
ib = [var[0].clone(), torch.zeros_like(var[0])]
lc.bcast_(ib)
mine = var[0].clone() if r == 0 else torch.zeros_like(var[0])
tc.bcast_([mine])
assert torch.equal(mine, var[0]) and torch.equal(ib[1], var[0])
sends = [[torch.full((2 + s + 3 * d,), 10 * s + d, dtype=torch.int64) for d in range(2)] for s in range(2)]
got = tc.all_to_all([sends[r]])[0]
want = lc.all_to_all(sends)[r]
assert all(torch.equal(a, b) for a, b in zip(got, want)), (got, want)
# flat blocks with sizes known on both sides
flat = [torch.cat(sends[s]) for s in range(2)]
ss = [[2 + s + 3 * d for d in range(2)] for s in range(2)]
rs = [[2 + s + 3 * d for s in range(2)] for d in range(2)]
got = tc.all_to_all_flat([flat[r]], [ss[r]], [rs[r]])[0]
want = lc.all_to_all_flat(flat, ss, rs)[r]
assert torch.equal(got, want) and torch.equal(want, torch.cat([sends[s][r] for s in range(2)])), (got, want)
dist.barrier()
dist.destroy_process_group()
print("ok", r)
"""


def test_torch_comm_matches_local_comm_gloo(tmp_path):
    """The sharded sparse path's collectives (distributed.py TorchComm, the
    NCCL path) agree with the in-process LocalComm the GPU tests use:
    dtype-preserving reductions, object all-gather, variable-length gather
    to rank 0, broadcast, variable-size all-to-all. gloo, world_size 2."""
    script = tmp_path / "c.py"
    script.write_text(COMM_SCRIPT)
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [subprocess.Popen([sys.executable, str(script), str(ROOT), str(port), str(r)],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=240) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
        assert "ok" in o


@pytest.mark.parametrize("kind,n,seed", [("square", 3000, 1), ("disk", 2000, 2), ("circle", 500, 3),
                                          ("collinear", 300, 4), ("square", 2, 5), ("square", 1, 6)])
def test_harness_monotone_chain_matches_oracle(oracle_mod, kind, n, seed):
    """The harness's self-contained restatement of oracle::monotone_chain
    (oracle.hpp:40-79) has the oracle's vertex set; strictly_inside agrees
    with the hull (vertices are not strictly inside, the centroid of a
    non-degenerate hull is)."""
    from paper_1508_05931_b200 import generate
    from paper_1508_05931_b200.harness import monotone_chain, same_vertex_set, strictly_inside

    xs, ys = generate(kind, n, seed)
    hull = monotone_chain(xs, ys)
    idx = oracle_mod.monotone_chain(xs, ys).astype(np.int64)
    assert same_vertex_set(hull, np.stack([xs[idx], ys[idx]], 1))
    assert not strictly_inside(hull, hull[:, 0], hull[:, 1]).any()
    if len(hull) >= 3:
        c = hull.mean(0)
        assert strictly_inside(hull, np.array([c[0]]), np.array([c[1]]))[0]


def test_mt64_jump_ahead_host():
    """The on-device generator's jump-ahead (mt64_jump.cpp): the jumped
    mt19937_64 state reproduces a sequentially advanced std::mt19937_64."""
    from paper_1508_05931_b200 import _native as N
    lib = N.load()
    for seed, blocks in [(1, 0), (1, 1), (1, 6), (7, 37), (2**63 + 5, 3)]:
        assert lib.gscan_mt64_jump_check(seed, blocks) == 0, (seed, blocks)
