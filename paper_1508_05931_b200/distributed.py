"""Sharded hull across ranks (one process per GPU, torch.distributed/NCCL).

Rank r owns a contiguous shard [offset_r, offset_r + n_r) of the input
(global input order = rank-major), so index ties resolve exactly as on one
device. The exchange follows the north star's simple form:
  1. every rank reduces its five extreme points (K1), an all-gather of
     15 doubles per rank, and every rank combines them with the reference's
     tie rules (strict compares, lowest global index; prefilter.hpp:28-39,
     angular.hpp:40-49);
  2. every rank filters its shard against the GLOBAL quadrilateral (K2) --
     the round-1 result is therefore identical to the single-device one;
  3. the survivors (x, y, global index) are gathered to rank 0 in rank order,
     which runs the rest of the pipeline (round 1 disabled: it already ran).
Step 3 is an all-gather of the survivor set, which is cheap for disks and
20M-point squares but not for on-circle inputs; the distributed sample sort /
multi-select of SURVEY.md 8e is the planned replacement.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .hull2d import Engine, PipelineConfig, StageStats


def _combine(recs: np.ndarray) -> np.ndarray:
    """recs: (R, 3, 5) = (global idx, x, y) per rank -> (3, 5) global extremes."""
    out = np.zeros((3, 5))
    R = recs.shape[0]
    for k in range(5):
        best = None
        for r in range(R):
            gi, x, y = recs[r, 0, k], recs[r, 1, k], recs[r, 2, k]
            cand = (gi, x, y)
            if best is None:
                best = cand
                continue
            bi, bx, by = best
            if k == 0:
                better = x < bx or (x == bx and gi < bi)
            elif k == 1:
                better = y < by or (y == by and gi < bi)
            elif k == 2:
                better = x > bx or (x == bx and gi < bi)
            elif k == 3:
                better = y > by or (y == by and gi < bi)
            else:
                better = y < by or (y == by and (x < bx or (x == bx and gi < bi)))
            if better:
                best = cand
        out[:, k] = best
    return out


def sharded_hull(eng: Engine, d_xs: torch.Tensor, d_ys: torch.Tensor, offset: int,
                 cfg: PipelineConfig | None = None, group=None):
    """Hull of the union of all ranks' shards. Returns (global indices as a
    numpy uint64 array, StageStats) on rank 0 and (None, None) elsewhere."""
    cfg = cfg or PipelineConfig()
    lib = eng._lib
    n = int(d_xs.numel())
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = d_xs.device
    if cfg.enable_round1:
        ex = N.gscan_extremes()
        rc = lib.gscan_shard_extremes(eng.handle, C.c_void_p(d_xs.data_ptr()),
                                      C.c_void_p(d_ys.data_ptr()), n, C.byref(ex))
        if rc:
            eng._raise(rc, "shard_extremes")
        mine = torch.tensor([[float(offset + ex.idx[k]) for k in range(5)], list(ex.x), list(ex.y)],
                            dtype=torch.float64, device=dev)
        allr = torch.empty((world, 3, 5), dtype=torch.float64, device=dev)
        dist.all_gather_into_tensor(allr, mine, group=group)
        g = _combine(allr.cpu().numpy())
        gex = N.gscan_extremes()
        for k in range(5):
            gex.idx[k] = int(g[0, k])
            gex.x[k] = g[1, k]
            gex.y[k] = g[2, k]
        surv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        n1 = C.c_uint64()
        rc = lib.gscan_shard_round1(eng.handle, C.c_void_p(d_xs.data_ptr()),
                                    C.c_void_p(d_ys.data_ptr()), n, C.byref(gex),
                                    C.c_void_p(surv.data_ptr()), C.byref(n1))
        if rc:
            eng._raise(rc, "shard_round1")
        loc = surv[: n1.value].long()
        sx, sy = d_xs[loc], d_ys[loc]
        sg = loc + offset
    else:
        sx, sy = d_xs, d_ys
        sg = torch.arange(offset, offset + n, device=dev, dtype=torch.int64)
    cnt = torch.tensor([sx.numel(), n], dtype=torch.int64, device=dev)
    both = torch.empty((world, 2), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(both, cnt, group=group)
    both = both.cpu().tolist()
    counts = [b[0] for b in both]
    n_global = sum(b[1] for b in both)
    mx = max(counts)
    pack = torch.zeros((3, mx), dtype=torch.float64, device=dev)
    pack[0, : sx.numel()] = sx
    pack[1, : sy.numel()] = sy
    pack[2, : sg.numel()] = sg.double()  # exact below 2^53
    gathered = torch.empty((world, 3, mx), dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(gathered, pack, group=group)
    if rank != 0:
        return None, None
    parts = [gathered[r, :, : counts[r]] for r in range(world)]
    allp = torch.cat(parts, dim=1)
    gx = allp[0].contiguous()
    gy = allp[1].contiguous()
    gidx = allp[2].long()
    m = int(gx.numel())
    out = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    rest = PipelineConfig(cfg.chunk_count, False, cfg.enable_round2, cfg.chunked)
    k, st = eng.hull_device(gx.data_ptr(), gy.data_ptr(), m, out.data_ptr(), m, rest)
    hull_global = gidx[out[:k].long()].cpu().numpy().astype(np.uint64)
    stats = StageStats(**{**st.__dict__, "n_input": n_global})
    return hull_global, stats
