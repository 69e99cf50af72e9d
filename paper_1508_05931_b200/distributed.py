"""Sharded hull across ranks (one process per GPU, torch.distributed/NCCL).

Rank r owns a contiguous shard [offset_r, offset_r + n_r) of the input
(global input order = rank-major), so index ties resolve exactly as on one
device. Two paths, both exact:

* ``sparse_sharded`` (default): every rank runs the sparse
  round-2 pipeline (csrc/sparse.cuh) on its own shard through the
  ``gscan_dist_*`` phases, and only small things move between ranks:

  =====================  ==========================================  =========
  exchange               what                                         size
  =====================  ==========================================  =========
  extremes               5 extreme points per rank (all-gather)       120 B
  sample cells           pseudo-angle sample histogram (sum)          8 KB
  bucket histogram       global ranks of every bucket (sum)           192 KB
  farthest point P_l     best (dist2, index) record per rank          40 B
  P_l's in-bucket rank   points of its bucket ordered before it       8 B
  walk-angle maxima      per-bucket phi maximum (max) + phi range     384 KB
  gathered points        buckets holding slice seeds -> rank 0        ~MBs
  prefix maxima          candidate thresholds (rank 0 -> all)         384 KB
  candidates             points the walk can keep -> rank 0           ~MBs
  duplicate check        64-bit hashes, partition k -> rank k         8 B/pt
  =====================  ==========================================  =========

  Rank 0 then walks the gathered points and candidates exactly, certifies
  the skipped points, and runs Graham. No rank ever holds another rank's
  survivors, so 1B points scale.
* the survivor gather (``survivor_gather``): K1/K2 per shard, then all
  survivors to rank 0. It is the exact fallback whenever the sparse path
  declines (tie for P_l, possible duplicates, a certificate that does not
  hold, near-convex input, capacity).

The collectives go through a small interface (``Comm``) so that the same
orchestration runs under NCCL (``TorchComm``, one rank per process) or as R
simulated ranks inside one process (``LocalComm``, used by the GPU tests on a
single device).
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .hull2d import Engine, PipelineConfig, StageStats

_U32 = torch.int32  # uint32 payloads travel as int32 bit patterns
_DBG = bool(int(__import__("os").environ.get("GSCAN_DIST_DEBUG", "0") or 0))


def _combine(recs: np.ndarray) -> np.ndarray:
    """recs: (R, 3, 5) = (global idx, x, y) per rank -> (3, 5) global extremes
    with the reference's tie rules (strict compares, lowest global index;
    prefilter.hpp:28-39, angular.hpp:40-49)."""
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


def _combine_best(recs) -> tuple[tuple | None, int]:
    """Per-rank (d2_bits, global idx, ties, x, y) -> the global farthest point
    (split_regions, angular.hpp:197-204: first maximal dist2 = lowest index
    among equals) and the number of points at that distance."""
    best, ties = None, 0
    for d2, gi, t, x, y in recs:
        if t == 0:
            continue
        if best is None or d2 > best[0]:
            best, ties = (d2, gi, x, y), t
        elif d2 == best[0]:
            ties += t
            if gi < best[1]:
                best = (d2, gi, x, y)
    return best, ties


# ---------------------------------------------------------------------------
# collectives
class Comm:
    """Collectives over R ranks. Every method takes one value per rank held by
    this process (``len(local) == len(self.ranks)``) and returns one per rank."""

    world: int
    ranks: list[int]

    def allreduce(self, ts: list[torch.Tensor], op: str) -> list[torch.Tensor]:
        raise NotImplementedError

    def allgather_obj(self, objs: list) -> list:
        """-> the list of all R objects (same on every rank)."""
        raise NotImplementedError

    def allgather_i64(self, rows: list) -> np.ndarray:
        """Fixed-length int64 rows (one per local rank, same length everywhere)
        -> (R, L) int64 array on every rank: one tensor all-gather, no pickling.
        Doubles travel as their bit patterns (_i64 / _f64)."""
        raise NotImplementedError

    def gather_root(self, ts: list[torch.Tensor]) -> list[torch.Tensor] | None:
        """Variable-length 1-D tensors -> rank 0 gets all R (rank order); others None."""
        raise NotImplementedError

    def bcast_root(self, t: torch.Tensor | None, like: list[torch.Tensor]) -> list[torch.Tensor]:
        raise NotImplementedError

    def all_to_all(self, sends: list[list[torch.Tensor]]) -> list[list[torch.Tensor]]:
        """sends[k][r] from local rank k to rank r -> recv[k][s] from rank s."""
        raise NotImplementedError


class LocalComm(Comm):
    """R simulated ranks in one process (tensors on one device)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))

    def allreduce(self, ts, op):
        st = torch.stack(ts)
        r = {"sum": lambda: st.sum(0, dtype=st.dtype), "max": lambda: st.max(0).values,
             "min": lambda: st.min(0).values}[op]()
        return [r.clone() for _ in ts]

    def allgather_obj(self, objs):
        return list(objs)

    def allgather_i64(self, rows):
        return np.stack([np.asarray(r, dtype=np.int64) for r in rows])

    def gather_root(self, ts):
        return [t.clone() for t in ts]

    def bcast_root(self, t, like):
        return [t.clone() for _ in like]

    def all_to_all(self, sends):
        return [[sends[s][r].clone() for s in range(self.world)] for r in range(self.world)]


class TorchComm(Comm):
    """torch.distributed (NCCL on GPUs, gloo on CPU): this process is one rank."""

    _OPS = {"sum": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ranks = [self.rank]
        # gloo (CPU backend, e.g. ranks sharing one GPU in tests) stages device
        # tensors through host memory; NCCL moves them directly
        self.stage = dist.get_backend(group) == "gloo"
        self.cdev = torch.device("cpu") if self.stage else torch.device(
            "cuda", torch.cuda.current_device())

    def _out(self, t):  # a tensor as the backend takes it
        return t.cpu() if self.stage else t

    def allreduce(self, ts, op):
        (t,) = ts
        w = self._out(t).clone()
        dist.all_reduce(w, op=self._OPS[op], group=self.group)
        return [w.to(t.device)]

    def allgather_obj(self, objs):
        (o,) = objs
        out = [None] * self.world
        dist.all_gather_object(out, o, group=self.group)
        return out

    def allgather_i64(self, rows):
        (r,) = rows
        t = torch.as_tensor(np.asarray(r, dtype=np.int64), device=self.cdev)
        out = torch.empty((self.world, t.numel()), dtype=torch.int64, device=self.cdev)
        if self.stage:
            dist.all_gather(list(out.unbind(0)), t, group=self.group)
        else:
            dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()

    def gather_root(self, ts):
        (t,) = ts
        ns = self.allgather_i64([[t.numel()]])[:, 0].tolist()
        mx = max(max(ns), 1)
        pad = torch.zeros(mx, dtype=t.dtype, device=self.cdev)
        pad[: t.numel()] = self._out(t)
        bufs = [torch.empty(mx, dtype=t.dtype, device=self.cdev) for _ in range(self.world)] \
            if self.rank == 0 else None
        dist.gather(pad, gather_list=bufs, dst=0, group=self.group)
        if self.rank != 0:
            return None
        return [bufs[r][: ns[r]].to(t.device) for r in range(self.world)]

    def bcast_root(self, t, like):
        (ref,) = like
        buf = self._out(t).clone() if self.rank == 0 else torch.empty_like(self._out(ref))
        dist.broadcast(buf, 0, group=self.group)
        return [buf.to(ref.device)]

    def all_to_all(self, sends):
        (row,) = sends
        dev = row[0].device
        sizes = [int(x.numel()) for x in row]
        rs = [int(v) for v in self.allgather_i64([sizes])[:, self.rank]]
        out = torch.empty(sum(rs), dtype=row[0].dtype, device=self.cdev)
        if self.stage:  # gloo: point-to-point through host memory
            outs = list(torch.split(out, rs))
            reqs = []
            for r in range(self.world):
                if r == self.rank:
                    outs[r].copy_(row[r].cpu())
                    continue
                reqs.append(dist.isend(row[r].cpu().contiguous(), r, group=self.group))
                reqs.append(dist.irecv(outs[r], r, group=self.group))
            for q in reqs:
                q.wait()
        else:
            dist.all_to_all_single(out, torch.cat(list(row)), output_split_sizes=rs,
                                   input_split_sizes=sizes, group=self.group)
        return [[x.to(dev) for x in torch.split(out, rs)]]


# ---------------------------------------------------------------------------
def _i64(x: float) -> int:
    """A double's bit pattern as int64 (exact through the int64 collectives)."""
    return int(np.array([x], dtype=np.float64).view(np.int64)[0])


def _f64(v) -> float:
    return float(np.array([v], dtype=np.int64).view(np.float64)[0])


def _u64(v) -> int:
    return int(v) & 0xFFFFFFFFFFFFFFFF


def _s64(v) -> int:
    """A uint64 as the int64 with the same bits (for the int64 collectives)."""
    v = int(v) & 0xFFFFFFFFFFFFFFFF
    return v - (1 << 64) if v >= 1 << 63 else v


def _ck(eng: Engine, rc: int, what: str):
    if rc:
        eng._raise(rc, what)


def _ready(dev) -> None:
    """The phases run on the handle's own stream: tensors torch (or NCCL) just
    wrote must be complete first."""
    torch.cuda.synchronize(dev)


def _extremes(engines, shards, offsets, comm: Comm) -> N.gscan_extremes:
    recs = []
    for eng, (dx, dy), off in zip(engines, shards, offsets):
        ex = N.gscan_extremes()
        _ready(dx.device)
        _ck(eng, eng._lib.gscan_shard_extremes(eng.handle, C.c_void_p(dx.data_ptr()),
                                               C.c_void_p(dy.data_ptr()), dx.numel(), C.byref(ex)),
            "shard_extremes")
        recs.append([off + ex.idx[k] for k in range(5)] + [_i64(v) for v in ex.x]
                    + [_i64(v) for v in ex.y])
    allr = comm.allgather_i64(recs)  # (R, 15): global indices, x bits, y bits
    g = _combine(np.stack([np.array([[float(r[k]) for k in range(5)],
                                     [_f64(r[5 + k]) for k in range(5)],
                                     [_f64(r[10 + k]) for k in range(5)]]) for r in allr]))
    gex = N.gscan_extremes()
    for k in range(5):
        gex.idx[k] = int(g[0, k])
        gex.x[k] = g[1, k]
        gex.y[k] = g[2, k]
    return gex


last_decline = ""  # why the last sparse_sharded call declined (diagnostics)


def _declined(why: str):
    global last_decline
    last_decline = why
    return None


def _agree(comm: Comm, local_ok: list[bool]) -> bool:
    """Every rank's verdict -> one decision all ranks take together."""
    return bool(comm.allgather_i64([[int(bool(v))] for v in local_ok]).all())


def sparse_sharded(engines: list[Engine], shards, offsets: list[int], n_global: int,
                   cfg: PipelineConfig, comm: Comm):
    """The sharded sparse path. Returns ``(hull_global_indices, stats)`` on rank 0
    and ``(None, None)`` elsewhere when it served the call, or ``None`` when it
    declined (every rank then gets None and takes the survivor gather)."""
    global last_decline
    last_decline = ""
    dev = shards[0][0].device
    ccfg = cfg._c()
    gex = _extremes(engines, shards, offsets, comm)
    i32 = lambda n: torch.empty(n, dtype=_U32, device=dev)  # noqa: E731

    # 1. sample cells -> sum
    cells = []
    for eng, (dx, dy), off in zip(engines, shards, offsets):
        t = i32(N.SP_CELLS)
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_begin(eng.handle, C.c_void_p(dx.data_ptr()),
                                           C.c_void_p(dy.data_ptr()), dx.numel(), off, C.byref(gex),
                                           C.byref(ccfg), C.c_void_p(t.data_ptr())), "dist_begin")
        cells.append(t)
    cells = comm.allreduce(cells, "sum")

    # 2. bucket histogram -> sum; farthest point -> best; round-1 survivors -> sum
    hists, bests, n1s = [], [], []
    for eng, cl in zip(engines, cells):
        hst = i32(N.SP_BUCKETS)
        b = N.gscan_dist_best()
        n1 = C.c_uint64()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_hist(eng.handle, C.c_void_p(cl.data_ptr()),
                                          C.c_void_p(hst.data_ptr()), C.byref(b), C.byref(n1)),
            "dist_hist")
        hists.append(hst)
        bests.append((int(b.d2_bits), int(b.idx), int(b.ties), float(b.x), float(b.y)))
        n1s.append(int(n1.value))
    hists = comm.allreduce(hists, "sum")
    rows = [[_s64(bb[0]), _s64(bb[1]), bb[2], _i64(bb[3]), _i64(bb[4]), n]
            for bb, n in zip(bests, n1s)]
    allb = comm.allgather_i64(rows)
    best, ties = _combine_best([(_u64(r[0]), _u64(r[1]), int(r[2]), _f64(r[3]), _f64(r[4]))
                                for r in allb])
    n1 = int(allb[:, 5].sum())
    fail = 0
    if best is None:
        fail |= N.SP_FAIL_FEW
    elif ties != 1:
        fail |= N.SP_FAIL_TIE
    if n1 * 10 > n_global * 9:
        fail |= N.SP_FAIL_MANY
    if fail:
        return _declined(f"P_l: fail bits {fail:#x} (no point, a tie, or >= 90% of the points survive round 1)")
    pl = N.gscan_dist_best(best[0], best[1], ties, 0, best[2], best[3])

    # 3. P_l's rank inside its bucket -> sum
    lbs, fails = [], []
    for eng, hst in zip(engines, hists):
        lb, f = C.c_uint64(), C.c_uint32()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_plan(eng.handle, C.c_void_p(hst.data_ptr()), C.byref(pl), 0,
                                          C.byref(lb), C.byref(f)), "dist_plan")
        lbs.append(int(lb.value))
        fails.append(int(f.value))
    allv = comm.allgather_i64([[a, b] for a, b in zip(lbs, fails)])
    if allv[:, 1].any():
        return _declined(f"ranking P_l: fail bits {allv[:, 1].tolist()}")
    l_below = int(allv[:, 0].sum())

    # 4. F3: walk-angle maxima -> max, phi range -> min/max; gathered counts
    phis, rng, ngs, fails = [], [], [], []
    for eng in engines:
        pm = i32(N.SP_BUCKETS)
        pr = (C.c_uint32 * 2)()
        ng, f = C.c_uint64(), C.c_uint32()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_phi(eng.handle, l_below, C.c_void_p(pm.data_ptr()), pr,
                                         C.byref(ng), C.byref(f)), "dist_phi")
        phis.append(pm.to(torch.int64) & 0xFFFFFFFF)
        rng.append((int(pr[0]), int(pr[1])))
        ngs.append(int(ng.value))
        fails.append(int(f.value))
    allv = comm.allgather_i64([[a[0], a[1], b] for a, b in zip(rng, fails)])
    if allv[:, 2].any():
        return _declined(f"F3: fail bits {allv[:, 2].tolist()}")
    if _DBG:
        print(f"[dist] n1={n1} l_below={l_below} n_g={ngs} hist_sum={int(hists[0].to(torch.int64).sum())}")
    phi_lo = int(allv[:, 0].min())
    phi_hi = int(allv[:, 1].max())
    phis = comm.allreduce(phis, "max")

    # duplicate check: this rank's hashes by partition; partition range k -> rank k
    sends, cnts = [], []
    for eng in engines:
        pc = i32(N.SP_PARTS)
        ptr, nh = C.c_uint64(), C.c_uint64()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_dup_local(eng.handle, C.c_void_p(pc.data_ptr()), C.byref(ptr),
                                               C.byref(nh)), "dist_dup_local")
        parted = _wrap_u64(ptr.value, int(nh.value), dev)
        pcl = pc.to(torch.int64)
        bounds = [(k * N.SP_PARTS) // comm.world for k in range(comm.world + 1)]
        offs = torch.zeros(N.SP_PARTS + 1, dtype=torch.int64, device=dev)
        offs[1:] = torch.cumsum(pcl, 0)
        row, crow = [], []
        for k in range(comm.world):
            a, b = int(offs[bounds[k]]), int(offs[bounds[k + 1]])
            row.append(parted[a:b].clone())
            crow.append(pc[bounds[k]:bounds[k + 1]].clone())
        sends.append(row)
        cnts.append(crow)
    recv = comm.all_to_all(sends)
    rcnt = comm.all_to_all(cnts)
    dups = []
    for li, eng in enumerate(engines):
        k = comm.ranks[li]
        lo, hi = (k * N.SP_PARTS) // comm.world, ((k + 1) * N.SP_PARTS) // comm.world
        mat = torch.zeros((comm.world, N.SP_PARTS), dtype=_U32, device=dev)
        for s in range(comm.world):
            mat[s, lo:hi] = rcnt[li][s]
        blob = torch.cat(recv[li]) if sum(x.numel() for x in recv[li]) else torch.zeros(1, dtype=torch.int64, device=dev)
        nrecv = sum(x.numel() for x in recv[li])
        d = C.c_uint32()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_dup_check(eng.handle, C.c_void_p(blob.data_ptr()), nrecv,
                                               C.c_void_p(mat.data_ptr()), comm.world, C.byref(d)),
            "dist_dup_check")
        dups.append(int(d.value))
    if comm.allgather_i64([[d] for d in dups]).any():
        return _declined("possible duplicate points (hash partition exchange)")

    # 5. gathered points -> rank 0 (records {x, y, global index, bucket})
    def export(candidates: int, counts):
        out = []
        for eng, cnt in zip(engines, counts):
            xs = torch.empty(max(cnt, 1), dtype=torch.float64, device=dev)
            ys = torch.empty_like(xs)
            gi, gb = i32(max(cnt, 1)), i32(max(cnt, 1))
            n = C.c_uint64()
            _ready(dev)
            _ck(eng, eng._lib.gscan_dist_export(eng.handle, candidates, C.c_void_p(xs.data_ptr()),
                                                C.c_void_p(ys.data_ptr()), C.c_void_p(gi.data_ptr()),
                                                C.c_void_p(gb.data_ptr()), C.byref(n)),
                "dist_export")
            k = int(n.value)
            out.append((xs[:k], ys[:k], gi[:k].to(torch.int64) & 0xFFFFFFFF, gb[:k]))
        return out

    def to_root(recs):
        parts = [comm.gather_root([r[j] for r in recs]) for j in range(4)]
        if parts[0] is None:
            return None
        x = torch.cat(parts[0])
        y = torch.cat(parts[1])
        gi = torch.cat(parts[2])
        gb = torch.cat(parts[3])
        order = torch.argsort(gi)
        return x[order], y[order], gi[order], gb[order]

    groot = to_root(export(0, ngs))
    if _DBG and groot is not None:
        print(f"[dist] gathered at root {groot[0].numel()} unique idx {torch.unique(groot[2]).numel()}")
    root = 0 in comm.ranks
    r0 = comm.ranks.index(0) if root else None
    pref = None
    if root:
        gx, gy, gg, gb = groot
        n_g = int(gx.numel())
        X = torch.cat([torch.tensor([gex.x[4]], dtype=torch.float64, device=dev), gx])
        Y = torch.cat([torch.tensor([gex.y[4]], dtype=torch.float64, device=dev), gy])
        lpos = int(torch.searchsorted(gg, torch.tensor([pl.idx], device=dev)).item())
        eng0 = engines[r0]
        if lpos < n_g and int(gg[lpos]) == pl.idx:  # P_l is a gathered point
            pref = i32(N.SP_BUCKETS)
            pr = (C.c_uint32 * 2)(phi_lo, phi_hi)
            f = C.c_uint32()
            pmx = phis[r0].to(_U32)
            _ready(dev)
            rc = eng0._lib.gscan_dist_slices(eng0.handle, C.c_void_p(X.data_ptr()),
                                             C.c_void_p(Y.data_ptr()), n_g,
                                             C.c_void_p(gb.data_ptr()), 1 + lpos,
                                             C.c_void_p(pmx.data_ptr()), pr,
                                             C.c_void_p(pref.data_ptr()), C.byref(f))
            if rc == N.GSCAN_E_CAPACITY or (rc == 0 and f.value):
                pref = None
                _declined(f"dist_slices: rc {rc}, fail bits {f.value:#x}")
            else:
                _ck(eng0, rc, "dist_slices")
    if not _agree(comm, [pref is not None if comm.ranks[k] == 0 else True
                         for k in range(len(engines))]):
        return _declined(last_decline or "rank 0 could not sort the gathered points")
    prefs = comm.bcast_root(pref, [i32(N.SP_BUCKETS) for _ in engines])

    # 6. candidates -> rank 0
    ncs, fails = [], []
    for eng, pm in zip(engines, prefs):
        nc, f = C.c_uint64(), C.c_uint32()
        _ready(dev)
        _ck(eng, eng._lib.gscan_dist_cand(eng.handle, C.c_void_p(pm.data_ptr()), C.byref(nc),
                                          C.byref(f)), "dist_cand")
        ncs.append(int(nc.value))
        fails.append(int(f.value))
    allv = comm.allgather_i64([[a, b] for a, b in zip(ncs, fails)])
    m_global = int(hists[0].to(torch.int64).sum())
    n_cand = int(allv[:, 0].sum())
    if allv[:, 1].any() or n_cand > max(m_global // 8, 65536):
        return _declined(f"F4: fail bits {allv[:, 1].tolist()}, candidates {n_cand} of {m_global}")
    croot = to_root(export(1, ncs))

    # 7. rank 0: walk, certificate, Graham
    result = None
    if root:
        cx, cy, cg, cb = croot
        n_c = int(cx.numel())
        X2 = torch.cat([X, cx])
        Y2 = torch.cat([Y, cy])
        gidx = torch.cat([torch.tensor([gex.idx[4]], dtype=torch.int64, device=dev), gg, cg])
        hull = i32(max(1 + n_g + n_c, 1))
        hn, nr, f = C.c_uint64(), C.c_uint64(), C.c_uint32()
        _ready(dev)
        rc = eng0._lib.gscan_dist_finish(eng0.handle, C.c_void_p(X2.data_ptr()),
                                         C.c_void_p(Y2.data_ptr()), n_g, n_c,
                                         C.c_void_p(cb.data_ptr()), C.c_void_p(hull.data_ptr()),
                                         hull.numel(), C.byref(hn), C.byref(nr), C.byref(f))
        if rc == N.GSCAN_E_CAPACITY or (rc == 0 and f.value):
            result = None
            _declined(f"dist_finish: rc {rc}, fail bits {f.value:#x}")
        else:
            _ck(eng0, rc, "dist_finish")
            k = int(hn.value)
            hv = gidx[hull[:k].to(torch.int64) & 0xFFFFFFFF].cpu().numpy().astype(np.uint64)
            st = StageStats(n_input=n_global, n_after_round1=n1, n_after_round2=int(nr.value),
                            hull_size=k)
            result = (hv, st)
    if not _agree(comm, [result is not None if comm.ranks[k] == 0 else True
                         for k in range(len(engines))]):
        return _declined(last_decline or "rank 0: walk, certificate or Graham declined")
    return result if root else (None, None)


class _DevBuf:
    """__cuda_array_interface__ view of a device buffer owned by a handle."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def _wrap_u64(ptr: int, n: int, dev) -> torch.Tensor:
    """n uint64 (as int64) at device address ptr, copied out of the handle."""
    if n == 0:
        return torch.zeros(0, dtype=torch.int64, device=dev)
    return torch.as_tensor(_DevBuf(ptr, n), device=dev).clone()


# ---------------------------------------------------------------------------
def survivor_gather(eng: Engine, d_xs: torch.Tensor, d_ys: torch.Tensor, offset: int,
                    cfg: PipelineConfig, comm: TorchComm):
    """K1/K2 per shard, every survivor (x, y, global index) to rank 0, which runs
    the rest with round 1 disabled (it already ran)."""
    lib = eng._lib
    n = int(d_xs.numel())
    rank, world = comm.rank, comm.world
    group = comm.group
    dev = d_xs.device
    if cfg.enable_round1:
        ex = N.gscan_extremes()
        _ck(eng, lib.gscan_shard_extremes(eng.handle, C.c_void_p(d_xs.data_ptr()),
                                          C.c_void_p(d_ys.data_ptr()), n, C.byref(ex)), "shard_extremes")
        allr = comm.allgather_i64([[offset + ex.idx[k] for k in range(5)] +
                                   [_i64(v) for v in ex.x] + [_i64(v) for v in ex.y]])
        g = _combine(np.stack([np.array([[float(r[k]) for k in range(5)],
                                         [_f64(r[5 + k]) for k in range(5)],
                                         [_f64(r[10 + k]) for k in range(5)]]) for r in allr]))
        gex = N.gscan_extremes()
        for k in range(5):
            gex.idx[k] = int(g[0, k])
            gex.x[k] = g[1, k]
            gex.y[k] = g[2, k]
        surv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        n1 = C.c_uint64()
        _ck(eng, lib.gscan_shard_round1(eng.handle, C.c_void_p(d_xs.data_ptr()),
                                        C.c_void_p(d_ys.data_ptr()), n, C.byref(gex),
                                        C.c_void_p(surv.data_ptr()), C.byref(n1)), "shard_round1")
        loc = surv[: n1.value].long()
        sx, sy = d_xs[loc], d_ys[loc]
        sg = loc + offset
    else:
        sx, sy = d_xs, d_ys
        sg = torch.arange(offset, offset + n, device=dev, dtype=torch.int64)
    n_global = int(comm.allgather_i64([[n]])[:, 0].sum())
    # survivors go to rank 0 only (the other ranks hold nothing extra)
    px = comm.gather_root([sx.contiguous()])
    py = comm.gather_root([sy.contiguous()])
    pg = comm.gather_root([sg.contiguous()])
    if rank != 0:
        return None, None
    gx = torch.cat(px).contiguous()
    gy = torch.cat(py).contiguous()
    gidx = torch.cat(pg).long()
    m = int(gx.numel())
    out = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    rest = PipelineConfig(cfg.chunk_count, False, cfg.enable_round2, cfg.chunked)
    k, st = eng.hull_device(gx.data_ptr(), gy.data_ptr(), m, out.data_ptr(), m, rest)
    hull_global = gidx[out[:k].long()].cpu().numpy().astype(np.uint64)
    stats = StageStats(**{**st.__dict__, "n_input": n_global})
    return hull_global, stats


def _default_toggles(cfg: PipelineConfig) -> bool:
    return cfg.enable_round1 and cfg.enable_round2 and cfg.chunked


def sharded_hull(eng: Engine, d_xs: torch.Tensor, d_ys: torch.Tensor, offset: int,
                 cfg: PipelineConfig | None = None, group=None):
    """Hull of the union of all ranks' shards. Returns (global indices as a
    numpy uint64 array, StageStats) on rank 0 and (None, None) elsewhere."""
    cfg = cfg or PipelineConfig()
    comm = TorchComm(group)
    n = int(d_xs.numel())
    sizes = comm.allgather_i64([[n]])[:, 0].tolist()
    n_global = sum(sizes)
    # global indices are 32-bit on the device (every rank knows n_global, so
    # all of them take the same path)
    if (_default_toggles(cfg) and 65536 <= n_global < 0xFFFFFFFF and min(sizes) > 0
            and d_xs.is_cuda):
        res = sparse_sharded([eng], [(d_xs, d_ys)], [offset], n_global, cfg, comm)
        if res is not None:
            return res
    return survivor_gather(eng, d_xs, d_ys, offset, cfg, comm)


def simulate_sharded(engines: list[Engine], xs: torch.Tensor, ys: torch.Tensor,
                     cfg: PipelineConfig | None = None, bounds: list[int] | None = None):
    """All R ranks in this process on one device (LocalComm): the sharded
    sparse path exactly as R GPUs would run it. Returns (indices, stats) or
    None when it declined. bounds: shard boundaries [0, ..., n] (default
    equal shards)."""
    cfg = cfg or PipelineConfig()
    R = len(engines)
    n = int(xs.numel())
    offs = list(bounds) if bounds is not None else [n * r // R for r in range(R + 1)]
    assert len(offs) == R + 1 and offs[0] == 0 and offs[-1] == n
    shards = [(xs[offs[r]:offs[r + 1]].contiguous(), ys[offs[r]:offs[r + 1]].contiguous())
              for r in range(R)]
    return sparse_sharded(engines, shards, offs[:R], n, cfg, LocalComm(R))
