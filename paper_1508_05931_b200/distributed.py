"""Sharded hull across ranks (one process per GPU, torch.distributed/NCCL).

Rank r owns a contiguous shard [offset_r, offset_r + n_r) of the input
(global input order = rank-major), so index ties resolve exactly as on one
device. Two paths, both exact:

* ``sparse_sharded`` (default): every rank runs the sparse
  round-2 pipeline (csrc/sparse.cuh) on its own shard through the
  enqueue-only ``gscan_dist_enq_*`` phases, and only small things move
  between ranks. Device-side data plane: per-phase records are all-gathered
  and combined by the next phase on the device, the fixed-size collectives
  run in place on the handle's buffers, all on one stream; the host waits
  for the device three times per call (sizes of the variable exchanges, the
  candidate counts, rank 0's verdict):

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
  the skipped points (when the certificate does not hold, every rank runs
  F6 on its own shard against rank 0's broadcast round-2 output), and runs
  Graham. No rank ever holds another rank's survivors, so 1B points scale.
* the survivor gather (``survivor_gather``): K1/K2 per shard, then all
  survivors to rank 0. It is the exact fallback whenever the sparse path
  declines (tie for P_l, possible duplicates, a failed distributed F6,
  near-convex input, capacity).

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


# ---------------------------------------------------------------------------
# collectives
class Comm:
    """Collectives over R ranks. Every method takes one value per rank held by
    this process (``len(local) == len(self.ranks)``) and returns one per rank."""

    world: int
    ranks: list[int]

    def allreduce(self, ts: list[torch.Tensor], op: str) -> list[torch.Tensor]:
        raise NotImplementedError

    def allgather_i64(self, rows: list) -> np.ndarray:
        """Fixed-length int64 rows (one per local rank, same length everywhere)
        -> (R, L) int64 array on every rank: one tensor all-gather, no pickling.
        Doubles travel as their bit patterns (_i64 / _f64)."""
        raise NotImplementedError

    def gather_root(self, ts: list[torch.Tensor], sizes: list[int] | None = None) -> list[torch.Tensor] | None:
        """Variable-length 1-D tensors -> rank 0 gets all R (rank order); others
        None. sizes: every rank's length when the caller knows them (no size
        exchange)."""
        raise NotImplementedError

    def bcast_root(self, t: torch.Tensor | None, like: list[torch.Tensor]) -> list[torch.Tensor]:
        raise NotImplementedError

    def all_to_all(self, sends: list[list[torch.Tensor]]) -> list[list[torch.Tensor]]:
        """sends[k][r] from local rank k to rank r -> recv[k][s] from rank s."""
        raise NotImplementedError

    # in-place device collectives, ordered on the current stream (no host wait
    # under NCCL): the device-side data plane of sparse_sharded
    def allreduce_(self, ts: list[torch.Tensor], op: str) -> None:
        raise NotImplementedError

    def allgather_(self, rows: list[torch.Tensor], outs: list[torch.Tensor]) -> None:
        """rows[k] (L) of local rank k -> every outs[k] (R * L), rank-major."""
        raise NotImplementedError

    def bcast_(self, ts: list[torch.Tensor]) -> None:
        """Rank 0's tensor into every rank's (same shape)."""
        raise NotImplementedError

    def all_to_all_flat(self, inps: list[torch.Tensor], send_sizes: list[list[int]],
                        recv_sizes: list[list[int]]) -> list[torch.Tensor]:
        """inps[k]: local rank k's blocks for ranks 0..R-1 back to back
        (send_sizes[k][r] elements each) -> per local rank the blocks from
        ranks 0..R-1 back to back (recv_sizes[k][s] each; sizes known)."""
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

    def allgather_i64(self, rows):
        return np.stack([np.asarray(r, dtype=np.int64) for r in rows])

    def gather_root(self, ts, sizes=None):
        return [t.clone() for t in ts]

    def bcast_root(self, t, like):
        return [t.clone() for _ in like]

    def all_to_all(self, sends):
        return [[sends[s][r].clone() for s in range(self.world)] for r in range(self.world)]

    def allreduce_(self, ts, op):
        st = torch.stack(ts)
        r = {"sum": lambda: st.sum(0, dtype=st.dtype), "max": lambda: st.max(0).values,
             "min": lambda: st.min(0).values}[op]()
        for t in ts:
            t.copy_(r)

    def allgather_(self, rows, outs):
        cat = torch.cat(rows)
        for o in outs:
            o.copy_(cat)

    def bcast_(self, ts):
        for t in ts[1:]:
            t.copy_(ts[0])

    def all_to_all_flat(self, inps, send_sizes, recv_sizes):
        blocks = [list(torch.split(inp[: sum(sz)], sz)) for inp, sz in zip(inps, send_sizes)]
        return [torch.cat([blocks[s][r] for s in range(self.world)]) for r in range(self.world)]


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

    def allgather_i64(self, rows):
        (r,) = rows
        t = torch.as_tensor(np.asarray(r, dtype=np.int64), device=self.cdev)
        out = torch.empty((self.world, t.numel()), dtype=torch.int64, device=self.cdev)
        if self.stage:
            dist.all_gather(list(out.unbind(0)), t, group=self.group)
        else:
            dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().numpy()

    def gather_root(self, ts, sizes=None):
        (t,) = ts
        ns = list(sizes) if sizes is not None else self.allgather_i64([[t.numel()]])[:, 0].tolist()
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

    def allreduce_(self, ts, op):
        (t,) = ts
        if self.stage:
            w = t.cpu()
            dist.all_reduce(w, op=self._OPS[op], group=self.group)
            t.copy_(w)
        else:
            dist.all_reduce(t, op=self._OPS[op], group=self.group)

    def allgather_(self, rows, outs):
        (r,), (o,) = rows, outs
        if self.stage:
            w = torch.empty((self.world, r.numel()), dtype=r.dtype)
            dist.all_gather(list(w.unbind(0)), r.cpu(), group=self.group)
            o.copy_(w.view(-1))
        else:
            dist.all_gather_into_tensor(o, r, group=self.group)

    def bcast_(self, ts):
        (t,) = ts
        if self.stage:
            w = t.cpu()
            dist.broadcast(w, 0, group=self.group)
            t.copy_(w)
        else:
            dist.broadcast(t, 0, group=self.group)

    def all_to_all_flat(self, inps, send_sizes, recv_sizes):
        (inp,), (ss,), (rs,) = inps, send_sizes, recv_sizes
        ss, rs = [int(v) for v in ss], [int(v) for v in rs]
        out = torch.empty(sum(rs), dtype=inp.dtype, device=inp.device)
        if self.stage:  # gloo: point-to-point through host memory
            src = list(torch.split(inp[: sum(ss)].cpu(), ss))
            outs = list(torch.split(torch.empty(sum(rs), dtype=inp.dtype), rs))
            reqs = []
            for r in range(self.world):
                if r == self.rank:
                    outs[r].copy_(src[r])
                    continue
                reqs.append(dist.isend(src[r].contiguous(), r, group=self.group))
                reqs.append(dist.irecv(outs[r], r, group=self.group))
            for q in reqs:
                q.wait()
            out.copy_(torch.cat(outs))
        else:
            dist.all_to_all_single(out, inp[: sum(ss)], output_split_sizes=rs,
                                   input_split_sizes=ss, group=self.group)
        return [out]


# ---------------------------------------------------------------------------
def _i64(x: float) -> int:
    """A double's bit pattern as int64 (exact through the int64 collectives)."""
    return int(np.array([x], dtype=np.float64).view(np.int64)[0])


def _f64(v) -> float:
    return float(np.array([v], dtype=np.int64).view(np.float64)[0])


def _ck(eng: Engine, rc: int, what: str):
    if rc:
        eng._raise(rc, what)


last_decline = ""  # why the last sparse_sharded call declined (diagnostics)


def _declined(why: str):
    global last_decline
    last_decline = why
    return None


# ---------------------------------------------------------------------------
# device-side data plane: record words (include/gscan.h, sparse.cuh kRx*)
_RX_F2, _RX_PLAN, _RX_F3, _RX_F4, _RX_VER = 16, 24, 28, 36, 40
_SIGN = -(1 << 31)  # int32 0x80000000: unsigned order <-> signed order


def _view(ptr: int, n: int, dtype: torch.dtype, dev) -> torch.Tensor:
    """A torch view (no copy) of n elements of a handle-owned device buffer."""
    ts = {torch.int64: "<i8", torch.int32: "<i4", torch.float64: "<f8"}[dtype]
    if n == 0:
        return torch.empty(0, dtype=dtype, device=dev)
    return torch.as_tensor(_DevBuf(ptr, n, ts), device=dev)


class _Bufs:
    """One rank's gscan_dist_bufs as device tensor views."""

    def __init__(self, eng: Engine, R: int, dev):
        b = N.gscan_dist_bufs()
        _ck(eng, eng._lib.gscan_dist_buffers(eng.handle, C.byref(b)), "dist_buffers")
        self.raw = b
        self.L = int(b.rec_len)
        self.rec = _view(b.rec, self.L, torch.int64, dev)
        self.recs = _view(b.recs, R * self.L, torch.int64, dev)
        self.ext = _view(b.ext, 15, torch.int64, dev)
        self.cells = _view(b.cells, int(b.cells_n), torch.int32, dev)
        self.hist = _view(b.hist, int(b.buckets), torch.int32, dev)
        self.phimax = _view(b.phimax, int(b.buckets), torch.int32, dev)
        self.pref = _view(b.pref, int(b.buckets) + 1, torch.int32, dev)
        self.part_counts = _view(b.part_counts, int(b.parts), torch.int32, dev)


def _bind_stream(engines: list[Engine], dev) -> torch.cuda.Stream:
    """One torch stream for every handle of this process: the phases, the
    collectives and the torch ops between them are then ordered on it without
    host waits (simulated ranks share it, so they serialise on it too)."""
    s = getattr(engines[0], "_dist_stream", None)
    if s is None or any(getattr(e, "_dist_stream", None) is not s for e in engines):
        s = torch.cuda.Stream(dev)
        for e in engines:
            _ck(e, e._lib.gscan_set_stream(e.handle, C.c_void_p(s.cuda_stream)), "set_stream")
            e._dist_stream = s
    return s


def sparse_sharded(engines: list[Engine], shards, offsets: list[int], n_global: int,
                   cfg: PipelineConfig, comm: Comm):
    """The sharded sparse path. Returns ``(hull_global_indices, stats)`` on rank 0
    and ``(None, None)`` elsewhere when it served the call, or ``None`` when it
    declined (every rank then gets None and takes the survivor gather).

    Device-side data plane: the ``gscan_dist_enq_*`` phases only enqueue;
    each writes a fixed record that the next phase combines on the device
    after an all-gather, and the fixed-size exchanges run in place on the
    handle's buffers, all on one stream. The host waits for the device at
    three points (sizes of the hash all-to-all and of the gathered points;
    candidate counts; rank 0's verdict), plus one when the certificate does
    not hold and the shards run F6."""
    global last_decline
    last_decline = ""
    dev = shards[0][0].device
    stream = _bind_stream(engines, dev)
    stream.wait_stream(torch.cuda.current_stream(dev))  # the shards were written there
    with torch.cuda.stream(stream):
        res = _sparse_sharded(engines, shards, offsets, n_global, cfg, comm, dev)
    torch.cuda.current_stream(dev).wait_stream(stream)
    return res


def _sparse_sharded(engines, shards, offsets, n_global, cfg, comm, dev):
    R = comm.world
    ccfg = cfg._c()
    bufs = []
    for eng, (dx, dy), off in zip(engines, shards, offsets):
        _ck(eng, eng._lib.gscan_dist_enq_begin(eng.handle, C.c_void_p(dx.data_ptr()),
                                               C.c_void_p(dy.data_ptr()), dx.numel(), off,
                                               C.byref(ccfg)), "dist_enq_begin")
        bufs.append(_Bufs(eng, R, dev))
    L = bufs[0].L

    def gather_recs():
        comm.allgather_([b.rec for b in bufs], [b.recs for b in bufs])

    def each(fn, what, *args):
        for eng in engines:
            _ck(eng, getattr(eng._lib, fn)(eng.handle, *args), what)

    # extremes -> global (device); sample cells -> sum; F2: histogram -> sum,
    # P_l records; plan: P_l's in-bucket rank; F3: walk-angle maxima -> max
    gather_recs()
    each("gscan_dist_enq_sample", "dist_enq_sample", R)
    comm.allreduce_([b.cells for b in bufs], "sum")
    each("gscan_dist_enq_f2", "dist_enq_f2")
    comm.allreduce_([b.hist for b in bufs], "sum")
    gather_recs()
    each("gscan_dist_enq_plan", "dist_enq_plan", R, n_global)
    gather_recs()
    each("gscan_dist_enq_f3", "dist_enq_f3", R)
    for b in bufs:
        b.phimax.bitwise_xor_(_SIGN)
    comm.allreduce_([b.phimax for b in bufs], "max")
    for b in bufs:
        b.phimax.bitwise_xor_(_SIGN)
    gather_recs()

    # duplicate check, step 1: hashes by partition; partition range k -> rank k
    each("gscan_dist_enq_dup_local", "dist_enq_dup_local", R)
    P = N.SP_PARTS
    bounds = [(k * P) // R for k in range(R + 1)]
    widths = [bounds[r + 1] - bounds[r] for r in range(R)]
    send_tot, cnt_recv = [], []
    for li, b in enumerate(bufs):
        pc = b.part_counts.to(torch.int64)
        send_tot.append(torch.stack([pc[bounds[r]:bounds[r + 1]].sum() for r in range(R)]))
    me = comm.ranks
    cnt_recv = comm.all_to_all_flat([b.part_counts for b in bufs], [widths] * len(bufs),
                                    [[widths[k]] * R for k in me])
    recv_tot = [c.to(torch.int64).view(R, widths[k]).sum(1) for c, k in zip(cnt_recv, me)]

    # host sync 1
    pack = torch.cat([bufs[0].recs[: R * L]] + send_tot + recv_tot).cpu().numpy()
    recs = pack[: R * L].reshape(R, L)
    off = R * L
    send_sz = [pack[off + R * k: off + R * (k + 1)].tolist() for k in range(len(bufs))]
    off += R * len(bufs)
    recv_sz = [pack[off + R * k: off + R * (k + 1)].tolist() for k in range(len(bufs))]
    fail = int(np.bitwise_or.reduce(recs[:, _RX_F3 + 3]))
    if fail:
        return _declined(f"fail bits {fail:#x} (P_l, its rank or F3)")
    n1 = int(recs[:, _RX_F2 + 5].sum())
    M = int(recs[0, _RX_PLAN + 2])
    n_g = [int(v) for v in recs[:, _RX_F3 + 2]]
    if _DBG:
        print(f"[dist] n1={n1} M={M} n_g={n_g}")

    # duplicate check, step 2: the hash blocks; the receiver checks its partitions
    parted = [_view(b.raw.parted, max(int(sum(sz)), 1), torch.int64, dev)[: int(sum(sz))]
              for b, sz in zip(bufs, send_sz)]
    recv = comm.all_to_all_flat(parted, send_sz, recv_sz)
    for li, (eng, k) in enumerate(zip(engines, me)):
        lo, hi = bounds[k], bounds[k + 1]
        mat = torch.zeros((R, P), dtype=_U32, device=dev)
        mat[:, lo:hi] = cnt_recv[li].view(R, hi - lo)
        blob = recv[li] if recv[li].numel() else torch.zeros(1, dtype=torch.int64, device=dev)
        _ck(eng, eng._lib.gscan_dist_enq_dup_check(eng.handle, C.c_void_p(blob.data_ptr()),
                                                   int(recv[li].numel()), C.c_void_p(mat.data_ptr()),
                                                   R), "dist_enq_dup_check")

    # gathered points -> rank 0 (records {x, y, global index, bucket}; sizes known)
    def export(which: int, counts: list[int]):
        out = []
        for eng, k in zip(engines, me):
            cnt = counts[k]
            xs = torch.empty(max(cnt, 1), dtype=torch.float64, device=dev)
            ys = torch.empty_like(xs)
            gi = torch.empty(max(cnt, 1), dtype=_U32, device=dev)
            gb = torch.empty_like(gi)
            _ck(eng, eng._lib.gscan_dist_enq_export(eng.handle, which, C.c_void_p(xs.data_ptr()),
                                                    C.c_void_p(ys.data_ptr()),
                                                    C.c_void_p(gi.data_ptr()),
                                                    C.c_void_p(gb.data_ptr())), "dist_enq_export")
            out.append((xs[:cnt], ys[:cnt], gi[:cnt], gb[:cnt]))
        parts = [comm.gather_root([r[j] for r in out], sizes=counts) for j in range(4)]
        if parts[0] is None:
            return None
        x, y = torch.cat(parts[0]), torch.cat(parts[1])
        gi = torch.cat(parts[2]).to(torch.int64) & 0xFFFFFFFF
        gb = torch.cat(parts[3])
        order = torch.argsort(gi)
        return x[order], y[order], gi[order], gb[order].contiguous()

    groot = export(0, n_g)
    root = 0 in me
    r0 = me.index(0) if root else None
    if root:
        eng0, b0 = engines[r0], bufs[r0]
        gx, gy, gg, gb = groot
        ng = int(sum(n_g))
        X = torch.cat([b0.ext[9:10].view(torch.float64), gx])
        Y = torch.cat([b0.ext[14:15].view(torch.float64), gy])
        rc = eng0._lib.gscan_dist_enq_slices(eng0.handle, C.c_void_p(X.data_ptr()),
                                             C.c_void_p(Y.data_ptr()), ng, C.c_void_p(gb.data_ptr()),
                                             C.c_void_p(gg.data_ptr()), M)
        if rc == N.GSCAN_E_CAPACITY:  # rank 0 cannot hold them: every rank declines after F4
            b0.pref[-1].fill_(N.SP_FAIL_CAP)
        else:
            _ck(eng0, rc, "dist_enq_slices")
    comm.bcast_([b.pref for b in bufs])
    each("gscan_dist_enq_cand", "dist_enq_cand")
    gather_recs()

    # host sync 2
    recs = bufs[0].recs[: R * L].view(R, L).cpu().numpy()
    fail = int(np.bitwise_or.reduce(recs[:, _RX_F4 + 1]))
    n_c = [int(v) for v in recs[:, _RX_F4]]
    if fail or sum(n_c) > max((M - 1) // 8, 65536):
        return _declined(f"F4 / duplicate check / rank 0: fail bits {fail:#x}, candidates "
                         f"{sum(n_c)} of {M - 1}")
    croot = export(1, n_c)

    # rank 0: walk, certificate, Graham (its own host wait); its verdict to every rank
    msg = torch.zeros(3, dtype=torch.int64, device=dev)
    hull_x = None
    if root:
        cx, cy, cg, cb = croot
        X2, Y2 = torch.cat([X, cx]), torch.cat([Y, cy])
        gidx = torch.cat([b0.ext[4:5], gg, cg])
        hull = torch.empty(max(X2.numel(), 1), dtype=_U32, device=dev)
        hn, nr, stat, f = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        rc = eng0._lib.gscan_dist_root_finish(eng0.handle, C.c_void_p(X2.data_ptr()),
                                              C.c_void_p(Y2.data_ptr()), ng, int(sum(n_c)),
                                              C.c_void_p(cb.data_ptr()), M,
                                              C.c_void_p(hull.data_ptr()), hull.numel(),
                                              C.byref(hn), C.byref(nr), C.byref(stat), C.byref(f))
        if rc == N.GSCAN_E_CAPACITY:
            stat.value = 2
            _declined(f"dist_root_finish: {eng0._lib.gscan_last_error(eng0.handle).decode()}")
        else:
            _ck(eng0, rc, "dist_root_finish")
            if stat.value == 2:
                _declined(f"rank 0 walk / certificate / Graham: fail bits {f.value:#x}")
        status, n_r, k = int(stat.value), int(nr.value), int(hn.value)
        msg[0], msg[1] = status, n_r  # device fills, no host wait
        if status != 2:
            hull_x = gidx[hull[:k].to(torch.int64) & 0xFFFFFFFF]
    msgs = [msg if comm.ranks[k] == 0 else torch.zeros(3, dtype=torch.int64, device=dev)
            for k in range(len(engines))]
    comm.bcast_(msgs)
    if not root:
        status, n_r, _ = (int(v) for v in msgs[0].cpu().tolist())  # host sync 3
    if status == 2:
        return _declined(last_decline or "rank 0: walk, certificate or Graham declined")
    if status == 1:
        # the certificate did not prove the skipped points: every rank checks
        # its own (distributed F6) against rank 0's round-2 output
        nb = N.SP_BUCKETS
        vb = []
        for b, k in zip(bufs, me):
            if k == 0:
                vb.append((_view(b.raw.rlo, nb + 1, torch.int32, dev),
                           _view(b.raw.rx, n_r, torch.float64, dev),
                           _view(b.raw.ry, n_r, torch.float64, dev)))
            else:
                vb.append((torch.empty(nb + 1, dtype=torch.int32, device=dev),
                           torch.empty(n_r, dtype=torch.float64, device=dev),
                           torch.empty(n_r, dtype=torch.float64, device=dev)))
        for j in range(3):
            comm.bcast_([v[j] for v in vb])
        for eng, (rl, rx, ry) in zip(engines, vb):
            _ck(eng, eng._lib.gscan_dist_enq_verify(eng.handle, C.c_void_p(rl.data_ptr()),
                                                    C.c_void_p(rx.data_ptr()),
                                                    C.c_void_p(ry.data_ptr())), "dist_enq_verify")
        gather_recs()
        recs = bufs[0].recs[: R * L].view(R, L).cpu().numpy()  # host sync 4
        vfail = int(np.bitwise_or.reduce(recs[:, _RX_VER + 1]))
        if vfail:
            return _declined(f"distributed F6: {int(recs[:, _RX_VER].sum())} skipped points "
                             f"would not be discarded (fail bits {vfail:#x})")
    if not root:
        return None, None
    hv = hull_x.cpu().numpy().astype(np.uint64)  # the output
    return hv, StageStats(n_input=n_global, n_after_round1=n1, n_after_round2=n_r,
                          hull_size=int(hv.size))


class _DevBuf:
    """__cuda_array_interface__ view of a device buffer owned by a handle."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i8"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


# ---------------------------------------------------------------------------
def survivor_gather(eng: Engine, d_xs: torch.Tensor, d_ys: torch.Tensor, offset: int,
                    cfg: PipelineConfig, comm: TorchComm):
    """K1/K2 per shard, every survivor (x, y, global index) to rank 0, which runs
    the rest with round 1 disabled (it already ran)."""
    stream = _bind_stream([eng], d_xs.device)  # the handle's work and the torch ops in one order
    stream.wait_stream(torch.cuda.current_stream(d_xs.device))
    with torch.cuda.stream(stream):
        res = _survivor_gather(eng, d_xs, d_ys, offset, cfg, comm)
    torch.cuda.current_stream(d_xs.device).wait_stream(stream)
    return res


def _survivor_gather(eng: Engine, d_xs: torch.Tensor, d_ys: torch.Tensor, offset: int,
                     cfg: PipelineConfig, comm: TorchComm):
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


def sample_sort_sharded(engines: list[Engine], shards, offsets: list[int], n_global: int,
                        cfg: PipelineConfig, comm: Comm):
    """The exact fallback as a distributed sample sort ("a
    distributed sample sort when the survivor set is large", e.g. points on a
    circle, where the sparse path declines). Every rank keeps its round-1
    survivors (global quad), keys them exactly (gscan_shard_keys: atan2 from
    the global anchor) and routes them by key range to the rank that sorts
    that range (splitters from a key sample; equal keys stay on one rank, so
    ties and duplicates are resolved where they meet). Each rank sorts and
    deduplicates its range with the bucket sort (gscan_stage_sorted over the
    received points plus the anchor, in global-index order: index ties break
    as on one device). The sorted runs, concatenated in rank order, are the
    reference's annotated buffer; rank 0 runs split_regions, round 2 and
    Graham on it (gscan_hull_sorted). Returns (indices, stats) on rank 0,
    (None, None) elsewhere."""
    dev = shards[0][0].device
    stream = _bind_stream(engines, dev)  # the handles' work and the torch ops in one order
    stream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(stream):
        res = _sample_sort(engines, shards, offsets, n_global, cfg, comm, dev)
    torch.cuda.current_stream(dev).wait_stream(stream)
    return res


def _sample_sort(engines, shards, offsets, n_global, cfg, comm, dev):
    R = comm.world
    me = comm.ranks
    # global extremes (the reference's tie rules)
    recs = []
    for eng, (dx, dy), off in zip(engines, shards, offsets):
        ex = N.gscan_extremes()
        _ck(eng, eng._lib.gscan_shard_extremes(eng.handle, C.c_void_p(dx.data_ptr()),
                                               C.c_void_p(dy.data_ptr()), dx.numel(), C.byref(ex)),
            "shard_extremes")
        recs.append([off + ex.idx[k] for k in range(5)] + [_i64(v) for v in ex.x]
                    + [_i64(v) for v in ex.y])
    allr = comm.allgather_i64(recs)
    g = _combine(np.stack([np.array([[float(r[k]) for k in range(5)],
                                     [_f64(r[5 + k]) for k in range(5)],
                                     [_f64(r[10 + k]) for k in range(5)]]) for r in allr]))
    gex = N.gscan_extremes()
    for k in range(5):
        gex.idx[k] = int(g[0, k])
        gex.x[k] = g[1, k]
        gex.y[k] = g[2, k]
    a_x, a_y, a_i = float(g[1, 4]), float(g[2, 4]), int(g[0, 4])
    # round-1 survivors and their exact keys; a key sample for the splitters
    S = 1024
    kept, n1s, samples = [], [], []
    for eng, (dx, dy), off in zip(engines, shards, offsets):
        n = int(dx.numel())
        surv = torch.empty(max(n, 1), dtype=_U32, device=dev)
        n1 = C.c_uint64()
        _ck(eng, eng._lib.gscan_shard_round1(eng.handle, C.c_void_p(dx.data_ptr()),
                                             C.c_void_p(dy.data_ptr()), n, C.byref(gex),
                                             C.c_void_p(surv.data_ptr()), C.byref(n1)), "shard_round1")
        m = int(n1.value)
        n1s.append(m)
        keys = torch.empty(max(m, 1), dtype=torch.int64, device=dev)
        _ck(eng, eng._lib.gscan_shard_keys(eng.handle, C.c_void_p(dx.data_ptr()),
                                           C.c_void_p(dy.data_ptr()), C.c_void_p(surv.data_ptr()), m,
                                           C.byref(gex), C.c_void_p(keys.data_ptr())), "shard_keys")
        loc = surv[:m].to(torch.int64) & 0xFFFFFFFF
        keys = keys[:m]
        keep = keys != -1  # points equal to the anchor: annotate drops them
        loc, keys = loc[keep], keys[keep]
        kept.append((dx[loc], dy[loc], loc + off, keys))
        pick = torch.linspace(0, max(keys.numel() - 1, 0), S, device=dev).long() if keys.numel() \
            else torch.zeros(0, dtype=torch.int64, device=dev)
        row = keys[pick].tolist() if keys.numel() else []
        samples.append(row + [np.iinfo(np.int64).max] * (S - len(row)))
    allS = comm.allgather_i64(samples).ravel()
    allS = np.sort(allS[allS != np.iinfo(np.int64).max])
    if allS.size == 0:
        split = torch.zeros(0, dtype=torch.int64, device=dev)
    else:
        split = torch.as_tensor(allS[[(k * allS.size) // R for k in range(1, R)]], device=dev)
    # route the survivors by key range (counts first: the receivers' sizes)
    sends, cnts = [], []
    for (x, y, gi, keys) in kept:
        dest = torch.searchsorted(split, keys, right=True)
        order = torch.argsort(dest, stable=True)
        sends.append((x[order], y[order], gi[order]))
        cnts.append(torch.bincount(dest, minlength=R).tolist())
    cm = comm.allgather_i64(cnts)  # (R senders, R receivers)
    send_sz = [cnts[k] for k in range(len(kept))]
    recv_sz = [cm[:, r].tolist() for r in me]
    rx = comm.all_to_all_flat([sd[0] for sd in sends], send_sz, recv_sz)
    ry = comm.all_to_all_flat([sd[1] for sd in sends], send_sz, recv_sz)
    rg = comm.all_to_all_flat([sd[2] for sd in sends], send_sz, recv_sz)
    # each rank: its key range sorted and deduplicated, in global-index order
    runs = []
    for eng, x, y, gi in zip(engines, rx, ry, rg):
        X = torch.cat([torch.tensor([a_x], dtype=torch.float64, device=dev), x])
        Y = torch.cat([torch.tensor([a_y], dtype=torch.float64, device=dev), y])
        G = torch.cat([torch.tensor([a_i], dtype=torch.int64, device=dev), gi])
        o = torch.argsort(G)
        X, Y, G = X[o].contiguous(), Y[o].contiguous(), G[o]
        m = int(X.numel())
        out = torch.empty(m, dtype=_U32, device=dev)
        ln = C.c_uint64()
        _ck(eng, eng._lib.gscan_stage_sorted(eng.handle, C.c_void_p(X.data_ptr()),
                                             C.c_void_p(Y.data_ptr()), m, C.c_void_p(out.data_ptr()),
                                             C.byref(ln)), "stage_sorted")
        pos = out[1: int(ln.value)].to(torch.int64) & 0xFFFFFFFF  # 0: the anchor
        runs.append((X[pos], Y[pos], G[pos]))
    sizes = comm.allgather_i64([[int(r[0].numel()), n1] for r, n1 in zip(runs, n1s)])
    rsz = sizes[:, 0].tolist()
    n1_total = int(sizes[:, 1].sum())
    parts = [comm.gather_root([r[j] for r in runs], sizes=rsz) for j in range(3)]
    if parts[0] is None:
        return None, None
    eng0 = engines[me.index(0)]
    BX = torch.cat([torch.tensor([a_x], dtype=torch.float64, device=dev)] + parts[0]).contiguous()
    BY = torch.cat([torch.tensor([a_y], dtype=torch.float64, device=dev)] + parts[1]).contiguous()
    BG = torch.cat([torch.tensor([a_i], dtype=torch.int64, device=dev)] + parts[2])
    M = int(BX.numel())
    out = torch.empty(M, dtype=_U32, device=dev)
    hn, n2 = C.c_uint64(), C.c_uint64()
    ccfg = cfg._c()
    _ck(eng0, eng0._lib.gscan_hull_sorted(eng0.handle, C.c_void_p(BX.data_ptr()),
                                          C.c_void_p(BY.data_ptr()), M, C.byref(ccfg),
                                          C.c_void_p(out.data_ptr()), M, C.byref(hn), C.byref(n2)),
        "hull_sorted")
    k = int(hn.value)
    hv = BG[out[:k].to(torch.int64) & 0xFFFFFFFF].cpu().numpy().astype(np.uint64)
    return hv, StageStats(n_input=n_global, n_after_round1=n1_total,
                          n_after_round2=int(n2.value), hull_size=k)


def simulate_sample_sort(engines: list[Engine], xs: torch.Tensor, ys: torch.Tensor,
                         cfg: PipelineConfig | None = None, bounds: list[int] | None = None):
    """The distributed sample sort with all R ranks in this process (LocalComm)."""
    cfg = cfg or PipelineConfig()
    R = len(engines)
    n = int(xs.numel())
    offs = list(bounds) if bounds is not None else [n * r // R for r in range(R + 1)]
    shards = [(xs[offs[r]:offs[r + 1]].contiguous(), ys[offs[r]:offs[r + 1]].contiguous())
              for r in range(R)]
    return sample_sort_sharded(engines, shards, offs[:R], n, cfg, LocalComm(R))


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
    if cfg.enable_round1 and n_global < 0xFFFFFFFF and d_xs.is_cuda and min(sizes) > 0:
        return sample_sort_sharded([eng], [(d_xs, d_ys)], [offset], n_global, cfg, comm)
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
