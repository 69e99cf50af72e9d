// gScan hull kernels for sm_100a. Each kernel cites the reference stage it
// replaces (/root/reference/proj/include/hull2d/...). Data layout in HBM is
// SoA float64 (xs, ys) in, uint32 input indices through the pipeline.
#pragma once
#include <cuda_runtime.h>
#include <float.h>
#include <stdint.h>

#include "device_common.cuh"

namespace gscan {

// Result of K1 (extremes + anchor), device resident.
struct ExtResult {
  uint32_t idx[5];  // i_minx, i_miny, i_maxx, i_maxy, anchor
  uint32_t pad;
  double qx[4], qy[4];
  double ax, ay;
};

// Per-call device counters (one cache line each would be overkill; these
// are touched by a handful of threads).
struct Counters {
  uint32_t n1;          // round-1 survivors
  uint32_t tile_ticket; // dynamic tile ids for look-back kernels
  uint32_t ext_ticket;  // last-block detection for K1
  uint32_t dead;        // duplicates removed during the bucket sort
  uint32_t n_oversize;  // buckets too large for the shared-memory sort
  uint32_t n2;          // round-2 survivors
  uint32_t hull;        // hull size
  uint32_t longest;     // split_regions().longest (buffer position)
  uint32_t m_total;     // annotated buffer size M (anchor included)
  uint32_t graham_fail; // certificate failures (diagnostics)
  uint32_t anchor_dups; // survivors coinciding with the anchor
  uint32_t pad[5];
  uint64_t tstamp[6];   // stage boundaries (%globaltimer ns) of a graph-replayed call
};

// ===========================================================================
// K1: find_extremes (prefilter.hpp:28-39) + select_anchor (angular.hpp:40-49)
// in one pass. Strict compares with lowest-index ties. The global lowest
// point is select_anchor(round-1 survivors) as well: it can never be strictly
// inside the quadrilateral, and compaction keeps order.
struct ExtAcc {
  double minx, miny, maxx, maxy, ly, lx;
  uint32_t iminx, iminy, imaxx, imaxy, il;
};

// +/-inf start values: every finite point beats them (non-finite input is a
// precondition of the reference, SPEC.md), so a push is compare + select.
__device__ __forceinline__ void ext_init(ExtAcc& a) {
  a.minx = a.miny = a.ly = a.lx = __longlong_as_double(0x7ff0000000000000ll);
  a.maxx = a.maxy = __longlong_as_double((long long)0xfff0000000000000ull);
  a.iminx = a.iminy = a.imaxx = a.imaxy = a.il = 0xffffffffu;
}

// Within one thread indices only grow, so strict compares keep the first.
__device__ __forceinline__ void ext_push(ExtAcc& a, double x, double y, uint32_t i) {
  const bool b0 = x < a.minx, b1 = y < a.miny, b2 = x > a.maxx, b3 = y > a.maxy;
  const bool b4 = y < a.ly || (y == a.ly && x < a.lx);
  a.minx = b0 ? x : a.minx; a.iminx = b0 ? i : a.iminx;
  a.miny = b1 ? y : a.miny; a.iminy = b1 ? i : a.iminy;
  a.maxx = b2 ? x : a.maxx; a.imaxx = b2 ? i : a.imaxx;
  a.maxy = b3 ? y : a.maxy; a.imaxy = b3 ? i : a.imaxy;
  a.ly = b4 ? y : a.ly; a.lx = b4 ? x : a.lx; a.il = b4 ? i : a.il;
}

__device__ __forceinline__ bool arg_better_min(double v, uint32_t i, double bv, uint32_t bi) {
  if (i == 0xffffffffu) return false;
  if (bi == 0xffffffffu) return true;
  return v < bv || (v == bv && i < bi);
}
__device__ __forceinline__ bool arg_better_max(double v, uint32_t i, double bv, uint32_t bi) {
  if (i == 0xffffffffu) return false;
  if (bi == 0xffffffffu) return true;
  return v > bv || (v == bv && i < bi);
}

__device__ __forceinline__ void ext_merge(ExtAcc& a, const ExtAcc& b) {
  if (arg_better_min(b.minx, b.iminx, a.minx, a.iminx)) { a.minx = b.minx; a.iminx = b.iminx; }
  if (arg_better_min(b.miny, b.iminy, a.miny, a.iminy)) { a.miny = b.miny; a.iminy = b.iminy; }
  if (arg_better_max(b.maxx, b.imaxx, a.maxx, a.imaxx)) { a.maxx = b.maxx; a.imaxx = b.imaxx; }
  if (arg_better_max(b.maxy, b.imaxy, a.maxy, a.imaxy)) { a.maxy = b.maxy; a.imaxy = b.imaxy; }
  bool take = false;
  if (b.il != 0xffffffffu) {
    if (a.il == 0xffffffffu) take = true;
    else if (b.ly < a.ly) take = true;
    else if (b.ly == a.ly && (b.lx < a.lx || (b.lx == a.lx && b.il < a.il))) take = true;
  }
  if (take) { a.ly = b.ly; a.lx = b.lx; a.il = b.il; }
}

__device__ __forceinline__ ExtAcc ext_shfl(const ExtAcc& a, int o) {
  ExtAcc b;
  b.minx = __shfl_xor_sync(0xffffffffu, a.minx, o);
  b.miny = __shfl_xor_sync(0xffffffffu, a.miny, o);
  b.maxx = __shfl_xor_sync(0xffffffffu, a.maxx, o);
  b.maxy = __shfl_xor_sync(0xffffffffu, a.maxy, o);
  b.ly = __shfl_xor_sync(0xffffffffu, a.ly, o);
  b.lx = __shfl_xor_sync(0xffffffffu, a.lx, o);
  b.iminx = __shfl_xor_sync(0xffffffffu, a.iminx, o);
  b.iminy = __shfl_xor_sync(0xffffffffu, a.iminy, o);
  b.imaxx = __shfl_xor_sync(0xffffffffu, a.imaxx, o);
  b.imaxy = __shfl_xor_sync(0xffffffffu, a.imaxy, o);
  b.il = __shfl_xor_sync(0xffffffffu, a.il, o);
  return b;
}

__device__ __forceinline__ void ext_finish(ExtAcc acc, const double* __restrict__ xs,
                                           const double* __restrict__ ys,
                                           ExtAcc* __restrict__ partials,
                                           ExtResult* __restrict__ out, Counters* __restrict__ ctr);

// Grid-stride over 128-bit pairs of (xs, ys) with 4 pairs in flight per
// thread; block partials are reduced by the last CTA to finish.
template <bool kVec>
__global__ void __launch_bounds__(kBlock) k_extremes(const double* __restrict__ xs,
                                                     const double* __restrict__ ys, uint32_t n,
                                                     ExtAcc* __restrict__ partials,
                                                     ExtResult* __restrict__ out,
                                                     Counters* __restrict__ ctr) {
  pdl_wait();
  ExtAcc acc;
  ext_init(acc);
  const uint32_t tid = blockIdx.x * kBlock + threadIdx.x;
  const uint32_t nthreads = gridDim.x * kBlock;
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    const uint32_t npairs = n / 2;
    uint32_t p = tid;
    for (; p + 3 * nthreads < npairs; p += 4 * nthreads) {
      double2 vx[4], vy[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        vx[u] = __ldcs(&x2[p + u * nthreads]);
        vy[u] = __ldcs(&y2[p + u * nthreads]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = 2 * (p + u * nthreads);
        ext_push(acc, vx[u].x, vy[u].x, i);
        ext_push(acc, vx[u].y, vy[u].y, i + 1);
      }
    }
    for (; p < npairs; p += nthreads) {
      const double2 vx = __ldcs(&x2[p]), vy = __ldcs(&y2[p]);
      ext_push(acc, vx.x, vy.x, 2 * p);
      ext_push(acc, vx.y, vy.y, 2 * p + 1);
    }
    if ((n & 1) && tid == 0) ext_push(acc, xs[n - 1], ys[n - 1], n - 1);
  } else {
    for (uint32_t i = tid; i < n; i += nthreads) ext_push(acc, xs[i], ys[i], i);
  }
  ext_finish(acc, xs, ys, partials, out, ctr);
}

// Block reduction of the per-thread accumulators, then the last CTA to finish
// reduces the block partials and writes the result (any block size <= 1024).
__device__ __forceinline__ void ext_finish(ExtAcc acc, const double* __restrict__ xs,
                                           const double* __restrict__ ys,
                                           ExtAcc* __restrict__ partials,
                                           ExtResult* __restrict__ out, Counters* __restrict__ ctr) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ext_merge(acc, ext_shfl(acc, o));
  __shared__ ExtAcc s_w[32];
  const int nwarps = (int)(blockDim.x >> 5);
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_w[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nwarps; ++w) ext_merge(acc, s_w[w]);
    partials[blockIdx.x] = acc;
    __threadfence();
    const uint32_t t = atomicAdd(&ctr->ext_ticket, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  // last CTA: reduce all partials
  __threadfence();
  ExtAcc a;
  ext_init(a);
  for (uint32_t b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    ExtAcc pb;
    const volatile ExtAcc* vp = &partials[b];
    pb.minx = vp->minx; pb.miny = vp->miny; pb.maxx = vp->maxx; pb.maxy = vp->maxy;
    pb.ly = vp->ly; pb.lx = vp->lx;
    pb.iminx = vp->iminx; pb.iminy = vp->iminy; pb.imaxx = vp->imaxx; pb.imaxy = vp->imaxy;
    pb.il = vp->il;
    ext_merge(a, pb);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ext_merge(a, ext_shfl(a, o));
  __syncthreads();
  if (lane == 0) s_w[warp] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nwarps; ++w) ext_merge(a, s_w[w]);
    out->idx[0] = a.iminx; out->idx[1] = a.iminy; out->idx[2] = a.imaxx; out->idx[3] = a.imaxy;
    out->idx[4] = a.il;
    for (int k = 0; k < 4; ++k) { out->qx[k] = xs[out->idx[k]]; out->qy[k] = ys[out->idx[k]]; }
    out->ax = a.lx;
    out->ay = a.ly;
    ctr->ext_ticket = 0;  // ready for the next launch
  }
}

// K1 as a bulk-copy pipeline (XYRing, device_common.cuh): one CTA per SM
// streams tiles of kExtTile points of xs and ys through a kExtStages-deep
// shared-memory ring; every warp is a consumer and the last warp to finish
// reading a stage refills it, so no CTA-wide barrier sits on the per-tile path
// and kExtStages x 32 KB are in flight per SM regardless of occupancy. Each
// warp releases its stage as soon as the values are in registers. Tiles go to
// CTAs round-robin; the remainder (< one tile) is read directly by the last
// CTA. Within a thread indices only grow (tile order, then pair order), as
// ext_push requires. Needs 16-byte aligned xs, ys.
#ifndef GSCAN_EXT_TILE
#define GSCAN_EXT_TILE 2048
#endif
constexpr int kExtTile = GSCAN_EXT_TILE;  // points per tile (2048: 16 KB of x + 16 KB of y)
#ifndef GSCAN_EXT_STAGES
#define GSCAN_EXT_STAGES 4
#endif
constexpr int kExtStages = GSCAN_EXT_STAGES;
#ifndef GSCAN_EXT_THREADS
#define GSCAN_EXT_THREADS 512
#endif
#ifndef GSCAN_EXT_ACC
#define GSCAN_EXT_ACC 4
#endif
constexpr int kExtThreads = GSCAN_EXT_THREADS;  // 512: 2 pairs (4 points) per thread per tile
constexpr int kExtAcc = GSCAN_EXT_ACC;          // independent accumulators per thread
using ExtRing = XYRing<kExtTile, kExtStages>;
constexpr size_t kExtSmem = ExtRing::kSmem + 64;

__global__ void __launch_bounds__(kExtThreads, 1) k_extremes_tma(const double* __restrict__ xs,
                                                           const double* __restrict__ ys, uint32_t n,
                                                           ExtAcc* __restrict__ partials,
                                                           ExtResult* __restrict__ out,
                                                           Counters* __restrict__ ctr) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char ext_smem[];
  ExtRing ring;
  ring.setup(ext_smem, xs, ys, n);
  ring.start();
  __syncthreads();
  // four independent accumulators (one per point of a thread's tile share):
  // shorter dependency chains; each still sees increasing indices
  ExtAcc acc[kExtAcc];
#pragma unroll
  for (int a = 0; a < kExtAcc; ++a) ext_init(acc[a]);
  for (uint32_t k = 0; k < ring.mine; ++k) {
    ring.wait(k);
    const double2* x2 = reinterpret_cast<const double2*>(ring.tx(k));
    const double2* y2 = reinterpret_cast<const double2*>(ring.ty(k));
    constexpr int kPairs = kExtTile / 2 / kExtThreads;
    double2 vx[kPairs], vy[kPairs];
#pragma unroll
    for (int u = 0; u < kPairs; ++u) {
      vx[u] = x2[threadIdx.x + u * kExtThreads];
      vy[u] = y2[threadIdx.x + u * kExtThreads];
    }
    ring.release(k);
    const uint32_t i0 = ring.tile_start(k) + 2 * threadIdx.x;
#pragma unroll
    for (int u = 0; u < kPairs; ++u) {
      const uint32_t i = i0 + 2 * u * kExtThreads;
      ext_push(acc[(2 * u) % kExtAcc], vx[u].x, vy[u].x, i);
      ext_push(acc[(2 * u + 1) % kExtAcc], vx[u].y, vy[u].y, i + 1);
    }
  }
  if (blockIdx.x == gridDim.x - 1)
    for (uint32_t i = (n / kExtTile) * kExtTile + threadIdx.x; i < n; i += kExtThreads)
      ext_push(acc[0], xs[i], ys[i], i);
#pragma unroll
  for (int a = 1; a < kExtAcc; ++a) ext_merge(acc[0], acc[a]);
  ext_finish(acc[0], xs, ys, partials, out, ctr);
}

// Overlapped ingest (gscan_hull_f64): K1 ran per H2D chunk (chunk c's points
// are global indices off[c] ..); merge the chunk results in index order with
// find_extremes' / select_anchor's rules (strict compares: on equal values
// the earlier chunk, i.e. the lower index, keeps it).
__global__ void k_ext_merge(const ExtResult* __restrict__ parts, const uint32_t* __restrict__ off,
                            uint32_t nparts, ExtResult* __restrict__ out) {
  if (threadIdx.x != 0) return;
  ExtResult r = parts[0];
  for (int k = 0; k < 5; ++k) r.idx[k] += off[0];
  for (uint32_t c = 1; c < nparts; ++c) {
    const ExtResult& p = parts[c];
    if (p.qx[0] < r.qx[0]) { r.qx[0] = p.qx[0]; r.qy[0] = p.qy[0]; r.idx[0] = off[c] + p.idx[0]; }
    if (p.qy[1] < r.qy[1]) { r.qx[1] = p.qx[1]; r.qy[1] = p.qy[1]; r.idx[1] = off[c] + p.idx[1]; }
    if (p.qx[2] > r.qx[2]) { r.qx[2] = p.qx[2]; r.qy[2] = p.qy[2]; r.idx[2] = off[c] + p.idx[2]; }
    if (p.qy[3] > r.qy[3]) { r.qx[3] = p.qx[3]; r.qy[3] = p.qy[3]; r.idx[3] = off[c] + p.idx[3]; }
    if (p.ay < r.ay || (p.ay == r.ay && p.ax < r.ax)) {
      r.ax = p.ax; r.ay = p.ay; r.idx[4] = off[c] + p.idx[4];
    }
  }
  *out = r;
}

// ===========================================================================
// K2: classify_quad (prefilter.hpp:47-63) fused with the stable compaction
// `compact` (prefilter.hpp:65-76). Each tile of 4096 points is read exactly
// once (128-bit loads), ranked with warp ballots, and its survivors' input
// indices are placed with a decoupled look-back; no flag array exists.
constexpr int kFilterPairs = 8;  // double2 per thread -> 16 points per thread
constexpr int kFilterTile = kBlock * kFilterPairs * 2;

__device__ __forceinline__ bool quad_keep(const double* qx, const double* qy, const double* ex,
                                          const double* ey, double x, double y) {
  // flag 0 iff strictly Left of all four directed edges (short-circuit as in
  // the reference; the result is the same either way)
  if (!(cross_edge(qx[0], qy[0], ex[0], ey[0], x, y) > 0.0)) return true;
  if (!(cross_edge(qx[1], qy[1], ex[1], ey[1], x, y) > 0.0)) return true;
  if (!(cross_edge(qx[2], qy[2], ex[2], ey[2], x, y) > 0.0)) return true;
  if (!(cross_edge(qx[3], qy[3], ex[3], ey[3], x, y) > 0.0)) return true;
  return false;
}

// kOrdered = true: decoupled look-back, survivors in input order (stage API,
// prefilter.hpp:65-76 compact). kOrdered = false: each CTA reserves its output
// range with one atomic -- the pipeline's choice, because every later stage
// orders points by (angle, dist2, input index) and never by survivor slot.
template <bool kVec, bool kOrdered>
__global__ void __launch_bounds__(kBlock, 3) k_filter_compact(
    const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n,
    const ExtResult* __restrict__ ext, int enable_round1, uint64_t* __restrict__ status,
    uint32_t* __restrict__ out_idx, Counters* __restrict__ ctr) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_cnt[kFilterPairs][kWarps];
  __shared__ uint32_t s_excl, s_total;
  __shared__ uint32_t s_out[kFilterTile];
  if (threadIdx.x == 0) s_tile = kOrdered ? atomicAdd(&ctr->tile_ticket, 1u) : blockIdx.x;
  double qx[4], qy[4], ex[4], ey[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { qx[k] = ext->qx[k]; qy[k] = ext->qy[k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) {  // edge q_k -> q_{k+1}, same subtraction as cross()
    ex[k] = __dsub_rn(qx[(k + 1) & 3], qx[k]);
    ey[k] = __dsub_rn(qy[(k + 1) & 3], qy[k]);
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * (uint32_t)kFilterTile;  // first point of the tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();

  uint32_t b0[kFilterPairs], b1[kFilterPairs];
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    double2 vx[kFilterPairs], vy[kFilterPairs];
#pragma unroll
    for (int k = 0; k < kFilterPairs; ++k) {
      const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
      if (i0 + 1 < n) {
        vx[k] = __ldcs(&x2[i0 >> 1]);
        vy[k] = __ldcs(&y2[i0 >> 1]);
      } else if (i0 < n) {
        vx[k].x = xs[i0]; vy[k].x = ys[i0]; vx[k].y = 0.0; vy[k].y = 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < kFilterPairs; ++k) {
      const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
      const bool k0 = i0 < n && (!enable_round1 || quad_keep(qx, qy, ex, ey, vx[k].x, vy[k].x));
      const bool k1 =
          i0 + 1 < n && (!enable_round1 || quad_keep(qx, qy, ex, ey, vx[k].y, vy[k].y));
      b0[k] = __ballot_sync(0xffffffffu, k0);
      b1[k] = __ballot_sync(0xffffffffu, k1);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kFilterPairs; ++k) {
      const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
      bool k0 = false, k1 = false;
      if (i0 < n) k0 = !enable_round1 || quad_keep(qx, qy, ex, ey, xs[i0], ys[i0]);
      if (i0 + 1 < n) k1 = !enable_round1 || quad_keep(qx, qy, ex, ey, xs[i0 + 1], ys[i0 + 1]);
      b0[k] = __ballot_sync(0xffffffffu, k0);
      b1[k] = __ballot_sync(0xffffffffu, k1);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kFilterPairs; ++k) s_cnt[k][warp] = __popc(b0[k]) + __popc(b1[k]);
  }
  __syncthreads();
  // exclusive scan of the 64 (stripe, warp) counts in point order, by warp 0
  if (warp == 0) {
    uint32_t v0 = s_cnt[lane >> 3][lane & 7];
    uint32_t v1 = s_cnt[4 + (lane >> 3)][lane & 7];
    uint32_t x0 = v0, x1 = v1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xffffffffu, x0, o);
      const uint32_t y1 = __shfl_up_sync(0xffffffffu, x1, o);
      if (lane >= o) { x0 += y0; x1 += y1; }
    }
    const uint32_t tot0 = __shfl_sync(0xffffffffu, x0, 31);
    const uint32_t tot1 = __shfl_sync(0xffffffffu, x1, 31);
    s_cnt[lane >> 3][lane & 7] = x0 - v0;
    s_cnt[4 + (lane >> 3)][lane & 7] = tot0 + x1 - v1;
    const uint32_t agg = tot0 + tot1;
    if (kOrdered) {
      const uint64_t excl = lookback_exclusive(status, tile, agg);
      if (lane == 0) {
        s_excl = (uint32_t)excl;
        s_total = agg;
        if (base + kFilterTile >= n) ctr->n1 = (uint32_t)(excl + agg);  // last tile
      }
    } else if (lane == 0) {
      s_excl = agg ? atomicAdd(&ctr->n1, agg) : 0u;
      s_total = agg;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kFilterPairs; ++k) {
    const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
    uint32_t r = s_cnt[k][warp] + __popc(b0[k] & lt) + __popc(b1[k] & lt);
    if (b0[k] & (1u << lane)) s_out[r++] = i0;
    if (b1[k] & (1u << lane)) s_out[r] = i0 + 1;
  }
  __syncthreads();
  const uint32_t total = s_total, off = s_excl;
  for (uint32_t r = threadIdx.x; r < total; r += kBlock) out_idx[off + r] = s_out[r];
}

// ===========================================================================
// K3: polar keys (annotate's key map, angular.hpp:135-146 / polar_key,
// geom.hpp:38-43) for every round-1 survivor, with the anchor coincidence
// test (geom.hpp:39) and a bucket histogram for the angle sort. The key is
// the bit pattern of glibc's atan2 result (angles lie in [0, pi] because the
// anchor is the lowest point; -0.0 is folded onto +0.0 so it ties with 0.0 as
// in the reference's double compare). Monotone bucket map: floor(angle*B/pi).
__device__ __forceinline__ uint32_t bucket_of(uint64_t key, double scale, uint32_t nb) {
  const double b = __dmul_rn(bitsd(key), scale);
  const uint32_t bi = (uint32_t)b;
  return bi < nb ? bi : nb - 1;
}

__global__ void __launch_bounds__(kBlock) k_keys(const double* __restrict__ xs,
                                                 const double* __restrict__ ys,
                                                 const uint32_t* __restrict__ surv,
                                                 const ExtResult* __restrict__ ext,
                                                 const Counters* __restrict__ ctr_in,
                                                 uint64_t* __restrict__ keys,
                                                 uint32_t* __restrict__ rank,
                                                 uint32_t* __restrict__ hist, double scale,
                                                 uint32_t nb, Counters* __restrict__ ctr) {
  const uint32_t n1 = ctr_in->n1;
  const double ax = ext->ax, ay = ext->ay;
  const int lane = threadIdx.x & 31;
  uint32_t drops = 0;
  for (uint32_t j = blockIdx.x * kBlock + threadIdx.x; j < n1; j += gridDim.x * kBlock) {
    const uint32_t i = surv[j];
    const double x = xs[i], y = ys[i];
    uint64_t key;
    uint32_t b;
    if (x == ax && y == ay) {
      key = kKeyDrop;
      b = nb;
      ++drops;
    } else {
      const double dx = __dsub_rn(x, ax), dy = __dsub_rn(y, ay);
      const double ang = glibc_atan2(dy, dx);
      key = (ang == 0.0) ? 0ull : dbits(ang);
      b = bucket_of(key, scale, nb);
    }
    keys[j] = key;
    // warp-aggregated claim of a slot inside the bucket: rank = arrival order
    const uint32_t active = __activemask();
    const uint32_t peers = __match_any_sync(active, b);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(&hist[b], (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, leader);
    rank[j] = base + __popc(peers & lanemask_lt());
  }
  if (drops) atomicAdd(&ctr->anchor_dups, drops);
}

// ===========================================================================
// K2+K3 fused (the pipeline's round-1 kernel): classify_quad + compact
// (prefilter.hpp:47-76) AND, for each survivor, its polar key (geom.hpp:38-43
// via the glibc-identical atan2), its angle bucket and its arrival rank in the
// bucket. The FP64 key work hides under the tile's HBM stream. Each CTA
// reserves its output range with one atomic (survivor order is irrelevant:
// the sort orders by (angle, dist2, input index)).
constexpr int kFusedPairs = 4;                       // 8 points per thread
constexpr int kFusedTile = kBlock * kFusedPairs * 2; // 2048 points per CTA

template <bool kVec>
__global__ void __launch_bounds__(kBlock, 3) k_filter_keys(
    const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n,
    const ExtResult* __restrict__ ext, int enable_round1, double scale, uint32_t nb,
    uint32_t* __restrict__ hist, uint32_t* __restrict__ out_idx, uint64_t* __restrict__ keys,
    uint32_t* __restrict__ rank, Counters* __restrict__ ctr) {
  __shared__ uint32_t s_cnt[kFusedPairs][kWarps];
  __shared__ uint32_t s_excl, s_total;
  __shared__ uint32_t s_idx[kFusedTile];
  __shared__ uint32_t s_rank[kFusedTile];
  __shared__ uint64_t s_key[kFusedTile];
  double qx[4], qy[4], ex[4], ey[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { qx[k] = ext->qx[k]; qy[k] = ext->qy[k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    ex[k] = __dsub_rn(qx[(k + 1) & 3], qx[k]);
    ey[k] = __dsub_rn(qy[(k + 1) & 3], qy[k]);
  }
  const double ax = ext->ax, ay = ext->ay;
  const uint32_t base = blockIdx.x * (uint32_t)kFusedTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  double vx[kFusedPairs][2], vy[kFusedPairs][2];
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
#pragma unroll
    for (int k = 0; k < kFusedPairs; ++k) {
      const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
      if (i0 + 1 < n) {
        const double2 a = __ldcs(&x2[i0 >> 1]), b = __ldcs(&y2[i0 >> 1]);
        vx[k][0] = a.x; vx[k][1] = a.y; vy[k][0] = b.x; vy[k][1] = b.y;
      } else if (i0 < n) {
        vx[k][0] = xs[i0]; vy[k][0] = ys[i0]; vx[k][1] = 0.0; vy[k][1] = 0.0;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < kFusedPairs; ++k) {
      const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        vx[k][h] = (i0 + h < n) ? xs[i0 + h] : 0.0;
        vy[k][h] = (i0 + h < n) ? ys[i0 + h] : 0.0;
      }
    }
  }
  uint32_t b0[kFusedPairs], b1[kFusedPairs];
#pragma unroll
  for (int k = 0; k < kFusedPairs; ++k) {
    const uint32_t i0 = base + 2u * (k * kBlock + threadIdx.x);
    const bool k0 = i0 < n && (!enable_round1 || quad_keep(qx, qy, ex, ey, vx[k][0], vy[k][0]));
    const bool k1 = i0 + 1 < n && (!enable_round1 || quad_keep(qx, qy, ex, ey, vx[k][1], vy[k][1]));
    b0[k] = __ballot_sync(0xffffffffu, k0);
    b1[k] = __ballot_sync(0xffffffffu, k1);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kFusedPairs; ++k) s_cnt[k][warp] = __popc(b0[k]) + __popc(b1[k]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 32 (stripe, warp) counts in point order
    const uint32_t v = s_cnt[lane >> 3][lane & 7];
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
    s_cnt[lane >> 3][lane & 7] = x - v;
    if (lane == 0) {
      s_total = tot;
      s_excl = tot ? atomicAdd(&ctr->n1, tot) : 0u;
    }
  }
  __syncthreads();
  // keys for this thread's survivors; rank = arrival order in the bucket
  uint32_t drops = 0;
#pragma unroll
  for (int k = 0; k < kFusedPairs; ++k) {
    uint32_t r = s_cnt[k][warp] + __popc(b0[k] & lt) + __popc(b1[k] & lt);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t m = h ? b1[k] : b0[k];
      if (m & (1u << lane)) {
        const double x = vx[k][h], y = vy[k][h];
        uint64_t key;
        uint32_t b;
        if (x == ax && y == ay) {
          key = kKeyDrop;
          b = nb;
          ++drops;
        } else {
          const double ang = glibc_atan2(__dsub_rn(y, ay), __dsub_rn(x, ax));
          key = (ang == 0.0) ? 0ull : dbits(ang);
          b = bucket_of(key, scale, nb);
        }
        s_idx[r] = base + 2u * (k * kBlock + threadIdx.x) + h;
        s_key[r] = key;
        s_rank[r] = atomicAdd(&hist[b], 1u);
        ++r;
      }
    }
  }
  if (drops) atomicAdd(&ctr->anchor_dups, drops);
  __syncthreads();
  const uint32_t total = s_total, off = s_excl;
  for (uint32_t r = threadIdx.x; r < total; r += kBlock) {
    out_idx[off + r] = s_idx[r];
    keys[off + r] = s_key[r];
    rank[off + r] = s_rank[r];
  }
}

// ===========================================================================
// Device-wide exclusive scan of uint32 counts (decoupled look-back); used for
// bucket offsets. out[i] = sum(in[0..i)); out[n] = total when n_out > n.
// Tiles are striped (coalesced loads and stores; striped_exclusive).
constexpr int kScanItems = 8;
constexpr int kScanTile = kBlock * kScanItems;

__global__ void __launch_bounds__(kBlock) k_scan_u32(const uint32_t* __restrict__ in, uint32_t n,
                                                     uint32_t* __restrict__ out,
                                                     uint64_t* __restrict__ status,
                                                     Counters* __restrict__ ctr) {
  pdl_wait();
  __shared__ uint32_t s_tile, s_excl, s_rows[kScanItems * kWarps + 1];
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile_ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kScanTile;  // striped: item (k, t) = base + k * kBlock + t
  uint32_t v[kScanItems], ex[kScanItems];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint32_t i = base + k * kBlock + threadIdx.x;
    v[k] = i < n ? in[i] : 0u;
  }
  const uint32_t total = striped_exclusive<kScanItems>(v, ex, s_rows);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, total);
    if (threadIdx.x == 0) s_excl = (uint32_t)e;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const uint32_t i = base + k * kBlock + threadIdx.x;
    if (i <= n) out[i] = s_excl + ex[k];  // out[n] = grand total
  }
}

// Scatter each survivor to its slot (bucket start + arrival rank from K3) as
// ONE 32-byte record {key, x, y, input index} written with a single 256-bit
// store (STG.E.256): a full L2 sector per point, so the random write needs
// no read-for-ownership of a partially written sector; no atomics.
struct __align__(32) PtRec {
  uint64_t key;
  double x, y;
  uint32_t idx;
  uint32_t pad;
};

__device__ __forceinline__ void st_rec256(PtRec* p, uint64_t key, double x, double y, uint32_t idx) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
               "r"((uint32_t)key), "r"((uint32_t)(key >> 32)),
               "r"((uint32_t)dbits(x)), "r"((uint32_t)(dbits(x) >> 32)),
               "r"((uint32_t)dbits(y)), "r"((uint32_t)(dbits(y) >> 32)), "r"(idx), "r"(0u));
}

__device__ __forceinline__ PtRec ld_rec256(const PtRec* p) {
  uint32_t v[8];
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "l"(p));
  PtRec r;
  r.key = (uint64_t)v[0] | ((uint64_t)v[1] << 32);
  r.x = bitsd((uint64_t)v[2] | ((uint64_t)v[3] << 32));
  r.y = bitsd((uint64_t)v[4] | ((uint64_t)v[5] << 32));
  r.idx = v[6];
  r.pad = v[7];
  return r;
}

constexpr int kScatterItems = 4;

__global__ void __launch_bounds__(kBlock) k_scatter(const double* __restrict__ xs,
                                                    const double* __restrict__ ys,
                                                    const uint64_t* __restrict__ keys,
                                                    const uint32_t* __restrict__ rank,
                                                    const uint32_t* __restrict__ surv,
                                                    const Counters* __restrict__ ctr,
                                                    const uint32_t* __restrict__ bstart,
                                                    double scale, uint32_t nb,
                                                    PtRec* __restrict__ rec) {
  const uint32_t n1 = ctr->n1;
  const uint32_t stride = gridDim.x * kBlock * kScatterItems;
  for (uint32_t j0 = blockIdx.x * kBlock * kScatterItems + threadIdx.x; j0 < n1; j0 += stride) {
    // three dependent load levels, issued kScatterItems-wide for MLP
    uint64_t key[kScatterItems];
    uint32_t i[kScatterItems], rk[kScatterItems], pos[kScatterItems];
    double x[kScatterItems], y[kScatterItems];
#pragma unroll
    for (int u = 0; u < kScatterItems; ++u) {
      const uint32_t j = j0 + u * kBlock;
      key[u] = kKeyDrop;
      if (j < n1) { key[u] = keys[j]; i[u] = surv[j]; rk[u] = rank[j]; }
    }
#pragma unroll
    for (int u = 0; u < kScatterItems; ++u) {
      if (key[u] != kKeyDrop) {
        pos[u] = bstart[bucket_of(key[u], scale, nb)] + rk[u];
        x[u] = xs[i[u]];
        y[u] = ys[i[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < kScatterItems; ++u)
      if (key[u] != kKeyDrop) st_rec256(&rec[pos[u]], key[u], x[u], y[u], i[u]);
  }
}

// ===========================================================================
// K4: per-bucket total-order sort = sort_by_angle's stable (angle, dist2)
// order (angular.hpp:154-194) with the input index as the final tie-break
// (equivalent to stability over the index-ordered survivors), plus annotate's
// dedup (angular.hpp:118-133): exact duplicates share (angle, dist2), so the
// later occurrences inside an equal-key run are dropped.
// Writes the annotated buffer (positions 1.. ; 0 is the anchor).
constexpr int kSortBlock = 128;
constexpr int kSortCap = 2048;   // CTA path capacity (shared memory)

struct BucketBest {  // farthest point candidate for split_regions
  uint64_t d2bits;
  uint32_t pos;
  uint32_t pad;
};

__device__ __forceinline__ bool key_less(uint64_t ka, double da, uint32_t ia, uint64_t kb,
                                         double db, uint32_t ib) {
  if (ka != kb) return ka < kb;
  if (da != db) return da < db;
  return ia < ib;
}

__device__ __forceinline__ void best_merge(uint64_t& bb, uint32_t& bp, uint64_t ob, uint32_t op) {
  if (op == 0xffffffffu) return;
  if (bp == 0xffffffffu || ob > bb || (ob == bb && op < bp)) { bb = ob; bp = op; }
}

// Block-wide (max dist2, first position) -> partial[slot].
template <int kThreads>
__device__ __forceinline__ void block_best(uint64_t bb, uint32_t bp, BucketBest* partial) {
  __shared__ uint64_t s_b[kThreads / 32];
  __shared__ uint32_t s_p[kThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ob = __shfl_xor_sync(0xffffffffu, bb, o);
    const uint32_t op = __shfl_xor_sync(0xffffffffu, bp, o);
    best_merge(bb, bp, ob, op);
  }
  if ((threadIdx.x & 31) == 0) { s_b[threadIdx.x >> 5] = bb; s_p[threadIdx.x >> 5] = bp; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kThreads / 32; ++w) best_merge(bb, bp, s_b[w], s_p[w]);
    partial->d2bits = bb;
    partial->pos = bp;
  }
}

// K4a: block-cooperative sort of 256 consecutive buckets (~2-5 keys each):
// the block loads its buckets' records contiguously into shared memory; each
// key's rank inside its bucket is counted against its bucket peers by the
// total order (angle bits, dist2, input index), and a key is a duplicate iff
// an equal point with a lower index shares its bucket (equal points always
// share angle and dist2). Blocks whose buckets hold more than kBlockCap keys
// defer those buckets to K4b.
constexpr int kBucketsPerBlock = 128;
constexpr int kBlockCap = 1024;

__global__ void __launch_bounds__(kBlock) k_bucket_sort_block(
    const uint32_t* __restrict__ bstart, const PtRec* __restrict__ rec,
    const ExtResult* __restrict__ ext, double scale,
    uint32_t nb, double* __restrict__ A_x, double* __restrict__ A_y,
    uint32_t* __restrict__ A_idx, BucketBest* __restrict__ partials,
    uint32_t* __restrict__ oversize, Counters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
  double* s_d2 = reinterpret_cast<double*>(s_key + kBlockCap);
  double* s_x = s_d2 + kBlockCap;
  double* s_y = s_x + kBlockCap;
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_y + kBlockCap);
  uint16_t* s_lb = reinterpret_cast<uint16_t*>(s_idx + kBlockCap);
  __shared__ uint32_t s_bs[kBucketsPerBlock + 1];
  const uint32_t b0 = blockIdx.x * kBucketsPerBlock;
  const uint32_t nbk = min((uint32_t)kBucketsPerBlock, nb - b0);
  for (uint32_t t = threadIdx.x; t <= nbk; t += kBlock) s_bs[t] = bstart[b0 + t];
  __syncthreads();
  uint64_t bb = 0;
  uint32_t bp = 0xffffffffu, dead = 0;
  const double ax = ext->ax, ay = ext->ay;
  __shared__ uint32_t s_win;
  // windows of consecutive buckets holding at most kBlockCap keys (usually
  // one window covers all kBucketsPerBlock buckets)
  uint32_t lb0 = 0;
  while (lb0 < nbk) {
    // largest lb1 with s_bs[lb1] - s_bs[lb0] <= kBlockCap (bucket starts are monotone)
    if (threadIdx.x == 0) s_win = lb0;
    __syncthreads();
    for (uint32_t t = lb0 + 1 + threadIdx.x; t <= nbk; t += kBlock)
      if (s_bs[t] - s_bs[lb0] <= (uint32_t)kBlockCap) atomicMax(&s_win, t);
    __syncthreads();
    if (threadIdx.x == 0 && s_win == lb0) {  // one bucket above capacity: defer to K4b
      if (s_bs[lb0 + 1] > s_bs[lb0]) oversize[atomicAdd(&ctr->n_oversize, 1u)] = b0 + lb0;
      s_win = (lb0 + 1) | 0x80000000u;
    }
    __syncthreads();
    const uint32_t wv = s_win;
    const uint32_t lb1 = wv & 0x7fffffffu;
    if (!(wv & 0x80000000u)) {
      const uint32_t e0 = s_bs[lb0], cnt = s_bs[lb1] - e0;
      for (uint32_t t = threadIdx.x; t < cnt; t += kBlock) {
        const PtRec r = ld_rec256(&rec[e0 + t]);
        s_key[t] = r.key;
        s_idx[t] = r.idx;
        s_x[t] = r.x;
        s_y[t] = r.y;
        s_d2[t] = dist2_rn(__dsub_rn(r.x, ax), __dsub_rn(r.y, ay));
        s_lb[t] = (uint16_t)(bucket_of(r.key, scale, nb) - b0);
      }
      __syncthreads();
      for (uint32_t t = threadIdx.x; t < cnt; t += kBlock) {
        const uint32_t lb = s_lb[t];
        const uint32_t sb = s_bs[lb] - e0, se = s_bs[lb + 1] - e0;
        const uint64_t kt = s_key[t];
        const double dt = s_d2[t], xt = s_x[t], yt = s_y[t];
        const uint32_t it = s_idx[t];
        uint32_t r = 0;
        bool is_dead = false;
        // key_less(j, t), reading dist2, index and coordinates only on equal
        // keys: equal points have equal keys and dist2 (the anchor's copies
        // were dropped), so a duplicate is always found in the last branch
        for (uint32_t j = sb; j < se; ++j) {
          const uint64_t kj = s_key[j];
          if (kj != kt) { r += kj < kt; continue; }
          const double dj = s_d2[j];
          if (dj != dt) { r += dj < dt; continue; }
          const uint32_t ij = s_idx[j];
          r += ij < it;
          is_dead |= (ij < it && s_x[j] == xt && s_y[j] == yt);
        }
        const uint32_t pos = 1 + e0 + sb + r;
        A_x[pos] = xt;
        A_y[pos] = yt;
        A_idx[pos] = is_dead ? kDead : it;
        if (is_dead) ++dead;
        else best_merge(bb, bp, dbits(dt), pos);
      }
    }
    __syncthreads();
    lb0 = lb1;
  }
  if (dead) atomicAdd(&ctr->dead, dead);
  block_best<kBlock>(bb, bp, &partials[blockIdx.x]);
}

// K4b: CTA per oversize bucket (grid-stride over the deferred list): rank
// sort in shared memory up to kSortCap keys, heap sort in global memory
// beyond that (degenerate inputs: long equal-angle runs). Same dedup/output.
__device__ __forceinline__ bool rec_less(const PtRec* k, double ax, double ay, uint32_t a,
                                         uint32_t b) {
  if (k[a].key != k[b].key) return k[a].key < k[b].key;
  const double da = dist2_rn(__dsub_rn(k[a].x, ax), __dsub_rn(k[a].y, ay));
  const double db = dist2_rn(__dsub_rn(k[b].x, ax), __dsub_rn(k[b].y, ay));
  if (da != db) return da < db;
  return k[a].idx < k[b].idx;
}

__global__ void __launch_bounds__(kSortBlock) k_bucket_sort_cta(
    const uint32_t* __restrict__ bstart, PtRec* __restrict__ rec,
    const ExtResult* __restrict__ ext, const uint32_t* __restrict__ oversize,
    const Counters* __restrict__ ctr_in, double* __restrict__ A_x, double* __restrict__ A_y,
    uint32_t* __restrict__ A_idx, BucketBest* __restrict__ partials, Counters* __restrict__ ctr) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
  double* s_d2 = reinterpret_cast<double*>(s_key + kSortCap);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_d2 + kSortCap);
  uint32_t* s_rank = s_idx + kSortCap;
  const uint32_t nov = ctr_in->n_oversize;
  const double ax = ext->ax, ay = ext->ay;
  uint64_t bb = 0;
  uint32_t bp = 0xffffffffu, dead = 0;
  for (uint32_t w = blockIdx.x; w < nov; w += gridDim.x) {
    const uint32_t b = oversize[w];
    const uint32_t start = bstart[b], s = bstart[b + 1] - start;
    const PtRec* R = rec + start;
    if (s <= (uint32_t)kSortCap) {
      __syncthreads();
      for (uint32_t t = threadIdx.x; t < s; t += kSortBlock) {
        s_key[t] = R[t].key;
        s_idx[t] = R[t].idx;
        s_d2[t] = dist2_rn(__dsub_rn(R[t].x, ax), __dsub_rn(R[t].y, ay));
      }
      __syncthreads();
      for (uint32_t e = threadIdx.x; e < s; e += kSortBlock) {
        const uint64_t ke = s_key[e];
        const double de = s_d2[e];
        const uint32_t ie = s_idx[e];
        uint32_t r = 0;
        for (uint32_t j = 0; j < s; ++j) r += key_less(s_key[j], s_d2[j], s_idx[j], ke, de, ie);
        s_rank[r] = e;
      }
      __syncthreads();
      for (uint32_t r = threadIdx.x; r < s; r += kSortBlock) {
        const uint32_t e = s_rank[r];
        const double px = R[e].x, py = R[e].y;
        bool is_dead = false;
        for (int32_t q = (int32_t)r - 1; q >= 0; --q) {
          const uint32_t f = s_rank[q];
          if (s_key[f] != s_key[e] || s_d2[f] != s_d2[e]) break;
          if (R[f].x == px && R[f].y == py) { is_dead = true; break; }
        }
        const uint32_t pos = 1 + start + r;
        A_x[pos] = px;
        A_y[pos] = py;
        A_idx[pos] = is_dead ? kDead : s_idx[e];
        if (is_dead) ++dead;
        else best_merge(bb, bp, dbits(s_d2[e]), pos);
      }
    } else if (threadIdx.x == 0) {
      PtRec* k = rec + start;
      auto sift = [&](uint32_t root, uint32_t len) {
        while (true) {
          uint32_t c = 2 * root + 1;
          if (c >= len) break;
          if (c + 1 < len && rec_less(k, ax, ay, c, c + 1)) ++c;
          if (!rec_less(k, ax, ay, root, c)) break;
          const PtRec t = k[root]; k[root] = k[c]; k[c] = t;
          root = c;
        }
      };
      for (int64_t r = (int64_t)s / 2 - 1; r >= 0; --r) sift((uint32_t)r, s);
      for (uint32_t len = s; len > 1; --len) {
        const PtRec t = k[0]; k[0] = k[len - 1]; k[len - 1] = t;
        sift(0, len - 1);
      }
      uint32_t run_start = 0;
      double prev_d2 = 0.0;
      for (uint32_t r = 0; r < s; ++r) {
        const double px = k[r].x, py = k[r].y;
        const double d2 = dist2_rn(__dsub_rn(px, ax), __dsub_rn(py, ay));
        if (r > 0 && (k[r - 1].key != k[r].key || prev_d2 != d2)) run_start = r;
        prev_d2 = d2;
        bool is_dead = false;
        for (uint32_t q = run_start; q < r; ++q)
          if (k[q].x == px && k[q].y == py) { is_dead = true; break; }
        const uint32_t pos = 1 + start + r;
        A_x[pos] = px;
        A_y[pos] = py;
        A_idx[pos] = is_dead ? kDead : k[r].idx;
        if (is_dead) ++dead;
        else best_merge(bb, bp, dbits(d2), pos);
      }
    }
  }
  if (dead) atomicAdd(&ctr->dead, dead);
  block_best<kSortBlock>(bb, bp, &partials[blockIdx.x]);
}

// Anchor into position 0 of the annotated buffer, M = 1 + sorted count.
__global__ void k_put_anchor(const ExtResult* __restrict__ ext, const uint32_t* __restrict__ bstart,
                             uint32_t nb, double* A_x, double* A_y, uint32_t* A_idx,
                             Counters* __restrict__ ctr) {
  A_x[0] = ext->ax;
  A_y[0] = ext->ay;
  A_idx[0] = ext->idx[4];
  ctr->m_total = 1 + bstart[nb];
}

// split_regions (angular.hpp:197-204): first position >= 1 with maximal
// dist2, from the per-block partial bests of the sort kernels.
__global__ void __launch_bounds__(1024) k_longest(const BucketBest* __restrict__ best,
                                                  uint32_t nb, Counters* __restrict__ ctr) {
  uint64_t bb = 0;
  uint32_t bp = 0xffffffffu;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    const BucketBest r = best[b];
    if (r.pos == 0xffffffffu) continue;
    if (bp == 0xffffffffu || r.d2bits > bb || (r.d2bits == bb && r.pos < bp)) {
      bb = r.d2bits; bp = r.pos;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ob = __shfl_xor_sync(0xffffffffu, bb, o);
    const uint32_t op = __shfl_xor_sync(0xffffffffu, bp, o);
    if (op != 0xffffffffu && (bp == 0xffffffffu || ob > bb || (ob == bb && op < bp))) {
      bb = ob; bp = op;
    }
  }
  __shared__ uint64_t s_b[32];
  __shared__ uint32_t s_p[32];
  if ((threadIdx.x & 31) == 0) { s_b[threadIdx.x >> 5] = bb; s_p[threadIdx.x >> 5] = bp; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      if (s_p[w] != 0xffffffffu && (bp == 0xffffffffu || s_b[w] > bb || (s_b[w] == bb && s_p[w] < bp))) {
        bb = s_b[w]; bp = s_p[w];
      }
    }
    ctr->longest = bp;
  }
}

// Position-wise split_regions over a compacted buffer (used after duplicates
// were removed, when bucket positions shifted).
__global__ void k_longest_scan(const double* __restrict__ A_x, const double* __restrict__ A_y,
                               uint32_t m, unsigned long long* __restrict__ best_bits,
                               uint32_t* __restrict__ best_pos, int phase) {
  const double ax = A_x[0], ay = A_y[0];
  for (uint32_t p = 1 + blockIdx.x * blockDim.x + threadIdx.x; p < m; p += gridDim.x * blockDim.x) {
    const double d2 = dist2_rn(__dsub_rn(A_x[p], ax), __dsub_rn(A_y[p], ay));
    if (phase == 0) atomicMax(best_bits, (unsigned long long)dbits(d2));
    else if (dbits(d2) == *best_bits) atomicMin(best_pos, p);
  }
}

// ===========================================================================
// Stable compaction by flag (generic): keeps entries whose keep(i) is true,
// preserving order; copies (x, y, idx) triples. Used for duplicate removal
// (keep = idx != kDead) and for stable_compact after round 2
// (discard.hpp:128-145, keep = flag).
constexpr int kCompactItems = 8;
constexpr int kCompactTile = kBlock * kCompactItems;

template <int kMode>  // 0: keep idx != kDead; 1: keep flags[i] != 0
__global__ void __launch_bounds__(kBlock) k_compact_xyi(
    const double* __restrict__ in_x, const double* __restrict__ in_y,
    const uint32_t* __restrict__ in_i, const uint8_t* __restrict__ flags, const uint32_t* n_dev,
    uint32_t n_host, double* __restrict__ out_x, double* __restrict__ out_y,
    uint32_t* __restrict__ out_i, uint64_t* __restrict__ status, Counters* __restrict__ ctr,
    uint32_t* __restrict__ n_out) {
  __shared__ uint32_t s_tile, s_excl, s_rows[kCompactItems * kWarps + 1];
  const uint32_t n = n_dev ? *n_dev : n_host;
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile_ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kCompactTile;  // striped: item (k, t) = base + k * kBlock + t
  bool keep[kCompactItems];
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    const uint32_t i = base + k * kBlock + threadIdx.x;
    bool kp = false;
    if (i < n) kp = (kMode == 0) ? (in_i[i] != kDead) : (flags[i] != 0);
    keep[k] = kp;
  }
  uint32_t rk[kCompactItems];
  const uint32_t total = striped_keep_ranks<kCompactItems>(keep, rk, s_rows);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, total);
    if (threadIdx.x == 0) {
      s_excl = (uint32_t)e;
      if (base + kCompactTile >= n) *n_out = (uint32_t)(e + total);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    if (keep[k]) {
      const uint32_t i = base + k * kBlock + threadIdx.x, o = s_excl + rk[k];
      out_x[o] = in_x[i];
      out_y[o] = in_y[i];
      out_i[o] = in_i[i];
    }
  }
}

// ===========================================================================
// K5: round-2 region walks (discard.hpp:36-66, 79-124) -- one warp per slice.
// A step discards P iff orient(temp, P_l, P) is Left (right region) / Right
// (left region); otherwise P becomes temp. Equivalently P is kept iff its
// direction from P_l does not turn back past temp's, so the kept points are
// the running maxima (minima) of the angle theta(P) of P - P_l. The warp
// speculates 32 steps at once with a max-scan over a floating-point theta,
// then VERIFIES every step with the exact predicate against the temp the
// speculation implies; the prefix up to the first disagreement is exact by
// induction, the disagreeing step takes the exact decision, and the walk
// resumes after it. Results are identical to the sequential loop; theta only
// decides how many steps one iteration commits.
struct SliceGeom {
  uint32_t l;         // longest (buffer position)
  uint32_t m;         // buffer size M
  uint32_t chunked;
  uint32_t n_right;   // slices in the right region
  uint32_t n_left;    // slices in the left region
  uint32_t step_r, step_l;
  uint32_t pad;
};

__device__ __forceinline__ double walk_theta(double px, double py, double lx, double ly, double ux,
                                             double uy) {
  const double vx = px - lx, vy = py - ly;
  return atan2(ux * vy - uy * vx, ux * vx + uy * vy);
}

__global__ void __launch_bounds__(kBlock) k_round2_walk(const double* __restrict__ A_x,
                                                        const double* __restrict__ A_y,
                                                        SliceGeom g, uint8_t* __restrict__ flags) {
  const uint32_t slice = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (slice >= g.n_right + g.n_left) return;
  uint32_t seed, start, count;
  int dir;
  if (slice < g.n_right) {
    dir = 1;
    if (g.chunked) {
      const uint32_t begin = 1 + slice * g.step_r;
      const uint32_t end = min(begin + g.step_r, g.l);
      seed = begin; start = begin + 1; count = end - begin - 1;
    } else {
      seed = 0; start = 1; count = g.l - 1;
    }
  } else {
    dir = -1;
    const uint32_t s = slice - g.n_right;
    const uint32_t m_left = g.m - 1 - g.l;
    if (g.chunked) {
      const uint32_t pos = s * g.step_l;
      seed = g.m - 1 - pos;
      const uint32_t off = min(pos + g.step_l - 1, m_left - 1);
      const uint32_t lo = g.m - 1 - off;
      start = seed - 1; count = seed - lo;
    } else {
      seed = g.m - 1; start = g.m - 2; count = g.m - 2 - g.l;
    }
  }
  if (count == 0) return;
  const double lx = A_x[g.l], ly = A_y[g.l];
  const double ux = A_x[0] - lx, uy = A_y[0] - ly;  // theta measured from P_l -> anchor
  const double sgn = (dir > 0) ? 1.0 : -1.0;        // left region: running minimum
  double tx = A_x[seed], ty = A_y[seed];
  double tth = sgn * walk_theta(tx, ty, lx, ly, ux, uy);
  const uint32_t lt = lanemask_lt();
  uint32_t i = 0;
  while (i < count) {
    const uint32_t off = i + lane;
    const bool valid = off < count;
    const uint32_t pos = (dir > 0) ? start + off : start - off;
    double px = 0.0, py = 0.0, th = -1e300;
    if (valid) {
      px = A_x[pos];
      py = A_y[pos];
      th = sgn * walk_theta(px, py, lx, ly, ux, uy);
    }
    // exclusive running max of theta (speculated temp angle before this step)
    double ex = th;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double v = __shfl_up_sync(0xffffffffu, ex, o);
      if (lane >= o) ex = fmax(ex, v);
    }
    double run = __shfl_up_sync(0xffffffffu, ex, 1);
    run = (lane == 0) ? tth : fmax(run, tth);
    const bool cand_keep = valid && th >= run;
    const uint32_t kmask = __ballot_sync(0xffffffffu, cand_keep);
    const uint32_t before = kmask & lt;
    const int src = before ? (31 - __clz(before)) : -1;
    const double sx = __shfl_sync(0xffffffffu, px, src < 0 ? 0 : src);
    const double sy = __shfl_sync(0xffffffffu, py, src < 0 ? 0 : src);
    const double cx = (src < 0) ? tx : sx, cy = (src < 0) ? ty : sy;
    const double c = cross_rn(cx, cy, lx, ly, px, py);
    const bool exact_discard = (dir > 0) ? (c > 0.0) : (c < 0.0);
    const bool mismatch = valid && (exact_discard == cand_keep);
    const uint32_t mm = __ballot_sync(0xffffffffu, mismatch);
    const int f = mm ? (__ffs(mm) - 1) : 32;
    if (valid && lane < f && !cand_keep) flags[pos] = 0;
    if (f < 32) {
      if (lane == f && exact_discard) flags[pos] = 0;
      const bool keep_f = !__shfl_sync(0xffffffffu, exact_discard, f);
      const int new_src = keep_f ? f : __shfl_sync(0xffffffffu, src, f);
      if (new_src >= 0) {
        tx = __shfl_sync(0xffffffffu, px, new_src);
        ty = __shfl_sync(0xffffffffu, py, new_src);
        tth = __shfl_sync(0xffffffffu, th, new_src);
      }
      i += f + 1;
    } else {
      if (kmask) {
        const int last = 31 - __clz(kmask);
        tx = __shfl_sync(0xffffffffu, px, last);
        ty = __shfl_sync(0xffffffffu, py, last);
        tth = __shfl_sync(0xffffffffu, th, last);
      }
      i += 32;
    }
  }
}

// K5 (block version): one CTA per slice, 1024 walk steps per window. Same
// speculate-then-verify contract as the warp version above, with a block-wide
// max-scan of (phi', walk index): phi' is a pseudo-angle of P - P_l (one
// division, monotone in the true angle; sign-flipped for the left region),
// the running maximum's element is the speculated temp of every step, each
// step is verified with the exact orient(), and the window restarts after the
// first disagreement with the exact decision applied.
constexpr int kWalkBlock = 256;
constexpr int kWalkItems = 4;
constexpr int kWalkWin = kWalkBlock * kWalkItems;

__device__ __forceinline__ double pseudo_angle(double px, double py, double lx, double ly,
                                               double ux, double uy) {
  const double vx = px - lx, vy = py - ly;
  const double c = ux * vx + uy * vy;   // along P_l -> anchor
  const double sn = ux * vy - uy * vx;  // across
  const double as = fabs(sn), den = fabs(c) + as;
  if (den == 0.0) return 0.0;
  const double t = 1.0 - c / den;      // [0, 2], increasing with the angle from u
  return sn >= 0.0 ? t : -t;
}

struct MaxPair {  // running maximum by (phi, walk index): the latest maximum wins
  double v;
  int32_t k;
};
__device__ __forceinline__ MaxPair mp_max(MaxPair a, MaxPair b) {
  return (b.v > a.v || (b.v == a.v && b.k > a.k)) ? b : a;
}

__global__ void __launch_bounds__(kWalkBlock) k_round2_block(const double* __restrict__ A_x,
                                                             const double* __restrict__ A_y,
                                                             SliceGeom g,
                                                             uint8_t* __restrict__ flags) {
  const uint32_t slice = blockIdx.x;
  uint32_t seed, start, count;
  int dir;
  if (slice < g.n_right) {
    dir = 1;
    if (g.chunked) {
      const uint32_t begin = 1 + slice * g.step_r;
      const uint32_t end = min(begin + g.step_r, g.l);
      seed = begin; start = begin + 1; count = end - begin - 1;
    } else {
      seed = 0; start = 1; count = g.l - 1;
    }
  } else {
    dir = -1;
    const uint32_t sl = slice - g.n_right;
    const uint32_t m_left = g.m - 1 - g.l;
    if (g.chunked) {
      const uint32_t pos = sl * g.step_l;
      seed = g.m - 1 - pos;
      const uint32_t off = min(pos + g.step_l - 1, m_left - 1);
      const uint32_t lo = g.m - 1 - off;
      start = seed - 1; count = seed - lo;
    } else {
      seed = g.m - 1; start = g.m - 2; count = g.m - 2 - g.l;
    }
  }
  if (count == 0) return;
  __shared__ MaxPair s_wm[kWalkBlock / 32];
  __shared__ int32_t s_first;
  __shared__ MaxPair s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double lx = A_x[g.l], ly = A_y[g.l];
  const double ux = A_x[0] - lx, uy = A_y[0] - ly;
  const double sgn = (dir > 0) ? 1.0 : -1.0;
  // walk index -1 = the seed; position of walk index k: start +- k
  auto wpos = [&](int32_t k) -> uint32_t {
    return k < 0 ? seed : ((dir > 0) ? start + (uint32_t)k : start - (uint32_t)k);
  };
  MaxPair carry;
  carry.v = sgn * pseudo_angle(A_x[seed], A_y[seed], lx, ly, ux, uy);
  carry.k = -1;
  int32_t w0 = 0;
  while (w0 < (int32_t)count) {
    // load this thread's kWalkItems consecutive walk steps
    double px[kWalkItems], py[kWalkItems], ph[kWalkItems];
    bool val[kWalkItems];
    const int32_t k0 = w0 + threadIdx.x * kWalkItems;
#pragma unroll
    for (int u = 0; u < kWalkItems; ++u) {
      const int32_t k = k0 + u;
      val[u] = k < (int32_t)count;
      if (val[u]) {
        const uint32_t p = wpos(k);
        px[u] = A_x[p];
        py[u] = A_y[p];
        ph[u] = sgn * pseudo_angle(px[u], py[u], lx, ly, ux, uy);
      } else {
        px[u] = py[u] = 0.0;
        ph[u] = -1e300;
      }
    }
    // thread aggregate, then block exclusive max-scan
    MaxPair agg{-1e300, INT32_MIN};
#pragma unroll
    for (int u = 0; u < kWalkItems; ++u)
      if (val[u]) agg = mp_max(agg, MaxPair{ph[u], k0 + u});
    MaxPair inc = agg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      MaxPair y;
      y.v = __shfl_up_sync(0xffffffffu, inc.v, o);
      y.k = __shfl_up_sync(0xffffffffu, inc.k, o);
      if (lane >= o) inc = mp_max(inc, y);
    }
    if (lane == 31) s_wm[warp] = inc;
    if (threadIdx.x == 0) s_first = INT32_MAX;
    __syncthreads();
    MaxPair ex = carry;
    for (int w = 0; w < warp; ++w) ex = mp_max(ex, s_wm[w]);
    MaxPair prev;
    prev.v = __shfl_up_sync(0xffffffffu, inc.v, 1);
    prev.k = __shfl_up_sync(0xffffffffu, inc.k, 1);
    if (lane > 0) ex = mp_max(ex, prev);
    // per step: speculated temp = running max before it; verify exactly
    bool cand_keep[kWalkItems], ex_disc[kWalkItems];
    int32_t tk[kWalkItems];
#pragma unroll
    for (int u = 0; u < kWalkItems; ++u) {
      tk[u] = ex.k;
      cand_keep[u] = val[u] && ph[u] >= ex.v;
      ex_disc[u] = false;
      if (val[u]) {
        const uint32_t tp = wpos(ex.k);
        const double c = cross_rn(A_x[tp], A_y[tp], lx, ly, px[u], py[u]);
        ex_disc[u] = (dir > 0) ? (c > 0.0) : (c < 0.0);
        if (ex_disc[u] == cand_keep[u]) atomicMin(&s_first, k0 + u);
        ex = mp_max(ex, MaxPair{ph[u], k0 + u});
      }
    }
    __syncthreads();
    const int32_t f = s_first;
#pragma unroll
    for (int u = 0; u < kWalkItems; ++u) {
      const int32_t k = k0 + u;
      if (!val[u] || k > f) continue;
      const bool disc = (k < f) ? !cand_keep[u] : ex_disc[u];
      if (disc) flags[wpos(k)] = 0;
      if (k == f) {  // the exact decision fixes the temp after step f
        MaxPair nc;
        if (ex_disc[u]) {
          const uint32_t tp = wpos(tk[u]);
          nc.v = sgn * pseudo_angle(A_x[tp], A_y[tp], lx, ly, ux, uy);
          nc.k = tk[u];
        } else {
          nc.v = ph[u];
          nc.k = k;
        }
        s_carry = nc;
      }
    }
    if (f == INT32_MAX) {
      // whole window verified: carry = running max through the window
      MaxPair tot = carry;
      for (int w = 0; w < kWalkBlock / 32; ++w) tot = mp_max(tot, s_wm[w]);
      carry = tot;
      w0 += kWalkWin;
      __syncthreads();
    } else {
      __syncthreads();
      carry = s_carry;
      w0 = f + 1;
    }
  }
}

// ===========================================================================
// K7 (v1): graham_finalize (pipeline.hpp:57-67) -- the exact sequential stack
// scan, run by one device thread (no host stage).
__global__ void k_graham_seq(const double* __restrict__ R_x, const double* __restrict__ R_y,
                             const uint32_t* __restrict__ R_i, const uint32_t* n_dev,
                             uint32_t* __restrict__ stack, uint32_t* __restrict__ out_idx,
                             Counters* __restrict__ ctr) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  const uint32_t n = *n_dev;
  uint32_t top = 0;
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;  // stack[top-1], stack[top-2]
  for (uint32_t i = 0; i < n; ++i) {
    const double px = R_x[i], py = R_y[i];
    while (top >= 2 && !(cross_rn(s2x, s2y, s1x, s1y, px, py) > 0.0)) {
      --top;
      s1x = s2x; s1y = s2y;
      if (top >= 2) { const uint32_t q = stack[top - 2]; s2x = R_x[q]; s2y = R_y[q]; }
    }
    stack[top++] = i;
    s2x = s1x; s2y = s1y;
    s1x = px; s1y = py;
  }
  for (uint32_t k = 0; k < top; ++k) out_idx[k] = R_i[stack[k]];
  ctr->hull = top;
}

// Device self-check: glibc-identical atan2.
__global__ void k_atan2(const double* __restrict__ y, const double* __restrict__ x,
                        double* __restrict__ out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = glibc_atan2(y[i], x[i]);
}

}  // namespace gscan
