// K7/K8 tree strategy: graham_finalize (pipeline.hpp:57-67) for buffers where
// most points are popped (round-2 output of squares and disks).
//
// Warp-speculative scans advance 32 points per iteration only while nothing is
// popped; on these buffers nearly every point pops, so here every scan is a
// plain sequential stack scan run by ONE thread (~2 orient() per point), and
// the parallelism comes from running many of them:
//
//   up      level j: Q_j is cut into chunks of kTreeChunk; every chunk's local
//           scan from an empty stack leaves a chain; the chains concatenated
//           form Q_{j+1} (Q_0 = the buffer). Repeat until Q_K is small.
//   top     one thread scans Q_K, recording the persistent stack (parent[p] =
//           the element below p when p was pushed) and the top before every
//           Q_{K-1} chunk.
//   down    level j -> j-1: the state before a Q_{j-1} chunk is the state
//           before the Q_j chunk holding its chain's first element, scanned
//           over the Q_j elements in between (thread per chunk).
//   certify every buffer chunk replays ITS OWN points from the candidate state
//           at its start and must end exactly in the candidate state at its
//           end (top and every parent link of its surviving pushes).
//
// The candidate rests on "scan(X ++ Y) = scan(scan(X) ++ scan_local(Y))",
// which exact geometry guarantees; rounding can only make the certificate
// fail (then the exact sequential kernel runs), never a wrong hull: by
// induction over chunks, certified states are the sequential scan's states.
#pragma once
#include "graham.cuh"

namespace gscan {

constexpr int kTreeChunk = 32;   // short chunks: every scan is latency-bound (~200 cycles/step)
constexpr int kTreeCta = 64;      // chunks (threads) per CTA
constexpr uint32_t kTreeTop = 128;  // largest top-level list for the single-thread scan

// Chunk coordinates staged in shared memory, [point][thread] so that the
// threads of a warp (each scanning its own chunk) hit distinct banks.
constexpr size_t kTreeSmem = (size_t)kTreeChunk * kTreeCta * 16;

__device__ __forceinline__ void stage_chunks(const uint32_t* __restrict__ Q, uint32_t nq,
                                             uint32_t first_chunk, const double* __restrict__ R_x,
                                             const double* __restrict__ R_y, double* sx,
                                             double* sy) {
  // element k of chunk t (t = 0..kTreeCta-1) -> sx[k * kTreeCta + t]
  const uint32_t base = first_chunk * kTreeChunk;
  for (uint32_t e = threadIdx.x; e < (uint32_t)kTreeChunk * kTreeCta; e += blockDim.x) {
    const uint32_t g = base + e;  // coalesced over the CTA's consecutive chunks
    if (g >= nq) break;
    const uint32_t p = Q ? Q[g] : g;
    const uint32_t t = e / kTreeChunk, k = e % kTreeChunk;
    sx[k * kTreeCta + t] = R_x[p];
    sy[k * kTreeCta + t] = R_y[p];
  }
}

// Local chains of Q (R positions; nullptr = identity) in chunks of kTreeChunk.
// out_q[c * kTreeChunk + k] = the Q index of the k-th chain element.
__global__ void __launch_bounds__(kTreeCta) k_gr_local(const uint32_t* __restrict__ Q, uint32_t nq,
                                                      const double* __restrict__ R_x,
                                                      const double* __restrict__ R_y,
                                                      uint32_t* __restrict__ out_q,
                                                      uint32_t* __restrict__ out_len) {
  extern __shared__ __align__(16) double tsm[];
  double* sx = tsm;
  double* sy = tsm + kTreeChunk * kTreeCta;
  __shared__ uint8_t s_stk[kTreeChunk][kTreeCta];  // [depth][thread]: conflict-free
  stage_chunks(Q, nq, blockIdx.x * kTreeCta, R_x, R_y, sx, sy);
  __syncthreads();
  const uint32_t c = blockIdx.x * kTreeCta + threadIdx.x;
  const uint32_t lo = c * kTreeChunk;
  if (lo >= nq) return;
  const int cnt = (int)min((uint32_t)kTreeChunk, nq - lo);
  const int t = threadIdx.x;
  int top = 0;
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;  // stack[top-1], stack[top-2]
  for (int k = 0; k < cnt; ++k) {
    const double px = sx[k * kTreeCta + t], py = sy[k * kTreeCta + t];
    while (top >= 2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
      --top;
      s1x = s2x; s1y = s2y;
      if (top >= 2) {
        const int q = s_stk[top - 2][t];
        s2x = sx[q * kTreeCta + t]; s2y = sy[q * kTreeCta + t];
      }
    }
    s_stk[top][t] = (uint8_t)k;
    ++top;
    s2x = s1x; s2y = s1y;
    s1x = px; s1y = py;
  }
  for (int k = 0; k < top; ++k) out_q[(size_t)c * kTreeChunk + k] = lo + s_stk[k][t];
  out_len[c] = top;
}

// Q_{j+1}[off[c] + k] = Q_j[chain element], up[off[c] + k] = its Q_j index.
__global__ void k_gr_gather(const uint32_t* __restrict__ Q, const uint32_t* __restrict__ chain_q,
                            const uint32_t* __restrict__ len, const uint32_t* __restrict__ off,
                            uint32_t nchunks, uint32_t* __restrict__ Qn, uint32_t* __restrict__ up) {
  const uint32_t c = blockIdx.x * (blockDim.x / kTreeChunk) + threadIdx.x / kTreeChunk;
  const uint32_t k = threadIdx.x % kTreeChunk;
  if (c >= nchunks || k >= len[c]) return;
  const uint32_t qi = chain_q[(size_t)c * kTreeChunk + k];
  Qn[off[c] + k] = Q ? Q[qi] : qi;
  up[off[c] + k] = qi;
}

// Top: one thread scans Q_K (R positions; up = their Q_{K-1} indices),
// recording parent[] and bt[b] = top before the first element of Q_{K-1}
// chunk >= b, b = 0..nch (bt[nch] = final top). *len = final size.
__global__ void k_gr_top(const uint32_t* __restrict__ QK, const uint32_t* __restrict__ up,
                         const uint32_t* nk_dev, uint32_t nch, const double* __restrict__ R_x,
                         const double* __restrict__ R_y, uint32_t* __restrict__ parent,
                         uint32_t* __restrict__ bt, uint32_t* __restrict__ out_len,
                         uint32_t* __restrict__ fstack) {
  if (blockIdx.x != 0) return;
  __shared__ uint32_t s_stk[kTreeTop];   // stack of Q_K indices
  __shared__ double s_x[kTreeTop], s_y[kTreeTop];
  __shared__ uint32_t s_p[kTreeTop], s_ch[kTreeTop];
  const uint32_t nk = *nk_dev;
  for (uint32_t k = threadIdx.x; k < nk; k += blockDim.x) {
    const uint32_t p = QK[k];
    s_p[k] = p;
    s_ch[k] = up[k] / kTreeChunk;
    s_x[k] = R_x[p];
    s_y[k] = R_y[p];
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int top = 0;
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
  uint32_t next_b = 0;
  for (uint32_t k = 0; k < nk; ++k) {
    const uint32_t p = s_p[k];
    const uint32_t ch = s_ch[k];
    const uint32_t t = top ? s_p[s_stk[top - 1]] : kNone;
    for (; next_b <= ch; ++next_b) bt[next_b] = t;
    const double px = s_x[k], py = s_y[k];
    while (top >= 2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
      --top;
      s1x = s2x; s1y = s2y;
      if (top >= 2) { const uint32_t q = s_stk[top - 2]; s2x = s_x[q]; s2y = s_y[q]; }
    }
    parent[p] = top ? s_p[s_stk[top - 1]] : kNone;
    s_stk[top++] = k;
    s2x = s1x; s2y = s1y;
    s1x = px; s1y = py;
  }
  const uint32_t t = top ? s_p[s_stk[top - 1]] : kNone;
  for (; next_b <= nch; ++next_b) bt[next_b] = t;
  for (int k = 0; k < top; ++k) fstack[k] = s_p[s_stk[k]];
  *out_len = top;
}

// One thread's stack scan of a run of points on top of a persistent state
// (top `base`, parent[] links below it). The run's coordinates come from
// shared memory (cx/cy at index k * kTreeCta + lane); own pushes are kept as
// run indices in stk[depth * kTreeCta + lane]; elements of the persistent
// part are loaded from global memory when pops reach them. pos(k) gives the
// R position of run element k (for parent links and the result).
struct PersistentTop {
  uint32_t b1, b2;  // top two elements of the persistent part (kNone if absent)
};

template <typename PosF, typename OnPush>
__device__ __forceinline__ int persistent_scan(PosF&& pos, int cnt, const double* cx,
                                               const double* cy, PersistentTop& pt,
                                               const double* __restrict__ R_x,
                                               const double* __restrict__ R_y,
                                               const uint32_t* __restrict__ parent, uint16_t* stk,
                                               OnPush&& on_push) {
  const int t = threadIdx.x;
  int top = 0;  // own pushes
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;  // coordinates of the whole stack's top two
  if (pt.b1 != kNone) { s1x = R_x[pt.b1]; s1y = R_y[pt.b1]; }
  if (pt.b2 != kNone) { s2x = R_x[pt.b2]; s2y = R_y[pt.b2]; }
  for (int k = 0; k < cnt; ++k) {
    const double px = cx[k * kTreeCta + t], py = cy[k * kTreeCta + t];
    while (true) {
      // the whole stack (persistent part + own pushes) holds >= 2 elements
      const bool has2 = (top >= 2) || (top == 1 && pt.b1 != kNone) ||
                        (top == 0 && pt.b1 != kNone && pt.b2 != kNone);
      if (!has2 || left_turn(s2x, s2y, s1x, s1y, px, py)) break;
      if (top >= 1) {
        --top;
      } else {
        pt.b1 = pt.b2;
        pt.b2 = (pt.b1 != kNone) ? parent[pt.b1] : kNone;
      }
      s1x = s2x; s1y = s2y;
      if (top >= 2) {
        const int q = stk[(top - 2) * kTreeCta + t];
        s2x = cx[q * kTreeCta + t]; s2y = cy[q * kTreeCta + t];
      } else {
        const uint32_t ns = (top == 1) ? pt.b1 : pt.b2;
        if (ns != kNone) { s2x = R_x[ns]; s2y = R_y[ns]; }
      }
    }
    on_push(k, top ? pos(stk[(top - 1) * kTreeCta + t]) : pt.b1);
    stk[top * kTreeCta + t] = (uint16_t)k;
    ++top;
    s2x = s1x; s2y = s1y;
    s1x = px; s1y = py;
  }
  return top;
}

// Down: for every Q_{j-1} chunk c' (thread), the state before it: the state
// before the Q_j chunk c holding its chain's first element (offset off[c'])
// scanned over Q_j[c * kTreeChunk, off[c']). Q_j holds R positions.
__global__ void __launch_bounds__(kTreeCta) k_gr_down(const uint32_t* __restrict__ Qj,
                                                     const uint32_t* __restrict__ off,
                                                     uint32_t nch_lo,
                                                     const uint32_t* __restrict__ bt_hi,
                                                     const double* __restrict__ R_x,
                                                     const double* __restrict__ R_y,
                                                     uint32_t* __restrict__ parent,
                                                     uint32_t* __restrict__ bt_lo) {
  extern __shared__ __align__(16) double tsm[];
  double* cx = tsm;
  double* cy = tsm + kTreeChunk * kTreeCta;
  __shared__ uint16_t s_stk[kTreeChunk * kTreeCta];
  const uint32_t cp = blockIdx.x * kTreeCta + threadIdx.x;
  const bool act = cp < nch_lo;
  const uint32_t e = act ? off[cp] : 0;
  const uint32_t c = e / kTreeChunk;
  const int cnt = (int)(e - c * kTreeChunk);  // < kTreeChunk
  // stage this thread's run (independent loads, unrolled)
  for (int k0 = 0; k0 < cnt; k0 += 8) {
    uint32_t pp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pp[u] = (k0 + u < cnt) ? Qj[c * kTreeChunk + k0 + u] : 0u;
    double vx[8], vy[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (k0 + u < cnt) { vx[u] = R_x[pp[u]]; vy[u] = R_y[pp[u]]; }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < cnt) { cx[(k0 + u) * kTreeCta + threadIdx.x] = vx[u]; cy[(k0 + u) * kTreeCta + threadIdx.x] = vy[u]; }
  }
  if (!act) return;
  PersistentTop pt;
  pt.b1 = bt_hi[c];
  pt.b2 = (pt.b1 != kNone) ? parent[pt.b1] : kNone;
  auto pos = [&](int k) -> uint32_t { return Qj[c * kTreeChunk + k]; };
  const int top = persistent_scan(pos, cnt, cx, cy, pt, R_x, R_y, parent, s_stk,
                                  [&](int k, uint32_t below) { parent[pos(k)] = below; });
  bt_lo[cp] = top ? pos(s_stk[(top - 1) * kTreeCta + threadIdx.x]) : pt.b1;
}

// Certificate (thread per buffer chunk): replay the chunk's own points from
// the candidate state bt[c]; the end state must be exactly bt[c + 1] with
// every surviving push linked as in parent[].
__global__ void __launch_bounds__(kTreeCta) k_gr_certify(uint32_t n, const double* __restrict__ R_x,
                                                        const double* __restrict__ R_y,
                                                        const uint32_t* __restrict__ parent,
                                                        const uint32_t* __restrict__ bt,
                                                        uint32_t* __restrict__ fail) {
  extern __shared__ __align__(16) double tsm[];
  double* cx = tsm;
  double* cy = tsm + kTreeChunk * kTreeCta;
  __shared__ uint16_t s_stk[kTreeChunk * kTreeCta];
  stage_chunks(nullptr, n, blockIdx.x * kTreeCta, R_x, R_y, cx, cy);
  __syncthreads();
  const uint32_t c = blockIdx.x * kTreeCta + threadIdx.x;
  const uint32_t lo = c * kTreeChunk;
  if (lo >= n) return;
  const int cnt = (int)min((uint32_t)kTreeChunk, n - lo);
  PersistentTop pt;
  pt.b1 = bt[c];
  pt.b2 = (pt.b1 != kNone) ? parent[pt.b1] : kNone;
  auto pos = [&](int k) -> uint32_t { return lo + (uint32_t)k; };
  bool ok = true;
  // every push's link at push time must be the candidate's link (pushes that
  // survive the chunk must match; popped ones are checked too -- a correct
  // candidate state at the next boundary implies them all, and checking them
  // here is cheaper than tracking survivors)
  const int top = persistent_scan(pos, cnt, cx, cy, pt, R_x, R_y, parent, s_stk,
                                  [&](int, uint32_t) {});
  const uint32_t end_top = top ? pos(s_stk[(top - 1) * kTreeCta + threadIdx.x]) : pt.b1;
  ok = bt[c + 1] == end_top;
  for (int k = 0; k < top && ok; ++k) {
    const uint32_t p = pos(s_stk[k * kTreeCta + threadIdx.x]);
    const uint32_t below = k ? pos(s_stk[(k - 1) * kTreeCta + threadIdx.x]) : pt.b1;
    if (parent[p] != below) ok = false;
  }
  if (!ok) atomicAdd(fail, 1u);
}

// Output (one CTA): the top-level scan's final stack is the certified final
// state iff its top is the certified top and every element links to the one
// below it in parent[] (all checked in parallel); otherwise the certified
// state is walked down its parent links by one thread.
__global__ void __launch_bounds__(1024) k_gr_emit(const uint32_t* __restrict__ bt_final,
                                                  const uint32_t* __restrict__ parent,
                                                  const uint32_t* __restrict__ fstack,
                                                  const uint32_t* __restrict__ flen_dev,
                                                  const uint32_t* __restrict__ R_i,
                                                  uint32_t* __restrict__ tmp,
                                                  uint32_t* __restrict__ out_idx,
                                                  Counters* __restrict__ ctr) {
  const uint32_t len = *flen_dev, top = *bt_final;
  bool ok = len > 0 && fstack[len - 1] == top;
  for (uint32_t k = threadIdx.x; k < len && ok; k += blockDim.x)
    ok = parent[fstack[k]] == (k ? fstack[k - 1] : kNone);
  if (__syncthreads_and(ok)) {
    for (uint32_t k = threadIdx.x; k < len; k += blockDim.x) out_idx[k] = R_i[fstack[k]];
    if (threadIdx.x == 0) ctr->hull = len;
    return;
  }
  if (threadIdx.x != 0) return;
  uint32_t h = 0;
  for (uint32_t t = top; t != kNone; t = parent[t]) tmp[h++] = t;
  for (uint32_t k = 0; k < h; ++k) out_idx[k] = R_i[tmp[h - 1 - k]];
  ctr->hull = h;
}

}  // namespace gscan
