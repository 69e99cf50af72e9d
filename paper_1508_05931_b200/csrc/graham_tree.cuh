// K7/K8 tree strategy: graham_finalize (pipeline.hpp:57-67) for buffers where
// most points are popped (round-2 output of squares and disks), as ONE kernel
// (one CTA, no host round trips).
//
// Warp-speculative scans advance 32 points per iteration only while nothing is
// popped; on these buffers nearly every point pops, so here every scan is a
// plain sequential stack scan run by ONE thread (~2 orient() per point), and
// the parallelism comes from running many short ones:
//
//   up      level j: Q_j (R positions; Q_0 = the buffer) is cut into chunks of
//           kTreeChunk; every chunk's scan from an empty stack leaves a chain;
//           the chains concatenated form Q_{j+1}. Repeat until Q_K is small.
//   top     one thread scans Q_K, recording the persistent stack (parent[p] =
//           the element below p when p was pushed) and the top before every
//           Q_{K-1} chunk.
//   down    level j -> j-1: the state before a Q_{j-1} chunk is the state
//           before the Q_j chunk holding its chain's first element, scanned
//           over the Q_j elements in between (thread per chunk).
//   certify every buffer chunk replays ITS OWN points from the candidate state
//           at its start and must end exactly in the candidate state at its
//           end (top and every parent link of its surviving pushes).
//   emit    the certified final state; if any chunk failed, the same CTA runs
//           the exact sequential scan instead.
//
// The candidate rests on "scan(X ++ Y) = scan(scan(X) ++ scan_local(Y))",
// which exact geometry guarantees; rounding can only make the certificate
// fail, never a wrong hull: by induction over chunks, certified states are the
// sequential scan's states.
#pragma once
#include "graham.cuh"

namespace gscan {

constexpr int kTreeChunk = 32;      // level-0 chunk (many CTAs); also the staging capacity
constexpr int kTreeChunkHi = 32;    // chunk of levels >= 1 (8 and 16 measured slower: per-level overhead dominates)
constexpr int kTreeThreads = 256;   // one CTA; chunks are processed in waves of this many
constexpr uint32_t kTreeTop = 128;  // largest top-level list for the single-thread scan
constexpr int kTreeMaxLevels = 32;
// shared memory: per thread a chunk's coordinates [k][t] and an index stack
// per-thread slot: chunk coordinates + positions (21 B per point) + the
// persistent-stack cache (20 B per cached element)
constexpr size_t tree_smem(int threads) {
  return (size_t)kTreeChunk * threads * (8 + 8 + 4 + 1) + (size_t)8 * threads * (4 + 8 + 8);
}
constexpr size_t kTreeSmem = tree_smem(256);

struct TreeLevel {
  uint32_t* Q;    // R positions (nullptr: identity, level 0)
  uint32_t* up;   // Q_{j-1} index of each element (level >= 1)
  uint32_t* off;  // chain offsets of this level's chunks in Q_{j+1} (nch + 1)
  uint32_t* bt;   // top before each chunk (nch + 1)
  uint32_t nq, nch;
};

// Workspace carved from one device buffer by the host; the kernel checks every
// level size against its capacity.
struct TreeWork {
  uint32_t* parent;  // N
  uint32_t* tmp;     // N (stack of the top-level / fallback scan)
  uint32_t* chainq;  // N: chain elements of the current level (Q index), chunk-strided
  uint32_t* chainp;  // N: the same elements' R positions
  uint32_t* len;     // ceil(N / kTreeChunk) + 1
  uint32_t* fstack;  // kTreeTop
  uint32_t* Qbuf[kTreeMaxLevels + 1];
  uint32_t* upbuf[kTreeMaxLevels + 1];
  uint32_t* offbuf[kTreeMaxLevels + 1];
  uint32_t* btbuf[kTreeMaxLevels + 1];
  uint32_t cap[kTreeMaxLevels + 1];  // element capacity of level j's Q / up
};

// CTA-wide exclusive scan of cnt uint32 (in place); returns the total.
__device__ uint32_t tree_scan(uint32_t* a, uint32_t cnt, uint32_t* s_w, uint32_t* s_carry) {
  if (threadIdx.x == 0) *s_carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (uint32_t base = 0; base < cnt; base += blockDim.x) {
    const uint32_t i = base + threadIdx.x;
    const uint32_t v = i < cnt ? a[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint32_t wv = lane < nw ? s_w[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wv, o);
        if (lane >= o) wv += y;
      }
      if (lane < nw) s_w[lane] = wv;
    }
    __syncthreads();
    const uint32_t carry = *s_carry;
    if (i < cnt) a[i] = carry + (warp ? s_w[warp - 1] : 0u) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) *s_carry = carry + s_w[nw - 1];
    __syncthreads();
  }
  return *s_carry;
}

// Stage up to kTreeChunk coordinates of run elements pos(0..cnt) into this
// thread's slots [k][t] (8 independent loads in flight).
template <int kStride, typename PosF>
__device__ __forceinline__ void tree_stage(PosF&& pos, int cnt, const double* __restrict__ R_x,
                                           const double* __restrict__ R_y, double* cx, double* cy,
                                           uint32_t* cp) {
  const int t = threadIdx.x;
  for (int k0 = 0; k0 < cnt; k0 += 8) {
    uint32_t pp[8];
    double vx[8], vy[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) pp[u] = (k0 + u < cnt) ? pos(k0 + u) : 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      vx[u] = (k0 + u < cnt) ? R_x[pp[u]] : 0.0;
      vy[u] = (k0 + u < cnt) ? R_y[pp[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (k0 + u < cnt) {
        cx[(k0 + u) * kStride + t] = vx[u];
        cy[(k0 + u) * kStride + t] = vy[u];
        if (cp) cp[(k0 + u) * kStride + t] = pp[u];
      }
  }
}

// One thread's stack scan of a staged run on top of a persistent state (top
// element b1, parent[] links below). The persistent state's top kTreePC
// elements (positions and coordinates) are first walked into a per-thread
// shared-memory cache pc[d * kStride + t] (d = depth, 0 = b1), so the pops
// that reach into it -- divergent, one per thread -- read shared memory;
// deeper elements come from global memory. Own pushes are kept as run
// indices in stk[depth * kStride + t]. on_push(k, below_run_index or -1 =
// persistent top) is called for every push. On return b1 = the persistent
// part's top. Returns the number of own pushes left.
constexpr int kTreePC = 8;

template <int kStride>
struct TreeCache {
  uint32_t* pos;  // [kTreePC][kStride]
  double* x;
  double* y;
};

template <int kStride, typename OnPush>
__device__ __forceinline__ int tree_scan_run(int cnt, const double* cx, const double* cy,
                                             uint32_t& b1, const double* __restrict__ R_x,
                                             const double* __restrict__ R_y,
                                             const uint32_t* __restrict__ parent, uint8_t* stk,
                                             TreeCache<kStride> pc, OnPush&& on_push) {
  const int t = threadIdx.x;
  // walk the persistent top into the cache (dependent parent loads, once)
  int ncached = 0;
  {
    uint32_t p = b1;
    uint32_t pp[kTreePC];
#pragma unroll
    for (int d = 0; d < kTreePC; ++d) {
      pp[d] = p;
      if (p != kNone) { ncached = d + 1; p = parent[p]; }
    }
    double vx[kTreePC], vy[kTreePC];
#pragma unroll
    for (int d = 0; d < kTreePC; ++d) {
      vx[d] = (d < ncached) ? R_x[pp[d]] : 0.0;
      vy[d] = (d < ncached) ? R_y[pp[d]] : 0.0;
    }
#pragma unroll
    for (int d = 0; d < kTreePC; ++d) {
      pc.pos[d * kStride + t] = (d < ncached) ? pp[d] : kNone;
      pc.x[d * kStride + t] = vx[d];
      pc.y[d * kStride + t] = vy[d];
    }
  }
  // persistent element at depth d (d >= pd: already popped above it)
  int pd = 0;  // persistent elements popped
  uint32_t deep = kNone;  // position at depth pd when pd >= ncached (global walk)
  auto pers_pos = [&](int d) -> uint32_t {  // d in {pd, pd + 1}
    if (d < kTreePC) return pc.pos[d * kStride + t];
    return kNone;  // handled by the caller through `deep`
  };
  uint32_t p1 = pers_pos(0);
  uint32_t p2 = (ncached >= 2) ? pers_pos(1) : kNone;
  int top = 0;
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
  if (p1 != kNone) { s1x = pc.x[t]; s1y = pc.y[t]; }
  if (p2 != kNone) {
    if (kTreePC >= 2) { s2x = pc.x[kStride + t]; s2y = pc.y[kStride + t]; }
  }
  // One flat loop, each iteration one pop or one push: a warp of divergent
  // scans then costs max over lanes of (pushes + pops) iterations instead of
  // the sum over points of the lanes' largest pop run.
  int k = 0;
  double px = 0, py = 0;
  if (cnt > 0) { px = cx[t]; py = cy[t]; }
  while (k < cnt) {
    const bool has2 = (top >= 2) || (top == 1 && p1 != kNone) ||
                      (top == 0 && p1 != kNone && p2 != kNone);
    if (has2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
      if (top >= 1) {
        --top;
      } else {  // pop the persistent top
        ++pd;
        p1 = p2;
        const int d2 = pd + 1;  // depth of the new second element
        if (d2 < ncached) {
          p2 = pc.pos[d2 * kStride + t];
        } else if (p1 != kNone && d2 >= kTreePC) {
          p2 = parent[p1];
          deep = p2;
        } else {
          p2 = kNone;
        }
      }
      s1x = s2x; s1y = s2y;
      if (top >= 2) {
        const int q = stk[(top - 2) * kStride + t];
        s2x = cx[q * kStride + t]; s2y = cy[q * kStride + t];
      } else if (top == 1) {
        if (p1 != kNone) {
          if (pd < kTreePC) { s2x = pc.x[pd * kStride + t]; s2y = pc.y[pd * kStride + t]; }
          else { s2x = R_x[p1]; s2y = R_y[p1]; }
        }
      } else {
        if (p2 != kNone) {
          const int d2 = pd + 1;
          if (d2 < kTreePC) { s2x = pc.x[d2 * kStride + t]; s2y = pc.y[d2 * kStride + t]; }
          else { s2x = R_x[p2]; s2y = R_y[p2]; }
        }
      }
      continue;
    }
    on_push(k, top ? (int)stk[(top - 1) * kStride + t] : -1, p1);
    stk[top * kStride + t] = (uint8_t)k;
    ++top;
    s2x = s1x; s2y = s1y;
    s1x = px; s1y = py;
    if (++k < cnt) { px = cx[k * kStride + t]; py = cy[k * kStride + t]; }
  }
  (void)deep;
  b1 = p1;
  return top;
}

// Shared-memory carve-up of one tree kernel: staging (coords, positions,
// index stack) and the persistent cache, all [element][thread].
template <int kStride>
struct TreeSmem {
  double *cx, *cy;
  uint32_t* cp;
  uint8_t* stk;
  TreeCache<kStride> pc;
  __device__ explicit TreeSmem(double* base) {
    cx = base;
    cy = cx + kTreeChunk * kStride;
    pc.x = cy + kTreeChunk * kStride;
    pc.y = pc.x + 8 * kStride;
    cp = reinterpret_cast<uint32_t*>(pc.y + 8 * kStride);
    pc.pos = cp + kTreeChunk * kStride;
    stk = reinterpret_cast<uint8_t*>(pc.pos + 8 * kStride);
  }
};

// ---------------------------------------------------------------------------
// Level 0, many CTAs: chains of the buffer's chunks (thread per chunk).
constexpr int kTreeCta = 64;
constexpr size_t kTreeCtaSmem = tree_smem(kTreeCta);

__global__ void __launch_bounds__(kTreeCta) k_gr_local0(uint32_t N, const double* __restrict__ R_x,
                                                       const double* __restrict__ R_y,
                                                       TreeWork w) {
  extern __shared__ __align__(16) double tsm[];
  TreeSmem<kTreeCta> sm(tsm);
  uint8_t* stk = sm.stk;
  const uint32_t c = blockIdx.x * kTreeCta + threadIdx.x;
  const uint32_t lo = c * kTreeChunk;
  if (lo >= N) return;
  const int cnt = (int)min((uint32_t)kTreeChunk, N - lo);
  tree_stage<kTreeCta>([&](int k) { return lo + (uint32_t)k; }, cnt, R_x, R_y, sm.cx, sm.cy, nullptr);
  uint32_t b1 = kNone;
  const int top = tree_scan_run<kTreeCta>(cnt, sm.cx, sm.cy, b1, R_x, R_y, w.parent, stk, sm.pc,
                                          [](int, int, uint32_t) {});
  for (int k = 0; k < top; ++k) {
    const uint32_t q = lo + stk[k * kTreeCta + threadIdx.x];
    w.chainq[lo + k] = q;
    w.chainp[lo + k] = q;
  }
  w.offbuf[0][c] = (uint32_t)top;
}

// Middle, ONE CTA: Q_1 from the level-0 chains, levels >= 1 up, the top-level
// scan, and the down-sweep to level 1 (bt_1). info[0] = 1: no shrink.
__global__ void __launch_bounds__(kTreeThreads, 1) k_gr_mid(
    const double* __restrict__ R_x, const double* __restrict__ R_y, uint32_t N, TreeWork w,
    uint32_t* __restrict__ info) {
  extern __shared__ __align__(16) double tsm[];
  TreeSmem<kTreeThreads> sm(tsm);
  double* cx = sm.cx;
  double* cy = sm.cy;
  uint32_t* cp = sm.cp;
  uint8_t* stk = sm.stk;
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  __shared__ TreeLevel L[kTreeMaxLevels + 1];
  __shared__ int s_K, s_bad;
  const int t = threadIdx.x;
  long long t_start = clock64();
  if (t == 0) {
    L[0].Q = nullptr;
    L[0].up = nullptr;
    L[0].nq = N;
    s_K = -1;
    s_bad = 0;
    info[0] = 0;
    info[2] = 0;
  }
  __syncthreads();
  for (int j = 0; j < kTreeMaxLevels; ++j) {
    const uint32_t nq = L[j].nq;
    const uint32_t cs = (j == 0) ? kTreeChunk : kTreeChunkHi;
    const uint32_t nch = (nq + cs - 1) / cs;
    if (t == 0) {
      L[j].nch = nch;
      L[j].off = w.offbuf[j];
      L[j].bt = w.btbuf[j];
    }
    __syncthreads();
    const uint32_t* Q = L[j].Q;
    if (j > 0) {  // level-0 chains come from k_gr_local0
      for (uint32_t c0 = 0; c0 < nch; c0 += kTreeThreads) {
        const uint32_t c = c0 + t;
        if (c < nch) {
          const uint32_t lo = c * cs;
          const int cnt = (int)min(cs, nq - lo);
          tree_stage<kTreeThreads>([&](int k) { return Q[lo + k]; }, cnt, R_x, R_y, cx, cy, cp);
          uint32_t b1 = kNone;
          const int top = tree_scan_run<kTreeThreads>(cnt, cx, cy, b1, R_x, R_y, w.parent, stk,
                                                      sm.pc, [](int, int, uint32_t) {});
          for (int k = 0; k < top; ++k) {
            const int e = stk[k * kTreeThreads + t];
            w.chainq[lo + k] = lo + e;
            w.chainp[lo + k] = cp[e * kTreeThreads + t];
          }
          L[j].off[c] = (uint32_t)top;
        }
      }
    }
    __syncthreads();
    const uint32_t total = tree_scan(L[j].off, nch, s_w, &s_carry);
    if (t == 0) {
      L[j].off[nch] = total;
      const bool shrink =
          (j == 0) ? (total * 20ull <= (uint64_t)nq * 17) : (total * 10ull <= (uint64_t)nq * 9);
      if (!shrink || total > w.cap[j + 1] || j + 1 > kTreeMaxLevels - 1) s_bad = 1;
      L[j + 1].Q = w.Qbuf[j + 1];
      L[j + 1].up = w.upbuf[j + 1];
      L[j + 1].nq = total;
    }
    __syncthreads();
    if (s_bad) break;
    for (uint32_t c = t; c < nch; c += kTreeThreads) {
      const uint32_t o = L[j].off[c], ln = L[j].off[c + 1] - o;
      for (uint32_t k0 = 0; k0 < ln; k0 += 8) {
        uint32_t qv[8], pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          qv[u] = (k0 + u < ln) ? w.chainq[c * cs + k0 + u] : 0u;
          pv[u] = (k0 + u < ln) ? w.chainp[c * cs + k0 + u] : 0u;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (k0 + u < ln) { L[j + 1].Q[o + k0 + u] = pv[u]; L[j + 1].up[o + k0 + u] = qv[u]; }
      }
    }
    __syncthreads();
    if (total <= kTreeTop) {
      if (t == 0) s_K = j + 1;
      __syncthreads();
      break;
    }
  }
  const int K = s_K;
  if (s_bad || K < 1) {  // no shrink: the host takes another strategy
    if (t == 0) { info[0] = 1; info[3] = 0; }
    return;
  }
  if (t == 0) {
    info[8] = (uint32_t)(clock64() - t_start);
    for (int j = 0; j <= K && j < 6; ++j) info[10 + j] = L[j].nq;
  }
  // ---- top: one thread over Q_K, staged in shared memory by all ----
  {
    const TreeLevel& tl = L[K];
    const TreeLevel& ll = L[K - 1];
    const uint32_t nk = tl.nq;  // <= kTreeTop
    uint32_t* s_p = cp;         // reuse the staging area
    uint32_t* s_ch = cp + kTreeTop;
    uint32_t* s_st = cp + 2 * kTreeTop;
    for (uint32_t k = t; k < nk; k += kTreeThreads) {
      const uint32_t p = tl.Q[k];
      s_p[k] = p;
      s_ch[k] = tl.up[k] / (K - 1 == 0 ? kTreeChunk : kTreeChunkHi);
      cx[k] = R_x[p];
      cy[k] = R_y[p];
    }
    __syncthreads();
    if (t == 0) {
      int top = 0;
      double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
      uint32_t next_b = 0;
      for (uint32_t k = 0; k < nk; ++k) {
        const uint32_t p = s_p[k];
        const uint32_t tp = top ? s_p[s_st[top - 1]] : kNone;
        for (; next_b <= s_ch[k]; ++next_b) ll.bt[next_b] = tp;
        const double px = cx[k], py = cy[k];
        while (top >= 2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
          --top;
          s1x = s2x; s1y = s2y;
          if (top >= 2) { const uint32_t q = s_st[top - 2]; s2x = cx[q]; s2y = cy[q]; }
        }
        w.parent[p] = top ? s_p[s_st[top - 1]] : kNone;
        s_st[top++] = k;
        s2x = s1x; s2y = s1y;
        s1x = px; s1y = py;
      }
      const uint32_t tp = top ? s_p[s_st[top - 1]] : kNone;
      for (; next_b <= ll.nch; ++next_b) ll.bt[next_b] = tp;
      for (int k = 0; k < top; ++k) w.fstack[k] = s_p[s_st[k]];
      info[1] = (uint32_t)top;
    }
    __syncthreads();
  }
  if (t == 0) info[9] = (uint32_t)(clock64() - t_start);
  // ---- down: level j -> j-1, for j >= 2 (level 1 -> 0 runs on many CTAs) ----
  for (int j = K - 1; j >= 2; --j) {
    const TreeLevel& hl = L[j];
    const TreeLevel& ll = L[j - 1];
    for (uint32_t c0 = 0; c0 < ll.nch; c0 += kTreeThreads) {
      const uint32_t cq = c0 + t;
      if (cq < ll.nch) {
        const uint32_t e = ll.off[cq];
        const uint32_t c = e / kTreeChunkHi;  // level j >= 2 > 0
        const int cnt = (int)(e - c * kTreeChunkHi);
        const uint32_t* Qj = hl.Q + c * kTreeChunkHi;
        tree_stage<kTreeThreads>([&](int k) { return Qj[k]; }, cnt, R_x, R_y, cx, cy, cp);
        uint32_t b1 = hl.bt[c];
        const int top = tree_scan_run<kTreeThreads>(
            cnt, cx, cy, b1, R_x, R_y, w.parent, stk, sm.pc, [&](int k, int below, uint32_t ptop) {
              w.parent[cp[k * kTreeThreads + t]] = below >= 0 ? cp[below * kTreeThreads + t] : ptop;
            });
        ll.bt[cq] = top ? cp[stk[(top - 1) * kTreeThreads + t] * kTreeThreads + t] : b1;
      }
    }
    __syncthreads();
    if (t == 0) ll.bt[ll.nch] = hl.bt[hl.nch];
    __syncthreads();
  }
  if (t == 0) {
    // K == 1: the top-level scan already wrote the level-0 boundary states;
    // else the level-0 boundary after the last chunk is the final top
    if (K >= 2) w.btbuf[0][(N + kTreeChunk - 1) / kTreeChunk] = L[1].bt[L[1].nch];
    info[3] = K;
    info[16] = (uint32_t)(clock64() - t_start);
  }
}

// Down 1 -> 0, many CTAs: the state before every buffer chunk.
__global__ void __launch_bounds__(kTreeCta) k_gr_down0(uint32_t N, const double* __restrict__ R_x,
                                                      const double* __restrict__ R_y, TreeWork w,
                                                      const uint32_t* __restrict__ info) {
  extern __shared__ __align__(16) double tsm[];
  TreeSmem<kTreeCta> sm(tsm);
  double* cx = sm.cx;
  double* cy = sm.cy;
  uint32_t* cp = sm.cp;
  uint8_t* stk = sm.stk;
  if (info[0] || info[3] < 2) return;  // K == 1: level-0 states come from the top scan
  const uint32_t nch0 = (N + kTreeChunk - 1) / kTreeChunk;
  const uint32_t cq = blockIdx.x * kTreeCta + threadIdx.x;
  if (cq >= nch0) return;
  const uint32_t* off0 = w.offbuf[0];
  const uint32_t* bt1 = w.btbuf[1];
  const uint32_t* Q1 = w.Qbuf[1];
  const uint32_t e = off0[cq];
  const uint32_t c = e / kTreeChunkHi;  // chunks of Q_1
  const int cnt = (int)(e - c * kTreeChunkHi);
  const uint32_t* Qj = Q1 + c * kTreeChunkHi;
  const int t = threadIdx.x;
  tree_stage<kTreeCta>([&](int k) { return Qj[k]; }, cnt, R_x, R_y, cx, cy, cp);
  uint32_t b1 = bt1[c];
  const int top = tree_scan_run<kTreeCta>(cnt, cx, cy, b1, R_x, R_y, w.parent, stk, sm.pc,
                                          [&](int k, int below, uint32_t ptop) {
                                            w.parent[cp[k * kTreeCta + t]] =
                                                below >= 0 ? cp[below * kTreeCta + t] : ptop;
                                          });
  w.btbuf[0][cq] = top ? cp[stk[(top - 1) * kTreeCta + t] * kTreeCta + t] : b1;
}

// Certificate, many CTAs (thread per buffer chunk); failures counted in info[2].
__global__ void __launch_bounds__(kTreeCta) k_gr_cert(uint32_t N, const double* __restrict__ R_x,
                                                     const double* __restrict__ R_y, TreeWork w,
                                                     uint32_t* __restrict__ info,
                                                     uint32_t debug_corrupt) {
  extern __shared__ __align__(16) double tsm[];
  TreeSmem<kTreeCta> sm(tsm);
  double* cx = sm.cx;
  double* cy = sm.cy;
  uint8_t* stk = sm.stk;
  if (info[0]) return;
  const uint32_t nch0 = (N + kTreeChunk - 1) / kTreeChunk;
  const uint32_t c = blockIdx.x * kTreeCta + threadIdx.x;
  if (c >= nch0) return;
  const uint32_t* bt = w.btbuf[0];
  const uint32_t lo = c * kTreeChunk;
  const int cnt = (int)min((uint32_t)kTreeChunk, N - lo);
  tree_stage<kTreeCta>([&](int k) { return lo + (uint32_t)k; }, cnt, R_x, R_y, cx, cy, nullptr);
  uint32_t b1 = bt[c];
  const int top = tree_scan_run<kTreeCta>(cnt, cx, cy, b1, R_x, R_y, w.parent, stk, sm.pc,
                                          [](int, int, uint32_t) {});
  const uint32_t end_top = top ? lo + stk[(top - 1) * kTreeCta + threadIdx.x] : b1;
  uint32_t want = bt[c + 1];
  if (debug_corrupt && c + 1 == nch0) want = bt[c];  // falsified final state
  bool ok = want == end_top;
  // surviving pushes must link as in parent[] (loads issued 8 at a time)
  for (int k0 = 0; k0 < top && ok; k0 += 8) {
    uint32_t lk[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      lk[u] = (k0 + u < top) ? w.parent[lo + stk[(k0 + u) * kTreeCta + threadIdx.x]] : 0u;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int k = k0 + u;
      if (k < top) ok = ok && lk[u] == (k ? lo + stk[(k - 1) * kTreeCta + threadIdx.x] : b1);
    }
  }
  if (!ok) atomicAdd(&info[2], 1u);
}

// Output (one CTA): the top-level scan's final stack is the certified final
// state iff its top is the certified top and every element links to the one
// below it (checked in parallel); otherwise the certified state is walked
// down its links. Certificate failures: the exact sequential scan (one
// thread), the reference loop itself.
__global__ void __launch_bounds__(1024) k_gr_emit(uint32_t N, const double* __restrict__ R_x,
                                                  const double* __restrict__ R_y,
                                                  const uint32_t* __restrict__ R_i, TreeWork w,
                                                  const uint32_t* __restrict__ info,
                                                  uint32_t* __restrict__ out_idx,
                                                  Counters* __restrict__ ctr) {
  if (info[0]) return;
  const uint32_t t = threadIdx.x;
  if (info[2]) {
    if (t != 0) return;
    uint32_t top = 0;
    double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
    for (uint32_t i = 0; i < N; ++i) {
      const double px = R_x[i], py = R_y[i];
      while (top >= 2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
        --top;
        s1x = s2x; s1y = s2y;
        if (top >= 2) { const uint32_t q = w.tmp[top - 2]; s2x = R_x[q]; s2y = R_y[q]; }
      }
      w.tmp[top++] = i;
      s2x = s1x; s2y = s1y;
      s1x = px; s1y = py;
    }
    for (uint32_t k = 0; k < top; ++k) out_idx[k] = R_i[w.tmp[k]];
    ctr->hull = top;
    return;
  }
  const uint32_t nch0 = (N + kTreeChunk - 1) / kTreeChunk;
  const uint32_t len = info[1], ftop = w.btbuf[0][nch0];
  bool ok = len > 0 && w.fstack[len - 1] == ftop;
  for (uint32_t k = t; k < len && ok; k += blockDim.x)
    ok = w.parent[w.fstack[k]] == (k ? w.fstack[k - 1] : kNone);
  if (__syncthreads_and(ok)) {
    for (uint32_t k = t; k < len; k += blockDim.x) out_idx[k] = R_i[w.fstack[k]];
    if (t == 0) ctr->hull = len;
    return;
  }
  if (t != 0) return;
  uint32_t h = 0;
  for (uint32_t p = ftop; p != kNone; p = w.parent[p]) w.tmp[h++] = p;
  for (uint32_t k = 0; k < h; ++k) out_idx[k] = R_i[w.tmp[h - 1 - k]];
  ctr->hull = h;
}

}  // namespace gscan
