// K7/K8 tree strategy: graham_finalize (pipeline.hpp:57-67) for buffers where
// most points are popped (round-2 output of squares and disks).
//
// Warp-speculative scans advance 32 points per iteration only while nothing is
// popped; on these buffers nearly every point pops, so here every scan is a
// plain sequential stack scan run by ONE thread, and the parallelism comes
// from running many short ones:
//
//   up      level j: Q_j (R positions + coordinates; Q_0 = the buffer) is cut
//           into chunks of kTreeChunk; every chunk's scan from an empty stack
//           leaves a chain; the chains concatenated form Q_{j+1}. Repeat until
//           Q_K is small.
//   top     one thread scans Q_K, recording the persistent stack (parent[p] =
//           the element below p when p was pushed) and the state before every
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
//
// Stack representation inside one scan: shared-memory rows [0, top) of the
// thread's column (coordinates, R position, chunk index), on top of a chain in
// global memory that starts at B (the element below row 0) and continues
// through parent[]. A state handed between levels is a boundary record: its
// top kTreePC rows (bottom-aligned) and the element below them. The chunk's
// own points are staged in rows kTreePC.. and pushes overwrite rows in place
// (a push lands at row <= kTreePC + k, never above the next unread point), so
// the common pop and push are one shared-memory access each.
#pragma once
#include "graham.cuh"

namespace gscan {

#ifndef GSCAN_TREE_CS1
#define GSCAN_TREE_CS1 32
#endif
#ifndef GSCAN_TREE_CS_HI
#define GSCAN_TREE_CS_HI 32
#endif
constexpr int kTreeChunk0 = 16;     // level 0 (the buffer): the widest level and the certificate
constexpr int kTreeChunk = GSCAN_TREE_CS1;     // level 1 (many CTAs)
constexpr int kTreeChunkHi = GSCAN_TREE_CS_HI;  // levels >= 2 (one CTA)
__host__ __device__ constexpr uint32_t tree_cs(int j) {
  return j == 0 ? kTreeChunk0 : (j == 1 ? kTreeChunk : kTreeChunkHi);
}
constexpr int kTreeThreads = 256;   // the middle CTA; chunks are processed in waves of this many
constexpr uint32_t kTreeTop = 128;       // levels stop shrinking once this small
constexpr uint32_t kTreeTopMax = 3072;   // largest top level (a level that stops
                                         // shrinking is mostly final-hull vertices)
constexpr int kTreeMaxLevels = 24;
constexpr int kTreePC = 8;          // stack rows carried in a boundary record
constexpr int kTreeRows = kTreePC + (kTreeChunk > kTreeChunkHi ? kTreeChunk : kTreeChunkHi);
constexpr uint32_t kTreeHiCap = 1u << 18;  // level >= 1 capacity (larger: another strategy)
constexpr uint8_t kTreeRec = 0xff;  // chunk index of a row loaded from a record
constexpr int kTreeInfoWords = 48;  // info[] words (cleared by k_gr_setup, read back by the host)

// shared memory: per thread kTreeRows rows of (x, y, position, chunk index)
constexpr size_t tree_smem(int threads) { return (size_t)kTreeRows * threads * (8 + 8 + 4 + 1); }
constexpr size_t kTreeSmem = tree_smem(kTreeThreads);

// Boundary records of one level: the state before each chunk.
struct TreeRec {
  uint32_t* n;      // rows recorded (<= kTreePC)
  uint32_t* below;  // element below the recorded rows (kNone: none)
  uint32_t* pos;    // [c * kTreePC + d], d = 0 the deepest recorded row
  double* x;
  double* y;
};

struct TreeLevel {
  uint32_t* Qp;  // R positions (level >= 1)
  double* Qx;
  double* Qy;
  uint32_t* up;   // Q_{j-1} index of each element (level >= 1)
  uint32_t* off;  // chain offsets of this level's chunks in Q_{j+1} (nch + 1)
  uint32_t* bt;   // top before each chunk (nch + 1)
  TreeRec rec;
  uint32_t nq, nch;
  uint32_t cs;  // chunk length
};

// Workspace carved from one device buffer by the host; the kernel checks every
// level size against its capacity.
struct TreeWork {
  uint32_t* parent;  // N
  uint32_t* tmp;     // N (fallback stack; top-scan boundary tops)
  uint32_t* chainq;  // N: chain elements of the current level (Q index), chunk-strided
  uint32_t* chainp;  // N: their R positions
  double* chainx;    // N: their coordinates
  double* chainy;
  uint32_t* fstack;  // kTreeTopMax
  uint32_t* Qp[kTreeMaxLevels + 1];
  double* Qx[kTreeMaxLevels + 1];
  double* Qy[kTreeMaxLevels + 1];
  uint32_t* up[kTreeMaxLevels + 1];
  uint32_t* off[kTreeMaxLevels + 1];
  uint32_t* bt[kTreeMaxLevels + 1];
  TreeRec rec[kTreeMaxLevels + 1];
  uint32_t cap[kTreeMaxLevels + 1];  // element capacity of level j
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

// The thread's rows, [row][thread] so any mix of rows across a warp is
// bank-conflict free.
template <int T>
struct TreeRows {
  double* X;
  double* Y;
  uint32_t* P;
  uint8_t* K;
  __device__ explicit TreeRows(double* base) {
    X = base;
    Y = X + kTreeRows * T;
    P = reinterpret_cast<uint32_t*>(Y + kTreeRows * T);
    K = reinterpret_cast<uint8_t*>(P + kTreeRows * T);
  }
  __device__ __forceinline__ int at(int row) const { return row * T + (int)threadIdx.x; }
};

// Stage run elements [base, base + cnt) into rows kTreePC + k (16 loads in
// flight). qp == nullptr: positions are base + k (level 0).
template <int T>
__device__ __forceinline__ void tree_stage(const TreeRows<T>& r, const uint32_t* __restrict__ qp,
                                           const double* __restrict__ qx,
                                           const double* __restrict__ qy, uint32_t base, int cnt) {
  for (int k0 = 0; k0 < cnt; k0 += 16) {
    double vx[16], vy[16];
    uint32_t vp[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const bool in = k0 + u < cnt;
      vx[u] = in ? qx[base + k0 + u] : 0.0;
      vy[u] = in ? qy[base + k0 + u] : 0.0;
      vp[u] = in ? (qp ? qp[base + k0 + u] : base + k0 + u) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (k0 + u < cnt) {
        const int a = r.at(kTreePC + k0 + u);
        r.X[a] = vx[u];
        r.Y[a] = vy[u];
        r.P[a] = vp[u];
        r.K[a] = (uint8_t)(k0 + u);
      }
  }
}

// Rows [0, n) from boundary record c; returns n, sets B.
template <int T>
__device__ __forceinline__ int tree_load_rec(const TreeRows<T>& r, const TreeRec& rec, uint32_t c,
                                             uint32_t& B) {
  const int n = (int)rec.n[c];
  B = rec.below[c];
  uint32_t vp[kTreePC];
  double vx[kTreePC], vy[kTreePC];
#pragma unroll
  for (int d = 0; d < kTreePC; ++d) {
    vp[d] = rec.pos[(size_t)c * kTreePC + d];
    vx[d] = rec.x[(size_t)c * kTreePC + d];
    vy[d] = rec.y[(size_t)c * kTreePC + d];
  }
#pragma unroll
  for (int d = 0; d < kTreePC; ++d)
    if (d < n) {
      const int a = r.at(d);
      r.X[a] = vx[d];
      r.Y[a] = vy[d];
      r.P[a] = vp[d];
      r.K[a] = kTreeRec;
    }
  return n;
}

// Boundary record c from the stack rows [0, top) above B.
template <int T>
__device__ __forceinline__ void tree_store_rec(const TreeRows<T>& r, int top, uint32_t B,
                                               const TreeRec& rec, uint32_t c) {
  const int n = min(top, kTreePC), r0 = top - n;
  rec.n[c] = (uint32_t)n;
  rec.below[c] = r0 > 0 ? r.P[r.at(r0 - 1)] : B;
  for (int d = 0; d < n; ++d) {
    const int a = r.at(r0 + d);
    rec.pos[(size_t)c * kTreePC + d] = r.P[a];
    rec.x[(size_t)c * kTreePC + d] = r.X[a];
    rec.y[(size_t)c * kTreePC + d] = r.Y[a];
  }
}

// One thread's stack scan over the staged points (rows kTreePC + k, k < cnt)
// on top of rows [0, top) and the chain below B. Every iteration is one pop
// or one push (a warp of divergent scans costs max over lanes of pushes +
// pops). on_push(k, position, below position) is called for every push.
// lo_own ends at the lowest row holding a surviving push of this scan.
// Returns the final top; B is updated when the scan pops below row 0.
template <int T, typename OnPush>
__device__ __forceinline__ int tree_scan_rows(const TreeRows<T>& r, int top, uint32_t& B, int cnt,
                                              const uint32_t* __restrict__ parent,
                                              const double* __restrict__ R_x,
                                              const double* __restrict__ R_y, int& lo_own,
                                              OnPush&& on_push) {
  double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
  bool h1, h2;
  uint32_t q2 = kNone;  // position of s2 while it is B or below (top <= 1)
  if (top >= 2) {
    s1x = r.X[r.at(top - 1)]; s1y = r.Y[r.at(top - 1)];
    s2x = r.X[r.at(top - 2)]; s2y = r.Y[r.at(top - 2)];
    h1 = h2 = true;
  } else if (top == 1) {
    s1x = r.X[r.at(0)]; s1y = r.Y[r.at(0)];
    h1 = true;
    h2 = B != kNone;
    q2 = B;
    if (h2) { s2x = R_x[B]; s2y = R_y[B]; }
  } else {
    h1 = B != kNone;
    h2 = false;
    if (h1) {
      s1x = R_x[B]; s1y = R_y[B];
      q2 = parent[B];
      h2 = q2 != kNone;
      if (h2) { s2x = R_x[q2]; s2y = R_y[q2]; }
    }
  }
  int k = 0;
  double px = 0, py = 0;
  if (cnt > 0) { px = r.X[r.at(kTreePC)]; py = r.Y[r.at(kTreePC)]; }
  // One loop shape for pops and pushes (the lanes of a warp pop and push
  // independently; separate paths cost a warp both of them per iteration).
  // Both candidates for the step's one new value -- the new second element
  // of a pop (row top - 3) and the next staged point of a push (row kTreePC
  // + k + 1) -- are loaded before the turn test, so their latency overlaps
  // it. Pops that reach B or the chain below it take the branch with the
  // global loads.
  while (k < cnt) {
    const int a3 = r.at(max(top - 3, 0));
    const int an = r.at(min(kTreePC + k + 1, kTreeRows - 1));
    const double l3x = r.X[a3], l3y = r.Y[a3];
    const double lnx = r.X[an], lny = r.Y[an];
    const bool pop = h2 && !left_turn(s2x, s2y, s1x, s1y, px, py);
    if (pop && top < 3 && (top != 2 || B != kNone)) {
      s1x = s2x; s1y = s2y;
      if (top == 2) {  // new s1 = row 0, s2 = B
        top = 1;
        q2 = B;
        h2 = true;
        s2x = R_x[B]; s2y = R_y[B];
      } else if (top == 1) {  // new s1 = B, s2 = parent[B]
        top = 0;
        q2 = parent[B];
        h2 = q2 != kNone;
        if (h2) { s2x = R_x[q2]; s2y = R_y[q2]; }
      } else {  // pop B itself
        B = q2;
        q2 = parent[B];
        h2 = q2 != kNone;
        if (h2) { s2x = R_x[q2]; s2y = R_y[q2]; }
      }
      continue;
    }
    if (!pop) {  // push p onto row top (<= kTreePC + k: the rows loaded above stay intact)
      const int a = r.at(top);
      const uint32_t pp = r.P[r.at(kTreePC + k)];
      on_push(k, pp, top >= 1 ? r.P[r.at(top - 1)] : B);
      r.X[a] = px;
      r.Y[a] = py;
      r.P[a] = pp;
      r.K[a] = (uint8_t)k;
      if (top < lo_own) lo_own = top;
    }
    if (pop) {  // the new second element: row top - 3 (none when top == 2: B is kNone)
      h2 = top >= 3;
      --top;
      s1x = s2x; s1y = s2y;
      s2x = l3x; s2y = l3y;
    } else {
      ++top;
      s2x = s1x; s2y = s1y;
      h2 = h1;
      s1x = px; s1y = py;
      h1 = true;
      ++k;
      px = lnx; py = lny;
    }
    if (top == 1) q2 = B;
  }
  return top;
}

struct TreeNoPush {
  __device__ __forceinline__ void operator()(int, uint32_t, uint32_t) const {}
};

// Chain of a scan from an empty stack: rows [0, top) -> chunk-strided temp
// (Q index = lo + chunk index, or the position on level 0).
template <int T>
__device__ __forceinline__ void tree_put_chain(const TreeRows<T>& r, int top, uint32_t lo,
                                               bool level0, const TreeWork& w) {
  for (int i = 0; i < top; ++i) {
    const int a = r.at(i);
    const uint32_t p = r.P[a];
    w.chainq[lo + i] = level0 ? p : lo + r.K[a];
    w.chainp[lo + i] = p;
    w.chainx[lo + i] = r.X[a];
    w.chainy[lo + i] = r.Y[a];
  }
}

// ---------------------------------------------------------------------------
// info[] layout (device, read back once by the host):
//   [0] declined (another strategy, or the sparse path failed)  [1] final
//   stack length  [2] certificate failures  [3] K  [4] N (buffer size, set
//   by k_gr_setup from the host or from the sparse path's device state)
//   [8..9, 16] diagnostics clocks  [10 + j] size of Q_j  [20..43] diagnostics
// Every kernel reads N from info[4], so the whole strategy can be enqueued
// before N is known on the host (inside the sparse path's CUDA graph); the
// many-CTA kernels loop grid-stride over chunks.
constexpr int kTreeCta = 64;
constexpr size_t kTreeCtaSmem = tree_smem(kTreeCta);

__device__ __forceinline__ TreeLevel tree_level(const TreeWork& w, int j, uint32_t nq) {
  TreeLevel L;
  L.Qp = w.Qp[j];
  L.Qx = w.Qx[j];
  L.Qy = w.Qy[j];
  L.up = w.up[j];
  L.off = w.off[j];
  L.bt = w.bt[j];
  L.rec = w.rec[j];
  L.nq = nq;
  L.cs = tree_cs(j);
  L.nch = (nq + L.cs - 1) / L.cs;
  return L;
}

__device__ __forceinline__ uint32_t tree_nq(const uint32_t* info, int j) {
  return j == 0 ? info[4] : info[10 + j];
}

// Setup: info[] cleared, N = *n_dev (sparse path: its round-2 size) or
// n_host; declined when `st_fail` (the sparse path failed) is set, when
// disabled, or when N exceeds the workspace.
__global__ void k_gr_setup(const uint32_t* __restrict__ n_dev, uint32_t n_host,
                           const uint32_t* __restrict__ st_fail, uint32_t n_max, uint32_t disable,
                           uint32_t* __restrict__ info) {
  pdl_wait();
  const uint32_t t = threadIdx.x;
  if (t < kTreeInfoWords && t != 4 && t != 0) info[t] = 0;
  if (t == 0) {
    const uint32_t N = n_dev ? *n_dev : n_host;
    info[4] = N;
    info[0] = (disable || (st_fail && *st_fail) || N == 0 || N > n_max) ? 1u : 0u;
  }
}

// Up, many CTAs (levels 0 and 1): chains of level j's chunks (thread per
// chunk) into the chunk-strided temp, lengths into off[j].
__global__ void __launch_bounds__(kTreeCta) k_gr_up(int j, const double* __restrict__ R_x,
                                                   const double* __restrict__ R_y, TreeWork w,
                                                   const uint32_t* __restrict__ info) {
  pdl_wait();
  extern __shared__ __align__(16) double tsm[];
  const TreeRows<kTreeCta> r(tsm);
  if (info[0]) return;
  const uint32_t nq = tree_nq(info, j);
  const uint32_t cs = tree_cs(j);
  for (uint32_t c = blockIdx.x * kTreeCta + threadIdx.x; c * cs < nq; c += gridDim.x * kTreeCta) {
    const uint32_t lo = c * cs;
    const int cnt = (int)min(cs, nq - lo);
    if (j == 0) tree_stage<kTreeCta>(r, nullptr, R_x, R_y, lo, cnt);
    else tree_stage<kTreeCta>(r, w.Qp[j], w.Qx[j], w.Qy[j], lo, cnt);
    uint32_t B = kNone;
    int lo_own = kTreeRows;
    const int top =
        tree_scan_rows<kTreeCta>(r, 0, B, cnt, w.parent, R_x, R_y, lo_own, TreeNoPush{});
    tree_put_chain<kTreeCta>(r, top, lo, j == 0, w);
    w.off[j][c] = (uint32_t)top;
  }
}

// Exclusive scan of level j's chain lengths (one CTA), Q_{j+1}'s size, and
// the shrink check (info[0]: the tree strategy declines).
__global__ void __launch_bounds__(1024) k_gr_scan(int j, TreeWork w, uint32_t* __restrict__ info) {
  pdl_wait();
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  if (info[0]) return;
  const uint32_t nq = tree_nq(info, j);
  const uint32_t nch = (nq + tree_cs(j) - 1) / tree_cs(j);
  const uint32_t total = tree_scan(w.off[j], nch, s_w, &s_carry);
  if (threadIdx.x == 0) {
    w.off[j][nch] = total;
    const bool shrink =
        (j == 0) ? (total * 20ull <= (uint64_t)nq * 17) : (total * 10ull <= (uint64_t)nq * 9);
    // a stalled level is the top level if the warp top scan can take it
    // (k_gr_mid decides); level 0 must shrink (else the buffer is in convex
    // position and the junction strategy is the right one)
    if ((!shrink && (j == 0 || total > kTreeTopMax)) || total > w.cap[j + 1]) info[0] = 1;
    info[11 + j] = total;
  }
}

// Level j chains -> Q_{j+1} (up index, position, coordinates): a warp per
// chunk, lanes over the chain, so loads and stores are coalesced.
__device__ __forceinline__ void tree_gather_chunk(const TreeWork& w, int j, uint32_t c) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t o = w.off[j][c], ln = w.off[j][c + 1] - o;
  const uint32_t s = c * tree_cs(j) + lane;
  if (lane < ln) {
    const uint32_t q = w.chainq[s], p = w.chainp[s];
    const double x = w.chainx[s], y = w.chainy[s];
    w.up[j + 1][o + lane] = q;
    w.Qp[j + 1][o + lane] = p;
    w.Qx[j + 1][o + lane] = x;
    w.Qy[j + 1][o + lane] = y;
  }
}

__global__ void __launch_bounds__(256) k_gr_gather(int j, TreeWork w,
                                                  const uint32_t* __restrict__ info) {
  pdl_wait();
  if (info[0]) return;
  const uint32_t nch = (tree_nq(info, j) + tree_cs(j) - 1) / tree_cs(j);
  for (uint32_t c = blockIdx.x * 8 + (threadIdx.x >> 5); c < nch; c += gridDim.x * 8)
    tree_gather_chunk(w, j, c);
}

// One down step for lower chunk cq: the state before it is the state before
// the upper chunk holding its chain's first element, scanned over the upper
// elements in between; pushes write parent[]. Writes the lower top + record.
template <int T>
__device__ __forceinline__ void tree_down_one(const TreeRows<T>& r, const TreeLevel& hl,
                                              const TreeLevel& ll, uint32_t cq,
                                              const double* __restrict__ R_x,
                                              const double* __restrict__ R_y, uint32_t* parent) {
  const uint32_t e = ll.off[cq];
  const uint32_t c = e / hl.cs;
  const int cnt = (int)(e - c * hl.cs);
  tree_stage<T>(r, hl.Qp, hl.Qx, hl.Qy, c * hl.cs, cnt);
  uint32_t B;
  const int n0 = tree_load_rec<T>(r, hl.rec, c, B);
  int lo_own = kTreeRows;
  const int top = tree_scan_rows<T>(r, n0, B, cnt, parent, R_x, R_y, lo_own,
                                    [&](int, uint32_t p, uint32_t below) { parent[p] = below; });
  ll.bt[cq] = top ? r.P[r.at(top - 1)] : B;
  tree_store_rec<T>(r, top, B, ll.rec, cq);
}

// Middle, ONE CTA: levels >= 2 up (Q_1 and Q_2 come from the many-CTA
// kernels), the top-level scan, and the down-sweep to level 2.
__global__ void __launch_bounds__(kTreeThreads, 1) k_gr_mid(
    const double* __restrict__ R_x, const double* __restrict__ R_y, TreeWork w,
    uint32_t* __restrict__ info) {
  pdl_wait();
  extern __shared__ __align__(16) double tsm[];
  const TreeRows<kTreeThreads> r(tsm);
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  __shared__ uint32_t s_nq[kTreeMaxLevels + 1];
  __shared__ int s_K, s_bad;
  const int t = threadIdx.x;
  long long t_start = clock64();
  if (info[0]) return;  // declined, or level 0 or 1 did not shrink
#ifdef GSCAN_TREE_PRINT
  __shared__ long long s_clk[64];
#endif
  if (t == 0) {
    s_nq[0] = info[4];
    s_nq[1] = info[11];
    s_nq[2] = info[12];
    // top level: small enough, or the first level that stops shrinking
    const bool stall2 = (uint64_t)s_nq[2] * 10 > (uint64_t)s_nq[1] * 9;
    s_K = s_nq[1] <= kTreeTop ? 1 : ((s_nq[2] <= kTreeTop || stall2) ? 2 : -1);
    s_bad = s_K == 2 && s_nq[2] > kTreeTopMax;
  }
  __syncthreads();
  if (s_bad) {
    if (t == 0) { info[0] = 1; info[3] = 0; }
    return;
  }
  for (int j = 2; s_K < 0 && j < kTreeMaxLevels; ++j) {
    const TreeLevel L = tree_level(w, j, s_nq[j]);
    for (uint32_t c0 = 0; c0 < L.nch; c0 += kTreeThreads) {
      const uint32_t c = c0 + t;
      if (c < L.nch) {
        const uint32_t lo = c * L.cs;
        const int cnt = (int)min(L.cs, L.nq - lo);
#ifdef GSCAN_TREE_PRINT
        if (t == 0) s_clk[j * 8 + 0] = clock64() - t_start;
#endif
        tree_stage<kTreeThreads>(r, L.Qp, L.Qx, L.Qy, lo, cnt);
#ifdef GSCAN_TREE_PRINT
        if (t == 0) s_clk[j * 8 + 1] = clock64() - t_start;
#endif
        uint32_t B = kNone;
        int lo_own = kTreeRows;
        const int top = tree_scan_rows<kTreeThreads>(r, 0, B, cnt, w.parent, R_x, R_y, lo_own,
                                                     TreeNoPush{});
#ifdef GSCAN_TREE_PRINT
        if (t == 0) s_clk[j * 8 + 2] = clock64() - t_start;
#endif
        tree_put_chain<kTreeThreads>(r, top, lo, false, w);
        L.off[c] = (uint32_t)top;
#ifdef GSCAN_TREE_PRINT
        if (t == 0) s_clk[j * 8 + 3] = clock64() - t_start;
#endif
      }
    }
    __syncthreads();
#ifdef GSCAN_TREE_PRINT
    if (t == 0) s_clk[j * 8 + 4] = clock64() - t_start;
#endif
    const uint32_t total = tree_scan(L.off, L.nch, s_w, &s_carry);
    if (t == 0) {
      L.off[L.nch] = total;
      const bool stall = total * 10ull > (uint64_t)L.nq * 9;
      if ((stall && total > kTreeTopMax) || total > w.cap[j + 1] || j + 1 > kTreeMaxLevels - 1)
        s_bad = 1;
      s_nq[j + 1] = total;
      if (stall) s_K = j + 1;  // the top level (before the s_K assignment below)
      if (j + 1 < 6) info[10 + j + 1] = total;  // diagnostics
    }
    __syncthreads();
    if (s_bad) break;
#ifdef GSCAN_TREE_PRINT
    if (t == 0) s_clk[j * 8 + 5] = clock64() - t_start;
#endif
    for (uint32_t c = t >> 5; c < L.nch; c += kTreeThreads / 32) tree_gather_chunk(w, j, c);
    __syncthreads();
    if (t == 0) {
      if (j < 12) info[20 + j] = (uint32_t)(clock64() - t_start);  // diagnostics
      if (s_nq[j + 1] <= kTreeTop) s_K = j + 1;
    }
    __syncthreads();
  }
  const int K = s_K;
  if (s_bad || K < 1) {  // no shrink: the host takes another strategy
    if (t == 0) { info[0] = 1; info[3] = 0; }
    return;
  }
  if (t == 0) {
    info[8] = (uint32_t)(clock64() - t_start);
    for (int j = 3; j <= K && j < 6; ++j) info[10 + j] = s_nq[j];
  }
  // ---- top: warp 0 scans Q_K (<= kTreeTopMax, staged in shared memory),
  // 32 points per iteration while nothing pops (the scan of k_graham_local);
  // it records below(k), the element each point is pushed onto. The state
  // before a Q_{K-1} boundary is "top = the previous element", so all threads
  // then turn below() into parent[], boundary tops and records. ----
  {
    const TreeLevel tl = tree_level(w, K, s_nq[K]);
    const TreeLevel ll = tree_level(w, K - 1, s_nq[K - 1]);
    const uint32_t nk = tl.nq;
    double* s_x = r.X;                        // [kTreeTopMax]
    double* s_y = r.Y;
    double* st_x = r.X + kTreeTopMax;         // the stack
    double* st_y = r.Y + kTreeTopMax;
    uint32_t* s_p = r.P;                      // R position of each Q_K element
    uint32_t* s_par = r.P + kTreeTopMax;      // below(k) as a Q_K index (kNone: none)
    uint32_t* st_i = r.P + 2 * kTreeTopMax;   // the stack (Q_K indices)
    uint32_t* bk = w.tmp;                     // Q_K index of the top before each boundary
    for (uint32_t k = t; k < nk; k += kTreeThreads) {
      s_p[k] = tl.Qp[k];
      s_x[k] = tl.Qx[k];
      s_y[k] = tl.Qy[k];
    }
    __syncthreads();
    if (nk <= kTreeTop && t == 0) {  // small (pop-heavy) top level: one thread is faster
      int top = 0;
      double s1x = 0, s1y = 0, s2x = 0, s2y = 0;
      for (uint32_t k = 0; k < nk; ++k) {
        const double px = s_x[k], py = s_y[k];
        while (top >= 2 && !left_turn(s2x, s2y, s1x, s1y, px, py)) {
          --top;
          s1x = s2x; s1y = s2y;
          if (top >= 2) { s2x = st_x[top - 2]; s2y = st_y[top - 2]; }
        }
        s_par[k] = top ? st_i[top - 1] : kNone;
        st_x[top] = px;
        st_y[top] = py;
        st_i[top++] = k;
        s2x = s1x; s2y = s1y;
        s1x = px; s1y = py;
      }
      for (int k = 0; k < top; ++k) w.fstack[k] = s_p[st_i[k]];
      info[1] = (uint32_t)top;
      const uint32_t ftop = top ? s_p[st_i[top - 1]] : kNone;
      for (int j = 0; j < K; ++j) w.bt[j][(s_nq[j] + tree_cs(j) - 1) / tree_cs(j)] = ftop;
    }
    if (nk > kTreeTop && t < 32) {
      const int lane = t;
      int top = 0;
      int i = 0;
      while (i < (int)nk) {
        const int j = i + lane;
        const bool valid = j < (int)nk;
        const double px = valid ? s_x[j] : 0.0, py = valid ? s_y[j] : 0.0;
        const int depth = top + lane;  // stack size before pushing j if all earlier lanes pushed
        bool ok = true;
        if (valid && depth >= 2) {
          double ax, ay, bx, by;
          if (lane >= 2) { ax = s_x[j - 2]; ay = s_y[j - 2]; bx = s_x[j - 1]; by = s_y[j - 1]; }
          else if (lane == 1) { ax = st_x[top - 1]; ay = st_y[top - 1]; bx = s_x[j - 1]; by = s_y[j - 1]; }
          else { ax = st_x[top - 2]; ay = st_y[top - 2]; bx = st_x[top - 1]; by = st_y[top - 1]; }
          ok = left_turn(ax, ay, bx, by, px, py);
        }
        const uint32_t fm = __ballot_sync(0xffffffffu, valid && !ok);
        const int nvalid = min(32, (int)nk - i);
        const int f = fm ? (__ffs(fm) - 1) : 32;
        const int commit = min(f, nvalid);
        if (lane < commit) {
          st_x[top + lane] = px;
          st_y[top + lane] = py;
          st_i[top + lane] = (uint32_t)j;
          s_par[j] = lane ? (uint32_t)(j - 1) : (top ? st_i[top - 1] : kNone);
        }
        top += commit;
        __syncwarp();
        if (f < nvalid) {
          const double fx = __shfl_sync(0xffffffffu, px, f), fy = __shfl_sync(0xffffffffu, py, f);
          int newtop;
          int dhi = top - 1;
          while (true) {
            const int d = dhi - lane;
            const bool l = d >= 1 && left_turn(st_x[d - 1], st_y[d - 1], st_x[d], st_y[d], fx, fy);
            const uint32_t m = __ballot_sync(0xffffffffu, l);
            if (m) { newtop = dhi - (__ffs(m) - 1) + 1; break; }
            if (dhi - 31 <= 1) { newtop = min(top, 1); break; }
            dhi -= 32;
          }
          __syncwarp();  // every lane's stack reads happen before lane 0 overwrites the top
          if (lane == 0) {
            st_x[newtop] = fx;
            st_y[newtop] = fy;
            st_i[newtop] = (uint32_t)(i + f);
            s_par[i + f] = newtop ? st_i[newtop - 1] : kNone;
          }
          top = newtop + 1;
          i += f + 1;
        } else {
          i += nvalid;
        }
        __syncwarp();
      }
      for (int k = lane; k < top; k += 32) w.fstack[k] = s_p[st_i[k]];
      if (lane == 0) {
        info[1] = (uint32_t)top;
        // every level's boundary after its last chunk holds the final top
        const uint32_t ftop = top ? s_p[st_i[top - 1]] : kNone;
        for (int j = 0; j < K; ++j) w.bt[j][(s_nq[j] + tree_cs(j) - 1) / tree_cs(j)] = ftop;
      }
    }
    __syncthreads();
    for (uint32_t k = t; k < nk; k += kTreeThreads) {
      const uint32_t below = s_par[k];
      w.parent[s_p[k]] = below != kNone ? s_p[below] : kNone;
      // boundaries b in (chunk(k - 1), chunk(k)] start at element k
      const uint32_t ch = tl.up[k] / tree_cs(K - 1);
      const uint32_t b0 = k ? tl.up[k - 1] / tree_cs(K - 1) + 1 : 0;
      for (uint32_t b = b0; b <= ch; ++b) bk[b] = k ? k - 1 : kNone;
      if (k + 1 == nk)
        for (uint32_t b = ch + 1; b <= ll.nch; ++b) bk[b] = k;
    }
    if (nk == 0)
      for (uint32_t b = t; b <= ll.nch; b += kTreeThreads) bk[b] = kNone;
    __syncthreads();
    for (uint32_t b = t; b < ll.nch; b += kTreeThreads) {
      uint32_t e[kTreePC];
      uint32_t q = bk[b];
      int n = 0;
      for (; n < kTreePC && q != kNone; ++n) { e[n] = q; q = s_par[q]; }
      ll.bt[b] = n ? s_p[e[0]] : kNone;
      ll.rec.n[b] = (uint32_t)n;
      ll.rec.below[b] = q != kNone ? s_p[q] : kNone;
      for (int d = 0; d < n; ++d) {  // bottom-aligned: d = 0 deepest
        const uint32_t qq = e[n - 1 - d];
        ll.rec.pos[(size_t)b * kTreePC + d] = s_p[qq];
        ll.rec.x[(size_t)b * kTreePC + d] = s_x[qq];
        ll.rec.y[(size_t)b * kTreePC + d] = s_y[qq];
      }
    }
    __syncthreads();
  }
  if (t == 0) info[9] = (uint32_t)(clock64() - t_start);
  // ---- down: level j -> j-1 for j >= 3 (2 -> 1 and 1 -> 0 run on many CTAs) ----
  for (int j = K - 1; j >= 3; --j) {
    const TreeLevel hl = tree_level(w, j, s_nq[j]);
    const TreeLevel ll = tree_level(w, j - 1, s_nq[j - 1]);
    for (uint32_t c0 = 0; c0 < ll.nch; c0 += kTreeThreads) {
      const uint32_t cq = c0 + t;
      if (cq < ll.nch) tree_down_one<kTreeThreads>(r, hl, ll, cq, R_x, R_y, w.parent);
    }
    __syncthreads();
    if (t == 0 && j < 12) info[32 + j] = (uint32_t)(clock64() - t_start);  // diagnostics
  }
  if (t == 0) {
    info[3] = K;
    info[16] = (uint32_t)(clock64() - t_start);
#ifdef GSCAN_TREE_PRINT
    for (int j = 2; j < 4; ++j) printf("lvl %d: stage %lld-%lld scan -%lld put -%lld | all chunks %lld | offs scan %lld | next level %u\n", j, s_clk[j*8], s_clk[j*8+1], s_clk[j*8+2], s_clk[j*8+3], s_clk[j*8+4], s_clk[j*8+5], info[20 + j]);
    printf("mid K=%d nq %u %u %u %u %u %u | up2 %u up3 %u up4 %u | upend %u top %u | down %u %u %u | end %u\n", K,
           s_nq[0], s_nq[1], s_nq[2], s_nq[3], s_nq[4], s_nq[5], info[22], info[23], info[24], info[8], info[9],
           info[35], info[34], info[33], info[16]);
#endif
  }
}

// Down j -> j-1 (j = 2, 1), many CTAs: the state before every level j-1
// chunk. Runs when the top level is above j - 1.
__global__ void __launch_bounds__(kTreeCta) k_gr_down(int j, const double* __restrict__ R_x,
                                                     const double* __restrict__ R_y, TreeWork w,
                                                     const uint32_t* __restrict__ info) {
  pdl_wait();
  extern __shared__ __align__(16) double tsm[];
  const TreeRows<kTreeCta> r(tsm);
  if (info[0] || (int)info[3] <= j) return;
  const TreeLevel hl = tree_level(w, j, tree_nq(info, j));
  const TreeLevel ll = tree_level(w, j - 1, tree_nq(info, j - 1));
  for (uint32_t cq = blockIdx.x * kTreeCta + threadIdx.x; cq < ll.nch; cq += gridDim.x * kTreeCta)
    tree_down_one<kTreeCta>(r, hl, ll, cq, R_x, R_y, w.parent);
}

// Certificate, many CTAs (thread per buffer chunk); failures counted in info[2].
__global__ void __launch_bounds__(kTreeCta) k_gr_cert(const double* __restrict__ R_x,
                                                     const double* __restrict__ R_y, TreeWork w,
                                                     uint32_t* __restrict__ info,
                                                     uint32_t debug_corrupt) {
  pdl_wait();
  extern __shared__ __align__(16) double tsm[];
  const TreeRows<kTreeCta> r(tsm);
  if (info[0]) return;
  const uint32_t N = info[4];
  const uint32_t nch0 = (N + kTreeChunk0 - 1) / kTreeChunk0;
  const uint32_t* bt = w.bt[0];
  uint32_t fails = 0;
  for (uint32_t c = blockIdx.x * kTreeCta + threadIdx.x; c < nch0; c += gridDim.x * kTreeCta) {
    const uint32_t lo = c * kTreeChunk0;
    const int cnt = (int)min((uint32_t)kTreeChunk0, N - lo);
    tree_stage<kTreeCta>(r, nullptr, R_x, R_y, lo, cnt);
    uint32_t B;
    const int n0 = tree_load_rec<kTreeCta>(r, w.rec[0], c, B);
    int lo_own = kTreeRows;
    const int top =
        tree_scan_rows<kTreeCta>(r, n0, B, cnt, w.parent, R_x, R_y, lo_own, TreeNoPush{});
    const uint32_t end_top = top ? r.P[r.at(top - 1)] : B;
    uint32_t want = bt[c + 1];
    if (debug_corrupt && c + 1 == nch0) want = bt[c];  // falsified final state
    bool ok = want == end_top;
    // surviving pushes must link as in parent[] (loads issued 8 at a time)
    for (int k0 = lo_own; k0 < top && ok; k0 += 8) {
      uint32_t lk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) lk[u] = (k0 + u < top) ? w.parent[r.P[r.at(k0 + u)]] : 0u;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = k0 + u;
        if (k < top) ok = ok && lk[u] == (k ? r.P[r.at(k - 1)] : B);
      }
    }
    fails += ok ? 0u : 1u;
  }
  if (fails) atomicAdd(&info[2], fails);
}

// Output (one CTA): the top-level scan's final stack is the certified final
// state iff its top is the certified top and every element links to the one
// below it (checked in parallel); otherwise the certified state is walked
// down its links. Certificate failures: the exact sequential scan (one
// thread), the reference loop itself.
__global__ void __launch_bounds__(1024) k_gr_emit(const double* __restrict__ R_x,
                                                  const double* __restrict__ R_y,
                                                  const uint32_t* __restrict__ R_i, TreeWork w,
                                                  const uint32_t* __restrict__ info,
                                                  uint32_t* __restrict__ out_idx,
                                                  Counters* __restrict__ ctr) {
  pdl_wait();
  if (info[0]) return;
  const uint32_t N = info[4];
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
  const uint32_t nch0 = (N + kTreeChunk0 - 1) / kTreeChunk0;
  const uint32_t len = info[1], ftop = w.bt[0][nch0];
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
