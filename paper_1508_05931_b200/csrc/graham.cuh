// K7/K8: graham_finalize (pipeline.hpp:57-67) on the device, in parallel,
// with an exact certificate.
//
// The reference scan is sequential and uses a non-robust predicate, so the
// output must equal THE SEQUENTIAL STACK, not just "the hull". Scheme:
//   1. chunk-local scans: every chunk of kChunk consecutive buffer points runs
//      the stack scan from an empty stack; its final stack (local chain) is kept.
//   2. candidate: per-boundary junction merges of neighbouring chains, run
//      in parallel and validated (junction strategy; points in convex
//      position); if a junction would reach below its neighbour's chain, a
//      sequential scan over the (much shorter) concatenation of all local
//      chains instead (sequential strategy). Either way the candidate defines a stack state at
//      every chunk boundary, stored as a persistent stack: boundary_top[c]
//      (top element before chunk c) and parent[p] (element below p).
//   3. certificate: every chunk replays ITS OWN points with the real
//      predicate from the candidate state at its start boundary and must end
//      in exactly the candidate state at its end boundary (compared node by
//      node). By induction over chunks, all-certified means the candidate's
//      final state is the sequential scan's output, bit for bit. Any failure
//      falls back to the exact sequential kernel.
#pragma once
#include "device_common.cuh"

namespace gscan {

constexpr int kChunk = 128;          // points per chunk (certificate granularity)
constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ bool left_turn(double ax, double ay, double bx, double by, double cx,
                                          double cy) {
  return cross_rn(ax, ay, bx, by, cx, cy) > 0.0;
}

// Step 1: chunk-local stack scans, one thread per chunk (the top two stack
// entries live in registers). Output: chain positions into
// chain[c*kChunk ...], chain_len[c].
__global__ void __launch_bounds__(128) k_graham_local(const double* __restrict__ R_x,
                                                       const double* __restrict__ R_y, uint32_t n,
                                                       uint32_t* __restrict__ chain,
                                                       uint32_t* __restrict__ chain_len) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lo = c * kChunk;
  if (lo >= n) return;
  const uint32_t cnt = min((uint32_t)kChunk, n - lo);
  const double* x = R_x + lo;
  const double* y = R_y + lo;
  uint8_t st[kChunk];
  int top = 0;
  double x1 = 0, y1 = 0, x2 = 0, y2 = 0;  // stack[top-1], stack[top-2]
  for (uint32_t i = 0; i < cnt; ++i) {
    const double px = x[i], py = y[i];
    while (top >= 2 && !left_turn(x2, y2, x1, y1, px, py)) {
      --top;
      x1 = x2; y1 = y2;
      if (top >= 2) { x2 = x[st[top - 2]]; y2 = y[st[top - 2]]; }
    }
    st[top++] = (uint8_t)i;
    x2 = x1; y2 = y1;
    x1 = px; y1 = py;
  }
  for (int k = 0; k < top; ++k) chain[lo + k] = lo + st[k];
  chain_len[c] = top;
}

// Gather chains into a dense list: out[off[c] + k] = chain[c*kChunk + k].
__global__ void k_gather_chains(const uint32_t* __restrict__ chain,
                                const uint32_t* __restrict__ chain_len,
                                const uint32_t* __restrict__ off, uint32_t nchunks,
                                uint32_t* __restrict__ out) {
  const uint32_t c = blockIdx.x * (blockDim.x / kChunk) + threadIdx.x / kChunk;
  const uint32_t k = threadIdx.x % kChunk;
  if (c >= nchunks) return;
  if (k < chain_len[c]) out[off[c] + k] = chain[c * kChunk + k];
}

// Step 2a, sequential strategy: stack scan over the candidate list Q (buffer
// positions, increasing) by one thread. Records parent[] for every push and
// the top before each level-0 chunk boundary. The final stack goes to out.
__global__ void k_graham_candidate_seq(const double* __restrict__ R_x,
                                       const double* __restrict__ R_y,
                                       const uint32_t* __restrict__ Q, const uint32_t* q_dev,
                                       uint32_t n_points, uint32_t* __restrict__ parent,
                                       uint32_t* __restrict__ btop, uint32_t* __restrict__ stack,
                                       uint32_t* __restrict__ out_len) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const uint32_t q = *q_dev;
  const uint32_t nchunks = (n_points + kChunk - 1) / kChunk;
  uint32_t top = 0;
  uint32_t next_b = 0;  // next boundary to record
  uint32_t t1 = kNone, t2 = kNone;  // stack[top-1], stack[top-2] positions
  double x1 = 0, y1 = 0, x2 = 0, y2 = 0;
  uint32_t pn = q ? Q[0] : 0;
  double pnx = q ? R_x[pn] : 0, pny = q ? R_y[pn] : 0;
  for (uint32_t i = 0; i < q; ++i) {
    const uint32_t p = pn;
    const double px = pnx, py = pny;
    if (i + 1 < q) {  // prefetch
      pn = Q[i + 1];
      pnx = R_x[pn];
      pny = R_y[pn];
    }
    const uint32_t cb = p / kChunk;
    while (next_b <= cb) btop[next_b++] = t1;
    while (top >= 2 && !left_turn(x2, y2, x1, y1, px, py)) {
      --top;
      t1 = t2; x1 = x2; y1 = y2;
      if (top >= 2) {
        t2 = stack[top - 2];
        x2 = R_x[t2];
        y2 = R_y[t2];
      } else {
        t2 = kNone;
      }
    }
    parent[p] = t1;
    stack[top++] = p;
    t2 = t1; x2 = x1; y2 = y1;
    t1 = p; x1 = px; y1 = py;
  }
  while (next_b <= nchunks) btop[next_b++] = t1;
  *out_len = top;
}

// Step 2b, junction strategy (thread per chunk c >= 1): merge L_c onto
// L_{c-1} as the sequential scan would, assuming nothing below L_{c-1}'s
// surviving part is touched; record pops k_c, dropped prefix e_c and the
// lowest L_{c-1} index examined (validated against e_{c-1} afterwards).
__global__ void k_graham_junction(const double* __restrict__ R_x, const double* __restrict__ R_y,
                                  const uint32_t* __restrict__ chain,
                                  const uint32_t* __restrict__ chain_len, uint32_t nchunks,
                                  uint32_t* __restrict__ jk, uint32_t* __restrict__ je,
                                  int32_t* __restrict__ jmin) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  if (c == 0) { jk[0] = 0; je[0] = 0; jmin[0] = 0; return; }
  const uint32_t* A = chain + (c - 1) * kChunk;
  const uint32_t* B = chain + c * kChunk;
  const int la = chain_len[c - 1], lb = chain_len[c];
  // stack = A[0..atop) ++ Bs[0..bt)
  int atop = la;
  uint32_t Bs[kChunk];
  uint8_t Bj[kChunk];
  int bt = 0;
  int minacc = la;  // lowest A index examined
  int j = 0;
  for (; j < lb; ++j) {
    const uint32_t p = B[j];
    const double px = R_x[p], py = R_y[p];
    while (true) {
      const int size = atop + bt;
      if (size < 2) {
        if (c != 1) minacc = -1;  // would need the state below A: invalid speculation
        break;                    // c == 1: A = L_0 is the bottom of the true stack
      }
      uint32_t s1, s2;
      if (bt >= 2) { s1 = Bs[bt - 1]; s2 = Bs[bt - 2]; }
      else if (bt == 1) { s1 = Bs[0]; s2 = A[atop - 1]; minacc = min(minacc, atop - 1); }
      else { s1 = A[atop - 1]; s2 = A[atop - 2]; minacc = min(minacc, atop - 2); }
      if (left_turn(R_x[s2], R_y[s2], R_x[s1], R_y[s1], px, py)) break;
      if (bt > 0) --bt; else --atop;
    }
    if (minacc < 0 && c != 1) break;
    Bs[bt] = p;
    Bj[bt] = (uint8_t)j;
    ++bt;
    if (j >= 1 && bt >= 2 && Bj[bt - 2] == j - 1) { ++j; break; }  // settled: rest appends
  }
  jk[c] = la - atop;
  je[c] = (minacc < 0) ? 0 : (uint32_t)Bj[0];
  jmin[c] = minacc;
}

// Validate junctions and build the persistent candidate: parent[] for every
// kept chain element, boundary tops, and kept flags for the final stack.
__global__ void k_graham_junction_apply(const uint32_t* __restrict__ chain,
                                        const uint32_t* __restrict__ chain_len, uint32_t nchunks,
                                        const uint32_t* __restrict__ jk,
                                        const uint32_t* __restrict__ je,
                                        const int32_t* __restrict__ jmin,
                                        uint32_t* __restrict__ parent, uint32_t* __restrict__ btop,
                                        uint32_t* __restrict__ keep_len,
                                        uint32_t* __restrict__ fail) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > nchunks) return;
  if (c == nchunks) {  // boundary after the last chunk
    btop[nchunks] = chain[(nchunks - 1) * kChunk + chain_len[nchunks - 1] - 1];
    return;
  }
  const uint32_t* L = chain + c * kChunk;
  const int len = chain_len[c];
  const int e = je[c];
  const int kill_top = (c + 1 < nchunks) ? (int)jk[c + 1] : 0;  // popped by the next junction
  if (c > 0) {
    const int la = chain_len[c - 1];
    const int e_prev = je[c - 1];
    const int k = jk[c];
    if (jmin[c] < e_prev || (c >= 2 && la - k <= e_prev)) atomicAdd(fail, 1u);
    const int below = la - 1 - k;  // A's top after the junction pops (c == 1 may empty A)
    parent[L[e]] = (below >= 0) ? chain[(c - 1) * kChunk + below] : kNone;
    btop[c] = chain[(c - 1) * kChunk + la - 1];
  } else {
    parent[L[0]] = kNone;
    btop[0] = kNone;
  }
  for (int i = e + 1; i < len; ++i) parent[L[i]] = L[i - 1];
  if (e + kill_top > len - 1 && c + 1 < nchunks) atomicAdd(fail, 1u);
  keep_len[c] = (uint32_t)max(0, len - kill_top - e);
}

__global__ void k_graham_junction_emit(const uint32_t* __restrict__ chain,
                                       const uint32_t* __restrict__ je,
                                       const uint32_t* __restrict__ keep_len,
                                       const uint32_t* __restrict__ off, uint32_t nchunks,
                                       uint32_t* __restrict__ stack) {
  const uint32_t c = blockIdx.x * (blockDim.x / kChunk) + threadIdx.x / kChunk;
  const uint32_t k = threadIdx.x % kChunk;
  if (c >= nchunks) return;
  if (k < keep_len[c]) stack[off[c] + k] = chain[c * kChunk + je[c] + k];
}

// Step 3: certificate. Thread per chunk: replay the chunk's points from the
// candidate state at its start and compare with the candidate state at its end.
__global__ void __launch_bounds__(128) k_graham_certify(const double* __restrict__ R_x,
                                                        const double* __restrict__ R_y,
                                                        uint32_t n, const uint32_t* __restrict__ parent,
                                                        const uint32_t* __restrict__ btop,
                                                        uint32_t* __restrict__ fail) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lo = c * kChunk;
  if (lo >= n) return;
  const uint32_t cnt = min((uint32_t)kChunk, n - lo);
  uint32_t base = btop[c];
  uint32_t nw[kChunk];
  int len = 0;
  bool ok = true;
  for (uint32_t i = 0; i < cnt && ok; ++i) {
    const uint32_t p = lo + i;
    const double px = R_x[p], py = R_y[p];
    while (true) {
      // the top two elements: nw[] first, then the base chain
      uint32_t s1, s2;
      if (len >= 2) { s1 = nw[len - 1]; s2 = nw[len - 2]; }
      else if (len == 1) { s1 = nw[0]; s2 = base; }
      else { s1 = base; s2 = (base == kNone) ? kNone : parent[base]; }
      if (s1 == kNone || s2 == kNone) break;  // fewer than two on the stack
      if (left_turn(R_x[s2], R_y[s2], R_x[s1], R_y[s1], px, py)) break;
      if (len > 0) --len; else base = parent[base];
    }
    nw[len++] = p;
  }
  // compare with the candidate end state
  uint32_t t = btop[c + 1];
  for (int k = len - 1; k >= 0 && ok; --k) {
    if (t != nw[k]) ok = false;
    else t = parent[t];
  }
  if (ok && t != base) ok = false;
  if (!ok) atomicAdd(fail, 1u);
}

// Output: positions in R -> input indices.
__global__ void k_graham_emit(const uint32_t* __restrict__ stack, const uint32_t* __restrict__ len_dev,
                              const uint32_t* __restrict__ R_i, uint32_t* __restrict__ out_idx,
                              Counters* __restrict__ ctr) {
  const uint32_t len = *len_dev;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < len; k += gridDim.x * blockDim.x)
    out_idx[k] = R_i[stack[k]];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hull = len;
}

}  // namespace gscan
