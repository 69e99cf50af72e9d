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
#include <cooperative_groups.h>

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
// ---------------------------------------------------------------------------
// Warp-cooperative stack scan. A sequential scan step costs ~160-280 cycles on
// B200 even from shared memory (8-cycle FP64 latency x a 3-deep predicate +
// branch), so every scan below advances 32 points per warp iteration: lane k
// tests the turn (P[k-2], P[k-1], P[k]) assuming all earlier points of the
// window were pushed without pops; the prefix up to the first failing lane f
// is committed (those tests ARE the sequential tests), point f takes its pop
// loop -- found in parallel as the first Left turn (S[d-1], S[d], P[f]) going
// down the stack -- and the window restarts after f. Identical decisions to
// the sequential loop, in order.

// Chunk-local scans (step 1): one warp per chunk, points staged in shared memory.
constexpr int kLocalWarps = 4;

__global__ void __launch_bounds__(kLocalWarps * 32) k_graham_local(const double* __restrict__ R_x,
                                                                   const double* __restrict__ R_y,
                                                                   uint32_t n,
                                                                   uint32_t* __restrict__ chain,
                                                                   uint32_t* __restrict__ chain_len) {
  __shared__ double s_px[kLocalWarps][kChunk], s_py[kLocalWarps][kChunk];
  __shared__ double s_sx[kLocalWarps][kChunk], s_sy[kLocalWarps][kChunk];
  __shared__ uint8_t s_si[kLocalWarps][kChunk];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kLocalWarps + w;
  const uint32_t lo = c * kChunk;
  if (lo >= n) return;
  const int cnt = (int)min((uint32_t)kChunk, n - lo);
  double* px_ = s_px[w];
  double* py_ = s_py[w];
  double* sx = s_sx[w];
  double* sy = s_sy[w];
  uint8_t* si = s_si[w];
  for (int k = lane; k < cnt; k += 32) { px_[k] = R_x[lo + k]; py_[k] = R_y[lo + k]; }
  __syncwarp();
  int top = 0;
  int i = 0;
  while (i < cnt) {
    const int j = i + lane;
    const bool valid = j < cnt;
    const double px = valid ? px_[j] : 0.0, py = valid ? py_[j] : 0.0;
    const int depth = top + lane;  // stack size before pushing j if all earlier lanes pushed
    bool ok = true;
    if (valid && depth >= 2) {
      double ax, ay, bx, by;  // prev2, prev1
      if (lane >= 2) { ax = px_[j - 2]; ay = py_[j - 2]; bx = px_[j - 1]; by = py_[j - 1]; }
      else if (lane == 1) { ax = sx[top - 1]; ay = sy[top - 1]; bx = px_[j - 1]; by = py_[j - 1]; }
      else { ax = sx[top - 2]; ay = sy[top - 2]; bx = sx[top - 1]; by = sy[top - 1]; }
      ok = left_turn(ax, ay, bx, by, px, py);
    }
    const uint32_t fm = __ballot_sync(0xffffffffu, valid && !ok);
    const int nvalid = min(32, cnt - i);
    const int f = fm ? (__ffs(fm) - 1) : 32;
    const int commit = min(f, nvalid);
    if (lane < commit) { sx[top + lane] = px; sy[top + lane] = py; si[top + lane] = (uint8_t)j; }
    top += commit;
    __syncwarp();
    if (f < nvalid) {
      const double fx = __shfl_sync(0xffffffffu, px, f), fy = __shfl_sync(0xffffffffu, py, f);
      int newtop;
      int dhi = top - 1;
      while (true) {
        const int d = dhi - lane;
        const bool l = d >= 1 && left_turn(sx[d - 1], sy[d - 1], sx[d], sy[d], fx, fy);
        const uint32_t m = __ballot_sync(0xffffffffu, l);
        if (m) { newtop = dhi - (__ffs(m) - 1) + 1; break; }
        if (dhi - 31 <= 1) { newtop = min(top, 1); break; }
        dhi -= 32;
      }
      __syncwarp();  // every lane's stack reads happen before lane 0 overwrites the top
      if (lane == 0) { sx[newtop] = fx; sy[newtop] = fy; si[newtop] = (uint8_t)(i + f); }
      top = newtop + 1;
      i += f + 1;
    } else {
      i += nvalid;
    }
    __syncwarp();
  }
  for (int k = lane; k < top; k += 32) chain[lo + k] = lo + si[k];
  if (lane == 0) chain_len[c] = top;
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
constexpr int kSeqBatch = 256;           // Q elements staged per batch
constexpr int kSeqStack = 4096;          // candidate stack capacity (shared memory)
constexpr size_t kCandSmem = (size_t)2 * kSeqBatch * (8 + 8 + 4) + (size_t)kSeqStack * (8 + 8 + 4);

// Step 2a, sequential strategy: the stack scan over the concatenated chains
// Q (buffer positions, increasing), warp-cooperative as above. Records the
// persistent candidate: parent[p] for every push and btop[b] = top before the
// first Q element of chunk >= b. *out_len = final size, or kNone if the stack
// outgrew shared memory (the host then takes the exact fallback).
__global__ void __launch_bounds__(32) k_graham_candidate_seq(
    const double* __restrict__ R_x, const double* __restrict__ R_y,
    const uint32_t* __restrict__ Q, const uint32_t* q_dev, uint32_t n_points,
    uint32_t* __restrict__ parent, uint32_t* __restrict__ btop, uint32_t* __restrict__ stack,
    uint32_t* __restrict__ out_len) {
  extern __shared__ __align__(16) unsigned char csm[];
  double* s_qx = reinterpret_cast<double*>(csm);        // [2][kSeqBatch]
  double* s_qy = s_qx + 2 * kSeqBatch;
  double* sx = s_qy + 2 * kSeqBatch;                     // [kSeqStack]
  double* sy = sx + kSeqStack;
  uint32_t* s_qp = reinterpret_cast<uint32_t*>(sy + kSeqStack);  // [2][kSeqBatch]
  uint32_t* sp = s_qp + 2 * kSeqBatch;                             // [kSeqStack]
  const uint32_t q = *q_dev;
  const uint32_t nchunks = (n_points + kChunk - 1) / kChunk;
  const int lane = threadIdx.x;
  auto load_batch = [&](uint32_t b, int buf) {
#pragma unroll
    for (int k = 0; k < kSeqBatch / 32; ++k) {
      const uint32_t i = b * kSeqBatch + k * 32 + lane;
      if (i < q) {
        const uint32_t p = Q[i];
        s_qp[buf * kSeqBatch + k * 32 + lane] = p;
        s_qx[buf * kSeqBatch + k * 32 + lane] = R_x[p];
        s_qy[buf * kSeqBatch + k * 32 + lane] = R_y[p];
      }
    }
  };
  const uint32_t nbatch = (q + kSeqBatch - 1) / kSeqBatch;
  if (nbatch) load_batch(0, 0);
  __syncwarp();
  int top = 0;
  int64_t last_chunk = -1;   // chunk of the previous Q element (boundaries recorded up to it)
  bool overflow = false;
  for (uint32_t bt = 0; bt < nbatch && !overflow; ++bt) {
    const int buf = bt & 1;
    if (bt + 1 < nbatch) load_batch(bt + 1, buf ^ 1);
    const double* qx = s_qx + buf * kSeqBatch;
    const double* qy = s_qy + buf * kSeqBatch;
    const uint32_t* qp = s_qp + buf * kSeqBatch;
    const int cnt = (int)min((uint32_t)kSeqBatch, q - bt * kSeqBatch);
    int i = 0;
    while (i < cnt) {
      if (top + 32 >= kSeqStack) { overflow = true; break; }
      const int j = i + lane;
      const bool valid = j < cnt;
      const double px = valid ? qx[j] : 0.0, py = valid ? qy[j] : 0.0;
      const uint32_t pp = valid ? qp[j] : 0u;
      const int depth = top + lane;
      bool ok = true;
      double ax = 0, ay = 0, bx = 0, by = 0;
      if (valid && depth >= 2) {
        if (lane >= 2) { ax = qx[j - 2]; ay = qy[j - 2]; bx = qx[j - 1]; by = qy[j - 1]; }
        else if (lane == 1) { ax = sx[top - 1]; ay = sy[top - 1]; bx = qx[j - 1]; by = qy[j - 1]; }
        else { ax = sx[top - 2]; ay = sy[top - 2]; bx = sx[top - 1]; by = sy[top - 1]; }
        ok = left_turn(ax, ay, bx, by, px, py);
      }
      const uint32_t fm = __ballot_sync(0xffffffffu, valid && !ok);
      const int nvalid = min(32, cnt - i);
      const int f = fm ? (__ffs(fm) - 1) : 32;
      const int commit = min(f, nvalid);
      const int upto = min(f + 1, nvalid);  // lanes whose "state before" is known
      // top before processing lane k: previous lane's point, or the stack top
      const uint32_t prev_pos = (lane >= 1) ? ((j - 1 >= 0) ? qp[j - 1] : 0u)
                                            : (top >= 1 ? sp[top - 1] : kNone);
      const uint32_t prev_top = (lane == 0) ? (top >= 1 ? sp[top - 1] : kNone) : prev_pos;
      // boundaries crossed before lane k: (chunk of previous element, chunk of k]
      if (lane < upto) {
        const int64_t pc = (lane == 0) ? last_chunk : (int64_t)(qp[j - 1] / kChunk);
        const int64_t cc = pp / kChunk;
        for (int64_t b2 = pc + 1; b2 <= cc; ++b2) btop[b2] = prev_top;
      }
      if (lane < commit) {
        sx[top + lane] = px; sy[top + lane] = py; sp[top + lane] = pp;
        stack[top + lane] = pp;
        parent[pp] = prev_top;
      }
      last_chunk = __shfl_sync(0xffffffffu, (int64_t)(pp / kChunk), max(upto - 1, 0));
      top += commit;
      __syncwarp();
      if (f < nvalid) {
        const double fx = __shfl_sync(0xffffffffu, px, f), fy = __shfl_sync(0xffffffffu, py, f);
        const uint32_t fp = __shfl_sync(0xffffffffu, pp, f);
        int newtop;
        int dhi = top - 1;
        while (true) {
          const int d = dhi - lane;
          const bool l = d >= 1 && left_turn(sx[d - 1], sy[d - 1], sx[d], sy[d], fx, fy);
          const uint32_t m = __ballot_sync(0xffffffffu, l);
          if (m) { newtop = dhi - (__ffs(m) - 1) + 1; break; }
          if (dhi - 31 <= 1) { newtop = min(top, 1); break; }
          dhi -= 32;
        }
        __syncwarp();  // every lane's stack reads happen before lane 0 overwrites the top
        if (lane == 0) {
          sx[newtop] = fx; sy[newtop] = fy; sp[newtop] = fp;
          stack[newtop] = fp;
          parent[fp] = newtop >= 1 ? sp[newtop - 1] : kNone;
        }
        top = newtop + 1;
        i += f + 1;
      } else {
        i += nvalid;
      }
      __syncwarp();
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (overflow) {
      *out_len = kNone;
    } else {
      const uint32_t t1 = top >= 1 ? sp[top - 1] : kNone;
      for (int64_t b2 = last_chunk + 1; b2 <= (int64_t)nchunks; ++b2) btop[b2] = t1;
      *out_len = top;
    }
  }
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
  // a warp per chunk: the chain's links are independent, so the lanes write
  // them together (coalesced chain reads; a thread per chunk walking its
  // chain was bound by the strided loads)
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (c > nchunks) return;
  if (c == nchunks) {  // boundary after the last chunk
    if (lane == 0) btop[nchunks] = chain[(nchunks - 1) * kChunk + chain_len[nchunks - 1] - 1];
    return;
  }
  const uint32_t* L = chain + c * kChunk;
  const int len = chain_len[c];
  const int e = je[c];
  if (lane == 0) {
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
    if (e + kill_top > len - 1 && c + 1 < nchunks) atomicAdd(fail, 1u);
    keep_len[c] = (uint32_t)max(0, len - kill_top - e);
  }
  for (int i = e + 1 + (int)lane; i < len; i += 32) parent[L[i]] = L[i - 1];
}

__global__ void __launch_bounds__(256) k_graham_junction_emit(const uint32_t* __restrict__ chain,
                                                           const uint32_t* __restrict__ je,
                                                           const uint32_t* __restrict__ keep_len,
                                                           const uint32_t* __restrict__ off,
                                                           uint32_t nchunks,
                                                           uint32_t* __restrict__ stack) {
  // a warp per chunk, kChunk / 32 elements per lane: the chunk's offsets are
  // read once and the element copies are independent (in flight together)
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (c >= nchunks) return;
  const uint32_t len = keep_len[c], o = off[c];
  const uint32_t* src = chain + (size_t)c * kChunk + je[c];
  constexpr int kPer = kChunk / 32;
  uint32_t v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t k = lane + 32u * u;
    v[u] = k < len ? src[k] : 0u;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const uint32_t k = lane + 32u * u;
    if (k < len) stack[o + k] = v[u];
  }
}

// Step 3: certificate. Thread per chunk: replay the chunk's points from the
// candidate state at its start and compare with the candidate state at its end.
// Step 3: certificate, one warp per chunk. The stack is the candidate state
// at the chunk's start boundary (persistent: btop[c], parent[]) with the
// chunk's own pushes in shared memory on top; the replay uses the same
// warp-cooperative scan (pops into the persistent part go one at a time).
// The end state must be exactly the candidate state at the next boundary:
// btop[c+1] == last push, parent[] links every push to the one below it, and
// the lowest push sits on the surviving persistent part.
constexpr int kCertWarps = 4;

__global__ void __launch_bounds__(kCertWarps * 32) k_graham_certify(
    const double* __restrict__ R_x, const double* __restrict__ R_y, uint32_t n,
    const uint32_t* __restrict__ parent, const uint32_t* __restrict__ btop,
    uint32_t* __restrict__ fail) {
  __shared__ double s_px[kCertWarps][kChunk], s_py[kCertWarps][kChunk];
  __shared__ double s_sx[kCertWarps][kChunk], s_sy[kCertWarps][kChunk];
  __shared__ uint8_t s_si[kCertWarps][kChunk];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t c = blockIdx.x * kCertWarps + w;
  const uint32_t lo = c * kChunk;
  if (lo >= n) return;
  const int cnt = (int)min((uint32_t)kChunk, n - lo);
  double* px_ = s_px[w];
  double* py_ = s_py[w];
  double* sx = s_sx[w];
  double* sy = s_sy[w];
  uint8_t* si = s_si[w];
  for (int k = lane; k < cnt; k += 32) { px_[k] = R_x[lo + k]; py_[k] = R_y[lo + k]; }
  // persistent part: base = its top, (b1x, b1y) its coords, pb = parent, (b2x, b2y)
  uint32_t base = btop[c];
  uint32_t pb = kNone;
  double b1x = 0, b1y = 0, b2x = 0, b2y = 0;
  auto load_base = [&]() {
    pb = kNone;
    if (base != kNone) {
      b1x = R_x[base]; b1y = R_y[base];
      pb = parent[base];
      if (pb != kNone) { b2x = R_x[pb]; b2y = R_y[pb]; }
    }
  };
  load_base();
  __syncwarp();
  int top = 0;  // pushes of this chunk on top of the persistent part
  int i = 0;
  while (i < cnt) {
    const int j = i + lane;
    const bool valid = j < cnt;
    const double px = valid ? px_[j] : 0.0, py = valid ? py_[j] : 0.0;
    // stack below lane j (assuming earlier lanes pushed): elements at depth 1 and 2
    bool has2;
    double ax, ay, bx, by;
    if (lane >= 2) { has2 = true; ax = px_[j - 2]; ay = py_[j - 2]; bx = px_[j - 1]; by = py_[j - 1]; }
    else if (lane == 1) {
      bx = px_[j - 1]; by = py_[j - 1];
      if (top >= 1) { has2 = true; ax = sx[top - 1]; ay = sy[top - 1]; }
      else { has2 = base != kNone; ax = b1x; ay = b1y; }
    } else {
      if (top >= 2) { has2 = true; ax = sx[top - 2]; ay = sy[top - 2]; bx = sx[top - 1]; by = sy[top - 1]; }
      else if (top == 1) { has2 = base != kNone; ax = b1x; ay = b1y; bx = sx[0]; by = sy[0]; }
      else { has2 = base != kNone && pb != kNone; ax = b2x; ay = b2y; bx = b1x; by = b1y; }
    }
    bool ok = true;
    if (valid && has2) ok = left_turn(ax, ay, bx, by, px, py);
    const uint32_t fm = __ballot_sync(0xffffffffu, valid && !ok);
    const int nvalid = min(32, cnt - i);
    const int f = fm ? (__ffs(fm) - 1) : 32;
    const int commit = min(f, nvalid);
    if (lane < commit) { sx[top + lane] = px; sy[top + lane] = py; si[top + lane] = (uint8_t)j; }
    top += commit;
    __syncwarp();
    if (f < nvalid) {
      const double fx = __shfl_sync(0xffffffffu, px, f), fy = __shfl_sync(0xffffffffu, py, f);
      // pops within this chunk's pushes (d >= 1: both in smem; d == 0: below is base)
      int newtop = -1;
      int dhi = top - 1;
      while (dhi >= 0) {
        const int d = dhi - lane;
        bool l = false;
        if (d >= 1) l = left_turn(sx[d - 1], sy[d - 1], sx[d], sy[d], fx, fy);
        else if (d == 0) l = (base == kNone) || left_turn(b1x, b1y, sx[0], sy[0], fx, fy);
        const uint32_t m = __ballot_sync(0xffffffffu, l);
        if (m) { newtop = dhi - (__ffs(m) - 1) + 1; break; }
        if (dhi - 31 <= 0) break;
        dhi -= 32;
      }
      if (newtop < 0) {
        // all pushes popped (or none existed): pop the persistent part one by one
        newtop = 0;
        while (base != kNone && pb != kNone && !left_turn(b2x, b2y, b1x, b1y, fx, fy)) {
          base = pb;
          load_base();
        }
      }
      if (lane == 0) { sx[newtop] = fx; sy[newtop] = fy; si[newtop] = (uint8_t)(i + f); }
      top = newtop + 1;
      i += f + 1;
    } else {
      i += nvalid;
    }
    __syncwarp();
  }
  // end state == candidate state at boundary c + 1
  bool ok = true;
  for (int k = lane; k < top; k += 32) {
    const uint32_t pk = lo + si[k];
    const uint32_t below = (k == 0) ? base : lo + si[k - 1];
    if (parent[pk] != below) ok = false;
  }
  if (lane == 0 && btop[c + 1] != (top ? lo + si[top - 1] : base)) ok = false;
  if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicAdd(fail, 1u);
}

// ---------------------------------------------------------------------------
// Step 2c, prefix strategy (square/disk-like inputs, where the boundary states
// stay small): every boundary state at once by a Hillis-Steele inclusive scan
// of the chunk chains under X (+) Y = Scan(X ++ Y), log2(chunks) rounds in one
// cooperative kernel. state[c] after the last round is the candidate stack
// after chunk c. States are explicit position lists of capacity `cap`; any
// overflow sets *ovf and the host takes another path. Associativity of (+) is
// what the exact geometry guarantees; the certificate checks every state, so
// rounding can only cost a fallback, never a wrong hull.

// Warp-cooperative scan of `cnt` points (positions pts[0..cnt)) onto the
// explicit stack st[0..top) (positions; coordinates gathered from R).
// Returns the new top. `cap` bounds the stack; returns -1 on overflow.
__device__ int warp_scan_onto(const double* __restrict__ R_x, const double* __restrict__ R_y,
                              uint32_t* st, int top, const uint32_t* pts, int cnt, int cap) {
  const int lane = threadIdx.x & 31;
  int i = 0;
  while (i < cnt) {
    if (top + 32 > cap) return -1;
    const int j = i + lane;
    const bool valid = j < cnt;
    const uint32_t pp = valid ? pts[j] : 0u;
    const double px = valid ? R_x[pp] : 0.0, py = valid ? R_y[pp] : 0.0;
    const int depth = top + lane;
    // previous two in the speculative chain
    const double q1x = __shfl_up_sync(0xffffffffu, px, 1), q1y = __shfl_up_sync(0xffffffffu, py, 1);
    const double q2x = __shfl_up_sync(0xffffffffu, px, 2), q2y = __shfl_up_sync(0xffffffffu, py, 2);
    bool ok = true;
    if (valid && depth >= 2) {
      double ax, ay, bx, by;
      if (lane >= 2) { ax = q2x; ay = q2y; bx = q1x; by = q1y; }
      else if (lane == 1) { ax = R_x[st[top - 1]]; ay = R_y[st[top - 1]]; bx = q1x; by = q1y; }
      else {
        ax = R_x[st[top - 2]]; ay = R_y[st[top - 2]];
        bx = R_x[st[top - 1]]; by = R_y[st[top - 1]];
      }
      ok = left_turn(ax, ay, bx, by, px, py);
    }
    const uint32_t fm = __ballot_sync(0xffffffffu, valid && !ok);
    const int nvalid = min(32, cnt - i);
    const int f = fm ? (__ffs(fm) - 1) : 32;
    const int commit = min(f, nvalid);
    if (lane < commit) st[top + lane] = pp;
    top += commit;
    __syncwarp();
    if (f < nvalid) {
      const double fx = __shfl_sync(0xffffffffu, px, f), fy = __shfl_sync(0xffffffffu, py, f);
      const uint32_t fp = __shfl_sync(0xffffffffu, pp, f);
      int newtop;
      int dhi = top - 1;
      while (true) {
        const int d = dhi - lane;
        bool l = false;
        if (d >= 1) {
          const uint32_t a = st[d - 1], b = st[d];
          l = left_turn(R_x[a], R_y[a], R_x[b], R_y[b], fx, fy);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, l);
        if (m) { newtop = dhi - (__ffs(m) - 1) + 1; break; }
        if (dhi - 31 <= 1) { newtop = min(top, 1); break; }
        dhi -= 32;
      }
      __syncwarp();  // every lane's stack reads happen before lane 0 overwrites the top
      if (lane == 0) st[newtop] = fp;
      top = newtop + 1;
      i += f + 1;
    } else {
      i += nvalid;
    }
    __syncwarp();
  }
  return top;
}

constexpr int kPrefixWarps = 4;

__global__ void __launch_bounds__(kPrefixWarps * 32) k_graham_prefix(
    const double* __restrict__ R_x, const double* __restrict__ R_y,
    const uint32_t* __restrict__ chain, const uint32_t* __restrict__ chain_len, uint32_t nchunks,
    uint32_t* __restrict__ stA, uint32_t* __restrict__ stB, uint32_t* __restrict__ lenA,
    uint32_t* __restrict__ lenB, uint32_t cap, uint32_t* __restrict__ ovf,
    uint32_t* __restrict__ which) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  // round 0 input: the chunk chains
  for (uint32_t c = gw; c < nchunks; c += nw) {
    const uint32_t l = chain_len[c];
    for (uint32_t k = lane; k < l; k += 32) stA[(size_t)c * cap + k] = chain[(size_t)c * kChunk + k];
    if (lane == 0) lenA[c] = l;
  }
  grid.sync();
  uint32_t* in = stA;
  uint32_t* out = stB;
  uint32_t* lin = lenA;
  uint32_t* lout = lenB;
  int rounds = 0;
  for (uint32_t off = 1; off < nchunks; off <<= 1, ++rounds) {
    for (uint32_t c = gw; c < nchunks; c += nw) {
      uint32_t* o = out + (size_t)c * cap;
      const uint32_t lc = lin[c];
      if (c < off) {
        for (uint32_t k = lane; k < lc; k += 32) o[k] = in[(size_t)c * cap + k];
        if (lane == 0) lout[c] = lc;
        continue;
      }
      const uint32_t la = lin[c - off];
      for (uint32_t k = lane; k < la; k += 32) o[k] = in[(size_t)(c - off) * cap + k];
      __syncwarp();
      const int t = warp_scan_onto(R_x, R_y, o, (int)la, in + (size_t)c * cap, (int)lc, (int)cap);
      if (lane == 0) {
        if (t < 0) { atomicAdd(ovf, 1u); lout[c] = 0; }
        else lout[c] = (uint32_t)t;
      }
    }
    grid.sync();
    uint32_t* tp = in; in = out; out = tp;
    tp = lin; lin = lout; lout = tp;
  }
  if (gw == 0 && lane == 0) *which = rounds & 1;  // 0: results in A, 1: in B
}

// Certificate for explicit states: warp per chunk c replays the chunk's
// points from state[c-1] (empty for c = 0) and must produce state[c] exactly.
__global__ void __launch_bounds__(kCertWarps * 32) k_graham_certify_explicit(
    const double* __restrict__ R_x, const double* __restrict__ R_y, uint32_t n,
    const uint32_t* __restrict__ st, const uint32_t* __restrict__ len, uint32_t cap,
    uint32_t* __restrict__ scratch, uint32_t* __restrict__ fail) {
  const int lane = threadIdx.x & 31;
  const uint32_t c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lo = c * kChunk;
  if (lo >= n) return;
  const uint32_t cnt = min((uint32_t)kChunk, n - lo);
  uint32_t* work = scratch + (size_t)c * (cap + kChunk + 32);
  uint32_t lp = 0;
  if (c > 0) {
    lp = len[c - 1];
    for (uint32_t k = lane; k < lp; k += 32) work[k] = st[(size_t)(c - 1) * cap + k];
  }
  uint32_t* pts = work + cap + 32;
  for (uint32_t k = lane; k < cnt; k += 32) pts[k] = lo + k;
  __syncwarp();
  const int t = warp_scan_onto(R_x, R_y, work, (int)lp, pts, (int)cnt, (int)(cap + 32));
  bool ok = (t >= 0) && (uint32_t)t == len[c];
  if (ok) {
    for (uint32_t k = lane; k < (uint32_t)t; k += 32)
      if (work[k] != st[(size_t)c * cap + k]) ok = false;
  }
  if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicAdd(fail, 1u);
}

__global__ void k_graham_emit_explicit(const uint32_t* __restrict__ st,
                                       const uint32_t* __restrict__ len, uint32_t last, uint32_t cap,
                                       const uint32_t* __restrict__ R_i, uint32_t* __restrict__ out_idx,
                                       Counters* __restrict__ ctr) {
  const uint32_t l = len[last];
  const uint32_t* s = st + (size_t)last * cap;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < l; k += gridDim.x * blockDim.x)
    out_idx[k] = R_i[s[k]];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hull = l;
}

// Output: positions in R -> input indices.
__global__ void k_graham_emit(const uint32_t* __restrict__ stack, const uint32_t* __restrict__ len_dev,
                              const uint32_t* __restrict__ R_i, uint32_t* __restrict__ out_idx,
                              Counters* __restrict__ ctr) {
  const uint32_t len = *len_dev;
  const uint32_t nth = gridDim.x * blockDim.x;
  uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  for (; k + 3 * nth < len; k += 4 * nth) {  // four independent gathers in flight
    uint32_t p[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p[u] = stack[k + u * nth];
    uint32_t q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = R_i[p[u]];
#pragma unroll
    for (int u = 0; u < 4; ++u) out_idx[k + u * nth] = q[u];
  }
  for (; k < len; k += nth) out_idx[k] = R_i[stack[k]];
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr->hull = len;
}

}  // namespace gscan
