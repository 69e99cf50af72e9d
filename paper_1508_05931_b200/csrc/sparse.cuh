// Sparse round 2: the pipeline's default path (gscan.cu run_sparse).
//
// The reference sorts EVERY round-1 survivor by (angle, dist2) and then walks
// 2 x chunk_count slices of that order (angular.hpp:154-194,
// discard.hpp:90-124); on a 20M square 13.3M survivors are sorted and 21K
// remain. Only the slice STRUCTURE needs every survivor -- slices are cut by
// rank -- and ranks need only counts. So this path:
//
//   map        a strided sample of round-1 survivors -> angle buckets of about
//              equal occupancy (k_sp_sample / k_sp_cdf / k_sp_theta).
//   F2         one pass (k_sp_hist): round-1 test, each survivor's bucket
//              (a monotone function of its glibc atan2 key, sp_bucket) into
//              a per-CTA shared-memory histogram and a per-point u16 code,
//              argmax dist2 (split_regions' P_l).
//   plan       bucket starts = exact ranks of every bucket; P_l's exact
//              position from its own bucket (codes-only pass k_sp_lrank);
//              slice steps; every bucket that holds a slice seed (or P_l) is
//              GATHERED: all its points are sorted exactly.
//   F3         one pass (k_sp_phi): gathered points are emitted; every other
//              survivor folds its walk angle phi (angle of P - P_l) into a
//              per-CTA bucket maximum; every survivor's 64-bit coordinate
//              hash goes to a per-CTA list (duplicate check).
//   sort G     gathered points exactly ordered -> every seed and, per
//              non-gathered bucket, the running maximum of phi over
//              everything before it in its slice (k_sp_slices).
//   F4         one pass (k_sp_cand): a non-gathered survivor whose phi is not
//              below its bucket's prefix maximum (minus kSpTol) is a
//              CANDIDATE.
//   walk       candidates + gathered points, exactly ordered, walked slice
//              by slice with the reference's exact predicate (k_sp_walk).
//   F6         one pass (k_sp_verify): every survivor that was NOT walked
//              must be discarded by the reference walk: strictly inside
//              against every kept point that can be its walk state
//              (discard.hpp:36-66), checked with the exact predicate.
//   dups       the hash lists are partitioned (k_sp_dup_part) and checked
//              for equal hashes (k_sp_dups): annotate's dedup
//              (angular.hpp:118-133) would change ranks.
//
// Why the result is the reference's, bit for bit: by induction along each
// slice, the reference's walk state before any point equals the last kept
// point before it. Walked points see that state in our walk too (skipped
// points never become state because they are discarded), and every skipped
// point is verified to be discarded against every state it could see. Any
// doubt -- a tie for P_l, a possible duplicate, a failed verification, an
// oversized bucket -- sets a fail bit and the call reruns the full sort
// path, which is exact by construction. The fast path never guesses.
#pragma once
#include "kernels.cuh"

namespace gscan {

constexpr uint32_t kSpBuckets = 48u * 1024u;  // coarse angle buckets (u32 smem arrays)
constexpr int kSpThreads = 512;               // persistent streaming CTAs, one per SM
constexpr uint32_t kSpPartBits = 11;          // duplicate-check hash partitions
constexpr uint32_t kSpParts = 1u << kSpPartBits;
constexpr double kSpTol = 1e-6;               // candidate tolerance on phi (pseudo-angle units)
constexpr double kSpPhiStoreErr = 1.2e-7;     // |phi| <= 2 stored as float: rounding <= 2^-23
constexpr uint32_t kSpGatherCap = 4096;       // largest bucket sorted in smem
constexpr uint32_t kSpPartChunk = 8192;       // entries per partitioning chunk (smem)
constexpr size_t kSpDupPartSmem = (size_t)kSpPartChunk * 8 + (size_t)kSpParts * 16;  // out + cnt/off/cursor/base

enum : uint32_t {
  kSpFailTie = 1u,        // several points share the maximal dist2
  kSpFailStep = 2u,       // (unused)
  kSpFailTiny = 4u,       // a region with <= 1 point (reference skips its walk)
  kSpFailDup = 8u,        // possible duplicate points (dedup changes ranks)
  kSpFailVerify = 16u,    // a skipped point would not be discarded
  kSpFailCap = 32u,       // a gathered bucket / dup partition exceeds capacity
  kSpFailInternal = 64u,  // inconsistent counts (should not happen)
  kSpFailFew = 128u,      // too few points for the bucket structure
  kSpFailMany = 256u,     // too many walk candidates (the full sort is faster)
};
// more than m / kSpManyDiv candidates after F4: decline (the full sort is faster)
constexpr uint32_t kSpManyDiv = 8;

struct SpD2 {        // per-CTA farthest-point candidate
  uint64_t d2;       // bits of dist2 (non-negative double: bit order = value order)
  uint32_t idx;      // input index
  uint32_t ties;     // points of this CTA at exactly d2
};

struct SpState {
  double lx, ly;       // P_l
  uint64_t d2max;
  uint32_t l_idx;      // input index of P_l
  uint32_t ties;
  uint32_t m;          // points in buckets = M - 1 (anchor excluded, no dedup)
  uint32_t M;
  uint32_t b_l;
  uint32_t l;          // exact position of P_l
  uint32_t l_below;    // points of P_l's bucket ordered before P_l
  uint32_t l_check;    // P_l's position as found by the gathered sort
  uint32_t step_r, step_l, n_right, n_left;
  uint32_t fail;
  uint32_t n_g;        // gathered elements emitted
  uint32_t n_c;        // candidates emitted
  uint32_t n_gb;       // gathered buckets
  uint32_t n_w;        // walk array size (anchor included)
  uint32_t n_r;        // kept (round-2 output size)
  uint32_t dups;
  uint32_t verify_fail;
  uint32_t why;        // first internal-failure site (debug)
  uint32_t n_bigc;     // candidate buckets sorted by the CTA sorter
  uint32_t max_g;      // largest gathered bucket
  uint32_t need_verify;  // 1: the error-bound certificate did not hold -> run F6
  uint32_t k_max;      // most kept points in one slice
  uint32_t phi_lo, phi_hi;  // range of phi over bucketed survivors (ordered floats)
  uint64_t rho2_bits;  // min |v|^2 over kept slice points (bits; non-negative double)
  double r02;          // (1e-3 * bounding-box diagonal)^2: closer points are always walked
  double dmax2;        // bounding-box diagonal^2
  uint32_t cert;       // 1: certificate holds (F6 skipped)
  uint32_t n_bigg;     // gathered buckets for the bitonic sorter
  uint32_t n_hugeg;    // gathered buckets above kSpGatherCap (global-scratch sorter)
  uint32_t n_exc;      // F2 points left to the exact pass (k_sp_f2_patch)
};

// ---------------------------------------------------------------------------
// Bucket map. Buckets are angle intervals: bucket(A) = #{k in [1, nb-1] :
// th[k] <= A} for the glibc atan2 key angle A (-0 folded) and an increasing
// table th[] -- monotone in A, so buckets never invert the reference order,
// whatever th[] holds. th[] is chosen per call so that buckets hold about
// equal numbers of survivors: th[k] = theta(Finv(k/nb)) where s(dx, dy) =
// (1 - dx/(|dx|+dy))/2 is a pseudo-angle (monotone in the angle, theta its
// inverse) and F is a piecewise-linear CDF of s over kSpCells cells, built
// from a fixed sample of round-1 survivors (k_sp_sample).
// Fast path: v = F(s)*nb from one approximate division; bucket = floor(v)
// unless v is within kSpGuard of an integer -- s is within 1e-13 of s(A)
// (division and glibc atan2 errors, the latter < 1 ulp), and even a cell
// holding every point moves v by < 1e-5 per 1e-13 of s -- else the exact key
// is computed and compared with th[].
constexpr int kSpCells = 2048;
constexpr double kSpGuardV = 1e-4;

__device__ __forceinline__ uint64_t angle_key(double dx, double dy) {
  const double a = glibc_atan2(dy, dx);
  return (a == 0.0) ? 0ull : dbits(a);
}

// 1/d to a few ulps: hardware approximation + two Newton steps (the error
// squares per step). Used only where a guard band, the certificate's e_phi
// term or the exact verification absorbs the error.
__device__ __forceinline__ double sp_rcp(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = __fma_rn(-d, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-d, r, 1.0);
  return __fma_rn(r, e, r);
}

// pseudo-angle s in [0, 1] (approximate; < 0 when undefined)
__device__ __forceinline__ double sp_s(double dx, double dy) {
  const double den = __dadd_rn(fabs(dx), dy);
  if (!(den > 1e-290)) return -1.0;
  return __dmul_rn(__dsub_rn(1.0, __dmul_rn(dx, sp_rcp(den))), 0.5);
}

// cdf: kSpCells + 1 increasing values from 0 to 1 (shared memory)
__device__ __forceinline__ uint32_t sp_bucket(double dx, double dy, const double* __restrict__ cdf,
                                              const double* __restrict__ th) {
  const double s = sp_s(dx, dy);
  uint32_t k = 0;
  if (s >= 0.0 && s <= 1.0) {
    const double u = __dmul_rn(s, (double)kSpCells);
    uint32_t j = (uint32_t)u;
    if (j > kSpCells - 1) j = kSpCells - 1;
    const double c0 = cdf[j], c1 = cdf[j + 1];
    const double v = __dmul_rn(__fma_rn(__dsub_rn(u, (double)j), __dsub_rn(c1, c0), c0),
                               (double)kSpBuckets);
    if (v >= 0.0 && v < (double)kSpBuckets) {
      k = (uint32_t)v;
      const double f = __dsub_rn(v, (double)k);
      if (f > kSpGuardV && f < 1.0 - kSpGuardV) return k;
    } else if (v >= (double)kSpBuckets) {
      k = kSpBuckets - 1;
    }
  }
  const double a = bitsd(angle_key(dx, dy));
  while (k > 0 && a < th[k]) --k;
  while (k + 1 < kSpBuckets && a >= th[k + 1]) ++k;
  return k;
}

__device__ __forceinline__ uint32_t ord_f(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
// 0 encodes "no value" (below every float)
__device__ __forceinline__ double unord_f(uint32_t u) {
  if (u == 0) return -1e300;
  return (double)__uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Coordinate hash with -0.0 folded onto +0.0 (annotate's CoordSet compares
// folded bits, angular.hpp:99-101): equal points hash equally.
// 64-bit coordinate hash with -0.0 folded onto +0.0 (annotate's CoordSet
// compares folded bits, angular.hpp:99-101): equal points hash equally, so
// equal hashes are the only possible duplicates.
// splitmix64's finalizer: a bijection of 64-bit words with full avalanche
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}

__device__ __forceinline__ uint64_t coord_hash64(double x, double y) {
  // x + 0.0 folds -0.0 onto +0.0 and leaves every other finite x unchanged
  const uint64_t a = dbits(__dadd_rn(x, 0.0)), b = dbits(__dadd_rn(y, 0.0));
  // mix(a + rotl(b, 32)): y's high bits land in the word's low half, where x's
  // doubles of structured inputs (integer lattices: ~40 trailing zero bits)
  // are zero, so such inputs do not collide before the bijective mix -- a
  // linear a*C1 + b*C2 kept only their top bits. A collision of distinct
  // points only makes the sparse path decline, never a wrong result.
  const uint64_t z = mix64(a + ((b << 32) | (b >> 32)));
  return z == ~0ull ? 0ull : z;  // ~0 marks an empty slot / padding
}


// Walk angle of P around P_l, measured from u = anchor - P_l (kernels.cuh
// pseudo_angle), signed by region: right region keeps running maxima of
// +phi, left region of -phi.
__device__ __forceinline__ double sp_phi(double px, double py, double lx, double ly, double ux,
                                         double uy, bool right) {
  const double vx = __dsub_rn(px, lx), vy = __dsub_rn(py, ly);
  const double c = __fma_rn(ux, vx, __dmul_rn(uy, vy));   // along P_l -> anchor
  const double sn = __fma_rn(ux, vy, -__dmul_rn(uy, vx)); // across
  const double den = fabs(c) + fabs(sn);
  if (!(den > 1e-290)) return 0.0;
  const double t = 1.0 - c * sp_rcp(den);                 // [0, 2], increasing with the angle
  const double p = sn >= 0.0 ? t : -t;
  return right ? p : -p;
}

// Raw walk angle (pseudo-angle of P - P_l from u, CCW positive) and |P - P_l|^2.
__device__ __forceinline__ double sp_phi_raw(double px, double py, double lx, double ly, double ux,
                                             double uy, double* v2) {
  const double vx = __dsub_rn(px, lx), vy = __dsub_rn(py, ly);
  *v2 = __fma_rn(vx, vx, __dmul_rn(vy, vy));
  const double c = __fma_rn(ux, vx, __dmul_rn(uy, vy));
  const double sn = __fma_rn(ux, vy, -__dmul_rn(uy, vx));
  const double den = fabs(c) + fabs(sn);
  if (!(den > 1e-290)) return 0.0;
  const double t = 1.0 - c * sp_rcp(den);
  return sn >= 0.0 ? t : -t;
}

// Streaming helper: visits every point i of [0, n) once across the grid,
// 128-bit loads, kPairs pairs in flight per thread. f(x, y, i).
template <bool kVec, int kPairs, typename F>
__device__ __forceinline__ void sp_stream(const double* __restrict__ xs,
                                          const double* __restrict__ ys, uint32_t n, F&& f) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nth = gridDim.x * blockDim.x;
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    const uint32_t np = n / 2;
    uint32_t p = tid;
    for (; p + (kPairs - 1) * nth < np; p += kPairs * nth) {
      double2 vx[kPairs], vy[kPairs];
#pragma unroll
      for (int u = 0; u < kPairs; ++u) {
        vx[u] = __ldcs(&x2[p + u * nth]);
        vy[u] = __ldcs(&y2[p + u * nth]);
      }
#pragma unroll
      for (int u = 0; u < kPairs; ++u) {
        const uint32_t i = 2 * (p + u * nth);
        f(vx[u].x, vy[u].x, i);
        f(vx[u].y, vy[u].y, i + 1);
      }
    }
    for (; p < np; p += nth) {
      const double2 vx = __ldcs(&x2[p]), vy = __ldcs(&y2[p]);
      f(vx.x, vy.x, 2 * p);
      f(vx.y, vy.y, 2 * p + 1);
    }
    if ((n & 1) && tid == nth - 1) f(xs[n - 1], ys[n - 1], n - 1);
  } else {
    for (uint32_t i = tid; i < n; i += nth) f(xs[i], ys[i], i);
  }
}

// Same visit order, with each point's u16 bucket code from F2 (0xffff: not
// in the buffer). f(x, y, code, i).
template <bool kVec, int kPairs, typename F>
__device__ __forceinline__ void sp_stream_coded(const double* __restrict__ xs,
                                                const double* __restrict__ ys,
                                                const uint16_t* __restrict__ codes, uint32_t n,
                                                F&& f) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nth = gridDim.x * blockDim.x;
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(codes);
    const uint32_t np = n / 2;
    uint32_t p = tid;
    for (; p + (kPairs - 1) * nth < np; p += kPairs * nth) {
      double2 vx[kPairs], vy[kPairs];
      uint32_t vc[kPairs];
#pragma unroll
      for (int u = 0; u < kPairs; ++u) vc[u] = __ldcs(&c2[p + u * nth]);
#pragma unroll
      for (int u = 0; u < kPairs; ++u) {
        vx[u] = __ldcs(&x2[p + u * nth]);
        vy[u] = __ldcs(&y2[p + u * nth]);
      }
#pragma unroll
      for (int u = 0; u < kPairs; ++u) {
        const uint32_t i = 2 * (p + u * nth);
        f(vx[u].x, vy[u].x, vc[u] & 0xffffu, i);
        f(vx[u].y, vy[u].y, vc[u] >> 16, i + 1);
      }
    }
    for (; p < np; p += nth) {
      const uint32_t vc = c2[p];
      const double2 vx = __ldcs(&x2[p]), vy = __ldcs(&y2[p]);
      f(vx.x, vy.x, vc & 0xffffu, 2 * p);
      f(vx.y, vy.y, vc >> 16, 2 * p + 1);
    }
    if ((n & 1) && tid == nth - 1) f(xs[n - 1], ys[n - 1], (uint32_t)codes[n - 1], n - 1);
  } else {
    for (uint32_t i = tid; i < n; i += nth) f(xs[i], ys[i], (uint32_t)codes[i], i);
  }
}
constexpr uint32_t kSpNoCode = 0xffffu;
constexpr uint32_t kSpCandCode = 0xfffeu;  // set by F4 on candidates

struct SpQuad {  // round-1 quadrilateral with hoisted edge vectors + anchor
  double qx[4], qy[4], ex[4], ey[4], ax, ay;
  uint32_t aidx;
};

__device__ __forceinline__ void load_quad(const ExtResult* ext, SpQuad& q) {
#pragma unroll
  for (int k = 0; k < 4; ++k) { q.qx[k] = ext->qx[k]; q.qy[k] = ext->qy[k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    q.ex[k] = __dsub_rn(q.qx[(k + 1) & 3], q.qx[k]);
    q.ey[k] = __dsub_rn(q.qy[(k + 1) & 3], q.qy[k]);
  }
  q.ax = ext->ax;
  q.ay = ext->ay;
  q.aidx = ext->idx[4];
}

// ===========================================================================
// Bucket map construction (after K1): a fixed strided sample of the input,
// its round-1 survivors' pseudo-angles counted in kSpCells cells ->
// piecewise-linear CDF (every cell gets a small floor so it stays strictly
// increasing) -> th[k] = theta(Finv(k/nb)).
constexpr uint32_t kSpSample = 1u << 17;

__global__ void __launch_bounds__(1024) k_sp_sample(const double* __restrict__ xs,
                                                    const double* __restrict__ ys, uint32_t n,
                                                    const ExtResult* __restrict__ ext,
                                                    uint32_t* __restrict__ cell_cnt) {
  pdl_wait();
  __shared__ uint32_t s_cnt[kSpCells];
  for (uint32_t j = threadIdx.x; j < kSpCells; j += blockDim.x) s_cnt[j] = 0;
  SpQuad q;
  load_quad(ext, q);
  __syncthreads();
  const uint32_t ns = min(n, kSpSample);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < ns; k += gridDim.x * blockDim.x) {
    const uint32_t i = (uint32_t)(((uint64_t)k * n) / ns);
    const double x = xs[i], y = ys[i];
    if (!quad_keep(q.qx, q.qy, q.ex, q.ey, x, y) || (x == q.ax && y == q.ay)) continue;
    const double sv = sp_s(__dsub_rn(x, q.ax), __dsub_rn(y, q.ay));
    if (sv < 0.0 || sv > 1.0) continue;
    uint32_t j = (uint32_t)(sv * kSpCells);
    if (j > kSpCells - 1) j = kSpCells - 1;
    atomicAdd(&s_cnt[j], 1u);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < kSpCells; j += blockDim.x)
    if (s_cnt[j]) atomicAdd(&cell_cnt[j], s_cnt[j]);
}

// One CTA of kSpCells/2 threads (two cells each): inclusive scan of the
// floored counts -> CDF.
// n > 0: also the early speed decision -- when >= 95% of the sampled points
// survive round 1 (near-convex input) nearly all will be walk candidates and
// the full sort is faster; decline before F2.
__global__ void __launch_bounds__(kSpCells / 2) k_sp_cdf(const uint32_t* __restrict__ cell_cnt,
                                                         double* __restrict__ cdf, uint32_t n,
                                                         SpState* __restrict__ st) {
  pdl_wait();
  __shared__ double s_w[32];
  const double floor_w = 0.02;  // per-cell floor, in sample units
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double a = (double)cell_cnt[2 * threadIdx.x] + floor_w;
  const double b = (double)cell_cnt[2 * threadIdx.x + 1] + floor_w;
  double x = a + b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  if (warp == 0) {
    double t = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_w[lane] = t;
  }
  __syncthreads();
  const double incl = x + (warp ? s_w[warp - 1] : 0.0), tot = s_w[31];
  const uint32_t j = 2 * threadIdx.x;
  cdf[j + 1] = (incl - b) / tot;
  cdf[j + 2] = (j + 2 == kSpCells) ? 1.0 : incl / tot;
  if (threadIdx.x == 0) {
    cdf[0] = 0.0;
    const double kept = tot - floor_w * kSpCells;  // sampled round-1 survivors
    const uint32_t ns = min(n, kSpSample);
    if (n > 0 && kept * 100.0 > (double)ns * 95.0) atomicOr(&st->fail, kSpFailMany);
  }
}

__global__ void __launch_bounds__(256) k_sp_theta(const double* __restrict__ cdf,
                                                  double* __restrict__ th,
                                                  SpState* __restrict__ st) {
  pdl_wait();
  __shared__ double s_cdf[kSpCells + 1];
  for (uint32_t j = threadIdx.x; j <= kSpCells; j += blockDim.x) s_cdf[j] = cdf[j];
  __syncthreads();
  auto theta_of = [&](uint32_t kk) -> double {
    if (kk == 0) return 0.0;
    if (kk >= kSpBuckets) return 3.141592653589793;
    const double y = (double)kk / (double)kSpBuckets;
    uint32_t lo = 0, hi = kSpCells - 1;  // cell j with cdf[j] <= y < cdf[j+1]
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (s_cdf[mid] <= y) lo = mid;
      else hi = mid - 1;
    }
    const double fr = (y - s_cdf[lo]) / (s_cdf[lo + 1] - s_cdf[lo]);
    const double sv = ((double)lo + fr) / (double)kSpCells;
    const double t = 1.0 - 2.0 * sv;
    return atan2(1.0 - fabs(t), t);
  };
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= kSpBuckets;
       k += gridDim.x * blockDim.x) {
    const double a = theta_of(k);
    th[k] = a;
    if (k > 0 && !(a > theta_of(k - 1))) atomicOr(&st->fail, kSpFailInternal);
  }
}

// Column reduction of per-CTA arrays: out[b] = sum / max over rows.
template <bool kMax>
__global__ void k_sp_reduce_cols(const uint32_t* __restrict__ part, uint32_t rows, uint32_t cols,
                                 uint32_t* __restrict__ out) {
  pdl_wait();
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= cols) return;
  uint32_t v = 0;
  for (uint32_t r = 0; r < rows; ++r) {
    const uint32_t x = part[(size_t)r * cols + b];
    v = kMax ? max(v, x) : v + x;
  }
  out[b] = v;
}

// F2's per-point work for B points at once, as branch-free phases (quad test,
// pseudo-angle, CDF lookup) so the independent FP64 chains interleave; only
// the rare guard-band case branches (sp_bucket's exact fallback). Same
// arithmetic, same result as visiting the points one by one.
template <int B, bool kHist>
__device__ __forceinline__ void f2_batch(const double (&x)[B], const double (&y)[B],
                                         const uint32_t (&idx)[B], uint32_t (&code)[B],
                                         const SpQuad& q, const double* s_cdf,
                                         const double* __restrict__ th, uint32_t* s_hist,
                                         uint32_t& n1, uint64_t& bd2, uint32_t& bidx,
                                         uint32_t& bties) {
  double dx[B], dy[B], u[B];
  bool live[B], oks[B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    bool inside = true;  // strictly Left of all four edges (classify_quad flag 0)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      inside = inside & (cross_edge(q.qx[e], q.qy[e], q.ex[e], q.ey[e], x[k], y[k]) > 0.0);
    n1 += inside ? 0u : 1u;
    live[k] = !inside && !(x[k] == q.ax && y[k] == q.ay);
    dx[k] = __dsub_rn(x[k], q.ax);
    dy[k] = __dsub_rn(y[k], q.ay);
    const double den = __dadd_rn(fabs(dx[k]), dy[k]);
    const bool okd = den > 1e-290;
    const double sv = __dmul_rn(__dsub_rn(1.0, __dmul_rn(dx[k], sp_rcp(okd ? den : 1.0))), 0.5);
    oks[k] = okd && sv >= 0.0 && sv <= 1.0;
    u[k] = __dmul_rn(oks[k] ? sv : 0.0, (double)kSpCells);
  }
  bool fast[B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    uint32_t j = (uint32_t)u[k];
    if (j > kSpCells - 1) j = kSpCells - 1;
    const double c0 = s_cdf[j], c1 = s_cdf[j + 1];
    const double v = __dmul_rn(__fma_rn(__dsub_rn(u[k], (double)j), __dsub_rn(c1, c0), c0),
                               (double)kSpBuckets);
    const bool inr = v >= 0.0 && v < (double)kSpBuckets;
    const uint32_t b = inr ? (uint32_t)v : (v >= (double)kSpBuckets ? kSpBuckets - 1 : 0u);
    const double f = __dsub_rn(v, (double)b);
    fast[k] = oks[k] && inr && f > kSpGuardV && f < 1.0 - kSpGuardV;
    code[k] = oks[k] ? b : 0u;
  }
#pragma unroll
  for (int k = 0; k < B; ++k) {
    if (!live[k]) { code[k] = kSpNoCode; continue; }
    uint32_t b = code[k];
    if (!fast[k]) {  // exact key against th[] (sp_bucket's fallback)
      const double a = bitsd(angle_key(dx[k], dy[k]));
      while (b > 0 && a < th[b]) --b;
      while (b + 1 < kSpBuckets && a >= th[b + 1]) ++b;
    }
    code[k] = b;
    if (kHist) atomicAdd(&s_hist[b], 1u);
    const uint64_t d2 = dbits(dist2_rn(dx[k], dy[k]));
    const uint32_t i = idx[k];
    if (bidx == 0xffffffffu || d2 > bd2) { bd2 = d2; bidx = i; bties = 1; }
    else if (d2 == bd2) { ++bties; if (i < bidx) bidx = i; }
  }
}

// ===========================================================================
// F2 screen. Most of F2's FP64 work (the four quad crosses, the CDF
// lookup and the guard test: ~48 FP64 instructions and 4 FP64 conversions
// per point in the plain path) is replaced by FP32 arithmetic with a proven
// error bound; only the pseudo-angle's cell coordinate stays in FP64. A point
// whose screened result lies within its error bound of a decision boundary is
// UNCERTAIN and takes the exact path (f2_exact: the plain per-point code),
// ~2e-4 of the points.
//
// Quad (classify_quad, prefilter.hpp:47-63). The reference's cross for edge e
// is R_e = ex*(y - qy) - ey*(x - qx) in double. With dx = x - ax, dy = y - ay
// (double, then rounded to float: fx, fy) and K_e = ex*qdy - ey*qdx
// (qd = q_e - anchor), the float value c_e = fma(EX, fy, fma(-EY, fx, -K_e))
// differs from the double cross by at most
//   4.1u (|ex||dy| + |ey||dx| + |K_e|) + O(2^-53) terms,  u = 2^-24,
// and |dx| <= DX, |dy| <= DY (bounding box of the input around the anchor).
// B_e = 8u (|ex| DY + |ey| DX + |K_e|) + 2^-100 covers that, plus the extra
// rounding of pre-scaling the coefficients by 1/B_e: c'_e = c_e / B_e, so
// min_e c'_e > 1 proves every cross > 0 (inside: flag 0) and min_e c'_e < -1
// proves one cross < 0 (kept). A zero edge (ex = ey = 0) has cross exactly 0:
// kept, encoded as c'_e = -2.
//
// Bucket (sp_bucket). The cell coordinate u = 1024 (1 - dx/(|dx| + dy))
// (= s * kSpCells) is formed in double (rcp.approx + one Newton step: error
// <= 1024 * 2^-39.8 = 1.1e-9), split exactly into the cell j = floor(u) and
// t = u - j in [0, 1] (t = 1 when u is an integer and the tie rounds down:
// the piecewise-linear map is continuous, so cell j at t = 1 is cell j + 1 at
// t = 0), and t is rounded to float (error <= 2^-25). Per cell the table
// holds I_j + phi_j = nb * cdf[j] (phi_j in [0, 1) as float) and the slope
// S_j = nb * (cdf[j+1] - cdf[j]) (float), and v = phi_j + t * S_j in float
// errs from the exact piecewise-linear value by at most 1.5e-7 S_j + 1.1e-7
// (t, S and phi rounding, the fma; a cell mix-up near a breakpoint stays
// inside the bound by continuity). The double path trusts floor(v_d) when
// frac(v_d) is 1e-4 away from an integer; the screen trusts floor(v_f) only
// when frac(v_f) is g_j = 1.03e-4 + 2e-7 S_j away, so floor(v_f) = floor(v_d)
// and the double path's own condition holds: the screened bucket IS
// sp_bucket's result.
//
// P_l (argmax dist2): a survivor whose float dist2 (error <= 5u) is below
// (1 - 16u) times the best dist2 seen by its warp (or by the quad vertices,
// which all survive) cannot be the maximum or tie it; only the others
// compute dist2 in double.
//
// Preconditions of the quad screen (checked per CTA, else every point takes
// the exact path): the box extents DX, DY in [2^-50, 2^50] and finite scaled
// coefficients.
constexpr float kF2G1 = 2.0e-7f;
constexpr float kF2G0 = 1.03e-4f;
constexpr float kF2Magic = 12582912.0f;          // 1.5 * 2^23: v + magic rounds v to an integer
constexpr int kF2MagicBits = 0x4B400000;
constexpr double kF2MagicD = 6755399441055744.0;  // 1.5 * 2^52

struct F2Float {
  float ex[4], ey[4], k[4];  // scaled: c'_e = ex*fy - ey*fx - k
  float thr0;                // lower bound of max dist2 (quad vertices), screened
  bool on;
};

// a float threshold t with t <= d2 * (1 - 16u) for the double d2 (0 when tiny):
// a survivor whose float dist2 (relative error <= 5u) is below t is below d2
__device__ __forceinline__ float f2_thr(double d2) {
  const float tf = __fmul_rn(__double2float_rz(d2), 1.0f - 16.0f * 5.9604645e-8f);
  return tf < 1e-27f ? 0.f : tf;
}

__device__ __forceinline__ void f2_float_setup(const SpQuad& q, F2Float& f) {
  // bounding box from the extremes (minx, miny, maxx, maxy) around the anchor
  const double DX = fmax(fabs(q.qx[0] - q.ax), fabs(q.qx[2] - q.ax));
  const double DY = fabs(q.qy[3] - q.ay);
  bool on = fmax(DX, DY) >= 0x1p-50 && fmax(DX, DY) <= 0x1p50;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const double ex = q.ex[e], ey = q.ey[e];
    const double qdx = q.qx[e] - q.ax, qdy = q.qy[e] - q.ay;
    const double K = ex * qdy - ey * qdx;
    if (ex == 0.0 && ey == 0.0) {
      f.ex[e] = 0.f; f.ey[e] = 0.f; f.k[e] = 2.f;
      continue;
    }
    const double B = 0x1p-21 * (fabs(ex) * DY + fabs(ey) * DX + fabs(K)) + 0x1p-100;  // 8u
    const double ib = 1.0 / B;
    f.ex[e] = (float)(ex * ib);
    f.ey[e] = (float)(ey * ib);
    f.k[e] = (float)(K * ib);
    on = on && isfinite(f.ex[e]) && isfinite(f.ey[e]) && isfinite(f.k[e]) && B >= 0x1p-90;
  }
  f.on = on;
  // every quad vertex survives round 1 (it lies on two edges): the maximal
  // dist2 is at least theirs (the anchor itself is not bucketed)
  double m = 0.0;
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (!(q.qx[e] == q.ax && q.qy[e] == q.ay))
      m = fmax(m, dist2_rn(__dsub_rn(q.qx[e], q.ax), __dsub_rn(q.qy[e], q.ay)));
  f.thr0 = f2_thr(m);
}

// Bucket table: entry j (cell j of the CDF, 0..kSpCells; entry kSpCells
// extrapolates the last cell: v >= nb there, always uncertain)
// = {I_j - magic bits, phi_j - 0.5, S_j, 0.5 - g_j}
// with I_j + phi_j = nb * cdf[j] (phi_j in [0, 1)), S_j = nb * (cdf[j+1] -
// cdf[j]) and g_j = kF2G0 + kF2G1 * S_j: v - 0.5 = (phi_j - 0.5) + t * S_j,
// rounded to the nearest integer by the magic add, is floor(v), and the
// fraction of v is g_j away from an integer iff |v - 0.5 - round| < 0.5 - g_j.
__device__ __forceinline__ void f2_table_setup(const double* __restrict__ cdf, float4* s_tab,
                                               uint32_t tid, uint32_t nthreads) {
  const double nb = (double)kSpBuckets;
  for (uint32_t r = tid; r <= (uint32_t)kSpCells; r += nthreads) {
    const uint32_t j = r < (uint32_t)kSpCells ? r : (uint32_t)kSpCells - 1;
    const double V = nb * cdf[r];
    const double I = floor(V);
    const float S = (float)(nb * cdf[j + 1] - nb * cdf[j]);
    s_tab[r] = make_float4(__int_as_float((int)I - kF2MagicBits), (float)(V - I) - 0.5f, S,
                           0.5f - fmaf(S, kF2G1, kF2G0));
  }
}

// The exact per-point F2 work (the plain path's visit): returns the code
// (kSpNoCode when not bucketed) and whether the point survives round 1.
__device__ __noinline__ uint32_t f2_exact(double x, double y, uint32_t i, const SpQuad& q,
                                          const double* __restrict__ cdf,
                                          const double* __restrict__ th, uint32_t& kept,
                                          uint64_t& bd2, uint32_t& bidx, uint32_t& bties) {
  kept = quad_keep(q.qx, q.qy, q.ex, q.ey, x, y) ? 1u : 0u;
  if (!kept) return kSpNoCode;
  if (x == q.ax && y == q.ay) return kSpNoCode;
  const double dx = __dsub_rn(x, q.ax), dy = __dsub_rn(y, q.ay);
  const uint32_t b = sp_bucket(dx, dy, cdf, th);
  const uint64_t d2 = dbits(dist2_rn(dx, dy));
  if (bidx == 0xffffffffu || d2 > bd2) { bd2 = d2; bidx = i; bties = 1; }
  else if (d2 == bd2) { ++bties; if (i < bidx) bidx = i; }
  return b;
}

// B points through the screen: first every point's screen, branch-free, so
// the B independent FP64/FP32 chains interleave; then the rare uncertain
// points and the dist2 candidates take their exact paths. Fills code[].
template <int B>
__device__ __forceinline__ void f2_points(const double (&x)[B], const double (&y)[B],
                                          const uint32_t (&idx)[B], uint32_t (&code)[B], const SpQuad& q, const F2Float& F,
                                          const float4* s_tab, const double* __restrict__ cdf,
                                          const double* __restrict__ th, uint32_t& n1,
                                          uint64_t& bd2, uint32_t& bidx, uint32_t& bties,
                                          float thr, uint32_t* __restrict__ exc_list,
                                          uint32_t exc_cap, uint32_t* __restrict__ exc_n) {
  uint32_t sure = 0, inside = 0, cand = 0;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    const double dx = __dsub_rn(x[k], q.ax), dy = __dsub_rn(y[k], q.ay);
    const float fx = __double2float_rn(dx), fy = __double2float_rn(dy);
    float m = fmaf(F.ex[0], fy, fmaf(-F.ey[0], fx, -F.k[0]));
#pragma unroll
    for (int e = 1; e < 4; ++e) m = fminf(m, fmaf(F.ex[e], fy, fmaf(-F.ey[e], fx, -F.k[e])));
    // cell coordinate in double, split exactly into j = floor(u) and t = u - j
    const double den = __dadd_rn(fabs(dx), dy);
    double r;  // 1/den: rcp.approx (2^-19.9) + one Newton step (2^-39.8): u errs <= 1.1e-9
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
    r = __fma_rn(r, __fma_rn(-den, r, 1.0), r);
    const double u = fma(-1024.0, __dmul_rn(dx, r), 1023.5);  // u - 0.5
    const double w = __dadd_rn(u, kF2MagicD);                  // round(u - 0.5) = floor(u)
    const int j = (int)__double2loint(w);
    const float t = __double2float_rn(__dadd_rn(__dsub_rn(u, __dsub_rn(w, kF2MagicD)), 0.5));
    const bool okr = (uint32_t)j <= (uint32_t)kSpCells;
    const float4 E = s_tab[okr ? j : 0];
    const float v = fmaf(t, E.z, E.y);  // v - 0.5
    const float w2 = __fadd_rn(v, kF2Magic);
    const float dd = __fsub_rn(v, __fsub_rn(w2, kF2Magic));
    const uint32_t bk = (uint32_t)(__float_as_int(E.x) + __float_as_int(w2));
    const bool in = F.on && m > 1.f;
    const bool ok = F.on && m < -1.f && den > 1e-280 && okr && fabsf(dd) < E.w && bk < kSpBuckets;
    const bool cd = fmaf(fx, fx, __fmul_rn(fy, fy)) >= thr;
    code[k] = in ? kSpNoCode : (ok ? bk : 0xffffffffu);
    inside |= (in ? 1u : 0u) << k;
    sure |= (ok ? 1u : 0u) << k;
    cand |= (ok && cd ? 1u : 0u) << k;
  }
  n1 += __popc(sure);
  // exceptions: uncertain points, and sure survivors that may be the farthest
  const uint32_t exc = (~(sure | inside) | cand) & ((1u << B) - 1u);
  if (exc == 0) return;
#pragma unroll
  for (int k = 0; k < B; ++k) {
    if (!((exc >> k) & 1u)) continue;
    if (!((sure >> k) & 1u)) {  // uncertain (~2e-4 of the points): listed for the exact pass
      const uint32_t slot = atomicAdd(exc_n, 1u);
      if (slot < exc_cap) exc_list[slot] = idx[k];
      code[k] = kSpNoCode;  // k_sp_f2_patch writes its code
    } else {  // may be (or tie) the farthest point
      const uint64_t d2 = dbits(dist2_rn(__dsub_rn(x[k], q.ax), __dsub_rn(y[k], q.ay)));
      const uint32_t i = idx[k];
      if (bidx == 0xffffffffu || d2 > bd2) { bd2 = d2; bidx = i; bties = 1; }
      else if (d2 == bd2) { ++bties; if (i < bidx) bidx = i; }
    }
  }
}

// ===========================================================================
// F2: round 1 + bucket histogram + argmax dist2 + hash-partition counts.
// The quad test is classify_quad (prefilter.hpp:47-63); n_after_round1 counts
// every survivor (pipeline.hpp:93); points equal to the anchor leave the
// buffer (annotate, angular.hpp:118-133) and are not bucketed.
// kHist = false: no shared-memory histogram (the codes are counted by
// k_sp_hist_codes), so two CTAs fit an SM.
template <bool kVec, bool kHist>
__global__ void __launch_bounds__(kSpThreads, kHist ? 1 : 2) k_sp_hist(
    const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n,
    const ExtResult* __restrict__ ext, const double* __restrict__ cdf,
    const double* __restrict__ th, uint16_t* __restrict__ codes, uint32_t* __restrict__ hist_part,
    SpD2* __restrict__ d2part, Counters* __restrict__ ctr, const SpState* __restrict__ st) {
  pdl_wait();
  extern __shared__ uint32_t s_hist[];  // kSpBuckets (kHist)
  if (st->fail) return;  // declined from the sample (k_sp_cdf)
  __shared__ double s_cdf[kSpCells + 1];
  if (kHist)
    for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) s_hist[b] = 0;
  for (uint32_t j = threadIdx.x; j <= kSpCells; j += blockDim.x) s_cdf[j] = cdf[j];
  SpQuad q;
  load_quad(ext, q);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  uint32_t n1 = 0, bidx = 0xffffffffu, bties = 0;
  uint64_t bd2 = 0;
  auto visit = [&](double x, double y, uint32_t i) -> uint32_t {
    if (!quad_keep(q.qx, q.qy, q.ex, q.ey, x, y)) return kSpNoCode;
    ++n1;
    if (x == q.ax && y == q.ay) return kSpNoCode;
    const double dx = __dsub_rn(x, q.ax), dy = __dsub_rn(y, q.ay);
    const uint32_t b = sp_bucket(dx, dy, s_cdf, th);
    if (kHist) atomicAdd(&s_hist[b], 1u);
    const uint64_t d2 = dbits(dist2_rn(dx, dy));
    if (bidx == 0xffffffffu || d2 > bd2) { bd2 = d2; bidx = i; bties = 1; }
    else if (d2 == bd2) { ++bties; if (i < bidx) bidx = i; }
    return b;
  };
  {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nth = gridDim.x * blockDim.x;
    if (kVec) {
      const double2* x2 = reinterpret_cast<const double2*>(xs);
      const double2* y2 = reinterpret_cast<const double2*>(ys);
      uint32_t* c2 = reinterpret_cast<uint32_t*>(codes);
      const uint32_t np = n / 2;
      uint32_t p = tid;
      constexpr int kP = kHist ? 4 : 2;  // the split variant runs twice the warps
      for (; p + (kP - 1) * nth < np; p += kP * nth) {
        double2 vx[kP], vy[kP];
#pragma unroll
        for (int u = 0; u < kP; ++u) {
          vx[u] = __ldcs(&x2[p + u * nth]);
          vy[u] = __ldcs(&y2[p + u * nth]);
        }
        if (kHist) {
#pragma unroll
          for (int g = 0; g < kP; g += 2) {  // batches of 4 points (8 measured slower)
            const double bx[4] = {vx[g].x, vx[g].y, vx[g + 1].x, vx[g + 1].y};
            const double by[4] = {vy[g].x, vy[g].y, vy[g + 1].x, vy[g + 1].y};
            const uint32_t i0 = 2 * (p + g * nth), i1 = 2 * (p + (g + 1) * nth);
            const uint32_t bi[4] = {i0, i0 + 1, i1, i1 + 1};
            uint32_t bc[4];
            f2_batch<4, kHist>(bx, by, bi, bc, q, s_cdf, th, s_hist, n1, bd2, bidx, bties);
            c2[p + g * nth] = bc[0] | (bc[1] << 16);
            c2[p + (g + 1) * nth] = bc[2] | (bc[3] << 16);
          }
        } else {
#pragma unroll
          for (int g = 0; g < kP; ++g) {  // 2-point batches: 64 registers
            const double bx[2] = {vx[g].x, vx[g].y};
            const double by[2] = {vy[g].x, vy[g].y};
            const uint32_t i0 = 2 * (p + g * nth);
            const uint32_t bi[2] = {i0, i0 + 1};
            uint32_t bc[2];
            f2_batch<2, kHist>(bx, by, bi, bc, q, s_cdf, th, s_hist, n1, bd2, bidx, bties);
            c2[p + g * nth] = bc[0] | (bc[1] << 16);
          }
        }
      }
      for (; p < np; p += nth) {
        const double2 vx = __ldcs(&x2[p]), vy = __ldcs(&y2[p]);
        const uint32_t c0 = visit(vx.x, vy.x, 2 * p);
        const uint32_t c1 = visit(vx.y, vy.y, 2 * p + 1);
        c2[p] = c0 | (c1 << 16);
      }
      if ((n & 1) && tid == nth - 1) codes[n - 1] = (uint16_t)visit(xs[n - 1], ys[n - 1], n - 1);
    } else {
      for (uint32_t i = tid; i < n; i += nth) codes[i] = (uint16_t)visit(xs[i], ys[i], i);
    }
  }
  // block reductions: n1 (sum), (d2 max, ties)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    const uint64_t od = __shfl_xor_sync(0xffffffffu, bd2, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const uint32_t ot = __shfl_xor_sync(0xffffffffu, bties, o);
    if (oi != 0xffffffffu) {
      if (bidx == 0xffffffffu || od > bd2) { bd2 = od; bidx = oi; bties = ot; }
      else if (od == bd2) { bties += ot; if (oi < bidx) bidx = oi; }
    }
  }
  __shared__ uint64_t s_d[32];
  __shared__ uint32_t s_i[32], s_t[32], s_n[32];
  if (lane == 0) { s_d[warp] = bd2; s_i[warp] = bidx; s_t[warp] = bties; s_n[warp] = n1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tot += s_n[w];
      if (w == 0) continue;
      if (s_i[w] == 0xffffffffu) continue;
      if (bidx == 0xffffffffu || s_d[w] > bd2) { bd2 = s_d[w]; bidx = s_i[w]; bties = s_t[w]; }
      else if (s_d[w] == bd2) { bties += s_t[w]; if (s_i[w] < bidx) bidx = s_i[w]; }
    }
    d2part[blockIdx.x] = SpD2{bd2, bidx, bidx == 0xffffffffu ? 0u : bties};
    if (tot) atomicAdd(&ctr->n1, tot);
  }
  if (kHist) {
    uint32_t* hp = hist_part + (size_t)blockIdx.x * kSpBuckets;
    for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) hp[b] = s_hist[b];
  }
}

// F2 as a bulk-copy pipeline (the default for aligned inputs): one CTA per
// SM, kF2Cons consumer threads plus one producer warp. The producer streams
// tiles of kF2Tile points of xs and ys into a kF2Stages-deep shared-memory
// ring with cp.async.bulk, completed on full[] mbarriers; each consumer warp
// releases a stage on empty[] when it is done with it, so there is no
// CTA-wide barrier per tile and the bytes in flight (kF2Stages x 32 KB per
// SM) do not depend on registers or occupancy. Tiles go to CTAs round-robin;
// the remainder (< one tile) is read directly by the last CTA. The per-point
// work is the F2 screen with its exact fallback (f2_point / f2_exact);
// outputs are identical to k_sp_hist<kVec, false>.
#ifndef GSCAN_F2_CONS
#define GSCAN_F2_CONS 512
#endif
#ifndef GSCAN_F2_PAIRS
#define GSCAN_F2_PAIRS 3
#endif
// threads per CTA (all consumers; one CTA per SM) and point pairs per thread
// per tile. Measured on C2 (us): 512x3 103.6, 512x2 107.3, 384x3 109.3,
// 256x4 111.9, 768x1 117.7, 640x1 124.1, 1024x1 128.2: the FP64/FP32 chains
// of several points per thread interleave, more warps with fewer points do not
constexpr int kF2Cons = GSCAN_F2_CONS;
constexpr int kF2Pairs = GSCAN_F2_PAIRS;
constexpr int kF2Tile = 2 * kF2Pairs * kF2Cons;
constexpr int kF2Stages = 4;
using F2Ring = XYRing<kF2Tile, kF2Stages>;
constexpr size_t kF2RingSmem = F2Ring::kSmem + (size_t)(kSpCells + 1) * 16;

__global__ void __launch_bounds__(kF2Cons, 1) k_sp_hist_ring(
    const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n,
    const ExtResult* __restrict__ ext, const double* __restrict__ cdf,
    const double* __restrict__ th, uint16_t* __restrict__ codes, SpD2* __restrict__ d2part,
    Counters* __restrict__ ctr, SpState* __restrict__ st, uint32_t* __restrict__ exc_list,
    uint32_t exc_cap) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char f2_smem[];
  if (st->fail) return;  // declined from the sample (k_sp_cdf)
  F2Ring ring;
  ring.setup(f2_smem + (size_t)(kSpCells + 1) * 16, xs, ys, n);
  float4* s_tab = reinterpret_cast<float4*>(f2_smem);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ring.start();
  f2_table_setup(cdf, s_tab, threadIdx.x, blockDim.x);
  SpQuad q;
  load_quad(ext, q);
  F2Float F;
  f2_float_setup(q, F);
  __syncthreads();
  uint32_t n1 = 0, bidx = 0xffffffffu, bties = 0;
  uint64_t bd2 = 0;
  float thr = F.thr0;
  uint32_t* c2 = reinterpret_cast<uint32_t*>(codes);
#ifndef GSCAN_F2_DEBUG
#define GSCAN_F2_DEBUG 0  // 1: no compute (ring + stores only), 2: no memory (tile 0 reused)
#endif
  for (uint32_t k = 0; k < ring.mine; ++k) {
    if (GSCAN_F2_DEBUG != 2 || k == 0) ring.wait(GSCAN_F2_DEBUG == 2 ? 0 : k);
    const double2* x2 = reinterpret_cast<const double2*>(ring.tx(GSCAN_F2_DEBUG == 2 ? 0 : k));
    const double2* y2 = reinterpret_cast<const double2*>(ring.ty(k));
    const uint32_t i0 = ring.tile_start(k);
    double2 vx[kF2Pairs], vy[kF2Pairs];
#pragma unroll
    for (int u = 0; u < kF2Pairs; ++u) {
      vx[u] = x2[threadIdx.x + u * kF2Cons];
      vy[u] = y2[threadIdx.x + u * kF2Cons];
    }
    if (GSCAN_F2_DEBUG != 2) ring.release(k);
    if (GSCAN_F2_DEBUG == 1) {
#pragma unroll
      for (int u = 0; u < kF2Pairs; ++u)
        c2[i0 / 2 + threadIdx.x + u * kF2Cons] = vx[u].x > 2.0 || vy[u].y > 2.0 ? 1u : 0u;
      continue;
    }
    double bx[2 * kF2Pairs], by[2 * kF2Pairs];
    uint32_t bi[2 * kF2Pairs], bc[2 * kF2Pairs];
#pragma unroll
    for (int u = 0; u < kF2Pairs; ++u) {
      bx[2 * u] = vx[u].x; bx[2 * u + 1] = vx[u].y;
      by[2 * u] = vy[u].x; by[2 * u + 1] = vy[u].y;
      bi[2 * u] = i0 + 2 * (threadIdx.x + u * kF2Cons);
      bi[2 * u + 1] = bi[2 * u] + 1;
    }
    f2_points<2 * kF2Pairs>(bx, by, bi, bc, q, F, s_tab, cdf, th, n1, bd2, bidx, bties, thr,
                            exc_list, exc_cap, &st->n_exc);
#pragma unroll
    for (int u = 0; u < kF2Pairs; ++u) c2[bi[2 * u] / 2] = bc[2 * u] | (bc[2 * u + 1] << 16);
    // warp-wide screen threshold: a point below the warp's best cannot be the
    // maximum or tie it (non-negative float bits order as the values)
    const float mine_t = bidx != 0xffffffffu ? f2_thr(bitsd(bd2)) : 0.f;
    thr = fmaxf(thr, __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(mine_t))));
  }
  // remainder (< one tile): listed for the exact pass as well
  if (blockIdx.x == gridDim.x - 1) {
    for (uint32_t i = (n / kF2Tile) * kF2Tile + threadIdx.x; i < n; i += kF2Cons) {
      const uint32_t slot = atomicAdd(&st->n_exc, 1u);
      if (slot < exc_cap) exc_list[slot] = i;
    }
  }
  // block reductions: n1 (sum), (d2 max, ties) -- as k_sp_hist
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    const uint64_t od = __shfl_xor_sync(0xffffffffu, bd2, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const uint32_t ot = __shfl_xor_sync(0xffffffffu, bties, o);
    if (oi != 0xffffffffu) {
      if (bidx == 0xffffffffu || od > bd2) { bd2 = od; bidx = oi; bties = ot; }
      else if (od == bd2) { bties += ot; if (oi < bidx) bidx = oi; }
    }
  }
  __shared__ uint64_t s_d[32];
  __shared__ uint32_t s_i[32], s_t[32], s_n[32];
  if (lane == 0) { s_d[warp] = bd2; s_i[warp] = bidx; s_t[warp] = bties; s_n[warp] = n1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tot += s_n[w];
      if (w == 0) continue;
      if (s_i[w] == 0xffffffffu) continue;
      if (bidx == 0xffffffffu || s_d[w] > bd2) { bd2 = s_d[w]; bidx = s_i[w]; bties = s_t[w]; }
      else if (s_d[w] == bd2) { bties += s_t[w]; if (s_i[w] < bidx) bidx = s_i[w]; }
    }
    d2part[blockIdx.x] = SpD2{bd2, bidx, bidx == 0xffffffffu ? 0u : bties};
    if (tot) atomicAdd(&ctr->n1, tot);
  }
}

// F2's exact pass over the points its screen left uncertain (and the tail
// of the last tile): f2_exact per listed point -- round-1 survival, bucket
// code (a 2-byte store; F2 wrote kSpNoCode there), its dist2 into this
// kernel's own P_l partials (d2part[blockIdx.x] of the slice passed in). A
// list that overflowed declines the call (kSpFailCap: only inputs outside
// the screen's preconditions get there).
__global__ void __launch_bounds__(256) k_sp_f2_patch(
    const double* __restrict__ xs, const double* __restrict__ ys,
    const ExtResult* __restrict__ ext, const double* __restrict__ cdf,
    const double* __restrict__ th, uint16_t* __restrict__ codes,
    const uint32_t* __restrict__ exc_list, uint32_t exc_cap, SpD2* __restrict__ d2part,
    Counters* __restrict__ ctr, SpState* __restrict__ st) {
  pdl_wait();
  if (st->fail) return;
  const uint32_t ne = st->n_exc;
  if (ne > exc_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 11u); }
    return;
  }
  SpQuad q;
  load_quad(ext, q);
  uint32_t n1 = 0, bidx = 0xffffffffu, bties = 0;
  uint64_t bd2 = 0;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < ne; e += gridDim.x * blockDim.x) {
    const uint32_t i = exc_list[e];
    uint32_t kept;
    const uint32_t c = f2_exact(xs[i], ys[i], i, q, cdf, th, kept, bd2, bidx, bties);
    n1 += kept;
    codes[i] = (uint16_t)c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    const uint64_t od = __shfl_xor_sync(0xffffffffu, bd2, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const uint32_t ot = __shfl_xor_sync(0xffffffffu, bties, o);
    if (oi != 0xffffffffu) {
      if (bidx == 0xffffffffu || od > bd2) { bd2 = od; bidx = oi; bties = ot; }
      else if (od == bd2) { bties += ot; if (oi < bidx) bidx = oi; }
    }
  }
  __shared__ uint64_t s_d[8];
  __shared__ uint32_t s_i[8], s_t[8], s_n[8];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) { s_d[warp] = bd2; s_i[warp] = bidx; s_t[warp] = bties; s_n[warp] = n1; }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      tot += s_n[w];
      if (w == 0 || s_i[w] == 0xffffffffu) continue;
      if (bidx == 0xffffffffu || s_d[w] > bd2) { bd2 = s_d[w]; bidx = s_i[w]; bties = s_t[w]; }
      else if (s_d[w] == bd2) { bties += s_t[w]; if (s_i[w] < bidx) bidx = s_i[w]; }
    }
    d2part[blockIdx.x] = SpD2{bd2, bidx, bidx == 0xffffffffu ? 0u : bties};
    if (tot) atomicAdd(&ctr->n1, tot);
  }
}

// Bucket histogram from F2's codes (2 B/pt): per-CTA shared-memory counts.
__global__ void __launch_bounds__(1024, 1) k_sp_hist_codes(const uint16_t* __restrict__ codes,
                                                           uint32_t n, uint32_t* __restrict__ hist_part,
                                                           const SpState* __restrict__ st) {
  pdl_wait();
  extern __shared__ uint32_t s_hist[];  // kSpBuckets
  if (st->fail) return;
  for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) s_hist[b] = 0;
  __syncthreads();
  const uint4* c8 = reinterpret_cast<const uint4*>(codes);  // 8 codes per 16 B
  const uint32_t n8 = n / 8;
  const uint32_t nth = gridDim.x * blockDim.x;
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < n8; p += nth) {
    const uint4 v = __ldcs(&c8[p]);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lo = w[k] & 0xffffu, hi = w[k] >> 16;
      if (lo != kSpNoCode) atomicAdd(&s_hist[lo], 1u);
      if (hi != kSpNoCode) atomicAdd(&s_hist[hi], 1u);
    }
  }
  for (uint32_t i = n8 * 8 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth)
    if (codes[i] != kSpNoCode) atomicAdd(&s_hist[codes[i]], 1u);
  __syncthreads();
  uint32_t* hp = hist_part + (size_t)blockIdx.x * kSpBuckets;
  for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) hp[b] = s_hist[b];
}

// ceil(a / b) for b > 0
__device__ __forceinline__ uint32_t cdiv(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

// Does [lo, hi] (positions, lo <= hi) contain 1 + s*step for some s >= 0?
__device__ __forceinline__ bool has_right_seed(uint32_t lo, uint32_t hi, uint32_t step) {
  if (step == 0) return false;
  const uint32_t a = lo - 1, b = hi - 1;  // offsets from position 1
  return (b / step) * step >= a;
}
// Does [lo, hi] contain M-1 - s*step for some s >= 0?
__device__ __forceinline__ bool has_left_seed(uint32_t lo, uint32_t hi, uint32_t M, uint32_t step) {
  if (step == 0) return false;
  const uint32_t a = M - 1 - hi, b = M - 1 - lo;
  return (b / step) * step >= a;
}

// ===========================================================================
// Plan. Slices follow discard_chunked (discard.hpp:90-124): right region
// positions 1..l-1 cut every step_r = ceil((l-1)/c) from position 1; left
// region l+1..M-1 cut every step_l = ceil((M-1-l)/c) downward from M-1.
// (a) P_l from the per-CTA partials (split_regions, angular.hpp:197-204:
// first maximal dist2 -- a tie would need the exact order, so it declines).
__global__ void __launch_bounds__(256) k_sp_plan_pl(const double* __restrict__ xs,
                                                    const double* __restrict__ ys,
                                                    const SpD2* __restrict__ d2part, uint32_t nparts,
                                                    SpState* __restrict__ st,
                                                    const Counters* __restrict__ ctr, uint32_t n) {
  pdl_wait();
  // >= 90% of the points survive round 1 (near-convex input): nearly all would
  // be walk candidates, the full sort is faster (a speed decision)
  if (threadIdx.x == 0 && (uint64_t)ctr->n1 * 10 > (uint64_t)n * 9) atomicOr(&st->fail, kSpFailMany);
  // a call that declined before F2 (k_sp_cdf) or inside it left the partials
  // of an earlier call: their indices may lie beyond this input
  __syncthreads();
  if (*(volatile const uint32_t*)&st->fail) return;  // block-uniform after the barrier
  __shared__ uint64_t s_d[8];
  __shared__ uint32_t s_i[8], s_t[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t bd = 0;
  uint32_t bi = 0xffffffffu, bt = 0;
  for (uint32_t c = threadIdx.x; c < nparts; c += blockDim.x) {
    const SpD2 p = d2part[c];
    if (p.idx == 0xffffffffu) continue;
    if (bi == 0xffffffffu || p.d2 > bd) { bd = p.d2; bi = p.idx; bt = p.ties; }
    else if (p.d2 == bd) { bt += p.ties; if (p.idx < bi) bi = p.idx; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t od = __shfl_xor_sync(0xffffffffu, bd, o);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    const uint32_t ot = __shfl_xor_sync(0xffffffffu, bt, o);
    if (oi != 0xffffffffu) {
      if (bi == 0xffffffffu || od > bd) { bd = od; bi = oi; bt = ot; }
      else if (od == bd) { bt += ot; if (oi < bi) bi = oi; }
    }
  }
  if (lane == 0) { s_d[warp] = bd; s_i[warp] = bi; s_t[warp] = bt; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < 8; ++w) {
    if (s_i[w] == 0xffffffffu) continue;
    if (bi == 0xffffffffu || s_d[w] > bd) { bd = s_d[w]; bi = s_i[w]; bt = s_t[w]; }
    else if (s_d[w] == bd) { bt += s_t[w]; if (s_i[w] < bi) bi = s_i[w]; }
  }
  st->d2max = bd;
  st->l_idx = bi;
  st->ties = bt;
  if (bi == 0xffffffffu) st->fail |= kSpFailFew;
  else if (bt != 1) st->fail |= kSpFailTie;
  if (bi != 0xffffffffu) { st->lx = xs[bi]; st->ly = ys[bi]; }
}

// (b) after the bucket scan: M and P_l's bucket.
__global__ void k_sp_plan_bl(const ExtResult* __restrict__ ext, const double* __restrict__ cdf,
                             const double* __restrict__ th, const uint32_t* __restrict__ bstart,
                             SpState* __restrict__ st) {
  pdl_wait();
  if (threadIdx.x != 0) return;
  const uint32_t m = bstart[kSpBuckets];
  st->m = m;
  st->M = m + 1;
  if (st->fail) return;
  st->b_l = sp_bucket(__dsub_rn(st->lx, ext->ax), __dsub_rn(st->ly, ext->ay), cdf, th);
  // bounding box of the input: qx[0] = min x, qy[1] = min y, qx[2] = max x, qy[3] = max y
  const double wx = ext->qx[2] - ext->qx[0], wy = ext->qy[3] - ext->qy[1];
  const double d2 = (wx * wx + wy * wy) * (1.0 + 1e-9);
  st->dmax2 = d2;
  st->r02 = 1e-6 * d2;
  st->phi_lo = 0xffffffffu;
  st->phi_hi = 0u;
  st->rho2_bits = 0x7fefffffffffffffull;
}

// (c) P_l's exact position: the points of its bucket ordered before it by the
// total order (angle key, dist2, index) -- a codes-only pass; only P_l's
// bucket (~m/nb points) computes keys.
__global__ void __launch_bounds__(256) k_sp_lrank(const double* __restrict__ xs,
                                                  const double* __restrict__ ys,
                                                  const uint16_t* __restrict__ codes, uint32_t n,
                                                  uint32_t base, const ExtResult* __restrict__ ext,
                                                  SpState* __restrict__ st) {
  pdl_wait();
  // base: global index of point 0 (a shard's offset; 0 on one device)
  if (st->fail) return;
  const uint32_t b_l = st->b_l, l_idx = st->l_idx;
  const double ax = ext->ax, ay = ext->ay;
  const double ldx = __dsub_rn(st->lx, ax), ldy = __dsub_rn(st->ly, ay);
  const uint64_t lkey = angle_key(ldx, ldy);
  const double ld2 = dist2_rn(ldx, ldy);
  uint32_t below = 0;
  const uint32_t nth = gridDim.x * blockDim.x;
  auto visit = [&](uint32_t code, uint32_t i) {
    if (code != b_l || base + i == l_idx) return;
    const double dx = __dsub_rn(xs[i], ax), dy = __dsub_rn(ys[i], ay);
    below += key_less(angle_key(dx, dy), dist2_rn(dx, dy), base + i, lkey, ld2, l_idx);
  };
  // 16-byte loads (8 codes), 4 in flight; the tail below n8 * 8 point by point
  const uint4* c8 = reinterpret_cast<const uint4*>(codes);
  const uint32_t n8 = n / 8;
  const uint32_t key2 = b_l | (b_l << 16);
  for (uint32_t q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < n8; q0 += 4 * nth) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = q0 + u * nth < n8 ? __ldcs(&c8[q0 + u * nth]) : make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // SWAR test: does either 16-bit half equal b_l?
        const uint32_t x = w[k] ^ key2;
        if ((x & 0xffffu) && (x >> 16)) continue;
        const uint32_t i = 8 * (q0 + u * nth) + 2 * k;
        visit(w[k] & 0xffffu, i);
        visit(w[k] >> 16, i + 1);
      }
    }
  }
  for (uint32_t i = n8 * 8 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth)
    visit(codes[i], i);
  if (below) atomicAdd(&st->l_below, below);
}


// (e) gathered buckets: P_l's bucket and every bucket holding a seed.
__global__ void __launch_bounds__(256) k_sp_gbits(const uint32_t* __restrict__ bstart,
                                                  uint64_t chunk_count, SpState* __restrict__ st,
                                                  uint32_t* __restrict__ gbits,
                                                  uint32_t* __restrict__ glist) {
  pdl_wait();
  // a thread per bucket, a warp per bitmap word
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;  // kSpBuckets is a multiple of 256
  const uint32_t lane = threadIdx.x & 31;
  bool g = false;
  // slice geometry from the exact l (discard.hpp:90-124), computed by every
  // thread, stored by one
  bool ok = !st->fail;
  const uint32_t b_l = st->b_l, M = st->M;
  const uint32_t l = 1 + bstart[b_l] + st->l_below;
  const uint32_t cc = (uint32_t)(chunk_count < 0xffffffffull ? chunk_count : 0xffffffffull);
  const uint32_t mr = l - 1, ml = M - 1 - l;
  if (ok && (mr < 2 || ml < 2)) {
    if (b == 0) atomicOr(&st->fail, kSpFailTiny);
    ok = false;
  }
  const uint32_t sr = ok ? cdiv(mr, cc) : 1u, sl = ok ? cdiv(ml, cc) : 1u;
  if (ok && b == 0) {
    st->l = l;
    st->step_r = sr;
    st->n_right = cdiv(mr, sr);
    st->step_l = sl;
    st->n_left = cdiv(ml, sl);
  }
  if (ok) {
    const uint32_t lo = 1 + bstart[b], hi = bstart[b + 1];
    if (hi >= lo) {  // non-empty
      g = (b == b_l);
      if (b < b_l) g = has_right_seed(lo, hi, sr);
      if (b > b_l) g = has_left_seed(lo, hi, M, sl);
    }
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, g);
  if (lane == 0) gbits[b >> 5] = bits;
  uint32_t at = 0;
  if (lane == 0 && bits) at = atomicAdd(&st->n_gb, (uint32_t)__popc(bits));
  at = __shfl_sync(0xffffffffu, at, 0);
  if (g) glist[at + __popc(bits & lanemask_lt())] = b;
}

__device__ __forceinline__ bool sp_gathered(const uint32_t* g, uint32_t b) {
  return (g[b >> 5] >> (b & 31)) & 1u;
}

// Per-CTA emission regions: CTA c of a streaming pass owns slots
// [c * cap, (c + 1) * cap); cap bounds the points one CTA visits. Slots are
// claimed with a shared-memory counter (warp-aggregated), so the streaming
// loops never wait on a global atomic.
__device__ __forceinline__ uint32_t warp_claim(uint32_t* s_counter, bool want) {
  const uint32_t act = __activemask();
  const uint32_t em = __ballot_sync(act, want);
  if (!em) return 0;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(em) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(s_counter, (uint32_t)__popc(em));
  base = __shfl_sync(act, base, leader);
  return base + __popc(em & lanemask_lt());
}

// Full-warp claim of cnt slots per lane: one shared-memory atomic per warp;
// returns this lane's first slot. All 32 lanes must call it.
__device__ __forceinline__ uint32_t warp_scan_claim(uint32_t* s_counter, uint32_t cnt, uint32_t lane) {
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  uint32_t base = 0;
  if (lane == 31 && incl) base = atomicAdd(s_counter, incl);
  base = __shfl_sync(0xffffffffu, base, 31);
  return base + incl - cnt;
}

// ===========================================================================
// F3: gathered points are emitted (index, bucket); other survivors fold phi
// into the per-CTA bucket maximum; every bucketed survivor's 64-bit hash goes
// to the CTA's hash list, counted per partition.
// kMax = false: no shared-memory bucket maxima (k_sp_phimax_codes computes
// them from the stored phi), so the CTA runs 1024 threads.
#ifndef GSCAN_F3_THREADS
#define GSCAN_F3_THREADS 512
#endif
#ifndef GSCAN_F3_P
#define GSCAN_F3_P 4
#endif
// F3 (k_sp_phi with the bucket maxima): 512 threads, 4 point pairs in flight.
// Measured on C2 (k_sp_phi 187 us): 640 threads 191 us, 768 threads 207 us
// (80 registers), 1024 threads with 2 pairs 187 us -- more warps do not help.
constexpr int kSpF3Threads = GSCAN_F3_THREADS;
template <bool kVec, bool kMax>
__global__ void __launch_bounds__(kMax ? kSpF3Threads : 1024, 1) k_sp_phi(
    const double* __restrict__ xs, const double* __restrict__ ys,
    const uint16_t* __restrict__ codes, uint32_t n, uint32_t cap, const ExtResult* __restrict__ ext,
    const uint32_t* __restrict__ gbits, SpState* __restrict__ st, uint32_t* __restrict__ phi_part,
    uint32_t* __restrict__ g_idx, uint32_t* __restrict__ g_b, uint32_t* __restrict__ g_count,
    double* __restrict__ g_x, double* __restrict__ g_y,  // gathered coordinates (same slots)
    uint64_t* __restrict__ hlist, uint32_t* __restrict__ h_count, uint32_t* __restrict__ part_cnt,
    float* __restrict__ phi32, uint32_t pad) {
  pdl_wait();
  // pad = 3: the partition counts are written rounded up to whole sectors (4
  // entries; k_sp_dup_part<true>), pad = 0: exact (the sharded exchange)
  extern __shared__ uint32_t s_phi[];  // kSpBuckets (kMax)
  __shared__ uint32_t s_g[kSpBuckets / 32];
  __shared__ uint32_t s_part[2][kSpParts];  // per half-CTA hash list
  __shared__ uint32_t s_ng, s_nh[2];
  if (st->fail) return;
  if (kMax)
    for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) s_phi[b] = 0;
  for (uint32_t w = threadIdx.x; w < kSpBuckets / 32; w += blockDim.x) s_g[w] = gbits[w];
  for (uint32_t p = threadIdx.x; p < 2 * kSpParts; p += blockDim.x) s_part[0][p] = 0;
  if (threadIdx.x == 0) { s_ng = 0; s_nh[0] = 0; s_nh[1] = 0; }
  // two hash lists per CTA (threads [0, 256) and [256, 512)) of cap / 2 slots
  // each, so the duplicate check's work items are finer than the CTAs
  const uint32_t half = threadIdx.x >= blockDim.x / 2 ? 1u : 0u;
  const size_t hbase = (size_t)(2 * blockIdx.x + half) * (cap / 2);
  const double lx = st->lx, ly = st->ly;
  const double ux = __dsub_rn(ext->ax, lx), uy = __dsub_rn(ext->ay, ly);
  const uint32_t b_l = st->b_l;
  const double r02 = st->r02;
  const size_t base = (size_t)blockIdx.x * cap;
  float plo = 3.0f, phi_ = -3.0f;  // phi range, already rounded outward (rd / ru)
  __syncthreads();
  auto visit = [&](double x, double y, uint32_t b, uint32_t i) {
    const bool surv = b != kSpNoCode;
    bool emit = false;
    uint64_t h = 0;
    if (surv) {
      h = coord_hash64(x, y);
      atomicAdd(&s_part[half][(uint32_t)(h >> (64 - kSpPartBits))], 1u);
      double v2;
      const double raw = sp_phi_raw(x, y, lx, ly, ux, uy, &v2);
      plo = fminf(plo, __double2float_rd(raw));
      phi_ = fmaxf(phi_, __double2float_ru(raw));
      if (sp_gathered(s_g, b)) {
        emit = true;
      } else if (v2 >= r02) {  // points within r0 of P_l never raise a maximum (certificate)
        // stored signed and rounded down: the value the bucket maxima take,
        // within the certificate's storage error (kSpPhiStoreErr, |phi| < 2)
        const float sv = __double2float_rd(b < b_l ? raw : -raw);
        if (kMax) atomicMax(&s_phi[b], ord_f(sv));
        phi32[i] = sv;  // F4 reads it instead of recomputing
      } else {
        phi32[i] = __int_as_float(0x7fc00000);  // NaN: always a candidate
      }
    }
    const uint32_t jh = warp_claim(&s_nh[half], surv);
    if (surv) hlist[hbase + jh] = h;
    const uint32_t jg = warp_claim(&s_ng, emit);
    if (emit) { g_idx[base + jg] = i; g_b[base + jg] = b; g_x[base + jg] = x; g_y[base + jg] = y; }
  };
  // batch of 4 points: the same work as visit() in branch-free phases, and one
  // warp-scan claim per batch instead of a ballot claim per point
  auto batch = [&](const double (&x)[4], const double (&y)[4], const uint32_t (&b)[4],
                   const uint32_t (&idx)[4]) {
    double raw[4], v2[4];
    uint64_t h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      h[k] = coord_hash64(x[k], y[k]);
      const double vx = __dsub_rn(x[k], lx), vy = __dsub_rn(y[k], ly);
      v2[k] = __fma_rn(vx, vx, __dmul_rn(vy, vy));
      const double c = __fma_rn(ux, vx, __dmul_rn(uy, vy));
      const double sn = __fma_rn(ux, vy, -__dmul_rn(uy, vx));
      const double den = fabs(c) + fabs(sn);
      const bool okd = den > 1e-290;
      const double t = 1.0 - c * sp_rcp(okd ? den : 1.0);
      raw[k] = okd ? (sn >= 0.0 ? t : -t) : 0.0;  // sp_phi_raw
    }
    uint32_t nh = 0, ng = 0;
    bool gat[4];
    float pv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool surv = b[k] != kSpNoCode;
      gat[k] = false;
      pv[k] = 0.0f;  // read by F4 only for bucketed, non-gathered points
      if (!surv) continue;
      ++nh;
      atomicAdd(&s_part[half][(uint32_t)(h[k] >> (64 - kSpPartBits))], 1u);
      plo = fminf(plo, __double2float_rd(raw[k]));
      phi_ = fmaxf(phi_, __double2float_ru(raw[k]));
      gat[k] = sp_gathered(s_g, b[k]);
      if (gat[k]) {
        ++ng;
      } else if (v2[k] >= r02) {  // points within r0 of P_l never raise a maximum (certificate)
        const float sv = __double2float_rd(b[k] < b_l ? raw[k] : -raw[k]);
        if (kMax) atomicMax(&s_phi[b[k]], ord_f(sv));
        pv[k] = sv;  // F4 reads it instead of recomputing
      } else {
        pv[k] = __int_as_float(0x7fc00000);  // NaN: always a candidate
      }
    }
    // every point's slot is written (whole sectors: no read-for-merge of
    // partially written ones when L2 evicts them)
#pragma unroll
    for (int k = 0; k < 4; ++k) phi32[idx[k]] = pv[k];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t at = warp_scan_claim(&s_nh[half], nh, lane);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (b[k] != kSpNoCode) hlist[hbase + at++] = h[k];
    if (__any_sync(0xffffffffu, ng != 0)) {
      uint32_t ag = warp_scan_claim(&s_ng, ng, lane);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (gat[k]) {
          g_idx[base + ag] = idx[k];
          g_b[base + ag] = b[k];
          g_x[base + ag] = x[k];
          g_y[base + ag] = y[k];
          ++ag;
        }
    }
  };
  {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nth = gridDim.x * blockDim.x;
    const uint32_t lane = threadIdx.x & 31;
    if (kVec) {
      const double2* x2 = reinterpret_cast<const double2*>(xs);
      const double2* y2 = reinterpret_cast<const double2*>(ys);
      const uint32_t* c2 = reinterpret_cast<const uint32_t*>(codes);
      const uint32_t np = n / 2;
      uint32_t p = tid;
      constexpr int kP = kMax ? GSCAN_F3_P : 2;  // fewer loads in flight at 32 warps
      // warp-uniform bound: the batch claims are warp-synchronous
      for (; (p - lane) + 31 + (kP - 1) * nth < np; p += kP * nth) {
        double2 vx[kP], vy[kP];
        uint32_t vc[kP];
#pragma unroll
        for (int u = 0; u < kP; ++u) vc[u] = __ldcs(&c2[p + u * nth]);
#pragma unroll
        for (int u = 0; u < kP; ++u) {
          vx[u] = __ldcs(&x2[p + u * nth]);
          vy[u] = __ldcs(&y2[p + u * nth]);
        }
#pragma unroll
        for (int g = 0; g < kP; g += 2) {
          const double bx[4] = {vx[g].x, vx[g].y, vx[g + 1].x, vx[g + 1].y};
          const double by[4] = {vy[g].x, vy[g].y, vy[g + 1].x, vy[g + 1].y};
          const uint32_t bb[4] = {vc[g] & 0xffffu, vc[g] >> 16, vc[g + 1] & 0xffffu, vc[g + 1] >> 16};
          const uint32_t i0 = 2 * (p + g * nth), i1 = 2 * (p + (g + 1) * nth);
          const uint32_t bi[4] = {i0, i0 + 1, i1, i1 + 1};
          batch(bx, by, bb, bi);
        }
      }
      for (; p < np; p += nth) {
        const uint32_t vc = c2[p];
        const double2 vx = __ldcs(&x2[p]), vy = __ldcs(&y2[p]);
        visit(vx.x, vy.x, vc & 0xffffu, 2 * p);
        visit(vx.y, vy.y, vc >> 16, 2 * p + 1);
      }
      if ((n & 1) && tid == nth - 1) visit(xs[n - 1], ys[n - 1], (uint32_t)codes[n - 1], n - 1);
    } else {
      for (uint32_t i = tid; i < n; i += nth) visit(xs[i], ys[i], (uint32_t)codes[i], i);
    }
  }
  __syncthreads();
  if (kMax) {
    uint32_t* pp = phi_part + (size_t)blockIdx.x * kSpBuckets;
    for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) pp[b] = s_phi[b];
  }
  for (uint32_t p = threadIdx.x; p < kSpParts; p += blockDim.x)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh)  // partition-major over the 2G lists
      part_cnt[(size_t)p * 2 * gridDim.x + 2 * blockIdx.x + hh] = (s_part[hh][p] + pad) & ~pad;
  if (threadIdx.x == 0) {
    g_count[blockIdx.x] = s_ng;
    h_count[2 * blockIdx.x] = s_nh[0];
    h_count[2 * blockIdx.x + 1] = s_nh[1];
    atomicAdd(&st->n_g, s_ng);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    plo = fminf(plo, __shfl_xor_sync(0xffffffffu, plo, o));
    phi_ = fmaxf(phi_, __shfl_xor_sync(0xffffffffu, phi_, o));
  }
  if ((threadIdx.x & 31) == 0 && plo <= phi_) {
    atomicMin(&st->phi_lo, ord_f(plo));
    atomicMax(&st->phi_hi, ord_f(phi_));
  }
}

// Bucket maxima of the stored walk angles (F3 with kMax = false): a light
// pass over the codes and phi (6 B/pt) with the shared-memory maxima F3
// would have kept. Gathered buckets and points within r0 (NaN) are skipped.
__global__ void __launch_bounds__(1024, 1) k_sp_phimax_codes(const uint16_t* __restrict__ codes,
                                                             const float* __restrict__ phi32,
                                                             const uint32_t* __restrict__ gbits,
                                                             uint32_t n, const SpState* __restrict__ st,
                                                             uint32_t* __restrict__ phi_part) {
  pdl_wait();
  extern __shared__ uint32_t s_phi[];  // kSpBuckets
  __shared__ uint32_t s_g[kSpBuckets / 32];
  if (st->fail) return;
  for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) s_phi[b] = 0;
  for (uint32_t w = threadIdx.x; w < kSpBuckets / 32; w += blockDim.x) s_g[w] = gbits[w];
  __syncthreads();
  auto visit = [&](uint32_t b, float ph) {
    if (b != kSpNoCode && !sp_gathered(s_g, b) && !isnan(ph)) atomicMax(&s_phi[b], ord_f(ph));
  };
  const uint4* c8 = reinterpret_cast<const uint4*>(codes);
  const float4* p4 = reinterpret_cast<const float4*>(phi32);
  const uint32_t n8 = n / 8, nth = gridDim.x * blockDim.x;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n8; q += nth) {
    const uint4 c = __ldcs(&c8[q]);
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    if (((w[0] & w[1] & w[2] & w[3]) == 0xffffffffu)) continue;  // no survivor among the 8
    const float4 a = __ldcs(&p4[2 * q]), bq = __ldcs(&p4[2 * q + 1]);
    const float f[8] = {a.x, a.y, a.z, a.w, bq.x, bq.y, bq.z, bq.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      visit(w[k] & 0xffffu, f[2 * k]);
      visit(w[k] >> 16, f[2 * k + 1]);
    }
  }
  for (uint32_t i = n8 * 8 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth)
    visit(codes[i], phi32[i]);
  __syncthreads();
  uint32_t* pp = phi_part + (size_t)blockIdx.x * kSpBuckets;
  for (uint32_t b = threadIdx.x; b < kSpBuckets; b += blockDim.x) pp[b] = s_phi[b];
}

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// Side-stream work distribution. The side kernels run one CTA per SM with
// enough shared memory reserved that no Graham-tail CTA fits beside them;
// CTAs placed on the first n_free SMs leave at once, so those SMs stay free
// for the main stream's latency-bound kernels. Work items come from a ticket.
__device__ __forceinline__ bool side_take(uint32_t* ticket, uint32_t* s_item, uint32_t n_items,
                                          uint32_t& w) {
  if (threadIdx.x == 0) *s_item = atomicAdd(ticket, 1u);
  __syncthreads();
  w = *s_item;
  __syncthreads();  // everyone has read it (and finished the previous item)
  return w < n_items;
}

// Duplicate check, step 1: work item c moves hash list c (F3-CTA c / 2, half
// c % 2; cap slots each) into the partitions. The list's run of partition p
// starts at the partition-major exclusive scan of the counts (part_off[p * C
// + c]); the CTA owns those runs, so the cursors live in shared memory.
// Chunks of kSpPartChunk entries are grouped by partition in shared memory and
// written run by run.
// kPad (the single-GPU check): the counts were rounded up to whole 32-byte
// sectors (4 entries) by k_sp_phi, and every store covers whole, aligned
// sectors: a partition's last count % 4 entries of a chunk are carried to the
// next chunk in shared memory, and the list's final carries are written with
// ~0 padding (skipped by k_sp_dups). Stores of partial sectors cost DRAM
// read-for-merge traffic that slowed the concurrent main path by ~60 us.
constexpr size_t kSpDupPartSmemPad = ((size_t)kSpPartChunk + 3 * kSpParts) * 8 +
                                     (size_t)kSpParts * 3 * 8 + (size_t)kSpParts * 6 * 4;

template <bool kPad>
__global__ void __launch_bounds__(1024) k_sp_dup_part(const uint64_t* __restrict__ hlist,
                                                      const uint32_t* __restrict__ h_count,
                                                      uint32_t cap, uint32_t C,
                                                      const uint32_t* __restrict__ part_off,
                                                      const SpState* __restrict__ st,
                                                      uint64_t* __restrict__ parted,
                                                      uint32_t* __restrict__ ticket, uint32_t n_free,
                                                      const uint64_t* __restrict__ list_base) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr uint32_t kOut = kSpPartChunk + (kPad ? 3 * kSpParts : 0);
  uint64_t* s_out = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_carry = s_out + kOut;  // [p * 3 + i] (kPad)
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_carry + (kPad ? 3 * kSpParts : 0));
  uint32_t* s_off = s_cnt + kSpParts;   // where the chunk's entries of p go in s_out
  uint32_t* s_cur = s_off + kSpParts;   // next parted slot of p
  uint32_t* s_base = s_cur + kSpParts;  // s_out index t of p -> parted[s_base[p] + t]
  uint32_t* s_cc = s_base + kSpParts;   // carried entries of p (kPad)
  uint32_t* s_lim = s_cc + kSpParts;    // s_out indices of p below s_lim[p] are stored (kPad)
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_item;
  if (st->fail || sm_id() < n_free) return;
  uint32_t c;
  while (side_take(ticket, &s_item, C, c)) {
    const uint32_t cnt = h_count[c];
    const uint64_t* src = hlist + (list_base ? list_base[c] : (size_t)c * cap);
    for (uint32_t p = threadIdx.x; p < kSpParts; p += blockDim.x) {
      s_cur[p] = part_off[(size_t)p * C + c];
      s_cnt[p] = 0;
      if (kPad) s_cc[p] = 0;
    }
    // chunk = 8 entries per thread, kept in registers with their rank among
    // the chunk's entries of the same partition (the counting atomic's return);
    // the next chunk's loads are issued before the current one is written
    uint64_t hv[8], nv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t t = threadIdx.x + u * blockDim.x;
      nv[u] = t < cnt ? src[t] : 0ull;
    }
    __syncthreads();
    for (uint32_t c0 = 0; c0 < cnt; c0 += kSpPartChunk) {
      const uint32_t len = min(kSpPartChunk, cnt - c0);
      uint32_t rk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        hv[u] = nv[u];
        const uint32_t t = threadIdx.x + u * blockDim.x;
        rk[u] = t < len ? atomicAdd(&s_cnt[(uint32_t)(hv[u] >> (64 - kSpPartBits))], 1u) : 0u;
      }
      const uint32_t n0 = c0 + kSpPartChunk;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t t = n0 + threadIdx.x + u * blockDim.x;
        nv[u] = t < cnt ? src[t] : 0ull;
      }
      __syncthreads();
      // exclusive scan of the group sizes (chunk count + carry; kSpParts = 2
      // x blockDim); the owner of partitions 2t, 2t+1 also places their
      // carries, clears their counts and advances their cursors
      uint32_t ntot;
      {
        const uint32_t q0 = 2 * threadIdx.x, q1 = q0 + 1;
        const uint32_t cc0 = kPad ? s_cc[q0] : 0u, cc1 = kPad ? s_cc[q1] : 0u;
        const uint32_t a = s_cnt[q0] + cc0, b = s_cnt[q1] + cc1;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        uint32_t x = a + b;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        // every warp scans the 32 warp totals itself (no second barrier);
        // s_w is rewritten only after the next chunk's first barrier
        uint32_t wv = s_w[lane];
        const uint32_t w0 = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, wv, o);
          if (lane >= o) wv += y;
        }
        ntot = __shfl_sync(0xffffffffu, wv, 31);
        const uint32_t wex = __shfl_sync(0xffffffffu, wv - w0, warp);  // totals of warps < warp
        const uint32_t e0 = x - (a + b) + wex, e1 = e0 + a;
        const uint32_t c0_ = s_cur[q0], c1_ = s_cur[q1];
        s_base[q0] = c0_ - e0;
        s_base[q1] = c1_ - e1;
        s_cnt[q0] = 0;
        s_cnt[q1] = 0;
        if constexpr (kPad) {
          for (uint32_t i = 0; i < cc0; ++i) s_out[e0 + i] = s_carry[q0 * 3 + i];
          for (uint32_t i = 0; i < cc1; ++i) s_out[e1 + i] = s_carry[q1 * 3 + i];
          s_off[q0] = e0 + cc0;
          s_off[q1] = e1 + cc1;
          s_lim[q0] = e0 + (a & ~3u);
          s_lim[q1] = e1 + (b & ~3u);
          s_cc[q0] = a & 3u;
          s_cc[q1] = b & 3u;
          s_cur[q0] = c0_ + (a & ~3u);
          s_cur[q1] = c1_ + (b & ~3u);
        } else {
          s_off[q0] = e0;
          s_off[q1] = e1;
          s_cur[q0] = c0_ + a;
          s_cur[q1] = c1_ + b;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t t = threadIdx.x + u * blockDim.x;
        if (t < len) s_out[s_off[(uint32_t)(hv[u] >> (64 - kSpPartBits))] + rk[u]] = hv[u];
      }
      __syncthreads();
      // the next chunk's counting touches only s_cnt, cleared above; its scan
      // rewrites the other arrays and s_out only after every thread passed
      // its first barrier, i.e. finished this loop
      for (uint32_t t = threadIdx.x; t < ntot; t += blockDim.x) {
        const uint64_t h = s_out[t];
        const uint32_t p = (uint32_t)(h >> (64 - kSpPartBits));
        if (!kPad || t < s_lim[p]) parted[s_base[p] + t] = h;
        else s_carry[p * 3 + (t - s_lim[p])] = h;
      }
    }
    __syncthreads();  // the item's carries, cursors and counters are final
    if (kPad) {  // the list's last partial sectors, padded
      for (uint32_t p = threadIdx.x; p < kSpParts; p += blockDim.x) {
        const uint32_t cc = s_cc[p];
        if (cc) {
          uint64_t* d = parted + s_cur[p];
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) d[i] = i < cc ? s_carry[p * 3 + i] : ~0ull;
        }
      }
    }
  }
}

// Duplicate check, step 2: a partition per work item, open-addressing set in
// shared memory. The CTA's kSpDupGroups thread groups take items
// independently (named barriers), so one group's load and barrier latencies
// hide behind the others' probing. A slot holds 32 bits: a 17-bit tag (hash
// bits 32..48; the slot is a range reduction of bits 0..31, the partition the
// top bits) and the entry's 15-bit index in its partition; equal tags are
// confirmed on the full 64-bit hash (one load, a few per call). An equal hash
// means a possible duplicate -> the full path (exact). Partitions over the
// table's load limit are checked in rounds over sub-ranges of the hash.
// Partitions of 2^15 entries or more (above ~67M round-1 survivors) use an
// 11-bit tag and a 21-bit index (more confirmations, same result); 2^21 - 1
// entries or more (above ~4G survivors) set kSpFailCap.
#ifndef GSCAN_DUPS_G
#define GSCAN_DUPS_G 2
#endif
constexpr uint32_t kSpDupGroups = GSCAN_DUPS_G;
constexpr uint32_t kSpDupGT = 1024 / kSpDupGroups;                       // threads per group
// slots per group table: C2 measured 16384 -> 103 us, 20480 -> 92, 24576 -> 88,
// 26624 -> 89 (k_sp_dups; shorter probe runs, the warp loops max over lanes)
#ifndef GSCAN_DUPS_SLOTS
#define GSCAN_DUPS_SLOTS (kSpDupGroups == 2 ? 24576u : 12288u)
#endif
constexpr uint32_t kSpDupGSlots = GSCAN_DUPS_SLOTS;
constexpr uint32_t kSpDupGRound = 8192;  // entries per round (load <= 1/3 at 24576 slots)
constexpr uint32_t kSpDupIdxBits = 15;     // index bits of a slot (tag: the other 17)
constexpr uint32_t kSpDupIdxBitsBig = 21;  // partitions of 2^15 entries or more
static_assert(32 + (32 - kSpDupIdxBits) <= 64 - kSpPartBits, "tag bits overlap the partition");
constexpr size_t kSpDupSmem = (size_t)kSpDupGroups * kSpDupGSlots * 4;

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ bool named_sync_or(uint32_t id, uint32_t n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\tselp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}

// One group's shared-memory hash-set pass over arr[0, n) (entries ~0 are
// sector padding): rounds of <= kSpDupGRound entries, each round the entries
// whose bits 0-15 select it (disjoint from the slot bits 18-31, the tag bits
// 32-48 and the partition bits 53-63, so a round's entries spread over the
// whole table). Equal hashes -> *dup; a skewed round -> *full.
__device__ __forceinline__ void dup_set_pass(const uint64_t* __restrict__ arr, uint32_t n,
                                             uint32_t* tab, uint32_t gt, uint32_t bar,
                                             bool& dup, bool& full, SpState* st) {
  constexpr uint32_t kGT = kSpDupGT, kB = 8;  // entries per thread per batch
#ifdef GSCAN_DUPS_FORCE_BIG  // test builds: the large-partition encoding everywhere
  const uint32_t ib = kSpDupIdxBitsBig;
#else
  const uint32_t ib = n < (1u << kSpDupIdxBits) ? kSpDupIdxBits : kSpDupIdxBitsBig;  // uniform
#endif
  const uint32_t imask = (1u << ib) - 1, tmask = (1u << (32 - ib)) - 1;
  if (n >= imask) {
    full = true;
    if (gt == 0) atomicMax(&st->why, 8u);
    return;
  }
  const uint32_t rounds = (n + kSpDupGRound - 1) / kSpDupGRound;
  for (uint32_t r = 0; r < rounds; ++r) {  // uniform over the group (named barriers)
    // the first batch's loads are in flight while the table is cleared
    uint64_t hv[kB];
#pragma unroll
    for (uint32_t u = 0; u < kB; ++u) {
      const uint32_t e = gt + u * kGT;
      hv[u] = e < n ? arr[e] : ~0ull;
    }
    named_sync(bar, kGT);  // the previous round's (or pass's) probes are done
    uint4* t4 = reinterpret_cast<uint4*>(tab);
    for (uint32_t k = gt; k < kSpDupGSlots / 4; k += kGT) t4[k] = make_uint4(~0u, ~0u, ~0u, ~0u);
    named_sync(bar, kGT);
    for (uint32_t e0 = gt; e0 < n; e0 += kB * kGT) {
      if (e0 != gt) {
#pragma unroll
        for (uint32_t u = 0; u < kB; ++u) {
          const uint32_t e = e0 + u * kGT;
          hv[u] = e < n ? arr[e] : ~0ull;
        }
      }
#pragma unroll
      for (uint32_t u = 0; u < kB; ++u) {
        const uint64_t h = hv[u];
        const uint32_t e = e0 + u * kGT;
        if (e >= n || h == ~0ull || dup || full) continue;  // ~0: sector padding
        if (rounds > 1) {
          const uint32_t mid = (uint32_t)h & 0xffffu;
          if ((uint32_t)(((uint64_t)mid * rounds) >> 16) != r) continue;
        }
        const uint32_t tag = (uint32_t)(h >> 32) & tmask;
        const uint32_t v = (tag << ib) | e;  // never ~0u: e < imask
        uint32_t slot = (uint32_t)(((uint64_t)(uint32_t)h * kSpDupGSlots) >> 32);
        for (uint32_t probe = 0;; ++probe) {
          if (probe == kSpDupGSlots / 2) {  // a skewed round
            full = true;
            atomicMax(&st->why, 9u);
            break;
          }
          const uint32_t prev = atomicCAS(&tab[slot], ~0u, v);
          if (prev == ~0u) break;
          if ((prev >> ib) == tag && arr[prev & imask] == h) {
            dup = true;
            break;
          }
          slot = slot + 1 == kSpDupGSlots ? 0u : slot + 1;
        }
      }
    }
  }
}

// Partitions of more than kSpDupMaxRounds rounds (inputs above ~100M points;
// 1B square: 322K hashes per partition, whose 40 rounds would each re-read the
// whole partition) are first split by hash bits 0-8 into up to 512
// sub-partitions of ~kSpDupSubTarget entries in a global scratch area of
// `gcap` entries per (CTA, group) (L2-resident), then each sub-partition goes
// through the shared-memory pass in about one round.
constexpr uint32_t kSpDupMaxRounds = 2;
constexpr uint32_t kSpDupSubTarget = 6144;
constexpr uint32_t kSpDupMaxSub = 512;

__global__ void __launch_bounds__(1024) k_sp_dups(const uint64_t* __restrict__ parted,
                                                 const uint32_t* __restrict__ part_off,
                                                 uint32_t nparts_cta, SpState* __restrict__ st,
                                                 uint32_t* __restrict__ ticket, uint32_t n_free,
                                                 uint64_t* __restrict__ gscr = nullptr,
                                                 uint32_t gcap = 0, bool discard = false) {
  extern __shared__ uint32_t s_tab[];  // kSpDupGroups x kSpDupGSlots
  __shared__ uint32_t s_next[kSpDupGroups];
  __shared__ uint32_t s_sub[kSpDupGroups][kSpDupMaxSub + 1];  // counts -> offsets
  __shared__ uint32_t s_cur[kSpDupGroups][kSpDupMaxSub];
  if (st->fail || sm_id() < n_free) return;
  constexpr uint32_t kGT = kSpDupGT;
  const uint32_t grp = threadIdx.x / kGT, gt = threadIdx.x % kGT, bar = 1 + grp;
  uint32_t* tab = s_tab + grp * kSpDupGSlots;
  uint32_t* sub = s_sub[grp];
  uint32_t* cur = s_cur[grp];
  uint64_t* scr = gscr ? gscr + (size_t)(blockIdx.x * kSpDupGroups + grp) * gcap : nullptr;
  const uint32_t total = part_off[(size_t)kSpParts * nparts_cta];  // the scan's total
  bool dup = false, full = false;
  if (gt == 0) s_next[grp] = atomicAdd(ticket, 1u);
  named_sync(bar, kGT);
  uint32_t p = s_next[grp];
  while (p < kSpParts) {
    const uint32_t lo = part_off[(size_t)p * nparts_cta];
    const uint32_t hi = (p + 1 < kSpParts) ? part_off[(size_t)(p + 1) * nparts_cta] : total;
    named_sync(bar, kGT);  // the group has read s_next
    // the next item's ticket is taken now and read after the closing barrier
    if (gt == 0) s_next[grp] = atomicAdd(ticket, 1u);
    const uint32_t n = hi - lo;
    const uint32_t nrounds = (n + kSpDupGRound - 1) / kSpDupGRound;
    if (scr && nrounds > kSpDupMaxRounds && n <= gcap) {
      uint32_t ns = 1;
      while (ns < kSpDupMaxSub && ns * kSpDupSubTarget < n) ns <<= 1;
      for (uint32_t k = gt; k <= ns; k += kGT) sub[k] = 0;
      named_sync(bar, kGT);
      for (uint32_t e = lo + gt; e < hi; e += kGT) {
        const uint64_t h = parted[e];
        if (h != ~0ull) atomicAdd(&sub[(uint32_t)h & (ns - 1)], 1u);
      }
      named_sync(bar, kGT);
      if (gt < 32) {  // exclusive scan of the ns counts by one warp
        uint32_t carry = 0;
        for (uint32_t base = 0; base < ns; base += 32) {
          const uint32_t v = base + gt < ns ? sub[base + gt] : 0u;
          uint32_t x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if ((int)gt >= o) x += y;
          }
          if (base + gt < ns) { sub[base + gt] = carry + x - v; cur[base + gt] = carry + x - v; }
          carry += __shfl_sync(0xffffffffu, x, 31);
        }
        if (gt == 0) sub[ns] = carry;
      }
      named_sync(bar, kGT);
      for (uint32_t e = lo + gt; e < hi; e += kGT) {
        const uint64_t h = parted[e];
        if (h != ~0ull) scr[atomicAdd(&cur[(uint32_t)h & (ns - 1)], 1u)] = h;
      }
      __threadfence_block();
      named_sync(bar, kGT);
      for (uint32_t j = 0; j < ns && !dup && !full; ++j)
        dup_set_pass(scr + sub[j], sub[j + 1] - sub[j], tab, gt, bar, dup, full, st);
    } else {
      dup_set_pass(parted + lo, n, tab, gt, bar, dup, full, st);
    }
    if (named_sync_or(bar, kGT, dup || full)) break;  // also publishes s_next
    if (discard) {
      // the partition is dead once checked: drop its whole 128-byte lines
      // from L2 without a write-back (lines shared with a neighbouring
      // partition stay); otherwise ~100 MB of dirty lines are written back
      // when the next call's first pass evicts them
      const size_t l0 = ((size_t)lo * 8 + 127) / 128, l1 = (size_t)hi * 8 / 128;
      const char* base = reinterpret_cast<const char*>(parted);
      for (size_t l = l0 + gt; l < l1; l += kGT)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(base + l * 128) : "memory");
    }
    p = s_next[grp];
  }
  if (dup) { atomicAdd(&st->dups, 1u); atomicOr(&st->fail, kSpFailDup); }
  if (full) atomicOr(&st->fail, kSpFailCap);
}

// Side-stream completion check. k_sp_dup_part and k_sp_dups hand out work by
// tickets and leave at once on the SMs reserved for the main stream
// (sm_id() < n_free); if the scheduler placed every CTA there (SM subsets
// under MIG/MPS, n_free >= the SM count), some lists or partitions were never
// examined. Every item is claimed before the ticket passes the item count, so
// fewer tickets than items declines the call (a possible duplicate unchecked).
__global__ void k_sp_side_check(const uint32_t* __restrict__ work, uint32_t n_lists,
                                SpState* __restrict__ st) {
  if (st->fail) return;
  if (work[0] < n_lists || work[1] < kSpParts) {
    atomicOr(&st->fail, kSpFailCap);
    atomicMax(&st->why, 10u);
  }
}

// Emitted elements (per-CTA regions) -> bucket slots start[b] + rank as
// 32-byte records {exact key, x, y, idx, bucket}; the glibc-exact atan2 runs
// here, densely. rank: arrival order (atomic on cnt[b]); with store_rank the
// rank is only recorded (first phase of a two-phase placement).
template <int kPhase>  // 0: rank + scatter (start known), 1: rank only, 2: scatter with stored rank
__global__ void __launch_bounds__(256) k_sp_emit_place(
    const double* __restrict__ xs, const double* __restrict__ ys, const uint32_t* __restrict__ e_idx,
    const uint32_t* __restrict__ e_b, uint32_t* __restrict__ e_rank,
    const uint32_t* __restrict__ e_count, uint32_t cap, uint32_t* __restrict__ cnt,
    const uint32_t* __restrict__ start, const ExtResult* __restrict__ ext,
    SpState* __restrict__ st, PtRec* __restrict__ rec,
    const double* __restrict__ e_x = nullptr, const double* __restrict__ e_y = nullptr,
    uint32_t wcap = 0xffffffffu) {
  pdl_wait();
  // e_x, e_y: the emitted points' coordinates in the region slots (F3 writes
  // them for gathered points, so no random reads of xs, ys); else xs[i], ys[i]
  if (st->fail) return;
  // the walk-side buffers hold wcap elements (large inputs, gscan.cu reserve):
  // gathered points, then gathered + candidate points, must fit
  if ((kPhase == 0 && (uint64_t)st->n_g + 2 > wcap) ||
      (kPhase == 1 && (uint64_t)st->n_g + st->n_c + 2 > wcap)) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
      atomicOr(&st->fail, kSpFailCap);
      atomicMax(&st->why, 7u);
    }
    return;
  }
  if (kPhase == 1 && st->n_c > max(st->m / kSpManyDiv, 65536u)) {
    // after F4: too many candidates (points near a circle); the full sort is
    // faster -- decline, every CTA sees the same count
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicOr(&st->fail, kSpFailMany);
    return;
  }
  const uint32_t c = blockIdx.y;
  const uint32_t ne = e_count[c];
  const size_t base = (size_t)c * cap;
  const double ax = ext->ax, ay = ext->ay;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < ne; k += gridDim.x * blockDim.x) {
    const uint32_t b = e_b[base + k];
    uint32_t r;
    if (kPhase == 2) r = e_rank[base + k];
    else r = atomicAdd(&cnt[b], 1u);
    if (kPhase == 1) { e_rank[base + k] = r; continue; }
    const uint32_t i = e_idx[base + k];
    PtRec o;
    o.x = e_x ? e_x[base + k] : xs[i];
    o.y = e_y ? e_y[base + k] : ys[i];
    o.key = angle_key(__dsub_rn(o.x, ax), __dsub_rn(o.y, ay));
    o.idx = i;
    o.pad = b;
    rec[start[b] + r] = o;
  }
}

// CTA-wide exact sort of one bucket's records (cnt <= kSpGatherCap) in shared
// memory: bitonic sort of a permutation under the total order (angle key,
// dist2, input index) -- the reference's stable (angle, dist2) order,
// angular.hpp:154-194. out(rank, x, y, idx) receives every element; returns
// true when two elements are equal points (annotate's dedup would drop one).
constexpr int kSpSortThreads = 512;
constexpr size_t kSpSortSmem = (size_t)kSpGatherCap * (8 + 8 + 8 + 8 + 4 + 2);

template <uint32_t kCap = kSpGatherCap, typename Out>
__device__ bool cta_sort_bucket(const PtRec* __restrict__ R, uint32_t cnt, double ax, double ay,
                                unsigned char* smem, Out&& out) {
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
  double* s_d2 = reinterpret_cast<double*>(s_key + kCap);
  double* s_x = s_d2 + kCap;
  double* s_y = s_x + kCap;
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_y + kCap);
  uint16_t* s_perm = reinterpret_cast<uint16_t*>(s_idx + kCap);
  uint32_t P = 32;
  while (P < cnt) P <<= 1;
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
    s_perm[t] = (uint16_t)t;
    if (t < cnt) {
      const PtRec r = ld_rec256(&R[t]);
      s_key[t] = r.key;
      s_x[t] = r.x;
      s_y[t] = r.y;
      s_idx[t] = r.idx;
      s_d2[t] = dist2_rn(__dsub_rn(r.x, ax), __dsub_rn(r.y, ay));
    }
  }
  __syncthreads();
  auto less = [&](uint32_t a, uint32_t b) -> bool {
    if (a >= cnt) return false;
    if (b >= cnt) return true;
    return key_less(s_key[a], s_d2[a], s_idx[a], s_key[b], s_d2[b], s_idx[b]);
  };
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint32_t ea = s_perm[i], eb = s_perm[ixj];
          const bool up = (i & k) == 0;
          if (up ? less(eb, ea) : less(ea, eb)) { s_perm[i] = (uint16_t)eb; s_perm[ixj] = (uint16_t)ea; }
        }
      }
      __syncthreads();
    }
  }
  bool dup = false;
  for (uint32_t r = threadIdx.x; r < cnt; r += blockDim.x) {
    const uint32_t e = s_perm[r];
    for (int32_t q = (int32_t)r - 1; q >= 0; --q) {  // equal points share (key, dist2)
      const uint32_t f = s_perm[q];
      if (s_key[f] != s_key[e] || s_d2[f] != s_d2[e]) break;
      if (s_x[f] == s_x[e] && s_y[f] == s_y[e]) { dup = true; break; }
    }
    out(r, s_x[e], s_y[e], s_idx[e]);
  }
  return dup;
}

// CTA-wide exact sort of one bucket (cnt <= kCap) in O(cnt): the angle keys
// are spread over cnt sub-buckets by linear interpolation between the
// bucket's min and max key (monotone in the key, so sub-buckets never invert
// the order), counted, and every element is ranked against the members of its
// own sub-bucket (about one) by the total order (angle key, dist2, input
// index) -- the reference's stable (angle, dist2) order, angular.hpp:154-194.
// out(rank, x, y, idx) receives every element; returns true when two elements
// are equal points (annotate's dedup would drop one). Sub-buckets above
// kSubMax members (clustered keys) flag `slow`: the caller re-sorts bitonically.
// `smem` may also be a global-memory scratch area (k_sp_sort_gathered_huge):
// the arrays are then laid out for `cap` elements instead of kCap.
// In global memory the counts and the member list are built with atomics,
// which are performed in L2: their reads bypass L1 (kGlobal, __ldcg).
template <uint32_t kCap, bool kGlobal = false, typename Out>
__device__ bool cta_sort_bucket_sub(const PtRec* __restrict__ R, uint32_t cnt, double ax, double ay,
                                    unsigned char* smem, bool* slow, Out&& out,
                                    uint32_t cap = kCap) {
  auto ld = [](const uint32_t* p) -> uint32_t { return kGlobal ? __ldcg(p) : *p; };
  constexpr uint32_t kSubMax = kCap;  // never slow: clustered keys cost O(k^2) in their group
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem);
  double* s_d2 = reinterpret_cast<double*>(s_key + cap);
  double* s_x = s_d2 + cap;
  double* s_y = s_x + cap;
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_y + cap);
  uint32_t* s_sub = s_idx + cap;     // element -> sub-bucket
  uint32_t* s_start = s_sub + cap;   // sub-bucket counts -> starts (cap + 1)
  uint32_t* s_list = s_start + cap + 1;  // members grouped by sub-bucket
  __shared__ uint64_t s_kmin, s_kmax;
  __shared__ uint32_t s_w[32], s_big;
  if (threadIdx.x == 0) { s_kmin = ~0ull; s_kmax = 0; s_big = 0; }
  __syncthreads();
  uint64_t lmin = ~0ull, lmax = 0;
  for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
    const PtRec r = ld_rec256(&R[t]);
    s_key[t] = r.key;
    s_x[t] = r.x;
    s_y[t] = r.y;
    s_idx[t] = r.idx;
    s_d2[t] = dist2_rn(__dsub_rn(r.x, ax), __dsub_rn(r.y, ay));
    lmin = r.key < lmin ? r.key : lmin;
    lmax = r.key > lmax ? r.key : lmax;
  }
  for (uint32_t t = threadIdx.x; t <= cnt; t += blockDim.x) s_start[t] = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a2 = __shfl_xor_sync(0xffffffffu, lmin, o), b2 = __shfl_xor_sync(0xffffffffu, lmax, o);
    lmin = a2 < lmin ? a2 : lmin;
    lmax = b2 > lmax ? b2 : lmax;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin((unsigned long long*)&s_kmin, (unsigned long long)lmin);
    atomicMax((unsigned long long*)&s_kmax, (unsigned long long)lmax);
  }
  __syncthreads();
  // keys are non-negative doubles: value order = bit order
  const double kmin = bitsd(s_kmin), kmax = bitsd(s_kmax);
  const double scale = (kmax > kmin) ? (double)cnt / (kmax - kmin) : 0.0;
  for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
    uint32_t j = (uint32_t)((bitsd(s_key[t]) - kmin) * scale);
    j = j < cnt ? j : cnt - 1;
    s_sub[t] = j;
    atomicAdd(&s_start[j], 1u);
  }
  __syncthreads();
  // exclusive scan of the sub-bucket counts (CTA-wide, chunked)
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t carry = 0;
    for (uint32_t base = 0; base < cnt; base += blockDim.x) {
      const uint32_t i = base + threadIdx.x;
      const uint32_t v = i < cnt ? ld(&s_start[i]) : 0u;
      if (v > kSubMax) s_big = 1;
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
      if (i < cnt) s_start[i] = carry + (warp ? s_w[warp - 1] : 0u) + x - v;
      carry += s_w[nw - 1];
      __syncthreads();
    }
    if (threadIdx.x == 0) s_start[cnt] = carry;
  }
  __syncthreads();
  if (s_big) { *slow = true; return false; }
  // group members by sub-bucket (order inside a group is irrelevant: ranks
  // come from comparisons), using s_d2's sign-free spare? no: a cursor copy
  for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
    const uint32_t j = s_sub[t];
    // claim a slot: the group's first free position (groups are tiny)
    const uint32_t g0 = ld(&s_start[j]), g1 = ld(&s_start[j + 1]);
    for (uint32_t q = g0; q < g1; ++q)
      if (atomicCAS(&s_list[q], 0xffffffffu, t) == 0xffffffffu) break;
  }
  __syncthreads();
  bool dup = false;
  for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) {
    const uint32_t j = s_sub[t];
    const uint32_t g0 = ld(&s_start[j]), g1 = ld(&s_start[j + 1]);
    const uint64_t kt = s_key[t];
    const double dt = s_d2[t];
    const uint32_t it = s_idx[t];
    uint32_t r = g0;
    for (uint32_t q = g0; q < g1; ++q) {
      const uint32_t u = ld(&s_list[q]);
      if (u == t) continue;
      r += key_less(s_key[u], s_d2[u], s_idx[u], kt, dt, it);
      dup |= (s_key[u] == kt && s_d2[u] == dt && s_x[u] == s_x[t] && s_y[u] == s_y[t]);
    }
    out(r, s_x[t], s_y[t], it);
  }
  return dup;
}

// Gathered buckets up to kSpSmallCap points (CTA per bucket, sub-bucket sort,
// 4 CTAs per SM); clustered or larger buckets go to the bitonic sorter.
// Exact positions 1 + bstart[b] + rank in the annotated-buffer space A;
// records P_l's position.
// 512 (8 CTAs/SM) measured on C2: k_sp_sort_gathered 37 -> 28 us but the
// buckets of 513-1024 points move to the big sorter (6 -> 14 us); net <= 4 us
#ifndef GSCAN_SMALL_CAP
#define GSCAN_SMALL_CAP 1024
#endif
constexpr uint32_t kSpSmallCap = GSCAN_SMALL_CAP;
constexpr int kSpSmallThreads = 256;
constexpr size_t kSpSmallSmem = (size_t)kSpSmallCap * (8 + 8 + 8 + 8 + 4 + 4 + 4 + 4) + 16;

__global__ void __launch_bounds__(kSpSmallThreads) k_sp_sort_gathered(
    const uint32_t* __restrict__ glist, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ gs, const uint32_t* __restrict__ hist,
    const uint32_t* __restrict__ gcnt,
    const PtRec* __restrict__ rec, const ExtResult* __restrict__ ext, SpState* __restrict__ st,
    uint32_t* __restrict__ big, double* __restrict__ A_x, double* __restrict__ A_y,
    uint32_t* __restrict__ A_i) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  if (st->fail) return;
  const uint32_t ngb = st->n_gb, l_idx = st->l_idx;
  const double ax = ext->ax, ay = ext->ay;
  uint32_t* s_list = reinterpret_cast<uint32_t*>(smem + (size_t)kSpSmallCap * (8 + 8 + 8 + 8 + 4 + 4)) +
                     kSpSmallCap + 1;
  for (uint32_t g = blockIdx.x; g < ngb; g += gridDim.x) {
    const uint32_t b = glist[g];
    const uint32_t s0 = bstart[b], g0 = gs[b], cnt = hist[b];
    if (gcnt[b] != cnt) {  // every point of a gathered bucket must have been emitted
      if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailInternal); atomicMax(&st->why, 1u); }
      return;
    }
    if (threadIdx.x == 0) atomicMax(&st->max_g, cnt);
    if (cnt > kSpSmallCap) {
      if (threadIdx.x == 0) big[atomicAdd(&st->n_bigg, 1u)] = b;
      continue;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) s_list[t] = 0xffffffffu;
    bool slow = false;
    const bool dup = cta_sort_bucket_sub<kSpSmallCap>(rec + g0, cnt, ax, ay, smem, &slow,
                                                      [&](uint32_t r, double x, double y, uint32_t idx) {
      const uint32_t q = 1 + g0 + r;  // storage; the position is 1 + s0 + r
      A_x[q] = x;
      A_y[q] = y;
      A_i[q] = idx;
      if (idx == l_idx) st->l_check = 1 + s0 + r;
    });
    if (slow) {
      if (threadIdx.x == 0) big[atomicAdd(&st->n_bigg, 1u)] = b;
      continue;
    }
    if (dup) atomicOr(&st->fail, kSpFailDup);
  }
}

// Gathered buckets above kSpSmallCap (up to kSpGatherCap): the same O(n)
// sub-bucket sort with a larger shared-memory footprint.
constexpr size_t kSpBigSmem = (size_t)kSpGatherCap * (8 + 8 + 8 + 8 + 4 + 4 + 4 + 4) + 16;

__global__ void __launch_bounds__(kSpSortThreads) k_sp_sort_gathered_big(
    const uint32_t* __restrict__ big, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ gs, const uint32_t* __restrict__ hist,
    const PtRec* __restrict__ rec,
    const ExtResult* __restrict__ ext, SpState* __restrict__ st, double* __restrict__ A_x,
    double* __restrict__ A_y, uint32_t* __restrict__ A_i, uint32_t* __restrict__ huge,
    uint32_t huge_cap) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  if (st->fail) return;
  const uint32_t nbig = st->n_bigg, l_idx = st->l_idx;
  const double ax = ext->ax, ay = ext->ay;
  uint32_t* s_list = reinterpret_cast<uint32_t*>(smem + (size_t)kSpGatherCap * (8 + 8 + 8 + 8 + 4 + 4)) +
                     kSpGatherCap + 1;
  for (uint32_t g = blockIdx.x; g < nbig; g += gridDim.x) {
    const uint32_t b = big[g];
    const uint32_t s0 = bstart[b], g0 = gs[b], cnt = hist[b];
    if (cnt > kSpGatherCap) {  // above the shared-memory sorter: global scratch (below)
      if (cnt > huge_cap) {  // no scratch (small input) or too large for it: decline
        if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 4u); }
        return;
      }
      if (threadIdx.x == 0) huge[atomicAdd(&st->n_hugeg, 1u)] = b;
      continue;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) s_list[t] = 0xffffffffu;
    bool slow = false;
    const bool dup = cta_sort_bucket_sub<kSpGatherCap>(rec + g0, cnt, ax, ay, smem, &slow,
                                                       [&](uint32_t r, double x, double y, uint32_t idx) {
      const uint32_t q = 1 + g0 + r;
      A_x[q] = x;
      A_y[q] = y;
      A_i[q] = idx;
      if (idx == l_idx) st->l_check = 1 + s0 + r;
    });
    if (dup) atomicOr(&st->fail, kSpFailDup);
  }
}

// Gathered buckets above kSpGatherCap (inputs above ~80M points, where the
// fixed kSpBuckets buckets hold ~n/48K points each): the same O(n)
// sub-bucket sort, its arrays in a per-CTA global-memory scratch area of
// `cap` elements (kSpHugeBytes per element, L2-resident at these sizes). A
// bucket above `cap`, or a sub-bucket above kSpGatherCap members (clustered
// keys), declines (kSpFailCap).
constexpr size_t kSpHugeBytes = 8 + 8 + 8 + 8 + 4 + 4 + 4 + 4;

__global__ void __launch_bounds__(kSpSortThreads) k_sp_sort_gathered_huge(
    const uint32_t* __restrict__ huge, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ gs, const uint32_t* __restrict__ hist,
    const PtRec* __restrict__ rec, const ExtResult* __restrict__ ext, SpState* __restrict__ st,
    double* __restrict__ A_x, double* __restrict__ A_y, uint32_t* __restrict__ A_i,
    unsigned char* __restrict__ scratch, uint32_t cap) {
  pdl_wait();
  if (st->fail) return;
  const uint32_t nh = st->n_hugeg, l_idx = st->l_idx;
  const double ax = ext->ax, ay = ext->ay;
  unsigned char* scr = scratch + (size_t)blockIdx.x * ((size_t)cap * kSpHugeBytes + 16);
  uint32_t* s_list = reinterpret_cast<uint32_t*>(scr + (size_t)cap * (8 + 8 + 8 + 8 + 4 + 4)) + cap + 1;
  for (uint32_t g = blockIdx.x; g < nh; g += gridDim.x) {
    const uint32_t b = huge[g];
    const uint32_t s0 = bstart[b], g0 = gs[b], cnt = hist[b];
    if (cnt > cap) {
      if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 4u); }
      return;
    }
    __syncthreads();
    for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) s_list[t] = 0xffffffffu;
    __threadfence_block();
    bool slow = false;
    const bool dup = cta_sort_bucket_sub<kSpGatherCap, true>(rec + g0, cnt, ax, ay, scr, &slow,
                                                       [&](uint32_t r, double x, double y, uint32_t idx) {
      const uint32_t q = 1 + g0 + r;
      A_x[q] = x;
      A_y[q] = y;
      A_i[q] = idx;
      if (idx == l_idx) st->l_check = 1 + s0 + r;
    }, cap);
    if (slow) {
      if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 6u); }
      return;
    }
    if (dup) atomicOr(&st->fail, kSpFailDup);
  }
}

// Position -> bucket (the non-empty bucket holding it: the largest b with
// bstart[b] <= pos - 1, else 0) for two positions at once, by a whole warp
// (pa, pb warp-uniform): each step the 32 lanes probe 32 evenly spaced
// buckets of the remaining range and the ballot keeps the last one at or
// below the target,
// so 4 dependent loads replace a binary search's 16 (bstart is non-decreasing;
// bucket lo of the range always qualifies).
__device__ __forceinline__ void bucket_of_pos2_warp(const uint32_t* __restrict__ bstart,
                                                    uint32_t pa, uint32_t pb, int lane,
                                                    uint32_t& ba, uint32_t& bb) {
  uint32_t la = 0, na = kSpBuckets, lb = 0, nb = kSpBuckets;
  while (na > 1 || nb > 1) {
    const uint32_t sa = (na + 31) / 32, sb = (nb + 31) / 32;
    const uint32_t qa = la + lane * sa, qb = lb + lane * sb;
    const bool oka = lane == 0 || (qa < la + na && bstart[qa] <= pa - 1);
    const bool okb = lane == 0 || (qb < lb + nb && bstart[qb] <= pb - 1);
    const uint32_t ma = __ballot_sync(0xffffffffu, oka), mb = __ballot_sync(0xffffffffu, okb);
    const uint32_t ea = la + na, eb = lb + nb;
    la += (31 - __clz(ma)) * sa;
    lb += (31 - __clz(mb)) * sb;
    na = min(sa, ea - la);
    nb = min(sb, eb - lb);
  }
  ba = la;
  bb = lb;
}

// Slice s (global numbering: right 0..n_right-1, left n_right + s): positions
// [lo, hi] and its seed.
struct SliceSpan {
  uint32_t lo, hi, seed;
  bool right;
};
__device__ __forceinline__ SliceSpan slice_span(const SpState& st, uint32_t s) {
  SliceSpan r;
  if (s < st.n_right) {
    r.right = true;
    r.lo = 1 + s * st.step_r;
    r.hi = min(r.lo + st.step_r, st.l) - 1;
    r.seed = r.lo;
  } else {
    r.right = false;
    const uint32_t k = s - st.n_right;
    const uint32_t ml = st.M - 1 - st.l;
    r.hi = st.M - 1 - k * st.step_l;
    r.lo = st.M - 1 - min(k * st.step_l + st.step_l - 1, ml - 1);
    r.seed = r.hi;
  }
  return r;
}

// One warp per slice: the head of the slice (its points inside the seed's
// gathered bucket, exact positions), then an exclusive running maximum of
// phi over the slice's buckets in walk order -> prefmax[b] and slice_of[b]
// for every non-gathered bucket. Gathered buckets inside a slice (possible
// when the step was ambiguous) contribute nothing (conservative).
__global__ void __launch_bounds__(256) k_sp_slices(
    const SpState* __restrict__ st_, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ gs, const uint32_t* __restrict__ gbits,
    const uint32_t* __restrict__ phimax,
    const double* __restrict__ A_x, const double* __restrict__ A_y,
    const ExtResult* __restrict__ ext, uint32_t* __restrict__ prefmax,
    uint32_t* __restrict__ slice_of) {
  pdl_wait();
  const SpState st = *st_;
  if (st.fail) return;
  const uint32_t s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= st.n_right + st.n_left) return;
  const SliceSpan sp = slice_span(st, s);
  const double lx = st.lx, ly = st.ly;
  const double ux = __dsub_rn(ext->ax, lx), uy = __dsub_rn(ext->ay, ly);
  uint32_t bs, be;  // the seed's bucket, the bucket of the slice's last walk position
  bucket_of_pos2_warp(bstart, sp.seed, sp.right ? sp.hi : sp.lo, lane, bs, be);
  // head: slice positions inside the seed's bucket
  uint32_t h0, h1;  // inclusive position range
  if (sp.right) { h0 = sp.seed; h1 = min(sp.hi, bstart[bs + 1]); }
  else { h0 = max(sp.lo, 1 + bstart[bs]); h1 = sp.seed; }
  double hm = -1e300;
  const uint32_t qd = gs[bs] - bstart[bs];  // position -> storage in the seed's bucket
  for (uint32_t p = h0 + lane; p <= h1; p += 32) {
    double v2;
    const double raw = sp_phi_raw(A_x[p + qd], A_y[p + qd], lx, ly, ux, uy, &v2);
    if (v2 >= st.r02) hm = fmax(hm, sp.right ? raw : -raw);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hm = fmax(hm, __shfl_xor_sync(0xffffffffu, hm, o));
  uint32_t run = ord_f(__double2float_rd(hm));
  // buckets after the seed's bucket up to the bucket holding the slice's last
  // walk position; a non-gathered one there ends exactly at the slice end
  // (otherwise it would hold the next seed and be gathered)
  if (sp.right) {
    for (uint32_t b0 = bs + 1; b0 <= be; b0 += 32) {
      const uint32_t b = b0 + lane;
      const bool in = b <= be && !sp_gathered(gbits, b);
      uint32_t v = in ? phimax[b] : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = max(inc, y);
      }
      const uint32_t up = __shfl_up_sync(0xffffffffu, inc, 1);
      const uint32_t excl = max(run, lane ? up : 0u);
      if (in) { prefmax[b] = excl; slice_of[b] = s; }
      run = max(run, __shfl_sync(0xffffffffu, inc, 31));
    }
  } else {
    // walk order descending: buckets bs-1 down to be
    for (int32_t b0 = (int32_t)bs - 1; b0 >= (int32_t)be; b0 -= 32) {
      const int32_t b = b0 - lane;
      const bool in = b >= (int32_t)be && !sp_gathered(gbits, (uint32_t)b);
      uint32_t v = in ? phimax[b] : 0u;
      uint32_t inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc = max(inc, y);
      }
      const uint32_t up = __shfl_up_sync(0xffffffffu, inc, 1);
      const uint32_t excl = max(run, lane ? up : 0u);
      if (in) { prefmax[b] = excl; slice_of[b] = s; }
      run = max(run, __shfl_sync(0xffffffffu, inc, 31));
    }
  }
}

// ===========================================================================
// F4: candidates = non-gathered survivors whose phi is not below their
// bucket's exclusive prefix maximum (minus kSpTol); emitted to the CTA's
// region and marked in the codes (the verification skips them).
__device__ __forceinline__ bool sp_is_candidate(double ph, uint32_t pm, bool drop) {
  return !drop && ph >= unord_f(pm) - kSpTol;
}

constexpr int kSpCandThreads = 1024;

// Candidate thresholds per bucket: prefmax - tol, rounded down to float (a
// lower threshold only adds candidates); gathered buckets get +inf (never
// candidates here).
__global__ void k_sp_thresholds(const uint32_t* __restrict__ gbits,
                                const uint32_t* __restrict__ prefmax, const SpState* __restrict__ st,
                                float* __restrict__ thr) {
  pdl_wait();
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= kSpBuckets || st->fail) return;
  const bool g = (gbits[b >> 5] >> (b & 31)) & 1u;
  thr[b] = g ? __int_as_float(0x7f800000) : __double2float_rd(unord_f(prefmax[b]) - kSpTol);
}

__global__ void __launch_bounds__(kSpCandThreads, 1) k_sp_cand(
    uint16_t* __restrict__ codes, const float* __restrict__ phi32, uint32_t n, uint32_t cap,
    const float* __restrict__ thr_g,
    SpState* __restrict__ st, uint32_t* __restrict__ c_idx, uint32_t* __restrict__ c_b,
    uint32_t* __restrict__ c_count, bool drop) {
  pdl_wait();
  // thresholds prefmax - tol, rounded down to float (a lower threshold only
  // adds candidates); gathered buckets get +inf (never candidates here)
  extern __shared__ __align__(16) float s_thr[];  // kSpBuckets
  __shared__ uint32_t s_nc;
  if (st->fail) return;
  {  // thresholds precomputed by k_sp_thresholds: a 16-byte copy into shared memory
    const float4* t4 = reinterpret_cast<const float4*>(thr_g);
    float4* s4 = reinterpret_cast<float4*>(s_thr);
    for (uint32_t q = threadIdx.x; q < kSpBuckets / 4; q += blockDim.x) s4[q] = __ldg(&t4[q]);
  }
  if (threadIdx.x == 0) s_nc = 0;
  const size_t base = (size_t)blockIdx.x * cap;
  __syncthreads();
  auto visit = [&](float ph, uint32_t b, uint32_t i) {
    // gathered buckets (threshold +inf) never emit here; NaN phi (within r0 of
    // P_l) compares false -> candidate
    bool emit = false;
    if (b != kSpNoCode) {
      const float thr = s_thr[b];
      emit = !drop && thr != __int_as_float(0x7f800000) && !(ph < thr);  // ph is signed
    }
    const uint32_t j = warp_claim(&s_nc, emit);
    if (emit) {
      c_idx[base + j] = i;
      c_b[base + j] = b;
      codes[i] = (uint16_t)kSpCandCode;
    }
  };
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nth = gridDim.x * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t* c2 = reinterpret_cast<const uint32_t*>(codes);
  const float2* p2 = reinterpret_cast<const float2*>(phi32);
  const uint32_t np = n / 2;
  uint32_t p = tid;
  // main loop, warp-uniform bound: 8 points per thread are tested first; a
  // warp without a candidate (the common case) claims nothing
  for (; (p - lane) + 31 + 3 * nth < np; p += 4 * nth) {
    uint32_t vc[4];
    float2 vp[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) vc[u] = __ldcs(&c2[p + u * nth]);
#pragma unroll
    for (int u = 0; u < 4; ++u) vp[u] = __ldcs(&p2[p + u * nth]);
    uint32_t em = 0, ne = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t b = hh ? vc[u] >> 16 : vc[u] & 0xffffu;
        const float ph = hh ? vp[u].y : vp[u].x;
        bool e = false;
        if (b != kSpNoCode) {
          const float thr = s_thr[b];
          e = !drop && thr != __int_as_float(0x7f800000) && !(ph < thr);
        }
        em |= (e ? 1u : 0u) << (2 * u + hh);
        ne += e ? 1u : 0u;
      }
    }
    if (__any_sync(0xffffffffu, ne != 0)) {
      uint32_t at = warp_scan_claim(&s_nc, ne, lane);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          if ((em >> (2 * u + hh)) & 1u) {
            const uint32_t i = 2 * (p + u * nth) + hh;
            c_idx[base + at] = i;
            c_b[base + at] = hh ? vc[u] >> 16 : vc[u] & 0xffffu;
            codes[i] = (uint16_t)kSpCandCode;
            ++at;
          }
    }
  }
  for (; p < np; p += nth) {
    const uint32_t vc = c2[p];
    const float2 vp = p2[p];
    visit(vp.x, vc & 0xffffu, 2 * p);
    visit(vp.y, vc >> 16, 2 * p + 1);
  }
  if ((n & 1) && tid == nth - 1) visit(phi32[n - 1], codes[n - 1], n - 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    c_count[blockIdx.x] = s_nc;
    atomicAdd(&st->n_c, s_nc);
  }
}

// Walk-array bucket sizes: gathered buckets bring all their points, others
// their candidates.
__global__ void k_sp_wcount(const uint32_t* __restrict__ gbits, const uint32_t* __restrict__ hist,
                            const uint32_t* __restrict__ ccnt, uint32_t* __restrict__ wcnt) {
  pdl_wait();
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < kSpBuckets) wcnt[b] = sp_gathered(gbits, b) ? hist[b] : ccnt[b];
}

__device__ __forceinline__ uint32_t slice_of_pos(const SpState& st, uint32_t p) {
  if (p == 0 || p == st.l) return kNone;
  if (p < st.l) return (p - 1) / st.step_r;
  return st.n_right + (st.M - 1 - p) / st.step_l;
}

// Candidates, warp per bucket: up to 32 per bucket are ranked in registers
// by the exact total order and written to the walk array W at
// 1 + wstart[b] + rank; larger buckets go to a list for the CTA sorter.
// Equal points -> fail.
__global__ void __launch_bounds__(256) k_sp_place_cand(
    const PtRec* __restrict__ crec, const uint32_t* __restrict__ cstart,
    const uint32_t* __restrict__ wstart, const uint32_t* __restrict__ slice_of,
    const ExtResult* __restrict__ ext, SpState* __restrict__ st, uint32_t* __restrict__ big,
    double* __restrict__ W_x, double* __restrict__ W_y, uint32_t* __restrict__ W_i,
    uint32_t* __restrict__ W_b, uint32_t* __restrict__ W_s, uint8_t* __restrict__ flags) {
  pdl_wait();
  if (st->fail) return;
  const double ax = ext->ax, ay = ext->ay;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < kSpBuckets; b += nwarps) {
    const uint32_t c0 = cstart[b], cnt = cstart[b + 1] - c0;
    if (cnt == 0) continue;
    const uint32_t sl = slice_of[b];
    if (sl == kNone) {
      if (lane == 0) { atomicOr(&st->fail, kSpFailInternal); atomicMax(&st->why, 3u); }
      continue;
    }
    if (cnt > 32) {
      if (lane == 0) big[atomicAdd(&st->n_bigc, 1u)] = b;
      continue;
    }
    PtRec r{};
    double d = 0.0;
    if ((uint32_t)lane < cnt) {
      r = ld_rec256(&crec[c0 + lane]);
      d = dist2_rn(__dsub_rn(r.x, ax), __dsub_rn(r.y, ay));
    }
    uint32_t rk = 0;
    bool dup = false;
    for (uint32_t k = 0; k < cnt; ++k) {
      const uint64_t ok = __shfl_sync(0xffffffffu, r.key, k);
      const double od = __shfl_sync(0xffffffffu, d, k);
      const uint32_t oi = __shfl_sync(0xffffffffu, r.idx, k);
      const double ox = __shfl_sync(0xffffffffu, r.x, k);
      const double oy = __shfl_sync(0xffffffffu, r.y, k);
      if ((uint32_t)lane < cnt && k != (uint32_t)lane) {
        rk += key_less(ok, od, oi, r.key, d, r.idx);
        dup |= (ox == r.x && oy == r.y);
      }
    }
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(&st->fail, kSpFailDup);
    if ((uint32_t)lane < cnt) {
      const uint32_t w = 1 + wstart[b] + rk;
      W_x[w] = r.x;
      W_y[w] = r.y;
      W_i[w] = r.idx;
      W_b[w] = b;
      W_s[w] = sl;
      flags[w] = 1;
    }
  }
}

// Candidate buckets with more than 32 candidates: CTA sub-bucket sorter.
__global__ void __launch_bounds__(kSpSortThreads) k_sp_sort_cand_big(
    const uint32_t* __restrict__ big, const PtRec* __restrict__ crec,
    const uint32_t* __restrict__ cstart, const uint32_t* __restrict__ wstart,
    const uint32_t* __restrict__ slice_of, const ExtResult* __restrict__ ext,
    SpState* __restrict__ st, double* __restrict__ W_x, double* __restrict__ W_y,
    uint32_t* __restrict__ W_i, uint32_t* __restrict__ W_b, uint32_t* __restrict__ W_s,
    uint8_t* __restrict__ flags, unsigned char* __restrict__ scratch, uint32_t scap) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem[];
  if (st->fail) return;
  const uint32_t nbig = st->n_bigc;
  const double ax = ext->ax, ay = ext->ay;
  uint32_t* s_list = reinterpret_cast<uint32_t*>(smem + (size_t)kSpGatherCap * (8 + 8 + 8 + 8 + 4 + 4)) +
                     kSpGatherCap + 1;
  // buckets above kSpGatherCap (large inputs): the global scratch area of
  // this CTA (k_sp_sort_gathered_huge's, which has finished by now)
  unsigned char* scr = scratch ? scratch + (size_t)blockIdx.x * ((size_t)scap * kSpHugeBytes + 16) : nullptr;
  uint32_t* g_list = scr ? reinterpret_cast<uint32_t*>(scr + (size_t)scap * (8 + 8 + 8 + 8 + 4 + 4)) + scap + 1
                         : nullptr;
  for (uint32_t g = blockIdx.x; g < nbig; g += gridDim.x) {
    const uint32_t b = big[g];
    const uint32_t c0 = cstart[b], cnt = cstart[b + 1] - c0;
    const bool huge = cnt > kSpGatherCap;
    if (huge && cnt > scap) {
      if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 5u); }
      return;
    }
    const uint32_t w0 = 1 + wstart[b], sl = slice_of[b];
    auto out = [&](uint32_t r, double x, double y, uint32_t idx) {
      W_x[w0 + r] = x;
      W_y[w0 + r] = y;
      W_i[w0 + r] = idx;
      W_b[w0 + r] = b;
      W_s[w0 + r] = sl;
      flags[w0 + r] = 1;
    };
    __syncthreads();
    bool slow = false, dup;
    if (!huge) {
      for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) s_list[t] = 0xffffffffu;
      dup = cta_sort_bucket_sub<kSpGatherCap>(crec + c0, cnt, ax, ay, smem, &slow, out);
    } else {
      for (uint32_t t = threadIdx.x; t < cnt; t += blockDim.x) g_list[t] = 0xffffffffu;
      __threadfence_block();
      dup = cta_sort_bucket_sub<kSpGatherCap, true>(crec + c0, cnt, ax, ay, scr, &slow, out, scap);
      if (slow) {
        if (threadIdx.x == 0) { atomicOr(&st->fail, kSpFailCap); atomicMax(&st->why, 6u); }
        return;
      }
    }
    if (dup) atomicOr(&st->fail, kSpFailDup);
  }
}

// Gathered buckets: copy their exactly placed points from A to W (CTA per
// gathered bucket); W[0] = anchor.
__global__ void __launch_bounds__(256) k_sp_place_gathered(
    const uint32_t* __restrict__ glist, const uint32_t* __restrict__ bstart,
    const uint32_t* __restrict__ gs, const uint32_t* __restrict__ hist,
    const uint32_t* __restrict__ wstart,
    const double* __restrict__ A_x, const double* __restrict__ A_y,
    const uint32_t* __restrict__ A_i, const ExtResult* __restrict__ ext, SpState* __restrict__ st_,
    double* __restrict__ W_x, double* __restrict__ W_y, uint32_t* __restrict__ W_i,
    uint32_t* __restrict__ W_b, uint32_t* __restrict__ W_s, uint8_t* __restrict__ flags) {
  pdl_wait();
  const SpState st = *st_;
  if (st.fail) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    flags[0] = 1;
    W_x[0] = ext->ax;
    W_y[0] = ext->ay;
    W_i[0] = ext->idx[4];
    W_b[0] = kNone;
    W_s[0] = kNone;
    st_->n_w = 1 + wstart[kSpBuckets];
    if (st.l_check != st.l) { atomicOr(&st_->fail, kSpFailInternal); atomicMax(&st_->why, 2u); }
  }
  for (uint32_t g = blockIdx.x; g < st.n_gb; g += gridDim.x) {
    const uint32_t b = glist[g];
    const uint32_t s0 = bstart[b], g0 = gs[b], cnt = hist[b], w0 = wstart[b];
    for (uint32_t r = threadIdx.x; r < cnt; r += blockDim.x) {
      const uint32_t p = 1 + s0 + r, q = 1 + g0 + r, w = 1 + w0 + r;
      W_x[w] = A_x[q];
      W_y[w] = A_y[q];
      W_i[w] = A_i[q];
      W_b[w] = b;
      W_s[w] = slice_of_pos(st, p);
      flags[w] = 1;
    }
  }
}

// Slice segments in W: seg_lo[s] = first W index of slice s, seg_hi[s] = one
// past its last (slices are contiguous because W is exactly ordered).
__global__ void k_sp_segments(const uint32_t* __restrict__ W_s, const SpState* __restrict__ st,
                              uint32_t* __restrict__ seg_lo, uint32_t* __restrict__ seg_hi) {
  pdl_wait();
  if (st->fail) return;
  const uint32_t nw = st->n_w;
  for (uint32_t j = 1 + blockIdx.x * blockDim.x + threadIdx.x; j < nw; j += gridDim.x * blockDim.x) {
    const uint32_t s = W_s[j];
    if (s == kNone) continue;
    if (W_s[j - 1] != s) seg_lo[s] = j;
    if (j + 1 == nw || W_s[j + 1] != s) seg_hi[s] = j + 1;
  }
}

// Round-2 walk (discard.hpp:36-66) of one slice over its walked points in W:
// CTA per slice; the speculate-and-verify scheme of k_round2_block with an
// explicit segment. Right slices walk ascending from their first element,
// left slices descending from their last.
__global__ void __launch_bounds__(kWalkBlock) k_sp_walk(
    const double* __restrict__ A_x, const double* __restrict__ A_y,
    const uint32_t* __restrict__ seg_lo, const uint32_t* __restrict__ seg_hi,
    const SpState* __restrict__ st_, const ExtResult* __restrict__ ext,
    uint8_t* __restrict__ flags) {
  pdl_wait();
  const SpState& st = *st_;
  if (st.fail) return;
  const uint32_t slice = blockIdx.x;
  if (slice >= st.n_right + st.n_left) return;
  const uint32_t lo = seg_lo[slice], hi = seg_hi[slice];
  const int dir = slice < st.n_right ? 1 : -1;
  const uint32_t seed = dir > 0 ? lo : hi - 1;
  const uint32_t start = dir > 0 ? lo + 1 : hi - 2;
  const uint32_t count = hi - lo - 1;
  if (count == 0 || count > 0x7fffffffu) return;
  __shared__ MaxPair s_wm[kWalkBlock / 32];
  __shared__ int32_t s_first;
  __shared__ MaxPair s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double lx = st.lx, ly = st.ly;
  const double ux = ext->ax - lx, uy = ext->ay - ly;
  const double sgn = (dir > 0) ? 1.0 : -1.0;
  auto wpos = [&](int32_t k) -> uint32_t {
    return k < 0 ? seed : ((dir > 0) ? start + (uint32_t)k : start - (uint32_t)k);
  };
  MaxPair carry;
  carry.v = sgn * pseudo_angle(A_x[seed], A_y[seed], lx, ly, ux, uy);
  carry.k = -1;
  int32_t w0 = 0;
  while (w0 < (int32_t)count) {
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
      if (k == f) {
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

// R bucket index: rlo[b] = first R position whose bucket >= b (anchor = -1).
__global__ void k_sp_rlo(const uint32_t* __restrict__ R_b, const SpState* __restrict__ st,
                         uint32_t* __restrict__ rlo) {
  pdl_wait();
  if (st->fail) return;
  const uint32_t nr = st->n_r;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= nr; j += gridDim.x * blockDim.x) {
    const int64_t prev = (j == 0) ? -2 : (j == 1 ? -1 : (int64_t)R_b[j - 1]);
    const int64_t cur = (j == nr) ? (int64_t)kSpBuckets : (j == 0 ? -1 : (int64_t)R_b[j]);
    for (int64_t b = prev + 1; b <= cur; ++b)
      if (b >= 0) rlo[b] = j;
  }
}

// ===========================================================================
// Error-bound certificate: when it holds, every survivor that was not walked
// is PROVABLY discarded by the reference walk, and F6 is skipped.
// Setting (right region; left mirrored): p not walked means phi(p) <
// prefmax(b) - kSpTol, where prefmax(b) <= phi(q*) for a point q* earlier in
// p's slice with |q* - P_l| >= r0 (F3 / k_sp_slices exclude closer points,
// F4 walks them). alpha = exact angle of P - P_l. The reference's orient() is
// off by at most 4.3 eps |v(t)| |q - t| (two rounded differences, two
// products, one difference), so one decision moves the walk state's alpha
// backwards by at most asin(4.3 eps (1 + |v(t)| / |v(q)|)): once when q* is
// decided and once per later state change (<= K_max kept points per slice);
// p is discarded once alpha(state) - alpha(p) exceeds the same bound for p.
// dphi/dalpha <= 1, so a phi gap bounds the alpha gap. Therefore
//   kSpTol > K_max * asin(4.3 eps (1 + D / rho)) + 2 asin(4.3 eps (1 + D / r0)) + 2 e_phi + e_f
// (e_f: F4 reads phi(p) stored as a float by F3)
// (D: bounding-box diagonal, rho: closest kept slice point to P_l, e_phi: phi
// evaluation error) proves every skipped point discarded, provided all angle
// gaps stay below pi - 1e-3 (checked from the phi range).
__global__ void __launch_bounds__(256) k_sp_cert_stats(const double* __restrict__ R_x,
                                                       const double* __restrict__ R_y,
                                                       const uint32_t* __restrict__ R_s,
                                                       SpState* __restrict__ st) {
  pdl_wait();
  if (st->fail) return;
  const uint32_t nr = st->n_r;
  const double lx = st->lx, ly = st->ly;
  uint64_t best = 0x7fefffffffffffffull;
  uint32_t kmax = 0;
  for (uint32_t j = 1 + blockIdx.x * blockDim.x + threadIdx.x; j < nr; j += gridDim.x * blockDim.x) {
    const uint32_t sl = R_s[j];
    if (sl == kNone) continue;  // anchor / P_l
    const double vx = __dsub_rn(R_x[j], lx), vy = __dsub_rn(R_y[j], ly);
    const uint64_t v2 = dbits(vx * vx + vy * vy);
    best = v2 < best ? v2 : best;
    if (R_s[j - 1] != sl) {  // first kept point of its slice: count the run
      uint32_t k = j + 1;
      while (k < nr && R_s[k] == sl) ++k;
      kmax = max(kmax, k - j);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ob = __shfl_xor_sync(0xffffffffu, best, o);
    best = ob < best ? ob : best;
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin((unsigned long long*)&st->rho2_bits, (unsigned long long)best);
    atomicMax(&st->k_max, kmax);
  }
}

__device__ __forceinline__ double angle_of_pseudo(double ph) {
  const double a = fabs(ph);
  const double t = (a <= 1.0) ? atan2(a, 1.0 - a) : 3.141592653589793 - atan2(2.0 - a, a - 1.0);
  return ph >= 0.0 ? t : -t;
}

__global__ void k_sp_cert_decide(SpState* __restrict__ st, bool force_verify) {
  pdl_wait();
  if (threadIdx.x != 0 || st->fail) return;
  const double eps = 1.1102230246251565e-16;
  const double D = sqrt(st->dmax2) * (1.0 + 1e-9);
  const double r0 = sqrt(st->r02) * (1.0 - 1e-9);
  const double rho = sqrt(bitsd(st->rho2_bits)) * (1.0 - 1e-9);
  bool ok = !force_verify && rho > 0.0 && r0 > 0.0 && st->phi_lo != 0xffffffffu;
  if (ok) {
    const double x1 = 4.3 * eps * (1.0 + D / rho), x2 = 4.3 * eps * (1.0 + D / r0);
    ok = x1 < 0.01 && x2 < 0.01;
    const double m = (double)(st->k_max + 1) * x1 * 1.01 + 2.0 * x2 * 1.01 + 2.0 * 1e-11 +
                     kSpPhiStoreErr;
    ok = ok && m < kSpTol;
    const double w = angle_of_pseudo((double)unord_f(st->phi_hi) + 1e-9) -
                     angle_of_pseudo((double)unord_f(st->phi_lo) - 1e-9);
    ok = ok && w < 3.141592653589793 - 1e-3;
  }
  st->cert = ok ? 1u : 0u;
  st->need_verify = ok ? 0u : 1u;
}

// ===========================================================================
// F6: every survivor that was not walked must be discarded by the reference
// walk. Its walk state is the last kept point before it in its slice: the
// last kept point before its bucket or a kept point of its own bucket
// (discard.hpp:44-50, 58-64); it must be strictly inside against all of them.
// The kept points' loads are issued for 8 points at once (memory-level
// parallelism).
template <bool kVec>
__global__ void __launch_bounds__(kSpThreads, 1) k_sp_verify(
    const double* __restrict__ xs, const double* __restrict__ ys,
    const uint16_t* __restrict__ codes, uint32_t n, const uint32_t* __restrict__ gbits,
    const uint32_t* __restrict__ rlo, const double* __restrict__ R_x,
    const double* __restrict__ R_y, SpState* __restrict__ st) {
  pdl_wait();
  extern __shared__ uint32_t s_rlo[];  // kSpBuckets + 1
  __shared__ uint32_t s_g[kSpBuckets / 32];
  if (st->fail || !st->need_verify) return;
  for (uint32_t b = threadIdx.x; b <= kSpBuckets; b += blockDim.x) s_rlo[b] = rlo[b];
  for (uint32_t w = threadIdx.x; w < kSpBuckets / 32; w += blockDim.x) s_g[w] = gbits[w];
  const double lx = st->lx, ly = st->ly;
  const uint32_t b_l = st->b_l;
  __syncthreads();
  uint32_t bad = 0;
  auto check8 = [&](const double* px, const double* py, const uint32_t* pc, int cnt) {
    uint32_t jb[8], j0[8], j1[8];
    bool act[8];
    double tx[8], ty[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t b = pc[u];
      act[u] = u < cnt && b < kSpCandCode && !sp_gathered(s_g, b);
      jb[u] = 0;
      j0[u] = j1[u] = 0;
      if (act[u]) {
        j0[u] = s_rlo[b];
        j1[u] = s_rlo[b + 1];
        jb[u] = (b < b_l) ? j0[u] - 1 : j1[u];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      tx[u] = act[u] ? R_x[jb[u]] : 0.0;
      ty[u] = act[u] ? R_y[jb[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (!act[u]) continue;
      const bool right = pc[u] < b_l;
      double c = cross_rn(tx[u], ty[u], lx, ly, px[u], py[u]);
      bool ok = right ? (c > 0.0) : (c < 0.0);
      for (uint32_t j = j0[u]; j < j1[u]; ++j) {
        c = cross_rn(R_x[j], R_y[j], lx, ly, px[u], py[u]);
        ok = ok && (right ? (c > 0.0) : (c < 0.0));
      }
      bad += !ok;
    }
  };
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nth = gridDim.x * blockDim.x;
  if (kVec) {
    const double2* x2 = reinterpret_cast<const double2*>(xs);
    const double2* y2 = reinterpret_cast<const double2*>(ys);
    const uint32_t* c2 = reinterpret_cast<const uint32_t*>(codes);
    const uint32_t np = n / 2;
    for (uint32_t p = tid; p < np; p += 4 * nth) {
      double px[8], py[8];
      uint32_t pc[8];
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = p + u * nth;
        if (q < np) {
          const uint32_t cw = __ldcs(&c2[q]);
          pc[2 * u] = cw & 0xffffu;
          pc[2 * u + 1] = cw >> 16;
          cnt = 2 * u + 2;
        } else {
          pc[2 * u] = pc[2 * u + 1] = kSpNoCode;
        }
      }
      // coordinates only for pairs that hold a point to verify
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t q = p + u * nth;
        const bool need = (pc[2 * u] < kSpCandCode) || (pc[2 * u + 1] < kSpCandCode);
        if (q < np && need) {
          const double2 vx = __ldcs(&x2[q]), vy = __ldcs(&y2[q]);
          px[2 * u] = vx.x; px[2 * u + 1] = vx.y;
          py[2 * u] = vy.x; py[2 * u + 1] = vy.y;
        } else {
          px[2 * u] = px[2 * u + 1] = py[2 * u] = py[2 * u + 1] = 0.0;
          pc[2 * u] = pc[2 * u + 1] = kSpNoCode;
        }
      }
      check8(px, py, pc, cnt);
    }
    if ((n & 1) && tid == nth - 1) {
      double px[8] = {xs[n - 1]}, py[8] = {ys[n - 1]};
      uint32_t pc[8] = {codes[n - 1]};
      check8(px, py, pc, 1);
    }
  } else {
    for (uint32_t i0 = tid * 8; i0 < n; i0 += nth * 8) {
      double px[8], py[8];
      uint32_t pc[8];
      const int cnt = (int)min(8u, n - i0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool v = u < cnt;
        pc[u] = v ? codes[i0 + u] : kSpNoCode;
        px[u] = (v && pc[u] < kSpCandCode) ? xs[i0 + u] : 0.0;
        py[u] = (v && pc[u] < kSpCandCode) ? ys[i0 + u] : 0.0;
      }
      check8(px, py, pc, cnt);
    }
  }
  if (bad) {
    atomicAdd(&st->verify_fail, bad);
    atomicOr(&st->fail, kSpFailVerify);
  }
}

// Stable compaction of the walk array by its keep flags (stable_compact,
// discard.hpp:128-145), carrying bucket ids; n from / to the state.
__global__ void __launch_bounds__(kBlock) k_sp_compact(
    const double* __restrict__ in_x, const double* __restrict__ in_y,
    const uint32_t* __restrict__ in_i, const uint32_t* __restrict__ in_b,
    const uint32_t* __restrict__ in_s, const uint8_t* __restrict__ flags, SpState* __restrict__ st,
    double* __restrict__ out_x, double* __restrict__ out_y, uint32_t* __restrict__ out_i,
    uint32_t* __restrict__ out_b, uint32_t* __restrict__ out_s, uint64_t* __restrict__ status,
    Counters* __restrict__ ctr) {
  pdl_wait();
  __shared__ uint32_t s_tile, s_excl, s_rows[kCompactItems * kWarps + 1];
  if (st->fail) return;
  const uint32_t n = st->n_w;
  if (threadIdx.x == 0) s_tile = atomicAdd(&ctr->tile_ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t base = tile * kCompactTile;  // striped: item (k, t) = base + k * kBlock + t
  if (base >= n) return;
  bool keep[kCompactItems];
#pragma unroll
  for (int k = 0; k < kCompactItems; ++k) {
    const uint32_t i = base + k * kBlock + threadIdx.x;
    keep[k] = i < n && flags[i] != 0;
  }
  uint32_t rk[kCompactItems];
  const uint32_t total = striped_keep_ranks<kCompactItems>(keep, rk, s_rows);
  if (threadIdx.x < 32) {
    const uint64_t e = lookback_exclusive(status, tile, total);
    if (threadIdx.x == 0) {
      s_excl = (uint32_t)e;
      if (base + kCompactTile >= n) st->n_r = (uint32_t)(e + total);
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
      out_b[o] = in_b[i];
      out_s[o] = in_s[i];
    }
  }
}


// ===========================================================================
// Sharded sparse path (distributed.py): conversions between a
// rank's per-CTA emission regions and compact records {x, y, global index,
// bucket} that travel between ranks.

// Regions (e_idx, e_b, e_count; cap slots per region, G regions) -> compact
// records; *n_out counts (order is arbitrary: the receiver sorts by index).
__global__ void __launch_bounds__(256) k_sp_export(
    const double* __restrict__ xs, const double* __restrict__ ys,
    const uint32_t* __restrict__ e_idx, const uint32_t* __restrict__ e_b,
    const uint32_t* __restrict__ e_count, uint32_t cap, uint32_t base, const SpState* __restrict__ st,
    double* __restrict__ ox, double* __restrict__ oy, uint32_t* __restrict__ oi,
    uint32_t* __restrict__ ob, uint32_t* __restrict__ n_out) {
  if (st->fail) return;
  const uint32_t c = blockIdx.y;
  const uint32_t ne = e_count[c];
  const size_t rb = (size_t)c * cap;
  for (uint32_t k0 = blockIdx.x * blockDim.x; k0 < ne; k0 += gridDim.x * blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    const bool have = k < ne;
    const uint32_t act = __ballot_sync(0xffffffffu, have);
    uint32_t at = 0;
    if ((threadIdx.x & 31) == 0 && act) at = atomicAdd(n_out, (uint32_t)__popc(act));
    at = __shfl_sync(0xffffffffu, at, 0) + __popc(act & lanemask_lt());
    if (have) {
      const uint32_t i = e_idx[rb + k];
      ox[at] = xs[i];
      oy[at] = ys[i];
      oi[at] = base + i;
      ob[at] = e_b[rb + k];
    }
  }
}

// Compact items j < n (buckets b_in[j]) -> regions: item j goes to region
// j / per (per = ceil(n / G) <= cap) as index idx0 + j.
__global__ void __launch_bounds__(256) k_sp_fill_regions(uint32_t n, uint32_t idx0,
                                                         const uint32_t* __restrict__ b_in,
                                                         uint32_t G, uint32_t cap,
                                                         uint32_t* __restrict__ e_idx,
                                                         uint32_t* __restrict__ e_b,
                                                         uint32_t* __restrict__ e_count) {
  const uint32_t per = (n + G - 1) / G;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < G; c += gridDim.x * blockDim.x)
    e_count[c] = c * per < n ? min(per, n - c * per) : 0u;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const uint32_t c = j / per, k = j - c * per;
    e_idx[(size_t)c * cap + k] = idx0 + j;
    e_b[(size_t)c * cap + k] = b_in[j];
  }
}


// Sizes of the gathered buckets (storage of rank 0's gathered records).
__global__ void k_sp_gsize(const uint32_t* __restrict__ gbits, const uint32_t* __restrict__ hist,
                           uint32_t* __restrict__ out) {
  pdl_wait();
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < kSpBuckets) out[b] = sp_gathered(gbits, b) ? hist[b] : 0u;
}

// Received hash blocks (R sources; cnt[r * kSpParts + p] entries of
// partition p from source r, block r = its partitions in order) -> the
// partition-major count table for the partitioning kernel, block sizes and
// block bases.
__global__ void k_sp_recv_plan(const uint32_t* __restrict__ cnt, uint32_t R,
                               uint32_t* __restrict__ pm, uint32_t* __restrict__ h_count,
                               uint64_t* __restrict__ list_base) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < kSpParts * R) {
    const uint32_t p = t / R, r = t - p * R;
    pm[t] = cnt[(size_t)r * kSpParts + p];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint64_t acc = 0;
    for (uint32_t r = 0; r < R; ++r) {
      uint32_t sz = 0;
      for (uint32_t p = 0; p < kSpParts; ++p) sz += cnt[(size_t)r * kSpParts + p];
      h_count[r] = sz;
      list_base[r] = acc;
      acc += sz;
    }
  }
}

// ===========================================================================
// Sharded path, device-side data plane (gscan_dist_enq_*): every rank writes
// its per-phase scalars into a fixed record of kDistRecLen int64 words; the
// host all-gathers the records on the handle's stream (NCCL) and the next
// phase combines them ON THE DEVICE, so a call needs host round trips only
// where a variable-size exchange needs its sizes. Word layout:
//   [0, 15)   extremes: global index (5), x bits (5), y bits (5)
//   [16, 23)  F2: dist2 bits, global index of P_l (-1: none), ties, x bits,
//             y bits, round-1 survivors, fail (locally decided P_l bits masked)
//   [24, 27)  plan: points of P_l's bucket ordered before it, fail, M
//   [28, 32)  F3: phi_lo, phi_hi, gathered points, fail
//   [36, 38)  F4: candidates, fail (includes the duplicate check)
//   [40, 42)  F6: points that would not be discarded, fail
constexpr int kDistRecLen = 64;
constexpr int kRxExt = 0, kRxF2 = 16, kRxPlan = 24, kRxF3 = 28, kRxF4 = 36, kRxVer = 40;

__global__ void k_dist_rec_ext(const ExtResult* __restrict__ ext, uint32_t base,
                               int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < 4; ++k) {
    rec[kRxExt + k] = (int64_t)base + ext->idx[k];
    rec[kRxExt + 5 + k] = (int64_t)dbits(ext->qx[k]);
    rec[kRxExt + 10 + k] = (int64_t)dbits(ext->qy[k]);
  }
  rec[kRxExt + 4] = (int64_t)base + ext->idx[4];
  rec[kRxExt + 9] = (int64_t)dbits(ext->ax);
  rec[kRxExt + 14] = (int64_t)dbits(ext->ay);
}

// Global extremes from R records with find_extremes' / select_anchor's rules
// (strict compares; equal values: the lowest global index; prefilter.hpp:28-39,
// angular.hpp:40-49). ext_out: the combined record (host/rank 0 reads it).
__global__ void k_dist_apply_ext(const int64_t* __restrict__ recs, uint32_t R,
                                 ExtResult* __restrict__ ext, int64_t* __restrict__ ext_out) {
  if (threadIdx.x != 0) return;
  for (int k = 0; k < 5; ++k) {
    int64_t bi = recs[kRxExt + k];
    double bx = bitsd((uint64_t)recs[kRxExt + 5 + k]), by = bitsd((uint64_t)recs[kRxExt + 10 + k]);
    for (uint32_t r = 1; r < R; ++r) {
      const int64_t* q = recs + (size_t)r * kDistRecLen;
      const int64_t gi = q[kRxExt + k];
      const double x = bitsd((uint64_t)q[kRxExt + 5 + k]), y = bitsd((uint64_t)q[kRxExt + 10 + k]);
      bool better;
      if (k == 0) better = x < bx || (x == bx && gi < bi);
      else if (k == 1) better = y < by || (y == by && gi < bi);
      else if (k == 2) better = x > bx || (x == bx && gi < bi);
      else if (k == 3) better = y > by || (y == by && gi < bi);
      else better = y < by || (y == by && (x < bx || (x == bx && gi < bi)));
      if (better) { bi = gi; bx = x; by = y; }
    }
    ext->idx[k] = (uint32_t)bi;
    if (k < 4) { ext->qx[k] = bx; ext->qy[k] = by; }
    else { ext->ax = bx; ext->ay = by; }
    ext_out[k] = bi;
    ext_out[5 + k] = (int64_t)dbits(bx);
    ext_out[10 + k] = (int64_t)dbits(by);
  }
}

__global__ void k_dist_rec_f2(const SpState* __restrict__ st, const Counters* __restrict__ ctr,
                              uint32_t base, int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  const bool have = st->l_idx != 0xffffffffu;
  rec[kRxF2 + 0] = (int64_t)st->d2max;
  rec[kRxF2 + 1] = have ? (int64_t)base + st->l_idx : -1;
  rec[kRxF2 + 2] = have ? st->ties : 0;
  rec[kRxF2 + 3] = (int64_t)dbits(st->lx);
  rec[kRxF2 + 4] = (int64_t)dbits(st->ly);
  rec[kRxF2 + 5] = ctr->n1;
  // P_l's tie / none / too-many bits are decided again over all ranks
  rec[kRxF2 + 6] = st->fail & ~(kSpFailTie | kSpFailFew | kSpFailMany);
}

// The global farthest point (split_regions, angular.hpp:197-204: the first
// maximal dist2 = the lowest global index among equals), its tie count and
// the global fail bits, into every rank's state.
__global__ void k_dist_apply_best(const int64_t* __restrict__ recs, uint32_t R, uint64_t n_global,
                                  SpState* __restrict__ st) {
  if (threadIdx.x != 0) return;
  bool found = false;
  uint64_t bd = 0, n1 = 0;
  int64_t bi = -1, bx = 0, by = 0;
  uint32_t ties = 0, fail = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const int64_t* q = recs + (size_t)r * kDistRecLen + kRxF2;
    n1 += (uint64_t)q[5];
    fail |= (uint32_t)q[6];
    const uint32_t t = (uint32_t)q[2];
    if (t == 0) continue;
    const uint64_t d2 = (uint64_t)q[0];
    if (!found || d2 > bd) {
      found = true; bd = d2; bi = q[1]; bx = q[3]; by = q[4]; ties = t;
    } else if (d2 == bd) {
      ties += t;
      if (q[1] < bi) { bi = q[1]; bx = q[3]; by = q[4]; }
    }
  }
  if (!found) fail |= kSpFailFew;
  else if (ties != 1) fail |= kSpFailTie;
  if (n1 * 10 > n_global * 9) fail |= kSpFailMany;
  st->d2max = bd;
  st->l_idx = found ? (uint32_t)bi : 0xffffffffu;
  st->ties = ties;
  st->lx = bitsd((uint64_t)bx);
  st->ly = bitsd((uint64_t)by);
  st->fail = fail;
}

__global__ void k_dist_rec_plan(const SpState* __restrict__ st, int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  rec[kRxPlan + 0] = st->l_below;
  rec[kRxPlan + 1] = st->fail;
  rec[kRxPlan + 2] = st->M;
}

__global__ void k_dist_apply_plan(const int64_t* __restrict__ recs, uint32_t R,
                                  SpState* __restrict__ st) {
  if (threadIdx.x != 0) return;
  uint64_t lb = 0;
  uint32_t fail = 0;
  for (uint32_t r = 0; r < R; ++r) {
    lb += (uint64_t)recs[(size_t)r * kDistRecLen + kRxPlan + 0];
    fail |= (uint32_t)recs[(size_t)r * kDistRecLen + kRxPlan + 1];
  }
  st->l_below = (uint32_t)lb;
  st->fail |= fail;
}

__global__ void k_dist_rec_f3(const SpState* __restrict__ st, int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  rec[kRxF3 + 0] = st->phi_lo;
  rec[kRxF3 + 1] = st->phi_hi;
  rec[kRxF3 + 2] = st->n_g;
  rec[kRxF3 + 3] = st->fail;
}

// phi range over all ranks (ordered-float encodings compare as uint32)
__global__ void k_dist_apply_f3(const int64_t* __restrict__ recs, uint32_t R,
                                SpState* __restrict__ st) {
  if (threadIdx.x != 0) return;
  uint32_t lo = 0xffffffffu, hi = 0, fail = 0;
  for (uint32_t r = 0; r < R; ++r) {
    const int64_t* q = recs + (size_t)r * kDistRecLen + kRxF3;
    lo = min(lo, (uint32_t)q[0]);
    hi = max(hi, (uint32_t)q[1]);
    fail |= (uint32_t)q[3];
  }
  st->phi_lo = lo;
  st->phi_hi = hi;
  st->fail |= fail;
}

// Hash counts per partition (part_off scanned over nl lists; its total at
// part_off[kSpParts * nl]).
__global__ void k_dist_part_totals(const uint32_t* __restrict__ part_off, uint32_t nl,
                                   uint32_t* __restrict__ out) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= kSpParts) return;
  const uint32_t lo = part_off[(size_t)p * nl];
  const uint32_t hi = part_off[(size_t)(p + 1) * nl];
  out[p] = hi - lo;
}

__global__ void k_dist_set_fail(SpState* __restrict__ st, uint32_t bits, uint32_t why) {
  if (threadIdx.x != 0) return;
  st->fail |= bits;
  if (why) atomicMax(&st->why, why);
}

// Rank 0, before sorting the gathered points: P_l's position in X (index 0
// = the anchor, 1.. the gathered points sorted by global index gi[0, n_g)).
__global__ void k_dist_find_pl(const int64_t* __restrict__ gi, uint32_t n_g,
                               SpState* __restrict__ st, ExtResult* __restrict__ ext) {
  if (threadIdx.x != 0 || st->fail) return;
  const int64_t want = st->l_idx;
  uint32_t lo = 0, hi = n_g;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) / 2;
    if (gi[mid] < want) lo = mid + 1;
    else hi = mid;
  }
  if (lo < n_g && gi[lo] == want) {
    st->l_idx = 1 + lo;
    ext->idx[4] = 0;
  } else {  // P_l is always in a gathered bucket; anything else is inconsistent
    st->fail |= kSpFailInternal;
    atomicMax(&st->why, 12u);
  }
}

// Rank 0's prefix maxima and its fail word -> the broadcast block
__global__ void k_dist_pref_out(const uint32_t* __restrict__ prefmax, const SpState* __restrict__ st,
                                uint32_t* __restrict__ out) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= kSpBuckets; b += gridDim.x * blockDim.x)
    out[b] = b < kSpBuckets ? prefmax[b] : st->fail;
}

// ... and back on every rank (before F4)
__global__ void k_dist_pref_in(const uint32_t* __restrict__ in, uint32_t* __restrict__ prefmax,
                               SpState* __restrict__ st) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < kSpBuckets; b += gridDim.x * blockDim.x)
    prefmax[b] = in[b];
  if (blockIdx.x == 0 && threadIdx.x == 0) st->fail |= in[kSpBuckets];
}

__global__ void k_dist_rec_f4(const SpState* __restrict__ st, int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  rec[kRxF4 + 0] = st->n_c;
  rec[kRxF4 + 1] = st->fail;
}

// Distributed F6: rank 0's round-2 output and bucket offsets are broadcast;
// every rank verifies its own shard's skipped points against them.
__global__ void k_dist_verify_prep(SpState* __restrict__ st) {
  if (threadIdx.x != 0) return;
  st->need_verify = 1;
  st->verify_fail = 0;
}

__global__ void k_dist_rec_ver(const SpState* __restrict__ st, int64_t* __restrict__ rec) {
  if (threadIdx.x != 0) return;
  rec[kRxVer + 0] = st->verify_fail;
  rec[kRxVer + 1] = st->fail;
}

}  // namespace gscan
