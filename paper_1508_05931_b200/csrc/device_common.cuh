// Device primitives shared by the gScan kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "glibc_atan2.h"

namespace gscan {

// Programmatic dependent launch: kernels of the sparse path's chain are
// launched with programmatic stream serialization (launch_pdl in gscan.cu),
// so the next grid is staged while the current one drains; every such kernel
// first waits here for its predecessor's completion and memory (a no-op when
// launched normally).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

constexpr int kBlock = 256;   // threads per CTA for the streaming kernels
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kDead = 0xffffffffu;        // index marker: duplicate dropped
constexpr uint64_t kKeyDrop = ~0ull;           // sort key marker: coincides with anchor

// ---------------------------------------------------------------------------
// Exact predicates. Every op is an explicit round-to-nearest intrinsic so the
// compiler cannot contract a*b-c*d into an FMA: the reference's cross() is
// plain double arithmetic without FMA (geom.hpp:19-21).

// (b.x-a.x)(c.y-a.y) - (b.y-a.y)(c.x-a.x), geom.hpp:19-21.
__device__ __forceinline__ double cross_rn(double ax, double ay, double bx, double by, double cx,
                                           double cy) {
  return __dsub_rn(__dmul_rn(__dsub_rn(bx, ax), __dsub_rn(cy, ay)),
                   __dmul_rn(__dsub_rn(by, ay), __dsub_rn(cx, ax)));
}

// Same value with the edge vector (ex, ey) = (b.x-a.x, b.y-a.y) precomputed
// (identical rounding: the subtraction is the same operation).
__device__ __forceinline__ double cross_edge(double ax, double ay, double ex, double ey, double cx,
                                             double cy) {
  return __dsub_rn(__dmul_rn(ex, __dsub_rn(cy, ay)), __dmul_rn(ey, __dsub_rn(cx, ax)));
}

// dist2 = dx*dx + dy*dy, geom.hpp:42 (no FMA).
__device__ __forceinline__ double dist2_rn(double dx, double dy) {
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

__device__ __forceinline__ uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
__device__ __forceinline__ double bitsd(uint64_t u) { return __longlong_as_double((long long)u); }

// ---------------------------------------------------------------------------
// Decoupled look-back (single-pass chained scan) over per-tile aggregates.
// Status word: bits 62-63 = flag, low 62 bits = value.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagPre = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  *reinterpret_cast<volatile uint64_t*>(p) = v;
}

// Called by all 32 lanes of ONE warp. Publishes `agg` for `tile` and returns
// the exclusive prefix of all earlier tiles (same value in every lane).
__device__ __forceinline__ uint64_t lookback_exclusive(uint64_t* status, uint32_t tile,
                                                       uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) {
      __threadfence();
      st_volatile(&status[0], kFlagPre | agg);
    }
    return 0;
  }
  if (lane == 0) {
    __threadfence();
    st_volatile(&status[tile], kFlagAgg | agg);
  }
  uint64_t excl = 0;
  int64_t look = (int64_t)tile - 1;
  while (true) {
    const int64_t t = look - lane;
    uint64_t w = kFlagPre;  // lanes past tile 0 read as an empty prefix
    if (t >= 0) {
      do {
        w = ld_volatile(&status[t]);
      } while ((w >> 62) == 0);
    }
    const uint32_t pre_mask = __ballot_sync(0xffffffffu, (w & kFlagPre) != 0);
    const int first_pre = pre_mask ? (__ffs(pre_mask) - 1) : 32;
    uint64_t v = (lane <= first_pre && t >= 0) ? (w & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (pre_mask) break;
    look -= 32;
  }
  if (lane == 0) {
    __threadfence();
    st_volatile(&status[tile], kFlagPre | (excl + agg));
  }
  return excl;
}


// ---- bulk copies (TMA, non-tensor) into shared memory, mbarrier-completed ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive (count 1) and add the transaction bytes the pending copies will deliver
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// plain arrive (count 1), e.g. a consumer warp releasing a ring stage
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// global -> shared, `bytes` a multiple of 16, both addresses 16 B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- XY tile ring: SoA (xs, ys) streamed through shared memory ----
// Each CTA takes tiles b, b + G, b + 2G, ... of kT points. Stage st holds
// one tile of xs and one of ys, filled by two bulk copies completed on
// full[st]. There is no producer warp: the LAST warp to finish reading a
// stage (a shared-memory counter) refills it with the CTA's tile k + kS, so
// every warp is a consumer, warps never wait on each other except through the
// data, and kS tiles are in flight per CTA. Needs 16-byte aligned xs, ys.
template <int kT, int kS>
struct XYRing {
  static constexpr size_t kSmem = (size_t)kS * kT * 16 + (size_t)kS * 16 + (size_t)kS * 4;
  double* sx;        // [kS][kT]
  double* sy;        // [kS][kT]
  uint64_t* full;    // [kS] the stage's tile has landed (bulk-copy transaction bytes)
  uint64_t* empty;   // [kS] every thread has read the stage (one arrival per thread)
  uint32_t* cnt;     // [kS] arrivals so far: elects the last warp as the refiller
  const double* xs;
  const double* ys;
  uint32_t mine;     // tiles of this CTA
  uint32_t nwarps;

  __device__ __forceinline__ void setup(unsigned char* smem, const double* x, const double* y,
                                        uint32_t n) {
    sx = reinterpret_cast<double*>(smem);
    sy = sx + (size_t)kS * kT;
    full = reinterpret_cast<uint64_t*>(sy + (size_t)kS * kT);
    empty = full + kS;
    cnt = reinterpret_cast<uint32_t*>(empty + kS);
    xs = x;
    ys = y;
    const uint32_t ntiles = n / kT;
    mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
    nwarps = blockDim.x >> 5;
  }
  __device__ __forceinline__ uint32_t tile_start(uint32_t k) const {
    return (blockIdx.x + k * gridDim.x) * (uint32_t)kT;
  }
  __device__ __forceinline__ void issue(uint32_t k) {
    const uint32_t st = k % kS;
    const size_t t0 = tile_start(k);
    mbar_expect_tx(&full[st], 2u * kT * 8u);
    bulk_g2s(sx + (size_t)st * kT, xs + t0, kT * 8u, &full[st]);
    bulk_g2s(sy + (size_t)st * kT, ys + t0, kT * 8u, &full[st]);
  }
  // thread 0: barriers and the first kS tiles (the caller then __syncthreads)
  __device__ __forceinline__ void start() {
    if (threadIdx.x == 0) {
      for (int k = 0; k < kS; ++k) {
        mbar_init(&full[k], 1);
        mbar_init(&empty[k], blockDim.x);
        cnt[k] = 0;
      }
      mbar_fence_init();
      for (uint32_t k = 0; k < (uint32_t)kS && k < mine; ++k) issue(k);
    }
  }
  __device__ __forceinline__ void wait(uint32_t k) { mbar_wait(&full[k % kS], (k / kS) & 1u); }
  __device__ __forceinline__ const double* tx(uint32_t k) const { return sx + (size_t)(k % kS) * kT; }
  __device__ __forceinline__ const double* ty(uint32_t k) const { return sy + (size_t)(k % kS) * kT; }
  // The calling warp is done reading tile k (its values are in registers): its
  // threads arrive on empty[st] (release); the last warp to arrive -- elected by the
  // counter -- waits for that phase (acquire: every warp's reads of the stage
  // are ordered before), fences the async proxy and refills the stage.
  __device__ __forceinline__ void release(uint32_t k) {
    const uint32_t st = k % kS;
    mbar_arrive(&empty[st]);  // every thread: its own reads are released
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      if (atomicAdd(&cnt[st], 1u) == nwarps - 1) {
        cnt[st] = 0;
        mbar_wait(&empty[st], (k / kS) & 1u);
        if (k + kS < mine) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // reads before the async writes
          issue(k + kS);
        }
      }
    }
  }
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Tiles of kBlock x ITEMS items in STRIPED order (item (k, t) = base + k *
// kBlock + t): every warp-wide load and store of a row is coalesced. The
// exclusive scan of the ITEMS x kWarps row counts (row-major = index order),
// by warp 0: s_rows[r] becomes the exclusive offset of row r and
// s_rows[ITEMS * kWarps] the tile total. All threads call it.
template <int ITEMS>
__device__ __forceinline__ uint32_t striped_rows_scan(uint32_t* s_rows) {
  __syncthreads();  // the row counts are written
  if ((threadIdx.x >> 5) == 0) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t carry = 0;
#pragma unroll
    for (int b = 0; b < ITEMS * kWarps; b += 32) {
      const bool in = b + (int)lane < ITEMS * kWarps;
      const uint32_t v = in ? s_rows[b + lane] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if ((int)lane >= o) x += y;
      }
      if (in) s_rows[b + lane] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) s_rows[ITEMS * kWarps] = carry;
  }
  __syncthreads();
  return s_rows[ITEMS * kWarps];
}

// Ranks (index order) of the kept items of a striped tile; returns the tile's
// kept count. s_rows: ITEMS * kWarps + 1 words.
template <int ITEMS>
__device__ __forceinline__ uint32_t striped_keep_ranks(const bool (&keep)[ITEMS], uint32_t (&rank)[ITEMS],
                                                       uint32_t* s_rows) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bal[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    bal[k] = __ballot_sync(0xffffffffu, keep[k]);
    if (lane == 0) s_rows[k * kWarps + warp] = __popc(bal[k]);
  }
  const uint32_t total = striped_rows_scan<ITEMS>(s_rows);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) rank[k] = s_rows[k * kWarps + warp] + __popc(bal[k] & lanemask_lt());
  return total;
}

// Exclusive prefix (index order) of per-item counts of a striped tile;
// returns the tile total.
template <int ITEMS>
__device__ __forceinline__ uint32_t striped_exclusive(const uint32_t (&v)[ITEMS], uint32_t (&ex)[ITEMS],
                                                      uint32_t* s_rows) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    uint32_t x = v[k];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)lane >= o) x += y;
    }
    incl[k] = x;
    if (lane == 31) s_rows[k * kWarps + warp] = x;
  }
  const uint32_t total = striped_rows_scan<ITEMS>(s_rows);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) ex[k] = s_rows[k * kWarps + warp] + incl[k] - v[k];
  return total;
}

}  // namespace gscan
