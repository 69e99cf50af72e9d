// On-device gen_square: the reference's input
// sequence, bit for bit, generated on the GPU.
//
// gen_square(n, seed) (datagen.hpp:32-41) draws x then y for every point
// from one std::mt19937_64 through uniform_real_distribution<double>(0, 1),
// i.e. libstdc++'s generate_canonical<double, 53>: one 64-bit engine output
// y per value, (double)y (round to nearest) * 2^-64, and 1 - 2^-53 in place of
// 1.0 (random.tcc:3349-3381, GCC 13). Word w of the engine's output stream is
// point w / 2's x (w even) or y (w odd).
//
// The stream is cut into generators of kMtL words. Generator g starts from
// the engine state after g * kMtL words, obtained by jump-ahead (mt64_jump.h):
// k_mt_jump doubles the set of known states per launch (states [2^b, 2^(b+1))
// = jump by 2^b * kMtL of states [0, 2^b)), each jump the XOR of the stream
// windows selected by the jump polynomial's coefficients. k_mt_gen then runs
// each generator's engine sequentially, one 312-word block at a time in two
// parallel phases (words 0-155 depend only on the previous block, 156-311 on
// the first phase), tempers, converts and stores only the shard's points.
#pragma once
#include <cstdint>

namespace gscan {

constexpr int kMtN = 312;
constexpr int kMtM = 156;
constexpr int kMtDeg = 19937;
constexpr int kMtWords = (kMtDeg + 1 + 63) / 64;       // jump polynomial words
constexpr int kMtStream = kMtN + 64 * kMtN;           // >= kMtDeg + kMtN words of stream per jump
constexpr uint64_t kMtL = 1ull << 20;                 // words per generator
constexpr int kMtThreads = 320;
constexpr size_t kMtJumpSmem = (size_t)kMtStream * 8;

__device__ __forceinline__ uint64_t mt_twist(uint64_t a, uint64_t b) {
  const uint64_t y = (a & (~0ull << 31)) | (b & ((1ull << 31) - 1));
  return (y >> 1) ^ ((b & 1u) ? 0xB5026F5AA96619E9ull : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// generate_canonical<double, 53> with one 64-bit draw, then * (1 - 0) + 0
__device__ __forceinline__ double mt_canonical(uint64_t y) {
  const double d = __dmul_rn(__ull2double_rn(y), 0x1p-64);
  return d >= 1.0 ? 0x1.fffffffffffffp-1 : d;
}

// x[m0, m0 + 312) known -> x[m0 + 312, m0 + 624), CTA-wide (all threads call)
__device__ __forceinline__ void mt_block_smem(uint64_t* x, uint32_t m0) {
  for (uint32_t k = threadIdx.x; k < (uint32_t)kMtM; k += blockDim.x)
    x[m0 + kMtN + k] = x[m0 + kMtM + k] ^ mt_twist(x[m0 + k], x[m0 + k + 1]);
  __syncthreads();
  for (uint32_t k = kMtM + threadIdx.x; k < (uint32_t)kMtN; k += blockDim.x)
    x[m0 + kMtN + k] = x[m0 + kMtM + k] ^ mt_twist(x[m0 + k], x[m0 + k + 1]);
  __syncthreads();
}

// states[2^b + i] = T^(2^b * kMtL) states[i], i < count (one CTA per i).
__global__ void __launch_bounds__(kMtThreads, 1) k_mt_jump(uint64_t* __restrict__ states,
                                                          uint32_t half, uint32_t count,
                                                          const uint64_t* __restrict__ poly) {
  extern __shared__ uint64_t mt_x[];  // kMtStream words of stream
  const uint32_t i = blockIdx.x;
  if (i >= count) return;
  for (uint32_t k = threadIdx.x; k < (uint32_t)kMtN; k += blockDim.x) mt_x[k] = states[(size_t)i * kMtN + k];
  __syncthreads();
  for (uint32_t m0 = 0; m0 + 2 * kMtN <= (uint32_t)kMtStream; m0 += kMtN) mt_block_smem(mt_x, m0);
  // word k of the jumped state = XOR of stream[j + k] over the set coefficients j
  if (threadIdx.x < (uint32_t)kMtN) {
    const uint32_t k = threadIdx.x;
    uint64_t acc = 0;
    for (int w = 0; w < kMtWords; ++w) {
      uint64_t bits = __ldg(&poly[w]);
      while (bits) {
        const int b = __ffsll((long long)bits) - 1;
        bits &= bits - 1;
        acc ^= mt_x[w * 64 + b + k];
      }
    }
    states[((size_t)half + i) * kMtN + k] = acc;
  }
}

// Generator g (= g0 + blockIdx.x) writes the points of words
// [g * kMtL, (g + 1) * kMtL) that fall in [2 lo, 2 hi) to xs/ys[p - lo].
__global__ void __launch_bounds__(kMtThreads) k_mt_gen(const uint64_t* __restrict__ states, uint64_t g0,
                                                     uint64_t lo, uint64_t hi, double* __restrict__ xs,
                                                     double* __restrict__ ys) {
  __shared__ uint64_t buf[2][kMtN];
  const uint64_t g = g0 + blockIdx.x;
  for (uint32_t k = threadIdx.x; k < (uint32_t)kMtN; k += blockDim.x) buf[0][k] = states[(size_t)g * kMtN + k];
  __syncthreads();
  const uint64_t w_lo = 2 * lo, w_hi = 2 * hi;
  const uint64_t gw0 = g * kMtL;
  const uint64_t wb = gw0 > w_lo ? gw0 : w_lo;              // first word this CTA stores
  const uint64_t we = (gw0 + kMtL) < w_hi ? gw0 + kMtL : w_hi;  // end
  // blocks before wb are generated but not stored
  const uint64_t nblk = (we - gw0 + kMtN - 1) / kMtN;
  int cur = 0;
  for (uint64_t bl = 0; bl < nblk; ++bl) {
    const uint64_t* o = buf[cur];
    uint64_t* nw = buf[cur ^ 1];
    for (uint32_t k = threadIdx.x; k < (uint32_t)kMtM; k += blockDim.x)
      nw[k] = o[k + kMtM] ^ mt_twist(o[k], o[k + 1]);
    __syncthreads();
    for (uint32_t k = kMtM + threadIdx.x; k < (uint32_t)kMtN; k += blockDim.x)
      nw[k] = nw[k - kMtM] ^ mt_twist(o[k], k + 1 < (uint32_t)kMtN ? o[k + 1] : nw[0]);
    __syncthreads();
    const uint64_t w0 = gw0 + bl * kMtN;  // word index of nw[0]
    if (w0 + kMtN > wb) {
      for (uint32_t k = threadIdx.x; k < (uint32_t)kMtN; k += blockDim.x) {
        const uint64_t w = w0 + k;
        if (w < wb || w >= we) continue;
        const double v = mt_canonical(mt_temper(nw[k]));
        const uint64_t p = (w >> 1) - lo;
        if (w & 1) ys[p] = v;
        else xs[p] = v;
      }
    }
    cur ^= 1;
  }
}

}  // namespace gscan
