// Read bandwidth of the producer/consumer bulk-copy ring (F2/K1 layout):
// one producer lane fills S stages of T points (x and y tiles, 2 bulk
// copies each) on full[] mbarriers; C consumer warps read the tile from
// shared memory and release it on empty[]. Sweeps T, S, CTAs per SM.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su(b)), "r"(par) : "memory");
}

template <int T, int S, int C>
__global__ void __launch_bounds__(C * 32 + 32) k_ring(const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n, double* out, int work) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sx = (double*)sm;
  double* sy = sx + (size_t)S * T;
  uint64_t* full = (uint64_t*)(sy + (size_t)S * T);
  uint64_t* empty = full + S;
  const uint32_t nt = n / T;
  const uint32_t mine = nt > blockIdx.x ? (nt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[k])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[k])), "r"(C));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  double s = 0;
  if (warp == C) {
    if (lane == 0)
      for (uint32_t k = 0; k < mine; ++k) {
        const uint32_t st = k % S;
        if (k >= S) wait(&empty[st], ((k / S) - 1) & 1);
        const size_t t0 = (size_t)(blockIdx.x + k * gridDim.x) * T;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(T * 16));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sx + (size_t)st * T)), "l"(xs + t0), "r"(T * 8), "r"(su(&full[st])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sy + (size_t)st * T)), "l"(ys + t0), "r"(T * 8), "r"(su(&full[st])) : "memory");
      }
  } else {
    for (uint32_t k = 0; k < mine; ++k) {
      const uint32_t st = k % S;
      wait(&full[st], (k / S) & 1);
      const double2* x2 = (const double2*)(sx + (size_t)st * T);
      const double2* y2 = (const double2*)(sy + (size_t)st * T);
      for (int p = threadIdx.x; p < T / 2; p += C * 32) {
        double2 a = x2[p], b = y2[p];
        double v = a.x * b.y + a.y * b.x;
        for (int w = 0; w < work; ++w) v = v * 1.0000001 + 1e-9;
        s += v;
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])) : "memory");
    }
  }
  if (s == 1.2345) out[0] = s;
}

// the XYRing scheme: no producer warp, the last warp to release a stage refills it
template <int T, int S, int C>
__global__ void __launch_bounds__(C * 32) k_ring_last(const double* __restrict__ xs, const double* __restrict__ ys, uint32_t n, double* out, int work) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* sx = (double*)sm;
  double* sy = sx + (size_t)S * T;
  uint64_t* full = (uint64_t*)(sy + (size_t)S * T);
  uint32_t* cnt = (uint32_t*)(full + S);
  const uint32_t nt = n / T;
  const uint32_t mine = nt > blockIdx.x ? (nt - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint32_t lane = threadIdx.x & 31;
  auto issue = [&](uint32_t k) {
    const uint32_t st = k % S;
    const size_t t0 = (size_t)(blockIdx.x + k * gridDim.x) * T;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(T * 16));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sx + (size_t)st * T)), "l"(xs + t0), "r"(T * 8), "r"(su(&full[st])) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sy + (size_t)st * T)), "l"(ys + t0), "r"(T * 8), "r"(su(&full[st])) : "memory");
  };
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[k]))); cnt[k] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;");
    for (uint32_t k = 0; k < S && k < mine; ++k) issue(k);
  }
  __syncthreads();
  double s = 0;
  for (uint32_t k = 0; k < mine; ++k) {
    const uint32_t st = k % S;
    wait(&full[st], (k / S) & 1);
    const double2* x2 = (const double2*)(sx + (size_t)st * T);
    const double2* y2 = (const double2*)(sy + (size_t)st * T);
    double2 a[T / 2 / (C * 32)], b[T / 2 / (C * 32)];
    for (int u = 0; u < T / 2 / (C * 32); ++u) { a[u] = x2[threadIdx.x + u * C * 32]; b[u] = y2[threadIdx.x + u * C * 32]; }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&cnt[st], 1u) == C - 1) {
        cnt[st] = 0;
        if (k + S < mine) { __threadfence_block(); asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); issue(k + S); }
      }
    }
    for (int u = 0; u < T / 2 / (C * 32); ++u) {
      double v = a[u].x * b[u].y + a[u].y * b[u].x;
      for (int w = 0; w < work; ++w) v = v * 1.0000001 + 1e-9;
      s += v;
    }
  }
  if (s == 1.2345) out[0] = s;
}

template <int T, int S, int C>
void run_last(const double* xs, const double* ys, uint32_t n, double* out, int sms, int work) {
  const size_t smem = (size_t)S * T * 16 + S * 12;
  auto k = k_ring_last<T, S, C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    k<<<sms, C * 32, smem>>>(xs, ys, n, out, work);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r) best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  printf("LAST T=%5d S=%d C=%2d work=%d: %7.1f us  %6.0f GB/s %s\n", T, S, C, work, best * 1e3, n * 16.0 / (best * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
}

template <int T, int S, int C>
void run(const double* xs, const double* ys, uint32_t n, double* out, int sms, int per_sm, int work) {
  const size_t smem = (size_t)S * T * 16 + 2 * S * 8;
  auto k = k_ring<T, S, C>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(a);
    k<<<sms * per_sm, C * 32 + 32, smem>>>(xs, ys, n, out, work);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r) best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  printf("T=%5d S=%d C=%2d ctas/sm=%d work=%d smem=%6zu: %7.1f us  %6.0f GB/s %s\n", T, S, C, per_sm, work, smem, best * 1e3,
         n * 16.0 / (best * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
}

__global__ void k_fill(double* a, uint32_t n, uint64_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t z = (i + seed * 0x9E3779B97F4A7C15ull) * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31; z *= 0x94D049BB133111EBull; z ^= z >> 29;
    a[i] = (z >> 11) * 0x1.0p-53;
  }
}

int main() {
  const uint32_t n = 20000000;
  double *xs, *ys, *out;
  cudaMalloc(&xs, n * 8ull); cudaMalloc(&ys, n * 8ull); cudaMalloc(&out, 8);
  cudaMemset(xs, 0, n * 8ull); cudaMemset(ys, 0, n * 8ull);
  if (getenv("RINGBW_RANDOM")) {  // uniform doubles in [0, 1) instead of zeros
    k_fill<<<1184, 256>>>(xs, n, 1);
    k_fill<<<1184, 256>>>(ys, n, 2);
    cudaDeviceSynchronize();
  }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int work : {0, 8, 32}) {
    run_last<3072, 4, 16>(xs, ys, n, out, sms, work);
    run_last<2048, 4, 16>(xs, ys, n, out, sms, work);
    run_last<2048, 6, 16>(xs, ys, n, out, sms, work);
    run<2048, 4, 16>(xs, ys, n, out, sms, 1, work);
  }
  for (int work : {0, 8}) {
    run<1920, 4, 15>(xs, ys, n, out, sms, 1, work);
    run<1920, 6, 15>(xs, ys, n, out, sms, 1, work);
    run<3840, 3, 15>(xs, ys, n, out, sms, 1, work);
    run<4096, 3, 16>(xs, ys, n, out, sms, 1, work);
    run<1024, 4, 8>(xs, ys, n, out, sms, 2, work);
    run<1024, 6, 8>(xs, ys, n, out, sms, 2, work);
    run<2048, 3, 8>(xs, ys, n, out, sms, 2, work);
    run<512, 8, 4>(xs, ys, n, out, sms, 4, work);
  }
  return 0;
}
