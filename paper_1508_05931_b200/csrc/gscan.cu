#include <chrono>
// Host orchestration and C-ABI of the B200 gScan hull path (include/gscan.h).
//
// One call = the reference's full_pipeline (pipeline.hpp:72-123) as a chain
// of sm_100a kernels on one stream:
//   K1 extremes+anchor -> K2 quad filter + stable compaction -> K3 polar keys
//   + bucket histogram -> bucket offsets (scan) -> scatter -> K4 per-bucket
//   sort + dedup -> split_regions -> K5 round-2 walks -> stable compaction
//   -> K7 Graham scan.
// Sizes that steer launches are read back at most twice per call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/gscan.h"
#include "kernels.cuh"
#include "graham.cuh"
#include "sparse.cuh"
#include "graham_tree.cuh"
#include "mtgen.cuh"
#include "mt64_jump.h"

using namespace gscan;

namespace {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ~ns of GPU time (profiling mode only; see run_sparse)
#ifdef GSCAN_STAMP
__global__ void k_stamp(unsigned long long* p) { *p = globaltimer_ns(); }
double g_host[4], g_host_prev_gap = 0, g_host_last_exit = 0;
void host_mark(int k) {
  const double t = std::chrono::duration<double, std::micro>(
                       std::chrono::steady_clock::now().time_since_epoch()).count();
  static std::vector<double> hrows;
  if (k == 0 && g_host_last_exit > 0) {
    hrows.push_back(g_host[1] - g_host[0]);
    hrows.push_back(g_host[2] - g_host[1]);
    hrows.push_back(g_host[3] - g_host[2]);
    hrows.push_back(t - g_host_last_exit);
    if (hrows.size() == 4 * 40) {
      for (size_t r = 0; r < hrows.size(); r += 4)
        fprintf(stderr, "[host] entry->launch %.1f, launch->sync return %.1f, sync return->exit %.1f, exit->entry %.1f us\n",
                hrows[r], hrows[r + 1], hrows[r + 2], hrows[r + 3]);
      hrows.clear();
    }
  }
  g_host[k] = t;
  if (k == 3) g_host_last_exit = t;
}
#endif
// The hull (count read on the device) into the caller's buffer, capacity-bounded.
__global__ void k_copy_out(const uint32_t* __restrict__ src, const Counters* __restrict__ ctr,
                           uint32_t* __restrict__ dst, uint64_t cap) {
  const uint64_t k = min((uint64_t)ctr->hull, cap);
  for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_busy_wait(unsigned long long ns) {
  const unsigned long long t0 = globaltimer_ns();
  while (globaltimer_ns() - t0 < ns) __nanosleep(1000);
}

constexpr double kPi = 3.14159265358979323846;

struct KernelTime {
  const char* name;
  cudaEvent_t a, b;
};

}  // namespace

struct SpGraphKey {
  const double* xs = nullptr;
  const double* ys = nullptr;
  uint32_t n = 0;
  uint64_t chunks = 0;
  uint32_t debug = 0;
  bool dup = true;
  bool k1_done = false;  // extremes already computed (overlapped ingest)
  // buffers the full-sort path may swap (stage_annotate_sort): the graph bakes
  // their addresses in, so they are part of the key
  const void* bufs[7] = {};  // + the tree workspace
  bool operator==(const SpGraphKey& o) const {
    for (int k = 0; k < 7; ++k)
      if (bufs[k] != o.bufs[k]) return false;
    return xs == o.xs && ys == o.ys && n == o.n && chunks == o.chunks && debug == o.debug &&
           dup == o.dup && k1_done == o.k1_done;
  }
};

struct gscan_handle {
  int device = 0;
  // on-device gen_square (mtgen.cuh): engine states per generator, jump table
  uint64_t* mt_states = nullptr;
  uint64_t mt_states_cap = 0;  // generators
  uint64_t* mt_jtab = nullptr;
  int mt_jtab_nb = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;          // duplicate check runs here, overlapping the tail
  cudaStream_t cap_stream = nullptr;    // CUDA graph capture
  cudaEvent_t ev_f3 = nullptr, ev_dup = nullptr, ev_part = nullptr;
  bool own_stream = false;
  int sm_count = 148;
  uint64_t cap = 0;  // points
  uint64_t nb_cap = 0;
  // large mode (cap > kFullSortMaxN): the buffers only the full sort needs at
  // full size are sized for the sparse path's walk (wcap elements), and the
  // full-sort fallback is unavailable on one device
  bool large = false;
  uint64_t wcap = 0;
  uint64_t host_cap = 0;  // d_xs/d_ys (host entry only), allocated on first use
  // overlapped ingest: copy stream, per-chunk events, chunk extremes
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_chunk[8] = {};
  ExtResult* ext_parts = nullptr;
  uint32_t* ext_off = nullptr;
  ExtAcc* ext_pp = nullptr;       // per-chunk K1 partials (sm_count each)
  Counters* ext_pctr = nullptr;   // per-chunk tickets
  bool k1_done = false;           // the next run_sparse may skip K1
  std::string err;
  uint64_t launches = 0;
  bool profiling = false;
  std::vector<KernelTime> ktimes;
  size_t kt_used = 0;

  // device buffers
  double *d_xs = nullptr, *d_ys = nullptr;
  uint32_t* surv = nullptr;
  uint64_t* keys = nullptr;
  uint32_t* rank = nullptr;
  PtRec* rec = nullptr;
  double *A_x = nullptr, *A_y = nullptr;
  uint32_t* A_i = nullptr;
  double *C_x = nullptr, *C_y = nullptr;
  uint32_t* C_i = nullptr;
  uint8_t* flags = nullptr;
  uint32_t* stack = nullptr;
  uint32_t* d_out = nullptr;
  // the caller's device output of the current gscan_hull_f64_device call:
  // the sparse path copies the hull there on the device before its one sync
  uint32_t* user_out = nullptr;
  uint64_t user_cap = 0;
  bool user_out_done = false;
  uint64_t* status = nullptr;
  uint64_t status_cap = 0;
  uint32_t *hist = nullptr, *bstart = nullptr, *cursor = nullptr, *oversize = nullptr;
  BucketBest* best = nullptr;  // per-block partials of the sort kernels
  uint64_t best_cap = 0;
  // Graham scratch
  uint32_t *g_chain = nullptr, *g_len = nullptr, *g_off = nullptr, *g_q0 = nullptr, *g_q1 = nullptr;
  uint32_t *g_parent = nullptr, *g_btop = nullptr, *g_jk = nullptr, *g_je = nullptr;
  int32_t* g_jmin = nullptr;
  uint32_t *g_keep = nullptr, *g_misc = nullptr;  // misc: [0] fail, [1] len, [2] ovf, [3] which
  uint32_t *g_stA = nullptr, *g_stB = nullptr, *g_lenA = nullptr, *g_lenB = nullptr,
           *g_scr = nullptr;
  uint64_t g_st_cap = 0, g_len_cap = 0;  // entries per state buffer / per length array
  ExtAcc* partials = nullptr;
  ExtResult* ext = nullptr;
  Counters* ctr = nullptr;
  unsigned long long* scratch64 = nullptr;  // [0] max bits, [1] min pos (as u32 in low half)
  Counters* h_ctr = nullptr;  // pinned mirror
  uint32_t* h_out = nullptr;  // pinned staging for indices
  uint64_t h_out_cap = 0;
  cudaEvent_t ev[8] = {};
  uint32_t debug = 0;  // GSCAN_DEBUG_* test hooks
  uint32_t graham_fails = 0;
  uint32_t graham_path = 0;  // 0 sequential kernel, 1 chains+certificate, 2 junctions+certificate

  // sparse round-2 path (sparse.cuh)
  int sp_grid = 0;
  double* sp_th = nullptr;   // bucket boundary angles, kSpBuckets + 1 (per call)
  double* sp_cdf = nullptr;  // sampled pseudo-angle CDF, kSpCells + 1 (per call)
  uint32_t* sp_cells = nullptr;  // sample counts per cell
  uint32_t* sp_big = nullptr;    // candidate buckets for the CTA sorter
  uint32_t* sp_bigg = nullptr;   // gathered buckets for the CTA sorter
  uint32_t* sp_hugeg = nullptr;  // gathered buckets above kSpGatherCap
  unsigned char* sp_huge_scr = nullptr;  // their per-CTA global scratch (sm_count areas)
  uint32_t sp_huge_cap = 0;      // elements per area (0: inputs too small to need it)
  uint64_t* sp_dup_scr = nullptr;  // duplicate check: sub-partition scratch of large partitions
  uint32_t sp_dup_scap = 0;        // entries per (CTA, group) area
  uint32_t* sp_exc = nullptr;      // F2 screen: points for the exact pass
  uint32_t sp_exc_cap = 0;
  uint32_t *sp_gcount = nullptr, *sp_ccount = nullptr, *sp_hcount = nullptr;  // per-CTA emissions
  uint64_t* sp_dup2 = nullptr;   // partitioned hash list (n)
  uint64_t* sp_side_status = nullptr;  // look-back status of the side stream's scan
  uint32_t* sp_side_work = nullptr;    // work tickets of the two side kernels
  Counters* sp_side_ticket = nullptr;
  bool sp_debug = false, sp_no_dup = false;
  // captured CUDA graph of the sparse path (sparse_enqueue)
  bool use_graphs = true, sp_graph_ok = false;
  cudaGraphExec_t sp_graph_exec = nullptr;
  SpGraphKey sp_key{};
  uint64_t sp_graph_launches = 0;
  uint32_t sp_cert = 0;
  uint16_t* sp_codes = nullptr;  // per-point bucket code (n)
  float* sp_phi32 = nullptr;     // per-point walk angle from F3 (n)
  uint32_t *sp_hist_part = nullptr, *sp_phi_part = nullptr, *sp_part_off = nullptr;
  SpD2* sp_d2 = nullptr;
  uint32_t *sp_hist = nullptr, *sp_bstart = nullptr, *sp_gbits = nullptr, *sp_glist = nullptr,
           *sp_gcnt = nullptr, *sp_phimax = nullptr, *sp_prefmax = nullptr, *sp_slice = nullptr,
           *sp_ccnt = nullptr, *sp_cstart = nullptr, *sp_wcnt = nullptr, *sp_wstart = nullptr,
           *sp_rlo = nullptr;
  uint32_t *sp_seglo = nullptr, *sp_seghi = nullptr;
  uint64_t sp_seg_cap = 0;
  SpState* sp_st = nullptr;
  SpState* h_sp = nullptr;  // pinned mirror
  // n-sized
  uint32_t *sp_eb = nullptr, *sp_Wb = nullptr, *sp_Ws = nullptr, *sp_Rb = nullptr, *sp_Rs = nullptr;
  double *sp_gx = nullptr, *sp_gy = nullptr;  // gathered points' coordinates (F3 region slots)
  uint64_t* sp_dup = nullptr;  // per-CTA hash lists (n)
  uint32_t sp_used = 0, sp_fail = 0, sp_walked = 0, sp_calls = 0, sp_fallbacks = 0;
  // Graham tree strategy pool (graham_tree.cuh)
  uint32_t* tw_pool = nullptr;  // tree strategy workspace (graham_tree.cuh)
  uint32_t tw_nmax = 0, tw_nch1 = 0;
  TreeWork tw{};
  uint32_t* h_info = nullptr;   // pinned mirror of the tree strategy's info words
  // sharded sparse path (gscan_dist_*): this rank's shard and scratch
  const double* dist_xs = nullptr;
  const double* dist_ys = nullptr;
  uint32_t dist_n = 0, dist_base = 0;
  uint64_t dist_chunks = 0;
  float* sp_thr = nullptr;  // F4 candidate thresholds per bucket
  // look-back state of the sparse path's scans, one slot per use, cleared once
  // per call (sp_seg_init) instead of two memsets per scan
  uint64_t* lb_status = nullptr;
  Counters* lb_ctr = nullptr;
  uint64_t lb_stride = 0;  // status words per slot
  uint32_t *sp_gs = nullptr, *sp_gsz = nullptr, *dist_ctr = nullptr, *dist_pm = nullptr,
           *dist_hc = nullptr;
  uint64_t* dist_lb = nullptr;
  // device-side data plane (gscan_dist_enq_*): this rank's record, the
  // gathered records of all ranks, the combined extremes, partition counts
  // and the prefix-maxima broadcast block
  int64_t *dist_rec = nullptr, *dist_recs = nullptr, *dist_ext = nullptr;
  uint32_t *dist_pc = nullptr, *dist_pref = nullptr;
};

namespace {

int fail(gscan_handle* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  return code;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(h, GSCAN_E_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void free_buffers(gscan_handle* h) {
  h->sp_graph_ok = false;
  dfree(h->surv); dfree(h->keys); dfree(h->rank);
  dfree(h->rec); dfree(h->A_x); dfree(h->A_y); dfree(h->A_i); dfree(h->C_x); dfree(h->C_y);
  dfree(h->C_i); dfree(h->flags); dfree(h->stack); dfree(h->d_out); dfree(h->status);
  dfree(h->hist); dfree(h->bstart); dfree(h->cursor); dfree(h->oversize); dfree(h->best);
  dfree(h->g_chain); dfree(h->g_len); dfree(h->g_off); dfree(h->g_q0); dfree(h->g_q1);
  dfree(h->g_parent); dfree(h->g_btop); dfree(h->g_jk); dfree(h->g_je); dfree(h->g_jmin);
  dfree(h->g_keep); dfree(h->g_misc);
  dfree(h->g_stA); dfree(h->g_stB); dfree(h->g_lenA); dfree(h->g_lenB); dfree(h->g_scr);
  dfree(h->lb_status); dfree(h->lb_ctr); dfree(h->sp_eb); dfree(h->sp_gx); dfree(h->sp_gy); dfree(h->sp_Wb); dfree(h->sp_Ws); dfree(h->sp_Rb); dfree(h->sp_Rs); dfree(h->sp_dup);
  dfree(h->sp_codes); dfree(h->sp_phi32); dfree(h->sp_dup2); dfree(h->tw_pool); dfree(h->sp_huge_scr); dfree(h->sp_dup_scr); dfree(h->sp_exc);
  h->tw_nmax = 0;
  h->g_st_cap = 0;
  h->g_len_cap = 0;
  h->cap = 0;
  h->nb_cap = 0;
  h->status_cap = 0;
}

constexpr uint32_t kCtaSortGrid = 296;

uint32_t buckets_for(uint64_t n) {
  uint64_t want = (n + 7) / 8;
  uint32_t nb = 1;
  while (nb < want && nb < (1u << 24)) nb <<= 1;
  return nb;
}

// Per-CTA emission regions of the sparse streaming passes: CTA c owns
// [c * cap, (c + 1) * cap), cap bounding the points one CTA visits.
uint32_t sparse_region_cap(const gscan_handle* h, uint64_t n) {
  uint64_t cap = 0;
  for (const uint64_t t : {(uint64_t)kSpThreads, (uint64_t)kSpCandThreads}) {
    const uint64_t nth = (uint64_t)h->sp_grid * t;
    cap = std::max<uint64_t>(cap, 2ull * t * ((n / 2 + nth - 1) / nth) + 2);
  }
  return (uint32_t)cap;
}

// look-back slots of the sparse path's scans (scan_u32_slot)
enum LbSlot { kLbBstart = 0, kLbGs, kLbCstart, kLbWstart, kLbCompact, kLbSlots };

constexpr uint64_t kSparseMinN = 1u << 16;  // smaller inputs take the full sort

// Above this many points one device runs the sparse path only: the full
// sort's per-point buffers (~120 B/pt) would not fit next to the input and
// the sparse path's own (~50 B/pt) at 1B points. GSCAN_LARGE_MIN (dev/tests)
// lowers the threshold.
constexpr uint64_t kFullSortMaxN = 400000000ull;

uint64_t full_sort_max(void) {
  const char* v = getenv("GSCAN_LARGE_MIN");
  return (v && *v) ? strtoull(v, nullptr, 10) : kFullSortMaxN;
}

int reserve(gscan_handle* h, uint64_t n) {
  if (n <= h->cap) return GSCAN_OK;
  free_buffers(h);
  const uint64_t m = n + 1;
  h->large = n > full_sort_max();
  // walk-side buffers: full size, or in large mode the sparse path's bound on
  // gathered + candidate points (checked on the device, k_sp_emit_place)
  h->wcap = h->large ? std::max<uint64_t>(n / 12, 1ull << 23) : m;
  const uint64_t mw = h->wcap;
  // the sparse path's emission regions may span more slots than points
  const uint64_t mr = std::max<uint64_t>(m, (uint64_t)h->sp_grid * sparse_region_cap(h, n) + 64);
  CU(cudaMalloc(&h->surv, mr * 4));
  CU(cudaMalloc(&h->keys, mw * 8));
  CU(cudaMalloc(&h->rank, mr * 4));
  CU(cudaMalloc(&h->rec, mw * sizeof(PtRec)));
  CU(cudaMalloc(&h->A_x, mw * 8));
  CU(cudaMalloc(&h->A_y, mw * 8));
  CU(cudaMalloc(&h->A_i, mw * 4));
  CU(cudaMalloc(&h->C_x, mw * 8));
  CU(cudaMalloc(&h->C_y, mw * 8));
  CU(cudaMalloc(&h->C_i, mw * 4));
  CU(cudaMalloc(&h->flags, mw));
  CU(cudaMalloc(&h->stack, mw * 4));
  CU(cudaMalloc(&h->d_out, mw * 4));
  const uint32_t nb = buckets_for(n);
  h->nb_cap = nb;
  CU(cudaMalloc(&h->hist, (nb + 2) * 4));
  CU(cudaMalloc(&h->bstart, (nb + 2) * 4));
  CU(cudaMalloc(&h->cursor, (nb + 2) * 4));
  CU(cudaMalloc(&h->oversize, (nb + 2) * 4));
  h->best_cap = (nb + kBucketsPerBlock - 1) / kBucketsPerBlock + kCtaSortGrid + 1;
  CU(cudaMalloc(&h->best, h->best_cap * sizeof(BucketBest)));
  const uint64_t nch = (mw + kChunk - 1) / kChunk + 2;
  CU(cudaMalloc(&h->g_chain, mw * 4));
  CU(cudaMalloc(&h->g_len, nch * 4));
  CU(cudaMalloc(&h->g_off, (nch + 1) * 4));
  CU(cudaMalloc(&h->g_q0, mw * 4));
  CU(cudaMalloc(&h->g_q1, mw * 4));
  CU(cudaMalloc(&h->g_parent, mw * 4));
  CU(cudaMalloc(&h->g_btop, (nch + 1) * 4));
  CU(cudaMalloc(&h->g_jk, nch * 4));
  CU(cudaMalloc(&h->g_je, nch * 4));
  CU(cudaMalloc(&h->g_jmin, nch * 4));
  CU(cudaMalloc(&h->g_keep, nch * 4));
  CU(cudaMalloc(&h->g_misc, 256));
  const uint64_t tiles = std::max((m + kCompactTile - 1) / kCompactTile,
                                  (uint64_t)(nb + 2 + kScanTile - 1) / kScanTile) + 64 +
                         // the sharded path scans kSpParts x (hash lists | ranks) counts
                         ((uint64_t)kSpParts * std::max(2 * h->sm_count, 64) + kScanTile) / kScanTile;
  h->status_cap = tiles;
  CU(cudaMalloc(&h->status, tiles * 8));
  h->lb_stride = std::max<uint64_t>((kSpBuckets + 2 + kScanTile - 1) / kScanTile,
                                    m / kCompactTile + 2) + 2;
  CU(cudaMalloc(&h->lb_status, (size_t)kLbSlots * h->lb_stride * 8));
  CU(cudaMalloc(&h->lb_ctr, (size_t)kLbSlots * sizeof(Counters)));
  CU(cudaMalloc(&h->sp_eb, mr * 4));
  CU(cudaMalloc(&h->sp_gx, mr * 8));
  CU(cudaMalloc(&h->sp_gy, mr * 8));
  CU(cudaMalloc(&h->sp_Wb, mw * 4));
  CU(cudaMalloc(&h->sp_Ws, mw * 4));
  CU(cudaMalloc(&h->sp_Rb, mw * 4));
  CU(cudaMalloc(&h->sp_Rs, mw * 4));
  CU(cudaMalloc(&h->sp_dup, (mr + 4096) * 8));
  // partitioned hashes: the runs are padded to whole sectors (k_sp_dup_part<true>)
  CU(cudaMalloc(&h->sp_dup2, (m + 4096 + 3ull * kSpParts * 2 * (uint64_t)h->sm_count) * 8));
  // gathered buckets above the shared-memory sorter (about n1 / kSpBuckets
  // points each, n1 / n ~ 1/3 - 2/3 for squares): per-CTA global scratch for
  // up to 8x the mean bucket of n points (1B square, seed 1: mean gathered
  // bucket 13.8K, largest 88.7K = 4.4x n / kSpBuckets)
  h->sp_huge_cap = 0;
  if (n >= kSparseMinN) {
    h->sp_huge_cap = (uint32_t)std::max<uint64_t>(2 * kSpGatherCap, 8 * (n / kSpBuckets) + 64);
    CU(cudaMalloc(&h->sp_huge_scr,
                  (size_t)h->sm_count * ((size_t)h->sp_huge_cap * kSpHugeBytes + 16)));
  }
  // duplicate check of partitions above kSpDupMaxRounds rounds (n1 / kSpParts
  // hashes each, n1 <= n): sub-partition scratch for up to 2x the mean
  // partition of n points
  h->sp_dup_scap = 0;
  if (n / kSpParts > (uint64_t)kSpDupMaxRounds * kSpDupGRound) {
    h->sp_dup_scap = (uint32_t)(2 * (n / kSpParts) + 4096);
    CU(cudaMalloc(&h->sp_dup_scr, (size_t)h->sm_count * kSpDupGroups * h->sp_dup_scap * 8));
  }
  // F2's uncertain points (~2e-4 of them; more than n/32 declines)
  h->sp_exc_cap = (uint32_t)(n / 32 + 8192);
  CU(cudaMalloc(&h->sp_exc, (size_t)h->sp_exc_cap * 4));
  CU(cudaMalloc(&h->sp_codes, (m + 1) * sizeof(uint16_t)));
  CU(cudaMalloc(&h->sp_phi32, (m + 1) * sizeof(float)));
  h->cap = n;
  return GSCAN_OK;
}

// Development switches: set and not "0".
bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && strcmp(v, "0") != 0;
}

// ---- launch bookkeeping (counts every kernel; optional per-kernel events) ----
struct Launch {
  gscan_handle* h;
  const char* name;
  KernelTime* kt = nullptr;
  cudaStream_t st;
  Launch(gscan_handle* hh, const char* nm, cudaStream_t s = nullptr)
      : h(hh), name(nm), st(s ? s : hh->stream) {
    ++h->launches;
    if (h->profiling) {
      if (h->kt_used == h->ktimes.size()) {
        KernelTime t{};
        cudaEventCreate(&t.a);
        cudaEventCreate(&t.b);
        h->ktimes.push_back(t);
      }
      kt = &h->ktimes[h->kt_used++];
      kt->name = nm;
      cudaEventRecord(kt->a, st);
    }
  }
  ~Launch() {
    if (kt) cudaEventRecord(kt->b, st);
  }
};

// A kernel of the sparse path's chain, launched with programmatic stream
// serialization: the grid is staged while its predecessor drains and starts
// with pdl_wait() (device_common.cuh). Captured into the sparse graph as a
// programmatic dependency edge.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // errors: cudaGetLastError
}

// Exclusive scan on a pre-cleared look-back slot (no memsets: one graph node).
int scan_u32_slot(gscan_handle* h, const uint32_t* in, uint32_t n, uint32_t* out, int slot,
                  cudaStream_t s) {
  const uint64_t tiles = (n + 1 + kScanTile - 1) / kScanTile;
  if (tiles > h->lb_stride) return fail(h, GSCAN_E_INTERNAL, "look-back slot too small");
  Launch L(h, "k_scan_u32", s);
  launch_pdl(k_scan_u32, tiles, kBlock, 0, s, in, n, out, h->lb_status + (size_t)slot * h->lb_stride,
                                      h->lb_ctr + slot);
  return GSCAN_OK;
}

int reset_lookback(gscan_handle* h, uint64_t tiles) {
  if (tiles > h->status_cap) return fail(h, GSCAN_E_INTERNAL, "look-back status too small");
  CU(cudaMemsetAsync(h->status, 0, tiles * 8, h->stream));
  CU(cudaMemsetAsync(&h->ctr->tile_ticket, 0, 4, h->stream));
  return GSCAN_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int sync_counters(gscan_handle* h) {
  CU(cudaMemcpyAsync(h->h_ctr, h->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

#define TRY(x)                  \
  do {                          \
    int rc_ = (x);              \
    if (rc_ != GSCAN_OK) return rc_; \
  } while (0)

// K1 + K2 (round 1). Leaves survivors in h->surv and n1 in ctr. With
// `quad_override` (distributed use: the quadrilateral of the GLOBAL extremes),
// K1 is skipped and the given ExtResult is used.
int stage_round1(gscan_handle* h, const double* xs, const double* ys, uint32_t n, int enable,
                 const ExtResult* quad_override = nullptr, bool ordered = false) {
  const bool vec = aligned16(xs) && aligned16(ys);
  if (quad_override) {
    CU(cudaMemcpyAsync(h->ext, quad_override, sizeof(ExtResult), cudaMemcpyHostToDevice, h->stream));
  } else {
    const uint32_t grid =
        std::max(1u, std::min<uint32_t>((n + kBlock * 8 - 1) / (kBlock * 8), h->sm_count * 8));
    Launch L(h, "k_extremes");
    if (vec) k_extremes<true><<<grid, kBlock, 0, h->stream>>>(xs, ys, n, h->partials, h->ext, h->ctr);
    else k_extremes<false><<<grid, kBlock, 0, h->stream>>>(xs, ys, n, h->partials, h->ext, h->ctr);
  }
  const uint64_t tiles = (n + kFilterTile - 1) / kFilterTile;
  if (ordered) TRY(reset_lookback(h, tiles));
  {
    Launch L(h, "k_filter_compact");
#define K2_ARGS xs, ys, n, h->ext, enable, h->status, h->surv, h->ctr
    if (vec && ordered) k_filter_compact<true, true><<<tiles, kBlock, 0, h->stream>>>(K2_ARGS);
    else if (vec) k_filter_compact<true, false><<<tiles, kBlock, 0, h->stream>>>(K2_ARGS);
    else if (ordered) k_filter_compact<false, true><<<tiles, kBlock, 0, h->stream>>>(K2_ARGS);
    else k_filter_compact<false, false><<<tiles, kBlock, 0, h->stream>>>(K2_ARGS);
#undef K2_ARGS
  }
  CU(cudaGetLastError());
  return GSCAN_OK;
}

// K1 + fused K2/K3 (pipeline path): extremes, then filter + keys + bucket
// ranks in one pass. Leaves survivors/keys/ranks and n1, hist filled.
int stage_round1_keys(gscan_handle* h, const double* xs, const double* ys, uint32_t n, int enable,
                      bool ext_ready = false) {
  const bool vec = aligned16(xs) && aligned16(ys);
  if (!ext_ready) {  // else h->ext already holds this input's extremes (declined sparse attempt)
    const uint32_t grid =
        std::max(1u, std::min<uint32_t>((n + kBlock * 8 - 1) / (kBlock * 8), h->sm_count * 8));
    Launch L(h, "k_extremes");
    if (vec) k_extremes<true><<<grid, kBlock, 0, h->stream>>>(xs, ys, n, h->partials, h->ext, h->ctr);
    else k_extremes<false><<<grid, kBlock, 0, h->stream>>>(xs, ys, n, h->partials, h->ext, h->ctr);
  }
  const uint32_t nb = buckets_for(n);
  const double scale = (double)nb / kPi;
  CU(cudaMemsetAsync(h->hist, 0, (nb + 1) * 4, h->stream));
  const uint64_t tiles = (n + kFusedTile - 1) / kFusedTile;
  {
    Launch L(h, "k_filter_keys");
#define KF_ARGS xs, ys, n, h->ext, enable, scale, nb, h->hist, h->surv, h->keys, h->rank, h->ctr
    if (vec) k_filter_keys<true><<<tiles, kBlock, 0, h->stream>>>(KF_ARGS);
    else k_filter_keys<false><<<tiles, kBlock, 0, h->stream>>>(KF_ARGS);
#undef KF_ARGS
  }
  CU(cudaGetLastError());
  return GSCAN_OK;
}

// K3 .. K4: keys, bucket offsets, scatter, per-bucket sort + dedup, anchor
// at position 0, split_regions. Leaves the annotated buffer in A_*.
int stage_annotate_sort(gscan_handle* h, const double* xs, const double* ys, uint32_t n,
                        int t_annot_ev, int t_sort_ev, bool keys_done = false) {
  const uint32_t nb = buckets_for(n);
  const double scale = (double)nb / kPi;
  if (!keys_done) CU(cudaMemsetAsync(h->hist, 0, (nb + 1) * 4, h->stream));
  if (!keys_done) {
    const uint32_t grid = std::max(1u, std::min<uint32_t>((n + kBlock - 1) / kBlock, h->sm_count * 16));
    Launch L(h, "k_keys");
    k_keys<<<grid, kBlock, 0, h->stream>>>(xs, ys, h->surv, h->ext, h->ctr, h->keys, h->rank,
                                           h->hist, scale, nb, h->ctr);
  }
  if (t_annot_ev >= 0) CU(cudaEventRecord(h->ev[t_annot_ev], h->stream));
  const uint64_t stiles = (nb + 1 + kScanTile - 1) / kScanTile;
  TRY(reset_lookback(h, stiles));
  {
    Launch L(h, "k_scan_u32");
    k_scan_u32<<<stiles, kBlock, 0, h->stream>>>(h->hist, nb, h->bstart, h->status, h->ctr);
  }
  {
    const uint32_t grid = std::max(1u, std::min<uint32_t>((n + kBlock - 1) / kBlock, h->sm_count * 16));
    Launch L(h, "k_scatter");
    k_scatter<<<grid, kBlock, 0, h->stream>>>(xs, ys, h->keys, h->rank, h->surv, h->ctr,
                                              h->bstart, scale, nb, h->rec);
  }
  const uint32_t tblocks = (nb + kBucketsPerBlock - 1) / kBucketsPerBlock;
  {
    const size_t smem = (size_t)kBlockCap * (8 + 8 + 8 + 8 + 4 + 2);
    Launch L(h, "k_bucket_sort_block");
    k_bucket_sort_block<<<tblocks, kBlock, smem, h->stream>>>(h->bstart, h->rec, h->ext, scale, nb,
                                                              h->A_x, h->A_y, h->A_i, h->best,
                                                              h->oversize, h->ctr);
  }
  {
    const size_t smem = (size_t)kSortCap * (8 + 8 + 4 + 4);
    Launch L(h, "k_bucket_sort_cta");
    k_bucket_sort_cta<<<kCtaSortGrid, kSortBlock, smem, h->stream>>>(
        h->bstart, h->rec, h->ext, h->oversize, h->ctr, h->A_x, h->A_y, h->A_i, h->best + tblocks,
        h->ctr);
  }
  {
    Launch L(h, "k_put_anchor");
    k_put_anchor<<<1, 1, 0, h->stream>>>(h->ext, h->bstart, nb, h->A_x, h->A_y, h->A_i, h->ctr);
  }
  {
    Launch L(h, "k_longest");
    k_longest<<<1, 1024, 0, h->stream>>>(h->best, tblocks + kCtaSortGrid, h->ctr);
  }
  CU(cudaGetLastError());
  TRY(sync_counters(h));
  if (h->h_ctr->dead) {
    // duplicates: compact the buffer, then split_regions over final positions
    const uint32_t m = h->h_ctr->m_total;
    const uint64_t tiles = (m + kCompactTile - 1) / kCompactTile;
    TRY(reset_lookback(h, tiles));
    {
      Launch L(h, "k_compact_dedup");
      k_compact_xyi<0><<<tiles, kBlock, 0, h->stream>>>(h->A_x, h->A_y, h->A_i, nullptr, nullptr,
                                                        m, h->C_x, h->C_y, h->C_i, h->status,
                                                        h->ctr, &h->ctr->m_total);
    }
    std::swap(h->A_x, h->C_x);
    std::swap(h->A_y, h->C_y);
    std::swap(h->A_i, h->C_i);
    TRY(sync_counters(h));
    const uint32_t m2 = h->h_ctr->m_total;
    CU(cudaMemsetAsync(h->scratch64, 0, 8, h->stream));
    CU(cudaMemsetAsync(h->scratch64 + 1, 0xff, 8, h->stream));
    const uint32_t grid = std::max(1u, std::min<uint32_t>((m2 + kBlock - 1) / kBlock, h->sm_count * 8));
    {
      Launch L(h, "k_longest_scan0");
      k_longest_scan<<<grid, kBlock, 0, h->stream>>>(h->A_x, h->A_y, m2, h->scratch64,
                                                     reinterpret_cast<uint32_t*>(h->scratch64 + 1), 0);
    }
    {
      Launch L(h, "k_longest_scan1");
      k_longest_scan<<<grid, kBlock, 0, h->stream>>>(h->A_x, h->A_y, m2, h->scratch64,
                                                     reinterpret_cast<uint32_t*>(h->scratch64 + 1), 1);
    }
    CU(cudaMemcpyAsync(&h->ctr->longest, h->scratch64 + 1, 4, cudaMemcpyDeviceToDevice, h->stream));
    TRY(sync_counters(h));
  }
  if (t_sort_ev >= 0) CU(cudaEventRecord(h->ev[t_sort_ev], h->stream));
  return GSCAN_OK;
}

// Round 2 over A_* (M entries). Result in R (pointers returned), n2 in ctr.
int stage_round2(gscan_handle* h, const gscan_config& cfg, double** Rx, double** Ry,
                 uint32_t** Ri) {
  const uint32_t m = h->h_ctr->m_total;
  if (!cfg.enable_round2 || m < 2) {
    *Rx = h->A_x; *Ry = h->A_y; *Ri = h->A_i;
    CU(cudaMemcpyAsync(&h->ctr->n2, &h->ctr->m_total, 4, cudaMemcpyDeviceToDevice, h->stream));
    return GSCAN_OK;
  }
  const uint32_t l = h->h_ctr->longest;
  if (l < 1 || l >= m) return fail(h, GSCAN_E_INTERNAL, "split index %u out of range (M=%u)", l, m);
  SliceGeom g{};
  g.l = l;
  g.m = m;
  g.chunked = cfg.chunked ? 1 : 0;
  const uint64_t c = cfg.chunk_count;
  const uint32_t m_right = l - 1, m_left = m - 1 - l;
  if (cfg.chunked) {
    if (m_right > 1) {
      g.step_r = (uint32_t)((m_right + c - 1) / c);
      g.n_right = (m_right + g.step_r - 1) / g.step_r;
    }
    if (m_left > 1) {
      g.step_l = (uint32_t)((m_left + c - 1) / c);
      g.n_left = (m_left + g.step_l - 1) / g.step_l;
    }
  } else {
    g.n_right = (l >= 2) ? 1 : 0;
    g.n_left = (l + 2 <= m - 1) ? 1 : 0;
  }
  CU(cudaMemsetAsync(h->flags, 1, m, h->stream));
  const uint32_t slices = g.n_right + g.n_left;
  if (slices) {
    Launch L(h, "k_round2_block");
    k_round2_block<<<slices, kWalkBlock, 0, h->stream>>>(h->A_x, h->A_y, g, h->flags);
  }
  const uint64_t tiles = (m + kCompactTile - 1) / kCompactTile;
  TRY(reset_lookback(h, tiles));
  {
    Launch L(h, "k_compact_round2");
    k_compact_xyi<1><<<tiles, kBlock, 0, h->stream>>>(h->A_x, h->A_y, h->A_i, h->flags, nullptr, m,
                                                      h->C_x, h->C_y, h->C_i, h->status, h->ctr,
                                                      &h->ctr->n2);
  }
  CU(cudaGetLastError());
  *Rx = h->C_x; *Ry = h->C_y; *Ri = h->C_i;
  return GSCAN_OK;
}


// Exclusive scan of n uint32 counts into out[0..n] (out[n] = total).
int scan_u32(gscan_handle* h, const uint32_t* in, uint32_t n, uint32_t* out) {
  const uint64_t tiles = (n + 1 + kScanTile - 1) / kScanTile;
  TRY(reset_lookback(h, tiles));
  Launch L(h, "k_scan_u32");
  k_scan_u32<<<tiles, kBlock, 0, h->stream>>>(in, n, out, h->status, h->ctr);
  return GSCAN_OK;
}

int read_u32(gscan_handle* h, const uint32_t* d, uint32_t* v) {
  CU(cudaMemcpyAsync(&h->h_ctr->pad[0], d, 4, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  *v = h->h_ctr->pad[0];
  return GSCAN_OK;
}

// K7/K8 (graham.cuh): candidate + certificate; exact sequential fallback.
// Leaves the hull (input indices) in h->d_out and its size in ctr->hull.
// Candidate strategies: junctions (convex-position inputs: chains don't
// shrink), prefix scan of explicit states (chains shrink: square/disk), and
// the warp sequential scan over the chains (prefix states too large).
constexpr uint64_t kPrefixBudget = 1ull << 26;  // entries per explicit-state buffer

int graham_seq_fallback(gscan_handle* h, const double* Rx, const double* Ry, const uint32_t* Ri) {
  h->graham_path |= 4;
  Launch L(h, "k_graham_seq");
  k_graham_seq<<<1, 32, 0, h->stream>>>(Rx, Ry, Ri, &h->ctr->n2, h->stack, h->d_out, h->ctr);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int graham_prefix(gscan_handle* h, const double* Rx, const double* Ry, const uint32_t* Ri,
                  uint32_t N, uint32_t nch, uint32_t q0, bool* done) {
  *done = false;
  const uint64_t cap = (uint64_t)q0 + 64;
  const uint64_t need = (uint64_t)nch * cap;
  const uint64_t need_scr = (uint64_t)nch * (cap + kChunk + 32);
  if (need > kPrefixBudget) return GSCAN_OK;
  if (need_scr > h->g_st_cap || need > h->g_st_cap || nch > h->g_len_cap) {
    dfree(h->g_stA); dfree(h->g_stB); dfree(h->g_lenA); dfree(h->g_lenB); dfree(h->g_scr);
    const uint64_t c2 = std::max(need_scr, need) * 5 / 4 + 1024;
    const uint64_t l2 = (uint64_t)nch * 5 / 4 + 64;
    CU(cudaMalloc(&h->g_stA, c2 * 4));
    CU(cudaMalloc(&h->g_stB, c2 * 4));
    CU(cudaMalloc(&h->g_scr, c2 * 4));
    CU(cudaMalloc(&h->g_lenA, l2 * 4));
    CU(cudaMalloc(&h->g_lenB, l2 * 4));
    h->g_st_cap = c2;
    h->g_len_cap = l2;
  }
  uint32_t* ovf = h->g_misc + 2;
  uint32_t* which = h->g_misc + 3;
  CU(cudaMemsetAsync(ovf, 0, 8, h->stream));
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_graham_prefix, kPrefixWarps * 32, 0));
  const uint32_t want = (nch + kPrefixWarps - 1) / kPrefixWarps;
  const uint32_t grid = std::max(1u, std::min<uint32_t>(want, (uint32_t)(per_sm * h->sm_count)));
  uint32_t capu = (uint32_t)cap;
  void* args[] = {(void*)&Rx, (void*)&Ry, (void*)&h->g_chain, (void*)&h->g_len, (void*)&nch,
                  (void*)&h->g_stA, (void*)&h->g_stB, (void*)&h->g_lenA, (void*)&h->g_lenB,
                  (void*)&capu, (void*)&ovf, (void*)&which};
  {
    Launch L(h, "k_graham_prefix");
    CU(cudaLaunchCooperativeKernel((void*)k_graham_prefix, grid, kPrefixWarps * 32, args, 0,
                                   h->stream));
  }
  uint32_t fl[2];
  CU(cudaMemcpyAsync(fl, ovf, 8, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  if (fl[0]) return GSCAN_OK;  // overflow (cannot happen with cap = q0 + 64; kept as a guard)
  const uint32_t* st = fl[1] ? h->g_stB : h->g_stA;
  const uint32_t* len = fl[1] ? h->g_lenB : h->g_lenA;
  uint32_t* fail_d = h->g_misc;
  CU(cudaMemsetAsync(fail_d, 0, 4, h->stream));
  if (h->debug & GSCAN_DEBUG_CORRUPT_CANDIDATE) {
    // falsify the final state (empty it): the certificate must reject it
    CU(cudaMemsetAsync((void*)(len + nch - 1), 0, 4, h->stream));
  }
  {
    Launch L(h, "k_graham_certify_explicit");
    k_graham_certify_explicit<<<(nch + kCertWarps - 1) / kCertWarps, kCertWarps * 32, 0,
                                h->stream>>>(Rx, Ry, N, st, len, capu, h->g_scr, fail_d);
  }
  uint32_t fails;
  TRY(read_u32(h, fail_d, &fails));
  h->graham_fails = fails;
  h->graham_path = 3;
  if (fails || (h->debug & GSCAN_DEBUG_FORCE_FALLBACK)) return GSCAN_OK;
  {
    Launch L(h, "k_graham_emit_explicit");
    k_graham_emit_explicit<<<std::max(1u, std::min<uint32_t>((q0 + kBlock - 1) / kBlock, 1184)),
                             kBlock, 0, h->stream>>>(st, len, nch - 1, capu, Ri, h->d_out, h->ctr);
  }
  CU(cudaGetLastError());
  *done = true;
  return GSCAN_OK;
}

// Tree strategy (graham_tree.cuh) for pop-heavy buffers. Split in three so the
// sparse path can enqueue it inside its CUDA graph before the buffer size is
// known on the host: tree_workspace (allocation for up to n_max points),
// tree_enqueue (every kernel reads N from the device), tree_finish (after the
// stream synchronised: *done = false when the tree declined -- convex
// position, or N beyond the workspace -- and the caller then takes the
// junction / prefix / sequential strategies).
constexpr uint32_t kTreeMaxN = 1u << 22;  // larger buffers: the middle level would be too long

int tree_workspace(gscan_handle* h, uint32_t n_max) {
  if (h->tw_pool && h->tw_nmax >= n_max) return GSCAN_OK;
  const uint32_t N = std::max<uint32_t>(n_max, 1024);
  // level capacities: level 1 <= 0.85 N, then <= 0.9x per level, levels >= 1
  // at most kTreeHiCap (else the kernel declines)
  uint64_t caps[kTreeMaxLevels + 1];
  caps[0] = N;
  for (int j = 1; j <= kTreeMaxLevels; ++j)
    caps[j] = std::min<uint64_t>((j == 1 ? (uint64_t)N * 17 / 20 : caps[j - 1] * 9 / 10) + 64,
                                 kTreeHiCap);
  auto nchunks = [&](int j) { return caps[j] / tree_cs(j) + 2; };
  uint64_t need = 8ull * N + kTreeTopMax + 64 * 8;  // parent, tmp, chainq/p, chainx/y, fstack
  for (int j = 0; j <= kTreeMaxLevels; ++j) {
    if (j >= 1) need += 6 * caps[j] + 4 * 32;                // Qp, Qx, Qy, up
    need += nchunks(j) * (2 + 2 + 8 + 16 + 16) + 7 * 32;   // off, bt, rec
  }
  dfree(h->tw_pool);
  CU(cudaMalloc(&h->tw_pool, need * 4));
  uint32_t* pool = h->tw_pool;
  uint64_t used = 0;
  auto take = [&](uint64_t cnt) { uint32_t* p = pool + used; used += (cnt + 31) & ~31ull; return p; };
  auto take_d = [&](uint64_t cnt) { return reinterpret_cast<double*>(take(2 * cnt)); };
  TreeWork& w = h->tw;
  w = TreeWork{};
  w.parent = take(N);
  w.tmp = take(N);
  w.chainq = take(N);
  w.chainp = take(N);
  w.chainx = take_d(N);
  w.chainy = take_d(N);
  w.fstack = take(kTreeTopMax);
  for (int j = 0; j <= kTreeMaxLevels; ++j) {
    w.cap[j] = (uint32_t)caps[j];
    if (j >= 1) {
      w.Qp[j] = take(caps[j]);
      w.Qx[j] = take_d(caps[j]);
      w.Qy[j] = take_d(caps[j]);
      w.up[j] = take(caps[j]);
    }
    const uint64_t nc = nchunks(j);
    w.off[j] = take(nc);
    w.bt[j] = take(nc);
    w.rec[j].n = take(nc);
    w.rec[j].below = take(nc);
    w.rec[j].pos = take(nc * kTreePC);
    w.rec[j].x = take_d(nc * kTreePC);
    w.rec[j].y = take_d(nc * kTreePC);
  }
  if (used > need) return fail(h, GSCAN_E_INTERNAL, "tree pool overflow");
  h->tw_nmax = N;
  h->tw_nch1 = (uint32_t)(caps[1] / tree_cs(1) + 1);
  return GSCAN_OK;
}

// Enqueue the whole tree strategy on s. N = *n_dev (the sparse path's round-2
// size) or n_host; the kernels no-op when *st_fail is set or when disabled.
// The info words are copied to the pinned h->h_info at the end.
uint32_t side_free_sms();
int tree_enqueue(gscan_handle* h, const double* Rx, const double* Ry, const uint32_t* Ri,
                 const uint32_t* n_dev, uint32_t n_host, const uint32_t* st_fail, bool disable,
                 cudaStream_t s) {
  const TreeWork& w = h->tw;
  uint32_t* info = h->g_misc + 4;
  const uint32_t nch0 = (h->tw_nmax + kTreeChunk0 - 1) / kTreeChunk0;  // upper bounds
  // the grids loop grid-stride over chunks: one wave on the SMs the side
  // stream leaves free (CTAs sized by the workspace bound would mostly find
  // no chunk, in waves, each exit behind a read of info[])
  const uint32_t gmax = 4 * std::max(side_free_sms(), 16u);
  const uint32_t g0 = std::min((nch0 + kTreeCta - 1) / kTreeCta, gmax);
  const uint32_t g1 = std::min((h->tw_nch1 + kTreeCta - 1) / kTreeCta, gmax);
  const uint32_t dbg = (h->debug & GSCAN_DEBUG_CORRUPT_CANDIDATE) ? 1u : 0u;
  { Launch Lk(h, "k_gr_setup", s); launch_pdl(k_gr_setup, 1, 64, 0, s, n_dev, n_host, st_fail, h->tw_nmax, disable ? 1u : 0u, info); }
  for (int j = 0; j < 2; ++j) {  // levels 0 and 1 on many CTAs
    const uint32_t g = j ? g1 : g0, nch = j ? h->tw_nch1 : nch0;
    { Launch Lk(h, "k_gr_up", s); launch_pdl(k_gr_up, g, kTreeCta, kTreeCtaSmem, s, j, Rx, Ry, w, info); }
    { Launch Lk(h, "k_gr_scan", s); launch_pdl(k_gr_scan, 1, 1024, 0, s, j, w, info); }
    { Launch Lk(h, "k_gr_gather", s); launch_pdl(k_gr_gather, std::min((nch + 7) / 8, gmax), 256, 0, s, j, w, info); }
  }
  { Launch Lk(h, "k_gr_mid", s); launch_pdl(k_gr_mid, 1, kTreeThreads, kTreeSmem, s, Rx, Ry, w, info); }
  { Launch Lk(h, "k_gr_down", s); launch_pdl(k_gr_down, g1, kTreeCta, kTreeCtaSmem, s, 2, Rx, Ry, w, info); }
  { Launch Lk(h, "k_gr_down", s); launch_pdl(k_gr_down, g0, kTreeCta, kTreeCtaSmem, s, 1, Rx, Ry, w, info); }
  { Launch Lk(h, "k_gr_cert", s); launch_pdl(k_gr_cert, g0, kTreeCta, kTreeCtaSmem, s, Rx, Ry, w, info, dbg); }
  { Launch Lk(h, "k_gr_emit", s); launch_pdl(k_gr_emit, 1, 1024, 0, s, Rx, Ry, Ri, w, info, h->d_out, h->ctr); }
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(h->h_info, info, kTreeInfoWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  return GSCAN_OK;
}

// After the stream synchronised (h->h_info current).
int tree_finish(gscan_handle* h, const double* Rx, const double* Ry, const uint32_t* Ri,
                bool* done) {
  *done = false;
  const uint32_t* hi = h->h_info;
  if (h->sp_debug) {
    fprintf(stderr, "[tree] N=%u K=%u declined=%u sizes=%u,%u,%u,%u,%u,%u.. cycles: up=%u top=%u down=%u fails=%u\n",
            hi[4], hi[3], hi[0], hi[4], hi[11], hi[12], hi[13], hi[14], hi[15], hi[8],
            hi[9] - hi[8], hi[16] - hi[9], hi[2]);
    fprintf(stderr, "[tree] level ends (cycles): up");
    for (uint32_t j = 2; j < hi[3] && j < 12; ++j) fprintf(stderr, " %u", hi[20 + j]);
    fprintf(stderr, " | down");
    for (uint32_t j = hi[3] - 1; j >= 3 && j < 12; --j) fprintf(stderr, " %u", hi[32 + j]);
    fprintf(stderr, "\n");
  }
  if (hi[0]) return GSCAN_OK;  // declined
  h->graham_fails = hi[2];
  h->graham_path = 8 | (hi[2] ? 4 : 0);
  if (!hi[2] && (h->debug & GSCAN_DEBUG_FORCE_FALLBACK)) TRY(graham_seq_fallback(h, Rx, Ry, Ri));
  *done = true;
  return GSCAN_OK;
}

bool tree_forced_off(const gscan_handle* h) {
  return h->debug & (GSCAN_DEBUG_FORCE_JUNCTION | GSCAN_DEBUG_FORCE_SEQUENTIAL |
                     GSCAN_DEBUG_FORCE_PREFIX);
}

int stage_graham(gscan_handle* h, const double* Rx, const double* Ry, const uint32_t* Ri,
                 uint32_t N, bool skip_tree = false) {
  uint32_t* fail_d = h->g_misc;
  uint32_t* len_d = h->g_misc + 1;
  CU(cudaMemsetAsync(h->g_misc, 0, 16, h->stream));
  h->graham_path = 0;
  h->graham_fails = 0;
  if (N <= 2 * kChunk) {  // tiny buffer: the sequential kernel is the fastest exact path
    TRY(graham_seq_fallback(h, Rx, Ry, Ri));
    h->graham_path = 0;
    return GSCAN_OK;
  }
  if (!skip_tree && !tree_forced_off(h) && N <= kTreeMaxN) {
    bool done = false;
    TRY(tree_workspace(h, N));
    TRY(tree_enqueue(h, Rx, Ry, Ri, nullptr, N, nullptr, false, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    TRY(tree_finish(h, Rx, Ry, Ri, &done));
    if (done) return GSCAN_OK;
  }
  const uint32_t nch = (N + kChunk - 1) / kChunk;
  {
    Launch L(h, "k_graham_local");
    k_graham_local<<<(nch + kLocalWarps - 1) / kLocalWarps, kLocalWarps * 32, 0, h->stream>>>(
        Rx, Ry, N, h->g_chain, h->g_len);
  }
  TRY(scan_u32(h, h->g_len, nch, h->g_off));
  uint32_t q0;
  TRY(read_u32(h, h->g_off + nch, &q0));
  const bool force_j = h->debug & GSCAN_DEBUG_FORCE_JUNCTION;
  const bool force_s = h->debug & GSCAN_DEBUG_FORCE_SEQUENTIAL;
  const bool force_p = h->debug & GSCAN_DEBUG_FORCE_PREFIX;
  bool junction_ok = false;
  if (force_j || (!force_s && !force_p && q0 > N / 2)) {
    {
      Launch L(h, "k_graham_junction");
      k_graham_junction<<<(nch + 127) / 128, 128, 0, h->stream>>>(Rx, Ry, h->g_chain, h->g_len,
                                                                   nch, h->g_jk, h->g_je, h->g_jmin);
    }
    {
      Launch L(h, "k_graham_junction_apply");
      k_graham_junction_apply<<<(nch + 1 + 7) / 8, 256, 0, h->stream>>>(
          h->g_chain, h->g_len, nch, h->g_jk, h->g_je, h->g_jmin, h->g_parent, h->g_btop,
          h->g_keep, fail_d);
    }
    uint32_t jfail;
    TRY(read_u32(h, fail_d, &jfail));
    junction_ok = (jfail == 0) || force_j;
  }
  if (!junction_ok && !force_s) {
    bool done = false;
    TRY(graham_prefix(h, Rx, Ry, Ri, N, nch, q0, &done));
    if (done) return GSCAN_OK;
    if (h->graham_path == 3) return graham_seq_fallback(h, Rx, Ry, Ri);  // certificate failed
  }
  CU(cudaMemsetAsync(fail_d, 0, 4, h->stream));
  if (junction_ok) {
    h->graham_path = 2;
    TRY(scan_u32(h, h->g_keep, nch, h->g_off));
    {
      Launch L(h, "k_graham_junction_emit");
      k_graham_junction_emit<<<(nch + 7) / 8, 256, 0, h->stream>>>(
          h->g_chain, h->g_je, h->g_keep, h->g_off, nch, h->stack);
    }
    CU(cudaMemcpyAsync(len_d, h->g_off + nch, 4, cudaMemcpyDeviceToDevice, h->stream));
  } else {
    h->graham_path = 1;
    {
      Launch L(h, "k_gather_chains");
      k_gather_chains<<<(nch + 7) / 8, 8 * kChunk, 0, h->stream>>>(h->g_chain, h->g_len,
                                                                   h->g_off, nch, h->g_q0);
    }
    {
      Launch L(h, "k_graham_candidate_seq");
      k_graham_candidate_seq<<<1, 32, kCandSmem, h->stream>>>(Rx, Ry, h->g_q0, h->g_off + nch, N,
                                                              h->g_parent, h->g_btop, h->stack,
                                                              len_d);
    }
    uint32_t clen;
    TRY(read_u32(h, len_d, &clen));
    if (clen == kNone) return graham_seq_fallback(h, Rx, Ry, Ri);
  }
  if (h->debug & GSCAN_DEBUG_CORRUPT_CANDIDATE) {
    // drop the candidate's last boundary state: the certificate must reject it
    CU(cudaMemcpyAsync(h->g_btop + nch, h->g_btop + nch - 1, 4, cudaMemcpyDeviceToDevice,
                       h->stream));
  }
  {
    Launch L(h, "k_graham_certify");
    k_graham_certify<<<(nch + kCertWarps - 1) / kCertWarps, kCertWarps * 32, 0, h->stream>>>(
        Rx, Ry, N, h->g_parent, h->g_btop, fail_d);
  }
  uint32_t fails;
  TRY(read_u32(h, fail_d, &fails));
  h->graham_fails = fails;
  if (fails == 0 && !(h->debug & GSCAN_DEBUG_FORCE_FALLBACK)) {
    Launch L(h, "k_graham_emit");
    k_graham_emit<<<std::max(1u, std::min<uint32_t>((N + kBlock - 1) / kBlock, 1184)), kBlock, 0,
                    h->stream>>>(h->stack, len_d, Ri, h->d_out, h->ctr);
    CU(cudaGetLastError());
    return GSCAN_OK;
  }
  return graham_seq_fallback(h, Rx, Ry, Ri);
}

int validate(gscan_handle* h, uint64_t n, const gscan_config& cfg) {
  if (!h) return GSCAN_E_INVALID;
  if (n == 0) return fail(h, GSCAN_E_EMPTY_INPUT, "full_pipeline: no points");
  if (cfg.chunk_count == 0) return fail(h, GSCAN_E_ZERO_CHUNKS, "full_pipeline: chunk_count must be positive");
  if (n >= 0xffffffffull) return fail(h, GSCAN_E_TOO_LARGE, "n = %llu exceeds 2^32-2", (unsigned long long)n);
  return GSCAN_OK;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// ---------------------------------------------------------------------------
// Sparse round-2 path (sparse.cuh). Returns GSCAN_OK with *ok = false when the
// path declined (fail bits in h->sp_fail): the caller then runs the full sort.

bool sparse_eligible(const gscan_handle* h, uint64_t n, const gscan_config& cfg) {
  return n >= kSparseMinN && cfg.enable_round1 && cfg.enable_round2 && cfg.chunked &&
         !(h->debug & GSCAN_DEBUG_FULL_SORT);
}

double __longlong_as_double_host(uint64_t u) {
  double d;
  memcpy(&d, &u, 8);
  return d;
}
float unord_host(uint32_t u) {
  if (u == 0 || u == 0xffffffffu) return 0.f;
  const uint32_t b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

int sparse_init(gscan_handle* h) {
  if (h->sp_st) return GSCAN_OK;
  const uint32_t nb = kSpBuckets, G = (uint32_t)h->sp_grid;
  CU(cudaMalloc(&h->sp_th, (nb + 1) * 8));
  CU(cudaMalloc(&h->sp_cdf, (kSpCells + 1) * 8));
  CU(cudaMalloc(&h->sp_cells, kSpCells * 4));
  CU(cudaMalloc(&h->sp_big, nb * 4));
  CU(cudaMalloc(&h->sp_bigg, nb * 4));
  CU(cudaMalloc(&h->sp_hugeg, nb * 4));
  CU(cudaMalloc(&h->sp_gcount, G * 4));
  CU(cudaMalloc(&h->sp_side_status, ((kSpParts * 2 * G + 1 + kScanTile - 1) / kScanTile + 64) * 8));
  CU(cudaMalloc(&h->sp_side_ticket, sizeof(Counters)));
  CU(cudaMalloc(&h->sp_side_work, 4 * sizeof(uint32_t)));
  CU(cudaMalloc(&h->sp_ccount, G * 4));
  CU(cudaMalloc(&h->sp_hcount, 2 * G * 4));  // two hash lists per F3 CTA
  h->sp_debug = env_flag("GSCAN_SP_DEBUG");
  // measurement hook only: skipping the duplicate check is exact only for
  // duplicate-free inputs
  h->sp_no_dup = env_flag("GSCAN_SP_NODUP");
  CU(cudaMalloc(&h->sp_hist_part, (size_t)G * nb * 4));
  CU(cudaMalloc(&h->sp_phi_part, (size_t)G * nb * 4));
  CU(cudaMalloc(&h->sp_part_off, ((size_t)2 * G * kSpParts + 1) * 4));
  CU(cudaMalloc(&h->sp_d2, 2 * G * sizeof(SpD2)));
  uint32_t** nb_bufs[] = {&h->sp_hist, &h->sp_bstart, &h->sp_glist, &h->sp_gcnt, &h->sp_phimax,
                          &h->sp_prefmax, &h->sp_slice, &h->sp_ccnt, &h->sp_cstart, &h->sp_wcnt,
                          &h->sp_wstart, &h->sp_rlo};
  for (uint32_t** b : nb_bufs) CU(cudaMalloc(b, (nb + 2) * 4));
  CU(cudaMalloc(&h->sp_thr, (size_t)nb * 4));
  CU(cudaMalloc(&h->sp_gs, (nb + 2) * 4));
  CU(cudaMalloc(&h->sp_gsz, (nb + 2) * 4));
  CU(cudaMalloc(&h->sp_gbits, nb / 8));
  CU(cudaMalloc(&h->sp_st, sizeof(SpState)));
  CU(cudaMallocHost(&h->h_sp, sizeof(SpState)));
  return GSCAN_OK;
}

// Event record usable inside stream capture (as an external event node, so
// elapsed times still work after graph launches) and outside of it.
// Stage boundary k (0..5) of the sparse path: inside a captured graph a
// one-thread kernel stores %globaltimer into the counters (read back with
// them), since six cudaEventElapsedTime calls cost ~17 us of host time per
// call; outside a capture (profiling, no graphs) an event.
__global__ void k_tstamp(Counters* __restrict__ ctr, int k) { pdl_wait(); ctr->tstamp[k] = globaltimer_ns(); }
int stage_mark(gscan_handle* h, int k, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(s, &cs));
  if (cs == cudaStreamCaptureStatusActive) launch_pdl(k_tstamp, 1, 1, 0, s, h->ctr, k);
  else CU(cudaEventRecord(h->ev[k], s));
  return GSCAN_OK;
}

int rec_event(gscan_handle* h, cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(s, &cs));
  if (cs == cudaStreamCaptureStatusActive) CU(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));
  else CU(cudaEventRecord(e, s));
  return GSCAN_OK;
}

// The sparse path as segments over one context. sparse_enqueue runs them all
// in order (one device, one CUDA graph); the sharded path (gscan_dist_*) runs
// them per rank with the collectives of SURVEY.md 8e in between.
// F2 without its shared-memory histogram (two CTAs per SM) + a histogram
// pass over the codes
constexpr bool kF2Split = true;
#ifndef GSCAN_F2_RING
#define GSCAN_F2_RING 1
#endif
constexpr bool kF2Ring = GSCAN_F2_RING;  // F2 as a bulk-copy pipeline (k_sp_hist_ring)
constexpr uint32_t kF2PatchGrid = 64;    // CTAs (and P_l partials) of k_sp_f2_patch
// F3 without its shared-memory bucket maxima (1024 threads) + a maxima pass:
// measured slower (F3 192 us either way, + 46 us for k_sp_phimax_codes)
constexpr bool kF3Split = false;

struct SpCtx {
  const double* xs;
  const double* ys;
  uint32_t n;       // points of this device
  uint32_t base;    // global index of point 0 (a shard's offset; 0 on one device)
  uint64_t chunks;  // cfg.chunk_count
  uint64_t nslices;
  uint32_t G, cap, nb;
  size_t smem_nb;
  bool vec, drop;
  const uint32_t* gs;  // storage base of gathered buckets (bstart on one device)
  cudaStream_t s;
  bool sharded;        // a rank of the sharded path (decisions are global there)
};

SpCtx sp_ctx(gscan_handle* h, const double* xs, const double* ys, uint32_t n, uint64_t chunks) {
  SpCtx c{};
  c.xs = xs;
  c.ys = ys;
  c.n = n;
  c.base = 0;
  c.chunks = chunks;
  c.nslices = 2 * std::min<uint64_t>(chunks, n);
  c.G = (uint32_t)h->sp_grid;
  c.cap = sparse_region_cap(h, n);  // per-CTA emission region: bound on the points one CTA visits
  c.nb = kSpBuckets;
  c.smem_nb = (size_t)kSpBuckets * 4;
  c.vec = aligned16(xs) && aligned16(ys);
  c.drop = (h->debug & GSCAN_DEBUG_SPARSE_DROP) != 0;
  c.gs = h->sp_gs;  // compact storage of the gathered buckets (sp_seg_f3 / gscan_dist_slices)
  c.s = h->stream;
  c.sharded = false;
  return c;
}

// The call's cleared state in one kernel (one graph node instead of nine
// memset nodes): segments of 32-bit words set to a value.
struct InitSegs {
  uint32_t* p[9];
  uint64_t words[9];
  uint32_t val[9];
};
__global__ void __launch_bounds__(256) k_sp_init(InitSegs g) {
  pdl_wait();
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nth = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll 1
  for (int k = 0; k < 9; ++k) {
    uint32_t* p = g.p[k];
    const uint64_t n = g.words[k];
    const uint32_t v = g.val[k];
    // 16-byte stores where aligned (every segment starts 16-byte aligned)
    uint4* p4 = reinterpret_cast<uint4*>(p);
    const uint64_t n4 = n / 4;
    for (uint64_t i = tid; i < n4; i += nth) p4[i] = make_uint4(v, v, v, v);
    for (uint64_t i = n4 * 4 + tid; i < n; i += nth) p[i] = v;
  }
}

int sp_seg_init(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  static_assert(sizeof(Counters) % 16 == 0 && sizeof(SpState) % 4 == 0, "init segments");
  InitSegs g{};
  int k = 0;
  auto seg = [&](void* p, uint64_t bytes, uint32_t v) {
    g.p[k] = static_cast<uint32_t*>(p);
    g.words[k] = bytes / 4;
    g.val[k] = v;
    ++k;
  };
  seg(h->ctr, sizeof(Counters), 0u);
  seg(h->sp_st, sizeof(SpState), 0u);
  seg(h->sp_gcnt, c.nb * 4ull, 0u);
  seg(h->sp_ccnt, c.nb * 4ull, 0u);
  seg(h->sp_prefmax, c.nb * 4ull, 0u);
  seg(h->sp_slice, c.nb * 4ull, 0xffffffffu);
  seg(h->sp_cells, kSpCells * 4ull, 0u);
  seg(h->lb_status, (uint64_t)kLbSlots * h->lb_stride * 8, 0u);
  seg(h->lb_ctr, (uint64_t)kLbSlots * sizeof(Counters), 0u);
  {
    Launch L(h, "k_sp_init", s);
    launch_pdl(k_sp_init, 2 * h->sm_count, 256, 0, s, g);
  }
  TRY(stage_mark(h, 0, s));
  return GSCAN_OK;
}

int sp_seg_extremes(gscan_handle* h, const SpCtx& c) {
  if (c.vec && c.n >= (uint32_t)kExtTile) {  // bulk-copy pipeline, one CTA per SM
    Launch L(h, "k_extremes_tma", c.s);
    launch_pdl(k_extremes_tma, h->sm_count, kExtThreads, kExtSmem, c.s, c.xs, c.ys, c.n, h->partials, h->ext,
                                                           h->ctr);
    return GSCAN_OK;
  }
  const uint32_t grid =
      std::max(1u, std::min<uint32_t>((c.n + kBlock * 8 - 1) / (kBlock * 8), h->sm_count * 8));
  Launch L(h, "k_extremes", c.s);
  if (c.vec) launch_pdl(k_extremes<true>, grid, kBlock, 0, c.s, c.xs, c.ys, c.n, h->partials, h->ext, h->ctr);
  else launch_pdl(k_extremes<false>, grid, kBlock, 0, c.s, c.xs, c.ys, c.n, h->partials, h->ext, h->ctr);
  return GSCAN_OK;
}

int sp_seg_sample(gscan_handle* h, const SpCtx& c) {
  Launch L(h, "k_sp_sample", c.s);
  launch_pdl(k_sp_sample, kSpSample / 1024, 1024, 0, c.s, c.xs, c.ys, c.n, h->ext, h->sp_cells);
  return GSCAN_OK;
}

// bucket map from the sample cells, then F2 and P_l from the per-CTA partials
int sp_seg_f2(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  {
    Launch L(h, "k_sp_cdf", s);
    launch_pdl(k_sp_cdf, 1, kSpCells / 2, 0, s, h->sp_cells, h->sp_cdf, c.base == 0 && !c.sharded ? c.n : 0u,
                                        h->sp_st);
  }
  {
    Launch L(h, "k_sp_theta", s);
    launch_pdl(k_sp_theta, (c.nb + 1 + 255) / 256, 256, 0, s, h->sp_cdf, h->sp_th, h->sp_st);
  }
  const bool ring = kF2Ring && c.vec;
  const uint32_t g2 = ring ? c.G : (kF2Split ? 2 * c.G : c.G);  // F2 CTAs (d2 partials)
  if (ring) {
    Launch L(h, "k_sp_hist", s);
    launch_pdl(k_sp_hist_ring, g2, kF2Cons, kF2RingSmem, s, c.xs, c.ys, c.n, h->ext, h->sp_cdf, h->sp_th,
                                                         h->sp_codes, h->sp_d2, h->ctr, h->sp_st,
                                                         h->sp_exc, h->sp_exc_cap);
  } else {
    Launch L(h, "k_sp_hist", s);
#define A2 c.xs, c.ys, c.n, h->ext, h->sp_cdf, h->sp_th, h->sp_codes, h->sp_hist_part, h->sp_d2, h->ctr, \
           h->sp_st
    if (kF2Split) {
      if (c.vec) launch_pdl(k_sp_hist<true, false>, g2, kSpThreads, 0, s, A2);
      else launch_pdl(k_sp_hist<false, false>, g2, kSpThreads, 0, s, A2);
    } else {
      if (c.vec) launch_pdl(k_sp_hist<true, true>, g2, kSpThreads, c.smem_nb, s, A2);
      else launch_pdl(k_sp_hist<false, true>, g2, kSpThreads, c.smem_nb, s, A2);
    }
#undef A2
  }
  uint32_t nparts = g2;  // P_l partials
  if (ring) {  // the screen's uncertain points, exactly
    Launch L(h, "k_sp_f2_patch", s);
    launch_pdl(k_sp_f2_patch, kF2PatchGrid, 256, 0, s, c.xs, c.ys, h->ext, h->sp_cdf, h->sp_th, h->sp_codes,
                                              h->sp_exc, h->sp_exc_cap, h->sp_d2 + g2, h->ctr,
                                              h->sp_st);
    nparts += kF2PatchGrid;
  }
  if (kF2Split || ring) {
    Launch L(h, "k_sp_hist_codes", s);
    launch_pdl(k_sp_hist_codes, c.G, 1024, c.smem_nb, s, h->sp_codes, c.n, h->sp_hist_part, h->sp_st);
  }
  {
    Launch L(h, "k_sp_reduce_hist", s);
    launch_pdl(k_sp_reduce_cols<false>, (c.nb + 255) / 256, 256, 0, s, h->sp_hist_part, c.G, c.nb, h->sp_hist);
  }
  {
    Launch L(h, "k_sp_plan_pl", s);
    launch_pdl(k_sp_plan_pl, 1, 256, 0, s, c.xs, c.ys, h->sp_d2, nparts, h->sp_st, h->ctr, c.n);
  }
  return GSCAN_OK;
}

// bucket starts (exact ranks), P_l's bucket and its rank inside it
int sp_seg_plan(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  TRY(scan_u32_slot(h, h->sp_hist, c.nb, h->sp_bstart, kLbBstart, s));
  {
    Launch L(h, "k_sp_plan_bl", s);
    launch_pdl(k_sp_plan_bl, 1, 32, 0, s, h->ext, h->sp_cdf, h->sp_th, h->sp_bstart, h->sp_st);
  }
  {
    Launch L(h, "k_sp_lrank", s);
    launch_pdl(k_sp_lrank, h->sm_count * 8, 256, 0, s, c.xs, c.ys, h->sp_codes, c.n, c.base, h->ext,
                                               h->sp_st);
  }
  return GSCAN_OK;
}

// slice geometry, gathered buckets, then F3 (G in (surv, sp_eb), hash lists in sp_dup)
int sp_seg_f3(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  {
    Launch L(h, "k_sp_gbits", s);
    launch_pdl(k_sp_gbits, c.nb / 256, 256, 0, s, h->sp_bstart, c.chunks, h->sp_st, h->sp_gbits,
                                          h->sp_glist);
  }
  if (!c.sharded) {
    // gathered buckets stored compactly (gs[b]): their records and sorted
    // points stay L2-resident instead of being scattered over the global
    // position range (rank 0 of the sharded path does this in dist_slices)
    Launch L(h, "k_sp_gsize", s);
    launch_pdl(k_sp_gsize, (c.nb + 255) / 256, 256, 0, s, h->sp_gbits, h->sp_hist, h->sp_gsz);
  }
  if (!c.sharded) TRY(scan_u32_slot(h, h->sp_gsz, c.nb, h->sp_gs, kLbGs, s));
  TRY(stage_mark(h, 1, s));
  {
    Launch L(h, "k_sp_phi", s);
    const uint32_t t3 = kF3Split ? 1024u : (uint32_t)kSpF3Threads;
    const size_t sm3 = kF3Split ? 0 : c.smem_nb;
#define A3 c.xs, c.ys, h->sp_codes, c.n, c.cap, h->ext, h->sp_gbits, h->sp_st, h->sp_phi_part, h->surv, \
           h->sp_eb, h->sp_gcount, h->sp_gx, h->sp_gy, h->sp_dup, h->sp_hcount, h->sp_part_off, \
           h->sp_phi32, c.sharded ? 0u : 3u
    if (kF3Split) {
      if (c.vec) launch_pdl(k_sp_phi<true, false>, c.G, t3, sm3, s, A3);
      else launch_pdl(k_sp_phi<false, false>, c.G, t3, sm3, s, A3);
    } else {
      if (c.vec) launch_pdl(k_sp_phi<true, true>, c.G, t3, sm3, s, A3);
      else launch_pdl(k_sp_phi<false, true>, c.G, t3, sm3, s, A3);
    }
#undef A3
  }
  if (kF3Split) {
    Launch L(h, "k_sp_phimax_codes", s);
    launch_pdl(k_sp_phimax_codes, c.G, 1024, c.smem_nb, s, h->sp_codes, h->sp_phi32, h->sp_gbits, c.n,
                                                   h->sp_st, h->sp_phi_part);
  }
  {
    Launch L(h, "k_sp_reduce_phi", s);
    launch_pdl(k_sp_reduce_cols<true>, (c.nb + 255) / 256, 256, 0, s, h->sp_phi_part, c.G, c.nb, h->sp_phimax);
  }
  if (!c.sharded) TRY(rec_event(h, h->ev_part, s));  // the side stream's count scan forks here
  return GSCAN_OK;
}

// gathered points (regions (surv, sp_eb, sp_gcount) indexing gx/gy) sorted
// exactly; slice heads and the per-bucket prefix maxima
int sp_seg_sortg(gscan_handle* h, const SpCtx& c, const double* gx, const double* gy,
                 bool region_xy = true) {
  cudaStream_t s = c.s;
  {
    Launch L(h, "k_sp_place_g", s);
    launch_pdl(k_sp_emit_place<0>, dim3(16, c.G), 256, 0, s, gx, gy, h->surv, h->sp_eb, nullptr,
                                                     h->sp_gcount, c.cap, h->sp_gcnt, c.gs,
                                                     h->ext, h->sp_st, h->rec,
                                                     region_xy ? h->sp_gx : nullptr,
                                                     region_xy ? h->sp_gy : nullptr,
                                                     (uint32_t)std::min<uint64_t>(h->wcap, 0xffffffffu));
  }
  {
    Launch L(h, "k_sp_sort_gathered", s);
    launch_pdl(k_sp_sort_gathered, h->sm_count * (kSpSmallCap <= 512 ? 8 : 4), kSpSmallThreads, kSpSmallSmem, s, 
        h->sp_glist, h->sp_bstart, c.gs, h->sp_hist, h->sp_gcnt, h->rec, h->ext, h->sp_st,
        h->sp_bigg, h->A_x, h->A_y, h->A_i);
  }
  {
    Launch L(h, "k_sp_sort_gathered_big", s);
    launch_pdl(k_sp_sort_gathered_big, h->sm_count, kSpSortThreads, kSpBigSmem, s, 
        h->sp_bigg, h->sp_bstart, c.gs, h->sp_hist, h->rec, h->ext, h->sp_st, h->A_x, h->A_y,
        h->A_i, h->sp_hugeg, h->sp_huge_cap);
  }
  if (h->sp_huge_cap) {  // inputs large enough for buckets above kSpGatherCap
    Launch L(h, "k_sp_sort_gathered_huge", s);
    launch_pdl(k_sp_sort_gathered_huge, h->sm_count, kSpSortThreads, 0, s, 
        h->sp_hugeg, h->sp_bstart, c.gs, h->sp_hist, h->rec, h->ext, h->sp_st, h->A_x, h->A_y,
        h->A_i, h->sp_huge_scr, h->sp_huge_cap);
  }
  {
    Launch L(h, "k_sp_slices", s);
    launch_pdl(k_sp_slices, (uint32_t)((c.nslices * 32 + 255) / 256), 256, 0, s, 
        h->sp_st, h->sp_bstart, c.gs, h->sp_gbits, h->sp_phimax, h->A_x, h->A_y, h->ext,
        h->sp_prefmax, h->sp_slice);
  }
  TRY(stage_mark(h, 2, s));
  return GSCAN_OK;
}

// F4 -> C in (surv, sp_eb); codes of candidates marked
int sp_seg_f4(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  {
    Launch L(h, "k_sp_thresholds", s);
    launch_pdl(k_sp_thresholds, (kSpBuckets + 255) / 256, 256, 0, s, h->sp_gbits, h->sp_prefmax, h->sp_st,
                                                            h->sp_thr);
  }
  {
    Launch L(h, "k_sp_cand", s);
    launch_pdl(k_sp_cand, c.G, kSpCandThreads, c.smem_nb, s, h->sp_codes, h->sp_phi32, c.n, c.cap,
                                                     h->sp_thr, h->sp_st, h->surv, h->sp_eb,
                                                     h->sp_ccount, c.drop);
  }
  return GSCAN_OK;
}

// candidates (regions indexing cx/cy) + gathered points, exactly ordered and
// walked; the round-2 output compacted into A; the certificate's statistics
int sp_seg_walk(gscan_handle* h, const SpCtx& c, const double* cx, const double* cy,
                uint32_t n_walk_cap) {
  cudaStream_t s = c.s;
  const uint32_t nb = c.nb;
  {
    Launch L(h, "k_sp_rank_c", s);
    launch_pdl(k_sp_emit_place<1>, dim3(4, c.G), 256, 0, s, cx, cy, h->surv, h->sp_eb, h->rank,
                                                    h->sp_ccount, c.cap, h->sp_ccnt, nullptr,
                                                    h->ext, h->sp_st, h->rec, nullptr, nullptr,
                                                    (uint32_t)std::min<uint64_t>(h->wcap, 0xffffffffu));
  }
  TRY(scan_u32_slot(h, h->sp_ccnt, nb, h->sp_cstart, kLbCstart, s));
  {
    Launch L(h, "k_sp_place_c", s);
    launch_pdl(k_sp_emit_place<2>, dim3(4, c.G), 256, 0, s, cx, cy, h->surv, h->sp_eb, h->rank,
                                                    h->sp_ccount, c.cap, nullptr, h->sp_cstart,
                                                    h->ext, h->sp_st, h->rec, nullptr, nullptr,
                                                    0xffffffffu);
  }
  {
    Launch L(h, "k_sp_wcount", s);
    launch_pdl(k_sp_wcount, (nb + 255) / 256, 256, 0, s, h->sp_gbits, h->sp_hist, h->sp_ccnt, h->sp_wcnt);
  }
  TRY(scan_u32_slot(h, h->sp_wcnt, nb, h->sp_wstart, kLbWstart, s));
  {
    Launch L(h, "k_sp_place_cand", s);
    launch_pdl(k_sp_place_cand, nb / 8, 256, 0, s, h->rec, h->sp_cstart, h->sp_wstart, h->sp_slice,
                                           h->ext, h->sp_st, h->sp_big, h->C_x, h->C_y, h->C_i,
                                           h->sp_Wb, h->sp_Ws, h->flags);
  }
  {
    Launch L(h, "k_sp_sort_cand_big", s);
    launch_pdl(k_sp_sort_cand_big, h->sm_count, kSpSortThreads, kSpBigSmem, s, 
        h->sp_big, h->rec, h->sp_cstart, h->sp_wstart, h->sp_slice, h->ext, h->sp_st, h->C_x,
        h->C_y, h->C_i, h->sp_Wb, h->sp_Ws, h->flags, h->sp_huge_scr, h->sp_huge_cap);
  }
  {
    Launch L(h, "k_sp_place_gathered", s);
    launch_pdl(k_sp_place_gathered, h->sm_count * 4, 256, 0, s, 
        h->sp_glist, h->sp_bstart, c.gs, h->sp_hist, h->sp_wstart, h->A_x, h->A_y, h->A_i, h->ext,
        h->sp_st, h->C_x, h->C_y, h->C_i, h->sp_Wb, h->sp_Ws, h->flags);
  }
  TRY(stage_mark(h, 3, s));
  {
    Launch L(h, "k_sp_segments", s);
    launch_pdl(k_sp_segments, h->sm_count * 8, kBlock, 0, s, h->sp_Ws, h->sp_st, h->sp_seglo, h->sp_seghi);
  }
  {
    Launch L(h, "k_sp_walk", s);
    launch_pdl(k_sp_walk, (uint32_t)c.nslices, kWalkBlock, 0, s, h->C_x, h->C_y, h->sp_seglo, h->sp_seghi,
                                                         h->sp_st, h->ext, h->flags);
  }
  {
    const uint64_t tiles = (uint64_t)n_walk_cap / kCompactTile + 2;
    if (tiles > h->lb_stride) return fail(h, GSCAN_E_INTERNAL, "look-back slot too small");
    Launch L(h, "k_sp_compact", s);
    launch_pdl(k_sp_compact, (uint32_t)tiles, kBlock, 0, s, 
        h->C_x, h->C_y, h->C_i, h->sp_Wb, h->sp_Ws, h->flags, h->sp_st, h->A_x, h->A_y, h->A_i,
        h->sp_Rb, h->sp_Rs, h->lb_status + (size_t)kLbCompact * h->lb_stride, h->lb_ctr + kLbCompact);
  }
  // the duplicate check (side stream, sparse_dup_check) forks here, so it
  // overlaps the certificate and the Graham tail
  TRY(rec_event(h, h->ev_f3, s));
  {
    Launch L(h, "k_sp_rlo", s);
    launch_pdl(k_sp_rlo, h->sm_count * 8, kBlock, 0, s, h->sp_Rb, h->sp_st, h->sp_rlo);
  }
  {
    Launch L(h, "k_sp_cert_stats", s);
    launch_pdl(k_sp_cert_stats, h->sm_count, 256, 0, s, h->A_x, h->A_y, h->sp_Rs, h->sp_st);
  }
  {
    Launch L(h, "k_sp_cert_decide", s);
    launch_pdl(k_sp_cert_decide, 1, 32, 0, s, h->sp_st, c.drop || (h->debug & GSCAN_DEBUG_SPARSE_VERIFY));
  }
  return GSCAN_OK;
}

// F6 (one device only: it reads every survivor), then the read-back
int sp_seg_verify(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  {
    Launch L(h, "k_sp_verify", s);
#define A6 c.xs, c.ys, h->sp_codes, c.n, h->sp_gbits, h->sp_rlo, h->A_x, h->A_y, h->sp_st
    if (c.vec) launch_pdl(k_sp_verify<true>, c.G, kSpThreads, c.smem_nb + 4, s, A6);
    else launch_pdl(k_sp_verify<false>, c.G, kSpThreads, c.smem_nb + 4, s, A6);
#undef A6
  }
  return GSCAN_OK;
}

int sp_seg_tail(gscan_handle* h, const SpCtx& c) {
  cudaStream_t s = c.s;
  TRY(stage_mark(h, 4, s));
  CU(cudaMemcpyAsync(h->h_sp, h->sp_st, sizeof(SpState), cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&h->ctr->n2, &h->sp_st->n_r, 4, cudaMemcpyDeviceToDevice, s));
  // K7/K8 in the same graph: the tree strategy over the round-2 buffer, its
  // size read on the device; it no-ops when the sparse path failed
  TRY(tree_enqueue(h, h->A_x, h->A_y, h->A_i, &h->sp_st->n_r, 0, &h->sp_st->fail,
                   tree_forced_off(h), s));
  TRY(stage_mark(h, 5, s));
  return GSCAN_OK;
}

// Enqueues the whole sparse path up to and including the verification, the
// SpState read-back and Graham: no host round trip inside, fixed launch
// shapes for a given (input, n, config), so run_sparse replays it as one
// captured CUDA graph.
int sparse_enqueue(gscan_handle* h, const double* xs, const double* ys, uint32_t n,
                   const gscan_config& cfg) {
  const SpCtx c = sp_ctx(h, xs, ys, n, cfg.chunk_count);
  TRY(sp_seg_init(h, c));
  if (!h->k1_done) TRY(sp_seg_extremes(h, c));  // else h->ext came from the ingest
  TRY(sp_seg_sample(h, c));
  TRY(sp_seg_f2(h, c));
  TRY(sp_seg_plan(h, c));
  TRY(sp_seg_f3(h, c));
  TRY(sp_seg_sortg(h, c, xs, ys));
  TRY(sp_seg_f4(h, c));
  TRY(sp_seg_walk(h, c, xs, ys, n));
  TRY(sp_seg_verify(h, c));
  TRY(sp_seg_tail(h, c));
  return GSCAN_OK;
}

// Duplicate check on the low-priority side stream, forked inside the sparse
// graph after the compaction: it overlaps the certificate and the Graham tail
// (latency-bound kernels on few SMs) and joins the state read-back.
// The side kernels run one CTA per SM except on kSideFreeSms SMs, each
// reserving kSpSideSmem so that no Graham-tail CTA (kTreeCtaSmem) shares an SM
// with them: those latency-bound CTAs get SMs of their own (sparse.cuh
// side_take). Measured (C2): 16-36 free SMs equally good; two smaller side
// CTAs per SM, or leaving no SM free, slower; a side kernel that only occupies
// the SMs costs the main path ~30 us, the partitioning's partial-sector stores
// cost another ~60 us (DRAM read-for-merge) until its runs were padded to
// whole sectors (k_sp_dup_part<true>); forking later (inside the tree) is slower.
// k_sp_dups, which overlaps only the end of the tail, leaves 16 SMs free.
constexpr uint32_t kSideFreeSms = 32;
constexpr size_t kSpSideSmem = kSpDupPartSmemPad;  // 208 KB
static_assert(kSpSideSmem >= kSpDupPartSmem && kSpSideSmem >= kSpDupSmem && kSpSideSmem <= 226 * 1024,
              "side smem");
static_assert(kSpSideSmem + 1024 + kTreeCtaSmem + 1024 > 228 * 1024, "tree CTA would fit");
uint32_t side_free_sms() {
  static const int v = getenv("GSCAN_SIDE_FREE") ? atoi(getenv("GSCAN_SIDE_FREE")) : (int)kSideFreeSms;
  return (uint32_t)v;
}
// k_sp_dups overlaps only the end of the Graham tail (the one-CTA middle and
// the down and certificate kernels, few CTAs with work)
constexpr uint32_t kSideFreeSmsDups = 16;  // measured: 16 (0.974 ms) < 8 < 32 (0.983) < 4, 48
uint32_t side_free_sms_dups() {
  static const int v =
      getenv("GSCAN_SIDE_FREE2") ? atoi(getenv("GSCAN_SIDE_FREE2")) : (int)kSideFreeSmsDups;
  return (uint32_t)v;
}

int sparse_dup_check(gscan_handle* h, uint32_t n) {
  const uint32_t G = (uint32_t)h->sp_grid;
  const uint32_t nl = 2 * G;  // hash lists (k_sp_phi: two per CTA)
  static_assert(kSpPartChunk == 8 * 1024, "k_sp_dup_part: 8 entries per thread");
  const uint32_t cap = sparse_region_cap(h, n);
  // the scan of the partition counts needs only F3: it overlaps the main
  // stream's sorts and walk; the partitioning waits for the compaction
  CU(cudaStreamWaitEvent(h->side, h->ev_part, 0));  // recorded after k_sp_phi
  {
    const uint64_t tiles = ((uint64_t)kSpParts * nl + 1 + kScanTile - 1) / kScanTile;
    CU(cudaMemsetAsync(h->sp_side_status, 0, tiles * 8, h->side));
    CU(cudaMemsetAsync(h->sp_side_ticket, 0, sizeof(Counters), h->side));
    Launch L(h, "k_scan_u32(side)", h->side);
    k_scan_u32<<<tiles, kBlock, 0, h->side>>>(h->sp_part_off, kSpParts * nl, h->sp_part_off,
                                             h->sp_side_status, h->sp_side_ticket);
  }
  CU(cudaMemsetAsync(h->sp_side_work, 0, 2 * sizeof(uint32_t), h->side));
  CU(cudaStreamWaitEvent(h->side, h->ev_f3, 0));  // recorded after k_sp_compact
  {
    Launch L(h, "k_sp_dup_part", h->side);
    k_sp_dup_part<true><<<h->sm_count, 1024, kSpSideSmem, h->side>>>(
        h->sp_dup, h->sp_hcount, cap / 2, nl, h->sp_part_off, h->sp_st, h->sp_dup2, h->sp_side_work,
        side_free_sms(), nullptr);
  }
  {
    Launch L(h, "k_sp_dups", h->side);
    k_sp_dups<<<h->sm_count, 1024, kSpSideSmem, h->side>>>(h->sp_dup2, h->sp_part_off, nl, h->sp_st,
                                                              h->sp_side_work + 1, side_free_sms_dups(),
                                                              h->sp_dup_scr, h->sp_dup_scap, true);
  }
  {
    Launch L(h, "k_sp_side_check", h->side);
    k_sp_side_check<<<1, 32, 0, h->side>>>(h->sp_side_work, nl, h->sp_st);
  }
  CU(cudaEventRecord(h->ev_dup, h->side));
  return GSCAN_OK;
}

void sp_debug_print(const gscan_handle* h, const char* tag) {
  const SpState& sp = *h->h_sp;
  fprintf(stderr, "%s ", tag);
  fprintf(stderr,
            "[sparse] fail=%#x m=%u M=%u b_l=%u l=%u/%u l_idx=%u ties=%u step=%u,%u slices=%u+%u "
            "n_gb=%u n_g=%u max_g=%u n_c=%u n_w=%u n_r=%u dups=%u vfail=%u why=%u bigc=%u cert=%u kmax=%u rho=%.3g phi=[%.4f,%.4f]\n",
            sp.fail, sp.m, sp.M, sp.b_l, sp.l, sp.l_check, sp.l_idx, sp.ties, sp.step_r, sp.step_l,
            sp.n_right, sp.n_left, sp.n_gb, sp.n_g, sp.max_g, sp.n_c, sp.n_w, sp.n_r, sp.dups,
            sp.verify_fail, sp.why, sp.n_bigc, sp.cert, sp.k_max, sqrt(__longlong_as_double_host(sp.rho2_bits)),
            unord_host(sp.phi_lo), unord_host(sp.phi_hi));
  }

int run_sparse(gscan_handle* h, const double* xs, const double* ys, uint32_t n,
               const gscan_config& cfg, uint64_t* hull_size, gscan_stats* st, bool* ok) {
  *ok = false;
  TRY(sparse_init(h));
  ++h->sp_calls;
  const uint64_t c = cfg.chunk_count;
  const uint64_t nslices = 2 * std::min<uint64_t>(c, n);
  if (nslices + 2 > h->sp_seg_cap) {
    dfree(h->sp_seglo);
    dfree(h->sp_seghi);
    CU(cudaMalloc(&h->sp_seglo, (nslices + 2) * 4));
    CU(cudaMalloc(&h->sp_seghi, (nslices + 2) * 4));
    h->sp_seg_cap = nslices + 2;
    h->sp_graph_ok = false;
  }
  cudaStream_t s = h->stream;
  const bool dup_check = !h->sp_no_dup;
  // one captured graph per (input, n, config): replayed while unchanged
  SpGraphKey key{xs, ys, n, c, h->debug, dup_check, h->k1_done};
  TRY(tree_workspace(h, std::min<uint32_t>(n, kTreeMaxN)));  // no allocation inside the capture
  const void* bufs[7] = {h->A_x, h->A_y, h->A_i, h->C_x, h->C_y, h->C_i, h->tw_pool};
  for (int k = 0; k < 7; ++k) key.bufs[k] = bufs[k];
  bool graph_path = !(h->profiling || !h->use_graphs);
  if (!graph_path) {
    // profiling: a short busy kernel first keeps the stream occupied while the
    // host enqueues the per-kernel events and launches, so each event pair
    // brackets its kernel and not the host's launch latency
    if (h->profiling) k_busy_wait<<<1, 32, 0, s>>>(200000ull);
    TRY(sparse_enqueue(h, xs, ys, n, cfg));
  } else {
    if (!h->sp_graph_ok || !(key == h->sp_key)) {
      if (h->sp_graph_exec) { cudaGraphExecDestroy(h->sp_graph_exec); h->sp_graph_exec = nullptr; }
      h->sp_graph_ok = false;
      const uint64_t l0 = h->launches;
      // capture on the handle's private stream (the caller's stream may be
      // the legacy default stream, which cannot be captured)
      h->stream = h->cap_stream;
      cudaError_t be = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed);
      int rc = (be == cudaSuccess) ? sparse_enqueue(h, xs, ys, n, cfg) : GSCAN_E_CUDA;
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = (be == cudaSuccess) ? cudaStreamEndCapture(h->stream, &graph) : be;
      h->stream = s;
      cudaError_t ie = cudaErrorUnknown;
      if (rc == GSCAN_OK && ce == cudaSuccess) {
        ie = cudaGraphInstantiate(&h->sp_graph_exec, graph, 0);
      }
      if (graph) cudaGraphDestroy(graph);
      if (rc != GSCAN_OK || ce != cudaSuccess || ie != cudaSuccess) {
        // capture unavailable here: run without graphs from now on
        cudaGetLastError();
        if (h->sp_debug)
          fprintf(stderr, "[sparse] graph capture disabled: %s / %s / %s\n", h->err.c_str(),
                  cudaGetErrorString(ce), cudaGetErrorString(ie));
        h->use_graphs = false;
        graph_path = false;
        h->launches = l0;
        if (h->sp_graph_exec) { cudaGraphExecDestroy(h->sp_graph_exec); h->sp_graph_exec = nullptr; }
        TRY(sparse_enqueue(h, xs, ys, n, cfg));
        goto enqueued;
      }
      h->sp_graph_launches = h->launches - l0;
      h->launches = l0;
      h->sp_key = key;
      h->sp_graph_ok = true;
    }
#ifdef GSCAN_STAMP  // diagnostics build: when each stream finished, relative to the graph's start
    host_mark(1);
    static unsigned long long* stamp = nullptr;
    if (!stamp) cudaHostAlloc(&stamp, 64, cudaHostAllocMapped);
    k_stamp<<<1, 1, 0, s>>>(stamp + 2);
#endif
    CU(cudaGraphLaunch(h->sp_graph_exec, s));
#ifdef GSCAN_STAMP
    if (h->user_out) k_copy_out<<<8, 256, 0, s>>>(h->d_out, h->ctr, h->user_out, h->user_cap);
    k_stamp<<<1, 1, 0, s>>>(stamp + 0);
    if (dup_check) {
      TRY(sparse_dup_check(h, n));
      k_stamp<<<1, 1, 0, h->side>>>(stamp + 1);
      CU(cudaStreamWaitEvent(s, h->ev_dup, 0));
      CU(cudaMemcpyAsync(&h->h_sp->fail, &h->sp_st->fail, 4, cudaMemcpyDeviceToHost, s));
    }
    TRY(sync_counters(h));
    host_mark(2);
    static unsigned long long prev_end = 0;
    static std::vector<double> rows;
    rows.push_back((stamp[0] - stamp[2]) / 1e3);
    rows.push_back((stamp[1] - stamp[2]) / 1e3);
    rows.push_back(prev_end ? (stamp[2] - prev_end) / 1e3 : 0.0);
    prev_end = std::max(stamp[0], stamp[1]);
    if (rows.size() == 3 * 24) {  // one print per 24 calls (printing widens its own gap)
      for (size_t r = 0; r < rows.size(); r += 3)
        fprintf(stderr, "[stamp] main %.1f us side %.1f us gap before %.1f us\n", rows[r], rows[r + 1], rows[r + 2]);
      rows.clear();

    }
    h->launches += h->sp_graph_launches;
    goto read_back;
#endif
    h->launches += h->sp_graph_launches;
  }
enqueued:
  if (h->user_out) {  // the tree's hull straight into the caller's buffer (no second sync)
    k_copy_out<<<8, 256, 0, s>>>(h->d_out, h->ctr, h->user_out, h->user_cap);
    CU(cudaGetLastError());
  }
  if (dup_check) {
    // the duplicate check's verdict joins the state read-back: one sync
    TRY(sparse_dup_check(h, n));
    CU(cudaStreamWaitEvent(s, h->ev_dup, 0));
    CU(cudaMemcpyAsync(&h->h_sp->fail, &h->sp_st->fail, 4, cudaMemcpyDeviceToHost, s));
  }
  TRY(sync_counters(h));
#ifdef GSCAN_STAMP
read_back:
#endif
  const SpState sp = *h->h_sp;
  if (h->sp_debug) sp_debug_print(h, "[run]");
  h->sp_fail = sp.fail | ((sp.fail & kSpFailInternal) ? (sp.why << 16) : 0u);
  h->sp_walked = sp.n_w;
  h->sp_cert = sp.cert;
  if (sp.fail) {
    ++h->sp_fallbacks;
    return GSCAN_OK;
  }
  {
    h->graham_path = 0;
    h->graham_fails = 0;
    bool done = false;
    TRY(tree_finish(h, h->A_x, h->A_y, h->A_i, &done));
    h->user_out_done = done && h->user_out && !(h->debug & GSCAN_DEBUG_FORCE_FALLBACK);
    if (!done) {  // the tree declined: the other strategies, launched from here
      TRY(stage_graham(h, h->A_x, h->A_y, h->A_i, sp.n_r, /*skip_tree=*/true));
      if (graph_path) k_tstamp<<<1, 1, 0, s>>>(h->ctr, 5);
      else CU(cudaEventRecord(h->ev[5], s));
    }
    // the tree's result (hull count) came with the first read-back, unless
    // more work was launched since
    if (!done || (h->debug & GSCAN_DEBUG_FORCE_FALLBACK)) TRY(sync_counters(h));
  }
  const Counters& cc = *h->h_ctr;
  *hull_size = cc.hull;
  if (st) {
    st->n_input = n;
    st->n_after_round1 = cc.n1;
    st->n_after_round2 = sp.n_r;
    st->hull_size = cc.hull;
    if (graph_path) {  // the graph's stage stamps, read back with the counters
      const uint64_t* t = cc.tstamp;
      auto ms = [&](int a, int b) { return (float)((double)(t[b] - t[a]) * 1e-6); };
      st->t_round1_ms = ms(0, 1);
      st->t_annotate_ms = ms(1, 2);
      st->t_sort_ms = ms(2, 3);
      st->t_round2_ms = ms(3, 4);
      st->t_finalize_ms = ms(4, 5);
      st->t_total_ms = ms(0, 5);
    } else {
      st->t_round1_ms = ev_ms(h->ev[0], h->ev[1]);
      st->t_annotate_ms = ev_ms(h->ev[1], h->ev[2]);
      st->t_sort_ms = ev_ms(h->ev[2], h->ev[3]);
      st->t_round2_ms = ev_ms(h->ev[3], h->ev[4]);
      st->t_finalize_ms = ev_ms(h->ev[4], h->ev[5]);
      st->t_total_ms = ev_ms(h->ev[0], h->ev[5]);
    }
  }
  h->sp_used = 1;
  *ok = true;
  return GSCAN_OK;
}

// Full pipeline on device-resident SoA input. Hull indices left in h->d_out.
int run_pipeline(gscan_handle* h, const double* xs, const double* ys, uint64_t n64,
                 const gscan_config& cfg, uint64_t* hull_size, gscan_stats* st) {
  TRY(validate(h, n64, cfg));
  TRY(reserve(h, n64));
  const uint32_t n = (uint32_t)n64;
  h->launches = 0;
  h->kt_used = 0;
  h->sp_used = 0;
  h->sp_fail = 0;
  bool ext_ready = false;
  if (h->large && !sparse_eligible(h, n64, cfg))
    return fail(h, GSCAN_E_TOO_LARGE,
                "%llu points: above %llu points one device runs only the default configuration "
                "(sparse path); shard the input (distributed.sharded_hull)",
                (unsigned long long)n64, (unsigned long long)full_sort_max());
  if (sparse_eligible(h, n64, cfg)) {
    bool ok = false;
    TRY(run_sparse(h, xs, ys, n, cfg, hull_size, st, &ok));
    if (ok) return GSCAN_OK;
    if (h->large)
      return fail(h, GSCAN_E_TOO_LARGE,
                  "%llu points declined the sparse path (fail bits %#x); the full-sort fallback "
                  "needs more than one device's memory above %llu points: shard the input",
                  (unsigned long long)n64, h->sp_fail, (unsigned long long)full_sort_max());
    ext_ready = true;  // K1 ran on this input inside the sparse attempt
  }
  CU(cudaEventRecord(h->ev[0], h->stream));
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  TRY(stage_round1_keys(h, xs, ys, n, cfg.enable_round1, ext_ready));
  CU(cudaEventRecord(h->ev[1], h->stream));
  CU(cudaEventRecord(h->ev[2], h->stream));  // annotate (keys) is fused into round 1
  TRY(stage_annotate_sort(h, xs, ys, n, -1, 3, /*keys_done=*/true));
  double *Rx, *Ry;
  uint32_t* Ri;
  TRY(stage_round2(h, cfg, &Rx, &Ry, &Ri));
  CU(cudaEventRecord(h->ev[4], h->stream));
  TRY(sync_counters(h));
  TRY(stage_graham(h, Rx, Ry, Ri, h->h_ctr->n2));
  CU(cudaEventRecord(h->ev[5], h->stream));
  TRY(sync_counters(h));
  const Counters& c = *h->h_ctr;
  *hull_size = c.hull;
  if (st) {
    st->n_input = n64;
    st->n_after_round1 = c.n1;
    st->n_after_round2 = c.n2;
    st->hull_size = c.hull;
    st->t_round1_ms = ev_ms(h->ev[0], h->ev[1]);
    st->t_annotate_ms = ev_ms(h->ev[1], h->ev[2]);
    st->t_sort_ms = ev_ms(h->ev[2], h->ev[3]);
    st->t_round2_ms = ev_ms(h->ev[3], h->ev[4]);
    st->t_finalize_ms = ev_ms(h->ev[4], h->ev[5]);
    st->t_total_ms = ev_ms(h->ev[0], h->ev[5]);
  }
  return GSCAN_OK;
}

constexpr uint64_t kIngestMinN = 4u << 20;  // below this one copy + K1 is as fast
constexpr uint32_t kIngestChunks = 8;

int ingest_overlapped(gscan_handle* h, const double* xs, const double* ys, uint64_t n) {
  if (!h->copy) {
    CU(cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking));
    for (auto& e : h->ev_chunk) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CU(cudaMalloc(&h->ext_parts, kIngestChunks * sizeof(ExtResult)));
    CU(cudaMalloc(&h->ext_off, kIngestChunks * 4));
    CU(cudaMalloc(&h->ext_pp, (size_t)kIngestChunks * h->sm_count * sizeof(ExtAcc)));
    CU(cudaMalloc(&h->ext_pctr, kIngestChunks * sizeof(Counters)));
    CU(cudaMemset(h->ext_pctr, 0, kIngestChunks * sizeof(Counters)));
  }
  // chunk boundaries on whole K1 tiles (16-byte aligned starts)
  uint32_t off[kIngestChunks + 1];
  for (uint32_t k = 0; k <= kIngestChunks; ++k)
    off[k] = k == kIngestChunks ? (uint32_t)n
                                : (uint32_t)((n * k / kIngestChunks) / kExtTile * kExtTile);
  CU(cudaMemcpyAsync(h->ext_off, off, kIngestChunks * 4, cudaMemcpyHostToDevice, h->stream));
  // the copy stream starts after everything already on the handle's stream
  CU(cudaEventRecord(h->ev_chunk[0], h->stream));
  CU(cudaStreamWaitEvent(h->copy, h->ev_chunk[0], 0));
  for (uint32_t k = 0; k < kIngestChunks; ++k) {
    const size_t len = (size_t)(off[k + 1] - off[k]) * 8;
    CU(cudaMemcpyAsync(h->d_xs + off[k], xs + off[k], len, cudaMemcpyHostToDevice, h->copy));
    CU(cudaMemcpyAsync(h->d_ys + off[k], ys + off[k], len, cudaMemcpyHostToDevice, h->copy));
    CU(cudaEventRecord(h->ev_chunk[k], h->copy));
  }
  for (uint32_t k = 0; k < kIngestChunks; ++k) {
    CU(cudaStreamWaitEvent(h->stream, h->ev_chunk[k], 0));
    Launch L(h, "k_extremes_tma(ingest)");
    k_extremes_tma<<<h->sm_count, kExtThreads, kExtSmem, h->stream>>>(
        h->d_xs + off[k], h->d_ys + off[k], off[k + 1] - off[k], h->ext_pp + (size_t)k * h->sm_count,
        h->ext_parts + k, h->ext_pctr + k);
  }
  {
    Launch L(h, "k_ext_merge");
    k_ext_merge<<<1, 32, 0, h->stream>>>(h->ext_parts, h->ext_off, kIngestChunks, h->ext);
  }
  return GSCAN_OK;
}

gscan_config resolve(const gscan_config* cfg) {
  gscan_config c;
  gscan_config_default(&c);
  if (cfg) c = *cfg;
  return c;
}

std::mutex g_default_mu;
gscan_handle* g_default = nullptr;

}  // namespace

// ============================================================================
// C-ABI

// ---------------------------------------------------------------------------
// Sharded sparse path. Each rank runs the segments of the
// sparse path on its shard; the host (distributed.py) does the collectives
// between the phases: sample cells and the bucket histogram are summed, P_l
// is the best record over ranks, P_l's in-bucket rank and the phi maxima are
// reduced, gathered and candidate points travel to rank 0 as records {x, y,
// global index, bucket}, rank 0 broadcasts the prefix maxima, and the 64-bit
// hashes are exchanged by partition for the duplicate check. Every exchange is
// KB-MB sized; no rank ever holds another rank's survivors.
constexpr uint32_t kDistMaxRanks = 64;

int dist_init(gscan_handle* h) {
  if (h->dist_ctr) return GSCAN_OK;
  CU(cudaMalloc(&h->dist_ctr, 64));
  CU(cudaMalloc(&h->dist_pm, ((size_t)kSpParts * kDistMaxRanks + 2) * 4));
  CU(cudaMalloc(&h->dist_hc, kDistMaxRanks * 4));
  CU(cudaMalloc(&h->dist_lb, kDistMaxRanks * 8));
  CU(cudaMalloc(&h->dist_rec, kDistRecLen * 8));
  CU(cudaMalloc(&h->dist_recs, (size_t)kDistMaxRanks * kDistRecLen * 8));
  CU(cudaMalloc(&h->dist_ext, 16 * 8));
  CU(cudaMalloc(&h->dist_pc, kSpParts * 4));
  CU(cudaMalloc(&h->dist_pref, (kSpBuckets + 1) * 4));
  CU(cudaMemset(h->dist_rec, 0, kDistRecLen * 8));
  return GSCAN_OK;
}

SpCtx dist_ctx(gscan_handle* h) {
  SpCtx c = sp_ctx(h, h->dist_xs, h->dist_ys, h->dist_n, h->dist_chunks);
  c.base = h->dist_base;
  c.sharded = true;
  // after the plan the slice structure is the GLOBAL one (M = all ranks'
  // points): size the slice grids by it, not by this rank's shard
  if (h->h_sp && h->h_sp->M) c.nslices = 2 * std::min<uint64_t>(h->dist_chunks, h->h_sp->M);
  return c;
}

// slice segment arrays for the global slice count (rank 0's walk)
int dist_slices_ensure(gscan_handle* h, const SpCtx& c) {
  if (c.nslices + 2 <= h->sp_seg_cap) return GSCAN_OK;
  dfree(h->sp_seglo);
  dfree(h->sp_seghi);
  h->sp_seg_cap = 0;
  CU(cudaMalloc(&h->sp_seglo, (c.nslices + 2) * 4));
  CU(cudaMalloc(&h->sp_seghi, (c.nslices + 2) * 4));
  h->sp_seg_cap = c.nslices + 2;
  h->sp_graph_ok = false;
  return GSCAN_OK;
}

// fail word for the host: the internal-error site in the high half
uint32_t dist_fail(const gscan_handle* h) {
  const SpState& sp = *h->h_sp;
  return sp.fail | ((sp.fail & kSpFailInternal) ? (sp.why << 16) : 0u);
}

int dist_fill(gscan_handle* h, const SpCtx& c, uint32_t n_items, uint32_t idx0, const uint32_t* b,
              uint32_t* count) {
  if (n_items > 0 && (n_items + c.G - 1) / c.G > c.cap)
    return fail(h, GSCAN_E_CAPACITY, "sharded path: %u records exceed the emission regions", n_items);
  Launch L(h, "k_sp_fill_regions", c.s);
  k_sp_fill_regions<<<std::max(1u, std::min((n_items + 255) / 256, 4u * h->sm_count)), 256, 0, c.s>>>(
      n_items, idx0, b, c.G, c.cap, h->surv, h->sp_eb, count);
  return GSCAN_OK;
}

extern "C" {

void gscan_config_default(gscan_config* cfg) {
  if (!cfg) return;
  cfg->chunk_count = 1024;
  cfg->enable_round1 = 1;
  cfg->enable_round2 = 1;
  cfg->chunked = 1;
  cfg->reserved = 0;
}

const char* gscan_status_string(int s) {
  switch (s) {
    case GSCAN_OK: return "ok";
    case GSCAN_E_EMPTY_INPUT: return "empty input";
    case GSCAN_E_ZERO_CHUNKS: return "chunk_count must be positive";
    case GSCAN_E_CAPACITY: return "output capacity too small";
    case GSCAN_E_CUDA: return "CUDA error";
    case GSCAN_E_INVALID: return "invalid argument";
    case GSCAN_E_TOO_LARGE: return "input too large";
    case GSCAN_E_NO_DEVICE: return "no CUDA device";
    case GSCAN_E_INTERNAL: return "internal consistency check failed";
    case GSCAN_E_IO: return "I/O error";
    case GSCAN_E_PARSE: return "parse error";
    case GSCAN_E_NCCL: return "collective (NCCL) failure";
    default: return "unknown status";
  }
}

const char* gscan_last_error(const gscan_handle* h) { return h ? h->err.c_str() : ""; }
uint64_t gscan_last_launch_count(const gscan_handle* h) { return h ? h->launches : 0; }

int gscan_create(int device, gscan_handle** out) {
  if (!out) return GSCAN_E_INVALID;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return GSCAN_E_NO_DEVICE;
  gscan_handle* h = new gscan_handle();
  if (device < 0) cudaGetDevice(&device);
  h->device = device;
  int rc = GSCAN_OK;
  auto init = [&]() -> int {
    CU(cudaSetDevice(device));
    CU(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device));
    CU(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
    {
      // the duplicate check's stream; its SMs are partitioned explicitly
      // (side_free_sms). Measured: a high priority on either stream changes
      // nothing (C2, within 3 us).
      int lo = 0, hi = 0;
      CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      CU(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, lo));
    }
    CU(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_f3, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_part, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_dup, cudaEventDisableTiming));
    CU(cudaMalloc(&h->partials, sizeof(ExtAcc) * h->sm_count * 8));
    CU(cudaMalloc(&h->ext, sizeof(ExtResult)));
    CU(cudaMalloc(&h->ctr, sizeof(Counters)));
    CU(cudaMemset(h->ctr, 0, sizeof(Counters)));
    CU(cudaMalloc(&h->scratch64, 16));
    CU(cudaMallocHost(&h->h_ctr, sizeof(Counters)));
    CU(cudaMallocHost(&h->h_info, kTreeInfoWords * sizeof(uint32_t)));
    for (auto& e : h->ev) CU(cudaEventCreate(&e));
    CU(cudaFuncSetAttribute(k_graham_candidate_seq, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kCandSmem));
    CU(cudaFuncSetAttribute(k_bucket_sort_block, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kBlockCap * (8 + 8 + 8 + 8 + 4 + 2)));
    CU(cudaFuncSetAttribute(k_bucket_sort_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kSortCap * (8 + 8 + 4 + 4)));
    const int nbs = (int)(kSpBuckets * 4);
    CU(cudaFuncSetAttribute(k_sp_hist<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_hist<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_hist_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_hist_ring, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kF2RingSmem));
    CU(cudaFuncSetAttribute(k_extremes_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kExtSmem));
    CU(cudaFuncSetAttribute(k_sp_phi<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_phi<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_phimax_codes, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_cand, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs));
    CU(cudaFuncSetAttribute(k_sp_verify<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs + 4));
    CU(cudaFuncSetAttribute(k_sp_verify<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, nbs + 4));
    CU(cudaFuncSetAttribute(k_sp_sort_gathered, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpSmallSmem));
    CU(cudaFuncSetAttribute(k_sp_sort_gathered_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpBigSmem));
    CU(cudaFuncSetAttribute(k_sp_sort_cand_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpBigSmem));
    CU(cudaFuncSetAttribute(k_sp_dups, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpSideSmem));
    CU(cudaFuncSetAttribute(k_sp_dup_part<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpSideSmem));
    CU(cudaFuncSetAttribute(k_sp_dup_part<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kSpSideSmem));
    CU(cudaFuncSetAttribute(k_gr_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTreeSmem));
    CU(cudaFuncSetAttribute(k_gr_up, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTreeCtaSmem));
    CU(cudaFuncSetAttribute(k_gr_down, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTreeCtaSmem));
    CU(cudaFuncSetAttribute(k_gr_cert, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTreeCtaSmem));
    h->sp_grid = h->sm_count;
    h->use_graphs = !env_flag("GSCAN_NO_GRAPH");
    return GSCAN_OK;
  };
  rc = init();
  if (rc != GSCAN_OK) {
    gscan_destroy(h);
    return rc;
  }
  *out = h;
  return GSCAN_OK;
}

int gscan_destroy(gscan_handle* h) {
  if (!h) return GSCAN_OK;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  free_buffers(h);
  dfree(h->d_xs); dfree(h->d_ys);
  dfree(h->ext_parts); dfree(h->ext_off); dfree(h->ext_pp); dfree(h->ext_pctr);
  for (auto& e : h->ev_chunk) if (e) cudaEventDestroy(e);
  if (h->copy) cudaStreamDestroy(h->copy);
  dfree(h->partials); dfree(h->ext); dfree(h->ctr); dfree(h->scratch64);
  dfree(h->sp_th); dfree(h->sp_cdf); dfree(h->sp_cells); dfree(h->sp_big); dfree(h->sp_bigg); dfree(h->sp_hugeg); dfree(h->sp_gcount); dfree(h->sp_side_status); dfree(h->sp_side_ticket); dfree(h->sp_side_work); dfree(h->sp_ccount); dfree(h->sp_hcount); dfree(h->sp_hist_part); dfree(h->sp_phi_part); dfree(h->sp_part_off);
  dfree(h->sp_d2); dfree(h->sp_hist); dfree(h->sp_bstart); dfree(h->sp_gbits); dfree(h->sp_glist);
  dfree(h->sp_gcnt); dfree(h->sp_phimax); dfree(h->sp_prefmax); dfree(h->sp_slice);
  dfree(h->sp_ccnt); dfree(h->sp_cstart); dfree(h->sp_wcnt); dfree(h->sp_wstart); dfree(h->sp_rlo);
  dfree(h->sp_seglo); dfree(h->sp_seghi); dfree(h->sp_st);
  if (h->mt_states) cudaFree(h->mt_states);
  if (h->mt_jtab) cudaFree(h->mt_jtab);
  if (h->h_sp) cudaFreeHost(h->h_sp);
  if (h->h_ctr) cudaFreeHost(h->h_ctr);
  if (h->h_info) cudaFreeHost(h->h_info);
  dfree(h->tw_pool);
  dfree(h->sp_gs); dfree(h->sp_thr); dfree(h->sp_gsz); dfree(h->dist_ctr); dfree(h->dist_pm); dfree(h->dist_hc);
  dfree(h->dist_lb);
  dfree(h->dist_rec); dfree(h->dist_recs); dfree(h->dist_ext); dfree(h->dist_pc); dfree(h->dist_pref);
  if (h->h_out) cudaFreeHost(h->h_out);
  for (auto& e : h->ev) if (e) cudaEventDestroy(e);
  for (auto& k : h->ktimes) { cudaEventDestroy(k.a); cudaEventDestroy(k.b); }
  if (h->sp_graph_exec) cudaGraphExecDestroy(h->sp_graph_exec);
  if (h->side) { cudaStreamSynchronize(h->side); cudaStreamDestroy(h->side); }
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->ev_f3) cudaEventDestroy(h->ev_f3);
  if (h->ev_part) cudaEventDestroy(h->ev_part);
  if (h->ev_dup) cudaEventDestroy(h->ev_dup);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
  return GSCAN_OK;
}

int gscan_reserve(gscan_handle* h, uint64_t n) {
  if (!h) return GSCAN_E_INVALID;
  CU(cudaSetDevice(h->device));
  return reserve(h, n);
}

int gscan_set_stream(gscan_handle* h, void* stream) {
  if (!h) return GSCAN_E_INVALID;
  if (stream) {
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    h->stream = static_cast<cudaStream_t>(stream);
    h->own_stream = false;
  }
  return GSCAN_OK;
}

int gscan_set_debug(gscan_handle* h, uint32_t flags) {
  if (!h) return GSCAN_E_INVALID;
  h->debug = flags;
  return GSCAN_OK;
}

int gscan_last_graham_info(const gscan_handle* h, uint32_t* path, uint32_t* certificate_failures) {
  if (!h) return GSCAN_E_INVALID;
  if (path) *path = h->graham_path;
  if (certificate_failures) *certificate_failures = h->graham_fails;
  return GSCAN_OK;
}

int gscan_last_sparse_info(const gscan_handle* h, uint32_t* used, uint32_t* fail_bits,
                           uint32_t* n_walked) {
  if (!h) return GSCAN_E_INVALID;
  if (used) *used = h->sp_used;
  if (fail_bits) *fail_bits = h->sp_fail;
  if (n_walked) *n_walked = h->sp_walked;
  return GSCAN_OK;
}

// debug hook (not in the public header): copy the last sparse round-2 buffer
// (input indices) to the host
int gscan_debug_round2(gscan_handle* h, uint32_t* host_out, uint64_t cap, uint64_t* len,
                       uint32_t* w_out, uint8_t* f_out, uint64_t* wlen) {
  if (!h || !h->h_sp) return GSCAN_E_INVALID;
  const uint64_t m = std::min<uint64_t>(cap, h->h_sp->n_r);
  *len = h->h_sp->n_r;
  CU(cudaMemcpy(host_out, h->A_i, m * 4, cudaMemcpyDeviceToHost));
  const uint64_t w = std::min<uint64_t>(cap, h->h_sp->n_w);
  *wlen = h->h_sp->n_w;
  CU(cudaMemcpy(w_out, h->C_i, w * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(f_out, h->flags, w, cudaMemcpyDeviceToHost));
  return GSCAN_OK;
}

int gscan_set_profiling(gscan_handle* h, int enabled) {
  if (!h) return GSCAN_E_INVALID;
  h->profiling = enabled != 0;
  return GSCAN_OK;
}

int gscan_last_kernel_times(const gscan_handle* h, const char** names, double* ms, int cap) {
  if (!h) return 0;
  int k = 0;
  for (size_t i = 0; i < h->kt_used && k < cap; ++i, ++k) {
    if (names) names[k] = h->ktimes[i].name;
    if (ms) ms[k] = ev_ms(h->ktimes[i].a, h->ktimes[i].b);
  }
  return k;
}

int gscan_hull_f64_device(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                          const gscan_config* cfg, uint32_t* d_out_idx, uint64_t out_cap,
                          uint64_t* out_len, gscan_stats* stats) {
  if (!h || (!d_xs && n) || (!d_ys && n)) return GSCAN_E_INVALID;
  CU(cudaSetDevice(h->device));
  const gscan_config c = resolve(cfg);
  uint64_t hs = 0;
#ifdef GSCAN_STAMP
  host_mark(0);
#endif
  h->user_out = d_out_idx;
  h->user_cap = out_cap;
  h->user_out_done = false;
  const int rc = run_pipeline(h, d_xs, d_ys, n, c, &hs, stats);
  h->user_out = nullptr;
  TRY(rc);
  if (out_len) *out_len = hs;
  if (hs > out_cap) return fail(h, GSCAN_E_CAPACITY, "hull has %llu vertices, capacity %llu",
                                (unsigned long long)hs, (unsigned long long)out_cap);
  if (d_out_idx && hs && !h->user_out_done) {
    CU(cudaMemcpyAsync(d_out_idx, h->d_out, hs * 4, cudaMemcpyDeviceToDevice, h->stream));
    CU(cudaStreamSynchronize(h->stream));
  }
#ifdef GSCAN_STAMP
  host_mark(3);
#endif
  return GSCAN_OK;
}

constexpr uint64_t kWidenOnDevice = 1u << 16;
__global__ void k_widen_u32(const uint32_t* __restrict__ in, uint32_t n, uint64_t* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[i];
}

int gscan_hull_f64(gscan_handle* h, const double* xs, const double* ys, uint64_t n,
                   const gscan_config* cfg, uint64_t* out_idx, uint64_t out_cap,
                   uint64_t* out_len, gscan_stats* stats) {
  if (!h || (n && (!xs || !ys))) return GSCAN_E_INVALID;
  CU(cudaSetDevice(h->device));
  const gscan_config c = resolve(cfg);
  TRY(validate(h, n, c));
  TRY(reserve(h, n));
  if (n > h->host_cap) {  // device copy of host input, host entry only
    dfree(h->d_xs);
    dfree(h->d_ys);
    h->host_cap = 0;
    CU(cudaMalloc(&h->d_xs, (n + 1) * 8));
    CU(cudaMalloc(&h->d_ys, (n + 1) * 8));
    h->host_cap = n;
  }
  uint64_t hs = 0;
  // Overlapped ingest: the H2D copy in chunks on the
  // copy stream, K1 on every chunk as it lands (the only stage that does not
  // need all of the input), a merge, and the sparse path without its K1.
  const bool overlap = n >= kIngestMinN && sparse_eligible(h, n, c) && !h->profiling;
  if (overlap) {
    TRY(ingest_overlapped(h, xs, ys, n));
    h->k1_done = true;
  } else {
    CU(cudaMemcpyAsync(h->d_xs, xs, n * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(h->d_ys, ys, n * 8, cudaMemcpyHostToDevice, h->stream));
  }
  const int rc = run_pipeline(h, h->d_xs, h->d_ys, n, c, &hs, stats);
  h->k1_done = false;
  TRY(rc);
  if (out_len) *out_len = hs;
  if (hs > out_cap) return fail(h, GSCAN_E_CAPACITY, "hull has %llu vertices, capacity %llu",
                                (unsigned long long)hs, (unsigned long long)out_cap);
  if (!out_idx || hs == 0) return GSCAN_OK;
  if (hs >= kWidenOnDevice) {
    // large hulls (points on a circle): widen to uint64 on the device and copy
    // straight into the caller's buffer (a host loop over 20M entries took
    // ~20 ms); C_x is free once the pipeline has finished
    uint64_t* wide = reinterpret_cast<uint64_t*>(h->C_x);
    const uint32_t grid = std::max(1u, std::min<uint32_t>((uint32_t)((hs + 255) / 256), h->sm_count * 8));
    k_widen_u32<<<grid, 256, 0, h->stream>>>(h->d_out, (uint32_t)hs, wide);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out_idx, wide, hs * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return GSCAN_OK;
  }
  if (hs > h->h_out_cap) {
    if (h->h_out) cudaFreeHost(h->h_out);
    h->h_out = nullptr;
    CU(cudaMallocHost(&h->h_out, hs * 4));
    h->h_out_cap = hs;
  }
  CU(cudaMemcpyAsync(h->h_out, h->d_out, hs * 4, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  for (uint64_t i = 0; i < hs; ++i) out_idx[i] = h->h_out[i];
  return GSCAN_OK;
}

int gscan_hull(const double* xs, const double* ys, uint64_t n, uint64_t* out_idx,
               uint64_t out_cap, uint64_t* out_len) {
  std::lock_guard<std::mutex> lock(g_default_mu);
  if (!g_default) {
    const int rc = gscan_create(-1, &g_default);
    if (rc != GSCAN_OK) return rc;
  }
  return gscan_hull_f64(g_default, xs, ys, n, nullptr, out_idx, out_cap, out_len, nullptr);
}

// ---- stage entry points ----

int gscan_stage_extremes(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         uint64_t out[5]) {
  if (!h || !out) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  TRY(stage_round1(h, d_xs, d_ys, (uint32_t)n, 1));
  ExtResult r;
  CU(cudaMemcpyAsync(&r, h->ext, sizeof r, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  for (int k = 0; k < 5; ++k) out[k] = r.idx[k];
  return GSCAN_OK;
}

int gscan_stage_round1(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       uint32_t* d_out, uint64_t* n_out) {
  if (!h || !d_out || !n_out) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  if (h->large) return fail(h, GSCAN_E_TOO_LARGE, "stage entry points need n <= %llu", (unsigned long long)full_sort_max());
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  TRY(stage_round1(h, d_xs, d_ys, (uint32_t)n, 1, nullptr, /*ordered=*/true));
  TRY(sync_counters(h));
  *n_out = h->h_ctr->n1;
  CU(cudaMemcpyAsync(d_out, h->surv, (size_t)h->h_ctr->n1 * 4, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

int gscan_stage_sorted(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       uint32_t* d_out, uint64_t* len) {
  if (!h || !d_out || !len) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  if (h->large) return fail(h, GSCAN_E_TOO_LARGE, "stage entry points need n <= %llu", (unsigned long long)full_sort_max());
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  TRY(stage_round1(h, d_xs, d_ys, (uint32_t)n, 0));
  TRY(stage_annotate_sort(h, d_xs, d_ys, (uint32_t)n, -1, -1));
  const uint32_t m = h->h_ctr->m_total;
  *len = m;
  CU(cudaMemcpyAsync(d_out, h->A_i, (size_t)m * 4, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

int gscan_stage_discard(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                        uint64_t chunk_count, int chunked, uint8_t* d_flags, uint64_t* longest,
                        uint64_t* len) {
  if (!h || !d_flags || !longest || !len) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  c.chunk_count = chunk_count;
  c.chunked = chunked;
  c.enable_round1 = 0;
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  if (h->large) return fail(h, GSCAN_E_TOO_LARGE, "stage entry points need n <= %llu", (unsigned long long)full_sort_max());
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  TRY(stage_round1(h, d_xs, d_ys, (uint32_t)n, 0));
  TRY(stage_annotate_sort(h, d_xs, d_ys, (uint32_t)n, -1, -1));
  const uint32_t m = h->h_ctr->m_total;
  if (m < 2) return fail(h, GSCAN_E_INVALID, "split_regions: need at least 2 annotated points");
  double *Rx, *Ry;
  uint32_t* Ri;
  TRY(stage_round2(h, c, &Rx, &Ry, &Ri));
  CU(cudaMemcpyAsync(d_flags, h->flags, m, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  *longest = h->h_ctr->longest;
  *len = m;
  return GSCAN_OK;
}

int gscan_shard_extremes(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         gscan_extremes* out) {
  if (!h || !out) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  const bool vec = aligned16(d_xs) && aligned16(d_ys);
  const uint32_t nn = (uint32_t)n;
  const uint32_t grid =
      std::max(1u, std::min<uint32_t>((nn + kBlock * 8 - 1) / (kBlock * 8), h->sm_count * 8));
  {
    Launch L(h, "k_extremes");
    if (vec) k_extremes<true><<<grid, kBlock, 0, h->stream>>>(d_xs, d_ys, nn, h->partials, h->ext, h->ctr);
    else k_extremes<false><<<grid, kBlock, 0, h->stream>>>(d_xs, d_ys, nn, h->partials, h->ext, h->ctr);
  }
  ExtResult r;
  CU(cudaMemcpyAsync(&r, h->ext, sizeof r, cudaMemcpyDeviceToHost, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  for (int k = 0; k < 4; ++k) { out->idx[k] = r.idx[k]; out->x[k] = r.qx[k]; out->y[k] = r.qy[k]; }
  out->idx[4] = r.idx[4];
  out->x[4] = r.ax;
  out->y[4] = r.ay;
  return GSCAN_OK;
}

// ---- distributed sample sort (the survivor fallback of the sharded path) ----
// Exact sort keys (angular.hpp: atan2 of the vector from the global anchor;
// kKeyDrop for points equal to the anchor) of a list of this shard's points.
__global__ void k_dist_keys(const double* __restrict__ xs, const double* __restrict__ ys,
                            const uint32_t* __restrict__ idx, uint32_t m, double ax, double ay,
                            uint64_t* __restrict__ keys) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
    const uint32_t i = idx[j];
    const double x = xs[i], y = ys[i];
    uint64_t key = kKeyDrop;
    if (!(x == ax && y == ay)) {
      const double a = glibc_atan2(__dsub_rn(y, ay), __dsub_rn(x, ax));
      key = (a == 0.0) ? 0ull : dbits(a);
    }
    keys[j] = key;
  }
}

__global__ void k_sp_set_u32_host(uint32_t* __restrict__ p, uint32_t v) { *p = v; }
__global__ void k_iota(uint32_t* __restrict__ a, uint32_t m) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) a[j] = j;
}

int gscan_shard_keys(gscan_handle* h, const double* d_xs, const double* d_ys, const uint32_t* d_idx,
                     uint64_t m, const gscan_extremes* global, uint64_t* d_keys) {
  if (!h || !global || (m && (!d_xs || !d_ys || !d_idx || !d_keys))) return GSCAN_E_INVALID;
  if (m >= 0xffffffffull) return fail(h, GSCAN_E_TOO_LARGE, "m = %llu exceeds 2^32-2", (unsigned long long)m);
  CU(cudaSetDevice(h->device));
  if (m) {
    const uint32_t grid = std::max(1u, std::min<uint32_t>((uint32_t)((m + 255) / 256), h->sm_count * 8));
    Launch L(h, "k_dist_keys");
    k_dist_keys<<<grid, 256, 0, h->stream>>>(d_xs, d_ys, d_idx, (uint32_t)m, global->x[4], global->y[4],
                                             d_keys);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

// Round 2 and Graham over an annotated buffer that is already sorted and
// deduplicated (position 0 = the anchor): the last step of the distributed
// sample sort on rank 0. *d_out: hull as buffer positions.
int gscan_hull_sorted(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t M,
                      const gscan_config* cfg, uint32_t* d_out, uint64_t out_cap, uint64_t* hull_n,
                      uint64_t* n2) {
  if (!h || !cfg || !d_X || !d_Y || !d_out || !hull_n || !n2 || M == 0) return GSCAN_E_INVALID;
  TRY(validate(h, M, *cfg));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, M));
  if (h->large) return fail(h, GSCAN_E_TOO_LARGE, "sorted buffers above %llu points", (unsigned long long)full_sort_max());
  const uint32_t m = (uint32_t)M;
  cudaStream_t s = h->stream;
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), s));
  CU(cudaMemcpyAsync(h->A_x, d_X, (size_t)m * 8, cudaMemcpyDeviceToDevice, s));
  CU(cudaMemcpyAsync(h->A_y, d_Y, (size_t)m * 8, cudaMemcpyDeviceToDevice, s));
  const uint32_t grid = std::max(1u, std::min<uint32_t>((m + kBlock - 1) / kBlock, h->sm_count * 8));
  k_iota<<<grid, kBlock, 0, s>>>(h->A_i, m);
  k_sp_set_u32_host<<<1, 1, 0, s>>>(&h->ctr->m_total, m);
  // split_regions (angular.hpp:197-204): the first position of the largest dist2
  CU(cudaMemsetAsync(h->scratch64, 0, 8, s));
  CU(cudaMemsetAsync(h->scratch64 + 1, 0xff, 8, s));
  k_longest_scan<<<grid, kBlock, 0, s>>>(h->A_x, h->A_y, m, h->scratch64,
                                         reinterpret_cast<uint32_t*>(h->scratch64 + 1), 0);
  k_longest_scan<<<grid, kBlock, 0, s>>>(h->A_x, h->A_y, m, h->scratch64,
                                         reinterpret_cast<uint32_t*>(h->scratch64 + 1), 1);
  CU(cudaMemcpyAsync(&h->ctr->longest, h->scratch64 + 1, 4, cudaMemcpyDeviceToDevice, s));
  CU(cudaGetLastError());
  TRY(sync_counters(h));
  if (m < 2) CU(cudaMemsetAsync(&h->ctr->longest, 0, 4, s));
  double *Rx, *Ry;
  uint32_t* Ri;
  TRY(stage_round2(h, *cfg, &Rx, &Ry, &Ri));
  TRY(sync_counters(h));
  TRY(stage_graham(h, Rx, Ry, Ri, h->h_ctr->n2));
  TRY(sync_counters(h));
  const uint32_t hull = h->h_ctr->hull;
  *n2 = h->h_ctr->n2;
  *hull_n = hull;
  if (hull > out_cap) return fail(h, GSCAN_E_CAPACITY, "hull of %u vertices exceeds out_cap", hull);
  CU(cudaMemcpyAsync(d_out, h->d_out, (size_t)hull * 4, cudaMemcpyDeviceToDevice, s));
  CU(cudaStreamSynchronize(s));
  return GSCAN_OK;
}

int gscan_shard_round1(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       const gscan_extremes* global, uint32_t* d_out, uint64_t* n_out) {
  if (!h || !global || !d_out || !n_out) return GSCAN_E_INVALID;
  gscan_config c;
  gscan_config_default(&c);
  TRY(validate(h, n, c));
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  CU(cudaMemsetAsync(h->ctr, 0, sizeof(Counters), h->stream));
  ExtResult q{};
  for (int k = 0; k < 4; ++k) { q.idx[k] = 0; q.qx[k] = global->x[k]; q.qy[k] = global->y[k]; }
  q.ax = global->x[4];
  q.ay = global->y[4];
  TRY(stage_round1(h, d_xs, d_ys, (uint32_t)n, 1, &q, /*ordered=*/true));
  TRY(sync_counters(h));
  *n_out = h->h_ctr->n1;
  if (*n_out)
    CU(cudaMemcpyAsync(d_out, h->surv, (size_t)*n_out * 4, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

// ---- device-side data plane: enqueue-only phases (include/gscan.h) ----
// Nothing below waits for the device; the caller runs the collectives on
// the handle's stream between the phases and reads sizes back only where a
// variable-size exchange needs them.

int gscan_dist_enq_begin(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         uint64_t offset, const gscan_config* cfg) {
  if (!h || !cfg) return GSCAN_E_INVALID;
  TRY(validate(h, n, *cfg));
  if (offset + n >= 0xffffffffull) return fail(h, GSCAN_E_TOO_LARGE, "global index beyond 2^32-2");
  CU(cudaSetDevice(h->device));
  TRY(reserve(h, n));
  TRY(sparse_init(h));
  TRY(dist_init(h));
  h->h_sp->M = 0;
  const uint64_t nslices = 2 * std::min<uint64_t>(cfg->chunk_count, n);
  if (nslices + 2 > h->sp_seg_cap) {
    dfree(h->sp_seglo);
    dfree(h->sp_seghi);
    CU(cudaMalloc(&h->sp_seglo, (nslices + 2) * 4));
    CU(cudaMalloc(&h->sp_seghi, (nslices + 2) * 4));
    h->sp_seg_cap = nslices + 2;
    h->sp_graph_ok = false;
  }
  h->dist_xs = d_xs;
  h->dist_ys = d_ys;
  h->dist_n = (uint32_t)n;
  h->dist_base = (uint32_t)offset;
  h->dist_chunks = cfg->chunk_count;
  const SpCtx c = dist_ctx(h);
  TRY(sp_seg_init(h, c));
  TRY(sp_seg_extremes(h, c));
  k_dist_rec_ext<<<1, 32, 0, c.s>>>(h->ext, c.base, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_buffers(gscan_handle* h, gscan_dist_bufs* b) {
  if (!h || !b) return GSCAN_E_INVALID;
  if (!h->dist_rec) return fail(h, GSCAN_E_INVALID, "gscan_dist_buffers before gscan_dist_enq_begin");
  b->rec = h->dist_rec;
  b->recs = h->dist_recs;
  b->ext = h->dist_ext;
  b->cells = h->sp_cells;
  b->hist = h->sp_hist;
  b->phimax = h->sp_phimax;
  b->pref = h->dist_pref;
  b->part_counts = h->dist_pc;
  b->parted = h->sp_dup2;
  b->rlo = h->sp_rlo;
  b->rx = h->A_x;
  b->ry = h->A_y;
  b->stream = h->stream;
  b->rec_len = kDistRecLen;
  b->max_ranks = kDistMaxRanks;
  b->buckets = kSpBuckets;
  b->cells_n = kSpCells;
  b->parts = kSpParts;
  return GSCAN_OK;
}

int gscan_dist_enq_sample(gscan_handle* h, uint32_t R) {
  if (!h || R == 0 || R > kDistMaxRanks || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  k_dist_apply_ext<<<1, 32, 0, c.s>>>(h->dist_recs, R, h->ext, h->dist_ext);
  TRY(sp_seg_sample(h, c));
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_f2(gscan_handle* h) {
  if (!h || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  TRY(sp_seg_f2(h, c));
  k_dist_rec_f2<<<1, 32, 0, c.s>>>(h->sp_st, h->ctr, c.base, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_plan(gscan_handle* h, uint32_t R, uint64_t n_global) {
  if (!h || R == 0 || R > kDistMaxRanks || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  k_dist_apply_best<<<1, 32, 0, c.s>>>(h->dist_recs, R, n_global, h->sp_st);
  TRY(sp_seg_plan(h, c));
  k_dist_rec_plan<<<1, 32, 0, c.s>>>(h->sp_st, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_f3(gscan_handle* h, uint32_t R) {
  if (!h || R == 0 || R > kDistMaxRanks || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  k_dist_apply_plan<<<1, 32, 0, c.s>>>(h->dist_recs, R, h->sp_st);
  TRY(sp_seg_f3(h, c));
  k_dist_rec_f3<<<1, 32, 0, c.s>>>(h->sp_st, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_dup_local(gscan_handle* h, uint32_t R) {
  if (!h || R == 0 || R > kDistMaxRanks || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  const uint32_t nl = 2 * c.G;
  k_dist_apply_f3<<<1, 32, 0, c.s>>>(h->dist_recs, R, h->sp_st);
  TRY(scan_u32(h, h->sp_part_off, kSpParts * nl, h->sp_part_off));
  CU(cudaMemsetAsync(h->sp_side_work, 0, 2 * sizeof(uint32_t), c.s));
  k_sp_dup_part<false><<<h->sm_count, 1024, kSpSideSmem, c.s>>>(h->sp_dup, h->sp_hcount, c.cap / 2, nl,
                                                        h->sp_part_off, h->sp_st, h->sp_dup2,
                                                        h->sp_side_work, 0u, nullptr);
  k_dist_part_totals<<<(kSpParts + 255) / 256, 256, 0, c.s>>>(h->sp_part_off, nl, h->dist_pc);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_dup_check(gscan_handle* h, const uint64_t* d_recv, uint64_t n_recv,
                             const uint32_t* d_counts, uint32_t R) {
  if (!h || !d_counts || R == 0 || R > kDistMaxRanks || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  if (n_recv > (uint64_t)h->sp_grid * sparse_region_cap(h, h->dist_n)) {
    // more hashes than this rank's regions hold (uneven shards): a decline
    // every rank learns from the next record exchange
    k_dist_set_fail<<<1, 32, 0, c.s>>>(h->sp_st, kSpFailCap, 13u);
    return GSCAN_OK;
  }
  k_sp_recv_plan<<<(kSpParts * R + 255) / 256, 256, 0, c.s>>>(d_counts, R, h->dist_pm, h->dist_hc,
                                                               h->dist_lb);
  TRY(scan_u32(h, h->dist_pm, kSpParts * R, h->dist_pm));
  CU(cudaMemsetAsync(h->sp_side_work, 0, 2 * sizeof(uint32_t), c.s));
  k_sp_dup_part<false><<<h->sm_count, 1024, kSpSideSmem, c.s>>>(d_recv, h->dist_hc, 0u, R, h->dist_pm,
                                                        h->sp_st, h->sp_dup, h->sp_side_work, 0u,
                                                        h->dist_lb);
  k_sp_dups<<<h->sm_count, 1024, kSpSideSmem, c.s>>>(h->sp_dup, h->dist_pm, R, h->sp_st,
                                                     h->sp_side_work + 1, 0u, h->sp_dup_scr,
                                                     h->sp_dup_scap);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_export(gscan_handle* h, int candidates, double* d_x, double* d_y, uint32_t* d_idx,
                          uint32_t* d_b) {
  if (!h || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  CU(cudaMemsetAsync(h->dist_ctr, 0, 4, c.s));
  Launch L(h, "k_sp_export", c.s);
  k_sp_export<<<dim3(8, c.G), 256, 0, c.s>>>(c.xs, c.ys, h->surv, h->sp_eb,
                                             candidates ? h->sp_ccount : h->sp_gcount, c.cap, c.base,
                                             h->sp_st, d_x, d_y, d_idx, d_b, h->dist_ctr);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_slices(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t n_g,
                          const uint32_t* d_gb, const int64_t* d_gidx, uint64_t M) {
  if (!h || !d_X || !d_Y || !h->dist_rec) return GSCAN_E_INVALID;
  h->h_sp->M = (uint32_t)M;  // the global slice structure sizes rank 0's grids
  SpCtx c = dist_ctx(h);
  if (1 + n_g + 2 > std::min<uint64_t>(h->cap, h->wcap))
    return fail(h, GSCAN_E_CAPACITY, "sharded path: %llu gathered points exceed rank 0's buffers",
                (unsigned long long)n_g);
  TRY(dist_slices_ensure(h, c));
  k_dist_find_pl<<<1, 32, 0, c.s>>>(d_gidx, (uint32_t)n_g, h->sp_st, h->ext);
  k_sp_gsize<<<(kSpBuckets + 255) / 256, 256, 0, c.s>>>(h->sp_gbits, h->sp_hist, h->sp_gsz);
  TRY(scan_u32(h, h->sp_gsz, kSpBuckets, h->sp_gs));
  TRY(dist_fill(h, c, (uint32_t)n_g, 1, d_gb, h->sp_gcount));
  c.gs = h->sp_gs;
  TRY(sp_seg_sortg(h, c, d_X, d_Y, /*region_xy=*/false));
  k_dist_pref_out<<<(kSpBuckets + 256) / 256, 256, 0, c.s>>>(h->sp_prefmax, h->sp_st, h->dist_pref);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_dist_enq_cand(gscan_handle* h) {
  if (!h || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  k_dist_pref_in<<<(kSpBuckets + 255) / 256, 256, 0, c.s>>>(h->dist_pref, h->sp_prefmax, h->sp_st);
  TRY(sp_seg_f4(h, c));
  k_dist_rec_f4<<<1, 32, 0, c.s>>>(h->sp_st, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

// Rank 0: walk, certificate and Graham (synchronises). *status: 0 the hull
// is final, 1 the certificate did not hold (every rank runs F6 on its shard:
// gscan_dist_enq_verify), 2 declined (fail bits in *fail_out).
int gscan_dist_root_finish(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t n_g,
                           uint64_t n_c, const uint32_t* d_cb, uint64_t M, uint32_t* d_hull,
                           uint64_t hull_cap, uint64_t* hull_n, uint64_t* n_r, uint32_t* status,
                           uint32_t* fail_out) {
  if (!h || !d_X || !d_Y || !d_hull || !hull_n || !n_r || !status || !fail_out || !h->dist_rec)
    return GSCAN_E_INVALID;
  h->h_sp->M = (uint32_t)M;
  SpCtx c = dist_ctx(h);
  c.gs = h->sp_gs;
  *status = 2;
  *hull_n = 0;
  *n_r = 0;
  const uint64_t nw = 1 + n_g + n_c;
  if (nw + 2 > std::min<uint64_t>(h->cap, h->wcap))
    return fail(h, GSCAN_E_CAPACITY, "sharded path: %llu walk records exceed rank 0's buffers",
                (unsigned long long)nw);
  TRY(dist_slices_ensure(h, c));
  TRY(dist_fill(h, c, (uint32_t)n_c, (uint32_t)(1 + n_g), d_cb, h->sp_ccount));
  TRY(tree_workspace(h, (uint32_t)std::min<uint64_t>(nw, kTreeMaxN)));
  TRY(sp_seg_walk(h, c, d_X, d_Y, (uint32_t)nw));
  h->graham_path = 0;
  h->graham_fails = 0;
  TRY(sp_seg_tail(h, c));
  TRY(sync_counters(h));
  const SpState sp = *h->h_sp;
  *fail_out = dist_fail(h);
  *n_r = sp.n_r;
  if (sp.fail) return GSCAN_OK;
  bool done = false;
  TRY(tree_finish(h, h->A_x, h->A_y, h->A_i, &done));
  if (!done) {
    TRY(stage_graham(h, h->A_x, h->A_y, h->A_i, sp.n_r, /*skip_tree=*/true));
    TRY(sync_counters(h));
  }
  const uint32_t hull = h->h_ctr->hull;
  if (hull > hull_cap) return fail(h, GSCAN_E_CAPACITY, "hull of %u vertices exceeds out_cap", hull);
  CU(cudaMemcpyAsync(d_hull, h->d_out, (size_t)hull * 4, cudaMemcpyDeviceToDevice, h->stream));
  CU(cudaStreamSynchronize(h->stream));
  *hull_n = hull;
  *status = sp.need_verify ? 1u : 0u;
  return GSCAN_OK;
}

int gscan_dist_enq_verify(gscan_handle* h, const uint32_t* d_rlo, const double* d_Rx,
                          const double* d_Ry) {
  if (!h || !d_rlo || !d_Rx || !d_Ry || !h->dist_rec) return GSCAN_E_INVALID;
  const SpCtx c = dist_ctx(h);
  if (d_rlo != h->sp_rlo)
    CU(cudaMemcpyAsync(h->sp_rlo, d_rlo, (kSpBuckets + 1) * 4, cudaMemcpyDeviceToDevice, c.s));
  k_dist_verify_prep<<<1, 32, 0, c.s>>>(h->sp_st);
  {
    Launch L(h, "k_sp_verify", c.s);
#define A6 c.xs, c.ys, h->sp_codes, c.n, h->sp_gbits, h->sp_rlo, d_Rx, d_Ry, h->sp_st
    if (c.vec) k_sp_verify<true><<<c.G, kSpThreads, c.smem_nb + 4, c.s>>>(A6);
    else k_sp_verify<false><<<c.G, kSpThreads, c.smem_nb + 4, c.s>>>(A6);
#undef A6
  }
  k_dist_rec_ver<<<1, 32, 0, c.s>>>(h->sp_st, h->dist_rec);
  CU(cudaGetLastError());
  return GSCAN_OK;
}

int gscan_generate_square_device(gscan_handle* h, uint64_t seed, uint64_t lo, uint64_t hi,
                                 double* d_xs, double* d_ys) {
  if (!h || hi < lo || ((!d_xs || !d_ys) && hi > lo)) return GSCAN_E_INVALID;
  if (hi == lo) return GSCAN_OK;
  if (hi > (1ull << 40)) return fail(h, GSCAN_E_TOO_LARGE, "generator range above 2^40 points");
  CU(cudaSetDevice(h->device));
  const uint64_t P = (2 * hi - 1) / kMtL + 1;  // generators 0 .. P-1 (states of all of them)
  int nb = 0;
  while ((1ull << nb) < P) ++nb;
  const int nbt = std::max(nb, 1);
  if (nbt > h->mt_jtab_nb) {
    const std::vector<uint64_t>& tab = mt64::jump_table(kMtL, nbt);
    if (h->mt_jtab) CU(cudaFree(h->mt_jtab));
    h->mt_jtab = nullptr;
    CU(cudaMalloc(&h->mt_jtab, tab.size() * 8));
    CU(cudaMemcpy(h->mt_jtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));
    h->mt_jtab_nb = nbt;
  }
  if (P > h->mt_states_cap) {
    if (h->mt_states) CU(cudaFree(h->mt_states));
    h->mt_states = nullptr;
    CU(cudaMalloc(&h->mt_states, P * kMtN * 8));
    h->mt_states_cap = P;
  }
  static std::once_flag attr;
  std::call_once(attr, [] {
    cudaFuncSetAttribute(k_mt_jump, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMtJumpSmem);
  });
  uint64_t st0[kMtN];
  mt64::seed_state(seed, st0);
  CU(cudaMemcpyAsync(h->mt_states, st0, sizeof(st0), cudaMemcpyHostToDevice, h->stream));
  for (int b = 0; b < nb; ++b) {
    const uint64_t half = 1ull << b;
    const uint64_t count = std::min(half, P - half);
    Launch L(h, "k_mt_jump");
    k_mt_jump<<<(uint32_t)count, kMtThreads, kMtJumpSmem, h->stream>>>(
        h->mt_states, (uint32_t)half, (uint32_t)count, h->mt_jtab + (size_t)b * kMtWords);
  }
  const uint64_t g0 = (2 * lo) / kMtL;
  {
    Launch L(h, "k_mt_gen");
    k_mt_gen<<<(uint32_t)(P - g0), kMtThreads, 0, h->stream>>>(h->mt_states, g0, lo, hi, d_xs, d_ys);
  }
  CU(cudaGetLastError());
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

int gscan_device_atan2(gscan_handle* h, const double* d_y, const double* d_x, double* d_out,
                       uint64_t n) {
  if (!h || !d_y || !d_x || !d_out) return GSCAN_E_INVALID;
  CU(cudaSetDevice(h->device));
  if (n) {
    const uint32_t grid = (uint32_t)std::min<uint64_t>((n + kBlock - 1) / kBlock, h->sm_count * 16);
    k_atan2<<<grid, kBlock, 0, h->stream>>>(d_y, d_x, d_out, n);
    CU(cudaGetLastError());
  }
  CU(cudaStreamSynchronize(h->stream));
  return GSCAN_OK;
}

}  // extern "C"
