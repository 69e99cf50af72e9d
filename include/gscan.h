/* gscan.h -- C-ABI of the B200-native gScan 2D convex hull path.
 *
 * Drop-in boundary for the reference's hot path
 *   hull2d::full_pipeline(std::span<const Point2>, const PipelineConfig&) -> PipelineResult
 *   (/root/reference/proj/include/hull2d/pipeline.hpp:72-123)
 * re-expressed as the north-star entry `hull(xs, ys, n) -> ordered hull vertex
 * indices`. The reference is a header-only C++20 library with no exported
 * symbols, so these entry points are what its FFI (a ctypes/cffi/JNI/cgo
 * binding) would bind. Plain pointers and sizes only.
 *
 * Output semantics (pipeline.hpp:19-26): the CCW sequence of strict hull
 * vertices starting at the anchor (lowest point: min y, then min x),
 * collinear boundary points excluded, one vertex for a single distinct point,
 * two for a collinear set. Each vertex is reported as the index of its FIRST
 * occurrence in the input (the reference deduplicates keeping the first
 * occurrence, angular.hpp:115-133, and compacts stably, prefilter.hpp:65-76).
 * Results are bit-identical to the reference on the same input.
 *
 * Errors (errors.hpp:9-49 -> status codes): EmptyInput (pipeline.hpp:73) ->
 * GSCAN_E_EMPTY_INPUT, ZeroChunks (pipeline.hpp:74) -> GSCAN_E_ZERO_CHUNKS.
 * Non-finite coordinates are a precondition violation, as in the reference
 * (SPEC.md:330), and are not checked.
 *
 * Threading: calls on distinct handles are independent; calls on one handle
 * are serialised by the caller. The library owns device scratch per handle and
 * does not allocate per call once a handle has seen its largest n.
 */
#ifndef GSCAN_H
#define GSCAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GSCAN_ABI_VERSION 1

/* Status codes. */
enum {
    GSCAN_OK = 0,
    GSCAN_E_EMPTY_INPUT = 1, /* hull2d::EmptyInput  (pipeline.hpp:73) */
    GSCAN_E_ZERO_CHUNKS = 2, /* hull2d::ZeroChunks  (pipeline.hpp:74) */
    GSCAN_E_CAPACITY = 3,    /* out_cap < hull size; *out_len holds the size needed */
    GSCAN_E_CUDA = 4,        /* CUDA runtime failure (gscan_last_error has text) */
    GSCAN_E_INVALID = 5,     /* NULL pointer / bad argument */
    GSCAN_E_TOO_LARGE = 6,   /* n >= 2^32 (indices are 32-bit on the device) */
    GSCAN_E_NO_DEVICE = 7,   /* no CUDA device / extension built without GPU */
    GSCAN_E_INTERNAL = 8,    /* device-side consistency check failed */
    GSCAN_E_IO = 9,          /* hull2d::IoError (datagen.hpp: cannot open / read) */
    GSCAN_E_PARSE = 10,      /* hull2d::ParseError (datagen.hpp; line in gscan_io_error) */
    GSCAN_E_NCCL = 11        /* a collective of the sharded path failed (distributed.py) */
};

/* hull2d::PipelineConfig (pipeline.hpp:41-46). */
typedef struct gscan_config {
    uint64_t chunk_count;  /* slices per region in round 2; default 1024 */
    int32_t enable_round1; /* quadrilateral pretest; default 1 */
    int32_t enable_round2; /* sorted-region discard; default 1 */
    int32_t chunked;       /* 1: discard_chunked (default); 0: discard_sequential */
    int32_t reserved;      /* must be 0 */
} gscan_config;

/* hull2d::StageStats (pipeline.hpp:28-39). Times are device time measured
 * with CUDA events on the call's stream, per reference stage. */
typedef struct gscan_stats {
    uint64_t n_input;
    uint64_t n_after_round1; /* pre-dedup survivors of round 1 (pipeline.hpp:93) */
    uint64_t n_after_round2; /* post-dedup, post-round-2 buffer (pipeline.hpp:109) */
    uint64_t hull_size;
    double t_round1_ms;
    double t_annotate_ms;
    double t_sort_ms;
    double t_round2_ms;
    double t_finalize_ms;
    double t_total_ms;
} gscan_stats;

typedef struct gscan_handle gscan_handle;

/* Fills the reference defaults (chunk_count 1024, both rounds, chunked). */
void gscan_config_default(gscan_config* cfg);

/* Handle lifetime. device < 0 selects the current device. */
int gscan_create(int device, gscan_handle** out);
int gscan_destroy(gscan_handle* h);
/* Pre-allocates device scratch for inputs of up to n points. */
int gscan_reserve(gscan_handle* h, uint64_t n);
/* Uses `stream` (a cudaStream_t; NULL = the handle's own stream) for later calls. */
int gscan_set_stream(gscan_handle* h, void* stream);

/* Host-buffer entry: copies xs/ys (n doubles each) to the device, runs the
 * pipeline, copies the index list back. cfg may be NULL (defaults); stats may
 * be NULL. On GSCAN_E_CAPACITY nothing is written to out_idx. */
int gscan_hull_f64(gscan_handle* h, const double* xs, const double* ys, uint64_t n,
                   const gscan_config* cfg, uint64_t* out_idx, uint64_t out_cap,
                   uint64_t* out_len, gscan_stats* stats);

/* Device-buffer entry: d_xs/d_ys are device pointers; the index list is left
 * in d_out_idx (device, uint32). Synchronises the handle's stream before
 * returning (hull size is needed on the host). */
int gscan_hull_f64_device(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                          const gscan_config* cfg, uint32_t* d_out_idx, uint64_t out_cap,
                          uint64_t* out_len, gscan_stats* stats);

/* North-star convenience entry: hull(xs, ys, n) with a lazily created
 * per-process handle on the current device and the default config. */
int gscan_hull(const double* xs, const double* ys, uint64_t n, uint64_t* out_idx,
               uint64_t out_cap, uint64_t* out_len);

/* ---- stage entry points (device pointers), for stage-level parity ---- */

/* find_extremes (prefilter.hpp:28-39) + select_anchor on all points
 * (angular.hpp:40-49): out[0..3] = i_minx, i_miny, i_maxx, i_maxy; out[4] = anchor. */
int gscan_stage_extremes(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         uint64_t out[5]);
/* classify_quad + compact (prefilter.hpp:47-76): survivor input indices in
 * input order into d_out (device uint32, capacity n); *n_out = count. */
int gscan_stage_round1(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       uint32_t* d_out, uint64_t* n_out);
/* annotate + sort_by_angle (angular.hpp:118-194) of ALL n points (round 1
 * skipped): buffer entries as input indices into d_out (device uint32,
 * capacity n); *len = buffer size. */
int gscan_stage_sorted(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       uint32_t* d_out, uint64_t* len);
/* split_regions + discard flags (discard.hpp:79-124) over the sorted buffer of
 * all n points (round 1 skipped): d_flags (device uint8, capacity n) gets one
 * keep flag per buffer entry; *longest = split index. */
int gscan_stage_discard(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                        uint64_t chunk_count, int chunked, uint8_t* d_flags, uint64_t* longest,
                        uint64_t* len);

/* ---- sharded (multi-GPU) building blocks ---- */

/* The five extreme points of a shard: idx[] are indices into the shard
 * (add the shard offset for global ones), x[]/y[] their coordinates;
 * order i_minx, i_miny, i_maxx, i_maxy, lowest (min y, then min x). */
typedef struct gscan_extremes {
    uint64_t idx[5];
    double x[5];
    double y[5];
} gscan_extremes;

/* find_extremes + lowest point of one shard (device pointers). */
int gscan_shard_extremes(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         gscan_extremes* out);
/* classify_quad + compact of one shard against the GLOBAL quadrilateral
 * (prefilter.hpp:47-76): survivors' shard-local indices, in order, into d_out
 * (device uint32, capacity n); *n_out = count. Only global->x/y[0..3] are read. */
int gscan_shard_round1(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                       const gscan_extremes* global, uint32_t* d_out, uint64_t* n_out);

/* Distributed sample sort (the sharded path's survivor fallback, SURVEY.md
 * 8e: "a distributed sample sort when the survivor set is large", e.g. points
 * on a circle). Every rank: gscan_shard_round1 -> gscan_shard_keys (the exact
 * sort key of each survivor: atan2 from the global anchor, bits; UINT64_MAX
 * for points equal to the anchor) -> survivors routed by key ranges (sampled
 * splitters; equal keys stay on one rank) -> gscan_stage_sorted on the
 * received points plus the anchor, in global-index order (the bucket sort +
 * dedup) -> sorted runs to rank 0, whose concatenation is the reference's
 * annotated buffer -> rank 0: gscan_hull_sorted (split_regions, round 2,
 * Graham; d_out = hull as buffer positions). */
int gscan_shard_keys(gscan_handle* h, const double* d_xs, const double* d_ys, const uint32_t* d_idx,
                     uint64_t m, const gscan_extremes* global, uint64_t* d_keys);
int gscan_hull_sorted(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t M,
                      const gscan_config* cfg, uint32_t* d_out, uint64_t out_cap, uint64_t* hull_n,
                      uint64_t* n2);

/* ---- sharded sparse path (paper_1508_05931_b200/distributed.py) ----
 *
 * One handle per rank; rank r owns the contiguous shard [offset, offset + n)
 * of the global input (device pointers). The phases are enqueue-only:
 * nothing waits for the device. Each phase
 * writes this rank's scalars into a fixed record (gscan_dist_bufs.rec,
 * rec_len int64 words); the caller all-gathers the records into
 * gscan_dist_bufs.recs (R x rec_len) and runs the fixed-size collectives in
 * place on the handle's buffers, all on the handle's stream (NCCL), and the
 * next phase combines them on the device. The host reads back only the sizes
 * of the variable-size exchanges, at three points per call:
 *   gscan_dist_enq_begin       K1 on the shard            rec -> all-gather
 *   gscan_dist_enq_sample      global extremes; sample    cells -> sum
 *   gscan_dist_enq_f2          F2                         hist -> sum, rec -> all-gather
 *   gscan_dist_enq_plan        global P_l; P_l's rank     rec -> all-gather
 *   gscan_dist_enq_f3          F3                         phimax -> max (as uint32), rec -> all-gather
 *   gscan_dist_enq_dup_local   hashes by partition        counts -> all-to-all
 *   (host sync 1: fail word, gathered counts, hash block sizes)
 *   hashes -> all-to-all; gscan_dist_enq_dup_check; gscan_dist_enq_export(0)
 *   -> rank 0; rank 0: gscan_dist_enq_slices; pref -> broadcast
 *   gscan_dist_enq_cand        F4                         rec -> all-gather
 *   (host sync 2: fail word, candidate counts)
 *   gscan_dist_enq_export(1) -> rank 0; rank 0: gscan_dist_root_finish
 *   (host sync 3: rank 0's status broadcast)
 *   status 1 (certificate not proved): rlo, rx, ry of rank 0 -> broadcast;
 *   gscan_dist_enq_verify on every rank (distributed F6), rec -> all-gather.
 * gscan_dist_buffers is valid after gscan_dist_enq_begin. */
typedef struct gscan_dist_bufs {
    int64_t* rec;           /* this rank's record (rec_len words) */
    int64_t* recs;          /* all ranks' records (max_ranks x rec_len) */
    int64_t* ext;           /* combined extremes: global index (5), x bits (5), y bits (5) */
    uint32_t* cells;        /* sample cells (cells_n) */
    uint32_t* hist;         /* bucket histogram (buckets) */
    uint32_t* phimax;       /* walk-angle maxima, ordered-float encoding (buckets) */
    uint32_t* pref;         /* prefix maxima + rank 0's fail word (buckets + 1) */
    uint32_t* part_counts;  /* hashes per partition (parts) */
    uint64_t* parted;       /* this rank's hashes, partition-major */
    uint32_t* rlo;          /* round-2 output offsets per bucket (buckets + 1; rank 0) */
    double* rx;             /* round-2 output coordinates (rank 0) */
    double* ry;
    void* stream;           /* the handle's cudaStream_t */
    uint64_t rec_len, max_ranks, buckets, cells_n, parts;
} gscan_dist_bufs;

int gscan_dist_enq_begin(gscan_handle* h, const double* d_xs, const double* d_ys, uint64_t n,
                         uint64_t offset, const gscan_config* cfg);
int gscan_dist_buffers(gscan_handle* h, gscan_dist_bufs* bufs);
int gscan_dist_enq_sample(gscan_handle* h, uint32_t R);
int gscan_dist_enq_f2(gscan_handle* h);
int gscan_dist_enq_plan(gscan_handle* h, uint32_t R, uint64_t n_global);
int gscan_dist_enq_f3(gscan_handle* h, uint32_t R);
int gscan_dist_enq_dup_local(gscan_handle* h, uint32_t R);
int gscan_dist_enq_dup_check(gscan_handle* h, const uint64_t* d_recv, uint64_t n_recv,
                             const uint32_t* d_counts, uint32_t R);
int gscan_dist_enq_export(gscan_handle* h, int candidates, double* d_x, double* d_y,
                          uint32_t* d_idx, uint32_t* d_b);
int gscan_dist_enq_slices(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t n_g,
                          const uint32_t* d_gb, const int64_t* d_gidx, uint64_t M);
int gscan_dist_enq_cand(gscan_handle* h);
int gscan_dist_root_finish(gscan_handle* h, const double* d_X, const double* d_Y, uint64_t n_g,
                           uint64_t n_c, const uint32_t* d_cb, uint64_t M, uint32_t* d_hull,
                           uint64_t hull_cap, uint64_t* hull_n, uint64_t* n_r, uint32_t* status,
                           uint32_t* fail_out);
int gscan_dist_enq_verify(gscan_handle* h, const uint32_t* d_rlo, const double* d_Rx,
                          const double* d_Ry);

/* ---- device self-checks ---- */

/* glibc-identical atan2 (paper_1508_05931_b200/csrc/glibc_atan2.h) on the
 * device: out[i] = atan2(y[i], x[i]); device pointers. */
int gscan_device_atan2(gscan_handle* h, const double* d_y, const double* d_x, double* d_out,
                       uint64_t n);

/* ---- introspection ---- */
const char* gscan_status_string(int status);
const char* gscan_last_error(const gscan_handle* h);
/* Number of kernels the handle launched in its last pipeline call. */
uint64_t gscan_last_launch_count(const gscan_handle* h);
/* Per-kernel event timing of the last call (ms), `names` entries, in launch
 * order; returns the number of records (<= cap). Requires gscan_set_profiling. */
int gscan_set_profiling(gscan_handle* h, int enabled);
int gscan_last_kernel_times(const gscan_handle* h, const char** names, double* ms, int cap);

/* ---- test hooks (exercise the certificate and fallback paths) ---- */
enum {
    GSCAN_DEBUG_FORCE_JUNCTION = 1u << 0,   /* Graham candidate via junction merges */
    GSCAN_DEBUG_FORCE_SEQUENTIAL = 1u << 1, /* Graham candidate via chains-of-chains scan */
    GSCAN_DEBUG_CORRUPT_CANDIDATE = 1u << 2,/* falsify the candidate: certificate must fail */
    GSCAN_DEBUG_FORCE_FALLBACK = 1u << 3,   /* always finish with the sequential kernel */
    GSCAN_DEBUG_FORCE_PREFIX = 1u << 4,     /* Graham candidate via prefix scan of states */
    GSCAN_DEBUG_FULL_SORT = 1u << 5,        /* skip the sparse round-2 path: sort every survivor */
    GSCAN_DEBUG_SPARSE_DROP = 1u << 6,      /* sparse path walks no candidates: its verification
                                               must reject the result and the call falls back */
    GSCAN_DEBUG_SPARSE_VERIFY = 1u << 7     /* sparse path: always run the verification pass,
                                               even when the error-bound certificate holds */
};
int gscan_set_debug(gscan_handle* h, uint32_t flags);
/* path: 0 = sequential kernel only (tiny input), 1 = chain scan + certificate,
 * 2 = junctions + certificate, 3 = prefix-scanned states + certificate,
 * 8 = tree of thread-sequential chain scans + certificate (pop-heavy buffers);
 * bit 4 set = certificate failed or fallback forced. */
int gscan_last_graham_info(const gscan_handle* h, uint32_t* path, uint32_t* certificate_failures);

/* Sparse round-2 path of the last call (the default for n >= 65536 with the
 * default toggles): used = 1 when its result was returned; fail_bits != 0
 * when it declined and the full sort ran instead: 1 tie for the farthest
 * point, 4 a region with <= 1 point, 8 possible duplicates, 16 failed
 * verification, 32 capacity (a gathered or candidate bucket above its
 * sorter's scratch -- 8x the mean bucket of n points -- or with clustered
 * keys; a duplicate-check partition of 2^21 - 1 hashes or more, above ~4G
 * survivors; walk arrays too small in large mode; unfinished side-stream
 * work), 64 internal, 128 too few points, 256 too many
 * walk candidates (near-circular inputs: the full sort is faster);
 * n_walked = points it sorted and walked exactly (gathered + candidates +
 * anchor). */
int gscan_last_sparse_info(const gscan_handle* h, uint32_t* used, uint32_t* fail_bits,
                           uint32_t* n_walked);

/* ---- harness helpers (host) ---- */
enum { GSCAN_GEN_SQUARE = 0, GSCAN_GEN_DISK = 1, GSCAN_GEN_CIRCLE = 2, GSCAN_GEN_COLLINEAR = 3 };
/* datagen::gen_* (datagen.hpp:32-91), bit-identical to the reference. */
int gscan_generate(int kind, uint64_t n, uint64_t seed, double* xs, double* ys);
/* On-device gen_square (datagen.hpp:32-41): points
 * [lo, hi) of the reference's gen_square(n, seed) sequence (any n >= hi),
 * bit-identical to gscan_generate(GSCAN_GEN_SQUARE, ...), written to device
 * arrays d_xs[0 .. hi-lo), d_ys[0 .. hi-lo) on the handle's stream
 * (mt19937_64 jump-ahead + per-generator engines; synchronises the stream).
 * A rank of a sharded run generates only its own shard. */
int gscan_generate_square_device(gscan_handle* h, uint64_t seed, uint64_t lo, uint64_t hi,
                                 double* d_xs, double* d_ys);
/* Ingest. Plain-XY text and the OBJ vertex subset
 * restate hull2d::datagen::load_points / load_obj_projected
 * (datagen.hpp:111-168: std::from_chars, '#'/blank lines skipped, "v x y [z]"
 * vertex lines); GSCANSOA is the device path's binary layout ("GSCANSOA",
 * uint64 n, n doubles x, n doubles y, little-endian). gscan_load returns
 * malloc'd arrays (free with gscan_free); gscan_soa_count + gscan_soa_read
 * fill caller buffers (e.g. pinned memory for gscan_hull_f64). Errors:
 * GSCAN_E_IO, GSCAN_E_PARSE, GSCAN_E_EMPTY_INPUT; the message (with the line
 * number) from gscan_io_error (per thread). */
enum { GSCAN_FMT_XY = 0, GSCAN_FMT_OBJ = 1, GSCAN_FMT_SOA = 2 };
int gscan_load(const char* path, int format, double** xs, double** ys, uint64_t* n);
int gscan_soa_count(const char* path, uint64_t* n);
int gscan_soa_read(const char* path, double* xs, double* ys, uint64_t n);
int gscan_save_soa(const char* path, const double* xs, const double* ys, uint64_t n);
void gscan_free(void* p);
const char* gscan_io_error(void);
/* Host self-check of the generator's mt19937_64 jump-ahead: jumps `blocks`
 * x 2^20 words and compares the next 312 outputs with a sequentially
 * advanced std::mt19937_64. Returns the number of mismatches (0 = exact). */
int gscan_mt64_jump_check(uint64_t seed, uint64_t blocks);
/* tests/support.hpp:54-63 gen_grid. */
int gscan_generate_grid(uint64_t n, uint64_t seed, int lo, int hi, double* xs, double* ys);

#ifdef __cplusplus
}
#endif
#endif /* GSCAN_H */
