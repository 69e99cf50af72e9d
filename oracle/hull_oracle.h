/* TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the gScan hull path.
 *
 * Plain-C restatement of hull2d::full_pipeline
 * (/root/reference/proj/include/hull2d/pipeline.hpp:72-123) that tracks the
 * input index of every point so the hull comes back as the north-star index
 * list. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it; the product path never does.
 *
 * Parity is pinned two ways: against the golden
 * vectors in tests/golden/ generated from the reference itself
 * (oracle/_ref/libhull2d_ref.so, built from /root/reference headers), and
 * against that library directly whenever it is present.
 */
#ifndef GSCAN_HULL_ORACLE_H
#define GSCAN_HULL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PipelineConfig (pipeline.hpp:41-46). */
typedef struct oc_config {
    uint64_t chunk_count;  /* default 1024 */
    int32_t enable_round1; /* default 1 */
    int32_t enable_round2; /* default 1 */
    int32_t chunked;       /* default 1; 0 = discard_sequential */
    int32_t reserved;
} oc_config;

/* StageStats (pipeline.hpp:28-39). */
typedef struct oc_stats {
    uint64_t n_input, n_after_round1, n_after_round2, hull_size;
    double t_round1_ms, t_annotate_ms, t_sort_ms, t_round2_ms, t_finalize_ms, t_total_ms;
} oc_stats;

/* Optional stage dumps; any pointer may be NULL. Arrays must hold n entries. */
typedef struct oc_trace {
    uint64_t quad[4];     /* ExtremeQuad (input indices; valid iff round 1 on) */
    uint64_t anchor;      /* input index of the anchor */
    uint64_t *r1_idx;     /* round-1 survivors, input order */
    uint64_t *sorted_idx; /* annotated + angle-sorted buffer (pos 0 = anchor) */
    uint64_t sorted_len;
    uint64_t longest;     /* split_regions().longest, 0 if round 2 skipped */
    uint8_t *r2_flags;    /* discard flags over the sorted buffer */
    uint64_t *r2_idx;     /* buffer after round 2 */
} oc_trace;

enum { OC_OK = 0, OC_E_EMPTY_INPUT = 1, OC_E_ZERO_CHUNKS = 2, OC_E_CAPACITY = 3, OC_E_NOMEM = 4 };

void oc_config_default(oc_config *cfg);

/* full_pipeline over SoA input; out_idx receives the CCW hull as input
 * indices (first occurrence of each vertex), starting at the anchor. */
int oc_full_pipeline(const double *xs, const double *ys, uint64_t n, const oc_config *cfg,
                     uint64_t *out_idx, uint64_t out_cap, uint64_t *out_len, oc_stats *stats,
                     oc_trace *trace);

/* Stage functions for stage-level parity. */
int oc_find_extremes(const double *xs, const double *ys, uint64_t n, uint64_t quad[4]);
uint64_t oc_select_anchor(const double *xs, const double *ys, uint64_t n);
void oc_classify_quad(const double *xs, const double *ys, uint64_t n, const uint64_t quad[4],
                      uint8_t *flags);
/* Orientation predicate (geom.hpp:26-31): +1 Left, -1 Right, 0 Collinear. */
int oc_orient(double ax, double ay, double bx, double by, double cx, double cy);
/* polar_key angle (geom.hpp:38-43) via the host libm. */
double oc_atan2(double y, double x);
void oc_atan2_array(const double *y, const double *x, double *out, uint64_t n);

/* Andrew's monotone chain (oracle.hpp:40-68), as input indices. */
int oc_monotone_chain(const double *xs, const double *ys, uint64_t n, uint64_t *out_idx,
                      uint64_t out_cap, uint64_t *out_len);

#ifdef __cplusplus
}
#endif
#endif
