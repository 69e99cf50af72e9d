/* TEST INFRASTRUCTURE ONLY -- CPU parity oracle (see hull_oracle.h).
 *
 * A line-by-line *behavioural* restatement of the reference hull pipeline in
 * plain C, carrying input indices. Build with -ffp-contract=off (oracle/Makefile):
 * the reference binary contains no FMA, so neither may this one, or orient()
 * and dist2 round differently.
 */
#define _POSIX_C_SOURCE 199309L
#include "hull_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct { double x, y; } pt;

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec * 1e3 + (double)ts.tv_nsec * 1e-6;
}

void oc_config_default(oc_config *cfg) {
    cfg->chunk_count = 1024;
    cfg->enable_round1 = 1;
    cfg->enable_round2 = 1;
    cfg->chunked = 1;
    cfg->reserved = 0;
}

/* geom.hpp:19-21 cross(); geom.hpp:26-31 orient(). */
static double cross3(pt a, pt b, pt c) {
    return (b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x);
}
enum { LEFT = 1, RIGHT = -1, COLLINEAR = 0 };
static int orient3(pt a, pt b, pt c) {
    const double area = cross3(a, b, c);
    if (area > 0.0) return LEFT;
    if (area < 0.0) return RIGHT;
    return COLLINEAR;
}
int oc_orient(double ax, double ay, double bx, double by, double cx, double cy) {
    pt a = {ax, ay}, b = {bx, by}, c = {cx, cy};
    return orient3(a, b, c);
}
double oc_atan2(double y, double x) { return atan2(y, x); }
void oc_atan2_array(const double *y, const double *x, double *out, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) out[i] = atan2(y[i], x[i]);
}

/* prefilter.hpp:28-39 find_extremes: strict compares, lowest index on ties. */
static void find_extremes_pts(const pt *p, uint64_t n, uint64_t q[4]) {
    q[0] = q[1] = q[2] = q[3] = 0;
    for (uint64_t i = 1; i < n; ++i) {
        if (p[i].x < p[q[0]].x) q[0] = i;
        if (p[i].y < p[q[1]].y) q[1] = i;
        if (p[i].x > p[q[2]].x) q[2] = i;
        if (p[i].y > p[q[3]].y) q[3] = i;
    }
}

int oc_find_extremes(const double *xs, const double *ys, uint64_t n, uint64_t quad[4]) {
    if (n == 0) return OC_E_EMPTY_INPUT;
    quad[0] = quad[1] = quad[2] = quad[3] = 0;
    for (uint64_t i = 1; i < n; ++i) {
        if (xs[i] < xs[quad[0]]) quad[0] = i;
        if (ys[i] < ys[quad[1]]) quad[1] = i;
        if (xs[i] > xs[quad[2]]) quad[2] = i;
        if (ys[i] > ys[quad[3]]) quad[3] = i;
    }
    return OC_OK;
}

/* prefilter.hpp:47-63 classify_quad: 0 iff strictly Left of all four edges
 * minx->miny->maxx->maxy->minx. */
static void classify_pts(const pt *p, uint64_t n, const uint64_t q[4], uint8_t *flags) {
    const pt q0 = p[q[0]], q1 = p[q[1]], q2 = p[q[2]], q3 = p[q[3]];
    for (uint64_t i = 0; i < n; ++i) {
        const pt c = p[i];
        flags[i] = !(orient3(q0, q1, c) == LEFT && orient3(q1, q2, c) == LEFT &&
                     orient3(q2, q3, c) == LEFT && orient3(q3, q0, c) == LEFT);
    }
}

void oc_classify_quad(const double *xs, const double *ys, uint64_t n, const uint64_t quad[4],
                      uint8_t *flags) {
    const pt q0 = {xs[quad[0]], ys[quad[0]]}, q1 = {xs[quad[1]], ys[quad[1]]};
    const pt q2 = {xs[quad[2]], ys[quad[2]]}, q3 = {xs[quad[3]], ys[quad[3]]};
    for (uint64_t i = 0; i < n; ++i) {
        const pt c = {xs[i], ys[i]};
        flags[i] = !(orient3(q0, q1, c) == LEFT && orient3(q1, q2, c) == LEFT &&
                     orient3(q2, q3, c) == LEFT && orient3(q3, q0, c) == LEFT);
    }
}

/* angular.hpp:40-49 select_anchor: min y, then min x, then lowest index. */
static uint64_t anchor_pts(const pt *p, uint64_t n) {
    uint64_t best = 0;
    for (uint64_t i = 1; i < n; ++i) {
        if (p[i].y < p[best].y || (p[i].y == p[best].y && p[i].x < p[best].x)) best = i;
    }
    return best;
}

uint64_t oc_select_anchor(const double *xs, const double *ys, uint64_t n) {
    uint64_t best = 0;
    for (uint64_t i = 1; i < n; ++i) {
        if (ys[i] < ys[best] || (ys[i] == ys[best] && xs[i] < xs[best])) best = i;
    }
    return best;
}

/* angular.hpp:57-111 CoordSet: exact coordinates, -0.0 folded onto +0.0. */
typedef struct { uint64_t *x, *y; uint64_t mask; } coordset;
static const uint64_t kEmpty = ~(uint64_t)0;
static uint64_t fold_bits(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t u;
    memcpy(&u, &v, 8);
    return u;
}
static uint64_t mix64(uint64_t a, uint64_t b) {
    uint64_t z = a ^ (b * 0x9e3779b97f4a7c15ULL);
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
}
static int coordset_init(coordset *s, uint64_t expected) {
    uint64_t cap = 16;
    while (cap < expected * 2) cap *= 2;
    s->x = (uint64_t *)malloc(cap * 8);
    s->y = (uint64_t *)malloc(cap * 8);
    if (!s->x || !s->y) return 0;
    memset(s->x, 0xff, cap * 8);
    s->mask = cap - 1;
    return 1;
}
static void coordset_free(coordset *s) { free(s->x); free(s->y); }
static int coordset_insert(coordset *s, pt p) {
    const uint64_t xb = fold_bits(p.x), yb = fold_bits(p.y);
    uint64_t i = mix64(xb, yb) & s->mask;
    for (;;) {
        if (s->x[i] == kEmpty) { s->x[i] = xb; s->y[i] = yb; return 1; }
        if (s->x[i] == xb && s->y[i] == yb) return 0;
        i = (i + 1) & s->mask;
    }
}

/* Annotated buffer entry: point, polar key, input index. */
typedef struct { double angle, dist2; pt p; uint64_t idx; } entry;

/* angular.hpp:159-161: (angle, dist2) ascending; ties keep buffer order. */
static int entry_less(const entry *a, const entry *b) {
    return a->angle < b->angle || (a->angle == b->angle && a->dist2 < b->dist2);
}

/* Stable merge sort (any stable sort yields std::stable_sort's permutation). */
static void merge_sort(entry *a, entry *tmp, uint64_t n) {
    if (n < 2) return;
    const uint64_t run = 32;
    for (uint64_t lo = 0; lo < n; lo += run) {
        const uint64_t hi = lo + run < n ? lo + run : n;
        for (uint64_t i = lo + 1; i < hi; ++i) {
            entry e = a[i];
            uint64_t j = i;
            while (j > lo && entry_less(&e, &a[j - 1])) { a[j] = a[j - 1]; --j; }
            a[j] = e;
        }
    }
    entry *src = a, *dst = tmp;
    for (uint64_t width = run; width < n; width *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * width) {
            uint64_t mid = lo + width < n ? lo + width : n;
            uint64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            uint64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) dst[k++] = entry_less(&src[j], &src[i]) ? src[j++] : src[i++];
            while (i < mid) dst[k++] = src[i++];
            while (j < hi) dst[k++] = src[j++];
        }
        entry *t = src; src = dst; dst = t;
    }
    if (src != a) memcpy(a, src, n * sizeof(entry));
}

/* discard.hpp:36-49 walk_right / :53-66 walk_left. */
static void walk_right(const entry *b, uint64_t longest, uint64_t seed, uint64_t first,
                       uint64_t last, uint8_t *flags) {
    const pt pl = b[longest].p;
    uint64_t temp = seed;
    for (uint64_t i = first; i < last; ++i) {
        if (orient3(b[temp].p, pl, b[i].p) == LEFT) flags[i] = 0;
        else temp = i;
    }
}
static void walk_left(const entry *b, uint64_t longest, uint64_t seed, uint64_t hi, uint64_t lo,
                      uint8_t *flags) {
    const pt pl = b[longest].p;
    uint64_t temp = seed;
    for (uint64_t i = hi; i >= lo; --i) {
        if (orient3(b[temp].p, pl, b[i].p) == RIGHT) flags[i] = 0;
        else temp = i;
        if (i == 0) break;
    }
}

int oc_full_pipeline(const double *xs, const double *ys, uint64_t n, const oc_config *cfg_in,
                     uint64_t *out_idx, uint64_t out_cap, uint64_t *out_len, oc_stats *stats,
                     oc_trace *trace) {
    oc_config cfg;
    if (cfg_in) cfg = *cfg_in; else oc_config_default(&cfg);
    if (n == 0) return OC_E_EMPTY_INPUT;           /* pipeline.hpp:73 */
    if (cfg.chunk_count == 0) return OC_E_ZERO_CHUNKS; /* pipeline.hpp:74 */
    oc_stats st;
    memset(&st, 0, sizeof st);
    st.n_input = n;
    int rc = OC_OK;

    const double t0 = now_ms();
    pt *pts = (pt *)malloc(n * sizeof(pt));
    uint64_t *sidx = (uint64_t *)malloc(n * sizeof(uint64_t)); /* stage-1 input indices */
    if (!pts || !sidx) { free(pts); free(sidx); return OC_E_NOMEM; }
    uint64_t n1 = 0;
    if (cfg.enable_round1) { /* pipeline.hpp:87-92 */
        for (uint64_t i = 0; i < n; ++i) { pts[i].x = xs[i]; pts[i].y = ys[i]; }
        uint64_t q[4];
        find_extremes_pts(pts, n, q);
        uint8_t *flags = (uint8_t *)malloc(n);
        if (!flags) { free(pts); free(sidx); return OC_E_NOMEM; }
        classify_pts(pts, n, q, flags);
        for (uint64_t i = 0; i < n; ++i) /* compact, prefilter.hpp:65-76 */
            if (flags[i]) { pts[n1] = pts[i]; sidx[n1] = i; ++n1; }
        free(flags);
        if (trace) memcpy(trace->quad, q, sizeof q);
    } else {
        for (uint64_t i = 0; i < n; ++i) { pts[i].x = xs[i]; pts[i].y = ys[i]; sidx[i] = i; }
        n1 = n;
    }
    st.n_after_round1 = n1;
    if (trace && trace->r1_idx) memcpy(trace->r1_idx, sidx, n1 * sizeof(uint64_t));
    const double t1 = now_ms();

    /* annotate(stage1, select_anchor(stage1)), angular.hpp:118-148 */
    const uint64_t a = anchor_pts(pts, n1);
    const pt anchor = pts[a];
    entry *buf = (entry *)malloc(n1 * sizeof(entry));
    coordset seen;
    if (!buf || !coordset_init(&seen, n1)) { free(pts); free(sidx); free(buf); return OC_E_NOMEM; }
    uint64_t m = 0;
    buf[m].p = anchor; buf[m].idx = sidx[a]; buf[m].angle = 0.0; buf[m].dist2 = 0.0; ++m;
    coordset_insert(&seen, anchor);
    for (uint64_t i = 0; i < n1; ++i) {
        if (coordset_insert(&seen, pts[i])) { buf[m].p = pts[i]; buf[m].idx = sidx[i]; ++m; }
    }
    coordset_free(&seen);
    for (uint64_t i = 1; i < m; ++i) { /* polar_key, geom.hpp:38-43 */
        const double dx = buf[i].p.x - anchor.x, dy = buf[i].p.y - anchor.y;
        buf[i].angle = atan2(dy, dx);
        buf[i].dist2 = dx * dx + dy * dy;
    }
    free(pts);
    free(sidx);
    if (trace) trace->anchor = buf[0].idx;
    const double t2 = now_ms();

    /* sort_by_angle, angular.hpp:154-194 */
    if (m >= 3) {
        entry *tmp = (entry *)malloc((m - 1) * sizeof(entry));
        if (!tmp) { free(buf); return OC_E_NOMEM; }
        merge_sort(buf + 1, tmp, m - 1);
        free(tmp);
    }
    if (trace && trace->sorted_idx)
        for (uint64_t i = 0; i < m; ++i) trace->sorted_idx[i] = buf[i].idx;
    if (trace) { trace->sorted_len = m; trace->longest = 0; }
    const double t3 = now_ms();

    /* round 2, pipeline.hpp:102-108 */
    if (cfg.enable_round2 && m >= 2) {
        uint64_t l = 1; /* split_regions, angular.hpp:197-204 */
        for (uint64_t i = 2; i < m; ++i) if (buf[i].dist2 > buf[l].dist2) l = i;
        uint8_t *flags = (uint8_t *)malloc(m);
        if (!flags) { free(buf); return OC_E_NOMEM; }
        memset(flags, 1, m);
        if (cfg.chunked) { /* discard_chunked, discard.hpp:96-124 */
            const uint64_t c = cfg.chunk_count;
            const uint64_t m_right = l - 1;
            if (m_right > 1) {
                const uint64_t step = (m_right + c - 1) / c;
                for (uint64_t begin = 1; begin < l; begin += step) {
                    const uint64_t end = begin + step < l ? begin + step : l;
                    walk_right(buf, l, begin, begin + 1, end, flags);
                }
            }
            const uint64_t m_left = m - 1 - l;
            if (m_left > 1) {
                const uint64_t step = (m_left + c - 1) / c;
                for (uint64_t pos = 0; pos < m_left; pos += step) {
                    const uint64_t seed = m - 1 - pos;
                    const uint64_t off = pos + step - 1 < m_left - 1 ? pos + step - 1 : m_left - 1;
                    const uint64_t lo = m - 1 - off;
                    if (seed > lo) walk_left(buf, l, seed, seed - 1, lo, flags);
                }
            }
        } else { /* discard_sequential, discard.hpp:79-88 */
            if (l >= 2) walk_right(buf, l, 0, 1, l, flags);
            if (l + 2 <= m - 1) walk_left(buf, l, m - 1, m - 2, l + 1, flags);
        }
        if (trace) trace->longest = l;
        if (trace && trace->r2_flags) memcpy(trace->r2_flags, flags, m);
        uint64_t k = 0; /* stable_compact, discard.hpp:128-145 */
        for (uint64_t i = 0; i < m; ++i) if (flags[i]) buf[k++] = buf[i];
        m = k;
        free(flags);
    }
    st.n_after_round2 = m;
    if (trace && trace->r2_idx)
        for (uint64_t i = 0; i < m; ++i) trace->r2_idx[i] = buf[i].idx;
    const double t4 = now_ms();

    /* graham_finalize, pipeline.hpp:57-67 */
    uint64_t *stack = (uint64_t *)malloc(m * sizeof(uint64_t));
    if (!stack) { free(buf); return OC_E_NOMEM; }
    uint64_t top = 0;
    for (uint64_t i = 0; i < m; ++i) {
        while (top >= 2 && orient3(buf[stack[top - 2]].p, buf[stack[top - 1]].p, buf[i].p) != LEFT)
            --top;
        stack[top++] = i;
    }
    const double t5 = now_ms();
    st.hull_size = top;
    if (out_len) *out_len = top;
    if (top > out_cap || !out_idx) {
        rc = (top > out_cap) ? OC_E_CAPACITY : OC_OK;
    } else {
        for (uint64_t i = 0; i < top; ++i) out_idx[i] = buf[stack[i]].idx;
    }
    free(stack);
    free(buf);
    st.t_round1_ms = t1 - t0;
    st.t_annotate_ms = t2 - t1;
    st.t_sort_ms = t3 - t2;
    st.t_round2_ms = t4 - t3;
    st.t_finalize_ms = t5 - t4;
    st.t_total_ms = t5 - t0;
    if (stats) *stats = st;
    return rc;
}

/* oracle.hpp:40-68 monotone_chain over (x, y, idx)-sorted unique points; the
 * kept index of a duplicated coordinate is its first occurrence. */
typedef struct { double x, y; uint64_t idx; } lexpt;
static int lex_cmp(const void *pa, const void *pb) {
    const lexpt *a = (const lexpt *)pa, *b = (const lexpt *)pb;
    if (a->x < b->x) return -1;
    if (b->x < a->x) return 1;
    if (a->y < b->y) return -1;
    if (b->y < a->y) return 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}
int oc_monotone_chain(const double *xs, const double *ys, uint64_t n, uint64_t *out_idx,
                      uint64_t out_cap, uint64_t *out_len) {
    if (n == 0) return OC_E_EMPTY_INPUT;
    lexpt *p = (lexpt *)malloc(n * sizeof(lexpt));
    uint64_t *ring = (uint64_t *)malloc((n + 1) * sizeof(uint64_t));
    if (!p || !ring) { free(p); free(ring); return OC_E_NOMEM; }
    for (uint64_t i = 0; i < n; ++i) { p[i].x = xs[i]; p[i].y = ys[i]; p[i].idx = i; }
    qsort(p, n, sizeof(lexpt), lex_cmp);
    uint64_t u = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (u == 0 || !(p[i].x == p[u - 1].x && p[i].y == p[u - 1].y)) p[u++] = p[i];
    uint64_t r = 0;
    if (u == 1) {
        ring[r++] = 0;
    } else {
#define PT(k) ((pt){p[(k)].x, p[(k)].y})
        for (uint64_t i = 0; i < u; ++i) {
            while (r >= 2 && orient3(PT(ring[r - 2]), PT(ring[r - 1]), PT(i)) != LEFT) --r;
            ring[r++] = i;
        }
        const uint64_t lower = r;
        for (uint64_t i = u - 1; i-- > 0;) {
            while (r > lower && orient3(PT(ring[r - 2]), PT(ring[r - 1]), PT(i)) != LEFT) --r;
            ring[r++] = i;
        }
        --r;
        uint64_t start = 0; /* canonicalize: lowest (y, then x) vertex first */
        for (uint64_t i = 1; i < r; ++i) {
            const lexpt *a = &p[ring[i]], *b = &p[ring[start]];
            if (a->y < b->y || (a->y == b->y && a->x < b->x)) start = i;
        }
        if (start) {
            uint64_t *tmp = (uint64_t *)malloc(r * sizeof(uint64_t));
            for (uint64_t i = 0; i < r; ++i) tmp[i] = ring[(start + i) % r];
            memcpy(ring, tmp, r * sizeof(uint64_t));
            free(tmp);
        }
#undef PT
    }
    if (out_len) *out_len = r;
    int rc = OC_OK;
    if (r > out_cap) rc = OC_E_CAPACITY;
    else for (uint64_t i = 0; i < r; ++i) out_idx[i] = p[ring[i]].idx;
    free(p);
    free(ring);
    return rc;
}
