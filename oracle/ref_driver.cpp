// TEST INFRASTRUCTURE ONLY -- C-ABI wrapper around the *unmodified* reference.
//
// Compiled by oracle/Makefile against the read-only headers in
// /root/reference/proj/include with the reference's Release flags
// (-std=c++20 -O3 -DNDEBUG -pthread, no -march: no FMA contraction,
// SURVEY.md 7.1) into oracle/_ref/libhull2d_ref.so. This file contains no
// reference code; it only calls hull2d::full_pipeline and the stage functions
// and maps the returned Point2 vertices back to input indices (first
// occurrence), which is how the north-star index list is defined.
#include <cstdint>
#include <cstring>
#include <span>
#include <unordered_map>
#include <vector>

#include "hull2d/hull2d.hpp"

namespace {

using hull2d::Point2;

std::vector<Point2> to_points(const double* xs, const double* ys, uint64_t n) {
    std::vector<Point2> p(n);
    for (uint64_t i = 0; i < n; ++i) p[i] = {xs[i], ys[i]};
    return p;
}

uint64_t fold(double v) {
    if (v == 0.0) v = 0.0;
    uint64_t u;
    std::memcpy(&u, &v, 8);
    return u;
}

struct KeyHash {
    size_t operator()(const std::pair<uint64_t, uint64_t>& k) const {
        return std::hash<uint64_t>()(k.first * 0x9e3779b97f4a7c15ULL ^ k.second);
    }
};

// coordinate -> first input index holding it (IEEE equality, -0.0 == +0.0)
struct FirstIndex {
    std::unordered_map<std::pair<uint64_t, uint64_t>, uint64_t, KeyHash> map;
    FirstIndex(const double* xs, const double* ys, uint64_t n) {
        map.reserve(n * 2);
        for (uint64_t i = 0; i < n; ++i) map.emplace(std::make_pair(fold(xs[i]), fold(ys[i])), i);
    }
    uint64_t operator()(Point2 p) const { return map.at({fold(p.x), fold(p.y)}); }
};

int status_of(const hull2d::Error& e) {
    if (dynamic_cast<const hull2d::EmptyInput*>(&e)) return 1;
    if (dynamic_cast<const hull2d::ZeroChunks*>(&e)) return 2;
    return 9;
}

}  // namespace

extern "C" {

struct ref_stats {
    uint64_t n_input, n_after_round1, n_after_round2, hull_size;
    double t_round1_ms, t_annotate_ms, t_sort_ms, t_round2_ms, t_finalize_ms, t_total_ms;
};

// hull2d::full_pipeline (pipeline.hpp:72) on SoA input. out_idx may be NULL
// (timing runs): then only stats/out_len are produced.
int ref_full_pipeline(const double* xs, const double* ys, uint64_t n, uint64_t chunk_count,
                      int enable_round1, int enable_round2, int chunked, uint64_t* out_idx,
                      uint64_t out_cap, uint64_t* out_len, ref_stats* stats) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        hull2d::PipelineConfig cfg;
        cfg.chunk_count = chunk_count;
        cfg.enable_round1 = enable_round1 != 0;
        cfg.enable_round2 = enable_round2 != 0;
        cfg.chunked = chunked != 0;
        const hull2d::PipelineResult r = hull2d::full_pipeline(pts, cfg);
        if (stats) {
            stats->n_input = r.stats.n_input;
            stats->n_after_round1 = r.stats.n_after_round1;
            stats->n_after_round2 = r.stats.n_after_round2;
            stats->hull_size = r.stats.hull_size;
            stats->t_round1_ms = r.stats.t_round1_ms;
            stats->t_annotate_ms = r.stats.t_annotate_ms;
            stats->t_sort_ms = r.stats.t_sort_ms;
            stats->t_round2_ms = r.stats.t_round2_ms;
            stats->t_finalize_ms = r.stats.t_finalize_ms;
            stats->t_total_ms = r.stats.t_total_ms;
        }
        if (out_len) *out_len = r.hull.size();
        if (!out_idx) return 0;
        if (r.hull.size() > out_cap) return 3;
        const FirstIndex first(xs, ys, n);
        for (size_t i = 0; i < r.hull.size(); ++i) out_idx[i] = first(r.hull.vertices[i]);
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// oracle::monotone_chain (oracle.hpp:40-68) as first-occurrence indices.
int ref_monotone_chain(const double* xs, const double* ys, uint64_t n, uint64_t* out_idx,
                       uint64_t out_cap, uint64_t* out_len) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        const hull2d::Hull h = hull2d::oracle::monotone_chain(pts);
        *out_len = h.size();
        if (h.size() > out_cap) return 3;
        const FirstIndex first(xs, ys, n);
        for (size_t i = 0; i < h.size(); ++i) out_idx[i] = first(h.vertices[i]);
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// find_extremes (prefilter.hpp:28-39).
int ref_find_extremes(const double* xs, const double* ys, uint64_t n, uint64_t quad[4]) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        const hull2d::ExtremeQuad q = hull2d::find_extremes(pts);
        quad[0] = q.i_minx; quad[1] = q.i_miny; quad[2] = q.i_maxx; quad[3] = q.i_maxy;
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// classify_quad (prefilter.hpp:47-63) with find_extremes' quad.
int ref_classify(const double* xs, const double* ys, uint64_t n, uint8_t* flags) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        const hull2d::KeepFlags f = hull2d::classify_quad(pts, hull2d::find_extremes(pts));
        std::memcpy(flags, f.data(), n);
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// annotate + sort_by_angle (angular.hpp:118-194) of the given points, as the
// input indices of the buffer entries; returns the buffer size in *len.
int ref_sorted_buffer(const double* xs, const double* ys, uint64_t n, uint64_t* out_idx,
                      double* out_angle, double* out_dist2, uint64_t* len) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        hull2d::AnnotatedBuffer buf = hull2d::annotate(pts, hull2d::select_anchor(pts));
        hull2d::sort_by_angle(buf);
        const FirstIndex first(xs, ys, n);
        *len = buf.size();
        for (size_t i = 0; i < buf.size(); ++i) {
            out_idx[i] = first(buf.pts[i]);
            if (out_angle) out_angle[i] = buf.angle[i];
            if (out_dist2) out_dist2[i] = buf.dist2[i];
        }
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// split_regions + discard_{chunked,sequential} flags over the sorted buffer of
// the given points (discard.hpp:79-124); returns longest.
int ref_discard_flags(const double* xs, const double* ys, uint64_t n, uint64_t chunk_count,
                      int chunked, uint8_t* flags, uint64_t* longest) {
    try {
        const std::vector<Point2> pts = to_points(xs, ys, n);
        hull2d::AnnotatedBuffer buf = hull2d::annotate(pts, hull2d::select_anchor(pts));
        hull2d::sort_by_angle(buf);
        const size_t l = hull2d::split_regions(buf).longest;
        const hull2d::KeepFlags f = chunked ? hull2d::discard_chunked(buf, l, {chunk_count})
                                            : hull2d::discard_sequential(buf, l);
        std::memcpy(flags, f.data(), f.size());
        *longest = l;
        return 0;
    } catch (const hull2d::Error& e) {
        return status_of(e);
    }
}

// datagen::gen_{square,disk,circle,collinear} (datagen.hpp:32-91): kind 0..3.
int ref_generate(int kind, uint64_t n, uint64_t seed, double* xs, double* ys) {
    std::vector<Point2> p;
    switch (kind) {
        case 0: p = hull2d::datagen::gen_square(n, seed); break;
        case 1: p = hull2d::datagen::gen_disk(n, seed); break;
        case 2: p = hull2d::datagen::gen_circle(n, seed); break;
        case 3: p = hull2d::datagen::gen_collinear(n, seed); break;
        default: return 9;
    }
    for (uint64_t i = 0; i < n; ++i) { xs[i] = p[i].x; ys[i] = p[i].y; }
    return 0;
}

// The reference's loaders (datagen.hpp:111-168) for the ingest parity tests:
// 0 ok, 1 ParseError, 2 IoError, 3 EmptyInput; msg receives what().
int ref_load(const char* path, int obj, double* xs, double* ys, uint64_t cap, uint64_t* n,
             char* msg, uint64_t msg_cap) {
    auto put = [&](const char* m) {
        if (msg && msg_cap) { strncpy(msg, m, msg_cap - 1); msg[msg_cap - 1] = 0; }
    };
    try {
        const std::vector<Point2> p = obj ? hull2d::datagen::load_obj_projected(std::string(path))
                                          : hull2d::datagen::load_points(std::string(path));
        *n = p.size();
        for (uint64_t i = 0; i < p.size() && i < cap; ++i) { xs[i] = p[i].x; ys[i] = p[i].y; }
        put("");
        return 0;
    } catch (const hull2d::ParseError& e) { put(e.what()); return 1; }
    catch (const hull2d::IoError& e) { put(e.what()); return 2; }
    catch (const hull2d::EmptyInput& e) { put(e.what()); return 3; }
}

}  // extern "C"
