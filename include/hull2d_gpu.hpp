// hull2d_gpu.hpp -- C++20 drop-in for the reference's hot path.
//
// Mirrors the reference API of /root/reference/proj/include/hull2d/:
//   Point2 (geom.hpp:9-14), Hull / StageStats / PipelineConfig / PipelineResult
//   (pipeline.hpp:19-51), full_pipeline(std::span<const Point2>, const
//   PipelineConfig&) (pipeline.hpp:72), and the Error hierarchy
//   (errors.hpp:9-49) -- so reference-style code and tests switch by changing
//   the namespace. Everything runs on the GPU through the C-ABI in gscan.h
//   (link with libgscan.so); Hull additionally carries the first-occurrence
//   input index of every vertex (the north-star output).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "gscan.h"

namespace hull2d_gpu {

struct Point2 {
    double x = 0.0;
    double y = 0.0;
    friend constexpr bool operator==(const Point2&, const Point2&) = default;
};

struct Hull {
    std::vector<Point2> vertices;
    std::vector<uint64_t> indices;  // first occurrence of each vertex in the input
    std::size_t size() const { return vertices.size(); }
};

struct StageStats {
    std::size_t n_input = 0;
    std::size_t n_after_round1 = 0;
    std::size_t n_after_round2 = 0;
    std::size_t hull_size = 0;
    double t_round1_ms = 0.0;
    double t_annotate_ms = 0.0;
    double t_sort_ms = 0.0;
    double t_round2_ms = 0.0;
    double t_finalize_ms = 0.0;
    double t_total_ms = 0.0;
};

struct PipelineConfig {
    std::size_t chunk_count = 1024;
    bool enable_round1 = true;
    bool enable_round2 = true;
    bool chunked = true;
};

struct PipelineResult {
    Hull hull;
    StageStats stats;
};

// The error hierarchy. When the reference's errors.hpp is on the include
// path (-I<reference>/proj/include) the shim throws the reference's own types
// (hull2d::EmptyInput, hull2d::ZeroChunks, ... -- errors.hpp:9-49), so
// `CHECK_THROWS_AS(full_pipeline(...), hull2d::EmptyInput)` ports unchanged;
// otherwise it defines the same hierarchy in this namespace.
#if !defined(HULL2D_GPU_OWN_ERRORS) && __has_include(<hull2d/errors.hpp>)
}  // namespace hull2d_gpu
#include <hull2d/errors.hpp>
namespace hull2d_gpu {
#define HULL2D_GPU_REFERENCE_ERRORS 1
using hull2d::EmptyInput;
using hull2d::Error;
using hull2d::TooLarge;
using hull2d::ZeroChunks;
struct DeviceError : hull2d::Error {
    using hull2d::Error::Error;
};
#else
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct EmptyInput : Error {
    using Error::Error;
};
struct ZeroChunks : Error {
    using Error::Error;
};
struct TooLarge : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};
#endif

namespace detail {
[[noreturn]] inline void raise(int rc, const gscan_handle* h) {
    std::string msg = gscan_status_string(rc);
    if (h && *gscan_last_error(h)) msg = gscan_last_error(h);
    switch (rc) {
        case GSCAN_E_EMPTY_INPUT: throw EmptyInput(msg);
        case GSCAN_E_ZERO_CHUNKS: throw ZeroChunks(msg);
        case GSCAN_E_TOO_LARGE: throw TooLarge(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// One device handle (scratch + stream). Not thread-safe per instance.
class Engine {
public:
    explicit Engine(int device = -1) {
        const int rc = gscan_create(device, &h_);
        if (rc != GSCAN_OK) detail::raise(rc, nullptr);
    }
    ~Engine() { gscan_destroy(h_); }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    gscan_handle* handle() const { return h_; }

    PipelineResult full_pipeline(std::span<const Point2> points, const PipelineConfig& cfg = {}) {
        const std::size_t n = points.size();
        std::vector<double> xs(n), ys(n);
        for (std::size_t i = 0; i < n; ++i) {
            xs[i] = points[i].x;
            ys[i] = points[i].y;
        }
        gscan_config c{cfg.chunk_count, cfg.enable_round1, cfg.enable_round2, cfg.chunked, 0};
        std::vector<uint64_t> idx(n ? n : 1);
        uint64_t len = 0;
        gscan_stats st{};
        const int rc = gscan_hull_f64(h_, xs.data(), ys.data(), n, &c, idx.data(), idx.size(), &len,
                                      &st);
        if (rc != GSCAN_OK) detail::raise(rc, h_);
        PipelineResult r;
        idx.resize(len);
        r.hull.indices = std::move(idx);
        r.hull.vertices.reserve(len);
        for (uint64_t i : r.hull.indices) r.hull.vertices.push_back(points[i]);
        r.stats = {st.n_input,     st.n_after_round1, st.n_after_round2, st.hull_size,
                   st.t_round1_ms, st.t_annotate_ms,  st.t_sort_ms,      st.t_round2_ms,
                   st.t_finalize_ms, st.t_total_ms};
        return r;
    }

private:
    gscan_handle* h_ = nullptr;
};

// full_pipeline on the current device with a per-thread engine.
inline PipelineResult full_pipeline(std::span<const Point2> points, const PipelineConfig& cfg = {}) {
    thread_local Engine engine;
    return engine.full_pipeline(points, cfg);
}

}  // namespace hull2d_gpu
