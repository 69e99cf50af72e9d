// Reference-style checks through the C++ shim (include/hull2d_gpu.hpp), in the
// shape of /root/reference/proj/tests/test_pipeline.cpp: the same known
// answers, exceptions and stats invariants, on the GPU. Prints "ok" and exits
// 0 on success; built and run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numbers>
#include <random>
#include <vector>

#include "hull2d_gpu.hpp"

using namespace hull2d_gpu;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // test_pipeline.cpp:19-28 graham on a square / collinear input
    CHECK((full_pipeline(std::vector<Point2>{{0, 0}, {1, 0}, {1, 1}, {0, 1}}).hull.vertices ==
           std::vector<Point2>{{0, 0}, {1, 0}, {1, 1}, {0, 1}}));
    CHECK((full_pipeline(std::vector<Point2>{{0, 0}, {1, 0}, {2, 0}}).hull.vertices ==
           std::vector<Point2>{{0, 0}, {2, 0}}));
    // :36-47 three non-collinear points pass both rounds under every config
    const std::vector<Point2> tri{{0, 0}, {3, 1}, {1, 4}};
    for (const PipelineConfig cfg :
         {PipelineConfig{}, PipelineConfig{.chunk_count = 1}, PipelineConfig{.enable_round1 = false},
          PipelineConfig{.enable_round2 = false}, PipelineConfig{.chunked = false}}) {
        const auto r = full_pipeline(tri, cfg);
        CHECK(r.hull.size() == 3);
        CHECK(r.stats.n_after_round1 == 3);
        CHECK(r.stats.n_after_round2 == 3);
    }
    // :92-107 degenerate conventions and the error behaviour
    CHECK((full_pipeline(std::vector<Point2>{{2, 3}}).hull.vertices == std::vector<Point2>{{2, 3}}));
    CHECK((full_pipeline(std::vector<Point2>{{2, 3}, {0, 1}}).hull.vertices ==
           std::vector<Point2>{{0, 1}, {2, 3}}));
    CHECK((full_pipeline(std::vector<Point2>{{0, 0}, {1, 0}, {2, 0}, {1, 0}}).hull.vertices ==
           std::vector<Point2>{{0, 0}, {2, 0}}));
    const auto dup = full_pipeline(std::vector<Point2>(6, Point2{1, 1}));
    CHECK((dup.hull.vertices == std::vector<Point2>{{1, 1}}));
    CHECK(dup.stats.n_after_round2 == 1);
    CHECK(throws_as<EmptyInput>([] { full_pipeline(std::vector<Point2>{}); }));
    CHECK(throws_as<ZeroChunks>([] {
        PipelineConfig bad;
        bad.chunk_count = 0;
        full_pipeline(std::vector<Point2>{{0, 0}}, bad);
    }));
    // :73-81 on-circle input keeps every point through both rounds
    {
        std::vector<Point2> circle;
        std::mt19937_64 rng(1);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        for (int i = 0; i < 1000; ++i) {
            const double t = 2.0 * std::numbers::pi * unit(rng);
            circle.push_back({std::cos(t), std::sin(t)});
        }
        const auto r = full_pipeline(circle);
        CHECK(r.stats.n_after_round1 == 1000);
        CHECK(r.stats.n_after_round2 == 1000);
        CHECK(r.hull.size() == 1000);
    }
    // :125-137 stats consistency; every input point lies inside or on the hull
    {
        std::vector<Point2> pts(2000);
        std::mt19937_64 rng(8);
        std::uniform_real_distribution<double> unit(0.0, 1.0);
        for (auto& p : pts) {
            p.x = unit(rng);
            p.y = unit(rng);
        }
        const auto r = full_pipeline(pts);
        CHECK(r.stats.n_input == 2000);
        CHECK(r.stats.n_after_round2 <= r.stats.n_after_round1);
        CHECK(r.stats.hull_size == r.hull.size());
        CHECK(r.stats.t_total_ms >= 0.0);
        const auto& v = r.hull.vertices;
        for (const auto& p : pts) {
            bool inside = true;
            for (std::size_t i = 0; i < v.size() && inside; ++i) {
                const Point2 a = v[i], b = v[(i + 1) % v.size()];
                if ((b.x - a.x) * (p.y - a.y) - (b.y - a.y) * (p.x - a.x) < 0.0) inside = false;
            }
            CHECK(inside);
        }
        for (std::size_t i = 0; i < r.hull.size(); ++i) CHECK(pts[r.hull.indices[i]] == v[i]);
    }
    if (failures) {
        std::printf("%d failures\n", failures);
        return 1;
    }
    std::printf("ok\n");
    return 0;
}
