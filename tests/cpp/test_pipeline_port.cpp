// The reference's own degenerate-input and error checks
// (/root/reference/proj/tests/test_pipeline.cpp:92-107, "degenerate inputs
// follow the documented conventions") run unchanged against the GPU shim:
// the only edits are the includes, the namespace switch and a minimal CHECK /
// CHECK_THROWS_AS in place of Catch2 (absent here). The
// exceptions are the reference's types (hull2d::EmptyInput, hull2d::ZeroChunks
// from its errors.hpp), thrown by hull2d_gpu::full_pipeline. Built by
// __graft_entry__.build() where /root/reference exists; the binary travels to
// the GPU box (tests/test_gpu_cpp.py runs it).
#include <cstdio>
#include <vector>

#include <hull2d/errors.hpp>

#include "hull2d_gpu.hpp"

static_assert(HULL2D_GPU_REFERENCE_ERRORS, "the shim must throw the reference's error types");

using namespace hull2d_gpu;
using hull2d::EmptyInput;
using hull2d::ZeroChunks;

static int failures = 0;
#define CHECK(...)                                                                   \
    do {                                                                             \
        if (!(__VA_ARGS__)) {                                                        \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__);       \
            ++failures;                                                              \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, E)                                                     \
    do {                                                                             \
        bool ok_ = false;                                                            \
        try {                                                                        \
            (void)(expr);                                                            \
        } catch (const E&) {                                                         \
            ok_ = true;                                                              \
        } catch (...) {                                                              \
        }                                                                            \
        if (!ok_) {                                                                  \
            std::printf("FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__,    \
                        #expr, #E);                                                  \
            ++failures;                                                              \
        }                                                                            \
    } while (0)

int main() {
    // ---- test_pipeline.cpp:92-107, unchanged ----
    CHECK(full_pipeline(std::vector<Point2>{{2, 3}}).hull.vertices ==
          std::vector<Point2>{{2, 3}});
    CHECK(full_pipeline(std::vector<Point2>{{2, 3}, {0, 1}}).hull.vertices ==
          std::vector<Point2>{{0, 1}, {2, 3}});
    CHECK(full_pipeline(std::vector<Point2>{{0, 0}, {1, 0}, {2, 0}, {1, 0}}).hull.vertices ==
          std::vector<Point2>{{0, 0}, {2, 0}});
    const auto dup = full_pipeline(std::vector<Point2>(6, Point2{1, 1}));
    CHECK(dup.hull.vertices == std::vector<Point2>{{1, 1}});
    CHECK(dup.stats.n_after_round2 == 1);

    CHECK_THROWS_AS(full_pipeline(std::vector<Point2>{}), EmptyInput);
    PipelineConfig bad;
    bad.chunk_count = 0;
    CHECK_THROWS_AS(full_pipeline(std::vector<Point2>{{0, 0}}, bad), ZeroChunks);
    // ---- end of the reference's checks ----
    if (failures) {
        std::printf("%d failures\n", failures);
        return 1;
    }
    std::printf("ok\n");
    return 0;
}
