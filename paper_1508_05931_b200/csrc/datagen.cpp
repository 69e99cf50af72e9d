// Seeded synthetic point sets for the bench and parity harness (host side).
//
// Behaviourally identical to the reference generators
// (/root/reference/proj/include/hull2d/datagen.hpp:32-91) and the tests'
// integer grid (tests/support.hpp:54-63): the same libstdc++ engines and
// distributions, drawn in the same order, so a (kind, n, seed) triple yields
// the same bits on both sides. Output is SoA (xs, ys), the layout the device
// path consumes. OpenMP-free and single-threaded on purpose: the sequence is
// one mt19937_64 stream.
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <unordered_set>

#include "../../include/gscan.h"

extern "C" int gscan_generate(int kind, uint64_t n, uint64_t seed, double* xs, double* ys) {
    if (!xs || !ys) return GSCAN_E_INVALID;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    switch (kind) {
        case GSCAN_GEN_SQUARE:  // datagen.hpp:32-41
            for (uint64_t i = 0; i < n; ++i) {
                xs[i] = unit(rng);
                ys[i] = unit(rng);
            }
            return GSCAN_OK;
        case GSCAN_GEN_DISK:  // datagen.hpp:43-54
            for (uint64_t i = 0; i < n; ++i) {
                const double r = std::sqrt(unit(rng));
                const double theta = 2.0 * std::numbers::pi * unit(rng);
                xs[i] = r * std::cos(theta);
                ys[i] = r * std::sin(theta);
            }
            return GSCAN_OK;
        case GSCAN_GEN_CIRCLE: {  // datagen.hpp:58-71: distinct angles, resampled on collision
            std::unordered_set<double> used;
            used.reserve(2 * n);
            uint64_t k = 0;
            while (k < n) {
                const double theta = 2.0 * std::numbers::pi * unit(rng);
                if (!used.insert(theta).second) continue;
                xs[k] = std::cos(theta);
                ys[k] = std::sin(theta);
                ++k;
            }
            return GSCAN_OK;
        }
        case GSCAN_GEN_COLLINEAR: {  // datagen.hpp:75-91
            std::uniform_int_distribution<int> small(-8, 8);
            std::uniform_int_distribution<int> param(-1000, 1000);
            const double ox = small(rng);
            const double oy = small(rng);
            int dx = small(rng);
            int dy = small(rng);
            if (dx == 0 && dy == 0) dx = 1;
            for (uint64_t i = 0; i < n; ++i) {
                const double t = param(rng);
                xs[i] = ox + t * dx;
                ys[i] = oy + t * dy;
            }
            return GSCAN_OK;
        }
        default:
            return GSCAN_E_INVALID;
    }
}

// tests/support.hpp:54-63 gen_grid: integer points in [lo, hi]^2.
extern "C" int gscan_generate_grid(uint64_t n, uint64_t seed, int lo, int hi, double* xs,
                                   double* ys) {
    if (!xs || !ys || lo > hi) return GSCAN_E_INVALID;
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<int> coord(lo, hi);
    for (uint64_t i = 0; i < n; ++i) {
        xs[i] = coord(rng);
        ys[i] = coord(rng);
    }
    return GSCAN_OK;
}
