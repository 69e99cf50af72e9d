// mt19937_64 jump-ahead over GF(2), host side (used by the on-device
// generator, gscan_generate_square_device).
//
// The reference's inputs come from libstdc++'s std::mt19937_64 fed to
// uniform_real_distribution<double>(0, 1) (datagen.hpp:32-41: gen_square draws
// x then y per point). The engine is a linear recurrence over GF(2) on its
// 312-word state (19937 effective bits): x[i+312] = x[i+156] ^ twist(x[i],
// x[i+1]). Its characteristic polynomial phi (degree 19937) is recovered once
// with Berlekamp-Massey from 2 * 19937 output bits; jumping the state ahead by
// J words is g(T) with g = t^J mod phi, evaluated as the XOR of the windows
// [i, i + 312) of the word stream for every set coefficient g_i (the device
// does that part, k_mt_jump). Only the top 33 bits of a state's first word
// matter to the recurrence; a jumped state's low 31 bits of word 0 may differ
// from the sequential engine's, and they are never output (outputs start at
// x[312]).
#pragma once
#include <cstdint>
#include <vector>

namespace gscan {
namespace mt64 {

constexpr int kN = 312;
constexpr int kM = 156;
constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 1 + 63) / 64;  // 312 words hold a polynomial of degree <= 19937
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = ~0ull << 31;  // top 33 bits
constexpr uint64_t kLower = (1ull << 31) - 1;

// std::mt19937_64::seed(s): the initial 312-word state
void seed_state(uint64_t seed, uint64_t* st);
// t^(2^b * L) mod phi for b = 0 .. nb-1, kWords words each (cached per L)
const std::vector<uint64_t>& jump_table(uint64_t L, int nb);
// host reference of the device jump (tests / self-check): state <- g(T) state
void apply_jump_host(const uint64_t* g, uint64_t* state);

}  // namespace mt64
}  // namespace gscan
