// rng.h — the reference's Xorshift64Star (problems.hpp:19-46), shared by the
// host generators (problems.cpp) and the device generators (generate.cu).
//
// The state update s -> s ^= s>>12; s ^= s<<25; s ^= s>>27 is linear over
// GF(2)^64, so advancing by m draws is a 64x64 bit-matrix power:
// jump_table() holds T^(2^b) (column j = image of bit j) for b < 64 and
// jump() applies the powers of m's set bits.  Any worker can start at stream
// position m and reproduce the sequential stream bit for bit, which is what
// makes the parallel generators identical to the reference's serial ones.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define BKG_HD __host__ __device__ __forceinline__
#else
#define BKG_HD inline
#endif

namespace bkg {
namespace rng {

BKG_HD uint64_t seed_state(uint64_t seed) {  // SplitMix64 scramble of the seed
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z ? z : 0x9E3779B97F4A7C15ull;
}

BKG_HD uint64_t step(uint64_t s) {
  s ^= s >> 12;
  s ^= s << 25;
  s ^= s >> 27;
  return s;
}

BKG_HD uint64_t output(uint64_t s) { return s * 0x2545F4914F6CDD1Dull; }

// next(): advance, then scramble (the reference's order).
BKG_HD uint64_t next(uint64_t& s) {
  s = step(s);
  return output(s);
}

BKG_HD double unit(uint64_t& s) { return static_cast<double>(next(s) >> 11) * 0x1.0p-53; }

BKG_HD double symmetric(uint64_t& s) { return 2.0 * unit(s) - 1.0; }

// M v over GF(2): XOR of the columns selected by v's bits.
BKG_HD uint64_t apply(const uint64_t* cols, uint64_t v) {
  uint64_t r = 0;
  for (int j = 0; j < 64; ++j)
    if ((v >> j) & 1ull) r ^= cols[j];
  return r;
}

// table[b * 64 + j] = T^(2^b) e_j, b = 0..63.
inline void jump_table(uint64_t* table) {
  for (int j = 0; j < 64; ++j) table[j] = step(1ull << j);
  for (int b = 1; b < 64; ++b) {
    const uint64_t* prev = table + (b - 1) * 64;
    for (int j = 0; j < 64; ++j) table[b * 64 + j] = apply(prev, apply(prev, 1ull << j));
  }
}

// The state after m further steps.
BKG_HD uint64_t jump(const uint64_t* table, uint64_t s, uint64_t m) {
  for (int b = 0; m; ++b, m >>= 1)
    if (m & 1ull) s = apply(table + b * 64, s);
  return s;
}

}  // namespace rng
}  // namespace bkg
