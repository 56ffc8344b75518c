// mgp_device.cuh -- device-side building blocks for the Megopolis hot path (sm_100a).
//
// Random streams
//   megores : the reference's keyed splitmix64 hash (pkg/src/megores/rng.py:85-121),
//             reproduced bit-for-bit.  x(lane, t) = mix(seed + M_LANE) + lane*M_LANE + t*M_CTR,
//             h = mix(x); u = (h >> 11) * 2^-53.  The per-lane key is strength-reduced:
//             x(lane, t+1) = x(lane, t) + M_CTR.
//   philox  : Philox4x32-10 (key = seed, counter = {lane, t >> 2}); word t & 3 of the
//             block is draw t; u = word * 2^-32, uint_below(n) = (word * n) >> 32.
//
// Acceptance (pkg/src/megores/resample.py:118-122): accept j iff
//   !(w_j == 0 && w_k == 0) && u * w_k <= w_j       evaluated in IEEE binary64.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mgp {

constexpr uint64_t M_LANE = 0x9E3779B97F4A7C15ull;  // rng.py:45
constexpr uint64_t M_CTR = 0xD1B54A32D192ED03ull;   // rng.py:46
constexpr uint64_t M_SALT = 0x8CB92BA72F3D8DD7ull;  // rng.py:47
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ull;    // rng.py:48
constexpr uint64_t MIX2 = 0x94D049BB133111EBull;    // rng.py:49
constexpr uint64_t WARP_LANE_BASE = 1ull << 61;     // rng.py:42
constexpr uint64_t GLOBAL_OFFSET_LANE = 1ull << 62; // rng.py:43

constexpr uint32_t PHILOX_M0 = 0xD2511F53u, PHILOX_M1 = 0xCD9E8D57u;
constexpr uint32_t PHILOX_W0 = 0x9E3779B9u, PHILOX_W1 = 0xBB67AE85u;

enum Rng : int { RNG_MEGORES = 0, RNG_PHILOX = 1 };

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // rng.py:85-89
  x = (x ^ (x >> 30)) * MIX1;
  x = (x ^ (x >> 27)) * MIX2;
  return x ^ (x >> 31);
}

// mix(x) >> 11 with the final xorshift folded into the shift:
// (x ^ (x >> 31)) >> 11 == (x >> 11) ^ (x >> 42).
__device__ __forceinline__ uint64_t mix64_m53(uint64_t x) {
  x = (x ^ (x >> 30)) * MIX1;
  x = (x ^ (x >> 27)) * MIX2;
  return (x >> 11) ^ (x >> 42);
}

__host__ __device__ __forceinline__ uint64_t megores_base(uint64_t seed) { return mix64(seed + M_LANE); }

__host__ __device__ __forceinline__ uint64_t megores_key(uint64_t base, uint64_t lane, uint64_t t) {
  return base + lane * M_LANE + t * M_CTR;
}

// ---------------------------------------------------------------------------
// Philox4x32-10

struct P4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ P4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                    uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(PHILOX_M0, c0), lo0 = PHILOX_M0 * c0;
    uint32_t hi1 = __umulhi(PHILOX_M1, c2), lo1 = PHILOX_M1 * c2;
#else
    uint64_t p0 = (uint64_t)PHILOX_M0 * c0, p1 = (uint64_t)PHILOX_M1 * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0, hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += PHILOX_W0; k1 += PHILOX_W1;
  }
  return P4{c0, c1, c2, c3};
}

__host__ __device__ __forceinline__ uint32_t p4_word(const P4& p, uint32_t q) {
  return q == 0 ? p.x : q == 1 ? p.y : q == 2 ? p.z : p.w;
}

__host__ __device__ __forceinline__ P4 philox_block(uint64_t seed, uint64_t lane, uint64_t blk) {
  return philox4x32_10((uint32_t)lane, (uint32_t)(lane >> 32), (uint32_t)blk, (uint32_t)(blk >> 32),
                       (uint32_t)seed, (uint32_t)(seed >> 32));
}

// ---------------------------------------------------------------------------
// Exact draws (generic paths)

__host__ __device__ __forceinline__ double u01_from_hash(uint64_t h) {  // rng.py:105-108
  return (double)(h >> 11) * 0x1p-53;
}

// uint_below on a megores hash: int64(u01 * float(n)), clamped (rng.py:111-121)
__host__ __device__ __forceinline__ int64_t below_from_hash(uint64_t h, int64_t n) {
  int64_t v = (int64_t)(u01_from_hash(h) * (double)n);
  return v >= n ? n - 1 : v;
}

__host__ __device__ __forceinline__ double u01_from_word(uint32_t w) { return (double)w * 0x1p-32; }

__host__ __device__ __forceinline__ int64_t below_from_word(uint32_t w, int64_t n) {
  return (int64_t)(((uint64_t)w * (uint64_t)n) >> 32);
}

// Generic per-lane stream positioned at counter t (one draw per call).
template <int RNG>
struct Stream;

template <>
struct Stream<RNG_MEGORES> {
  uint64_t x;
  __device__ __forceinline__ Stream(uint64_t seed_base, uint64_t /*seed*/, uint64_t lane, uint64_t t)
      : x(megores_key(seed_base, lane, t)) {}
  __device__ __forceinline__ double u() { double r = u01_from_hash(mix64(x)); x += M_CTR; return r; }
  __device__ __forceinline__ int64_t below(int64_t n) { int64_t r = below_from_hash(mix64(x), n); x += M_CTR; return r; }
};

template <>
struct Stream<RNG_PHILOX> {
  uint64_t seed, lane, t;
  P4 blk;
  __device__ __forceinline__ Stream(uint64_t /*seed_base*/, uint64_t s, uint64_t l, uint64_t t0)
      : seed(s), lane(l), t(t0) { blk = philox_block(seed, lane, t >> 2); }
  __device__ __forceinline__ uint32_t word() {
    if ((t & 3) == 0) blk = philox_block(seed, lane, t >> 2);
    uint32_t r = p4_word(blk, (uint32_t)(t & 3));
    ++t;
    return r;
  }
  __device__ __forceinline__ double u() { return u01_from_word(word()); }
  __device__ __forceinline__ int64_t below(int64_t n) { return below_from_word(word(), n); }
};

// Single keyed draw (lane, t) without a running stream.
template <int RNG>
__device__ __forceinline__ int64_t draw_below(uint64_t seed_base, uint64_t seed, uint64_t lane, uint64_t t, int64_t n) {
  if (RNG == RNG_MEGORES) return below_from_hash(mix64(megores_key(seed_base, lane, t)), n);
  return below_from_word(p4_word(philox_block(seed, lane, t >> 2), (uint32_t)(t & 3)), n);
}

// ---------------------------------------------------------------------------
// Acceptance

// Exact rule, any weights (zeros, subnormals, f64).
__device__ __forceinline__ bool accepts(double u, double wk, double wj) {
  return !(wj == 0.0 && wk == 0.0) && (u * wk <= wj);
}

}  // namespace mgp
