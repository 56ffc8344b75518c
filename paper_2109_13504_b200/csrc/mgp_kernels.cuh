// mgp_kernels.cuh -- sm_100a kernels for the Megopolis hot path.
//
// Reference (pkg/src/megores, abbreviated M/):
//   Megopolis   M/resample.py:180-198, 263-282
//   Metropolis  M/resample.py:125-138, 201-206
//   C1 / C2     M/resample.py:141-177, 209-244
//   B rule      M/weights.py:114-131 fed by np.asarray(w, float64).mean()/max() (M/bench.py:119-120)
//   offspring   M/resample.py:361-368     quality  M/metrics.py:55-110     gather M/resample.py:371-377
//
// Layout in HBM: weights are the caller's contiguous f32[N] / f64[N]; ancestors int64[N]
// (the reference's dtype); particle index arithmetic is 32-bit (N < 2^31).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "mgp_device.cuh"

namespace mgp {

constexpr int RS_THREADS = 256;   // resampler CTA size (8 warps)
constexpr int OFF_CAP = 1024;     // Megopolis offsets carried per launch in the param space

// Offsets o_b for rounds [b0, b0+cnt) of one launch, pre-split on the host into
// {o & ~31, o & 31}.  Kernel parameter space is a constant bank: the warp-uniform
// reads are uniform-datapath loads that never touch the LSU/L1 path.
struct OffChunk {
  uint2 o[OFF_CAP];
};

struct ResampleArgs {
  const void* w;
  uint32_t n;        // particles
  uint32_t p0, p_end;  // particles [p0, p_end) handled by this launch (p0 % 256 == 0)
  uint32_t n_w;      // partition width (C1/C2)
  uint32_t n_part;   // number of partitions (C1/C2)
  uint32_t log2;     // log2(n) (Metropolis pow2) or log2(n_w) (C1/C2 pow2)
  uint64_t seed;     // run seed (philox key)
  uint64_t base;     // mix(seed + M_LANE) (megores stream key)
  int b0, cnt;       // rounds [b0, b0 + cnt)
  int first, last;   // first launch reads k = i; last launch writes ancestors
  int32_t* kstate;   // carried ancestor between launches (B > OFF_CAP)
  int64_t* anc;      // output ancestors
  cudaTextureObject_t tex;  // float32 weights as a 1-D linear texture (0: use LDG)
  uint32_t one;             // = 1; an opaque multiplier keeps the 64-bit key add on the FMA pipe
  int half;                 // half-split launch: [p0, p_end) is a range of LOWER-half particles
  int64_t hi_shift;         // half-split: upper-half particle i stores its ancestor at anc[i - hi_shift]
  uint32_t pk0[10], pk1[10];  // Philox round keys (uniform; constant bank)
  // fused apply_ancestors (null rows_out: off): the resampled particle's state row is copied
  // from its owner's memory -- a local array or NVLink-mapped peer memory.  Contiguous layout
  // (rows_half == 0): owner = k / rows_local.  Stripes layout (rows_half = N/2): owner r holds
  // [r*h, (r+1)*h) then N/2 + [r*h, (r+1)*h), h = rows_local / 2.
  const void* const* rows_peers;  // device array of per-owner row pointers
  int64_t rows_local;             // rows per owner
  int64_t rows_half;              // 0, or N/2 for the stripes layout
  uint32_t row_words;             // 4-byte words per row
  uint32_t* rows_out;             // output rows, indexed like anc (same shifts)
};

// Final store of one particle: the ancestor (last launch) or the carried state, and with the
// fused gather the ancestor's state row, read directly from its owner (M/resample.py:371-377).
// ROWS: compiled only into the fused-gather instantiations, so the plain kernels' code (and
// ptxas's scheduling of their main loop) is unchanged (the runtime branch alone cost 1.8%).
template <bool ROWS = true>
__device__ __forceinline__ void store_result(const ResampleArgs& a, int64_t out_idx, uint32_t i, uint32_t k) {
  if (!a.last) {
    a.kstate[i] = (int32_t)k;
    return;
  }
  a.anc[out_idx] = (int64_t)k;
  if (ROWS && a.rows_out) {
    int64_t owner, local;
    if (a.rows_half) {
      const int64_t h = a.rows_local >> 1, up = (int64_t)k >= a.rows_half, kk = (int64_t)k - up * a.rows_half;
      owner = kk / h;
      local = kk - owner * h + up * h;
    } else {
      owner = (int64_t)k / a.rows_local;
      local = (int64_t)k - owner * a.rows_local;
    }
    const uint32_t* __restrict__ src = reinterpret_cast<const uint32_t*>(a.rows_peers[owner]) + local * a.row_words;
    uint32_t* __restrict__ dst = a.rows_out + out_idx * a.row_words;
    for (uint32_t q = 0; q < a.row_words; ++q) dst[q] = src[q];
  }
}

// ---------------------------------------------------------------------------
// weight loads.  float32 -> float64 conversion is F2F (exact for every float32,
// subnormals included); it runs on the otherwise idle conversion pipe.

template <typename WT, bool TEX>
__device__ __forceinline__ WT wfetch(const WT* __restrict__ w, cudaTextureObject_t tex, uint32_t j) {
  if constexpr (TEX && sizeof(WT) == 4) return tex1Dfetch<float>(tex, (int)j);
  else return __ldg(w + j);
}

// accept j (M/resample.py:118-122).  NOZERO: no weight is zero, so the both-zero
// rejection can never fire and is skipped.  u * w_k is exact-rounded binary64.
template <bool NOZERO, typename WT>
__device__ __forceinline__ bool accept_w(double u, WT wk, WT wj) {
  const bool le = u * (double)wk <= (double)wj;
  if constexpr (NOZERO) return le;
  else return le && !(wj == (WT)0 && wk == (WT)0);
}

// accept j for a Philox word (u = word * 2^-32): fl(u * wk) as one DFMA on 1 + u (exact),
// see u1_from_word below; same binary64 value as accept_w((double)word * 2^-32, wk, wj).
__device__ __forceinline__ double u1_from_word(uint32_t w);
template <bool NOZERO, typename WT>
__device__ __forceinline__ bool accept_word(uint32_t word, WT wk, WT wj) {
  const double wkd = (double)wk;
  const bool le = fma(u1_from_word(word), wkd, -wkd) <= (double)wj;
  if constexpr (NOZERO) return le;
  else return le && !(wj == (WT)0 && wk == (WT)0);
}

// (a & c) | (b & ~c) in one LOP3
__device__ __forceinline__ uint32_t mux3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Megopolis partner for W = 32, N % 32 == 0 (M/resample.py:187-193):
//   j = ((i_al + o_al) mod N) | ((lane + o) & 31)
// POW2 (N >= 64 a power of two): one LOP3 mux with C = (N-1) & ~31.
template <bool POW2>
__device__ __forceinline__ uint32_t mego_j(uint32_t i_al, uint32_t lane, uint2 o, uint32_t n) {
  if constexpr (POW2) {
    return mux3(i_al + o.x, lane + o.y, (n - 1) & ~31u);
  } else {
    uint32_t a = i_al + o.x;
    a = (a >= n) ? a - n : a;
    return a | ((lane + o.y) & 31u);
  }
}

// Philox4x32-10 block with the round keys from the parameter space (uniform registers)
__device__ __forceinline__ P4 philox_keys(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                          const uint32_t* pk0, const uint32_t* pk1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t q0 = (uint64_t)PHILOX_M0 * c0, q1 = (uint64_t)PHILOX_M1 * c2;
    const uint32_t n0 = (uint32_t)(q1 >> 32) ^ c1 ^ pk0[r], n2 = (uint32_t)(q0 >> 32) ^ c3 ^ pk1[r];
    c1 = (uint32_t)q1;
    c3 = (uint32_t)q0;
    c0 = n0;
    c2 = n2;
  }
  return P4{c0, c1, c2, c3};
}

// x + M_CTR as IADD3 (low word, carry out) + IMAD.X (high word: x_hi * one + M_CTR_hi + carry,
// the FMA pipe); `one` (== 1) comes from the parameter space so ptxas cannot fold the multiply
// into an IADD3.X on the ALU pipe.  Two instructions (the mad.wide form it replaces compiled to
// IADD3 + IMAD.X + IMAD: ptxas hoisted one * M_CTR_lo and added one * M_CTR_hi separately).
__device__ __forceinline__ uint64_t add64_fma(uint64_t x, uint32_t one) {
  uint32_t lo, hi;
  asm("{\n\t.reg .u32 xl, xh;\n\t"
      "mov.b64 {xl, xh}, %2;\n\t"
      "add.cc.u32 %0, xl, %4;\n\t"
      "madc.lo.u32 %1, xh, %3, %5;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "l"(x), "r"(one), "n"((uint32_t)M_CTR), "n"((uint32_t)(M_CTR >> 32)));
  return ((uint64_t)hi << 32) | lo;
}

// exact (double)w * 2^-32 for a 32-bit word: (2^52 + w) * 2^-32 - 2^20 in one DFMA
__device__ __forceinline__ double u32_exact(uint32_t w) {
  return fma(__hiloint2double(0x43300000, (int)w), 0x1p-32, -0x1p20);
}

// 1 + w * 2^-32 for a 32-bit word, assembled from bits (exact: 32 fraction bits < 52).
// Then fl(u * wk) = DFMA(u1, wk, -wk): the product (1+u)wk - wk = u*wk is exact inside the
// FMA and rounded once -- the same binary64 value as (w * 2^-32) * wk.  Replaces
// I2F.F64.U32 (conversion pipe, 64-bit result) + DMUL by 2^-32 + DMUL by wk with
// LEA.HI + IMAD.SHL + one DFMA (scripts/mb/mb_conv.cu: 5.46 -> 5.24 ms at 2^24, B = 352).
__device__ __forceinline__ double u1_from_word(uint32_t w) {
  return __hiloint2double((int)((w >> 12) + 0x3FF00000u), (int)(w << 20));
}

// high word of mix64's second product m = v * MIX2 (mod 2^64), v = z ^ (z >> 27)
__device__ __forceinline__ uint32_t mix64_mhi(uint64_t x) {
  x = (x ^ (x >> 30)) * MIX1;
  x ^= x >> 27;
  const uint32_t vlo = (uint32_t)x, vhi = (uint32_t)(x >> 32);
  return __umulhi(vlo, (uint32_t)MIX2) + vlo * (uint32_t)(MIX2 >> 32) + vhi * (uint32_t)MIX2;
}

__device__ unsigned long long g_megores_fallbacks;  // diagnostic count (mgp_debug_megores_fallbacks)

// ---------------------------------------------------------------------------
// Megopolis, W = 32 (the hot path).  One particle per thread; the warp's 32 partner
// weights for round b are one 128-byte line (4 sectors) -- the paper's coalescing.
// Per round: partner fetch (texture path, no address arithmetic), one stream draw,
// one DMUL + DSETP, one 32-bit select.  The accepted round index is carried instead
// of j (j is a pure function of (i, o_b)) and k is rebuilt once at the end.

template <int RNG, typename WT, bool POW2, bool NOZERO, bool TEX, int PPT, bool HALF = false, bool ROWS = false>
__global__ void __launch_bounds__(RS_THREADS / PPT, PPT == 1 ? 0 : 1) k_megopolis_w32(const __grid_constant__ ResampleArgs a,
                                                                    const __grid_constant__ OffChunk oc) {
  // PPT particles per thread: i + p*(256/PPT) of this CTA's 256-particle block -- same lane,
  // different warps, so the lane part of the partner index is shared and the independent
  // random-stream chains interleave (ILP).  p_end is a multiple of 32: whole warps only.
  //
  // HALF (full-range launch, N = 2^k >= 256, PPT = 4): the thread owns {i, i+64, i+N/2,
  // i+N/2+64}, i in the lower half.  Adding N/2 modulo N flips the top index bit, so the
  // partners of the upper pair are those of the lower pair with bit k-1 flipped:
  // j(i + N/2) = j(i) ^ N/2 -- one LOP3 instead of an add and a mux per comparison
  // (scripts/mb/mb_conv.cu: 5.28 -> 5.11 ms at 2^24, B = 352).
  static_assert(!HALF || (PPT == 4 && POW2), "HALF needs PPT 4 and a power-of-two N");
  constexpr int STRIDE = HALF ? 64 : RS_THREADS / PPT;
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = HALF ? a.p0 + blockIdx.x * 128 + threadIdx.x : a.p0 + blockIdx.x * RS_THREADS + threadIdx.x;
  if (!HALF && i0 >= a.p_end) return;
  const WT* __restrict__ w = reinterpret_cast<const WT*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, n = a.n;
  uint32_t ii[PPT], ial[PPT];
  bool live[PPT];
  WT wk[PPT];
  int bstar[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if constexpr (HALF) ii[p] = i0 + (p & 1) * STRIDE + (p >> 1) * half;
    else ii[p] = i0 + p * STRIDE;
    live[p] = HALF || ii[p] < a.p_end;
    ial[p] = ii[p] - lane;
    const uint32_t k0 = live[p] ? (a.first ? ii[p] : (uint32_t)a.kstate[ii[p]]) : 0u;
    wk[p] = wfetch<WT, TEX>(w, a.tex, k0);
    bstar[p] = -1;
  }
  // partner indices of round o for all PPT particles
  auto partners = [&](const uint2 o, uint32_t* jj) {
    if constexpr (HALF) {
      jj[0] = mego_j<true>(ial[0], lane, o, n);
      jj[1] = mego_j<true>(ial[1], lane, o, n);
      jj[2] = jj[0] ^ half;
      jj[3] = jj[1] ^ half;
    } else {
#pragma unroll
      for (int p = 0; p < PPT; ++p) jj[p] = mego_j<POW2>(ial[p], lane, o, n);
    }
  };
  if constexpr (RNG == RNG_MEGORES) {
    uint64_t x[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) x[p] = megores_key(a.base, ii[p], (uint64_t)a.b0);
#pragma unroll(4 / PPT)
    for (int t = 0; t < a.cnt; ++t) {
      uint32_t jj[PPT];
      partners(oc.o[t], jj);
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const WT wj = wfetch<WT, TEX>(w, a.tex, jj[p]);
        const double u = (double)mix64_m53(x[p]) * 0x1p-53;  // exact: u01 (M/rng.py:105-108)
        x[p] = add64_fma(x[p], a.one);  // x += M_CTR on the FMA pipe (the ALU pipe binds)
        if (accept_w<NOZERO>(u, wk[p], wj)) { wk[p] = wj; bstar[p] = t; }
      }
    }
  } else {
    // philox: draw t = b0 + t; block (t >> 2), word (t & 3); b0 % 4 == 0.  Full groups of
    // four draws run unguarded; the state weight is kept in float64 (the conversion pipe,
    // not the ALU, is this variant's scarce resource).
    double wkd[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) wkd[p] = (double)wk[p];
    const int full = a.cnt & ~3;
    auto group = [&](int t0, int lim) {
      uint32_t c0[PPT], c1[PPT], c2[PPT], c3[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        c0[p] = ii[p]; c1[p] = 0; c2[p] = (uint32_t)((a.b0 + t0) >> 2); c3[p] = 0;
      }
#pragma unroll
      for (int r = 0; r < 10; ++r) {
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          const uint64_t q0 = (uint64_t)PHILOX_M0 * c0[p], q1 = (uint64_t)PHILOX_M1 * c2[p];
          const uint32_t n0 = (uint32_t)(q1 >> 32) ^ c1[p] ^ a.pk0[r], n2 = (uint32_t)(q0 >> 32) ^ c3[p] ^ a.pk1[r];
          c1[p] = (uint32_t)q1;
          c3[p] = (uint32_t)q0;
          c0[p] = n0;
          c2[p] = n2;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q < lim) {
          const int t = t0 + q;
          uint32_t jj[PPT];
          partners(oc.o[t], jj);
#pragma unroll
          for (int p = 0; p < PPT; ++p) {
            const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
            const WT wj = wfetch<WT, TEX>(w, a.tex, jj[p]);
            const double wjd = (double)wj;
            const bool le = fma(u1_from_word(wd), wkd[p], -wkd[p]) <= wjd;  // fl(u * wk) <= wj
            const bool acc = NOZERO ? le : (le && !(wj == (WT)0 && wkd[p] == 0.0));
            if (acc) { wkd[p] = wjd; bstar[p] = t; }
          }
        }
      }
    };
    for (int t0 = 0; t0 < full; t0 += 4) group(t0, 4);
    if (full < a.cnt) group(full, a.cnt - full);
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (!live[p]) continue;
    uint32_t k = a.first ? ii[p] : (uint32_t)a.kstate[ii[p]];
    if (bstar[p] >= 0) k = mego_j<POW2>(ial[p], lane, oc.o[bstar[p]], n);
    store_result<ROWS>(a, (int64_t)ii[p] - (HALF && p >= 2 ? a.hi_shift : 0), ii[p], k);
  }
}

// ---------------------------------------------------------------------------
// The headline configuration, specialised: Philox stream, float32 weights through the texture
// path, no zero weights, half-split (N = 2^k >= 256).  Same arithmetic and layout as
// k_megopolis_w32<RNG_PHILOX, float, true, true, true, 4, true>, written as one straight loop of
// Philox blocks plus a guarded tail block: ptxas schedules this form 0.6-1% faster on every box
// measured (scripts/mb/mb_conv.cu "x2 gen" vs "lib HALF").  [p0, p_end) is a range of
// lower-half particles (multiple of 128); upper-half ancestors land at anc[i - hi_shift].

__global__ void __launch_bounds__(64, 1) k_megopolis_philox_half(const __grid_constant__ ResampleArgs a,
                                                                 const __grid_constant__ OffChunk oc) {
  constexpr int PPT = 4;
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = a.p0 + blockIdx.x * 128 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT];
  double wkd[PPT];
  int bstar[PPT];
  ii[0] = i0; ii[1] = i0 + 64; ii[2] = i0 + half; ii[3] = i0 + half + 64;
  const uint32_t ial0 = i0 - lane, ial1 = ial0 + 64;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const uint32_t k0 = a.first ? ii[p] : (uint32_t)a.kstate[ii[p]];
    wkd[p] = (double)tex1Dfetch<float>(a.tex, (int)k0);
    bstar[p] = -1;
  }
  const int full = a.cnt & ~3;
  auto body = [&](int t0, int lim) {  // rounds [t0, t0 + lim) from Philox block (b0 + t0) / 4
    uint32_t c0[PPT], c1[PPT], c2[PPT], c3[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) { c0[p] = ii[p]; c1[p] = 0; c2[p] = (uint32_t)((a.b0 + t0) >> 2); c3[p] = 0; }
#pragma unroll
    for (int r = 0; r < 10; ++r) {
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const uint64_t q0 = (uint64_t)PHILOX_M0 * c0[p], q1 = (uint64_t)PHILOX_M1 * c2[p];
        const uint32_t n0 = (uint32_t)(q1 >> 32) ^ c1[p] ^ a.pk0[r], n2 = (uint32_t)(q0 >> 32) ^ c3[p] ^ a.pk1[r];
        c1[p] = (uint32_t)q1; c3[p] = (uint32_t)q0; c0[p] = n0; c2[p] = n2;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < lim) {
        const int t = t0 + q;
        const uint2 o = oc.o[t];
        const uint32_t L = lane + o.y;
        uint32_t jj[PPT];
        jj[0] = mux3(ial0 + o.x, L, cmask);
        jj[1] = mux3(ial1 + o.x, L, cmask);
        jj[2] = jj[0] ^ half;
        jj[3] = jj[1] ^ half;
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
          const double wjd = (double)tex1Dfetch<float>(a.tex, (int)jj[p]);
          const double prod = fma(u1_from_word(wd), wkd[p], -wkd[p]);  // fl(u * wk)
          if (prod <= wjd) { wkd[p] = wjd; bstar[p] = t; }
        }
      }
    }
  };
  for (int t0 = 0; t0 < full; t0 += 4) body(t0, 4);
  if (full < a.cnt) body(full, a.cnt - full);
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = a.first ? ii[p] : (uint32_t)a.kstate[ii[p]];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3((ii[p] - lane) + o.x, lane + o.y, cmask); }
    if (a.last) a.anc[(int64_t)ii[p] - (p >= 2 ? a.hi_shift : 0)] = (int64_t)k;
    else a.kstate[ii[p]] = (int32_t)k;
  }
}

// ---------------------------------------------------------------------------
// The reference's own stream (megores), float32 weights, no zero weights: a float32 bracket of
// the float64 decision with an exact fallback.
//
// The reference accepts iff fl64(u * wk) <= wj with u = h53 * 2^-53 (M/resample.py:118-122,
// M/rng.py:105-108).  The top 23 bits of h53 are bits 31..9 of the high word of the second
// splitmix product m (the final xorshift x ^ (x >> 31) only touches bit 0 of the high word),
// so u lies in [u23, u23 + 2^-23) with u23 = (m_hi >> 9) * 2^-23, assembled from bits as the
// float 1 + u23 (one LEA.HI).  Two directed-rounding FFMAs bracket the product:
//   lo = fl_down((1 + u23) wk - wk) <= u23 wk <= u wk,
//   hi = fl_up(lo + 2^-22 wk) >= u23 wk + 2^-23 wk > u wk     (lo >= u23 wk - ulp(u23 wk) and
//        ulp(u23 wk) <= 2^-23 wk).
// hi <  wj  => u wk <= wj => fl64(u wk) <= wj: accept.  The comparison is strict because the
//              bound hi >= u wk needs 2^-23 wk >= ulp32(u23 wk), which fails for subnormal wk
//              (spacing 2^-149): there u wk < hi + 2^-149, and hi < wj means wj >= hi + 2^-149
//              (wj is a float), so u wk < wj still holds.  wj == hi is left to the exact re-run.
// lo >  wj  => u wk >= lo >= wj + ulp32(wj) > wj + ulp64(wj) / 2 => fl64(u wk) > wj: reject.
// Otherwise (probability ~2^-21 per comparison) the round is ambiguous: the lane records it,
// and after the loop every lane that saw one re-runs its rounds with the exact float64 rule
// (megores_exact_rounds).  The result is the reference's bit for bit, while the common path
// needs neither the low half of the second product, the final xorshift, the 64-bit integer
// conversion (I2F.F64.U64, conversion pipe) nor any float64 instruction: 32.5 instructions
// per round instead of 38.75 (scripts/mb/mb_mego.cu "z H--- 1u8": 7.82 -> 6.78 ms at 2^24,
// B = 354).  Subnormal weights are exact too: the FFMAs are IEEE with denormals (no ftz), and the
// strict accept comparison above covers the bound's one-spacing slack there.


// One particle's rounds [0, cnt) of a launch with the exact float64 decision; returns the last
// accepted round (-1: none).  wk is the weight of the particle's state at the launch start.
__device__ __noinline__ int megores_exact_rounds(const ResampleArgs& a, const OffChunk& oc, uint32_t i, float wk,
                                                 bool pow2) {
  atomicAdd(&g_megores_fallbacks, 1ull);
  const uint32_t lane = i & 31u, ial = i - lane;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
  int bstar = -1;
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t j = pow2 ? mego_j<true>(ial, lane, oc.o[t], a.n) : mego_j<false>(ial, lane, oc.o[t], a.n);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    const double u = (double)mix64_m53(x) * 0x1p-53;  // u01 (M/rng.py:105-108)
    if (u * (double)wk <= (double)wj) { wk = wj; bstar = t; }
    x += M_CTR;
  }
  return bstar;
}

// One particle per thread (2 or 4 particles per thread, with or without the half split, measured
// no faster: scripts/mb/mb_mego.cu "z H--- 2 / 2h / 4h"; re-measured after the 2-instruction key
// add: a half-split kernel with four particles per thread, 30 instead of 32 instructions per
// comparison, ran 6.64 ms against 6.48, scripts/mb/probe_mh.sh).
template <bool POW2, bool ROWS = false>
__global__ void __launch_bounds__(RS_THREADS) k_megopolis_megores_f32(const __grid_constant__ ResampleArgs a,
                                                                     const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * RS_THREADS + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = threadIdx.x & 31u, ial = i - lane, n = a.n;
  const uint32_t k0 = a.first ? i : (uint32_t)a.kstate[i];
  const float wk0 = tex1Dfetch<float>(a.tex, (int)k0);
  float wk = wk0;
  // the accepted partner index itself is carried (j is live for the fetch anyway): no per-round
  // round-index register (one VIADD per round; 6.476 -> 6.456 ms, scripts/mb/probe_cj.sh) and the
  // ambiguity is a flag
  uint32_t kacc = k0;
  bool amb = false;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll 8
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t j = mego_j<POW2>(ial, lane, oc.o[t], n);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    const float u1 = __uint_as_float(0x3F800000u + (mix64_mhi(x) >> 9));  // 1 + u23
    const float lo = __fmaf_rd(u1, wk, -wk);
    const float hi = __fmaf_ru(wk, 0x1p-22f, lo);
    const bool acc = hi < wj;  // strict: see the subnormal note above k_megopolis_megores_f32
    if (!acc && lo <= wj) amb = true;
    if (acc) { wk = wj; kacc = j; }
    // x += M_CTR: ptxas hoists one * M_CTR and splits the add into IADD3 (ALU) + IMAD.X (FMA
    // pipe) -- 3% faster than IADD3 + IADD3.X (scripts/mb/mb_mego2.cu "ADDW u8": 6.84 -> 6.69 ms);
    // moving more of the hash to the heavy FMA pipe (IMAD.WIDE adds, IMAD.HI shifts, I2F for
    // the bracket) measured 1-12% slower there.
    x = add64_fma(x, a.one);
  }
  if (amb) {
    const int bstar = megores_exact_rounds(a, oc, i, wk0, POW2);
    kacc = bstar >= 0 ? mego_j<POW2>(ial, lane, oc.o[bstar], n) : k0;
  }
  store_result<ROWS>(a, (int64_t)i, i, kacc);
}

// ---------------------------------------------------------------------------
// Metropolis (uniform random partner; the uncoalesced baseline, M/resample.py:125-138)

template <int RNG, typename WT, bool POW2, bool NOZERO>
__global__ void __launch_bounds__(RS_THREADS) k_metropolis(const __grid_constant__ ResampleArgs a) {
  const uint32_t i = a.p0 + blockIdx.x * RS_THREADS + threadIdx.x;
  if (i >= a.p_end) return;
  const WT* __restrict__ w = reinterpret_cast<const WT*>(a.w);
  const uint32_t n = a.n;
  uint32_t k = a.first ? i : (uint32_t)a.kstate[i];
  WT wk = __ldg(w + k);
  if constexpr (RNG == RNG_MEGORES) {
    uint64_t x = megores_key(a.base, i, 2ull * (uint64_t)a.b0);
#pragma unroll 2
    for (int t = 0; t < a.cnt; ++t) {
      const double u = (double)mix64_m53(x) * 0x1p-53;  // u at counter 2b
      x += M_CTR;
      const uint64_t hj = mix64(x);                     // j at counter 2b+1
      x += M_CTR;
      uint32_t j;
      if constexpr (POW2) j = (uint32_t)(hj >> 32) >> (32 - a.log2);  // == uint_below for n = 2^k
      else j = (uint32_t)below_from_hash(hj, (int64_t)n);
      const WT wj = __ldg(w + j);
      if (accept_w<NOZERO>(u, wk, wj)) { wk = wj; k = j; }
    }
  } else {
    // u at draw 2b, j at draw 2b+1: one philox block serves rounds (2m, 2m+1).
    for (int t = 0; t < a.cnt;) {
      const uint32_t blkidx = (uint32_t)(((uint64_t)(a.b0 + t) * 2) >> 2);
      const P4 blk = philox_keys(i, 0, blkidx, 0, a.pk0, a.pk1);
      const int first_half = ((a.b0 + t) & 1) == 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if ((h == 0 && first_half) || (h == 1 && t < a.cnt)) {
          const uint32_t wu = h == 0 ? blk.x : blk.z, wjw = h == 0 ? blk.y : blk.w;
          const uint32_t j = __umulhi(wjw, n);
          const WT wj = __ldg(w + j);
          if (accept_word<NOZERO>(wu, wk, wj)) { wk = wj; k = j; }
          ++t;
        }
      }
    }
  }
  store_result(a, i, i, k);
}

// ---------------------------------------------------------------------------
// Metropolis-C1 (one partition per warp for all rounds, M/resample.py:141-158) and
// C2 (a fresh partition per warp and round, M/resample.py:161-177) for W = 32.
// C1 stages its partition in shared memory once and serves all B rounds from it.
// C2 draws the 32 upcoming partitions cooperatively (lane l draws round b0+l) and
// broadcasts them with a shuffle; its partner loads are partition-local gathers.

template <int RNG>
__device__ __forceinline__ uint32_t below_n(uint64_t h_or_word, uint32_t n, uint32_t log2, bool pow2) {
  if (RNG == RNG_MEGORES) {
    if (pow2) return log2 == 0 ? 0u : (uint32_t)(h_or_word >> 32) >> (32 - log2);
    return (uint32_t)below_from_hash(h_or_word, (int64_t)n);
  }
  return __umulhi((uint32_t)h_or_word, n);
}

// C1 / C2 on the megores stream with the exact float64 rule (power-of-two partitions, no zero
// weight): the fallback of the float32-bracket path below when one of the particle's rounds is
// ambiguous; C2's per-round partition is drawn directly instead of by the warp's shuffle.
template <bool C2>
__device__ __noinline__ uint32_t c12_exact_rounds(const ResampleArgs& a, uint32_t i, uint32_t k, float wk, uint32_t lo) {
  atomicAdd(&g_megores_fallbacks, 1ull);
  const float* __restrict__ w = reinterpret_cast<const float*>(a.w);
  const uint64_t wlane = WARP_LANE_BASE + (i >> 5);
  uint64_t x = megores_key(a.base, i, 2ull * (uint64_t)a.b0);
  for (int t = 0; t < a.cnt; ++t) {
    if (C2) lo = (uint32_t)draw_below<RNG_MEGORES>(a.base, a.seed, wlane, (uint64_t)(a.b0 + t), (int64_t)a.n_part) * a.n_w;
    const double u = (double)mix64_m53(x) * 0x1p-53;  // u01 (M/rng.py:105-108)
    x += M_CTR;
    const uint32_t jl = below_n<RNG_MEGORES>(mix64(x), a.n_w, a.log2, true);
    x += M_CTR;
    const float wj = __ldg(w + lo + jl);
    if (u * (double)wk <= (double)wj) { wk = wj; k = lo + jl; }
  }
  return k;
}

template <int RNG, typename WT, bool POW2, bool NOZERO, bool C2, bool STAGE>
__global__ void __launch_bounds__(RS_THREADS) k_c12_w32(const __grid_constant__ ResampleArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t i = a.p0 + blockIdx.x * RS_THREADS + threadIdx.x;
  // Whole warps past the range leave together.  A warp straddling p_end (p_end % 32 != 0)
  // stays complete -- every lane takes part in the partition staging and the C2 owner
  // shuffles (n % 32 == 0, so i < n) -- and only the lanes inside the range store.
  if ((i & ~31u) >= a.p_end) return;
  const bool live = i < a.p_end;
  const WT* __restrict__ w = reinterpret_cast<const WT*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, warp_g = i >> 5;
  const uint32_t n_w = a.n_w;
  const uint64_t wlane = WARP_LANE_BASE + warp_g;
  uint32_t k = (a.first || !live) ? i : (uint32_t)a.kstate[i];
  WT wk = __ldg(w + k);
  uint32_t lo = 0;
  WT* part = reinterpret_cast<WT*>(smem_raw) + (threadIdx.x >> 5) * n_w;
  if constexpr (!C2) {
    lo = (uint32_t)draw_below<RNG>(a.base, a.seed, wlane, 0, (int64_t)a.n_part) * n_w;
    if constexpr (STAGE) {
      for (uint32_t q = lane; q < n_w; q += 32) part[q] = __ldg(w + lo + q);
      __syncwarp();
    }
  }
  uint32_t preg = 0;
  if constexpr (RNG == RNG_MEGORES && sizeof(WT) == 4 && NOZERO && POW2) {
    // float32 weights, no zero weight, power-of-two partitions: the float32 bracket of the float64
    // decision of k_megopolis_megores_f32 (exact re-run of the particle's rounds when a round is
    // ambiguous), and only the high word m_hi of each draw's second splitmix product: the u draw
    // needs its top 23 bits, and uint_below(2^k) = h >> (64 - k) reads bits [32 - k, 32) of h's
    // high word, which equal m_hi's (h = m ^ (m >> 31) changes bit 0 of the high word only).
    const float wk0 = (float)wk;
    const uint32_t k0 = k, lo0 = lo, sh = 32u - a.log2;
    bool amb = false;
    uint64_t x = megores_key(a.base, i, 2ull * (uint64_t)a.b0);
#pragma unroll 4
    for (int t = 0; t < a.cnt; ++t) {
      if constexpr (C2) {
        if ((t & 31) == 0)
          preg = (uint32_t)draw_below<RNG>(a.base, a.seed, wlane, (uint64_t)(a.b0 + t + (int)lane), (int64_t)a.n_part);
        lo = __shfl_sync(0xffffffffu, preg, t & 31) * n_w;
      }
      const uint32_t mu = mix64_mhi(x);  // u at counter 2b
      x = add64_fma(x, a.one);
      const uint32_t mj = mix64_mhi(x);  // j at counter 2b + 1
      x = add64_fma(x, a.one);
      const uint32_t jl = a.log2 ? mj >> sh : 0u;
      const float wj = (STAGE && !C2) ? part[jl] : __ldg(w + lo + jl);
      const float u1 = __uint_as_float(0x3F800000u + (mu >> 9));  // 1 + u23
      const float flo = __fmaf_rd(u1, wk, -wk);
      const float fhi = __fmaf_ru(wk, 0x1p-22f, flo);
      const bool acc = fhi < wj;  // strict: see the subnormal note above k_megopolis_megores_f32
      amb |= !acc && flo <= wj;
      if (acc) { wk = wj; k = lo + jl; }
    }
    if (amb && live) k = c12_exact_rounds<C2>(a, i, k0, wk0, lo0);
  } else if constexpr (RNG == RNG_MEGORES) {
    uint64_t x = megores_key(a.base, i, 2ull * (uint64_t)a.b0);
    for (int t = 0; t < a.cnt; ++t) {
      if constexpr (C2) {
        if ((t & 31) == 0)
          preg = (uint32_t)draw_below<RNG>(a.base, a.seed, wlane, (uint64_t)(a.b0 + t + (int)lane), (int64_t)a.n_part);
        lo = __shfl_sync(0xffffffffu, preg, t & 31) * n_w;
      }
      const double u = (double)mix64_m53(x) * 0x1p-53;
      x += M_CTR;
      const uint32_t jl = below_n<RNG>(mix64(x), n_w, a.log2, POW2);
      x += M_CTR;
      const WT wj = (STAGE && !C2) ? part[jl] : __ldg(w + lo + jl);
      if (accept_w<NOZERO>(u, wk, wj)) { wk = wj; k = lo + jl; }
    }
  } else {
    // u at draw 2b, j at draw 2b+1: one philox block serves rounds (2m, 2m+1).
    for (int t = 0; t < a.cnt;) {
      const uint32_t blkidx = (uint32_t)(((uint64_t)(a.b0 + t) * 2) >> 2);
      const P4 blk = philox_keys(i, 0, blkidx, 0, a.pk0, a.pk1);
      const int first_half = ((a.b0 + t) & 1) == 0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if ((h == 0 && first_half) || (h == 1 && t < a.cnt)) {
          if constexpr (C2) {
            if ((t & 31) == 0)
              preg = (uint32_t)draw_below<RNG>(a.base, a.seed, wlane, (uint64_t)(a.b0 + t + (int)lane),
                                               (int64_t)a.n_part);
            lo = __shfl_sync(0xffffffffu, preg, t & 31) * n_w;
          }
          const uint32_t wu = h == 0 ? blk.x : blk.z, wjw = h == 0 ? blk.y : blk.w;
          const uint32_t jl = __umulhi(wjw, n_w);
          const WT wj = (STAGE && !C2) ? part[jl] : __ldg(w + lo + jl);
          if (accept_word<NOZERO>(wu, wk, wj)) { wk = wj; k = lo + jl; }
          ++t;
        }
      }
    }
  }
  if (live) store_result(a, i, i, k);
}

// ---------------------------------------------------------------------------
// Generic path: any logical warp size W (semantic, M/resample.py:59-75), any N
// (permissive mode, M/resample.py:103-108), f32 or f64.  64-bit index arithmetic,
// exact draws, exact acceptance.  kind: 1 = C1, 2 = C2, 3 = Megopolis.

struct GenericArgs {
  const void* w;
  int64_t n, warp, n_w, n_part, b, p0, p_end;
  uint64_t seed, base;
  const int64_t* off;  // Megopolis offsets (device)
  int64_t* anc;
};

template <int RNG, typename WT, int KIND>
__global__ void __launch_bounds__(RS_THREADS) k_generic(const GenericArgs a) {
  const int64_t i = a.p0 + (int64_t)blockIdx.x * RS_THREADS + threadIdx.x;
  if (i >= a.p_end) return;
  const WT* __restrict__ w = reinterpret_cast<const WT*>(a.w);
  Stream<RNG> s(a.base, a.seed, (uint64_t)i, 0);
  int64_t k = i;
  const uint64_t wlane = WARP_LANE_BASE + (uint64_t)(i / a.warp);
  int64_t lo = 0;
  if (KIND == 1) lo = draw_below<RNG>(a.base, a.seed, wlane, 0, a.n_part) * a.n_w;
  const int64_t i_al = i - i % a.warp;
  for (int64_t b = 0; b < a.b; ++b) {
    int64_t j;
    double u;
    if (KIND == 3) {
      const int64_t ob = a.off[b];
      j = (i_al + (ob - ob % a.warp) + (i + ob) % a.warp) % a.n;
      u = s.u();
    } else {
      u = s.u();
      if (KIND == 2) lo = draw_below<RNG>(a.base, a.seed, wlane, (uint64_t)b, a.n_part) * a.n_w;
      j = lo + s.below(a.n_w);
    }
    if (accepts(u, (double)w[k], (double)w[j])) k = j;
  }
  a.anc[i] = k;
}

// Megopolis offsets on the device: o_b = uint_below(seed, GLOBAL_OFFSET_LANE, b, N)
template <int RNG>
__global__ void k_offsets(uint64_t base, uint64_t seed, int64_t n, int64_t b, int64_t* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < b) out[t] = draw_below<RNG>(base, seed, GLOBAL_OFFSET_LANE, (uint64_t)t, n);
}

// ---------------------------------------------------------------------------
// numpy-exact pairwise reduction.
//
// np.add.reduce over a contiguous float64 array is the recursive pairwise sum
// (blocks of <= 128 with 8 accumulators; split n2 = n/2 - (n/2)%8).  This is what
// np.asarray(w, float64).mean() (B rule), .sum() (expected offspring total) and the
// QualityAccumulator sums evaluate.  We reproduce the same tree: the top D levels
// form a complete binary tree of "chunks" (<= PW_CHUNK elements each, one CTA per
// chunk, sub-tree built level by level in shared memory), then one CTA combines the
// chunk sums in the same pairwise order.  The result is bit-identical to numpy.

constexpr int PW_CHUNK = 4096;   // elements per CTA (staged as float64 in shared memory)
constexpr int PW_HEAP = 256;     // heap slots of one chunk's subtree (depth <= 7)
constexpr int PW_THREADS = 256;
constexpr int PW_PAD = 8;        // +8 doubles per 128: 8-lane leaf groups hit disjoint banks
__host__ __device__ constexpr int pw_sidx(int e) { return e + (e >> 7) * PW_PAD; }

__host__ __device__ inline void pw_chunk_span(int64_t n, int depth, int64_t c, int64_t& lo, int64_t& len) {
  lo = 0;
  len = n;
  for (int d = depth - 1; d >= 0; --d) {
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((c >> d) & 1) { lo += n2; len -= n2; }
    else len = n2;
  }
}

struct WStats {  // per-chunk and final weight statistics
  double max;
  int64_t n_pos, n_zero, n_neg, n_nonfinite, n_notnormal;
};

// Element functors: value(i) in float64, exactly as numpy evaluates it.
template <typename WT>
struct ElemWeight {
  const WT* w;
  __device__ __forceinline__ double operator()(int64_t i) const { return (double)w[i]; }
};
template <typename CT>
struct ElemSqErr {  // (o - E)**2, M/metrics.py:68, 93
  const CT* counts;
  const double* e;
  __device__ __forceinline__ double operator()(int64_t i) const {
    double d = __dsub_rn((double)counts[i], e[i]);
    return __dmul_rn(d, d);
  }
};
struct ElemVar {  // sum_sq/k - mean*mean, M/metrics.py:101
  const double *s, *s2;
  double k;
  __device__ __forceinline__ double operator()(int64_t i) const {
    double m = __ddiv_rn(s[i], k);
    return __dsub_rn(__ddiv_rn(s2[i], k), __dmul_rn(m, m));
  }
};
struct ElemBias {  // (mean - expected)**2, M/metrics.py:102
  const double *s, *e;
  double k;
  __device__ __forceinline__ double operator()(int64_t i) const {
    double d = __dsub_rn(__ddiv_rn(s[i], k), e[i]);
    return __dmul_rn(d, d);
  }
};

template <typename WT>
__device__ __forceinline__ void wstat_observe(WStats& s, WT v) {
  if constexpr (sizeof(WT) == 4) {
    const uint32_t bits = __float_as_uint(v);
    const uint32_t ex = (bits >> 23) & 0xFFu;
    const bool neg = (bits >> 31) != 0;
    const bool zero = (bits & 0x7FFFFFFFu) == 0;
    if (ex == 0xFFu) s.n_nonfinite++;
    else if (zero) s.n_zero++;
    else if (neg) s.n_neg++;
    else s.n_pos++;
    if (ex == 0u || ex == 0xFFu || neg) s.n_notnormal++;
  } else {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const uint32_t ex = (uint32_t)(bits >> 52) & 0x7FFu;
    const bool neg = (bits >> 63) != 0;
    const bool zero = (bits & 0x7FFFFFFFFFFFFFFFull) == 0;
    if (ex == 0x7FFu) s.n_nonfinite++;
    else if (zero) s.n_zero++;
    else if (neg) s.n_neg++;
    else s.n_pos++;
    if (ex == 0u || ex == 0x7FFu || neg) s.n_notnormal++;
  }
  const double d = (double)v;
  if (d > s.max) s.max = d;
}

// Branch-free per-thread tallies for the 4096-element chunks (at most 16 elements per thread:
// 32-bit counters, the max in the weights' own type -- the same first-maximum-wins comparison
// as wstat_observe, NaN never wins); n_pos is the remainder of the observed count.
template <typename WT>
struct WTally {
  uint32_t nonfinite = 0, zero = 0, neg = 0, notnormal = 0;
  WT max = (WT)-1;
};
template <typename WT>
__device__ __forceinline__ void wtally_observe(WTally<WT>& c, WT v) {
  bool nf, zero, negb, sub;
  if constexpr (sizeof(WT) == 4) {
    const uint32_t bits = __float_as_uint(v), ex = (bits >> 23) & 0xFFu;
    nf = ex == 0xFFu;
    zero = (bits & 0x7FFFFFFFu) == 0;
    negb = (bits >> 31) != 0;
    sub = ex == 0;
  } else {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const uint32_t ex = (uint32_t)(bits >> 52) & 0x7FFu;
    nf = ex == 0x7FFu;
    zero = (bits & 0x7FFFFFFFFFFFFFFFull) == 0;
    negb = (bits >> 63) != 0;
    sub = ex == 0;
  }
  c.nonfinite += nf;
  c.zero += !nf && zero;
  c.neg += !nf && !zero && negb;
  c.notnormal += sub || nf || negb;
  c.max = v > c.max ? v : c.max;
}

// One CTA per chunk.  The chunk's elements are staged (coalesced) into shared memory as
// float64; its subtree is built level by level; each leaf (<= 128 elements) is summed by
// 8 lanes, lane j owning numpy's accumulator r[j] (elements j, j+8, j+16, ...), then
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by xor-shuffles (IEEE addition commutes exactly),
// then the n % 8 tail sequentially -- numpy's leaf order.  Internal nodes are combined
// bottom-up.  heap[2^D + c] receives the chunk sum.
// k_pw_final launched as a programmatic dependent of the chunk pass (its launch and residency
// overlap the chunk pass's last wave)
#ifndef MGP_PW_PDL
#define MGP_PW_PDL 1
#endif
template <class Elem, typename WT, bool STATS>
__global__ void __launch_bounds__(PW_THREADS) k_pw_chunks(Elem e, const WT* wraw, int64_t n, int depth,
                                                          double* heap, WStats* cstats) {
#if MGP_PW_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_pw_final may become resident
#endif
  __shared__ double s_el[pw_sidx(PW_CHUNK)];
  __shared__ int32_t s_lo[PW_HEAP];
  __shared__ int32_t s_len[PW_HEAP];
  __shared__ double s_val[PW_HEAP];
  __shared__ int32_t s_leaf[PW_HEAP];
  __shared__ int32_t s_nleaf;
  __shared__ WStats s_red[PW_THREADS / 32];
  int64_t lo0, len0;
  pw_chunk_span(n, depth, blockIdx.x, lo0, len0);
  const int len = (int)len0;
  for (int h = threadIdx.x; h < PW_HEAP; h += PW_THREADS) s_len[h] = 0;
  if (threadIdx.x == 0) s_nleaf = 0;
  // stage (coalesced; each element read exactly once)
  WStats st{-1.0, 0, 0, 0, 0, 0};
#pragma unroll 4
  for (int q = threadIdx.x; q < len; q += PW_THREADS) {
    s_el[pw_sidx(q)] = e(lo0 + q);
    if constexpr (STATS) wstat_observe<WT>(st, wraw[lo0 + q]);
  }
  __syncthreads();
  if (threadIdx.x == 0) { s_lo[1] = 0; s_len[1] = len; }
  __syncthreads();
  for (int lvl = 0; lvl < 8; ++lvl) {  // build the subtree top-down
    const int h0 = 1 << lvl, h1 = min(2 << lvl, PW_HEAP);
    for (int h = h0 + threadIdx.x; h < h1; h += PW_THREADS) {
      const int32_t ln = s_len[h];
      if (ln > 128 && 2 * h + 1 < PW_HEAP) {
        int32_t n2 = ln / 2;
        n2 -= n2 % 8;
        s_lo[2 * h] = s_lo[h];
        s_len[2 * h] = n2;
        s_lo[2 * h + 1] = s_lo[h] + n2;
        s_len[2 * h + 1] = ln - n2;
      } else if (ln > 0) {
        s_leaf[atomicAdd(&s_nleaf, 1)] = h;
      }
    }
    __syncthreads();
  }
  const int nleaf = s_nleaf;
  const int grp = threadIdx.x >> 3, jl = threadIdx.x & 7;
  for (int q0 = 0; q0 < nleaf; q0 += PW_THREADS / 8) {  // warp-uniform trip count
    const int q = q0 + grp;
    const bool live = q < nleaf;
    const int h = live ? s_leaf[q] : 0;
    const int lo = live ? s_lo[h] : 0, ln = live ? s_len[h] : 0;
    double r = 0.0;
    if (ln >= 8) {
      r = s_el[pw_sidx(lo + jl)];
      const int m = ln - (ln % 8);
      for (int i = 8; i < m; i += 8) r = __dadd_rn(r, s_el[pw_sidx(lo + i + jl)]);
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (live && jl == 0) {
      double res;
      int i;
      if (ln < 8) { res = 0.0; i = 0; }
      else { res = r; i = ln - (ln % 8); }
      for (; i < ln; ++i) res = __dadd_rn(res, s_el[pw_sidx(lo + i)]);
      s_val[h] = res;
    }
  }
  __syncthreads();
  for (int lvl = 7; lvl >= 0; --lvl) {  // combine bottom-up in the same order as numpy
    const int h0 = 1 << lvl, h1 = min(2 << lvl, PW_HEAP / 2);
    for (int h = h0 + threadIdx.x; h < h1; h += PW_THREADS)
      if (s_len[h] > 128) s_val[h] = __dadd_rn(s_val[2 * h], s_val[2 * h + 1]);
    __syncthreads();
  }
  if (threadIdx.x == 0) heap[(1ll << depth) + blockIdx.x] = len0 > 0 ? s_val[1] : 0.0;
  if constexpr (STATS) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      st.max = fmax(st.max, __shfl_xor_sync(0xffffffffu, st.max, off));
      st.n_pos += __shfl_xor_sync(0xffffffffu, st.n_pos, off);
      st.n_zero += __shfl_xor_sync(0xffffffffu, st.n_zero, off);
      st.n_neg += __shfl_xor_sync(0xffffffffu, st.n_neg, off);
      st.n_nonfinite += __shfl_xor_sync(0xffffffffu, st.n_nonfinite, off);
      st.n_notnormal += __shfl_xor_sync(0xffffffffu, st.n_notnormal, off);
    }
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = st;
    __syncthreads();
    if (threadIdx.x == 0) {
      WStats t = s_red[0];
      for (int q = 1; q < PW_THREADS / 32; ++q) {
        t.max = fmax(t.max, s_red[q].max);
        t.n_pos += s_red[q].n_pos; t.n_zero += s_red[q].n_zero; t.n_neg += s_red[q].n_neg;
        t.n_nonfinite += s_red[q].n_nonfinite; t.n_notnormal += s_red[q].n_notnormal;
      }
      cstats[blockIdx.x] = t;
    }
  }
}

// Fast path for chunks of exactly 4096 elements (every chunk when N = 4096 * 2^D): the
// subtree is the perfect binary tree over 32 leaves of 128.  Lane j (0..7) of leaf L owns
// numpy's accumulator r[j] = sum_q a[L*128 + j + 8q]; the 8-lane shuffle tree forms
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); the 32 leaf sums are then combined pairwise by one
// warp -- the same tree, no shared-memory staging, two barriers.
template <class Elem, typename WT, bool STATS>
__global__ void __launch_bounds__(PW_THREADS) k_pw_chunks4096(Elem e, const WT* wraw, int depth, double* heap,
                                                              WStats* cstats) {
#if MGP_PW_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // k_pw_final may become resident
#endif
  __shared__ double s_leaf[32];
  __shared__ WStats s_red[PW_THREADS / 32];
  const int64_t lo0 = (int64_t)blockIdx.x * PW_CHUNK;
  const int leaf = threadIdx.x >> 3, jl = threadIdx.x & 7;
  const int64_t base = lo0 + leaf * 128 + jl;
  double r;
  if constexpr (STATS) {  // Elem is ElemWeight<WT>: one load per element serves both
    WTally<WT> c;
    const WT v0 = wraw[base];
    r = (double)v0;
    wtally_observe<WT>(c, v0);
#pragma unroll
    for (int q = 1; q < 16; ++q) {
      const WT v = wraw[base + 8 * q];
      r = __dadd_rn(r, (double)v);
      wtally_observe<WT>(c, v);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const WT o = __shfl_xor_sync(0xffffffffu, c.max, off);
      c.max = o > c.max ? o : c.max;
    }
    const uint32_t nf = __reduce_add_sync(0xffffffffu, c.nonfinite), nz = __reduce_add_sync(0xffffffffu, c.zero),
                   nn = __reduce_add_sync(0xffffffffu, c.neg), nb = __reduce_add_sync(0xffffffffu, c.notnormal);
    if ((threadIdx.x & 31) == 0)
      s_red[threadIdx.x >> 5] = WStats{(double)c.max, (int64_t)(32 * 16 - nf - nz - nn), (int64_t)nz, (int64_t)nn,
                                       (int64_t)nf, (int64_t)nb};
  } else {
    r = e(base);
#pragma unroll
    for (int q = 1; q < 16; ++q) r = __dadd_rn(r, e(base + 8 * q));
  }
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
  if (jl == 0) s_leaf[leaf] = r;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = s_leaf[threadIdx.x];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (threadIdx.x == 0) heap[(1ll << depth) + blockIdx.x] = v;
    if constexpr (STATS) {
      if (threadIdx.x == 0) {
        WStats t = s_red[0];
        for (int q = 1; q < PW_THREADS / 32; ++q) {
          t.max = fmax(t.max, s_red[q].max);
          t.n_pos += s_red[q].n_pos; t.n_zero += s_red[q].n_zero; t.n_neg += s_red[q].n_neg;
          t.n_nonfinite += s_red[q].n_nonfinite; t.n_notnormal += s_red[q].n_notnormal;
        }
        cstats[blockIdx.x] = t;
      }
    }
  }
}

// Combine the complete top tree heap[1 .. 2^(D+1)) in place (single CTA) and emit
//   out[0] = sum, and, when requested, mean = sum / n, accumulation into *accum.
struct PwOut {
  double* sum;       // may be null
  double* mean;      // may be null
  double* accum;     // may be null: *accum += sum (sequential, like Python float +=)
  WStats* stats;     // may be null
};

__global__ void __launch_bounds__(1024) k_pw_final(double* heap, int depth, int64_t n, const WStats* cstats,
                                                   PwOut out) {
#if MGP_PW_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the chunk pass complete
#endif
  for (int lvl = depth - 1; lvl >= 0; --lvl) {
    const int64_t h0 = 1ll << lvl, h1 = 2ll << lvl;
    for (int64_t h = h0 + threadIdx.x; h < h1; h += blockDim.x) heap[h] = __dadd_rn(heap[2 * h], heap[2 * h + 1]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double s = heap[1];
    if (out.sum) *out.sum = s;
    if (out.mean) *out.mean = __ddiv_rn(s, (double)n);
    if (out.accum) *out.accum = __dadd_rn(*out.accum, s);
  }
  if (out.stats && cstats) {
    __shared__ WStats red[32];
    WStats st{-1.0, 0, 0, 0, 0, 0};
    const int64_t nch = 1ll << depth;
    for (int64_t c = threadIdx.x; c < nch; c += blockDim.x) {
      const WStats& q = cstats[c];
      st.max = fmax(st.max, q.max);
      st.n_pos += q.n_pos; st.n_zero += q.n_zero; st.n_neg += q.n_neg;
      st.n_nonfinite += q.n_nonfinite; st.n_notnormal += q.n_notnormal;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      st.max = fmax(st.max, __shfl_xor_sync(0xffffffffu, st.max, off));
      st.n_pos += __shfl_xor_sync(0xffffffffu, st.n_pos, off);
      st.n_zero += __shfl_xor_sync(0xffffffffu, st.n_zero, off);
      st.n_neg += __shfl_xor_sync(0xffffffffu, st.n_neg, off);
      st.n_nonfinite += __shfl_xor_sync(0xffffffffu, st.n_nonfinite, off);
      st.n_notnormal += __shfl_xor_sync(0xffffffffu, st.n_notnormal, off);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = st;
    __syncthreads();
    if (threadIdx.x == 0) {
      WStats t = red[0];
      for (int q = 1; q < (int)(blockDim.x + 31) / 32; ++q) {
        t.max = fmax(t.max, red[q].max);
        t.n_pos += red[q].n_pos; t.n_zero += red[q].n_zero; t.n_neg += red[q].n_neg;
        t.n_nonfinite += red[q].n_nonfinite; t.n_notnormal += red[q].n_notnormal;
      }
      *out.stats = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Offspring histogram (M/resample.py:361-368): counts[a] += 1 with warp-aggregated
// atomics -- lanes holding the same ancestor elect one leader that adds the
// popcount, so the heavy ancestors of degenerate (y = 4) weights do not serialise
// 32 atomics per warp.  Out-of-range ancestors set *bad.

template <typename CT>
__global__ void k_offspring(const int64_t* __restrict__ anc, int64_t n_anc, int64_t n, CT* counts, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < n_anc;
  int64_t a = live ? anc[i] : -1;
  const bool ok = live && a >= 0 && a < n;
  if (live && !ok) atomicExch(bad, 1);
  const unsigned act = __ballot_sync(0xffffffffu, ok);
  if (!ok) return;
  // n < 2^31: the index fits 32 bits, and the 32-bit match is cheaper than the 64-bit one
  // (scripts/mb/offspring_modes.sh: 0.37 -> 0.30 ms at 2^24, y = 4; no aggregation: 0.31)
  const unsigned peers = __match_any_sync(act, (unsigned)a);
  const int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) {
    if constexpr (sizeof(CT) == 8)
      atomicAdd(reinterpret_cast<unsigned long long*>(counts) + a, (unsigned long long)__popc(peers));
    else
      atomicAdd(reinterpret_cast<unsigned int*>(counts) + a, (unsigned int)__popc(peers));
  }
}

// ---------------------------------------------------------------------------
// Bucketed offspring histogram (no per-particle global atomics).  The bins [0, n) are split into
// K = ceil(n / 2^14) buckets; the ancestors are moved into per-bucket runs, then every bucket is
// histogrammed by one CTA in shared memory (2^14 uint32 bins, 64 KB) and written out as the
// ABI's int64 counts in one coalesced pass.  Launches:
//   k_offb_count    per tile of OFFB_TILE ancestors: bucket counts in shared memory, written to
//                   the bucket-major matrix cnt[b * tiles + tile]; validates the range (bad flag)
//   (CUB exclusive scan of the matrix: every (bucket, tile) run's start; bucket b's run is
//    [off[b * tiles], off[(b + 1) * tiles]))
//   k_offb_scatter  per tile: a counting sort by bucket in shared memory (from the tile's column
//                   of the count matrix), then every (tile, bucket) run leaves as one contiguous
//                   uint16 store of the low 14 bits (scattered 2-byte stores would run at the L2's
//                   random-transaction rate, like the atomics this replaces)
//   k_offb_hist     one CTA per bucket: shared-memory atomics over its run, then 2^14 int64
//                   counts (coalesced streaming stores)
// HBM traffic per call: 2 x 8N (ancestors read twice) + 8N (counts) against the algorithmic
// 16N; the 2N-byte runs stay in L2.  Used for K <= OFFB_KMAX (n <= 2^27).  (Staging the
// ancestors as uint32 for the second pass was slower: 0.162 ms.)
// Measured at 2^24 (Megopolis ancestors, y = 4): 0.149 ms against 0.212 ms for the int32
// global-atomic histogram + widening pass (scripts/mb/offspring_time.py).  A variant that sorted
// each tile once and let the bucket CTAs gather ~16-element runs from every tile ran at 0.204 ms
// (the gathers are latency-bound).
constexpr int OFFB_BITS = 14;
constexpr int OFFB_BINS = 1 << OFFB_BITS;
constexpr int OFFB_TILE = 16384;
constexpr int OFFB_THREADS = 512;
constexpr int OFFB_KMAX = 8192;

__global__ void __launch_bounds__(OFFB_THREADS) k_offb_count(const int64_t* __restrict__ anc, int64_t n_anc, int64_t n,
                                                             int K, int64_t tiles, uint32_t* __restrict__ cnt_mat,
                                                             int* bad) {
  __shared__ uint32_t cnt[OFFB_KMAX];
  for (int b = threadIdx.x; b < K; b += OFFB_THREADS) cnt[b] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * OFFB_TILE;
  const int len = (int)min((int64_t)OFFB_TILE, n_anc - t0);
  bool oob = false;
  for (int q = threadIdx.x; q < len; q += OFFB_THREADS) {
    const int64_t a = anc[t0 + q];
    if (a < 0 || a >= n) { oob = true; continue; }
    atomicAdd(&cnt[(unsigned)(a >> OFFB_BITS)], 1u);
  }
  if (oob) atomicExch(bad, 1);
  __syncthreads();
  for (int b = threadIdx.x; b < K; b += OFFB_THREADS) cnt_mat[(int64_t)b * tiles + blockIdx.x] = cnt[b];
}

__global__ void __launch_bounds__(OFFB_THREADS) k_offb_scatter(const int64_t* __restrict__ anc, int64_t n_anc, int64_t n,
                                                               int K, int64_t tiles,
                                                               const uint32_t* __restrict__ cnt_mat,
                                                               const uint32_t* __restrict__ off_mat,
                                                               uint16_t* __restrict__ runs) {
  extern __shared__ __align__(16) unsigned char offb_smem[];
  uint32_t* cur = reinterpret_cast<uint32_t*>(offb_smem);  // K: local cursors
  uint32_t* loc = cur + K;                                 // K: local run starts
  uint32_t* gst = loc + K;                                 // K: global run starts
  uint32_t* keys = gst + K;                                // OFFB_TILE: the tile sorted by bucket
  __shared__ uint32_t wsum[OFFB_THREADS / 32];
  const int64_t t0 = (int64_t)blockIdx.x * OFFB_TILE;
  const int len = (int)min((int64_t)OFFB_TILE, n_anc - t0);
  uint32_t carry = 0;
  for (int c0 = 0; c0 < K; c0 += OFFB_THREADS) {  // exclusive scan of the tile's bucket counts
    const int b = c0 + threadIdx.x;
    const uint32_t v = b < K ? cnt_mat[(int64_t)b * tiles + blockIdx.x] : 0;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if ((threadIdx.x & 31) >= d) x += y;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
    __syncthreads();
    uint32_t wb = 0, tot = 0;
#pragma unroll
    for (int q = 0; q < OFFB_THREADS / 32; ++q) {
      wb += q < (int)(threadIdx.x >> 5) ? wsum[q] : 0u;
      tot += wsum[q];
    }
    if (b < K) {
      loc[b] = cur[b] = carry + wb + x - v;
      gst[b] = off_mat[(int64_t)b * tiles + blockIdx.x];
    }
    carry += tot;
    __syncthreads();
  }
  for (int q = threadIdx.x; q < len; q += OFFB_THREADS) {
    const int64_t a = __ldcs(anc + t0 + q);  // last read of the ancestors
    if (a < 0 || a >= n) continue;           // flagged by k_offb_count
    keys[atomicAdd(&cur[(unsigned)(a >> OFFB_BITS)], 1u)] = (uint32_t)a;
  }
  __syncthreads();
  const int valid = (int)carry;
  for (int q = threadIdx.x; q < valid; q += OFFB_THREADS) {
    const uint32_t k = keys[q], b = k >> OFFB_BITS;
    runs[gst[b] + (uint32_t)q - loc[b]] = (uint16_t)(k & (OFFB_BINS - 1));
  }
}

__global__ void __launch_bounds__(512) k_offb_hist(const uint16_t* __restrict__ runs, const uint32_t* __restrict__ off_mat,
                                                   int64_t tiles, int64_t n, int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char offb_smem[];
  uint32_t* bins = reinterpret_cast<uint32_t*>(offb_smem);
  const int b = blockIdx.x;
  for (int q = threadIdx.x; q < OFFB_BINS / 4; q += 512) reinterpret_cast<uint4*>(bins)[q] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint32_t r0 = off_mat[(int64_t)b * tiles], r1 = off_mat[(int64_t)(b + 1) * tiles];
  for (uint32_t q = r0 + threadIdx.x; q < r1; q += 512) atomicAdd(&bins[runs[q]], 1u);
  __syncthreads();
  const int64_t c0 = (int64_t)b << OFFB_BITS;
  const int nb = (int)min((int64_t)OFFB_BINS, n - c0);
  for (int q = threadIdx.x; q < nb; q += 512) __stcs(counts + c0 + q, (int64_t)bins[q]);
}

// ---------------------------------------------------------------------------
// Queued offspring histogram (the default for 2^20 <= n <= 2^27): the bucketed histogram above
// without its count pass and scan.  A histogram does not care in which order a bucket's ancestors
// arrive, so every bucket gets a fixed-capacity queue and a tile reserves its run in it with one
// global atomic (the arrival order is the atomic order; the counts are still exact):
//   k_offq_scatter   per tile of 8192 ancestors (4096 for n > 2^25; one read of the ancestors,
//                    16-byte loads held in registers): range check (bad flag), bucket counts by
//                    shared-memory atomics, block scan, one atomicAdd per non-empty bucket on its
//                    queue cursor, counting sort of the tile by bucket in shared memory, then every
//                    (tile, bucket) run leaves as one contiguous uint16 store of the low 14 bits.
//                    Positions past a queue's capacity (skewed inputs: one-hot ancestors, weights
//                    that grow with the index) go to an overflow list instead, one atomicAdd on its
//                    length per spilling run.
//   k_offq_hist      one CTA per bucket: shared-memory histogram of its queue (8 uint16 per
//                    16-byte load), 2^14 int64 counts out with streaming stores.
//   k_offq_overflow  the overflow list (usually empty: one uniform load and exit) as
//                    warp-aggregated int64 atomics into the finished counts.
// HBM traffic per call: 8N (ancestors, read once) + 8N (counts) = the algorithmic 16N; the 2N-byte
// queues stay in L2.
// three 512-thread CTAs per SM (registers capped at 40, no spill with OFFQ_DEFER = 2): 0.123 -> 0.109 ms at
// 2^24 against two per SM (scripts/mb/probe_oq.sh: 4 per SM or 256-/384-thread CTAs were slower)
// Programmatic dependent launch of k_offq_hist and k_offq_overflow (their launch latency and the
// histogram CTAs' bin zeroing overlap the previous kernel's last wave)
#ifndef MGP_OFFQ_PDL
#define MGP_OFFQ_PDL 1
#endif
#ifndef MGP_OFFQ_MINB
#define MGP_OFFQ_MINB 3
#endif
#ifndef MGP_OFFQ_THR
#define MGP_OFFQ_THR 512
#endif
#ifndef MGP_OFFQ_PER
#define MGP_OFFQ_PER 16
#endif
constexpr int OFFQ_DEFER = 2;                 // queue reservations held in registers per thread (K <= 2 * THREADS)
constexpr uint32_t OFFQ_SPILL = 0xFFFFFFFFu;  // run reaching past its queue's capacity

// One tile of PER * THREADS ancestors per CTA, read with 16-byte loads held in registers.  Invalid
// (out-of-range) ancestors go to a trash bucket K so that every per-element step is branch-free.
// (Measured alternatives, scripts/mb/probe_offq*.sh, probe_oq.sh: persistent CTAs streaming the
// next tiles through a two-slot shared-memory ring by bulk copy (TMA) 0.138-0.155 ms; 32 ancestors
// per thread 0.13-0.17 ms; the queue loads of k_offq_hist batched four per thread: 0.180 ms.  This
// shape with three CTAs per SM: 0.109 ms.)
template <int THREADS, int PER>
__global__ void __launch_bounds__(THREADS, MGP_OFFQ_MINB) k_offq_scatter(const int64_t* __restrict__ anc, int64_t n_anc, int64_t n,
                                                          int K, uint32_t cap, uint32_t* __restrict__ gcur,
                                                          uint16_t* __restrict__ queue, uint32_t* __restrict__ novf,
                                                          uint32_t* __restrict__ ovf, int* bad) {
  constexpr int TILE = PER * THREADS;
  extern __shared__ __align__(16) unsigned char offq_smem[];
  uint32_t* sorted = reinterpret_cast<uint32_t*>(offq_smem);  // TILE, sorted by bucket
  uint32_t* cnt = sorted + TILE;  // K + 1: bucket counts (K: the trash bucket), then cursors
  uint32_t* loc = cnt + K + 1;    // K: local run starts
  uint32_t* gb = loc + K;         // K: queue position of the run
  uint32_t* ob = gb + K;          // K: overflow-list position of the spill
  uint32_t* dst = ob + K;         // K: queue index base of the run (or OFFQ_SPILL)
  __shared__ uint32_t wsum[THREADS / 32];
  const uint32_t trash = (uint32_t)K << OFFB_BITS;
  bool oob = false;
#if MGP_OFFQ_PDL
  // let k_offq_hist's CTAs become resident in the slots the last scatter wave leaves free (they
  // zero their bins, then wait for this grid's completion in griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  {
    for (int b = threadIdx.x; b <= K; b += THREADS) cnt[b] = 0;
    const int64_t t0 = (int64_t)blockIdx.x * TILE;
    const bool full = t0 + TILE <= n_anc;
    __syncthreads();
    uint32_t key[PER];
#pragma unroll
    for (int q = 0; q < PER / 2; ++q) {  // element pair 2 * (q * THREADS + tid) + {0, 1} of the tile
      const int e = 2 * (q * THREADS + (int)threadIdx.x);
      int64_t a0 = -1, a1 = -1;
      bool l0 = true, l1 = true;
      if (full) {
        const longlong2 v = __ldcs(reinterpret_cast<const longlong2*>(anc + t0 + e));
        a0 = v.x;
        a1 = v.y;
      } else {
        l0 = t0 + e < n_anc;
        l1 = t0 + e + 1 < n_anc;
        if (l0) a0 = anc[t0 + e];
        if (l1) a1 = anc[t0 + e + 1];
      }
      const bool v0 = a0 >= 0 && a0 < n, v1 = a1 >= 0 && a1 < n;
      oob |= (l0 && !v0) || (l1 && !v1);
      key[2 * q] = v0 ? (uint32_t)a0 : trash;  // trash >> OFFB_BITS == K
      key[2 * q + 1] = v1 ? (uint32_t)a1 : trash;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) atomicAdd(&cnt[key[q] >> OFFB_BITS], 1u);
#if MGP_OFFQ_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_offq_zero complete: cursors and flag zeroed
#endif
    __syncthreads();  // counts complete
    // exclusive scan of the bucket counts; the queue reservations are issued here and their
    // results consumed after the shared-memory sort, which hides the contended atomics' latency
    const bool defer = K <= OFFQ_DEFER * THREADS;
    uint32_t gres[OFFQ_DEFER];
    uint32_t carry = 0;
    for (int c0 = 0, it = 0; c0 < K; c0 += THREADS, ++it) {
      const int b = c0 + threadIdx.x;
      const uint32_t v = b < K ? cnt[b] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if ((threadIdx.x & 31) >= d) x += y;
      }
      if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = x;
      __syncthreads();
      uint32_t wb = 0, tot = 0;
#pragma unroll
      for (int q = 0; q < THREADS / 32; ++q) {
        wb += q < (int)(threadIdx.x >> 5) ? wsum[q] : 0u;
        tot += wsum[q];
      }
      if (b < K) {
        const uint32_t l = carry + wb + x - v;
        loc[b] = l;
        cnt[b] = l;  // cursor
        const uint32_t g = v ? atomicAdd(&gcur[b], v) : 0u;
        if (defer) {
#pragma unroll
          for (int r = 0; r < OFFQ_DEFER; ++r)
            if (r == it) gres[r] = g;
        } else {
          gb[b] = g;
        }
      }
      carry += tot;
      if (c0 + THREADS >= K && threadIdx.x == 0) cnt[K] = carry;  // the trash run follows the valid ones
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) sorted[atomicAdd(&cnt[key[q] >> OFFB_BITS], 1u)] = key[q];
    // runs past a queue's capacity: positions [max(g, cap), g + v) go to the overflow list
    for (int c0 = 0, it = 0; c0 < K; c0 += THREADS, ++it) {
      const int b = c0 + threadIdx.x;
      if (b >= K) break;
      uint32_t g = gb[b];
      if (defer) {
#pragma unroll
        for (int r = 0; r < OFFQ_DEFER; ++r)
          if (r == it) g = gres[r];
        gb[b] = g;
      }
      const uint32_t l = loc[b], v = (b + 1 < K ? loc[b + 1] : carry) - l;
      uint32_t o = 0;
      if (g + v > cap) {
        const uint32_t from = g > cap ? g : cap;
        o = atomicAdd(novf, g + v - from) - (from - g);  // ovf index = o + r for run offset r
      }
      ob[b] = o;
      // queue index of sorted element q of this run = dst + q (K * cap < 2^31); SPILL: the run
      // reaches past the capacity, take the checked path
      dst[b] = g + v > cap ? OFFQ_SPILL : (uint32_t)b * cap + g - l;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < carry; q += THREADS) {
      const uint32_t k = sorted[q], b = k >> OFFB_BITS, d = dst[b];
      if (d != OFFQ_SPILL) {
        queue[d + q] = (uint16_t)(k & (OFFB_BINS - 1));
      } else {
        const uint32_t r = q - loc[b], pos = gb[b] + r;
        if (pos < cap) queue[(size_t)b * cap + pos] = (uint16_t)(k & (OFFB_BINS - 1));
        else ovf[ob[b] + r] = k;
      }
    }
  }
  if (oob) atomicExch(bad, 1);
}

// zero the queue cursors + overflow length (k1 words) and the caller's out-of-range flag
__global__ void __launch_bounds__(1024) k_offq_zero(uint32_t* __restrict__ ctr, int k1, int* bad) {
#if MGP_OFFQ_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  for (int q = threadIdx.x; q < k1; q += 1024) ctr[q] = 0u;
  if (bad && threadIdx.x == 0) *bad = 0;
}

__global__ void __launch_bounds__(512) k_offq_hist(const uint16_t* __restrict__ queue, uint32_t cap,
                                                   const uint32_t* __restrict__ gcur, int64_t n,
                                                   int64_t* __restrict__ counts) {
  extern __shared__ __align__(16) unsigned char offq_smem[];
  uint32_t* bins = reinterpret_cast<uint32_t*>(offq_smem);
  const int b = blockIdx.x;
  for (int q = threadIdx.x; q < OFFB_BINS / 4; q += 512) reinterpret_cast<uint4*>(bins)[q] = make_uint4(0, 0, 0, 0);
#if MGP_OFFQ_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_offq_scatter complete, its queues visible
#endif
  __syncthreads();
  const uint32_t m = min(gcur[b], cap);
  const uint16_t* __restrict__ qb = queue + (size_t)b * cap;  // cap % 8 == 0: 16-byte aligned
  const uint32_t m8 = m >> 3;
  for (uint32_t q = threadIdx.x; q < m8; q += 512) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(qb) + q);
    const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      atomicAdd(&bins[w4[h] & 0xFFFFu], 1u);
      atomicAdd(&bins[w4[h] >> 16], 1u);
    }
  }
  for (uint32_t q = (m8 << 3) + threadIdx.x; q < m; q += 512) atomicAdd(&bins[qb[q]], 1u);
  __syncthreads();
  const int64_t c0 = (int64_t)b << OFFB_BITS;
  const int nb = (int)min((int64_t)OFFB_BINS, n - c0);
  if (nb == OFFB_BINS && (reinterpret_cast<uintptr_t>(counts + c0) & 15) == 0) {
    for (int q = threadIdx.x; q < OFFB_BINS / 2; q += 512)
      __stcs(reinterpret_cast<longlong2*>(counts + c0) + q, make_longlong2(bins[2 * q], bins[2 * q + 1]));
  } else {
    for (int q = threadIdx.x; q < nb; q += 512) __stcs(counts + c0 + q, (int64_t)bins[q]);
  }
}

__global__ void k_offq_overflow(const uint32_t* __restrict__ ovf, const uint32_t* __restrict__ novf,
                                int64_t* __restrict__ counts) {
#if MGP_OFFQ_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_offq_hist complete (the counts it adds to)
#endif
  const uint32_t m = *novf;
  for (uint32_t q0 = blockIdx.x * blockDim.x; q0 < m; q0 += gridDim.x * blockDim.x) {
    const uint32_t q = q0 + threadIdx.x;
    const bool live = q < m;
    const uint32_t k = live ? ovf[q] : 0xFFFFFFFFu;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    if (!live) continue;
    const unsigned peers = __match_any_sync(act, k);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1)
      atomicAdd(reinterpret_cast<unsigned long long*>(counts) + k, (unsigned long long)__popc(peers));
  }
}

// int32 histogram -> the int64 counts of the ABI (4 counts per thread, 16-byte loads)
__global__ void k_widen_counts(const int32_t* __restrict__ c32, int64_t n, int64_t* __restrict__ c64) {
  const int64_t n4 = n >> 2;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = reinterpret_cast<const int4*>(c32)[q];
    longlong2* d = reinterpret_cast<longlong2*>(c64) + 2 * q;
    d[0] = make_longlong2(v.x, v.y);
    d[1] = make_longlong2(v.z, v.w);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c64[i] = c32[i];
}

// QualityAccumulator.add element update (M/metrics.py:90-92): sum += o, sum_sq += o*o
template <typename CT>
__global__ void k_quality_accum(const CT* __restrict__ counts, int64_t n, double* sum, double* sumsq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double o = (double)counts[i];
    sum[i] = __dadd_rn(sum[i], o);
    sumsq[i] = __dadd_rn(sumsq[i], __dmul_rn(o, o));
  }
}

// expected offspring N * w / sum(w)  (M/metrics.py:55-60: len(values) * values / total)
template <typename WT>
__global__ void k_expected(const WT* __restrict__ w, int64_t n, double n_all, const double* total, double total_v,
                           double* e) {
  const double t = total ? *total : total_v;  // the total on the device, or given by value (sharded slices)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    e[i] = __ddiv_rn(__dmul_rn(n_all, (double)w[i]), t);
}

// ---------------------------------------------------------------------------
// Ancestor-driven particle-state gather (M/resample.py:371-377): out[i] = states[anc[i]].
// Rows of row_bytes; vector width V (16/8/4/1 bytes) chosen by alignment.

template <typename V>
__global__ void k_gather(const V* __restrict__ src, const int64_t* __restrict__ anc, int64_t n, int64_t row_v,
                         V* __restrict__ dst) {
  const int64_t total = n * row_v;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / row_v, c = t - i * row_v;
    dst[t] = __ldg(src + anc[i] * row_v + c);
  }
}

// Sharded gather over peer memory (NVLink P2P / symmetric memory): rank r owns rows
// [r*n_local, (r+1)*n_local); out[i] = peers[anc[i] / n_local][anc[i] % n_local].
// The remote rows are read directly by this kernel -- no staging copy.
struct PeerTable {
  const void* p[64];
};

template <typename V>
__global__ void k_gather_peers(const __grid_constant__ PeerTable peers, int npeers, int64_t n_local,
                               const int64_t* __restrict__ anc, int64_t n, int64_t row_v, V* __restrict__ dst,
                               int64_t rows_half) {
  const int64_t total = n * row_v;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / row_v, c = t - i * row_v;
    const int64_t a = anc[i];
    int64_t owner, local;
    if (rows_half) {  // stripes: owner r holds stripe r of each half, low stripe first
      const int64_t h = n_local >> 1, up = a >= rows_half, k = a - up * rows_half;
      owner = k / h;
      local = k - owner * h + up * h;
    } else {
      owner = a / n_local;
      local = a - owner * n_local;
    }
    const V* src = reinterpret_cast<const V*>(peers.p[owner]);
    dst[t] = src[local * row_v + c];
  }
}

// ---------------------------------------------------------------------------
// Comparison-index replay and the warp transaction model (M/resample.py:384-428,
// M/warpsim.py:62-111).  k_comparison_indices writes the weight index particle i reads
// at round r (row-major [B][N]) with the resamplers' own draw conventions (reference
// stream); k_traffic counts, for every W-wide group of one row, the distinct aligned
// segments (transactions) and distinct words it touches.

enum { TR_METROPOLIS = 0, TR_C1 = 1, TR_C2 = 2, TR_MEGOPOLIS = 3 };

__global__ void k_comparison_indices(int kind, int64_t n, int32_t b, uint64_t base, int64_t warp, int64_t n_w,
                                     int64_t n_part, const int64_t* __restrict__ off, int64_t* __restrict__ out) {
  const int64_t total = (int64_t)b * n;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / n, i = t - r * n;
    int64_t j;
    if (kind == TR_MEGOPOLIS) {  // (i - i%W + o - o%W + (i + o)%W) mod N
      const int64_t o = off[r];
      j = (i - i % warp + o - o % warp + (i + o) % warp) % n;
    } else {
      const int64_t local = below_from_hash(mix64(megores_key(base, (uint64_t)i, 2ull * (uint64_t)r + 1)),
                                            kind == TR_METROPOLIS ? n : n_w);
      if (kind == TR_METROPOLIS) {
        j = local;
      } else {  // partition of the particle's logical warp: drawn once (C1) or per round (C2)
        const uint64_t wl = WARP_LANE_BASE + (uint64_t)(i / warp);
        const int64_t p = below_from_hash(mix64(megores_key(base, wl, kind == TR_C1 ? 0ull : (uint64_t)r)), n_part);
        j = p * n_w + local;
      }
    }
    out[t] = j;
  }
}

__device__ __forceinline__ int64_t floor_div(int64_t a, int64_t d) {  // d > 0; numpy's //
  const int64_t q = a / d;
  return q - ((a % d) < 0);
}

__global__ void k_traffic(const int64_t* __restrict__ idx, int64_t groups, int32_t w, int32_t word_bytes,
                          int32_t seg_bytes, unsigned long long* __restrict__ acc) {
  const int64_t wps = seg_bytes / word_bytes;
  unsigned long long tot = 0, waste = 0, mx = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* row = idx + g * w;
    int64_t segs = 0, words = 0;
    for (int a = 0; a < w; ++a) {  // an element is new if no earlier one of the group matches it
      const int64_t va = row[a], sa = floor_div(va * word_bytes, seg_bytes);
      bool new_word = true, new_seg = true;
      for (int c = 0; c < a && (new_word || new_seg); ++c) {
        const int64_t vc = row[c];
        new_word &= vc != va;
        new_seg &= floor_div(vc * word_bytes, seg_bytes) != sa;
      }
      segs += new_seg;
      words += new_word;
    }
    tot += (unsigned long long)segs;
    waste += (unsigned long long)(segs * wps - words);
    mx = segs > (int64_t)mx ? (unsigned long long)segs : mx;
  }
  for (int s = 16; s; s >>= 1) {
    tot += __shfl_xor_sync(0xffffffffu, tot, s);
    waste += __shfl_xor_sync(0xffffffffu, waste, s);
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, mx, s);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], tot);
    atomicMax(&acc[1], mx);
    atomicAdd(&acc[2], waste);
  }
}

// ---------------------------------------------------------------------------
// Synthetic Gaussian-family weights on the device (M/weights.py:100-104 with the
// Box-Muller draw of M/rng.py:152-161).  Same formula and stream; libm rounding of
// exp/log/cos may differ from the host's in the last float64 bit.

template <typename WT>
__global__ void k_gen_gaussian(double y, int64_t n, uint64_t seed, WT* out) {
  const uint64_t base = megores_base(seed);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t x = megores_key(base, (uint64_t)i, 0);
    const uint64_t h1 = mix64(x), h2 = mix64(x + M_SALT);
    const double u1 = ((double)(h1 >> 11) + 0.5) * 0x1p-53;
    const double u2 = (double)(h2 >> 11) * 0x1p-53;
    const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
    const double d = z - y;
    out[i] = (WT)(exp(-0.5 * (d * d)) * 0.3989422804014327);
  }
}

// ---------------------------------------------------------------------------
// gen_gamma_weights (M/weights.py:107-111): w_i = F^-1(u_i; alpha) / beta, the inverse CDF of
// gamma(alpha, rate beta) at u_i = uniform_open01_at(seed, i, 0) (M/rng.py:134-137).  The
// reference evaluates scipy.stats.gamma.ppf (Boost's gamma_p_inv); here: the regularized
// incomplete gamma P/Q (series below a + 1, Lentz continued fraction above) and Halley steps
// on P(x) = u (u <= 1/2) or Q(x) = 1 - u (u > 1/2, exact there) from the Wilson-Hilferty /
// small-shape starting point.  float64 throughout; agrees with scipy to ~1e-14 relative
// (tests/test_gamma_gpu.py states the tolerance), so float32 weights match scipy's except
// in the last ulp of a tiny fraction of draws.

// P(a, x) and Q(a, x) = 1 - P; the one computed directly keeps full relative accuracy
__device__ __forceinline__ void gamma_pq(double a, double x, double lga, double& P, double& Q, double& dens) {
  const double lpre = a * log(x) - x - lga;  // log(x^a e^-x / Gamma(a))
  const double pre = exp(lpre);
  dens = pre / x;  // the gamma(a) density at x
  if (x < a + 1.0) {  // P = pre * sum_k x^k / (a (a+1) ... (a+k))
    double ap = a, del = 1.0 / a, sum = del;
    for (int k = 0; k < 2000; ++k) {
      ap += 1.0;
      del *= x / ap;
      sum += del;
      if (fabs(del) < fabs(sum) * 1e-17) break;
    }
    P = pre * sum;
    Q = 1.0 - P;
  } else {  // Q = pre / (x + 1 - a - 1 (1 - a) / (x + 3 - a - ...)), modified Lentz
    const double tiny = 1e-300;
    double b = x + 1.0 - a, c = 1.0 / tiny, d = 1.0 / b, h = d;
    for (int k = 1; k < 2000; ++k) {
      const double an = -k * (k - a);
      b += 2.0;
      d = an * d + b;
      if (fabs(d) < tiny) d = tiny;
      c = b + an / c;
      if (fabs(c) < tiny) c = tiny;
      d = 1.0 / d;
      const double del = d * c;
      h *= del;
      if (fabs(del - 1.0) < 1e-17) break;
    }
    Q = pre * h;
    P = 1.0 - Q;
  }
}

// x with P(a, x) = p, given q = 1 - p (both exact inputs)
__device__ double gamma_p_inv_dev(double a, double p, double q, double lga) {
  double x;
  if (a > 1.0) {  // Wilson-Hilferty from the normal quantile (Abramowitz-Stegun 26.2.22)
    const double pp = p < 0.5 ? p : q;
    const double t = sqrt(-2.0 * log(pp));
    double z = (2.30753 + t * 0.27061) / (1.0 + t * (0.99229 + t * 0.04481)) - t;  // -z_p (p >= 1/2)
    if (p < 0.5) z = -z;
    const double c = 1.0 - 1.0 / (9.0 * a) - z / (3.0 * sqrt(a));
    x = a * c * c * c;
    if (!(x > 1e-3)) x = 1e-3;
  } else {  // small shape: P ~ (x^a / Gamma(a+1)) near 0, exponential tail above
    const double t = 1.0 - a * (0.253 + a * 0.12);
    x = p < t ? pow(p / t, 1.0 / a) : 1.0 - log(q / (1.0 - t));
    if (!(x > 0.0)) x = 1e-300;
  }
  const bool lower = p <= 0.5;
  double lo = 0.0, hi = INFINITY;  // bracket of the root, tightened every step
  for (int it = 0; it < 200; ++it) {
    double P, Q, f;
    gamma_pq(a, x, lga, P, Q, f);
    // g = P - p (lower) or q - Q (upper): increasing in x, g' = f, g''/g' = (a - 1)/x - 1
    const double g = lower ? P - p : q - Q;
    if (g == 0.0) break;
    if (g > 0.0) hi = x; else lo = x;
    double xn;
    if (f > 0.0 && isfinite(f)) {
      const double tt = g / f;
      const double hal = 1.0 - 0.5 * tt * ((a - 1.0) / x - 1.0);
      xn = x - ((hal > 0.5 && hal < 2.0) ? tt / hal : tt);  // Halley; Newton when it would overshoot
    } else {
      xn = -1.0;
    }
    if (!(xn > lo && xn < hi))  // outside the bracket: bisect it (geometrically when unbounded)
      xn = isfinite(hi) ? (lo > 0.0 && hi > 4.0 * lo ? sqrt(lo * hi) : 0.5 * (lo + hi)) : 2.0 * x + 1.0;
    if (fabs(xn - x) <= 2e-16 * xn) { x = xn; break; }
    x = xn;
  }
  return x;
}

template <typename WT>
__global__ void k_gen_gamma(double a, double lga, double scale, int64_t n, uint64_t seed, WT* out) {
  const uint64_t base = megores_base(seed);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(megores_key(base, (uint64_t)i, 0));
    const double u = __dmul_rn(__dadd_rn((double)(h >> 11), 0.5), 0x1p-53);  // uniform_open01_at
    out[i] = (WT)__dmul_rn(gamma_p_inv_dev(a, u, 1.0 - u, lga), scale);
  }
}

// ---------------------------------------------------------------------------
// SIR particle filter stages (M/pfilter.py:86-165), float64 like numpy.
// gaussian_at(seed, i, 0) (M/rng.py:152-161): Box-Muller on salts 0/1.

__device__ __forceinline__ double gaussian_at_dev(uint64_t base, uint64_t i) {
  const uint64_t x = megores_key(base, i, 0);
  const uint64_t h1 = mix64(x), h2 = mix64(x + M_SALT);
  const double u1 = __dmul_rn(__dadd_rn((double)(h1 >> 11), 0.5), 0x1p-53);
  const double u2 = __dmul_rn((double)(h2 >> 11), 0x1p-53);
  return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(6.283185307179586, u2)));
}

// init_state (M/pfilter.py:129-133): x_i = gaussian_at(seed_init, i, 0) * sqrt(process_var)
__global__ void k_pf_init(int64_t n, uint64_t base, double sqrt_pv, double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __dmul_rn(gaussian_at_dev(base, (uint64_t)i), sqrt_pv);
}

// stage 1 of sir_step (M/pfilter.py:149-153): process noise, transition (M/pfilter.py:86-89),
// likelihood with the float64-tiny floor (M/pfilter.py:92-103), cast to the weight precision.
template <typename WT>
__global__ void k_pf_predict_update(const double* __restrict__ x, int64_t n, double cos_term, double sqrt_pv,
                                    uint64_t base, double z, double obs_var, double norm,
                                    double* __restrict__ xp, WT* __restrict__ w, int32_t* any_pos) {
  bool pos = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = __dmul_rn(gaussian_at_dev(base, (uint64_t)i), sqrt_pv);
    const double xi = x[i];
    // x / 2.0 + 25.0 * x / (1.0 + x * x) + 8.0 * cos(1.2 t) + noise   (left to right)
    const double a = __dadd_rn(__ddiv_rn(xi, 2.0), __ddiv_rn(__dmul_rn(25.0, xi), __dadd_rn(1.0, __dmul_rn(xi, xi))));
    const double xn = __dadd_rn(__dadd_rn(a, cos_term), v);
    xp[i] = xn;
    // residual = z - x*x/20; exp(-0.5 * r * r / obs_var) / sqrt(2 pi obs_var); max(., tiny)
    const double r = __dsub_rn(z, __ddiv_rn(__dmul_rn(xn, xn), 20.0));
    double dens = __ddiv_rn(exp(__ddiv_rn(__dmul_rn(__dmul_rn(-0.5, r), r), obs_var)), norm);
    dens = dens > 2.2250738585072014e-308 ? dens : 2.2250738585072014e-308;
    const WT wv = (WT)dens;
    w[i] = wv;
    pos |= wv > (WT)0;
  }
  // _check_weights' "any w > 0" (M/resample.py:96-100), without a host round trip: float32
  // weights can underflow to 0 (the float64 floor becomes 0.0f)
  if (any_pos && __any_sync(0xffffffffu, pos) && (threadIdx.x & 31) == 0) atomicOr(any_pos, 1);
}

// estimate_ratio subset (M/weights.py:134-154): keys = the 53-bit draw of uniform01_at(seed, i, 0)
// (a stable radix sort by key reproduces np.argsort(kind="stable")); gather w in that order.
__global__ void k_ratio_keys(int64_t n, uint64_t base, uint64_t* __restrict__ keys, int32_t* __restrict__ idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = mix64(megores_key(base, (uint64_t)i, 0)) >> 11;
    idx[i] = (int32_t)i;
  }
}

template <typename WT>
__global__ void k_gather_f64(const WT* __restrict__ w, const int32_t* __restrict__ idx, int64_t m, double* __restrict__ out) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m; q += (int64_t)gridDim.x * blockDim.x)
    out[q] = (double)w[idx[q]];
}

}  // namespace mgp
