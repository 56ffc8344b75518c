// mgp_prefix.cuh -- the prefix-sum resamplers (M/resample.py:285-336) on sm_100a.
//
// multinomial and systematic_improved both search the inclusive prefix sum
// np.cumsum(values), which numpy evaluates as a SEQUENTIAL left-to-right scan in the
// weights' own dtype (M/resample.py:288-291): s_k = fl(s_{k-1} + w_k).  Its float32
// rounding is part of the reference's result (criterion 6, T/test_acceptance.py:109-176),
// so a tree scan is not acceptable.  The sequential scan is reproduced bit for bit and
// in parallel from one observation:
//
//   While the running sum s stays inside one binade [2^e, 2^(e+1)) (grid spacing
//   u_e = 2^(e - MANT)), s is an integer number of u_e and
//       fl(s + w) = s + inc_e(w),   inc_e(w) = round-half-even-free(w / u_e),
//   an exact integer that does not depend on s -- except when w / u_e lies exactly
//   half-way between integers, where round-to-nearest-even picks the neighbour that
//   makes s + inc even, i.e. inc depends on the parity of s.  So each element is a
//   two-state transducer on the parity of s (in units of u_e): (a0, a1) = increment
//   for parity 0 / 1.  Transducers compose associatively, so inside a binade the
//   sequential scan IS an ordered integer scan -- parallel and exact.
//
// Pipeline (chunks of PX_CHUNK elements, super-chunks of PX_SUPER chunks), three launches:
//   k_px_scan_aggregate  one read of the weights: per chunk the float64 sum and its exclusive
//                     prefix by decoupled look-back (the carry-in estimate), then the composed
//                     transducer for the 3 binades around the estimate (e0-1, e0, e0+1).  All
//                     three are needed: for skewed weights float32 drops whole addends below
//                     half an ulp, so the sequential sum drifts from the float64 estimate
//                     systematically (tens of percent at 2^24 Gaussian y=4 weights), not by a
//                     random-walk sqrt(n) ulps.  The last chunk of a super-chunk to finish
//                     composes the super-chunk's aggregates.
//   k_px_resolve      one CTA walks the super-chunks 32 at a time: from the true carry-in
//                     s (binade e, parity p) it scans the lanes' aggregates for e; every
//                     super-chunk whose end stays inside binade e is resolved in O(1); the
//                     first that leaves it is descended into (chunk windows), and the chunk
//                     the sum leaves its binade in is resolved -- and materialised -- element
//                     by element by the whole CTA (a handful per array: the running sum
//                     crosses each binade once)
//   k_px_materialize  per chunk, its carry-in (composed from its super-chunk's, or written by
//                     the resolver), then an ordered block scan of the transducers writes
//                     s_k = carry + units * u_e
// All arithmetic is integer or exact power-of-two scaling; the result equals np.cumsum.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "mgp_device.cuh"

namespace mgp {

// k_px_resolve and k_px_materialize launched as programmatic dependents of the kernel before
#ifndef MGP_PX_PDL
#define MGP_PX_PDL 1
#endif

constexpr int PX_THREADS = 256;
constexpr int PX_PER_THREAD = 4;
constexpr int PX_CHUNK = PX_THREADS * PX_PER_THREAD;  // 1024 elements per chunk
constexpr int PX_CAND = 3;                             // binades e0-1, e0, e0+1 per chunk
// Super-chunks: PX_SUPER consecutive chunks.  Their aggregate for a binade e is the ordered
// composition of the chunks' aggregates for e (when every chunk carries e among its three
// candidates); candidates E-1, E, E+1 with E the first chunk's e0.
constexpr int PX_SUPER = 32;
constexpr int32_t PX_EXC = -100000;                    // mode: chunk re-scanned sequentially
constexpr int64_t PX_SAT = (int64_t)1 << 61;           // saturation: "leaves the binade"

template <typename WT>
struct PxFp;
template <>
struct PxFp<float> {
  static constexpr int MANT = 23, EMIN = -126;
  __device__ static int expo(float s) {  // floor(log2 s) for normal s, EMIN for 0 / subnormal
    const int ex = (int)((__float_as_uint(s) >> 23) & 0xFFu);
    return ex == 0 ? EMIN : ex - 127;
  }
};
template <>
struct PxFp<double> {
  static constexpr int MANT = 52, EMIN = -1022;
  __device__ static int expo(double s) {
    const int ex = (int)(((unsigned long long)__double_as_longlong(s) >> 52) & 0x7FFull);
    return ex == 0 ? EMIN : ex - 1023;
  }
};

struct Tx {  // increment (in units of u_e) for incoming parity 0 / 1
  int64_t a0, a1;
};

__device__ __forceinline__ int64_t px_sat(int64_t x) { return x > PX_SAT ? PX_SAT : x; }

// A then B
__device__ __forceinline__ Tx px_compose(Tx A, Tx B) {
  Tx r;
  r.a0 = px_sat(A.a0 + ((A.a0 & 1) ? B.a1 : B.a0));
  r.a1 = px_sat(A.a1 + (((1 + A.a1) & 1) ? B.a1 : B.a0));
  return r;
}

__device__ __forceinline__ int64_t px_apply(Tx T, int64_t parity) { return parity ? T.a1 : T.a0; }

// Element transducer of weight w in binade e: w / u_e = M * 2^(ew - e) with M the integer
// significand (implicit bit included for normal w) -- an integer shift with an exact
// remainder, no floating point.  Weights >= 2^(e+1) leave the binade in one step: saturate.
// float32, branch-free and 32-bit: q = floor(M / 2^k), v = q rounded (ties flagged), for
// k = e - ew clamped to [0, 31] (k > 25 gives q = v = 0: M < 2^24 <= half), sat for k < 0.
struct PxInc32 {
  uint32_t q, v;
  bool tie, sat;
};
__device__ __forceinline__ PxInc32 px_inc32(float w, int e) {
  const uint32_t bits = __float_as_uint(w);
  const uint32_t ef = (bits >> 23) & 0xFFu;
  const uint32_t M = (bits & 0x7FFFFFu) | (ef ? 0x800000u : 0u);
  const int k = e - (ef ? (int)ef - 127 : -126);
  const uint32_t kc = (uint32_t)(k < 0 ? 0 : (k > 31 ? 31 : k));
  const uint32_t q = M >> kc, r = M & ((1u << kc) - 1u), half = (1u << kc) >> 1;
  PxInc32 d;
  d.q = q;
  d.v = q + (r > half ? 1u : 0u);
  d.tie = kc > 0 && r == half;
  d.sat = k < 0;
  return d;
}

// float32, four elements at once on the FMA pipe (the integer form above is ~13 ALU instructions
// per element and binade; the aggregate pass was ALU-bound at 82%): t = w * 2^(23-e) is exact,
// fl(t + 2^23) is t rounded to the nearest integer (ties to even) with unit spacing because
// t < 2^22, its low mantissa bits are that integer, and t - round(t) = +-0.5 (exact) flags a
// tie -- the same increments and tie flags as px_inc32.  Valid when every element is below
// 2^(e-1) (wmax_bits: the largest bit pattern; negative, non-finite and saturating elements fail
// it) and e >= -104 (2^(23-e) a normal float); otherwise the integer form.
__device__ __forceinline__ uint32_t px_inc4_f32(const float* v, int e, uint32_t wmax_bits, uint32_t* inc, bool& tie,
                                                bool& sat) {
  uint32_t s = 0;
  if (e >= -104 && wmax_bits < ((uint32_t)(e + 126) << 23)) {
    const float scale = __uint_as_float((uint32_t)(150 - e) << 23);  // 2^(23-e)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float y = __fmaf_rn(v[j], scale, 0x1p23f);
      const float r = __fadd_rn(y, -0x1p23f);
      tie |= fabsf(__fmaf_rn(v[j], scale, -r)) == 0.5f;
      inc[j] = __float_as_uint(y) - 0x4B000000u;
      s += inc[j];
    }
    return s;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const PxInc32 d = px_inc32(v[j], e);
    inc[j] = d.v;
    s += d.v;
    tie |= d.tie;
    sat |= d.sat;
  }
  return s;
}
// float64, the same on the FP64 pipe: t = w * 2^(52-e), fl(t + 2^52) for w < 2^(e-1), e >= -970.
// Returns false (nothing computed) when an element needs the integer form.
__device__ __forceinline__ bool px_inc4_f64(const double* v, int e, int64_t* inc, int64_t& sum, bool& tie) {
  const uint64_t wmax = max(max((uint64_t)__double_as_longlong(v[0]), (uint64_t)__double_as_longlong(v[1])),
                            max((uint64_t)__double_as_longlong(v[2]), (uint64_t)__double_as_longlong(v[3])));
  if (!(e >= -970 && wmax < ((uint64_t)(e + 1022) << 52))) return false;
  const double scale = __longlong_as_double((long long)(1075 - e) << 52);  // 2^(52-e)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double y = __fma_rn(v[j], scale, 0x1p52);
    const double r = __dadd_rn(y, -0x1p52);
    tie |= fabs(__fma_rn(v[j], scale, -r)) == 0.5;
    inc[j] = (int64_t)((uint64_t)__double_as_longlong(y) - 0x4330000000000000ull);
    sum += inc[j];
  }
  return true;
}
__device__ __forceinline__ uint32_t px_wmax_bits(const float* v) {
  return max(max(__float_as_uint(v[0]), __float_as_uint(v[1])), max(__float_as_uint(v[2]), __float_as_uint(v[3])));
}

// float64: the same branch-free form in 64 bits (M < 2^53; k clamped to [0, 63], k > 54 gives
// q = v = 0 because M < 2^53 <= half)
struct PxInc64 {
  uint64_t q, v;
  bool tie, sat;
};
__device__ __forceinline__ PxInc64 px_inc64(double w, int e) {
  const uint64_t bits = (uint64_t)__double_as_longlong(w);
  const uint32_t ef = (uint32_t)(bits >> 52) & 0x7FFu;
  const uint64_t M = (bits & 0xFFFFFFFFFFFFFull) | (ef ? (1ull << 52) : 0ull);
  const int k = e - (ef ? (int)ef - 1023 : -1022);
  const uint32_t kc = (uint32_t)(k < 0 ? 0 : (k > 63 ? 63 : k));
  const uint64_t q = M >> kc, r = M & ((1ull << kc) - 1ull), half = (1ull << kc) >> 1;
  PxInc64 d;
  d.q = q;
  d.v = q + (r > half ? 1ull : 0ull);
  d.tie = kc > 0 && r == half;
  d.sat = k < 0;
  return d;
}

// the per-dtype unit type of the crossing scan below: increments, their caps and the binade limit
template <typename WT>
struct PxScanT;
template <>
struct PxScanT<float> {
  using U = uint32_t;
  static constexpr U CAP = 1u << 25, LIM = (1u << 24) - 1u;  // 32 increments < 2^24 each: no overflow
  __device__ static PxInc32 inc(float w, int e) { return px_inc32(w, e); }
  __device__ static float at(U units, int e) {  // units * 2^(e-23), exact (subnormal spacing too)
    const int xe = e - 23;
    return __fmul_rn((float)units, xe >= -126 ? __uint_as_float((uint32_t)(xe + 127) << 23)
                                              : __uint_as_float(1u << (xe + 149)));
  }
};
template <>
struct PxScanT<double> {
  using U = uint64_t;
  static constexpr U CAP = 1ull << 54, LIM = (1ull << 53) - 1ull;
  __device__ static PxInc64 inc(double w, int e) { return px_inc64(w, e); }
  __device__ static double at(U units, int e);
};

template <typename WT>
__device__ __forceinline__ Tx px_elem(WT w, int e) {
  if constexpr (sizeof(WT) == 4) {  // tie: round half to even makes s + inc even
    const PxInc32 d = px_inc32(w, e);
    const int64_t a0 = d.tie ? (int64_t)(d.q + (d.q & 1u)) : (int64_t)d.v;
    const int64_t a1 = d.tie ? (int64_t)(d.q + ((d.q + 1u) & 1u)) : (int64_t)d.v;
    return d.sat ? Tx{PX_SAT, PX_SAT} : Tx{a0, a1};
  } else {
    const PxInc64 d = px_inc64(w, e);
    const int64_t a0 = d.tie ? (int64_t)(d.q + (d.q & 1ull)) : (int64_t)d.v;
    const int64_t a1 = d.tie ? (int64_t)(d.q + ((d.q + 1ull) & 1ull)) : (int64_t)d.v;
    return d.sat ? Tx{PX_SAT, PX_SAT} : Tx{a0, a1};
  }
}

// Same increment as a plain integer plus a tie flag (tie: inc = q, the transducer is
// {q + (q & 1), q + ((q + 1) & 1)}).  The fast paths below sum plain increments while no
// element of the warp / block is a tie -- the common case for real weights.
template <typename WT>
__device__ __forceinline__ int64_t px_inc(WT w, int e, bool& tie) {
  if constexpr (sizeof(WT) == 4) {
    const PxInc32 d = px_inc32(w, e);
    tie = d.tie;
    return d.sat ? PX_SAT : (int64_t)(d.tie ? d.q + (d.q & 1u) : d.v);
  }
  const Tx t = px_elem<WT>(w, e);
  tie = t.a0 != t.a1;
  return t.a0;  // the increment when !tie
}

__device__ __forceinline__ int64_t px_sat_add(int64_t a, int64_t b) { return px_sat(a + b); }

// A thread's PX_PER_THREAD (= 4) consecutive elements: one 16-byte (float32) or two 16-byte
// (float64) vector accesses when the array is 16-byte aligned and the four are in range (VEC,
// decided on the host), else element by element.  Vector loads/stores make every warp
// instruction cover whole 128-byte lines (scalar ones at a 16-byte stride touched each line
// four times, and the scalar stores wrote partial sectors).
static_assert(PX_PER_THREAD == 4, "vector accesses assume 4 elements per thread");
template <typename WT, bool VEC>
__device__ __forceinline__ void px_load4(const WT* __restrict__ w, int64_t base, int64_t n, WT* v) {
  if (VEC && base + 4 <= n) {
    if constexpr (sizeof(WT) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(w + base));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 q0 = __ldg(reinterpret_cast<const double2*>(w + base));
      const double2 q1 = __ldg(reinterpret_cast<const double2*>(w + base) + 1);
      v[0] = q0.x; v[1] = q0.y; v[2] = q1.x; v[3] = q1.y;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = base + j < n ? w[base + j] : (WT)0;
}
template <typename WT, bool VEC>
__device__ __forceinline__ void px_store4(WT* __restrict__ out, int64_t base, int64_t n, const WT* v) {
  if (VEC && base + 4 <= n) {
    if constexpr (sizeof(WT) == 4) {
      *reinterpret_cast<float4*>(out + base) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
      reinterpret_cast<double2*>(out + base)[0] = make_double2(v[0], v[1]);
      reinterpret_cast<double2*>(out + base)[1] = make_double2(v[2], v[3]);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (base + j < n) out[base + j] = v[j];
}

// ---------------------------------------------------------------------------

// ordered warp reduction (lane 0 receives lane 0 o lane 1 o ... o lane 31)
__device__ __forceinline__ Tx px_warp_reduce(Tx t) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Tx r;
    r.a0 = __shfl_down_sync(0xffffffffu, t.a0, d);
    r.a1 = __shfl_down_sync(0xffffffffu, t.a1, d);
    if ((threadIdx.x & 31) + d < 32 && ((threadIdx.x & 31) & (2 * d - 1)) == 0) t = px_compose(t, r);
  }
  return t;
}

// ordered inclusive warp scan (lane l receives lane 0 o ... o lane l)
__device__ __forceinline__ Tx px_warp_scan(Tx t) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    Tx l;
    l.a0 = __shfl_up_sync(0xffffffffu, t.a0, d);
    l.a1 = __shfl_up_sync(0xffffffffu, t.a1, d);
    if (lane >= d) t = px_compose(l, t);
  }
  return t;
}

template <typename WT, bool VEC>
__global__ void __launch_bounds__(PX_THREADS) k_px_chunk_sum(const WT* __restrict__ w, int64_t n, double* csum,
                                                             uint32_t* __restrict__ zero, int64_t zwords) {
  __shared__ double red[PX_THREADS / 32];
  WT v[PX_PER_THREAD];
  px_load4<WT, VEC>(w, (int64_t)blockIdx.x * PX_CHUNK + threadIdx.x * PX_PER_THREAD, n, v);
  // the counters / carries / modes the later passes expect zeroed (replaces a memset node)
  for (int64_t q = (int64_t)blockIdx.x * PX_THREADS + threadIdx.x; q < zwords; q += (int64_t)gridDim.x * PX_THREADS)
    zero[q] = 0u;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j) s += (double)v[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < PX_THREADS / 32; ++q) t += red[q];
    csum[blockIdx.x] = t;
  }
}

// Per chunk, the composed transducers for the 3 binades around the carry-in estimate (the
// exclusive prefix of the float64 chunk sums); the last chunk of each super-chunk to finish
// composes the super-chunk's aggregates (no separate super-chunk pass).  The estimate only
// chooses candidate binades: its rounding never reaches the result, which the resolver makes
// exact.  (A single-pass decoupled look-back for the estimate was measured: with 1024-element
// chunks the look-back distance is a whole wave of resident CTAs, 200 us at 2^24.)
template <typename WT, bool VEC>
__global__ void __launch_bounds__(PX_THREADS) k_px_aggregate(const WT* __restrict__ w, int64_t n, int64_t nch,
                                                             const double* __restrict__ est, int32_t* scnt,
                                                             int32_t* e0_out, Tx* agg, int32_t* se0, Tx* sagg) {
  __shared__ Tx red[PX_CAND][PX_THREADS / 32];
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t c = blockIdx.x;
  WT v[PX_PER_THREAD];
  px_load4<WT, VEC>(w, c * PX_CHUNK + tid * PX_PER_THREAD, n, v);
#if MGP_PX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the scan of the chunk sums complete
#endif
  const int e0 = PxFp<WT>::expo((WT)est[c]);
  uint32_t wmax = 0;
  if constexpr (sizeof(WT) == 4) wmax = px_wmax_bits(reinterpret_cast<const float*>(v));
#pragma unroll
  for (int k = 0; k < PX_CAND; ++k) {
    const int e = e0 - 1 + k;
    bool tie = false;
    int64_t sum = 0;
    Tx t;
    if constexpr (sizeof(WT) == 4) {
      // float32: every increment is < 2^24, so a warp's 128 of them sum exactly in 32 bits
      // (one REDUX); any saturating element saturates the warp's aggregate
      bool sat = false;
      uint32_t incs[PX_PER_THREAD];
      const uint32_t s32 = px_inc4_f32(reinterpret_cast<const float*>(v), e, wmax, incs, tie, sat);
      if (!__any_sync(0xffffffffu, tie)) {
        const bool any_sat = __any_sync(0xffffffffu, sat);
        const int64_t tot = (int64_t)__reduce_add_sync(0xffffffffu, s32);
        t = any_sat ? Tx{PX_SAT, PX_SAT} : Tx{tot, tot};
        if (lane == 0) red[k][wid] = t;
        continue;
      }
    } else {
      int64_t incs[PX_PER_THREAD];
      if (!px_inc4_f64(reinterpret_cast<const double*>(v), e, incs, sum, tie)) {
#pragma unroll
        for (int j = 0; j < PX_PER_THREAD; ++j) {
          bool tj;
          sum = px_sat_add(sum, px_inc<WT>(v[j], e, tj));
          tie |= tj;
        }
      }
    }
    if (__any_sync(0xffffffffu, tie)) {  // rounding ties in this warp: parity transducers
      t = Tx{0, 0};
#pragma unroll
      for (int j = 0; j < PX_PER_THREAD; ++j) t = px_compose(t, px_elem<WT>(v[j], e));
      t = px_warp_reduce(t);
    } else {  // plain saturating integer sum
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum = px_sat_add(sum, __shfl_xor_sync(0xffffffffu, sum, o));
      t = Tx{sum, sum};
    }
    if (lane == 0) red[k][wid] = t;
  }
  __syncthreads();
  if (tid < PX_CAND) {
    Tx t{0, 0};
    for (int q = 0; q < PX_THREADS / 32; ++q) t = px_compose(t, red[tid][q]);
    agg[c * PX_CAND + tid] = t;
    if (tid == 0) e0_out[c] = e0;
    __threadfence();  // the writers' stores are visible before the counter moves
  }
  // the last chunk of super-chunk sp to finish composes its aggregates
  __syncthreads();
  const int64_t sp = c / PX_SUPER;
  if (tid == 0) {
    const int64_t in_sp = min((int64_t)PX_SUPER, nch - sp * PX_SUPER);
    s_last = atomicAdd(scnt + sp, 1) == (int)in_sp - 1;
  }
  __syncthreads();
  if (!s_last || wid != 0) return;
  __threadfence();
  const int64_t cc = sp * PX_SUPER + lane;
  const bool valid = cc < nch;
  const int ec = valid ? __ldcg(e0_out + cc) : 0;
  const int E = __shfl_sync(0xffffffffu, ec, 0);
#pragma unroll
  for (int k = 0; k < PX_CAND; ++k) {
    const int e = E - 1 + k, kk = e - (ec - 1);
    Tx t{0, 0};  // chunks past the end: identity
    if (valid) {
      if (kk >= 0 && kk < PX_CAND) {
        t.a0 = __ldcg(&agg[cc * PX_CAND + kk].a0);
        t.a1 = __ldcg(&agg[cc * PX_CAND + kk].a1);
      } else {
        t = Tx{PX_SAT, PX_SAT};
      }
    }
    t = px_warp_reduce(t);
    if (lane == 0) sagg[sp * PX_CAND + k] = t;
  }
  if (lane == 0) se0[sp] = E;
}

// The running sum s in units of its binade's spacing (S = the integer significand) and
// that spacing u_e as a double, by bit manipulation (no division / ldexp on the resolver's
// critical path).
template <typename WT>
__device__ __forceinline__ int64_t px_units(WT s) {
  if constexpr (sizeof(WT) == 4) {
    const uint32_t b = __float_as_uint(s);
    return (int64_t)((b & 0x7FFFFFu) | ((b >> 23) & 0xFFu ? 0x800000u : 0u));
  } else {
    const uint64_t b = (uint64_t)__double_as_longlong(s);
    return (int64_t)((b & 0xFFFFFFFFFFFFFull) | ((b >> 52) & 0x7FFull ? (1ull << 52) : 0ull));
  }
}
__device__ __forceinline__ double px_ulp(int e, int mant) {  // 2^(e - mant), exact
  const int x = e - mant;
  return x >= -1022 ? __longlong_as_double((long long)(x + 1023) << 52) : __longlong_as_double(1ll << (x + 1074));
}
__device__ inline double PxScanT<double>::at(uint64_t units, int e) {  // exact: units < 2^53
  return (double)units * px_ulp(e, 52);
}

// The resolver runs as one CTA of PXR_THREADS threads.  Every warp walks the same windows (the
// same data, so the same results; only warp 0 writes), and the chunks the running sum leaves
// its binade in are resolved by the whole CTA together.  One pass: from the running sum s
// (binade e, S units) every thread sums its PXR_PER increments in binade e (saturating: only
// "does it leave the binade" matters); after one barrier every warp scans the 8 warp totals by
// shuffle, so every thread knows the warp the sum leaves the binade in, that warp finds the
// thread T by ballot, T adds its own elements (registers) sequentially from the exact carry
// (S + exclusive prefix) * u_e and publishes the new sum; a second barrier, and the next pass
// restarts after T's elements in the new binade.  A chunk still unresolved after PXR_PASSES
// passes (the first chunks of a sum that starts small cross a binade every few elements),
// rounding ties, or a non-finite sum: the rest of the chunk is staged in shared memory and
// added by one thread in numpy's order (~4 cycles per dependent add).  The result is numpy's
// sequential loop over the chunk.
constexpr int PXR_THREADS = 256;
// resolver profile (build with -DMGP_PX_PROF; read by mgp_debug_px_prof): thread 0 counts
// [0] super windows [1] their cycles [2] chunk windows [3] their cycles [4] crossing chunks
// [5] their cycles [6] block passes [7] sequential tails [8] tail elements [9] kernel cycles
__device__ unsigned long long g_px_prof[16];
#ifdef MGP_PX_PROF
#define PXP_T0() const long long pxp_t0 = clock64()
#define PXP_ADD(k, v) do { if (threadIdx.x == 0) g_px_prof[k] += (unsigned long long)(v); } while (0)
#define PXP_CYC(k) PXP_ADD(k, clock64() - pxp_t0)
#else
#define PXP_T0() do {} while (0)
#define PXP_ADD(k, v) do {} while (0)
#define PXP_CYC(k) do {} while (0)
#endif
constexpr int PXR_WARPS = PXR_THREADS / 32;
constexpr int PXR_PER = PX_CHUNK / PXR_THREADS;  // 4 elements per thread
constexpr int PXR_PASSES = 3;

template <typename U>
__device__ __forceinline__ U px_cap_add(U a, U b, U cap) { return a + b < cap ? a + b : cap; }

template <typename WT>
struct PxBlockScratch {
  typename PxScanT<WT>::U wsum[PXR_WARPS];
  int tie[PXR_WARPS];
  int p_new;
  WT s_new;
  WT buf[PX_CHUNK];  // the chunk, staged for the sequential tail
};

// prefix values of this thread's elements [p, len) from `run` units (binade e, all inside it)
template <typename WT>
__device__ __forceinline__ void px_write_run(WT* __restrict__ cum, int64_t c0, int p, int len,
                                             typename PxScanT<WT>::U run, const typename PxScanT<WT>::U* inc, int e) {
#pragma unroll
  for (int j = 0; j < PXR_PER; ++j) {
    const int idx = threadIdx.x * PXR_PER + j;
    if (idx >= p && idx < len) {
      run += inc[j];
      cum[c0 + idx] = PxScanT<WT>::at(run, e);
    }
  }
}

// cum != nullptr: also writes the chunk's prefix values (the resolver materialises the chunks the
// running sum leaves its binade in; k_px_materialize skips them)
template <typename WT>
__device__ WT px_chunk_block(const WT* __restrict__ w, int64_t n, int64_t c, WT s, PxBlockScratch<WT>& sh,
                             WT* __restrict__ cum) {
  using P = PxScanT<WT>;
  using U = typename P::U;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t c0 = c * (int64_t)PX_CHUNK;
  const int len = (int)((n - c0) < PX_CHUNK ? (n - c0) : (int64_t)PX_CHUNK);
  WT v[PXR_PER];
  px_load4<WT, false>(w, c0 + tid * PXR_PER, n, v);
#ifdef MGP_PX_PROF
  {
    const long long t0 = clock64();
    WT acc = v[0] + v[1] + v[2] + v[3];
    if (acc == (WT)-1.2345) sh.s_new = acc;  // forces the loads to land
    PXP_ADD(10, clock64() - t0);
  }
  const long long pxp_p0 = clock64();
#endif
  int p = 0;  // first chunk-local element not yet added (a multiple of PXR_PER)
  for (int pass = 0; pass < PXR_PASSES && p < len; ++pass) {
    if (!isfinite((double)s)) break;  // s is uniform: every thread leaves together
    const int e = PxFp<WT>::expo(s);
    const U S = (U)px_units<WT>(s);
    U t = 0, inc[PXR_PER];
    bool tie = false, sat = false;
    if constexpr (sizeof(WT) == 4) {  // elements before p (and past len: zero-filled) count 0
      float vm[PXR_PER];
#pragma unroll
      for (int j = 0; j < PXR_PER; ++j) vm[j] = tid * PXR_PER + j >= p ? (float)v[j] : 0.0f;
      t = px_inc4_f32(vm, e, px_wmax_bits(vm), inc, tie, sat);
    } else {
#pragma unroll
      for (int j = 0; j < PXR_PER; ++j) {
        const int idx = tid * PXR_PER + j;
        inc[j] = 0;
        if (idx >= p && idx < len) {
          const auto d = P::inc(v[j], e);
          inc[j] = d.v;
          t += d.v;
          tie |= d.tie;
          sat |= d.sat;
        }
      }
    }
    t = sat ? P::CAP : (t < P::CAP ? t : P::CAP);
    U x = t;  // inclusive warp scan, saturating at CAP
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const U y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x = px_cap_add(x, y, P::CAP);
    }
    U wex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) wex = 0;
    const unsigned tb = __ballot_sync(0xffffffffu, tie);
    if (lane == 31) sh.wsum[wid] = x;
    if (lane == 0) sh.tie[wid] = tb != 0u;
    __syncthreads();
    // every warp: the 8 warp totals on lanes 0..7, inclusive scan by shuffle
    U iw = lane < PXR_WARPS ? sh.wsum[lane] : (U)0;
    const bool anytie = __any_sync(0xffffffffu, lane < PXR_WARPS && sh.tie[lane]);
#pragma unroll
    for (int d = 1; d < PXR_WARPS; d <<= 1) {
      const U y = __shfl_up_sync(0xffffffffu, iw, d);
      if (lane >= d) iw = px_cap_add(iw, y, P::CAP);
    }
    if (anytie) break;  // uniform (every warp read the same flags)
    const U total = __shfl_sync(0xffffffffu, iw, PXR_WARPS - 1);
    U base = __shfl_sync(0xffffffffu, iw, wid > 0 ? wid - 1 : 0);
    if (wid == 0) base = 0;
    const unsigned wb = __ballot_sync(0xffffffffu, lane < PXR_WARPS && S + iw > P::LIM);
    if (!wb) {  // the rest of the chunk stays in binade e
      if (cum) px_write_run<WT>(cum, c0, p, len, S + base + wex, inc, e);
      s = P::at(S + total, e);
      p = len;
      break;
    }
    const int wT = __ffs(wb) - 1;  // the warp the sum leaves binade e in
    if (cum && wid < wT) px_write_run<WT>(cum, c0, p, len, S + base + wex, inc, e);
    if (wid == wT) {
      const U incl = px_cap_add(base, x, P::CAP), excl = px_cap_add(base, wex, P::CAP);
      const unsigned bm = __ballot_sync(0xffffffffu, S + incl > P::LIM);
      const int lT = __ffs(bm) - 1;
      if (cum && lane < lT) px_write_run<WT>(cum, c0, p, len, S + excl, inc, e);
      if (lane == lT) {
        WT r = P::at(S + excl, e);  // exact: <= LIM units
#pragma unroll
        for (int j = 0; j < PXR_PER; ++j) {  // this thread's elements, numpy's order
          const int idx = tid * PXR_PER + j;
          if (idx >= p && idx < len) {
            r = r + v[j];
            if (cum) cum[c0 + idx] = r;
          }
        }
        sh.s_new = r;
        sh.p_new = (tid + 1) * PXR_PER;
      }
    }
    __syncthreads();
    s = sh.s_new;
    p = sh.p_new;
    PXP_ADD(6, 1);
  }
#ifdef MGP_PX_PROF
  PXP_ADD(11, clock64() - pxp_p0);
  const long long pxp_q0 = clock64();
#endif
  if (p < len) {  // sequential tail, numpy's order
#ifdef MGP_PX_PROF
    if (tid == 0 && g_px_prof[7] < 3) g_px_prof[13 + g_px_prof[7]] = (unsigned long long)(c * 4096 + p);
#endif
    PXP_ADD(7, 1);
    PXP_ADD(8, len - p);
#pragma unroll
    for (int j = 0; j < PXR_PER; ++j) sh.buf[tid * PXR_PER + j] = v[j];
    __syncthreads();
    if (tid == 0) {  // groups of 8 through registers, the next group's loads issued before this
      WT r = s;        // group's dependent adds (the add chain, ~4 cycles per element, is the cost)
      int idx = p;
      WT g[8], h[8];
      if (idx + 8 <= len) {
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = sh.buf[idx + j];
      }
      for (; idx + 8 <= len; idx += 8) {
        const bool more = idx + 16 <= len;
        if (more) {
#pragma unroll
          for (int j = 0; j < 8; ++j) h[j] = sh.buf[idx + 8 + j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          r = r + g[j];
          g[j] = r;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sh.buf[idx + j] = g[j];  // the prefix values
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = h[j];
      }
      for (; idx < len; ++idx) {
        r = r + sh.buf[idx];
        sh.buf[idx] = r;
      }
      sh.s_new = r;
    }
    __syncthreads();
    s = sh.s_new;
    if (cum) {
#pragma unroll
      for (int j = 0; j < PXR_PER; ++j) {
        const int idx = tid * PXR_PER + j;
        if (idx >= p && idx < len) cum[c0 + idx] = sh.buf[idx];
      }
    }
  }
#ifdef MGP_PX_PROF
  PXP_ADD(12, clock64() - pxp_q0);
#endif
  __syncthreads();  // sh is reused by the next call
  return s;
}

// One window of up to 32 consecutive units (super-chunks or chunks) from carry-in s: lane l
// takes unit u0 + l (if u0 + l < uend) with its e0 / aggregates; returns the number f of
// leading units whose composed sum stays inside s's binade, the carry-in of lane l's unit
// (units of u_e, valid for l < f) and the carry-out after unit f-1.
struct PxWin {
  int f;
  int e;
  double ue;
  int64_t carry_units;  // this lane's carry-in, in units of u_e
  int64_t out_units;    // carry-out of unit f-1 (all lanes)
};

template <typename WT>
__device__ __forceinline__ PxWin px_window(WT s, int64_t u0, int64_t uend, const int32_t* __restrict__ e0s,
                                           const Tx* __restrict__ aggs) {
  constexpr int MANT = PxFp<WT>::MANT;
  const int lane = threadIdx.x & 31;
  const int64_t lim = ((int64_t)1 << (MANT + 1)) - 1;
  PxWin r;
  const bool fin = isfinite((double)s);
  r.e = PxFp<WT>::expo(s);
  r.ue = px_ulp(r.e, MANT);
  const int64_t S = fin ? px_units<WT>(s) : 0, p = S & 1;
  const int64_t u = u0 + lane;
  const bool valid = u < uend;
  // the unit's binade and all its candidate aggregates in one round trip (the resolver is a
  // chain of these windows: latency, not bandwidth, is its cost)
  const int64_t uu = valid ? u : u0;
  const int eu = e0s[uu];
  Tx cand[PX_CAND];
#pragma unroll
  for (int q = 0; q < PX_CAND; ++q) cand[q] = aggs[uu * PX_CAND + q];
  const int k = valid ? r.e - (eu - 1) : -1;
  const bool has = fin && valid && k >= 0 && k < PX_CAND;
  Tx t{PX_SAT, PX_SAT};
#pragma unroll
  for (int q = 0; q < PX_CAND; ++q)
    if (has && k == q) t = cand[q];
  if (!__any_sync(0xffffffffu, has && t.a0 != t.a1)) {
    // no rounding ties in the window (the common case): the transducers are plain increments,
    // a capped integer scan in the dtype's unit type (32-bit for float32) instead of the
    // parity composition (resolver profile: ~1100 -> ~400 cycles per window)
    using U = typename PxScanT<WT>::U;
    constexpr U CAP = PxScanT<WT>::CAP;
    U x = has ? (U)(t.a0 < (int64_t)CAP ? t.a0 : (int64_t)CAP) : CAP;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const U y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x = px_cap_add(x, y, CAP);
    }
    U ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = 0;
    const U out = (U)S + x;
    const unsigned bad = __ballot_sync(0xffffffffu, !(has && out <= (U)lim));
    r.f = bad ? __ffs(bad) - 1 : 32;
    r.carry_units = S + (int64_t)ex;
    r.out_units = r.f > 0 ? (int64_t)__shfl_sync(0xffffffffu, out, r.f - 1) : S;
    return r;
  }
  const Tx P = px_warp_scan(t);
  Tx Q;
  Q.a0 = __shfl_up_sync(0xffffffffu, P.a0, 1);
  Q.a1 = __shfl_up_sync(0xffffffffu, P.a1, 1);
  if (lane == 0) Q = Tx{0, 0};
  const int64_t out = S + px_apply(P, p);
  const unsigned bad = __ballot_sync(0xffffffffu, !(has && out <= lim));
  r.f = bad ? __ffs(bad) - 1 : 32;
  r.carry_units = S + px_apply(Q, p);
  r.out_units = r.f > 0 ? __shfl_sync(0xffffffffu, out, r.f - 1) : S;
  return r;
}

// One CTA.  Walks super-chunks 32 at a time; a super-chunk the sum leaves its binade in is
// descended into (chunk windows); a chunk the sum leaves its binade in is resolved and
// materialised by px_chunk_block.  Writes smode[sp] = binade e and scarry[sp] for every
// super-chunk resolved whole (k_px_materialize composes its chunks' carry-ins), and
// carry[c] / mode[c] for the chunks of descended super-chunks (PX_EXC for the ones it
// materialised).
constexpr int32_t PX_DESC = -200000;  // smode: descended into

constexpr int64_t PX_STAGE_MAX = 96 * 1024;  // shared-memory budget of the resolver's staging
__host__ __device__ __forceinline__ int64_t px_stage_bytes(int64_t nsup) {
  const int64_t b = nsup * (int64_t)(PX_CAND * sizeof(Tx) + sizeof(int32_t));
  return b <= PX_STAGE_MAX ? b : 0;
}
__device__ __forceinline__ uint32_t dyn_smem_size() {
  uint32_t r;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
  return r;
}

template <typename WT>
__global__ void __launch_bounds__(PXR_THREADS, 1) k_px_resolve(const WT* __restrict__ w, int64_t n, int64_t nch,
                                                            int64_t nsup, const int32_t* __restrict__ e0,
                                                            const Tx* __restrict__ agg, const int32_t* se0,
                                                            const Tx* sagg, WT* carry, int32_t* mode, WT* scarry,
                                                            int32_t* smode, WT* cum) {
  const int tid = threadIdx.x;
  const bool w0 = tid < 32;  // warp 0 writes; every warp computes the same windows
  __shared__ PxBlockScratch<WT> sh;
  // super-chunk aggregates staged in shared memory when the launch provides room (one bulk
  // copy instead of a global round trip per super window)
  extern __shared__ __align__(16) unsigned char px_smem[];
#if MGP_PX_PDL
  // k_px_materialize may launch now: its first wave loads its weights while this CTA runs and
  // then waits in griddepcontrol.wait for this grid
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_px_aggregate complete
#endif
  const bool staged = px_stage_bytes(nsup) != 0 && dyn_smem_size() >= px_stage_bytes(nsup);
  if (staged) {
    Tx* ssagg = reinterpret_cast<Tx*>(px_smem);
    int32_t* sse0 = reinterpret_cast<int32_t*>(ssagg + nsup * PX_CAND);
    for (int64_t q = tid; q < nsup * PX_CAND; q += PXR_THREADS) ssagg[q] = sagg[q];
    for (int64_t q = tid; q < nsup; q += PXR_THREADS) sse0[q] = se0[q];
    __syncthreads();
    se0 = sse0;
    sagg = ssagg;
  }
  WT s = (WT)0;
  int64_t sp = 0;
#ifdef MGP_PX_PROF
  const long long pxp_k0 = clock64();
#endif
  while (sp < nsup) {
    PXP_T0();
    const PxWin r = px_window<WT>(s, sp, nsup, se0, sagg);
    PXP_ADD(0, 1);
    PXP_CYC(1);
    if (w0 && tid < r.f) {
      scarry[sp + tid] = (WT)((double)r.carry_units * r.ue);
      smode[sp + tid] = r.e;
    }
    if (r.f > 0) s = (WT)((double)r.out_units * r.ue);
    sp += r.f;
    if (r.f == 32 || sp >= nsup) continue;
    // descend into super-chunk sp
    if (tid == 0) smode[sp] = PX_DESC;
    int64_t c = sp * PX_SUPER;
    const int64_t cend = min(nch, c + PX_SUPER);
    while (c < cend) {
      PXP_T0();
      const PxWin q = px_window<WT>(s, c, cend, e0, agg);
      PXP_ADD(2, 1);
      PXP_CYC(3);
      if (w0 && tid < q.f) {
        carry[c + tid] = (WT)((double)q.carry_units * q.ue);
        mode[c + tid] = q.e;
      }
      if (q.f > 0) s = (WT)((double)q.out_units * q.ue);
      c += q.f;
      if (c < cend) {  // chunk c leaves its binade: the whole CTA resolves and materialises it
        if (tid == 0) {
          carry[c] = s;
          mode[c] = PX_EXC;
        }
        {
          PXP_T0();
          s = px_chunk_block<WT>(w, n, c, s, sh, cum);
          PXP_ADD(4, 1);
          PXP_CYC(5);
        }
        ++c;
      }
    }
    ++sp;
  }
#ifdef MGP_PX_PROF
  PXP_ADD(9, clock64() - pxp_k0);
#endif
}

// Pass 2: per chunk, an ordered block scan of the transducers from the true carry-in writes
// s_k = carry + units * u_e.  The carry-in of a chunk inside a super-chunk the resolver settled
// whole (smode[sp] = its binade) is the super-chunk's carry-in composed with the aggregates of
// the chunks before it (one warp reduction here, replacing a separate expansion pass); inside a
// descended super-chunk the resolver wrote it (carry / mode), and the chunks the sum leaves its
// binade in (PX_EXC) were materialised by the resolver itself.
template <typename WT, bool VEC>
__global__ void __launch_bounds__(PX_THREADS) k_px_materialize(const WT* __restrict__ w, int64_t n,
                                                               const int32_t* __restrict__ e0,
                                                               const Tx* __restrict__ agg,
                                                               const WT* __restrict__ scarry,
                                                               const int32_t* __restrict__ smode,
                                                               const WT* __restrict__ carry,
                                                               const int32_t* __restrict__ mode, WT* __restrict__ cum) {
  constexpr int MANT = PxFp<WT>::MANT;
  __shared__ Tx wsum[PX_THREADS / 32];
  __shared__ WT s_carry;
  __shared__ int s_md;
  const int64_t c = blockIdx.x;
  const int64_t base = c * PX_CHUNK + threadIdx.x * PX_PER_THREAD;
  WT v[PX_PER_THREAD];
  px_load4<WT, VEC>(w, base, n, v);  // in flight while the carry-in is composed
#if MGP_PX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // k_px_resolve complete (carries, modes)
#endif
  if (threadIdx.x < 32) {
    // everything the carry-in may need in one round trip (independent loads), then select
    const int64_t sp = c / PX_SUPER;
    const int64_t cl = sp * PX_SUPER + threadIdx.x;  // chunks [sp * 32, c) of the super-chunk
    const bool in = cl < c;
    const int sm = smode[sp];
    const int ecl = in ? e0[cl] : 0;
    Tx cand[PX_CAND];
#pragma unroll
    for (int q = 0; q < PX_CAND; ++q) cand[q] = in ? agg[cl * PX_CAND + q] : Tx{0, 0};
    const WT sc = scarry[sp];
    const int md_c = mode[c];
    const WT carry_c = carry[c];
    if (sm == PX_DESC) {
      if (threadIdx.x == 0) {
        s_md = md_c;
        s_carry = carry_c;
      }
    } else {
      Tx t{0, 0};
      const int kq = sm - (ecl - 1);
#pragma unroll
      for (int q = 0; q < PX_CAND; ++q)
        if (in && kq == q) t = cand[q];
      t = px_warp_reduce(t);
      if (threadIdx.x == 0) {
        const int64_t S = px_units<WT>(sc);
        s_md = sm;
        s_carry = (WT)((double)(S + px_apply(t, S & 1)) * px_ulp(sm, MANT));
      }
    }
  }
  __syncthreads();
  const int md = s_md;
  const WT s0 = s_carry;
  if (md == PX_EXC) return;  // materialised by the resolver
  const int e = md;
  const double ue = px_ulp(e, MANT);
  const int64_t S = px_units<WT>(s0);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t inc[PX_PER_THREAD];
  int64_t tsum = 0;
  bool tie = false;
  if constexpr (sizeof(WT) == 4) {
    // float32: a resolved chunk keeps the running sum inside binade e, so every prefix is
    // U * 2^(e-23) with U < 2^24 -- 32-bit scan, and U is exact as a float (one FMUL by the
    // power of two, subnormal spacing included)
    uint32_t i32[PX_PER_THREAD];
    bool sat = false;  // a resolved chunk stays inside its binade: never set
    const float* vf = reinterpret_cast<const float*>(v);
    const uint32_t t32 = px_inc4_f32(vf, e, px_wmax_bits(vf), i32, tie, sat);
    if (!__syncthreads_or(tie)) {
      __shared__ uint32_t wt32[PX_THREADS / 32];
      uint32_t x = t32;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (lane == 31) wt32[wid] = x;
      __syncthreads();
      // warps before this one: the 8 totals on lanes 0..7, one masked REDUX
      const uint32_t wq = (lane < wid) ? wt32[lane & (PX_THREADS / 32 - 1)] : 0u;
      uint32_t U = (uint32_t)S + x - t32 + __reduce_add_sync(0xffffffffu, wq);
      const int xe = e - 23;
      const float uef = xe >= -126 ? __uint_as_float((uint32_t)(xe + 127) << 23) : __uint_as_float(1u << (xe + 149));
      WT o[PX_PER_THREAD];
#pragma unroll
      for (int j = 0; j < PX_PER_THREAD; ++j) {
        U += i32[j];
        o[j] = (WT)__fmul_rn((float)U, uef);
      }
      px_store4<WT, VEC>(cum, base, n, o);
      return;
    }
#pragma unroll
    for (int j = 0; j < PX_PER_THREAD; ++j) inc[j] = i32[j];
  } else {
    if (!px_inc4_f64(reinterpret_cast<const double*>(v), e, inc, tsum, tie)) {
#pragma unroll
      for (int j = 0; j < PX_PER_THREAD; ++j) {
        bool tj;
        inc[j] = px_inc<WT>(v[j], e, tj);
        tie |= tj;
        tsum += inc[j];  // a resolved chunk stays inside its binade: no saturation here
      }
    }
  }
  if (!__syncthreads_or(tie)) {  // no rounding ties in the chunk: plain exclusive integer scan
    __shared__ int64_t wtot[PX_THREADS / 32];
    int64_t x = tsum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wtot[wid] = x;
    __syncthreads();
    int64_t wq = (lane < wid) ? wtot[lane & (PX_THREADS / 32 - 1)] : 0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) wq += __shfl_xor_sync(0xffffffffu, wq, o);  // lanes 0..7 hold them
    int64_t U = S + x - tsum + __shfl_sync(0xffffffffu, wq, 0);
    WT o[PX_PER_THREAD];
#pragma unroll
    for (int j = 0; j < PX_PER_THREAD; ++j) {
      U += inc[j];
      o[j] = (WT)((double)U * ue);
    }
    px_store4<WT, VEC>(cum, base, n, o);
    return;
  }
  // exclusive ordered block scan of the per-thread transducers
  Tx te[PX_PER_THREAD];
  Tx t{0, 0};
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j) {
    te[j] = px_elem<WT>(v[j], e);
    t = px_compose(t, te[j]);
  }
  Tx incw = px_warp_scan(t);
  if (lane == 31) wsum[wid] = incw;
  __syncthreads();
  Tx pre{0, 0};
  for (int q = 0; q < wid; ++q) pre = px_compose(pre, wsum[q]);
  Tx ex;
  ex.a0 = __shfl_up_sync(0xffffffffu, incw.a0, 1);
  ex.a1 = __shfl_up_sync(0xffffffffu, incw.a1, 1);
  if (lane == 0) ex = Tx{0, 0};
  ex = px_compose(pre, ex);
  int64_t U = S + px_apply(ex, S & 1);
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j) {
    U += px_apply(te[j], U & 1);
    if (base + j < n) cum[base + j] = (WT)((double)U * ue);
  }
}


// ---------------------------------------------------------------------------
// Searches.  multinomial (M/resample.py:295-304): key_i = WT(uniform01_at(seed, i, 0) *
// total), ancestor = searchsorted(cum, key_i, "right") clamped to n-1.
// systematic_improved (M/resample.py:307-336): target_i = (i + u0) / n * total (float64),
// ancestor = first a with float64(cum[a]) >= target_i, else n-1.

// Searches of the prefix sum.
//
// multinomial (M/resample.py:295-304): key_i = WT(uniform01_at(seed, i, 0) * total) is
// uniform in [0, total), so a bucket index narrows every search: K buckets with boundary
// values bnd[b] = WT(total * b / K) (non-decreasing) and start[b] = upper_bound(cum, bnd[b]);
// a key in [bnd[b], bnd[b+1]) has its answer in [start[b], start[b+1]] (upper_bound is
// monotone).  The bucket is guessed from the key and corrected by exact comparisons against
// the stored boundaries, then ~log2(N/K) probes finish the search (vs log2 N).
constexpr int PXM_PER_BUCKET = 8;  // 16 -> 8: 292 -> 265 us of search at 2^24 (scripts/mb/search_time.py)

template <typename WT>
__device__ __forceinline__ int64_t pxs_upper(const WT* __restrict__ cum, int64_t lo, int64_t hi, WT key) {
  while (lo < hi) {  // first index in [lo, hi) with cum > key (hi if none)
    const int64_t mid = (lo + hi) >> 1;
    if (__ldg(cum + mid) <= key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// K is a power of two: b / K = b * 2^-log2(K) exactly, one DMUL instead of a DDIV sequence
template <typename WT>
__device__ __forceinline__ WT pxm_bound(double total, int64_t b, int64_t K) {
  return b >= K ? (WT)INFINITY : (WT)(total * ((double)b * __longlong_as_double((1023ll - (63 - __clzll(K))) << 52)));
}

template <typename WT>
__global__ void k_multinomial_buckets(const WT* __restrict__ cum, int64_t n, int64_t K, int32_t* __restrict__ start) {
#if MGP_PX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (px_search)
#endif
  const double total = (double)cum[n - 1];
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= K; b += (int64_t)gridDim.x * blockDim.x)
    start[b] = (int32_t)(b == 0 ? pxs_upper(cum, 0, n, (WT)0) - 0 : pxs_upper(cum, 0, n, pxm_bound<WT>(total, b, K)));
}

template <typename WT>
__global__ void k_multinomial(const WT* __restrict__ cum, int64_t n, uint64_t base, int64_t p0, int64_t p_end,
                              int64_t K, const int32_t* __restrict__ start, int64_t* __restrict__ anc) {
#if MGP_PX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (px_search)
#endif
  const double total = (double)cum[n - 1];
  const double kscale = (double)K / total;  // the bucket guess only: exact corrections follow
  for (int64_t i = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p_end; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(megores_key(base, (uint64_t)i, 0));
    const double ud = __dmul_rn((double)(h >> 11) * 0x1p-53, total);
    const WT key = (WT)ud;
    int64_t bk = (int64_t)((double)key * kscale);
    bk = bk < 0 ? 0 : (bk >= K ? K - 1 : bk);
    while (bk > 0 && key < pxm_bound<WT>(total, bk, K)) --bk;          // exact corrections
    while (bk < K - 1 && !(key < pxm_bound<WT>(total, bk + 1, K))) ++bk;
    // key >= bnd[bk] (bnd[0] = 0 <= key) and key < bnd[bk+1]: answer in [start[bk], start[bk+1]]
    const int64_t lo = bk == 0 ? 0 : start[bk];
    const int64_t hi = start[bk + 1];
    const int64_t a = pxs_upper(cum, lo, hi, key);
    anc[i] = a < n - 1 ? a : n - 1;
  }
}

// systematic_improved (M/resample.py:307-336): target_i = (i + u0) / n * total (float64) is
// monotone in i, so each thread takes a run of PXS_RUN consecutive particles: one binary
// search, then a galloping search from the previous answer for each next particle.  (A
// warp-interleaved run with coalesced stores was tried: the 32-strata gallops cost more.)
constexpr int PXS_RUN = 16;

template <typename WT>
__global__ void k_systematic(const WT* __restrict__ cum, int64_t n, double u0, int64_t p0, int64_t p_end,
                             int64_t* __restrict__ anc) {
#if MGP_PX_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a programmatic dependent (px_search)
#endif
  const double total = (double)cum[n - 1];
  const int64_t nrun = (p_end - p0 + PXS_RUN - 1) / PXS_RUN;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrun; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = p0 + r * PXS_RUN, i1 = min(p_end, i0 + PXS_RUN);
    int64_t a = 0;
    for (int64_t i = i0; i < i1; ++i) {
      const double target = __dmul_rn(__ddiv_rn(__dadd_rn((double)i, u0), (double)n), total);
      // first index >= a with float64(cum) >= target (targets are non-decreasing in i)
      int64_t lo = a, step = 1, hi = a;
      if (i == i0) {
        hi = n;
      } else {  // gallop: a, a+1, a+3, a+7, ... until cum >= target
        while (hi < n && (double)__ldg(cum + hi) < target) { lo = hi + 1; hi += step; step <<= 1; }
        if (hi > n) hi = n;
      }
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((double)__ldg(cum + mid) < target) lo = mid + 1;
        else hi = mid;
      }
      a = lo;
      anc[i] = a < n - 1 ? a : n - 1;
    }
  }
}

// systematic_oracle(w, u) (M/resample.py:339-354): the reference's sequential stratified loop
// for an explicit u.  Its comparison `cum[j] < target` has a float32 array element on the left
// and a Python float on the right; under NumPy 2 (NEP 50) the Python float is a weak scalar
// converted to float32, so for float32 weights the comparison is made in float32 against
// float32(target) -- the only difference from systematic_improved (float64 comparison).
template <typename WT>
__global__ void k_systematic_oracle(const WT* __restrict__ cum, int64_t n, double u, int64_t* __restrict__ anc) {
  const double total = (double)cum[n - 1];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double target = __dmul_rn(__ddiv_rn(__dadd_rn((double)i, u), (double)n), total);
    const WT key = (WT)target;  // float32 weights: the weak-scalar conversion; float64: exact
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(cum + mid) < key) lo = mid + 1;
      else hi = mid;
    }
    anc[i] = lo < n - 1 ? lo : n - 1;
  }
}

}  // namespace mgp
