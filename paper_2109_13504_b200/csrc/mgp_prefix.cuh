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
// Pipeline (chunks of PX_CHUNK elements):
//   k_px_chunk_sum    float64 chunk sums -> (CUB) exclusive prefix = carry-in estimates
//   k_px_aggregate    per chunk, the composed transducer for the 3 binades around the
//                     estimate (e0-1, e0, e0+1)
//   k_px_resolve      one warp walks the chunks 32 at a time: from the true carry-in s
//                     (binade e, parity p) it scans the lanes' aggregates for e; every
//                     chunk whose end stays inside binade e is resolved in O(1); the
//                     first chunk that leaves the binade (or lacks an aggregate for e)
//                     is scanned sequentially by one lane (a handful per array: the
//                     running sum crosses each binade once)
//   k_px_materialize  per chunk, an ordered block scan of the transducers from the true
//                     carry-in writes s_k = carry + units * u_e (sequential re-scan for
//                     the chunks the resolver scanned)
// All arithmetic is integer or exact power-of-two scaling; the result equals np.cumsum.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "mgp_device.cuh"

namespace mgp {

constexpr int PX_THREADS = 256;
constexpr int PX_PER_THREAD = 4;
constexpr int PX_CHUNK = PX_THREADS * PX_PER_THREAD;  // 1024 elements per chunk
constexpr int PX_CAND = 3;                             // binades e0-1, e0, e0+1 per chunk
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

// Element transducer of weight w in binade e.  Weights >= 2^(e+1) leave the binade in one
// step: saturate.  ldexp scaling is exact (w / u_e has at most MANT+1 significant bits).
template <typename WT>
__device__ __forceinline__ Tx px_elem(WT w, int e) {
  constexpr int MANT = PxFp<WT>::MANT;
  if (!((double)w < ldexp(1.0, e + 1))) return Tx{PX_SAT, PX_SAT};
  const double x = ldexp((double)w, MANT - e);
  const double m = floor(x);
  const double f = x - m;
  const int64_t mi = (int64_t)m;
  if (f < 0.5) return Tx{mi, mi};
  if (f > 0.5) return Tx{mi + 1, mi + 1};
  return Tx{mi + (mi & 1), mi + ((mi + 1) & 1)};  // tie: the result s + inc is even
}

// ---------------------------------------------------------------------------

template <typename WT>
__global__ void __launch_bounds__(PX_THREADS) k_px_chunk_sum(const WT* __restrict__ w, int64_t n, double* csum) {
  __shared__ double red[PX_THREADS / 32];
  const int64_t base = (int64_t)blockIdx.x * PX_CHUNK + threadIdx.x * PX_PER_THREAD;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j)
    if (base + j < n) s += (double)w[base + j];
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

template <typename WT>
__global__ void __launch_bounds__(PX_THREADS) k_px_aggregate(const WT* __restrict__ w, int64_t n,
                                                             const double* __restrict__ est, int32_t* e0_out,
                                                             Tx* agg) {
  __shared__ Tx red[PX_CAND][PX_THREADS / 32];
  const int64_t c = blockIdx.x;
  const WT carry_est = (WT)est[c];
  const int e0 = PxFp<WT>::expo(carry_est);
  const int64_t base = c * PX_CHUNK + threadIdx.x * PX_PER_THREAD;
  WT v[PX_PER_THREAD];
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j) v[j] = base + j < n ? w[base + j] : (WT)0;
#pragma unroll
  for (int k = 0; k < PX_CAND; ++k) {
    const int e = e0 - 1 + k;
    Tx t{0, 0};
#pragma unroll
    for (int j = 0; j < PX_PER_THREAD; ++j) t = px_compose(t, px_elem<WT>(v[j], e));
    t = px_warp_reduce(t);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = t;
  }
  __syncthreads();
  if (threadIdx.x < PX_CAND) {
    Tx t{0, 0};
    for (int q = 0; q < PX_THREADS / 32; ++q) t = px_compose(t, red[threadIdx.x][q]);
    agg[c * PX_CAND + threadIdx.x] = t;
  }
  if (threadIdx.x == 0) e0_out[c] = e0;
}

// One warp.  carry[c] / mode[c] receive every chunk's true carry-in and its binade (or
// PX_EXC when the chunk was scanned sequentially here).
template <typename WT>
__global__ void __launch_bounds__(32) k_px_resolve(const WT* __restrict__ w, int64_t n, int64_t nch,
                                                   const int32_t* __restrict__ e0, const Tx* __restrict__ agg,
                                                   WT* carry, int32_t* mode) {
  constexpr int MANT = PxFp<WT>::MANT;
  const int lane = threadIdx.x;
  const int64_t lim = ((int64_t)1 << (MANT + 1)) - 1;  // last unit of the binade
  WT s = (WT)0;
  int64_t c = 0;
  while (c < nch) {
    const int e = PxFp<WT>::expo(s);
    const double ue = ldexp(1.0, e - MANT);
    const int64_t S = isfinite((double)s) ? (int64_t)((double)s / ue) : 0;  // exact: s is a whole number of u_e
    const int64_t p = S & 1;
    const int64_t cc = c + lane;
    const bool valid = cc < nch;
    const int k = valid ? e - (e0[cc] - 1) : -1;
    const bool has = valid && k >= 0 && k < PX_CAND && isfinite((double)s);
    Tx t = has ? agg[cc * PX_CAND + k] : Tx{PX_SAT, PX_SAT};
    const Tx P = px_warp_scan(t);
    Tx Q;
    Q.a0 = __shfl_up_sync(0xffffffffu, P.a0, 1);
    Q.a1 = __shfl_up_sync(0xffffffffu, P.a1, 1);
    if (lane == 0) Q = Tx{0, 0};
    const int64_t out = S + px_apply(P, p);
    const bool safe = has && out <= lim;
    const unsigned bad = __ballot_sync(0xffffffffu, !safe);
    const int f = bad ? __ffs(bad) - 1 : 32;  // chunks c .. c+f-1 stay inside binade e
    if (lane < f) {
      carry[cc] = (WT)((double)(S + px_apply(Q, p)) * ue);
      mode[cc] = e;
    }
    if (f > 0) {
      const int64_t last = __shfl_sync(0xffffffffu, out, f - 1);
      s = (WT)((double)last * ue);
    }
    c += f;
    if (f < 32 && c < nch) {  // chunk c leaves binade e (or lacks its aggregate): sequential
      WT t2 = s;
      if (lane == 0) {
        carry[c] = s;
        mode[c] = PX_EXC;
        const int64_t end = min(n, (c + 1) * (int64_t)PX_CHUNK);
        for (int64_t q = c * (int64_t)PX_CHUNK; q < end; ++q) t2 = t2 + w[q];
      }
      s = __shfl_sync(0xffffffffu, t2, 0);
      c += 1;
    }
  }
}

template <typename WT>
__global__ void __launch_bounds__(PX_THREADS) k_px_materialize(const WT* __restrict__ w, int64_t n,
                                                               const WT* __restrict__ carry,
                                                               const int32_t* __restrict__ mode, WT* __restrict__ cum) {
  constexpr int MANT = PxFp<WT>::MANT;
  __shared__ Tx wsum[PX_THREADS / 32];
  const int64_t c = blockIdx.x;
  const int md = mode[c];
  const WT s0 = carry[c];
  const int64_t base = c * PX_CHUNK + threadIdx.x * PX_PER_THREAD;
  if (md == PX_EXC) {  // sequential (one thread), as numpy
    if (threadIdx.x == 0) {
      WT s = s0;
      const int64_t end = min(n, (c + 1) * (int64_t)PX_CHUNK);
      for (int64_t q = c * (int64_t)PX_CHUNK; q < end; ++q) {
        s = s + w[q];
        cum[q] = s;
      }
    }
    return;
  }
  const int e = md;
  const double ue = ldexp(1.0, e - MANT);
  const int64_t S = (int64_t)((double)s0 / ue);
  WT v[PX_PER_THREAD];
  Tx te[PX_PER_THREAD];
  Tx t{0, 0};
#pragma unroll
  for (int j = 0; j < PX_PER_THREAD; ++j) {
    v[j] = base + j < n ? w[base + j] : (WT)0;
    te[j] = px_elem<WT>(v[j], e);
    t = px_compose(t, te[j]);
  }
  // exclusive ordered block scan of the per-thread transducers
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Tx inc = px_warp_scan(t);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  Tx pre{0, 0};
  for (int q = 0; q < wid; ++q) pre = px_compose(pre, wsum[q]);
  Tx ex;
  ex.a0 = __shfl_up_sync(0xffffffffu, inc.a0, 1);
  ex.a1 = __shfl_up_sync(0xffffffffu, inc.a1, 1);
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

template <typename WT>
__global__ void k_multinomial(const WT* __restrict__ cum, int64_t n, uint64_t base, int64_t p0, int64_t p_end,
                              int64_t* __restrict__ anc) {
  const double total = (double)cum[n - 1];
  for (int64_t i = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p_end; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t h = mix64(megores_key(base, (uint64_t)i, 0));
    const double ud = __dmul_rn((double)(h >> 11) * 0x1p-53, total);
    const WT key = (WT)ud;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(cum + mid) <= key) lo = mid + 1;
      else hi = mid;
    }
    anc[i] = lo < n - 1 ? lo : n - 1;
  }
}

template <typename WT>
__global__ void k_systematic(const WT* __restrict__ cum, int64_t n, double u0, int64_t p0, int64_t p_end,
                             int64_t* __restrict__ anc) {
  const double total = (double)cum[n - 1];
  for (int64_t i = p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p_end; i += (int64_t)gridDim.x * blockDim.x) {
    const double target = __dmul_rn(__ddiv_rn(__dadd_rn((double)i, u0), (double)n), total);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((double)__ldg(cum + mid) < target) lo = mid + 1;
      else hi = mid;
    }
    anc[i] = lo < n - 1 ? lo : n - 1;
  }
}

}  // namespace mgp
