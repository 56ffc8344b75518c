// Microbenchmark of Megopolis kernel variants (megores stream, f32, W=32, pow2 N, fast path).
// Every variant must reproduce the library kernel's ancestors bit-for-bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
//        -I../../include -I../../paper_2109_13504_b200/csrc mb_mego.cu -o mb_mego
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "mgp_kernels.cuh"

using namespace mgp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------------------
// V1: balanced pipes.
//  - 64-bit x update from the loop counter (IMAD.WIDE on the FMA pipe)
//  - 64x64 multiply as 2 IMAD + 1 IMAD.WIDE with a {0, cross} addend
//  - u via I2F.RZ(h | 2^63) * 2^-64 - 0.5 (one DFMA, exact)
//  - j = mux(i_al + o_al, lane + o_lo, C) (n >= 64)

__device__ __forceinline__ uint64_t mulc64(uint64_t x, uint64_t c) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t cl = (uint32_t)c, ch = (uint32_t)(c >> 32);
  uint32_t t;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(t) : "r"(hi), "r"(cl));
  asm("mad.lo.u32 %0, %1, %2, %0;" : "+r"(t) : "r"(lo), "r"(ch));
  uint64_t q, p;
  asm("mov.b64 %0, {%1, %2};" : "=l"(q) : "r"(0u), "r"(t));
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(lo), "r"(cl), "l"(q));
  return p;
}

__device__ __forceinline__ double u_from_x_v1(uint64_t x) {
  x = (x ^ (x >> 30));
  x = mulc64(x, MIX1);
  x = (x ^ (x >> 27));
  x = mulc64(x, MIX2);
  uint64_t h = (x ^ (x >> 31)) | 0x8000000000000000ull;
  double d = __ull2double_rz(h);
  return fma(d, 0x1p-64, -0.5);
}

__global__ void __launch_bounds__(256) k_v1(const ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  double wk = f32n_to_f64(__ldg(w + i));
  int bstar = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t A = i_al + (o & ~31u), B = lane + (o & 31u);
    const uint32_t j = (A & cmask) | (B & ~cmask);
    const double wj = f32n_to_f64(__ldg(w + j));
    const uint64_t x = x0 + (uint64_t)(uint32_t)t * M_CTR;
    const double u = u_from_x_v1(x);
    if (u * wk <= wj) { wk = wj; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}

// V2: V1 but the state weight kept as f32 bits (one 32-bit select) and re-expanded.
__global__ void __launch_bounds__(256) k_v2(const ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t wkb = __ldg(w + i);
  int bstar = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t A = i_al + (o & ~31u), B = lane + (o & 31u);
    const uint32_t j = (A & cmask) | (B & ~cmask);
    const uint32_t wjb = __ldg(w + j);
    const uint64_t x = x0 + (uint64_t)(uint32_t)t * M_CTR;
    const double u = u_from_x_v1(x);
    if (u * f32n_to_f64(wkb) <= f32n_to_f64(wjb)) { wkb = wjb; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}

// V3: V1 with strength-reduced x (x += M_CTR) instead of the counter multiply.
__global__ void __launch_bounds__(256) k_v3(const ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  double wk = f32n_to_f64(__ldg(w + i));
  int bstar = -1;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t A = i_al + (o & ~31u), B = lane + (o & 31u);
    const uint32_t j = (A & cmask) | (B & ~cmask);
    const double wj = f32n_to_f64(__ldg(w + j));
    const double u = u_from_x_v1(x);
    x += M_CTR;
    if (u * wk <= wj) { wk = wj; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}

// V4: two particles per thread (i and i + 32*8*... same lane, next CTA-slice) for ILP.
__global__ void __launch_bounds__(128) k_v4(const ResampleArgs a, const __grid_constant__ OffChunk oc) {
  // thread handles particles i and i + 128 within a 256-particle block
  const uint32_t blk = a.p0 + blockIdx.x * 256;
  const uint32_t i0 = blk + threadIdx.x, i1 = i0 + 128;
  if (i0 >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, ia0 = i0 - lane, ia1 = i1 - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  double wk0 = f32n_to_f64(__ldg(w + i0)), wk1 = f32n_to_f64(__ldg(w + i1));
  int bs0 = -1, bs1 = -1;
  const uint64_t xa = megores_key(a.base, i0, (uint64_t)a.b0), xb = megores_key(a.base, i1, (uint64_t)a.b0);
#pragma unroll 2
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t B = lane + (o & 31u), oa = o & ~31u;
    const uint32_t j0 = ((ia0 + oa) & cmask) | (B & ~cmask);
    const uint32_t j1 = ((ia1 + oa) & cmask) | (B & ~cmask);
    const double wj0 = f32n_to_f64(__ldg(w + j0)), wj1 = f32n_to_f64(__ldg(w + j1));
    const uint64_t tc = (uint64_t)(uint32_t)t * M_CTR;
    const double u0 = u_from_x_v1(xa + tc), u1 = u_from_x_v1(xb + tc);
    if (u0 * wk0 <= wj0) { wk0 = wj0; bs0 = t; }
    if (u1 * wk1 <= wj1) { wk1 = wj1; bs1 = t; }
  }
  uint32_t k0 = i0, k1 = i1;
  if (bs0 >= 0) k0 = mego_j<true>(ia0, lane, oc.o[bs0], a.n);
  if (bs1 >= 0) k1 = mego_j<true>(ia1, lane, oc.o[bs1], a.n);
  a.anc[i0] = (int64_t)k0;
  a.anc[i1] = (int64_t)k1;
}


// ---------------------------------------------------------------------------
// V5..V8: single-LOP3 mux, DFMA u, 32-bit state select, F2F or texture partner fetch.

__device__ __forceinline__ uint32_t mux3(uint32_t a, uint32_t b, uint32_t c) {  // (a & c) | (b & ~c)
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

__device__ __forceinline__ double u_ref(uint64_t x) {  // library path: m53 + exponent hack
  return u53_fast(mix64_m53(x));
}
__device__ __forceinline__ double u_rz(uint64_t x) {   // I2F.RZ(h|2^63)*2^-64 - 0.5 (DFMA)
  x = (x ^ (x >> 30)) * MIX1;
  x = (x ^ (x >> 27)) * MIX2;
  const uint64_t h = (x ^ (x >> 31)) | 0x8000000000000000ull;
  return fma(__ull2double_rz(h), 0x1p-64, -0.5);
}

template <int UMODE, int WMODE, bool STATE32>
__global__ void __launch_bounds__(256) k_vx(const ResampleArgs a, const __grid_constant__ OffChunk oc,
                                            cudaTextureObject_t tex) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t wkb = __ldg(w + i);
  double wk = (double)__uint_as_float(wkb);
  int bstar = -1;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t j = mux3(i_al + (o & ~31u), lane + (o & 31u), cmask);
    double wj;
    uint32_t wjb = 0;
    if (WMODE == 0) { wjb = __ldg(w + j); wj = f32n_to_f64(wjb); }
    else if (WMODE == 1) { wjb = __ldg(w + j); wj = (double)__uint_as_float(wjb); }
    else { float f = tex1Dfetch<float>(tex, (int)j); wjb = __float_as_uint(f); wj = (double)f; }
    const double u = UMODE == 0 ? u_ref(x) : u_rz(x);
    x += M_CTR;
    const double wkd = STATE32 ? (double)__uint_as_float(wkb) : wk;
    if (u * wkd <= wj) { if (STATE32) wkb = wjb; else wk = wj; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}


// Combined candidates: exponent-hack u (exact), texture or F2F partner, mux, 32-bit state.
template <int WMODE, bool STATE32, int UNROLL, bool XMUL>
__global__ void __launch_bounds__(256) k_vy(const ResampleArgs a, const __grid_constant__ OffChunk oc,
                                            cudaTextureObject_t tex) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t* __restrict__ w = reinterpret_cast<const uint32_t*>(a.w);
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t wkb = __ldg(w + i);
  double wk = (double)__uint_as_float(wkb);
  int bstar = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
  uint64_t x = x0;
#pragma unroll UNROLL
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t j = mux3(i_al + (o & ~31u), lane + (o & 31u), cmask);
    double wj;
    uint32_t wjb;
    if (WMODE == 1) { wjb = __ldg(w + j); wj = (double)__uint_as_float(wjb); }
    else { float f = tex1Dfetch<float>(tex, (int)j); wjb = __float_as_uint(f); wj = (double)f; }
    const uint64_t xx = XMUL ? x0 + (uint64_t)(uint32_t)t * M_CTR : x;
    const double u = u_ref(xx);
    x += M_CTR;
    const double wkd = STATE32 ? (double)__uint_as_float(wkb) : wk;
    if (u * wkd <= wj) { if (STATE32) wkb = wjb; else wk = wj; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}


// ---- optimized candidates ------------------------------------------------------
// megores: texture partner fetch, F2F conversions, 32-bit state select, lop3 mux,
// u = (double)m * 2^-53 on the FP64 pipe (exact for every m, incl. m == 0).
template <bool XMUL>
__global__ void __launch_bounds__(256) k_vz(const ResampleArgs a, const __grid_constant__ OffChunk oc,
                                            cudaTextureObject_t tex) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  float wkf = tex1Dfetch<float>(tex, (int)i);
  int bstar = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
  uint64_t x = x0;
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint32_t o = oc.o[t];
    const uint32_t j = mux3(i_al + (o & ~31u), lane + (o & 31u), cmask);
    const float wjf = tex1Dfetch<float>(tex, (int)j);
    const uint64_t xx = XMUL ? x0 + (uint64_t)(uint32_t)t * M_CTR : x;
    x += M_CTR;
    const double u = (double)mix64_m53(xx) * 0x1p-53;
    if (u * (double)wkf <= (double)wjf) { wkf = wjf; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}

// philox: round keys in the param space (uniform), 4 draws per block.
struct PhiloxKeys { uint32_t k0[10], k1[10]; };
__global__ void __launch_bounds__(256) k_vp(const ResampleArgs a, const __grid_constant__ OffChunk oc,
                                            cudaTextureObject_t tex, const __grid_constant__ PhiloxKeys pk) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  float wkf = tex1Dfetch<float>(tex, (int)i);
  int bstar = -1;
  for (int t0 = 0; t0 < a.cnt; t0 += 4) {
    uint32_t c0 = i, c1 = 0, c2 = (uint32_t)((a.b0 + t0) >> 2), c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t p0 = (uint64_t)PHILOX_M0 * c0, p1 = (uint64_t)PHILOX_M1 * c2;
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ pk.k0[r], n2 = (uint32_t)(p0 >> 32) ^ c3 ^ pk.k1[r];
      c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
    }
    const uint32_t wd[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q;
      if (t < a.cnt) {
        const uint32_t o = oc.o[t];
        const uint32_t j = mux3(i_al + (o & ~31u), lane + (o & 31u), cmask);
        const float wjf = tex1Dfetch<float>(tex, (int)j);
        const double u = (double)wd[q] * 0x1p-32;
        if (u * (double)wkf <= (double)wjf) { wkf = wjf; bstar = t; }
      }
    }
  }
  uint32_t k = i;
  if (bstar >= 0) k = mego_j<true>(i_al, lane, oc.o[bstar], a.n);
  a.anc[i] = (int64_t)k;
}

// ---------------------------------------------------------------------------

template <class K>
float time_it(K launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<float> ts;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main(int argc, char** argv) {
  const int logn = argc > 1 ? atoi(argv[1]) : 24;
  const int B = argc > 2 ? atoi(argv[2]) : 354;
  const uint32_t n = 1u << logn;
  const uint64_t seed = 7;
  float* w;
  int64_t *anc0, *anc1;
  CK(cudaMalloc(&w, sizeof(float) * n));
  CK(cudaMalloc(&anc0, sizeof(int64_t) * n));
  CK(cudaMalloc(&anc1, sizeof(int64_t) * n));
  k_gen_gaussian<float><<<148 * 32, 256>>>(4.0, n, 20240, w);
  CK(cudaDeviceSynchronize());
  static OffChunk oc;
  const uint64_t base = megores_base(seed);
  for (int t = 0; t < B; ++t) oc.o[t] = (uint32_t)below_from_hash(mix64(megores_key(base, GLOBAL_OFFSET_LANE, t)), n);
  ResampleArgs a{};
  a.w = w; a.n = n; a.p0 = 0; a.p_end = n; a.seed = seed; a.base = base; a.b0 = 0; a.cnt = B;
  a.first = 1; a.last = 1; a.anc = anc0;
  const unsigned grid = n / 256;
  auto ref = [&]() { k_megopolis_w32<0, float, true, true><<<grid, 256>>>(a, oc); };
  float t0 = time_it(ref, 7);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  const double cmp = (double)n * B;
  printf("N=2^%d B=%d  ref  %.3f ms  %.3f Gcmp/s\n", logn, B, t0, cmp / t0 / 1e6);
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("%-4s %.3f ms  %.3f Gcmp/s  speedup %.3f  mismatches %zu\n", name, ms, cmp / ms / 1e6, t0 / ms, bad);
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
  ResampleArgs b = a;
  b.anc = anc1;
  check("v1", time_it([&]() { k_v1<<<grid, 256>>>(b, oc); }, 7));
  check("v2", time_it([&]() { k_v2<<<grid, 256>>>(b, oc); }, 7));
  check("v3", time_it([&]() { k_v3<<<grid, 256>>>(b, oc); }, 7));
  check("v4", time_it([&]() { k_v4<<<grid, 128>>>(b, oc); }, 7));
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = w;
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = sizeof(float) * n;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  check("u0w0", time_it([&]() { k_vx<0, 0, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u1w0", time_it([&]() { k_vx<1, 0, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u0w1", time_it([&]() { k_vx<0, 1, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u1w1", time_it([&]() { k_vx<1, 1, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u1w1s", time_it([&]() { k_vx<1, 1, true><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u0w2", time_it([&]() { k_vx<0, 2, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("u1w2", time_it([&]() { k_vx<1, 2, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y1s4", time_it([&]() { k_vy<1, true, 4, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y2s4", time_it([&]() { k_vy<2, true, 4, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y2d4", time_it([&]() { k_vy<2, false, 4, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y2s8", time_it([&]() { k_vy<2, true, 8, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y2s2", time_it([&]() { k_vy<2, true, 2, false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("y2s4m", time_it([&]() { k_vy<2, true, 4, true><<<grid, 256>>>(b, oc, tex); }, 7));
  check("vz", time_it([&]() { k_vz<false><<<grid, 256>>>(b, oc, tex); }, 7));
  check("vzm", time_it([&]() { k_vz<true><<<grid, 256>>>(b, oc, tex); }, 7));
  {
    // philox reference (library kernel) vs optimized philox
    static OffChunk ocp;
    for (int t = 0; t < B; ++t) ocp.o[t] = (uint32_t)below_from_word(p4_word(philox_block(seed, GLOBAL_OFFSET_LANE, t >> 2), t & 3), n);
    ResampleArgs c = a; c.anc = anc0;
    float tpl = time_it([&]() { k_megopolis_w32<1, float, true, true><<<grid, 256>>>(c, ocp); }, 7);
    CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
    PhiloxKeys pk;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) { pk.k0[r] = k0; pk.k1[r] = k1; k0 += PHILOX_W0; k1 += PHILOX_W1; }
    printf("philox lib %.3f ms\n", tpl);
    float tvp = time_it([&]() { k_vp<<<grid, 256>>>(b, ocp, tex, pk); }, 7);
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("vp (philox opt) %.3f ms  %.3f Gcmp/s  vs megores ref %.3f  mismatches %zu\n", tvp, cmp / tvp / 1e6, t0 / tvp, bad);
  }
  {
    float tp = time_it([&]() { k_megopolis_w32<1, float, true, true><<<grid, 256>>>(b, oc); }, 7);
    printf("philox(lib) %.3f ms  %.3f Gcmp/s  vs megores ref %.3f\n", tp, cmp / tp / 1e6, t0 / tp);
  }
  check("u1w2s", time_it([&]() { k_vx<1, 2, true><<<grid, 256>>>(b, oc, tex); }, 7));
  return 0;
}
