// Microbenchmark of Megopolis kernel variants vs the library kernel (megores stream, f32, W=32,
// pow2 N, no zero weights).  Every variant must reproduce the library's ancestors bit for bit.
// Earlier exploratory variants (bit-hack conversions, LDG vs texture, unroll sweeps) are in git
// history; DESIGN.md section 4 summarises what they showed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
//        -I../../include -I../../paper_2109_13504_b200/csrc mb_mego.cu -o mb_mego
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "mgp_kernels.cuh"

using namespace mgp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---- variants of k_megopolis_megores_f32 (PPT 1) ----
// z = y * MIX1 (mod 2^64) as IMAD.WIDE.U32(ylo, C_lo, {0, t}) with t = yhi*C_lo + ylo*C_hi
__device__ __forceinline__ uint64_t mul64_wide(uint64_t y, uint64_t c) {
  uint64_t r;
  asm("{\n\t.reg .u32 lo, hi, t, z;\n\t.reg .u64 a;\n\t"
      "mov.b64 {lo, hi}, %1;\n\t"
      "mul.lo.u32 t, hi, %2;\n\t"
      "mad.lo.u32 t, lo, %3, t;\n\t"
      "mov.u32 z, 0;\n\t"
      "mov.b64 a, {z, t};\n\t"
      "mad.wide.u32 %0, lo, %2, a;\n\t}"
      : "=l"(r) : "l"(y), "r"((uint32_t)c), "r"((uint32_t)(c >> 32)));
  return r;
}
template <int MUL>
__device__ __forceinline__ uint32_t mhi_v(uint64_t x) {
  x ^= x >> 30;
  x = MUL ? mul64_wide(x, MIX1) : x * MIX1;
  x ^= x >> 27;
  const uint32_t vlo = (uint32_t)x, vhi = (uint32_t)(x >> 32);
  return __umulhi(vlo, (uint32_t)MIX2) + vlo * (uint32_t)(MIX2 >> 32) + vhi * (uint32_t)MIX2;
}
// FADD: uf1u = uf1 + 2^-23 on the FMA pipe; MUL: wide multiply; XF: x += M_CTR on the FMA pipe;
// AMBP: ambiguity flag as a predicated store of the round
template <bool FADD, int MUL, bool XF, bool AMBP, int UNR>
__global__ void __launch_bounds__(256) k_mv(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = i & 31u, ial = i - lane, cmask = (a.n - 1) & ~31u;
  float wk = tex1Dfetch<float>(a.tex, (int)i);
  const float wk0 = wk;
  int bstar = -1, ambt = -1;
  bool amb = false;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll UNR
  for (int t = 0; t < a.cnt; ++t) {
    const uint2 o = oc.o[t];
    const uint32_t j = mux3(ial + o.x, lane + o.y, cmask);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    const uint32_t top = mhi_v<MUL>(x) >> 9;
    const float u1 = __uint_as_float(0x3F800000u + top);
    const float u1u = FADD ? __fadd_rn(u1, 0x1p-23f) : __uint_as_float(0x3F800001u + top);
    const float lo = __fmaf_rd(u1, wk, -wk);
    const float hi = __fmaf_ru(u1u, wk, -wk);
    const bool acc = hi <= wj;
    if (AMBP) { if (!acc && lo <= wj) ambt = t; }
    else amb |= !acc && lo <= wj;
    if (acc) { wk = wj; bstar = t; }
    x = XF ? add64_fma(x, a.one) : x + M_CTR;
  }
  if (AMBP ? ambt >= 0 : amb) bstar = megores_exact_rounds(a, oc, i, wk0, true);
  uint32_t k = i;
  if (bstar >= 0) k = mux3(ial + oc.o[bstar].x, lane + oc.o[bstar].y, cmask);
  a.anc[i] = (int64_t)k;
}

struct OffChunkX { uint4 o[1024]; };  // {o & ~31, o & 31, lo(t*M_CTR), hi(t*M_CTR)}
__device__ __forceinline__ uint32_t imad_add(uint32_t a, uint32_t b, uint32_t one) {
  uint32_t r; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(b), "r"(one), "r"(a)); return r;
}
__device__ __forceinline__ uint32_t imad_hi(uint32_t a, uint32_t m) {  // (a * m) >> 32
  uint32_t r; asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(m)); return r;
}
// x0 + c (64-bit) as IMAD.WIDE.U32(one, c_lo, x0) + IMAD(one, c_hi, hi)
__device__ __forceinline__ uint64_t add64_wide(uint64_t x0, uint32_t clo, uint32_t chi, uint32_t one) {
  uint64_t r;
  asm("{\n\t.reg .u32 lo, hi;\n\t"
      "mad.wide.u32 %0, %1, %2, %3;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "mad.lo.u32 hi, %1, %4, hi;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "r"(one), "r"(clo), "l"(x0), "r"(chi));
  return r;
}
// IDX: index adds on the FMA pipe; XW: x = x0 + C_t (param) on the FMA pipe; SH: the high-word
// shifts of both xorshifts as IMAD.HI (m = 4, 32 from the parameter space); AMBP: predicated amb
template <bool IDX, bool XW, bool SH, bool AMBP>
__global__ void __launch_bounds__(256) k_mw(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunkX oc,
                                           const __grid_constant__ OffChunk oc2, uint32_t m4, uint32_t m32) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = i & 31u, ial = i - lane, cmask = (a.n - 1) & ~31u, one = a.one;
  float wk = tex1Dfetch<float>(a.tex, (int)i);
  const float wk0 = wk;
  int bstar = -1, ambt = -1;
  bool amb = false;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
  uint64_t x = x0;
#pragma unroll 4
  for (int t = 0; t < a.cnt; ++t) {
    const uint4 o = oc.o[t];
    const uint32_t j = IDX ? mux3(imad_add(ial, o.x, one), imad_add(lane, o.y, one), cmask) : mux3(ial + o.x, lane + o.y, cmask);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    const uint64_t xx = XW ? add64_wide(x0, o.z, o.w, one) : x;
    uint64_t y;
    if (SH) {
      const uint32_t lo = (uint32_t)xx, hi = (uint32_t)(xx >> 32);
      y = ((uint64_t)(hi ^ imad_hi(hi, m4)) << 32) | (uint32_t)(lo ^ ((uint32_t)(xx >> 30)));
    } else y = xx ^ (xx >> 30);
    uint64_t z = y * MIX1, v;
    if (SH) {
      const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
      v = ((uint64_t)(hi ^ imad_hi(hi, m32)) << 32) | (uint32_t)(lo ^ ((uint32_t)(z >> 27)));
    } else v = z ^ (z >> 27);
    const uint32_t vlo = (uint32_t)v, vhi = (uint32_t)(v >> 32);
    const uint32_t top = (__umulhi(vlo, (uint32_t)MIX2) + vlo * (uint32_t)(MIX2 >> 32) + vhi * (uint32_t)MIX2) >> 9;
    const float u1 = __uint_as_float(0x3F800000u + top);
    const float u1u = __fadd_rn(u1, 0x1p-23f);
    const float lo = __fmaf_rd(u1, wk, -wk);
    const float hi = __fmaf_ru(u1u, wk, -wk);
    const bool acc = hi <= wj;
    if (AMBP) { if (!acc && lo <= wj) ambt = t; }
    else amb |= !acc && lo <= wj;
    if (acc) { wk = wj; bstar = t; }
    if (!XW) x += M_CTR;
  }
  if (AMBP ? ambt >= 0 : amb) bstar = megores_exact_rounds(a, oc2, i, wk0, true);
  uint32_t k = i;
  if (bstar >= 0) k = mux3(ial + oc.o[bstar].x, lane + oc.o[bstar].y, cmask);
  a.anc[i] = (int64_t)k;
}

// x = x0 + c with add.cc / addc
__device__ __forceinline__ uint64_t add64_cc(uint64_t x0, uint32_t clo, uint32_t chi) {
  uint64_t r;
  asm("{\n\t.reg .u32 a, b, lo, hi;\n\t"
      "mov.b64 {a, b}, %1;\n\t"
      "add.cc.u32 lo, a, %2;\n\t"
      "addc.u32 hi, b, %3;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "l"(x0), "r"(clo), "r"(chi));
  return r;
}
// HI1: upper bound from lo (hi = fl_up(lo + wk 2^-22)); XC: x = x0 + C_t (param, add.cc);
// PPT / HALF as the library kernel
template <bool HI1, int XC, int PPT, bool HALF, int UNR, bool LEAH = false, int MINB = 0>
__global__ void __launch_bounds__(256 / PPT, MINB) k_mz(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunkX oc,
                                                 const __grid_constant__ OffChunk ocx) {
  constexpr int PH = HALF ? PPT / 2 : PPT;
  constexpr int STRIDE = HALF ? 128 / PH : 256 / PPT;
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = HALF ? a.p0 + blockIdx.x * 128 + threadIdx.x : a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT], ial[PPT];
  float wk[PPT], wk0[PPT];
  int bstar[PPT], ambt[PPT];
  uint64_t x0[PPT], x[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ii[p] = HALF ? i0 + (p % PH) * STRIDE + (p / PH) * half : i0 + p * STRIDE;
    ial[p] = ii[p] - lane;
    wk[p] = wk0[p] = tex1Dfetch<float>(a.tex, (int)ii[p]);
    bstar[p] = -1; ambt[p] = -1;
    x[p] = x0[p] = megores_key(a.base, ii[p], (uint64_t)a.b0);
  }
#pragma unroll UNR
  for (int t = 0; t < a.cnt; ++t) {
    const uint4 o = oc.o[t];
    const uint2 ot = make_uint2(o.z, o.w);  // XC 2/3: {t, 1}
    uint32_t jj[PPT];
#pragma unroll
    for (int p = 0; p < PH; ++p) jj[p] = mux3(ial[p] + o.x, lane + o.y, cmask);
#pragma unroll
    for (int p = PH; p < PPT; ++p) jj[p] = jj[p - PH] ^ half;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const float wj = tex1Dfetch<float>(a.tex, (int)jj[p]);
      uint64_t xx;
      if (XC == 1) xx = add64_cc(x0[p], o.z, o.w);
      else if (XC == 2) xx = x0[p] + (uint64_t)ot.x * M_CTR;
      else if (XC == 3) {
        asm("{\n\t.reg .u32 lo, hi;\n\t"
            "mad.wide.u32 %0, %1, %2, %3;\n\t"
            "mov.b64 {lo, hi}, %0;\n\t"
            "mad.lo.u32 hi, %1, %4, hi;\n\t"
            "mov.b64 %0, {lo, hi};\n\t}"
            : "=l"(xx) : "r"(ot.x), "r"((uint32_t)M_CTR), "l"(x0[p]), "r"((uint32_t)(M_CTR >> 32)));
      } else xx = x[p];
      float u1;
      if (LEAH) u1 = __uint_as_float(__umulhi(mix64_mhi(xx), o.w) + 0x3F800000u);  // o.w = 2^23 (opaque)
      else u1 = __uint_as_float(0x3F800000u + (mix64_mhi(xx) >> 9));
      const float lo = __fmaf_rd(u1, wk[p], -wk[p]);
      const float hi = HI1 ? __fmaf_ru(wk[p], 0x1p-22f, lo) : __fmaf_ru(__fadd_rn(u1, 0x1p-23f), wk[p], -wk[p]);
      const bool acc = hi <= wj;
      if (!acc && lo <= wj) ambt[p] = t;
      if (acc) { wk[p] = wj; bstar[p] = t; }
      if (XC == 0) x[p] += M_CTR;
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (ambt[p] >= 0) bstar[p] = megores_exact_rounds(a, ocx, ii[p], wk0[p], true);
    uint32_t k = ii[p];
    if (bstar[p] >= 0) k = mux3(ial[p] + oc.o[bstar[p]].x, lane + oc.o[bstar[p]].y, cmask);
    a.anc[ii[p]] = (int64_t)k;
  }
}

// FP64 bracket: u1 = 1 + m_hi 2^-32 from bits; true u in [(m_hi - 1) 2^-32, (m_hi + 2) 2^-32)
// (bit 0 of the final xorshift's high word may differ from m_hi's).  WKD: state weight kept in
// float64 (2 SELs) instead of float32 + F2F per round.
template <bool WKD, int UNR>
__global__ void __launch_bounds__(256) k_md(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, ial = i - lane, cmask = (a.n - 1) & ~31u;
  const float wk0 = tex1Dfetch<float>(a.tex, (int)i);
  float wk = wk0;
  double wkd = (double)wk0;
  int bstar = -1, ambt = -1;
  uint64_t x = megores_key(a.base, i, (uint64_t)a.b0);
#pragma unroll UNR
  for (int t = 0; t < a.cnt; ++t) {
    const uint2 o = oc.o[t];
    const uint32_t j = mux3(ial + o.x, lane + o.y, cmask);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    const double wjd = (double)wj;
    const uint32_t m = mix64_mhi(x);
    const double u1 = __hiloint2double((int)((m >> 12) + 0x3FF00000u), (int)(m << 20));  // 1 + m 2^-32
    const double wkc = WKD ? wkd : (double)wk;
    const double lo = __fma_rd(__dadd_rn(u1, -0x1p-32), wkc, -wkc);
    const double hi = __fma_ru(__dadd_rn(u1, 0x1p-31), wkc, -wkc);
    const bool acc = hi <= wjd;
    if (!acc && lo <= wjd) ambt = t;
    if (acc) { if (WKD) wkd = wjd; else wk = wj; bstar = t; }
    x += M_CTR;
  }
  if (ambt >= 0) bstar = megores_exact_rounds(a, oc, i, wk0, true);
  uint32_t k = i;
  if (bstar >= 0) k = mux3(ial + oc.o[bstar].x, lane + oc.o[bstar].y, cmask);
  a.anc[i] = (int64_t)k;
}

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
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = w;
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = sizeof(float) * n;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));

  static OffChunk oc;
  const uint64_t base = megores_base(seed);
  for (int t = 0; t < B; ++t) {
    const uint32_t o = (uint32_t)below_from_hash(mix64(megores_key(base, GLOBAL_OFFSET_LANE, t)), n);
    oc.o[t] = make_uint2(o & ~31u, o & 31u);
  }
  ResampleArgs a{};
  a.w = w; a.n = n; a.p0 = 0; a.p_end = n; a.seed = seed; a.base = base; a.b0 = 0; a.cnt = B;
  a.first = 1; a.last = 1; a.anc = anc0; a.tex = tex; a.one = 1;
  const unsigned grid = n / 256;
  const double cmp = (double)n * B;
  float t0 = time_it([&]() { k_megopolis_w32<0, float, true, true, true, 1><<<grid, 256>>>(a, oc); }, 7);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  printf("N=2^%d B=%d  lib megores PPT1  %.3f ms  %.1f Gcmp/s\n", logn, B, t0, cmp / t0 / 1e6);
  ResampleArgs b = a;
  b.anc = anc1;
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("%-14s %.3f ms  %.1f Gcmp/s  speedup %.3f  mismatches %zu\n", name, ms, cmp / ms / 1e6, t0 / ms, bad);
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
  ResampleArgs bh = b;
  bh.p0 = 0; bh.p_end = n / 2; bh.hi_shift = 0;
  check("f32 PPT1", time_it([&]() { k_megopolis_megores_f32<true, 1, false><<<grid, 256>>>(b, oc); }, 7));
  check("f32 PPT2", time_it([&]() { k_megopolis_megores_f32<true, 2, false><<<grid, 128>>>(b, oc); }, 7));
  check("f32 PPT2 half", time_it([&]() { k_megopolis_megores_f32<true, 2, true><<<n / 256, 128>>>(bh, oc); }, 7));
  check("f32 PPT4 half", time_it([&]() { k_megopolis_megores_f32<true, 4, true><<<n / 256, 64>>>(bh, oc); }, 7));
  check("f32 PPT4", time_it([&]() { k_megopolis_megores_f32<true, 4, false><<<grid, 64>>>(b, oc); }, 7));
  b.one = 1;
  static OffChunkX ox;
  for (int t = 0; t < B; ++t) { const uint64_t c = (uint64_t)t * M_CTR; ox.o[t] = make_uint4(oc.o[t].x, oc.o[t].y, (uint32_t)c, (uint32_t)(c >> 32)); }
  static OffChunkX oxt;
  for (int t = 0; t < B; ++t) oxt.o[t] = make_uint4(oc.o[t].x, oc.o[t].y, (uint32_t)t, 1u);
  static OffChunkX oxl;
  for (int t = 0; t < B; ++t) oxl.o[t] = make_uint4(oc.o[t].x, oc.o[t].y, 0u, 1u << 23);
  check("d f 4", time_it([&]() { k_md<false, 4><<<grid, 256>>>(b, oc); }, 7));
  check("d d 4", time_it([&]() { k_md<true, 4><<<grid, 256>>>(b, oc); }, 7));
  check("d f 8", time_it([&]() { k_md<false, 8><<<grid, 256>>>(b, oc); }, 7));
  check("d d 8", time_it([&]() { k_md<true, 8><<<grid, 256>>>(b, oc); }, 7));
  check("z H--- 1u8 L", time_it([&]() { k_mz<true, 0, 1, false, 8, true><<<grid, 256>>>(b, oxl, oc); }, 7));
  check("z H--- 1u4 L", time_it([&]() { k_mz<true, 0, 1, false, 4, true><<<grid, 256>>>(b, oxl, oc); }, 7));
  check("z H--- 1u8 m4", time_it([&]() { k_mz<true, 0, 1, false, 8, false, 4><<<grid, 256>>>(b, oxl, oc); }, 7));
  check("z H--- 1u8 m6", time_it([&]() { k_mz<true, 0, 1, false, 8, false, 6><<<grid, 256>>>(b, oxl, oc); }, 7));
  check("z H--- 1u8 L m6", time_it([&]() { k_mz<true, 0, 1, false, 8, true, 6><<<grid, 256>>>(b, oxl, oc); }, 7));
  check("z HT-- 1", time_it([&]() { k_mz<true, 2, 1, false, 4><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z HW-- 1", time_it([&]() { k_mz<true, 3, 1, false, 4><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z HW-- 1u8", time_it([&]() { k_mz<true, 3, 1, false, 8><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z HW-- 4h", time_it([&]() { k_mz<true, 3, 4, true, 2><<<n / 256, 64>>>(bh, oxt, oc); }, 7));
  check("z ---- 1", time_it([&]() { k_mz<false, 0, 1, false, 4><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z H--- 1", time_it([&]() { k_mz<true, 0, 1, false, 4><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z HX-- 1", time_it([&]() { k_mz<true, 1, 1, false, 4><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("z H--- 2", time_it([&]() { k_mz<true, 0, 2, false, 2><<<grid, 128>>>(b, oxt, oc); }, 7));
  check("z H--- 2h", time_it([&]() { k_mz<true, 0, 2, true, 2><<<n / 256, 128>>>(bh, oxt, oc); }, 7));
  check("z H--- 4h", time_it([&]() { k_mz<true, 0, 4, true, 2><<<n / 256, 64>>>(bh, oxt, oc); }, 7));
  check("z HX-- 2h", time_it([&]() { k_mz<true, 1, 2, true, 2><<<n / 256, 128>>>(bh, oxt, oc); }, 7));
  check("z H--- 1u8", time_it([&]() { k_mz<true, 0, 1, false, 8><<<grid, 256>>>(b, oxt, oc); }, 7));
  check("w ----", time_it([&]() { k_mw<false, false, false, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w I---", time_it([&]() { k_mw<true, false, false, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w -X--", time_it([&]() { k_mw<false, true, false, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w --S-", time_it([&]() { k_mw<false, false, true, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w ---A", time_it([&]() { k_mw<false, false, false, true><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w IX--", time_it([&]() { k_mw<true, true, false, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w IXS-", time_it([&]() { k_mw<true, true, true, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w IXSA", time_it([&]() { k_mw<true, true, true, true><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("w I-S-", time_it([&]() { k_mw<true, false, true, false><<<grid, 256>>>(b, ox, oc, 4, 32); }, 7));
  check("v F", time_it([&]() { k_mv<true, 0, false, false, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v FM", time_it([&]() { k_mv<true, 1, false, false, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v FMX", time_it([&]() { k_mv<true, 1, true, false, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v FMA", time_it([&]() { k_mv<true, 1, false, true, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v FMXA", time_it([&]() { k_mv<true, 1, true, true, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v MA", time_it([&]() { k_mv<false, 1, false, true, 4><<<grid, 256>>>(b, oc); }, 7));
  check("v FMA u2", time_it([&]() { k_mv<true, 1, false, true, 2><<<grid, 256>>>(b, oc); }, 7));
  check("v FMA u8", time_it([&]() { k_mv<true, 1, false, true, 8><<<grid, 256>>>(b, oc); }, 7));
  check("lib PPT4 half", time_it([&]() { k_megopolis_w32<0, float, true, true, true, 4, true><<<n / 256, 64>>>(bh, oc); }, 7));
  return 0;
}
