// Round-2 microbenchmark of k_megopolis_megores_f32 variants (megores stream, f32, W=32, pow2 N,
// no zero weights).  The kernel is ALU-pipe bound (ncu: ALU 78%, 16.5 ALU warp-instructions per
// round, math-pipe-throttle 4.3 stalls/issue), so every variant moves ALU work elsewhere:
//   PMOV : wk / bstar / amb updates as predicated moves (FMA-pipe IMAD.MOV) instead of FSEL/SEL
//   ADDW : x += M_CTR as IMAD.WIDE.U32 + IMAD (heavy FMA pipe) instead of IADD3 + IADD3.X
//   PPT2 : two particles per thread, half split (j(i + N/2) = j(i) ^ N/2)
// Every variant must reproduce the library's ancestors bit for bit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
//        -I../../include -I../../paper_2109_13504_b200/csrc mb_mego2.cu -o mb_mego2
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "mgp_kernels.cuh"

using namespace mgp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// predicated moves: if (p) { wk = wj; bstar = t; }   (and the ambiguity record)
__device__ __forceinline__ void pmov_acc(float hi, float wj, float& wk, int& bstar, int t) {
  asm("{\n\t.reg .pred p;\n\t"
      "setp.le.f32 p, %2, %3;\n\t"
      "@p mov.b32 %0, %3;\n\t"
      "@p mov.b32 %1, %4;\n\t}"
      : "+f"(wk), "+r"(bstar) : "f"(hi), "f"(wj), "r"(t));
}
__device__ __forceinline__ void pmov_amb(float lo, float hi, float wj, int& amb, int t) {
  asm("{\n\t.reg .pred p, q;\n\t"
      "setp.le.f32 p, %1, %3;\n\t"
      "setp.gtu.f32 q, %2, %3;\n\t"
      "and.pred p, p, q;\n\t"
      "@p mov.b32 %0, %4;\n\t}"
      : "+r"(amb) : "f"(lo), "f"(hi), "f"(wj), "r"(t));
}

template <bool PMOV, bool ADDW, int PPT, int UNR>
__global__ void __launch_bounds__(256 / PPT) k_v(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = PPT == 2 ? a.p0 + blockIdx.x * 128 + threadIdx.x : a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT];
  float wk[PPT], wk0[PPT];
  int bstar[PPT], amb[PPT];
  uint64_t x[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ii[p] = i0 + p * half;
    wk[p] = wk0[p] = tex1Dfetch<float>(a.tex, (int)ii[p]);
    bstar[p] = -1; amb[p] = -1;
    x[p] = megores_key(a.base, ii[p], (uint64_t)a.b0);
  }
  const uint32_t ial = i0 - lane;
#pragma unroll UNR
  for (int t = 0; t < a.cnt; ++t) {
    const uint2 o = oc.o[t];
    uint32_t jj[PPT];
    jj[0] = mux3(ial + o.x, lane + o.y, cmask);
    if (PPT == 2) jj[PPT - 1] = jj[0] ^ half;
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
      const float wj = tex1Dfetch<float>(a.tex, (int)jj[p]);
      const float u1 = __uint_as_float(0x3F800000u + (mix64_mhi(x[p]) >> 9));
      const float lo = __fmaf_rd(u1, wk[p], -wk[p]);
      const float hi = __fmaf_ru(wk[p], 0x1p-22f, lo);
      if (PMOV) {
        pmov_amb(lo, hi, wj, amb[p], t);
        pmov_acc(hi, wj, wk[p], bstar[p], t);
      } else {
        const bool acc = hi <= wj;
        if (!acc && lo <= wj) amb[p] = t;
        if (acc) { wk[p] = wj; bstar[p] = t; }
      }
      x[p] = ADDW ? add64_fma(x[p], a.one) : x[p] + M_CTR;
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    if (amb[p] >= 0) bstar[p] = megores_exact_rounds(a, oc, ii[p], wk0[p], true);
    uint32_t k = ii[p];
    if (bstar[p] >= 0) k = mux3((ii[p] - lane) + oc.o[bstar[p]].x, lane + oc.o[bstar[p]].y, cmask);
    a.anc[ii[p]] = (int64_t)k;
  }
}


struct OffT { uint32_t t[1024]; };
__device__ __forceinline__ uint32_t imad_hi(uint32_t a, uint32_t m) {  // (a * m) >> 32 on the FMA pipe
  uint32_t r; asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(m)); return r;
}
// XC: x = x0 + t * M_CTR as IMAD.WIDE.U32(t, C_lo, x0) + IMAD(t, C_hi, hi), t read from the param
//     space each round (ptxas cannot strength-reduce it into an IADD3 chain)
// SH: bit 0 -> (hi >> 27) as IMAD.HI(hi, 32); bit 1 -> (hi >> 30) as IMAD.HI(hi, 4)
// I2F: u bracket from I2F.U32.RZ (conversion pipe) instead of LEA.HI (ALU)
template <bool XC, int SH, bool I2F, int UNR>
__global__ void __launch_bounds__(256) k_w(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc,
                                          const __grid_constant__ OffT ot, uint32_t m4, uint32_t m32) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, cmask = (a.n - 1) & ~31u, ial = i - lane;
  float wk = tex1Dfetch<float>(a.tex, (int)i);
  const float wk0 = wk;
  int bstar = -1, amb = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
  uint64_t x = x0;
#pragma unroll UNR
  for (int t = 0; t < a.cnt; ++t) {
    const uint2 o = oc.o[t];
    const uint32_t j = mux3(ial + o.x, lane + o.y, cmask);
    const float wj = tex1Dfetch<float>(a.tex, (int)j);
    uint64_t xx;
    if (XC) {
      const uint32_t tt = ot.t[t];
      asm("{\n\t.reg .u32 lo, hi;\n\t"
          "mad.wide.u32 %0, %1, %2, %3;\n\t"
          "mov.b64 {lo, hi}, %0;\n\t"
          "mad.lo.u32 hi, %1, %4, hi;\n\t"
          "mov.b64 %0, {lo, hi};\n\t}"
          : "=l"(xx) : "r"(tt), "r"((uint32_t)M_CTR), "l"(x0), "r"((uint32_t)(M_CTR >> 32)));
    } else xx = x;
    uint32_t xl = (uint32_t)xx, xh = (uint32_t)(xx >> 32);
    // z = x ^ (x >> 30)
    uint32_t zl = xl ^ (uint32_t)(xx >> 30);
    uint32_t zh = xh ^ ((SH & 2) ? imad_hi(xh, m4) : (xh >> 30));
    uint64_t y = (((uint64_t)zh << 32) | zl) * MIX1;
    uint32_t yl = (uint32_t)y, yh = (uint32_t)(y >> 32);
    uint32_t vl = yl ^ (uint32_t)(y >> 27);
    uint32_t vh = yh ^ ((SH & 1) ? imad_hi(yh, m32) : (yh >> 27));
    const uint32_t m = __umulhi(vl, (uint32_t)MIX2) + vl * (uint32_t)(MIX2 >> 32) + vh * (uint32_t)MIX2;
    float lo, hi;
    if (I2F) {
      const float uf = __uint2float_rz(m);
      const float up = __fmaf_rd(uf, 0x1p-32f, -0x1p-32f);
      lo = __fmul_rd(up, wk);
      hi = __fmaf_ru(wk, 0x1.004p-22f, lo);
    } else {
      const float u1 = __uint_as_float(0x3F800000u + (m >> 9));
      lo = __fmaf_rd(u1, wk, -wk);
      hi = __fmaf_ru(wk, 0x1p-22f, lo);
    }
    const bool acc = hi <= wj;
    if (!acc && lo <= wj) amb = t;
    if (acc) { wk = wj; bstar = t; }
    if (!XC) x += M_CTR;
  }
  if (amb >= 0) bstar = megores_exact_rounds(a, oc, i, wk0, true);
  uint32_t k = i;
  if (bstar >= 0) k = mux3(ial + oc.o[bstar].x, lane + oc.o[bstar].y, cmask);
  a.anc[i] = (int64_t)k;
}

// PFMA: the accept updates as predicated FMA-pipe instructions (FFMA wj*1+0, IMAD t*1+0 with
// opaque 1 / 0 from the parameter space, so ptxas cannot turn them back into FSEL / SEL);
// AMBB: ambiguity as a bool (predicate accumulation) instead of a recorded round
template <bool PFMA, bool AMBB, bool ADDW, int UNR>
__global__ void __launch_bounds__(256) k_p(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc,
                                          float onef, float zerof, uint32_t onei, uint32_t zeroi) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u, cmask = (a.n - 1) & ~31u, ial = i - lane;
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
    const float u1 = __uint_as_float(0x3F800000u + (mix64_mhi(x) >> 9));
    const float lo = __fmaf_rd(u1, wk, -wk);
    const float hi = __fmaf_ru(wk, 0x1p-22f, lo);
    if (AMBB) amb |= (lo <= wj) && !(hi <= wj);
    else if (!(hi <= wj) && lo <= wj) ambt = t;
    if (PFMA) {
      asm("{\n\t.reg .pred p;\n\t"
          "setp.le.f32 p, %2, %3;\n\t"
          "@p fma.rn.f32 %0, %3, %5, %6;\n\t"
          "@p mad.lo.u32 %1, %4, %7, %8;\n\t}"
          : "+f"(wk), "+r"(bstar) : "f"(hi), "f"(wj), "r"(t), "f"(onef), "f"(zerof), "r"(onei), "r"(zeroi));
    } else {
      if (hi <= wj) { wk = wj; bstar = t; }
    }
    x = ADDW ? add64_fma(x, a.one) : x + M_CTR;
  }
  if (AMBB ? amb : ambt >= 0) bstar = megores_exact_rounds(a, oc, i, wk0, true);
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
  float t0 = time_it([&]() { k_megopolis_megores_f32<true><<<grid, 256>>>(a, oc); }, 7);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  printf("N=2^%d B=%d  lib megores_f32  %.3f ms  %.1f Gcmp/s\n", logn, B, t0, cmp / t0 / 1e6);
  ResampleArgs b = a;
  b.anc = anc1;
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("%-18s %.3f ms  %.1f Gcmp/s  speedup %.3f  mismatches %zu\n", name, ms, cmp / ms / 1e6, t0 / ms, bad);
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
  for (int rep = 0; rep < 2; ++rep) {
    check("p base ADDW", time_it([&]() { k_p<false, false, true, 8><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
    check("p PFMA ADDW", time_it([&]() { k_p<true, false, true, 8><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
    check("p AMBB ADDW", time_it([&]() { k_p<false, true, true, 8><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
    check("p PFMA AMBB ADDW", time_it([&]() { k_p<true, true, true, 8><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
    check("p PFMA AMBB", time_it([&]() { k_p<true, true, false, 8><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
    check("p PFMA AMBB ADDW u4", time_it([&]() { k_p<true, true, true, 4><<<grid, 256>>>(b, oc, 1.f, 0.f, 1u, 0u); }, 7));
  }
  return 0;
}
