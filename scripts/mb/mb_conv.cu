// Microbenchmark: conversion strategies in the Philox Megopolis kernel (f32, W=32, pow2 N,
// no zero weights).  Every variant must reproduce the library kernel's ancestors bit for bit.
//   CU (uniform):   0 = I2F.F64.U32 + DMUL 2^-32 (+ DMUL by w_k)       [library]
//                   1 = u1 = 1 + word*2^-32 assembled from bits; fl(u*w_k) = DFMA(u1, w_k, -w_k)
//   CW (weight):    0 = F2F.F64.F32                                     [library]
//                   1 = D-domain: the f32 bit pattern b reinterpreted as the double
//                       {hi = b >> 3, lo = b << 29} == w * 2^-896 exactly (all weights normal)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
//        -I../../include -I../../paper_2109_13504_b200/csrc mb_conv.cu -o mb_conv
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "mgp_kernels.cuh"

using namespace mgp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ double u1_bits(uint32_t wd) {  // 1 + wd * 2^-32, exact
  return __hiloint2double((int)((wd >> 12) + 0x3FF00000u), (int)(wd << 20));
}
__device__ __forceinline__ double dbits(uint32_t b) {  // f32 bits -> double (w * 2^-896)
  return __hiloint2double((int)(b >> 3), (int)(b << 29));
}

template <int PPT, int CU, int CW, int MINB, int SU = 0>
__global__ void __launch_bounds__(256 / PPT, MINB) k_var(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  constexpr int STRIDE = 256 / PPT;
  const uint32_t i0 = a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT], ial[PPT];
  double wkd[PPT];
  int bstar[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ii[p] = i0 + p * STRIDE;
    ial[p] = ii[p] - lane;
    const float f = tex1Dfetch<float>(a.tex, (int)ii[p]);
    wkd[p] = CW ? dbits(__float_as_uint(f)) : (double)f;
    bstar[p] = -1;
  }
  const double one_d = __hiloint2double((int)(a.one * 0x3FF00000u), 0);
  const int full = a.cnt & ~3;
  for (int t0 = 0; t0 < full; t0 += 4) {
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
      const int t = t0 + q;
      const uint2 o = oc.o[t];
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
        const uint32_t j = mux3(ial[p] + o.x, lane + o.y, cmask);
        const float f = tex1Dfetch<float>(a.tex, (int)j);
        const double wjd = CW ? dbits(__float_as_uint(f)) : (double)f;
        double prod;
        if (CU) prod = fma(u1_bits(wd), wkd[p], -wkd[p]);
        else prod = ((double)wd * 0x1p-32) * wkd[p];
        if (SU == 0) {
          if (prod <= wjd) { wkd[p] = wjd; bstar[p] = t; }
        } else if (SU == 1) {  // predicated DMUL by an opaque 1.0 (FP64 pipe) instead of 2 FSEL
          asm("{\n\t.reg .pred q;\n\tsetp.le.f64 q, %2, %3;\n\t@q mul.rn.f64 %0, %3, %4;\n\t@q mov.b32 %1, %5;\n\t}"
              : "+d"(wkd[p]), "+r"(bstar[p]) : "d"(prod), "d"(wjd), "d"(one_d), "r"(t));
        } else {  // + bstar through a predicated IMAD (FMA pipe)
          asm("{\n\t.reg .pred q;\n\tsetp.le.f64 q, %2, %3;\n\t@q mul.rn.f64 %0, %3, %4;\n\t@q mad.lo.u32 %1, %5, %6, 0;\n\t}"
              : "+d"(wkd[p]), "+r"(bstar[p]) : "d"(prod), "d"(wjd), "d"(one_d), "r"(t), "r"(a.one));
        }
      }
    }
  }
  // (B % 4 == 0 in this harness)
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = ii[p];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3(ial[p] + o.x, lane + o.y, cmask); }
    a.anc[ii[p]] = (int64_t)k;
  }
}


// Duplicated weights (w2[x] = w[x mod N] for x < 2N): the partner index needs no wrap,
// j_p = ial_p + X with X = o_al + ((lane + o_lo) & 31) shared by the thread's particles.
template <int PPT, int MINB>
__global__ void __launch_bounds__(256 / PPT, MINB) k_dup(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  constexpr int STRIDE = 256 / PPT;
  const uint32_t i0 = a.p0 + blockIdx.x * 256 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT], ial[PPT];
  double wkd[PPT];
  int bstar[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ii[p] = i0 + p * STRIDE;
    ial[p] = ii[p] - lane;
    wkd[p] = (double)tex1Dfetch<float>(a.tex, (int)ii[p]);
    bstar[p] = -1;
  }
  const int full = a.cnt & ~3;
  for (int t0 = 0; t0 < full; t0 += 4) {
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
      const int t = t0 + q;
      const uint2 o = oc.o[t];
      const uint32_t X = o.x + ((lane + o.y) & 31u);
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
        const double wjd = (double)tex1Dfetch<float>(a.tex, (int)(ial[p] + X));
        const double prod = fma(u1_bits(wd), wkd[p], -wkd[p]);
        if (prod <= wjd) { wkd[p] = wjd; bstar[p] = t; }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = ii[p];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3(ial[p] + o.x, lane + o.y, cmask); }
    a.anc[ii[p]] = (int64_t)k;
  }
}


// Full-range variant: thread owns particles {i, i+64, i+N/2, i+N/2+64}.  Partners of
// i + N/2 are those of i with the top index bit flipped: j(i + N/2) = j(i) ^ N/2.
// GEN: general launch state (first/kstate/last, tail rounds).
template <int MINB, bool GEN = false, bool ONELOOP = false, bool KST = true>
__global__ void __launch_bounds__(64, MINB) k_x2(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  constexpr int PPT = 4;
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = blockIdx.x * 128 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT];
  double wkd[PPT];
  int bstar[PPT];
  ii[0] = i0; ii[1] = i0 + 64; ii[2] = i0 + half; ii[3] = i0 + half + 64;
  const uint32_t ial0 = i0 - lane, ial1 = ial0 + 64;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const uint32_t k0 = (GEN && KST) ? (a.first ? ii[p] : (uint32_t)a.kstate[ii[p]]) : ii[p];
    wkd[p] = (double)tex1Dfetch<float>(a.tex, (int)k0);
    bstar[p] = -1;
  }
  const int full = a.cnt & ~3;
  auto body = [&](int t0, int lim) {
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
          const double prod = fma(u1_bits(wd), wkd[p], -wkd[p]);
          if (prod <= wjd) { wkd[p] = wjd; bstar[p] = t; }
        }
      }
    }
  };
  if (ONELOOP) {
    for (int t0 = 0; t0 < a.cnt; t0 += 4) body(t0, min(4, a.cnt - t0));
  } else {
    for (int t0 = 0; t0 < full; t0 += 4) body(t0, 4);
    if (GEN && full < a.cnt) body(full, a.cnt - full);
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = (GEN && KST) ? (a.first ? ii[p] : (uint32_t)a.kstate[ii[p]]) : ii[p];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3((ii[p] - lane) + o.x, lane + o.y, cmask); }
    if (!GEN || !KST || a.last) a.anc[ii[p]] = (int64_t)k;
    else a.kstate[ii[p]] = (int32_t)k;
  }
}


// Software-pipelined half-split: the Philox block of the next group is computed in the same
// basic block as the compares of the current one.  PPT 4 ({i, i+64, i+N/2, i+N/2+64}) or
// PPT 2 ({i, i+N/2}).  No tail (B % 4 == 0 harness).
template <int PPT, int MINB>
__global__ void __launch_bounds__(PPT == 4 ? 64 : 128, MINB) k_sp(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t half = a.n >> 1;
  constexpr int LOWC = PPT == 4 ? 128 : 128;  // lower-half particles per CTA
  const uint32_t i0 = blockIdx.x * LOWC + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT];
  if (PPT == 4) { ii[0] = i0; ii[1] = i0 + 64; ii[2] = i0 + half; ii[3] = i0 + half + 64; }
  else { ii[0] = i0; ii[1] = i0 + half; }
  const uint32_t ial0 = i0 - lane, ial1 = ial0 + 64;
  double wkd[PPT];
  int bstar[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) { wkd[p] = (double)tex1Dfetch<float>(a.tex, (int)ii[p]); bstar[p] = -1; }
  auto philox = [&](int t0, uint32_t (&c0)[PPT], uint32_t (&c1)[PPT], uint32_t (&c2)[PPT], uint32_t (&c3)[PPT]) {
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
  };
  uint32_t c0[PPT], c1[PPT], c2[PPT], c3[PPT];
  philox(0, c0, c1, c2, c3);
  const int full = a.cnt & ~3;
  for (int t0 = 0; t0 < full; t0 += 4) {
    uint32_t d0[PPT], d1[PPT], d2[PPT], d3[PPT];
    philox(t0 + 4, d0, d1, d2, d3);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int t = t0 + q;
      const uint2 o = oc.o[t];
      const uint32_t L = lane + o.y;
      uint32_t jj[PPT];
      jj[0] = mux3(ial0 + o.x, L, cmask);
      if (PPT == 4) { jj[1] = mux3(ial1 + o.x, L, cmask); jj[2] = jj[0] ^ half; jj[3] = jj[1] ^ half; }
      else jj[1] = jj[0] ^ half;
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
        const double wjd = (double)tex1Dfetch<float>(a.tex, (int)jj[p]);
        if (fma(u1_bits(wd), wkd[p], -wkd[p]) <= wjd) { wkd[p] = wjd; bstar[p] = t; }
      }
    }
#pragma unroll
    for (int p = 0; p < PPT; ++p) { c0[p] = d0[p]; c1[p] = d1[p]; c2[p] = d2[p]; c3[p] = d3[p]; }
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = ii[p];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3((ii[p] - lane) + o.x, lane + o.y, cmask); }
    a.anc[ii[p]] = (int64_t)k;
  }
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
  const int B = argc > 2 ? atoi(argv[2]) : 352;  // multiple of 4 for this harness
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
  for (int t = 0; t < B; ++t) {
    const uint32_t o = (uint32_t)below_from_word(p4_word(philox_block(seed, GLOBAL_OFFSET_LANE, t >> 2), t & 3), n);
    oc.o[t] = make_uint2(o & ~31u, o & 31u);
  }
  ResampleArgs a{};
  a.w = w; a.n = n; a.p0 = 0; a.p_end = n; a.seed = seed; a.base = megores_base(seed); a.b0 = 0; a.cnt = B;
  a.first = 1; a.last = 1; a.anc = anc0; a.tex = tex; a.one = 1;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) { a.pk0[r] = k0; a.pk1[r] = k1; k0 += PHILOX_W0; k1 += PHILOX_W1; }
  const unsigned grid = n / 256;
  const double cmp = (double)n * B;
  const double alg = (double)n * (B + 1) * 4 + (double)n * 8;
  float t0 = time_it([&]() { k_megopolis_w32<1, float, true, true, true, 4><<<grid, 64>>>(a, oc); }, 9);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  printf("N=2^%d B=%d  lib(ppt4) %.3f ms  %.1f Gcmp/s  alg %.0f GB/s\n", logn, B, t0, cmp / t0 / 1e6, alg / t0 / 1e6);
  ResampleArgs b = a;
  b.anc = anc1;
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("%-14s %.3f ms  %.1f Gcmp/s  alg %.0f GB/s  speedup %.3f  mismatches %zu\n", name, ms, cmp / ms / 1e6,
           alg / ms / 1e6, t0 / ms, bad);
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
#define RUN(P, U, W, M, S) check("p" #P " u" #U " w" #W " m" #M " s" #S, time_it([&]() { k_var<P, U, W, M, S><<<grid, 256 / P>>>(b, oc); }, 9))
  RUN(4, 1, 0, 1, 0);
  check("lib HALF", time_it([&]() { k_megopolis_w32<1, float, true, true, true, 4, true><<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 p4", time_it([&]() { k_x2<1><<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 gen", time_it([&]() { k_x2<1, true><<<n / 256, 64>>>(b, oc); }, 9));
  {  // wave quantisation probe: grids of whole waves (148 SMs x CTAs per SM) vs the full grid
    int bps = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_megopolis_w32<1, float, true, true, true, 4, true>, 64, 0));
    const int slots = 148 * bps, full = (int)(n / 256);
    for (int g : {full, full / slots * slots, full / slots * slots - slots / 2}) {
      float ms = time_it([&]() { k_megopolis_w32<1, float, true, true, true, 4, true><<<g, 64>>>(b, oc); }, 9);
      printf("grid %d (%.2f waves of %d): %.3f ms, %.4f ms per 1000 CTAs\n", g, (double)g / slots, slots, ms,
             ms / g * 1000);
    }
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  }
  check("lib philox_half", time_it([&]() { k_megopolis_philox_half<<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 gen m11", time_it([&]() { k_x2<11, true><<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 gen m12", time_it([&]() { k_x2<12, true><<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 gen m14", time_it([&]() { k_x2<14, true><<<n / 256, 64>>>(b, oc); }, 9));
  check("sp p4", time_it([&]() { k_sp<4, 1><<<n / 256, 64>>>(b, oc); }, 9));
  check("sp p2", time_it([&]() { k_sp<2, 1><<<n / 256, 128>>>(b, oc); }, 9));
  check("x2 gen nokst", time_it([&]() { k_x2<1, true, false, false><<<n / 256, 64>>>(b, oc); }, 9));
  check("x2 gen", time_it([&]() { k_x2<1, true><<<n / 256, 64>>>(b, oc); }, 9));
  {
    float* w2;
    CK(cudaMalloc(&w2, sizeof(float) * 2 * n));
    CK(cudaMemcpy(w2, w, sizeof(float) * n, cudaMemcpyDeviceToDevice));
    CK(cudaMemcpy(w2 + n, w, sizeof(float) * n, cudaMemcpyDeviceToDevice));
    cudaResourceDesc rd2 = rd;
    rd2.res.linear.devPtr = w2;
    rd2.res.linear.sizeInBytes = sizeof(float) * 2 * n;
    cudaTextureObject_t tex2 = 0;
    CK(cudaCreateTextureObject(&tex2, &rd2, &td, nullptr));
    ResampleArgs d = b;
    d.tex = tex2;
    check("dup p4", time_it([&]() { k_dup<4, 1><<<grid, 64>>>(d, oc); }, 9));
    check("dup p2", time_it([&]() { k_dup<2, 1><<<grid, 128>>>(d, oc); }, 9));
    check("dup p8", time_it([&]() { k_dup<8, 1><<<grid, 32>>>(d, oc); }, 9));
    float tc = time_it([&]() { CK(cudaMemcpyAsync(w2, w, sizeof(float) * n, cudaMemcpyDeviceToDevice));
                               CK(cudaMemcpyAsync(w2 + n, w, sizeof(float) * n, cudaMemcpyDeviceToDevice)); }, 9);
    printf("duplicate copy %.3f ms\n", tc);
  }
  return 0;
}
