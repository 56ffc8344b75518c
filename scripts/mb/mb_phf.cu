// Microbenchmark: the Philox Megopolis kernel with a float32 bracket of the float64 decision
// (the megores kernel's idea applied to the Philox stream), against the library's
// k_megopolis_philox_half (float64 DFMA decision).  Every variant must reproduce the library's
// ancestors bit for bit.
//
// Decision: accept iff fl64(u wk) <= wj, u = word 2^-32.  With u23 = top 23 bits of word,
// lo = RD(u23 wk) <= u wk < hi = RU(wk 2^-22 + lo):  hi <= wj => accept; lo > wj => reject
// (lo >= wj + ulp32(wj) > wj + ulp64(wj)/2); otherwise ambiguous (~2^-21 per comparison).
// AMB 0: per Philox block (4 rounds x 4 particles) an ambiguity flag; a block that saw one is
//        re-run from its saved state with the exact float64 rule (words still in registers).
// AMB 1: the exact float64 decision inline under a per-comparison branch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false \
//        -I../../include -I../../paper_2109_13504_b200/csrc mb_phf.cu -o mb_phf
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "mgp_kernels.cuh"

using namespace mgp;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ unsigned long long g_redo;

template <int AMB, int MINB>
__global__ void __launch_bounds__(64, MINB) k_phf(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  constexpr int PPT = 4;
  const uint32_t half = a.n >> 1;
  const uint32_t i0 = a.p0 + blockIdx.x * 128 + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT];
  float wk[PPT];
  int bstar[PPT];
  ii[0] = i0; ii[1] = i0 + 64; ii[2] = i0 + half; ii[3] = i0 + half + 64;
  const uint32_t ial0 = i0 - lane, ial1 = ial0 + 64;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    wk[p] = tex1Dfetch<float>(a.tex, (int)ii[p]);
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
    float wks[PPT];
    int bss[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) { wks[p] = wk[p]; bss[p] = bstar[p]; }
    bool amb = false;
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
          const float wj = tex1Dfetch<float>(a.tex, (int)jj[p]);
          const float u1 = __uint_as_float(0x3F800000u + (wd >> 9));  // 1 + u23
          const float lo = __fmaf_rd(u1, wk[p], -wk[p]);
          const float hi = __fmaf_ru(wk[p], 0x1p-22f, lo);
          bool acc = hi <= wj;
          if (AMB == 1) {
            if (!acc && lo <= wj) {  // rare: the exact rule
              const double wkd = (double)wk[p];
              acc = fma(u1_from_word(wd), wkd, -wkd) <= (double)wj;
            }
          } else {
            amb |= !acc && lo <= wj;
          }
          if (acc) { wk[p] = wj; bstar[p] = t; }
        }
      }
    }
    if (AMB == 0 && amb) {  // rare: re-run the block's rounds exactly from the saved state
      atomicAdd(&g_redo, 1ull);
#pragma unroll
      for (int p = 0; p < PPT; ++p) { wk[p] = wks[p]; bstar[p] = bss[p]; }
      for (int q = 0; q < lim; ++q) {
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
          const float wj = tex1Dfetch<float>(a.tex, (int)jj[p]);
          const double wkd = (double)wk[p];
          if (fma(u1_from_word(wd), wkd, -wkd) <= (double)wj) { wk[p] = wj; bstar[p] = t; }
        }
      }
    }
  };
  for (int t0 = 0; t0 < full; t0 += 4) body(t0, 4);
  if (full < a.cnt) body(full, a.cnt - full);
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    uint32_t k = ii[p];
    if (bstar[p] >= 0) { const uint2 o = oc.o[bstar[p]]; k = mux3((ii[p] - lane) + o.x, lane + o.y, cmask); }
    a.anc[(int64_t)ii[p] - (p >= 2 ? a.hi_shift : 0)] = (int64_t)k;
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
  const int B = argc > 2 ? atoi(argv[2]) : 354;
  const double y = argc > 3 ? atof(argv[3]) : 4.0;
  const uint32_t n = 1u << logn;
  const uint64_t seed = 7;
  float* w;
  int64_t *anc0, *anc1;
  CK(cudaMalloc(&w, sizeof(float) * n));
  CK(cudaMalloc(&anc0, sizeof(int64_t) * n));
  CK(cudaMalloc(&anc1, sizeof(int64_t) * n));
  k_gen_gaussian<float><<<148 * 32, 256>>>(y, n, 20240, w);
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
  a.w = w; a.n = n; a.p0 = 0; a.p_end = n / 2; a.seed = seed; a.base = megores_base(seed); a.b0 = 0; a.cnt = B;
  a.first = 1; a.last = 1; a.anc = anc0; a.tex = tex; a.one = 1; a.half = 1; a.hi_shift = 0;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) { a.pk0[r] = k0; a.pk1[r] = k1; k0 += PHILOX_W0; k1 += PHILOX_W1; }
  const double cmp = (double)n * B;
  float t0 = time_it([&]() { k_megopolis_philox_half<<<n / 256, 64>>>(a, oc); }, 9);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  printf("N=2^%d B=%d y=%.1f  lib philox_half %.3f ms  %.1f Gcmp/s\n", logn, B, y, t0, cmp / t0 / 1e6);
  ResampleArgs b = a;
  b.anc = anc1;
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    unsigned long long redo = 0;
    CK(cudaMemcpyFromSymbol(&redo, g_redo, sizeof redo));
    printf("%-16s %.3f ms  %.1f Gcmp/s  speedup %.3f  mismatches %zu  redo-blocks %llu\n", name, ms, cmp / ms / 1e6,
           t0 / ms, bad, redo);
    unsigned long long z = 0;
    CK(cudaMemcpyToSymbol(g_redo, &z, sizeof z));
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
  check("f32 blockredo", time_it([&]() { k_phf<0, 1><<<n / 256, 64>>>(b, oc); }, 9));
  check("f32 inline", time_it([&]() { k_phf<1, 1><<<n / 256, 64>>>(b, oc); }, 9));
  check("f32 blockredo m2", time_it([&]() { k_phf<0, 2><<<n / 256, 64>>>(b, oc); }, 9));
  check("f32 inline m2", time_it([&]() { k_phf<1, 2><<<n / 256, 64>>>(b, oc); }, 9));
  check("f32 blockredo m12", time_it([&]() { k_phf<0, 12><<<n / 256, 64>>>(b, oc); }, 9));
  check("f32 inline m12", time_it([&]() { k_phf<1, 12><<<n / 256, 64>>>(b, oc); }, 9));
  return 0;
}
