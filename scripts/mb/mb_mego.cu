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

// state = wk * 2^-53 in float64 (exact for float32 weights), predicated update;
// TPARAM: the round counter comes from the parameter space (defeats strength reduction of
// the 64-bit key update onto the ALU pipe).
struct OffChunk4 { uint4 o[1024]; };  // {o_al, o_lo, t, 0}
template <bool TPARAM, int UNROLL>
__global__ void __launch_bounds__(256) k_vw(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk4 oc) {
  const uint32_t i = a.p0 + blockIdx.x * 256 + threadIdx.x;
  if (i >= a.p_end) return;
  const uint32_t lane = threadIdx.x & 31u, i_al = i - lane;
  const uint32_t cmask = (a.n - 1) & ~31u;
  double wks = (double)tex1Dfetch<float>(a.tex, (int)i) * 0x1p-53;
  int bstar = -1;
  const uint64_t x0 = megores_key(a.base, i, (uint64_t)a.b0);
  uint64_t x = x0;
#pragma unroll UNROLL
  for (int t = 0; t < a.cnt; ++t) {
    const uint4 o = oc.o[t];
    const uint32_t j = mux3(i_al + o.x, lane + o.y, cmask);
    const double wj = (double)tex1Dfetch<float>(a.tex, (int)j);
    const uint64_t xx = TPARAM ? x0 + (uint64_t)o.z * M_CTR : x;
    x += M_CTR;
    const double p = (double)mix64_m53(xx) * wks;  // == fl(u * wk) exactly
    if (p <= wj) { wks = wj * 0x1p-53; bstar = t; }
  }
  uint32_t k = i;
  if (bstar >= 0) { const uint4 o = oc.o[bstar]; k = mux3(i_al + o.x, lane + o.y, cmask); }
  a.anc[i] = (int64_t)k;
}


// Philox, two particles per thread (i and i + 128 of a 256-particle block): two independent
// Philox chains interleaved per thread.
template <int PPT>
__global__ void __launch_bounds__(256 / PPT) k_vp2(const __grid_constant__ ResampleArgs a, const __grid_constant__ OffChunk oc) {
  const uint32_t blk = a.p0 + blockIdx.x * 256;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t cmask = (a.n - 1) & ~31u;
  uint32_t ii[PPT], ial[PPT];
  double wkd[PPT];
  int bstar[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    ii[p] = blk + threadIdx.x + p * (256 / PPT);
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
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        const uint32_t wd = q == 0 ? c0[p] : q == 1 ? c1[p] : q == 2 ? c2[p] : c3[p];
        const uint32_t j = mux3(ial[p] + o.x, lane + o.y, cmask);
        const double wjd = (double)tex1Dfetch<float>(a.tex, (int)j);
        if (((double)wd * 0x1p-32) * wkd[p] <= wjd) { wkd[p] = wjd; bstar[p] = t; }
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
  static OffChunk4 o4;
  const uint64_t base = megores_base(seed);
  for (int t = 0; t < B; ++t) {
    const uint32_t o = (uint32_t)below_from_hash(mix64(megores_key(base, GLOBAL_OFFSET_LANE, t)), n);
    oc.o[t] = make_uint2(o & ~31u, o & 31u);
    o4.o[t] = make_uint4(o & ~31u, o & 31u, (uint32_t)t, 0u);
  }
  ResampleArgs a{};
  a.w = w; a.n = n; a.p0 = 0; a.p_end = n; a.seed = seed; a.base = base; a.b0 = 0; a.cnt = B;
  a.first = 1; a.last = 1; a.anc = anc0; a.tex = tex;
  const unsigned grid = n / 256;
  const double cmp = (double)n * B;
  float t0 = time_it([&]() { k_megopolis_w32<0, float, true, true, true><<<grid, 256>>>(a, oc); }, 7);
  std::vector<int64_t> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  printf("N=2^%d B=%d  lib  %.3f ms  %.1f Gcmp/s\n", logn, B, t0, cmp / t0 / 1e6);
  ResampleArgs b = a;
  b.anc = anc1;
  auto check = [&](const char* name, float ms) {
    CK(cudaMemcpy(h1.data(), anc1, 8ull * n, cudaMemcpyDeviceToHost));
    size_t bad = 0;
    for (uint32_t q = 0; q < n; ++q) bad += h0[q] != h1[q];
    printf("%-6s %.3f ms  %.1f Gcmp/s  speedup %.3f  mismatches %zu\n", name, ms, cmp / ms / 1e6, t0 / ms, bad);
    CK(cudaMemset(anc1, 0xff, 8ull * n));
  };
  {
    static OffChunk ocp;
    for (int t = 0; t < B; ++t) {
      const uint32_t o = (uint32_t)below_from_word(p4_word(philox_block(seed, GLOBAL_OFFSET_LANE, t >> 2), t & 3), n);
      ocp.o[t] = make_uint2(o & ~31u, o & 31u);
    }
    ResampleArgs c = a;
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; ++r) { c.pk0[r] = k0; c.pk1[r] = k1; k0 += PHILOX_W0; k1 += PHILOX_W1; }
    c.anc = anc0;
    float tp = time_it([&]() { k_megopolis_w32<1, float, true, true, true><<<grid, 256>>>(c, ocp); }, 7);
    CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
    printf("philox lib %.3f ms\n", tp);
    ResampleArgs d = c; d.anc = anc1;
    float t1 = time_it([&]() { k_vp2<1><<<grid, 256>>>(d, ocp); }, 7);
    check("vp2_1", t1);
    float t2 = time_it([&]() { k_vp2<2><<<grid, 128>>>(d, ocp); }, 7);
    check("vp2_2", t2);
    CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  }
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  t0 = time_it([&]() { k_megopolis_w32<0, float, true, true, true><<<grid, 256>>>(a, oc); }, 3);
  CK(cudaMemcpy(h0.data(), anc0, 8ull * n, cudaMemcpyDeviceToHost));
  check("vw4", time_it([&]() { k_vw<false, 4><<<grid, 256>>>(b, o4); }, 7));
  check("vwt4", time_it([&]() { k_vw<true, 4><<<grid, 256>>>(b, o4); }, 7));
  check("vwt2", time_it([&]() { k_vw<true, 2><<<grid, 256>>>(b, o4); }, 7));
  check("vwt8", time_it([&]() { k_vw<true, 8><<<grid, 256>>>(b, o4); }, 7));
  return 0;
}
