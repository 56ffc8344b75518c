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
  check("vw4", time_it([&]() { k_vw<false, 4><<<grid, 256>>>(b, o4); }, 7));
  check("vwt4", time_it([&]() { k_vw<true, 4><<<grid, 256>>>(b, o4); }, 7));
  check("vwt2", time_it([&]() { k_vw<true, 2><<<grid, 256>>>(b, o4); }, 7));
  check("vwt8", time_it([&]() { k_vw<true, 8><<<grid, 256>>>(b, o4); }, 7));
  return 0;
}
