// Measurement probe (not on the product path): the read bandwidth the Megopolis kernel's
// roofline is quoted against.  bench.py loads libmgp_probe.so and times these launches with
// CUDA events on its own stream:
//
//   * mgpp_read_stream: every CTA streams float4 lines over an array of `bytes` (L1 bypassed
//     with ld.global.cg, so each load is an L2 request), `reps` passes per launch, grid-stride
//     with 4 independent loads in flight per thread.  For an array the L2 holds (the 64 MiB
//     float32 weights at N = 2^24) this is the L2 -> SM read bandwidth; for a 1+ GiB array it
//     is the HBM read bandwidth.
//   * mgpp_megopolis_read: the Megopolis access shape without its arithmetic -- round b, warp
//     w reads the 128-byte line (w*32 + o_b) mod N (M/resample.py:187-193), one float per lane
//     through the texture path like k_megopolis_philox_half -- i.e. the best a kernel issuing
//     exactly the Megopolis loads can do on this chip.
//
// Built by paper_2109_13504_b200/build.py next to libmgp.so (same nvcc flags).

#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ float4 ld_cg(const float4* p) {
  float4 v;
  asm volatile("ld.global.cg.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

__global__ void __launch_bounds__(512) k_read_stream(const float4* __restrict__ a, int64_t n4, int reps, float* sink) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  float acc = 0.f;
  for (int r = 0; r < reps; ++r) {
    int64_t i = t0;
    for (; i + 3 * stride < n4; i += 4 * stride) {
      const float4 v0 = ld_cg(a + i), v1 = ld_cg(a + i + stride), v2 = ld_cg(a + i + 2 * stride),
                   v3 = ld_cg(a + i + 3 * stride);
      acc += (v0.x + v1.y) + (v2.z + v3.w);
    }
    for (; i < n4; i += stride) acc += ld_cg(a + i).x;
  }
  if (acc == 1234.5f) sink[t0] = acc;  // never true for the probe's data: keeps the loads live
}

// the Megopolis load stream: thread (CTA c, lane l) of warp w handles particles
// i = w*32 + l over a grid-stride loop; per round one texture fetch of w[(i & ~31) + o_b + l]
__global__ void __launch_bounds__(256) k_megopolis_read(cudaTextureObject_t tex, uint32_t n, const uint32_t* off,
                                                         int b, float* sink) {
  const uint32_t lane = threadIdx.x & 31u;
  float acc = 0.f;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t base = i & ~31u;
    for (int r = 0; r < b; ++r) {
      const uint32_t o = __ldg(off + r);
      const uint32_t j = ((base + (o & ~31u)) & (n - 1)) | ((lane + o) & 31u);
      acc += tex1Dfetch<float>(tex, (int)j);
    }
  }
  if (acc == 1234.5f) sink[0] = acc;
}

}  // namespace

extern "C" {

int mgpp_read_stream(const void* d_a, int64_t bytes, int reps, int blocks, float* d_sink, void* stream) {
  if (!d_a || bytes < 16 || reps < 1 || blocks < 1) return -1;
  k_read_stream<<<blocks, 512, 0, (cudaStream_t)stream>>>((const float4*)d_a, bytes / 16, reps, d_sink);
  return (int)cudaGetLastError();
}

// n a power of two; d_off: b offsets (device); the texture is built and destroyed per call
int mgpp_megopolis_read(const float* d_w, uint32_t n, const uint32_t* d_off, int b, int blocks, float* d_sink,
                        void* stream) {
  if (!d_w || !d_off || n < 32 || (n & (n - 1)) || b < 1 || blocks < 1) return -1;
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = const_cast<float*>(d_w);
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = sizeof(float) * (size_t)n;
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  cudaError_t e = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  if (e != cudaSuccess) return (int)e;
  k_megopolis_read<<<blocks, 256, 0, (cudaStream_t)stream>>>(tex, n, d_off, b, d_sink);
  e = cudaGetLastError();
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaDestroyTextureObject(tex);
  return (int)e;
}

}  // extern "C"
