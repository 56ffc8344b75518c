// Per-SASS-instruction throughput on B200 (cycles per warp-instruction per SM sub-partition).
// 8 independent dependency chains per thread, 64 warps per SM, long unrolled loops.
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int ITERS = 2048;

#define CHAINS8(OP) OP(a0) OP(a1) OP(a2) OP(a3) OP(a4) OP(a5) OP(a6) OP(a7)
#define RING8(OP) OP(a0, a1) OP(a1, a2) OP(a2, a3) OP(a3, a4) OP(a4, a5) OP(a5, a6) OP(a6, a7) OP(a7, a0)

template <int K>
__global__ void __launch_bounds__(256) kop(uint64_t* out, uint32_t s1, uint32_t s2, long long* cyc) {
  __syncthreads();
  long long c0 = clock64();
  unsigned long long g0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 ^ 9, a5 = a0 + 11, a6 = a0 * 13, a7 = a0 + 17;
  uint32_t b0 = a0 + 1, b1 = a1 + 2, b2 = a2 + 3, b3 = a3 + 4, b4 = a4 + 5, b5 = a5 + 6, b6 = a6 + 7, b7 = a7 + 8;
  uint64_t dd = a0; double d0 = a0, d1 = a1, d2 = a2, d3 = a3, d4 = a4, d5 = a5, d6 = a6, d7 = a7;
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (K == 0) {  // LOP3 (xor)
#define OP(a, b) asm volatile("xor.b32 %0, %0, %1;" : "+r"(a) : "r"(b));
        RING8(OP)
#undef OP
      } else if (K == 1) {  // SHF.R.U32.HI
#define OP(a, b) asm volatile("shr.b32 %0, %1, %2;" : "=r"(a) : "r"(b), "r"(s1));
        RING8(OP)
#undef OP
      } else if (K == 2) {  // funnel shift SHF.R.W
#define OP(a, b) asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(s1));
        RING8(OP)
#undef OP
      } else if (K == 3) {  // IMAD
#define OP(a, b) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(s2));
        RING8(OP)
#undef OP
      } else if (K == 4) {  // IMAD.WIDE
#define OP(a, b) { uint64_t t; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(t) : "r"(a), "r"(b), "l"(dd)); dd = t; a = (uint32_t)t; }
        RING8(OP)
#undef OP
      } else if (K == 5) {  // IMAD.HI
#define OP(a, b) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(s2));
        RING8(OP)
#undef OP
      } else if (K == 6) {  // IADD3
#define OP(a, b) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
        RING8(OP)
#undef OP
      } else if (K == 7) {  // DMUL
#define OPD(d) asm volatile("mul.rn.f64 %0, %0, %0;" : "+d"(d));
        OPD(d0) OPD(d1) OPD(d2) OPD(d3) OPD(d4) OPD(d5) OPD(d6) OPD(d7)
#undef OPD
      } else if (K == 8) {  // I2F.F64.U64
#define OPC(a, b) { uint64_t v; asm volatile("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(a), "r"(b)); double t; asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(t) : "l"(v)); asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "d"(t)); }
        OPC(a0, a1) OPC(a2, a3) OPC(a4, a5) OPC(a6, a7) OPC(a1, a2) OPC(a3, a4) OPC(a5, a6) OPC(a7, a0)
#undef OPC
      } else if (K == 9) {  // F2F.F64.F32
#define OPC(a, b) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(__uint_as_float(a))); asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(b), "=r"(a) : "d"(t)); }
        OPC(a0, a1) OPC(a2, a3) OPC(a4, a5) OPC(a6, a7) OPC(a1, a2) OPC(a3, a4) OPC(a5, a6) OPC(a7, a0)
#undef OPC
      } else if (K == 10) {  // SEL via selp
#define OP(a, b) asm volatile("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.b32 %0, %2, %3, p;}" : "=r"(a) : "r"(s2), "r"(b), "r"(a));
        RING8(OP)
#undef OP
      } else if (K == 11) {  // 3-input LOP3
#define OP(a, b) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(b1));
        RING8(OP)
#undef OP
      } else if (K == 12) {  // IADD/VIADD with immediate
#define OP(a, b) asm volatile("add.u32 %0, %1, 12345;" : "=r"(a) : "r"(b));
        RING8(OP)
#undef OP
      } else if (K == 13) {  // mixed: LOP3 and IMAD alternating (dual pipe)
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a0) : "r"(a1));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a1) : "r"(a2), "r"(s2));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a2) : "r"(a3));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a3) : "r"(a4), "r"(s2));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a4) : "r"(a5));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a5) : "r"(a6), "r"(s2));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a6) : "r"(a7));
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a7) : "r"(a0), "r"(s2));
      } else if (K == 14) {  // FFMA (fma-lite eligible)
#define OPF(a) { float f = __uint_as_float(a); asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0001f), "f"(0.5f)); a = __float_as_uint(f); }
        CHAINS8(OPF)
#undef OPF
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    cyc[0] = clock64() - c0;
    cyc[1] = (long long)(g1 - g0);
  }
  out[blockIdx.x * 256 + threadIdx.x] = (uint64_t)(a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7) +
                                        dd + (uint64_t)(d0 + d1 + d2 + d3 + d4 + d5 + d6 + d7);
}

template <int K>
void run(const char* name, uint64_t* out, long long* cyc, int sms, int nop) {
  const int blocks = sms * 8 * 4;  // several waves
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kop<K><<<blocks, 256>>>(out, 3, 5, cyc);
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  kop<K><<<blocks, 256>>>(out, 3, 5, cyc);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  long long h[2];
  CK(cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost));
  const double ghz = (double)h[0] / (double)h[1];
  const double warp_instr = (double)blocks * 8 * ITERS * nop;  // op instructions
  const double smsp_cycles = ms * 1e-3 * ghz * 1e9 * sms * 4;
  printf("%-14s %7.3f ms  clk %.3f GHz  %.2f cycles per warp-op per SMSP\n", name, ms, ghz, smsp_cycles / warp_instr);
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  uint64_t* out;
  long long* cyc;
  CK(cudaMalloc(&out, sizeof(uint64_t) * sms * 32 * 256));
  CK(cudaMalloc(&cyc, sizeof(long long) * sms * 8));
  run<0>("LOP3 xor", out, cyc, sms, 18);
  run<11>("LOP3 3-in", out, cyc, sms, 32);
  run<1>("SHF.R.U32", out, cyc, sms, 32);
  run<2>("SHF funnel", out, cyc, sms, 32);
  run<6>("IADD reg", out, cyc, sms, 32);
  run<12>("IADD imm", out, cyc, sms, 4);
  run<10>("SEL", out, cyc, sms, 32);
  run<3>("IMAD", out, cyc, sms, 32);
  run<4>("IMAD.WIDE+x", out, cyc, sms, 32);
  run<5>("IMAD.HI", out, cyc, sms, 32);
  run<13>("LOP3|IMAD mix", out, cyc, sms, 32);
  run<14>("FFMA", out, cyc, sms, 32);
  run<7>("DMUL", out, cyc, sms, 32);
  run<8>("I2F.F64.U64+", out, cyc, sms, 32);
  run<9>("F2F.F64.F32+", out, cyc, sms, 32);
  return 0;
}
