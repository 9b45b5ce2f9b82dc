// ubench_xu.cu -- throughput of the epilogue's instruction classes on this GPU
// (MUFU ex2/tanh/rcp, f32->f16 conversions, f16->f32, FFMA), ops/clk/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_xu tools/ubench_xu.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>

#define CHAINS 8
#define ITERS 4096

template <int OP>
__global__ void k(float *out, float seed) {
  float v[CHAINS];
  uint32_t u[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    v[c] = seed + 0.001f * (threadIdx.x + c);
    u[c] = threadIdx.x * 7 + c;
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
      if (OP == 1) asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[c]));
      if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(v[c]));
      if (OP == 3) {
        uint32_t r;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[c]), "f"(v[c]));
        u[c] ^= r;
        v[c] = __uint_as_float(u[c] & 0x3f7fffff);
      }
      if (OP == 4) {
        unsigned short r;
        asm volatile("cvt.rn.f16.f32 %0, %1;" : "=h"(r) : "f"(v[c]));
        u[c] ^= r;
        v[c] = __uint_as_float(u[c] & 0x3f7fffff);
      }
      if (OP == 5) {
        float r;
        asm volatile("cvt.f32.f16 %0, %1;" : "=f"(r) : "h"((unsigned short)u[c]));
        u[c] += __float_as_uint(r);
      }
      if (OP == 6) asm volatile("fma.rn.f32 %0, %0, 0f3F800001, 0f3C000000;" : "+f"(v[c]));
      if (OP == 7) {  // integer ops only (alu): and + add
        u[c] = (u[c] & 0x7fffe000u) + 0x1234u;
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += v[c] + (float)u[c];
  if (s == 12345.f) out[0] = s;
}

template <int OP>
void run(const char *name, float *out, int sms, int clk_khz) {
  int blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<OP><<<blocks, threads>>>(out, 0.5f);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(out, 0.5f);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * CHAINS * ITERS;
  double per_clk_sm = ops / (ms * 1e-3) / sms / (clk_khz * 1e3);
  printf("%-28s %8.3f ms  %7.1f ops/clk/SM (at %d MHz)\n", name, ms, per_clk_sm, clk_khz / 1000);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *out;
  cudaMalloc(&out, 4);
  printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
  run<0>("ex2.approx.ftz.f32", out, p.multiProcessorCount, clk);
  run<1>("tanh.approx.f32", out, p.multiProcessorCount, clk);
  run<2>("rcp.approx.ftz.f32", out, p.multiProcessorCount, clk);
  run<3>("cvt.rn.f16x2.f32 (+2 alu)", out, p.multiProcessorCount, clk);
  run<4>("cvt.rn.f16.f32 (+2 alu)", out, p.multiProcessorCount, clk);
  run<5>("cvt.f32.f16 (+1 alu)", out, p.multiProcessorCount, clk);
  run<6>("fma.rn.f32", out, p.multiProcessorCount, clk);
  run<7>("and+add (alu)", out, p.multiProcessorCount, clk);
  return 0;
}
