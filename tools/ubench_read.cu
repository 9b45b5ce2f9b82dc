// Microbenchmark: HBM streaming-read rate of the load paths the kernels use --
// (a) LDG.128 from many warps (registers), (b) cp.async.bulk into a shared-memory
// ring per SM (the TMA / bulk-copy engine), (c) cp.async.cg (LSU) into shared
// memory -- over a 1 GiB fp32 buffer (> L2), each element read once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ubench_read tools/ubench_read.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2407_09486_b200/csrc/common.cuh"
using namespace enova;
namespace enova {
void set_error(const std::string &) {}
enova_status cuda_status(cudaError_t, const char *) { return ENOVA_ERR_CUDA; }
void count_launch() {}
}

// (a) LDG: every thread streams float4 with U loads in flight
template <int U>
__global__ void __launch_bounds__(512) k_ldg(const float4 *__restrict__ x, size_t n4, float *out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(x + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) { const float4 v = __ldcs(x + i); acc += v.x + v.y + v.z + v.w; }
  if (acc == 1.2345f) out[0] = acc;
}

// (b) bulk copies: one CTA per SM, a producer thread keeps S chunks of CH bytes in
// flight, 512 consumer threads sum each chunk from shared memory
template <int S, int CH>
__global__ void __launch_bounds__(544, 1) k_bulk(const uint8_t *__restrict__ x, size_t bytes, float *out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[S], empty[S];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 16); }
    fence_mbar_init();
  }
  __syncthreads();
  const size_t per = (bytes / gridDim.x) / CH * CH;
  const uint8_t *base = x + (size_t)blockIdx.x * per;
  const int nch = (int)(per / CH);
  if (tid >= 512) {
    if (tid == 512)
      for (int k = 0; k < nch; ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(&empty[s], ((k / S) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], CH);
        bulk_g2s(sm + (size_t)s * CH, base + (size_t)k * CH, CH, &full[s]);
      }
    return;
  }
  float acc = 0.f;
  for (int k = 0; k < nch; ++k) {
    const int s = k % S;
    mbar_wait(&full[s], (k / S) & 1);
    const float4 *c = reinterpret_cast<const float4 *>(sm + (size_t)s * CH);
    for (int i = tid; i < CH / 16; i += 512) { const float4 v = c[i]; acc += v.x + v.y + v.z + v.w; }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 1.2345f) out[0] = acc;
}

// (c) cp.async.cg 16 B per thread-op into a shared ring, D groups in flight
template <int D>
__global__ void __launch_bounds__(512, 1) k_lsu(const uint8_t *__restrict__ x, size_t bytes, float *out) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int CH = 32768;   // bytes per group (64 B per thread)
  const int tid = threadIdx.x;
  const size_t per = (bytes / gridDim.x) / CH * CH;
  const uint8_t *base = x + (size_t)blockIdx.x * per;
  const int nch = (int)(per / CH);
  auto issue = [&](int k) {
    const uint32_t dst = smem_u32(sm + (size_t)(k % (D + 1)) * CH);
    for (int i = tid; i < CH / 16; i += 512)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16u * i),
                   "l"(base + (size_t)k * CH + 16 * (size_t)i) : "memory");
  };
  for (int k = 0; k < D; ++k) { if (k < nch) issue(k); asm volatile("cp.async.commit_group;" ::: "memory"); }
  float acc = 0.f;
  for (int k = 0; k < nch; ++k) {
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    __syncthreads();
    const float4 *c = reinterpret_cast<const float4 *>(sm + (size_t)(k % (D + 1)) * CH);
    for (int i = tid; i < CH / 16; i += 512) { const float4 v = c[i]; acc += v.x + v.y + v.z + v.w; }
    if (k + D < nch) issue(k + D);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const size_t bytes = (size_t)1 << 30;
  uint8_t *x;
  float *out;
  cudaMalloc(&x, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(x, 0, bytes);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char *name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-44s %7.1f GB/s  (%s)\n", name, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const size_t n4 = bytes / 16;
  timeit("LDG.128 U=4  2x512 thr/SM", [&] { k_ldg<4><<<2 * sms, 512>>>((const float4 *)x, n4, out); });
  timeit("LDG.128 U=8  2x512 thr/SM", [&] { k_ldg<8><<<2 * sms, 512>>>((const float4 *)x, n4, out); });
  timeit("LDG.128 U=8  4x512 thr/SM", [&] { k_ldg<8><<<4 * sms, 512>>>((const float4 *)x, n4, out); });
  timeit("LDG.128 U=16 2x512 thr/SM", [&] { k_ldg<16><<<2 * sms, 512>>>((const float4 *)x, n4, out); });
  cudaFuncSetAttribute(k_bulk<5, 32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 32768);
  cudaFuncSetAttribute(k_bulk<3, 65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536);
  cudaFuncSetAttribute(k_bulk<12, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
  timeit("bulk 5 x 32 KB, 1 CTA/SM", [&] { k_bulk<5, 32768><<<sms, 544, 5 * 32768>>>(x, bytes, out); });
  timeit("bulk 3 x 64 KB, 1 CTA/SM", [&] { k_bulk<3, 65536><<<sms, 544, 3 * 65536>>>(x, bytes, out); });
  timeit("bulk 12 x 16 KB, 1 CTA/SM", [&] { k_bulk<12, 16384><<<sms, 544, 12 * 16384>>>(x, bytes, out); });
  cudaFuncSetAttribute(k_lsu<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 32768);
  cudaFuncSetAttribute(k_lsu<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
  timeit("cp.async.cg 4 x 32 KB groups, 1 CTA/SM", [&] { k_lsu<4><<<sms, 512, 5 * 32768>>>(x, bytes, out); });
  timeit("cp.async.cg 5 x 32 KB groups, 1 CTA/SM", [&] { k_lsu<5><<<sms, 512, 6 * 32768>>>(x, bytes, out); });
  return 0;
}
