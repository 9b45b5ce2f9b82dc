// Microbenchmark: back-to-back tcgen05.mma cta_group::1 kind::f16 M=128 N=128
// K=16 from shared memory (one CTA), no-swizzle vs SWIZZLE_128B A/B operands.
// Prints cycles per MMA.  nvcc -gencode arch=compute_100a,code=sm_100a -I../include
#include <cstdio>
#include "../paper_2407_09486_b200/csrc/common.cuh"
using namespace enova;
namespace enova {
void set_error(const std::string &) {}
enova_status cuda_status(cudaError_t, const char *) { return ENOVA_ERR_CUDA; }
void count_launch() {}
}
__device__ __forceinline__ uint64_t sd_sw128(uint32_t a) {
  return ((uint64_t)((a >> 4) & 0x3FFF)) | (1ull << 16) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61);
}
template <int MODE>   // 0: A,B no-swizzle; 1: A sw128, B no-swizzle; 2: both sw128; 3: 1 + commit every 4 MMAs; 4: 1 + commit every MMA
__global__ void kbench(int nmma, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar, bar2[8];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 8; ++i) mbar_init(&bar2[i], 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&slot, 128);
  fence_proxy_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    const uint32_t id = make_idesc_f16(128, 128);
    unsigned long long t0 = clock64();
    for (int q = 0; q < nmma; ++q) {
      const int j = q & 3;
      uint64_t ad, bd;
      if (MODE == 0) { ad = make_sdesc(a + (q & 7) * 4096, 2048, 128); bd = make_sdesc(b + (q & 7) * 4096, 2048, 128); }
      else if (MODE == 1) { ad = sd_sw128(a + ((q >> 2) & 1) * 16384 + 32 * j); bd = make_sdesc(b + (q & 7) * 4096, 2048, 128); }
      else if (MODE == 2) { ad = sd_sw128(a + ((q >> 2) & 1) * 16384 + 32 * j); bd = sd_sw128(b + ((q >> 2) & 1) * 16384 + 32 * j); }
      else { ad = sd_sw128(a + ((q >> 2) & 1) * 16384 + 32 * j); bd = make_sdesc(b + (q & 7) * 4096, 2048, 128); }
      mma_f16_ss(tmem, ad, bd, id, q > 0);
      if (MODE == 3 && j == 3) mma_commit(&bar2[(q >> 2) & 7]);
      if (MODE == 4) mma_commit(&bar2[q & 7]);
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[MODE] = (t1 - t0);
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 128);
}
int main() {
  unsigned long long *d, h[5];
  cudaMalloc(&d, 64);
  const int n = 4096;
  cudaFuncSetAttribute(kbench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(kbench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(kbench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(kbench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(kbench<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) {
    kbench<0><<<1, 128, 65536>>>(n, d);
    kbench<1><<<1, 128, 65536>>>(n, d);
    kbench<2><<<1, 128, 65536>>>(n, d);
    kbench<3><<<1, 128, 65536>>>(n, d);
    kbench<4><<<1, 128, 65536>>>(n, d);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  printf("cycles per M128N128K16 MMA: noswz %.1f  A-sw128/B-noswz %.1f  both-sw128 %.1f  "
         "commit/4 %.1f  commit/1 %.1f\n",
         h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
}
