// Microbenchmark + layout check: tcgen05.mma cta_group::2 kind::f16 with the A
// operand in TENSOR MEMORY ("TS" form) vs shared memory ("SS" form).
//
// Layout hypothesis checked here (K2 v5 keeps h and mu in TMEM this way): A row m
// of the pair tile lives in lane (m mod 128) of CTA (m / 128); 32-bit column c of
// a K=16 step holds the fp16 pair (k = 2c in the low half, k = 2c+1 in the high
// half), so a K=16 step spans 8 consecutive columns.  B (K-major, no swizzle) is
// split N/2 rows per CTA as in K2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/ubench_ts tools/ubench_ts.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_fp16.h>
#include "../paper_2407_09486_b200/csrc/common.cuh"
#include "../paper_2407_09486_b200/csrc/layout.h"
using namespace enova;
namespace enova {
void set_error(const std::string &) {}
enova_status cuda_status(cudaError_t, const char *) { return ENOVA_ERR_CUDA; }
void count_launch() {}
}

__device__ __forceinline__ void mma_ts_pair(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

// check: D[256 x N] = A[256 x K] B[N x K]^T with A in TMEM, K = KS*16
template <int N, int KS>
__global__ void __cluster_dims__(2, 1, 1) kcheck(const __half *A, const __half *B, float *D) {
  __shared__ __align__(1024) uint8_t bs[(N / 2) * KS * 16 * 2];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const uint32_t rank = cluster_ctarank();
  // B half (rows rank*N/2 ..) as a K-step image
  for (int i = threadIdx.x; i < (N / 2) * KS * 16; i += blockDim.x) {
    const int nl = i / (KS * 16), k = i % (KS * 16);
    *reinterpret_cast<__half *>(bs + kmajor_step_offset(nl, k, N / 2)) =
        B[(rank * (N / 2) + nl) * KS * 16 + k];
  }
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  cluster_sync_all();
  if (threadIdx.x < 32) tmem_alloc_pair(&slot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = rank * 128 + warp * 32 + lane;
  const uint32_t a_col = 128;   // A at columns [128, 128 + 8 KS)
  {
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16) + a_col;
    for (int c = 0; c < 8 * KS; c += 8) {
      float v[8];
      for (int j = 0; j < 8; ++j) {
        const __half lo = A[row * KS * 16 + 2 * (c + j)], hi = A[row * KS * 16 + 2 * (c + j) + 1];
        v[j] = __uint_as_float((uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16));
      }
      tmem_st8(la + c, v);
    }
    tmem_wait_st();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t id = make_idesc_f16(256, N);
    for (int s = 0; s < KS; ++s) {
      const uint64_t bd = make_sdesc(smem_u32(bs) + s * 32 * (N / 2), 16 * (N / 2), 128);
      mma_ts_pair(tmem, tmem + a_col + 8 * s, bd, id, s > 0);
    }
    mma_commit_pair(&done, 3);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  {
    const uint32_t la = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c = 0; c < N; c += 8) {
      float v[8];
      tmem_ld8(la + c, v);
      tmem_wait_ld();
      for (int j = 0; j < 8; ++j) D[row * N + c + j] = v[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 256);
}

// throughput: nmma back-to-back M256 N K16 MMAs, A from TMEM (TS) or smem (SS)
template <int N, bool TS, int NACC = 1>
__global__ void __cluster_dims__(2, 1, 1) kbench(int nmma, unsigned long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&done, 1); fence_mbar_init(); }
  fence_proxy_async_smem();
  cluster_sync_all();
  if (threadIdx.x < 32) tmem_alloc_pair(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  cluster_sync_all();
  if (cluster_ctarank() == 0 && threadIdx.x == 0) {
    const uint32_t id = make_idesc_f16(256, N);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    unsigned long long t0 = clock64();
    for (int q = 0; q < nmma; ++q) {
      const uint64_t bd = make_sdesc(b + (q & 7) * 2048, 16 * (N / 2), 128);
      const uint32_t d = tmem + (uint32_t)((q % NACC) * N);   // NACC independent accumulators
      if (TS) mma_ts_pair(d, tmem + 256 + 8 * (q & 15), bd, id, q >= NACC);
      else mma_f16_pair(d, make_sdesc(a + (q & 7) * 4096, 2048, 128), bd, id, q >= NACC);
    }
    mma_commit_pair(&done, 3);
    mbar_wait(&done, 0);
    out[0] = clock64() - t0;
  } else {
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (threadIdx.x < 32) tmem_dealloc_pair(tmem, 512);
}

template <int N, int KS>
static int check() {
  const int K = KS * 16;
  std::vector<__half> hA(256 * K), hB(N * K);
  std::vector<float> fA(256 * K), fB(N * K), hD(256 * N);
  srand(1234 + N + KS);
  for (int i = 0; i < 256 * K; ++i) { fA[i] = (float)((rand() % 17) - 8) / 8.f; hA[i] = __float2half(fA[i]); }
  for (int i = 0; i < N * K; ++i) { fB[i] = (float)((rand() % 13) - 6) / 4.f; hB[i] = __float2half(fB[i]); }
  __half *dA, *dB; float *dD;
  cudaMalloc(&dA, hA.size() * 2); cudaMalloc(&dB, hB.size() * 2); cudaMalloc(&dD, hD.size() * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, hD.size() * 4);
  kcheck<N, KS><<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)fA[m * K + k] * fB[n * K + k];
      const double err = fabs(r - hD[m * N + n]);
      maxerr = fmax(maxerr, err);
      if (err > 1e-3) ++bad;
    }
  printf("TS check N=%d K=%d: %s, mismatches %d, max |err| %.3g (D[0][0]=%g D[255][N-1]=%g)\n", N, K,
         cudaGetErrorString(e), bad, maxerr, hD[0], hD[256 * N - 1]);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

template <int N, bool TS, int NACC = 1>
static double bench() {
  unsigned long long *d, h = 0;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(kbench<N, TS, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  const int n = 4096;
  for (int rep = 0; rep < 2; ++rep) kbench<N, TS, NACC><<<2, 128, 65536>>>(n, d);
  cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return h / (double)n;
}

int main() {
  int bad = check<32, 1>() + check<32, 8>() + check<128, 2>();
  printf("cycles per M256 K16 MMA: N=128 SS %.1f TS %.1f | N=32 SS %.1f TS %.1f\n", bench<128, false>(),
         bench<128, true>(), bench<32, false>(), bench<32, true>());
  printf("independent accumulators (TS): N=32 x2 %.1f x4 %.1f x8 %.1f | N=64 x1 %.1f x2 %.1f | N=16 x1 %.1f x4 %.1f | N=256 x1 %.1f\n",
         bench<32, true, 2>(), bench<32, true, 4>(), bench<32, true, 8>(), bench<64, true, 1>(),
         bench<64, true, 2>(), bench<16, true, 1>(), bench<16, true, 4>(), bench<256, true, 1>());
  printf("independent accumulators (SS): N=32 x4 %.1f | N=128 x2 %.1f\n", bench<32, false, 4>(),
         bench<128, false, 2>());
  printf("%s\n", bad ? "TS LAYOUT MISMATCH" : "TS layout ok");
  return bad != 0;
}
