// ring.cu -- K6: streaming mirror ring (a-10).
// Each instance keeps 2W samples; sample of tick k goes to slots (k mod W) and
// (k mod W) + W, so the W samples ending at tick k are always contiguous:
// ring + ((k+1) mod W) * M.  One thread per 16 bytes of the new sample.
#include "common.cuh"

namespace enova {

__global__ void k_ring_push(float *__restrict__ ring, int64_t n, int W, int M,
                            const float *__restrict__ sample, int64_t tick) {
  const int G = M / 4;
  const int64_t total = n * G;
  const int slot = (int)(tick % W);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / G;
    const int g = (int)(e - i * G);
    const float4 v = __ldg(reinterpret_cast<const float4 *>(sample + i * M) + g);
    float4 *r = reinterpret_cast<float4 *>(ring + i * (int64_t)(2 * W) * M);
    r[(int64_t)slot * G + g] = v;
    r[(int64_t)(slot + W) * G + g] = v;
  }
}

enova_status ring_push(float *ring, int64_t n, int W, int M, const float *sample, int64_t tick,
                       cudaStream_t st) {
  if (n == 0) return ENOVA_OK;
  int64_t total = n * (M / 4);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ENOVA_LAUNCH(k_ring_push, blocks, 256, 0, st, ring, n, W, M, sample, tick);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

}  // namespace enova
