// flags.cu -- a-6 for windows that were scored before the threshold existed.
//
// "if the KL-divergence exceeds this threshold, ... the Mean Difference (MD)
// ... determines whether to scale up or down" (
// DESIGN.md R-9, R-10): flag = 0 if score <= z_q, else +1 if MD >= 0, else -1.
// The calibration windows of a step are scored (with MD) BEFORE the POT fit
// that needs their scores; once the fit has written the device threshold this
// kernel applies the same rule to them, so every window of the step ends with
// a score, an MD and a flag.  The comparison is the score kernels' own:
// (double)score > z_q, MD >= 0.f.  Pure HBM streaming: 8 B read + 1 B written
// per window, 16 windows per thread with 128-bit loads.
#include "common.cuh"

namespace enova {

__global__ void __launch_bounds__(256) k_apply_flags(const float *__restrict__ scores,
                                                     const float *__restrict__ md, int64_t n,
                                                     const double *__restrict__ z_q_dev,
                                                     int8_t *__restrict__ flags) {
  const double zq = __ldg(z_q_dev);
  const int64_t i0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 16;
  if (i0 >= n) return;
  if (i0 + 16 <= n && ((reinterpret_cast<uintptr_t>(scores) | reinterpret_cast<uintptr_t>(md) |
                        reinterpret_cast<uintptr_t>(flags)) & 15) == 0) {
    float s[16], m[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 a = __ldg(reinterpret_cast<const float4 *>(scores + i0) + k);
      const float4 b = __ldg(reinterpret_cast<const float4 *>(md + i0) + k);
      s[4 * k] = a.x; s[4 * k + 1] = a.y; s[4 * k + 2] = a.z; s[4 * k + 3] = a.w;
      m[4 * k] = b.x; m[4 * k + 1] = b.y; m[4 * k + 2] = b.z; m[4 * k + 3] = b.w;
    }
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = 4 * k + u;
        const int8_t f = ((double)s[e] > zq) ? (m[e] >= 0.f ? 1 : -1) : 0;
        v |= (uint32_t)(uint8_t)f << (8 * u);
      }
      w[k] = v;
    }
    *reinterpret_cast<uint4 *>(flags + i0) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    for (int64_t i = i0; i < n && i < i0 + 16; ++i)
      flags[i] = ((double)scores[i] > zq) ? (md[i] >= 0.f ? 1 : -1) : 0;
  }
}

enova_status apply_flags(const float *scores, const float *md, int64_t n,
                         const enova_threshold *thr_dev, int8_t *flags, cudaStream_t st) {
  if (n == 0) return ENOVA_OK;
  const int64_t threads = (n + 15) / 16;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  ENOVA_LAUNCH(k_apply_flags, grid, 256, 0, st, scores, md, n, &thr_dev->z_q, flags);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

}  // namespace enova
