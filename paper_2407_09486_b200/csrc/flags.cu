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

// two segments (e.g. the calibration and the detection windows of a step) in one
// launch: blocks [0, nb1) flag segment 1, the rest segment 2
__global__ void __launch_bounds__(256) k_apply_flags2(const float *__restrict__ s1,
                                                      const float *__restrict__ m1, int64_t n1,
                                                      int8_t *__restrict__ f1, unsigned nb1,
                                                      const float *__restrict__ s2,
                                                      const float *__restrict__ m2, int64_t n2,
                                                      int8_t *__restrict__ f2,
                                                      const double *__restrict__ z_q_dev) {
  const double zq = __ldg(z_q_dev);
  const bool first = blockIdx.x < nb1;
  const float *s = first ? s1 : s2;
  const float *m = first ? m1 : m2;
  int8_t *f = first ? f1 : f2;
  const int64_t n = first ? n1 : n2;
  const int64_t i0 = ((int64_t)(first ? blockIdx.x : blockIdx.x - nb1) * blockDim.x + threadIdx.x) * 16;
  if (i0 >= n) return;
  if (i0 + 16 <= n && ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(m) |
                        reinterpret_cast<uintptr_t>(f)) & 15) == 0) {
    float a[16], b[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 x = __ldg(reinterpret_cast<const float4 *>(s + i0) + k);
      const float4 y = __ldg(reinterpret_cast<const float4 *>(m + i0) + k);
      a[4 * k] = x.x; a[4 * k + 1] = x.y; a[4 * k + 2] = x.z; a[4 * k + 3] = x.w;
      b[4 * k] = y.x; b[4 * k + 1] = y.y; b[4 * k + 2] = y.z; b[4 * k + 3] = y.w;
    }
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t v = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = 4 * k + u;
        const int8_t fl = ((double)a[e] > zq) ? (b[e] >= 0.f ? 1 : -1) : 0;
        v |= (uint32_t)(uint8_t)fl << (8 * u);
      }
      w[k] = v;
    }
    *reinterpret_cast<uint4 *>(f + i0) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
    for (int64_t i = i0; i < n && i < i0 + 16; ++i)
      f[i] = ((double)s[i] > zq) ? (m[i] >= 0.f ? 1 : -1) : 0;
  }
}

enova_status apply_flags2(const float *s1, const float *m1, int64_t n1, int8_t *f1,
                          const float *s2, const float *m2, int64_t n2, int8_t *f2,
                          const enova_threshold *thr_dev, cudaStream_t st) {
  const unsigned nb1 = (unsigned)(((n1 + 15) / 16 + 255) / 256);
  const unsigned nb2 = (unsigned)(((n2 + 15) / 16 + 255) / 256);
  if (nb1 + nb2 == 0) return ENOVA_OK;
  ENOVA_LAUNCH(k_apply_flags2, nb1 + nb2, 256, 0, st, s1, m1, n1, f1, nb1, s2, m2, n2, f2,
               &thr_dev->z_q);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
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
