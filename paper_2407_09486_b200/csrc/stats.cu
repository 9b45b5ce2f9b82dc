// stats.cu -- K1: per-(instance, metric) normalisation statistics (a-1).
//
// "The input metrics are normalized prior to being fed into the VAE"
// (PAPER.md:282); per-dimension z-score with stats from the training horizon
// reused at inference, std floored at 1e-6 (R-4).
// One CTA per instance streams its [T_cal][M] block with coalesced 128-bit
// loads, twice (mean, then centred second moment), accumulating in fp64 with
// a fixed reduction order; results are rounded to fp32.
#include "common.cuh"

namespace enova {

__global__ void __launch_bounds__(1024) k_series_stats(const float *__restrict__ X, int64_t ld, int M, int64_t T_cal,
                               float *__restrict__ mean_out, float *__restrict__ std_out,
                               unsigned long long *__restrict__ counters) {
  extern __shared__ double red[];  // [nslots][M]
  __shared__ double mean_s[256];
  const int G = M / 4;
  const int g = threadIdx.x % G;
  const int slot = threadIdx.x / G;
  const int nslots = blockDim.x / G;
  const int64_t inst = blockIdx.x;
  const float4 *base = reinterpret_cast<const float4 *>(X + inst * ld);

  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  int bad = 0;
  int64_t t = slot;
  for (; t + 3 * nslots < T_cal; t += 4 * nslots) {   // 4 independent 128-bit loads in flight
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(base + (t + u * nslots) * G + g);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= !(isfinite(v[u].x) && isfinite(v[u].y) && isfinite(v[u].z) && isfinite(v[u].w));
      s0 += v[u].x; s1 += v[u].y; s2 += v[u].z; s3 += v[u].w;
    }
  }
  for (; t < T_cal; t += nslots) {
    float4 v = __ldg(base + t * G + g);
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    s0 += v.x; s1 += v.y; s2 += v.z; s3 += v.w;
  }
  red[slot * M + 4 * g + 0] = s0;
  red[slot * M + 4 * g + 1] = s1;
  red[slot * M + 4 * g + 2] = s2;
  red[slot * M + 4 * g + 3] = s3;
  bad = __syncthreads_or(bad);
  if (threadIdx.x < M) {
    double s = 0;
    for (int k = 0; k < nslots; ++k) s += red[k * M + threadIdx.x];
    mean_s[threadIdx.x] = s / (double)T_cal;
  }
  __syncthreads();
  const double m0 = mean_s[4 * g], m1 = mean_s[4 * g + 1], m2 = mean_s[4 * g + 2],
               m3 = mean_s[4 * g + 3];
  s0 = s1 = s2 = s3 = 0;
  for (t = slot; t + 3 * nslots < T_cal; t += 4 * nslots) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(base + (t + u * nslots) * G + g);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double d0 = v[u].x - m0, d1 = v[u].y - m1, d2 = v[u].z - m2, d3 = v[u].w - m3;
      s0 += d0 * d0; s1 += d1 * d1; s2 += d2 * d2; s3 += d3 * d3;
    }
  }
  for (; t < T_cal; t += nslots) {
    float4 v = __ldg(base + t * G + g);
    double d0 = v.x - m0, d1 = v.y - m1, d2 = v.z - m2, d3 = v.w - m3;
    s0 += d0 * d0; s1 += d1 * d1; s2 += d2 * d2; s3 += d3 * d3;
  }
  __syncthreads();
  red[slot * M + 4 * g + 0] = s0;
  red[slot * M + 4 * g + 1] = s1;
  red[slot * M + 4 * g + 2] = s2;
  red[slot * M + 4 * g + 3] = s3;
  __syncthreads();
  if (threadIdx.x < M) {
    double s = 0;
    for (int k = 0; k < nslots; ++k) s += red[k * M + threadIdx.x];
    double sd = sqrt(s / (double)T_cal);
    if (sd < 1e-6) {
      atomicAdd(counters + 0, 1ull);
      sd = 1e-6;
    }
    mean_out[inst * M + threadIdx.x] = (float)mean_s[threadIdx.x];
    std_out[inst * M + threadIdx.x] = (float)sd;
  }
  if (threadIdx.x == 0 && bad) atomicAdd(counters + 1, 1ull);
}

enova_status compute_stats(const enova_series *s, int64_t t_cal_end, float *mean, float *stdv,
                           int64_t *n_degenerate, void *ws, cudaStream_t st) {
  const int M = s->n_metrics;
  const int G = M / 4;
  const int nthreads = G * (1024 / G);
  const int nslots = nthreads / G;
  unsigned long long *counters = static_cast<unsigned long long *>(ws);
  ENOVA_CUDA_TRY(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st));
  size_t smem = (size_t)nslots * M * sizeof(double);
  k_series_stats<<<(unsigned)s->n_instances, nthreads, smem, st>>>(
      s->metrics, s->ld_instance, M, t_cal_end, mean, stdv, counters);
  ENOVA_CUDA_TRY(cudaGetLastError());
  unsigned long long h[2];
  ENOVA_CUDA_TRY(cudaMemcpyAsync(h, counters, sizeof(h), cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
  if (n_degenerate) *n_degenerate = (int64_t)h[0];
  if (h[1]) {
    set_error("non-finite metric value in the calibration horizon");
    return ENOVA_ERR_NONFINITE;
  }
  return ENOVA_OK;
}

}  // namespace enova
