// stats.cu -- K1: per-(instance, metric) normalisation statistics (a-1).
//
// "The input metrics are normalized prior to being fed into the VAE"
// (PAPER.md:282); per-dimension z-score with stats from the training horizon
// reused at inference, std floored at 1e-6 (R-4).
//
// One HBM pass: the calibration horizon of each instance is split into
// `nchunk` contiguous time chunks, one CTA each, streamed with coalesced
// 128-bit loads (4 in flight per thread, ragged tail predicated; 2 CTAs per SM).  Each thread accumulates the SHIFTED
// sums S1 = sum(x - K), S2 = sum((x - K)^2) in fp64, with K = the series' first
// sample (the same shift in every chunk, so chunk sums simply add); the CTA
// reduces them in a fixed order and the last CTA of the instance (ticket)
// combines the chunks in chunk order: mean = K + S1/n, var = S2/n - (S1/n)^2.
// With fp32 data and K inside the series' range this equals the two-pass fp64
// result to ~1e-16 relative, far below the fp32 rounding that follows.
#include "common.cuh"

namespace enova {

constexpr int kStatsThreads = 512;
constexpr int kStatsMaxChunks = 16;

// workspace: [0, 256) diag counters | tickets u32[N] | partial sums f64[N][nchunk][2][M]
static inline int stats_max_chunks(int64_t n) {
  if (n <= 0) return 1;
  int64_t c = (1024 + n - 1) / n;
  return (int)(c < 1 ? 1 : c > kStatsMaxChunks ? kStatsMaxChunks : c);
}

size_t stats_workspace_bytes(int64_t n, int m) {
  if (n < 0) n = 0;
  return 256 + align_up((size_t)n * 4, 256) +
         align_up((size_t)n * stats_max_chunks(n) * 2 * m * sizeof(double), 256);
}

template <bool kPow2Group>
__global__ void __launch_bounds__(kStatsThreads, 2) k_series_stats(
    const float *__restrict__ X, int64_t ld, int M, int64_t T_cal, int nchunk,
    float *__restrict__ mean_out, float *__restrict__ std_out, unsigned long long *diag,
    unsigned int *ticket, double *part) {
  extern __shared__ double red[];  // [nwarps or nslots][2][M]
  __shared__ bool last;
  const int G = M / 4;
  const int g = threadIdx.x % G;
  const int slot = threadIdx.x / G;
  const int nslots = blockDim.x / G;
  const int64_t inst = blockIdx.x / nchunk;
  const int chunk = blockIdx.x % nchunk;
  const float4 *base = reinterpret_cast<const float4 *>(X + inst * ld);
  const int64_t t0 = T_cal * chunk / nchunk, t1 = T_cal * (chunk + 1) / nchunk;
  const float4 K = __ldg(base + g);   // shift: the series' first sample

  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, q0 = 0, q1 = 0, q2 = 0, q3 = 0;
  int bad = 0;
  auto acc = [&](const float4 v) {
    bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
    const double d0 = (double)v.x - K.x, d1 = (double)v.y - K.y, d2 = (double)v.z - K.z,
                 d3 = (double)v.w - K.w;
    a0 += d0; a1 += d1; a2 += d2; a3 += d3;
    q0 = fma(d0, d0, q0); q1 = fma(d1, d1, q1); q2 = fma(d2, d2, q2); q3 = fma(d3, d3, q3);
  };
  for (int64_t t = t0 + slot; t < t1; t += 4 * nslots) {   // 4 x 128-bit loads in flight
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u * nslots < t1) v[u] = __ldg(base + (t + u * nslots) * G + g);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t + u * nslots < t1) acc(v[u]);
  }
  double v8[8] = {a0, a1, a2, a3, q0, q1, q2, q3};
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int nred;   // partial sums per output left in red[] (summed below in index order)
  if (kPow2Group) {
    // G a power of two <= 32 (M in {8, ..., 128}), full warps: fixed-order
    // shuffle tree over the slots of a warp (lanes with the same g), then one
    // row of red[] per warp
    for (int o = G; o < 32; o <<= 1)
#pragma unroll
      for (int k = 0; k < 8; ++k) v8[k] += __shfl_xor_sync(0xffffffffu, v8[k], o);
    if (lane < G) {
      double *r = red + (size_t)warp * 2 * M;
      r[4 * g + 0] = v8[0]; r[4 * g + 1] = v8[1]; r[4 * g + 2] = v8[2]; r[4 * g + 3] = v8[3];
      r[M + 4 * g + 0] = v8[4]; r[M + 4 * g + 1] = v8[5]; r[M + 4 * g + 2] = v8[6]; r[M + 4 * g + 3] = v8[7];
    }
    nred = blockDim.x >> 5;
  } else {
    // any G (M a multiple of 4 up to 256, partial last warp allowed): one row
    // of red[] per slot, then a fixed-order pairwise tree over the slots in
    // shared memory (row s += row s + half), so the result does not depend on
    // warp boundaries
    double *r = red + (size_t)slot * 2 * M;
    r[4 * g + 0] = v8[0]; r[4 * g + 1] = v8[1]; r[4 * g + 2] = v8[2]; r[4 * g + 3] = v8[3];
    r[M + 4 * g + 0] = v8[4]; r[M + 4 * g + 1] = v8[5]; r[M + 4 * g + 2] = v8[6]; r[M + 4 * g + 3] = v8[7];
    int rows = nslots;
    while (rows > 1) {
      const int half = (rows + 1) >> 1;
      __syncthreads();
      for (int e = threadIdx.x; e < (rows - half) * 2 * M; e += blockDim.x)
        red[e] += red[(size_t)half * 2 * M + e];
      rows = half;
    }
    nred = 1;
  }
  bad = __syncthreads_or(bad);
  double *pc = part + ((size_t)inst * nchunk + chunk) * 2 * M;
  for (int e = threadIdx.x; e < 2 * M; e += blockDim.x) {   // fixed-order sum over rows
    double s = 0;
    for (int k = 0; k < nred; ++k) s += red[(size_t)k * 2 * M + e];
    pc[e] = s;
  }
  if (threadIdx.x == 0 && bad) atomicAdd(diag + 1, 1ull);   // chunks with a non-finite sample
  // last CTA of this instance combines the chunks in chunk order
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket + inst, 1u) == (unsigned)nchunk - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    const double *p0 = part + (size_t)inst * nchunk * 2 * M;
    double s1 = 0, s2 = 0;
    for (int c = 0; c < nchunk; ++c) {
      s1 += *(volatile const double *)(p0 + (size_t)c * 2 * M + j);
      s2 += *(volatile const double *)(p0 + (size_t)c * 2 * M + M + j);
    }
    const double n = (double)T_cal;
    const double kj = (double)__ldg(X + inst * ld + j);
    const double m1 = s1 / n;
    double var = s2 / n - m1 * m1;
    if (var < 0) var = 0;
    double sd = sqrt(var);
    if (sd < 1e-6) {
      atomicAdd(diag + 0, 1ull);
      sd = 1e-6;
    }
    mean_out[inst * M + j] = (float)(kj + m1);
    std_out[inst * M + j] = (float)sd;
  }
}

// diag[0] = series whose std was floored, diag[1] = (instance, chunk) blocks
// holding a non-finite sample (> 0 <=> ENOVA_ERR_NONFINITE).
enova_status compute_stats_async(const enova_series *s, int64_t t_cal_end, float *mean,
                                 float *stdv, unsigned long long *diag_dev, void *ws,
                                 size_t ws_bytes, cudaStream_t st) {
  const int64_t N = s->n_instances;
  const int M = s->n_metrics;
  if (ws_bytes < stats_workspace_bytes(N, M)) {
    set_error("stats workspace too small (size it with enova_stats_workspace_bytes)");
    return ENOVA_ERR_WORKSPACE;
  }
  char *b = static_cast<char *>(ws);
  unsigned long long *diag = diag_dev ? diag_dev : reinterpret_cast<unsigned long long *>(b);
  unsigned int *ticket = reinterpret_cast<unsigned int *>(b + 256);
  double *part = reinterpret_cast<double *>(b + 256 + align_up((size_t)N * 4, 256));
  int dev = 0, sms = 148;
  ENOVA_CUDA_TRY(cudaGetDevice(&dev));
  ENOVA_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // chunks per instance: the smallest count (>= one wave of 2 CTAs per SM) whose
  // last wave is at least 85% full, so no SM idles through a ragged tail wave
  const int64_t slots = 2 * (int64_t)sms;
  int64_t nchunk = (slots + N - 1) / N;
  for (int64_t c = nchunk; c <= stats_max_chunks(N); ++c) {
    const int64_t rem = (N * c) % slots;
    if (rem == 0 || rem >= (slots * 85) / 100) {
      nchunk = c;
      break;
    }
  }
  if (nchunk > stats_max_chunks(N)) nchunk = stats_max_chunks(N);
  if (nchunk > t_cal_end / 64) nchunk = t_cal_end / 64;
  if (nchunk < 1) nchunk = 1;
  const int G = M / 4;
  const int nthreads = G * (kStatsThreads / G);
  const int nslots = nthreads / G;
  if (diag_dev) ENOVA_CUDA_TRY(cudaMemsetAsync(diag_dev, 0, 2 * sizeof(unsigned long long), st));
  ENOVA_CUDA_TRY(cudaMemsetAsync(b, 0, 256 + (size_t)N * 4, st));   // diag (own) + tickets
  const bool pow2 = (G & (G - 1)) == 0 && G <= 32;
  const size_t smem = (size_t)(pow2 ? nthreads / 32 : nslots) * 2 * M * sizeof(double);
  auto kern = pow2 ? k_series_stats<true> : k_series_stats<false>;
  if (smem > 48 * 1024)
    ENOVA_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  ENOVA_LAUNCH(kern, (unsigned)(N * nchunk), nthreads, smem, st, s->metrics,
               s->ld_instance, M, t_cal_end, (int)nchunk, mean, stdv, diag, ticket, part);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

enova_status compute_stats(const enova_series *s, int64_t t_cal_end, float *mean, float *stdv,
                           int64_t *n_degenerate, void *ws, size_t ws_bytes, cudaStream_t st) {
  enova_status r = compute_stats_async(s, t_cal_end, mean, stdv, nullptr, ws, ws_bytes, st);
  if (r) return r;
  unsigned long long h[2];
  ENOVA_CUDA_TRY(cudaMemcpyAsync(h, ws, sizeof(h), cudaMemcpyDeviceToHost, st));
  ENOVA_CUDA_TRY(cudaStreamSynchronize(st));
  if (n_degenerate) *n_degenerate = (int64_t)h[0];
  if (h[1]) {
    set_error("non-finite metric value in the calibration horizon");
    return ENOVA_ERR_NONFINITE;
  }
  return ENOVA_OK;
}

}  // namespace enova
