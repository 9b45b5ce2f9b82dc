// train.cu -- NEXT-3: semi-supervised training of the detector (Eq. 9).
//
// "ENOVA optimizes the evidence of variational lower bound (ELBO)
//   L_vae = 1/|D| sum_i l_i E_q log p(m|z) - (1 + l_i)/2 beta(k) KL(q(z|m_i) || p(z))
// ... l_i = 1 indicates that m_i is normal ... beta(k) from PI control"
// (R-24, R-25).
//
// One training step over a batch of B windows of a series (window ids g =
// instance * nw + (t - t_begin), id < 0 = padding row):
//   gather   x = fp16_RN(clamp((X - mean) / std, +-1e4)) as fp32 -- exactly the
//            detector input of the score kernels (R-17), one row per window
//   forward  h = tanh(x W1^T + b1); [mu | lv] = h [Wmu; Wlv]^T + b;
//            z = mu + exp(lv / 2) eps (reparameterisation, eps an input);
//            a3 = tanh(z W3^T + b3); m' = a3 W4^T + b4;
//            log p = -1/2 ||x - m'||^2 - D/2 log 2 pi; KL = 1/2 sum(mu^2 + e^lv - 1 - lv)
//   backward the analytic gradient of L (the oracle's order: dm', dW4, da3,
//            dW3, dz, dmu/dlv with the KL and reparameterisation terms, dWheads,
//            dh, dW1; bias gradients as fixed-order column sums)
//   update   Adam ascent on L, then beta(k+1) from the PI controller on the
//            batch's mean KL of normal rows.
// The GEMMs (8 per step) are plain dense products with no fusion opportunity
// worth a custom kernel at these shapes (K = D, H, Z or the batch): they go to
// cuBLAS (fp32 FFMA by default -- parity against the fp64 oracle -- or TF32
// tensor cores on request).  Everything element-wise or row-wise is fused into
// this file's kernels; every reduction is in a fixed order, so a step is
// deterministic.
#include <cublas_v2.h>
#include <math.h>

#include <vector>

#include "common.cuh"

struct enova_trainer_s {
  int W, M, H, Z, D, max_batch, device;
  cublasHandle_t blas;
  // flat parameter / gradient / Adam layout (param_offsets order below)
  float *params, *grads, *adam_m, *adam_v;
  int64_t n_params;
  int64_t off[10];   // w1 b1 wmu bmu wlv blv w3 b3 w4 b4 inside the flat buffers
  // activations [B][.]
  float *x, *h, *heads, *z, *a3, *mp, *da3, *dz, *dheads, *dh;
  double *rowv;      // [B][2]: log p, KL per row
  double *state;     // [0] beta, [1] integral, [2] adam t, [3] n_valid
  double *stats;     // [4] L, beta used, KL normal mean, ELBO normal mean
  void *blas_ws;
};

namespace enova {

constexpr size_t kBlasWs = 4u << 20;

// param_offsets: the caller's view (oracle order); inside, the two head
// matrices Wmu, Wlv are adjacent ([2Z][H] heads image) so one GEMM serves both
enum { P_W1 = 0, P_B1, P_WMU, P_BMU, P_WLV, P_BLV, P_W3, P_B3, P_W4, P_B4 };

static void layout(enova_trainer_s *t) {
  const int64_t D = t->D, H = t->H, Z = t->Z;
  int64_t o = 0;
  auto take = [&](int64_t n) { int64_t r = o; o += (n + 63) / 64 * 64; return r; };
  t->off[P_W1] = take(H * D);
  t->off[P_WMU] = take(2 * Z * H);         // [Wmu ; Wlv] contiguous
  t->off[P_WLV] = t->off[P_WMU] + Z * H;
  t->off[P_W3] = take(H * Z);
  t->off[P_W4] = take(D * H);
  t->off[P_B1] = take(H);
  t->off[P_BMU] = take(2 * Z);             // [bmu ; blv] contiguous
  t->off[P_BLV] = t->off[P_BMU] + Z;
  t->off[P_B3] = take(H);
  t->off[P_B4] = take(D);
  t->n_params = o;
}

// row-major C[m x n] = op(A)[m x k] op(B)[k x n] (+ beta C); lda/ldb/ldc = row
// strides of the stored matrices
static enova_status rm_gemm(cublasHandle_t hb, bool ta, bool tb, int m, int n, int k,
                            const float *A, int lda, const float *B, int ldb, float *C, int ldc,
                            float beta = 0.f) {
  const float one = 1.f;
  cublasStatus_t s = cublasSgemm(hb, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N,
                                 n, m, k, &one, B, ldb, A, lda, &beta, C, ldc);
  if (s != CUBLAS_STATUS_SUCCESS) {
    set_error("cublasSgemm failed (status " + std::to_string((int)s) + ")");
    return ENOVA_ERR_CUDA;
  }
  return ENOVA_OK;
}

// ------------------------------------------------------------- kernels ----
// x rows of the batch: the score kernels' detector input (R-17), zero rows for
// padding ids; state[3] = number of valid rows (fixed-order count, one CTA)
__global__ void k_tr_gather(const float *__restrict__ X, int64_t ld, int64_t t_begin, int64_t nw,
                            int64_t n_win, const float *__restrict__ mean,
                            const float *__restrict__ stdv, int W, int M,
                            const int64_t *__restrict__ ids, int B, float *__restrict__ x) {
  const int D = W * M;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * D) return;
  const int b = (int)(e / D), k = (int)(e - (int64_t)b * D);
  const int64_t g = ids[b];
  float v = 0.f;
  if (g >= 0 && g < n_win) {
    const int64_t inst = g / nw, wi = g - inst * nw;
    const int tau = k / M, j = k - tau * M;
    const int64_t t = t_begin + wi - (W - 1) + tau;
    const float raw = X[inst * ld + t * M + j];
    float zz = __fdiv_rn(__fsub_rn(raw, mean[inst * M + j]), stdv[inst * M + j]);
    zz = fminf(fmaxf(zz, -1e4f), 1e4f);
    v = __half2float(__float2half_rn(zz));
  }
  x[e] = v;
}

__global__ void k_tr_count(const int64_t *__restrict__ ids, int B, int64_t n_win,
                           double *__restrict__ state) {
  __shared__ int cnt[32];
  int c = 0;
  for (int b = threadIdx.x; b < B; b += blockDim.x) c += (ids[b] >= 0 && ids[b] < n_win);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) cnt[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += cnt[w];
    state[3] = (double)s;
  }
}

// y = tanh(y + bias[col]) over [B][C]
__global__ void k_tr_bias_tanh(float *__restrict__ y, const float *__restrict__ bias, int B, int C) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * C) return;
  y[e] = tanhf(y[e] + bias[e % C]);
}

// per row: mu, lv (+ biases, in place in heads [B][2Z]), z = mu + exp(lv/2) eps,
// KL of the row
__global__ void k_tr_latent(float *__restrict__ heads, const float *__restrict__ bheads,
                            const float *__restrict__ eps, int B, int Z, float *__restrict__ z,
                            double *__restrict__ rowv) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  float *hr = heads + (int64_t)b * 2 * Z;
  double kl = 0.0;
  for (int q = 0; q < Z; ++q) {
    const float mu = hr[q] + bheads[q];
    const float lv = hr[Z + q] + bheads[Z + q];
    hr[q] = mu;
    hr[Z + q] = lv;
    z[(int64_t)b * Z + q] = mu + expf(0.5f * lv) * eps[(int64_t)b * Z + q];
    kl += 0.5 * ((double)mu * mu + (double)expm1f(lv) - (double)lv);
  }
  rowv[2 * b + 1] = kl;
}

// per row (one warp): r = x - (m' + b4); log p; dm' = c r with c = l / n_valid
// written over mp
__global__ void k_tr_recon(const float *__restrict__ x, float *__restrict__ mp,
                           const float *__restrict__ b4, const int8_t *__restrict__ labels,
                           const int64_t *__restrict__ ids, int64_t n_win, int B, int D,
                           const double *__restrict__ state, double *__restrict__ rowv) {
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const bool valid = ids[b] >= 0 && ids[b] < n_win;
  const double nv = state[3] > 0 ? state[3] : 1.0;
  const float c = valid ? (float)((double)labels[ids[b]] / nv) : 0.f;
  double ss = 0.0;
  for (int k = lane; k < D; k += 32) {
    const int64_t e = (int64_t)b * D + k;
    const float r = x[e] - (mp[e] + b4[k]);
    ss += (double)r * r;
    mp[e] = c * r;
  }
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) rowv[2 * b] = -0.5 * ss - 0.5 * (double)D * 1.8378770664093453;   // log(2 pi)
}

// d = d * (1 - y^2) over [B][C] (tanh derivative)
__global__ void k_tr_dtanh(float *__restrict__ d, const float *__restrict__ y, int B, int C) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * C) return;
  const float v = y[e];
  d[e] = d[e] * (1.f - v * v);
}

// per row: dmu = dz - k mu; dlv = dz eps exp(lv/2)/2 - k expm1(lv)/2 with
// k = (1 + l)/2 beta / n_valid (0 for padding rows: dz is 0 there too)
__global__ void k_tr_dlatent(const float *__restrict__ dz, const float *__restrict__ heads,
                             const float *__restrict__ eps, const int8_t *__restrict__ labels,
                             const int64_t *__restrict__ ids, int64_t n_win, int B, int Z,
                             const double *__restrict__ state, const double *__restrict__ beta_in,
                             float *__restrict__ dheads) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const bool valid = ids[b] >= 0 && ids[b] < n_win;
  const double nv = state[3] > 0 ? state[3] : 1.0;
  const double beta = *beta_in;
  const float k = valid ? (float)(0.5 * (1.0 + (double)labels[ids[b]]) * beta / nv) : 0.f;
  for (int q = 0; q < Z; ++q) {
    const float mu = heads[(int64_t)b * 2 * Z + q], lv = heads[(int64_t)b * 2 * Z + Z + q];
    const float g = dz[(int64_t)b * Z + q];
    dheads[(int64_t)b * 2 * Z + q] = g - k * mu;
    dheads[(int64_t)b * 2 * Z + Z + q] =
        g * eps[(int64_t)b * Z + q] * 0.5f * expf(0.5f * lv) - k * 0.5f * expm1f(lv);
  }
}

// out[c] = sum_b A[b][c] (fixed order over rows)
__global__ void k_tr_colsum(const float *__restrict__ A, int B, int C, float *__restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  float s = 0.f;
  for (int b = 0; b < B; ++b) s += A[(int64_t)b * C + c];
  out[c] = s;
}

// L, stats of the batch (one CTA, fixed order)
__global__ void k_tr_stats(const double *__restrict__ rowv, const int8_t *__restrict__ labels,
                           const int64_t *__restrict__ ids, int64_t n_win, int B,
                           const double *__restrict__ state, const double *__restrict__ beta_in,
                           double *__restrict__ stats, double *__restrict__ kl_normal_out) {
  if (threadIdx.x != 0) return;
  const double beta = *beta_in;
  double L = 0.0, kln = 0.0, eln = 0.0;
  int nn = 0;
  for (int b = 0; b < B; ++b) {
    if (!(ids[b] >= 0 && ids[b] < n_win)) continue;
    const double l = labels[ids[b]], lp = rowv[2 * b], kl = rowv[2 * b + 1];
    L += l * lp - 0.5 * (1.0 + l) * beta * kl;
    if (l > 0) {
      kln += kl;
      eln += lp - kl;
      ++nn;
    }
  }
  const double nv = state[3] > 0 ? state[3] : 1.0;
  stats[0] = L / nv;
  stats[1] = beta;
  stats[2] = nn ? kln / nn : 0.0;
  stats[3] = nn ? eln / nn : 0.0;
  *kl_normal_out = stats[2];
}

// Adam ascent on the flat parameters; t read from state[2] (incremented by
// k_tr_pi after the step)
__global__ void k_tr_adam(float *__restrict__ p, const float *__restrict__ g,
                          float *__restrict__ m, float *__restrict__ v, int64_t n,
                          const double *__restrict__ state, double lr, double b1, double b2,
                          double eps) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double t = state[2] + 1.0;
  const double c1 = 1.0 - pow(b1, t), c2 = 1.0 - pow(b2, t);
  const double gi = g[i];
  const double mi = b1 * (double)m[i] + (1.0 - b1) * gi;
  const double vi = b2 * (double)v[i] + (1.0 - b2) * gi * gi;
  m[i] = (float)mi;
  v[i] = (float)vi;
  p[i] = (float)((double)p[i] + lr * (mi / c1) / (sqrt(vi / c2) + eps));
}

// beta(k+1) from the PI controller (R-24); Adam step count + 1
__global__ void k_tr_pi(double *__restrict__ state, const double *__restrict__ kl_normal,
                        double setpoint, double kp, double ki, double beta_max, int fixed_mode,
                        double beta_fixed) {
  if (threadIdx.x != 0) return;
  state[2] += 1.0;
  if (fixed_mode) {
    state[0] = beta_fixed;
    return;
  }
  const double e = *kl_normal - setpoint;
  const double I = state[1] + e;
  const double b = kp * e + ki * I;
  if (b >= 0.0 && b <= beta_max) state[1] = I;
  state[0] = fmin(beta_max, fmax(0.0, b));
}

__global__ void k_tr_set(double *p, double v) { *p = v; }

// ---------------------------------------------------------------- host ----
static enova_status forward_backward(enova_trainer_s *t, const enova_series *s,
                                     const int64_t *ids, const int8_t *labels, int B,
                                     const float *eps, const double *beta_dev, cudaStream_t st) {
  const int D = t->D, H = t->H, Z = t->Z, W = t->W, M = t->M;
  const int64_t nw = s->t_end - s->t_begin, n_win = s->n_instances * nw;
  float *P = t->params, *G = t->grads;
  if (cublasSetStream(t->blas, st) != CUBLAS_STATUS_SUCCESS) {
    set_error("cublasSetStream failed");
    return ENOVA_ERR_CUDA;
  }
  auto grid = [](int64_t n, int b) { return (unsigned)((n + b - 1) / b); };
  enova_status r;
  ENOVA_LAUNCH(k_tr_count, 1, 256, 0, st, ids, B, n_win, t->state);
  ENOVA_LAUNCH(k_tr_gather, grid((int64_t)B * D, 256), 256, 0, st, s->metrics, s->ld_instance,
               s->t_begin, nw, n_win, s->norm_mean, s->norm_std, W, M, ids, B, t->x);
  // ---- forward
  if ((r = rm_gemm(t->blas, false, true, B, H, D, t->x, D, P + t->off[P_W1], D, t->h, H))) return r;
  ENOVA_LAUNCH(k_tr_bias_tanh, grid((int64_t)B * H, 256), 256, 0, st, t->h, P + t->off[P_B1], B, H);
  if ((r = rm_gemm(t->blas, false, true, B, 2 * Z, H, t->h, H, P + t->off[P_WMU], H, t->heads,
                   2 * Z)))
    return r;
  ENOVA_LAUNCH(k_tr_latent, grid(B, 128), 128, 0, st, t->heads, P + t->off[P_BMU], eps, B, Z,
               t->z, t->rowv);
  if ((r = rm_gemm(t->blas, false, true, B, H, Z, t->z, Z, P + t->off[P_W3], Z, t->a3, H))) return r;
  ENOVA_LAUNCH(k_tr_bias_tanh, grid((int64_t)B * H, 256), 256, 0, st, t->a3, P + t->off[P_B3], B, H);
  if ((r = rm_gemm(t->blas, false, true, B, D, H, t->a3, H, P + t->off[P_W4], H, t->mp, D))) return r;
  ENOVA_LAUNCH(k_tr_recon, grid(B, 8), 256, 0, st, t->x, t->mp, P + t->off[P_B4], labels, ids,
               n_win, B, D, t->state, t->rowv);
  // ---- backward (t->mp now holds dL/dm')
  if ((r = rm_gemm(t->blas, true, false, D, H, B, t->mp, D, t->a3, H, G + t->off[P_W4], H))) return r;
  ENOVA_LAUNCH(k_tr_colsum, grid(D, 128), 128, 0, st, t->mp, B, D, G + t->off[P_B4]);
  if ((r = rm_gemm(t->blas, false, false, B, H, D, t->mp, D, P + t->off[P_W4], H, t->da3, H)))
    return r;
  ENOVA_LAUNCH(k_tr_dtanh, grid((int64_t)B * H, 256), 256, 0, st, t->da3, t->a3, B, H);
  if ((r = rm_gemm(t->blas, true, false, H, Z, B, t->da3, H, t->z, Z, G + t->off[P_W3], Z))) return r;
  ENOVA_LAUNCH(k_tr_colsum, grid(H, 128), 128, 0, st, t->da3, B, H, G + t->off[P_B3]);
  if ((r = rm_gemm(t->blas, false, false, B, Z, H, t->da3, H, P + t->off[P_W3], Z, t->dz, Z)))
    return r;
  ENOVA_LAUNCH(k_tr_dlatent, grid(B, 128), 128, 0, st, t->dz, t->heads, eps, labels, ids, n_win,
               B, Z, t->state, beta_dev, t->dheads);
  if ((r = rm_gemm(t->blas, true, false, 2 * Z, H, B, t->dheads, 2 * Z, t->h, H, G + t->off[P_WMU],
                   H)))
    return r;
  ENOVA_LAUNCH(k_tr_colsum, grid(2 * Z, 128), 128, 0, st, t->dheads, B, 2 * Z, G + t->off[P_BMU]);
  if ((r = rm_gemm(t->blas, false, false, B, H, 2 * Z, t->dheads, 2 * Z, P + t->off[P_WMU], H,
                   t->dh, H)))
    return r;
  ENOVA_LAUNCH(k_tr_dtanh, grid((int64_t)B * H, 256), 256, 0, st, t->dh, t->h, B, H);
  if ((r = rm_gemm(t->blas, true, false, H, D, B, t->dh, H, t->x, D, G + t->off[P_W1], D))) return r;
  ENOVA_LAUNCH(k_tr_colsum, grid(H, 128), 128, 0, st, t->dh, B, H, G + t->off[P_B1]);
  ENOVA_LAUNCH(k_tr_stats, 1, 32, 0, st, t->rowv, labels, ids, n_win, B, t->state, beta_dev,
               t->stats, t->state + 4);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

static enova_status check_step_args(enova_trainer_s *t, const enova_series *s, const int64_t *ids,
                                    const int8_t *labels, int B, const float *eps) {
  if (!t || !s || !ids || !labels || !eps || B < 1 || B > t->max_batch) {
    set_error("train step: trainer, series, ids, labels, eps required; 1 <= batch <= max_batch");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (s->n_metrics != t->M || !s->metrics || !s->norm_mean || !s->norm_std ||
      s->t_begin < t->W - 1 || s->t_end < s->t_begin || s->t_end > s->n_steps ||
      s->ld_instance < s->n_steps * (int64_t)s->n_metrics) {
    set_error("train step: series shape, range or statistics invalid for this trainer");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return ENOVA_OK;
}

}  // namespace enova

using namespace enova;

extern "C" {

enova_status enova_trainer_create(enova_trainer_t *out, int32_t window, int32_t n_metrics,
                                  int32_t hidden, int32_t latent, int32_t max_batch, int device) {
  if (!out || window < 1 || n_metrics < 1 || hidden < 1 || latent < 1 || max_batch < 1) {
    set_error("enova_trainer_create: positive sizes required");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  ENOVA_CUDA_TRY(cudaSetDevice(device));
  enova_trainer_s *t = new enova_trainer_s();
  t->W = window;
  t->M = n_metrics;
  t->H = hidden;
  t->Z = latent;
  t->D = window * n_metrics;
  t->max_batch = max_batch;
  t->device = device;
  layout(t);
  const int64_t B = max_batch, D = t->D, H = hidden, Z = latent;
  std::vector<void **> bufs;
  std::vector<size_t> sizes;
  auto add = [&](void **p, size_t bytes) { bufs.push_back(p); sizes.push_back(bytes); };
  add((void **)&t->params, t->n_params * 4);
  add((void **)&t->grads, t->n_params * 4);
  add((void **)&t->adam_m, t->n_params * 4);
  add((void **)&t->adam_v, t->n_params * 4);
  add((void **)&t->x, B * D * 4);
  add((void **)&t->h, B * H * 4);
  add((void **)&t->heads, B * 2 * Z * 4);
  add((void **)&t->z, B * Z * 4);
  add((void **)&t->a3, B * H * 4);
  add((void **)&t->mp, B * D * 4);
  add((void **)&t->da3, B * H * 4);
  add((void **)&t->dz, B * Z * 4);
  add((void **)&t->dheads, B * 2 * Z * 4);
  add((void **)&t->dh, B * H * 4);
  add((void **)&t->rowv, B * 2 * 8);
  add((void **)&t->state, 8 * 8);
  add((void **)&t->stats, 4 * 8);
  add(&t->blas_ws, kBlasWs);
  for (size_t i = 0; i < bufs.size(); ++i) {
    cudaError_t e = cudaMalloc(bufs[i], sizes[i] ? sizes[i] : 8);
    if (e != cudaSuccess) {
      for (size_t j = 0; j < i; ++j) cudaFree(*bufs[j]);
      delete t;
      return cuda_status(e, "cudaMalloc (trainer)");
    }
  }
  cudaMemset(t->grads, 0, t->n_params * 4);
  cudaMemset(t->state, 0, 8 * 8);
  cudaMemset(t->stats, 0, 4 * 8);
  if (cublasCreate(&t->blas) != CUBLAS_STATUS_SUCCESS ||
      cublasSetWorkspace(t->blas, t->blas_ws, kBlasWs) != CUBLAS_STATUS_SUCCESS ||
      cublasSetMathMode(t->blas, CUBLAS_PEDANTIC_MATH) != CUBLAS_STATUS_SUCCESS) {
    for (auto p : bufs) cudaFree(*p);
    delete t;
    set_error("cuBLAS initialisation failed");
    return ENOVA_ERR_CUDA;
  }
  *out = t;
  return ENOVA_OK;
}

void enova_trainer_destroy(enova_trainer_t t) {
  if (!t) return;
  cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  cublasDestroy(t->blas);
  void *ps[] = {t->params, t->grads, t->adam_m, t->adam_v, t->x, t->h, t->heads, t->z, t->a3,
                t->mp, t->da3, t->dz, t->dheads, t->dh, t->rowv, t->state, t->stats, t->blas_ws};
  for (void *p : ps) cudaFree(p);
  delete t;
}

int64_t enova_trainer_param_offsets(enova_trainer_t t, int64_t *offsets10) {
  if (!t) return 0;
  if (offsets10)
    for (int i = 0; i < 10; ++i) offsets10[i] = t->off[i];
  return t->n_params;
}

enova_status enova_trainer_set_math(enova_trainer_t t, int32_t math) {
  if (!t || (math != 0 && math != 1)) {
    set_error("enova_trainer_set_math: 0 (fp32) or 1 (TF32 tensor cores)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cublasStatus_t s = cublasSetMathMode(t->blas, math ? CUBLAS_TF32_TENSOR_OP_MATH
                                                     : CUBLAS_PEDANTIC_MATH);
  if (s != CUBLAS_STATUS_SUCCESS) {
    set_error("cublasSetMathMode failed");
    return ENOVA_ERR_CUDA;
  }
  return ENOVA_OK;
}

// params <- the caller's detector (device fp32, include/enova.h layouts); Adam
// moments, step count and the PI state are reset (beta(0) = beta0)
enova_status enova_trainer_load(enova_trainer_t t, const enova_detector *det, double beta0,
                                void *stream) {
  if (!t || !det || det->window != t->W || det->n_metrics != t->M || det->hidden != t->H ||
      det->latent != t->Z) {
    set_error("enova_trainer_load: detector shape does not match the trainer");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t D = t->D, H = t->H, Z = t->Z;
  const float *src[10] = {det->enc_w1, det->enc_b1, det->enc_wmu, det->enc_bmu, det->enc_wlv,
                          det->enc_blv, det->dec_w1, det->dec_b1, det->dec_w2, det->dec_b2};
  const int64_t n[10] = {H * D, H, Z * H, Z, Z * H, Z, H * Z, H, D * H, D};
  for (int i = 0; i < 10; ++i) {
    if (!src[i]) {
      set_error("enova_trainer_load: NULL detector tensor");
      return ENOVA_ERR_INVALID_ARGUMENT;
    }
    ENOVA_CUDA_TRY(cudaMemcpyAsync(t->params + t->off[i], src[i], n[i] * 4,
                                   cudaMemcpyDeviceToDevice, st));
  }
  ENOVA_CUDA_TRY(cudaMemsetAsync(t->adam_m, 0, t->n_params * 4, st));
  ENOVA_CUDA_TRY(cudaMemsetAsync(t->adam_v, 0, t->n_params * 4, st));
  ENOVA_CUDA_TRY(cudaMemsetAsync(t->state, 0, 8 * 8, st));
  ENOVA_LAUNCH(k_tr_set, 1, 1, 0, st, t->state, beta0);
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

// the trained parameters -> the caller's detector buffers (device fp32, written)
enova_status enova_trainer_store(enova_trainer_t t, const enova_detector *det, void *stream) {
  if (!t || !det || det->window != t->W || det->n_metrics != t->M || det->hidden != t->H ||
      det->latent != t->Z) {
    set_error("enova_trainer_store: detector shape does not match the trainer");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t D = t->D, H = t->H, Z = t->Z;
  float *dst[10] = {const_cast<float *>(det->enc_w1), const_cast<float *>(det->enc_b1),
                    const_cast<float *>(det->enc_wmu), const_cast<float *>(det->enc_bmu),
                    const_cast<float *>(det->enc_wlv), const_cast<float *>(det->enc_blv),
                    const_cast<float *>(det->dec_w1), const_cast<float *>(det->dec_b1),
                    const_cast<float *>(det->dec_w2), const_cast<float *>(det->dec_b2)};
  const int64_t n[10] = {H * D, H, Z * H, Z, Z * H, Z, H * Z, H, D * H, D};
  for (int i = 0; i < 10; ++i) {
    if (!dst[i]) {
      set_error("enova_trainer_store: NULL detector tensor");
      return ENOVA_ERR_INVALID_ARGUMENT;
    }
    ENOVA_CUDA_TRY(cudaMemcpyAsync(dst[i], t->params + t->off[i], n[i] * 4,
                                   cudaMemcpyDeviceToDevice, st));
  }
  return ENOVA_OK;
}

enova_status enova_train_gradient(enova_trainer_t t, const enova_series *s, const int64_t *ids,
                                  const int8_t *labels, int32_t batch, const float *eps,
                                  double beta, float *grad_out, double *stats_out,
                                  void *stream) {
  enova_status r = check_step_args(t, s, ids, labels, batch, eps);
  if (r) return r;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ENOVA_LAUNCH(k_tr_set, 1, 1, 0, st, t->state + 5, beta);
  if ((r = forward_backward(t, s, ids, labels, batch, eps, t->state + 5, st))) return r;
  if (grad_out)
    ENOVA_CUDA_TRY(cudaMemcpyAsync(grad_out, t->grads, t->n_params * 4, cudaMemcpyDeviceToDevice, st));
  if (stats_out)
    ENOVA_CUDA_TRY(cudaMemcpyAsync(stats_out, t->stats, 4 * 8, cudaMemcpyDeviceToDevice, st));
  return ENOVA_OK;
}

enova_status enova_train_step(enova_trainer_t t, const enova_series *s, const int64_t *ids,
                              const int8_t *labels, int32_t batch, const float *eps,
                              const enova_train_config *cfg, double *stats_out, void *stream) {
  enova_status r = check_step_args(t, s, ids, labels, batch, eps);
  if (r) return r;
  if (!cfg || !(cfg->lr > 0) || !(cfg->beta_max >= 0)) {
    set_error("enova_train_step: config required (lr > 0, beta_max >= 0)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if ((r = forward_backward(t, s, ids, labels, batch, eps, t->state, st))) return r;
  const unsigned nb = (unsigned)((t->n_params + 255) / 256);
  ENOVA_LAUNCH(k_tr_adam, nb, 256, 0, st, t->params, t->grads, t->adam_m, t->adam_v, t->n_params,
               t->state, cfg->lr, cfg->adam_beta1, cfg->adam_beta2, cfg->adam_eps);
  ENOVA_LAUNCH(k_tr_pi, 1, 1, 0, st, t->state, t->state + 4, cfg->kl_setpoint, cfg->kp, cfg->ki,
               cfg->beta_max, cfg->beta_mode, cfg->beta_fixed);
  if (stats_out)
    ENOVA_CUDA_TRY(cudaMemcpyAsync(stats_out, t->stats, 4 * 8, cudaMemcpyDeviceToDevice, st));
  ENOVA_CUDA_TRY(cudaGetLastError());
  return ENOVA_OK;
}

}  // extern "C"
