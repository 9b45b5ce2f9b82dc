// abi.cu -- the C ABI of libenova (include/enova.h): argument validation,
// workspace sizing and launch sequencing.  No allocation on the hot path.
#include <math.h>

#include <atomic>
#include <string>

#include "comm.h"
#include "common.cuh"
#include "layout.h"

namespace enova {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const std::string &msg) { g_last_error = msg; }

enova_status cuda_status(cudaError_t e, const char *what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return ENOVA_ERR_CUDA;
}

enova_status prepare_detector(const enova_detector *det, const DetLayout &L, void *ws,
                              cudaStream_t st);
enova_status compute_stats(const enova_series *s, int64_t t_cal_end, float *mean, float *stdv,
                           int64_t *n_degenerate, void *ws, size_t ws_bytes, cudaStream_t st);
enova_status compute_stats_async(const enova_series *s, int64_t t_cal_end, float *mean,
                                 float *stdv, unsigned long long *diag_dev, void *ws,
                                 size_t ws_bytes, cudaStream_t st);
size_t stats_workspace_bytes(int64_t n, int m);
void set_forced_kernel(int k);
int64_t pot_sampled_offset();
int64_t pot_fit_stamp_offset();
enova_status apply_flags(const float *scores, const float *md, int64_t n,
                         const enova_threshold *thr_dev, int8_t *flags, cudaStream_t st);
enova_status launch_score(const enova_series *s, const DetLayout &L, const void *det_ws,
                          float *scores, float *md, int8_t *flags, double z_q, const double *z_q_dev,
                          cudaStream_t st);
enova_status fit_threshold(const float *scores, int64_t n_local, double q0, double q,
                           enova_comm_t comm, enova_threshold *out, void *ws, size_t ws_bytes,
                           int64_t n_global_max, cudaStream_t st);
enova_status fit_threshold_async(const float *scores, int64_t n, double q0, double q,
                                 enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                 int64_t n_global_max, cudaStream_t st);
size_t threshold_workspace_bytes(int64_t n_max, double q0, int world);
enova_status fit_threshold_dist_async(const float *scores, int64_t n_local, int64_t n, double q0,
                                      double q, enova_comm_t comm, enova_threshold *out_dev,
                                      void *ws, size_t ws_bytes, int64_t n_global_max,
                                      cudaStream_t st);
enova_status fit_threshold_comm_async(const float *scores, int64_t n_local, int64_t n, double q0,
                                      double q, enova_comm_t comm, enova_threshold *out_dev,
                                      void *ws, size_t ws_bytes, int64_t n_global_max,
                                      cudaStream_t st);
void set_pair_trace(void *t);
void pot_stamp_offsets(int64_t *n_off, int64_t *st_off);
enova_status ring_push(float *ring, int64_t n, int W, int M, const float *sample, int64_t tick,
                       cudaStream_t st);
size_t stream_ring_bytes(int64_t n, int W, int M);
enova_status spot_update(const float *scores, const int8_t *flags, int64_t n, void *ws,
                         size_t ws_bytes, int64_t n_global_max, double q0, cudaStream_t st);
enova_status spot_refit(double q, enova_threshold *out_dev, void *ws, size_t ws_bytes,
                        int64_t n_global_max, double q0, cudaStream_t st);
enova_status select_flagged(const int8_t *flags, int64_t n, int64_t *ids, long long *count_dev,
                            void *scratch, cudaStream_t st);
size_t select_flagged_scratch_bytes(int64_t n);
enova_status launch_explain_rows(const enova_series *s, const DetLayout &L, const void *det_ws,
                                 const int64_t *rows_dev, int64_t n_rows, float *md_metric,
                                 float *scores, float *md, cudaStream_t st);
bool rows_path_ok(const DetLayout &L);
enova_status stream_step(void *ring, int64_t n, int64_t tick, const DetLayout &L,
                         const void *det_ws, const float *sample, const float *mean,
                         const float *stdv, const double *z_q_dev, int8_t *flags, float *scores,
                         float *md, cudaStream_t st);
enova_status point_adjust_counts(const int8_t *labels, int64_t ld_labels, const int8_t *flags,
                                 int64_t n_inst, int64_t t_begin, int64_t nw,
                                 unsigned long long *counts_dev, cudaStream_t st);
enova_status stream_push(void *ring, int64_t n, int W, int M, const float *sample,
                         const float *mean, const float *stdv, int64_t tick, cudaStream_t st);
enova_status stream_detect(const void *ring, int64_t n, int64_t tick, const DetLayout &L,
                           const void *det_ws, const double *z_q_dev, int8_t *flags, float *scores,
                           float *md, cudaStream_t st, const float *sample = nullptr,
                           const float *mean = nullptr, const float *stdv = nullptr);

static inline bool aligned(const void *p, size_t a) {
  return (reinterpret_cast<uintptr_t>(p) % a) == 0;
}

static enova_status check_detector(const enova_detector *det, DetLayout *L) {
  if (!det) {
    set_error("detector is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_layout(det->window, det->n_metrics, det->hidden, det->latent, L)) {
    set_error("detector shape outside the fast-path envelope (M in {8, 16, 32, 64}, W even "
              "2..256, H in {32,64,128}, 1<=Z<=16)");
    return ENOVA_ERR_UNSUPPORTED;
  }
  return ENOVA_OK;
}

static enova_status check_det_ptrs(const enova_detector *d) {
  if (!d->enc_w1 || !d->enc_b1 || !d->enc_wmu || !d->enc_bmu || !d->enc_wlv || !d->enc_blv ||
      !d->dec_w1 || !d->dec_b1 || !d->dec_w2 || !d->dec_b2) {
    set_error("detector weight pointer is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return ENOVA_OK;
}

static enova_status check_series_base(const enova_series *s) {
  if (!s || !s->metrics) {
    set_error("series or series->metrics is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (s->n_instances < 0 || s->n_steps < 0 || s->n_metrics <= 0 || (s->n_metrics % 8) != 0) {
    set_error("bad series sizes (n_metrics must be a positive multiple of 8)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (s->ld_instance < s->n_steps * (int64_t)s->n_metrics || (s->ld_instance % 4) != 0) {
    set_error("ld_instance must be >= n_steps*n_metrics and a multiple of 4");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!aligned(s->metrics, 16)) {
    set_error("metrics must be 16-byte aligned");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return ENOVA_OK;
}

static enova_status check_series_windows(const enova_series *s, const DetLayout &L) {
  enova_status r = check_series_base(s);
  if (r) return r;
  if (s->n_metrics != L.M) {
    set_error("series n_metrics != detector n_metrics");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (s->n_steps < L.W) {
    set_error("insufficient history: n_steps < window");
    return ENOVA_ERR_INSUFFICIENT_HISTORY;
  }
  if (s->t_begin < L.W - 1) {
    set_error("insufficient history: t_begin < window - 1");
    return ENOVA_ERR_INSUFFICIENT_HISTORY;
  }
  if (s->t_end < s->t_begin || s->t_end > s->n_steps) {
    set_error("window range must satisfy t_begin <= t_end <= n_steps");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!s->norm_mean || !s->norm_std || !aligned(s->norm_mean, 16) || !aligned(s->norm_std, 16)) {
    set_error("norm_mean / norm_std are required and must be 16-byte aligned");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  return ENOVA_OK;
}

static enova_status sticky() {
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) return cuda_status(e, "pending CUDA error");
  return ENOVA_OK;
}

}  // namespace enova

using namespace enova;

extern "C" {

int enova_abi_version(void) { return ENOVA_ABI_VERSION; }

// diagnostic (not part of enova.h): record a %globaltimer pipeline trace of CTA
// pair 0 of the next CTA-pair score launches into a device buffer of
// 2 x 512 x 16 uint64 (NULL disables)
void enova_internal_set_trace(void *dev_buf) { enova::set_pair_trace(dev_buf); }
// diagnostic (not in enova.h): where k_pot writes its %globaltimer phase stamps
// in the threshold workspace (PotGlobal is at offset 0)
// diagnostic (not in enova.h): byte offset of the int flag "the last selection ran
// on the sampled candidates" in the threshold workspace
int64_t enova_internal_pot_sampled_offset(void) { return enova::pot_sampled_offset(); }
// diagnostic: byte offset of the int "stamp index at the start of the fit"
int64_t enova_internal_pot_fit_stamp_offset(void) { return enova::pot_fit_stamp_offset(); }
void enova_internal_pot_stamp_offsets(int64_t *n_off, int64_t *st_off) {
  enova::pot_stamp_offsets(n_off, st_off);
}

uint64_t enova_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

enova_status enova_flag_scores_async(const float *scores, const float *md, int64_t n,
                                     const enova_threshold *thr_dev, int8_t *flags, void *stream) {
  if (n < 0) {
    enova::set_error("n < 0");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n > 0 && (!scores || !md || !flags)) {
    enova::set_error("scores / md / flags must be non-NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!thr_dev || !enova::aligned(thr_dev, 8)) {
    enova::set_error("device threshold missing or misaligned");
    return ENOVA_ERR_UNCALIBRATED;
  }
  enova_status r = enova::sticky();
  if (r) return r;
  return enova::apply_flags(scores, md, n, thr_dev, flags, static_cast<cudaStream_t>(stream));
}

enova_status enova_set_score_kernel(int which) {
  if (which < 0 || which > 3) {
    enova::set_error("enova_set_score_kernel: which must be 0 (auto), 1 (stream), 2 (pair) or 3 (rows)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova::set_forced_kernel(which);
  return ENOVA_OK;
}

const char *enova_last_error(void) { return g_last_error.c_str(); }

const char *enova_status_string(enova_status s) {
  switch (s) {
    case ENOVA_OK: return "ENOVA_OK";
    case ENOVA_ERR_INVALID_ARGUMENT: return "ENOVA_ERR_INVALID_ARGUMENT";
    case ENOVA_ERR_UNSUPPORTED: return "ENOVA_ERR_UNSUPPORTED";
    case ENOVA_ERR_INSUFFICIENT_HISTORY: return "ENOVA_ERR_INSUFFICIENT_HISTORY";
    case ENOVA_ERR_TOO_FEW_EXCEEDANCES: return "ENOVA_ERR_TOO_FEW_EXCEEDANCES";
    case ENOVA_ERR_NONFINITE: return "ENOVA_ERR_NONFINITE";
    case ENOVA_ERR_UNCALIBRATED: return "ENOVA_ERR_UNCALIBRATED";
    case ENOVA_ERR_CUDA: return "ENOVA_ERR_CUDA";
    case ENOVA_ERR_NCCL: return "ENOVA_ERR_NCCL";
    case ENOVA_ERR_WORKSPACE: return "ENOVA_ERR_WORKSPACE";
  }
  return "ENOVA_ERR_UNKNOWN";
}

size_t enova_detector_workspace_bytes(const enova_detector *det) {
  DetLayout L;
  if (!det || !det_layout(det->window, det->n_metrics, det->hidden, det->latent, &L)) return 0;
  return L.total;
}

enova_status enova_prepare_detector(const enova_detector *det, void *det_ws, size_t det_ws_bytes,
                                    void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if ((r = check_det_ptrs(det))) return r;
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("detector workspace missing, too small or not 256-byte aligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  return prepare_detector(det, L, det_ws, static_cast<cudaStream_t>(stream));
}

size_t enova_stats_workspace_bytes(int64_t n_instances, int32_t n_metrics) {
  if (n_metrics < 1) n_metrics = 1;
  return stats_workspace_bytes(n_instances, n_metrics);
}

static enova_status check_stats_args(const enova_series *series, int64_t t_cal_end,
                                     const float *mean, const float *std, const void *ws,
                                     size_t ws_bytes) {
  enova_status r = check_series_base(series);
  if (r) return r;
  if (series->n_metrics > 256) {
    set_error("n_metrics > 256");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (t_cal_end < 1 || t_cal_end > series->n_steps) {
    set_error("t_cal_end must be in [1, n_steps]");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!mean || !std) {
    set_error("mean / std outputs are NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!ws || !aligned(ws, 256) ||
      ws_bytes < stats_workspace_bytes(series->n_instances, series->n_metrics)) {
    set_error("stats workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  return sticky();
}

enova_status enova_compute_stats(const enova_series *series, int64_t t_cal_end, float *mean,
                                 float *std, int64_t *n_degenerate, void *ws, size_t ws_bytes,
                                 void *stream) {
  enova_status r = check_stats_args(series, t_cal_end, mean, std, ws, ws_bytes);
  if (r) return r;
  if (series->n_instances == 0) {
    if (n_degenerate) *n_degenerate = 0;
    return ENOVA_OK;
  }
  return compute_stats(series, t_cal_end, mean, std, n_degenerate, ws, ws_bytes,
                       static_cast<cudaStream_t>(stream));
}

enova_status enova_compute_stats_async(const enova_series *series, int64_t t_cal_end, float *mean,
                                       float *std, int64_t *diag_dev, void *ws, size_t ws_bytes,
                                       void *stream) {
  enova_status r = check_stats_args(series, t_cal_end, mean, std, ws, ws_bytes);
  if (r) return r;
  if (diag_dev && !aligned(diag_dev, 8)) {
    set_error("diag_dev must be 8-byte aligned");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (series->n_instances == 0) {
    if (diag_dev) ENOVA_CUDA_TRY(cudaMemsetAsync(diag_dev, 0, 16, st));
    return ENOVA_OK;
  }
  return compute_stats_async(series, t_cal_end, mean, std,
                             reinterpret_cast<unsigned long long *>(diag_dev), ws, ws_bytes, st);
}

enova_status enova_score_windows(const enova_series *series, const enova_detector *det,
                                 const void *det_ws, size_t det_ws_bytes, float *scores,
                                 float *md, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if ((r = check_series_windows(series, L))) return r;
  const bool empty = series->n_instances == 0 || series->t_end == series->t_begin;
  if (!scores && !empty) {
    set_error("scores output is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  if (empty) return ENOVA_OK;
  return launch_score(series, L, det_ws, scores, md, nullptr, 0.0, nullptr,
                      static_cast<cudaStream_t>(stream));
}

size_t enova_threshold_workspace_bytes(int64_t n_global_max, double init_quantile) {
  if (n_global_max < 1) n_global_max = 1;
  return threshold_workspace_bytes(n_global_max, init_quantile, 0);
}

size_t enova_threshold_comm_workspace_bytes(int64_t n_global_max, double init_quantile,
                                            int32_t world) {
  if (n_global_max < 1) n_global_max = 1;
  if (world < 1) world = 1;
  return threshold_workspace_bytes(n_global_max, init_quantile, world);
}

enova_status enova_fit_threshold_comm_async(const float *scores, int64_t n_local, int64_t n_global,
                                            int64_t n_global_max, double init_quantile,
                                            double risk_q, enova_comm_t comm,
                                            enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                            void *stream) {
  if (!comm || !out_dev || n_local < 0 || (n_local > 0 && !scores) || n_global < 1 ||
      !aligned(out_dev, 8)) {
    set_error("bad fit_threshold_comm_async arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!(init_quantile >= 0.0 && init_quantile < 1.0) || !(risk_q > 0.0 && risk_q < 1.0)) {
    set_error("init_quantile must be in [0,1) and risk_q in (0,1)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n_global_max < n_global) n_global_max = n_global;
  if (!ws || !aligned(ws, 256)) {
    set_error("threshold workspace missing or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = sticky();
  if (r) return r;
  return fit_threshold_comm_async(scores, n_local, n_global, init_quantile, risk_q, comm, out_dev,
                                  ws, ws_bytes, n_global_max, static_cast<cudaStream_t>(stream));
}

enova_status enova_fit_threshold_dist_async(const float *scores, int64_t n_local, int64_t n_global,
                                            int64_t n_global_max, double init_quantile,
                                            double risk_q, enova_comm_t comm,
                                            enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                            void *stream) {
  if (!comm || !out_dev || n_local < 0 || (n_local > 0 && !scores) || n_global < 1 ||
      !aligned(out_dev, 8)) {
    set_error("bad fit_threshold_dist_async arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!(init_quantile >= 0.0 && init_quantile < 1.0) || !(risk_q > 0.0 && risk_q < 1.0)) {
    set_error("init_quantile must be in [0,1) and risk_q in (0,1)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n_global_max < n_global) n_global_max = n_global;
  if (!ws || !aligned(ws, 256)) {
    set_error("threshold workspace missing or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = sticky();
  if (r) return r;
  return fit_threshold_dist_async(scores, n_local, n_global, init_quantile, risk_q, comm, out_dev,
                                  ws, ws_bytes, n_global_max, static_cast<cudaStream_t>(stream));
}

enova_status enova_fit_threshold(const float *scores, int64_t n_local, int64_t n_global_max,
                                 double init_quantile, double risk_q, enova_comm_t comm,
                                 enova_threshold *out, void *ws, size_t ws_bytes, void *stream) {
  if (!out || n_local < 0 || (n_local > 0 && !scores)) {
    set_error("bad fit_threshold arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!(init_quantile >= 0.0 && init_quantile < 1.0) || !(risk_q > 0.0 && risk_q < 1.0)) {
    set_error("init_quantile must be in [0,1) and risk_q in (0,1)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n_global_max < n_local) n_global_max = n_local;
  if (!ws || !aligned(ws, 256)) {
    set_error("threshold workspace missing or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = sticky();
  if (r) return r;
  return fit_threshold(scores, n_local, init_quantile, risk_q, comm, out, ws, ws_bytes,
                       n_global_max, static_cast<cudaStream_t>(stream));
}

enova_status enova_fit_threshold_async(const float *scores, int64_t n, int64_t n_global_max,
                                       double init_quantile, double risk_q,
                                       enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                       void *stream) {
  if (!out_dev || n < 1 || !scores || !aligned(out_dev, 8)) {
    set_error("bad fit_threshold_async arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!(init_quantile >= 0.0 && init_quantile < 1.0) || !(risk_q > 0.0 && risk_q < 1.0)) {
    set_error("init_quantile must be in [0,1) and risk_q in (0,1)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (n_global_max < n) n_global_max = n;
  if (!ws || !aligned(ws, 256)) {
    set_error("threshold workspace missing or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  enova_status r = sticky();
  if (r) return r;
  return fit_threshold_async(scores, n, init_quantile, risk_q, out_dev, ws, ws_bytes,
                             n_global_max, static_cast<cudaStream_t>(stream));
}

enova_status enova_detect(const enova_series *series, const enova_detector *det,
                          const void *det_ws, size_t det_ws_bytes, const enova_threshold *thr,
                          int8_t *flags, float *scores_opt, float *md_opt, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if ((r = check_series_windows(series, L))) return r;
  if (!thr || !isfinite(thr->z_q)) {
    set_error("threshold missing or not finite");
    return ENOVA_ERR_UNCALIBRATED;
  }
  const bool empty = series->n_instances == 0 || series->t_end == series->t_begin;
  if (!flags && !empty) {
    set_error("flags output is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  if (empty) return ENOVA_OK;
  return launch_score(series, L, det_ws, scores_opt, md_opt, flags, thr->z_q, nullptr,
                      static_cast<cudaStream_t>(stream));
}

enova_status enova_detect_async(const enova_series *series, const enova_detector *det,
                                const void *det_ws, size_t det_ws_bytes,
                                const enova_threshold *thr_dev, int8_t *flags, float *scores_opt,
                                float *md_opt, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if ((r = check_series_windows(series, L))) return r;
  if (!thr_dev || !aligned(thr_dev, 8)) {
    set_error("device threshold missing or misaligned");
    return ENOVA_ERR_UNCALIBRATED;
  }
  const bool empty = series->n_instances == 0 || series->t_end == series->t_begin;
  if (!flags && !empty) {
    set_error("flags output is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  if (empty) return ENOVA_OK;
  return launch_score(series, L, det_ws, scores_opt, md_opt, flags, 0.0, &thr_dev->z_q,
                      static_cast<cudaStream_t>(stream));
}

enova_status enova_ring_push(float *ring, int64_t n_instances, int32_t window, int32_t n_metrics,
                             const float *sample, int64_t tick, void *stream) {
  if (!ring || !sample || n_instances < 0 || window < 1 || n_metrics < 1 || tick < 0 ||
      (n_metrics % 4) != 0 || !aligned(ring, 16) || !aligned(sample, 16)) {
    set_error("bad ring_push arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return ring_push(ring, n_instances, window, n_metrics, sample, tick,
                   static_cast<cudaStream_t>(stream));
}

size_t enova_stream_ring_bytes(int64_t n_instances, int32_t window, int32_t n_metrics) {
  if (n_instances < 0 || window < 2 || window > 256 || (window % 2) != 0 ||
      !(n_metrics == 8 || n_metrics == 16 || n_metrics == 32 || n_metrics == 64))
    return 0;
  return stream_ring_bytes(n_instances, window, n_metrics);
}

enova_status enova_stream_push(void *ring, int64_t n_instances, int32_t window, int32_t n_metrics,
                               const float *sample, const float *norm_mean, const float *norm_std,
                               int64_t tick, void *stream) {
  if (enova_stream_ring_bytes(n_instances, window, n_metrics) == 0) {
    set_error("stream ring: bad shape (W even 2..256, M in {8,16,32,64})");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (!ring || !sample || !norm_mean || !norm_std || tick < 0 || !aligned(ring, 256) ||
      !aligned(sample, 16) || !aligned(norm_mean, 16) || !aligned(norm_std, 16)) {
    set_error("bad stream_push arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return stream_push(ring, n_instances, window, n_metrics, sample, norm_mean, norm_std, tick,
                     static_cast<cudaStream_t>(stream));
}

enova_status enova_stream_detect(const void *ring, int64_t n_instances, int64_t tick,
                                 const enova_detector *det, const void *det_ws,
                                 size_t det_ws_bytes, const enova_threshold *thr_dev,
                                 int8_t *flags, float *scores_opt, float *md_opt, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if (enova_stream_ring_bytes(n_instances, L.W, L.M) == 0) {
    set_error("stream ring: bad shape (M in {8,16,32,64})");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (!ring || !aligned(ring, 256) || n_instances < 0) {
    set_error("stream ring missing or misaligned");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (tick < L.W - 1) {
    set_error("stream_detect needs W pushed ticks (tick >= W-1)");
    return ENOVA_ERR_INSUFFICIENT_HISTORY;
  }
  if (flags && (!thr_dev || !aligned(thr_dev, 8))) {
    set_error("device threshold missing or misaligned");
    return ENOVA_ERR_UNCALIBRATED;
  }
  if (!flags && !scores_opt && !md_opt && n_instances > 0) {
    set_error("no output requested");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  return stream_detect(ring, n_instances, tick, L, det_ws, thr_dev ? &thr_dev->z_q : nullptr,
                       flags, scores_opt, md_opt, static_cast<cudaStream_t>(stream));
}

enova_status enova_stream_step(void *ring, int64_t n_instances, int64_t tick, const float *sample,
                               const float *norm_mean, const float *norm_std,
                               const enova_detector *det, const void *det_ws,
                               size_t det_ws_bytes, const enova_threshold *thr_dev,
                               int8_t *flags, float *scores_opt, float *md_opt, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if (enova_stream_ring_bytes(n_instances, L.W, L.M) == 0) {
    set_error("stream ring: bad shape (M in {8,16,32,64})");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (!ring || !aligned(ring, 256) || n_instances < 0 ||
      (n_instances > 0 && (!sample || !norm_mean || !norm_std || !aligned(sample, 16) ||
                           !aligned(norm_mean, 16) || !aligned(norm_std, 16)))) {
    set_error("bad stream_step arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (tick < L.W - 1) {
    set_error("stream_step needs W-1 earlier pushed ticks (tick >= W-1)");
    return ENOVA_ERR_INSUFFICIENT_HISTORY;
  }
  if (flags && (!thr_dev || !aligned(thr_dev, 8))) {
    set_error("device threshold missing or misaligned");
    return ENOVA_ERR_UNCALIBRATED;
  }
  if (!flags && !scores_opt && !md_opt && n_instances > 0) {
    set_error("no output requested");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  return stream_step(ring, n_instances, tick, L, det_ws, sample, norm_mean, norm_std,
                     thr_dev ? &thr_dev->z_q : nullptr, flags, scores_opt, md_opt,
                     static_cast<cudaStream_t>(stream));
}

enova_status enova_spot_update(const float *scores, const int8_t *flags, int64_t n, void *ws,
                               size_t ws_bytes, int64_t n_global_max, double init_quantile,
                               void *stream) {
  if (n < 0 || !ws || !aligned(ws, 256) || n_global_max <= 0 || !(init_quantile > 0.0) ||
      !(init_quantile < 1.0) || (n > 0 && (!scores || !flags))) {
    set_error("bad spot_update arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return spot_update(scores, flags, n, ws, ws_bytes, n_global_max, init_quantile,
                     static_cast<cudaStream_t>(stream));
}

enova_status enova_spot_refit(double risk_q, enova_threshold *out_dev, void *ws, size_t ws_bytes,
                              int64_t n_global_max, double init_quantile, void *stream) {
  if (!out_dev || !aligned(out_dev, 8) || !ws || !aligned(ws, 256) || n_global_max <= 0 ||
      !(risk_q > 0.0) || !(risk_q < 1.0) || !(init_quantile > 0.0) || !(init_quantile < 1.0)) {
    set_error("bad spot_refit arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return spot_refit(risk_q, out_dev, ws, ws_bytes, n_global_max, init_quantile,
                    static_cast<cudaStream_t>(stream));
}

size_t enova_select_flagged_scratch_bytes(int64_t n) {
  return n < 0 ? 0 : select_flagged_scratch_bytes(n);
}

enova_status enova_select_flagged(const int8_t *flags, int64_t n, int64_t *ids_out,
                                  int64_t *count_dev, void *scratch, void *stream) {
  if (n < 0 || !count_dev || !aligned(count_dev, 8) ||
      (n > 0 && (!flags || !ids_out || !scratch || !aligned(ids_out, 8)))) {
    set_error("bad select_flagged arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return select_flagged(flags, n, ids_out, reinterpret_cast<long long *>(count_dev), scratch,
                        static_cast<cudaStream_t>(stream));
}

enova_status enova_explain_windows(const enova_series *series, const enova_detector *det,
                                   const void *det_ws, size_t det_ws_bytes, const int64_t *ids_dev,
                                   int64_t n_ids, float *md_metric, float *scores_opt,
                                   float *md_opt, void *stream) {
  DetLayout L;
  enova_status r = check_detector(det, &L);
  if (r) return r;
  if ((r = check_series_windows(series, L))) return r;
  if (!rows_path_ok(L)) {
    set_error("explain_windows supports M in {8, 16}");
    return ENOVA_ERR_UNSUPPORTED;
  }
  if (n_ids < 0 || (n_ids > 0 && (!ids_dev || !md_metric))) {
    set_error("bad explain_windows arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!det_ws || det_ws_bytes < L.total || !aligned(det_ws, 256)) {
    set_error("prepared-detector workspace missing, too small or misaligned");
    return ENOVA_ERR_WORKSPACE;
  }
  if ((r = sticky())) return r;
  return launch_explain_rows(series, L, det_ws, ids_dev, n_ids, md_metric, scores_opt, md_opt,
                             static_cast<cudaStream_t>(stream));
}

enova_status enova_point_adjusted_counts(const int8_t *labels, int64_t ld_labels,
                                         const int8_t *flags, int64_t n_instances,
                                         int64_t t_begin, int64_t n_windows,
                                         uint64_t *counts_dev, void *stream) {
  if (!counts_dev || !aligned(counts_dev, 8) || n_instances < 0 || n_windows < 0 || t_begin < 0 ||
      ld_labels < t_begin + n_windows || (n_instances > 0 && n_windows > 0 && (!labels || !flags))) {
    set_error("bad point_adjusted_counts arguments");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  enova_status r = sticky();
  if (r) return r;
  return point_adjust_counts(labels, ld_labels, flags, n_instances, t_begin, n_windows,
                             reinterpret_cast<unsigned long long *>(counts_dev),
                             static_cast<cudaStream_t>(stream));
}

}  // extern "C"
