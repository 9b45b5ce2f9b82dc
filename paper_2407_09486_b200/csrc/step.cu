// step.cu -- the whole detection hot path of one batch as ONE stream-ordered
// call (enova_step_enqueue), with the threshold fit overlapped with the
// detection scores.
//
// Dependencies of a step:
//   stats (a-1) -> calibration scores + MD (a-2..a-5) -> POT fit (a-7..a-9)
//   stats (a-1) -> detection scores + MD (a-2..a-5)
//   fit + all scores -> flags (a-6) of every window
// The detection scores do not need the threshold -- only their flags do -- so
// the fit (a latency-bound cooperative kernel: radix passes, grid barriers, an
// fp64 root search; ~0.1 ms at c2 whatever its grid) need not stall the SMs.
// In the overlapped mode the fit runs on a side stream with a reduced grid
// (pot_ctas CTAs in 2-CTA clusters, i.e. whole TPCs) while the detection scores
// of the first `concurrent_instances` instances run on the remaining TPCs
// (a capped CTA-pair launch); the rest of the detection scores follow on the
// whole device, then one launch flags the calibration and detection windows.
// Every output is bit-identical to the sequential order (scores do not depend
// on the launch that computes them; the fit depends on its grid only through
// the summation order, deterministic for a given pot_ctas).  Fork and join are
// events, so the whole step captures into one CUDA graph.
#include "comm.h"
#include "common.cuh"

struct enova_step_s {
  int device, sms;
  cudaStream_t aux;
  cudaEvent_t fork, join;
  int pot_ctas;                 // 0: sequential (fit on every SM, then detection)
  int64_t concurrent_instances; // detection instances scored next to the fit
  int fit_mode;                 // communicator: 0 replicated fit, 1 distributed fit
};

namespace enova {
void set_pair_cap(int pairs);
void set_pot_grid(int ctas, int cluster);
enova_status apply_flags(const float *scores, const float *md, int64_t n,
                         const enova_threshold *thr_dev, int8_t *flags, cudaStream_t st);
enova_status apply_flags2(const float *s1, const float *m1, int64_t n1, int8_t *f1,
                          const float *s2, const float *m2, int64_t n2, int8_t *f2,
                          const enova_threshold *thr_dev, cudaStream_t st);

namespace {
struct Overrides {   // thread-local launch overrides, reset on every exit path
  ~Overrides() {
    set_pair_cap(0);
    set_pot_grid(0, 0);
  }
};
}  // namespace
}  // namespace enova

using namespace enova;

extern "C" {

enova_status enova_step_create(enova_step_t *out, int device) {
  if (!out) {
    set_error("enova_step_create: out is NULL");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  ENOVA_CUDA_TRY(cudaSetDevice(device));
  enova_step_s *s = new enova_step_s();
  s->device = device;
  s->pot_ctas = 0;
  s->fit_mode = 0;
  s->concurrent_instances = 0;
  cudaError_t e = cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device);
  int lo = 0, hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s->aux, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->join, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete s;
    return cuda_status(e, "enova_step_create");
  }
  *out = s;
  return ENOVA_OK;
}

void enova_step_destroy(enova_step_t s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->aux);
  cudaEventDestroy(s->fork);
  cudaEventDestroy(s->join);
  cudaStreamDestroy(s->aux);
  delete s;
}

enova_status enova_step_configure(enova_step_t s, int32_t pot_ctas, int64_t concurrent_instances) {
  if (!s || pot_ctas < 0 || concurrent_instances < 0 || (pot_ctas % 2) != 0 ||
      pot_ctas >= s->sms) {
    set_error("enova_step_configure: pot_ctas even in [0, SMs), concurrent_instances >= 0");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  s->pot_ctas = pot_ctas;
  s->concurrent_instances = concurrent_instances;
  return ENOVA_OK;
}

enova_status enova_step_set_fit_mode(enova_step_t s, int32_t fit_mode) {
  if (!s || fit_mode < 0 || fit_mode > 1) {
    set_error("enova_step_set_fit_mode: fit_mode 0 (replicated) or 1 (distributed)");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  s->fit_mode = fit_mode;
  return ENOVA_OK;
}

enova_status enova_step_enqueue(enova_step_t s, const enova_step_args *a, void *stream) {
  if (!s || !a || !a->series || !a->det) {
    set_error("enova_step_enqueue: step, args, series and detector are required");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const enova_series &X = *a->series;
  const int W = a->det->window;
  const int64_t N = X.n_instances, T = X.n_steps, tcal = a->t_cal_end;
  if (tcal < W || tcal > T) {
    set_error("enova_step_enqueue: t_cal_end must be in [window, n_steps]");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  const int64_t n_cal = N * (tcal - (W - 1)), n_det = N * (T - tcal);
  if (s->pot_ctas > 0 && n_det > 0 && (!a->scores || !a->md)) {
    set_error("enova_step_enqueue: the overlapped step needs the detection scores and md outputs");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  if (!a->cal_scores || !a->cal_md || !a->cal_flags || !a->thr_dev || (n_det > 0 && !a->flags)) {
    set_error("enova_step_enqueue: cal_scores, cal_md, cal_flags, thr_dev and flags are required");
    return ENOVA_ERR_INVALID_ARGUMENT;
  }
  Overrides guard;
  enova_status r;
  // a-1: statistics over the calibration horizon
  if ((r = enova_compute_stats_async(&X, tcal, a->mean, a->std, a->stats_diag, a->stats_ws,
                                     a->stats_ws_bytes, st)))
    return r;
  // a-2..a-5 on the calibration windows (scores + MD; flagged after the fit)
  enova_series cal = X;
  cal.t_begin = W - 1;
  cal.t_end = tcal;
  cal.norm_mean = a->mean;
  cal.norm_std = a->std;
  if ((r = enova_score_windows(&cal, a->det, a->det_ws, a->det_ws_bytes, a->cal_scores, a->cal_md,
                               st)))
    return r;
  enova_series det = cal;
  det.t_begin = tcal;
  det.t_end = T;
  auto fit = [&](cudaStream_t fs) -> enova_status {
    if (a->comm && s->fit_mode == 1)
      return enova_fit_threshold_dist_async(a->cal_scores, n_cal, a->n_global, a->n_global_max,
                                            a->init_quantile, a->risk_q, a->comm, a->thr_dev,
                                            a->thr_ws, a->thr_ws_bytes, fs);
    if (a->comm)
      return enova_fit_threshold_comm_async(a->cal_scores, n_cal, a->n_global, a->n_global_max,
                                            a->init_quantile, a->risk_q, a->comm, a->thr_dev,
                                            a->thr_ws, a->thr_ws_bytes, fs);
    return enova_fit_threshold_async(a->cal_scores, n_cal, a->n_global_max, a->init_quantile,
                                     a->risk_q, a->thr_dev, a->thr_ws, a->thr_ws_bytes, fs);
  };
  if (s->pot_ctas == 0 || n_det == 0) {
    // sequential: fit on every SM, then the detection windows with inline flags
    if ((r = fit(st))) return r;
    if ((r = apply_flags(a->cal_scores, a->cal_md, n_cal, a->thr_dev, a->cal_flags, st))) return r;
    return enova_detect_async(&det, a->det, a->det_ws, a->det_ws_bytes, a->thr_dev, a->flags,
                              a->scores, a->md, st);
  }
  // overlapped: fork the fit onto the side stream with a reduced grid
  ENOVA_CUDA_TRY(cudaEventRecord(s->fork, st));
  ENOVA_CUDA_TRY(cudaStreamWaitEvent(s->aux, s->fork, 0));
  // a fit grid of <= 16 CTAs runs as one cluster (cluster barriers instead of
  // grid barriers through global memory); larger grids as whole TPCs
  set_pot_grid(s->pot_ctas, s->pot_ctas <= 16 ? s->pot_ctas : 2);
  r = fit(s->aux);
  set_pot_grid(0, 0);
  if (r) return r;
  ENOVA_CUDA_TRY(cudaEventRecord(s->join, s->aux));
  // detection scores: the first instances on the TPCs the fit leaves free, then
  // the rest on the whole device (no flags yet: they need z_q)
  const int64_t a1 = s->concurrent_instances < N ? s->concurrent_instances : N;
  const int64_t nw = T - tcal;
  if (a1 > 0) {
    enova_series d1 = det;
    d1.n_instances = a1;
    set_pair_cap((s->sms - s->pot_ctas) / 2);
    r = enova_score_windows(&d1, a->det, a->det_ws, a->det_ws_bytes, a->scores, a->md, st);
    set_pair_cap(0);
    if (r) return r;
  }
  if (a1 < N) {
    enova_series d2 = det;
    d2.n_instances = N - a1;
    d2.metrics = X.metrics + a1 * X.ld_instance;
    d2.norm_mean = a->mean + a1 * X.n_metrics;
    d2.norm_std = a->std + a1 * X.n_metrics;
    if ((r = enova_score_windows(&d2, a->det, a->det_ws, a->det_ws_bytes, a->scores + a1 * nw,
                                 a->md + a1 * nw, st)))
      return r;
  }
  ENOVA_CUDA_TRY(cudaStreamWaitEvent(st, s->join, 0));
  // a-6 for every window of the step, one launch
  return apply_flags2(a->cal_scores, a->cal_md, n_cal, a->cal_flags, a->scores, a->md, n_det,
                      a->flags, a->thr_dev, st);
}

}  // extern "C"
