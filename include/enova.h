/*
 * enova.h -- C ABI of the B200-native ENOVA performance-detection hot path.
 *
 * ENOVA (arXiv 2407.09486) detects anomalous service performance with a VAE
 * over normalised monitoring metrics, scores each input by the KL divergence
 * of the posterior from the prior, sets the anomaly threshold with the
 * peaks-over-threshold (POT) method, and uses the Mean Difference (MD) between
 * the input and its reconstruction to decide scale-up vs scale-down
 * (PAPER.md:282-297).  This library runs that path over a fleet's metric
 * tensor [instances x T x M] with sliding windows of length W.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; R-n = reading n in
 * DESIGN.md (where the paper is silent or ambiguous).
 *
 * Conventions (every entry point):
 *  - All tensors are caller-owned.  Pointers documented "device" must be CUDA
 *    device pointers on the current device; "host" pointers are host memory.
 *    The library never allocates device memory on the hot path; scratch lives
 *    in caller-provided workspaces sized by the *_workspace_bytes functions
 *    (256-byte aligned; one workspace per concurrent stream).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    score/detect/stats/ring_push are stream-ordered and asynchronous;
 *    enova_compute_stats synchronises only to return n_degenerate;
 *    enova_fit_threshold is synchronous and returns with *out filled.
 *    The *_async variants (stats, single-GPU threshold, detect) never
 *    synchronise: their status and results stay in device memory, so a whole
 *    pipeline step can be enqueued back to back or captured in a CUDA graph.
 *  - Argument and shape errors are detected before any launch; outputs are
 *    then untouched.  Sticky CUDA / NCCL errors surface as ENOVA_ERR_CUDA /
 *    ENOVA_ERR_NCCL; enova_last_error() returns a thread-local detail string.
 *    No C++ exception crosses the ABI.
 *  - Fast-path envelope (else ENOVA_ERR_UNSUPPORTED, there is no fallback):
 *    M in {8, 16, 32, 64}; W even, 2 <= W <= 256; H in {32, 64, 128};
 *    1 <= Z <= 16.
 *  - Precision is part of the contract (R-17): the detector is defined on fp16
 *    tensor-core operands.  enc_w1, enc_wmu, enc_wlv and dec_w1 are rounded to
 *    fp16 (RNE) by enova_prepare_detector; the normalised input is
 *    x = fp16_RNE(clamp(fp32((fp32(X - mean)) / std), +-1e4)).  Everything after
 *    that is carried with fp32 accumulation (h and mu as hi+lo fp16 pairs).
 */
#ifndef ENOVA_H_
#define ENOVA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENOVA_ABI_VERSION 1

typedef enum {
  ENOVA_OK = 0,
  ENOVA_ERR_INVALID_ARGUMENT = 1,   /* null pointer, bad size, misalignment          */
  ENOVA_ERR_UNSUPPORTED = 2,        /* shape outside the fast-path envelope           */
  ENOVA_ERR_INSUFFICIENT_HISTORY = 3, /* T < W, or a window range needs t < W-1 */
  ENOVA_ERR_TOO_FEW_EXCEEDANCES = 4,  /* fewer than 10 POT peaks       */
  ENOVA_ERR_NONFINITE = 5,          /* NaN/Inf in the calibration horizon (R-18)       */
  ENOVA_ERR_UNCALIBRATED = 6,       /* threshold missing or not finite         */
  ENOVA_ERR_CUDA = 7,
  ENOVA_ERR_NCCL = 8,
  ENOVA_ERR_WORKSPACE = 9           /* workspace too small or misaligned               */
} enova_status;

/* Detector parameters (VAE; topology S:547, R-5).  Device pointers,
 * fp32, row-major [out][in], read-only.  D = window * n_metrics, flattened
 * time-major k = tau*M + j with tau = 0 the oldest sample of the window (R-1). */
typedef struct {
  int32_t window, n_metrics, hidden, latent;   /* W, M, H, Z                    */
  const float *enc_w1, *enc_b1;    /* [H][D], [H]      encoder hidden layer    */
  const float *enc_wmu, *enc_bmu;  /* [Z][H], [Z]      posterior mean head     */
  const float *enc_wlv, *enc_blv;  /* [Z][H], [Z]      posterior log-variance  */
  const float *dec_w1, *dec_b1;    /* [H][Z], [H]      decoder hidden layer    */
  const float *dec_w2, *dec_b2;    /* [D][H], [D]      linear output m'        */
} enova_detector;

/* A fleet's metric tensor and the window range to score.
 * metrics: device fp32, instance i occupies [i*ld_instance, i*ld_instance + T*M),
 * row-major [T][M]; 16-byte aligned, ld_instance % 4 == 0, ld_instance >= T*M.
 * Windows ENDING at t in [t_begin, t_end) are scored (window = samples
 * t-W+1 .. t, R-2); requires W-1 <= t_begin <= t_end <= T.
 * Per-window outputs are laid out [N][t_end - t_begin] (index t - t_begin).
 * norm_mean / norm_std: device fp32 [N][M] from enova_compute_stats over the
 * calibration horizon, frozen for detection and streaming (R-4);
 * REQUIRED by score/detect. */
typedef struct {
  const float *metrics;
  int64_t n_instances, n_steps, ld_instance;
  int64_t t_begin, t_end;
  const float *norm_mean, *norm_std;
  int32_t n_metrics, reserved;     /* M; must equal detector.n_metrics */
} enova_series;

/* POT threshold (P:297 citing Siffer et al. 2017, R-11..R-13).
 * t = initial threshold (order statistic), (gamma, sigma) = GPD MLE of the
 * peaks, z_q = final threshold at risk q, n = scores used, n_peaks = N_t,
 * method 0 = GPD root (gamma != 0), 1 = exponential candidate (gamma == 0). */
typedef struct {
  double init_quantile, risk_q, t, gamma, sigma, z_q;
  int64_t n, n_peaks;
  int32_t method, reserved;
} enova_threshold;

typedef struct enova_comm_s *enova_comm_t;

/* ---------------------------------------------------------------- K0 ----
 * Bytes of the prepared-detector image (fp16 canonical UMMA operand images of
 * W1, [Wmu|Wlv], W3; fp32 biases; w_bar = 1^T W_dec2 and b_bar = sum b_dec2
 * accumulated in fp64).  0 if the detector is outside the envelope. */
size_t enova_detector_workspace_bytes(const enova_detector *det);

/* Build the prepared-detector image into det_ws (device, caller-owned, must
 * stay alive and unmodified while score/detect use it).  Asynchronous. */
enova_status enova_prepare_detector(const enova_detector *det, void *det_ws,
                                    size_t det_ws_bytes, void *stream);

/* ---------------------------------------------------------------- a-1 ----
 * Per-(instance, metric) mean and population std over samples [0, t_cal_end)
 * ("input metrics are normalized prior"; R-4), accumulated in
 * fp64 (one pass of shifted sums, time chunks combined in a fixed order) and
 * rounded to fp32; std floored at 1e-6.  mean/std: device fp32 [N][M].
 * *n_degenerate (host, may be NULL): series whose std was floored.
 * Reads series->metrics / n_instances / n_steps / ld_instance / n_metrics only.
 * ws: device scratch of enova_stats_workspace_bytes(N, M) bytes, 256-aligned.
 * Returns ENOVA_ERR_NONFINITE if any sample in the horizon is NaN/Inf (R-18);
 * synchronises the stream. */
size_t enova_stats_workspace_bytes(int64_t n_instances, int32_t n_metrics);
enova_status enova_compute_stats(const enova_series *series, int64_t t_cal_end, float *mean, float *std,
                                 int64_t *n_degenerate, void *ws, size_t ws_bytes,
                                 void *stream);
/* Stream-ordered variant (no synchronisation).  diag_dev (device int64[2], may
 * be NULL): [0] = series whose std was floored, [1] > 0 iff a sample in the
 * horizon is NaN/Inf (what enova_compute_stats reports as
 * ENOVA_ERR_NONFINITE).  Argument errors are still returned synchronously. */
enova_status enova_compute_stats_async(const enova_series *series, int64_t t_cal_end, float *mean,
                                       float *std, int64_t *diag_dev, void *ws, size_t ws_bytes,
                                       void *stream);

/* ------------------------------------------------------------ a-2..a-5 ----
 * KL score (R-6) and MD (R-8) of every window in
 * the series range.  scores, md: device fp32 [N][t_end - t_begin] (md may be
 * NULL).  det_ws: the image from enova_prepare_detector for `det`. */
enova_status enova_score_windows(const enova_series *series, const enova_detector *det,
                                 const void *det_ws, size_t det_ws_bytes,
                                 float *scores, float *md, void *stream);

/* ------------------------------------------------------------ a-7..a-9 ----
 * Fleet-wide POT threshold over calibration scores.  scores: device fp32
 * [n_local] (this rank's shard).  comm == NULL: single GPU.  With a comm, all
 * ranks call collectively; integer histograms are all-reduced and score tails
 * all-gathered in rank order, so *out is bit-identical on every rank and for
 * every world size.  Argument / workspace errors are detected per rank before
 * the first collective: give every rank the same n_global_max (a rank that
 * returns early leaves the others waiting in a collective, as with NCCL).
 * n_global_max bounds sum(n_local) over ranks and must be
 * the value the workspace was sized with: enova_threshold_workspace_bytes
 * without a comm, enova_threshold_comm_workspace_bytes(.., world) with one.
 * out: host.  Synchronous.
 * ENOVA_ERR_TOO_FEW_EXCEEDANCES if fewer than 10 scores exceed t. */
size_t enova_threshold_workspace_bytes(int64_t n_global_max, double init_quantile);
size_t enova_threshold_comm_workspace_bytes(int64_t n_global_max, double init_quantile,
                                            int32_t world);
enova_status enova_fit_threshold(const float *scores, int64_t n_local, int64_t n_global_max,
                                 double init_quantile, double risk_q, enova_comm_t comm,
                                 enova_threshold *out, void *ws, size_t ws_bytes,
                                 void *stream);
/* Single-GPU, stream-ordered variant (one cooperative kernel, no host sync).
 * out_dev: DEVICE enova_threshold written by the kernel; out_dev->reserved holds
 * the enova_status of the fit (ENOVA_OK, ENOVA_ERR_TOO_FEW_EXCEEDANCES,
 * ENOVA_ERR_WORKSPACE, ENOVA_ERR_UNSUPPORTED) and z_q is NaN unless it is
 * ENOVA_OK, so enova_detect_async flags nothing from a failed fit.  Argument
 * errors are returned synchronously. */
enova_status enova_fit_threshold_async(const float *scores, int64_t n, int64_t n_global_max,
                                       double init_quantile, double risk_q,
                                       enova_threshold *out_dev, void *ws, size_t ws_bytes,
                                       void *stream);

/* Fleet-wide, stream-ordered variant (§8e): no host synchronisation, so the
 * whole call -- k_pot phase launches and the NCCL collectives between them
 * (3 histogram allreduces, an allgather of tail counts, an allgather of
 * fixed-size fp32 tail slots of capacity ~(1 - init_quantile) * n_global_max
 * per rank) -- can be captured in a CUDA graph.  n_global: sum of n_local over
 * the ranks, identical on every rank (e.g. from enova_comm_sum_i64 once at
 * setup).  out_dev / status as enova_fit_threshold_async; bit-identical to the
 * single-GPU fit of the rank-ordered concatenation of the shards. */
enova_status enova_fit_threshold_comm_async(const float *scores, int64_t n_local,
                                            int64_t n_global, int64_t n_global_max,
                                            double init_quantile, double risk_q,
                                            enova_comm_t comm, enova_threshold *out_dev,
                                            void *ws, size_t ws_bytes, void *stream);

/* Distributed-fit variant: the same selection
 * phases and collectives, then every rank fits the GPD on ITS OWN tail -- no
 * tail gather: one cooperative launch per fit step (statistics, grid scan,
 * certified refinement passes, candidates; a fixed sequence of 17 launches,
 * steps after convergence return at once) with an all-gather of the ranks'
 * pass totals (6 KB per rank) between steps, summed by every rank in rank
 * order.  z_q is bit-identical across the ranks of one communicator and equal
 * across world sizes up to the fp64 summation order (the replicated
 * enova_fit_threshold_comm_async is bit-identical across world sizes).  The
 * fit's work per rank is its own tail: the replicated fit's Amdahl term at large
 * world sizes.  Workspace, arguments, out_dev and status as
 * enova_fit_threshold_comm_async. */
enova_status enova_fit_threshold_dist_async(const float *scores, int64_t n_local,
                                            int64_t n_global, int64_t n_global_max,
                                            double init_quantile, double risk_q,
                                            enova_comm_t comm, enova_threshold *out_dev,
                                            void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------ a-2..a-6 ----
 * Score every window of the series range and flag it ("An anomaly is
 * detected if the KL-divergence ... exceeds this threshold", MD decides
 * "scale up or down", R-9, R-10):
 *   flag = 0 if score <= z_q; +1 (scale up) if MD >= 0; -1 (scale down) otherwise.
 * flags: device int8 [N][t_end - t_begin]; scores_opt / md_opt may be NULL.
 * thr: host; ENOVA_ERR_UNCALIBRATED if thr is NULL or z_q is not finite. */
enova_status enova_detect(const enova_series *series, const enova_detector *det,
                          const void *det_ws, size_t det_ws_bytes,
                          const enova_threshold *thr, int8_t *flags,
                          float *scores_opt, float *md_opt, void *stream);
/* As enova_detect with the threshold in DEVICE memory (e.g. the out_dev of
 * enova_fit_threshold_async); z_q is read by the kernel.  A NaN z_q (failed
 * fit) flags nothing. */
enova_status enova_detect_async(const enova_series *series, const enova_detector *det,
                                const void *det_ws, size_t det_ws_bytes,
                                const enova_threshold *thr_dev, int8_t *flags,
                                float *scores_opt, float *md_opt, void *stream);

/* a-6 on windows scored before the threshold existed (the calibration windows
 * of a step: scored with MD, then the POT fit runs on their scores): flags[i]
 * = 0 if scores[i] <= z_q, else +1 if md[i] >= 0, else -1 (PAPER.md:297
 * "exceeds this threshold", "scale up or down"; R-9, R-10) --
 * the comparison the score kernels make, with z_q read from the device
 * threshold (a failed fit has z_q = NaN: nothing is flagged).  scores, md:
 * device fp32 [n]; flags: device int8 [n]; all caller-owned.  Stream-ordered,
 * capturable.  ENOVA_ERR_INVALID_ARGUMENT for n < 0 or NULL buffers with
 * n > 0; ENOVA_ERR_UNCALIBRATED without a (8-byte aligned) thr_dev. */
enova_status enova_flag_scores_async(const float *scores, const float *md, int64_t n,
                                     const enova_threshold *thr_dev, int8_t *flags, void *stream);

/* ----------------------------------------------------------------- a-10 ----
 * Streaming ("executed in streaming computing framework"): a mirror
 * ring of 2W samples per instance, device fp32 [N][2W][M].  enova_ring_push
 * writes sample[N][M] (device) for tick `tick` at ring slots (tick mod W) and
 * (tick mod W) + W.  After the push of tick k >= W-1, the window ending at
 * tick k is the contiguous view ring + ((k+1) mod W)*M with ld_instance =
 * 2*W*M, n_steps = W, t_begin = W-1, t_end = W: pass it to enova_detect. */
enova_status enova_ring_push(float *ring, int64_t n_instances, int32_t window,
                             int32_t n_metrics, const float *sample, int64_t tick,
                             void *stream);

/* ------------------------------------------------ a-10, ingest-normalised ----
 * Streaming fast path: each new sample is normalised ONCE when it
 * arrives, with the frozen calibration statistics (R-4), into an fp16
 * mirror ring, so a tick scores every instance's newest window with no
 * re-normalisation and half the HBM bytes of the fp32 ring; the window's GEMM1
 * operand is fed to the tensor cores by TMA straight from the ring.  Results
 * are bit-identical to enova_detect on the same windows (same quantisation x =
 * fp16_RNE(clamp((X - mean)/std)), same sample-sum association).
 *
 * ring: device, 256-byte aligned, enova_stream_ring_bytes(N, W, M) bytes,
 * caller-owned, opaque to the caller: per instance a row of fp16 x (2W slots
 * of M metrics, the sample of tick k at slots k mod W and (k mod W) + W, the row
 * pitch padded off powers of two) followed (at a 256-byte boundary) by the fp32
 * per-sample sums s = sum_j x_j, 2W per instance (padded pitch).
 * M in {8, 16, 32, 64}.
 * enova_stream_push: sample device fp32 [N][M] (16-byte aligned) for tick
 * `tick` (>= 0); norm_mean / norm_std device fp32 [N][M] (enova_compute_stats).
 * enova_stream_detect: after pushes of ticks tick-W+1 .. tick (tick >= W-1),
 * scores / MD / flags of the window ending at `tick` of every instance:
 * outputs device [N] (scores_opt, md_opt may be NULL); thr_dev: DEVICE
 * enova_threshold (e.g. from enova_fit_threshold_async), required when flags
 * is not NULL; a NaN z_q flags nothing.  Both are stream-ordered and capturable
 * in CUDA graphs (one graph per ring phase tick mod W). */
size_t enova_stream_ring_bytes(int64_t n_instances, int32_t window, int32_t n_metrics);
/* One launch per tick: enova_stream_push of `sample` (tick `tick`) fused into
 * enova_stream_detect of the windows ending at `tick` (each CTA ingests its own
 * instances' samples, then TMA-loads their windows).  Same results as the two
 * calls; requires the pushes of ticks tick-W+1 .. tick-1 before. */
enova_status enova_stream_step(void *ring, int64_t n_instances, int64_t tick, const float *sample,
                               const float *norm_mean, const float *norm_std,
                               const enova_detector *det, const void *det_ws,
                               size_t det_ws_bytes, const enova_threshold *thr_dev,
                               int8_t *flags, float *scores_opt, float *md_opt, void *stream);
enova_status enova_stream_push(void *ring, int64_t n_instances, int32_t window, int32_t n_metrics,
                               const float *sample, const float *norm_mean, const float *norm_std,
                               int64_t tick, void *stream);
enova_status enova_stream_detect(const void *ring, int64_t n_instances, int64_t tick,
                                 const enova_detector *det, const void *det_ws,
                                 size_t det_ws_bytes, const enova_threshold *thr_dev,
                                 int8_t *flags, float *scores_opt, float *md_opt, void *stream);

/* ------------------------------------------------------ NEXT-2, online SPOT ----
 * Streaming threshold updates (SPOT, Siffer et al. 2017 -- the method PAPER.md:297
 * cites for the POT threshold; R-23, tick-synchronous): the SPOT state
 * is the single-GPU threshold workspace left by enova_fit_threshold_async on the
 * calibration scores (peaks Y, N_t, t, and the observation count n), sized with
 * an n_global_max large enough for the calibration plus the streamed scores.
 * Per tick: flag the tick's scores against the current threshold
 * (enova_stream_detect / enova_detect_async with thr_dev), then
 * enova_spot_update(scores, flags) appends every NON-anomalous score above t to
 * Y in index order (anomalies never update the model) and adds the number of
 * non-anomalous scores to n; enova_spot_refit re-fits the GPD on the grown Y and
 * writes the new device threshold (same as enova_fit_threshold_async's out_dev)
 * -- call it every tick (exact SPOT semantics per tick) or periodically.  The
 * peak capacity is ceil((1 - init_quantile) n_global_max) + 16 (calibration
 * peaks included).  Peaks beyond it are dropped; the next refit -- and every
 * later one until a new calibration fit -- does not fit the truncated set and
 * writes ENOVA_ERR_WORKSPACE to out_dev->reserved with z_q = NaN (so no window
 * is flagged against a biased threshold).  Both stream-ordered and capturable;
 * single GPU. */
enova_status enova_spot_update(const float *scores, const int8_t *flags, int64_t n, void *ws,
                               size_t ws_bytes, int64_t n_global_max, double init_quantile,
                               void *stream);
enova_status enova_spot_refit(double risk_q, enova_threshold *out_dev, void *ws, size_t ws_bytes,
                              int64_t n_global_max, double init_quantile, void *stream);

/* ----------------------------------------------------- NEXT-1, explanation ----
 * Per-metric root cause of flagged windows ("the root cause could
 * be localized to the lack of GPU memory for KV cache"): for each
 * listed window, the per-metric mean difference
 *   MD_j = (1/W) sum_tau (x_{tau,j} - m'_{tau,j}),  j = 0..M-1
 * between the normalised input x and the decoder reconstruction m' (P:297's MD
 * resolved per metric; MD = mean_j MD_j), computed by the column-sum identity per
 * metric (w_bar_j = sum_tau W_dec2[tau*M + j, :], exact algebra, R-8) on the
 * tensor-core row kernel.
 * enova_select_flagged: ids_out (device int64, capacity n) receives the
 * indices i of flags[i] != 0 in ascending order (flags device int8 [n], e.g.
 * the [N][nw] output of enova_detect flattened); *count_dev (device int64) the
 * number.  scratch: device, enova_select_flagged_scratch_bytes(n) bytes.
 * enova_explain_windows: ids_dev (device int64 [n_ids]) are window ids
 * g = instance * nw + (t - t_begin) of the series range (nw = t_end - t_begin);
 * md_metric: device fp32 [n_ids][M]; scores_opt / md_opt: device fp32 [n_ids]
 * (bit-identical to the batch kernels' score / MD of the same window).
 * M in {8, 16}.  Both stream-ordered. */
size_t enova_select_flagged_scratch_bytes(int64_t n);
enova_status enova_select_flagged(const int8_t *flags, int64_t n, int64_t *ids_out,
                                  int64_t *count_dev, void *scratch, void *stream);
enova_status enova_explain_windows(const enova_series *series, const enova_detector *det,
                                   const void *det_ws, size_t det_ws_bytes, const int64_t *ids_dev,
                                   int64_t n_ids, float *md_metric, float *scores_opt,
                                   float *md_opt, void *stream);

/* ----------------------------------------------------- NEXT-4, evaluation ----
 * Point-adjusted detection counts ("we adopt a point-adjusted
 * approach"; the rule as SPEC.md:530-533 states it, R-21): for each
 * contiguous true-anomaly segment containing at least one predicted point,
 * every point of the segment counts as predicted; then pointwise counts.
 * Points are the window end times t in [t_begin, t_begin + n_windows) of every
 * instance: prediction = flags[i][t - t_begin] != 0 (device int8 [N][n_windows],
 * the enova_detect output), truth = labels[i*ld_labels + t] != 0 (device int8,
 * ld_labels >= t_begin + n_windows).  Segments are clipped to the range and
 * never cross instances.  counts_dev: device uint64[4] = {TP, FP, FN, TN}
 * (overwritten), so precision = TP/(TP+FP), recall = TP/(TP+FN); exact integers,
 * summable across ranks.  Stream-ordered. */
enova_status enova_point_adjusted_counts(const int8_t *labels, int64_t ld_labels,
                                         const int8_t *flags, int64_t n_instances,
                                         int64_t t_begin, int64_t n_windows,
                                         uint64_t *counts_dev, void *stream);

/* ------------------------------------------------------------ the step ----
 * One pass of the whole hot path over one batch, as
 * ONE stream-ordered, graph-capturable call: statistics over [0, t_cal_end) ->
 * scores + MD of the calibration windows (ending in [W-1, t_cal_end)) -> the
 * (fleet-wide with `comm`) POT threshold on them -> scores + MD of the
 * detection windows (ending in [t_cal_end, T)) -> the flags of EVERY window
 * (PAPER.md:282, 297).  The step object owns a high-priority side stream and
 * two events (created at setup).  enova_step_configure(step, pot_ctas,
 * concurrent_instances): pot_ctas = 0 runs the stages in sequence (the fit on
 * every SM); pot_ctas > 0 (even) runs the fit on pot_ctas CTAs in 2-CTA
 * clusters on the side stream while the detection scores of the first
 * concurrent_instances instances run on the remaining TPCs, then the rest of
 * the detection scores, then one flag launch for all windows.  Outputs are
 * identical in both modes except for the fit's summation order (deterministic
 * for a given pot_ctas).  All buffers are caller-owned device memory in the
 * layouts of the single calls above (mean/std [N][M]; cal_* [N][t_cal_end-W+1];
 * scores/md/flags [N][T-t_cal_end]; thr_dev an enova_threshold); stats_diag is
 * the device int64[2] of enova_compute_stats_async.  n_global / n_global_max:
 * the calibration score count over all ranks / the threshold workspace sizing
 * (single GPU: both N*(t_cal_end-W+1) or larger).  Errors of the single calls
 * propagate unchanged; the overlapped mode needs scores and md. */
typedef struct enova_step_s *enova_step_t;
typedef struct {
  const enova_series *series;        /* metrics; norm_mean / norm_std / t_begin / t_end ignored */
  int64_t t_cal_end;
  const enova_detector *det;
  const void *det_ws;
  size_t det_ws_bytes;
  double init_quantile, risk_q;
  enova_comm_t comm;                 /* NULL = single GPU */
  int64_t n_global, n_global_max;
  float *mean, *std;
  int64_t *stats_diag;
  void *stats_ws;
  size_t stats_ws_bytes;
  float *cal_scores, *cal_md;
  int8_t *cal_flags;
  enova_threshold *thr_dev;
  void *thr_ws;
  size_t thr_ws_bytes;
  float *scores, *md;
  int8_t *flags;
} enova_step_args;
enova_status enova_step_create(enova_step_t *out, int device);
enova_status enova_step_configure(enova_step_t step, int32_t pot_ctas, int64_t concurrent_instances);
/* fit_mode (communicator steps): 0 = replicated fit on the gathered tails
 * (enova_fit_threshold_comm_async, default), 1 = distributed fit
 * (enova_fit_threshold_dist_async). */
enova_status enova_step_set_fit_mode(enova_step_t step, int32_t fit_mode);
enova_status enova_step_enqueue(enova_step_t step, const enova_step_args *args, void *stream);
void enova_step_destroy(enova_step_t step);

/* ------------------------------------------------------ NEXT-3, training ----
 * Semi-supervised training of the detector by Eq. 9:
 *   L = 1/B sum_i l_i log p(x_i | z_i) - (1 + l_i)/2 beta(k) KL(q(z|x_i) || N(0, I))
 * with l_i = +1 (normal or unlabelled) / -1 (labelled anomaly), the single-sample
 * reparameterised z_i = mu_i + exp(lv_i / 2) eps_i (eps an input, device fp32
 * [batch][latent]), the unit-variance Gaussian likelihood log p = -1/2 ||x -
 * m'(z)||^2 - D/2 log 2 pi and beta(k) from a PI controller
 * on the batch's mean KL of normal rows (R-24):
 *   e = KL - kl_setpoint, I += e while unclamped, beta = clamp(kp e + ki I, 0, beta_max)
 * (beta_mode 1: beta = beta_fixed).  Adam ascent on L (lr, adam_beta1/2,
 * adam_eps).  A window row is the score kernels' detector input x of the window
 * with id g = instance * nw + (t - t_begin) of the series range (nw = t_end -
 * t_begin); ids < 0 or >= n_instances * nw are padding rows (ignored; B counts
 * the valid rows).  The trainer owns its fp32 master parameters, Adam moments,
 * PI state, activations (max_batch rows) and a cuBLAS handle -- all allocated
 * at create (setup time; the step never allocates).  The GEMMs run in cuBLAS
 * (fp32 FFMA by default; enova_trainer_set_math(t, 1) allows TF32 tensor cores);
 * the element-wise / row-wise work and every reduction are the library's own
 * deterministic kernels.  All calls are stream-ordered on `stream`.
 *   enova_trainer_load:  parameters <- det (device fp32 tensors, include layouts);
 *                        Adam moments, step count and PI integral reset, beta = beta0.
 *   enova_trainer_store: parameters -> det's tensors (device fp32, WRITTEN).
 *   enova_train_step:    one Eq. 9 step on the `batch` rows ids (device int64)
 *                        with labels indexed BY WINDOW ID (device int8 [n_instances
 *                        * nw], +1 / -1) and eps, then Adam + PI update; stats_out (optional, device
 *                        fp64 [4]) = {L, beta used, mean KL of normal rows, their
 *                        mean log p - KL}.
 *   enova_train_gradient: dL/dtheta at the given beta, no update (parity checks):
 *                        grad_out device fp32 [enova_trainer_param_offsets(t, off)]
 *                        with tensor i of (enc_w1, enc_b1, enc_wmu, enc_bmu, enc_wlv,
 *                        enc_blv, dec_w1, dec_b1, dec_w2, dec_b2) at offset off[i].
 * Errors: ENOVA_ERR_INVALID_ARGUMENT for shapes / NULL inputs / batch outside
 * [1, max_batch]; ENOVA_ERR_CUDA for allocation, cuBLAS or launch failures. */
typedef struct enova_trainer_s *enova_trainer_t;
typedef struct {
  double lr, adam_beta1, adam_beta2, adam_eps;
  double kl_setpoint, kp, ki, beta_max;
  int32_t beta_mode;        /* 0 = PI controller, 1 = fixed beta_fixed */
  int32_t reserved;
  double beta_fixed;
} enova_train_config;
enova_status enova_trainer_create(enova_trainer_t *out, int32_t window, int32_t n_metrics,
                                  int32_t hidden, int32_t latent, int32_t max_batch, int device);
void enova_trainer_destroy(enova_trainer_t t);
int64_t enova_trainer_param_offsets(enova_trainer_t t, int64_t *offsets10);
enova_status enova_trainer_set_math(enova_trainer_t t, int32_t math);
enova_status enova_trainer_load(enova_trainer_t t, const enova_detector *det, double beta0,
                                void *stream);
enova_status enova_trainer_store(enova_trainer_t t, const enova_detector *det, void *stream);
enova_status enova_train_step(enova_trainer_t t, const enova_series *series, const int64_t *ids,
                              const int8_t *labels, int32_t batch, const float *eps,
                              const enova_train_config *cfg, double *stats_out, void *stream);
enova_status enova_train_gradient(enova_trainer_t t, const enova_series *series,
                                  const int64_t *ids, const int8_t *labels, int32_t batch,
                                  const float *eps, double beta, float *grad_out,
                                  double *stats_out, void *stream);

/* ------------------------------------------------------------ comm (§8e) ----
 * NCCL communicator for the fleet-wide threshold.  Rank 0 creates the 128-byte
 * unique id; the caller broadcasts it (e.g. torch.distributed) and every rank
 * calls enova_comm_create with its own device.  NCCL is loaded at run time
 * (libnccl.so.2); ENOVA_ERR_NCCL if it is unavailable. */
enova_status enova_comm_unique_id(void *out128);
enova_status enova_comm_create(enova_comm_t *comm, int rank, int world, const void *id128,
                               int device);
/* In-process communicator: comms[0..world) are `world` ranks that live in ONE
 * process on `device`, each driven by its own host thread (collectives
 * rendezvous on the host and are ordered across the ranks' streams with
 * events).  Runs the multi-rank threshold path on one GPU; not graph-capturable.
 * The ranks' grid-synchronising threshold kernels are serialised on the device
 * (they must never share the SMs).  world <= 16.  Destroy every handle with
 * enova_comm_destroy. */
enova_status enova_comm_create_local(enova_comm_t *comms, int world, int device);
/* Synchronous sum of one int64 over the ranks (collective; setup-time helper:
 * it allocates and frees 256 B of device scratch, so keep it off the hot path). */
enova_status enova_comm_sum_i64(enova_comm_t comm, int64_t in, int64_t *out, void *stream);
void enova_comm_destroy(enova_comm_t comm);
/* Failure handling of the fleet collectives (SURVEY §5, §8b conventions).
 * Every host-side wait on a communicator is bounded by its timeout (default
 * 300 s; enova_comm_set_timeout, seconds > 0): enova_fit_threshold with a
 * communicator, enova_comm_sum_i64 and enova_comm_wait poll the stream and
 * ncclCommGetAsyncError instead of blocking in cudaStreamSynchronize.  An
 * asynchronous NCCL error or an expired timeout (a peer rank died or stalled)
 * aborts the communicator (ncclCommAbort: no rank stays blocked in a
 * collective) and returns ENOVA_ERR_NCCL; every later call on it returns
 * ENOVA_ERR_NCCL too, and enova_comm_destroy only frees the handle.  The local
 * backend bounds its host rendezvous the same way.
 * enova_comm_wait(comm, stream): bounded wait for the work enqueued on `stream`
 * (e.g. a captured fleet step replayed with fit_threshold_comm_async inside)
 * before reading its results on the host. */
enova_status enova_comm_set_timeout(enova_comm_t comm, double seconds);
enova_status enova_comm_wait(enova_comm_t comm, void *stream);

/* ------------------------------------------------------------- misc ---- */
const char *enova_status_string(enova_status s);
/* Number of CUDA kernels this library has launched in this process (all
 * devices, monotonically increasing; diagnostic for benchmarks). */
uint64_t enova_kernel_launches(void);
/* Diagnostic kernel override for the windowed scoring calls (score_windows,
 * detect*): 0 = choose by shape (default), 1 = W1-streaming kernel, 2 = CTA-pair
 * kernel, 3 = instance-batched row kernel (where the shape allows; otherwise
 * the choice by shape).  Process-wide; used by A/B and parity tests only.
 * ENOVA_ERR_INVALID_ARGUMENT for any other value. */
enova_status enova_set_score_kernel(int which);
const char *enova_last_error(void);
int enova_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ENOVA_H_ */
