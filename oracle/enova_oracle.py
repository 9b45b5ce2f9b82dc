"""ENOVA performance-detection oracle: plain, slow, fp64 NumPy.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module.  The product path (``paper_2407_09486_b200``) never imports it and
shares no code with it; the two meet only at the seeded input generators in
``paper_2407_09486_b200/synth.py``.

What it computes (citations are PAPER.md line numbers ``P:n`` and SPEC.md line
numbers ``S:n``; readings ``R-n`` are listed in DESIGN.md):

1. ``series_stats``   per-(instance, metric) mean / population std over the
   calibration horizon, std floored at 1e-6 ("input metrics are
   normalized prior"; R-4).
2. ``normalise_x16``  z = (X - mean) / std in fp32, clamped to +-1e4, rounded to
   fp16: the detector input x (R-4, R-17).  ``normalise_exact`` is the
   fp64-only variant used for the disclosed "exact" comparison.
3. ``window_matrix``  window ending at t = the W samples t-W+1 .. t, flattened
   time-major k = tau*M + j, tau = 0 oldest ("[x_{t-w} ... x_t]";
   S:66-74; R-1, R-2).
4. ``encoder``        h = tanh(W1 x + b1); mu = Wmu h + bmu; lv = Wlv h + blv
   (P:282 VAE encoder q_phi(z|m); S:547 two-layer tanh MLP; R-5).
5. ``kl_score``       KL(N(mu, diag e^lv) || N(0, I)) = 1/2 sum(mu^2 + e^lv - 1 - lv)
   ("focuses on the KL-divergence"; R-6).
6. ``decoder`` / ``mean_difference``  m' = W_dec2 tanh(W3 mu + b3) + b_dec2
   (explicit, full D-wide); MD = mean_k (x_k - m'_k) ("Mean Difference
   (MD) between the input metrics m and the reconstructed metrics m'";
   S:524; R-7, R-8).
7. ``pot_threshold``  peaks-over-threshold (P:297 citing Siffer et al. 2017;
   S:232-240): t = S_(floor(q0 n)); Y = {s - t : s > t};
   GPD MLE by Grimshaw's reduction (``gpd_grimshaw``); z_q (R-11 .. R-13).
8. ``flags``          0 if score <= z_q, else +1 (scale up) if MD >= 0 else -1
   ("exceeds this threshold", "scale up or down"; S:484, S:521-529;
   R-9, R-10).
7b. ``spot_classic`` / ``spot_ticks``  NEXT-2 online threshold: SPOT (Siffer
   et al. 2017, Algorithm 1, the method P:297 cites), per observation; and its
   tick-synchronous form (R-23) that the GPU implements.
9b. ``per_metric_mean_difference``  NEXT-1 explanation: MD_j = (1/W) sum_tau
   (x_{tau,j} - m'_{tau,j}) per metric with the explicit D-wide decoder (P:297's
   MD resolved per metric, the root-cause reading of P:512; MD = mean_j MD_j).
9. ``point_adjusted_counts``  NEXT-4 evaluation: point-adjusted TP/FP/FN/TN of
   the flags against anomaly labels ("we adopt a point-adjusted
   approach"; the rule as S:530-533 states it; R-21).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): SPEC worked examples
(tests/golden/spec_examples.json), KL closed forms and a quadrature check of
the Gaussian KL integral, constructed detectors with closed-form outputs
(zero encoder, mean detector, single-tap selector, perfect-reconstruction MD,
and a full-path selector detector whose log-variance head Wlv h and decoder
hidden layer W3 mu are both non-zero),
window locality, an independent scipy GPD MLE and a brute-force likelihood
grid for the tail fit, the exp(1) analytic quantile, and order statistics by
full sort.  Parity unpinned: absolute scores of a *trained* detector (the
paper publishes no weights or data) -- see DESIGN.md.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

STD_FLOOR = 1e-6
Z_CLAMP = 1.0e4           # R-4 (fp16 range; paper silent)


class InsufficientHistory(ValueError):
    """T < W."""


class TooFewExceedances(ValueError):
    """Fewer than 10 peaks above the initial threshold."""


# ----------------------------------------------------------------------------
# 1-3. normalisation and windows
# ----------------------------------------------------------------------------

def series_stats(X: np.ndarray, t_cal_end: int):
    """Mean and population std of each (instance, metric) series over samples
    [0, t_cal_end), two-pass in fp64; std floored at 1e-6 and both rounded to
    fp32 (the precision the detector consumes them in, R-4).

    Returns (mean32 [N, M], std32 [N, M], n_degenerate) where n_degenerate
    counts series whose fp64 std is below the floor ("flagged")."""
    X = np.asarray(X)
    if t_cal_end < 1 or t_cal_end > X.shape[1]:
        raise ValueError("t_cal_end out of range")
    seg = X[:, :t_cal_end, :].astype(np.float64)
    mean = seg.mean(axis=1)
    var = ((seg - mean[:, None, :]) ** 2).mean(axis=1)
    std = np.sqrt(var)
    n_deg = int(np.count_nonzero(std < STD_FLOOR))
    std = np.maximum(std, STD_FLOOR)
    return mean.astype(np.float32), std.astype(np.float32), n_deg


def normalise_x16(X: np.ndarray, mean32: np.ndarray, std32: np.ndarray) -> np.ndarray:
    """Detector input x = fp16_RNE(clamp(fp32((fp32(X - mean)) / std), +-1e4)).

    fp32 arithmetic is IEEE (numpy float32 ops are correctly rounded), so this
    is the exact quantisation the detector is defined on (R-17).  Returned as
    fp64 (every fp16 value is exact in fp64)."""
    X32 = np.asarray(X, dtype=np.float32)
    d = X32 - mean32[:, None, :].astype(np.float32)
    z = d / std32[:, None, :].astype(np.float32)
    z = np.clip(z, np.float32(-Z_CLAMP), np.float32(Z_CLAMP))
    return z.astype(np.float16).astype(np.float64)


def normalise_exact(X: np.ndarray, mean: np.ndarray, std: np.ndarray) -> np.ndarray:
    """fp64 z-score without any rounding (the disclosed 'exact' comparison)."""
    z = (np.asarray(X, np.float64) - np.asarray(mean, np.float64)[:, None, :]) \
        / np.asarray(std, np.float64)[:, None, :]
    return np.clip(z, -Z_CLAMP, Z_CLAMP)


def window(samples: np.ndarray, w: int, end_index: int) -> np.ndarray:
    """SPEC.md core.window: the last w samples ending at end_index (inclusive).
    samples: [T, M]."""
    if w < 1:
        raise ValueError("w must be >= 1")
    if end_index < w - 1 or end_index >= len(samples):
        raise InsufficientHistory(f"need {w} samples ending at {end_index}")
    return samples[end_index - w + 1:end_index + 1]


def window_matrix(x: np.ndarray, W: int, t_begin: int, t_end: int) -> np.ndarray:
    """All windows of every instance ending at t in [t_begin, t_end), each
    flattened time-major (k = tau*M + j, tau = 0 is the oldest sample).
    x: [N, T, M] -> [N, t_end - t_begin, W*M]."""
    N, T, M = x.shape
    if T < W:
        raise InsufficientHistory(f"T={T} < W={W}")
    if not (W - 1 <= t_begin <= t_end <= T):
        raise ValueError("window range out of bounds")
    out = np.empty((N, t_end - t_begin, W * M), dtype=x.dtype)
    for r, t in enumerate(range(t_begin, t_end)):
        out[:, r, :] = x[:, t - W + 1:t + 1, :].reshape(N, W * M)
    return out


# ----------------------------------------------------------------------------
# 4-6. detector forward, KL score, mean difference
# ----------------------------------------------------------------------------

@dataclass
class Detector:
    """Detector parameters in fp64.  Tensor-core operands (W1, Wmu, Wlv, W3) are
    the fp16 rounding of the caller's fp32 values (R-17); biases and the output
    layer stay at the caller's fp32 values."""
    W: int
    M: int
    H: int
    Z: int
    w1: np.ndarray
    b1: np.ndarray
    wmu: np.ndarray
    bmu: np.ndarray
    wlv: np.ndarray
    blv: np.ndarray
    w3: np.ndarray
    b3: np.ndarray
    w4: np.ndarray
    b4: np.ndarray

    @staticmethod
    def from_weights(d: dict) -> "Detector":
        f16 = lambda a: np.asarray(a, np.float32).astype(np.float16).astype(np.float64)
        f64 = lambda a: np.asarray(a, np.float32).astype(np.float64)
        return Detector(int(d["window"]), int(d["n_metrics"]), int(d["hidden"]), int(d["latent"]),
                        f16(d["enc_w1"]), f64(d["enc_b1"]), f16(d["enc_wmu"]), f64(d["enc_bmu"]),
                        f16(d["enc_wlv"]), f64(d["enc_blv"]), f16(d["dec_w1"]), f64(d["dec_b1"]),
                        f64(d["dec_w2"]), f64(d["dec_b2"]))


def encoder(det: Detector, xw: np.ndarray, round_h: bool = False):
    """q_phi(z|m): h = tanh(W1 x + b1); mu = Wmu h + bmu; lv = Wlv h + blv.
    round_h=True is the 'fp16-boundary' debug mode (h rounded to one fp16)."""
    h = np.tanh(xw @ det.w1.T + det.b1)
    if round_h:
        h = h.astype(np.float16).astype(np.float64)
    mu = h @ det.wmu.T + det.bmu
    lv = h @ det.wlv.T + det.blv
    return mu, lv


def kl_score(mu: np.ndarray, lv: np.ndarray) -> np.ndarray:
    """KL(N(mu, diag(exp lv)) || N(0, I)) = 1/2 sum_z (mu^2 + expm1(lv) - lv),
    summed over the last axis; clamped at 0 against rounding."""
    s = 0.5 * np.sum(mu * mu + np.expm1(lv) - lv, axis=-1)
    return np.maximum(s, 0.0)


def decoder(det: Detector, mu: np.ndarray, round_mu: bool = False) -> np.ndarray:
    """p_theta(m|z) mean at z = mu (R-7): m' = W_dec2 tanh(W3 mu + b3) + b_dec2."""
    if round_mu:
        mu = mu.astype(np.float16).astype(np.float64)
    a3 = np.tanh(mu @ det.w3.T + det.b3)
    return a3 @ det.w4.T + det.b4


def mean_difference(xw: np.ndarray, mprime: np.ndarray) -> np.ndarray:
    """MD = mean over all D window entries of (x - m')  (R-8)."""
    return np.mean(xw - mprime, axis=-1)


def score_windows(X: np.ndarray, weights: dict, mean32: np.ndarray, std32: np.ndarray,
                  t_begin: int, t_end: int, mode: str = "x16"):
    """Scores and MD for every window of every instance ending in [t_begin, t_end).

    mode: 'x16' (the contract), 'exact' (x = fp64 z), 'fp16h' (debug: h and mu
    rounded to single fp16).  Returns fp64 arrays [N, t_end - t_begin]."""
    det = weights if isinstance(weights, Detector) else Detector.from_weights(weights)
    X = np.asarray(X)
    N, T, M = X.shape
    if M != det.M:
        raise ValueError("metric count mismatch")
    if T < det.W:
        raise InsufficientHistory(f"T={T} < W={det.W}")
    if mode == "exact":
        x = normalise_exact(X, mean32, std32)
    else:
        x = normalise_x16(X, mean32, std32)
    n = t_end - t_begin
    scores = np.empty((N, n))
    md = np.empty((N, n))
    for i in range(N):                       # one instance at a time bounds memory
        xw = window_matrix(x[i:i + 1], det.W, t_begin, t_end)[0]
        mu, lv = encoder(det, xw, round_h=(mode == "fp16h"))
        scores[i] = kl_score(mu, lv)
        md[i] = mean_difference(xw, decoder(det, mu, round_mu=(mode == "fp16h")))
    return scores, md


def per_metric_mean_difference(X: np.ndarray, weights: dict, mean32: np.ndarray,
                               std32: np.ndarray, t_begin: int, t_end: int,
                               mode: str = "x16") -> np.ndarray:
    """NEXT-1: per-metric MD of every window ending in [t_begin, t_end):
    MD_j = mean over the window's W samples of (x_{tau,j} - m'_{tau,j}), with
    m' the explicit D-wide reconstruction.  [N, n, M] fp64."""
    det = weights if isinstance(weights, Detector) else Detector.from_weights(weights)
    X = np.asarray(X)
    N, T, M = X.shape
    x = normalise_exact(X, mean32, std32) if mode == "exact" else normalise_x16(X, mean32, std32)
    n = t_end - t_begin
    out = np.empty((N, n, M))
    for i in range(N):
        xw = window_matrix(x[i:i + 1], det.W, t_begin, t_end)[0]         # [n, W*M]
        mu, _ = encoder(det, xw)
        resid = xw - decoder(det, mu)                                   # [n, W*M], k = tau*M + j
        out[i] = resid.reshape(n, det.W, M).mean(axis=1)
    return out


def flags(score: np.ndarray, md: np.ndarray, z_q: float) -> np.ndarray:
    """0 = normal; +1 = anomaly with MD >= 0 (overload -> scale up); -1 =
    anomaly with MD < 0 (underload -> scale down).  Strict '>' (R-10), MD = 0
    goes to scale-up (R-9)."""
    anomalous = np.asarray(score) > z_q
    direction = np.where(np.asarray(md) >= 0.0, 1, -1)
    return np.where(anomalous, direction, 0).astype(np.int8)


# ----------------------------------------------------------------------------
# 7. peaks-over-threshold with a Grimshaw GPD MLE
# ----------------------------------------------------------------------------

GRID_POINTS = 64
BISECTIONS = 60


def initial_threshold(scores: np.ndarray, q0: float):
    """t = S_(k), k = floor(q0 * n), 0-based ascending order statistic (R-12)."""
    s = np.sort(np.asarray(scores, dtype=np.float32).astype(np.float64), kind="stable")
    n = s.size
    k = int(math.floor(float(q0) * float(n)))
    if not (0 <= k < n):
        raise ValueError("init_quantile out of range")
    return float(s[k]), k


def peaks(scores: np.ndarray, t: float) -> np.ndarray:
    """Y = {s - t : s > t} in fp64, index order (ties at t excluded, R-12)."""
    s = np.asarray(scores, dtype=np.float32).astype(np.float64)
    return s[s > t] - t


def _w_terms(Y: np.ndarray, x: float):
    """Grimshaw's u(x) = mean 1/(1+xY) and v(x) = 1 + mean log1p(xY), returned
    as P = u - 1 = mean(-xY/(1+xY)) and L = v - 1 = mean(log1p(xY)) so that
    w(x) = u v - 1 = P + L + P L is evaluated without the cancellation of
    forming u v - 1 directly (R-13)."""
    xy = x * Y
    P = float(np.mean(-xy / (1.0 + xy)))
    L = float(np.mean(np.log1p(xy)))
    return P, L


def grimshaw_w(Y: np.ndarray, x: float) -> float:
    P, L = _w_terms(Y, x)
    return P + L + P * L


def grid_points(Y: np.ndarray):
    """The fixed 64-point scan grids of the two root brackets (R-13):
    left  x in (-1/Ymax, 0): x = (-1/Ymax)(1 - theta), theta linear in [1e-8, 1-1e-8];
    right x in (0, 2(Ybar - Ymin)/Ymin^2): log-spaced from 1e-12/Ybar."""
    Ymax, Ymin, Ybar = float(Y.max()), float(Y.min()), float(Y.mean())
    th = np.array([1e-8 + k * ((1.0 - 2e-8) / (GRID_POINTS - 1)) for k in range(GRID_POINTS)])
    left = (-1.0 / Ymax) * (1.0 - th)
    a = 1e-12 / Ybar
    b = 2.0 * (Ybar - Ymin) / (Ymin * Ymin)
    if b > a:
        la, lb = math.log(a), math.log(b)
        right = np.array([math.exp(la + k * ((lb - la) / (GRID_POINTS - 1)))
                          for k in range(GRID_POINTS)])
    else:
        right = np.empty(0)
    return left, right


def _bisect(Y, lo, hi, wlo):
    for _ in range(BISECTIONS):
        mid = 0.5 * (lo + hi)
        wm = grimshaw_w(Y, mid)
        if (wm > 0) == (wlo > 0):
            lo, wlo = mid, wm
        else:
            hi = mid
    return 0.5 * (lo + hi)


def grimshaw_roots(Y: np.ndarray):
    """All sign changes of w on both grids, each bisected 60 times."""
    roots = []
    for grid in grid_points(Y):
        if grid.size == 0:
            continue
        w = [grimshaw_w(Y, float(x)) for x in grid]
        for k in range(len(grid) - 1):
            if w[k] == 0.0:
                roots.append(float(grid[k]))
            elif w[k] * w[k + 1] < 0.0:
                roots.append(_bisect(Y, float(grid[k]), float(grid[k + 1]), w[k]))
        if w[-1] == 0.0:
            roots.append(float(grid[-1]))
    return roots


def gpd_loglik(Y: np.ndarray, gamma: float, sigma: float) -> float:
    """GPD log-likelihood of exceedances Y (Grimshaw / SPOT form)."""
    n = Y.size
    if sigma <= 0:
        return -math.inf
    if gamma == 0.0:
        return -n * math.log(sigma) - float(np.sum(Y)) / sigma
    z = gamma * Y / sigma
    if np.any(1.0 + z <= 0.0):
        return -math.inf
    return -n * math.log(sigma) - (1.0 + 1.0 / gamma) * float(np.sum(np.log1p(z)))


def gpd_grimshaw(Y: np.ndarray):
    """GPD MLE (gamma, sigma) by Grimshaw's reduction.  Candidates: every root
    x of w (gamma = v(x) - 1, sigma = gamma / x) plus the exponential
    candidate (gamma = 0, sigma = Ybar).  Max log-likelihood wins; ties go to
    the smaller |gamma|.  Returns (gamma, sigma, method) with method 0 = GPD
    root, 1 = exponential."""
    Y = np.asarray(Y, dtype=np.float64)
    cands = [(0.0, float(Y.mean()), 1)]
    for x in grimshaw_roots(Y):
        if x == 0.0:
            continue
        _, L = _w_terms(Y, x)
        gamma = L
        if gamma == 0.0:
            continue
        sigma = gamma / x
        if sigma > 0:
            cands.append((gamma, sigma, 0))
    best = None
    best_ll = -math.inf
    for g, s, m in cands:
        if g == 0.0:
            ll = gpd_loglik(Y, 0.0, s)
        else:
            # gamma*Y/sigma == x*Y; evaluate with x to avoid re-rounding
            x = g / s
            ll = -Y.size * math.log(s) - (1.0 + 1.0 / g) * float(np.sum(np.log1p(x * Y)))
        if best is None or ll > best_ll or (ll == best_ll and abs(g) < abs(best[0])):
            best, best_ll = (g, s, m), ll
    return best


def pot_quantile(t: float, gamma: float, sigma: float, n: int, n_peaks: int, q: float) -> float:
    """z_q = t + (sigma/gamma)((q n / N_t)^(-gamma) - 1), or t - sigma ln(q n / N_t)
    when gamma = 0 (Siffer et al. 2017 POT quantile)."""
    r = float(q) * float(n) / float(n_peaks)
    lr = math.log(r)
    if gamma == 0.0:
        return t - sigma * lr
    return t + (sigma / gamma) * math.expm1(-gamma * lr)


def pot_threshold(scores: np.ndarray, init_quantile: float = 0.98, risk_q: float = 1e-3) -> dict:
    """Fit the fleet-wide POT threshold on calibration scores."""
    s = np.asarray(scores).ravel()
    n = s.size
    t, _ = initial_threshold(s, init_quantile)
    Y = peaks(s, t)
    if Y.size < 10:
        raise TooFewExceedances(f"only {Y.size} peaks above t={t}")
    gamma, sigma, method = gpd_grimshaw(Y)
    z_q = pot_quantile(t, gamma, sigma, n, Y.size, risk_q)
    return dict(init_quantile=float(init_quantile), risk_q=float(risk_q), t=t, gamma=gamma,
                sigma=sigma, z_q=z_q, n=n, n_peaks=int(Y.size), method=method)


# ----------------------------------------------------------------------------
# 7b. online SPOT (NEXT-2; P:297 citing Siffer et al. 2017; R-23)
# ----------------------------------------------------------------------------

def spot_classic(init_scores, stream, init_quantile=0.98, risk_q=1e-3):
    """SPOT, Algorithm 1 of the cited paper, one observation at a time:
    calibrate (t, GPD, z_q) on the initial batch with k = n observations; then
    for each x: x > z_q -> anomaly (no update); elif x > t -> add the peak
    x - t, k += 1, refit, recompute z_q; else k += 1.  Returns (flags, z_q
    after every observation)."""
    init = np.asarray(init_scores, dtype=np.float32).ravel()
    thr = pot_threshold(init, init_quantile, risk_q)
    t, z = thr["t"], thr["z_q"]
    Y = list(peaks(init, t))
    k = init.size
    out_f, out_z = [], []
    for x in np.asarray(stream, dtype=np.float32).ravel():
        xd = float(x)
        if xd > z:
            out_f.append(True)
        else:
            out_f.append(False)
            if xd > t:
                Y.append(xd - t)
                k += 1
                g, s_, _ = gpd_grimshaw(np.asarray(Y))
                z = pot_quantile(t, g, s_, k, len(Y), risk_q)
            else:
                k += 1
        out_z.append(z)
    return np.array(out_f), np.array(out_z)


def spot_ticks(init_scores, ticks, init_quantile=0.98, risk_q=1e-3, refit_every=1):
    """Tick-synchronous SPOT (R-23): every score of a tick is flagged against
    the threshold current at the tick's start; then the tick's non-anomalous
    scores above t are added to Y in index order and k grows by the number of
    non-anomalous scores; every `refit_every` ticks the GPD is refitted if a
    peak arrived since the last fit.
    Returns a list of (flags, threshold dict after the tick)."""
    init = np.asarray(init_scores, dtype=np.float32).ravel()
    thr = pot_threshold(init, init_quantile, risk_q)
    t, z = thr["t"], thr["z_q"]
    Y = list(peaks(init, t))
    k = init.size
    res = []
    cur = dict(thr)
    added = 0
    for it, tick in enumerate(ticks):
        x = np.asarray(tick, dtype=np.float32).ravel().astype(np.float64)
        fl = x > z
        normal = x[~fl]
        new = normal[normal > t] - t
        Y.extend(list(new))
        added += int(new.size)
        k += int(normal.size)
        # scheduled refit, only if a peak arrived since the last fit (Algorithm 1
        # refits exactly when a peak is added)
        if (it + 1) % refit_every == 0 and added > 0:
            added = 0
            g, s_, m = gpd_grimshaw(np.asarray(Y))
            z = pot_quantile(t, g, s_, k, len(Y), risk_q)
            cur = dict(t=t, gamma=g, sigma=s_, z_q=z, n=k, n_peaks=len(Y), method=m)
        res.append((fl, dict(cur)))
    return res


# ----------------------------------------------------------------------------
# whole pipeline (c1-sized inputs)
# ----------------------------------------------------------------------------

def detect_pipeline(X: np.ndarray, weights: dict, t_cal_end: int,
                    init_quantile: float = 0.98, risk_q: float = 1e-3, mode: str = "x16"):
    """stats over [0, t_cal_end) -> scores of windows ending in [W-1, t_cal_end)
    -> POT threshold -> scores/MD/flags of windows ending in [t_cal_end, T)."""
    W = int(weights["window"] if isinstance(weights, dict) else weights.W)
    T = np.asarray(X).shape[1]
    mean32, std32, n_deg = series_stats(X, t_cal_end)
    cal, _ = score_windows(X, weights, mean32, std32, W - 1, t_cal_end, mode)
    thr = pot_threshold(cal, init_quantile, risk_q)
    sc, md = score_windows(X, weights, mean32, std32, t_cal_end, T, mode)
    return dict(mean=mean32, std=std32, n_degenerate=n_deg, cal_scores=cal, threshold=thr,
                scores=sc, md=md, flags=flags(sc, md, thr["z_q"]))


# ----------------------------------------------------------------------------
# 9. point-adjusted evaluation (NEXT-4, R-21)
# ----------------------------------------------------------------------------

def point_adjusted_counts(labels, preds):
    """One sequence: (TP, FP, FN, TN) after point adjustment.  S:532-533: "for
    each contiguous true-anomaly segment containing >= 1 predicted point, all
    points of that segment count as correctly predicted; then pointwise"."""
    labels = [bool(v) for v in labels]
    preds = [bool(v) for v in preds]
    if len(labels) != len(preds):
        raise ValueError("length mismatch")
    adjusted = list(preds)
    i, n = 0, len(labels)
    while i < n:
        if labels[i]:
            j = i
            while j < n and labels[j]:
                j += 1
            if any(preds[i:j]):                                  # segment detected
                for k in range(i, j):
                    adjusted[k] = True
            i = j
        else:
            i += 1
    tp = sum(1 for a, p in zip(labels, adjusted) if a and p)
    fp = sum(1 for a, p in zip(labels, adjusted) if not a and p)
    fn = sum(1 for a, p in zip(labels, adjusted) if a and not p)
    tn = sum(1 for a, p in zip(labels, adjusted) if not a and not p)
    return tp, fp, fn, tn


def precision_recall_f1(tp, fp, fn):
    prec = tp / (tp + fp) if tp + fp else 0.0
    rec = tp / (tp + fn) if tp + fn else 0.0
    f1 = 2 * prec * rec / (prec + rec) if prec + rec else 0.0
    return prec, rec, f1


def fleet_point_adjusted_counts(labels: np.ndarray, flags: np.ndarray, t_begin: int):
    """labels [N][T] (!= 0 = anomaly), flags [N][nw] of the windows ending at
    t_begin .. t_begin + nw - 1: counts summed over instances (segments are
    per instance and clipped to the evaluated range)."""
    nw = flags.shape[1]
    tot = [0, 0, 0, 0]
    for i in range(flags.shape[0]):
        c = point_adjusted_counts(labels[i, t_begin:t_begin + nw], flags[i])
        tot = [a + b for a, b in zip(tot, c)]
    return tuple(tot)
