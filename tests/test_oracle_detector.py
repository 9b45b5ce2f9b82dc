"""Pins of the oracle's normalisation, windows, encoder/KL and MD against what
the paper/spec and the mathematics fix (not against the oracle itself)."""
import json
import math
import os
import statistics

import numpy as np
import pytest
from scipy import integrate

from oracle import enova_oracle as O
from paper_2407_09486_b200 import synth
from tests import detectors

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- windows ----
@pytest.mark.parametrize("ex", GOLD["window"], ids=lambda e: e["cite"])
def test_spec_window_examples(ex):
    samples = np.arange(ex["n_samples"] * 3, dtype=np.float64).reshape(ex["n_samples"], 3)
    if "expect_rows" in ex:
        w = O.window(samples, ex["w"], ex["end"])
        assert np.array_equal(w, samples[ex["expect_rows"]])
    else:
        with pytest.raises(O.InsufficientHistory):
            O.window(samples, ex["w"], ex["end"])


def test_window_matrix_is_time_major_oldest_first():
    # X[i, t, j] = 1e4*i + 10*t + j identifies every entry: window ending at t,
    # entry k = tau*M + j must be sample (t - W + 1 + tau, j)
    N, T, M, W = 2, 40, 8, 6
    i, t, j = np.meshgrid(np.arange(N), np.arange(T), np.arange(M), indexing="ij")
    X = 1e4 * i + 10.0 * t + j
    xw = O.window_matrix(X, W, W - 1, T)
    assert xw.shape == (N, T - W + 1, W * M)
    for ii in range(N):
        for r, tend in enumerate(range(W - 1, T)):
            for tau in range(W):
                for jj in range(M):
                    assert xw[ii, r, tau * M + jj] == 1e4 * ii + 10.0 * (tend - W + 1 + tau) + jj


def test_window_count_and_insufficient_history():
    X = np.zeros((1, 31, 8))
    with pytest.raises(O.InsufficientHistory):
        O.window_matrix(X, 32, 31, 31)
    X = np.zeros((1, 100, 8))
    assert O.window_matrix(X, 32, 31, 100).shape[1] == 100 - 32 + 1


# ----------------------------------------------------------- normalisation ----
def test_stats_match_textbook_population_std():
    X = synth.metric_trace(3, 300, 8, seed=11)
    mean32, std32, nd = O.series_stats(X, 200)
    for i in range(3):
        for j in range(8):
            col = [float(v) for v in X[i, :200, j]]
            assert mean32[i, j] == np.float32(statistics.fmean(col))
            assert abs(std32[i, j] - statistics.pstdev(col)) <= 1e-6 * max(1.0, statistics.pstdev(col))
    assert nd == 0


def test_standardised_data_unchanged():
    r = np.random.default_rng(1)
    X = r.standard_normal((2, 500, 8))
    X = (X - X.mean(axis=1, keepdims=True)) / X.std(axis=1, keepdims=True)
    mean, std, _ = O.series_stats(X, 500)
    z = O.normalise_exact(X, mean.astype(np.float64) * 0, std.astype(np.float64) * 0 + 1)
    assert np.max(np.abs(z - X)) < 1e-9
    # and the stats of standardised data are (0, 1) to fp32 rounding
    assert np.max(np.abs(mean)) < 1e-6 and np.max(np.abs(std - 1)) < 1e-6


def test_constant_dimension_zero_and_flagged():
    X = np.random.default_rng(2).standard_normal((2, 100, 8)).astype(np.float32)
    X[1, :, 3] = 7.25
    mean, std, nd = O.series_stats(X, 100)
    assert nd == 1 and std[1, 3] == np.float32(O.STD_FLOOR)
    x = O.normalise_x16(X, mean, std)
    assert np.all(x[1, :, 3] == 0.0)


def test_normalised_mean_zero():
    X = synth.metric_trace(2, 400, 16, seed=3).astype(np.float64)
    mean, std, _ = O.series_stats(X, 400)
    m64 = X.mean(axis=1)
    s64 = X.std(axis=1)
    z = O.normalise_exact(X, m64, s64)
    assert np.max(np.abs(z.mean(axis=1))) < 1e-9


def test_x16_is_fp16_rounding_of_fp32_zscore():
    # x must be representable in fp16 and within half an fp16 ulp (+ fp32
    # rounding) of the exact z-score (R-17)
    X = synth.metric_trace(2, 300, 8, seed=4)
    mean, std, _ = O.series_stats(X, 300)
    x = O.normalise_x16(X, mean, std)
    assert np.array_equal(x, x.astype(np.float16).astype(np.float64))
    z = O.normalise_exact(X, mean, std)
    ulp = np.spacing(np.abs(z).astype(np.float16)).astype(np.float64)
    assert np.all(np.abs(x - z) <= 0.5 * ulp + 1e-6 * np.abs(z) + 1e-7)


# -------------------------------------------------------------------- KL ----
@pytest.mark.parametrize("ex", [e for e in GOLD["score"] if "kl" in e], ids=lambda e: e["cite"])
def test_kl_closed_forms(ex):
    assert O.kl_score(np.array(ex["mu"]), np.array(ex["lv"])) == pytest.approx(ex["kl"], abs=1e-15)


@pytest.mark.parametrize("mu,lv", [(0.3, -0.7), (-1.2, 0.4), (2.0, 1.5), (0.0, -2.0)])
def test_kl_equals_quadrature_of_the_kl_integral(mu, lv):
    # KL(q||p) = integral q(z) log(q(z)/p(z)) dz, q = N(mu, e^lv), p = N(0,1)
    s = math.exp(0.5 * lv)
    q = lambda z: math.exp(-0.5 * ((z - mu) / s) ** 2) / (s * math.sqrt(2 * math.pi))
    lp = lambda z: -0.5 * z * z - 0.5 * math.log(2 * math.pi)
    lq = lambda z: -0.5 * ((z - mu) / s) ** 2 - math.log(s) - 0.5 * math.log(2 * math.pi)
    val, _ = integrate.quad(lambda z: q(z) * (lq(z) - lp(z)), mu - 40 * s, mu + 40 * s, limit=400)
    assert O.kl_score(np.array([mu]), np.array([lv])) == pytest.approx(val, rel=1e-8, abs=1e-12)


def test_kl_nonnegative_random():
    r = np.random.default_rng(5)
    mu = r.standard_normal((10000, 16)) * 3
    lv = r.standard_normal((10000, 16)) * 3
    assert np.all(O.kl_score(mu, lv) >= 0)


# ------------------------------------------------------ constructed detectors ----
W, M, H, Z = 32, 8, 32, 4      # the c1 "tiny" detector (SPEC.md:547 sizes)


def _fp16_trace(N, T, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal((N, T, M)).astype(np.float16).astype(np.float32)


def _unit_stats(N):
    return np.zeros((N, M), np.float32), np.ones((N, M), np.float32)


def test_zero_encoder_gives_constant_score():
    d = detectors.zeros(W, M, H, Z)
    d["enc_bmu"][:] = np.array([0.5, -0.25, 1.0, 0.0], np.float32)
    d["enc_blv"][:] = np.array([0.125, -0.5, 0.0, 1.0], np.float32)
    X = _fp16_trace(2, 200, 6)
    s, _ = O.score_windows(X, d, *_unit_stats(2), W - 1, 200)
    b, l = d["enc_bmu"].astype(np.float64), d["enc_blv"].astype(np.float64)
    expect = 0.5 * sum(b[z] ** 2 + math.expm1(l[z]) - l[z] for z in range(Z))
    assert np.allclose(s, expect, rtol=0, atol=1e-15)


def test_mean_detector_closed_form():
    d = detectors.mean_detector(W, M, H, Z, alpha=4.0, beta=2.0, b1=0.25, bmu0=0.5)
    X = _fp16_trace(1, 120, 7)
    s, md = O.score_windows(X, d, *_unit_stats(1), W - 1, 120)
    for r, t in enumerate(range(W - 1, 120)):
        m = float(np.mean(X[0, t - W + 1:t + 1, :].astype(np.float64)))
        mu0 = 2.0 * math.tanh(4.0 * m + 0.25) + 0.5
        assert s[0, r] == pytest.approx(0.5 * mu0 * mu0, rel=1e-12, abs=1e-15)
        assert md[0, r] == pytest.approx(m, rel=1e-12, abs=1e-15)   # zero decoder -> MD = mean(x)


@pytest.mark.parametrize("tau,j", [(0, 0), (0, 7), (5, 2), (31, 0), (31, 7)])
def test_tap_selector_orientation(tau, j):
    d = detectors.tap_selector(W, M, H, Z, tau, j, a=0.75)
    X = _fp16_trace(1, 100, 8)
    s, _ = O.score_windows(X, d, *_unit_stats(1), W - 1, 100)
    for r, t in enumerate(range(W - 1, 100)):
        v = float(X[0, t - W + 1 + tau, j])          # tau = 0 is the oldest sample
        assert s[0, r] == pytest.approx(0.5 * math.tanh(0.75 * v) ** 2, rel=1e-12, abs=1e-15)


def test_md_zero_on_perfect_reconstruction():
    # "zero score on a perfectly reconstructed window": decoder outputs b_dec2 = c,
    # input window x == c  ->  MD = 0 exactly
    d = detectors.zeros(W, M, H, Z)
    d["dec_b2"][:] = np.float32(0.625)
    X = np.full((1, 80, M), 0.625, np.float32)
    _, md = O.score_windows(X, d, *_unit_stats(1), W - 1, 80)
    assert np.all(md == 0.0)


def test_md_decoder_column_sum_closed_form():
    # W3 = 0, b3 = d -> a3 = tanh(d) constant; W_dec2[:, 0] = 1, rest 0 ->
    # m'_k = tanh(d_0) + b_dec2_k  ->  MD = mean(x) - tanh(d_0) - mean(b_dec2)
    d = detectors.zeros(W, M, H, Z)
    d["dec_b1"][:] = np.float32(0.5)
    d["dec_w2"][:, 0] = np.float32(1.0)
    d["dec_b2"][:] = np.linspace(-1, 1, W * M).astype(np.float16).astype(np.float32)
    X = _fp16_trace(1, 90, 9)
    _, md = O.score_windows(X, d, *_unit_stats(1), W - 1, 90)
    bm = float(np.mean(d["dec_b2"].astype(np.float64)))
    for r, t in enumerate(range(W - 1, 90)):
        m = float(np.mean(X[0, t - W + 1:t + 1, :].astype(np.float64)))
        assert md[0, r] == pytest.approx(m - math.tanh(0.5) - bm, rel=1e-12, abs=1e-14)


def full_path_closed_form(d, xbar, drop_wlv=False, decoder_input="mu"):
    """Scalar restatement of the full_path_detector's score and MD for a window
    of mean xbar (written from the selector structure, not from the oracle's
    matrix code): exercises W1, Wmu, Wlv (lv head) and the decoder's
    hidden layer W3 fed with mu (R-7)."""
    Hh, Zz = d["hidden"], d["latent"]
    D = d["window"] * d["n_metrics"]
    f = lambda a: float(np.float32(a))
    h = [math.tanh(f(d["enc_w1"][k, 0]) * D * xbar + f(d["enc_b1"][k])) for k in range(Hh)]
    mu = [f(d["enc_bmu"][z]) for z in range(Zz)]
    lv = [f(d["enc_blv"][z]) for z in range(Zz)]
    mu[0] += 1.5 * h[2]
    mu[1] += -0.75 * h[5]
    if not drop_wlv:
        lv[0] += 0.5 * h[3]
        lv[2] += -1.25 * h[1]
    score = 0.5 * sum(mu[z] ** 2 + math.expm1(lv[z]) - lv[z] for z in range(Zz))
    lat = mu if decoder_input == "mu" else lv
    a3_4 = math.tanh(0.875 * lat[1] + f(d["dec_b1"][4]))
    a3_0 = math.tanh(f(d["dec_b1"][0]))
    bbar = float(np.mean(d["dec_b2"].astype(np.float64)))
    md = xbar - (0.625 * a3_4 - 0.5 * a3_0) - bbar
    return score, md


@pytest.mark.parametrize("shape", [(32, 8, 32, 4), (16, 16, 64, 8), (8, 8, 128, 16)])
def test_full_path_detector_closed_form(shape):
    """Pins the log-variance head (Wlv h, which every other constructed detector
    zeroes) and the decoder hidden layer W3 fed with mu (not lv, not a sample):
    dropping Wlv h, swapping mu/lv into the decoder, or transposing a selector
    changes the closed form."""
    Wn, Mn, Hn, Zn = shape
    d = detectors.full_path_detector(Wn, Mn, Hn, Zn)
    r = np.random.default_rng(21)
    T = 3 * Wn + 17
    X = (r.standard_normal((1, T, Mn)) * 0.7).astype(np.float16).astype(np.float32)
    s, md = O.score_windows(X, d, np.zeros((1, Mn), np.float32), np.ones((1, Mn), np.float32),
                            Wn - 1, T)
    for r_, t in enumerate(range(Wn - 1, T)):
        xbar = float(np.mean(X[0, t - Wn + 1:t + 1, :].astype(np.float64)))
        es, em = full_path_closed_form(d, xbar)
        assert s[0, r_] == pytest.approx(es, rel=1e-12, abs=1e-14)
        assert md[0, r_] == pytest.approx(em, rel=1e-12, abs=1e-14)


def test_full_path_detector_distinguishes_plausible_mistakes():
    """The closed form separates the mistakes the mean/tap/zero detectors cannot:
    lv = blv (Wlv h dropped) and lv fed to the decoder in place of mu; an oracle
    without Wlv (run here on the detector with Wlv zeroed) misses the pin."""
    d = detectors.full_path_detector(32, 8, 32, 4)
    for xbar in (-1.0, 0.3, 2.0):
        es, em = full_path_closed_form(d, xbar)
        assert abs(es - full_path_closed_form(d, xbar, drop_wlv=True)[0]) > 1e-3
        assert abs(em - full_path_closed_form(d, xbar, decoder_input="lv")[1]) > 1e-3
    d0 = dict(d)
    d0["enc_wlv"] = np.zeros_like(d["enc_wlv"])
    X = np.full((1, 40, 8), 0.5, np.float32)
    s0, _ = O.score_windows(X, d0, np.zeros((1, 8), np.float32), np.ones((1, 8), np.float32), 31, 40)
    assert abs(s0[0, 0] - full_path_closed_form(d, 0.5)[0]) > 1e-3


def test_window_locality_and_permutation_equivariance():
    wts = synth.detector_weights(W, M, H, Z, seed=1)
    X = synth.metric_trace(3, 200, M, seed=2)
    mean, std, _ = O.series_stats(X, 200)
    s0, m0 = O.score_windows(X, wts, mean, std, W - 1, 200)
    X2 = X.copy()
    tstar = 90
    X2[1, tstar, 3] += 10 * std[1, 3]
    s1, m1 = O.score_windows(X2, wts, mean, std, W - 1, 200)
    changed = np.nonzero((s1[1] != s0[1]) | (m1[1] != m0[1]))[0] + (W - 1)
    assert changed.min() >= tstar and changed.max() <= tstar + W - 1
    assert np.array_equal(s1[[0, 2]], s0[[0, 2]])
    perm = [2, 0, 1]
    sp, mp = O.score_windows(X[perm], wts, mean[perm], std[perm], W - 1, 200)
    assert np.array_equal(sp, s0[perm]) and np.array_equal(mp, m0[perm])


def test_outlier_scores_above_normals():         # S:514 (10-sigma outlier)
    d = detectors.mean_detector(W, M, H, Z, alpha=1.0, beta=2.0)
    r = np.random.default_rng(10)
    wins = 0
    trials = 200
    for k in range(trials):
        X = r.standard_normal((1, 2 * W, M)).astype(np.float32)
        X[0, -W:, :] += 10.0
        s, _ = O.score_windows(X, d, *_unit_stats(1), W - 1, 2 * W)
        wins += s[0, -1] > s[0, 0]
    assert wins >= 0.99 * trials


def test_surge_and_drop_flags():
    d = detectors.mean_detector(W, M, H, Z, alpha=1.0, beta=2.0)
    r = np.random.default_rng(12)
    T = 4000
    X = r.standard_normal((1, T, M)).astype(np.float32)
    X[0, 3000:3000 + W, :] += 5.0        # overload: all load metrics +5 sigma
    X[0, 3500:3500 + W, :] -= 3.0        # underload: -3 sigma
    out = O.detect_pipeline(X, d, t_cal_end=2000)
    f = out["flags"][0]
    idx = lambda t: t - 2000
    assert f[idx(3000 + W - 1)] == 1
    assert f[idx(3500 + W - 1)] == -1
    # below threshold -> (false, none); direction != none iff anomaly
    anomalous = out["scores"][0] > out["threshold"]["z_q"]
    assert np.array_equal(f != 0, anomalous)
    # monotone in tau: raising the threshold never adds flags
    for zq in np.linspace(out["threshold"]["z_q"], out["threshold"]["z_q"] * 3, 5):
        f2 = O.flags(out["scores"], out["md"], zq)
        assert np.all((f2 != 0) <= (out["flags"] != 0))


# ------------------------------------------------------------- NEXT-1 pins ----
def _mdm_setup(seed=4):
    from paper_2407_09486_b200 import synth as S
    X = S.metric_trace(2, 300, 8, seed=seed)
    w = S.detector_weights(16, 8, 32, 4, seed=seed)
    mean, std, _ = O.series_stats(X, 150)
    return X, w, mean, std


def test_per_metric_md_averages_to_md():
    """MD = mean_j MD_j (the definitions of P:297's MD and its per-metric split)."""
    X, w, mean, std = _mdm_setup()
    mdm = O.per_metric_mean_difference(X, w, mean, std, 15, 300)
    _, md = O.score_windows(X, w, mean, std, 15, 300)
    assert np.max(np.abs(mdm.mean(axis=-1) - md)) < 1e-12


def test_per_metric_md_closed_form_constant_decoder():
    """Zero decoder weights, b_dec2[tau*M + j] = c_j: m'_{tau,j} = c_j, so
    MD_j = mean_tau x_{tau,j} - c_j -- pins the (tau, j) orientation of the
    time-major flattening."""
    X, w, mean, std = _mdm_setup(5)
    W, M = 16, 8
    c = np.array([0.5, -0.25, 1.0, 0.0, 2.0, -1.5, 0.125, 0.75], np.float32)
    w = dict(w)
    w["dec_w2"] = np.zeros_like(w["dec_w2"])
    w["dec_b2"] = np.tile(c, W).astype(np.float32)
    mdm = O.per_metric_mean_difference(X, w, mean, std, W - 1, 300)
    x = O.normalise_x16(X, mean, std)
    for i in range(2):
        for r, t in enumerate(range(W - 1, 300)):
            ref = x[i, t - W + 1:t + 1, :].mean(axis=0) - c
            assert np.allclose(mdm[i, r], ref, atol=1e-12)


def test_per_metric_md_localises_a_single_metric_surge():
    """A +8 sigma surge on metric j* only (zero decoder) makes MD_{j*} the
    largest per-metric deviation of the windows covering it (P:512 root cause)."""
    X, w, mean, std = _mdm_setup(6)
    w = dict(w)
    w["dec_w2"] = np.zeros_like(w["dec_w2"])
    w["dec_b2"] = np.zeros_like(w["dec_b2"])
    js = 5
    X = X.copy()
    X[0, 200:216, js] = mean[0, js] + 8 * std[0, js]
    mdm = O.per_metric_mean_difference(X, w, mean, std, 215, 216)
    assert int(np.argmax(mdm[0, 0])) == js
