"""Pins of the training oracle (NEXT-3, Eq. 9; oracle/enova_train_oracle.py)
against what the paper/spec and the mathematics fix -- not against itself."""
import math

import numpy as np
import pytest
from numpy.polynomial.hermite_e import hermegauss
from scipy import stats

from oracle import enova_train_oracle as T
from paper_2407_09486_b200 import synth


def _setup(W=2, M=8, H=32, Z=4, B=3, seed=0):
    w = synth.detector_weights(W, M, H, Z, seed=seed)
    p = T.as_params(w)
    r = np.random.default_rng(seed + 1)
    x = r.standard_normal((B, W * M)) * 0.8
    eps = r.standard_normal((B, Z))
    return w, p, x, eps


def test_gradient_matches_central_finite_differences():
    """dL/dtheta for EVERY parameter against central finite differences
    on a 3-row dataset, <= 1e-4 relative (mixed labels, beta != 0, 1)."""
    w, p, x, eps = _setup(B=3, seed=3)
    labels = np.array([1.0, -1.0, 1.0])
    beta = 0.37
    _, g, _, _ = T.elbo_grad(p, x, labels, eps, beta)
    h = 1e-6
    for name in T.PARAMS:
        flat = p[name].reshape(-1)
        gg = g[name].reshape(-1)
        fd = np.empty_like(flat)
        for i in range(flat.size):
            old = flat[i]
            flat[i] = old + h
            lp = T.elbo(p, x, labels, eps, beta)[0]
            flat[i] = old - h
            lm = T.elbo(p, x, labels, eps, beta)[0]
            flat[i] = old
            fd[i] = (lp - lm) / (2 * h)
        err = np.linalg.norm(gg - fd) / max(np.linalg.norm(fd), 1e-300)
        assert err <= 1e-4, f"{name}: relative gradient error {err:.2e}"


def _plain_elbo_independent(p, x, eps):
    """Plain VAE ELBO, coded independently of the oracle: the expectation term
    as scipy Gaussian log-densities of x under N(m'(z), I), the KL term as a
    Gauss-Hermite quadrature of E_q[log q(z) - log p(z)] per latent dimension."""
    h = np.tanh(x @ p["enc_w1"].T + p["enc_b1"])
    mu = h @ p["enc_wmu"].T + p["enc_bmu"]
    lv = h @ p["enc_wlv"].T + p["enc_blv"]
    s = np.sqrt(np.exp(lv))
    z = mu + s * eps
    mp = np.tanh(z @ p["dec_w1"].T + p["dec_b1"]) @ p["dec_w2"].T + p["dec_b2"]
    logp = stats.norm.logpdf(x, loc=mp, scale=1.0).sum(axis=1)
    nodes, wts = hermegauss(80)                 # E_{u~N(0,1)} f(u) = sum w f(u) / sqrt(2 pi)
    kl = np.zeros(x.shape[0])
    for i in range(x.shape[0]):
        for d in range(mu.shape[1]):
            u = mu[i, d] + s[i, d] * nodes
            f = stats.norm.logpdf(u, mu[i, d], s[i, d]) - stats.norm.logpdf(u, 0.0, 1.0)
            kl[i] += np.sum(wts * f) / math.sqrt(2 * math.pi)
    return float(np.mean(logp - kl))


def test_all_normal_beta1_equals_plain_elbo():
    """with every label +1 and beta = 1, Eq. 9 is the standard ELBO (1e-9)."""
    w, p, x, eps = _setup(B=5, seed=7)
    L, _, _ = T.elbo(p, x, np.ones(5), eps, 1.0)
    ref = _plain_elbo_independent(p, x, eps)
    assert L == pytest.approx(ref, rel=1e-9, abs=1e-9)


def test_anomaly_rows_have_no_kl_term():
    """the (1 + l)/2 weight -- an anomaly row (l = -1) contributes no KL
    term, so with only anomaly rows L does not depend on beta and equals
    -mean(log p); the encoder's KL gradient vanishes for them."""
    w, p, x, eps = _setup(B=4, seed=9)
    lab = -np.ones(4)
    L0, logp, _ = T.elbo(p, x, lab, eps, 0.0)
    L1, _, _ = T.elbo(p, x, lab, eps, 0.9)
    assert L0 == L1 == pytest.approx(-np.mean(logp), rel=1e-15)
    _, g0, _, _ = T.elbo_grad(p, x, lab, eps, 0.0)
    _, g1, _, _ = T.elbo_grad(p, x, lab, eps, 0.9)
    for k in T.PARAMS:
        assert np.array_equal(g0[k], g1[k])


def test_label_sign_flips_reconstruction_term():
    """Eq. 9: l_i multiplies the expectation term -- flipping a row's label from
    +1 to -1 flips the sign of its log-likelihood contribution."""
    w, p, x, eps = _setup(B=1, seed=11)
    Lp, logp, kl = T.elbo(p, x, np.array([1.0]), eps, 0.25)
    Ln, _, _ = T.elbo(p, x, np.array([-1.0]), eps, 0.25)
    assert Lp == pytest.approx(logp[0] - 0.25 * kl[0], rel=1e-14)
    assert Ln == pytest.approx(-logp[0], rel=1e-14)


def test_beta_pi_hand_computed_sequence():
    """R-24 (P:288 'beta(k) from PI control', S:548 constants): e = KL - setpoint,
    I += e while beta is unclamped, beta = clamp(Kp e + Ki I, 0, 1)."""
    pi = T.BetaPI(setpoint=2.0, kp=0.01, ki=0.001)
    seq = [12.0, 12.0, 1.0, 150.0, 150.0, 2.0]
    got = [pi.update(v) for v in seq]
    # k=0: e=10, I=10 -> 0.1 + 0.01 = 0.11
    # k=1: e=10, I=20 -> 0.1 + 0.02 = 0.12
    # k=2: e=-1, I=19 -> -0.01 + 0.019 = 0.009
    # k=3: e=148, I=167 -> 1.48 + 0.167 > 1 -> clamp 1, I held at 19
    # k=4: same -> 1 (I stays 19)
    # k=5: e=0, I=19 -> 0.019
    exp = [0.11, 0.12, 0.009, 1.0, 1.0, 0.019]
    assert got == pytest.approx(exp, abs=1e-15)
    pi2 = T.BetaPI(setpoint=2.0)
    assert pi2.update(-50.0) == 0.0 and pi2.integral == 0.0    # clamped low, no windup


def test_adam_first_step_is_signed_lr():
    """Bias-corrected Adam: the first step moves every parameter by
    lr * g / (|g| + eps) (ascent direction)."""
    p = {"a": np.array([1.0, -2.0, 0.5])}
    g = {"a": np.array([3.0, -1e-3, 0.0])}
    opt = T.AdamAscent(p, lr=1e-3, eps=1e-8)
    opt.step(p, g)
    exp = np.array([1.0, -2.0, 0.5]) + 1e-3 * g["a"] / (np.abs(g["a"]) + 1e-8)
    assert np.allclose(p["a"], exp, rtol=0, atol=1e-15)


def test_training_curve_non_decreasing():
    """the training-set ELBO of normal rows rises over training (100-step
    moving average non-decreasing within stochastic tolerance) on synthetic
    windows."""
    W, M, H, Z = 2, 8, 32, 4
    X, lab = synth.spec_benchmark(4, 3000, seed=5)
    x = X[:, 1:, :].reshape(-1, M)
    win = np.concatenate([X[:, :-1, :], X[:, 1:, :]], axis=2).reshape(-1, W * M)
    labels = np.where(lab[:, 1:].reshape(-1) != 0, -1.0, 1.0)
    normal = labels > 0
    win, labels = win[normal], labels[normal]
    r = np.random.default_rng(2)
    batch, steps = 64, 1200
    order = np.concatenate([r.permutation(len(win)) for _ in range(steps * batch // len(win) + 1)])
    order = order[:steps * batch]
    eps = r.standard_normal((steps * batch, Z))
    w = synth.detector_weights(W, M, H, Z, seed=5)
    _, hist = T.train(w, win, labels, order, eps, batch, lr=2e-3)
    L = np.array([h[3] for h in hist])          # plain ELBO of the normal rows
    ma = np.convolve(L, np.ones(100) / 100, mode="valid")
    assert ma[-1] > ma[0] + 1.0
    # non-decreasing within stochastic tolerance: no 100-step average falls more
    # than 1 nat below the running maximum of the earlier ones
    assert np.all(ma >= np.maximum.accumulate(ma) - 1.0)


def test_spec_benchmark_point_adjusted_f1():
    """S:544 / S:701 at the oracle level: Eq. 9 training (tests/train_bench.py
    schedule: 30 epochs, batch 64, Adam 3e-3, PI beta) on the synthetic benchmark's contaminated calibration
    half with 50% of the anomaly segments labelled, POT on the normal
    calibration windows, then detection on the second half: point-adjusted
    F1 >= 0.90 and a held-out normal false-positive rate <= 2 q."""
    from oracle import enova_oracle as O
    from tests import train_bench as TB
    X, lab, tl = TB.data()
    mean, std, _ = O.series_stats(X, TB.TCAL)
    x = O.normalise_x16(X, mean, std)
    win = O.window_matrix(x, TB.W, TB.W - 1, TB.TCAL).reshape(-1, TB.W * TB.M)
    l = TB.train_labels(tl)
    order, steps = TB.schedule(len(win), TB.EPOCHS, TB.BATCH)
    w0 = synth.detector_weights(TB.W, TB.M, TB.H, TB.Z, seed=TB.SEED)
    p, hist = T.train(w0, win, l, order, TB.noise(steps, TB.BATCH), TB.BATCH, lr=TB.LR)
    wts = dict(w0)
    wts.update({k: p[k].astype(np.float32) for k in T.PARAMS})
    cal, _ = O.score_windows(X, wts, mean, std, TB.W - 1, TB.TCAL)
    thr = O.pot_threshold(cal[TB.normal_cal_mask(lab)], 0.98, 1e-3)
    sc, md = O.score_windows(X, wts, mean, std, TB.TCAL, TB.T)
    ev = TB.evaluate(O.flags(sc, md, thr["z_q"]), lab)
    assert ev["f1"] >= 0.90, ev
    assert ev["fp_rate_normal"] <= ev["fp_rate_bound"], ev
