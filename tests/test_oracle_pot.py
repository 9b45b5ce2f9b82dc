"""Pins of the oracle's peaks-over-threshold fit
against analytic quantiles, an independent MLE (scipy) and brute force."""
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import enova_oracle as O
from paper_2407_09486_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def gpd_sample(n, xi, sigma, seed):
    r = np.random.default_rng(seed)
    u = r.uniform(size=n)
    if xi == 0:
        return -sigma * np.log(u)
    return sigma / xi * (u ** (-xi) - 1.0)


def test_exp1_threshold_spec_example():             # S:238, acceptance #9
    ex = GOLD["fit_tail_pot"][0]
    s = np.random.default_rng(0).exponential(1.0, ex["n"]).astype(np.float32)
    thr = O.pot_threshold(s, 0.98, ex["risk_q"])
    assert abs(thr["z_q"] - ex["expect"]) / ex["expect"] < ex["rel_tol"]
    # tighter closed form: t -> ln 50, gamma -> 0, z_q -> ln 1000
    assert thr["t"] == pytest.approx(math.log(50), rel=0.03)
    assert thr["z_q"] == pytest.approx(math.log(1000), rel=0.02)


def test_xi_zero_recovered():
    s = np.random.default_rng(1).exponential(2.0, 200_000).astype(np.float32)
    thr = O.pot_threshold(s, 0.98, 1e-3)
    assert abs(thr["gamma"]) < GOLD["fit_tail_pot"][1]["xi_tol"]


def test_too_few_exceedances():
    s = np.random.default_rng(2).exponential(1.0, 400)
    with pytest.raises(O.TooFewExceedances):
        O.pot_threshold(s, 0.98, 1e-3)      # 400 - 392 - 1 = 7 peaks


def test_initial_threshold_is_the_order_statistic():
    r = np.random.default_rng(3)
    s = np.round(r.exponential(1.0, 50_001), 2).astype(np.float32)   # many ties
    t, k = O.initial_threshold(s, 0.98)
    assert k == math.floor(0.98 * 50_001)
    s64 = s.astype(np.float64)
    assert np.count_nonzero(s64 < t) <= k < np.count_nonzero(s64 <= t)
    Y = O.peaks(s, t)
    assert Y.size == np.count_nonzero(s64 > t) and np.all(Y > 0)


@pytest.mark.parametrize("xi,sigma", [(0.3, 1.0), (-0.2, 2.0), (0.0, 0.5), (0.1, 3.0)])
def test_gpd_mle_matches_scipy_and_truth(xi, sigma):
    Y = gpd_sample(20_000, xi, sigma, seed=int(100 * (xi + 1)))
    g, s, _ = O.gpd_grimshaw(Y)
    c_sp, _, s_sp = stats.genpareto.fit(Y, floc=0)
    ll_ours = O.gpd_loglik(Y, g, s)
    ll_sp = O.gpd_loglik(Y, c_sp, s_sp)
    assert ll_ours >= ll_sp - 1e-6 * abs(ll_sp)          # ours is a true maximum
    assert g == pytest.approx(c_sp, abs=2e-3)
    assert s == pytest.approx(s_sp, rel=2e-3)
    se = 1.0 / math.sqrt(Y.size)                           # sampling error scale
    assert abs(g - xi) < 6 * se * (1 + xi)
    assert abs(s / sigma - 1) < 8 * se


def test_gpd_mle_beats_brute_force_grid():
    Y = gpd_sample(300, 0.2, 1.5, seed=7)
    g, s, _ = O.gpd_grimshaw(Y)
    best = -math.inf
    for gg in np.linspace(-0.6, 1.0, 321):
        for ss in np.exp(np.linspace(math.log(0.3), math.log(6.0), 321)):
            best = max(best, O.gpd_loglik(Y, float(gg), float(ss)))
    assert O.gpd_loglik(Y, g, s) >= best - 1e-9


def test_grimshaw_root_is_a_stationary_point():
    Y = gpd_sample(5000, 0.25, 1.0, seed=8)
    roots = O.grimshaw_roots(Y)
    assert roots
    for x in roots:
        assert abs(O.grimshaw_w(Y, x)) < 1e-10
    # score equations of the GPD log-likelihood vanish at the fitted (gamma, sigma)
    g, s, m = O.gpd_grimshaw(Y)
    assert m == 0
    eps = 1e-6
    dg = (O.gpd_loglik(Y, g + eps, s) - O.gpd_loglik(Y, g - eps, s)) / (2 * eps)
    ds = (O.gpd_loglik(Y, g, s * (1 + eps)) - O.gpd_loglik(Y, g, s * (1 - eps))) / (2 * eps)
    assert abs(dg) < 1e-2 and abs(ds) < 1e-2


def test_threshold_invariants():
    s = synth.score_mixture(400_000, seed=9)
    zs = [O.pot_threshold(s, 0.98, q)["z_q"] for q in (1e-2, 3e-3, 1e-3, 1e-4)]
    t = O.pot_threshold(s, 0.98, 1e-3)["t"]
    assert all(z >= t for z in zs)
    assert all(a <= b for a, b in zip(zs, zs[1:]))


def test_calibration_false_positive_rate():         # S:520 held-out FP <= 2 q
    q = 1e-3
    r = np.random.default_rng(11)
    cal = r.exponential(1.0, 500_000).astype(np.float32)
    held = r.exponential(1.0, 2_000_000).astype(np.float32)
    z = O.pot_threshold(cal, 0.98, q)["z_q"]
    fp = np.mean(held > z)
    assert 0.5 * q <= fp <= 2 * q
    assert math.exp(-z) == pytest.approx(q, rel=0.2)     # analytic tail of exp(1)


def test_quantile_formula_closed_forms():
    # gamma = 0: z = t - sigma ln(q n / N_t);  gamma != 0: GPD tail quantile
    assert O.pot_quantile(1.0, 0.0, 2.0, 1000, 20, 1e-3) == pytest.approx(1.0 - 2.0 * math.log(0.05))
    g, sg = 0.3, 1.5
    z = O.pot_quantile(2.0, g, sg, 10_000, 200, 1e-3)
    # P(S > z) = (N_t/n) * (1 + g (z - t)/sg)^(-1/g) must equal q
    assert (200 / 10_000) * (1 + g * (z - 2.0) / sg) ** (-1 / g) == pytest.approx(1e-3, rel=1e-12)


# ------------------------------------------------------------- NEXT-2 pins ----
def test_spot_ticks_of_one_equal_classic_spot():
    """The tick-synchronous SPOT the GPU implements (R-23) reduces to the cited
    per-observation SPOT (Algorithm 1) when every tick holds one score."""
    rng = np.random.default_rng(2)
    init = rng.exponential(1.0, 5000).astype(np.float32)
    stream = rng.exponential(1.0, 300).astype(np.float32)
    stream[[50, 120, 200]] = 40.0                     # anomalies: never update the model
    f1, z1 = O.spot_classic(init, stream)
    res = O.spot_ticks(init, [[v] for v in stream])
    f2 = np.array([r[0][0] for r in res])
    z2 = np.array([r[1]["z_q"] for r in res])
    assert np.array_equal(f1, f2) and np.array_equal(z1, z2)
    assert f1[[50, 120, 200]].all()


def test_spot_threshold_stays_calibrated_on_a_stationary_stream():
    """exp(1) stream: z_q stays within 10% of ln(1/q) (S:238's bar) while the
    peak set grows, and anomalies (> z_q) are a fraction ~q of the stream."""
    rng = np.random.default_rng(3)
    init = rng.exponential(1.0, 20000).astype(np.float32)
    ticks = [rng.exponential(1.0, 2000).astype(np.float32) for _ in range(10)]
    res = O.spot_ticks(init, ticks, refit_every=2)
    for fl, thr in res:
        assert abs(thr["z_q"] - math.log(1000.0)) < 0.1 * math.log(1000.0)
    frac = np.mean(np.concatenate([fl for fl, _ in res]))
    assert frac < 5e-3
    assert res[-1][1]["n_peaks"] > 400 and res[-1][1]["n"] > 20000
