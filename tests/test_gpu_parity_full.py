"""GPU parity, round 2: exhaustive full-size comparisons and the edge cases the
round-1 suite did not reach.  Every comparison is the CUDA path (through the C
ABI) against the fp64 oracle on the same seeded inputs, with the tolerances of
tests/test_gpu_parity.py (north_star):

* c2 at full size in the bench's launch configuration (Pipeline, CUDA graph):
  EVERY one of the 2 543 872 windows -- calibration and detection scores and
  MD, the threshold fitted on the ORACLE's calibration scores, and the
  oracle's flags outside the R-19 band;
* a c3 instance block, every window;
* the +-1e4 z clamp (R-4) reached the way the paper's case study reaches it: a
  metric constant through the calibration horizon (std floored to 1e-6,
  SPEC.md:491-492) that later steps (GPU memory 90% -> 95%);
* the full-path selector detector (Wlv and W3 non-zero) against its closed form;
* stats for metric counts whose 4-metric groups are not a power of two;
* the 'exact'-oracle deviation (x = fp64 z) reported, not gating.

Results of the exhaustive runs are written to gpurun_out/ as JSON (committed
under profiles/ by the round's validation pass).
"""
import json
import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from oracle import enova_oracle as O
from paper_2407_09486_b200 import synth
from tests import detectors
from tests.test_gpu_parity import MD_ATOL, MD_RTOL, SCORE_ATOL, SCORE_RTOL, cuda

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# z_q fitted on the GPU's scores vs on the oracle's: t is an order statistic of
# scores that carry <= ~5e-6 relative error (measured max 4e-6 at c2) and the
# GPD fit is smooth in them, so the end-to-end z_q differs at that scale; 1e-5
# is 100x inside the north_star flag band (1e-3 z_q).  On IDENTICAL scores the
# bound is 1e-9.
Z_Q_E2E_RTOL = 1e-5
OUT = os.path.join(ROOT, "gpurun_out")


@pytest.fixture(scope="module")
def E():
    from paper_2407_09486_b200 import build as B
    B.build()
    import paper_2407_09486_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def _record(name, payload):
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(payload, f, indent=1, sort_keys=True)


def oracle_windows(X, wts, mean, std, tb, te, mode="x16", workers=None):
    """O.score_windows over every instance, instances spread over threads
    (NumPy releases the GIL in its kernels); same arithmetic as one call."""
    N = X.shape[0]
    workers = workers or max(1, min(16, (os.cpu_count() or 2)))
    sc = np.empty((N, te - tb))
    md = np.empty((N, te - tb))

    def one(i):
        s_, m_ = O.score_windows(X[i:i + 1], wts, mean[i:i + 1], std[i:i + 1], tb, te, mode)
        sc[i], md[i] = s_[0], m_[0]

    with ThreadPoolExecutor(max_workers=workers) as ex:
        list(ex.map(one, range(N)))
    return sc, md


def parity_stats(gpu_sc, gpu_md, ref_sc, ref_md):
    g = np.asarray(gpu_sc, np.float64)
    rel = np.abs(g - ref_sc) / np.maximum(np.abs(ref_sc), 1e-12)
    bad_s = int(np.count_nonzero(np.abs(g - ref_sc) > SCORE_RTOL * np.abs(ref_sc) + SCORE_ATOL))
    dm = np.abs(np.asarray(gpu_md, np.float64) - ref_md)
    bad_m = int(np.count_nonzero(dm > MD_ATOL + MD_RTOL * np.abs(ref_md)))
    return {"windows": int(g.size), "score_rel_max": float(rel.max()),
            "score_rel_p99_99": float(np.percentile(rel, 99.99)),
            "score_rel_median": float(np.median(rel)), "score_violations": bad_s,
            "md_abs_max": float(dm.max()), "md_violations": bad_m}


def band_of(ref_sc, ref_md, z_q):
    return (np.abs(ref_sc - z_q) <= 1e-3 * abs(z_q)) | (
        (np.abs(ref_md) <= 1e-4) & (ref_sc > z_q * (1 - 1e-3)))


# --------------------------------------------------------------- c2 exhaustive ----
def test_c2_full_size_exhaustive(E):
    """Every window of c2 (256 x T=10 000, W=64, benchmark detector) in the bench's
    graph-captured Pipeline against the oracle: stats, calibration and detection
    scores and MD, the threshold (on the oracle's own calibration scores, and on
    the GPU's), and the oracle's flags for every window outside the band."""
    cfg = synth.CONFIGS["c2"]
    N, T, M = cfg["n_instances"], cfg["n_steps"], cfg["n_metrics"]
    W, H, Z = cfg["window"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2)   # bench.py's trace
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    pipe = E.Pipeline(det, N, T, tcal)
    pipe.capture(Xc)
    pipe.replay()
    torch.cuda.synchronize()
    res = pipe.result()
    om, os_, ond = O.series_stats(X, tcal)
    assert np.max(np.abs(res.mean.cpu().numpy().view(np.int32) - om.view(np.int32))) <= 1
    assert np.max(np.abs(res.std.cpu().numpy().view(np.int32) - os_.view(np.int32))) <= 1
    # the oracle on the oracle's stats (x16 contract)
    rc, rcm = oracle_windows(X, wts, om, os_, W - 1, tcal)
    rd, rdm = oracle_windows(X, wts, om, os_, tcal, T)
    cal = parity_stats(res.cal_scores.cpu().numpy(), res.cal_md.cpu().numpy(), rc, rcm)
    dtc = parity_stats(res.scores.cpu().numpy(), res.md.cpu().numpy(), rd, rdm)
    # threshold end to end: oracle fit on the ORACLE's scores vs the GPU fit on its own
    o_ref = O.pot_threshold(rc, 0.98, 1e-3)
    o_gpu = O.pot_threshold(res.cal_scores.cpu().numpy(), 0.98, 1e-3)
    g = res.threshold
    zr = o_ref["z_q"]
    # flags: the oracle's flags (its scores, MD and threshold) outside the band
    fd_ref = O.flags(rd, rdm, zr)
    fc_ref = O.flags(rc, rcm, zr)
    bd, bc = band_of(rd, rdm, zr), band_of(rc, rcm, zr)
    mis_d = int(((res.flags.cpu().numpy() != fd_ref) & ~bd).sum())
    mis_c = int(((res.cal_flags.cpu().numpy() != fc_ref) & ~bc).sum())
    report = {"config": "c2 full size, bench Pipeline (CUDA graph)", "calibration": cal,
              "detection": dtc,
              "threshold": {"gpu_z_q": g["z_q"], "oracle_on_oracle_scores_z_q": zr,
                            "rel_diff_end_to_end": abs(g["z_q"] - zr) / zr,
                            "oracle_on_gpu_scores_z_q": o_gpu["z_q"],
                            "rel_diff_identical_scores": abs(g["z_q"] - o_gpu["z_q"]) / o_gpu["z_q"],
                            "t_equal": g["t"] == o_ref["t"], "n_peaks": g["n_peaks"],
                            "n_peaks_oracle": o_ref["n_peaks"]},
              "flags": {"detection_mismatch_outside_band": mis_d, "detection_in_band": int(bd.sum()),
                        "calibration_mismatch_outside_band": mis_c,
                        "calibration_in_band": int(bc.sum()),
                        "flagged_gpu": int((res.flags.cpu().numpy() != 0).sum()
                                           + (res.cal_flags.cpu().numpy() != 0).sum()),
                        "flagged_oracle": int((fd_ref != 0).sum() + (fc_ref != 0).sum())}}
    _record("c2_exhaustive_parity.json", report)
    assert cal["score_violations"] == 0 and cal["md_violations"] == 0, report
    assert dtc["score_violations"] == 0 and dtc["md_violations"] == 0, report
    assert abs(g["z_q"] - o_gpu["z_q"]) <= 1e-9 * o_gpu["z_q"], report
    assert abs(g["z_q"] - zr) <= Z_Q_E2E_RTOL * zr, report
    assert mis_d == 0 and mis_c == 0, report


def test_c3_instance_block_exhaustive(E):
    """Eight instances of c3's per-GPU shard (T = 50 000), every window against
    the oracle, in the bench's Pipeline launch configuration."""
    cfg = synth.CONFIGS["c3"]
    N, T, M = 8, cfg["n_steps"], cfg["n_metrics"]
    W, H, Z = cfg["window"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2, instance_offset=3 * 512 + 77)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    pipe = E.Pipeline(det, N, T, tcal)
    pipe.capture(Xc)
    pipe.replay()
    torch.cuda.synchronize()
    res = pipe.result()
    om, os_, _ = O.series_stats(X, tcal)
    rc, rcm = oracle_windows(X, wts, om, os_, W - 1, tcal)
    rd, rdm = oracle_windows(X, wts, om, os_, tcal, T)
    cal = parity_stats(res.cal_scores.cpu().numpy(), res.cal_md.cpu().numpy(), rc, rcm)
    dtc = parity_stats(res.scores.cpu().numpy(), res.md.cpu().numpy(), rd, rdm)
    zr = O.pot_threshold(rc, 0.98, 1e-3)["z_q"]
    bd = band_of(rd, rdm, zr)
    mis = int(((res.flags.cpu().numpy() != O.flags(rd, rdm, zr)) & ~bd).sum())
    _record("c3_block_exhaustive_parity.json",
            {"config": "c3 shard block: 8 instances x T=50000", "calibration": cal, "detection": dtc,
             "z_q_gpu": res.threshold["z_q"], "z_q_oracle": zr, "flag_mismatch_outside_band": mis})
    assert cal["score_violations"] == 0 and cal["md_violations"] == 0
    assert dtc["score_violations"] == 0 and dtc["md_violations"] == 0
    assert abs(res.threshold["z_q"] - zr) <= Z_Q_E2E_RTOL * zr
    assert mis == 0


# ----------------------------------------------------------------- clamp ----
@pytest.mark.parametrize("W,M,H,Z", [(64, 16, 128, 16), (32, 8, 32, 4)], ids=lambda v: str(v))
def test_clamp_region_matches_oracle(E, W, M, H, Z):
    """A metric held constant through calibration has its std floored to 1e-6
    (SPEC.md:491-492); a later step (PAPER.md:512's GPU memory 90% -> 95%) gives
    |z| ~ 5e4, clamped to +-1e4 (R-4).  Scores, MD and flags of the whole
    pipeline against the oracle, with the clamp asserted to fire."""
    N, T, tcal = 3, 1400, 700
    X = synth.metric_trace(N, T, M, seed=101 + W)
    j1, j2 = 5 % M, 3 % M
    X[1, :, j1] = np.float32(0.9)
    X[1, 900:, j1] = np.float32(0.95)          # step up after calibration
    X[2, :, j2] = np.float32(0.5)
    X[2, 1000:, j2] = np.float32(0.45)         # step down
    X[0, :, 0] = np.float32(3.0)
    X[0, 800:803, 0] = np.float32(-2.0)        # a 3-sample dip inside the window
    wts = synth.detector_weights(W, M, H, Z, seed=102 + W)
    det = E.PreparedDetector(wts)
    res = E.run_pipeline(cuda(X), det, tcal)
    ref = O.detect_pipeline(X, wts, tcal)
    assert res.n_degenerate == ref["n_degenerate"] == 3
    x = O.normalise_x16(X, ref["mean"], ref["std"])
    assert np.max(x) == 1.0e4 and np.min(x) == -1.0e4, "the clamp must fire"
    st = parity_stats(res.scores.cpu().numpy(), res.md.cpu().numpy(), ref["scores"], ref["md"])
    assert st["score_violations"] == 0 and st["md_violations"] == 0, st
    zq = ref["threshold"]["z_q"]
    assert abs(res.threshold["z_q"] - zq) <= Z_Q_E2E_RTOL * zq
    band = band_of(ref["scores"], ref["md"], zq)
    mism = (res.flags.cpu().numpy() != ref["flags"]) & ~band
    assert not mism.any(), f"{mism.sum()} flag mismatches in the clamp case"
    # the clamped windows are scored (finite) and the steps are detected in direction
    assert np.all(np.isfinite(res.scores.cpu().numpy()))
    clamped = np.abs(x[:, tcal:, :]).max(axis=2) >= 1.0e4          # [N, T - tcal] samples
    assert clamped[1, 900 - tcal] and clamped[2, 1000 - tcal]


# --------------------------------------------------- full-path detector ----
@pytest.mark.parametrize("W,M,H,Z", [(32, 8, 32, 4), (64, 16, 128, 16), (16, 32, 64, 8)],
                         ids=lambda v: str(v))
def test_full_path_detector_closed_form_gpu(E, W, M, H, Z):
    """Wlv and W3 non-zero: the GPU's scores / MD against the scalar closed form
    (tests/test_oracle_detector.full_path_closed_form) and the oracle."""
    from tests.test_oracle_detector import full_path_closed_form
    d = detectors.full_path_detector(W, M, H, Z)
    r = np.random.default_rng(5)
    T = 3 * W + 150
    X = (r.standard_normal((2, T, M)) * 0.7).astype(np.float16).astype(np.float32)
    zeros = torch.zeros((2, M), dtype=torch.float32, device="cuda")
    ones = torch.ones((2, M), dtype=torch.float32, device="cuda")
    sc, md = E.score_windows(cuda(X), E.PreparedDetector(d), zeros, ones)
    sc, md = sc.cpu().numpy(), md.cpu().numpy()
    es = np.empty_like(sc, dtype=np.float64)
    em = np.empty_like(md, dtype=np.float64)
    for i in range(2):
        for k, t in enumerate(range(W - 1, T)):
            es[i, k], em[i, k] = full_path_closed_form(d, float(np.mean(X[i, t - W + 1:t + 1].astype(np.float64))))
    st = parity_stats(sc, md, es, em)
    assert st["score_violations"] == 0 and st["md_violations"] == 0, st
    rs, rmd = O.score_windows(X, d, np.zeros((2, M), np.float32), np.ones((2, M), np.float32), W - 1, T)
    st2 = parity_stats(sc, md, rs, rmd)
    assert st2["score_violations"] == 0 and st2["md_violations"] == 0, st2


# ------------------------------------------------------------ stats, any M ----
@pytest.mark.parametrize("M", [24, 48, 256, 8, 128])
def test_stats_any_metric_count(E, M):
    """M / 4 not a power of two (24, 48) or above a warp (256): the fixed-order
    shared-memory reduction path, against the oracle to <= 1 fp32 ulp."""
    N, T = 5, 2100
    X = synth.metric_trace(N, T, 16, seed=M).astype(np.float32)
    X = np.concatenate([X] * (M // 16 + 1), axis=2)[:, :, :M].copy()
    X += np.arange(M, dtype=np.float32)[None, None, :] * 0.25
    X[3, :, M - 1] = 2.5                               # degenerate
    mean, std, nd = E.compute_stats(cuda(X), 1500)
    om, os_, ond = O.series_stats(X, 1500)
    assert nd == ond
    assert np.max(np.abs(mean.cpu().numpy().view(np.int32) - om.view(np.int32))) <= 1
    assert np.max(np.abs(std.cpu().numpy().view(np.int32) - os_.view(np.int32))) <= 1


def test_m48_detector_rejected(E):
    """M = 48 (metric groups not a power of two) is outside the scoring
    envelope: ENOVA_ERR_UNSUPPORTED, never silently wrong scores."""
    wts = synth.detector_weights(16, 48, 64, 8, seed=48)
    with pytest.raises(E.EnovaError) as ei:
        E.PreparedDetector(wts)
    assert ei.value.name == "ENOVA_ERR_UNSUPPORTED"


# ------------------------------------------------------ a-6 on scored windows ----
def test_flag_scores_async_rule(E):
    r = np.random.default_rng(3)
    n = 100_003                                          # ragged tail of the 16-wide path
    s = r.exponential(1.0, n).astype(np.float32)
    m = r.standard_normal(n).astype(np.float32)
    m[::97] = 0.0                                        # MD = 0 -> scale up (R-9)
    thr = {"z_q": 2.5, "t": 1.0, "gamma": 0.0, "sigma": 1.0, "n": 1, "n_peaks": 10,
           "init_quantile": 0.98, "risk_q": 1e-3, "method": 1}
    f = E.flag_scores_async(cuda(s), cuda(m), E.threshold_to_device(thr)).cpu().numpy()
    assert np.array_equal(f, O.flags(s.astype(np.float64), m.astype(np.float64), 2.5))
    s[5] = np.float32(2.5)                               # exactly at z_q: not anomalous (strict >)
    f = E.flag_scores_async(cuda(s), cuda(m), E.threshold_to_device(thr)).cpu().numpy()
    assert f[5] == 0
    thr["z_q"] = float("nan")                            # failed fit: nothing flagged
    f = E.flag_scores_async(cuda(s), cuda(m), E.threshold_to_device(thr)).cpu().numpy()
    assert not f.any()


def test_explain_invalid_ids_are_nan(E):
    W, M, H, Z = 32, 8, 32, 4
    X = synth.metric_trace(2, 200, M, seed=8)
    wts = synth.detector_weights(W, M, H, Z, seed=8)
    det = E.PreparedDetector(wts)
    mean, std, _ = E.compute_stats(cuda(X), 100)
    nw = 200 - (W - 1)
    ids = torch.tensor([0, -1, 2 * nw, 5, 2 * nw - 1, 10 ** 12], dtype=torch.int64)   # CPU tensor
    mdm, sc, md = E.explain_windows(cuda(X), det, mean, std, ids)
    sc, md, mdm = sc.cpu().numpy(), md.cpu().numpy(), mdm.cpu().numpy()
    bad = [1, 2, 5]
    assert np.all(np.isnan(sc[bad])) and np.all(np.isnan(md[bad])) and np.all(np.isnan(mdm[bad]))
    good = [0, 3, 4]
    ref_s, ref_m = E.score_windows(cuda(X), det, mean, std)
    flat_s, flat_m = ref_s.reshape(-1).cpu().numpy(), ref_m.reshape(-1).cpu().numpy()
    g = np.array([0, 5, 2 * nw - 1])
    assert np.array_equal(sc[good], flat_s[g]) and np.array_equal(md[good], flat_m[g])


# --------------------------------------------------------- exact deviation ----
def test_exact_mode_deviation_reported(E):
    """The disclosed cost of the fp16 input contract (SURVEY §8c 'exact' mode,
    BASELINE.md §2): GPU vs the oracle with x = fp64 z, on c1 (every window) and
    on 16 c2 instances (every window).  Reported in gpurun_out/ -- the gate is
    only that the deviation stays inside the precision study's envelope."""
    import __graft_entry__ as G
    out = {}
    cfg = synth.CONFIGS["c1"]
    W, M, H, Z = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace(cfg["n_instances"], cfg["n_steps"], M, seed=synth.DEFAULT_SEED + 1)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 1)
    tcal = X.shape[1] // 2
    res = E.run_pipeline(cuda(X), E.PreparedDetector(wts), tcal)
    ref = O.detect_pipeline(X, wts, tcal)
    out["c1"] = G.exact_deviation(res.scores.cpu().numpy(), res.flags.cpu().numpy(), X, wts,
                                  ref["mean"], ref["std"], tcal, X.shape[1], ref["threshold"]["z_q"])
    cfg = synth.CONFIGS["c2"]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    X = synth.metric_trace(16, T, M, seed=synth.DEFAULT_SEED + 2)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2
    res = E.run_pipeline(cuda(X), E.PreparedDetector(wts), tcal)
    om, os_, _ = O.series_stats(X, tcal)
    zq = O.pot_threshold(oracle_windows(X, wts, om, os_, W - 1, tcal)[0], 0.98, 1e-3)["z_q"]
    out["c2_16_instances"] = G.exact_deviation(res.scores.cpu().numpy(), res.flags.cpu().numpy(),
                                               X, wts, om, os_, tcal, T, zq)
    out["note"] = ("GPU vs oracle 'exact' mode (x = fp64 z, no fp16 input rounding): relative "
                   "score deviation and flag mismatches outside the R-19 band; reported, not "
                   "gating (the contract is the x16 oracle, SURVEY §8c c-17)")
    _record("exact_deviation.json", out)
    print(json.dumps(out))
    for k in ("c1", "c2_16_instances"):
        # reported, not gating: only sanity (finite, fp16-input scale) and no
        # flag disagreement outside the band
        assert math.isfinite(out[k]["max"]) and out[k]["median"] < 1e-3
        assert out[k]["flag_mismatch_outside_band"] == 0


# ----------------------------------------------- sampled one-pass selection ----
def _sampled_flag(E, ws):
    import ctypes as C
    from paper_2407_09486_b200 import _lib
    L = _lib.lib()
    L.enova_internal_pot_sampled_offset.restype = C.c_int64
    off = int(L.enova_internal_pot_sampled_offset())
    return int(ws.buf[off:off + 4].cpu().numpy().view(np.int32)[0])


@pytest.mark.parametrize("kind", ["mixture", "sorted", "reversed", "ties", "blocks", "negative",
                                  "straddle"])
def test_sampled_selection_exact(E, kind):
    """n >= 2^22 takes the sampled path (strided sample -> lo, ONE full pass
    compacting the candidates, radix passes on the candidates only).  The
    threshold must equal the oracle's on any ordering of the scores --
    including sorted input (every candidate in the last CTAs) and heavy ties
    at the quantile -- with t, n, N_t exact and z_q within 1e-9."""
    n = (1 << 22) + 12345
    r = np.random.default_rng(17)
    s = synth.score_mixture(n, seed=5)
    if kind == "sorted":
        s = np.sort(s)
    elif kind == "reversed":
        s = np.sort(s)[::-1].copy()
    elif kind == "ties":
        s = np.round(s, 1).astype(np.float32)
    elif kind == "negative":      # every score < 0: the scan's general (key) path, lo < 2^31
        s = (s - 60.0).astype(np.float32)
    elif kind == "straddle":      # the quantile just below 0, the tail crossing 0 (-0.0 included)
        s = (s - np.float32(np.quantile(s, 0.985))).astype(np.float32)
        s[::1000] = np.float32(-0.0)
    elif kind == "blocks":        # the tail concentrated in a few contiguous blocks
        s = np.sort(s)
        cut = int(0.97 * n)
        tail = s[cut:].copy()
        s = s[:cut]
        r.shuffle(s)
        pos = [int(p * len(s)) for p in (0.1, 0.55, 0.9)]
        parts = np.array_split(tail, 3)
        for p, t in sorted(zip(pos, parts), reverse=True):
            s = np.concatenate([s[:p], t, s[p:]])
    ws = E.ThresholdWorkspace(n)
    g = E.fit_threshold(cuda(s), 0.98, 1e-3, workspace=ws)
    assert _sampled_flag(E, ws) == 1, "the sampled path should have run"
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert g["t"] == o["t"] and g["n"] == o["n"] and g["n_peaks"] == o["n_peaks"]
    assert abs(g["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])
    # and identical to the full-pass selection of a workspace without candidates
    # (the same scores in a vector too short for sampling would change n: compare
    # the fit inputs instead -- t and N_t above are exact)


def test_sampled_selection_fallback(E):
    """A sample that misjudges the quantile: a score vector whose strided sample
    points all fall on small values while the real 98% quantile is high (values
    at the sample's stride positions are zero) -- the count below lo exceeds k,
    every CTA falls back to the full passes, and the result is still exact."""
    n = 1 << 22
    s = synth.score_mixture(n, seed=9)
    nb = torch.cuda.get_device_properties(0).multi_processor_count
    chunk = ((n + nb - 1) // nb + 3) // 4 * 4
    idx = []
    for b in range(nb):
        b0, b1 = min(n, b * chunk), min(n, b * chunk + chunk)
        ln = b1 - b0
        ns = min(2048, ln)
        idx.extend(b0 + np.arange(ns, dtype=np.int64) * ln // ns)
    idx = np.array(idx)
    s[idx] = 100.0 + np.arange(len(idx), dtype=np.float32) * 1e-3   # every sampled score on top
    ws = E.ThresholdWorkspace(n)
    g = E.fit_threshold(cuda(s), 0.98, 1e-3, workspace=ws)
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert g["t"] == o["t"] and g["n_peaks"] == o["n_peaks"]
    assert abs(g["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])
    assert _sampled_flag(E, ws) == 0, "lo above the quantile must fall back"


def test_binned_fit_deterministic(E):
    """The log2(Y) bins are int64 fixed-point sums (integer atomics, order-free):
    repeated fits of the same scores -- binned grid pass, binned Halley start,
    certifying fp64 passes -- give bit-identical thresholds (a replicated fleet
    fit must agree bit for bit on every rank)."""
    n = 6_000_000
    s = cuda(np.random.default_rng(7).gamma(2.0, 1.0, n).astype(np.float32))
    ws = E.ThresholdWorkspace(n)
    a = [E.fit_threshold(s, 0.98, 1e-3, workspace=ws) for _ in range(3)]
    assert a[0]["n_peaks"] >= 100_000
    for b in a[1:]:
        assert b["z_q"] == a[0]["z_q"] and b["gamma"] == a[0]["gamma"] and b["sigma"] == a[0]["sigma"]


# --------------------------------------------- binned grid pass (N_t >= 1e5) ----
@pytest.mark.parametrize("kind", ["exp", "gpd_heavy", "gpd_neg", "gpd_neg45", "ties", "wide"])
def test_binned_grid_fit_matches_oracle(E, kind):
    """The fit's binned grid pass (k_pot PH_GRIDBIN: N_t >= 1e5 peaks; the non-pole
    grid points evaluated over a log2 histogram of Y with the second-order
    correction, certified signs, uncertain points re-evaluated in fp64 -- R-13)
    on tails of different shapes: exponential, heavy (xi = 0.5), bounded
    (xi = -0.2 and -0.45: roots near the pole, many Y in the hybrid pole points'
    exact high bins), heavy ties, and a tail spanning ~30 octaves.  6M scores ->
    120k peaks; t, N_t and the method exact, z_q within 1e-9 of the oracle's
    fp64 scan + bisection."""
    n = 6_000_000
    r = np.random.default_rng(101)
    if kind == "exp":
        s = r.exponential(1.0, n)
    elif kind == "gpd_heavy":
        s = 2.0 / 0.5 * (r.uniform(size=n) ** -0.5 - 1.0)
    elif kind == "gpd_neg":
        s = 2.0 / -0.2 * (r.uniform(size=n) ** 0.2 - 1.0)
    elif kind == "gpd_neg45":     # strongly bounded: the root near the pole x -> -1/Ymax,
        s = 2.0 / -0.45 * (r.uniform(size=n) ** 0.45 - 1.0)   # many Y in the exact high bins
    elif kind == "ties":
        s = np.round(r.exponential(1.0, n), 3)
    else:   # tail values from ~1e-6 to ~1e3 above t
        s = np.exp(r.normal(0.0, 3.0, n))
    s = s.astype(np.float32)
    g = E.fit_threshold(cuda(s), 0.98, 1e-3)
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert o["n_peaks"] >= 100_000            # the binned path runs
    assert g["t"] == o["t"] and g["n_peaks"] == o["n_peaks"]
    assert g["method"] == o["method"]
    assert abs(g["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"]), (g, o)
