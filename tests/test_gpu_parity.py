"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded inputs.  Tolerances (north_star):
  scores  |d| <= 1e-3 |ref| + 1e-6         (every window)
  md      |d| <= 1e-4 + 1e-3 |ref|
  flags   identical outside |score_ref - z_q| <= 1e-3 z_q and |md_ref| <= 1e-4
  stats   bitwise (fp64-accumulated, rounded to fp32) up to 1 fp32 ulp
  z_q     |d| <= 1e-9 z_q on identical scores
"""
import math

import numpy as np
import pytest
import torch

from oracle import enova_oracle as O
from paper_2407_09486_b200 import synth
from tests import detectors

pytestmark = pytest.mark.gpu

SCORE_RTOL, SCORE_ATOL = 1e-3, 1e-6
MD_ATOL, MD_RTOL = 1e-4, 1e-3


@pytest.fixture(scope="module")
def E():
    from paper_2407_09486_b200 import build as B
    B.build()
    import paper_2407_09486_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def assert_scores(gpu, ref, what="scores"):
    gpu = np.asarray(gpu, np.float64)
    err = np.abs(gpu - ref)
    tol = SCORE_RTOL * np.abs(ref) + SCORE_ATOL
    bad = np.count_nonzero(err > tol)
    assert bad == 0, f"{what}: {bad} windows outside tolerance; max rel {np.max(err / (np.abs(ref) + 1e-12)):.3e}"
    return float(np.max(err / (np.abs(ref) + 1e-12)))


def assert_md(gpu, ref):
    err = np.abs(np.asarray(gpu, np.float64) - ref)
    bad = np.count_nonzero(err > MD_ATOL + MD_RTOL * np.abs(ref))
    assert bad == 0, f"md: {bad} windows outside tolerance; max abs {err.max():.3e}"


def assert_flags(gpu_flags, ref_flags, ref_scores, ref_md, z_q):
    band = (np.abs(ref_scores - z_q) <= 1e-3 * abs(z_q)) | (
        (np.abs(ref_md) <= 1e-4) & (ref_scores > z_q * (1 - 1e-3)))
    g = np.asarray(gpu_flags)
    mism = (g != ref_flags) & ~band
    assert not mism.any(), f"{mism.sum()} flag mismatches outside the band"
    return int(band.sum())


# ------------------------------------------------------------------ a-1 ----
def test_stats_match_oracle(E):
    X = synth.metric_trace(8, 3000, 16, seed=21)
    X[5, :, 7] = 3.5                                    # degenerate series
    mean, std, nd = E.compute_stats(cuda(X), 1500)
    om, os_, ond = O.series_stats(X, 1500)
    gm, gs = mean.cpu().numpy(), std.cpu().numpy()
    assert nd == ond == 1
    assert np.max(np.abs(gm.view(np.int32) - om.view(np.int32))) <= 1
    assert np.max(np.abs(gs.view(np.int32) - os_.view(np.int32))) <= 1


def test_stats_nonfinite_rejected(E):
    X = synth.metric_trace(2, 300, 8, seed=22)
    X[1, 100, 2] = np.nan
    with pytest.raises(E.EnovaError) as ei:
        E.compute_stats(cuda(X), 300)
    assert ei.value.name == "ENOVA_ERR_NONFINITE"
    X[1, 100, 2] = 0.0
    X[0, 250, 0] = np.inf          # outside the horizon [0, 200): accepted
    E.compute_stats(cuda(X), 200)


# ------------------------------------------------------------ a-2..a-5 ----
SHAPES = [  # (W, M, H, Z)
    (32, 8, 32, 4),       # c1 "tiny" (SPEC sizes)
    (64, 16, 128, 16),    # c2..c5 benchmark detector
    (16, 32, 64, 8),
    (8, 64, 32, 16),
    (64, 16, 64, 5),
    (2, 8, 32, 1),
    (10, 16, 128, 9),
    (128, 32, 128, 16),   # W1 half > 128 KB: W1-streaming kernel
]


@pytest.mark.parametrize("W,M,H,Z", SHAPES, ids=lambda v: str(v))
def test_scores_match_oracle_shapes(E, W, M, H, Z):
    N, T = 3, 700 + W                          # ragged last tile per instance
    X = synth.metric_trace(N, T, M, seed=W * 1000 + M + H + Z)
    wts = synth.detector_weights(W, M, H, Z, seed=H + Z)
    mean, std, _ = O.series_stats(X, T // 2)
    det = E.PreparedDetector(wts)
    for tb, te in ((W - 1, T), (W - 1 + 37, T - 11), (T - 5, T), (W + 3, W + 3)):
        sc, md = E.score_windows(cuda(X), det, cuda(mean), cuda(std), tb, te)
        rs, rmd = O.score_windows(X, wts, mean, std, tb, te)
        assert sc.shape == (N, te - tb)
        if te > tb:
            assert_scores(sc.cpu().numpy(), rs)
            assert_md(md.cpu().numpy(), rmd)


def test_streaming_kernel_matches_oracle_c2_slice(E):
    """The W1-streaming kernel (forced with enova_set_score_kernel) on the
    benchmark detector."""
    X = synth.metric_trace(4, 800, 16, seed=9)
    w = synth.detector_weights(64, 16, 128, 16, seed=9)
    m, s, _ = O.series_stats(X, 400)
    d = E.PreparedDetector(w)
    with E.force_score_kernel("stream"):
        sc, md = E.score_windows(cuda(X), d, cuda(m), cuda(s))
    rs, rmd = O.score_windows(X, w, m, s, 63, 800)
    assert_scores(sc.cpu().numpy(), rs, "stream-kernel scores")
    assert_md(md.cpu().numpy(), rmd)


ROW_SHAPES = [(32, 8, 32, 4), (64, 16, 128, 16), (64, 16, 64, 5), (2, 8, 32, 1), (10, 16, 128, 9),
              (24, 8, 64, 16)]


@pytest.mark.parametrize("W,M,H,Z", ROW_SHAPES, ids=lambda v: str(v))
def test_row_kernel_matches_oracle_and_pair_kernel(E, W, M, H, Z):
    """The instance-batched row kernel (forced with enova_set_score_kernel) on
    multi-window ranges with ragged tiles: within tolerance of
    the oracle, and BIT-identical to the windowed CTA-pair kernel (same epilogue
    arithmetic and window-sum association), so streamed and batch scores agree."""
    N, T = 5, 300 + W
    seed = 7 * W + M + H + Z
    X = synth.metric_trace(N, T, M, seed=seed)
    wts = synth.detector_weights(W, M, H, Z, seed=seed)
    mean, std, _ = O.series_stats(X, T // 2)
    tb, te = W - 1 + 3, T - 2
    det = E.PreparedDetector(wts)
    sc_p, md_p = E.score_windows(cuda(X), det, cuda(mean), cuda(std), tb, te)
    fl_p = E.detect(cuda(X), det, cuda(mean), cuda(std), {"z_q": 2.0}, tb, te)
    with E.force_score_kernel("rows"):
        sc_r, md_r = E.score_windows(cuda(X), det, cuda(mean), cuda(std), tb, te)
        fl_r = E.detect(cuda(X), det, cuda(mean), cuda(std), {"z_q": 2.0}, tb, te)
    got = dict(sc=sc_r.cpu().numpy(), md=md_r.cpu().numpy(), fl=fl_r.cpu().numpy())
    rs, rmd = O.score_windows(X, wts, mean, std, tb, te)
    assert_scores(got["sc"], rs, "row-kernel scores")
    assert_md(got["md"], rmd)
    assert np.array_equal(got["sc"], sc_p.cpu().numpy()), "row kernel scores != pair kernel scores"
    assert np.array_equal(got["md"], md_p.cpu().numpy()), "row kernel md != pair kernel md"
    assert np.array_equal(got["fl"], fl_p.cpu().numpy())


def test_strided_instances_and_large_values(E):
    W, M, H, Z = 64, 16, 128, 16
    N, T = 4, 900
    X = synth.metric_trace(N, T, M, seed=5)
    X[2, 300:340, :] *= 50.0                    # far outliers -> clamp region / saturation
    pad = np.zeros((N, T * M + 64), np.float32)
    pad[:, :T * M] = X.reshape(N, -1)
    Xt = cuda(pad)[:, :T * M].view(N, T, M)      # ld_instance = T*M + 64
    wts = synth.detector_weights(W, M, H, Z)
    mean, std, _ = O.series_stats(X, 450)
    det = E.PreparedDetector(wts)
    sc, md = E.score_windows(Xt, det, cuda(mean), cuda(std))
    rs, rmd = O.score_windows(X, wts, mean, std, W - 1, T)
    assert_scores(sc.cpu().numpy(), rs)
    assert_md(md.cpu().numpy(), rmd)


def test_constructed_detectors(E):
    W, M, H, Z = 32, 8, 32, 4
    r = np.random.default_rng(3)
    X = r.standard_normal((2, 300, M)).astype(np.float16).astype(np.float32)
    zeros_m, ones_s = cuda(np.zeros((2, M), np.float32)), cuda(np.ones((2, M), np.float32))
    d = detectors.zeros(W, M, H, Z)
    d["enc_bmu"][:] = [0.5, -0.25, 1.0, 0.0]
    d["enc_blv"][:] = [0.125, -0.5, 0.0, 1.0]
    sc, _ = E.score_windows(cuda(X), E.PreparedDetector(d), zeros_m, ones_s)
    expect = 0.5 * sum(b * b + math.expm1(l) - l for b, l in zip(d["enc_bmu"], d["enc_blv"]))
    assert np.allclose(sc.cpu().numpy(), expect, rtol=1e-6, atol=0)
    for tau, j in ((0, 0), (5, 3), (31, 7)):
        d = detectors.tap_selector(W, M, H, Z, tau, j, a=0.75)
        sc, _ = E.score_windows(cuda(X), E.PreparedDetector(d), zeros_m, ones_s)
        t = np.arange(W - 1, 300)
        v = X[:, t - W + 1 + tau, j].astype(np.float64)
        assert_scores(sc.cpu().numpy(), 0.5 * np.tanh(0.75 * v) ** 2, f"tap {tau},{j}")
    d = detectors.zeros(W, M, H, Z)
    d["dec_b2"][:] = 0.625
    Xc = np.full((1, 80, M), 0.625, np.float32)
    _, md = E.score_windows(cuda(Xc), E.PreparedDetector(d), zeros_m[:1], ones_s[:1])
    assert np.all(md.cpu().numpy() == 0.0)           # perfect reconstruction -> MD = 0


# ------------------------------------------------------------ a-7..a-9 ----
@pytest.mark.parametrize("kind,n", [("mixture", 2_000_000), ("exp", 100_000), ("gpd_neg", 300_000),
                                    ("ties", 50_001), ("small", 600)])
def test_threshold_on_identical_scores(E, kind, n):
    r = np.random.default_rng(7)
    if kind == "mixture":
        s = synth.score_mixture(n, seed=77)
    elif kind == "exp":
        s = r.exponential(1.0, n).astype(np.float32)
    elif kind == "gpd_neg":
        s = (2.0 / -0.2 * (r.uniform(size=n) ** 0.2 - 1.0)).astype(np.float32)
    elif kind == "ties":
        s = np.round(r.exponential(1.0, n), 2).astype(np.float32)
    else:
        s = r.exponential(1.0, n).astype(np.float32)
    g = E.fit_threshold(cuda(s), 0.98, 1e-3)
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert g["t"] == o["t"]
    assert g["n"] == o["n"] and g["n_peaks"] == o["n_peaks"]
    assert g["method"] == o["method"]
    assert abs(g["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])
    assert abs(g["gamma"] - o["gamma"]) <= 1e-7 * max(1.0, abs(o["gamma"]))
    assert abs(g["sigma"] - o["sigma"]) <= 1e-9 * o["sigma"]


def test_threshold_too_few_exceedances(E):
    s = np.random.default_rng(1).exponential(1.0, 400).astype(np.float32)
    with pytest.raises(E.EnovaError) as ei:
        E.fit_threshold(cuda(s), 0.98, 1e-3)
    assert ei.value.name == "ENOVA_ERR_TOO_FEW_EXCEEDANCES"


def test_threshold_c5_full_size(E):
    n = synth.CONFIGS["c5"]["n_scores"]
    s = synth.score_mixture(n)
    g = E.fit_threshold(cuda(s), 0.98, 1e-3)
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert g["t"] == o["t"] and g["n_peaks"] == o["n_peaks"]
    assert abs(g["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])


def test_comm_world1_matches_single_gpu(E):
    s = synth.score_mixture(500_000, seed=3)
    comm = E.Comm.create(0, 1, torch.cuda.current_device())
    try:
        a = E.fit_threshold(cuda(s), 0.98, 1e-3, comm=comm)
    finally:
        comm.destroy()
    b = E.fit_threshold(cuda(s), 0.98, 1e-3)
    assert a == b


# ------------------------------------------------------ whole path ----
def test_c1_pipeline_matches_oracle(E):
    cfg = synth.CONFIGS["c1"]
    W, M, H, Z = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace(cfg["n_instances"], cfg["n_steps"], M, seed=synth.DEFAULT_SEED + 1)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 1)
    T = X.shape[1]
    tcal = T // 2
    det = E.PreparedDetector(wts)
    res = E.run_pipeline(cuda(X), det, tcal)
    ref = O.detect_pipeline(X, wts, tcal)
    assert np.array_equal(res.mean.cpu().numpy(), ref["mean"])
    assert_scores(res.cal_scores.cpu().numpy(), ref["cal_scores"], "calibration scores")
    assert_scores(res.scores.cpu().numpy(), ref["scores"])
    assert_md(res.md.cpu().numpy(), ref["md"])
    # end to end: threshold fitted on GPU scores vs on oracle scores
    assert res.threshold["n"] == ref["threshold"]["n"]
    assert abs(res.threshold["z_q"] - ref["threshold"]["z_q"]) <= 1e-3 * ref["threshold"]["z_q"]
    assert_flags(res.flags.cpu().numpy(), ref["flags"], ref["scores"], ref["md"],
                 ref["threshold"]["z_q"])


def test_c2_full_size_sampled(E):
    """c2 at full size in the bench's launch configuration; the oracle checks a
    seeded sample of windows one by one, and flags are checked everywhere."""
    cfg = synth.CONFIGS["c2"]
    N, T, M = cfg["n_instances"], cfg["n_steps"], cfg["n_metrics"]
    W, H, Z = cfg["window"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace(N, T, M, seed=synth.DEFAULT_SEED + 2)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2
    det = E.PreparedDetector(wts)
    res = E.run_pipeline(cuda(X), det, tcal)
    mean32, std32 = res.mean.cpu().numpy(), res.std.cpu().numpy()
    om, os_, _ = O.series_stats(X, tcal)
    assert np.max(np.abs(mean32.view(np.int32) - om.view(np.int32))) <= 1
    r = np.random.default_rng(11)
    gs, gmd = res.scores.cpu().numpy(), res.md.cpu().numpy()
    inst = r.integers(0, N, 400)
    for i in np.unique(inst):
        ts = np.sort(r.choice(np.arange(tcal, T), 4, replace=False))
        for t in ts:
            rs, rmd = O.score_windows(X[i:i + 1], wts, om[i:i + 1], os_[i:i + 1], t, t + 1)
            assert_scores(gs[i, t - tcal:t - tcal + 1], rs[0], f"inst {i} t {t}")
            assert_md(gmd[i, t - tcal:t - tcal + 1], rmd[0])
    # fleet threshold from the GPU's own calibration scores equals the oracle fit of them
    o = O.pot_threshold(res.cal_scores.cpu().numpy(), 0.98, 1e-3)
    assert abs(res.threshold["z_q"] - o["z_q"]) <= 1e-9 * o["z_q"]
    # flags are exactly the rule applied to the GPU's scores/MD
    f = O.flags(gs, gmd, res.threshold["z_q"])
    assert np.array_equal(res.flags.cpu().numpy(), f)


def test_detect_invariants(E):
    W, M, H, Z = 64, 16, 128, 16
    X = synth.metric_trace(6, 2500, M, seed=31)
    wts = synth.detector_weights(W, M, H, Z, seed=31)
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc, 1250)
    sc, md = E.score_windows(Xc, det, mean, std)
    s_np = sc.cpu().numpy()
    zq = float(np.quantile(s_np, 0.99))
    prev = None
    for z in (zq, zq * 1.1, zq * 1.5):
        f = E.detect(Xc, det, mean, std, {"z_q": z}).cpu().numpy()
        assert np.array_equal(f != 0, s_np > z)                    # direction != 0 iff anomaly
        assert np.array_equal(f[f != 0], np.where(md.cpu().numpy() >= 0, 1, -1)[f != 0])
        if prev is not None:
            assert np.all((f != 0) <= (prev != 0))                  # monotone in the threshold
        prev = f
    perm = [3, 1, 5, 0, 2, 4]
    sp, mp = E.score_windows(cuda(X[perm]), det, mean[perm].contiguous(), std[perm].contiguous())
    assert torch.equal(sp, sc[perm]) and torch.equal(mp, md[perm])  # bitwise equivariance
    sc2, md2 = E.score_windows(Xc, det, mean, std)
    assert torch.equal(sc2, sc) and torch.equal(md2, md)           # deterministic
    X2 = X.copy()
    X2[2, 1000, 4] += 7 * float(std[2, 4])
    s3, _ = E.score_windows(cuda(X2), det, mean, std)
    ch = torch.nonzero((s3 != sc).any(dim=0)).flatten().cpu().numpy() + W - 1
    assert ch.min() >= 1000 and ch.max() <= 1000 + W - 1            # window locality
    with pytest.raises(E.EnovaError) as ei:
        E.detect(Xc, det, mean, std, {"z_q": float("nan")})
    assert ei.value.name == "ENOVA_ERR_UNCALIBRATED"
    with pytest.raises(E.EnovaError) as ei:
        E.score_windows(Xc[:, :50], det, mean, std)
    assert ei.value.name == "ENOVA_ERR_INSUFFICIENT_HISTORY"


def test_surge_and_drop_flags(E):                 # S:527-529 with a constructed detector
    W, M, H, Z = 32, 8, 32, 4
    d = detectors.mean_detector(W, M, H, Z, alpha=1.0, beta=2.0)
    r = np.random.default_rng(12)
    T = 4000
    X = r.standard_normal((1, T, M)).astype(np.float32)
    X[0, 3000:3000 + W, :] += 5.0
    X[0, 3500:3500 + W, :] -= 3.0
    det = E.PreparedDetector(d)
    res = E.run_pipeline(cuda(X), det, 2000)
    f = res.flags.cpu().numpy()[0]
    assert f[3000 + W - 1 - 2000] == 1 and f[3500 + W - 1 - 2000] == -1
    ref = O.detect_pipeline(X, d, 2000)
    assert_flags(f[None], ref["flags"], ref["scores"], ref["md"], ref["threshold"]["z_q"])


# ----------------------------------------------------------------- a-10 ----
def test_streaming_ring_matches_batch(E):
    W, M, H, Z = 64, 16, 128, 16
    N, T = 300, 200
    X = synth.metric_trace(N, T, M, seed=41)
    wts = synth.detector_weights(W, M, H, Z, seed=41)
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc, 150)
    thr = {"z_q": 2.0}
    fb, sb, mb = E.detect(Xc, det, mean, std, thr, return_scores=True)
    ring = torch.zeros((N, 2 * W, M), dtype=torch.float32, device="cuda")
    for k in range(T):
        E.ring_push(ring, Xc[:, k, :].contiguous(), k)
        if k >= W - 1:
            view = E.ring_view(ring, k)
            f, s, m = E.detect(view, det, mean, std, thr, W - 1, W, return_scores=True)
            assert torch.equal(s[:, 0], sb[:, k - W + 1])
            assert torch.equal(f[:, 0], fb[:, k - W + 1])


@pytest.mark.parametrize("W,M,H,Z,N", [(64, 16, 128, 16, 300), (32, 8, 32, 4, 130), (16, 32, 64, 8, 70),
                                       (20, 8, 64, 8, 200), (40, 16, 128, 16, 129)],
                         ids=lambda v: str(v))
def test_stream_ring_matches_batch_and_oracle(E, W, M, H, Z, N):
    """a-10 fast path: ingest-normalised fp16 ring + TMA-fed row kernel.  Every
    tick's scores / MD / flags equal the batch detect() of the same windows bit
    for bit (M <= 16: same epilogue and association as the CTA-pair kernel) and
    match the oracle within the parity tolerances."""
    T = W + 40
    X = synth.metric_trace(N, T, M, seed=W + M + N)
    wts = synth.detector_weights(W, M, H, Z, seed=W + M + N)
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc, T)
    thr = {"z_q": 1.5, "t": 1.0, "gamma": 0.0, "sigma": 1.0, "n": 1, "n_peaks": 10,
           "init_quantile": 0.98, "risk_q": 1e-3, "method": 1}
    thr_dev = E.threshold_to_device(thr)
    fb, sb, mb = E.detect(Xc, det, mean, std, thr, return_scores=True)
    rs, rmd = O.score_windows(X, wts, mean.cpu().numpy(), std.cpu().numpy(), W - 1, T)
    ring = E.StreamRing(det, mean, std)
    ring2 = E.StreamRing(det, mean, std)           # fused push + detect (enova_stream_step)
    for k in range(T):
        ring.push(Xc[:, k, :].contiguous(), k)
        if k < W - 1:
            ring2.push(Xc[:, k, :].contiguous(), k)
        if k >= W - 1:
            f, s_, m_ = ring.detect(k, thr_dev)
            f2, s2, m2 = ring2.step(Xc[:, k, :].contiguous(), k, thr_dev)
            assert torch.equal(f, f2) and torch.equal(s_, s2) and torch.equal(m_, m2), k
            j = k - W + 1
            assert_scores(s_.cpu().numpy(), rs[:, j], "stream scores")
            assert_md(m_.cpu().numpy(), rmd[:, j])
            if M <= 16:
                assert torch.equal(s_, sb[:, j]), f"tick {k}: stream scores != batch"
                assert torch.equal(m_, mb[:, j]), f"tick {k}: stream md != batch"
                assert torch.equal(f, fb[:, j])


# ------------------------------------------- stream-ordered / graph path ----
def test_async_pipeline_matches_sync_and_oracle(E):
    """Pipeline (enova_step: stats -> calibration scores + MD -> fit -> detection
    scores + MD -> every flag) in sequence gives bitwise the result of the
    synchronous calls, eagerly and as a CUDA graph; the overlapped step (the fit
    on a reduced grid next to the detection scores) gives the same scores, MD,
    flags and calibration flags bit for bit and z_q up to the fit's summation
    order (1e-12)."""
    W, M, H, Z = 64, 16, 128, 16
    N, T = 12, 3000
    X = synth.metric_trace(N, T, M, seed=51)
    wts = synth.detector_weights(W, M, H, Z, seed=51)
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    ref = E.run_pipeline(Xc, det, T // 2)
    pipe = E.Pipeline(det, N, T, T // 2, overlap=False)
    pipe.enqueue(Xc)
    res = pipe.result()
    assert res.threshold == ref.threshold
    assert torch.equal(res.mean, ref.mean) and torch.equal(res.std, ref.std)
    assert torch.equal(res.cal_scores, ref.cal_scores)
    assert torch.equal(res.flags, ref.flags) and torch.equal(res.scores, ref.scores)
    assert torch.equal(res.md, ref.md)
    assert torch.equal(res.cal_md, ref.cal_md) and torch.equal(res.cal_flags, ref.cal_flags)
    pipe.flags.zero_()
    pipe.capture(Xc)
    for _ in range(2):
        pipe.replay()
    res2 = pipe.result()
    assert res2.threshold == ref.threshold and torch.equal(res2.flags, ref.flags)
    o = O.pot_threshold(ref.cal_scores.cpu().numpy(), 0.98, 1e-3)
    assert abs(res2.threshold["z_q"] - o["z_q"]) <= 1e-9 * o["z_q"]
    for pot, conc in ((24, 5), (32, 12), (16, 0), (8, 3)):
        po = E.Pipeline(det, N, T, T // 2, pot_ctas=pot, concurrent_instances=conc)
        po.capture(Xc)
        po.replay()
        r3 = po.result()
        assert torch.equal(r3.scores, ref.scores) and torch.equal(r3.md, ref.md)
        assert torch.equal(r3.flags, ref.flags) and torch.equal(r3.cal_flags, ref.cal_flags)
        assert r3.threshold["t"] == ref.threshold["t"]
        assert r3.threshold["n_peaks"] == ref.threshold["n_peaks"]
        assert abs(r3.threshold["z_q"] - ref.threshold["z_q"]) <= 1e-12 * ref.threshold["z_q"]


def test_async_failures_are_reported_on_device(E):
    s = np.random.default_rng(1).exponential(1.0, 400).astype(np.float32)
    thr = E.fit_threshold_async(cuda(s), 0.98, 1e-3)
    with pytest.raises(E.EnovaError) as ei:
        E.threshold_from_device(thr)
    assert ei.value.name == "ENOVA_ERR_TOO_FEW_EXCEEDANCES"
    from paper_2407_09486_b200 import _lib
    t = _lib.Threshold.from_buffer_copy(bytes(thr.cpu().numpy().tobytes()))
    assert math.isnan(t.z_q)
    # a failed fit flags nothing
    W, M, H, Z = 32, 8, 32, 4
    X = synth.metric_trace(2, 400, M, seed=52)
    det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=52))
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc, 200)
    f, _, _ = E.detect_async(Xc, det, mean, std, thr)
    assert int((f != 0).sum()) == 0
    # non-finite calibration data is reported through diag
    X[1, 10, 3] = np.inf
    diag = torch.zeros(2, dtype=torch.int64, device="cuda")
    E.compute_stats_async(cuda(X), 200, diag=diag)
    with pytest.raises(E.EnovaError) as ei:
        E.check_stats_diag(diag)
    assert ei.value.name == "ENOVA_ERR_NONFINITE"


def test_stats_chunked_one_pass_matches_oracle(E):
    """One-pass shifted sums over time chunks: many instances (1 chunk each) and
    few long ones (up to 16 chunks), incl. a degenerate and an offset series."""
    # (20000, 100, 8) and (5000, 80, 24): > 64 instance segments per CTA, so the
    # deferred tickets / combines are flushed mid-range (kStatsDefer) as well as
    # at the end; M = 24 takes the non-power-of-two reduction
    for N, T, M in ((1, 20000, 8), (3, 9000, 32), (700, 300, 16), (20000, 100, 8), (5000, 80, 24)):
        X = synth.metric_trace(N, T, M, seed=53 + N)
        X[0, :, 1] = 7.25                                    # constant -> floored
        X[-1, :, 0] += 1e4                                   # large offset vs spread
        mean, std, nd = E.compute_stats(cuda(X), T // 2 + 3)
        om, os_, ond = O.series_stats(X, T // 2 + 3)
        assert nd == ond
        assert np.max(np.abs(mean.cpu().numpy().view(np.int32) - om.view(np.int32))) <= 1
        assert np.max(np.abs(std.cpu().numpy().view(np.int32) - os_.view(np.int32))) <= 1


# ------------------------------------------------------------------ NEXT-4 ----
def test_point_adjusted_counts_match_oracle(E):
    """Point-adjusted TP/FP/FN/TN on the GPU (one warp per instance, 32-point
    ballots with segments carried across chunks) equal the oracle's exactly:
    random segment structures incl. segments crossing and filling 32-point
    chunks and the range ends, several t_begin, plus a real detect run against
    the synthetic injected-event labels."""
    rng = np.random.default_rng(11)
    for trial in range(12):
        N, T = int(rng.integers(1, 40)), int(rng.integers(33, 400))
        tb = int(rng.integers(0, T // 3))
        nw = T - tb - int(rng.integers(0, 5))
        lab = np.zeros((N, T), np.int8)
        for i in range(N):
            for _ in range(int(rng.integers(0, 6))):
                a = int(rng.integers(0, T))
                lab[i, a:a + int(rng.integers(1, 80))] = rng.choice([-1, 1])
        if trial == 0:
            lab[:, :] = 1                       # one segment over everything
        fl = ((rng.random((N, nw)) < rng.uniform(0, 0.3)) * rng.choice([-1, 1])).astype(np.int8)
        got = E.point_adjusted_counts(cuda(lab), cuda(fl), tb).cpu().tolist()
        ref = O.fleet_point_adjusted_counts(lab, fl, tb)
        assert tuple(got) == ref, (trial, got, ref)
    # a detect run against the generator's labels (c1-shaped detector)
    X, labels = synth.metric_trace(6, 3000, 8, seed=17, return_labels=True)
    d = detectors.mean_detector(32, 8, 32, 4, alpha=4.0, beta=2.0) if hasattr(detectors, "mean_detector") \
        else synth.detector_weights(32, 8, 32, 4, seed=17)
    det = E.PreparedDetector(d)
    res = E.run_pipeline(cuda(X), det, 1500)
    fl = res.flags
    got = E.point_adjusted_counts(cuda(labels), fl, 1500).cpu().tolist()
    ref = O.fleet_point_adjusted_counts(labels, fl.cpu().numpy(), 1500)
    assert tuple(got) == ref
    m = E.point_adjusted_f1(cuda(labels), fl, 1500)
    assert 0.0 <= m["precision"] <= 1.0 and 0.0 <= m["recall"] <= 1.0


# ------------------------------------------------------------------ NEXT-1 ----
@pytest.mark.parametrize("W,M,H,Z", [(64, 16, 128, 16), (32, 8, 32, 4), (24, 8, 64, 9)],
                         ids=lambda v: str(v))
def test_explain_windows_match_oracle(E, W, M, H, Z):
    """select_flagged = np.flatnonzero; explain_windows gives per-metric MD within
    the MD tolerance of the oracle's explicit D-wide decoder, and scores / MD
    bit-identical to the batch detect of the same windows."""
    N, T = 7, 260 + W
    X = synth.metric_trace(N, T, M, seed=W + H)
    wts = synth.detector_weights(W, M, H, Z, seed=W + H)
    mean, std, _ = O.series_stats(X, T // 2)
    det = E.PreparedDetector(wts)
    tb, te = W - 1 + 5, T - 3
    thr = {"z_q": 1.0}
    fl, sc, md = E.detect(cuda(X), det, cuda(mean), cuda(std), thr, tb, te, return_scores=True)
    ids = E.select_flagged(fl)
    assert np.array_equal(ids.cpu().numpy(), np.flatnonzero(fl.cpu().numpy().reshape(-1)))
    rng = np.random.default_rng(W)
    extra = rng.choice(N * (te - tb), size=300, replace=False)
    for sel in (ids, torch.from_numpy(np.sort(extra)).cuda()):
        if sel.numel() == 0:
            continue
        mdm, s2, m2 = E.explain_windows(cuda(X), det, cuda(mean), cuda(std), sel, tb, te)
        g = sel.cpu().numpy()
        assert torch.equal(s2, sc.reshape(-1)[sel]) and torch.equal(m2, md.reshape(-1)[sel])
        ref = O.per_metric_mean_difference(X, wts, mean, std, tb, te).reshape(-1, M)[g]
        err = np.abs(mdm.cpu().numpy() - ref)
        assert np.all(err <= 1e-4 + 1e-3 * np.abs(ref)), err.max()


# ------------------------------------------------------------------ NEXT-2 ----
@pytest.mark.parametrize("refit_every", [1, 3])
def test_spot_ticks_match_oracle(E, refit_every):
    """Online SPOT on the device state (calibration fit -> per-tick appends of the
    non-anomalous peaks -> refits) tracks the oracle's tick-synchronous SPOT:
    identical flags, t, n and N_t, z_q within 1e-9 relative, after every tick."""
    init = synth.score_mixture(200_000, seed=21)
    ticks = [synth.score_mixture(2000, seed=22, offset=2000 * k) for k in range(10)]
    ticks[4][[7, 900]] = 80.0                        # anomalies never enter the model
    ref = O.spot_ticks(init, ticks, refit_every=refit_every)
    spot = E.Spot(200_000, stream_peaks=20_000)
    spot.calibrate(cuda(init))
    z0 = spot.threshold()
    r0 = O.pot_threshold(init)
    assert z0["n_peaks"] == r0["n_peaks"] and abs(z0["z_q"] - r0["z_q"]) <= 1e-9 * r0["z_q"]
    for k, tick in enumerate(ticks):
        sc = cuda(tick)
        z = spot.threshold()["z_q"]
        fl = (sc.double() > z).to(torch.int8)
        spot.update(sc, fl)
        if (k + 1) % refit_every == 0:
            spot.refit()
        got = spot.threshold()
        rfl, rthr = ref[k]
        assert np.array_equal(fl.cpu().numpy().astype(bool), rfl), k
        assert got["n"] == rthr["n"] and got["n_peaks"] == rthr["n_peaks"], (k, got, rthr)
        assert got["t"] == rthr["t"]
        assert abs(got["z_q"] - rthr["z_q"]) <= 1e-9 * rthr["z_q"], (k, got["z_q"], rthr["z_q"])


def test_spot_capacity_overflow_reported(E):
    """Peaks beyond the SPOT capacity are not silently dropped: the refit after
    the overflow (and every later one) reports ENOVA_ERR_WORKSPACE with a NaN
    z_q instead of fitting the truncated peak set; a new calibration clears it."""
    init = synth.score_mixture(50_000, seed=31)
    spot = E.Spot(50_000, stream_peaks=100)
    spot.calibrate(cuda(init))
    base = spot.threshold()
    t = base["t"]
    tick = cuda(np.full(300, t + 0.5, np.float32))        # 300 normal peaks > capacity 100
    spot.update(tick, torch.zeros(300, dtype=torch.int8, device="cuda"))
    spot.refit()
    with pytest.raises(E.EnovaError):
        spot.threshold()
    raw = spot.thr.cpu().numpy().tobytes()
    from paper_2407_09486_b200._lib import Threshold
    th = Threshold.from_buffer_copy(raw)
    assert math.isnan(th.z_q) and th.reserved == 9      # ENOVA_ERR_WORKSPACE
    spot.refit()                                          # still reported
    with pytest.raises(E.EnovaError):
        spot.threshold()
    spot.calibrate(cuda(init))                            # a new calibration clears it
    assert spot.threshold()["z_q"] == base["z_q"]
    # within capacity: no error
    spot.update(cuda(np.full(50, t + 0.5, np.float32)), torch.zeros(50, dtype=torch.int8, device="cuda"))
    spot.refit()
    assert spot.threshold()["n_peaks"] == base["n_peaks"] + 50


# ------------------------------------------------------- full-size configs ----
def test_c3_shard_full_size_sampled(E):
    """c3's per-GPU shard at full size (512 instances x T=50 000, 25.5M windows) in
    the bench's graph-captured Pipeline: sampled windows one by one against the
    oracle, the fleet threshold against the oracle fit of the same 12.8M
    calibration scores, and every flag against the rule."""
    cfg = synth.CONFIGS["c3"]
    N, T, M = cfg["n_instances"] // 8, cfg["n_steps"], cfg["n_metrics"]
    W, H, Z = cfg["window"], cfg["hidden"], cfg["latent"]
    X = synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2, instance_offset=3 * N)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    pipe = E.Pipeline(det, N, T, tcal)
    pipe.capture(Xc)
    pipe.replay()
    torch.cuda.synchronize()
    res = pipe.result()
    r = np.random.default_rng(13)
    om, os_, _ = O.series_stats(X, tcal)
    gs, gmd = res.scores.cpu().numpy(), res.md.cpu().numpy()
    for i in np.unique(r.integers(0, N, 60)):
        for t in np.sort(r.choice(np.arange(tcal, T), 3, replace=False)):
            rs, rmd = O.score_windows(X[i:i + 1], wts, om[i:i + 1], os_[i:i + 1], t, t + 1)
            assert_scores(gs[i, t - tcal:t - tcal + 1], rs[0], f"inst {i} t {t}")
            assert_md(gmd[i, t - tcal:t - tcal + 1], rmd[0])
    o = O.pot_threshold(res.cal_scores.cpu().numpy(), 0.98, 1e-3)
    assert res.threshold["n_peaks"] == o["n_peaks"] and res.threshold["t"] == o["t"]
    assert abs(res.threshold["z_q"] - o["z_q"]) <= 1e-9 * o["z_q"]
    assert np.array_equal(res.flags.cpu().numpy(), O.flags(gs, gmd, res.threshold["z_q"]))


def test_c4_streaming_full_size(E):
    """c4 at full size: 10 000 instances, fused stream ticks (enova_stream_step)
    against the oracle on a sample of instances per tick and against batch
    detect bit for bit."""
    cfg = synth.CONFIGS["c4"]
    n, M, W, H, Z = cfg["n_instances"], cfg["n_metrics"], cfg["window"], cfg["hidden"], cfg["latent"]
    t_hist, ticks = 256, 4
    X = synth.metric_trace_parallel(n, t_hist + ticks, M, seed=synth.DEFAULT_SEED + 4)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 4)
    det = E.PreparedDetector(wts)
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc[:, :t_hist], t_hist)
    thr = {"z_q": 3.0}
    thr_dev = E.threshold_to_device(thr)
    ring = E.StreamRing(det, mean, std)
    for t in range(t_hist - W + 1, t_hist):
        ring.push(Xc[:, t].contiguous(), t)
    m_np, s_np = mean.cpu().numpy(), std.cpu().numpy()
    r = np.random.default_rng(4)
    for t in range(t_hist, t_hist + ticks):
        f, sc, md = ring.step(Xc[:, t].contiguous(), t, thr_dev)
        fb, sb, mb = E.detect(Xc[:, t - W + 1:t + 1].contiguous(), det, mean, std, thr, W - 1, W,
                              return_scores=True)
        assert torch.equal(sc, sb[:, 0]) and torch.equal(md, mb[:, 0]) and torch.equal(f, fb[:, 0])
        idx = np.sort(r.choice(n, 50, replace=False))
        rs, rmd = O.score_windows(X[idx][:, t - W + 1:t + 1], wts, m_np[idx], s_np[idx], W - 1, W)
        assert_scores(sc.cpu().numpy()[idx], rs[:, 0], f"tick {t}")
        assert_md(md.cpu().numpy()[idx], rmd[:, 0])
