"""GPU: NEXT-3 training (Eq. 9) through the C ABI against the fp64 training
oracle (oracle/enova_train_oracle.py), and the SPEC synthetic benchmark end to
end through the hot path and the NEXT-4 evaluator.

Tolerances (derived from the arithmetic): the GPU step is fp32
(cuBLAS FFMA GEMMs, fp32 element-wise, fp64 row reductions) against fp64, sums
of at most a few thousand terms -> normwise relative gradient error ~1e-6;
gated at 1e-4 per tensor.  After 20 Adam steps the parameters agree to 1e-3
normwise (Adam divides by sqrt(v), which amplifies the relative error of
near-zero gradient components)."""
import json
import os

import numpy as np
import pytest
import torch

from oracle import enova_oracle as O
from oracle import enova_train_oracle as T
from paper_2407_09486_b200 import synth
from tests import train_bench as TB

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def E():
    from paper_2407_09486_b200 import build as B
    B.build()
    import paper_2407_09486_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _case(W, M, H, Z, N=3, Tn=400, seed=1):
    X = synth.metric_trace(N, Tn, M, seed=seed)
    w = synth.detector_weights(W, M, H, Z, seed=seed)
    tcal = Tn // 2
    mean, std, _ = O.series_stats(X, tcal)
    x = O.normalise_x16(X, mean, std)
    win = O.window_matrix(x, W, W - 1, Tn).reshape(-1, W * M)       # ids g = i * nw + r
    return X, w, mean, std, win


@pytest.mark.parametrize("W,M,H,Z,B", [(2, 8, 32, 4, 64), (32, 8, 32, 4, 256), (8, 16, 64, 16, 200)],
                         ids=lambda v: str(v))
def test_gradient_matches_oracle(E, W, M, H, Z, B):
    X, w, mean, std, win = _case(W, M, H, Z)
    n = win.shape[0]
    r = np.random.default_rng(W + B)
    ids = r.choice(n, B, replace=False).astype(np.int64)
    ids[[3, 17]] = -1                                       # padding rows are ignored
    labels = np.where(r.uniform(size=n) < 0.1, -1, 1).astype(np.int8)
    eps = r.standard_normal((B, Z)).astype(np.float32)
    beta = 0.4
    tr = E.Trainer(W, M, H, Z, max_batch=B)
    try:
        tr.load(w)
        g = tr.gradient(cuda(X), cuda(mean), cuda(std), W - 1, X.shape[1], cuda(ids), cuda(labels),
                        cuda(eps), beta)
        stats = tr.stats.cpu().numpy()
    finally:
        tr.destroy()
    keep = ids >= 0
    p = T.as_params(w)
    L, go, kln, eln = T.elbo_grad(p, win[ids[keep]], labels[ids[keep]].astype(np.float64),
                                  eps[keep].astype(np.float64), beta)
    for k in T.PARAMS:
        a = g[k].cpu().numpy().astype(np.float64)
        d = np.linalg.norm(a - go[k]) / max(np.linalg.norm(go[k]), 1e-30)
        assert d <= 1e-4, f"{k}: normwise relative gradient error {d:.2e}"
    assert stats[0] == pytest.approx(L, rel=1e-5)
    assert stats[2] == pytest.approx(kln, rel=1e-5)
    assert stats[3] == pytest.approx(eln, rel=1e-5)


def test_adam_and_pi_steps_match_oracle(E):
    """20 steps of Eq. 9 + Adam + the PI controller (beta starts at 0 and moves)."""
    W, M, H, Z, B = 4, 8, 32, 4, 128
    X, w, mean, std, win = _case(W, M, H, Z, N=2, Tn=600, seed=4)
    n = win.shape[0]
    r = np.random.default_rng(5)
    labels = np.where(r.uniform(size=n) < 0.05, -1, 1).astype(np.int8)
    steps = 20
    order = np.concatenate([r.permutation(n)[:B] for _ in range(steps)]).astype(np.int64)
    eps = r.standard_normal((steps * B, Z)).astype(np.float32)
    cfg = E.train_config(lr=2e-3, latent=Z, kl_setpoint=0.5)   # low setpoint: beta moves
    tr = E.Trainer(W, M, H, Z, max_batch=B)
    try:
        tr.load(w)
        hist = tr.fit(cuda(X), cuda(mean), cuda(std), W - 1, X.shape[1], cuda(labels),
                      cuda(order), cuda(eps), B, cfg, history=True).cpu().numpy()
        got = {k: v.cpu().numpy().astype(np.float64) for k, v in tr.weights().items()
               if k in T.PARAMS}
    finally:
        tr.destroy()
    p, ohist = T.train(w, win, labels.astype(np.float64), order, eps.astype(np.float64), B,
                       lr=2e-3, setpoint=0.5)
    betas_o = np.array([h[1] for h in ohist])
    assert np.max(np.abs(hist[:, 1] - betas_o)) <= 1e-4
    assert betas_o.max() > 0.0                                # the controller acted
    assert np.allclose(hist[:, 0], [h[0] for h in ohist], rtol=1e-3, atol=1e-3)
    for k in T.PARAMS:
        d = np.linalg.norm(got[k] - p[k]) / max(np.linalg.norm(p[k]), 1e-30)
        assert d <= 1e-3, f"{k}: {d:.2e}"


def test_spec_benchmark_f1_on_gpu(E):
    """S:544 / S:701 on the GPU: train with the CUDA trainer, then the hot path
    (stats -> calibration scores -> POT on the normal calibration windows ->
    flags of the detection half) and the NEXT-4 point-adjusted evaluator:
    F1 >= 0.90 and a held-out normal false-positive rate <= 2 q."""
    X, lab, tl = TB.data()
    W, M, H, Z = TB.W, TB.M, TB.H, TB.Z
    Xc = cuda(X)
    mean, std, _ = E.compute_stats(Xc, TB.TCAL)
    nw = TB.TCAL - (W - 1)
    l = cuda(TB.train_labels(tl).astype(np.int8))
    order, steps = TB.schedule(X.shape[0] * nw, TB.EPOCHS, TB.BATCH)
    eps = TB.noise(steps, TB.BATCH)
    w0 = synth.detector_weights(W, M, H, Z, seed=TB.SEED)
    tr = E.Trainer(W, M, H, Z, max_batch=TB.BATCH)
    cfg = E.train_config(lr=TB.LR, latent=Z)
    try:
        tr.load(w0)
        import time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hist = tr.fit(Xc, mean, std, W - 1, TB.TCAL, l, cuda(order), cuda(eps), TB.BATCH, cfg,
                      history=True)
        torch.cuda.synchronize()
        train_s = time.perf_counter() - t0
        wts = tr.weights()
    finally:
        tr.destroy()
    det = E.PreparedDetector(wts)
    cal, _ = E.score_windows(Xc, det, mean, std, W - 1, TB.TCAL)
    normal = cuda(TB.normal_cal_mask(lab))
    thr = E.fit_threshold(cal[normal].contiguous(), 0.98, 1e-3)
    flags = E.detect(Xc, det, mean, std, thr, TB.TCAL, TB.T)
    pa = E.point_adjusted_f1(cuda(lab), flags, TB.TCAL)
    ev = TB.evaluate(flags.cpu().numpy(), lab)
    assert (pa["tp"], pa["fp"], pa["fn"], pa["tn"]) == (ev["tp"], ev["fp"], ev["fn"], ev["tn"])
    rep = {"benchmark": f"SPEC S:544 synthetic (16 x 8000, W=2, M=8, H=32, Z=4), {TB.EPOCHS} epochs, batch {TB.BATCH}, Adam {TB.LR}",
           "train_s": train_s, "steps": steps, "final_beta": float(hist[-1, 1]),
           "z_q": thr["z_q"], **ev}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "train_f1.json"), "w") as f:
        json.dump(rep, f, indent=1)
    print(json.dumps(rep))
    assert ev["f1"] >= 0.90, rep
    assert ev["fp_rate_normal"] <= ev["fp_rate_bound"], rep


def test_trainer_argument_errors(E):
    tr = E.Trainer(2, 8, 32, 4, max_batch=8)
    try:
        X = cuda(np.zeros((1, 50, 8), np.float32))
        m = torch.zeros((1, 8), device="cuda")
        s = torch.ones((1, 8), device="cuda")
        ids = torch.zeros(9, dtype=torch.int64, device="cuda")                 # > max_batch
        lab = torch.ones(49, dtype=torch.int8, device="cuda")
        eps = torch.zeros((9, 4), device="cuda")
        with pytest.raises(E.EnovaError) as ei:
            tr.gradient(X, m, s, 1, 50, ids, lab, eps, 1.0)
        assert ei.value.name == "ENOVA_ERR_INVALID_ARGUMENT"
    finally:
        tr.destroy()
