"""Constructed detectors with closed-form outputs (test helpers, no method
arithmetic).  Every matrix entry is fp16-representable so the detector's
fp16 operand rounding (R-17) is lossless."""
import numpy as np


def zeros(W, M, H, Z):
    D = W * M
    f = np.float32
    return dict(window=W, n_metrics=M, hidden=H, latent=Z,
                enc_w1=np.zeros((H, D), f), enc_b1=np.zeros(H, f),
                enc_wmu=np.zeros((Z, H), f), enc_bmu=np.zeros(Z, f),
                enc_wlv=np.zeros((Z, H), f), enc_blv=np.zeros(Z, f),
                dec_w1=np.zeros((H, Z), f), dec_b1=np.zeros(H, f),
                dec_w2=np.zeros((D, H), f), dec_b2=np.zeros(D, f))


def mean_detector(W, M, H, Z, alpha=1.0, beta=2.0, b1=0.0, bmu0=0.0):
    """Every W1 row = alpha/D * 1, Wmu = beta * e_1 selector, Wlv = 0:
    score = 1/2 (beta*tanh(alpha*mean(x) + b1) + bmu0)^2 (+ 0 from the
    other coordinates); decoder = 0 so MD = mean(x)."""
    d = zeros(W, M, H, Z)
    D = W * M
    d["enc_w1"][:] = np.float32(alpha / D)
    d["enc_b1"][:] = np.float32(b1)
    d["enc_wmu"][0, 0] = np.float32(beta)
    d["enc_bmu"][0] = np.float32(bmu0)
    return d


def tap_selector(W, M, H, Z, tau, j, a=0.75):
    """W1[0, tau*M + j] = a: mu_0 = tanh(a * x[t-W+1+tau, j]),
    score = 1/2 tanh(a * x[t-W+1+tau, j])^2."""
    d = zeros(W, M, H, Z)
    d["enc_w1"][0, tau * M + j] = np.float32(a)
    d["enc_wmu"][0, 0] = np.float32(1.0)
    return d
