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


def full_path_detector(W, M, H, Z):
    """Every weight matrix of the path non-zero, each a sparse selector, with
    a closed form per window (``full_path_closed_form``):
      W1 row k = a_k/D * 1           -> h_k = tanh(a_k mean(x) + b1_k)
      Wmu[0, 2] = 1.5, Wmu[1, 5] = -0.75  -> mu_0 = 1.5 h_2 + bmu_0, mu_1 = -0.75 h_5 + bmu_1
      Wlv[0, 3] = 0.5, Wlv[2, 1] = -1.25  -> lv_0 = 0.5 h_3 + blv_0, lv_2 = -1.25 h_1 + blv_2
      W3[4, 1] = 0.875                    -> a3_4 = tanh(0.875 mu_1 + b3_4), a3_j = tanh(b3_j)
      Wdec2[:, 4] = 0.625, Wdec2[:, 0] = -0.5 -> m'_k = 0.625 a3_4 - 0.5 a3_0 + bdec2_k
    Needs H >= 6, Z >= 3.  All entries fp16-representable."""
    if H < 6 or Z < 3:
        raise ValueError("full_path_detector needs H >= 6 and Z >= 3")
    d = zeros(W, M, H, Z)
    D = W * M
    f = np.float32
    a = [(k % 7 + 1) * 0.5 for k in range(H)]
    for k in range(H):
        d["enc_w1"][k, :] = f(a[k] / D)
        d["enc_b1"][k] = f(((k % 5) - 2) * 0.125)
    d["enc_wmu"][0, 2] = f(1.5)
    d["enc_wmu"][1, 5] = f(-0.75)
    d["enc_bmu"][:] = np.array([((z % 3) - 1) * 0.25 for z in range(Z)], f)
    d["enc_wlv"][0, 3] = f(0.5)
    d["enc_wlv"][2, 1] = f(-1.25)
    d["enc_blv"][:] = np.array([((z % 4) - 1.5) * 0.25 for z in range(Z)], f)
    d["dec_w1"][4, 1] = f(0.875)
    d["dec_b1"][:] = np.array([((k % 3) - 1) * 0.375 for k in range(H)], f)
    d["dec_w2"][:, 4] = f(0.625)
    d["dec_w2"][:, 0] = f(-0.5)
    d["dec_b2"][:] = np.array([((k % 9) - 4) * 0.0625 for k in range(D)], f)
    return d
