"""ENOVA detector training oracle (NEXT-3): Eq. 9's semi-supervised ELBO with a
PI-controlled beta(k), plain, slow, fp64 NumPy.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` may import this module; the product path never does.  It shares
no code with the CUDA path (``paper_2407_09486_b200/csrc/train.cu``).

What it computes (``P:n`` = PAPER.md line, ``S:n`` = SPEC.md line, ``R-n`` =
DESIGN.md reading):

* ``elbo``       Eq. 9 on a batch of windows x_i with labels l_i:
      L = (1/B) sum_i [ l_i * log p(x_i | z_i) - (1 + l_i)/2 * beta * KL_i ]
  with the reparameterised single-sample estimate z_i = mu_i + exp(lv_i / 2) eps_i
  of the expectation ("gradient ascent with the reparameterization
  trick ... single-sample Monte-Carlo"), the unit-variance Gaussian likelihood
  log p(x|z) = -1/2 ||x - m'(z)||^2 - D/2 log 2 pi, and
  KL = 1/2 sum (mu^2 + e^lv - 1 - lv) against the N(0, I) prior (R-6).  The
  encoder / decoder are the detector's (enova_oracle.encoder / decoder
  topology: h = tanh(W1 x + b1), [mu | lv] = heads(h), m' = W4 tanh(W3 z + b3)
  + b4), here with the SAMPLE z in the decoder (training) where detection uses
  z = mu (R-7).  The noise eps is an input (drawn by the caller).
* ``elbo_grad``  the analytic gradient of L with respect to every parameter,
  back-propagated by hand step by step in the forward's order (no autodiff).
* ``beta_pi``    beta(k) "from PI control": the error of the k-th
  iteration e_k = KLbar_k - setpoint (KLbar = mean KL of the batch's normal
  rows), integral I_k = I_{k-1} + e_k, beta_k = clamp(Kp e_k + Ki I_k, 0,
  beta_max) with the integral held (anti-windup) while beta is clamped; SPEC
  S:548's constants setpoint = 0.5 Z nats, Kp = 0.01, Ki = 0.001, beta in
  [0, 1] (reading R-24).
* ``adam_ascent`` Adam (step 1e-3; betas 0.9 / 0.999, eps 1e-8 --
  the method's customary constants) maximising L.
* ``train``      epochs x batches of the above over given window ids in a
  given order (the permutation and the noise are inputs).

Pins (tests/test_oracle_train.py): the gradient against central finite
differences on a 3-row dataset (<= 1e-4 relative), Eq. 9 with every
label +1 and beta = 1 against an independently coded plain ELBO (scipy
Gaussian log-densities and a Gauss-Hermite quadrature of the KL integral,
S:540, 1e-9), the (1 + l)/2 weight (an anomaly row has no KL term), the
PI controller and Adam against hand-computed sequences, and the training
curve.
"""
from __future__ import annotations

import math

import numpy as np

PARAMS = ("enc_w1", "enc_b1", "enc_wmu", "enc_bmu", "enc_wlv", "enc_blv",
          "dec_w1", "dec_b1", "dec_w2", "dec_b2")


def as_params(weights: dict) -> dict:
    """fp64 copies of the trainable parameters (include/enova.h layouts)."""
    return {k: np.array(weights[k], dtype=np.float64) for k in PARAMS}


def forward(p: dict, x: np.ndarray, eps: np.ndarray):
    """Training forward of a batch x [B, D] with noise eps [B, Z]."""
    h = np.tanh(x @ p["enc_w1"].T + p["enc_b1"])
    mu = h @ p["enc_wmu"].T + p["enc_bmu"]
    lv = h @ p["enc_wlv"].T + p["enc_blv"]
    sd = np.exp(0.5 * lv)
    z = mu + sd * eps
    a3 = np.tanh(z @ p["dec_w1"].T + p["dec_b1"])
    mp = a3 @ p["dec_w2"].T + p["dec_b2"]
    D = x.shape[1]
    logp = -0.5 * np.sum((x - mp) ** 2, axis=1) - 0.5 * D * math.log(2.0 * math.pi)
    kl = 0.5 * np.sum(mu * mu + np.expm1(lv) - lv, axis=1)
    return dict(h=h, mu=mu, lv=lv, sd=sd, z=z, a3=a3, mp=mp, logp=logp, kl=kl)


def elbo(p: dict, x: np.ndarray, labels: np.ndarray, eps: np.ndarray, beta: float):
    """Eq. 9: returns (L, per-row logp, per-row KL)."""
    f = forward(p, x, eps)
    l = np.asarray(labels, dtype=np.float64)
    L = float(np.mean(l * f["logp"] - 0.5 * (1.0 + l) * beta * f["kl"]))
    return L, f["logp"], f["kl"]


def elbo_grad(p: dict, x: np.ndarray, labels: np.ndarray, eps: np.ndarray, beta: float):
    """dL/dtheta of Eq. 9 for every parameter, by hand-written back-propagation
    (same order as the forward).  Returns (L, grads dict, mean KL of the rows
    with l = +1, their mean plain ELBO log p - KL)."""
    f = forward(p, x, eps)
    B = x.shape[0]
    l = np.asarray(labels, dtype=np.float64)
    L = float(np.mean(l * f["logp"] - 0.5 * (1.0 + l) * beta * f["kl"]))
    c = (l / B)[:, None]                       # weight of log p per row
    k = (0.5 * (1.0 + l) * beta / B)[:, None]  # weight of -KL per row
    g = {}
    # log p = -1/2 ||x - m'||^2  ->  dL/dm' = c (x - m')
    d_mp = c * (x - f["mp"])
    g["dec_w2"] = d_mp.T @ f["a3"]
    g["dec_b2"] = d_mp.sum(axis=0)
    d_a3 = d_mp @ p["dec_w2"]
    d_pre3 = d_a3 * (1.0 - f["a3"] ** 2)
    g["dec_w1"] = d_pre3.T @ f["z"]
    g["dec_b1"] = d_pre3.sum(axis=0)
    d_z = d_pre3 @ p["dec_w1"]
    # z = mu + exp(lv/2) eps ; -KL term: d(-KL)/dmu = -mu, d(-KL)/dlv = -(e^lv - 1)/2
    d_mu = d_z - k * f["mu"]
    d_lv = d_z * eps * 0.5 * f["sd"] - k * 0.5 * np.expm1(f["lv"])
    g["enc_wmu"] = d_mu.T @ f["h"]
    g["enc_bmu"] = d_mu.sum(axis=0)
    g["enc_wlv"] = d_lv.T @ f["h"]
    g["enc_blv"] = d_lv.sum(axis=0)
    d_h = d_mu @ p["enc_wmu"] + d_lv @ p["enc_wlv"]
    d_pre1 = d_h * (1.0 - f["h"] ** 2)
    g["enc_w1"] = d_pre1.T @ x
    g["enc_b1"] = d_pre1.sum(axis=0)
    normal = l > 0
    kl_normal = float(f["kl"][normal].mean()) if normal.any() else 0.0
    elbo_normal = float((f["logp"] - f["kl"])[normal].mean()) if normal.any() else 0.0
    return L, g, kl_normal, elbo_normal


class BetaPI:
    """beta(k) from a PI controller on the KL of the normal rows (R-24)."""

    def __init__(self, setpoint: float, kp: float = 0.01, ki: float = 0.001,
                 beta_max: float = 1.0, beta0: float = 0.0):
        self.setpoint, self.kp, self.ki, self.beta_max = setpoint, kp, ki, beta_max
        self.integral = 0.0
        self.beta = beta0

    def update(self, kl_normal: float) -> float:
        e = kl_normal - self.setpoint
        integral = self.integral + e
        b = self.kp * e + self.ki * integral
        if 0.0 <= b <= self.beta_max:
            self.integral = integral           # anti-windup: integrate only unclamped
        self.beta = min(self.beta_max, max(0.0, b))
        return self.beta


class AdamAscent:
    """Adam maximising the objective: theta += lr * mhat / (sqrt(vhat) + eps)."""

    def __init__(self, params: dict, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.m = {k: np.zeros_like(v) for k, v in params.items()}
        self.v = {k: np.zeros_like(v) for k, v in params.items()}
        self.t = 0

    def step(self, params: dict, grads: dict):
        self.t += 1
        c1 = 1.0 - self.b1 ** self.t
        c2 = 1.0 - self.b2 ** self.t
        for k in params:
            self.m[k] = self.b1 * self.m[k] + (1.0 - self.b1) * grads[k]
            self.v[k] = self.b2 * self.v[k] + (1.0 - self.b2) * grads[k] ** 2
            mhat = self.m[k] / c1
            vhat = self.v[k] / c2
            params[k] = params[k] + self.lr * mhat / (np.sqrt(vhat) + self.eps)


def train(weights: dict, windows: np.ndarray, labels: np.ndarray, order: np.ndarray,
          eps: np.ndarray, batch: int, lr: float = 1e-3, setpoint: float | None = None,
          kp: float = 0.01, ki: float = 0.001, beta_max: float = 1.0, log_every: int = 0):
    """Train on `windows` [n, D] (detector inputs x, e.g. enova_oracle.normalise_x16
    windows) with labels [n] in {+1, -1}.  `order` [steps * batch] lists the
    window index of every row of every step (epochs concatenated, ragged last
    batch of an epoch allowed via -1 padding rows that are skipped); `eps`
    [steps * batch, Z] the noise of every row.  Returns (params, history) with
    history = [(L, beta, kl_normal, elbo_normal)] per step."""
    p = as_params(weights)
    Z = p["enc_bmu"].size
    pi = BetaPI(0.5 * Z if setpoint is None else setpoint, kp, ki, beta_max)
    opt = AdamAscent(p, lr)
    hist = []
    steps = len(order) // batch
    for s in range(steps):
        idx = order[s * batch:(s + 1) * batch]
        keep = idx >= 0
        idx = idx[keep]
        e = eps[s * batch:(s + 1) * batch][keep]
        L, g, kln, eln = elbo_grad(p, windows[idx], labels[idx], e, pi.beta)
        opt.step(p, g)
        hist.append((L, pi.beta, kln, eln))
        pi.update(kln)
        if log_every and s % log_every == 0:
            print(f"step {s}: L {L:.4f} beta {pi.beta:.4f} KL(normal) {kln:.4f}")
    return p, hist
