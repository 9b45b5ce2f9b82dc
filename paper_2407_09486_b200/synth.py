"""Seeded synthetic inputs shared by the tests, the bench and the oracle checks.

This module holds NO arithmetic of the detection method (no normalisation, no
detector forward, no threshold).  It only draws inputs:

* ``metric_trace``   -- a fleet's monitoring tensor ``[instances, T, M]`` fp32,
  shaped like the paper's workload: one sample per minute (1440 points/day,
  PAPER.md:482), diurnal load, injected surges and drops (the case study's
  KV-cache surge), Table II metrics plus
  KV-cache utilisation.
* ``detector_weights`` -- random-init VAE detector parameters (Xavier normal),
  rounded to fp16-representable fp32 values (reading R-17).
* ``score_mixture``  -- the c5 threshold-calibration score vector.

Every draw uses a counter-based generator (numpy Philox) keyed by
``(seed, instance)`` or ``(seed, chunk)`` so any shard or subset of the fleet
regenerates bit-identically on any rank.  The recipe is stated in DESIGN.md
("Input recipe").
"""
from __future__ import annotations

import math

import numpy as np
from scipy.signal import lfilter

DEFAULT_SEED = 0x240709486

# Metric channel order: SPEC.md:90 field order n_f,n_r,n_a,n_p,t_r,m_u,g_u
# (Table II) + KV-cache utilisation.
BASE_METRICS = ("n_f", "n_r", "n_a", "n_p", "t_r", "m_u", "g_u", "kv")
EXTRA_METRICS = ("tokens_s", "ttft", "tpot", "queue_time", "prefill_tok_s",
                 "decode_tok_s", "power_w", "sm_occupancy")

STEPS_PER_DAY = 1440          # PAPER.md:482 (1440 points per day)
STEPS_PER_WEEK = 7 * STEPS_PER_DAY


def _rng(*key: int) -> np.random.Generator:
    k = np.array([int(x) & 0xFFFFFFFFFFFFFFFF for x in key] + [0] * (2 - len(key)),
                 dtype=np.uint64)[:2]
    return np.random.Generator(np.random.Philox(key=k))


def fp16_representable(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest fp16 value, returned as fp32."""
    return np.asarray(a, dtype=np.float32).astype(np.float16).astype(np.float32)


def metric_trace(n_instances: int, n_steps: int, n_metrics: int = 16,
                 seed: int = DEFAULT_SEED, instance_offset: int = 0,
                 return_labels: bool = False):
    """Synthetic fleet trace ``[n_instances, n_steps, n_metrics]`` fp32.

    Instance ``g = instance_offset + i`` is drawn from Philox(seed, g) only, so
    a shard ``[a, b)`` of a fleet equals rows ``a..b`` of the whole fleet.
    Labels (int8, +1 surge / -1 drop / 0 normal) are returned on request.
    """
    if n_metrics % 8 != 0 or n_metrics < 8:
        raise ValueError("n_metrics must be a positive multiple of 8")
    N, T, M = int(n_instances), int(n_steps), int(n_metrics)
    t = np.arange(T, dtype=np.float64)
    lam = np.empty((N, T))
    arrivals = np.empty((N, T))
    noise = np.empty((N, T, M))
    labels = np.zeros((N, T), dtype=np.int8)
    par = np.empty((N, 8))
    for i in range(N):
        r = _rng(seed, instance_offset + i)
        L = r.uniform(2.0, 20.0)                  # base load, req/s
        cap = L * r.uniform(1.3, 2.0)             # capacity, req/s
        A = r.uniform(0.3, 0.7)                   # diurnal amplitude
        phi = r.uniform(0.0, STEPS_PER_DAY)       # diurnal phase
        t_r0 = r.uniform(0.5, 3.0)                # base execution time, s
        mns = math.floor(cap * t_r0 * r.uniform(1.0, 1.5)) + 1   # max_num_seqs
        m0 = r.uniform(0.3, 0.6)
        out_len = r.uniform(150.0, 500.0)
        par[i] = (L, cap, t_r0, mns, m0, out_len, A, phi)
        e = r.standard_normal(T)
        ar1 = lfilter([math.sqrt(1.0 - 0.81)], [1.0, -0.9], e)
        lam_i = (L * (1.0 + A * np.sin(2 * np.pi * (t + phi) / STEPS_PER_DAY))
                 * (1.0 + 0.1 * np.sin(2 * np.pi * t / STEPS_PER_WEEK))
                 * np.exp(0.05 * ar1))
        # injected events: Poisson, ~1 per 2880 steps; surge p=0.6, drop p=0.4
        n_ev = r.poisson(T / 2880.0)
        for _ in range(n_ev):
            s = int(r.integers(0, T))
            d = int(r.integers(5, 61))
            if r.uniform() < 0.6:
                lam_i[s:s + d] *= r.uniform(1.5, 3.0)
                labels[i, s:s + d] = 1
            else:
                lam_i[s:s + d] *= r.uniform(0.05, 0.4)
                labels[i, s:s + d] = -1
        lam[i] = lam_i
        arrivals[i] = r.poisson(60.0 * lam_i) / 60.0
        noise[i] = r.standard_normal((T, M))

    L, cap, t_r0, mns, m0, out_len = (par[:, k:k + 1] for k in range(6))
    # pending queue (Lindley recursion): grows when arrivals exceed capacity
    #
    Q = np.empty((N, T))
    served = np.empty((N, T))
    q = np.zeros(N)
    capv = cap[:, 0]
    for k in range(T):
        want = arrivals[:, k] + q / 60.0
        sv = np.minimum(want, capv)
        q = np.maximum(0.0, q + 60.0 * (arrivals[:, k] - capv))
        served[:, k] = sv
        Q[:, k] = q
    ns = noise
    g_u = np.clip(served / cap + 0.02 * ns[..., 6], 0.0, 1.0)
    t_r = t_r0 * (1.0 + 0.5 * g_u ** 2) + Q / (60.0 * cap) + 0.01 * t_r0 * ns[..., 4]
    n_r = np.minimum(served * t_r, mns) * (1.0 + 0.02 * ns[..., 1])
    n_f = served * (1.0 + 0.02 * ns[..., 0])
    n_a = arrivals + 0.01 * L * ns[..., 2]
    n_p = Q + np.abs(0.5 * ns[..., 3])
    k_mem = (0.9 - m0) / mns
    m_u = np.clip(m0 + k_mem * n_r + 0.01 * ns[..., 5], 0.0, 1.0)   # Eq. 6 linear form
    kv = np.clip(n_r / mns + 0.02 * Q / (60.0 * cap) + 0.01 * ns[..., 7], 0.0, 1.0)
    chans = [n_f, n_r, n_a, n_p, t_r, m_u, g_u, kv]
    # extra channels (M >= 16): derived from the above with independent noise
    j = 8
    while len(chans) < M:
        nz = ns[..., j]
        which = (j - 8) % 8
        if which == 0:
            c = n_f * out_len * (1.0 + 0.03 * nz)                     # tokens/s
        elif which == 1:
            c = 0.2 + Q / (60.0 * cap) + 0.02 * g_u + 0.01 * nz        # TTFT
        elif which == 2:
            c = 0.02 * (1.0 + g_u) * (1.0 + 0.02 * nz)                 # TPOT
        elif which == 3:
            c = Q / (60.0 * cap) + 0.005 * np.abs(nz)                  # queue time
        elif which == 4:
            c = n_a * 400.0 * (1.0 + 0.03 * nz)                        # prefill tokens/s
        elif which == 5:
            c = n_f * out_len * (1.0 + 0.03 * nz)                      # decode tokens/s
        elif which == 6:
            c = 200.0 + 500.0 * g_u + 5.0 * nz                         # power, W
        else:
            c = np.clip(0.9 * g_u + 0.02 * nz, 0.0, 1.0)               # SM occupancy
        chans.append(c)
        j += 1
    X = np.stack(chans[:M], axis=-1).astype(np.float32)
    if return_labels:
        return X, labels
    return X


def detector_weights(window: int, n_metrics: int, hidden: int, latent: int,
                     seed: int = DEFAULT_SEED) -> dict:
    """Random-init detector (SPEC.md:547 topology: D -> H -> (mu, logvar) Z;
    Z -> H -> D, tanh, linear output), Xavier normal N(0, 1/fan_in), logvar
    head 0.3/sqrt(fan_in), biases N(0, 0.1^2); all rounded to fp16-representable
    fp32.  Layouts follow include/enova.h (row-major [out][in])."""
    D = window * n_metrics
    r = _rng(seed, 0xDE7EC7)
    def g(shape, std):
        return fp16_representable(r.standard_normal(shape) * std)
    return dict(
        window=window, n_metrics=n_metrics, hidden=hidden, latent=latent,
        enc_w1=g((hidden, D), 1.0 / math.sqrt(D)), enc_b1=g((hidden,), 0.1),
        enc_wmu=g((latent, hidden), 1.0 / math.sqrt(hidden)), enc_bmu=g((latent,), 0.1),
        enc_wlv=g((latent, hidden), 0.3 / math.sqrt(hidden)), enc_blv=g((latent,), 0.1),
        dec_w1=g((hidden, latent), 1.0 / math.sqrt(latent)), dec_b1=g((hidden,), 0.1),
        dec_w2=g((D, hidden), 1.0 / math.sqrt(hidden)), dec_b2=g((D,), 0.1),
    )


# c5 mixture constants: bulk = 0.5 * chi2_16 (KL of a 16-dim posterior with
# mu ~ N(0, I), lv = 0); tail weight 1e-3 from u99 + GPD(xi=0.25, sigma=2),
# u99 = 0.5 * chi2_16 99th percentile = 0.5 * 31.99993 (scipy.stats.chi2.ppf).
C5_TAIL_WEIGHT = 1e-3
def _trace_block(args):
    n, T, M, seed, off, labels = args
    return metric_trace(n, T, M, seed=seed, instance_offset=off, return_labels=labels)


def metric_trace_parallel(n_instances: int, n_steps: int, n_metrics: int = 16,
                          seed: int = DEFAULT_SEED, instance_offset: int = 0,
                          workers: int | None = None, block: int = 32,
                          return_labels: bool = False):
    """``metric_trace`` generated over a process pool in instance blocks; equal
    to the serial call bit for bit (every instance has its own Philox stream)."""
    import os
    from concurrent.futures import ProcessPoolExecutor
    N = int(n_instances)
    if workers is None:
        try:
            workers = len(os.sched_getaffinity(0))
        except AttributeError:
            workers = os.cpu_count() or 1
    if workers <= 1 or N <= block:
        return metric_trace(N, n_steps, n_metrics, seed=seed, instance_offset=instance_offset,
                            return_labels=return_labels)
    jobs = [(min(block, N - a), n_steps, n_metrics, seed, instance_offset + a, return_labels)
            for a in range(0, N, block)]
    out = np.empty((N, int(n_steps), int(n_metrics)), dtype=np.float32)
    lab = np.empty((N, int(n_steps)), dtype=np.int8) if return_labels else None
    import multiprocessing as mp
    # forkserver: the caller may be multi-threaded (torch), where fork() can deadlock
    with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("forkserver")) as ex:
        a = 0
        for blk in ex.map(_trace_block, jobs):
            if return_labels:
                blk, lb = blk
                lab[a:a + blk.shape[0]] = lb
            out[a:a + blk.shape[0]] = blk
            a += blk.shape[0]
    return (out, lab) if return_labels else out


C5_U99 = 0.5 * 31.999926908815176
C5_XI, C5_SIGMA = 0.25, 2.0
_CHUNK = 1 << 20


def score_mixture(n: int, seed: int = DEFAULT_SEED + 5, offset: int = 0) -> np.ndarray:
    """c5 calibration scores, elements [offset, offset+n) of an infinite seeded
    stream (chunked Philox so shards regenerate identically), fp32."""
    out = np.empty(n, dtype=np.float32)
    pos = offset
    w = 0
    while w < n:
        c = pos // _CHUNK
        lo = pos - c * _CHUNK
        take = min(_CHUNK - lo, n - w)
        r = _rng(seed, c)
        bulk = 0.5 * r.chisquare(16, _CHUNK)
        u = r.uniform(size=_CHUNK)
        v = r.uniform(size=_CHUNK)
        tail = C5_U99 + C5_SIGMA / C5_XI * (v ** (-C5_XI) - 1.0)
        vals = np.where(u < C5_TAIL_WEIGHT, tail, bulk)
        out[w:w + take] = vals[lo:lo + take]
        w += take
        pos += take
    return out


# Paper-scale configurations (BASELINE.json "configs").
CONFIGS = {
    "c1": dict(n_instances=1, n_steps=2000, n_metrics=8, window=32, hidden=32, latent=4),
    "c2": dict(n_instances=256, n_steps=10000, n_metrics=16, window=64, hidden=128, latent=16),
    "c3": dict(n_instances=4096, n_steps=50000, n_metrics=16, window=64, hidden=128, latent=16),
    "c4": dict(n_instances=10000, n_steps=64, n_metrics=16, window=64, hidden=128, latent=16),
    "c5": dict(n_scores=100_000_000),
}


# SPEC.md's synthetic detection benchmark: normals from a
# correlated 8-dim Gaussian (Table II's 7 metrics + KV-cache utilisation),
# anomalies injected as level shifts of the load metrics in contiguous
# segments, ~1% of the points; half of the anomaly segments carry a label for
# the semi-supervised training of Eq. 9.  Magnitudes (the spec
# leaves them open): surges +U(5, 10) sigma, drops -U(5, 10) sigma on
# n_f, n_r, n_a, n_p and kv; segment lengths U{5..30}; gaps Exp(mean 1500).
SPEC_BENCH_RHO = 0.6
SPEC_BENCH_LOAD = (0, 1, 2, 3, 7)


def spec_benchmark(n_instances: int, n_steps: int, seed: int = DEFAULT_SEED,
                   instance_offset: int = 0, return_train_labels: bool = False):
    """Returns (X [N, T, 8] fp32, labels [N, T] int8 +1 surge / -1 drop / 0), and
    with return_train_labels also l [N, T] int8 (+1 normal or unlabelled, -1 a
    point of a LABELLED anomaly segment: 50% of the segments, drawn per segment)."""
    N, T, M = int(n_instances), int(n_steps), 8
    C = SPEC_BENCH_RHO ** np.abs(np.subtract.outer(np.arange(M), np.arange(M)))
    Lc = np.linalg.cholesky(C)
    X = np.empty((N, T, M), np.float32)
    lab = np.zeros((N, T), np.int8)
    tl = np.ones((N, T), np.int8)
    load = list(SPEC_BENCH_LOAD)
    for i in range(N):
        r = _rng(seed ^ 0x5BEC, instance_offset + i)
        x = r.standard_normal((T, M)) @ Lc.T
        t = 0
        while True:
            t += int(r.exponential(1500.0))
            if t >= T:
                break
            d = int(r.integers(5, 31))
            sgn = 1 if r.uniform() < 0.6 else -1
            mag = r.uniform(5.0, 10.0)
            x[t:t + d, load] += sgn * mag
            lab[i, t:t + d] = sgn
            if r.uniform() < 0.5:
                tl[i, t:t + d] = -1
            t += d
        X[i] = x.astype(np.float32)
    if return_train_labels:
        return X, lab, tl
    return X, lab


def noise_normal(n: int, z: int, seed: int, step: int) -> np.ndarray:
    """The reparameterisation noise eps [n, z] of training step `step` (fp32)."""
    return _rng(seed ^ 0xE95, step).standard_normal((n, z)).astype(np.float32)


def epoch_order(n: int, seed: int, epoch: int) -> np.ndarray:
    """The window order of training epoch `epoch` (a permutation of [0, n))."""
    return _rng(seed ^ 0x0DE, epoch).permutation(n).astype(np.int64)
