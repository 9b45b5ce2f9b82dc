"""NEXT-3 robustness sweep on the GPU trainer (diagnostic, not a test): point-
adjusted F1 of the SPEC synthetic benchmark over seeds and schedules.

  python tools/train_sweep.py [epochs,lr,batch ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402
from tests import train_bench as TB  # noqa: E402


def run(X, lab, tl, epochs, lr, batch, seed, n_inst):
    W, M, H, Z = TB.W, TB.M, TB.H, TB.Z
    Xc = torch.from_numpy(X).cuda()
    mean, std, _ = E.compute_stats(Xc, TB.TCAL)
    nw = TB.TCAL - (W - 1)
    n = X.shape[0] * nw
    l = torch.from_numpy(TB.train_labels(tl).astype(np.int8)).cuda()
    r = np.random.default_rng(1000 + seed)
    per = -(-n // batch) * batch
    order = np.full(epochs * per, -1, np.int64)
    for e in range(epochs):
        order[e * per:e * per + n] = r.permutation(n)
    steps = len(order) // batch
    eps = r.standard_normal((steps * batch, Z)).astype(np.float32)
    w0 = synth.detector_weights(W, M, H, Z, seed=TB.SEED + seed)
    tr = E.Trainer(W, M, H, Z, max_batch=batch)
    tr.load(w0)
    t0 = time.perf_counter()
    tr.fit(Xc, mean, std, W - 1, TB.TCAL, l, torch.from_numpy(order).cuda(),
           torch.from_numpy(eps).cuda(), batch, E.train_config(lr=lr, latent=Z))
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    wts = tr.weights()
    tr.destroy()
    det = E.PreparedDetector(wts)
    cal, _ = E.score_windows(Xc, det, mean, std, W - 1, TB.TCAL)
    normal = torch.from_numpy(lab[:, W - 1:TB.TCAL] == 0).cuda()
    thr = E.fit_threshold(cal[normal].contiguous(), 0.98, 1e-3)
    flags = E.detect(Xc, det, mean, std, thr, TB.TCAL, TB.T)
    pa = E.point_adjusted_f1(torch.from_numpy(lab).cuda(), flags, TB.TCAL)
    return pa["f1"], pa["precision"], pa["recall"], ts


def main():
    cfgs = [a.split(",") for a in sys.argv[1:]] or [["10", "3e-3", "64"]]
    out = []
    for n_inst in (16,):
        X, lab, tl = synth.spec_benchmark(n_inst, TB.T, seed=TB.SEED, return_train_labels=True)
        for c in cfgs:
            ep, lr, b = int(c[0]), float(c[1]), int(c[2])
            f1s = []
            for seed in range(8):
                f1, p, rc, ts = run(X, lab, tl, ep, lr, b, seed, n_inst)
                f1s.append(f1)
                print(json.dumps(dict(n=n_inst, epochs=ep, lr=lr, batch=b, seed=seed, f1=f1, p=p,
                                      r=rc, train_s=ts)), flush=True)
            out.append(dict(epochs=ep, lr=lr, batch=b, f1_min=min(f1s), f1_median=float(np.median(f1s))))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
