"""Minimal c2 pipeline driver for ncu captures (never a bench number).

  ncu --set full -k regex:k_score -s 2 -c 1 -o gpurun_out/prof python tools/profile_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = synth.CONFIGS["c2"]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    N = cfg["n_instances"]
    X = torch.from_numpy(synth.metric_trace(N, T, M, seed=synth.DEFAULT_SEED + 2)).cuda()
    det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2))
    for _ in range(steps):
        E.run_pipeline(X, det, T // 2)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
