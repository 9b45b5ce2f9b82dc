"""Minimal c5 threshold driver for ncu captures (never a bench number)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    s = torch.from_numpy(synth.score_mixture(synth.CONFIGS["c5"]["n_scores"])).cuda()
    ws = E.ThresholdWorkspace(s.numel())
    thr = torch.zeros(E.api.THRESHOLD_BYTES, dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        E.fit_threshold_async(s, workspace=ws, out=thr)
    torch.cuda.synchronize()
    print(E.threshold_from_device(thr))


if __name__ == "__main__":
    main()
