"""Time the CTA-pair scorer alone on the c2 calibration range (diagnostic A/B
driver for tools/k2_ab.sh; never a bench number): prints the mean of 20
back-to-back launches after 3 warm-ups, CUDA events on the launching stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402

cfg = synth.CONFIGS["c2"]
W, M, H, Z, T, N = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"], cfg["n_instances"]
X = torch.from_numpy(synth.metric_trace(N, T, M, seed=7)).cuda()
det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=7))
mean, std, _ = E.compute_stats(X, T // 2)
for _ in range(3):
    E.score_windows(X, det, mean, std, W - 1, T // 2)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    E.score_windows(X, det, mean, std, W - 1, T // 2)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nwin = N * (T // 2 - W + 1)
print(f"{os.environ.get('ENOVA_NVCC_FLAGS', '') or 'base'}: {ms:.4f} ms/launch  "
      f"{274432 * nwin / ms / 1e9:.1f} TFLOP/s")
