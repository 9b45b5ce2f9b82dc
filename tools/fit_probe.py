"""Probe of enova_fit_threshold on the c2 calibration-score shape (1.26M scores):
wall time per call and the device-state trace (not a bench number)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_09486_b200 as E
from paper_2407_09486_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1263872
s = torch.from_numpy(synth.score_mixture(n, seed=3)).cuda()
ws = E.ThresholdWorkspace(n, 0.98)
for _ in range(3):
    thr = E.fit_threshold(s, workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    thr = E.fit_threshold(s, workspace=ws)
torch.cuda.synchronize()
print(f"n={n} fit wall {1e3*(time.perf_counter()-t0)/20:.3f} ms  n_peaks={thr['n_peaks']} gamma={thr['gamma']:.6f}")
