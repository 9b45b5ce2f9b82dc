"""Diagnostic (build with ENOVA_NVCC_FLAGS=-DENOVA_FIT_STAMPS): the binned Halley
steps of the last fit -- per pass and root the relative step |x_new - x| / |x|
(negative when the step left the fp64 bracket and was clamped) -- read from the
k_pot stamp slots 72..88, for the c5 mixture and the binned-test tails."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import _lib, synth  # noqa: E402


def show(s, label):
    import ctypes as C
    ws = E.ThresholdWorkspace(s.numel())
    t = E.fit_threshold(s, 0.98, 1e-3, workspace=ws)
    no, so = C.c_int64(), C.c_int64()
    _lib.lib().enova_internal_pot_stamp_offsets(C.byref(no), C.byref(so))
    st = ws.buf[so.value:so.value + 8 * 96].cpu().numpy().view(np.uint64)
    d = st[72:88].view(np.float64).reshape(4, 4)
    nr = int(st[88])
    print(f"[{label}] n_peaks={t['n_peaks']} z_q={t['z_q']:.6f} gamma={t['gamma']:.5f} roots refined={nr}")
    for it in range(4):
        print("  pass", it, " ".join(f"{v:+.3e}" for v in d[it, :max(nr, 1)]))


def main():
    show(torch.from_numpy(synth.score_mixture(100_000_000)).cuda(), "c5 mixture")
    r = np.random.default_rng(101)
    show(torch.from_numpy(r.exponential(1.0, 6_000_000).astype(np.float32)).cuda(), "exp 6M")
    show(torch.from_numpy(r.gamma(2.0, 1.0, 6_000_000).astype(np.float32)).cuda(), "gamma 6M")


if __name__ == "__main__":
    main()
