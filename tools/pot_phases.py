"""Phase timeline of the threshold kernel k_pot (diagnostic, run under gpurun).

Scores the c2 calibration windows, then runs enova_fit_threshold_async a few
times and prints CTA 0's %globaltimer stamps at every phase boundary / fit pass
(PotGlobal.stamps, threshold.cu) plus the event-timed launch duration.
Also runs the c5 mixture (100M scores) when "--c5" is given.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402



def _offsets():
    import ctypes as C
    from paper_2407_09486_b200 import _lib
    no, so = C.c_int64(), C.c_int64()
    _lib.lib().enova_internal_pot_stamp_offsets(C.byref(no), C.byref(so))
    return no.value, so.value


def report(scores, label, reps=5):
    ws = E.ThresholdWorkspace(scores.numel())
    thr = torch.zeros(E.api.THRESHOLD_BYTES, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        E.fit_threshold_async(scores, workspace=ws, out=thr)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        E.fit_threshold_async(scores, workspace=ws, out=thr)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    OFF_NSTAMPS, OFF_STAMPS = _offsets()
    head = ws.buf[:OFF_STAMPS + 8 * 98].cpu().numpy()
    n = int(head[OFF_NSTAMPS:OFF_NSTAMPS + 4].view(np.int32)[0])
    passes = int(head[OFF_NSTAMPS + 4:OFF_NSTAMPS + 8].view(np.int32)[0])
    allst = head[OFF_STAMPS:OFF_STAMPS + 8 * 98].view(np.uint64)
    st = allst[:min(n, 95)].astype(np.int64)
    k0 = int(allst[95])
    first = int(~allst[96] & np.uint64(0xFFFFFFFFFFFFFFFF))
    last = int(allst[97])
    print(f"  CTA0 entry -> first stamp {(st[0]-k0)/1e3:.1f} us; first CTA start -> CTA0 entry "
          f"{(k0-first)/1e3:.1f} us; last stamp -> last CTA end {(last-st[-1])/1e3:.1f} us; "
          f"first start -> last end {(last-first)/1e3:.1f} us")
    d = np.diff(st) / 1e3
    t = E.threshold_from_device(thr)
    print(f"[{label}] n={scores.numel()} peaks={t['n_peaks']} launch median {np.median(ms)*1e3:.1f} us; "
          f"stamps={n} refine passes={passes}; total stamped {(st[-1]-st[0])/1e3:.1f} us")
    print("  deltas (us):", " ".join(f"{x:.1f}" for x in d))


def main():
    cfg = synth.CONFIGS["c2"]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    X = torch.from_numpy(synth.metric_trace(256, T, M, seed=synth.DEFAULT_SEED + 2)).cuda()
    det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2))
    mean, std, _ = E.compute_stats(X, T // 2)
    cal, _ = E.score_windows(X, det, mean, std, W - 1, T // 2, with_md=False)
    report(cal.reshape(-1), "c2 calibration")
    mix = torch.from_numpy(synth.score_mixture(2_000_000)).cuda()
    report(mix, "mixture 2M")
    if "--c5" in sys.argv:
        big = torch.from_numpy(synth.score_mixture(100_000_000)).cuda()
        report(big, "c5 100M", reps=3)


if __name__ == "__main__":
    main()
