"""Diagnostic: where the c2 threshold fit's launch time goes (not a bench).

Times k_pot (fit_threshold_async on the c2 calibration score count) with CUDA
events: (a) back to back, (b) right after a K2 calibration launch, and reads
the kernel's own %globaltimer span (first CTA start -> last CTA end)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import _lib, synth  # noqa: E402


def main():
    cfg = synth.CONFIGS["c2"]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    N = cfg["n_instances"]
    X = torch.from_numpy(synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2)).cuda()
    det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2))
    tcal = T // 2
    mean, std, _ = E.compute_stats(X, tcal)
    cal, md = E.score_windows(X, det, mean, std, W - 1, tcal)
    ws = E.ThresholdWorkspace(cal.numel())
    thr = torch.zeros(E.api.THRESHOLD_BYTES, dtype=torch.uint8, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()

    def span():
        no, so = C.c_int64(), C.c_int64()
        _lib.lib().enova_internal_pot_stamp_offsets(C.byref(no), C.byref(so))
        head = ws.buf[:so.value + 8 * 96].cpu().numpy()
        st = head[so.value:so.value + 8 * 96].view(np.uint64).astype(np.int64)
        # t_first_start (complemented), t_last_end follow the stamps
        return st

    for mode in ("back_to_back", "after_k2"):
        for _ in range(3):
            E.fit_threshold_async(cal, workspace=ws, out=thr)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            if mode == "after_k2":
                E.score_windows(X, det, mean, std, W - 1, tcal, out=(cal, md))
            a, b = ev(), ev()
            a.record(s)
            E.fit_threshold_async(cal, workspace=ws, out=thr)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        print(mode, "event us: median %.1f min %.1f" % (np.median(ts), np.min(ts)))
    # kernel span from the device stamps of the last launch
    no, so = C.c_int64(), C.c_int64()
    _lib.lib().enova_internal_pot_stamp_offsets(C.byref(no), C.byref(so))
    raw = ws.buf[:4096].cpu().numpy()
    ns = int(raw[no.value:no.value + 4].view(np.int32)[0])
    st = raw[so.value:so.value + 8 * 96].view(np.uint64).astype(np.int64)
    print("stamps", ns, "CTA0 span us %.1f" % ((st[ns - 1] - st[0]) / 1e3),
          "deltas", np.round(np.diff(st[:ns]) / 1e3, 1).tolist())


if __name__ == "__main__":
    main()
