"""Diagnostic (not the bench): c2 step time of the sequential and the overlapped
enova_step (threshold fit on pot_ctas CTAs next to the detection scores of the
first `concurrent` instances), CUDA graphs, L2 flushed between steps; outputs
checked equal to the sequential step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import synth  # noqa: E402


def time_pipe(pipe, X, flush, reps=20):
    pipe.capture(X)
    for _ in range(3):
        pipe.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        pipe.replay()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), pipe.result()


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = synth.CONFIGS[wl]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    N = 256 if wl == "c2" else cfg["n_instances"] // 8
    X = torch.from_numpy(synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2)).cuda()
    det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    base = E.Pipeline(det, N, T, T // 2, overlap=False)
    t0, r0 = time_pipe(base, X, flush)
    ref = (r0.scores.clone(), r0.md.clone(), r0.flags.clone(), r0.cal_flags.clone(), r0.threshold)
    print(f"{wl} sequential: {t0 * 1e3:.1f} us  z_q {r0.threshold['z_q']:.9f}", flush=True)
    pots = [int(v) for v in os.environ.get('POTS', '16,32,48').split(',')]
    fracs = [float(v) for v in os.environ.get('FRACS', '0.2,0.3,0.4,0.5').split(',')]
    for pot in pots:
        for frac in fracs:
            p = E.Pipeline(det, N, T, T // 2, pot_ctas=pot, concurrent_instances=int(frac * N))
            t, r = time_pipe(p, X, flush)
            same = (torch.equal(r.scores, ref[0]) and torch.equal(r.md, ref[1]))
            dz = abs(r.threshold["z_q"] - ref[4]["z_q"]) / ref[4]["z_q"]
            fl = int((r.flags != ref[2]).sum()) + int((r.cal_flags != ref[3]).sum())
            print(f"{wl} overlap pot_ctas={pot} concurrent={frac:.1f}: {t * 1e3:.1f} us "
                  f"({t0 / t:.3f}x)  scores/md equal {same}  dz_q {dz:.1e}  flag diffs {fl}",
                  flush=True)
            del p


if __name__ == "__main__":
    main()
