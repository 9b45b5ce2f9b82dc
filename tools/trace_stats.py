"""Timeline of CTA 0 of K1 (k_series_stats), c2 shape: chunk issue / arrival
and per-instance segment epilogues.  Diagnostic only (enova_internal_set_trace)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["ENOVA_NVCC_FLAGS"] = "-DENOVA_TRACE"   # stamps are compiled out by default
from paper_2407_09486_b200 import build as _B  # noqa: E402
_B.build()
import paper_2407_09486_b200 as E
from paper_2407_09486_b200 import _lib, synth


def main():
    cfg = synth.CONFIGS["c2"]
    N, T, M = cfg["n_instances"], cfg["n_steps"], cfg["n_metrics"]
    X = torch.from_numpy(synth.metric_trace_parallel(N, T, M, seed=3)).cuda()
    for _ in range(3):
        E.compute_stats(X, T // 2)
    torch.cuda.synchronize()
    tr = torch.zeros(96, dtype=torch.int64, device="cuda")
    L = _lib.lib()
    L.enova_internal_set_trace.argtypes = [C.c_void_p]
    L.enova_internal_set_trace(C.c_void_p(tr.data_ptr()))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    E.compute_stats(X, T // 2)
    e1.record()
    torch.cuda.synchronize()
    L.enova_internal_set_trace(None)
    t = tr.cpu().numpy().astype(np.float64)
    z = t[0]
    f = lambda i: f"{(t[i] - z) / 1e3:.2f}" if t[i] else "-"
    print(f"call {e0.elapsed_time(e1) * 1e3:.1f} us (incl. host)")
    print("chunk issued (us):", " ".join(f(1 + k) for k in range(24)))
    print("chunk ready  (us):", " ".join(f(32 + k) for k in range(24)))
    print("segment epilogue start/end (us):", " ".join(f"{f(64 + 2 * s)}/{f(65 + 2 * s)}" for s in range(8)))
    print("end", f(95))


if __name__ == "__main__":
    main()
