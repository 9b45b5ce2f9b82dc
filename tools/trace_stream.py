"""Timeline of CTA 0 of the TMA-fed stream row kernel (k_stream_rows), c4 shape.
Diagnostic only (uses enova_internal_set_trace)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["ENOVA_NVCC_FLAGS"] = "-DENOVA_TRACE"   # stamps are compiled out by default
from paper_2407_09486_b200 import build as _B  # noqa: E402
_B.build()
import paper_2407_09486_b200 as E
from paper_2407_09486_b200 import _lib, synth
cfg = synth.CONFIGS["c4"]
W, M, H, Z, N = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else cfg["n_instances"]
T = 200
X = torch.from_numpy(synth.metric_trace(N, T, M, seed=3)).cuda()   # serial: no process pool in a script without a main guard
det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=3))
mean, std, _ = E.compute_stats(X, T)
ring = E.StreamRing(det, mean, std)
for k in range(W):
    ring.push(X[:, k].contiguous(), k)
thr = E.threshold_to_device({"z_q": 2.0})
for _ in range(3):
    ring.detect(W - 1, thr)
torch.cuda.synchronize()
busy = "--busy" in sys.argv
if busy:   # keep the GPU busy right before the traced launch (clock ramp-up)
    for _ in range(200):
        ring.detect(W - 1, thr)
tr = torch.zeros(96, dtype=torch.int64, device="cuda")
L = _lib.lib()
L.enova_internal_set_trace.argtypes = [C.c_void_p]
L.enova_internal_set_trace(C.c_void_p(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ring.detect(W - 1, thr)
e1.record()
torch.cuda.synchronize()
L.enova_internal_set_trace(None)
t = tr.cpu().numpy().astype(np.float64)
names = ["start", "prod: first A TMA", "prod: last A TMA", "mma: first", "mma: last G1",
         "rows: window sums", "rows: G1 done", "rows: E1 done", "rows: G2 done", "rows: E2 done",
         "rows: G3 done", "rows: E3 done"]
print(f"launch {e0.elapsed_time(e1) * 1e3:.1f} us")
for i, nm in enumerate(names):
    print(f"{nm:22s} {(t[i] - t[0]) / 1e3:8.2f} us")
print("E2 detail (us): tmem loaded %.2f, KL+pack+stores %.2f, fences+syncwarp %.2f" % tuple((t[i] - t[0]) / 1e3 for i in (12, 13, 14)))
print("A TMA issued (us):", " ".join(f"{(t[16 + g] - t[0]) / 1e3:.2f}" for g in range(16)))
print("A ready at MMA (us):", " ".join(f"{(t[36 + g] - t[0]) / 1e3:.2f}" for g in range(16)))

print("W1 stage issued (us):", " ".join(f"{(t[56 + g] - t[0]) / 1e3:.2f}" for g in range(16)))
print("W1 ready at MMA (us):", " ".join(f"{(t[72 + g] - t[0]) / 1e3:.2f}" for g in range(16)))
