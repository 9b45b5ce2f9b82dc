"""Pipeline timeline of the CTA-pair scorer (CTA pair 0, %globaltimer ns).
Diagnostic only: rebuilds libenova.so with -DENOVA_TRACE (the stamps are
compiled out of the default build); rebuild without it afterwards."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
os.environ["ENOVA_NVCC_FLAGS"] = "-DENOVA_TRACE"
from paper_2407_09486_b200 import build as _B  # noqa: E402
_B.build()
import paper_2407_09486_b200 as E  # noqa: E402
from paper_2407_09486_b200 import _lib, synth  # noqa: E402
cfg = synth.CONFIGS["c2"]
W, M, H, Z, T, N = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"], cfg["n_instances"]
X = torch.from_numpy(synth.metric_trace(N, T, M, seed=7)).cuda()
det = E.PreparedDetector(synth.detector_weights(W, M, H, Z, seed=7))
mean, std, _ = E.compute_stats(X, T // 2)
tr = torch.zeros(4 * 512 * 16, dtype=torch.int64, device="cuda")
E.score_windows(X, det, mean, std, W - 1, T // 2)
_lib.lib().enova_internal_set_trace.argtypes = [C.c_void_p]
_lib.lib().enova_internal_set_trace(C.c_void_p(tr.data_ptr()))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
E.score_windows(X, det, mean, std, W - 1, T // 2)
e1.record()
torch.cuda.synchronize()
print("traced launch", e0.elapsed_time(e1) * 1e3, "us")
_lib.lib().enova_internal_set_trace(None)
t = tr.view(4, 512, 16).cpu().numpy().astype(np.float64)
for c in range(4):
    st, en = t[c, 500, 15], t[c, 501, 15]
    n = int((t[c, :500, 14] > 0).sum())
    first = t[c, 0, 0] if c % 2 == 0 else t[c, 0, 13]
    print(f"cta slot {c}: kernel body {(en - st) / 1e3:.1f} us, prologue to first iter {(t[c, 0, 1] - st) / 1e3 if c % 2 == 0 else 0:.1f} us, iterations {n}")
gstart = min(t[c, 500, 15] for c in range(4)); gend = max(t[c, 501, 15] for c in range(4))
names = {0: "mma: iter start", 1: "mma: planes ready", 2: "mma: G1 issued", 3: "mma: h ready(G2 i-1)",
         4: "mma: G2 issued", 5: "mma: mu+dec ready (G3 i-2)", 6: "epi: E1 wait start", 7: "epi: E1 acc full",
         8: "epi: E1 done", 9: "epi: E3 dec full", 10: "epi: E3 done", 11: "epi: E2 heads full",
         12: "epi: E2 done", 13: "stage: start wait", 14: "stage: sx done"}
a = t[0]
n = int((a[:, 14] > 0).sum())
print("iterations", n, "period", np.diff(a[5:n - 2, 0]).mean(), "ns")
t0 = a[10, 0]
for it in range(10, 12):
    ev = []
    for k in range(15):
        for cta in (0, 1):
            arr = t[cta]
            if arr[it, k] > 0 and (cta == 0 or k >= 6):
                ev.append(((arr[it, k] - t0) / 1e3, f"c{cta} {names[k]} [tile/iter {it}]"))
    for x, nme in sorted(ev):
        print(f"   {x:8.3f}  {nme}")

print("staging detail (CTA0), us: waits-done -> planes-loop-done -> planes_full -> sx done")
for it in range(8, 16):
    r = t[0, 256 + it]
    print(f"  tile {it}: start {(t[0, it, 13] - t0) / 1e3:7.3f} waits-done {(r[0] - t0) / 1e3:7.3f} loop {(r[1] - t0) / 1e3:7.3f} full {(r[2] - t0) / 1e3:7.3f} sx {(t[0, it, 14] - t0) / 1e3:7.3f}")
print("per-tile summary (CTA0, us rel. to tile-10 MMA start):")
print("  tile | mma start  planes  G1    h     G2    mu/dec | stg wait-done loop full | E1 acc  E1 done | E2 hf  E2 done | E3 df  E3 done")
for it in range(8, 16):
    a = t[0]; r = a[256 + it]
    f = lambda v: f"{(v - t0) / 1e3:6.2f}"
    print(f"  {it:4d} | {f(a[it,0])} {f(a[it,1])} {f(a[it,2])} {f(a[it,3])} {f(a[it,4])} {f(a[it,5])} | {f(r[0])} {f(r[1])} {f(r[2])} | {f(a[it,7])} {f(a[it,8])} | {f(a[it,11])} {f(a[it,12])} | {f(a[it,9])} {f(a[it,10])}")
