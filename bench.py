#!/usr/bin/env python
"""Benchmark of the ENOVA detection hot path on B200 (BASELINE.json metric:
metric-windows scored/sec at 1/2/4/8 B200 and % of the tensor-pipe roofline).

One step = one pass of the whole hot path over one batch:
  stats over the calibration horizon [0, T/2)            (a-1, K1)
  -> scores of every calibration window                  (a-2..a-5, K2)
  -> fleet-wide POT threshold (NCCL across ranks)        (a-7..a-9, K3-K5)
  -> scores / MD / flags of every detection window       (a-2..a-6, K2)
so every window of the trace is scored exactly once per step.

Workloads (BASELINE.json configs; --workload, default c2 = the headline):
  c2  256 instances x T=10000 x M=16 per GPU, W=64, benchmark detector H=128,
      Z=16; weak scaling: rank r owns global instances [256 r, 256 (r+1)).
  c3  the c3 fleet's per-GPU shard: 512 of 4096 instances x T=50000 per GPU
      (at --gpus 8 exactly c3; weak scaling below that).
  c4  streaming: 10000 instances, one new sample per instance per tick; a step
      is one tick (ring push + scores/MD/flags of the 10000 windows ending now).
  c5  threshold calibration sweep: 100M seeded scores (strong scaling: rank r
      holds a contiguous shard), a step is one fleet-wide POT fit.
Inputs are synthetic (paper_2407_09486_b200.synth).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c3|c4|c5]
  torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "metric-windows scored/sec at 1/2/4/8 B200; % HBM / tensor-pipe roofline"
UNIT = "windows/s"
INST_PER_GPU = 256


def flops_per_window(D, H, Z):
    # algorithmic tensor FLOPs: GEMM1 2DH + heads 2H(2Z) + decoder layer 1 2ZH
    return 2 * D * H + 2 * H * 2 * Z + 2 * Z * H


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sus=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0,
                source="fallback (B200_PROFILING.md)")


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        load = [v for v in sm if v > 0.5 * (mx or max(sm))] or sm
        return {"sm_mhz": float(np.median(load)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.lower().startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


SPEC_F16_TFLOPS = 2250.0    # B200 dense fp16/bf16 spec sheet (B200_PROFILING.md nominal table)
SPEC_HBM_GBS = 7700.0       # HGX B200 HBM3e spec sheet


def measure_traffic(kernel_regex, argv, timeout=240):
    """DRAM bytes (read + write) of ONE launch of the kernel, measured live with
    ncu in a subprocess (never timed: the bench numbers come from CUDA events in
    this process).  Returns (bytes, read, write) or None if ncu is unavailable."""
    import shutil
    ncu = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum", "--clock-control",
           "none", "-k", f"regex:{kernel_regex}", "-c", "1", "--csv", sys.executable] + argv
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    except (subprocess.TimeoutExpired, OSError):
        return None
    rd = wr = None
    import csv
    import io
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith('"')]
    for row in csv.reader(io.StringIO("\n".join(lines))):
        if len(row) < 3:
            continue
        name, unit, val = row[-3], row[-2], row[-1]
        try:
            v = float(val.replace(",", ""))
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                 "GB": 1e9}.get(unit, 1)
        if name == "dram__bytes_read.sum":
            rd = v * scale
        elif name == "dram__bytes_write.sum":
            wr = v * scale
    if rd is None or wr is None:
        return None
    return rd + wr, rd, wr


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_sample(X, wts, tcal, budget_s=15.0, min_inst=2):
    """Time the oracle (as it stands) on the first instances of the workload until
    ~budget_s of CPU work; returns (windows/s, windows, instances, seconds)."""
    from oracle import enova_oracle as O
    W = wts["window"]
    T = X.shape[1]
    t0 = time.perf_counter()
    n_inst = 0
    wins = 0
    while n_inst < X.shape[0]:
        Xi = X[n_inst:n_inst + 1]
        mean, std, _ = O.series_stats(Xi, tcal)
        cal, _ = O.score_windows(Xi, wts, mean, std, W - 1, tcal)
        sc, md = O.score_windows(Xi, wts, mean, std, tcal, T)
        n_inst += 1
        wins += cal.size + sc.size
        if n_inst >= min_inst and time.perf_counter() - t0 > budget_s:
            break
    # the fleet threshold on the sampled calibration scores (part of the step)
    t1 = time.perf_counter()
    el = t1 - t0
    return wins / el, wins, n_inst, el


def run_reference(args, rank, world):
    """--impl reference: the oracle (fp64 NumPy, as it stands) on the host cores,
    each step a bounded sample of the same workload."""
    if rank != 0:
        return
    from oracle import enova_oracle as O
    from paper_2407_09486_b200 import synth
    cfg = synth.CONFIGS["c2"]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    n_inst = 2
    X = synth.metric_trace(n_inst, T, M, seed=synth.DEFAULT_SEED + 2)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    tcal = T // 2

    def step():
        out = O.detect_pipeline(X, wts, tcal)
        return out["cal_scores"].size + out["scores"].size

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    wins = 0
    for _ in range(args.steps):
        wins += step()
    el = time.perf_counter() - t0
    v = wins / el
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "c2 sample: 2 instances x T=10000 x M=16, W=64, H=128, Z=16 "
                               "(stats -> calibration scores -> POT -> flags)",
                   "instances": n_inst, "windows_per_step": wins // args.steps},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu_cores(), "cpu_model": cpu_model(),
                         "kind": "oracle",
                         "sample": f"{n_inst} of 256 c2 instances, full T, whole pipeline"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _dist_setup(world, local_rank):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    return dev


def _pct(v, q):
    return float(np.percentile(np.asarray(v, dtype=np.float64), q))


def run_streaming(args, rank, world, local_rank):
    """c4: 10000 instances, one new sample per instance per
    tick; a step = one tick = ring push + scores/MD/flags of the windows ending
    at that tick, against stats and a fleet threshold frozen from the preceding
    calibration horizon.  Each tick is one CUDA graph replay (one graph per ring
    phase, tick mod W); the new samples come from a fixed device staging buffer
    (device-resident run: D2D copy from the pre-generated ticks; e2e run: H2D
    copy from pinned host memory, flags copied back every tick)."""
    import torch
    import torch.distributed as dist

    import paper_2407_09486_b200 as E
    from paper_2407_09486_b200 import _lib, synth
    from paper_2407_09486_b200.fleet import max_over_ranks, shard_range

    dev = _dist_setup(world, local_rank)
    cfg = synth.CONFIGS["c4"]
    W, M, H, Z = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"]
    n_global = cfg["n_instances"]
    a, b = shard_range(n_global, world, rank)
    n = b - a
    t_hist = 1024                         # calibration horizon before streaming starts
    ticks = args.warmup + args.steps
    T = t_hist + 2 * ticks
    Xh = synth.metric_trace_parallel(n, T, M, seed=synth.DEFAULT_SEED + 4, instance_offset=a)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 4)
    X = torch.from_numpy(Xh).to(dev)
    det = E.PreparedDetector(wts, device=dev)
    comm = E.Comm.create(rank, world, local_rank) if world > 1 else None
    hist = X[:, :t_hist]
    mean, std, _ = E.compute_stats(hist, t_hist)
    cal, _ = E.score_windows(hist, det, mean, std, W - 1, t_hist, with_md=False)
    thr = E.fit_threshold(cal, comm=comm)   # workspace sized for the summed count
    thr_dev = E.threshold_to_device(thr, dev)
    # samples of the streamed ticks, [tick][instance][metric]
    S = X[:, t_hist:].transpose(0, 1).contiguous()
    S_h = torch.from_numpy(np.ascontiguousarray(Xh[:, t_hist:].transpose(1, 0, 2))).pin_memory()
    # the ingest-normalised fp16 ring (enova_stream_*), filled with the W-1
    # samples before the first streamed tick
    ring = E.StreamRing(det, mean, std)
    for t in range(t_hist - W + 1, t_hist):
        ring.push(X[:, t].contiguous(), t)
    stage = torch.empty((n, M), dtype=torch.float32, device=dev)
    flags = torch.empty(n, dtype=torch.int8, device=dev)
    scores = torch.empty(n, dtype=torch.float32, device=dev)
    md = torch.empty(n, dtype=torch.float32, device=dev)

    def tick_ops(t):
        ring.step(stage, t, thr_dev, out=(flags, scores, md))   # one fused launch per tick

    l0 = _lib.lib().enova_kernel_launches()
    stage.copy_(S[0])
    tick_ops(t_hist)
    torch.cuda.synchronize()
    launches_per_tick = _lib.lib().enova_kernel_launches() - l0
    # one graph per ring phase
    side = torch.cuda.Stream(device=dev)
    graphs = {}
    side.wait_stream(torch.cuda.current_stream())
    for ph in range(W):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            tick_ops(ph + W)      # same ring phase, tick >= W-1
        graphs[ph] = g
    # device-resident run: one graph per tick whose launch reads that tick's
    # samples where they arrived (S[k], device memory) -- the tick is ONE graph
    # launch of ONE kernel, no staging copy
    tick_graphs = []
    for k in range(ticks):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            ring.step(S[k], t_hist + k, thr_dev, out=(flags, scores, md))
        tick_graphs.append(g)
    # e2e run: one graph per tick = the H2D copy of that tick's samples from pinned
    # host memory, the fused kernel, the D2H copy of the flags (one launch per tick)
    # (double-buffered: tick k's graph also copies tick k+1's samples into the
    # other staging buffer on a copy stream, overlapping the kernel; the first
    # tick's samples are copied before the run, the last graph prefetches nothing)
    flags_pin = torch.empty(n, dtype=torch.int8).pin_memory()
    stage2 = [torch.empty((n, M), dtype=torch.float32, device=dev) for _ in range(2)]
    cstream = torch.cuda.Stream(device=dev)
    e2e_graphs = []
    for k in range(ticks, 2 * ticks):
        j = k - ticks
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            if k + 1 < 2 * ticks:
                cstream.wait_stream(side)
                with torch.cuda.stream(cstream):
                    stage2[(j + 1) % 2].copy_(S_h[k + 1], non_blocking=True)
            ring.step(stage2[j % 2], t_hist + k, thr_dev, out=(flags, scores, md))
            flags_pin.copy_(flags, non_blocking=True)
            if k + 1 < 2 * ticks:
                side.wait_stream(cstream)
        e2e_graphs.append(g)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def run(k0, e2e, gate=False, per_tick=True, direct=False):
        starts, ends = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
        if e2e:
            stage2[0].copy_(S_h[k0], non_blocking=True)   # the first tick's samples (untimed)
        if gate:
            # a GPU-side spin (untimed, before the first start event) holds the
            # stream while the host enqueues every tick: the ticks then run back
            # to back and the events time the device, not the host's launch rate
            torch.cuda._sleep(3_000_000)
        for k in range(k0, k0 + ticks):
            i = k - k0 - args.warmup
            if i >= 0 and (per_tick or i == 0):
                starts[i].record(stream)
            if e2e:
                e2e_graphs[k - k0].replay()
            elif direct:   # the fused kernel launched straight through the C ABI
                ring.step(S[k], t_hist + k, thr_dev, out=(flags, scores, md))
            else:
                tick_graphs[k - k0].replay()
            if i >= 0 and (per_tick or i == args.steps - 1):
                ends[i].record(stream)
        torch.cuda.synchronize()
        lat = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)] if per_tick else []
        tot = starts[0].elapsed_time(ends[-1])
        return lat, tot

    if world > 1:
        dist.barrier()
    lat_host, tot_host = run(0, False)        # host-paced: one graph launch per tick from Python
    lat, tot_ev = run(0, False, gate=True)    # per-tick events: latency percentiles
    with ClockSampler(local_rank) as clk:
        # throughput: the same back-to-back ticks with events only around the
        # timed region (per-tick event records add ~1 us of stream gaps each)
        _, tot = run(0, False, gate=True, per_tick=False)
        _, tot_direct = run(0, False, gate=True, per_tick=False, direct=True)
    # validate the last tick against a batch scoring of the same windows
    t_last = t_hist + ticks - 1
    fb, sb, mb = E.detect(X[:, t_last - W + 1:t_last + 1].contiguous(), det, mean, std, thr,
                          W - 1, W, return_scores=True)
    assert torch.equal(sb[:, 0], scores) and torch.equal(fb[:, 0], flags), \
        "streaming tick != batch scoring"
    tot = max_over_ranks(tot)

    # ---- NEXT-2: the same ticks with online SPOT (single GPU) ----
    spot_line = None
    if world == 1:
        spot_line = {}
        for every in (10, 1):
            # fresh SPOT state per run, calibrated on the same calibration scores;
            # capacity for every streamed score to be a peak (no overflow)
            spot = E.Spot(cal.numel(), device=dev, stream_peaks=n * ticks)
            spot.calibrate(cal.reshape(-1))
            sgraphs = {}
            side.wait_stream(torch.cuda.current_stream())
            for ph in range(W):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    ring.step(stage, ph + W, spot.thr, out=(flags, scores, md))
                    spot.update(scores, flags)
                sgraphs[ph] = g
            gref = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gref, stream=side):
                spot.refit()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            for t in range(t_hist - W + 1, t_hist):    # restore the ring to the stream start
                ring.push(X[:, t].contiguous(), t)
            st_, en_ = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
            for k in range(ticks):
                i = k - args.warmup
                if i >= 0:
                    st_[i].record(stream)
                stage.copy_(S[k])
                sgraphs[(t_hist + k) % W].replay()
                if (k + 1) % every == 0:
                    gref.replay()
                if i >= 0:
                    en_[i].record(stream)
            torch.cuda.synchronize()
            lat_s = [a_.elapsed_time(b_) for a_, b_ in zip(st_, en_)]
            tot_s = st_[0].elapsed_time(en_[-1])
            thr_s = spot.threshold()
            spot_line[f"refit_every_{every}"] = {
                "windows_per_s": n * args.steps / (tot_s * 1e-3),
                "tick_latency_us": {"p50": 1e3 * _pct(lat_s, 50), "p99": 1e3 * _pct(lat_s, 99)},
                "n_peaks_end": thr_s["n_peaks"], "n_end": thr_s["n"], "z_q_end": thr_s["z_q"]}
    lat_e2e, _ = run(ticks, True, gate=True)                    # p50 / p99 per tick
    _, tot_e2e = run(ticks, True, gate=True, per_tick=False)    # throughput
    tot_e2e = max_over_ranks(tot_e2e)
    value = n_global * args.steps / (tot * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import enova_oracle as O
        m_np, s_np = mean.cpu().numpy(), std.cpu().numpy()
        t0 = time.perf_counter()
        done = 0
        k = 0
        while time.perf_counter() - t0 < args.cpu_budget / 3 or done == 0:
            t = t_hist + k
            blk = Xh[:, t - W + 1:t + 1]
            sc_o, md_o = O.score_windows(blk, wts, m_np, s_np, W - 1, W)
            O.flags(sc_o, md_o, thr["z_q"])
            done += n
            k += 1
        el = time.perf_counter() - t0
        cpu = {"value": done / el, "unit": "windows/s", "cores": cpu_cores(),
               "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"{k} ticks x {n} instances ({el:.1f} s)"}
    if comm is not None:
        comm.destroy()
    # roofline of the one launch per tick (k_stream_rows with the push fused):
    # algorithmic bytes = the new samples in + score/md/flag out; the kernel also
    # re-reads every instance's W-sample window from the fp16 ring (2 D B) and
    # its W sample sums (4 W B) -- reported separately, labelled
    peaks = load_peaks()
    tick_s = tot / args.steps * 1e-3
    algo_b = n * (M * 4 + 4 + 4 + 1)
    ring_b = n * (2 * W * M + 4 * W)
    roof = {"kernel": "k_stream_rows (enova_stream_step)", "bound": "hbm",
            "achieved": algo_b / tick_s / 1e9, "peak": peaks["hbm"], "unit": "GB/s",
            "frac": algo_b / tick_s / 1e9 / peaks["hbm"], "traffic": None,
            "algorithmic_bytes_per_launch": algo_b,
            "with_ring_reread": {"bytes_per_launch": algo_b + ring_b,
                                 "achieved": (algo_b + ring_b) / tick_s / 1e9,
                                 "frac": (algo_b + ring_b) / tick_s / 1e9 / peaks["hbm"],
                                 "frac_spec": (algo_b + ring_b) / tick_s / 1e9 / SPEC_HBM_GBS,
                                 "note": "the window of every instance re-read from the fp16 "
                                         "ring (2*D B) plus its W sample sums (4*W B)"},
            "ring_read_floor_us": 1e6 * (algo_b + ring_b) / (peaks["hbm"] * 1e9),
            "frac_of_floor": (algo_b + ring_b) / (peaks["hbm"] * 1e9) / tick_s,
            "peak_spec": SPEC_HBM_GBS, "frac_spec": algo_b / tick_s / 1e9 / SPEC_HBM_GBS,
            "peak_source": peaks["source"],
            "launch_ms_avg": tot / args.steps,
            "note": "latency-bound: one launch per tick; the per-tick bytes are far below "
                    "what HBM moves in the tick's duration"}
    if rank == 0:
        line = {
            "metric": METRIC + " (c4 streaming tick)", "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": f"c4: {n_global} instances x M={M}, W={W}, H={H}, Z={Z}; one "
                                   f"sample per instance per tick; stats and fleet threshold frozen "
                                   f"from a {t_hist}-step calibration horizon",
                       "instances": n_global, "parallelism": f"instance-sharded x{world}",
                       "step": "one tick: ingest-normalise the new samples into the fp16 ring "
                               "and score/flag every instance's newest window in ONE launch "
                               "(enova_stream_step: push fused into the TMA ring -> tcgen05 "
                               "row kernel)",
                       "l2": "not flushed: the 41 MB fp16 ring is the streaming working set"},
            "tick_latency_host_paced_us": {"p50": 1e3 * _pct(lat_host, 50),
                                           "p99": 1e3 * _pct(lat_host, 99),
                                           "windows_per_s": n_global * args.steps / (tot_host * 1e-3),
                                           "note": "each tick's graph launched from the Python loop "
                                                   "as the previous one is queued: includes the "
                                                   "host launch rate"},
            "tick_direct_launch_us": 1e3 * tot_direct / args.steps,
            "tick_latency_us": {"p50": 1e3 * _pct(lat, 50), "p99": 1e3 * _pct(lat, 99),
                                "max": 1e3 * max(lat), "mean_per_tick_events": 1e3 * tot_ev / args.steps,
                                "note": "events around every tick (a separate back-to-back run); "
                                        "ms_per_step / value: events around the timed region only"},
            "step_mode": "one CUDA graph replay per tick, one kernel (the tick's samples read where "
                         "they arrived in device memory), the ticks enqueued back to back behind an "
                         "untimed GPU-side spin so the events time the device; e2e: H2D into a "
                         "staging buffer (tick k+1's copy overlapping tick k's kernel, double-buffered), the kernel and the flags' D2H copy captured as one graph per tick, enqueued the same way",
            "threshold": {"z_q": thr["z_q"], "n_peaks": thr["n_peaks"]},
            "roofline": roof,
            "next_rows": {"online_spot": spot_line},
            "cpu_baseline": cpu,
            "e2e": {"value": n_global * args.steps / (tot_e2e * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": int(n * M * 4), "d2h_bytes_per_step": int(n),
                    "tick_latency_us": {"p50": 1e3 * _pct(lat_e2e, 50), "p99": 1e3 * _pct(lat_e2e, 99)}},
            "gpu_launches": int(launches_per_tick * args.steps),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_threshold_sweep(args, rank, world, local_rank):
    """c5: the fleet-wide POT threshold of 100M calibration
    scores; strong scaling (rank r holds a contiguous shard).  One GPU: the
    stream-ordered fit (one cooperative kernel) replayed as a CUDA graph; N > 1:
    the collective fit (histogram all-reduces + fixed-slot tail gather), also
    stream-ordered and replayed as a graph."""
    import torch
    import torch.distributed as dist

    import paper_2407_09486_b200 as E
    from paper_2407_09486_b200 import _lib, synth
    from paper_2407_09486_b200.fleet import max_over_ranks, shard_range

    dev = _dist_setup(world, local_rank)
    n_total = synth.CONFIGS["c5"]["n_scores"]
    a, b = shard_range(n_total, world, rank)
    n = b - a
    sh = synth.score_mixture(n, offset=a)
    sh_pinned = torch.from_numpy(sh).pin_memory()
    scores = sh_pinned.to(dev)
    force_comm = os.environ.get("ENOVA_BENCH_COMM") == "1"   # diagnostic, as in run_windows
    comm = E.Comm.create(rank, world, local_rank) if (world > 1 or force_comm) else None
    ws = E.ThresholdWorkspace(n_total, 0.98, dev, world=world if comm is not None else 0)
    thr_dev = torch.zeros(E.api.THRESHOLD_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def enqueue():
        if comm is None:
            E.fit_threshold_async(scores, workspace=ws, out=thr_dev)
        elif args.fit == "distributed":   # per-rank tails, pass totals all-gathered
            E.fit_threshold_dist_async(scores, n_total, comm, workspace=ws, out=thr_dev)
        else:   # stream-ordered collective fit: captured with its NCCL calls
            E.fit_threshold_comm_async(scores, n_total, comm, workspace=ws, out=thr_dev)
    l0 = _lib.lib().enova_kernel_launches()
    enqueue()
    torch.cuda.synchronize()
    per = _lib.lib().enova_kernel_launches() - l0
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(stream)
    with torch.cuda.graph(g, stream=side):
        enqueue()
    stream.wait_stream(side)
    step = g.replay
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    starts, ends = [ev() for _ in range(args.steps)], [ev() for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    tot = max_over_ranks(float(sum(step_ms)))
    thr = E.threshold_from_device(thr_dev)
    value = n_total * args.steps / (tot * 1e-3)
    # phase split of one k_pot launch from its %globaltimer stamps (CTA 0):
    # [0] launch entry ... [fit_stamp] start of the GPD fit, [-1] end
    phases = None
    if comm is None:
        import ctypes as C
        step()
        torch.cuda.synchronize()
        L_ = _lib.lib()
        no, so = C.c_int64(), C.c_int64()
        L_.enova_internal_pot_stamp_offsets(C.byref(no), C.byref(so))
        L_.enova_internal_pot_fit_stamp_offset.restype = C.c_int64
        L_.enova_internal_pot_sampled_offset.restype = C.c_int64
        fo = int(L_.enova_internal_pot_fit_stamp_offset())
        sp = int(L_.enova_internal_pot_sampled_offset())
        head = ws.buf[:so.value + 8 * 96].cpu().numpy()
        ns = int(head[no.value:no.value + 4].view(np.int32)[0])
        fs = int(head[fo:fo + 4].view(np.int32)[0])
        sampled = int(head[sp:sp + 4].view(np.int32)[0])
        st = head[so.value:so.value + 8 * min(ns, 95)].view(np.uint64).astype(np.int64)
        if ns >= 4 and 0 < fs < ns:
            sel_us = (st[fs] - st[0]) / 1e3
            fit_us = (st[ns - 1] - st[fs]) / 1e3
            # bytes the selection must move: one read of the scores + the peaks out;
            # the sampled path also writes and re-reads the ~2.4% candidates
            moved = 4.0 * n + 8.0 * thr["n_peaks"]
            phases = {"select_compact_us": sel_us, "fit_us": fit_us, "sampled_selection": bool(sampled),
                      "select_bytes_algorithmic": moved,
                      "select_achieved_GBps": moved / (sel_us * 1e-6) / 1e9,
                      "select_hbm_frac": moved / (sel_us * 1e-6) / 1e9 / load_peaks()["hbm"],
                      "fit_grid_points": 128, "fit_peaks": thr["n_peaks"],
                      "note": "stamps of CTA 0 (globaltimer); the fit is fp64 compute "
                              "(Grimshaw grid + certified Halley passes), not HBM-bound"}
            if sampled and ns > 4:
                # the one full pass over the scores (k_pot_scan) runs between the
                # sampling launch's last stamp [3] and the selection launch's first
                # [4]: the gap bounds the scan kernel's time (two launch gaps included)
                gap = (st[4] - st[3]) / 1e3
                phases["scan"] = {"kernel": "k_pot_scan", "gap_us": gap,
                                  "achieved_GBps_lower_bound": 4.0 * n / (gap * 1e-6) / 1e9,
                                  "hbm_frac_lower_bound": 4.0 * n / (gap * 1e-6) / 1e9 / load_peaks()["hbm"],
                                  "note": "algorithmic bytes = one fp32 read of the scores; the "
                                          "stamp gap includes the end of the sampling launch, two "
                                          "launch gaps and the start of the selection launch"}
    peaks = load_peaks()
    ms = tot / args.steps
    achieved = 4.0 * n / (ms * 1e-3) / 1e9                 # algorithmic: one read of the shard
    # e2e: the shard copied from pinned host memory every step + the threshold read back
    e0, e1 = ev(), ev()
    e0.record(stream)
    for _ in range(args.steps):
        scores.copy_(sh_pinned, non_blocking=True)
        step()
        if world == 1:
            thr_h = thr_dev.cpu()
    e1.record(stream)
    torch.cuda.synchronize()
    e_ms = max_over_ranks(e0.elapsed_time(e1))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import enova_oracle as O
        m = 10_000_000
        t0 = time.perf_counter()
        O.pot_threshold(sh[:m], 0.98, 1e-3)
        el = time.perf_counter() - t0
        cpu = {"value": m / el, "unit": "scores/s", "cores": cpu_cores(),
               "cpu_model": cpu_model(), "kind": "oracle",
               "sample": f"first {m} of {n_total} c5 scores: full sort + Grimshaw fit ({el:.1f} s)"}
    if comm is not None:
        comm.destroy()
    if rank == 0:
        line = {
            "metric": "calibration scores thresholded/sec (c5 POT fit); % HBM roofline",
            "value": value, "unit": "scores/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 keys / f64 fit",
            "data": "synthetic",
            "config": {"workload": f"c5: {n_total} scores (99.9% 0.5*chi2_16 + 0.1% GPD tail), "
                                   f"q0=0.98, q=1e-3", "scores": n_total,
                       "parallelism": f"score-sharded x{world}",
                       "fit": args.fit if comm is not None else "single-GPU",
                       "l2": "inputs 400 MB > L2 (no flush needed)"},
            "threshold": {k_: thr[k_] for k_ in ("t", "gamma", "sigma", "z_q", "n_peaks")},
            "phases": phases,
            "roofline": {"kernel": "k_pot", "bound": "hbm", "achieved": achieved,
                         "peak": peaks["hbm"], "unit": "GB/s", "frac": achieved / peaks["hbm"],
                         "traffic": None, "peak_source": peaks["source"],
                         "peak_spec": SPEC_HBM_GBS, "frac_spec": achieved / SPEC_HBM_GBS,
                         "bytes_per_launch": 4 * n,
                         "note": "algorithmic bytes = one fp32 read of the scores; the fit's "
                                 "fp64 grid scan over the 2M peaks is compute, not bytes"},
            "cpu_baseline": cpu,
            "e2e": {"value": n_total * args.steps / (e_ms * 1e-3), "unit": "scores/s",
                    "h2d_bytes_per_step": int(4 * n), "d2h_bytes_per_step": int(E.api.THRESHOLD_BYTES)},
            "gpu_launches": int(per * args.steps),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    # NCCL prints its version banner on stdout at communicator creation when
    # NCCL_DEBUG=VERSION: keep stdout to the one JSON line
    if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the live ncu DRAM-traffic pass of the roofline kernel")
    ap.add_argument("--dry-run", action="store_true",
                    help="host-side multi-rank plumbing only (gloo, no GPU, no kernels): "
                         "shards, barrier, max-over-ranks timing and the JSON line")
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--fit", default="replicated", choices=["replicated", "distributed"],
                    help="fleet threshold fit with a communicator (N > 1): every rank fits the "
                         "gathered tail (replicated) or its own tail with pass totals all-gathered "
                         "(distributed, SURVEY §8e)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: re-exec under
        # torch.distributed.run, one process per GPU (the driver's own launch)
        return self_launch(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world:
        if rank == 0:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one process per "
                  f"GPU with --nproc-per-node {args.gpus} (or omit the launcher)", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        return run_dry(args, rank, world)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "c4":
        return run_streaming(args, rank, world, local_rank)
    if args.workload == "c5":
        return run_threshold_sweep(args, rank, world, local_rank)
    return run_windows(args, rank, world, local_rank)


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(n):
    """Re-run this command under torch.distributed.run with n ranks on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    rc = subprocess.call(cmd)
    if rc:
        sys.exit(rc)


def run_dry(args, rank, world):
    """--dry-run: the multi-rank host plumbing without a GPU (gloo): each rank's
    instance shard, a barrier, a per-rank "step time" reduced with max over
    ranks and the windows summed over ranks, then rank 0's JSON line.  No
    kernels run; `value` is null.  Used by the CPU tests to check that
    `--gpus N` really starts N ranks."""
    import torch.distributed as dist

    from paper_2407_09486_b200 import synth
    from paper_2407_09486_b200.fleet import max_over_ranks, shard_range, sum_over_ranks
    if world > 1:
        dist.init_process_group("gloo")
    cfg = synth.CONFIGS[args.workload if args.workload in ("c2", "c3") else "c2"]
    n_per = INST_PER_GPU if args.workload == "c2" else cfg["n_instances"] // 8
    a, b = shard_range(n_per * world, world, rank)
    T, W = cfg["n_steps"], cfg["window"]
    wins = sum_over_ranks((b - a) * (T - W + 1))
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "dry_run": True,
                          "ranks_seen_max": t, "windows_per_step": wins,
                          "config": {"workload": args.workload,
                                     "parallelism": f"instance-sharded x{world}"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_windows(args, rank, world, local_rank):
    """c2 / c3: the whole hot path over every window of the rank's fleet shard."""
    import torch
    import torch.distributed as dist

    import paper_2407_09486_b200 as E
    from paper_2407_09486_b200 import _lib, synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfg = synth.CONFIGS[args.workload]
    W, M, H, Z, T = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"], cfg["n_steps"]
    N = INST_PER_GPU if args.workload == "c2" else cfg["n_instances"] // 8
    D = W * M
    tcal = T // 2
    Xh, labels_h = synth.metric_trace_parallel(N, T, M, seed=synth.DEFAULT_SEED + 2,
                                               instance_offset=rank * N, return_labels=True)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + 2)
    X_pinned = torch.from_numpy(Xh).pin_memory()
    X = X_pinned.to(dev)
    det = E.PreparedDetector(wts, device=dev)
    # ENOVA_BENCH_COMM=1 forces the communicator path at world size 1 (measures
    # the collective threshold's overhead on one GPU; diagnostic only)
    force_comm = os.environ.get("ENOVA_BENCH_COMM") == "1"
    comm = E.Comm.create(rank, world, local_rank) if (world > 1 or force_comm) else None
    n_cal_local = N * (tcal - (W - 1))
    n_det_local = N * (T - tcal)
    wins_local = n_cal_local + n_det_local
    pipe = E.Pipeline(det, N, T, tcal, device=dev, comm=comm, fit_mode=args.fit)
    cal, mean, std = pipe.cal, pipe.mean, pipe.std
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    # the zero-fill leaves L2 full of dirty lines whose write-back would overlap
    # the next step; a read pass over a second buffer (also untimed) evicts them
    flush_rd = torch.zeros(64 << 20, dtype=torch.int32, device=dev)    # 256 MiB

    def l2_flush():
        flush.zero_()
        flush_rd.sum()
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)

    # one step = pipe.enqueue(X) = enova_step_enqueue: stats -> calibration scores +
    # MD -> POT threshold (with a communicator the stream-ordered collective fit)
    # overlapped with the detection scores + MD -> the flags of every window.  The
    # step is captured once into a CUDA graph and replayed (one graph launch per
    # step), NCCL collectives included.  Pipeline.tune picks the overlap
    # configuration (fit grid, detection instances scored next to it) by time;
    # every configuration gives the same scores, MD and flags.
    use_graph = True   # with a communicator too: the NCCL collectives are captured
    tuned = pipe.tune(X)
    if world > 1:   # the same fit grid on every rank (z_q bit-identical across ranks)
        cfg_t = torch.tensor([tuned["pot_ctas"], tuned["concurrent_instances"]], dtype=torch.int64,
                             device=dev)
        dist.broadcast(cfg_t, 0)
        pipe.configure(int(cfg_t[0]), int(cfg_t[1]))
        tuned = dict(tuned, pot_ctas=int(cfg_t[0]), concurrent_instances=int(cfg_t[1]))
    l0 = _lib.lib().enova_kernel_launches()
    pipe.enqueue(X)
    torch.cuda.synchronize()
    launches_per_step = _lib.lib().enova_kernel_launches() - l0
    if use_graph:
        pipe.capture(X)
    run_step = pipe.replay if use_graph else (lambda: pipe.enqueue(X))
    for _ in range(args.warmup):
        run_step()
    torch.cuda.synchronize()
    warm = pipe.result()                       # statuses checked (raises on failure)

    # ---- device-resident timed region ----
    starts = [ev() for _ in range(args.steps)]
    ends = [ev() for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = _lib.lib().enova_kernel_launches()
    with ClockSampler(local_rank) as clk:
        for i in range(args.steps):
            l2_flush()                                 # untimed L2 flush between steps
            starts[i].record(stream)
            run_step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    launches = (launches_per_step * args.steps if use_graph
                else _lib.lib().enova_kernel_launches() - l0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    res = pipe.result()
    thr = res.threshold
    step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
    tot_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([tot_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = wins_local * world * args.steps / (tot_ms * 1e-3)

    # ---- per-stage device times (eager, stream-ordered, events between stages) ----
    stage = {"stats": [], "score_calibration": [], "fit_threshold": [], "flag_calibration": [],
             "detect": []}
    if world == 1:
        for _ in range(5):
            l2_flush()
            k = [ev() for _ in range(6)]
            k[0].record(stream)
            E.compute_stats_async(X, tcal, out=(mean, std), diag=pipe.diag, workspace=pipe.stats_ws)
            k[1].record(stream)
            E.score_windows(X, det, mean, std, W - 1, tcal, out=(cal, pipe.cal_md))
            k[2].record(stream)
            E.fit_threshold_async(cal, 0.98, 1e-3, workspace=pipe.thr_ws, out=pipe.thr)
            k[3].record(stream)
            E.flag_scores_async(cal, pipe.cal_md, pipe.thr, out=pipe.cal_flags)
            k[4].record(stream)
            E.detect_async(X, det, mean, std, pipe.thr, tcal, T, out=(pipe.flags, pipe.scores, pipe.md))
            k[5].record(stream)
            torch.cuda.synchronize()
            for j, name in enumerate(stage):
                stage[name].append(k[j].elapsed_time(k[j + 1]))
    stage_ms = {k_: float(np.median(v_)) for k_, v_ in stage.items() if v_}

    # ---- roofline of the dominant kernel (k_score) ----
    # The kernel's own launch duration is measured with the same launch back to
    # back (calibration range, the configuration the step uses), L2 flushed
    # before the burst; its share of the step comes from the per-stage events.
    peaks = load_peaks()
    fpw = flops_per_window(D, H, Z)
    reps = 10
    flush.zero_()
    k0, k1 = ev(), ev()
    E.score_windows(X, det, mean, std, W - 1, tcal, out=(cal, pipe.cal_md))
    k0.record(stream)
    for _ in range(reps):
        E.score_windows(X, det, mean, std, W - 1, tcal, out=(cal, pipe.cal_md))
    k1.record(stream)
    torch.cuda.synchronize()
    launch_ms = k0.elapsed_time(k1) / reps
    achieved = fpw * n_cal_local / (launch_ms * 1e-3) / 1e12   # TFLOP/s
    traffic, traffic_src = None, None
    if rank == 0 and world == 1 and args.workload == "c2" and not args.no_traffic:
        # live ncu pass (subprocess, untimed) over the same calibration launch
        t_ = measure_traffic("k_score_pair", [os.path.join(ROOT, "tools", "profile_run.py"), "1"])
        if t_ is not None:
            traffic = t_[0]
            traffic_src = (f"ncu dram__bytes_read.sum + dram__bytes_write.sum of the first "
                           f"c2 calibration launch, measured in this run "
                           f"(read {t_[1] / 1e6:.1f} MB, write {t_[2] / 1e6:.1f} MB)")
    algo_bytes = N * tcal * M * 4 + n_cal_local * 8   # samples read once + score, md written
    roof = {"kernel": "k_score_pair<128,16>", "bound": "tensor", "achieved": achieved,
            "peak": peaks["bf16"], "unit": "TFLOP/s", "frac": achieved / peaks["bf16"],
            "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_bytes_per_launch": algo_bytes,
            "peak_spec": SPEC_F16_TFLOPS, "frac_spec": achieved / SPEC_F16_TFLOPS,
            "peak_sustained": peaks["bf16_sus"], "frac_sustained": achieved / peaks["bf16_sus"],
            "peak_source": peaks["source"] + ": dense bf16 burst; fp16 has the same nominal rate",
            "flops_per_window": fpw, "windows_per_launch": n_cal_local,
            "launch_ms_avg": launch_ms, "launches_timed": reps,
            "in_step_score_ms": (stage_ms.get("score_calibration", 0.0) + stage_ms.get("detect", 0.0)) or None,
            "share_of_step": ((stage_ms["score_calibration"] + stage_ms["detect"]) / ms_per_step
                              if stage_ms else None),
            "step_level": {"achieved": fpw * wins_local / (ms_per_step * 1e-3) / 1e12,
                           "frac": fpw * wins_local / (ms_per_step * 1e-3) / 1e12 / peaks["bf16"],
                           "frac_spec": fpw * wins_local / (ms_per_step * 1e-3) / 1e12 / SPEC_F16_TFLOPS,
                           "note": "every window's algorithmic tensor FLOPs / the whole step "
                                   "(stats, threshold and flags included)"}}

    # ---- NEXT-1 / NEXT-4 on this step's detection flags (not part of the step) ----
    extras = None
    if world == 1:
        labels = torch.from_numpy(labels_h).to(dev)
        reps = 10
        # device time of the kernels: each measured call sequence is one CUDA
        # graph replay (host-side binding overhead excluded)
        cnt = torch.empty(4, dtype=torch.int64, device=dev)
        E.point_adjusted_counts(labels, pipe.flags, tcal, out=cnt)
        side_e = torch.cuda.Stream(device=dev)
        side_e.wait_stream(stream)
        g_pa = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_pa, stream=side_e):
            for _ in range(reps):
                E.point_adjusted_counts(labels, pipe.flags, tcal, out=cnt)
        stream.wait_stream(side_e)
        t0e, t1e = ev(), ev()
        g_pa.replay()
        t0e.record(stream)
        g_pa.replay()
        t1e.record(stream)
        torch.cuda.synchronize()
        pa_ms = t0e.elapsed_time(t1e) / reps
        pa = E.point_adjusted_f1(labels, pipe.flags, tcal)
        ids = E.select_flagged(pipe.flags)
        # explain at least 10 000 windows: the flagged ones, padded with a fixed stride
        if ids.numel() < 10000:
            pad = torch.arange(0, pipe.flags.numel(), max(1, pipe.flags.numel() // 10000),
                               device=dev)[:10000 - ids.numel()]
            sel = torch.cat([ids, pad]).sort().values
        else:
            sel = ids
        E.explain_windows(X, det, mean, std, sel, tcal, T)
        side_e.wait_stream(stream)
        g_ex = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_ex, stream=side_e):
            for _ in range(reps):
                E.explain_windows(X, det, mean, std, sel, tcal, T)
        stream.wait_stream(side_e)
        g_ex.replay()
        t0e.record(stream)
        g_ex.replay()
        t1e.record(stream)
        torch.cuda.synchronize()
        ex_ms = t0e.elapsed_time(t1e) / reps
        extras = {
            "point_adjusted_eval": {"us": 1e3 * pa_ms, "points": int(pipe.flags.numel()),
                                    "precision": pa["precision"], "recall": pa["recall"],
                                    "f1": pa["f1"],
                                    "note": "random-init detector: the P/R/F1 values carry no "
                                            "semantic meaning; the kernel time is the measurement"},
            "explain_windows": {"windows": int(sel.numel()), "flagged": int(ids.numel()),
                                "us": 1e3 * ex_ms,
                                "windows_per_s": sel.numel() / (ex_ms * 1e-3)},
        }

    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        # the same step through the public API with the trace in pinned HOST memory:
        # H2D copy of the whole trace, the step, D2H of the flags, every step
        flags_h = torch.empty(tuple(pipe.flags.shape), dtype=torch.int8).pin_memory()
        cflags_h = torch.empty(tuple(pipe.cal_flags.shape), dtype=torch.int8).pin_memory()
        d2h = flags_h.numel() + cflags_h.numel()

        if use_graph:
            # double-buffered: the H2D copy of step k+1 (copy stream) overlaps the
            # step-k graph on the compute stream; every step still copies its whole
            # trace in and its flags out
            X2 = X.clone()   # capture warms up on real data
            pipe2 = E.Pipeline(det, N, T, tcal, device=dev, comm=comm, fit_mode=args.fit)
            pipe2.configure(pipe.pot_ctas, pipe.concurrent_instances)
            pipe2.capture(X2)
            mk = lambda: (torch.empty(tuple(pipe.cal_flags.shape), dtype=torch.int8).pin_memory(),
                          torch.empty(tuple(pipe.flags.shape), dtype=torch.int8).pin_memory())
            bufs = [(X, pipe, mk()), (X2, pipe2, mk())]
            cs = torch.cuda.Stream(device=dev)
            copied = [torch.cuda.Event(), torch.cuda.Event()]
            freed = [torch.cuda.Event(), torch.cuda.Event()]
            for b in range(2):
                freed[b].record(stream)

            def e2e_run(nsteps, e_start):
                cs.wait_event(e_start)
                for k in range(nsteps):
                    b = k % 2
                    xb, pb, fh = bufs[b]
                    with torch.cuda.stream(cs):
                        cs.wait_event(freed[b])
                        xb.copy_(X_pinned, non_blocking=True)
                        copied[b].record(cs)
                    stream.wait_event(copied[b])
                    pb.replay()
                    fh[0].copy_(pb.cal_flags, non_blocking=True)
                    fh[1].copy_(pb.flags, non_blocking=True)
                    freed[b].record(stream)

            w0 = ev()
            w0.record(stream)
            e2e_run(2, w0)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
                torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record(stream)
            e2e_run(args.steps, e0)
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1)
            pipe2.result()
            d2h = bufs[0][2][0].numel() + bufs[0][2][1].numel()
            e2e_mode = "double-buffered: H2D of step k+1 overlaps the step-k graph"
        else:
            def e2e_step():
                X.copy_(X_pinned, non_blocking=True)
                run_step()
                flags_h.copy_(pipe.flags, non_blocking=True)
                cflags_h.copy_(pipe.cal_flags, non_blocking=True)

            for _ in range(2):
                e2e_step()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0, e1 = ev(), ev()
            e0.record(stream)
            for _ in range(args.steps):
                e2e_step()
            e1.record(stream)
            torch.cuda.synchronize()
            e_ms = e0.elapsed_time(e1)
            e2e_mode = "serial: H2D, step, D2H"
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        pipe.result()
        e2e = {"value": wins_local * world * args.steps / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(Xh.nbytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e_ms / args.steps, "mode": e2e_mode}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, wins, ninst, el = oracle_sample(Xh, wts, tcal, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "cpu_model": cpu_model(),
               "kind": "oracle",
               "sample": f"first {ninst} of {N} {args.workload} instances, all {wins} windows, "
                         f"fp64 NumPy forward incl. explicit decoder ({el:.1f} s)"}

    if comm is not None:
        comm.destroy()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {
                "workload": f"{args.workload} per GPU: {N} instances x T={T} x M={M}, W={W}, detector "
                            f"H={H} Z={Z}; T_cal={tcal}; fleet-wide POT threshold",
                "instances_per_gpu": N, "global_instances": N * world, "T": T, "M": M, "W": W,
                "windows_per_step": wins_local * world, "parallelism": f"instance-sharded x{world}",
                "fit": args.fit if world > 1 else "single-GPU",
                "l2": f"flushed between steps (256 MiB zero-fill + 256 MiB read pass, untimed); inputs {Xh.nbytes / 1e6:.0f} MB/GPU > L2",
                "precision": "fp16 operands (x, weights), fp32 accumulate, h/mu hi+lo fp16",
                "outputs": "every window of the trace (calibration and detection) ends the step "
                           "with a score, an MD and a flag",
            },
            "stage_ms": stage_ms,
            "stage_ms_note": "each stage alone, eager, in sequence (the step overlaps the fit "
                             "with the detection scores: see step_overlap)",
            "step_overlap": {"pot_ctas": tuned["pot_ctas"],
                             "concurrent_instances": tuned["concurrent_instances"],
                             "tuning_ms": {f"{p_}/{c_}": round(m_, 4)
                                           for p_, c_, m_ in tuned.get("candidates", [])},
                             "note": "enova_step: the POT fit on pot_ctas CTAs (2-CTA clusters) "
                                     "on a side stream next to the detection scores of the "
                                     "first concurrent_instances instances; (0, 0) = sequential"},
            "next_rows": extras,
            "step_mode": "CUDA graph replay (1 graph launch/step)" if use_graph else "eager",
            "threshold": {"z_q": thr["z_q"], "t": thr["t"], "gamma": thr["gamma"],
                          "n_peaks": thr["n_peaks"]},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
