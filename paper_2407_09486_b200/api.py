"""Python surface of the ENOVA detection hot path (same names as the C ABI in
include/enova.h).  Tensors are CUDA fp32; torch provides memory, streams and
process groups; libenova.so does all the work."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Detector, Series, StepArgs, Threshold, TrainConfig, check, lib

_WEIGHT_KEYS = ("enc_w1", "enc_b1", "enc_wmu", "enc_bmu", "enc_wlv", "enc_blv",
                "dec_w1", "dec_b1", "dec_w2", "dec_b2")


def _stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _require_cuda(t: torch.Tensor, name: str, dtype=torch.float32):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")


_KERNELS = {"auto": 0, "stream": 1, "pair": 2, "rows": 3}


class force_score_kernel:
    """Diagnostic context manager: force the windowed scoring kernel ("stream",
    "pair", "rows" or "auto") for the calls inside (enova_set_score_kernel)."""

    def __init__(self, name: str):
        self.k = _KERNELS[name]

    def __enter__(self):
        check(lib().enova_set_score_kernel(self.k))
        return self

    def __exit__(self, *a):
        check(lib().enova_set_score_kernel(0))


class PreparedDetector:
    """Detector weights on the GPU plus their prepared fp16 operand image (K0)."""

    def __init__(self, weights: dict, device=None, stream=None):
        device = torch.device(device or "cuda")
        self.window = int(weights["window"])
        self.n_metrics = int(weights["n_metrics"])
        self.hidden = int(weights["hidden"])
        self.latent = int(weights["latent"])
        self.tensors = {}
        for k in _WEIGHT_KEYS:
            v = weights[k]
            if isinstance(v, np.ndarray):
                v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))
            self.tensors[k] = v.to(device=device, dtype=torch.float32).contiguous()
        self.struct = Detector(self.window, self.n_metrics, self.hidden, self.latent,
                               *[self.tensors[k].data_ptr() for k in _WEIGHT_KEYS])
        self.ws_bytes = int(lib().enova_detector_workspace_bytes(C.byref(self.struct)))
        if self.ws_bytes == 0:
            raise _lib.EnovaError(2, "detector shape outside the fast-path envelope")
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        check(lib().enova_prepare_detector(C.byref(self.struct), C.c_void_p(self.ws.data_ptr()),
                                           self.ws_bytes, _stream_ptr(stream)))


def _series(metrics: torch.Tensor, mean=None, std=None, t_begin=0, t_end=0) -> Series:
    _require_cuda(metrics, "metrics")
    if metrics.dim() != 3:
        raise ValueError("metrics must be [instances, T, M]")
    N, T, M = metrics.shape
    if metrics.stride(2) != 1 or metrics.stride(1) != M:
        raise ValueError("metrics rows must be contiguous [T][M] per instance")
    ld = metrics.stride(0) if N > 1 else T * M
    for name, v in (("mean", mean), ("std", std)):
        if v is not None:
            _require_cuda(v, name)
            if v.device != metrics.device:
                raise ValueError(f"{name} must be on {metrics.device}")
            if tuple(v.shape) != (N, M) or not v.is_contiguous():
                raise ValueError(f"{name} must be a contiguous [{N}, {M}] tensor")
    s = Series(metrics.data_ptr(), N, T, ld, int(t_begin), int(t_end),
               mean.data_ptr() if mean is not None else None,
               std.data_ptr() if std is not None else None, M, 0)
    return s


def compute_stats(metrics: torch.Tensor, t_cal_end: int, *, out=None, stream=None):
    """a-1: per-(instance, metric) mean / std over [0, t_cal_end)."""
    N, T, M = metrics.shape
    s = _series(metrics)
    if out is None:
        mean = torch.empty((N, M), dtype=torch.float32, device=metrics.device)
        std = torch.empty((N, M), dtype=torch.float32, device=metrics.device)
    else:
        mean, std = out
    ws = StatsWorkspace(N, M, metrics.device)
    ndeg = C.c_int64(0)
    check(lib().enova_compute_stats(C.byref(s), int(t_cal_end), C.c_void_p(mean.data_ptr()),
                                    C.c_void_p(std.data_ptr()), C.byref(ndeg),
                                    C.c_void_p(ws.buf.data_ptr()), ws.nbytes, _stream_ptr(stream)))
    return mean, std, int(ndeg.value)


class StatsWorkspace:
    """Scratch for enova_compute_stats / _async (sized by enova_stats_workspace_bytes)."""

    def __init__(self, n_instances: int, n_metrics: int, device=None):
        self.nbytes = int(lib().enova_stats_workspace_bytes(int(n_instances), int(n_metrics)))
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device or "cuda")


def compute_stats_async(metrics: torch.Tensor, t_cal_end: int, *, out=None, diag=None,
                        workspace: StatsWorkspace | None = None, stream=None):
    """a-1, stream-ordered (no host sync).  diag: device int64[2] = (degenerate
    series, non-finite flag) -- read it later (e.g. check_stats_diag)."""
    N, T, M = metrics.shape
    s = _series(metrics)
    if out is None:
        mean = torch.empty((N, M), dtype=torch.float32, device=metrics.device)
        std = torch.empty((N, M), dtype=torch.float32, device=metrics.device)
    else:
        mean, std = out
    if workspace is None:
        workspace = StatsWorkspace(N, M, metrics.device)
    check(lib().enova_compute_stats_async(
        C.byref(s), int(t_cal_end), C.c_void_p(mean.data_ptr()), C.c_void_p(std.data_ptr()),
        C.c_void_p(diag.data_ptr() if diag is not None else None),
        C.c_void_p(workspace.buf.data_ptr()), workspace.nbytes, _stream_ptr(stream)))
    return mean, std


def check_stats_diag(diag: torch.Tensor) -> int:
    """Host check of the diag of compute_stats_async: raises ENOVA_ERR_NONFINITE,
    returns the number of degenerate series."""
    d = diag.cpu().tolist()
    if d[1]:
        raise _lib.EnovaError(5, "non-finite metric value in the calibration horizon")
    return int(d[0])


def score_windows(metrics: torch.Tensor, det: PreparedDetector, mean: torch.Tensor,
                  std: torch.Tensor, t_begin: int | None = None, t_end: int | None = None,
                  *, with_md: bool = True, out=None, stream=None):
    """a-2..a-5: KL scores and MD of every window ending in [t_begin, t_end)."""
    N, T, M = metrics.shape
    tb = det.window - 1 if t_begin is None else int(t_begin)
    te = T if t_end is None else int(t_end)
    s = _series(metrics, mean, std, tb, te)
    nw = max(te - tb, 0)
    if out is None:
        scores = torch.empty((N, nw), dtype=torch.float32, device=metrics.device)
        md = torch.empty((N, nw), dtype=torch.float32, device=metrics.device) if with_md else None
    else:
        scores, md = out
    check(lib().enova_score_windows(C.byref(s), C.byref(det.struct), C.c_void_p(det.ws.data_ptr()),
                                    det.ws_bytes, C.c_void_p(scores.data_ptr()),
                                    C.c_void_p(md.data_ptr() if md is not None else None),
                                    _stream_ptr(stream)))
    return scores, md


class ThresholdWorkspace:
    """Scratch for enova_fit_threshold*, sized for up to n_global_max scores; with a
    communicator of `world` ranks it also holds the gathered tail slots."""

    def __init__(self, n_global_max: int, init_quantile: float = 0.98, device=None,
                 world: int = 0):
        self.n_global_max = int(n_global_max)
        self.init_quantile = float(init_quantile)
        self.world = int(world)
        if self.world > 0:
            self.nbytes = int(lib().enova_threshold_comm_workspace_bytes(
                self.n_global_max, self.init_quantile, self.world))
        else:
            self.nbytes = int(lib().enova_threshold_workspace_bytes(self.n_global_max,
                                                                    self.init_quantile))
        self.buf = torch.empty(self.nbytes, dtype=torch.uint8, device=device or "cuda")


def fit_threshold(scores: torch.Tensor, init_quantile: float = 0.98, risk_q: float = 1e-3,
                  comm: "Comm | None" = None, n_global_max: int | None = None,
                  workspace: ThresholdWorkspace | None = None, stream=None) -> dict:
    """a-7..a-9: fleet-wide POT threshold (synchronous; identical on all ranks)."""
    _require_cuda(scores, "scores")
    flat = scores.reshape(-1)
    if not flat.is_contiguous():
        flat = flat.contiguous()
    n_local = flat.numel()
    if workspace is None:
        if n_global_max is not None:
            nmax = int(n_global_max)
        elif comm is not None:   # every rank must size for the same total (collective)
            nmax = comm.sum_i64(n_local, stream=stream)
        else:
            nmax = n_local
        workspace = ThresholdWorkspace(max(nmax, 1), init_quantile, scores.device,
                                       world=comm.world if comm is not None else 0)
    out = Threshold()
    check(lib().enova_fit_threshold(C.c_void_p(flat.data_ptr()), n_local, workspace.n_global_max,
                                    float(init_quantile), float(risk_q),
                                    C.c_void_p(comm.handle if comm is not None else None),
                                    C.byref(out), C.c_void_p(workspace.buf.data_ptr()),
                                    workspace.nbytes, _stream_ptr(stream)))
    return out.as_dict()


THRESHOLD_BYTES = C.sizeof(Threshold)


def fit_threshold_async(scores: torch.Tensor, init_quantile: float = 0.98, risk_q: float = 1e-3,
                        *, workspace: ThresholdWorkspace | None = None, out=None,
                        stream=None) -> torch.Tensor:
    """a-7..a-8 on one GPU, stream-ordered: returns the DEVICE enova_threshold
    (uint8 tensor) written by the kernel; read it with threshold_from_device."""
    _require_cuda(scores, "scores")
    flat = scores.reshape(-1)
    if not flat.is_contiguous():
        flat = flat.contiguous()
    n = flat.numel()
    if workspace is None:
        workspace = ThresholdWorkspace(n, init_quantile, scores.device)
    thr = out if out is not None else torch.zeros(THRESHOLD_BYTES, dtype=torch.uint8,
                                                  device=scores.device)
    check(lib().enova_fit_threshold_async(
        C.c_void_p(flat.data_ptr()), n, workspace.n_global_max, float(init_quantile),
        float(risk_q), C.c_void_p(thr.data_ptr()), C.c_void_p(workspace.buf.data_ptr()),
        workspace.nbytes, _stream_ptr(stream)))
    return thr


def fit_threshold_comm_async(scores: torch.Tensor, n_global: int, comm: "Comm",
                             init_quantile: float = 0.98, risk_q: float = 1e-3, *,
                             workspace: ThresholdWorkspace | None = None, out=None,
                             stream=None) -> torch.Tensor:
    """a-7..a-9 across the ranks of `comm`, stream-ordered (no host sync; with
    NCCL it can be captured in a CUDA graph).  n_global: the total score count
    over all ranks (Comm.sum_i64 once at setup).  Returns the DEVICE
    enova_threshold (identical on every rank)."""
    _require_cuda(scores, "scores")
    flat = scores.reshape(-1)
    if not flat.is_contiguous():
        flat = flat.contiguous()
    if workspace is None:
        workspace = ThresholdWorkspace(n_global, init_quantile, scores.device, world=comm.world)
    thr = out if out is not None else torch.zeros(THRESHOLD_BYTES, dtype=torch.uint8,
                                                  device=scores.device)
    check(lib().enova_fit_threshold_comm_async(
        C.c_void_p(flat.data_ptr()), flat.numel(), int(n_global), workspace.n_global_max,
        float(init_quantile), float(risk_q), C.c_void_p(comm.handle), C.c_void_p(thr.data_ptr()),
        C.c_void_p(workspace.buf.data_ptr()), workspace.nbytes, _stream_ptr(stream)))
    return thr


def threshold_to_device(thr: dict, device=None) -> torch.Tensor:
    """A host threshold (fit_threshold's dict) as a DEVICE enova_threshold for
    detect_async (e.g. a fleet threshold frozen for streaming)."""
    t = _thr_struct(thr)
    t.reserved = 0
    raw = np.frombuffer(bytes(t), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to(device or "cuda")


def threshold_from_device(thr_dev: torch.Tensor) -> dict:
    """Read a device enova_threshold (synchronises); raises on a failed fit."""
    raw = bytes(thr_dev.cpu().numpy().tobytes())
    t = Threshold.from_buffer_copy(raw)
    if t.reserved != 0:
        raise _lib.EnovaError(int(t.reserved), "device threshold fit failed")
    return t.as_dict()


def detect_async(metrics: torch.Tensor, det: PreparedDetector, mean: torch.Tensor,
                 std: torch.Tensor, thr_dev: torch.Tensor, t_begin: int | None = None,
                 t_end: int | None = None, *, out=None, stream=None):
    """a-2..a-6 with the threshold read from device memory (no host sync)."""
    N, T, M = metrics.shape
    tb = det.window - 1 if t_begin is None else int(t_begin)
    te = T if t_end is None else int(t_end)
    s = _series(metrics, mean, std, tb, te)
    nw = max(te - tb, 0)
    if out is None:
        flags = torch.empty((N, nw), dtype=torch.int8, device=metrics.device)
        sc = md = None
    else:
        flags, sc, md = out
    check(lib().enova_detect_async(C.byref(s), C.byref(det.struct), C.c_void_p(det.ws.data_ptr()),
                                   det.ws_bytes, C.c_void_p(thr_dev.data_ptr()),
                                   C.c_void_p(flags.data_ptr()),
                                   C.c_void_p(sc.data_ptr() if sc is not None else None),
                                   C.c_void_p(md.data_ptr() if md is not None else None),
                                   _stream_ptr(stream)))
    return flags, sc, md


def flag_scores_async(scores: torch.Tensor, md: torch.Tensor, thr_dev: torch.Tensor, *,
                      out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """a-6 on already-scored windows (e.g. the calibration windows, scored before
    the fit): flags = 0 / +1 / -1 against the DEVICE threshold (no host sync)."""
    _require_cuda(scores, "scores")
    _require_cuda(md, "md")
    if scores.shape != md.shape or not scores.is_contiguous() or not md.is_contiguous():
        raise ValueError("scores and md: contiguous, same shape")
    flags = out if out is not None else torch.empty(scores.shape, dtype=torch.int8,
                                                    device=scores.device)
    _require_cuda(flags, "flags", torch.int8)
    if flags.shape != scores.shape or not flags.is_contiguous():
        raise ValueError("flags: contiguous, same shape as scores")
    check(lib().enova_flag_scores_async(C.c_void_p(scores.data_ptr()), C.c_void_p(md.data_ptr()),
                                        scores.numel(), C.c_void_p(thr_dev.data_ptr()),
                                        C.c_void_p(flags.data_ptr()), _stream_ptr(stream)))
    return flags


def _thr_struct(thr: dict) -> Threshold:
    t = Threshold()
    for k, _ in Threshold._fields_:
        if k in thr:
            setattr(t, k, thr[k])
    return t


def detect(metrics: torch.Tensor, det: PreparedDetector, mean: torch.Tensor, std: torch.Tensor,
           threshold: dict, t_begin: int | None = None, t_end: int | None = None, *,
           return_scores: bool = False, out=None, stream=None):
    """a-2..a-6: flags (+1 scale up / -1 scale down / 0) of every window."""
    N, T, M = metrics.shape
    tb = det.window - 1 if t_begin is None else int(t_begin)
    te = T if t_end is None else int(t_end)
    s = _series(metrics, mean, std, tb, te)
    nw = max(te - tb, 0)
    if out is None:
        flags = torch.empty((N, nw), dtype=torch.int8, device=metrics.device)
        sc = torch.empty((N, nw), dtype=torch.float32, device=metrics.device) if return_scores else None
        md = torch.empty((N, nw), dtype=torch.float32, device=metrics.device) if return_scores else None
    else:
        flags, sc, md = out
    thr = _thr_struct(threshold)
    check(lib().enova_detect(C.byref(s), C.byref(det.struct), C.c_void_p(det.ws.data_ptr()),
                             det.ws_bytes, C.byref(thr), C.c_void_p(flags.data_ptr()),
                             C.c_void_p(sc.data_ptr() if sc is not None else None),
                             C.c_void_p(md.data_ptr() if md is not None else None),
                             _stream_ptr(stream)))
    if return_scores:
        return flags, sc, md
    return flags


def ring_push(ring: torch.Tensor, sample: torch.Tensor, tick: int, stream=None):
    """a-10: append one sample per instance to the mirror ring [N][2W][M]."""
    _require_cuda(ring, "ring")
    _require_cuda(sample, "sample")
    N, W2, M = ring.shape
    check(lib().enova_ring_push(C.c_void_p(ring.data_ptr()), N, W2 // 2, M,
                                C.c_void_p(sample.data_ptr()), int(tick), _stream_ptr(stream)))


def ring_view(ring: torch.Tensor, tick: int) -> torch.Tensor:
    """The W samples ending at `tick` as a [N, W, M] strided view of the ring."""
    N, W2, M = ring.shape
    W = W2 // 2
    off = ((tick + 1) % W)
    return ring.as_strided((N, W, M), (W2 * M, M, 1), ring.storage_offset() + off * M)


class StreamRing:
    """a-10 fast path: the ingest-normalised fp16 mirror ring of a fleet
    (enova_stream_*).  push() normalises one new sample per instance with the
    frozen calibration statistics; detect() scores the window ending at a tick
    for every instance (bit-identical to detect() on the same windows)."""

    def __init__(self, det: PreparedDetector, mean: torch.Tensor, std: torch.Tensor, device=None):
        _require_cuda(mean, "mean")
        _require_cuda(std, "std")
        if mean.dim() != 2 or mean.shape[1] != det.n_metrics or tuple(std.shape) != tuple(mean.shape):
            raise ValueError(f"mean and std must both be [instances, {det.n_metrics}]")
        if std.device != mean.device:
            raise ValueError("mean and std must be on the same device")
        self.det, self.mean, self.std = det, mean.contiguous(), std.contiguous()
        self.n = int(mean.shape[0])
        self.W, self.M = det.window, det.n_metrics
        nbytes = int(lib().enova_stream_ring_bytes(self.n, self.W, self.M))
        if nbytes == 0:
            raise _lib.EnovaError(2, "stream ring: unsupported shape")
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device or mean.device)

    def push(self, sample: torch.Tensor, tick: int, stream=None):
        _require_cuda(sample, "sample")
        if tuple(sample.shape) != (self.n, self.M) or not sample.is_contiguous():
            raise ValueError(f"sample must be contiguous [{self.n}, {self.M}]")
        check(lib().enova_stream_push(C.c_void_p(self.buf.data_ptr()), self.n, self.W, self.M,
                                      C.c_void_p(sample.data_ptr()), C.c_void_p(self.mean.data_ptr()),
                                      C.c_void_p(self.std.data_ptr()), int(tick), _stream_ptr(stream)))

    def step(self, sample: torch.Tensor, tick: int, thr_dev: torch.Tensor | None = None, *,
             out=None, stream=None):
        """push(sample, tick) + detect(tick) in ONE launch (enova_stream_step)."""
        _require_cuda(sample, "sample")
        if tuple(sample.shape) != (self.n, self.M) or not sample.is_contiguous():
            raise ValueError(f"sample must be contiguous [{self.n}, {self.M}]")
        dev = self.buf.device
        if out is None:
            flags = torch.empty(self.n, dtype=torch.int8, device=dev) if thr_dev is not None else None
            sc = torch.empty(self.n, dtype=torch.float32, device=dev)
            md = torch.empty(self.n, dtype=torch.float32, device=dev)
        else:
            flags, sc, md = out
        ptr = lambda t: C.c_void_p(t.data_ptr() if t is not None else None)
        check(lib().enova_stream_step(C.c_void_p(self.buf.data_ptr()), self.n, int(tick),
                                      ptr(sample), ptr(self.mean), ptr(self.std),
                                      C.byref(self.det.struct), C.c_void_p(self.det.ws.data_ptr()),
                                      self.det.ws_bytes, ptr(thr_dev), ptr(flags), ptr(sc), ptr(md),
                                      _stream_ptr(stream)))
        return flags, sc, md

    def detect(self, tick: int, thr_dev: torch.Tensor | None = None, *, out=None, stream=None):
        """(flags, scores, md) of the windows ending at `tick`, each [n]; flags
        need a device threshold (threshold_to_device / fit_threshold_async)."""
        dev = self.buf.device
        if out is None:
            flags = torch.empty(self.n, dtype=torch.int8, device=dev) if thr_dev is not None else None
            sc = torch.empty(self.n, dtype=torch.float32, device=dev)
            md = torch.empty(self.n, dtype=torch.float32, device=dev)
        else:
            flags, sc, md = out
        ptr = lambda t: C.c_void_p(t.data_ptr() if t is not None else None)
        check(lib().enova_stream_detect(C.c_void_p(self.buf.data_ptr()), self.n, int(tick),
                                        C.byref(self.det.struct), C.c_void_p(self.det.ws.data_ptr()),
                                        self.det.ws_bytes, ptr(thr_dev), ptr(flags), ptr(sc), ptr(md),
                                        _stream_ptr(stream)))
        return flags, sc, md


class Spot:
    """NEXT-2 online SPOT state on one GPU: calibrate() fits the initial POT
    threshold (device-resident, `thr` usable by detect_async / StreamRing.detect);
    update(scores, flags) adds a tick's non-anomalous peaks; refit() re-fits.

    Capacity: the peak buffer holds the calibration peaks (<= ceil((1-q0) n_cal)
    + 16) plus `stream_peaks` streamed ones (default: as many again as the
    calibration).  Peaks beyond it are dropped and every later refit reports
    ENOVA_ERR_WORKSPACE (threshold() raises) until the next calibrate()."""

    def __init__(self, n_calibration: int, init_quantile: float = 0.98, risk_q: float = 1e-3,
                 device=None, stream_peaks: int | None = None):
        self.q0, self.q = float(init_quantile), float(risk_q)
        n_cal = int(n_calibration)
        if stream_peaks is None:
            stream_peaks = int(math.ceil((1.0 - self.q0) * n_cal)) + 16
        self.n_calibration = n_cal
        self.stream_peaks = int(stream_peaks)
        # the workspace cap is ceil((1 - q0) n_max) + 16 peaks
        n_max = n_cal + int(math.ceil(self.stream_peaks / max(1.0 - self.q0, 1e-12)))
        self.ws = ThresholdWorkspace(n_max, self.q0, device)
        self.thr = torch.zeros(THRESHOLD_BYTES, dtype=torch.uint8, device=device or "cuda")

    def calibrate(self, scores: torch.Tensor, stream=None):
        fit_threshold_async(scores, self.q0, self.q, workspace=self.ws, out=self.thr, stream=stream)
        return self.thr

    def update(self, scores: torch.Tensor, flags: torch.Tensor, stream=None):
        _require_cuda(scores, "scores")
        _require_cuda(flags, "flags", torch.int8)
        s, f = scores.reshape(-1), flags.reshape(-1)
        if s.numel() != f.numel() or not s.is_contiguous() or not f.is_contiguous():
            raise ValueError("scores and flags: contiguous, same length")
        check(lib().enova_spot_update(C.c_void_p(s.data_ptr()), C.c_void_p(f.data_ptr()), s.numel(),
                                      C.c_void_p(self.ws.buf.data_ptr()), self.ws.nbytes,
                                      self.ws.n_global_max, self.q0, _stream_ptr(stream)))

    def refit(self, stream=None):
        check(lib().enova_spot_refit(self.q, C.c_void_p(self.thr.data_ptr()),
                                     C.c_void_p(self.ws.buf.data_ptr()), self.ws.nbytes,
                                     self.ws.n_global_max, self.q0, _stream_ptr(stream)))
        return self.thr

    def threshold(self) -> dict:
        return threshold_from_device(self.thr)


def select_flagged(flags: torch.Tensor, stream=None) -> torch.Tensor:
    """NEXT-1 helper: ascending flat indices of the nonzero flags (device int64;
    synchronises once to read the count)."""
    _require_cuda(flags, "flags", torch.int8)
    f = flags.reshape(-1)
    n = f.numel()
    ids = torch.empty(max(n, 1), dtype=torch.int64, device=flags.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=flags.device)
    scratch = torch.empty(max(int(lib().enova_select_flagged_scratch_bytes(n)), 1),
                          dtype=torch.uint8, device=flags.device)
    check(lib().enova_select_flagged(C.c_void_p(f.data_ptr()), n, C.c_void_p(ids.data_ptr()),
                                     C.c_void_p(cnt.data_ptr()), C.c_void_p(scratch.data_ptr()),
                                     _stream_ptr(stream)))
    return ids[:int(cnt.item())]


def explain_windows(metrics: torch.Tensor, det: PreparedDetector, mean: torch.Tensor,
                    std: torch.Tensor, ids: torch.Tensor, t_begin: int | None = None,
                    t_end: int | None = None, *, stream=None):
    """NEXT-1: per-metric mean difference [n_ids, M] (+ score, MD) of the windows
    with ids g = instance * nw + (t - t_begin) of the range [t_begin, t_end)."""
    N, T, M = metrics.shape
    tb = det.window - 1 if t_begin is None else int(t_begin)
    te = T if t_end is None else int(t_end)
    s = _series(metrics, mean, std, tb, te)
    ids = ids.to(device=metrics.device, dtype=torch.int64).contiguous()
    n = ids.numel()
    mdm = torch.empty((n, M), dtype=torch.float32, device=metrics.device)
    sc = torch.empty(n, dtype=torch.float32, device=metrics.device)
    md = torch.empty(n, dtype=torch.float32, device=metrics.device)
    check(lib().enova_explain_windows(C.byref(s), C.byref(det.struct), C.c_void_p(det.ws.data_ptr()),
                                      det.ws_bytes, C.c_void_p(ids.data_ptr() if n else None), n,
                                      C.c_void_p(mdm.data_ptr()), C.c_void_p(sc.data_ptr()),
                                      C.c_void_p(md.data_ptr()), _stream_ptr(stream)))
    return mdm, sc, md


def point_adjusted_counts(labels: torch.Tensor, flags: torch.Tensor, t_begin: int, *,
                          out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """NEXT-4: device uint64[4] (as int64) = {TP, FP, FN, TN} of the point-adjusted
    evaluation of `flags` [N, nw] against `labels` [N, T] (int8, != 0 = anomaly)
    at the window end times t_begin .. t_begin + nw - 1."""
    _require_cuda(labels, "labels", torch.int8)
    _require_cuda(flags, "flags", torch.int8)
    if labels.dim() != 2 or flags.dim() != 2 or labels.shape[0] != flags.shape[0]:
        raise ValueError("labels [N, T] and flags [N, nw] expected")
    if labels.stride(1) != 1 or not flags.is_contiguous():
        raise ValueError("labels rows and flags must be contiguous")
    N, nw = flags.shape
    ld = labels.stride(0) if N > 1 else labels.shape[1]
    counts = out if out is not None else torch.empty(4, dtype=torch.int64, device=flags.device)
    check(lib().enova_point_adjusted_counts(C.c_void_p(labels.data_ptr()), ld,
                                            C.c_void_p(flags.data_ptr()), N, int(t_begin), nw,
                                            C.c_void_p(counts.data_ptr()), _stream_ptr(stream)))
    return counts


def point_adjusted_f1(labels: torch.Tensor, flags: torch.Tensor, t_begin: int, comm=None) -> dict:
    """Precision / recall / F1 (point-adjusted) of the flags; with a torch.distributed
    process group the integer counts are summed over ranks first (exact)."""
    c = point_adjusted_counts(labels, flags, t_begin)
    if comm is not None:
        import torch.distributed as dist
        dist.all_reduce(c, group=comm)
    tp, fp, fn, tn = (int(v) for v in c.cpu().tolist())
    prec = tp / (tp + fp) if tp + fp else 0.0
    rec = tp / (tp + fn) if tp + fn else 0.0
    f1 = 2 * prec * rec / (prec + rec) if prec + rec else 0.0
    return dict(tp=tp, fp=fp, fn=fn, tn=tn, precision=prec, recall=rec, f1=f1)


class Comm:
    """Communicator for the fleet-wide threshold (one per rank): NCCL (one process
    per GPU, `create`) or in-process (`create_local`: `world` ranks driven by host
    threads of one process on one GPU -- runs the multi-rank path on one device)."""

    def __init__(self, handle: int, rank: int, world: int, local: bool = False):
        self.handle, self.rank, self.world, self.local = handle, rank, world, local

    @staticmethod
    def create_local(world: int, device: int = 0) -> "list[Comm]":
        hs = (C.c_void_p * world)()
        check(lib().enova_comm_create_local(hs, int(world), int(device)))
        return [Comm(hs[r], r, world, local=True) for r in range(world)]

    def set_timeout(self, seconds: float):
        """Bound of every host-side wait on this communicator (default 300 s)."""
        check(lib().enova_comm_set_timeout(C.c_void_p(self.handle), float(seconds)))

    def wait(self, stream=None):
        """Bounded wait for the work enqueued on `stream`: a dead peer or an async
        NCCL error raises ENOVA_ERR_NCCL (the communicator is aborted) instead of
        hanging."""
        check(lib().enova_comm_wait(C.c_void_p(self.handle), _stream_ptr(stream)))

    def sum_i64(self, value: int, stream=None) -> int:
        """Synchronous sum of one integer over the ranks (collective)."""
        out = C.c_int64()
        check(lib().enova_comm_sum_i64(C.c_void_p(self.handle), int(value), C.byref(out),
                                       _stream_ptr(stream)))
        return int(out.value)

    @staticmethod
    def unique_id(rank: int, world: int, group=None) -> bytes:
        """Rank 0 draws the NCCL id (enova_comm_unique_id); every rank returns it."""
        from .fleet import broadcast_unique_id
        raw = None
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            check(lib().enova_comm_unique_id(buf))
            raw = bytes(buf)
        return broadcast_unique_id(raw, rank, world, group)

    @staticmethod
    def create(rank: int, world: int, device: int, group=None) -> "Comm":
        raw = (C.c_uint8 * 128)(*Comm.unique_id(rank, world, group))
        h = C.c_void_p()
        check(lib().enova_comm_create(C.byref(h), rank, world, raw, device))
        return Comm(h.value, rank, world)

    def destroy(self):
        if self.handle:
            lib().enova_comm_destroy(C.c_void_p(self.handle))
            self.handle = None


@dataclass
class PipelineResult:
    mean: torch.Tensor
    std: torch.Tensor
    n_degenerate: int
    cal_scores: torch.Tensor
    threshold: dict
    flags: torch.Tensor
    scores: torch.Tensor | None
    md: torch.Tensor | None
    cal_md: torch.Tensor | None = None
    cal_flags: torch.Tensor | None = None


def run_pipeline(metrics: torch.Tensor, det: PreparedDetector, t_cal_end: int,
                 init_quantile: float = 0.98, risk_q: float = 1e-3, comm: Comm | None = None,
                 workspace: ThresholdWorkspace | None = None, return_scores: bool = True,
                 stream=None) -> PipelineResult:
    """One pass of the whole hot path: stats over [0, t_cal_end) -> scores and MD
    of the calibration windows (ending in [W-1, t_cal_end)) -> fleet-wide POT
    threshold -> flags of the calibration windows -> flags (and scores/MD) of
    the windows ending in [t_cal_end, T)."""
    T = metrics.shape[1]
    mean, std, nd = compute_stats(metrics, t_cal_end, stream=stream)
    cal, cal_md = score_windows(metrics, det, mean, std, det.window - 1, t_cal_end,
                                stream=stream)
    thr = fit_threshold(cal, init_quantile, risk_q, comm=comm, workspace=workspace, stream=stream)
    thr_d = threshold_to_device(thr, metrics.device)
    if stream is not None:
        thr_d.record_stream(stream)
    cal_flags = flag_scores_async(cal, cal_md, thr_d, stream=stream)
    res = detect(metrics, det, mean, std, thr, t_cal_end, T, return_scores=return_scores,
                 stream=stream)
    if return_scores:
        flags, sc, md = res
    else:
        flags, sc, md = res, None, None
    return PipelineResult(mean, std, nd, cal, thr, flags, sc, md, cal_md, cal_flags)


def fit_threshold_dist_async(scores: torch.Tensor, n_global: int, comm: "Comm",
                             init_quantile: float = 0.98, risk_q: float = 1e-3, *,
                             workspace: ThresholdWorkspace | None = None, out=None,
                             stream=None) -> torch.Tensor:
    """The distributed-fit variant of fit_threshold_comm_async
    (enova_fit_threshold_dist_async): every rank fits on its own tail with the
    ranks' pass totals all-gathered between fit steps.  Returns the DEVICE
    enova_threshold (identical on every rank)."""
    _require_cuda(scores, "scores")
    flat = scores.reshape(-1)
    if not flat.is_contiguous():
        flat = flat.contiguous()
    if workspace is None:
        workspace = ThresholdWorkspace(n_global, init_quantile, scores.device, world=comm.world)
    thr = out if out is not None else torch.zeros(THRESHOLD_BYTES, dtype=torch.uint8,
                                                  device=scores.device)
    check(lib().enova_fit_threshold_dist_async(
        C.c_void_p(flat.data_ptr()), flat.numel(), int(n_global), workspace.n_global_max,
        float(init_quantile), float(risk_q), C.c_void_p(comm.handle), C.c_void_p(thr.data_ptr()),
        C.c_void_p(workspace.buf.data_ptr()), workspace.nbytes, _stream_ptr(stream)))
    return thr


class Pipeline:
    """The whole hot path for a fixed fleet shape, preallocated and stream-ordered:
    stats over [0, t_cal_end) -> calibration scores and MD -> single-GPU POT
    threshold (device-resident) -> flags of the calibration windows -> flags /
    scores / MD of the windows ending in [t_cal_end, T): every window of the
    trace ends the step with a score, an MD and a flag.  `enqueue` issues the step with no host synchronisation;
    `capture` records it into a CUDA graph that `replay` relaunches (one graph
    launch per step); `result` synchronises and checks the device statuses.
    With a communicator (fleet sharded over ranks) the threshold is the
    collective, stream-ordered enova_fit_threshold_comm_async: still no host
    synchronisation, and with NCCL the step (collectives included) is captured
    into the graph too; an in-process communicator's step is enqueued eagerly
    (one host thread per rank).  Construction with a communicator is collective
    (the global calibration score count is summed once)."""

    def __init__(self, det: PreparedDetector, n_instances: int, n_steps: int, t_cal_end: int,
                 init_quantile: float = 0.98, risk_q: float = 1e-3, return_scores: bool = True,
                 device=None, comm: "Comm | None" = None, overlap: bool = True,
                 pot_ctas: int = 32, concurrent_instances: int | None = None,
                 fit_mode: str = "replicated"):
        dev = torch.device(device or "cuda")
        # the overlapped step (enova_step: the fit on pot_ctas CTAs next to the
        # detection scores) needs the detection scores and MD buffers
        overlap = overlap and not (comm is not None and comm.local)
        return_scores = return_scores or overlap
        W, M = det.window, det.n_metrics
        self.det, self.N, self.T, self.M, self.tcal = det, int(n_instances), int(n_steps), M, int(t_cal_end)
        self.q0, self.q = float(init_quantile), float(risk_q)
        N, T, tcal = self.N, self.T, self.tcal
        self.mean = torch.empty((N, M), dtype=torch.float32, device=dev)
        self.std = torch.empty((N, M), dtype=torch.float32, device=dev)
        self.diag = torch.zeros(2, dtype=torch.int64, device=dev)
        self.cal = torch.empty((N, max(tcal - (W - 1), 0)), dtype=torch.float32, device=dev)
        self.cal_md = torch.empty_like(self.cal)
        self.cal_flags = torch.empty(tuple(self.cal.shape), dtype=torch.int8, device=dev)
        self.thr = torch.zeros(THRESHOLD_BYTES, dtype=torch.uint8, device=dev)
        self.flags = torch.empty((N, T - tcal), dtype=torch.int8, device=dev)
        self.scores = torch.empty((N, T - tcal), dtype=torch.float32, device=dev) if return_scores else None
        self.md = torch.empty((N, T - tcal), dtype=torch.float32, device=dev) if return_scores else None
        self.stats_ws = StatsWorkspace(N, M, dev)
        self.comm = comm
        if comm is not None:
            self.n_global = comm.sum_i64(self.cal.numel())
            self.thr_ws = ThresholdWorkspace(max(self.n_global, 1), self.q0, dev, world=comm.world)
        else:
            self.n_global = self.cal.numel()
            self.thr_ws = ThresholdWorkspace(max(self.cal.numel(), 1), self.q0, dev)
        self.graph = None
        self._graph_input = None
        h = C.c_void_p()
        check(lib().enova_step_create(C.byref(h), dev.index if dev.index is not None
                                      else torch.cuda.current_device()))
        self._step = h.value
        if fit_mode not in ("replicated", "distributed"):
            raise ValueError("fit_mode must be 'replicated' or 'distributed'")
        self.fit_mode = fit_mode
        check(lib().enova_step_set_fit_mode(C.c_void_p(self._step),
                                            1 if fit_mode == "distributed" else 0))
        self.overlap = bool(overlap)
        if concurrent_instances is None:
            concurrent_instances = (2 * N) // 5 if overlap else 0
        self.configure(pot_ctas if overlap else 0, concurrent_instances)

    def configure(self, pot_ctas: int, concurrent_instances: int):
        """Overlap of the fit with the detection scores (enova_step_configure):
        pot_ctas = 0 runs the stages in sequence."""
        check(lib().enova_step_configure(C.c_void_p(self._step), int(pot_ctas),
                                         int(concurrent_instances)))
        self.pot_ctas, self.concurrent_instances = int(pot_ctas), int(concurrent_instances)

    def tune(self, metrics: torch.Tensor, candidates=None, reps: int = 5) -> dict:
        """Pick the fastest step configuration on `metrics` (a fixed device buffer):
        each candidate (pot_ctas, concurrent_instances) -- (0, 0) is the sequential
        order -- is captured and replayed `reps` times; every candidate gives the
        same scores, MD and flags (the fit differs only in summation order), so
        the choice is by time alone.  Leaves the winner configured and captured."""
        if self.comm is not None and self.comm.local:
            return {"pot_ctas": 0, "concurrent_instances": 0, "ms": None}
        N = self.N
        if candidates is None:
            candidates = [(0, 0)]
            if self.overlap:
                for pot in (24, 32):
                    for frac in (0.15, 0.3, 0.45, 0.6, 0.75):
                        candidates.append((pot, int(frac * N)))
        s = torch.cuda.current_stream(metrics.device)
        best, timings = None, []
        for pot, conc in candidates:
            self.configure(pot, conc)
            self.capture(metrics)
            self.replay()
            s.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(reps):
                self.replay()
            b.record(s)
            s.synchronize()
            ms = a.elapsed_time(b) / reps
            timings.append((pot, conc, ms))
            if best is None or ms < best[2]:
                best = (pot, conc, ms)
        self.configure(best[0], best[1])
        self.capture(metrics)
        return {"pot_ctas": best[0], "concurrent_instances": best[1], "ms": best[2],
                "candidates": timings}

    def __del__(self):
        try:
            if getattr(self, "_step", None):
                lib().enova_step_destroy(C.c_void_p(self._step))
                self._step = None
        except Exception:   # noqa: BLE001 -- interpreter shutdown
            pass

    def enqueue(self, metrics: torch.Tensor, stream=None):
        """One step (enova_step_enqueue): stats -> calibration scores + MD -> fit
        (fleet-wide with a communicator) -> detection scores + MD -> every flag."""
        if tuple(metrics.shape) != (self.N, self.T, self.M):
            raise ValueError(f"metrics must be [{self.N}, {self.T}, {self.M}]")
        s = _series(metrics)
        ptr = lambda t: t.data_ptr() if t is not None else None
        a = StepArgs()
        a.series = C.cast(C.pointer(s), C.c_void_p)
        a.t_cal_end = self.tcal
        a.det = C.cast(C.pointer(self.det.struct), C.c_void_p)
        a.det_ws, a.det_ws_bytes = self.det.ws.data_ptr(), self.det.ws_bytes
        a.init_quantile, a.risk_q = self.q0, self.q
        a.comm = self.comm.handle if self.comm is not None else None
        a.n_global, a.n_global_max = self.n_global, self.thr_ws.n_global_max
        a.mean, a.std, a.stats_diag = ptr(self.mean), ptr(self.std), ptr(self.diag)
        a.stats_ws, a.stats_ws_bytes = self.stats_ws.buf.data_ptr(), self.stats_ws.nbytes
        a.cal_scores, a.cal_md, a.cal_flags = ptr(self.cal), ptr(self.cal_md), ptr(self.cal_flags)
        a.thr_dev = ptr(self.thr)
        a.thr_ws, a.thr_ws_bytes = self.thr_ws.buf.data_ptr(), self.thr_ws.nbytes
        a.scores, a.md, a.flags = ptr(self.scores), ptr(self.md), ptr(self.flags)
        self._args_keep = (s, a)
        check(lib().enova_step_enqueue(C.c_void_p(self._step), C.byref(a), _stream_ptr(stream)))

    def capture(self, metrics: torch.Tensor):
        """Record one step on `metrics` (a fixed device buffer) into a CUDA graph."""
        if self.comm is not None and self.comm.local:
            raise RuntimeError("an in-process communicator's collectives cannot be captured")
        side = torch.cuda.Stream(device=metrics.device)
        side.wait_stream(torch.cuda.current_stream(metrics.device))
        with torch.cuda.stream(side):
            self.enqueue(metrics)            # warm-up outside capture (one-time attributes)
        torch.cuda.current_stream(metrics.device).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            self.enqueue(metrics)
        self.graph, self._graph_input = g, metrics
        return g

    def replay(self):
        if self.graph is None:
            raise RuntimeError("capture() first")
        self.graph.replay()

    def result(self) -> PipelineResult:
        if self.comm is not None and not self.comm.local:
            self.comm.wait()          # bounded: a dead peer raises instead of hanging
        nd = check_stats_diag(self.diag)
        thr = threshold_from_device(self.thr)
        return PipelineResult(self.mean, self.std, nd, self.cal, thr, self.flags, self.scores,
                              self.md, self.cal_md, self.cal_flags)


# ------------------------------------------------------------------ NEXT-3 ----
TRAIN_PARAMS = _WEIGHT_KEYS


def train_config(lr=1e-3, latent=4, kl_setpoint=None, kp=0.01, ki=0.001, beta_max=1.0,
                 beta_fixed=None, adam_beta1=0.9, adam_beta2=0.999, adam_eps=1e-8) -> TrainConfig:
    """Eq. 9 training constants (SPEC.md:548-550 defaults; R-24): PI
    setpoint 0.5 * latent nats unless given; beta_fixed switches the PI off."""
    c = TrainConfig()
    c.lr, c.adam_beta1, c.adam_beta2, c.adam_eps = lr, adam_beta1, adam_beta2, adam_eps
    c.kl_setpoint = 0.5 * latent if kl_setpoint is None else kl_setpoint
    c.kp, c.ki, c.beta_max = kp, ki, beta_max
    c.beta_mode = 0 if beta_fixed is None else 1
    c.beta_fixed = 0.0 if beta_fixed is None else beta_fixed
    return c


class Trainer:
    """NEXT-3: Eq. 9 training state on one GPU (enova_trainer_*): fp32 master
    parameters, Adam moments, the PI-controlled beta, activations for up to
    max_batch windows, and a cuBLAS handle for the GEMMs."""

    def __init__(self, window: int, n_metrics: int, hidden: int, latent: int, max_batch: int,
                 device=None):
        dev = torch.device(device or "cuda")
        self.device = dev
        self.W, self.M, self.H, self.Z, self.max_batch = window, n_metrics, hidden, latent, max_batch
        h = C.c_void_p()
        check(lib().enova_trainer_create(C.byref(h), window, n_metrics, hidden, latent, max_batch,
                                         dev.index if dev.index is not None else
                                         torch.cuda.current_device()))
        self.handle = h.value
        off = (C.c_int64 * 10)()
        self.n_params = int(lib().enova_trainer_param_offsets(C.c_void_p(self.handle), off))
        self.offsets = list(off)
        self.stats = torch.zeros(4, dtype=torch.float64, device=dev)

    def _shapes(self):
        D, H, Z = self.W * self.M, self.H, self.Z
        return {"enc_w1": (H, D), "enc_b1": (H,), "enc_wmu": (Z, H), "enc_bmu": (Z,),
                "enc_wlv": (Z, H), "enc_blv": (Z,), "dec_w1": (H, Z), "dec_b1": (H,),
                "dec_w2": (D, H), "dec_b2": (D,)}

    def _struct(self, tensors: dict) -> Detector:
        return Detector(self.W, self.M, self.H, self.Z, *[tensors[k].data_ptr() for k in _WEIGHT_KEYS])

    def set_math(self, tf32: bool):
        check(lib().enova_trainer_set_math(C.c_void_p(self.handle), 1 if tf32 else 0))

    def load(self, weights: dict, beta0: float = 0.0, stream=None):
        t = {}
        for k in _WEIGHT_KEYS:
            v = weights[k]
            if isinstance(v, np.ndarray):
                v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))
            t[k] = v.to(device=self.device, dtype=torch.float32).contiguous()
        self._loaded = t          # keep alive until the stream-ordered copies ran
        check(lib().enova_trainer_load(C.c_void_p(self.handle), C.byref(self._struct(t)),
                                       float(beta0), _stream_ptr(stream)))

    def weights(self, stream=None) -> dict:
        """The current parameters as a detector weight dict (device fp32 tensors)."""
        out = {k: torch.empty(sh, dtype=torch.float32, device=self.device)
               for k, sh in self._shapes().items()}
        check(lib().enova_trainer_store(C.c_void_p(self.handle), C.byref(self._struct(out)),
                                        _stream_ptr(stream)))
        out.update(window=self.W, n_metrics=self.M, hidden=self.H, latent=self.Z)
        return out

    def _args(self, metrics, mean, std, t_begin, t_end, ids, labels, eps):
        s = _series(metrics, mean, std, t_begin, t_end)
        _require_cuda(ids, "ids", torch.int64)
        _require_cuda(labels, "labels", torch.int8)
        _require_cuda(eps, "eps")
        B = ids.numel()
        if labels.numel() != s.n_instances * max(s.t_end - s.t_begin, 0) or eps.numel() != B * self.Z:
            raise ValueError("ids [B], labels [n_windows of the range] (by window id), eps [B, latent]")
        if not labels.is_contiguous() or not ids.is_contiguous() or not eps.is_contiguous():
            raise ValueError("ids, labels and eps must be contiguous")
        return s, B

    def step(self, metrics, mean, std, t_begin, t_end, ids, labels, eps, cfg: TrainConfig,
             stream=None):
        s, B = self._args(metrics, mean, std, t_begin, t_end, ids, labels, eps)
        check(lib().enova_train_step(C.c_void_p(self.handle), C.byref(s), C.c_void_p(ids.data_ptr()),
                                     C.c_void_p(labels.data_ptr()), B, C.c_void_p(eps.data_ptr()),
                                     C.byref(cfg), C.c_void_p(self.stats.data_ptr()),
                                     _stream_ptr(stream)))
        return self.stats

    def gradient(self, metrics, mean, std, t_begin, t_end, ids, labels, eps, beta: float,
                 stream=None) -> dict:
        s, B = self._args(metrics, mean, std, t_begin, t_end, ids, labels, eps)
        g = torch.empty(self.n_params, dtype=torch.float32, device=self.device)
        check(lib().enova_train_gradient(C.c_void_p(self.handle), C.byref(s),
                                         C.c_void_p(ids.data_ptr()), C.c_void_p(labels.data_ptr()),
                                         B, C.c_void_p(eps.data_ptr()), float(beta),
                                         C.c_void_p(g.data_ptr()), C.c_void_p(self.stats.data_ptr()),
                                         _stream_ptr(stream)))
        out = {}
        for k, o in zip(_WEIGHT_KEYS, self.offsets):
            sh = self._shapes()[k]
            out[k] = g[o:o + int(np.prod(sh))].view(sh)
        return out

    def fit(self, metrics, mean, std, t_begin, t_end, labels_per_window: torch.Tensor,
            order: torch.Tensor, eps: torch.Tensor, batch: int, cfg: TrainConfig,
            history: bool = False, stream=None):
        """Every step of a schedule: order [steps * batch] window ids (-1 = padding)
        and eps [steps * batch, latent] (device), labels_per_window [n_windows] int8
        (+1 / -1) of the series range.  Returns the per-step stats [steps, 4] (device)
        when history is set."""
        steps = order.numel() // batch
        hist = torch.empty((steps, 4), dtype=torch.float64, device=self.device) if history else None
        for k in range(steps):
            sl = slice(k * batch, (k + 1) * batch)
            st = self.step(metrics, mean, std, t_begin, t_end, order[sl], labels_per_window,
                           eps[sl], cfg, stream=stream)
            if hist is not None:
                hist[k].copy_(st)
        return hist

    def destroy(self):
        if getattr(self, "handle", None):
            lib().enova_trainer_destroy(C.c_void_p(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:   # noqa: BLE001 -- interpreter shutdown
            pass
