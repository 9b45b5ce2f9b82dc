"""ctypes binding of libenova.so (include/enova.h).  Argument marshalling only:
every step of the detection path runs in the library's CUDA kernels.  torch
supplies device memory and streams.  There is no fallback: if the library is
missing or the GPU is absent the calls raise."""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libenova.so")

ENOVA_OK = 0
STATUS = {
    0: "ENOVA_OK", 1: "ENOVA_ERR_INVALID_ARGUMENT", 2: "ENOVA_ERR_UNSUPPORTED",
    3: "ENOVA_ERR_INSUFFICIENT_HISTORY", 4: "ENOVA_ERR_TOO_FEW_EXCEEDANCES",
    5: "ENOVA_ERR_NONFINITE", 6: "ENOVA_ERR_UNCALIBRATED", 7: "ENOVA_ERR_CUDA",
    8: "ENOVA_ERR_NCCL", 9: "ENOVA_ERR_WORKSPACE",
}

# every symbol include/enova.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "enova_detector_workspace_bytes", "enova_prepare_detector", "enova_stats_workspace_bytes",
    "enova_compute_stats", "enova_score_windows", "enova_threshold_workspace_bytes",
    "enova_fit_threshold", "enova_detect", "enova_ring_push", "enova_comm_unique_id",
    "enova_comm_create", "enova_comm_destroy", "enova_status_string", "enova_last_error",
    "enova_abi_version", "enova_kernel_launches", "enova_compute_stats_async",
    "enova_fit_threshold_async", "enova_detect_async", "enova_stream_ring_bytes",
    "enova_stream_push", "enova_stream_detect", "enova_point_adjusted_counts",
    "enova_select_flagged_scratch_bytes", "enova_select_flagged", "enova_explain_windows",
    "enova_spot_update", "enova_spot_refit", "enova_stream_step",
    "enova_threshold_comm_workspace_bytes", "enova_fit_threshold_comm_async",
    "enova_comm_create_local", "enova_comm_sum_i64", "enova_set_score_kernel",
    "enova_flag_scores_async", "enova_comm_set_timeout", "enova_comm_wait",
    "enova_trainer_create", "enova_trainer_destroy", "enova_trainer_param_offsets",
    "enova_trainer_set_math", "enova_trainer_load", "enova_trainer_store", "enova_train_step",
    "enova_train_gradient", "enova_step_create", "enova_step_configure", "enova_step_enqueue",
    "enova_step_destroy", "enova_fit_threshold_dist_async", "enova_step_set_fit_mode",
)


class EnovaError(RuntimeError):
    def __init__(self, status: int, detail: str):
        self.status = status
        self.name = STATUS.get(status, str(status))
        super().__init__(f"{self.name}: {detail}")


class Detector(C.Structure):
    _fields_ = [("window", C.c_int32), ("n_metrics", C.c_int32), ("hidden", C.c_int32),
                ("latent", C.c_int32),
                ("enc_w1", C.c_void_p), ("enc_b1", C.c_void_p),
                ("enc_wmu", C.c_void_p), ("enc_bmu", C.c_void_p),
                ("enc_wlv", C.c_void_p), ("enc_blv", C.c_void_p),
                ("dec_w1", C.c_void_p), ("dec_b1", C.c_void_p),
                ("dec_w2", C.c_void_p), ("dec_b2", C.c_void_p)]


class TrainConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("adam_beta1", C.c_double), ("adam_beta2", C.c_double),
                ("adam_eps", C.c_double), ("kl_setpoint", C.c_double), ("kp", C.c_double),
                ("ki", C.c_double), ("beta_max", C.c_double), ("beta_mode", C.c_int32),
                ("reserved", C.c_int32), ("beta_fixed", C.c_double)]


class StepArgs(C.Structure):
    _fields_ = [("series", C.c_void_p), ("t_cal_end", C.c_int64), ("det", C.c_void_p),
                ("det_ws", C.c_void_p), ("det_ws_bytes", C.c_size_t),
                ("init_quantile", C.c_double), ("risk_q", C.c_double), ("comm", C.c_void_p),
                ("n_global", C.c_int64), ("n_global_max", C.c_int64),
                ("mean", C.c_void_p), ("std", C.c_void_p), ("stats_diag", C.c_void_p),
                ("stats_ws", C.c_void_p), ("stats_ws_bytes", C.c_size_t),
                ("cal_scores", C.c_void_p), ("cal_md", C.c_void_p), ("cal_flags", C.c_void_p),
                ("thr_dev", C.c_void_p), ("thr_ws", C.c_void_p), ("thr_ws_bytes", C.c_size_t),
                ("scores", C.c_void_p), ("md", C.c_void_p), ("flags", C.c_void_p)]


class Series(C.Structure):
    _fields_ = [("metrics", C.c_void_p), ("n_instances", C.c_int64), ("n_steps", C.c_int64),
                ("ld_instance", C.c_int64), ("t_begin", C.c_int64), ("t_end", C.c_int64),
                ("norm_mean", C.c_void_p), ("norm_std", C.c_void_p),
                ("n_metrics", C.c_int32), ("reserved", C.c_int32)]


class Threshold(C.Structure):
    _fields_ = [("init_quantile", C.c_double), ("risk_q", C.c_double), ("t", C.c_double),
                ("gamma", C.c_double), ("sigma", C.c_double), ("z_q", C.c_double),
                ("n", C.c_int64), ("n_peaks", C.c_int64), ("method", C.c_int32),
                ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libenova.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_2407_09486_b200.build)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        vp, i64, i32, dbl, sz = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_size_t
        P = C.POINTER
        sig = {
            "enova_detector_workspace_bytes": (sz, [P(Detector)]),
            "enova_prepare_detector": (C.c_int, [P(Detector), vp, sz, vp]),
            "enova_stats_workspace_bytes": (sz, [i64, i32]),
            "enova_compute_stats": (C.c_int, [P(Series), i64, vp, vp, P(i64), vp, sz, vp]),
            "enova_compute_stats_async": (C.c_int, [P(Series), i64, vp, vp, vp, vp, sz, vp]),
            "enova_fit_threshold_async": (C.c_int, [vp, i64, i64, dbl, dbl, vp, vp, sz, vp]),
            "enova_detect_async": (C.c_int, [P(Series), P(Detector), vp, sz, vp, vp, vp, vp, vp]),
            "enova_score_windows": (C.c_int, [P(Series), P(Detector), vp, sz, vp, vp, vp]),
            "enova_threshold_workspace_bytes": (sz, [i64, dbl]),
            "enova_fit_threshold": (C.c_int, [vp, i64, i64, dbl, dbl, vp, P(Threshold), vp, sz, vp]),
            "enova_detect": (C.c_int, [P(Series), P(Detector), vp, sz, P(Threshold), vp, vp, vp, vp]),
            "enova_ring_push": (C.c_int, [vp, i64, i32, i32, vp, i64, vp]),
            "enova_stream_ring_bytes": (sz, [i64, i32, i32]),
            "enova_point_adjusted_counts": (C.c_int, [vp, i64, vp, i64, i64, i64, vp, vp]),
            "enova_select_flagged_scratch_bytes": (sz, [i64]),
            "enova_spot_update": (C.c_int, [vp, vp, i64, vp, sz, i64, dbl, vp]),
            "enova_stream_step": (C.c_int, [vp, i64, i64, vp, vp, vp, P(Detector), vp, sz, vp, vp, vp, vp, vp]),
            "enova_spot_refit": (C.c_int, [dbl, vp, vp, sz, i64, dbl, vp]),
            "enova_select_flagged": (C.c_int, [vp, i64, vp, vp, vp, vp]),
            "enova_explain_windows": (C.c_int, [P(Series), P(Detector), vp, sz, vp, i64, vp, vp, vp, vp]),
            "enova_stream_push": (C.c_int, [vp, i64, i32, i32, vp, vp, vp, i64, vp]),
            "enova_stream_detect": (C.c_int, [vp, i64, i64, P(Detector), vp, sz, vp, vp, vp, vp, vp]),
            "enova_comm_unique_id": (C.c_int, [vp]),
            "enova_comm_create": (C.c_int, [P(vp), C.c_int, C.c_int, vp, C.c_int]),
            "enova_comm_destroy": (None, [vp]),
            "enova_comm_create_local": (C.c_int, [P(vp), C.c_int, C.c_int]),
            "enova_comm_sum_i64": (C.c_int, [vp, i64, P(i64), vp]),
            "enova_threshold_comm_workspace_bytes": (sz, [i64, dbl, i32]),
            "enova_fit_threshold_comm_async": (C.c_int, [vp, i64, i64, i64, dbl, dbl, vp, vp, vp,
                                                         sz, vp]),
            "enova_status_string": (C.c_char_p, [C.c_int]),
            "enova_last_error": (C.c_char_p, []),
            "enova_abi_version": (C.c_int, []),
            "enova_kernel_launches": (C.c_uint64, []),
            "enova_set_score_kernel": (C.c_int, [C.c_int]),
            "enova_flag_scores_async": (C.c_int, [vp, vp, i64, vp, vp, vp]),
            "enova_comm_set_timeout": (C.c_int, [vp, dbl]),
            "enova_trainer_create": (C.c_int, [P(vp), i32, i32, i32, i32, i32, C.c_int]),
            "enova_step_create": (C.c_int, [P(vp), C.c_int]),
            "enova_step_configure": (C.c_int, [vp, i32, i64]),
            "enova_step_set_fit_mode": (C.c_int, [vp, i32]),
            "enova_fit_threshold_dist_async": (C.c_int, [vp, i64, i64, i64, dbl, dbl, vp, vp, vp,
                                                         sz, vp]),
            "enova_step_enqueue": (C.c_int, [vp, P(StepArgs), vp]),
            "enova_step_destroy": (None, [vp]),
            "enova_trainer_destroy": (None, [vp]),
            "enova_trainer_param_offsets": (i64, [vp, P(i64)]),
            "enova_trainer_set_math": (C.c_int, [vp, i32]),
            "enova_trainer_load": (C.c_int, [vp, P(Detector), dbl, vp]),
            "enova_trainer_store": (C.c_int, [vp, P(Detector), vp]),
            "enova_train_step": (C.c_int, [vp, P(Series), vp, vp, i32, vp, P(TrainConfig), vp, vp]),
            "enova_train_gradient": (C.c_int, [vp, P(Series), vp, vp, i32, vp, dbl, vp, vp, vp]),
            "enova_comm_wait": (C.c_int, [vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
        return _lib


def check(status: int) -> None:
    if status != ENOVA_OK:
        detail = lib().enova_last_error()
        raise EnovaError(status, detail.decode() if detail else "")
