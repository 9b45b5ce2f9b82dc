"""B200-native ENOVA performance-detection hot path (arXiv 2407.09486).

Public API (thin binding over libenova.so, include/enova.h):
  PreparedDetector, compute_stats, score_windows, fit_threshold, detect,
  ring_push, ring_view, Comm, ThresholdWorkspace, run_pipeline; stream-ordered
  variants compute_stats_async, fit_threshold_async, detect_async,
  threshold_from_device, and Pipeline (preallocated step, CUDA-graph capture).
Seeded synthetic inputs live in ``paper_2407_09486_b200.synth``.
"""
__all__ = ["PreparedDetector", "compute_stats", "score_windows", "fit_threshold", "detect",
           "ring_push", "ring_view", "Comm", "ThresholdWorkspace", "run_pipeline",
           "EnovaError", "compute_stats_async", "fit_threshold_async", "fit_threshold_comm_async",
           "fit_threshold_dist_async",
           "detect_async",
           "threshold_from_device", "threshold_to_device", "check_stats_diag", "Pipeline",
           "StatsWorkspace", "StreamRing", "point_adjusted_counts", "point_adjusted_f1", "select_flagged",
           "explain_windows", "Spot", "force_score_kernel",
           "flag_scores_async", "Trainer", "train_config"]


def __getattr__(name):
    if name in __all__:
        from . import api
        from ._lib import EnovaError
        return EnovaError if name == "EnovaError" else getattr(api, name)
    raise AttributeError(name)
