#!/bin/bash
# Full GPU validation + evidence pass (run under gpurun): build, every GPU test,
# smoke, compute-sanitizer (memcheck / racecheck / synccheck) over the small GPU
# tests, bench lines for c2 (default), c3, c4, c5.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
K="test_scores_match_oracle_shapes or test_row_kernel_matches or test_stream_ring_matches_batch_and_oracle or test_threshold_on_identical_scores or test_stats_match_oracle or test_point_adjusted or test_c1_pipeline or test_explain_windows or test_spot_ticks or test_gradient_matches or test_distributed_fit_matches"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --target-processes all \
     python -m pytest tests -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/sanitizer_$tool.log | tail -2
done
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.jsonl 2> gpurun_out/bench_$w.err
done
python - <<'PY'
import json
for f in ["bench", "bench_c3", "bench_c4", "bench_c5"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.jsonl").read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f, d["value"], d["unit"], "ms", d.get("ms_per_step"), "frac", r.get("frac"), "e2e", (d.get("e2e") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
