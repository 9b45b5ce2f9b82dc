#!/bin/bash
# Round-2 profile pass (run under gpurun): ncu launch list of 2 c2 steps, ncu --set full
# of the hot kernels, compute-sanitizer (memcheck/racecheck/synccheck) over small GPU tests.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_pair -s 2 -c 1 \
   -f -o gpurun_out/prof_score python tools/profile_run.py 2 > gpurun_out/prof_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pot -s 1 -c 1 \
   -f -o gpurun_out/prof_pot python tools/profile_run.py 2 > gpurun_out/prof_pot.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_series_stats -s 1 -c 1 \
   -f -o gpurun_out/prof_stats python tools/profile_run.py 2 > gpurun_out/prof_stats.log 2>&1
K="test_scores_match_oracle_shapes or test_row_kernel_matches or test_stream_ring_matches_batch_and_oracle or test_threshold_on_identical_scores or test_stats_match_oracle or test_point_adjusted or test_c1_pipeline or test_explain_windows or test_spot_ticks or test_gradient_matches"
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --target-processes all \
     python -m pytest tests -m gpu -q -x -k "$K" -p no:cacheprovider > gpurun_out/sanitizer_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.log
done
tail -3 gpurun_out/sanitizer_*.log
