#!/bin/bash
# Round profile pass (run under gpurun): default bench line, workload lines,
# ncu launch list of 2 c2 steps, ncu --set full captures of the hot kernels.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/bench_$w.jsonl 2> gpurun_out/bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_run.py 2 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_score_pair -s 2 -c 1 \
   -f -o gpurun_out/prof_score python tools/profile_run.py 2 > gpurun_out/prof_score.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pot -s 1 -c 1 \
   -f -o gpurun_out/prof_pot python tools/profile_run.py 2 > gpurun_out/prof_pot.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_series_stats -s 1 -c 1 \
   -f -o gpurun_out/prof_stats python tools/profile_run.py 2 > gpurun_out/prof_stats.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stream_rows -s 5 -c 1 \
   -f -o gpurun_out/prof_stream python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof_stream.log 2>&1
./tools/ubench_mma > gpurun_out/ubench_mma.txt 2>&1 || true
python tools/pot_phases.py --c5 > gpurun_out/pot_phases.txt 2>&1
python tools/trace_pair.py > gpurun_out/trace_pair.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/build.log 2>&1   # back to the untraced build
python tools/trace_stream.py > gpurun_out/trace_stream.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/build.log 2>&1
cat gpurun_out/bench.jsonl
