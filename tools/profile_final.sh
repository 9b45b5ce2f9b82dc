#!/bin/bash
# End-of-round profile pass (run under gpurun): ncu launch list of 2 default
# bench steps, ncu --set full of the hot kernels (c2 K2, K1, k_pot; c5 k_pot fit
# launch; c4 k_stream_rows), trace of the K2 pipeline.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e > gpurun_out/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score_pair -s 2 -c 1 \
   -f -o gpurun_out/prof_score python tools/profile_run.py 2 > gpurun_out/prof_score.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_pot -s 1 -c 1 \
   -f -o gpurun_out/prof_pot python tools/profile_run.py 2 > gpurun_out/prof_pot.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_series_stats -s 1 -c 1 \
   -f -o gpurun_out/prof_stats python tools/profile_run.py 2 > gpurun_out/prof_stats.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_pot -s 1 -c 1 \
   -f -o gpurun_out/prof_pot5 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_pot5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_rows -s 5 -c 1 \
   -f -o gpurun_out/prof_stream python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof_stream.log 2>&1
timeout 300 python tools/pot_phases.py --c5 > gpurun_out/pot_phases.txt 2>&1
timeout 300 python tools/trace_pair.py > gpurun_out/trace_pair.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" >> gpurun_out/build.log 2>&1   # back to the untraced build
ls -la gpurun_out/*.ncu-rep
