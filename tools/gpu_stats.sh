mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "stats or c1_pipeline or async_pipeline" > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_series_stats -s 1 -c 1 -f -o gpurun_out/prof_stats python tools/profile_run.py 2 > gpurun_out/prof_stats.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-traffic --no-e2e > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
python -c "import json; d=json.loads(open('gpurun_out/bench.jsonl').readline()); print(d['value'], d['ms_per_step'], d['stage_ms'])"
