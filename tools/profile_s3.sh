#!/bin/bash
# Round-2 (session 3) evidence pass (run under gpurun): GPU tests, smoke, the
# four bench lines, the ingest microbenchmark, ncu launch list of the default
# bench and ncu --set full of the hot kernels (c2 K2, c2 k_pot, c5 k_pot_scan +
# k_pot, c4 k_stream_rows), k_pot phase stamps.  Outputs under gpurun_out/s3/.
O=gpurun_out/s3
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 600 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 600 python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 600 python bench.py --workload c4 > $O/bench_c4.jsonl 2> $O/bench_c4.err
timeout 600 python bench.py --workload c5 > $O/bench_c5.jsonl 2> $O/bench_c5.err
./tools/ubench_c4 > $O/ubench_c4.txt 2>&1
timeout 300 python tools/pot_phases.py --c5 > $O/pot_phases.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e > $O/launches_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_score_pair -s 2 -c 1 \
   -f -o $O/prof_score python tools/profile_run.py 2 > $O/prof_score.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_pot -s 1 -c 1 \
   -f -o $O/prof_pot python tools/profile_run.py 2 > $O/prof_pot.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_pot_scan -s 1 -c 1 \
   -f -o $O/prof_scan5 python tools/profile_c5.py 2 > $O/prof_scan5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k k_pot -s 1 -c 1 \
   -f -o $O/prof_pot5 python tools/profile_c5.py 2 > $O/prof_pot5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stream_rows -s 5 -c 1 \
   -f -o $O/prof_stream python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/prof_stream.log 2>&1
ls -la $O/*.ncu-rep
for f in $O/bench_c*.jsonl; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', 'value %.4g' % d['value'], 'ms %.4f' % d['ms_per_step'], 'frac', d.get('roofline',{}).get('frac'), 'tick', d.get('tick_latency_us'), 'clocks', d.get('clocks'))
"; done
