mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for f in replicated distributed; do
  ENOVA_BENCH_COMM=1 timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline --fit $f > gpurun_out/c5_$f.jsonl 2> gpurun_out/c5_$f.err
  python -c "import json; d=json.loads(open('gpurun_out/c5_$f.jsonl').read().strip().splitlines()[-1]); print('c5 comm1 $f', d['ms_per_step'], d['threshold']['z_q'])" || tail -3 gpurun_out/c5_$f.err
  ENOVA_BENCH_COMM=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-traffic --no-e2e --fit $f > gpurun_out/c2_$f.jsonl 2> gpurun_out/c2_$f.err
  python -c "import json; d=json.loads(open('gpurun_out/c2_$f.jsonl').read().strip().splitlines()[-1]); print('c2 comm1 $f', d['ms_per_step'], d['threshold']['z_q'], d['step_overlap']['pot_ctas'])" || tail -3 gpurun_out/c2_$f.err
done
timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5_single.jsonl 2> gpurun_out/c5_single.err
python -c "import json; d=json.loads(open('gpurun_out/c5_single.jsonl').readline()); print('c5 single', d['ms_per_step'], d['threshold']['z_q'], d['phases']['select_compact_us'], d['phases']['fit_us'])"
