#!/bin/bash
# Same-box A/B of compile-time k_pot variants on c5 (run under gpurun):
#   bash tools/c5_ab.sh "" "-DENOVA_X" ...
mkdir -p gpurun_out
for rep in 1 2; do
  for f in "$@"; do
    ENOVA_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo "build failed: $f"
    ENOVA_NVCC_FLAGS="$f" timeout 300 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c5ab.jsonl 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/c5ab.jsonl').read().strip().splitlines()[-1]); p=d['phases']; print('${f:-base}', 'ms', round(d['ms_per_step'],4), 'select_us', round(p['select_compact_us'],1), 'fit_us', round(p['fit_us'],1), 'z_q', d['threshold']['z_q'])" || echo "$f: failed"
  done
done | tee gpurun_out/c5_ab.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
