#!/bin/bash
# Same-box A/B of compile-time variants on the c4 streaming tick (run under gpurun):
#   bash tools/c4_ab.sh "" "-DENOVA_AB_X" ...   (each argument = ENOVA_NVCC_FLAGS; "" = base)
mkdir -p gpurun_out
for rep in 1 2; do
  for f in "$@"; do
    ENOVA_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo "build failed: $f"
    ENOVA_NVCC_FLAGS="$f" timeout 300 python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c4ab.jsonl 2>/dev/null
    python -c "import json,sys; d=json.loads(open('gpurun_out/c4ab.jsonl').read().strip().splitlines()[-1]); print('${f:-base}', 'tick p50 us', round(d['tick_latency_us']['p50'],2), 'p99', round(d['tick_latency_us']['p99'],2))" || echo "$f: failed"
  done
done | tee gpurun_out/c4_ab.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
