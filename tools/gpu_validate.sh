#!/bin/bash
# GPU validation pass (run under gpurun): build, GPU parity tests, smoke, bench
# lines.  Usage: tools/gpu_validate.sh [pytest -k expr]
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
K=${1:-}
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
else
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err
cat gpurun_out/bench.jsonl | head -c 3000
