#!/bin/bash
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 600 python bench.py --workload c5 --steps 10 --warmup 3 > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err
python tools/pot_phases.py --c5 > gpurun_out/pot_phases.txt 2>&1
tail -5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err
cat gpurun_out/bench.jsonl | head -c 3000
