#!/bin/bash
# Quick GPU check (run under gpurun): build, all GPU tests (stop at first failure), default bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
for l in open("gpurun_out/bench.jsonl"):
    d = json.loads(l)
    r = d.get("roofline", {})
    print("value", d["value"], "ms", d["ms_per_step"], "frac", r.get("frac"), "launch_ms", r.get("launch_ms_avg"), "stage", d.get("stage_ms"), "e2e", d.get("e2e", {}).get("value"))
PY
