#!/bin/bash
# Threshold-path GPU check (run under gpurun): build, all GPU tests, c5 + c2 bench lines, k_pot phase stamps.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
timeout 300 python tools/pot_phases.py > gpurun_out/pot_phases.txt 2>&1
tail -12 gpurun_out/pot_phases.txt
python - <<'PY'
import json
for f in ("gpurun_out/bench_c5.jsonl", "gpurun_out/bench_c2.jsonl"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "failed", e); continue
    print(f, "value %.4g ms %.4f" % (d["value"], d["ms_per_step"]), "phases", d.get("phases"), "stage", d.get("stage_ms"), "thr", d.get("threshold"))
PY
