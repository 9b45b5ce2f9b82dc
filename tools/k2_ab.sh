#!/bin/bash
# Same-box A/B of compile-time K2 variants (run under gpurun):
#   bash tools/k2_ab.sh "" "-DENOVA_AB_X" ...   (each argument = ENOVA_NVCC_FLAGS; "" = base)
# every timing run is bounded (a variant that deadlocks prints "timeout").
mkdir -p gpurun_out
for rep in 1 2; do
  for f in "$@"; do
    ENOVA_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo "build failed: $f"
    ENOVA_NVCC_FLAGS="$f" timeout 90 python tools/k2_time.py 2>&1 | tail -1 || echo "$f: timeout"
  done
done | tee gpurun_out/k2_ab.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
