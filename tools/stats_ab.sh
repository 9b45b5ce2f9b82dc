#!/bin/bash
# Same-box A/B of compile-time K1 variants by ncu kernel duration (run under gpurun):
#   bash tools/stats_ab.sh "" "-DENOVA_AB_X" ...
mkdir -p gpurun_out
for f in "$@"; do
  ENOVA_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  ENOVA_NVCC_FLAGS="$f" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_series_stats python tools/profile_run.py 3 2>/dev/null | grep gpu__time_duration | awk -F'"' -v f="${f:-base}" '{print f, $(NF-1)}' | tail -2
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
