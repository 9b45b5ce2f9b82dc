mkdir -p gpurun_out
for f in "" "-DENOVA_STATS_STAGES=10 -DENOVA_STATS_CHUNK=16384" "-DENOVA_STATS_STAGES=3 -DENOVA_STATS_CHUNK=65536" "-DENOVA_STATS_STAGES=12 -DENOVA_STATS_CHUNK=8192"; do
  ENOVA_NVCC_FLAGS="$f" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  ENOVA_NVCC_FLAGS="$f" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_series_stats python tools/profile_run.py 3 2>/dev/null | grep gpu__time_duration | awk -F'"' -v f="$f" '{print f, $(NF-1)}' | tail -2
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
