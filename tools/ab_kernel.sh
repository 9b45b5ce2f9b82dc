#!/bin/bash
# Same-box A/B of one kernel source (run under gpurun; boxes differ by a few %):
#   bash tools/ab_kernel.sh <tracked source> <alternative copy> [reps]
# builds and benches (c2, no cpu baseline / e2e) the current source (A) and the
# alternative (B) alternately; restores A.  Results: gpurun_out/ab_{A,B}_<i>.json
F=$1; ALT=$2; N=${3:-2}
cp "$F" /tmp/ab_a.cu
for i in $(seq 1 "$N"); do
  cp /tmp/ab_a.cu "$F"; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_A_$i.json 2>/dev/null
  cp "$ALT" "$F"; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_B_$i.json 2>/dev/null
done
cp /tmp/ab_a.cu "$F"; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
