#!/bin/bash
# Profiling recipe run on the GPU box (via gpurun) -- see profiles/README.md.
# Usage: scripts/gpu_profile.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
# every launch with its device time (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu \
  --realizations 200 > $OUT/launches_bench.log 2>&1
# full section set on the streaming step kernel (one launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_step -s 3 -c 1 \
  -o $OUT/prof_tile python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --realizations 200 \
  > $OUT/prof_tile.log 2>&1
# resident kernel (N = 64)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:resident -s 3 -c 1 \
  -o $OUT/prof_resident python bench.py --n 64 --steps 20 --warmup 3 --no-e2e --no-cpu \
  --realizations 148 > $OUT/prof_resident.log 2>&1
