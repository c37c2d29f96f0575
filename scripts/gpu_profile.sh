#!/bin/bash
# Profiling recipe run on the GPU box (via gpurun) -- summaries go to profiles/.
# Usage: scripts/gpu_profile.sh <tag> [kernel-regex]
set -u
TAG=${1:-r01}
KRE=${2:-band_step}
OUT=gpurun_out/$TAG
mkdir -p $OUT
# every launch with its device time (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu \
  --realizations 200 > $OUT/launches_bench.log 2>&1
# full section set on the streaming step kernel (one launch, bench-sized grid)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
  -o $OUT/prof_step python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --realizations 1000 \
  > $OUT/prof_step.log 2>&1
