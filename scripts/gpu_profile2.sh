#!/bin/bash
# ncu captures of the streaming kernels at the BASELINE sizes (run under gpurun).
# Usage: bash scripts/gpu_profile2.sh <tag>
set -u
TAG=${1:-p2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
B="python bench.py --no-e2e --no-cpu"
# launch list of the default bench workload (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_default.csv $B --steps 10 --warmup 3 > $OUT/launches_default.log 2>&1
full() {  # name, kernel regex, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
    -o $OUT/$1 $B --steps 4 --warmup 3 ${@:3} > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/$1_details.csv 2>/dev/null
}
full band2_fma_n256 band2 --fma --realizations 1000
full band_n1024 band --n 1024 --realizations 300
full band2_n512 band2 --n 512 --realizations 500
full generic_m3 taylor_order --m 3 --n 128 --realizations 64 --dt 0.015
ls -la $OUT
