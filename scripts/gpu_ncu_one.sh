#!/bin/bash
# ncu --set full of one launch of a kernel under bench.py; args: tag name regex bench-args...
set -u
TAG=$1; NAME=$2; KRE=$3; shift 3
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 3 -c 1 \
  -o $OUT/$NAME python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 "$@" > $OUT/$NAME.log 2>&1
ncu -i $OUT/$NAME.ncu-rep --page details --csv > $OUT/${NAME}_details.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page raw --csv > $OUT/${NAME}_raw.csv 2>/dev/null
ncu -i $OUT/$NAME.ncu-rep --page source --csv --print-source sass > $OUT/${NAME}_sass.csv 2>/dev/null
