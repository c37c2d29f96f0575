#!/bin/bash
# band4 size/noise matrix: device-timed lines for N = 256/512/1024 x tunnelling/both.
set -u
TAG=${1:-sizes}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for n in 256 512 1024; do
  R=$(( 1000 * 256 * 256 / (n * n) )); [ $n = 1024 ] && R=1250; [ $n = 512 ] && R=1000
  for t in tunneling both; do
    timeout 300 python bench.py --n $n --realizations $R --target $t --steps 20 --warmup 3 --no-e2e --no-cpu --no-secondary --no-other ${EXTRA:-} > $OUT/n${n}_$t.json 2>> $OUT/bench.err
  done
done
for f in $OUT/n*.json; do python -c "
import json; d=json.load(open('$f'))
print('$f', round(d['value']), round(d['roofline']['frac'],3))"; done
