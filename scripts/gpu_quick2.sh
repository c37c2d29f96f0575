#!/bin/bash
# Quick GPU check: pytest -m gpu (optionally -k), plus the configs[3] post-rate sweep.
set -u
TAG=${1:-q}
K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
else
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
for pr in 1 10 100; do
  timeout 300 python bench.py --config 3 --post-rate $pr --steps 100 --warmup 3 --no-e2e --no-cpu --no-other > $OUT/c3_post$pr.json 2>> $OUT/bench.err
done
tail -5 $OUT/pytest_gpu.log
for f in $OUT/c3_post*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['roofline']['kernel_share_of_step'])"; done
