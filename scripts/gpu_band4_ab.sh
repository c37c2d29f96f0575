#!/bin/bash
# band4 A/B pass: band4 parity tests + device-timed bench lines for configs[1..3].
set -u
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x -k "band4 or bench_parity or streaming or repeat" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for c in 2 3 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu --no-secondary > $OUT/c$c.json 2>> $OUT/bench.err
done
timeout 300 python bench.py --config 2 --backend rk4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary --no-other > $OUT/c2rk4.json 2>> $OUT/bench.err
tail -3 $OUT/pytest_gpu.log
for f in $OUT/c*.json; do python -c "
import json; d=json.load(open('$f')); o=d.get('other_arithmetic') or {}
print('$f', round(d['value']), round(d['roofline']['frac'],3), 'exact', round(o.get('value',0)))"; done
