#!/bin/bash
# plane3 (configs[4]) measurement: bench line + ncu --set full of one launch.
set -u
TAG=${1:-p3}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python bench.py --config 4 --steps 6 --warmup 3 --no-e2e --no-cpu --no-secondary > $OUT/c4.json 2> $OUT/c4.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plane3 -s 3 -c 1 -o $OUT/plane3 \
  python bench.py --config 4 --realizations 112 --steps 4 --warmup 3 --no-e2e --no-cpu --no-secondary --no-other > $OUT/ncu.log 2>&1
ncu -i $OUT/plane3.ncu-rep --page raw --csv > $OUT/plane3_raw.csv 2>/dev/null
ncu -i $OUT/plane3.ncu-rep --page details --csv > $OUT/plane3_details.csv 2>/dev/null
ncu -i $OUT/plane3.ncu-rep --page source --csv --print-source sass > $OUT/plane3_sass.csv 2>/dev/null
rm -f $OUT/plane3.ncu-rep
python -c "
import json; d=json.load(open('$OUT/c4.json')); o=d.get('other_arithmetic') or {}
print('c4', round(d['value']), round(d['roofline']['frac'],3), 'exact', round(o.get('value',0)), d['roofline']['kernel_ms_avg'])"
python scripts/ncu_summary.py $OUT/plane3_raw.csv
