#!/bin/bash
# A/B of two builds of libctqw.so on sweep cases:  ab_sweep.sh <libA> <libB> <rounds> <--only pattern>
A=$1; B=$2; N=$3; shift 3
for i in $(seq $N); do
  for L in $A $B; do
    CTQW_LIB=$L timeout 300 python scripts/sweep.py --quick "$@" 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l)
    if not d['exact']: print('$(basename $L)', d['case'], d['post_rate'], round(d['r_steps_per_s']))"
  done
done
