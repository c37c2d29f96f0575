#!/bin/bash
# A/B of two builds of libctqw.so on the kernel-only bench lines:
#   ab_bench.sh <libA> <libB> [rounds] [extra bench args...]
A=$1; B=$2; N=${3:-3}; shift 3
for i in $(seq $N); do
  for L in $A $B; do
    v=$(CTQW_LIB=$L timeout 300 python bench.py --no-e2e --no-cpu --no-secondary --no-other --steps 20 --warmup 5 "$@" 2>/dev/null \
        | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['roofline']['frac'],4))")
    echo "$(basename $L) $v"
  done
done
