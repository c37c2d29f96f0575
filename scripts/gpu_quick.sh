#!/bin/bash
# Quick GPU iteration: parity tests + bench exact/fma at N=256/512/1024.
set -u
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -25 $OUT/pytest_gpu.log
IFS=';' read -ra CASES <<< "${BENCH_CASES:-;--fma;--backend rk4;--n 512;--n 1024 --realizations 250;--n 512 --fma;--n 1024 --realizations 250 --fma}"
for args in "${CASES[@]}"; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 3 $args 2>>$OUT/bench.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); r=d['roofline']
    print('$args'.ljust(34), d['config']['n_sites'], '%.4g r-steps/s'%d['value'], 'frac %.3f'%r['frac'], r['kernel'], 'share %.3f'%r['kernel_share_of_step'], 'clk', d['clocks']['sm_mhz'])
" | tee -a $OUT/bench.txt
done
