#!/bin/bash
# One GPU call: parity tests, smoke, bench (exact + fma), quick sweep.
# Usage (under gpurun): bash scripts/gpu_check.sh <tag>
set -u
TAG=${1:-chk}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --fma --no-cpu --no-e2e > $OUT/bench_fma.json 2> $OUT/bench_fma.err
timeout 900 python scripts/sweep.py --quick > $OUT/sweep.jsonl 2> $OUT/sweep.err
tail -3 $OUT/pytest_gpu.log; cat $OUT/smoke.log | tail -3; cat $OUT/bench.json $OUT/bench_fma.json $OUT/sweep.jsonl
