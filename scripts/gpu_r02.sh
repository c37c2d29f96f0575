#!/bin/bash
# Round-2 GPU pass (run under gpurun): tests, smoke, bench (both arms), the
# launch list of the default bench, and ncu --set full of the headline kernel.
# Usage: bash scripts/gpu_r02.sh <tag> [pytest -k expr]
set -u
TAG=${1:-r02a}
K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
else
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_default.csv python bench.py --no-e2e --no-cpu --no-secondary --no-other \
  --steps 10 --warmup 3 > $OUT/launches_default.log 2>&1
full() {  # name, kernel regex, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 \
    -o $OUT/$1 python bench.py --no-e2e --no-cpu --no-secondary --no-other --steps 4 --warmup 3 ${@:3} > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/${1}_details.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/${1}_raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/${1}_sass.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
}
full band4_n1024_site_fma band4 --realizations 250
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_ref.json; tail -5 $OUT/bench.err
