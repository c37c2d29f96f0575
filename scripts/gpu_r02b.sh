#!/bin/bash
# Round-2 evidence pass (run under gpurun): GPU tests, smoke, both bench arms,
# the launch list of the default bench, the BASELINE sweep, and ncu --set full
# of the headline kernel (band4, configs[2]) and of resident64 (configs[0]).
set -u
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_default.csv python bench.py --no-e2e --no-cpu --no-secondary --no-other \
  --steps 10 --warmup 3 > $OUT/launches_default.log 2>&1
python scripts/launch_shares.py $OUT/launches_default.csv > $OUT/launch_shares.txt 2>&1
timeout 1500 python scripts/sweep.py --quick > $OUT/sweep.jsonl 2> $OUT/sweep.err
full() {  # name, kernel regex, skip, bench args
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
    -o $OUT/$1 python bench.py --no-e2e --no-cpu --no-secondary --no-other ${@:4} > $OUT/$1.log 2>&1
  ncu -i $OUT/$1.ncu-rep --page details --csv > $OUT/${1}_details.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page raw --csv > $OUT/${1}_raw.csv 2>/dev/null
  ncu -i $OUT/$1.ncu-rep --page source --csv --print-source sass > $OUT/${1}_sass.csv 2>/dev/null
  rm -f $OUT/$1.ncu-rep
  python scripts/ncu_summary.py $OUT/${1}_raw.csv > $OUT/${1}_summary.txt 2>&1
}
full band4_n1024_site_fma band4 3 --realizations 250 --steps 4 --warmup 3
full resident64_n64 resident64 3 --config 0 --realizations 148 --steps 200 --warmup 3
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_ref.json | cut -c1-400; head -12 $OUT/launch_shares.txt
