#!/bin/bash
# Full GPU evidence pass (run under gpurun): tests, smoke, bench (both arms),
# sweep, ncu launch list of the default bench, ncu --set full of each kernel.
set -u
TAG=${1:-r01c}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 1500 python scripts/sweep.py --quick > $OUT/sweep.jsonl 2> $OUT/sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_default.csv python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 > $OUT/launches_default.log 2>&1
for spec in "band4_n256_fma|band4|" "band4_n256_exact|band4|--exact" "band4_n1024_fma|band4|--n 1024 --realizations 250" \
            "band4_n256_rk4|band4|--backend rk4" "plane3_fma|plane3|--m 3 --n 128 --realizations 64 --dt 0.015" \
            "resident_n64|resident|--n 64 --realizations 1000"; do
  IFS='|' read -r name kre args <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o $OUT/$name python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 $args > $OUT/$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv --print-source sass > $OUT/${name}_sass.csv 2>/dev/null
  rm -f $OUT/$name.ncu-rep  # reports exceed the copy-back limit; the CSV exports stay
done
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/smoke.log; cat $OUT/bench.json $OUT/bench_ref.json $OUT/sweep.jsonl
