#!/bin/bash
# ncu evidence (run under gpurun): launch list of the default bench and
# --set full of each kernel; only CSV exports are kept (reports are large).
set -u
TAG=${1:-ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
[ -z "${NCU_SKIP_LAUNCHES:-}" ] && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_default.csv python bench.py --no-e2e --no-cpu --steps 10 --warmup 3 > $OUT/launches_default.log 2>&1
IFS=';' read -ra SPECS <<< "${NCU_SPECS:-band4_n256_fma|band4|;band4_n256_exact|band4|--exact;band4_n1024_fma|band4|--n 1024 --realizations 250;band4_n256_rk4|band4|--backend rk4;plane3_fma|plane3|--m 3 --n 128 --realizations 64 --dt 0.015;resident_n64|resident|--n 64 --realizations 1000}"
for spec in "${SPECS[@]}"; do
  IFS='|' read -r name kre args <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s 2 -c 1 \
    -o $OUT/$name python bench.py --no-e2e --no-cpu --steps 4 --warmup 3 $args > $OUT/$name.log 2>&1
  ncu -i $OUT/$name.ncu-rep --page details --csv > $OUT/${name}_details.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/${name}_raw.csv 2>/dev/null
  rm -f $OUT/$name.ncu-rep
done
ls -la $OUT
