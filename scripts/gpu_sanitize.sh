#!/bin/bash
# compute-sanitizer over the round-2 kernels (resident64 with the fused collection,
# packed_gram, the batched point reductions) and the earlier families.
set -u
OUT=gpurun_out/${1:-san}
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py ${WHICH:-resident64 gram points band4} \
    > $OUT/$tool.log 2>&1; echo "rc=$?" >> $OUT/$tool.log
  tail -3 $OUT/$tool.log
done
