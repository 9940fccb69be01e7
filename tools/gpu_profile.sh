#!/bin/bash
# ncu --set full capture of k_fused for the given configs (after a clean plain run).
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-p}
for c in ${PROFILE:-C2 C4}; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_fused} \
      -s ${SKIP:-3} -c 1 -o $OUT/${TAG}_$c -f $CMD > $OUT/ncu_${TAG}_$c.log 2>&1; echo "full $c rc=$?"
done
