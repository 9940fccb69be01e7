#!/bin/bash
# ONE ncu tool run per call: MODE=launches (launch list of the whole command)
# or MODE=full (ncu --set full of one kernel), after a clean run of the same
# command without ncu.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r01}
C=${CONFIG:-C2}
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > $OUT/plain_$C.log 2>&1 || { echo "plain run failed"; exit 1; }
if [ "${MODE:-full}" = launches ]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${TAG}_$C.csv $CMD > $OUT/ncu_launch_$C.log 2>&1
  echo "launch list $C rc=$?"
else
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
      -k regex:${KERNEL:-k_fused} -s ${SKIP:-3} -c 1 -o $OUT/${TAG}_${C}_${KERNEL:-k_fused} -f $CMD \
      > $OUT/ncu_full_$C.log 2>&1
  echo "full $C rc=$?"
fi
