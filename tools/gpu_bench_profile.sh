#!/bin/bash
# One gpurun call: full bench lines for every config, then per profiled config
# the ncu launch list and one `ncu --set full` capture of k_fused (each only
# after the same command exited 0 without ncu). Outputs land in gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r01}
for c in ${CONFIGS:-C2 C3 C4 C5 C1}; do
  timeout -s KILL 900 python bench.py --config $c --steps ${STEPS:-200} --warmup 10 \
     > $OUT/bench_${TAG}_$c.json 2> $OUT/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_${TAG}_reference.json 2>&1; echo "reference rc=$?"
for c in ${PROFILE:-C2 C3 C4}; do
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 && \
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${TAG}_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
  timeout -s KILL 300 $CMD > $OUT/plain2_$c.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:k_fused \
      -s 3 -c 1 -o $OUT/${TAG}_$c -f $CMD > $OUT/ncu_full_$c.log 2>&1; echo "full $c rc=$?"
done
