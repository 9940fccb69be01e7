#!/bin/bash
# One gpurun call: parity suite, full bench lines for every config + the
# reference arm, launch lists and one ncu --set full capture per profiled
# config (each after the same command exited 0 without ncu). -> gpurun_out/
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-r01}
timeout -s KILL 900 python -m pytest tests -q -m gpu -x --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.log)"
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 $OUT/smoke.log)"
CONFIGS=${CONFIGS:-C2 C3 C4 C5 C1} TAG=$TAG bash tools/gpu_bench_all.sh
for spec in ${PROFILE:-C2:k_fused C3:k_fused C4:k_fused C5:k_long_smem}; do
  c=${spec%%:*}; k=${spec##*:}
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 && \
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${TAG}_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k \
      -s 3 -c 1 -o $OUT/${TAG}_${c}_$k -f $CMD > $OUT/ncu_full_$c.log 2>&1; echo "full $c $k rc=$?"
done
