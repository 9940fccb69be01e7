#!/bin/bash
# ncu --set full of one kernel of one config (after a clean run of the same
# command). CONFIG, KERNEL, TAG, SKIP via env. -> gpurun_out/
set -u
OUT=gpurun_out; mkdir -p $OUT
C=${CONFIG:-C5}; K=${KERNEL:-k_esc_block}; TAG=${TAG:-dev}
CMD="python bench.py --config $C --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > $OUT/plain_$C.log 2>&1 || { echo "plain run failed"; tail -5 $OUT/plain_$C.log; exit 1; }
for k in $K; do
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k \
    -s ${SKIP:-3} -c 1 -o $OUT/${TAG}_${C}_$k -f $CMD > $OUT/ncu_full_${C}_$k.log 2>&1
echo "full $C $k rc=$?"
done
