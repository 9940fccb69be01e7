#!/bin/bash
# ncu --set full capture of one kernel of one config: tools/ncu_one.sh C5 k_fused tag
OUT=gpurun_out; mkdir -p $OUT
c=$1; k=$2; tag=${3:-x}
CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/${tag}_${c}_$k -f $CMD > $OUT/ncu_full_${c}_$k.log 2>&1; echo "full $c $k rc=$?"
