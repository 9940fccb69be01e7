#!/bin/bash
# ncu --set full captures of several kernels of one config: tools/ncu_multi.sh C5 tag k1 k2 ...
OUT=gpurun_out; mkdir -p $OUT
c=$1; tag=$2; shift 2
CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 || exit 1
for k in "$@"; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/${tag}_${c}_$k -f $CMD > $OUT/ncu_full_${c}_$k.log 2>&1; echo "full $c $k rc=$?"
done
