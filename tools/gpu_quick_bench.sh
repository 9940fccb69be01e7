#!/bin/bash
# quick bench lines (no e2e / cpu baseline) for CONFIGS
OUT=gpurun_out; mkdir -p $OUT
for c in ${CONFIGS:-C2 C3 C4 C5}; do
  timeout -s KILL 300 python bench.py --config $c --steps ${STEPS:-50} --warmup 5 --no-e2e --no-cpu-baseline > $OUT/qb_$c.json 2> $OUT/qb_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.load(open('$OUT/qb_$c.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'],d['roofline']['kernel'],d['roofline']['frac'])" 2>&1 | tail -1)"
done
