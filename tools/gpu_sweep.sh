#!/bin/bash
# C2 size sweep (grid side 32..2048, BASELINE configs[1]): one bench line per
# size (device step, e2e, roofline) -> gpurun_out/sweep_<tag>.jsonl
set -u
OUT=gpurun_out; mkdir -p $OUT
TAG=${TAG:-r01}
: > $OUT/sweep_$TAG.jsonl
for g in 32 64 128 256 512 1024 2048; do
  timeout -s KILL 300 python bench.py --config C2 --grid $g --steps ${STEPS:-100} --warmup 5 \
      --no-cpu-baseline --e2e-steps 5 2> $OUT/sweep_$g.err | tail -1 >> $OUT/sweep_$TAG.jsonl
  echo "grid $g rc=$?"
done
