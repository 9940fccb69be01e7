#!/bin/bash
# Full bench lines for every config and the reference arm (no profilers).
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${TAG:-r01}
for c in ${CONFIGS:-C2 C3 C4 C5 C1}; do
  timeout -s KILL 900 python bench.py --config $c --steps ${STEPS:-200} --warmup 10 \
     > $OUT/bench_${TAG}_$c.json 2> $OUT/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 3 \
   > $OUT/bench_${TAG}_reference.json 2> $OUT/bench_${TAG}_reference.err; echo "reference rc=$?"
timeout -s KILL 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err
echo "default rc=$?"
