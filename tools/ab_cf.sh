#!/bin/bash
# A/B on one box: count-free path vs counted path (SPMMM_NO_COUNT_FREE=1)
for c in ${CONFIGS:-C2 C3}; do
  for v in cf counted; do
    if [ $v = counted ]; then export SPMMM_NO_COUNT_FREE=1; else unset SPMMM_NO_COUNT_FREE; fi
    timeout -s KILL 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', d['ms_per_step'], d['kernel_ms'])"
  done
done
