#!/bin/bash
# e2e A/B on one box: pipelined blocks counted (default) vs count-free
for v in default pipecf; do
  if [ $v = pipecf ]; then export SPMMM_PIPE_COUNT_FREE=1; fi
  for c in ${CONFIGS:-C2 C3 C4}; do
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 9 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'pg', d['e2e_pageable']['ms_per_step'])"
  done
done
unset SPMMM_PIPE_COUNT_FREE
python bench.py --impl reference --steps 3 --warmup 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ref', d['value'])"
