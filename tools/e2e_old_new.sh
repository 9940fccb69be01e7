#!/bin/bash
# e2e of the current tree vs oldtree/ (a git worktree of an earlier commit) on one box
for t in old new; do
  d=$PWD; [ $t = old ] && d=$PWD/oldtree
  for c in ${CONFIGS:-C2 C4}; do
    (cd $d && timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 9 2>/dev/null) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $t', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'pg', d['e2e_pageable']['ms_per_step'])"
  done
done
