#!/bin/bash
# step and kernel times of each variants/<name>/libspmmm.so on one box
for c in ${CONFIGS:-C2 C3}; do
  for v in ${VARIANTS:-$(ls variants)}; do
    SPMMM_LIB_PATH=$PWD/variants/$v/libspmmm.so timeout -s KILL 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', d['ms_per_step'], ' '.join(f'{k[2:]}={v:.3f}' for k,v in d['kernel_ms'].items() if v > 0.02))"
  done
done
