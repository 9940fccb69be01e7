#!/bin/bash
# pipelined host path: parity tests, then e2e bench lines
OUT=gpurun_out; mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 600 -p no:cacheprovider -k "pipelined or drop_in or golden" > $OUT/pytest_pipe.log 2>&1
echo pytest_rc=$?; tail -3 $OUT/pytest_pipe.log
for c in ${CONFIGS:-C2 C3 C4 C5}; do
  timeout -s KILL 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps ${E2E:-5} > $OUT/e2e_$c.json 2> $OUT/e2e_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.load(open('$OUT/e2e_$c.json'));print(d['value'],d['ms_per_step'],d['e2e'])" 2>&1 | tail -1)"
done
