#!/bin/bash
# parity suite + quick per-config bench lines (no e2e / cpu baseline)
OUT=gpurun_out; mkdir -p $OUT
if [ -z "${NOTEST:-}" ]; then
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo pytest_rc=$?; tail -3 $OUT/pytest_gpu.log
fi
for c in ${CONFIGS:-C2 C3 C4 C5}; do
  timeout -s KILL 300 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_$c.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'],d['roofline']['frac'])" 2>&1 | tail -1)"
done
