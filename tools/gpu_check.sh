#!/bin/bash
# One gpurun call: the GPU test files given in $TESTS (default: all -m gpu),
# then the default bench line, then the functional 2-rank bench line.
OUT=gpurun_out; mkdir -p $OUT
timeout -s KILL 1500 python -m pytest ${TESTS:-tests} -q -m gpu -x --timeout 900 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu.log)"
if [ -z "${NOBENCH:-}" ]; then
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
timeout -s KILL 900 python bench.py --gpus 2 --backend gloo --config ${DCONF:-C3} --steps 5 --warmup 3 --e2e-steps 3 > $OUT/bench_g2.json 2> $OUT/bench_g2.err; echo "bench g2 rc=$?"
fi
