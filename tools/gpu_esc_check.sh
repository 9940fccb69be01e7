OUT=gpurun_out; mkdir -p $OUT
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider -k "esc or C5 or clustered or random_vs or golden" > $OUT/pytest_esc.log 2>&1
echo pytest_rc=$?; tail -5 $OUT/pytest_esc.log
for c in C5; do
  timeout -s KILL 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_$c.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'])" 2>&1 | tail -1)"
  SPMMM_NO_ESC=1 timeout -s KILL 300 python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_${c}_old.json 2> $OUT/bench_$c.err
  echo "$c old rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_${c}_old.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'])" 2>&1 | tail -1)"
done
SPMMM_SERIAL_ESC=1 timeout -s KILL 300 python bench.py --config C5 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline > $OUT/bench_C5_serial.json 2> $OUT/bench_C5.err
echo "C5 serial rc=$? $(python -c "import json;d=json.load(open('$OUT/bench_C5_serial.json'));print(d['value'],d['ms_per_step'],d['kernel_ms'])" 2>&1 | tail -1)"
