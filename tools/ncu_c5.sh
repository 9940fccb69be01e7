OUT=gpurun_out; mkdir -p $OUT
CMD="python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout -s KILL 300 $CMD > $OUT/plain_C5.log 2>&1 || exit 1
for k in k_fused k_copy_long k_esc_warp k_esc_plan k_count; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o $OUT/r02b_C5_$k -f $CMD > $OUT/ncu_full_C5_$k.log 2>&1; echo "full C5 $k rc=$?"
done
