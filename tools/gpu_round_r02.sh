#!/bin/bash
# One gpurun call: bench lines for every config + the reference arm + the
# default line, the C2 sweep, launch lists and ncu --set full captures of
# the dominant kernels (each only after its command exited 0 without ncu).
set -u
OUT=gpurun_out; mkdir -p $OUT/profiles
TAG=${TAG:-r02}
# the per-kernel DRAM bytes merge into the committed file's other entries
cp profiles/${TAG}_traffic.json $OUT/profiles/ 2>/dev/null
for c in ${CONFIGS:-C2 C3 C4 C5 C1}; do
  timeout -s KILL 900 python bench.py --config $c --steps ${STEPS:-200} --warmup 10 \
     > $OUT/bench_${TAG}_$c.json 2> $OUT/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout -s KILL 900 python bench.py --impl reference --steps 5 --warmup 3 \
   > $OUT/bench_${TAG}_reference.json 2> $OUT/bench_${TAG}_reference.err; echo "reference rc=$?"
timeout -s KILL 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err
echo "default rc=$?"
if [ -z "${NOSWEEP:-}" ]; then TAG=$TAG STEPS=200 bash tools/gpu_sweep.sh; fi
for spec in ${PROFILE:-C2:k_fused C2:k_prep C3:k_fused C4:k_fused C5:k_esc_block C5:k_esc_dom C5:k_esc_warp C5:k_esc_plan C5:k_fused C5:k_copy_long C5:k_count}; do
  c=${spec%%:*}; k=${spec##*:}
  CMD="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  if [ ! -f $OUT/launches_${TAG}_$c.csv ]; then
    timeout -s KILL 300 $CMD > $OUT/plain_$c.log 2>&1 && \
    timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches_${TAG}_$c.csv $CMD > $OUT/ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
    SPMMM_PROFILE_DIR=$OUT/profiles python tools/profile_commit.py launches $OUT/launches_${TAG}_$c.csv $c $TAG > /dev/null
  fi
  timeout -s KILL 300 $CMD > $OUT/plain2_$c.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:$k \
      -s 3 -c 1 -o $OUT/${TAG}_${c}_$k -f $CMD > $OUT/ncu_full_${c}_$k.log 2>&1; echo "full $c $k rc=$?"
  # the summaries are made on the box (the reports together pass gpurun_out's 64 MiB)
  SPMMM_PROFILE_DIR=$OUT/profiles python tools/profile_commit.py full $OUT/${TAG}_${c}_$k.ncu-rep $c $k $TAG \
      && rm -f $OUT/${TAG}_${c}_$k.ncu-rep
done
# the N > 1 path: one rank over NCCL (torchrun), and two ranks sharing the GPU over gloo
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 \
   --master-port=29561 bench.py --distributed --config C2 --steps 20 --warmup 5 \
   > $OUT/bench_${TAG}_dist1_nccl.json 2> $OUT/bench_${TAG}_dist1_nccl.err; echo "dist1 nccl rc=$?"
timeout -s KILL 900 python bench.py --gpus 2 --backend gloo --config C2 --steps 20 --warmup 5 \
   > $OUT/bench_${TAG}_dist2_gloo.json 2> $OUT/bench_${TAG}_dist2_gloo.err; echo "dist2 gloo rc=$?"
