OUT=gpurun_out/g41; mkdir -p $OUT
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_sync_$i.json 2>&1
DFS_EXPERIMENT_SKIP_FLAG_CHECK=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_nosync_$i.json 2>&1
done
DFS_EXPERIMENT_SKIP_FLAG_CHECK=1 python tools/step_timeline.py HY > $OUT/timeline_nosync.txt 2>&1
