#!/bin/bash
# Round-2 measurement batch on one B200 (run from the repo root under gpurun):
#   compute-sanitizer memcheck / racecheck / synccheck on small launches of every kernel,
#   bench lines (HY headline, C, W4, the W7 gamma sweep, W4/W7 trajectories), K5 SM cycles.
# Everything lands in gpurun_out/r2/.
OUT=gpurun_out/r2; mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "sanitize $tool rc=$?" >> $OUT/summary.txt
done
python bench.py --steps 20 --warmup 5 > $OUT/bench_HY.json 2> $OUT/bench_HY.err
for wl in C W4; do python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$wl.json 2>&1; done
for g in 0.30 0.25 0.20 0.15 0.10 0.05; do
  python bench.py --workload W7 --gamma $g --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_W7_g$g.json 2>&1
done
for wl in W4 W7; do python bench.py --workload $wl --trajectory --steps 50 --warmup 3 --no-cpu-baseline > $OUT/traj_$wl.json 2>&1; done
for wl in HY C; do bash tools/k5_cycles.sh "" r2 $wl >> $OUT/k5_cycles.txt 2>&1; done
echo done >> $OUT/summary.txt
