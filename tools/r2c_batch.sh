#!/bin/bash
# Round-2 measurement batch on one B200 after the K5 row-split rework (run from the repo root):
# GPU tests + smoke, bench lines (HY with the CPU baseline, C, W4, W7, W4/W7 trajectories),
# the reference arm, launch list + ncu --set full of one HY update step, sanitizers.
OUT=gpurun_out/${R2_OUT:-r2c}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_HY.json 2> $OUT/bench_HY.err
for wl in C W4 W7; do timeout 600 python bench.py --workload $wl --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_$wl.json 2>&1; done
for wl in W4 W7; do timeout 900 python bench.py --workload $wl --trajectory --steps 50 --warmup 3 --no-cpu-baseline > $OUT/traj_$wl.json 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python tools/profile_step.py HY > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:'attn_sm100|score_sm100|permute_kernel|topk|absmax|split_kernel|lut_ptr' -s 12 -c 12 \
  -o $OUT/prof python tools/profile_step.py HY > $OUT/ncu.log 2>&1
# compute-sanitizer (tools/sanitize.sh) is closed on the GPU pool since r2m; run it separately where allowed
echo done >> $OUT/summary.txt
