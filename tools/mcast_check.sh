# dense-step K/V multicast (DFS_ATTN_MCAST, default on) check: GPU tests, then the W7 50-step
# trajectory (12 dense steps) and a dense-only K5 power-capped loop with the in-tree library and
# the multicast-off variant (build/ab/lib_nomcast.so) on the same box
OUT=gpurun_out/${1:-mcast}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "gpu tests rc=$?" >> $OUT/summary.txt
for lib in "" build/ab/lib_nomcast.so "" build/ab/lib_nomcast.so; do
  DFS_B200_LIB=$lib timeout 900 python bench.py --workload W7 --trajectory --steps 50 --warmup 3 --no-cpu-baseline > $OUT/traj.json 2>&1
  python -c "import json; d=json.loads(open('$OUT/traj.json').read().strip().splitlines()[-1]); print('${lib:-in-tree}', round(d['ms_per_step'],3), d['per_step_kind_ms'], d['clocks'])" >> $OUT/summary.txt
done
