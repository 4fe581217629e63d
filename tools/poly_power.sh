# HY bench lines (CUDA-event ms/call, SM clock, board power) per exp2 MUFU/polynomial split:
# under the power cap wall time is cycles / clock(power), so the split is judged here too,
# not only by SM cycles (tools/poly_sweep.sh)
OUT=gpurun_out/${1:-polypow}; mkdir -p $OUT
for pp in 3 0 38 2 3; do
  DFS_ATTN_POLY=$pp timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $OUT/HY_$pp.json 2>&1
  python -c "import json,sys; d=json.loads(open('$OUT/HY_$pp.json').read().strip().splitlines()[-1]); print('$pp', round(d['ms_per_step'],3), d['clocks'])" >> $OUT/summary.txt
done
