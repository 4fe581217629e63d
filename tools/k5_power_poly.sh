# K5 alone under the power cap (tools/k5_power.py) per exp2 MUFU/polynomial split
OUT=gpurun_out/${1:-k5powpoly}; mkdir -p $OUT
for wl in HY C; do for pp in 3 0 38 2 516 3; do
  echo "$wl POLY=$pp: $(DFS_ATTN_POLY=$pp timeout 300 python tools/k5_power.py $wl 6 2>&1 | tail -1)" >> $OUT/summary.txt
done; done
