# K2 A/B: tools/permute_bench.py at C, W4 and HY for the in-tree library and each variant
OUT=gpurun_out/${1:-k2ab}; mkdir -p $OUT
for lib in "" $2; do for wl in C W4 HY; do
  echo "== ${lib:-in-tree} $wl" >> $OUT/summary.txt
  DFS_B200_LIB=$lib timeout 300 python tools/permute_bench.py $wl 20 >> $OUT/summary.txt 2>&1
done; done
