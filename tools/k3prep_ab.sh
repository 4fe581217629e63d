# K3 operand prep (absmax + split kernels) durations under ncu for the in-tree and variant libraries
OUT=gpurun_out/${1:-k3prep}; mkdir -p $OUT
for lib in "" $2; do
  DFS_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'absmax|split_kernel' -c 6 --csv python tools/score_bench.py HY 2 2>/dev/null | grep gpu__time | awk -F'","' -v l=${lib:-in-tree} '{gsub(/"/,"",$NF); print l, $5, $NF}' >> $OUT/summary.txt
done
