# power-capped K5 isolation: MMA+TMA side, MMA alone (no K/V loads), TMA alone (no MMAs), softmax alone
OUT=gpurun_out/${1:-k5powiso}; mkdir -p $OUT
for lib in build/ab/lib_skipsm.so build/ab/lib_mmaonly.so build/ab/lib_tmaonly.so build/ab/lib_skipmma.so; do
  echo "$lib: $(DFS_B200_LIB=$lib timeout 300 python tools/k5_power.py HY 6 2>&1 | tail -1)" >> $OUT/summary.txt
  bash tools/k5_cycles.sh $lib $(basename $lib .so) HY | grep cycles >> $OUT/summary.txt
done
