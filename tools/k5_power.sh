# board power / SM clock / ms per call of K5 alone and of its isolation builds at HY
OUT=gpurun_out/${1:-k5pow}; mkdir -p $OUT
for lib in "" build/ab/lib_skipsm.so build/ab/lib_skipmma.so build/ab/lib_nomufu.so ""; do
  echo "${lib:-in-tree}: $(DFS_B200_LIB=$lib timeout 300 python tools/k5_power.py HY 6 2>&1 | tail -1)" >> $OUT/summary.txt
done
