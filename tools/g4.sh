mkdir -p gpurun_out/g4
for lib in build/ab/lib_qt_SKIP_SOFTMAX.so build/ab/lib_noqt_SKIP_SOFTMAX.so build/ab/lib_qt_SKIP_MMA.so build/ab/lib_noqt_SKIP_MMA.so; do
  bash tools/k5_cycles.sh "$lib" "$lib" HY >> gpurun_out/g4/cycles.txt 2>&1
done
nvidia-smi --query-gpu=clocks.sm --format=csv >> gpurun_out/g4/cycles.txt
