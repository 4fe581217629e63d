# K5 SM cycles at C and HY across kept fractions: the slope is the per-block cost, the
# intercept the per-tile (epilogue / tile boundary) cost
OUT=gpurun_out/${1:-k5gamma}; mkdir -p $OUT
for g in 0.1 0.2 0.4 0.8; do K5_GAMMA=$g bash tools/k5_cycles.sh "" C_g$g C >> $OUT/cycles.txt 2>&1; done
for g in 0.05 0.1 0.2; do K5_GAMMA=$g bash tools/k5_cycles.sh "" HY_g$g HY >> $OUT/cycles.txt 2>&1; done
