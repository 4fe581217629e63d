# K5 timing bounds from deliberately wrong experiment builds (SM cycles at HY and C):
#   bash tools/k5_variant.sh nosum  paper_2605_23445_b200/csrc/attn_sm100.cu -DDFS_ATTN_NOSUM_EXPERIMENT
#   bash tools/k5_variant.sh nomufu paper_2605_23445_b200/csrc/attn_sm100.cu -DDFS_ATTN_NOMUFU_EXPERIMENT
# (the macros were applied to a scratch copy of the source for profiles/r2/bound_*_cycles.txt;
# they are not kept in the production source)
OUT=gpurun_out/${OUT:-bound}; mkdir -p $OUT
for lib in ${LIBS:-nosum nomufu}; do
  for wl in HY C; do bash tools/k5_cycles.sh "" base $wl >> $OUT/cycles.txt 2>&1; bash tools/k5_cycles.sh build/ab/lib_$lib.so $lib $wl >> $OUT/cycles.txt 2>&1; done
done
