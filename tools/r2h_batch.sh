#!/bin/bash
# Round-2 final measurement batch on one B200 (run from the repo root; R2_OUT names the subdir):
# the r2c batch (GPU tests, smoke, bench lines, trajectories, reference arm, ncu step capture,
# sanitizers) + the W7 sparsity sweep, a CUPTI step timeline and the PCIe probe.
R2_OUT=${R2_OUT:-r2h}
OUT=gpurun_out/$R2_OUT
R2_OUT=$R2_OUT bash tools/r2c_batch.sh
OUT=$OUT/w7 bash tools/w7_sweep.sh
timeout 300 python tools/step_timeline.py HY > $OUT/timeline_HY.txt 2>&1
timeout 300 python tools/pcie_probe.py > $OUT/pcie.txt 2>&1
echo batch-done >> $OUT/summary.txt
