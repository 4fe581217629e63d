# K4 change check: top-K / mask tests and parity pins, K4 duration at HY under ncu
OUT=gpurun_out/${1:-k4}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -k "topk or tie or mask or parity or pins or lut" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk -c 4 --csv python tools/profile_step.py HY 2>/dev/null | grep gpu__time | awk -F'","' '{gsub(/"/,"",$NF); print "topk", $NF}' >> $OUT/summary.txt
