mkdir -p gpurun_out/g11
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py tests/test_gpu_parity.py -x -q > gpurun_out/g11/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g11/summary.txt
for lib in "" build/ab/lib_rs2_SKIP_MMA.so; do bash tools/k5_cycles.sh "$lib" "${lib:-rs2}" HY >> gpurun_out/g11/cycles.txt 2>&1; done
bash tools/k5_cycles.sh "" rs2_C C >> gpurun_out/g11/cycles.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g11/bench_HY.json 2> gpurun_out/g11/bench_HY.err
