mkdir -p gpurun_out/g3
timeout 300 ./tools/mma_bw 2>&1 | grep -E "ring|K5:" > gpurun_out/g3/mma_bw.txt
timeout 900 python -m pytest tests/test_gpu_attn_sm100.py -x -q > gpurun_out/g3/pytest_attn.log 2>&1; echo "attn rc=$?" >> gpurun_out/g3/summary.txt
for lib in "" build/ab/lib_noqt.so; do bash tools/k5_cycles.sh "$lib" "${lib:-qt}" HY >> gpurun_out/g3/cycles.txt 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g3/bench_HY.json 2> gpurun_out/g3/bench_HY.err
DFS_B200_LIB=build/ab/lib_noqt.so timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g3/bench_HY_noqt.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g3/pytest.log 2>&1; echo "all rc=$?" >> gpurun_out/g3/summary.txt
