mkdir -p gpurun_out/g9
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > gpurun_out/g9/pytest_attn.log 2>&1; echo "attn rc=$?" >> gpurun_out/g9/summary.txt
for lib in "" build/ab/lib_colsplit.so build/ab/lib_rs_SKIP_MMA.so; do bash tools/k5_cycles.sh "$lib" "${lib:-rowsplit}" HY >> gpurun_out/g9/cycles.txt 2>&1; done
DFS_B200_LIB=build/ab/lib_trace.so timeout 300 python tools/trace_attn.py > gpurun_out/g9/trace.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g9/bench_HY.json 2> gpurun_out/g9/bench_HY.err
