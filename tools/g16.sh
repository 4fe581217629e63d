mkdir -p gpurun_out/g16
timeout 600 python -m pytest tests/test_gpu_attn_sm100.py -x -q > gpurun_out/g16/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g16/summary.txt
bash tools/k5_cycles.sh "" mma9 HY >> gpurun_out/g16/cycles.txt 2>&1
bash tools/k5_cycles.sh "" mma9_C C >> gpurun_out/g16/cycles.txt 2>&1
DFS_B200_LIB=build/ab/lib_trace.so timeout 300 python tools/trace_attn.py > gpurun_out/g16/trace.txt 2>&1
