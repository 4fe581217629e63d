mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g1/summary.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g1/bench_HY.json 2> gpurun_out/g1/bench_HY.err
timeout 300 python bench.py --workload C --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g1/bench_C.json 2>&1
timeout 300 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize.py > gpurun_out/g1/synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/g1/summary.txt
