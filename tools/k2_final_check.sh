OUT=gpurun_out/k2fin; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/summary.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_HY.json 2>&1
timeout 600 python bench.py --workload C --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_C.json 2>&1
timeout 300 python tools/permute_bench.py HY > $OUT/permute_HY.txt 2>&1
