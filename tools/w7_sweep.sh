# W7 (Wan2.1-14B 720p, 40 heads) bench lines across the north-star sparsity sweep (gamma = kept
# fraction 0.30 ... 0.05, i.e. 70-95 % block sparsity) into gpurun_out/${OUT:-w7}/
OUT=${OUT:-gpurun_out/w7}; mkdir -p $OUT
for g in 0.30 0.25 0.20 0.15 0.10 0.05; do
  timeout 600 python bench.py --workload W7 --gamma $g --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_W7_g$g.json 2>&1
done
