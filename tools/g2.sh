# microbenchmarks for the K5 redesign: UMMA rates with/without concurrent TMA, Q-in-TMEM; L2->SMEM TMA;
# dense ceilings (library SDPA, K5 dense); synccheck on the sanitizer build
mkdir -p gpurun_out/g2
timeout 300 ./tools/mma_bw > gpurun_out/g2/mma_bw.txt 2>&1
timeout 300 ./tools/tma_bw > gpurun_out/g2/tma_bw.txt 2>&1
timeout 300 python tools/sdpa_ceiling.py 32768 24 > gpurun_out/g2/sdpa.txt 2>&1
timeout 300 python tools/sdpa_ceiling.py 118800 8 >> gpurun_out/g2/sdpa.txt 2>&1
timeout 300 python tools/dense_probe.py > gpurun_out/g2/dense_probe.txt 2>&1
OUT=gpurun_out/g2 timeout 1200 bash tools/sanitize.sh > gpurun_out/g2/sanitize_summary.txt 2>&1
