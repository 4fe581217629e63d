OUT=gpurun_out/iso2 bash tools/k5_isolation.sh
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_sm100 -s 1 -c 1 -o gpurun_out/iso2/k5_C python tools/k5_once.py C > gpurun_out/iso2/ncu_C.log 2>&1
