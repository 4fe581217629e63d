# cuDNN SDPA (dense, library kernel) in SM cycles at N=32768, 24 heads, d=128: FLOP per SM-cycle
# for comparison with K5 (tools/k5_cycles.sh). Prints ncu's cycles and duration of the attention kernel.
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum,smsp__cycles_active.avg --clock-control none -k regex:'cudnn|fmha|flash|attn|sm100' -c 2 --csv \
  python tools/sdpa_ceiling.py 32768 24 2>/dev/null | grep -E "sm__cycles_elapsed.max|gpu__time|Kernel" | tail -8
