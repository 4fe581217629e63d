#!/bin/bash
# K5 dense vs cuDNN SDPA in SM cycles at d = 64 and d = 128 (tools/d64_ceiling.py): FLOP per
# SM-cycle of each kernel, immune to the power-capped clock. One launch of each per head dim.
ncu --metrics sm__cycles_elapsed.max,gpu__time_duration.sum --clock-control none \
  -k regex:'attn_sm100|cudnn|fmha|sm100_f' --launch-skip 0 -c 40 --csv \
  python tools/d64_ceiling.py "${1:-32768}" "${2:-24}" 2>/dev/null | grep -E "sm__cycles_elapsed.max" \
  | awk -F'","' '{gsub(/"/,"",$NF); print $5, $NF}'
