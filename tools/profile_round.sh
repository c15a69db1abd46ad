#!/bin/bash
# Round profile capture (run on the GPU box from the repo root):
#   1. the bench line of CONFIG (no profiler),
#   2. the ncu launch list of the same bench command (per-launch durations, cold, serialised),
#   3. one `ncu --set full` capture of the top kernel (KERNEL regex) on a tools/prof_run.py call.
# Outputs land in gpurun_out/<ROUND>_<CONFIG>_*; copy the summaries into profiles/.
set -e
R=${ROUND:-r01}; C=${CONFIG:-c2}; K=${KERNEL:-k_fused2d}; NF=${NFIELDS:-0}
mkdir -p gpurun_out
python bench.py --config "$C" --steps 10 --warmup 3 > "gpurun_out/${R}_${C}_bench.json"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file "gpurun_out/${R}_${C}_launches.csv" \
    python bench.py --config "$C" --steps 2 --warmup 1 --no-cpu-baseline > /dev/null
python tools/prof_run.py "$C" $NF 1 > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:$K" -c 1 \
    -o "gpurun_out/${R}_${C}_full" python tools/prof_run.py "$C" $NF 1 > "gpurun_out/${R}_${C}_ncu.log" 2>&1
echo done
