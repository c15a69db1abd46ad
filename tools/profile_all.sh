#!/bin/bash
# Round profile refresh (run on the GPU box from the repo root): bench line + ncu
# launch list + one `ncu --set full` capture per headline kernel, into gpurun_out/.
set -x
cd "$(dirname "$0")/.."
ROUND=${ROUND:-r01}
ROUND=$ROUND CONFIG=c2 KERNEL=k_fused2d bash tools/profile_round.sh
ROUND=$ROUND CONFIG=c3 KERNEL=k_fused2d bash tools/profile_round.sh
ROUND=$ROUND CONFIG=c5 KERNEL=k_fused2d bash tools/profile_round.sh
python tools/prof_run.py c2 0 1 > /dev/null
GRFC_ALG=0 ncu --set full --clock-control none --import-source on -k "regex:k_fused2d_alg1" -c 1 \
  -o gpurun_out/${ROUND}_c2alg1_full python tools/prof_run.py c2 0 1 > gpurun_out/${ROUND}_c2alg1_ncu.log 2>&1
python tools/prof_run.py c4 0 1 > /dev/null
ncu --set full --clock-control none --import-source on -k "regex:k_3d" -c 2 \
  -o gpurun_out/${ROUND}_c4_full python tools/prof_run.py c4 0 1 > gpurun_out/${ROUND}_c4_ncu.log 2>&1
echo done-all
