set -x
ROUND=r01 CONFIG=c2 KERNEL=k_fused2d bash tools/profile_round.sh
ROUND=r01 CONFIG=c3 KERNEL=k_fused2d bash tools/profile_round.sh
python tools/prof_run.py c2 0 1 > /dev/null
GRFC_ALG=0 ncu --set full --clock-control none --import-source on -k "regex:k_fused2d_alg1" -c 1 -o gpurun_out/r01_c2alg1_full python tools/prof_run.py c2 0 1 > gpurun_out/r01_c2alg1_ncu.log 2>&1
echo done-all
