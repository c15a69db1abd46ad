#!/bin/bash
# Pipe utilisation of the c2 kernel (ncu sections + the L1/shared data-pipe wavefront metric
# that DESIGN.md 8 builds on).
cd /root/repo
cat > /tmp/r.py <<'PY'
import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_1105_2737_b200 import grfc
plan = grfc.Plan((512,512),(1.0,1.0),grfc.Density.matern(2,1.5,0.1),grfc.ONE_FFT_OVERWRITE,grfc.F32,device=0)
out = plan.generate_tensor(0,0,1024)
for _ in range(2): plan.generate_tensor(0,0,1024,out=out)
torch.cuda.synchronize()
PY
timeout 300 ncu --section ComputeWorkloadAnalysis --section SchedulerStats --section WarpStateStats --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --clock-control none -k regex:k_fused2d -s 2 -c 1 python /tmp/r.py 2>&1 | sed -n '/Section: Compute/,$p'
timeout 300 ncu --metrics sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_issued.avg.per_cycle_active,smsp__warps_eligible.avg.per_cycle_active,smsp__warps_active.avg.per_cycle_active,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,sm__mio_inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_fma_pred_on_fp32x2.sum --clock-control none -k regex:k_fused2d -s 2 -c 1 python /tmp/r.py 2>&1 | grep -E "sm__|smsp__|l1tex__"
