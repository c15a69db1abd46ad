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
for v in "" "GRFC_DEFER=1 GRFC_RING_LA=4 GRFC_RING_SL=3" "GRFC_DEFER=1 GRFC_RING_LA=2 GRFC_RING_SL=3" "GRFC_RING_LA=4 GRFC_RING_SL=3"; do
  echo "== variant: $v"
  env $v timeout 200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_executed.avg.per_cycle_active --clock-control none -k regex:k_fused2d -s 2 -c 1 python /tmp/r.py 2>&1 | grep -E "duration|dram__|hit_rate|per_cycle" 
done
