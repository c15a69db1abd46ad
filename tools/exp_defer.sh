#!/bin/bash
# Deferral-schedule sweep (measurement 4). Needs a library built with
#   make -C paper_1105_2737_b200 build/libgrfc_xdefer.so XDEFS=-DGRFC_DEFER_BUILD=15
# and GRFC_LIB=paper_1105_2737_b200/build/libgrfc_xdefer.so: checks bit-identity against the
# default schedule on 1/40/300 fields, then sweeps the ring geometry on c2, c5 and c3.
cd /root/repo
cat > /tmp/t.py <<'PY'
import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_1105_2737_b200 import grfc
plan = grfc.Plan((512,512),(1.0,1.0),grfc.Density.matern(2,1.5,0.1),grfc.ONE_FFT_OVERWRITE,grfc.F32,device=0)
for n in (1, 40, 300):
    a = plan.generate_tensor(0,0,n).clone()
    b = plan.generate_tensor(0,0,n).clone()
    os.environ['GRFC_DEFER']='1'
    c = plan.generate_tensor(0,0,n).clone()
    os.environ['GRFC_RING_LA']='1'; os.environ['GRFC_RING_SL']='1'
    d = plan.generate_tensor(0,0,n).clone()
    for k in ('GRFC_DEFER','GRFC_RING_LA','GRFC_RING_SL'): os.environ.pop(k)
    torch.cuda.synchronize()
    print(n, 'default==default', torch.equal(a,b), 'defer==default', torch.equal(a,c), 'defer-small==default', torch.equal(a,d), float(a.abs().max()), flush=True)
PY
timeout 90 python /tmp/t.py 2>&1 | tail -4 | tee /tmp/t.out; grep -q '^300 ' /tmp/t.out || { echo CORRECTNESS RUN INCOMPLETE; exit 1; }
V=()
for la in 1 2 3 4 6 12; do for sl in 1 3; do V+=("GRFC_DEFER=1 GRFC_RING_LA=$la GRFC_RING_SL=$sl"); done; done
timeout 150 python tools/ab_env.py --config c2 "GRFC_DEFER=1" "${V[@]}" 2>&1
echo "--- c5"
timeout 150 python tools/ab_env.py --config c5 "GRFC_DEFER=1" "GRFC_DEFER=1 GRFC_RING_LA=1 GRFC_RING_SL=1" "GRFC_DEFER=1 GRFC_RING_LA=2 GRFC_RING_SL=1" "GRFC_DEFER=1 GRFC_RING_LA=3 GRFC_RING_SL=2"  "GRFC_DEFER=1 GRFC_RING_LA=4 GRFC_RING_SL=3" 2>&1
echo "--- c3"
timeout 150 python tools/ab_env.py --config c3 --iters 8 "GRFC_DEFER=1" "GRFC_DEFER=1 GRFC_RING_LA=1 GRFC_RING_SL=1" "GRFC_DEFER=1 GRFC_RING_LA=0 GRFC_RING_SL=0" 2>&1
