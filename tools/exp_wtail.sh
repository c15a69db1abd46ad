cd /root/repo
cat > /tmp/a.py <<'PY'
import os, sys, torch, statistics, hashlib
sys.path.insert(0, '/root/repo')
import bench
CFGS = sys.argv[1:] or ['c2','c5','c3']
from paper_1105_2737_b200 import grfc
for cfg in CFGS:
    c = bench.CONFIGS[cfg]
    fam = c["density"]; d = len(c["counts"])
    dens = grfc.Density.gaussian_cov(d, fam[1]) if fam[0] == "gauss" else grfc.Density.matern(d, fam[1], fam[2])
    plan = grfc.Plan(c["counts"], tuple(1.0 for _ in c["counts"]), dens, 1, grfc.F32, device=0)
    n = c["fields"]
    out = plan.generate_tensor(0,0,n)
    for _ in range(3): plan.generate_tensor(0,0,n,out=out)
    torch.cuda.synchronize()
    ts=[]
    for _ in range(15):
        a,b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); plan.generate_tensor(0,0,n,out=out); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    pts = n
    for x in c["counts"]: pts *= x
    ms = statistics.median(ts)
    h = hashlib.sha1(out[:: max(1, n//8)].contiguous().cpu().numpy().tobytes()).hexdigest()[:12]
    print(cfg, f"{ms:.4f} ms {pts/ms/1e6:.1f} Gpts/s min {min(ts):.4f} sha {h}", flush=True)
PY
for lib in paper_1105_2737_b200/lib/libgrfc.so paper_1105_2737_b200/build/libgrfc_xnowt.so paper_1105_2737_b200/lib/libgrfc.so paper_1105_2737_b200/build/libgrfc_xnowt.so; do echo "== $lib"; GRFC_LIB=$lib timeout 100 python /tmp/a.py c3 2>&1 | tail -3; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
