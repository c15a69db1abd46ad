import sys, itertools
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1105_2737_b200 import grfc
from oracle import pyoracle as po
port = po.Port()
def od(g):
    d = po.Density(); d.family, d.dim = g.family, g.dim
    for k in range(8): d.r[k], d.i[k] = g.r[k], g.i[k]
    return d
for counts in [(128,128,128), (256,128,128), (128,256,128), (128,128,256), (512,128,128), (128,512,128), (128,128,512), (256,256,256)]:
    for dt in (grfc.F32,):
        dens = grfc.Density.gaussian_cov(3, 0.03)
        plan = grfc.Plan(counts, (1.0,1.0,1.0), dens, 1, dt)
        got = plan.generate_tensor(4, 2, 1)[0].cpu().numpy().astype(np.float64)
        want, _ = port.synthesize(counts, (1.0,1.0,1.0), od(dens), 1, plan.dump_noise(4, 2))
        e = np.linalg.norm(got - want) / np.linalg.norm(want)
        print(counts, plan.path, "rel", e, "var got/want", (got**2).mean(), (want**2).mean(), flush=True)
