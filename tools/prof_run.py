"""Small driver for ncu captures: one (or a few) generate calls of a config.

    python tools/prof_run.py [config] [nfields] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import CONFIGS  # noqa: E402
from paper_1105_2737_b200 import grfc  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
nf = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else cfg["fields"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
alg = int(os.environ.get("GRFC_ALG", cfg["algs"][0]))
d = len(cfg["counts"])
fam = cfg["density"]
dens = grfc.Density.gaussian_cov(d, fam[1]) if fam[0] == "gauss" else grfc.Density.matern(d, fam[1], fam[2])
dtype = grfc.F64 if cfg["dtype"] == "f64" else grfc.F32
plan = grfc.Plan(cfg["counts"], (1.0,) * d, dens, alg, dtype)
out = torch.empty((nf,) + tuple(cfg["counts"]), dtype=torch.float64 if dtype == grfc.F64 else torch.float32,
                  device="cuda")
for _ in range(reps):
    plan.generate(0, 0, nf, out.data_ptr(), plan.points, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", plan.path, float(out[0].float().std()))
