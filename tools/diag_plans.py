import sys; sys.path.insert(0, '.')
from paper_1105_2737_b200 import grfc
for dt in (grfc.F32, grfc.F64):
    for n1 in (256, 512, 1024, 2048, 4096):
        for n2 in (256, 512, 1024, 2048, 4096):
            try:
                p = grfc.Plan((n1, n2), (1.0, 1.0), grfc.Density.matern(2, 1.5, 0.1), 1, dt)
            except Exception as e:
                print("FAIL", dt, n1, n2, e)
print("diag done")
