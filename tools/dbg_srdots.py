"""Debug: SR sweep dot sums vs exact on a few meshes (prints relative errors)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2010_03660_b200 as sten
from test_gpu_sr import _sweep_case, _pairs
from gpu_util import widen
for mesh in [(37, 29, 19), (130, 17, 9), (130, 17, 1), (128, 16, 1), (136, 16, 1), (130, 16, 1), (128, 17, 1)]:
    got, dots, ref, rh = _sweep_case(sten, "mixed", mesh)
    wide = [widen(a, "mixed") for a in (rh, got[1], got[3], got[4], got[5])]
    errs = []
    for d, (a, b) in enumerate(_pairs(*wide)):
        exact = float(np.vdot(a, b)); scale = float(np.vdot(np.abs(a), np.abs(b)))
        errs.append((dots[d] - exact) / scale)
    print(mesh, " ".join(f"{e:+.1e}" for e in errs), flush=True)
