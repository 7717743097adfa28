import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2010_03660_b200 as sten, oracle as orc
from gpu_util import from_gpu_vec, quantize_vec, to_gpu_vec, widen
POISSON = (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0)
for const in (True, False):
  for pack in (16, 8):
    for nslabs in (1, 3):
        nx, ny, nz = 1, 1, 3
        prec = "fp32"
        diag = np.full((nz, ny, nx), 6.0); offs = [np.full((nz, ny, nx), -1.0) for _ in range(6)]
        if const:
            st = sten.stencil_create_const(nx, ny, nz, POISSON, nslabs=nslabs)
        else:
            st = sten.stencil_create(nx, ny, nz, [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs], nslabs=nslabs)
        sten.set_sr_tiling(st, 0, 8, 2, 2, 3, pack)
        cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
        rng = np.random.default_rng(4)
        vec = lambda: quantize_vec(rng.uniform(-1, 1, (nz, ny, nx)), prec)
        rh, x, r, p = vec(), vec(), vec(), vec()
        v, q = orc.apply32_fma(cq, p), orc.apply32_fma(cq, r); y = orc.apply32_fma(cq, v)
        ts = [to_gpu_vec(a, prec) for a in (rh, x, r, p, v, q, y)]
        sten.sr_sweep(st, 0, (0.61, 0.93, -0.27), *ts)
        ref = orc.sr_sweep32(cq, (0.61, 0.93, -0.27), rh, x, r, p, v, q, y)
        names = "x r p v q y".split()
        bad = [n for n, g, w in zip(names, ts[1:], ref[:6]) if not np.array_equal(from_gpu_vec(g, prec), w)]
        print("const", const, "pack", pack, "nslabs", nslabs, "bad:", bad, "x gpu", from_gpu_vec(ts[1], prec).ravel(), "ref", ref[0].ravel(), "x in", x.ravel())
        st.close()
