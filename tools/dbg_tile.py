import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np, torch, inputs, oracle as orc
import paper_2010_03660_b200 as sten
from gpu_util import *
for (nx,ny,nz),til in [((45,23,17),(64,16,5,3)),((45,23,17),(64,4,64,4)),((45,23,17),(64,16,64,3)),((45,23,17),(64,16,5,4)),((64,23,17),(64,16,5,3)),((45,16,17),(64,16,5,3))]:
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, seed=3)
    st = gpu_stencil(diag, offs); sten.set_tiling(st, 0, *til)
    cq = oracle_coeffs(diag, offs, "fp32")
    v = quantize_vec(np.random.default_rng(1).uniform(-1, 1, (nz, ny, nx)), "fp32")
    vt = to_gpu_vec(v, "fp32"); yt = torch.empty_like(vt); sten.stencil_apply(st, 0, vt, yt)
    y = yt.cpu().numpy(); m = orc.apply32_fma(cq, v)
    bad = np.argwhere(y != m)
    print((nx,ny,nz), til, 'nbad', len(bad), bad[:5].tolist(), 'zs', sorted(set(bad[:,0].tolist()))[:20] if len(bad) else '')
