"""Small runs of every kernel family for compute-sanitizer (one tool per gpurun call):
3D classic solve (k_stencil H1/H2, k_h3_bulk, k_init), SR solve (k_sr, k_sr_last), 2D gather and
tiled SpMV (k_apply9, k_ring9, k_round9), 2D solve (persistent k_bicg9)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

torch.cuda.set_device(0)
nx, ny, nz = 70, 37, 24
diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=1, delta=0.1)
st = sten.stencil_create(nx, ny, nz, [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs])
b = torch.from_numpy(inputs.rhs_uniform(nx, ny, nz, seed=1)).cuda()
for prec, dt in ((sten.MIXED, torch.float16), (sten.FP32, torch.float32)):
    for sch in (sten.SCHED_CLASSIC, sten.SCHED_SR):
        sten.set_schedule(st, sch)
        x = torch.empty_like(b, dtype=dt)
        it, hist, status = sten.bicgstab_solve(st, prec, b.to(dt), None, 0.0, 6, x)
        print("3D", prec, sch, it, hist[-1])
st.close()
n2x, n2y = 300, 140
d2, o2 = inputs.problem_fields_2d(n2x, n2y, seed=2)
s2 = sten.stencil2d_create(n2x, n2y, [torch.from_numpy(d2).cuda()] + [torch.from_numpy(o).cuda() for o in o2])
b2 = torch.from_numpy(inputs.rhs_uniform_2d(n2x, n2y, seed=2)).cuda()
for prec, dt in ((sten.MIXED, torch.float16), (sten.FP32, torch.float32)):
    y = torch.empty_like(b2, dtype=dt)
    for tiles in ((1, 1), (7, 5), (40, 30)):
        sten.stencil2d_set_tiles(s2, *tiles)
        sten.stencil2d_apply(s2, prec, b2.to(dt), y)
    sten.stencil2d_set_tiles(s2, 1, 1)
    x2 = torch.empty_like(b2, dtype=dt)
    it, hist, status = sten.bicgstab2d_solve(s2, prec, b2.to(dt), None, 0.0, 6, x2)
    print("2D", prec, it, hist[-1])
s2.close()
torch.cuda.synchronize()
print("sanitize run ok")
