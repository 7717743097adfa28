"""One short 2D run at 22800^2 for ncu captures: a mixed BiCGStab of 2 iterations (k_init, then
k_bicg9<H1>, k_bicg9<H2>, k_h3 twice), a gather SpMV and a tiled (600 x 600) SpMV."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

n = 22800
diag, offs = icuda.fields2d_device(n, n, seed=1, delta=0.1)
st = sten.stencil2d_create(n, n, [diag] + offs)
del diag, offs
torch.cuda.empty_cache()
b = icuda.uniform_device(n, n, 1, seed=1, stream=0).view(n, n).half()
x = torch.empty_like(b)
it, hist, status = sten.bicgstab2d_solve(st, sten.MIXED, b, None, 0.0, 2, x)
sten.stencil2d_apply(st, sten.MIXED, b, x)
sten.stencil2d_set_tiles(st, 600, 600)
sten.stencil2d_apply(st, sten.MIXED, b, x)
st.close()
print("ok", it, hist)
