"""Quick 2D solve timing for kernel experiments: python tools/b2d_quick.py <tag|base> [n] [maxit]
(mixed and fp32 BiCGStab on the 2D stand-in, per-phase ms via stencil2d_set_timing)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

tag = sys.argv[1]
if tag != "base":
    sten.LIB_PATH = os.path.join(ROOT, "paper_2010_03660_b200", f"libsten_{tag}.so")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 22800
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 50
diag, offs = icuda.fields2d_device(n, n, seed=1, delta=0.1)
st = sten.stencil2d_create(n, n, [diag] + offs)
del diag, offs
torch.cuda.empty_cache()
b64 = icuda.uniform_device(n, n, 1, seed=1, stream=0).view(n, n)
for prec, dt in ((sten.MIXED, torch.float16), (sten.FP32, torch.float32)):
    b = b64.to(dt)
    x = torch.empty_like(b)
    sten.stencil2d_set_timing(st, True)
    sten.bicgstab2d_solve(st, prec, b, None, 0.0, 4, x)
    it, hist, status = sten.bicgstab2d_solve(st, prec, b, None, 0.0, maxit, x)
    ph, nit = sten.stencil2d_phase_ms(st)
    es = 2 if prec == sten.MIXED else 4
    tot = sum(ph)
    print(f"{tag} {'mixed' if es == 2 else 'fp32'} ms/it {tot:.4f} H1 {ph[0]:.4f} H2 {ph[1]:.4f} H3 {ph[2]:.4f} "
          f"frac33 {33 * es * n * n / (tot * 1e-3) / 6547.2e9:.4f} hist[-1] {hist[-1]:.3e}", flush=True)
    del b, x
st.close()
