"""R21 handover on the weakly dominant Fig. 8-like system (100x400x100 convection-diffusion, delta = 0,
the accuracy study's stand-in, profiles/r1_accuracy.md): mixed iterative refinement to 1e-6 with
short, loose inner solves (inner tol 0.1, <= 25 iterations) and SR / classic inner schedules; with
SR the first stagnation hands the inner solves over to the classic schedule.  GPU, through the C ABI:
  python tools/refine_handover.py  ->  one line per run"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import inputs  # noqa: E402
import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

nx, ny, nz = 100, 400, 100
for delta in (0.0, 0.1):
    diag, offs = icuda.fields_device(inputs.KIND_CD, nx, ny, nz, seed=1, delta=delta)
    st = sten.stencil_create(nx, ny, nz, [diag] + offs)
    b32 = icuda.uniform_device(nx, ny, nz, seed=1, stream=0).float()
    xo = torch.empty_like(b32)
    for sched, sname in ((1, "SR"), (0, "classic")):
        for inner_tol, inner_maxit, outer in ((0.1, 25, 60), (1e-2, 200, 30)):
            sten.set_schedule(st, sched)
            torch.cuda.synchronize()
            t = time.perf_counter()
            ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, outer, inner_tol, inner_maxit, xo)
            ms = (time.perf_counter() - t) * 1e3
            print(f"delta={delta} inner={sname} inner_tol={inner_tol} inner_maxit={inner_maxit}: {ko} outer, {ki} "
                  f"fp16 iterations, status {sten.STATUS_NAMES[status]}, handover at outer step "
                  f"{sten.get_stats(st)['handover']}, final {rh[-1]:.2e}, {ms:.1f} ms", flush=True)
    st.close()
