"""Accuracy study (the paper's Fig. 8) and
time to solution with iterative refinement.  Runs on the GPU through the C ABI;
writes profiles/<tag>_accuracy.md.

1. A Fig.8-like synthetic system (100x400x100, the shape of the paper's MFIX
   momentum system; seeded convection-diffusion, delta = 0 and 0.1): the
   recurrence residual of fp32 and mixed BiCGStab (both schedules) and the true
   residual of the mixed solution, per iteration.
2. 600x595x1536 (cfg 3 operator): device time to reach ||r||/||b|| <= 1e-6 with
   fp32 BiCGStab vs mixed iterative refinement (fp32 residual, fp16 inner solves).
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402


def hist_run(st, prec, b, maxit, sched, half=False):
    sten.set_schedule(st, sched)
    sten.set_dot_precision(st, sten.DOTS_HALF if half else sten.DOTS_MIXED)
    x = torch.empty_like(b)
    it, hist, status = sten.bicgstab_solve(st, prec, b, None, 0.0, maxit, x)
    sten.set_dot_precision(st, sten.DOTS_MIXED)
    return hist, x


def main(tag="r1"):
    out = [f"# {tag}: accuracy study and time to solution (B200, `python tools/accuracy_study.py`)\n"]
    nx, ny, nz = 100, 400, 100
    out.append(f"## 1. Fig. 8-like run: {nx}x{ny}x{nz} seeded convection-diffusion (stand-in for the MFIX "
               "momentum system, PAPER.md:591)\n")
    out.append("Recurrence residual ||r_i||/||b|| (R4) per iteration; `true16` is the fp64 true residual of the "
               "mixed x (computed on the GPU in fp32 through the refinement's residual step).\n")
    its = [0, 2, 4, 7, 10, 15, 20, 30, 40, 60]
    for delta in (0.0, 0.1):
        diag, offs = icuda.fields_device(inputs.KIND_CD, nx, ny, nz, seed=1, delta=delta)
        st = sten.stencil_create(nx, ny, nz, [diag] + offs)
        b32 = icuda.uniform_device(nx, ny, nz, seed=1, stream=0).float()
        b16 = b32.half()
        rows = {}
        for name, prec, b, sched in (("fp32 classic", sten.FP32, b32, 0), ("fp32 SR", sten.FP32, b32, 1),
                                     ("mixed classic", sten.MIXED, b16, 0), ("mixed SR", sten.MIXED, b16, 1),
                                     ("half-dot SR", sten.MIXED, b16, 2)):
            h, x = hist_run(st, prec, b, 60, min(sched, 1), half=sched == 2)
            rows[name] = h
            if prec == sten.MIXED:
                # true residual of the mixed solution: one refinement step with outer_maxit = 0 from x0 = x
                x32 = x.float()
                xo = torch.empty_like(x32)
                _, _, th, _ = sten.bicgstab_refine(st, b32, x32, 1e-30, 0, 1e-2, 1, xo)
                rows[name + " (true, final x)"] = th
        out.append(f"\n### delta = {delta}\n")
        out.append("| iteration | " + " | ".join(k for k in rows if "true" not in k) + " |")
        out.append("|---|" + "---|" * sum(1 for k in rows if "true" not in k))
        for i in its:
            out.append(f"| {i} | " + " | ".join(f"{rows[k][i]:.2e}" if i < len(rows[k]) else "-"
                                                for k in rows if "true" not in k) + " |")
        for k in rows:
            if "true" in k:
                out.append(f"\nTrue residual of the {k.split(' (')[0]} x after 60 iterations: {rows[k][0]:.2e}")
        # refinement on the same system
        sten.set_schedule(st, 1)
        xo = torch.empty_like(b32)
        ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, 30, 1e-2, 200, xo)
        out.append(f"\nIterative refinement (SR inner, inner tol 1e-2): {ko} outer steps, {ki} mixed iterations, "
                   f"status {sten.STATUS_NAMES[status]}; outer residuals " + ", ".join(f"{v:.1e}" for v in rh) + "\n")
        if delta == 0.0:  # the weakly dominant system: short, loose inner solves
            for sched, sname in ((1, "SR"), (0, "classic")):
                sten.set_schedule(st, sched)
                ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, 60, 0.1, 25, xo)
                out.append(f"Iterative refinement ({sname} inner, inner tol 0.1, <= 25 inner iterations): {ko} outer "
                           f"steps, {ki} mixed iterations, status {sten.STATUS_NAMES[status]}, final outer residual "
                           f"{rh[-1]:.1e}\n")
        st.close()
        del diag, offs
        torch.cuda.empty_cache()

    # 2. time to solution at the paper's mesh
    NX, NY, NZ = 600, 595, 1536
    out.append(f"\n## 2. Time to ||r||/||b|| <= 1e-6 at {NX}x{NY}x{NZ} (cfg 3 operator, delta = 0.1)\n")
    diag, offs = icuda.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
    st = sten.stencil_create(NX, NY, NZ, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    b32 = icuda.uniform_device(NX, NY, NZ, seed=1, stream=0).float()
    x32 = torch.empty_like(b32)
    out.append("| method | iterations | device time (ms) | achieved ||r||/||b|| |")
    out.append("|---|---|---|---|")
    for sched, name in ((1, "SR"), (0, "classic")):
        sten.set_schedule(st, sched)
        sten.bicgstab_solve(st, sten.FP32, b32, None, 1e-6, 500, x32)  # warm-up (graphs)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        it, hist, status = sten.bicgstab_solve(st, sten.FP32, b32, None, 1e-6, 500, x32)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        out.append(f"| fp32 BiCGStab ({name}) | {it} | {ms:.1f} | {hist[-1]:.2e} (recurrence) |")
        sten.bicgstab_refine(st, b32, None, 1e-6, 30, 1e-2, 200, x32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, 30, 1e-2, 200, x32)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        out.append(f"| mixed refinement ({name} inner, tol 1e-2) | {ko} outer / {ki} mixed | {ms:.1f} | "
                   f"{rh[-1]:.2e} (fp32 true) |")
    st.close()
    path = os.path.join(ROOT, "profiles", f"{tag}_accuracy.md")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
