"""BASELINE configs 1 and 2 (the small, L2-resident meshes): iterations and time to
the 1e-6 target, and the per-iteration device time of a fixed 100-iteration run
(CUDA events around the graph replays, tol = 0), for both schedules.  Config 1 is
the constant Poisson operator, so it also runs through stencil_create_const.
Writes profiles/<tag>_small.md."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import oracle as orc  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402


def run(st, b, sched, label, rows):
    sten.set_schedule(st, sched)
    x = torch.empty_like(b)
    sten.bicgstab_solve(st, sten.FP32, b, None, 1e-6, 2000, x)  # warm (graphs)
    it, hist, status = sten.bicgstab_solve(st, sten.FP32, b, None, 1e-6, 2000, x)
    ms_tts = sten.get_stats(st)["solve_ms"]
    sten.bicgstab_solve(st, sten.FP32, b, None, 0.0, 100, x)
    sten.bicgstab_solve(st, sten.FP32, b, None, 0.0, 100, x)
    us_it = sten.get_stats(st)["solve_ms"] * 1e3 / 100
    rows.append(f"| {label} | {'SR' if sched else 'classic'} | {it} | {sten.STATUS_NAMES[status]} | "
                f"{hist[-1]:.1e} | {ms_tts:.3f} | {us_it:.1f} |")


def main(tag="r1"):
    rows = [f"# {tag}: BASELINE configs 1 and 2 (fp32, tol 1e-6; L2-resident meshes)\n",
            "`solve_ms` is the device time of the whole solve (init + iterations + status polls every 8 "
            "iterations); `us/it` is from a fixed 100-iteration solve (one graph replay).\n",
            "| config | schedule | iterations | status | final hist | time to 1e-6 (ms) | us / iteration |",
            "|---|---|---|---|---|---|---|"]
    n = 32  # config 1: Poisson, b = A x_true
    diag, offs = inputs.problem_fields(inputs.KIND_POISSON, n, n, n)
    xt = inputs.rhs_uniform(n, n, n, seed=1)
    b1 = torch.from_numpy(orc.apply_raw64(diag, offs, xt).astype(np.float32)).cuda()
    st = sten.stencil_create(n, n, n, [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs])
    for sched in (sten.SCHED_SR, sten.SCHED_CLASSIC):
        run(st, b1, sched, "1: 32^3 Poisson (fields)", rows)
    st.close()
    stc = sten.stencil_create_const(n, n, n, (6.0, -1, -1, -1, -1, -1, -1))
    for sched in (sten.SCHED_SR, sten.SCHED_CLASSIC):
        run(stc, b1, sched, "1: 32^3 Poisson (constant operator)", rows)
    stc.close()
    n = 128  # config 2: convection-diffusion, delta = 0.1
    diag, offs = inputs.problem_fields(inputs.KIND_CD, n, n, n, seed=1, delta=0.1)
    b2 = torch.from_numpy(inputs.rhs_uniform(n, n, n, seed=1).astype(np.float32)).cuda()
    st = sten.stencil_create(n, n, n, [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs])
    for sched in (sten.SCHED_SR, sten.SCHED_CLASSIC):
        run(st, b2, sched, "2: 128^3 conv.-diff.", rows)
    st.close()
    out = "\n".join(rows) + "\n"
    print(out)
    with open(os.path.join(ROOT, "profiles", f"{tag}_small.md"), "w") as f:
        f.write(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
