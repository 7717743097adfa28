"""Quick start: the C ABI through the Python binding, on one B200.

    python examples/quickstart.py [nx ny nz]

1. build a 7-point convection-diffusion operator (diagonal + six couplings, fp64 on the device),
2. solve A x = b in the paper's mixed mode with the single-reduction schedule,
3. solve several right-hand sides with the host copies pipelined (bicgstab_solve_batch),
4. refine a mixed solve to an fp32 answer (bicgstab_refine),
5. check the true residual with the library's own SpMV.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402


def main(nx=128, ny=96, nz=64):
    icuda.build()
    # 1. the operator: diag a_P and couplings A_xm..A_zp of a seeded upwinded convection-diffusion
    #    stencil (inputs/ holds no arithmetic of the method, only the random fields)
    diag, offs = icuda.fields_device(inputs.KIND_CD, nx, ny, nz, seed=1, delta=0.1)
    st = sten.stencil_create(nx, ny, nz, [diag] + offs)  # Jacobi-scaled inside, fp32 + fp16 copies
    sten.set_schedule(st, sten.SCHED_SR)

    # 2. one mixed-precision solve to the paper's 1e-3
    b = icuda.uniform_device(nx, ny, nz, seed=1, stream=0)
    b16 = b.half()
    x16 = torch.empty_like(b16)
    it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b16, None, 1e-3, 200, x16)
    print(f"mixed: {it} iterations, status {sten.STATUS_NAMES[status]}, ||r||/||b|| = {hist[-1]:.2e}")

    # 3. a batch of right-hand sides from pinned host memory
    bs = [icuda.uniform_device(nx, ny, nz, seed=s, stream=0).half().cpu().pin_memory() for s in (2, 3, 4)]
    xs = [torch.empty_like(t).pin_memory() for t in bs]
    for i, (itb, hb, sb) in enumerate(sten.bicgstab_solve_batch(st, sten.MIXED, bs, xs, 1e-3, 200)):
        print(f"batch[{i}]: {itb} iterations, ||r||/||b|| = {hb[-1]:.2e}")

    # 4. mixed-precision iterative refinement to an fp32 answer
    b32 = b.float()
    x32 = torch.empty_like(b32)
    outer, inner, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, 20, 1e-2, 200, x32)
    print(f"refine: {outer} outer steps, {inner} mixed iterations, ||r||/||b|| = {rh[-1]:.2e}")

    # 5. the true residual of the refined x on the scaled system, by the library's SpMV
    ax = torch.empty_like(x32)
    sten.stencil_apply(st, sten.FP32, x32, ax)
    bhat = (b.double() / diag).float()
    true = float(torch.linalg.vector_norm((bhat - ax).double()) / torch.linalg.vector_norm(bhat.double()))
    print(f"true residual of the refined x: {true:.2e}")
    st.close()
    return hist[-1], rh[-1], true


if __name__ == "__main__":
    main(*(int(v) for v in sys.argv[1:4]))
