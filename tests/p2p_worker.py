"""One rank of the cross-process peer-memory solve (tests/test_gpu_multiproc.py).

Run as `python tests/p2p_worker.py RANK WORLD PORT OUTDIR PREC MAXIT TOL NX NY NZ SEED [SCHEDULE [OP]]`
(SCHEDULE sr, the default, classic, or classic_fused; OP fields, the default, or const: the skew
constant-coefficient operator of stencil_create_const).
Every rank uses cuda:0 (the one GPU here), owns planes [r nz/R, (r+1) nz/R) of the
mesh, builds its handle on a peer-memory-only communicator (sten_comm_create with
no NCCL id), exchanges the CUDA IPC records over gloo, and solves in host lockstep
(sten_set_host_barrier: a gloo barrier before every peer all-reduce's waiting
kernel, so no kernel ever waits on another process's kernel on the shared GPU).
Writes x, the history, iterations and status of its slab to OUTDIR/rank<R>.npz.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


CONST_SKEW = (3.0, -0.7, -0.4, -0.25, -0.55, -0.3, -0.5)  # the constant operator of test_gpu_const*.py


def main():
    rank, world, port = (int(v) for v in sys.argv[1:4])
    outdir, prec = sys.argv[4], sys.argv[5]
    maxit, tol = int(sys.argv[6]), float(sys.argv[7])
    nx, ny, nz, seed = (int(v) for v in sys.argv[8:12])
    schedule = sys.argv[12] if len(sys.argv) > 12 else "sr"
    op = sys.argv[13] if len(sys.argv) > 13 else "fields"
    import numpy as np
    import torch
    import torch.distributed as dist

    import inputs
    import paper_2010_03660_b200 as sten
    from gpu_util import from_gpu_vec, quantize_vec, to_gpu_vec

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    nzl = nz // world
    z0 = rank * nzl
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nzl, z0=z0, seed=seed, delta=0.1)
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nzl, z0=z0, seed=seed), prec)
    comm = sten.comm_create(None, world, rank, 0)
    if op == "const":
        st = sten.stencil_create_const(nx, ny, nz, CONST_SKEW, nslabs=1, comm=comm)
    else:
        coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
        st = sten.stencil_create(nx, ny, nz, coeffs, nslabs=1, comm=comm)
    torch.cuda.synchronize()
    dist.barrier()  # every rank's coefficients exist before anyone imports (sten.h)
    P = sten.FP32 if prec == "fp32" else sten.MIXED
    sten.set_schedule(st, sten.SCHED_SR if schedule == "sr" else sten.SCHED_CLASSIC)
    if schedule == "classic_fused":  # halos and sums stored by the phase kernels themselves
        sten.set_option(st, sten.OPT_CLASSIC_FUSED, 1)
    sten.p2p_setup(st, P)  # export, all_gather over gloo, import
    sten.set_host_barrier(st, lambda: dist.barrier())
    bt = to_gpu_vec(b, prec)
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, P, bt, None, tol, maxit, xt)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), x=from_gpu_vec(xt, prec), hist=hist, it=it, status=status,
             launches=sten.get_stats(st)["kernel_launches"])
    dist.barrier()  # nobody unmaps a peer's buffers while another rank may still touch them
    st.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
