"""libsten across PROCESSES (PAPER.md:193-195 z decomposition; PAPER.md:376-397 AllReduce).

Two processes share cuda:0 (the only GPU of the test box), each one rank of a
peer-memory-only communicator: rank r owns half of the z planes, imports the other
rank's CUDA IPC records (boundary-slab SR buffers, inbox, boundary coefficient
planes), and runs the fused SR solve - its sweep kernel stores its boundary planes
straight into the neighbour process's halo buffers and deposits its sums in both
processes' inboxes; the one-shot all-reduce is read by k_p2p_fin.  The solve runs
in host lockstep (sten_set_host_barrier + a gloo barrier), because kernels of two
processes on one GPU that wait on each other are not guaranteed to run together
(B200_PROFILING: Xid 109); with the barrier every flag is set before the waiting
kernel starts.  The result must be BITWISE the single-process solve on two
loopback slabs (same kernels, same slot order of the sums)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import inputs
from gpu_util import fields, from_gpu_vec, quantize_vec, to_gpu_vec, torch_cuda

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PREC = {"fp32": 0, "mixed": 1}


@pytest.fixture(scope="module")
def sten():
    import paper_2010_03660_b200 as s
    return s


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _run_ranks(tmp_path, world, prec, maxit, tol, nx, ny, nz, seed, schedule="sr", op="fields"):
    port = _free_port()
    procs = []
    for r in range(world):
        cmd = [sys.executable, os.path.join(ROOT, "tests", "p2p_worker.py"), str(r), str(world), str(port),
               str(tmp_path), prec, str(maxit), repr(tol), str(nx), str(ny), str(nz), str(seed), schedule, op]
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]
    return [np.load(os.path.join(tmp_path, f"rank{r}.npz")) for r in range(world)]


def _loopback(sten, prec, maxit, tol, nx, ny, nz, seed, world, schedule="sr", op="fields"):
    torch = torch_cuda()
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=seed), prec)
    if op == "const":
        from p2p_worker import CONST_SKEW
        st = sten.stencil_create_const(nx, ny, nz, CONST_SKEW, nslabs=world)
    else:
        diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=seed)
        coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
        st = sten.stencil_create(nx, ny, nz, coeffs, nslabs=world)
    if schedule == "sr":
        sten.set_schedule(st, sten.SCHED_SR)
        sten.set_sr_exchange(st, sten.XCHG_FUSED)
    else:  # the serial classic exchange: slab sums in slab order, like the peer-memory reduction
        sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, 0)
    bt = to_gpu_vec(b, prec)
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, PREC[prec], bt, None, tol, maxit, xt)
    x = from_gpu_vec(xt, prec)
    st.close()
    return x, it, hist, status


@pytest.mark.parametrize("prec,maxit,tol,mesh", [
    ("fp32", 12, 0.0, (40, 33, 24)),
    ("mixed", 12, 0.0, (40, 33, 24)),
    ("mixed", 40, 1e-3, (37, 29, 16)),  # stops on the tolerance: both ranks take the same decision
    ("fp32", 30, 1e-6, (64, 9, 10)),
])
def test_two_processes_fused_sr_equals_loopback_slabs(sten, tmp_path, prec, maxit, tol, mesh):
    nx, ny, nz = mesh
    seed = 5
    res = _run_ranks(tmp_path, 2, prec, maxit, tol, nx, ny, nz, seed)
    x_ref, it_ref, h_ref, s_ref = _loopback(sten, prec, maxit, tol, nx, ny, nz, seed, 2)
    for r in res:
        assert int(r["it"]) == it_ref and int(r["status"]) == s_ref
        assert np.array_equal(r["hist"], h_ref)
        assert int(r["launches"]) > 0
    x = np.concatenate([r["x"] for r in res], axis=0)
    assert x.shape == x_ref.shape
    assert np.array_equal(x, x_ref)
    if tol > 0:
        assert s_ref == sten.CONVERGED and it_ref < maxit and h_ref[-1] <= tol


@pytest.mark.parametrize("schedule", ["classic", "classic_fused"])
@pytest.mark.parametrize("prec,maxit,tol,mesh", [
    ("fp32", 10, 0.0, (40, 33, 24)),
    ("mixed", 10, 0.0, (40, 33, 24)),
    ("mixed", 40, 1e-3, (37, 29, 16)),
])
def test_two_processes_classic_equals_loopback_slabs(sten, tmp_path, prec, maxit, tol, mesh, schedule):
    """The headline schedule (Alg. 1 as printed) across two PROCESSES, host
    lockstep.  classic: the halo planes of r, p, v (before H1) and v' (before H2) pushed into the
    neighbour process's buffers through CUDA IPC, the three per-iteration all-reduces through the
    peer-memory inboxes.  classic_fused: no exchange at all - H1 stores its boundary planes of p', v'
    and H3 those of r straight into the neighbour process's halo planes, and the last CTA of every
    phase kernel deposits the slab's sums in both processes' inboxes (fused compute + collective).
    Both bitwise equal to the single-process solve on two loopback slabs with the serial exchange
    (the same kernels, slab sums added in the same order)."""
    nx, ny, nz = mesh
    seed = 6
    res = _run_ranks(tmp_path, 2, prec, maxit, tol, nx, ny, nz, seed, schedule)
    x_ref, it_ref, h_ref, s_ref = _loopback(sten, prec, maxit, tol, nx, ny, nz, seed, 2, "classic")
    for r in res:
        assert int(r["it"]) == it_ref and int(r["status"]) == s_ref
        assert np.array_equal(r["hist"], h_ref)
    x = np.concatenate([r["x"] for r in res], axis=0)
    assert np.array_equal(x, x_ref)
    if tol > 0:
        assert s_ref == sten.CONVERGED and it_ref < maxit and h_ref[-1] <= tol


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("nslabs,mesh", [(2, (40, 33, 24)), (3, (29, 17, 15)), (4, (64, 20, 16))])
def test_classic_fused_loopback_equals_serial(sten, prec, nslabs, mesh):
    """STEN_OPT_CLASSIC_FUSED on loopback slabs (one process): the phase kernels store the boundary
    planes into the neighbour slabs' halo planes and deposit their sums in the inbox slots; bitwise
    equal to the serial exchange (and the fused state survives repeated solves)."""
    torch = torch_cuda()
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=8)
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=8), prec)
    coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
    st = sten.stencil_create(nx, ny, nz, coeffs, nslabs=nslabs)
    bt = to_gpu_vec(b, prec)
    res = {}
    for mode in ("serial", "fused", "fused2"):
        sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, 0)
        sten.set_option(st, sten.OPT_CLASSIC_FUSED, 0 if mode == "serial" else 1)
        xt = torch.empty_like(bt)
        it, hist, status = sten.bicgstab_solve(st, PREC[prec], bt, None, 0.0, 12, xt)
        res[mode] = (from_gpu_vec(xt, prec), it, hist, status)
    for mode in ("fused", "fused2"):
        assert res[mode][1] == res["serial"][1] and res[mode][3] == res["serial"][3]
        assert np.array_equal(res[mode][2], res["serial"][2])
        assert np.array_equal(res[mode][0], res["serial"][0])
    assert sten.get_option(st, sten.OPT_CLASSIC_FUSED) == 1
    st.close()


def test_p2p_only_comm_refuses_what_needs_nccl(sten):
    """A peer-memory-only communicator: create checks the slab convention; a solve before
    sten_p2p_import and the apply are refused (no silent fallback)."""
    torch = torch_cuda()
    nx, ny, nz = 16, 8, 8
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz // 2, seed=3)
    comm = sten.comm_create(None, 2, 0, 0)
    coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
    with pytest.raises(sten.StenError):
        sten.stencil_create(nx, ny, 7, coeffs, comm=comm)  # 7 planes do not split over 2 ranks
    st = sten.stencil_create(nx, ny, nz, coeffs, comm=comm)
    assert st.nz == nz // 2
    b = torch.zeros(nz // 2, ny, nx, dtype=torch.float32, device="cuda")
    x = torch.empty_like(b)
    with pytest.raises(sten.StenError, match="p2p-only"):
        sten.bicgstab_solve(st, sten.FP32, b, None, 0.0, 3, x)  # nothing imported
    with pytest.raises(sten.StenError, match="p2p-only"):
        sten.stencil_apply(st, sten.FP32, b, x)
    st.close()
    comm.close()
    with pytest.raises(sten.StenError):
        sten.comm_create(None, 2, 0, 9999)  # no such device


@pytest.mark.parametrize("schedule", ["sr", "classic_fused"])
@pytest.mark.parametrize("prec", ["fp32", "mixed"])
def test_two_processes_constant_operator(sten, tmp_path, schedule, prec):
    """The constant-coefficient kernels (scalar couplings: k_sr<CC> with its fused halo stores, the classic
    tile kernels' CC + fused instance) across two processes, bitwise the loopback-slab solve."""
    nx, ny, nz = 45, 33, 20
    seed = 7
    res = _run_ranks(tmp_path, 2, prec, 12, 0.0, nx, ny, nz, seed, schedule, "const")
    x_ref, it_ref, h_ref, s_ref = _loopback(sten, prec, 12, 0.0, nx, ny, nz, seed, 2,
                                            "sr" if schedule == "sr" else "classic", "const")
    for r in res:
        assert int(r["it"]) == it_ref and int(r["status"]) == s_ref
        assert np.array_equal(r["hist"], h_ref)
    assert np.array_equal(np.concatenate([r["x"] for r in res], axis=0), x_ref)
