"""World-size-2 `gloo` tests of the multi-rank path on CPU (no GPU here).

1. Host plumbing: slab bounds, unique-id bootstrap, max-over-ranks timing.
2. The decomposition itself: a z-slab BiCGStab in fp64 across 2 processes, with
   halo planes exchanged by gloo send/recv and dot sums all-reduced, matches the
   monolithic oracle (O64).  This is the scheme libsten runs over NCCL
   (DESIGN.md §6): per-rank slabs of the global generator, halo planes of the
   SpMV input before each SpMV, one all-reduce per group of dots.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _plumbing_worker(rank, world, port, q):
    dist = _init(rank, world, port)
    from paper_2010_03660_b200 import dist as sd
    import paper_2010_03660_b200 as sten
    out = {"env": sd.rank_env(), "slab": sd.slab_of(rank, world, 1536 * world), "nb": sd.neighbours(rank, world)}
    try:
        uid = sd.broadcast_bytes(sten.comm_unique_id() if rank == 0 else None)
        out["uid"] = uid
    except Exception as e:  # libnccl missing on a CPU box: the bootstrap plumbing still works
        out["uid"] = sd.broadcast_bytes(bytes([7]) * 128 if rank == 0 else None)
        out["uid_note"] = str(e)
    out["max"] = sd.max_over_ranks(10.0 + rank)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_host_plumbing_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_plumbing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0]["slab"] == (0, 1536) and res[1]["slab"] == (1536, 1536)
    assert res[0]["nb"] == (None, 1) and res[1]["nb"] == (0, None)
    assert res[0]["uid"] == res[1]["uid"] and len(res[0]["uid"]) == 128
    assert res[0]["max"] == res[1]["max"] == 11.0


def _slab_solver_worker(rank, world, port, q, mesh, maxit):
    dist = _init(rank, world, port)
    import torch
    import oracle as orc
    from paper_2010_03660_b200 import dist as sd
    nx, ny, nz = mesh
    z0, nzl = sd.slab_of(rank, world, nz)
    below, above = sd.neighbours(rank, world)
    # this rank's planes of the global problem, from the generator's global index
    lo, hi = max(z0 - 1, 0), min(z0 + nzl + 1, nz)
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, hi - lo, z0=lo, seed=5, delta=0.0)
    cext = orc.jacobi_scale(diag, offs)  # couplings inside [lo, hi) kept; true mesh ends dropped
    c = [a[z0 - lo: z0 - lo + nzl] for a in cext]
    b = inputs.rhs_uniform(nx, ny, nzl, z0=z0, seed=5) / diag[z0 - lo: z0 - lo + nzl]

    def halo(v):  # one plane to/from each z-neighbour (gloo send/recv)
        ext = np.zeros((nzl + 2, ny, nx))
        ext[1:-1] = v
        reqs = []
        bot_in, top_in = torch.zeros(ny, nx, dtype=torch.float64), torch.zeros(ny, nx, dtype=torch.float64)
        if below is not None:
            reqs += [dist.isend(torch.from_numpy(v[0].copy()), below), dist.irecv(bot_in, below)]
        if above is not None:
            reqs += [dist.isend(torch.from_numpy(v[-1].copy()), above), dist.irecv(top_in, above)]
        for r in reqs:
            r.wait()
        ext[0], ext[-1] = bot_in.numpy(), top_in.numpy()
        return ext

    def apply(v):  # unit-diagonal SpMV of the slab, neighbours from the halo'd copy
        e = halo(v)
        u = v.copy()
        u[:, :, 1:] += c[0][:, :, 1:] * v[:, :, :-1]
        u[:, :, :-1] += c[1][:, :, :-1] * v[:, :, 1:]
        u[:, 1:, :] += c[2][:, 1:, :] * v[:, :-1, :]
        u[:, :-1, :] += c[3][:, :-1, :] * v[:, 1:, :]
        u += c[4] * e[:-2]
        u += c[5] * e[2:]
        return u

    def allsum(*vals):  # the scalar all-reduce of one phase
        t = torch.tensor(vals, dtype=torch.float64)
        dist.all_reduce(t)
        return t.numpy()

    x = np.zeros_like(b)
    r = b.copy()
    rh, p = r.copy(), r.copy()
    rho, bb = allsum(np.sum(rh * r), np.sum(b * b))
    nb = np.sqrt(bb)
    hist = [np.sqrt(allsum(np.sum(r * r))[0]) / nb]
    v = np.zeros_like(b)
    beta = omega = 0.0
    for i in range(1, maxit + 1):
        if i > 1:
            p = r + beta * (p - omega * v)
        v = apply(p)
        alpha = rho / allsum(np.sum(rh * v))[0]
        s = r - alpha * v
        t = apply(s)
        ts, tt = allsum(np.sum(t * s), np.sum(t * t))
        omega = ts / tt
        x = (x + alpha * p) + omega * s
        r = s - omega * t
        rhon, rr = allsum(np.sum(rh * r), np.sum(r * r))
        hist.append(np.sqrt(rr) / nb)
        beta = (rhon / rho) * (alpha / omega)
        rho = rhon
    q.put((rank, z0, x, np.array(hist)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_decomposed_bicgstab_matches_monolithic_oracle(orc, world):
    mesh, maxit = (9, 7, 12), 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_slab_solver_worker, args=(r, world, port, q, mesh, maxit)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=180) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.concatenate([r[2] for r in res])
    nx, ny, nz = mesh
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=5, delta=0.0)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=5) / diag
    ref = orc.bicgstab64(c, b, tol=0.0, maxit=maxit)
    assert np.allclose(res[0][3], res[1][3], rtol=0, atol=0)  # every rank sees the same scalars
    assert np.all(np.abs(res[0][3] - ref["hist"]) <= 1e-10 * ref["hist"])
    assert np.linalg.norm(x - ref["x"]) / np.linalg.norm(ref["x"]) <= 1e-10
