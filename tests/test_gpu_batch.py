"""bicgstab_solve_batch: n independent solves with pipelined host<->device copies
(include/sten.h).  Every system's x, history, iteration count and status must be
bitwise what bicgstab_solve gives for it alone, for pinned-host, pageable-host and
device vectors, both schedules and both precisions, with a tolerance stop that
ends the systems at different iterations."""
import numpy as np
import pytest

import inputs
from gpu_util import fields, gpu_stencil, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def _rhs(torch, n, shape, prec, seed):
    out = []
    for i in range(n):
        b = torch.from_numpy(inputs.rhs_uniform(shape[2], shape[1], shape[0], seed=seed + i)).float()
        out.append(b.half() if prec == 1 else b)
    return out


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("sched", [0, 1])
@pytest.mark.parametrize("where", ["pinned", "pageable", "device", "mixed"])
def test_batch_equals_single_solves(sten, prec, sched, where):
    torch = torch_cuda()
    nx, ny, nz = 45, 33, 20
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=4)
    st = gpu_stencil(diag, offs)
    sten.set_schedule(st, sched)
    tol, maxit = (1e-5, 60) if prec == 0 else (1e-3, 40)
    bs = _rhs(torch, 3, (nz, ny, nx), prec, seed=11)
    bs[1] = bs[1] * 0.5 + 0.25  # a different convergence path
    ref = []
    for b in bs:
        x = torch.empty_like(b).cuda()
        ref.append((*sten.bicgstab_solve(st, prec, b.cuda(), None, tol, maxit, x), x.cpu()))

    def place(t, i):
        mode = where if where != "mixed" else ("pinned", "device", "pageable")[i % 3]
        return t.pin_memory() if mode == "pinned" else (t.cuda() if mode == "device" else t.clone())
    bb = [place(b, i) for i, b in enumerate(bs)]
    xs = [place(torch.empty_like(b), i + 1) for i, b in enumerate(bs)]
    got = sten.bicgstab_solve_batch(st, prec, bb, xs, tol, maxit)
    for (it, h, stt), (rit, rh, rst, rx), x in zip(got, ref, xs):
        assert it == rit and stt == rst and np.array_equal(h, rh)
        assert torch.equal(x.cpu(), rx)
    st.close()


def test_batch_edge_cases(sten):
    torch = torch_cuda()
    diag, offs = fields(inputs.KIND_CD, 16, 8, 6)
    st = gpu_stencil(diag, offs)
    assert sten.bicgstab_solve_batch(st, 0, [], [], 0.0, 5) == []
    b = torch.zeros(6, 8, 16, dtype=torch.float32).pin_memory()
    x = torch.full_like(b, 7.0).pin_memory()
    (it, h, status), = sten.bicgstab_solve_batch(st, 0, [b], [x], 1e-6, 5)
    assert it == 0 and status == sten.CONVERGED and not torch.any(x)
    with pytest.raises(sten.StenError):
        sten.bicgstab_solve_batch(st, 0, [b], [x], -1.0, 5)
    with pytest.raises(sten.StenError):
        sten.bicgstab_solve_batch(st, 0, [b, b], [x], 0.0, 5)
    # maxit iterations exactly in benchmark mode, history NaN-free up to it
    b1 = torch.from_numpy(inputs.rhs_uniform(16, 8, 6, seed=2)).float().pin_memory()
    (it, h, status), (it2, h2, _) = sten.bicgstab_solve_batch(st, 0, [b1, b1], [x, torch.empty_like(x)], 0.0, 7)
    assert it == it2 == 7 and np.all(np.isfinite(h)) and np.array_equal(h, h2)
    st.close()


def test_quickstart_example_runs():
    """examples/quickstart.py (the user-facing walk-through) runs and reaches its targets."""
    import importlib.util
    import os
    torch_cuda()
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples", "quickstart.py")
    spec = importlib.util.spec_from_file_location("quickstart", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    h_mixed, h_refine, true = mod.main(64, 48, 32)
    assert h_mixed <= 1e-3 and h_refine <= 1e-6 and true <= 1e-5
