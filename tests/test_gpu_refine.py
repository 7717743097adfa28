"""GPU parity of the mixed-precision iterative refinement (bicgstab_refine, R21)
against the oracle (oracle.refine16): the same outer residual sequence within
the inner solves' rounding, fp32-level final accuracy, and the edge cases."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import fields, gpu_stencil, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def _refine(sten, st, b32, tol, outer, inner_tol, inner_maxit, x0=None, schedule=0):
    torch = torch_cuda()
    sten.set_schedule(st, schedule)
    bt = torch.from_numpy(np.ascontiguousarray(b32)).cuda()
    xt = torch.empty_like(bt)
    x0t = None if x0 is None else torch.from_numpy(np.ascontiguousarray(x0)).cuda()
    ko, ki, hist, status = sten.bicgstab_refine(st, bt, x0t, tol, outer, inner_tol, inner_maxit, xt)
    return xt.cpu().numpy(), ko, ki, hist, status


@pytest.mark.parametrize("schedule", [0, 1])
@pytest.mark.parametrize("mesh,delta", [((32, 32, 32), 0.1), ((40, 24, 18), 0.0), ((64, 64, 64), 0.1)])
def test_refinement_vs_oracle(sten, schedule, mesh, delta):
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=delta, seed=3)
    b = inputs.rhs_uniform(nx, ny, nz, seed=3).astype(np.float32)
    st = gpu_stencil(diag, offs)
    x, ko, ki, hist, status = _refine(sten, st, b, 1e-6, 30, 1e-2, 200, schedule=schedule)
    c64 = orc.jacobi_scale(diag, offs)
    bh = orc.scale_rhs(b, diag, "fp32")
    ref = orc.refine16(c64, bh, tol=1e-6, outer_maxit=30, inner_tol=1e-2, inner_maxit=200,
                       schedule="sr" if schedule else "classic")
    assert status == sten.CONVERGED == ref["status"]
    assert hist[-1] <= 1e-6 and abs(ko - ref["outer"]) <= 1
    # outer residuals: the first step is b_hat itself; each later one is set by
    # an inner solve stopped at 1e-2, whose rounding differs in the last bits
    assert hist[0] == pytest.approx(1.0, rel=1e-6)
    n = min(len(hist), len(ref["hist"])) - 1
    assert np.all(np.abs(np.log10(hist[1:n]) - np.log10(ref["hist"][1:n])) <= 0.5)
    c32 = [a.astype(np.float32).astype(np.float64) for a in c64]
    tr = orc.true_residual64(c32, bh.astype(np.float64), x.astype(np.float64))
    assert tr <= 2e-6
    assert np.linalg.norm(x - ref["x"]) <= 1e-4 * np.linalg.norm(ref["x"])
    st.close()


def test_refinement_edge_cases(sten):
    nx, ny, nz = 20, 12, 10
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=5)
    st = gpu_stencil(diag, offs)
    z = np.zeros((nz, ny, nx), np.float32)
    x, ko, ki, hist, status = _refine(sten, st, z, 1e-6, 10, 1e-2, 50, x0=np.ones_like(z))
    assert status == sten.CONVERGED and ko == 0 and not np.any(x)
    b = inputs.rhs_uniform(nx, ny, nz, seed=5).astype(np.float32)
    x1, ko1, _, h1, s1 = _refine(sten, st, b, 1e-6, 20, 1e-2, 50)
    x2, ko2, _, h2, s2 = _refine(sten, st, b, 1e-6, 20, 1e-2, 50, x0=x1 + np.float32(1e-3))
    assert s1 == s2 == sten.CONVERGED and h2[0] < 1e-1
    assert np.max(np.abs(x2 - x1)) <= 1e-5
    # outer_maxit = 0: only the initial residual
    x3, ko3, _, h3, s3 = _refine(sten, st, b, 1e-6, 0, 1e-2, 50)
    assert ko3 == 0 and s3 == sten.MAXIT and h3[0] == pytest.approx(1.0) and not np.any(x3)
    with pytest.raises(sten.StenError):
        _refine(sten, st, b, 0.0, 5, 1e-2, 50)
    st.close()


@pytest.mark.parametrize("schedule", [0, 1])
def test_refinement_slab_decomposed(sten, schedule):
    nx, ny, nz = 33, 21, 32
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=6)
    b = inputs.rhs_uniform(nx, ny, nz, seed=6).astype(np.float32)
    st1 = gpu_stencil(diag, offs)
    x1, ko1, _, h1, s1 = _refine(sten, st1, b, 1e-6, 20, 1e-2, 100, schedule=schedule)
    st2 = gpu_stencil(diag, offs, nslabs=4)
    x2, ko2, _, h2, s2 = _refine(sten, st2, b, 1e-6, 20, 1e-2, 100, schedule=schedule)
    assert s1 == s2 == sten.CONVERGED and abs(ko1 - ko2) <= 1
    assert np.linalg.norm(x2 - x1) <= 1e-5 * np.linalg.norm(x1)
    st1.close()
    st2.close()


@pytest.mark.parametrize("delta", [0.1, 0.0])
def test_sr_inner_stagnation_hands_over_to_classic(sten, delta):
    """R21 handover: with an unreachable tol the outer residual settles on the fp32 floor; the first
    stagnation switches the inner schedule (SR <-> classic; sten_stats.handover = that outer step)
    and the second stops with BREAKDOWN, as oracle.refine16 does."""
    nx, ny, nz = 40, 24, 18
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=delta, seed=3)
    b = inputs.rhs_uniform(nx, ny, nz, seed=3).astype(np.float32)
    st = gpu_stencil(diag, offs)
    c64 = orc.jacobi_scale(diag, offs)
    bh = orc.scale_rhs(b, diag, "fp32")
    c32 = [a.astype(np.float32).astype(np.float64) for a in c64]
    for schedule in (0, 1):
        x, ko, ki, hist, status = _refine(sten, st, b, 1e-12, 60, 1e-2, 200, schedule=schedule)
        ref = orc.refine16(c64, bh, tol=1e-12, outer_maxit=60, inner_tol=1e-2, inner_maxit=200,
                           schedule="sr" if schedule else "classic")
        k = sten.get_stats(st)["handover"]
        assert status == sten.BREAKDOWN == ref["status"]
        assert k >= 3 and ref["handover"] >= 3 and ko >= k + 3
        assert np.all(hist[k - 2:k + 1] >= 0.99 * np.min(hist[:k - 2]))
        assert hist[-1] <= 3e-7
        assert orc.true_residual64(c32, bh.astype(np.float64), x.astype(np.float64)) <= 3e-7
    st.close()


@pytest.mark.parametrize("schedule", [0, 1])
def test_nonfinite_inner_solve_adds_no_update(sten, schedule):
    """R21: an inner solve that ends NONFINITE adds nothing to x and halves the inner cap, as
    oracle.refine16 does (tests/test_oracle_refine.py: the same indefinite 6^3 system, whose first
    inner solve overflows within four iterations, early enough for both dot orders): the second outer residual is bitwise the first, x stays finite, the
    call ends on stagnation (BREAKDOWN) like the oracle's."""
    nx = ny = nz = 6
    rng = np.random.default_rng(5)
    diag = np.ones((nz, ny, nx))
    offs = [-30.0 * rng.uniform(0.5, 1.5, (nz, ny, nx)) for _ in range(6)]
    b = inputs.rhs_uniform(nx, ny, nz, seed=2).astype(np.float32)
    st = gpu_stencil(diag, offs)
    x, ko, ki, hist, status = _refine(sten, st, b, 1e-6, 20, 1e-2, 64, schedule=schedule)
    ref = orc.refine16(orc.jacobi_scale(diag, offs), b, tol=1e-6, outer_maxit=20, inner_tol=1e-2, inner_maxit=64,
                       schedule="sr" if schedule else "classic")
    assert ref["hist"][1] == ref["hist"][0]
    assert hist[0] == pytest.approx(1.0, rel=1e-6) and hist[1] == hist[0]
    assert status == sten.BREAKDOWN == ref["status"] and np.all(np.isfinite(x))
    st.close()
