"""Pins for the fp64 oracle (O64): Jacobi scaling, SpMV, BiCGStab.

Independent references only: a dense matrix assembled HERE by explicit
neighbour enumeration, numpy.linalg.solve (LAPACK) for exact solves, closed-
form Poisson eigenpairs, Krylov finite-termination theory, and the
true-vs-recurrence residual invariant.
"""
import numpy as np
import pytest

import inputs

DIRS = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]  # xm xp ym yp zm zp


def dense_scaled(diag, offs):
    """D^-1 A assembled entry by entry (test-side, no oracle code)."""
    nz, ny, nx = offs[0].shape
    n = nx * ny * nz
    M = np.zeros((n, n))
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                P = i + nx * (j + ny * k)
                M[P, P] = 1.0
                for d, (dx, dy, dz) in enumerate(DIRS):
                    ii, jj, kk = i + dx, j + dy, k + dz
                    if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                        Q = ii + nx * (jj + ny * kk)
                        M[P, Q] += offs[d][k, j, i] / (diag[k, j, i] if diag is not None else 1.0)
    return M


def random_fields(rng, nx, ny, nz):
    diag = rng.uniform(1.0, 3.0, (nz, ny, nx))
    offs = [rng.uniform(-1.0, 1.0, (nz, ny, nx)) for _ in range(6)]
    return diag, offs


MESHES = [(1, 1, 1), (1, 1, 2), (2, 1, 1), (1, 3, 1), (3, 4, 5), (8, 8, 8), (5, 2, 7)]


@pytest.mark.parametrize("mesh", MESHES)
def test_apply_matches_dense_assembly(orc, mesh):
    nx, ny, nz = mesh
    rng = np.random.default_rng(nx * 100 + ny * 10 + nz)
    diag, offs = random_fields(rng, nx, ny, nz)
    c = orc.jacobi_scale(diag, offs)
    M = dense_scaled(diag, offs)
    v = rng.uniform(-1, 1, (nz, ny, nx))
    u = orc.apply64(c, v)
    ref = M @ v.ravel()
    scale = np.abs(M) @ np.abs(v.ravel())
    assert np.all(np.abs(u.ravel() - ref) <= 1e-15 * 8 * scale + 1e-300)
    # scaled couplings are exactly off/diag in-mesh and +0 outside
    for d, (dx, dy, dz) in enumerate(DIRS):
        for k in range(nz):
            for j in range(ny):
                for i in range(nx):
                    inside = 0 <= i + dx < nx and 0 <= j + dy < ny and 0 <= k + dz < nz
                    want = offs[d][k, j, i] / diag[k, j, i] if inside else 0.0
                    assert c[d][k, j, i] == want


def test_zero_couplings_identity(orc):
    # all six couplings zero -> SpMV is the identity, bitwise
    rng = np.random.default_rng(5)
    c = [np.zeros((4, 3, 5)) for _ in range(6)]
    v = rng.uniform(-1, 1, (4, 3, 5))
    assert np.array_equal(orc.apply64(c, v), v)


def test_column_of_A_on_1x1x4(orc):
    # u = A e_j is column j of A
    rng = np.random.default_rng(6)
    diag, offs = random_fields(rng, 1, 1, 4)
    c = orc.jacobi_scale(diag, offs)
    M = dense_scaled(diag, offs)
    for jcol in range(4):
        e = np.zeros((4, 1, 1))
        e[jcol] = 1.0
        assert np.allclose(orc.apply64(c, e).ravel(), M[:, jcol], rtol=0, atol=1e-16)


def poisson_scaled(orc, nx, ny, nz):
    diag, offs = inputs.problem_fields(inputs.KIND_POISSON, nx, ny, nz)
    return orc.jacobi_scale(diag, offs)


def phi(nx, ny, nz, a, b, cc):
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (np.sin(a * np.pi * (i + 1) / (nx + 1)) * np.sin(b * np.pi * (j + 1) / (ny + 1))
            * np.sin(cc * np.pi * (k + 1) / (nz + 1)))


def lam(nx, ny, nz, a, b, cc):
    return 1.0 - (np.cos(a * np.pi / (nx + 1)) + np.cos(b * np.pi / (ny + 1)) + np.cos(cc * np.pi / (nz + 1))) / 3.0


@pytest.mark.parametrize("abc", [(1, 1, 1), (2, 3, 1), (5, 1, 4)])
def test_poisson_eigenvectors(orc, abc):
    nx, ny, nz = 9, 7, 6
    c = poisson_scaled(orc, nx, ny, nz)
    f = phi(nx, ny, nz, *abc)
    assert np.max(np.abs(orc.apply64(c, f) - lam(nx, ny, nz, *abc) * f)) <= 1e-14


@pytest.mark.parametrize("kind,delta", [(inputs.KIND_POISSON, 0.0), (inputs.KIND_CD, 0.1), (inputs.KIND_CD, 0.0)])
def test_solve_matches_dense_lu(orc, kind, delta):
    nx = ny = nz = 6
    diag, offs = inputs.problem_fields(kind, nx, ny, nz, seed=2, delta=delta)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=2)
    M = dense_scaled(diag, offs)
    x_lu = np.linalg.solve(M, b.ravel())
    res = orc.bicgstab64(c, b, tol=1e-13, maxit=500)
    assert res["status"] == orc.ORC_CONVERGED
    assert np.linalg.norm(res["x"].ravel() - x_lu) / np.linalg.norm(x_lu) <= 1e-10
    # the recurrence history is non-increasing "on average": final < first
    assert res["hist"][-1] <= 1e-13 < res["hist"][0]


def test_hand_lu_agrees_with_lapack():
    # an independent partial-pivot LU written here, as a second reference
    rng = np.random.default_rng(9)
    A = rng.uniform(-1, 1, (30, 30)) + 8 * np.eye(30)
    b = rng.uniform(-1, 1, 30)
    M = A.copy()
    y = b.copy()
    n = 30
    for kcol in range(n):
        piv = kcol + np.argmax(np.abs(M[kcol:, kcol]))
        M[[kcol, piv]] = M[[piv, kcol]]
        y[[kcol, piv]] = y[[piv, kcol]]
        for r in range(kcol + 1, n):
            f = M[r, kcol] / M[kcol, kcol]
            M[r, kcol:] -= f * M[kcol, kcol:]
            y[r] -= f * y[kcol]
    x = np.zeros(n)
    for r in range(n - 1, -1, -1):
        x[r] = (y[r] - M[r, r + 1:] @ x[r + 1:]) / M[r, r]
    assert np.allclose(x, np.linalg.solve(A, b), rtol=1e-12, atol=1e-14)


def test_krylov_termination_one_eigenvector(orc):
    nx, ny, nz = 7, 6, 5
    c = poisson_scaled(orc, nx, ny, nz)
    f = phi(nx, ny, nz, 1, 1, 1)
    res = orc.bicgstab64(c, f, tol=0.0, maxit=1)
    assert res["hist"][1] <= 1e-14
    assert np.max(np.abs(res["x"] - f / lam(nx, ny, nz, 1, 1, 1))) <= 1e-13


def test_krylov_termination_two_eigenvectors(orc):
    # r0 in a 2-D invariant subspace -> BiCG (=CG here, symmetric, rhat=r0)
    # terminates at step 2; BiCGStab's s-step keeps the residual in that space
    nx, ny, nz = 7, 6, 5
    c = poisson_scaled(orc, nx, ny, nz)
    f = phi(nx, ny, nz, 1, 1, 1) + 0.7 * phi(nx, ny, nz, 2, 1, 3)
    res = orc.bicgstab64(c, f, tol=0.0, maxit=2)
    assert res["hist"][2] <= 1e-13
    assert res["hist"][1] > 1e-6


def test_identity_lucky_exit(orc):
    # A = I converges after one iteration with x = b exactly
    rng = np.random.default_rng(11)
    c = [np.zeros((3, 4, 5)) for _ in range(6)]
    b = rng.uniform(-1, 1, (3, 4, 5))
    res = orc.bicgstab64(c, b, tol=1e-12, maxit=10)
    assert res["iters"] == 1 and res["status"] == orc.ORC_CONVERGED
    assert np.array_equal(res["x"], b)
    assert res["hist"][1] == 0.0


def test_two_unknown_upper_triangular(orc):
    # mesh (1,1,2), c_zp[0] = 0.5, c_zm[1] = 0, b = (1,1) -> x = (0.5, 1)
    c = [np.zeros((2, 1, 1)) for _ in range(6)]
    c[5][0, 0, 0] = 0.5
    b = np.ones((2, 1, 1))
    res = orc.bicgstab64(c, b, tol=1e-14, maxit=10)
    assert res["status"] == orc.ORC_CONVERGED
    assert np.allclose(res["x"].ravel(), [0.5, 1.0], rtol=0, atol=1e-14)


def test_x0_nonzero_reduces_to_same_solution(orc):
    nx, ny, nz = 5, 5, 5
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=4)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=4)
    x0 = inputs.rhs_uniform(nx, ny, nz, seed=5)
    r1 = orc.bicgstab64(c, b, tol=1e-12, maxit=200)
    r2 = orc.bicgstab64(c, b, x0=x0, tol=1e-12, maxit=200)
    assert np.allclose(r1["x"], r2["x"], rtol=0, atol=1e-10)
    # hist[0] refers to r0 = b - A x0 (R1)
    assert abs(r2["hist"][0] - orc.true_residual64(c, b, x0)) <= 1e-14


def test_manufactured_config1(orc):
    # BASELINE.json config 1: 32^3 Poisson, x_true ~ U(-1,1), b = A x_true, tol 1e-6
    n = 32
    diag, offs = inputs.problem_fields(inputs.KIND_POISSON, n, n, n)
    c = orc.jacobi_scale(diag, offs)
    xt = inputs.rhs_uniform(n, n, n, seed=1)
    b = orc.apply_raw64(diag, offs, xt)
    bh = b / diag  # scaled right-hand side (R3)
    res = orc.bicgstab64(c, bh, tol=1e-6, maxit=200)
    assert res["status"] == orc.ORC_CONVERGED
    assert 40 <= res["iters"] <= 120
    kappa = (1 - np.cos(np.pi / 33)) ** -1 * (1 + np.cos(np.pi / 33))  # lmax/lmin of D^-1 A
    err = np.linalg.norm(res["x"] - xt) / np.linalg.norm(xt)
    assert err <= kappa * 1e-6


def test_true_vs_recurrence_residual_invariant(orc):
    # for >= 20 fp64 iterations, recurrence and true residual agree
    nx, ny, nz = 10, 9, 8
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=7, delta=0.0)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=7)
    for it in (1, 5, 20, 35):
        res = orc.bicgstab64(c, b, tol=0.0, maxit=it)
        tr = orc.true_residual64(c, b, res["x"])
        assert abs(tr - res["hist"][it]) <= 1e-10


def test_convergence_sanity_many_seeds(orc):
    # SPEC.md:456-style sanity: the cd(delta=0.1) class converges for every seed
    nx, ny, nz = 8, 7, 6
    for seed in range(1, 21):
        diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=seed, delta=0.1)
        c = orc.jacobi_scale(diag, offs)
        b = inputs.rhs_uniform(nx, ny, nz, seed=seed)
        res = orc.bicgstab64(c, b, tol=1e-8, maxit=100)
        assert res["status"] == orc.ORC_CONVERGED, seed
        assert orc.true_residual64(c, b, res["x"]) <= 1e-7


def test_benchmark_mode_runs_exactly_maxit(orc):
    nx, ny, nz = 6, 6, 6
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=1)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=1)
    res = orc.bicgstab64(c, b, tol=0.0, maxit=30)
    assert res["iters"] == 30
    assert np.all(np.isfinite(res["hist"]))


def test_flop_accounting_matches_paper_table():
    # PAPER.md:399-417 Table "Operations per meshpoint per iteration"
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))
    t = g["ops_table"]
    sp = sum(r["sp_add"] + r["sp_mul"] for r in t["rows"])
    mixed16 = sum(r["hp_add"] + r["hp_mul"] for r in t["rows"])
    mixed32 = sum(r["sp_add_mixed"] for r in t["rows"])
    assert sp == 44 and mixed16 == 40 and mixed32 == 4
    from paper_2010_03660_b200.roofline import FLOPS_PER_POINT_ITER, PHASE_FLOPS
    assert FLOPS_PER_POINT_ITER == sp == sum(PHASE_FLOPS.values())
    # 44 * 600*595*1536 / 28.1us = 0.86 PFLOPS
    m = g["measured"]
    pf = FLOPS_PER_POINT_ITER * m["nx"] * m["ny"] * m["nz"] / (m["us_per_iter"] * 1e-6) / 1e15
    assert round(pf, 2) == m["pflops"]
    # 10Z words of fp16 at Z = 1536 "about 31KB out of 48KB"
    assert round(10 * 1536 * 2 / 1000) == g["storage"]["kb_used"]
