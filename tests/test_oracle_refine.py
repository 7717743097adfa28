"""Pins for the iterative-refinement oracle (oracle.refine16, R21).

Independent references: LAPACK on a dense matrix assembled here, the
identity operator (each step removes the fp16 rounding of the residual, a
factor <= 2^-10), b = 0, and the fp64 solution of the same fp32-quantised
system.
"""
import numpy as np
import pytest

import inputs
from test_oracle_o64 import dense_scaled


@pytest.mark.parametrize("kind,delta", [(inputs.KIND_POISSON, 0.0), (inputs.KIND_CD, 0.1), (inputs.KIND_CD, 0.0)])
@pytest.mark.parametrize("schedule", ["classic", "sr"])
def test_refinement_reaches_fp32_accuracy_vs_lapack(orc, kind, delta, schedule):
    nx = ny = nz = 6
    diag, offs = inputs.problem_fields(kind, nx, ny, nz, seed=2, delta=delta)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=2).astype(np.float32)
    c32 = [a.astype(np.float32).astype(np.float64) for a in c]  # the operator the fp32 residual uses
    M = dense_scaled(None, c32)
    x_lu = np.linalg.solve(M, b.astype(np.float64).ravel())
    res = orc.refine16(c, b, tol=1e-6, outer_maxit=30, inner_tol=1e-2, inner_maxit=60, schedule=schedule)
    assert res["status"] == orc.ORC_CONVERGED
    assert res["hist"][-1] <= 1e-6 and res["hist"][0] == 1.0
    assert np.all(np.diff(res["hist"]) < 0)  # the delta = 0.1 / Poisson classes refine monotonically
    kappa = np.linalg.cond(M)
    err = np.linalg.norm(res["x"].ravel() - x_lu) / np.linalg.norm(x_lu)
    assert err <= 4 * kappa * 1e-6
    # the mixed inner solves alone stall near fp16 resolution; refinement does not
    plain = orc.bicgstab16(orc.quantize_coeffs(c, "mixed"), orc.f16_from_double(b), tol=0.0, maxit=60)
    tr_plain = np.linalg.norm(b.ravel() - M @ orc.f16_to_double(plain["x"]).ravel()) / np.linalg.norm(b)
    assert tr_plain > 1e-5 > res["hist"][-1]


def test_identity_operator_each_step_removes_fp16_rounding(orc):
    rng = np.random.default_rng(3)
    c = [np.zeros((3, 4, 5)) for _ in range(6)]
    b = rng.uniform(-1, 1, (3, 4, 5)).astype(np.float32)
    res = orc.refine16(c, b, tol=1e-7, outer_maxit=10, inner_tol=1e-3, inner_maxit=5)
    assert res["status"] == orc.ORC_CONVERGED
    h = res["hist"]
    assert h[0] == 1.0 and np.all(h[1:] / h[:-1] <= 2.0 ** -10)
    assert np.max(np.abs(res["x"] - b)) <= 1e-7


def test_zero_rhs_and_x0(orc):
    nx, ny, nz = 5, 4, 3
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=4, delta=0.1)
    c = orc.jacobi_scale(diag, offs)
    z = orc.refine16(c, np.zeros((nz, ny, nx), np.float32), x0=np.ones((nz, ny, nx), np.float32))
    assert z["status"] == orc.ORC_CONVERGED and z["outer"] == 0 and not np.any(z["x"])
    b = inputs.rhs_uniform(nx, ny, nz, seed=4).astype(np.float32)
    a = orc.refine16(c, b, tol=1e-6, outer_maxit=20, inner_tol=1e-2)
    x0 = a["x"] + np.float32(1e-3)
    r = orc.refine16(c, b, x0=x0, tol=1e-6, outer_maxit=20, inner_tol=1e-2)
    assert r["status"] == orc.ORC_CONVERGED and r["hist"][0] < 1e-1
    assert np.max(np.abs(r["x"] - a["x"])) <= 1e-5


@pytest.mark.parametrize("kind,delta", [(inputs.KIND_POISSON, 0.0), (inputs.KIND_CD, 0.1), (inputs.KIND_CD, 0.0)])
def test_sr_inner_stagnation_hands_over_to_classic(orc, kind, delta):
    """R21: with an unreachable tol the outer residual settles on the fp32 floor of the system;
    the first stagnation switches the inner schedule (SR -> classic, classic -> SR) instead of
    stopping, and the second stagnation stops (BREAKDOWN).  The handover step is the first one
    ending three steps without a 1% gain on the best residual before them; x stays at LAPACK
    accuracy (4 kappa 1e-6)."""
    nx = ny = nz = 6
    diag, offs = inputs.problem_fields(kind, nx, ny, nz, seed=2, delta=delta)
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=2).astype(np.float32)
    M = dense_scaled(None, [a.astype(np.float32).astype(np.float64) for a in c])
    x_lu = np.linalg.solve(M, b.astype(np.float64).ravel())
    runs = [orc.refine16(c, b, tol=1e-12, outer_maxit=60, inner_tol=1e-2, inner_maxit=60, schedule=s)
            for s in ("classic", "sr")]
    for res in runs:
        assert res["status"] == orc.ORC_BREAKDOWN
        h, k = res["hist"], res["handover"]
        assert 3 <= k <= res["outer"] - 3
        assert np.all(h[k - 2:k + 1] >= 0.99 * np.min(h[:k - 2]))   # three steps without a 1% gain ...
        assert not any(np.all(h[j - 2:j + 1] >= 0.99 * np.min(h[:j - 2])) for j in range(3, k))  # ... first at k
    for res in runs:
        assert res["hist"][-1] <= 2e-7
        err = np.linalg.norm(res["x"].ravel() - x_lu) / np.linalg.norm(x_lu)
        assert err <= 4 * np.linalg.cond(M) * 1e-6


@pytest.mark.parametrize("schedule", ["classic", "sr"])
def test_nonfinite_inner_solve_adds_no_update(orc, schedule):
    """R21: an inner solve that ends NONFINITE (its fp16 scalars overflow, R7) adds nothing to x
    and halves the inner cap.  On an indefinite 6^3 system (couplings about -30 against a unit
    diagonal) the first inner solve, run here directly on r16 = rn16(b_hat / sigma), ends
    NONFINITE within four iterations; the refinement's second residual is then bitwise its first, x stays finite and
    the call ends on stagnation, not NONFINITE."""
    nx = ny = nz = 6
    rng = np.random.default_rng(5)
    diag = np.ones((nz, ny, nx))
    offs = [-30.0 * rng.uniform(0.5, 1.5, (nz, ny, nx)) for _ in range(6)]
    c = orc.jacobi_scale(diag, offs)
    b = inputs.rhs_uniform(nx, ny, nz, seed=2).astype(np.float32)
    sigma = 2.0 ** np.frexp(float(np.max(np.abs(b))))[1]
    d = orc.bicgstab16(orc.quantize_coeffs(c, "mixed"), orc.f16_from_double(b.astype(np.float64) / sigma),
                       tol=1e-2, maxit=64, schedule=schedule)
    assert d["status"] == orc.ORC_NONFINITE
    res = orc.refine16(c, b, tol=1e-6, outer_maxit=20, inner_tol=1e-2, inner_maxit=64, schedule=schedule)
    assert res["hist"][0] == 1.0 and res["hist"][1] == res["hist"][0]
    assert res["status"] == orc.ORC_BREAKDOWN and np.all(np.isfinite(res["x"]))
