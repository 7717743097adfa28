"""Pins for the mixed-precision oracle (O16): fp16 SpMV and the mixed BiCGStab.

References: O64 (itself pinned in test_oracle_o64.py) on IDENTICALLY quantised
inputs, the classical floating-point error bound of a chain of six FMAs, exact
special cases, and the paper's qualitative accuracy result (PAPER.md:586-598,
"Up to iteration 7 the mixed precision implementation tracks the 32-bit, but
then fails to reduce the residual further ... a plateau").
"""
import numpy as np
import pytest

import inputs

U16 = 2.0 ** -11  # unit roundoff of binary16


def setup_mixed(orc, kind, nx, ny, nz, delta=0.1, seed=1):
    diag, offs = inputs.problem_fields(kind, nx, ny, nz, seed=seed, delta=delta)
    c64 = orc.jacobi_scale(diag, offs)
    c16 = orc.quantize_coeffs(c64, "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=seed))
    bh16 = orc.scale_rhs(b16, diag, "mixed")
    cq = [orc.f16_to_double(a) for a in c16]
    return c16, bh16, cq, orc.f16_to_double(bh16)


def neighbour_abs_sum(cq, v):
    """|v_P| + sum_d |c_d v_nb| (test-side, with explicit shifts)."""
    nz, ny, nx = v.shape
    pad = np.zeros((nz + 2, ny + 2, nx + 2))
    pad[1:-1, 1:-1, 1:-1] = v
    nbs = [pad[1:-1, 1:-1, :-2], pad[1:-1, 1:-1, 2:], pad[1:-1, :-2, 1:-1], pad[1:-1, 2:, 1:-1],
           pad[:-2, 1:-1, 1:-1], pad[2:, 1:-1, 1:-1]]
    return np.abs(v) + sum(np.abs(c) * np.abs(nb) for c, nb in zip(cq, nbs))


@pytest.mark.parametrize("unfused", [False, True])
def test_spmv16_error_bound_vs_o64(orc, unfused):
    nx, ny, nz = 40, 33, 24
    c16, _, cq, _ = setup_mixed(orc, inputs.KIND_CD, nx, ny, nz, delta=0.0, seed=3)
    rng = np.random.default_rng(3)
    v16 = orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    vq = orc.f16_to_double(v16)
    u16 = orc.f16_to_double(orc.apply16(c16, v16, unfused=unfused))
    u64 = orc.apply64(cq, vq)
    err = np.abs(u16 - u64)
    # fused: 6 roundings of partial sums; unfused: 6 products + 6 sums
    k = 7 if not unfused else 13
    assert np.all(err <= k * U16 * neighbour_abs_sum(cq, vq))
    # north_star metric (R9): max|du| / max|u| <= 2e-3
    assert err.max() / np.abs(u64).max() <= 2e-3


def test_spmv16_identity_and_exactness(orc):
    rng = np.random.default_rng(4)
    v16 = orc.f16_from_double(rng.uniform(-1, 1, (3, 4, 5)))
    zeros = [np.zeros((3, 4, 5), np.uint16) for _ in range(6)]
    assert np.array_equal(orc.apply16(zeros, v16), v16)
    # small-integer data: every partial sum exact in fp16 -> equals O64 exactly
    c = [np.full((3, 4, 5), 0x3C00, np.uint16) for _ in range(6)]  # all couplings 1
    vi = orc.f16_from_double(rng.integers(-8, 8, (3, 4, 5)).astype(np.float64))
    cq = [orc.f16_to_double(a) for a in c]
    assert np.array_equal(orc.f16_to_double(orc.apply16(c, vi)), orc.apply64(cq, orc.f16_to_double(vi)))


def test_dot16_exact_for_representable_sums(orc):
    # fp16-exact data with an exactly representable fp32 sum == fp64
    rng = np.random.default_rng(5)
    a = orc.f16_from_double(rng.integers(-64, 64, (6, 5, 7)).astype(np.float64))
    b = orc.f16_from_double(rng.integers(-64, 64, (6, 5, 7)).astype(np.float64))
    assert orc.dot16(a, b) == float(np.sum(orc.f16_to_double(a) * orc.f16_to_double(b)))


def test_mixed_identity_converges_in_one(orc):
    rng = np.random.default_rng(6)
    c = [np.zeros((3, 4, 5), np.uint16) for _ in range(6)]
    b = orc.f16_from_double(rng.uniform(-1, 1, (3, 4, 5)))
    res = orc.bicgstab16(c, b, tol=1e-3, maxit=5)
    assert res["iters"] == 1 and res["status"] == orc.ORC_CONVERGED
    assert np.array_equal(res["x"], b)


def test_mixed_tracks_fp64_early(orc):
    c16, b16, cq, bq = setup_mixed(orc, inputs.KIND_CD, 20, 40, 20, delta=0.0)
    h16 = orc.bicgstab16(c16, b16, tol=0.0, maxit=6)["hist"]
    h64 = orc.bicgstab64(cq, bq, tol=0.0, maxit=6)["hist"]
    assert np.all(np.abs(h16 - h64) <= 0.05 * h64)


def test_mixed_plateau_while_fp64_converges(orc):
    # PAPER.md:591-592 on a synthetic stand-in (SPEC.md:600 class 20x40x20, delta=0)
    c16, b16, cq, bq = setup_mixed(orc, inputs.KIND_CD, 20, 40, 20, delta=0.0)
    r64 = orc.bicgstab64(cq, bq, tol=1e-6, maxit=200)
    assert r64["status"] == orc.ORC_CONVERGED
    for it in (20, 40):
        x16 = orc.bicgstab16(c16, b16, tol=0.0, maxit=it)["x"]
        tr = orc.true_residual64(cq, bq, orc.f16_to_double(x16))
        assert 1e-3 <= tr <= 1e-1, (it, tr)


def test_mixed_reaches_1e3_with_margin(orc):
    # north_star: mixed reaches a relative residual of 1e-3 (recurrence, R13)
    c16, b16, cq, bq = setup_mixed(orc, inputs.KIND_CD, 32, 32, 32, delta=0.1)
    res = orc.bicgstab16(c16, b16, tol=1e-3, maxit=200)
    assert res["status"] == orc.ORC_CONVERGED and res["iters"] <= 15


def test_fused_and_unfused_plateaus_agree(orc):
    c16, b16, cq, bq = setup_mixed(orc, inputs.KIND_CD, 24, 24, 24, delta=0.1)
    tr = []
    for unf in (False, True):
        x16 = orc.bicgstab16(c16, b16, tol=0.0, maxit=20, unfused=unf)["x"]
        tr.append(orc.true_residual64(cq, bq, orc.f16_to_double(x16)))
    assert 0.5 <= tr[0] / tr[1] <= 2.0


def test_spmv32_mirror_vs_o64(orc):
    nx, ny, nz = 17, 9, 11
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=8)
    c64 = orc.jacobi_scale(diag, offs)
    c32 = orc.quantize_coeffs(c64, "fp32")
    rng = np.random.default_rng(8)
    v32 = rng.uniform(-1, 1, (nz, ny, nx)).astype(np.float32)
    u32 = orc.apply32_fma(c32, v32).astype(np.float64)
    cq = [a.astype(np.float64) for a in c32]
    u64 = orc.apply64(cq, v32.astype(np.float64))
    assert np.all(np.abs(u32 - u64) <= 7 * 2.0 ** -24 * neighbour_abs_sum(cq, v32.astype(np.float64)))
    assert np.max(np.abs(u32 - u64)) / np.max(np.abs(u64)) <= 1e-6
