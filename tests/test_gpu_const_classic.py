"""The classic schedule (Alg. 1) on a constant-coefficient operator
(stencil_create_const: "no coefficient streams: 17 instead of 29
passes").  The tile kernels then take the six scaled couplings as scalars
(STEN_OPT_CLASSIC_CONST = 1, the default) and must give what the array kernels give on
the same handle (option 0) - bitwise on widened values, so +0 == -0 - and what the
oracle gives: the SpMV bitwise against apply16 / apply32_fma on the constant fields
(R5: couplings leaving the mesh dropped), the solve's history against O16 / O64."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import from_gpu_vec, quantize_vec, to_gpu_vec, torch_cuda, widen

pytestmark = pytest.mark.gpu
PREC = {"fp32": 0, "mixed": 1}
POISSON = (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0)
SKEW = (3.0, -0.7, -0.4, -0.25, -0.55, -0.3, -0.5)  # nonsymmetric constant operator


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def const_coeffs(c, nx, ny, nz, prec):
    diag = np.full((nz, ny, nx), c[0])
    offs = [np.full((nz, ny, nx), c[1 + d]) for d in range(6)]
    return orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec), diag


def _apply(sten, st, prec, v):
    torch = torch_cuda()
    vt = to_gpu_vec(v, prec)
    yt = torch.empty_like(vt)
    sten.stencil_apply(st, PREC[prec], vt, yt)
    return from_gpu_vec(yt, prec)


def _solve(sten, st, prec, b, tol, maxit, x0=None):
    torch = torch_cuda()
    bt = to_gpu_vec(b, prec)
    xt = torch.empty_like(bt)
    x0t = None if x0 is None else to_gpu_vec(x0, prec)
    it, hist, status = sten.bicgstab_solve(st, PREC[prec], bt, x0t, tol, maxit, xt)
    return widen(from_gpu_vec(xt, prec), prec), it, hist, status


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("mesh", [(37, 29, 18), (130, 17, 9), (1, 1, 6), (13, 40, 6), (300, 35, 12)])
@pytest.mark.parametrize("coef", [POISSON, SKEW])
@pytest.mark.parametrize("nslabs", [1, 3])
def test_const_apply_bitwise(sten, prec, mesh, coef, nslabs):
    """y = A_hat v through the scalar-coupling tile kernel: bitwise the oracle's FMA chain on
    the constant fields, at ragged x (nx not a multiple of the 16-B vector: lanes past nx
    must stay 0) and y tails, on one slab and on three loopback slabs."""
    nx, ny, nz = mesh
    if nz % nslabs:
        pytest.skip("nz not divisible")
    st = sten.stencil_create_const(nx, ny, nz, coef, nslabs=nslabs)
    assert sten.get_option(st, sten.OPT_CLASSIC_CONST) == 1
    cq, _ = const_coeffs(coef, nx, ny, nz, prec)
    v = quantize_vec(np.random.default_rng(nx * ny + nz).uniform(-1, 1, (nz, ny, nx)), prec)
    want = (orc.apply32_fma if prec == "fp32" else orc.apply16)(cq, v)
    got = _apply(sten, st, prec, v)
    assert np.array_equal(widen(got, prec), widen(want, prec))
    sten.set_option(st, sten.OPT_CLASSIC_CONST, 0)  # the array kernel on the same handle
    assert np.array_equal(widen(_apply(sten, st, prec, v), prec), widen(got, prec))
    st.close()


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("mesh,nslabs", [((48, 40, 36), 1), ((130, 21, 12), 1), ((37, 29, 18), 3)])
@pytest.mark.parametrize("coef", [POISSON, SKEW])
def test_const_classic_solve_equals_array_kernels(sten, prec, mesh, nslabs, coef):
    """Every H1 / H2 output feeds the next iteration, so equal x and history after 25
    iterations on the same handle mean every phase agreed (up to the sign of zero)."""
    nx, ny, nz = mesh
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=3), prec)
    st = sten.stencil_create_const(nx, ny, nz, coef, nslabs=nslabs)
    sten.set_schedule(st, sten.SCHED_CLASSIC)
    x1, it1, h1, s1 = _solve(sten, st, prec, b, 0.0, 25)
    sten.set_option(st, sten.OPT_CLASSIC_CONST, 0)
    x2, it2, h2, s2 = _solve(sten, st, prec, b, 0.0, 25)
    assert (it1, s1) == (it2, s2)
    assert np.array_equal(x1, x2)
    assert np.array_equal(h1, h2)
    st.close()


@pytest.mark.parametrize("mode", ["serial", "overlap", "fused"])
def test_const_classic_exchange_modes(sten, mode):
    """Three loopback slabs: the overlapped exchange and the fused peer-memory exchange
    (H1's boundary planes stored into the neighbours' halo planes by the scalar-coupling
    kernel) give the serial exchange's x and history."""
    nx, ny, nz = 45, 33, 18
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=5), "mixed")
    out = {}
    for m in ("serial", mode):
        st = sten.stencil_create_const(nx, ny, nz, SKEW, nslabs=3)
        sten.set_schedule(st, sten.SCHED_CLASSIC)
        sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, 1 if m == "overlap" else 0)
        sten.set_option(st, sten.OPT_CLASSIC_FUSED, 1 if m == "fused" else 0)
        out[m] = _solve(sten, st, "mixed", b, 0.0, 15)
        st.close()
    hs, hm = out["serial"][2], out[mode][2]
    if mode == "overlap":  # only the order in which the slabs' sums are added differs (fp16 amplifies it)
        assert np.all(np.abs(hm[:10] - hs[:10]) <= 5e-2 * hs[:10])
    else:
        assert np.array_equal(out["serial"][0], out[mode][0])
        assert np.array_equal(hs, hm)


@pytest.mark.parametrize("mesh,nhist", [((20, 40, 20), 12), ((45, 23, 17), 12), ((32, 32, 32), 12)])
@pytest.mark.parametrize("coef", [POISSON, SKEW])
def test_const_classic_mixed_history_vs_o16(sten, mesh, nhist, coef):
    """The north_star gate of the mixed mode (history within 5e-2 of the fp16-emulating
    oracle) on the constant operators.  These well-conditioned systems
    reach the fp16 floor (~5e-3 at the uniform right-hand side) by iteration ~14, after
    which both histories are rounding noise: R18's 12-iteration window of the classes that
    reach the floor sooner applies."""
    nx, ny, nz = mesh
    c16, diag = const_coeffs(coef, nx, ny, nz, "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=1))
    st = sten.stencil_create_const(nx, ny, nz, coef)
    x, it, hist, status = _solve(sten, st, "mixed", b16, 0.0, nhist)
    ref = orc.bicgstab16(c16, orc.scale_rhs(b16, diag, "mixed"), tol=0.0, maxit=nhist)
    n = min(len(hist), len(ref["hist"]))
    assert n == nhist + 1
    assert np.all(np.abs(hist[:n] - ref["hist"][:n]) <= 5e-2 * ref["hist"][:n])
    st.close()


def test_const_classic_fp32_vs_o64(sten):
    """fp32 to 1e-6 on the config-1 operator (32^3 Poisson): converged like the fp64 oracle,
    the early history within 1e-4, and x's true residual at the tolerance."""
    n = 32
    c32, diag = const_coeffs(POISSON, n, n, n, "fp32")
    b = inputs.rhs_uniform(n, n, n, seed=2).astype(np.float32)
    st = sten.stencil_create_const(n, n, n, POISSON)
    x, it, hist, status = _solve(sten, st, "fp32", b, 1e-6, 200)
    c64 = [c.astype(np.float64) for c in c32]
    bh = orc.scale_rhs(b, diag, "fp32").astype(np.float64)
    ref = orc.bicgstab64(c64, bh, tol=1e-6, maxit=200)
    assert status == sten.CONVERGED and hist[-1] <= 1e-6
    assert abs(it - ref["iters"]) <= max(3, 0.25 * ref["iters"])
    assert np.all(np.abs(hist[:11] - ref["hist"][:11]) <= 1e-4 * ref["hist"][:11])
    assert orc.true_residual64(c64, bh, x) <= 5e-6
    st.close()


def test_const_classic_x0_and_tol(sten):
    """x0 != 0 (r = b - A x0 through the scalar-coupling apply) and a tol stop: equal to the
    array kernels on the same handle."""
    nx, ny, nz = 40, 24, 16
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=7), "mixed")
    x0 = quantize_vec(np.random.default_rng(7).uniform(-0.1, 0.1, (nz, ny, nx)), "mixed")
    st = sten.stencil_create_const(nx, ny, nz, POISSON)
    r1 = _solve(sten, st, "mixed", b, 2e-3, 60, x0)
    sten.set_option(st, sten.OPT_CLASSIC_CONST, 0)
    r2 = _solve(sten, st, "mixed", b, 2e-3, 60, x0)
    assert r1[1] == r2[1] and r1[3] == r2[3] and np.array_equal(r1[2], r2[2])
    assert np.array_equal(r1[0], r2[0])
    assert r1[3] == sten.CONVERGED
    with pytest.raises(sten.StenError):
        sten.set_option(st, sten.OPT_CLASSIC_CONST, 2)
    st.close()
