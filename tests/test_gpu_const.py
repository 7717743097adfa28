"""Constant-coefficient operator (stencil_create_const): the
SR sweep without coefficient streams must equal the general kernel on the same
constant fields (bitwise: widened values, so +0 == -0), and the oracle."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import from_gpu_vec, gpu_stencil, quantize_vec, to_gpu_vec, torch_cuda, widen

pytestmark = pytest.mark.gpu
PREC = {"fp32": 0, "mixed": 1}
POISSON = (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0)
SKEW = (3.0, -0.7, -0.4, -0.25, -0.55, -0.3, -0.5)  # nonsymmetric constant operator


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def fields_const(c, nx, ny, nz):
    diag = np.full((nz, ny, nx), c[0])
    offs = [np.full((nz, ny, nx), c[1 + d]) for d in range(6)]
    return diag, offs


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("mesh", [(37, 29, 18), (130, 17, 9), (1, 1, 6), (13, 40, 6)])
@pytest.mark.parametrize("coef", [POISSON, SKEW])
@pytest.mark.parametrize("nslabs", [1, 3])
def test_const_sweep_equals_oracle(sten, prec, mesh, coef, nslabs):
    nx, ny, nz = mesh
    if nz % nslabs:
        pytest.skip("nz not divisible")
    torch = torch_cuda()
    st = sten.stencil_create_const(nx, ny, nz, coef, nslabs=nslabs)
    sten.set_sr_tiling(st, PREC[prec], 8, 2, 2, 3, 8 if nslabs == 3 else 16)
    diag, offs = fields_const(coef, nx, ny, nz)
    cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
    rng = np.random.default_rng(nx + nz)
    vec = lambda: quantize_vec(rng.uniform(-1, 1, (nz, ny, nx)), prec)
    rh, x, r, p = vec(), vec(), vec(), vec()
    ap = orc.apply32_fma if prec == "fp32" else orc.apply16
    v, q = ap(cq, p), ap(cq, r)
    y = ap(cq, v)
    ts = [to_gpu_vec(a, prec) for a in (rh, x, r, p, v, q, y)]
    dots = sten.sr_sweep(st, PREC[prec], (0.61, 0.93, -0.27), *ts)
    ref = (orc.sr_sweep32 if prec == "fp32" else orc.sr_sweep16)(cq, (0.61, 0.93, -0.27), rh, x, r, p, v, q, y)
    for g, w in zip(ts[1:], ref[:6]):
        assert np.array_equal(widen(from_gpu_vec(g, prec), prec), widen(w, prec))
    # the twelve sums see only mesh points (ragged x and y tails included)
    got = [widen(from_gpu_vec(t, prec), prec) for t in ts]
    rhw, rw, vw, qw, yw = got[0], got[2], got[4], got[5], got[6]
    pairs = [(rhw, vw), (rhw, rw), (rhw, qw), (rhw, yw), (qw, rw), (qw, vw), (yw, rw), (yw, vw), (qw, qw),
             (qw, yw), (yw, yw), (rw, rw)]
    for d, (a_, b_) in enumerate(pairs):
        assert abs(float(dots[d]) - float(np.vdot(a_, b_))) <= 1e-5 * float(np.vdot(np.abs(a_), np.abs(b_))) + 1e-30
    st.close()
    del torch


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
def test_const_solve_equals_general_kernel(sten, prec):
    torch = torch_cuda()
    nx, ny, nz = 48, 40, 36
    diag, offs = fields_const(POISSON, nx, ny, nz)
    b = quantize_vec(inputs.rhs_uniform(nx, ny, nz, seed=1), prec)
    out = {}
    for name in ("const", "general"):
        st = (sten.stencil_create_const(nx, ny, nz, POISSON) if name == "const" else gpu_stencil(diag, offs))
        sten.set_schedule(st, sten.SCHED_SR)
        sten.set_sr_tiling(st, PREC[prec], 16, 2, 2)  # the same geometry (and dot order) on both handles
        bt = to_gpu_vec(b, prec)
        xt = torch.empty_like(bt)
        it, hist, status = sten.bicgstab_solve(st, PREC[prec], bt, None, 0.0, 30, xt)
        out[name] = (widen(from_gpu_vec(xt, prec), prec), hist)
        # the classic schedule runs on the constant handle too (coefficient arrays)
        sten.set_schedule(st, sten.SCHED_CLASSIC)
        itc, histc, _ = sten.bicgstab_solve(st, PREC[prec], bt, None, 0.0, 10, xt)
        out[name + "_classic"] = histc
        st.close()
    assert np.array_equal(out["const"][0], out["general"][0])
    assert np.array_equal(out["const"][1], out["general"][1])
    assert np.array_equal(out["const_classic"], out["general_classic"])


def test_sr_needs_two_planes_per_slab(sten):
    st = sten.stencil_create_const(5, 4, 3, POISSON, nslabs=3)
    sten.set_schedule(st, sten.SCHED_SR)
    torch = torch_cuda()
    b = torch.zeros((3, 4, 5), dtype=torch.float32, device="cuda")
    with pytest.raises(sten.StenError):
        sten.bicgstab_solve(st, 0, b, None, 0.0, 2, torch.empty_like(b))
    st.close()


def test_const_invalid(sten):
    with pytest.raises(sten.StenError):
        sten.stencil_create_const(4, 4, 4, (0.0, -1, -1, -1, -1, -1, -1))
    with pytest.raises(sten.StenError):
        sten.stencil_create_const(4, 4, 4, (6.0, float("nan"), -1, -1, -1, -1, -1))
