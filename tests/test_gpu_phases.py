"""Classic-schedule phases H1 and H2 (Alg. 1) element by element.

sten_classic_phase runs ONE phase of the solve's kernels on caller vectors (same
tiling, slabs, halo exchange and its overlap as a solve).  The oracle side is the
composition of pinned primitives in the R10/R11 order:
  H1: p' = fma(beta_w, fma(-omega_w, v, p), r) (l.184), v' = A p' (l.176), (rhat, v') (l.177)
  H2: s = fma(-alpha_w, v, r) (l.178), t = A s (l.179), (t, s), (t, t) (l.180)
with fma = o16_fma (binary16, exact-then-round) or o32_fma_array (fmaf), A the
FMA-chain mirrors o16_apply_fused / o32_apply_fma, and the scalars rounded fp64 ->
fp32 -> working precision.  Vectors must be bitwise equal; the fp32 sums lie within
1e-5 * sum|a_i b_i| of fp64 reductions of the returned vectors (R13).
"""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import fields, from_gpu_vec, gpu_stencil, oracle_coeffs, quantize_vec, to_gpu_vec, torch_cuda, widen

pytestmark = pytest.mark.gpu
PREC = {"fp32": 0, "mixed": 1}
SCAL = (0.61, 0.93, -0.27)  # alpha, omega, beta


@pytest.fixture(scope="module")
def sten():
    import paper_2010_03660_b200 as s
    return s


def scal_w(x, prec):
    x32 = np.float32(x)
    return x32 if prec == "fp32" else orc.f16_from_double(np.array([float(x32)]))[0]


def oracle_phase(phase, cq, r, p, v, prec):
    al, om, be = (scal_w(t, prec) for t in SCAL)
    if prec == "fp32":
        neg = lambda a: np.float32(-a)  # noqa: E731
        fma = orc.fma32_array
        A = lambda u: orc.apply32_fma(cq, u)  # noqa: E731
    else:
        neg = lambda a: np.uint16(int(a) ^ 0x8000)  # noqa: E731
        fma = lambda a, b, c: orc.fma16_array(np.full(b.shape, a, np.uint16), b, c)  # noqa: E731
        A = lambda u: orc.apply16(cq, u)  # noqa: E731
    if phase == 1:
        out0 = fma(be, fma(neg(om), v, p), r)
    else:
        out0 = fma(neg(al), v, r)
    return out0, A(out0)


def vecs(nx, ny, nz, prec, seed):
    rng = np.random.default_rng(seed)
    return {n: quantize_vec(rng.uniform(-1, 1, (nz, ny, nx)), prec) for n in ("r", "p", "v", "rh")}


def run_phase(sten, st, prec, phase, V):
    torch = torch_cuda()
    t = {n: to_gpu_vec(a, prec) for n, a in V.items()}
    o0, o1 = torch.empty_like(t["r"]), torch.empty_like(t["r"])
    dots = sten.classic_phase(st, PREC[prec], phase, SCAL, t["r"], t["p"], t["v"], t["rh"], o0, o1)
    return from_gpu_vec(o0, prec), from_gpu_vec(o1, prec), dots


def check_dots(phase, dots, o0, o1, V, prec):
    w = lambda a: widen(a, prec).ravel()  # noqa: E731
    pairs = [(w(V["rh"]), w(o1))] if phase == 1 else [(w(o1), w(o0)), (w(o1), w(o1))]
    for d, (a, b) in zip(dots, pairs):
        assert abs(float(d) - float(a @ b)) <= 1e-5 * float(np.abs(a) @ np.abs(b)) + 1e-30


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("phase", [1, 2])
@pytest.mark.parametrize("mesh,ns", [((1, 1, 1), 1), ((45, 23, 17), 1), ((300, 40, 70), 1), ((129, 17, 9), 1),
                                     ((37, 21, 24), 2), ((37, 21, 24), 3), ((37, 21, 24), 12)])
def test_phase_bitwise_vs_oracle(sten, prec, phase, mesh, ns):
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=3)
    cq = oracle_coeffs(diag, offs, prec)
    V = vecs(nx, ny, nz, prec, 11)
    st = gpu_stencil(diag, offs, nslabs=ns)
    o0, o1, dots = run_phase(sten, st, prec, phase, V)
    w0, w1 = oracle_phase(phase, cq, V["r"], V["p"], V["v"], prec)
    assert np.array_equal(widen(o0, prec), widen(w0, prec))
    assert np.array_equal(widen(o1, prec), widen(w1, prec))
    check_dots(phase, dots, o0, o1, V, prec)
    if ns > 1:  # serial exchange: the same vectors, sums to rounding
        sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, 0)
        s0, s1, sd = run_phase(sten, st, prec, phase, V)
        assert np.array_equal(s0, o0) and np.array_equal(s1, o1)
        check_dots(phase, sd, s0, s1, V, prec)
    st.close()


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
def test_phase_tilings_and_segments(sten, prec):
    """Explicit tilings (row strips, 8-row tiles, per-thread coefficient loads, 1-plane chunks): the
    same vectors; the segment list follows the chunk plan."""
    nx, ny, nz = 150, 37, 13
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.0, seed=4)
    cq = oracle_coeffs(diag, offs, prec)
    V = vecs(nx, ny, nz, prec, 12)
    want = {ph: oracle_phase(ph, cq, V["r"], V["p"], V["v"], prec) for ph in (1, 2)}
    st = gpu_stencil(diag, offs)
    bx = 64 if prec == "fp32" else 128
    for tiling in ((0, 0, 0, 0), (bx, 8, 5, 3), (bx, 16, 1, 4), (nx, 2, 4, 3), (bx, 16, 13, 0)):
        sten.set_tiling(st, PREC[prec], *tiling)
        segs = sten.classic_segments(st, PREC[prec])
        assert segs[0] == 0 and all(b > a for a, b in zip(segs, segs[1:])) and segs[-1] < nz
        if tiling[2]:
            assert segs == list(range(0, nz, tiling[2]))
        for ph in (1, 2):
            o0, o1, dots = run_phase(sten, st, prec, ph, V)
            assert np.array_equal(widen(o0, prec), widen(want[ph][0], prec)), (tiling, ph)
            assert np.array_equal(widen(o1, prec), widen(want[ph][1], prec)), (tiling, ph)
            check_dots(ph, dots, o0, o1, V, prec)
    st.close()


def test_phase_argument_errors(sten):
    torch = torch_cuda()
    diag, offs = fields(inputs.KIND_CD, 8, 4, 3, seed=1)
    st = gpu_stencil(diag, offs)
    a = torch.zeros(3, 4, 8, device="cuda")
    with pytest.raises(sten.StenError):
        sten.classic_phase(st, sten.FP32, 3, SCAL, a, a, a, a, a, a)
    with pytest.raises(sten.StenError):
        sten.classic_phase(st, sten.FP32, 1, SCAL, a, None, a, None, a, a)
    st.close()
