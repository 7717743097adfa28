"""GPU parity of the half-dot SR sweep (STEN_DOTS_HALF, R22; SURVEY §8(f)
NEXT-4) against oracle/osr.c o16h_*.

  sweep : x, r, p, v, q, y bitwise equal to the oracle (the vector arithmetic is
          the mixed sweep's); the twelve sums within the fp32 reordering bound of
          the same fp16 column-segment pencils, |d| <= 1e-5 * sum|segment sums|,
          with the segments the library reports (sten_sr_segments) -- default
          plan, uniform chunks, ragged meshes, 8- and 16-row tiles
  solve : residual history within 5e-2 of O16-SR with the same half dots for
          the first iterations (the R20 rule of the mixed mode)
  API   : unsupported combinations are refused, not silently run as mixed
"""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import fields, from_gpu_vec, gpu_stencil, oracle_coeffs, quantize_vec, to_gpu_vec, torch_cuda, widen

pytestmark = pytest.mark.gpu
MIXED = 1


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def _sweep(sten, mesh, tiling=None, scalars=(0.61, 0.93, -0.27), seed=3, nslabs=1):
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.0, seed=seed)
    st = gpu_stencil(diag, offs, nslabs=nslabs)
    if nslabs > 1:
        sten.set_sr_exchange(st, sten.XCHG_SERIAL)
    if tiling:
        sten.set_sr_tiling(st, MIXED, *tiling)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    seg = sten.sr_segments(st, MIXED)
    cq = oracle_coeffs(diag, offs, "mixed")
    rng = np.random.default_rng(seed + 5)
    vec = lambda: quantize_vec(rng.uniform(-1, 1, (nz, ny, nx)), "mixed")
    rh, x, r, p = vec(), vec(), vec(), vec()
    v = orc.apply16(cq, p)
    q = orc.apply16(cq, r)
    y = orc.apply16(cq, v)
    ts = [to_gpu_vec(a, "mixed") for a in (rh, x, r, p, v, q, y)]
    dots = sten.sr_sweep(st, MIXED, scalars, *ts)
    got = [from_gpu_vec(t, "mixed") for t in ts[1:]]
    ref = orc.sr_sweep16(cq, scalars, rh, x, r, p, v, q, y, segments=seg)
    st.close()
    return got, dots, ref, seg


@pytest.mark.parametrize("mesh,tiling", [((37, 29, 19), None), ((130, 17, 40), (16, 2, 2, 16)),
                                         ((264, 20, 11), (8, 2, 2, 3)), ((5, 3, 2), None),
                                         ((129, 33, 70), (8, 3, 3, 9))])
def test_half_dot_sweep(sten, mesh, tiling):
    got, dots, ref, seg = _sweep(sten, mesh, tiling)
    if tiling:
        assert seg == list(range(0, mesh[2], tiling[3]))
    for name, g, w in zip(["x", "r", "p", "v", "q", "y"], got, ref[:6]):
        assert np.array_equal(widen(g, "mixed"), widen(w, "mixed")), name
    want, scale = ref[6], ref[7]
    for d in range(12):
        assert abs(float(dots[d]) - float(want[d])) <= 1e-5 * float(scale[d]) + 1e-30, (d, float(dots[d]), want[d])


def test_half_dot_sweep_slabs(sten):
    """Three loopback z-slabs: the pencils restart at every slab (and chunk) boundary."""
    got, dots, ref, seg = _sweep(sten, (37, 29, 30), (16, 2, 2, 7), nslabs=3)
    assert seg == [0, 7, 10, 17, 20, 27]
    for name, g, w in zip(["x", "r", "p", "v", "q", "y"], got, ref[:6]):
        assert np.array_equal(widen(g, "mixed"), widen(w, "mixed")), name
    for d in range(12):
        assert abs(float(dots[d]) - float(ref[6][d])) <= 1e-5 * float(ref[7][d]) + 1e-30, d


def test_half_dots_refuse_fused_exchange(sten):
    diag, offs = fields(inputs.KIND_CD, 16, 8, 8)
    st = gpu_stencil(diag, offs, nslabs=2)
    sten.set_sr_exchange(st, sten.XCHG_FUSED)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    torch = torch_cuda()
    b = torch.ones(8, 8, 16, dtype=torch.float16, device="cuda")
    x = torch.empty_like(b)
    sten.set_schedule(st, sten.SCHED_SR)
    with pytest.raises(sten.StenError, match="FUSED"):
        sten.bicgstab_solve(st, MIXED, b, None, 0.0, 3, x)
    sten.set_sr_exchange(st, sten.XCHG_OVERLAP)
    it, hist, status = sten.bicgstab_solve(st, MIXED, b, None, 0.0, 3, x)
    assert it == 3
    st.close()


def test_half_dots_differ_from_mixed(sten):
    """The mode really changes the sums (one long pencil per column: 40 fp16 adds)."""
    got_h, dots_h, _, _ = _sweep(sten, (64, 16, 40), (16, 2, 2, 40))
    torch = torch_cuda()
    nx, ny, nz = 64, 16, 40
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.0, seed=3)
    st = gpu_stencil(diag, offs)
    sten.set_sr_tiling(st, MIXED, 16, 2, 2, 40)
    cq = oracle_coeffs(diag, offs, "mixed")
    rng = np.random.default_rng(8)
    vec = lambda: quantize_vec(rng.uniform(-1, 1, (nz, ny, nx)), "mixed")
    rh, x, r, p = vec(), vec(), vec(), vec()
    v, q = orc.apply16(cq, p), orc.apply16(cq, r)
    y = orc.apply16(cq, v)
    dots_m = sten.sr_sweep(st, MIXED, (0.61, 0.93, -0.27), *[to_gpu_vec(a, "mixed") for a in (rh, x, r, p, v, q, y)])
    st.close()
    assert not np.array_equal(np.asarray(dots_h), np.asarray(dots_m))
    del torch


@pytest.mark.parametrize("mesh,delta,nhist", [((32, 32, 32), 0.1, 12), ((37, 29, 19), 0.0, 10)])
def test_half_dot_solve_history(sten, mesh, delta, nhist):
    torch = torch_cuda()
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=delta, seed=1)
    b16 = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=1))
    st = gpu_stencil(diag, offs)
    sten.set_schedule(st, sten.SCHED_SR)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    seg = sten.sr_segments(st, MIXED)
    bt = to_gpu_vec(b16, "mixed")
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, MIXED, bt, None, 0.0, nhist, xt)
    c16 = oracle_coeffs(diag, offs, "mixed")
    ref = orc.bicgstab16(c16, orc.scale_rhs(b16, diag, "mixed"), tol=0.0, maxit=nhist, schedule="sr", segments=seg)
    assert len(hist) == len(ref["hist"]) == nhist + 1
    assert np.all(np.abs(hist - ref["hist"]) <= 5e-2 * ref["hist"])
    st.close()


def test_half_dot_api_guards(sten):
    diag, offs = fields(inputs.KIND_CD, 16, 8, 6)
    st = gpu_stencil(diag, offs)
    with pytest.raises(sten.StenError):
        sten.set_dot_precision(st, 2)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    torch = torch_cuda()
    b = torch.ones(6, 8, 16, dtype=torch.float16, device="cuda")
    x = torch.empty_like(b)
    sten.set_schedule(st, sten.SCHED_CLASSIC)  # classic half (R28): the default tile kernels only
    sten.set_tiling(st, MIXED, 0, 8, 0, 0)
    with pytest.raises(sten.StenError, match="half dots"):
        sten.bicgstab_solve(st, MIXED, b, None, 0.0, 3, x)
    st.close()
    st = gpu_stencil(diag, offs)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    st2 = gpu_stencil(diag, offs, nslabs=2)  # and one slab
    sten.set_dot_precision(st2, sten.DOTS_HALF)
    with pytest.raises(sten.StenError, match="half dots"):
        sten.bicgstab_solve(st2, MIXED, b, None, 0.0, 3, x)
    st2.close()
    sten.set_schedule(st, sten.SCHED_SR)
    sten.set_sr_tiling(st, MIXED, 16, 2, 2, 0, 8)  # 8-B packs: not built with half dots
    with pytest.raises(sten.StenError, match="half dots"):
        sten.bicgstab_solve(st, MIXED, b, None, 0.0, 3, x)
    sten.set_sr_tiling(st, MIXED, 16, 2, 2, 0, 16)
    it, hist, status = sten.bicgstab_solve(st, MIXED, b, None, 0.0, 3, x)
    assert it == 3 and np.all(np.isfinite(hist))
    # fp32 solves ignore the setting
    bf, xf = b.float(), torch.empty(6, 8, 16, dtype=torch.float32, device="cuda")
    it, hist, status = sten.bicgstab_solve(st, 0, bf, None, 0.0, 3, xf)
    assert it == 3
    sten.set_dot_precision(st, sten.DOTS_MIXED)
    st.close()
    cst = sten.stencil_create_const(16, 8, 6, [6.0] + [-1.0] * 6)
    sten.set_schedule(cst, sten.SCHED_SR)
    sten.set_dot_precision(cst, sten.DOTS_HALF)
    with pytest.raises(sten.StenError, match="constant"):
        sten.bicgstab_solve(cst, MIXED, b, None, 0.0, 3, x)
    cst.close()


def test_half_dot_underflow_is_breakdown(sten):
    """R23: when every fp16 pencil of (r,r) underflows to 0 while (rhat, r) does not,
    the solve reports BREAKDOWN at that iteration - never a false CONVERGED - as the oracle does
    (tests/test_oracle_halfdots.py); with tol > 0 it stops there with BREAKDOWN."""
    torch = torch_cuda()
    n = 10
    diag, offs = fields(inputs.KIND_CD, n, n, n, delta=0.1, seed=2)
    b = quantize_vec(inputs.rhs_uniform(n, n, n, seed=2), "mixed")
    # the scaled system with b_hat = b (unit diagonal passed in): the RHS of the oracle pin
    st = gpu_stencil(None, [o / diag for o in offs], unit_diag=True)
    sten.set_schedule(st, sten.SCHED_SR)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    seg = sten.sr_segments(st, MIXED)
    bt = to_gpu_vec(b, "mixed")
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, MIXED, bt, None, 0.0, 40, xt)
    zero = np.flatnonzero(hist == 0.0)
    assert zero.size > 0
    k = int(zero[0])
    assert status == sten.BREAKDOWN and sten.get_stats(st)["event_iter"] == k
    it2, hist2, status2 = sten.bicgstab_solve(st, MIXED, bt, None, 1e-9, 40, xt)
    assert status2 == sten.BREAKDOWN and it2 == k and hist2[-1] == 0.0
    # the oracle with the library's segments underflows at the same point within the
    # fp32 reordering of the segment sums (its trajectory matches to 5e-2 until then)
    cq = oracle_coeffs(diag, offs, "mixed")
    ref = orc.bicgstab16(cq, b, tol=0.0, maxit=40, schedule="sr", segments=seg)
    assert ref["status"] == orc.ORC_BREAKDOWN and abs(ref["event_it"] - k) <= 1
    st.close()


# ---------------- the classic schedule (Alg. 1 as printed) with half dots (R28) ----------------
@pytest.mark.parametrize("mesh,delta,nhist", [((32, 32, 32), 0.1, 12), ((37, 29, 19), 0.0, 10),
                                              ((130, 33, 45), 0.1, 12)])
def test_classic_half_dot_solve_history(sten, mesh, delta, nhist):
    """The classic schedule with half dots against o16h_bicgstab over the library's own chunk plan
    (sten_classic_segments, one plan for H1, H2 and H3 in this mode): the history within 5e-2, and
    the same vectors as the classic mixed solve after one iteration except through the scalars."""
    torch = torch_cuda()
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=delta, seed=1)
    b16 = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=1))
    st = gpu_stencil(diag, offs)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    seg = sten.classic_segments(st, MIXED)
    bt = to_gpu_vec(b16, "mixed")
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, MIXED, bt, None, 0.0, nhist, xt)
    c16 = oracle_coeffs(diag, offs, "mixed")
    bh = orc.scale_rhs(b16, diag, "mixed")
    ref = orc.bicgstab16(c16, bh, tol=0.0, maxit=nhist, segments=seg)
    assert len(hist) == len(ref["hist"]) == nhist + 1
    assert np.all(np.abs(hist - ref["hist"]) <= 5e-2 * ref["hist"]), (hist, ref["hist"])
    mixed = orc.bicgstab16(c16, bh, tol=0.0, maxit=nhist)
    assert hist[0] == pytest.approx(mixed["hist"][0], rel=1e-6)  # the setup stays mixed
    assert not np.array_equal(hist, mixed["hist"])
    st.close()


@pytest.mark.parametrize("mesh", [(70, 37, 50), (130, 33, 45), (600, 7, 9)])
def test_classic_half_first_iteration_vectors(sten, mesh):
    """x_1 of the classic half solve within one fp16 ulp of o16h_bicgstab's (every vector op is the
    oracle's; alpha_1, omega_1 come from pencils whose fp32 sum order differs).  The two larger
    planes span two of k_h3s_half's 384-vector segments (the second one partial)."""
    torch = torch_cuda()
    nx, ny, nz = mesh
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz, delta=0.1, seed=4)
    b16 = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=4))
    st = gpu_stencil(diag, offs)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    seg = sten.classic_segments(st, MIXED)
    assert seg == list(range(0, nz, seg[1] if len(seg) > 1 else nz))
    bt = to_gpu_vec(b16, "mixed")
    xt = torch.empty_like(bt)
    _, hist, _ = sten.bicgstab_solve(st, MIXED, bt, None, 0.0, 1, xt)
    c16 = oracle_coeffs(diag, offs, "mixed")
    ref = orc.bicgstab16(c16, orc.scale_rhs(b16, diag, "mixed"), tol=0.0, maxit=1, segments=seg)
    xg, xo = widen(from_gpu_vec(xt, "mixed"), "mixed"), widen(ref["x"], "mixed")
    assert np.all(np.abs(xg - xo) <= np.spacing(np.abs(xo).astype(np.float16)).astype(np.float64) + 1e-12)
    # hist[1] = sqrt((r_1, r_1)) / ||b||: H3's (r,r) pencils over the same segments, summed in another order
    assert abs(hist[1] - ref["hist"][1]) <= 1e-3 * ref["hist"][1], (hist[1], ref["hist"][1])
    st.close()


def test_classic_half_underflow_is_breakdown(sten):
    """R23 with the classic half dots: the solve reports BREAKDOWN, never CONVERGED, where the
    pencils of (r,r) underflow (the oracle pin's system)."""
    torch = torch_cuda()
    n = 8
    diag, offs = fields(inputs.KIND_CD, n, n, n, delta=0.1, seed=1)
    b = quantize_vec(inputs.rhs_uniform(n, n, n, seed=1), "mixed")
    st = gpu_stencil(None, [o / diag for o in offs], unit_diag=True)
    sten.set_dot_precision(st, sten.DOTS_HALF)
    bt = to_gpu_vec(b, "mixed")
    xt = torch.empty_like(bt)
    it, hist, status = sten.bicgstab_solve(st, MIXED, bt, None, 1e-9, 40, xt)
    assert status == sten.BREAKDOWN and hist[-1] == 0.0
    st.close()
