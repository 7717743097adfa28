"""Parity at BASELINE.json's full size (600x595x1536, config 3/4), in the launch
configuration bench.py times (default tiling, 64-plane z chunks).

The oracle cannot hold the full mesh, so the SpMV is checked on SAMPLED outputs:
for each sampled point the oracle scales (o64_jacobi_scale) and applies
(o16/o32 mirrors) the 3x3x3 window around it, clipped to the global mesh, built
from the global generator (inputs.field_at) - the centre value of the window is
exactly the full-mesh value.  Samples cover mesh corners and faces, tile edges
(x = 127/128, y = 15/16), the z-chunk edges of the library's own chunk plan
(sten_classic_segments: every chunk start and the plane before it) and random
interior points.  The fused phases H1 and H2 (sten_classic_phase, the kernels a
solve launches) are sampled the same way against the oracle's composition of
pinned primitives on the window.  The solve is checked through properties that
hold at any size.
"""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

NX, NY, NZ = 600, 595, 1536


def chunk_edges(segs):
    zs = {0, 1, NZ - 2, NZ - 1}
    for z in segs:
        zs.update(z2 for z2 in (z - 1, z) if 0 <= z2 < NZ)
    return sorted(zs)


def sample_points(rng, n_random=600, zs=(0, 1, 63, 64, 127, 128, 1534, 1535)):
    pts = set()
    for x in (0, 1, 127, 128, 255, 256, 511, 512, 598, 599):
        for y in (0, 1, 15, 16, 593, 594):
            for z in zs:
                pts.add((x, y, z))
    for _ in range(n_random):
        pts.add((int(rng.integers(NX)), int(rng.integers(NY)), int(rng.integers(NZ))))
    return sorted(pts)


def window_value(pt, vfull_fn, prec):
    """Oracle value of (A_hat v) at one global point from its clipped 3x3x3 window."""
    x, y, z = pt
    x0, x1 = max(x - 1, 0), min(x + 2, NX)
    y0, y1 = max(y - 1, 0), min(y + 2, NY)
    z0, z1 = max(z - 1, 0), min(z + 2, NZ)
    kg, j, i = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag, offs = inputs.field_at(inputs.KIND_CD, NX, NY, i, j, kg, seed=1, delta=0.1)
    c64 = orc.jacobi_scale(diag, offs)  # window edges that are not mesh edges: coupling
    cq = orc.quantize_coeffs(c64, prec)  # dropped there, but never used for the centre
    v = vfull_fn(i, j, kg)
    u = orc.apply32_fma(cq, v) if prec == "fp32" else orc.apply16(cq, v)
    return u[z - z0, y - y0, x - x0]


@pytest.fixture(scope="module")
def full_problem():
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    ic.build()
    diag, offs = ic.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
    st = sten.stencil_create(NX, NY, NZ, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    yield st
    st.close()


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
def test_fullsize_spmv_sampled_bitwise(full_problem, prec):
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    # v = a seeded field on the full mesh (stream 7), rounded RN to fp32 on the device,
    # then (mixed) fp32 -> fp16 RN.  torch's fp64 -> fp16 would round twice (via fp32),
    # so both sides round through fp32 explicitly.
    v32 = ic.uniform_device(NX, NY, NZ, seed=3, stream=7, dtype="f32")
    vt = v32 if prec == "fp32" else v32.to(torch.float16)
    del v32
    yt = torch.empty_like(vt)
    sten.stencil_apply(st, sten.FP32 if prec == "fp32" else sten.MIXED, vt, yt)
    torch.cuda.synchronize()

    def vfull(i, j, kg):  # the same v values, recomputed on the host for a window
        idx = (i + NX * (j + NY * kg)).astype(np.uint64)
        v = inputs.uniform(3, 7, idx, -1.0, 1.0).astype(np.float32)
        return v if prec == "fp32" else orc.f16_from_double(v.astype(np.float64))

    segs = sten.classic_segments(st, sten.FP32 if prec == "fp32" else sten.MIXED)
    assert len(segs) > 1 and segs == sorted(segs)
    pts = sample_points(np.random.default_rng(11), zs=chunk_edges(segs))
    idx = torch.tensor([x + NX * (y + NY * z) for x, y, z in pts], device="cuda")
    got = yt.reshape(-1)[idx].cpu().numpy()
    if prec != "fp32":
        got = got.view(np.uint16)
    for k, pt in enumerate(pts):
        want = window_value(pt, vfull, prec)
        a = float(got[k]) if prec == "fp32" else orc.f16_to_double(np.array([got[k]]))[0]
        b = float(want) if prec == "fp32" else orc.f16_to_double(np.array([want]))[0]
        assert a == b, (pt, a, b)


PH_STREAMS = dict(r=21, p=22, v=23, rh=24)
PH_SCAL = (0.61, 0.93, -0.27)  # alpha, omega, beta


def _w(x, prec):  # scalar rounded fp64 -> fp32 -> working precision (R11)
    x32 = np.float32(x)
    return x32 if prec == "fp32" else orc.f16_from_double(np.array([float(x32)]))[0]


def window_phase(pt, phase, prec):
    """Oracle (out0, out1) of one classic phase at a global point from its clipped 3x3x3 window:
    out0 = p' (H1) or s (H2) element-wise, out1 = A out0 at the centre."""
    x, y, z = pt
    x0, x1 = max(x - 1, 0), min(x + 2, NX)
    y0, y1 = max(y - 1, 0), min(y + 2, NY)
    z0, z1 = max(z - 1, 0), min(z + 2, NZ)
    kg, j, i = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag, offs = inputs.field_at(inputs.KIND_CD, NX, NY, i, j, kg, seed=1, delta=0.1)
    cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
    idx = (i + NX * (j + NY * kg)).astype(np.uint64)
    V = {}
    for n, s_ in PH_STREAMS.items():
        v = inputs.uniform(9, s_, idx, -1.0, 1.0).astype(np.float32)
        V[n] = v if prec == "fp32" else orc.f16_from_double(v.astype(np.float64))
    al, om, be = (_w(t, prec) for t in PH_SCAL)
    if prec == "fp32":
        fma, neg = orc.fma32_array, (lambda a: np.float32(-a))
        A = lambda u: orc.apply32_fma(cq, u)  # noqa: E731
    else:
        fma = lambda a, b, c: orc.fma16_array(np.full(b.shape, a, np.uint16), b, c)  # noqa: E731
        neg = lambda a: np.uint16(int(a) ^ 0x8000)  # noqa: E731
        A = lambda u: orc.apply16(cq, u)  # noqa: E731
    out0 = fma(be, fma(neg(om), V["v"], V["p"]), V["r"]) if phase == 1 else fma(neg(al), V["v"], V["r"])
    out1 = A(out0)
    c = (z - z0, y - y0, x - x0)
    return out0[c], out1[c]


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
@pytest.mark.parametrize("phase", [1, 2])
def test_fullsize_phase_sampled_bitwise(full_problem, prec, phase):
    """H1 (p' = r + beta(p - omega v), v' = A p') and H2 (s = r - alpha v, t = A s) at 600x595x1536 in
    the bench's launch configuration, sampled bitwise; their sums against fp64 reductions."""
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    P = sten.FP32 if prec == "fp32" else sten.MIXED
    t = {}
    for n, s_ in PH_STREAMS.items():
        v32 = ic.uniform_device(NX, NY, NZ, seed=9, stream=s_, dtype="f32")
        t[n] = v32 if prec == "fp32" else v32.to(torch.float16)
        del v32
    o0, o1 = torch.empty_like(t["r"]), torch.empty_like(t["r"])
    dots = sten.classic_phase(st, P, phase, PH_SCAL, t["r"], t["p"], t["v"], t["rh"], o0, o1)
    torch.cuda.synchronize()
    pts = sample_points(np.random.default_rng(23), n_random=300, zs=chunk_edges(sten.classic_segments(st, P)))
    idx = torch.tensor([x + NX * (y + NY * z) for x, y, z in pts], device="cuda")
    g0, g1 = (o.reshape(-1)[idx].cpu().numpy() for o in (o0, o1))
    wid = (lambda a: float(a)) if prec == "fp32" else (lambda a: float(orc.f16_to_double(np.array([a]).view(np.uint16))[0]))
    for k, pt in enumerate(pts):
        w0, w1 = window_phase(pt, phase, prec)
        assert wid(g0[k]) == wid(w0) and wid(g1[k]) == wid(w1), (pt, phase)
    d0, d1 = o0.double().reshape(-1), o1.double().reshape(-1)
    pairs = [(t["rh"].double().reshape(-1), d1)] if phase == 1 else [(d1, d0), (d1, d1)]
    for got, (a, b) in zip(dots, pairs):
        exact, scale = float(torch.dot(a, b)), float(torch.dot(a.abs(), b.abs()))
        assert abs(float(got) - exact) <= 2e-5 * scale, (float(got), exact)


def test_fullsize_mixed_solve_properties(full_problem):
    """Config 3 in the bench's configuration: 100 fixed iterations, then a tol=1e-3 run."""
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    b = ic.uniform_device(NX, NY, NZ, seed=1, stream=0).half()
    x = torch.empty_like(b)
    it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 100, x)
    assert it == 100 and np.all(np.isfinite(hist))
    assert hist[0] == 1.0
    assert hist[10] < 2e-3  # converging like the oracle does on the same class at 32^3-128^3
    # determinism at full size
    x2 = torch.empty_like(b)
    it2, hist2, _ = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 100, x2)
    assert np.array_equal(hist, hist2) and torch.equal(x, x2)
    # config 3(b): tol = 1e-3 stops at the first history entry below it
    it3, hist3, status3 = sten.bicgstab_solve(st, sten.MIXED, b, None, 1e-3, 200, x2)
    assert status3 == sten.CONVERGED and hist3[-1] <= 1e-3 < hist3[-2] and it3 <= 15
    assert np.array_equal(hist3, hist[: it3 + 1])  # same trajectory as the fixed-iteration run


def test_fullsize_fp32_reaches_1e6(full_problem):
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    b = ic.uniform_device(NX, NY, NZ, seed=1, stream=0).float()
    x = torch.empty_like(b)
    it, hist, status = sten.bicgstab_solve(st, sten.FP32, b, None, 1e-6, 500, x)
    assert status == sten.CONVERGED and hist[-1] <= 1e-6 and it < 40
    # recurrence residual vs the true residual of the scaled system, at full size:
    # ||b_hat - A x|| / ||b_hat|| computed with the library's own SpMV (fp32)
    ax = torch.empty_like(x)
    sten.stencil_apply(st, sten.FP32, x, ax)
    # b_hat = b / a_P: a_P from the generator on the device
    dg, _ = ic.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
    bh = (b.double() / dg).float()
    del dg
    true_res = float(torch.linalg.vector_norm((bh - ax).double()) / torch.linalg.vector_norm(bh.double()))
    assert true_res <= 1e-5, true_res


def test_fullsize_loopback_slab_exchange_modes():
    """Config 3 on 2 loopback z-slabs (the multi-GPU decomposition's code on one GPU, at the size
    the scaling runs use): every classic exchange mode runs - serial, overlapped (side stream),
    fused (peer stores + inbox deposits) - and serial and fused agree bitwise, overlapped to the
    rounding of its different sum order; the SR sweep in its three exchange modes too."""
    torch = torch_cuda()
    import inputs.cuda as icuda
    import paper_2010_03660_b200 as sten
    diag, offs = icuda.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
    st = sten.stencil_create(NX, NY, NZ, [diag] + offs, nslabs=2)
    del diag, offs
    b = icuda.uniform_device(NX, NY, NZ, seed=1, stream=0).half()
    res = {}
    for mode, ov, fu in (("serial", 0, 0), ("overlap", 1, 0), ("fused", 0, 1)):
        sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, ov)
        sten.set_option(st, sten.OPT_CLASSIC_FUSED, fu)
        x = torch.empty_like(b)
        it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 4, x)
        res[mode] = (x, hist)
        assert it == 4 and np.all(np.isfinite(hist))
    assert torch.equal(res["serial"][0].view(torch.int16), res["fused"][0].view(torch.int16))
    assert np.array_equal(res["serial"][1], res["fused"][1])
    assert np.allclose(res["overlap"][1], res["serial"][1], rtol=1e-3)
    sten.set_schedule(st, sten.SCHED_SR)
    srh = {}
    for xm in (sten.XCHG_SERIAL, sten.XCHG_OVERLAP, sten.XCHG_FUSED):  # the SR exchange modes too
        sten.set_sr_exchange(st, xm)
        x = torch.empty_like(b)
        it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 4, x)
        assert it == 4 and np.allclose(hist, res["serial"][1], rtol=5e-2)
        srh[xm] = hist
    assert np.array_equal(srh[sten.XCHG_SERIAL], srh[sten.XCHG_FUSED])
    st.close()


@pytest.mark.parametrize("phase", [1, 2])
def test_fullsize_half_dot_phase(full_problem, phase):
    """Half dots (R22, R28; `bench.py --dots half`) at 600x595x1536: the phase's vectors bitwise those
    of the mixed-dot phase (only the sums differ), and its sums within 2e-5 of the sum of |segment
    sums| from the oracle's exact sum of the same fp16 column pencils (dot16h) over the library's
    chunk plan (one plan for the three phases in this mode)."""
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    t = {}
    for n, s_ in PH_STREAMS.items():
        t[n] = ic.uniform_device(NX, NY, NZ, seed=9, stream=s_, dtype="f32").to(torch.float16)
    outs = {}
    for mode in (sten.DOTS_MIXED, sten.DOTS_HALF):
        sten.set_dot_precision(st, mode)
        try:
            o0, o1 = torch.empty_like(t["r"]), torch.empty_like(t["r"])
            dots = sten.classic_phase(st, sten.MIXED, phase, PH_SCAL, t["r"], t["p"], t["v"], t["rh"], o0, o1)
            segs = sten.classic_segments(st, sten.MIXED)
        finally:
            sten.set_dot_precision(st, sten.DOTS_MIXED)
        outs[mode] = (o0, o1, dots, segs)
    o0, o1, dots, segs = outs[sten.DOTS_HALF]
    assert torch.equal(o0.view(torch.int16), outs[sten.DOTS_MIXED][0].view(torch.int16))
    assert torch.equal(o1.view(torch.int16), outs[sten.DOTS_MIXED][1].view(torch.int16))
    host = lambda a: a.cpu().numpy().view(np.uint16).reshape(NZ, NY, NX)  # noqa: E731
    h1 = host(o1)
    pairs = [(host(t["rh"]), h1)] if phase == 1 else [(h1, host(o0)), (h1, h1)]
    for got, (a, b) in zip(dots, pairs):
        want, absum = orc.dot16h(a, b, segs)
        assert abs(float(got) - want) <= 2e-5 * absum, (float(got), want, absum)
