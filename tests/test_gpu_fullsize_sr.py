"""SR-schedule parity at BASELINE.json's full size (600x595x1536, config 3) in the
launch configuration bench.py times (the SR defaults: 160-plane chunks with
64-plane tail chunks over the last 320 planes, 16-row tiles, unpadded rows).

One sweep (sten_sr_sweep) on seeded full-mesh inputs is checked on SAMPLED
outputs: the oracle runs o16_sr_sweep / o32_sr_sweep on the clipped 5x5x5 window
around each sampled point (y' = A A p' reaches two points), built from the global
generator; the window centre is exactly the full-mesh value.  Samples cover mesh
corners and faces, tile edges (x = 127/128, y = 15/16), every z-chunk edge of
the library's own SR chunk plan (sten_sr_segments: each chunk start and the plane
before it, including the long-to-tail transition) and random interior points.  The
twelve sums are checked against fp64 reductions of the returned vectors; the
solve through properties that hold at any size.
"""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

NX, NY, NZ = 600, 595, 1536
STREAMS = dict(rh=7, x=8, r=9, p=10, v=11, q=12, y=13)
SCAL = (0.61, 0.93, -0.27)


def chunk_edges(segs):
    zs = {0, 1, NZ - 2, NZ - 1}
    for z in segs:
        zs.update(z2 for z2 in (z - 1, z) if 0 <= z2 < NZ)
    return sorted(zs)


def sample_points(rng, zs, n_random=300):
    pts = set()
    for x in (0, 1, 127, 128, 511, 512, 598, 599):
        for y in (0, 1, 15, 16, 593, 594):
            for z in zs:
                pts.add((x, y, z))
    for _ in range(n_random):
        pts.add((int(rng.integers(NX)), int(rng.integers(NY)), int(rng.integers(NZ))))
    return sorted(pts)


def host_vec(name, i, j, kg, prec):
    idx = (i + NX * (j + NY * kg)).astype(np.uint64)
    v = inputs.uniform(5, STREAMS[name], idx, -1.0, 1.0).astype(np.float32)
    return v if prec == "fp32" else orc.f16_from_double(v.astype(np.float64))


def window_sweep(pt, prec):
    x, y, z = pt
    x0, x1 = max(x - 2, 0), min(x + 3, NX)
    y0, y1 = max(y - 2, 0), min(y + 3, NY)
    z0, z1 = max(z - 2, 0), min(z + 3, NZ)
    kg, j, i = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag, offs = inputs.field_at(inputs.KIND_CD, NX, NY, i, j, kg, seed=1, delta=0.1)
    cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
    vec = {n: host_vec(n, i, j, kg, prec) for n in STREAMS}
    fn = orc.sr_sweep32 if prec == "fp32" else orc.sr_sweep16
    out = fn(cq, SCAL, vec["rh"], vec["x"], vec["r"], vec["p"], vec["v"], vec["q"], vec["y"])
    return [o[z - z0, y - y0, x - x0] for o in out[:6]]


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
def test_fullsize_sr_sweep_sampled_bitwise(full_problem, prec):
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    P = sten.FP32 if prec == "fp32" else sten.MIXED
    ts = {}
    for n, s_ in STREAMS.items():
        v32 = ic.uniform_device(NX, NY, NZ, seed=5, stream=s_, dtype="f32")
        ts[n] = v32 if prec == "fp32" else v32.to(torch.float16)
        del v32
    order = ["rh", "x", "r", "p", "v", "q", "y"]
    dots = sten.sr_sweep(st, P, SCAL, *[ts[n] for n in order])
    torch.cuda.synchronize()
    segs = sten.sr_segments(st, P)
    if prec == "mixed":  # the bench's plan: long chunks, then the short tail chunks
        steps = [b - a for a, b in zip(segs, segs[1:])]
        assert len(set(steps)) == 2 and steps == sorted(steps, reverse=True), segs
    pts = sample_points(np.random.default_rng(17), chunk_edges(segs))
    idx = torch.tensor([x + NX * (y + NY * z) for x, y, z in pts], device="cuda")
    got = {n: ts[n].reshape(-1)[idx].cpu().numpy() for n in order[1:]}
    widen = (lambda a: a.astype(np.float64)) if prec == "fp32" else (lambda a: orc.f16_to_double(np.asarray(a)))
    for k, pt in enumerate(pts):
        want = window_sweep(pt, prec)
        for n, w in zip(order[1:], want):
            g = got[n][k] if prec == "fp32" else got[n][k:k + 1].view(np.uint16)
            assert float(np.asarray(widen(g)).ravel()[0]) == float(np.asarray(widen(np.asarray([w]))).ravel()[0]), (n, pt)
    # the twelve sums against fp64 reductions of the vectors the sweep returned
    d = {n: ts[n].double().reshape(-1) for n in ("rh", "r", "v", "q", "y")}
    pairs = [("rh", "v"), ("rh", "r"), ("rh", "q"), ("rh", "y"), ("q", "r"), ("q", "v"), ("y", "r"), ("y", "v"),
             ("q", "q"), ("q", "y"), ("y", "y"), ("r", "r")]
    for k, (a_, b_) in enumerate(pairs):
        exact = float(torch.dot(d[a_], d[b_]))
        scale = float(torch.dot(d[a_].abs(), d[b_].abs()))
        assert abs(float(dots[k]) - exact) <= 2e-5 * scale, (a_, b_, float(dots[k]), exact)


def test_fullsize_sr_solve_properties(full_problem):
    """Config 3 with the bench's schedule: 100 fixed iterations, then the tol = 1e-3 run;
    fp32 to 1e-6 with the true residual checked by the library's own SpMV."""
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = full_problem
    sten.set_schedule(st, sten.SCHED_SR)
    b = ic.uniform_device(NX, NY, NZ, seed=1, stream=0).half()
    x = torch.empty_like(b)
    it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 100, x)
    assert it == 100 and np.all(np.isfinite(hist)) and hist[0] == pytest.approx(1.0, rel=1e-6)
    assert hist[10] < 2e-3
    x2 = torch.empty_like(b)
    it2, hist2, _ = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 100, x2)
    assert np.array_equal(hist, hist2) and torch.equal(x, x2)  # deterministic at full size
    it3, hist3, status3 = sten.bicgstab_solve(st, sten.MIXED, b, None, 1e-3, 200, x2)
    assert status3 == sten.CONVERGED and hist3[-1] <= 1e-3 < hist3[-2] and it3 <= 15
    assert np.array_equal(hist3, hist[: it3 + 1])
    bf = ic.uniform_device(NX, NY, NZ, seed=1, stream=0).float()
    xf = torch.empty_like(bf)
    itf, histf, statusf = sten.bicgstab_solve(st, sten.FP32, bf, None, 1e-6, 500, xf)
    assert statusf == sten.CONVERGED and histf[-1] <= 1e-6 and itf < 40
    ax = torch.empty_like(xf)
    sten.stencil_apply(st, sten.FP32, xf, ax)
    dg, _ = ic.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
    bh = (bf.double() / dg).float()
    del dg
    tr = float(torch.linalg.vector_norm((bh - ax).double()) / torch.linalg.vector_norm(bh.double()))
    assert tr <= 1e-5, tr
    sten.set_schedule(st, sten.SCHED_CLASSIC)
