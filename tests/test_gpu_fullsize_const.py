"""The constant-coefficient classic path (NEXT-4, scalar-coupling tile kernels) at BASELINE.json's
full size, 600x595x1536, in the launch configuration `bench.py --operator poisson-const` times:
stencil_apply bitwise at sampled points (mesh corners and faces, tile edges, the chunk plan's
edges, random interior) against the oracle's FMA chain on the clipped 3x3x3 window of the
constant fields; a 12-iteration mixed solve (x and history) bitwise equal to the array kernels
on the same handle (STEN_OPT_CLASSIC_CONST = 0)."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import torch_cuda
from test_gpu_fullsize import NX, NY, NZ, chunk_edges, sample_points

pytestmark = pytest.mark.gpu
SKEW = (3.0, -0.7, -0.4, -0.25, -0.55, -0.3, -0.5)


@pytest.fixture(scope="module")
def const_problem():
    torch_cuda()
    import paper_2010_03660_b200 as sten
    st = sten.stencil_create_const(NX, NY, NZ, SKEW)
    yield st
    st.close()


def window_value(pt, vfull_fn, prec):
    x, y, z = pt
    x0, x1 = max(x - 1, 0), min(x + 2, NX)
    y0, y1 = max(y - 1, 0), min(y + 2, NY)
    z0, z1 = max(z - 1, 0), min(z + 2, NZ)
    kg, j, i = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag = np.full(i.shape, SKEW[0])
    offs = [np.full(i.shape, SKEW[1 + d]) for d in range(6)]
    # couplings leaving the window are dropped by jacobi_scale; the centre's all lie inside it
    # unless they leave the global mesh, where R5 drops them too
    cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
    u = orc.apply32_fma(cq, vfull_fn(i, j, kg)) if prec == "fp32" else orc.apply16(cq, vfull_fn(i, j, kg))
    return u[z - z0, y - y0, x - x0]


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
def test_fullsize_const_apply_sampled_bitwise(const_problem, prec):
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = const_problem
    P = sten.FP32 if prec == "fp32" else sten.MIXED
    assert sten.get_option(st, sten.OPT_CLASSIC_CONST) == 1
    v32 = ic.uniform_device(NX, NY, NZ, seed=3, stream=7, dtype="f32")
    vt = v32 if prec == "fp32" else v32.to(torch.float16)
    del v32
    yt = torch.empty_like(vt)
    sten.stencil_apply(st, P, vt, yt)
    torch.cuda.synchronize()

    def vfull(i, j, kg):
        idx = (i + NX * (j + NY * kg)).astype(np.uint64)
        v = inputs.uniform(3, 7, idx, -1.0, 1.0).astype(np.float32)
        return v if prec == "fp32" else orc.f16_from_double(v.astype(np.float64))

    pts = sample_points(np.random.default_rng(12), zs=chunk_edges(sten.classic_segments(st, P)))
    idx = torch.tensor([x + NX * (y + NY * z) for x, y, z in pts], device="cuda")
    got = yt.reshape(-1)[idx].cpu().numpy()
    if prec != "fp32":
        got = got.view(np.uint16)
    for k, pt in enumerate(pts):
        want = window_value(pt, vfull, prec)
        if prec == "fp32":
            a, b = float(got[k]), float(want)
        else:
            a = orc.f16_to_double(np.array([got[k]]))[0]
            b = orc.f16_to_double(np.array([want]))[0]
        assert a == b, (pt, a, b)


def test_fullsize_const_solve_equals_array_kernels(const_problem):
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = const_problem
    b = ic.uniform_device(NX, NY, NZ, seed=1, stream=0).to(torch.float16)
    out = []
    for opt in (1, 0):
        sten.set_option(st, sten.OPT_CLASSIC_CONST, opt)
        x = torch.empty_like(b)
        it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 12, x)
        out.append((x.float(), hist, it, status))
    sten.set_option(st, sten.OPT_CLASSIC_CONST, 1)
    assert out[0][2:] == out[1][2:]
    assert np.array_equal(out[0][1], out[1][1])
    assert torch.equal(out[0][0], out[1][0])
    assert np.all(np.isfinite(out[0][1])) and out[0][1][-1] < out[0][1][0]


def window_sr_const(pt, prec, streams, scal):
    """Oracle SR sweep (o16_sr_sweep / o32_sr_sweep) of the constant operator on the clipped 5x5x5
    window around one point (y' = A A p' reaches two points); the centre is the full-mesh value."""
    x, y, z = pt
    x0, x1 = max(x - 2, 0), min(x + 3, NX)
    y0, y1 = max(y - 2, 0), min(y + 3, NY)
    z0, z1 = max(z - 2, 0), min(z + 3, NZ)
    kg, j, i = np.meshgrid(np.arange(z0, z1), np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag = np.full(i.shape, SKEW[0])
    offs = [np.full(i.shape, SKEW[1 + d]) for d in range(6)]
    cq = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), prec)
    idx = (i + NX * (j + NY * kg)).astype(np.uint64)
    vec = {}
    for n, s_ in streams.items():
        v = inputs.uniform(5, s_, idx, -1.0, 1.0).astype(np.float32)
        vec[n] = v if prec == "fp32" else orc.f16_from_double(v.astype(np.float64))
    fn = orc.sr_sweep32 if prec == "fp32" else orc.sr_sweep16
    out = fn(cq, scal, vec["rh"], vec["x"], vec["r"], vec["p"], vec["v"], vec["q"], vec["y"])
    return [o[z - z0, y - y0, x - x0] for o in out[:6]]


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
def test_fullsize_const_sr_sweep_sampled_bitwise(const_problem, prec):
    """The constant-coefficient SR sweep (k_sr<CC>, the bench's `--operator poisson-const` SR field) at
    full size: x, r, p, v, q, y bitwise at sampled points (chunk edges of its own plan, tile edges of
    its 8-row tiles, faces, random) against the window oracle; the twelve sums against fp64
    reductions of the returned vectors."""
    torch = torch_cuda()
    import inputs.cuda as ic
    import paper_2010_03660_b200 as sten
    st = const_problem
    P = sten.FP32 if prec == "fp32" else sten.MIXED
    streams = dict(rh=7, x=8, r=9, p=10, v=11, q=12, y=13)
    scal = (0.61, 0.93, -0.27)
    ts = {}
    for n, s_ in streams.items():
        v32 = ic.uniform_device(NX, NY, NZ, seed=5, stream=s_, dtype="f32")
        ts[n] = v32 if prec == "fp32" else v32.to(torch.float16)
        del v32
    order = ["rh", "x", "r", "p", "v", "q", "y"]
    dots = sten.sr_sweep(st, P, scal, *[ts[n] for n in order])
    torch.cuda.synchronize()
    zs = chunk_edges(sten.sr_segments(st, P))
    rng = np.random.default_rng(23)
    pts = set()
    for x in (0, 1, 127, 128, 598, 599):
        for y in (0, 1, 7, 8, 15, 16, 593, 594):
            for z in zs:
                pts.add((x, y, z))
    for _ in range(300):
        pts.add((int(rng.integers(NX)), int(rng.integers(NY)), int(rng.integers(NZ))))
    pts = sorted(pts)
    idx = torch.tensor([x + NX * (y + NY * z) for x, y, z in pts], device="cuda")
    got = {n: ts[n].reshape(-1)[idx].cpu().numpy() for n in order[1:]}
    for n in order[1:]:
        if prec != "fp32":
            got[n] = got[n].view(np.uint16)
    wid = (lambda a: np.asarray(a, dtype=np.float64)) if prec == "fp32" else (lambda a: orc.f16_to_double(np.asarray(a)))
    for k, pt in enumerate(pts):
        want = window_sr_const(pt, prec, streams, scal)
        for n, w in zip(order[1:], want):
            assert float(wid([got[n][k]])[0]) == float(wid([w])[0]), (n, pt)
    d = {n: ts[n].double().reshape(-1) for n in ("rh", "r", "v", "q", "y")}
    pairs = [("rh", "v"), ("rh", "r"), ("rh", "q"), ("rh", "y"), ("q", "r"), ("q", "v"), ("y", "r"), ("y", "v"),
             ("q", "q"), ("q", "y"), ("y", "y"), ("r", "r")]
    for k, (a_, b_) in enumerate(pairs):
        exact = float(torch.dot(d[a_], d[b_]))
        scale = float(torch.dot(d[a_].abs(), d[b_].abs()))
        assert abs(float(dots[k]) - exact) <= 2e-5 * scale, (a_, b_, float(dots[k]), exact)
