"""The 2D 9-point SpMV at the paper's 2D geometry, 22800 x 22800, in the launch
configuration tools/bench_2d.py times - parity on SAMPLED outputs (the oracle cannot hold the
mesh): for each sampled point the oracle scales (o64_jacobi_scale9) and applies (the o16 / o32
FMA-chain mirrors) the 3x3 window around it, clipped to the mesh, built from the global generator
(inputs.field_at_2d); the centre value of the window is exactly the full-mesh value.  Samples
cover the mesh corners and edges, the CTA tile edges (x = 127/128 fp16 or 63/64 fp32, y = 31/32)
and random interior points.  The paper's tiled output-halo form at 600 x 600 tiles (the 38 x 38
per-core sub-blocks of PAPER.md:371) is checked against the gather: bitwise where the stencil stays
inside one tile, within the fp64 tolerance of the window on the tile edges (R24)."""
import numpy as np
import pytest

import inputs
import oracle as orc
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

N = 22800


@pytest.fixture(scope="module")
def setup():
    torch = torch_cuda()
    import inputs.cuda as icuda
    import paper_2010_03660_b200 as sten
    diag, offs = icuda.fields2d_device(N, N, seed=1, delta=0.1)
    st = sten.stencil2d_create(N, N, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    v64 = icuda.uniform_device(N, N, 1, seed=3, stream=0).view(N, N)
    yield sten, st, v64
    st.close()


def points(rng, bx):
    pts = set()
    for x in (0, 1, bx - 1, bx, 2 * bx - 1, 2 * bx, N - 2, N - 1):
        for y in (0, 1, 31, 32, 63, 64, N - 2, N - 1):
            pts.add((x, y))
    for _ in range(300):
        pts.add((int(rng.integers(N)), int(rng.integers(N))))
    return sorted(pts)


def window(pt, v_dev, prec):
    """(oracle value of A_hat v at pt, its fp64 value, |v_P| + sum_d |c_d v_nb|) from the clipped 3x3
    window; v read back from the device (the values the kernel used)."""
    x, y = pt
    x0, x1, y0, y1 = max(x - 1, 0), min(x + 2, N), max(y - 1, 0), min(y + 2, N)
    j, i = np.meshgrid(np.arange(y0, y1), np.arange(x0, x1), indexing="ij")
    diag, offs = inputs.field_at_2d(N, i, j, seed=1, delta=0.1)
    cq = orc.quantize_coeffs(orc.jacobi_scale9(diag, offs), prec)
    v = v_dev[y0:y1, x0:x1].cpu().numpy()
    if prec == "fp32":
        u = orc.apply9_32(cq, v)
        cw, vw = [a.astype(np.float64) for a in cq], v.astype(np.float64)
    else:
        v16 = v.view(np.uint16)
        u = orc.apply9_16(cq, v16).view(np.float16)
        cw, vw = [orc.f16_to_double(a) for a in cq], orc.f16_to_double(v16)
    u64 = orc.apply9_64(cw, vw)
    mag = orc.apply9_64([np.abs(a) for a in cw], np.abs(vw))  # |v_P| + sum |c_d v_nb|
    return u[y - y0, x - x0], u64[y - y0, x - x0], mag[y - y0, x - x0]


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
def test_apply9_fullsize_sampled_bitwise(setup, prec):
    torch = torch_cuda()
    sten, st, v64 = setup
    v = v64.to(torch.float16 if prec == "mixed" else torch.float32)
    u = torch.empty_like(v)
    sten.stencil2d_apply(st, sten.MIXED if prec == "mixed" else sten.FP32, v, u)
    bx = 128 if prec == "mixed" else 64
    bad = []
    for pt in points(np.random.default_rng(7), bx):
        ref, _, _ = window(pt, v, prec)
        got = u[pt[1], pt[0]].item()
        if not (float(got) == float(ref)):
            bad.append((pt, got, float(ref)))
    assert not bad, bad[:10]


@pytest.mark.parametrize("prec", ["mixed", "fp32"])
def test_tiled_600x600_fullsize_against_gather(setup, prec):
    torch = torch_cuda()
    sten, st, v64 = setup
    v = v64.to(torch.float16 if prec == "mixed" else torch.float32)
    P = sten.MIXED if prec == "mixed" else sten.FP32
    ug, ut = torch.empty_like(v), torch.empty_like(v)
    sten.stencil2d_set_tiles(st, 1, 1)
    sten.stencil2d_apply(st, P, v, ug)
    sten.stencil2d_set_tiles(st, 600, 600)
    try:
        sten.stencil2d_apply(st, P, v, ut)
    finally:
        sten.stencil2d_set_tiles(st, 1, 1)
    edges = np.array([(a * N) // 600 for a in range(1, 600)])
    on_edge = torch.zeros(N, dtype=torch.bool, device="cuda")
    e = torch.from_numpy(edges).cuda()
    on_edge[e] = True
    on_edge[e - 1] = True
    interior = ~(on_edge[:, None] | on_edge[None, :])
    # bitwise where the stencil stays inside one tile (the FMA chain of the gather)
    assert torch.equal(ug[interior], ut[interior])
    # tile edges: the output-halo sums within the componentwise rounding bound of their 13
    # roundings (8 FMAs, up to 4 halo additions, the +0 start) against fp64: |d| <= 13 eps m,
    # m = |v_P| + sum |c_d v_nb| (R19's componentwise check, with the tiled form's extra adds)
    rng = np.random.default_rng(11)
    eps = 2.0 ** -11 if prec == "mixed" else 2.0 ** -24
    checked = 0
    for _ in range(400):
        xe = int(edges[rng.integers(len(edges))]) - int(rng.integers(2))
        y = int(rng.integers(N))
        for pt in ((xe, y), (y, xe)):
            _, ref64, mag = window(pt, v, prec)
            got = float(ut[pt[1], pt[0]].item())
            assert abs(got - ref64) <= 13 * eps * mag, (pt, got, ref64, mag)
            checked += 1
    assert checked == 800
    # and the edge values really are the output-halo sums, not the gather's chain (some differ)
    assert not torch.equal(ug[~interior], ut[~interior])


def test_solve_fullsize_properties():
    """BiCGStab on the 2D operator at 22800 x 22800 (the bench's `next3_2d` configuration), mixed: the
    tol = 1e-3 run converges in a handful of iterations, deterministically, and x's true residual
    of the scaled system - b_hat = b / a_P and A_hat x through the library's fp32 apply, the
    difference and the norms in fp64 - is at the mixed level (as for the small meshes)."""
    torch = torch_cuda()
    import inputs.cuda as icuda
    import paper_2010_03660_b200 as sten
    diag, offs = icuda.fields2d_device(N, N, seed=1, delta=0.1)
    st = sten.stencil2d_create(N, N, [diag] + offs)
    del offs
    b64 = icuda.uniform_device(N, N, 1, seed=1, stream=0).view(N, N)
    b16 = b64.to(torch.float16)
    x = torch.empty_like(b16)
    it, hist, status = sten.bicgstab2d_solve(st, sten.MIXED, b16, None, 1e-3, 100, x)
    assert status == sten.CONVERGED and hist[-1] <= 1e-3 and it <= 20, (it, hist, status)
    x2 = torch.empty_like(b16)
    it2, hist2, status2 = sten.bicgstab2d_solve(st, sten.MIXED, b16, None, 1e-3, 100, x2)
    assert (it2, status2) == (it, status) and np.array_equal(hist2, hist) and torch.equal(x2.view(torch.int16),
                                                                                          x.view(torch.int16))
    y = torch.empty((N, N), dtype=torch.float32, device="cuda")
    sten.stencil2d_apply(st, sten.FP32, x.float(), y)
    bh = (b16.double() / diag.double().view(N, N)).half().double()  # b_hat = rn16(b / a_P) (R3)
    true = float(torch.linalg.vector_norm(bh - y.double()) / torch.linalg.vector_norm(bh))
    assert true <= 1e-2, true
    st.close()
