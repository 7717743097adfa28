"""GPU parity of the paper's tiled 2D SpMV (stencil2d_set_tiles + stencil2d_apply; NEXT-3,
PAPER.md:364-368, R24) against oracle/o2d.c apply9_tiles: bitwise against the fp32 /
fp16 mirrors of the output-halo algorithm (local products into the grown region, x round, then y
round) on tile grids with ragged, width-1 and height-1 tiles and with tiles spanning several CTAs;
fp64 tolerance of the result; the invalid tile counts; switching back to the gather."""
import numpy as np
import pytest

import oracle as orc
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def _case(nx, ny, seed, with_diag=True):
    rng = np.random.default_rng(seed)
    diag = rng.uniform(2.0, 4.0, (ny, nx)) if with_diag else None
    offs = [rng.uniform(-1, 1, (ny, nx)) * (1.0 if with_diag else 0.25) for _ in range(8)]
    v64 = rng.uniform(-1, 1, (ny, nx))
    return diag, offs, v64


def _wide(a, prec):
    return a.astype(np.float64) if prec == "fp32" else orc.f16_to_double(a.view(np.uint16))


CASES = [
    ((7, 5), (2, 1)), ((7, 5), (1, 2)), ((7, 5), (3, 2)), ((7, 5), (7, 5)), ((7, 5), (5, 4)),
    ((1, 1), (1, 1)), ((2, 9), (2, 9)), ((40, 3), (6, 3)),
    ((130, 33), (4, 5)), ((264, 70), (3, 3)), ((129, 65), (2, 7)), ((300, 8), (1, 8)), ((8, 300), (8, 1)),
    ((257, 129), (16, 9)),
]


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("mesh,tiles", CASES)
def test_tiled_apply_bitwise(sten, prec, mesh, tiles):
    torch = torch_cuda()
    nx, ny = mesh
    diag, offs, v64 = _case(nx, ny, nx * 31 + ny * 7 + tiles[0])
    coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
    st = sten.stencil2d_create(nx, ny, coeffs)
    sten.stencil2d_set_tiles(st, *tiles)
    cq = orc.quantize_coeffs(orc.jacobi_scale9(diag, offs), prec)
    if prec == "fp32":
        v = v64.astype(np.float32)
        vt = torch.from_numpy(v).cuda()
    else:
        v = orc.f16_from_double(v64)
        vt = torch.from_numpy(v.view(np.float16)).cuda()
    mirror = orc.apply9_tiles(cq, v, tiles, prec)
    yt = torch.empty_like(vt)
    sten.stencil2d_apply(st, sten.FP32 if prec == "fp32" else sten.MIXED, vt, yt)
    y = yt.cpu().numpy()
    if prec == "mixed":
        y = y.view(np.uint16)
    # bit patterns (signed zeros included: the tiled form skips out-of-tile terms, R24)
    assert np.array_equal(y.view(np.uint32 if prec == "fp32" else np.uint16),
                          mirror.view(np.uint32 if prec == "fp32" else np.uint16))
    # the tiled result is A v up to rounding: fp64 of the same quantised inputs
    c64 = [_wide(a, prec) for a in cq]
    u64 = orc.apply9_64(c64, _wide(v, prec))
    err = np.max(np.abs(_wide(y, prec) - u64)) / max(np.max(np.abs(u64)), 1e-300)
    assert err <= (1e-6 if prec == "fp32" else 2e-3)
    st.close()


def test_tiled_differs_from_gather_only_at_tile_edges(sten):
    """The output-halo sums round differently from the gather's FMA chain only at points whose
    stencil crosses a tile edge: interior points are bitwise the gather's."""
    torch = torch_cuda()
    nx, ny, TX, TY = 200, 90, 4, 3
    diag, offs, v64 = _case(nx, ny, 5)
    coeffs = [torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
    st = sten.stencil2d_create(nx, ny, coeffs)
    v = orc.f16_from_double(v64)
    vt = torch.from_numpy(v.view(np.float16)).cuda()
    yg, yt = torch.empty_like(vt), torch.empty_like(vt)
    sten.stencil2d_apply(st, sten.MIXED, vt, yg)
    sten.stencil2d_set_tiles(st, TX, TY)
    sten.stencil2d_apply(st, sten.MIXED, vt, yt)
    sten.stencil2d_set_tiles(st, 1, 1)  # back to the gather
    yg2 = torch.empty_like(vt)
    sten.stencil2d_apply(st, sten.MIXED, vt, yg2)
    assert torch.equal(yg.view(torch.int16), yg2.view(torch.int16))
    xe = {(a * nx) // TX for a in range(1, TX)}
    ye = {(b * ny) // TY for b in range(1, TY)}
    edge = np.zeros((ny, nx), bool)
    for x in xe:
        edge[:, x - 1:x + 1] = True
    for y in ye:
        edge[y - 1:y + 1, :] = True
    g = yg.cpu().numpy().view(np.uint16)
    t = yt.cpu().numpy().view(np.uint16)
    assert np.array_equal(g[~edge], t[~edge])
    assert np.any(g[edge] != t[edge])  # the rounding order really differs on the edges
    st.close()


def test_tiles_invalid(sten):
    nx, ny = 10, 4
    offs = [np.full((ny, nx), -0.1) for _ in range(8)]
    st = sten.stencil2d_create(nx, ny, [None] + offs)
    for tx, ty in [(0, 1), (1, 0), (11, 1), (1, 5), (-1, 2)]:
        with pytest.raises(sten.StenError):
            sten.stencil2d_set_tiles(st, tx, ty)
    sten.stencil2d_set_tiles(st, 10, 4)  # every tile one point
    x = np.random.default_rng(2).uniform(-1, 1, (ny, nx)).astype(np.float32)
    y = np.zeros_like(x)
    sten.stencil2d_apply(st, sten.FP32, x, y)
    cq = orc.quantize_coeffs(orc.jacobi_scale9(None, offs), "fp32")
    assert np.array_equal(y.view(np.uint32), orc.apply9_tiles(cq, x, (10, 4), "fp32").view(np.uint32))
    st.close()
