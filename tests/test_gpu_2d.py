"""GPU parity of the 2D 9-point SpMV (stencil2d_apply, NEXT-3) against oracle/o2d.c:
bitwise against the fp32 / fp16 FMA-chain mirrors on meshes with several tiles and
ragged tails, and max|du|/max|u| <= 1e-6 (fp32) / 2e-3 (fp16) against fp64 on the
same quantised inputs (the north_star SpMV tolerances, R9)."""
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


@pytest.mark.parametrize("prec", ["fp32", "mixed"])
@pytest.mark.parametrize("mesh", [(1, 1), (7, 5), (130, 33), (264, 70), (8, 300), (128, 32), (129, 65)])
@pytest.mark.parametrize("with_diag", [True, False])
def test_apply9_bitwise_and_tolerance(sten, prec, mesh, with_diag):
    torch = torch_cuda()
    nx, ny = mesh
    rng = np.random.default_rng(nx * 7 + ny)
    diag = rng.uniform(2.0, 4.0, (ny, nx)) if with_diag else None
    offs = [rng.uniform(-1, 1, (ny, nx)) * (0.25 if not with_diag else 1.0) for _ in range(8)]
    coeffs = [None if diag is None else torch.from_numpy(diag).cuda()] + [torch.from_numpy(o).cuda() for o in offs]
    st = sten.stencil2d_create(nx, ny, coeffs)
    c64 = orc.jacobi_scale9(diag, offs)
    cq = orc.quantize_coeffs(c64, prec)
    v64 = rng.uniform(-1, 1, (ny, nx))
    if prec == "fp32":
        v = v64.astype(np.float32)
        vt = torch.from_numpy(v).cuda()
        mirror = orc.apply9_32(cq, v)
    else:
        v = orc.f16_from_double(v64)
        vt = torch.from_numpy(v.view(np.float16)).cuda()
        mirror = orc.apply9_16(cq, v)
    yt = torch.empty_like(vt)
    ms = sten.stencil2d_apply(st, sten.FP32 if prec == "fp32" else sten.MIXED, vt, yt)
    assert ms >= 0.0
    y = yt.cpu().numpy()
    wide = (lambda a: a.astype(np.float64)) if prec == "fp32" else (lambda a: orc.f16_to_double(a.view(np.uint16)))
    assert np.array_equal(wide(y), wide(mirror if prec == "fp32" else mirror.view(np.float16)))
    u64 = orc.apply9_64([wide(a if prec == "fp32" else a.view(np.float16)) for a in cq], wide(v if prec == "fp32" else v.view(np.float16)))
    err = np.max(np.abs(wide(y) - u64)) / max(np.max(np.abs(u64)), 1e-300)
    assert err <= (1e-6 if prec == "fp32" else 2e-3)
    st.close()


def test_apply9_host_buffers_and_invalid(sten):
    torch = torch_cuda()
    nx, ny = 50, 20
    offs = [np.full((ny, nx), -0.1) for _ in range(8)]
    st = sten.stencil2d_create(nx, ny, [None] + offs)  # host coefficients
    x = np.random.default_rng(1).uniform(-1, 1, (ny, nx)).astype(np.float32)
    y = np.empty_like(x)
    sten.stencil2d_apply(st, sten.FP32, x, y)  # host vectors
    c32 = orc.quantize_coeffs(orc.jacobi_scale9(None, offs), "fp32")
    assert np.array_equal(y, orc.apply9_32(c32, x))
    st.close()
    with pytest.raises(sten.StenError):
        sten.stencil2d_create(0, 5, [None] + offs)
    del torch
