"""Pins for the 2D 9-point SpMV oracle (oracle/o2d.c, NEXT-3).

Independent references: a dense matrix assembled here by neighbour
enumeration (brute force), the closed-form eigenpairs of the 9-point
Laplacian on a rectangle, zero couplings = identity, and the fp16/fp32 mirrors
as the composition of the pinned single-rounding FMA primitives.
"""
import numpy as np
import pytest

D9 = [(-1, -1), (0, -1), (1, -1), (-1, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]


def dense9(diag, offs):
    ny, nx = offs[0].shape
    M = np.zeros((nx * ny, nx * ny))
    for j in range(ny):
        for i in range(nx):
            P = i + nx * j
            M[P, P] = 1.0
            for d, (dx, dy) in enumerate(D9):
                ii, jj = i + dx, j + dy
                if 0 <= ii < nx and 0 <= jj < ny:
                    M[P, ii + nx * jj] += offs[d][j, i] / (diag[j, i] if diag is not None else 1.0)
    return M


@pytest.mark.parametrize("mesh", [(1, 1), (1, 5), (4, 1), (3, 4), (9, 7), (16, 12)])
def test_apply9_matches_dense_assembly(orc, mesh):
    nx, ny = mesh
    rng = np.random.default_rng(nx * 31 + ny)
    diag = rng.uniform(1.0, 3.0, (ny, nx))
    offs = [rng.uniform(-1, 1, (ny, nx)) for _ in range(8)]
    c = orc.jacobi_scale9(diag, offs)
    v = rng.uniform(-1, 1, (ny, nx))
    M = dense9(diag, offs)
    scale = np.abs(M) @ np.abs(v.ravel())
    assert np.all(np.abs(orc.apply9_64(c, v).ravel() - M @ v.ravel()) <= 1e-15 * 10 * scale + 1e-300)
    for d, (dx, dy) in enumerate(D9):  # couplings leaving the mesh are exactly +0
        for j in range(ny):
            for i in range(nx):
                inside = 0 <= i + dx < nx and 0 <= j + dy < ny
                assert c[d][j, i] == (offs[d][j, i] / diag[j, i] if inside else 0.0)


@pytest.mark.parametrize("ab", [(1, 1), (2, 3), (5, 1)])
def test_nine_point_laplacian_eigenpairs(orc, ab):
    # A = 8 I - (all 8 neighbours), scaled by 1/8: eigenvectors sin(a pi (i+1)/(nx+1)) sin(b pi (j+1)/(ny+1)),
    # lambda = 1 - (2 cos ta + 2 cos tb + 4 cos ta cos tb) / 8  (product structure of the 3x3 all-ones stencil)
    nx, ny = 11, 8
    a, b = ab
    diag = np.full((ny, nx), 8.0)
    offs = [np.full((ny, nx), -1.0) for _ in range(8)]
    c = orc.jacobi_scale9(diag, offs)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    ta, tb = a * np.pi / (nx + 1), b * np.pi / (ny + 1)
    f = np.sin(ta * (i + 1)) * np.sin(tb * (j + 1))
    lam = 1.0 - (2 * np.cos(ta) + 2 * np.cos(tb) + 4 * np.cos(ta) * np.cos(tb)) / 8.0
    assert np.max(np.abs(orc.apply9_64(c, f) - lam * f)) <= 1e-14


def test_zero_couplings_identity(orc):
    rng = np.random.default_rng(2)
    v = rng.uniform(-1, 1, (6, 7))
    c = [np.zeros((6, 7)) for _ in range(8)]
    assert np.array_equal(orc.apply9_64(c, v), v)
    v16 = orc.f16_from_double(v)
    assert np.array_equal(orc.apply9_16([np.zeros((6, 7), np.uint16)] * 8, v16), v16)


def test_mirrors_are_fma_chains(orc):
    """fp16 mirror = the pinned binary16 fma applied term by term in the stated order;
    fp32 mirror within one rounding per term of the fp64 result."""
    nx, ny = 9, 6
    rng = np.random.default_rng(5)
    diag = rng.uniform(1.0, 3.0, (ny, nx))
    offs = [rng.uniform(-1, 1, (ny, nx)) for _ in range(8)]
    c = orc.jacobi_scale9(diag, offs)
    c16 = orc.quantize_coeffs(c, "mixed")
    v16 = orc.f16_from_double(rng.uniform(-1, 1, (ny, nx)))
    acc = v16.copy()
    for d, (dx, dy) in enumerate(D9):
        nb = np.zeros_like(v16)
        ys, ye = max(0, -dy), ny - max(0, dy)
        xs, xe = max(0, -dx), nx - max(0, dx)
        nb[ys:ye, xs:xe] = v16[ys + dy:ye + dy, xs + dx:xe + dx]
        acc = orc.fma16_array(c16[d], nb, acc)
    assert np.array_equal(orc.apply9_16(c16, v16), acc)
    c32 = orc.quantize_coeffs(c, "fp32")
    v32 = rng.uniform(-1, 1, (ny, nx)).astype(np.float32)
    u32 = orc.apply9_32(c32, v32)
    u64 = orc.apply9_64([a.astype(np.float64) for a in c32], v32.astype(np.float64))
    scale = sum(np.abs(a.astype(np.float64)) for a in c32) + 1.0
    assert np.all(np.abs(u32 - u64) <= 9 * 2.0 ** -24 * scale * np.max(np.abs(v32)))
