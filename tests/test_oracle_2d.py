"""Pins for the 2D 9-point oracle (oracle/o2d.c, NEXT-3): the gather
SpMV, the paper's tiled form with the output-halo rounds x then y (R24), and BiCGStab on the
2D operator (R25: dense LAPACK solve, Krylov termination on a closed-form eigenvector, A = I,
the true-vs-recurrence residual invariant, x0, the binary16 plateau).

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


# ------------------------------------------- the paper's tiled form (R24) --
TILINGS = [(1, 1), (2, 1), (1, 3), (2, 3), (3, 2), "cols", "points"]


def _grid(t, nx, ny):
    return (nx, 1) if t == "cols" else ((nx, ny) if t == "points" else t)


@pytest.mark.parametrize("mesh", [(9, 7), (1, 5), (6, 1), (13, 11)])
@pytest.mark.parametrize("tiling", TILINGS)
def test_tiled_apply_exact_on_dyadic_inputs(orc, mesh, tiling):
    """Couplings and v on the k/64 grid: every product and partial sum is exact in fp64 and fp32,
    so the tiled form (any tile grid, down to one point per tile) equals the dense product."""
    nx, ny = mesh
    TX, TY = _grid(tiling, nx, ny)
    if TX > nx or TY > ny:
        pytest.skip("more tiles than points")
    rng = np.random.default_rng(nx * 13 + ny)
    offs = [rng.integers(-64, 65, (ny, nx)) / 64.0 for _ in range(8)]
    c = orc.jacobi_scale9(None, offs)
    v = rng.integers(-64, 65, (ny, nx)) / 64.0
    want = dense9(None, offs) @ v.ravel()
    assert np.array_equal(orc.apply9_tiles(c, v, (TX, TY), "fp64").ravel(), want)
    c32 = [a.astype(np.float32) for a in c]
    got32 = orc.apply9_tiles(c32, v.astype(np.float32), (TX, TY), "fp32")
    assert np.array_equal(got32.ravel().astype(np.float64), want)


@pytest.mark.parametrize("tiling", TILINGS)
def test_tiled_apply_random_fp64_and_fp16_bounds(orc, tiling):
    nx, ny = 17, 12
    TX, TY = _grid(tiling, nx, ny)
    rng = np.random.default_rng(3)
    diag = rng.uniform(1.0, 3.0, (ny, nx))
    offs = [rng.uniform(-1, 1, (ny, nx)) for _ in range(8)]
    c = orc.jacobi_scale9(diag, offs)
    v = rng.uniform(-1, 1, (ny, nx))
    M = dense9(diag, offs)
    scale = (np.abs(M) @ np.abs(v.ravel())).reshape(ny, nx)
    assert np.all(np.abs(orc.apply9_tiles(c, v, (TX, TY), "fp64") - (M @ v.ravel()).reshape(ny, nx))
                  <= 16 * 2.0 ** -53 * scale)
    # binary16: at most 8 FMA roundings + 4 halo additions per output, each <= u = 2^-11 relative
    c16 = orc.quantize_coeffs(c, "mixed")
    v16 = orc.f16_from_double(v)
    u16 = orc.f16_to_double(orc.apply9_tiles(c16, v16, (TX, TY), "mixed"))
    cq = [orc.f16_to_double(a) for a in c16]
    exact = orc.apply9_64(cq, orc.f16_to_double(v16))
    sc = np.abs(orc.f16_to_double(v16)) + sum(np.abs(a) for a in cq) * np.max(np.abs(v))
    assert np.all(np.abs(u16 - exact) <= 13 * 2.0 ** -11 * sc)


def test_tiled_apply_one_tile_is_the_fma_chain(orc):
    """One tile: no exchange, every in-mesh product enters the chain in the d order - the
    GPU's gather mirror (equal up to the sign of zero)."""
    nx, ny = 11, 9
    rng = np.random.default_rng(4)
    c = orc.jacobi_scale9(rng.uniform(1.0, 3.0, (ny, nx)), [rng.uniform(-1, 1, (ny, nx)) for _ in range(8)])
    c16 = orc.quantize_coeffs(c, "mixed")
    v16 = orc.f16_from_double(rng.uniform(-1, 1, (ny, nx)))
    assert np.array_equal(orc.f16_to_double(orc.apply9_tiles(c16, v16, (1, 1), "mixed")),
                          orc.f16_to_double(orc.apply9_16(c16, v16)))
    c32 = orc.quantize_coeffs(c, "fp32")
    v32 = rng.uniform(-1, 1, (ny, nx)).astype(np.float32)
    assert np.array_equal(orc.apply9_tiles(c32, v32, (1, 1), "fp32"), orc.apply9_32(c32, v32))


def test_tiled_apply_round_order_at_a_tile_corner(orc):
    """2 x 2 tiles, the point P at the lower-left corner of the upper-right tile: its value is
    ((own chain + left tile's chain) + (lower tile's chain + lower-left tile's chain)) - the x round,
    then the y round carrying the diagonal product - composed here from the pinned
    binary16 fma/add on single points."""
    nx, ny = 6, 6  # tiles split at x = 3, y = 3
    rng = np.random.default_rng(9)
    c = orc.jacobi_scale9(rng.uniform(1.0, 3.0, (ny, nx)), [rng.uniform(-1, 1, (ny, nx)) for _ in range(8)])
    c16 = orc.quantize_coeffs(c, "mixed")
    v16 = orc.f16_from_double(rng.uniform(-1, 1, (ny, nx)))
    i, j = 3, 3
    owner = lambda ii, jj: (ii >= 3, jj >= 3)  # noqa: E731

    def chain(tile, start):
        acc = np.uint16(start)
        for d, (dx, dy) in enumerate(D9):
            ii, jj = i + dx, j + dy
            if 0 <= ii < nx and 0 <= jj < ny and owner(ii, jj) == tile:
                acc = orc.fma16_array(np.array([c16[d][j, i]]), np.array([v16[jj, ii]]), np.array([acc]))[0]
        return acc

    own = chain((True, True), v16[j, i])
    left, below, belowleft = chain((False, True), 0), chain((True, False), 0), chain((False, False), 0)
    add = lambda a, b: orc.add16_array(np.array([a], np.uint16), np.array([b], np.uint16))[0]  # noqa: E731
    want = add(add(own, left), add(below, belowleft))
    got = orc.apply9_tiles(c16, v16, (2, 2), "mixed")[j, i]
    assert orc.f16_to_double(np.array([got]))[0] == orc.f16_to_double(np.array([want]))[0]


# ------------------------------------------------------ 2D BiCGStab (R25) --
def _cd2d(orc, nx, ny, delta=0.1, seed=1):
    """The seeded 2D stand-in (inputs.problem_fields_2d) and its scaled couplings."""
    import inputs
    diag, offs = inputs.problem_fields_2d(nx, ny, seed=seed, delta=delta)
    return diag, offs, orc.jacobi_scale9(diag, offs)


@pytest.mark.parametrize("delta", [0.1, 0.0])
def test_bicgstab2d_matches_lapack(orc, delta):
    nx, ny = 12, 9
    diag, offs, c = _cd2d(orc, nx, ny, delta)
    import inputs
    b = inputs.rhs_uniform_2d(nx, ny, seed=2) / diag
    M = dense9(diag, offs)
    x_ref = np.linalg.solve(M, b.ravel())
    r = orc.bicgstab2d(c, b, tol=1e-13, maxit=500)
    assert r["status"] == orc.ORC_CONVERGED
    assert np.linalg.norm(r["x"].ravel() - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_bicgstab2d_krylov_termination_and_identity(orc):
    nx, ny = 11, 8
    diag = np.full((ny, nx), 8.0)
    offs = [np.full((ny, nx), -1.0) for _ in range(8)]
    c = orc.jacobi_scale9(diag, offs)
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    ta, tb = 2 * np.pi / (nx + 1), 3 * np.pi / (ny + 1)
    phi = np.sin(ta * (i + 1)) * np.sin(tb * (j + 1))
    lam = 1.0 - (2 * np.cos(ta) + 2 * np.cos(tb) + 4 * np.cos(ta) * np.cos(tb)) / 8.0
    r = orc.bicgstab2d(c, phi, tol=0.0, maxit=1)
    assert r["hist"][1] <= 1e-14 and np.max(np.abs(r["x"] - phi / lam)) <= 1e-13
    z = [np.zeros((ny, nx)) for _ in range(8)]
    b = np.random.default_rng(1).uniform(-1, 1, (ny, nx))
    r = orc.bicgstab2d(z, b, tol=1e-8, maxit=10)
    assert r["iters"] == 1 and r["status"] == orc.ORC_CONVERGED and np.array_equal(r["x"], b)
    b16 = orc.f16_from_double(b)
    r16 = orc.bicgstab2d([np.zeros((ny, nx), np.uint16)] * 8, b16, tol=1e-8, maxit=10, prec="mixed")
    assert r16["iters"] == 1 and np.array_equal(r16["x"], b16)


def test_bicgstab2d_true_vs_recurrence_residual_and_x0(orc):
    nx, ny = 20, 17
    diag, offs, c = _cd2d(orc, nx, ny, 0.0, seed=3)
    import inputs
    b = inputs.rhs_uniform_2d(nx, ny, seed=3) / diag
    nb = np.linalg.norm(b)
    for maxit in (1, 5, 20, 30):
        r = orc.bicgstab2d(c, b, tol=0.0, maxit=maxit)
        true = np.linalg.norm(b - orc.apply9_64(c, r["x"])) / nb
        assert abs(true - r["hist"][-1]) <= 1e-10, (maxit, true, r["hist"][-1])
    full = orc.bicgstab2d(c, b, tol=1e-10, maxit=400)
    x0 = full["x"] + 1e-3 * np.random.default_rng(0).uniform(-1, 1, (ny, nx))
    r = orc.bicgstab2d(c, b, x0=x0, tol=1e-10, maxit=400)
    assert r["status"] == orc.ORC_CONVERGED and r["iters"] < full["iters"]


def test_bicgstab2d_mixed_tracks_fp64_then_plateaus(orc):
    """The binary16 mode follows fp64 for the first iterations and reaches 1e-3 (the R15 reading
    on a delta = 0.1 system), with its true residual on the fp16 plateau."""
    nx, ny = 48, 40
    diag, offs, c = _cd2d(orc, nx, ny, 0.1, seed=4)
    import inputs
    b = inputs.rhs_uniform_2d(nx, ny, seed=4)
    c16 = orc.quantize_coeffs(c, "mixed")
    b16 = orc.f16_from_double(b / diag)
    r64 = orc.bicgstab2d([orc.f16_to_double(a) for a in c16], orc.f16_to_double(b16), tol=0.0, maxit=6)
    r16 = orc.bicgstab2d(c16, b16, tol=0.0, maxit=6, prec="mixed")
    assert np.all(np.abs(r16["hist"][:6] - r64["hist"][:6]) <= 2e-2 * r64["hist"][:6])
    r16 = orc.bicgstab2d(c16, b16, tol=1e-3, maxit=100, prec="mixed")
    assert r16["status"] == orc.ORC_CONVERGED and r16["hist"][-1] <= 1e-3
    x = orc.f16_to_double(r16["x"])
    bb = orc.f16_to_double(b16)
    true = np.linalg.norm(bb - orc.apply9_64([orc.f16_to_double(a) for a in c16], x)) / np.linalg.norm(bb)
    assert 1e-4 < true < 1e-2


# ------------------------------- 2D BiCGStab on the tiled SpMV (R24, R25) --
@pytest.mark.parametrize("tiles", [(2, 1), (3, 2), (5, 4), (12, 9)])
def test_bicgstab2d_tiled_matches_lapack_and_gather(orc, tiles):
    """The solve on the paper's tiled output-halo SpMV is the same algorithm on the same operator:
    it converges to LAPACK's solution, and its fp64 iterates follow the gather solve's to rounding
    (the tiling only re-associates the nine products at tile edges)."""
    nx, ny = 12, 9
    diag, offs, c = _cd2d(orc, nx, ny, 0.1)
    import inputs
    b = inputs.rhs_uniform_2d(nx, ny, seed=2) / diag
    x_ref = np.linalg.solve(dense9(diag, offs), b.ravel())
    r = orc.bicgstab2d(c, b, tol=1e-13, maxit=500, tiles=tiles)
    assert r["status"] == orc.ORC_CONVERGED
    assert np.linalg.norm(r["x"].ravel() - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
    g = orc.bicgstab2d(c, b, tol=0.0, maxit=8)
    t = orc.bicgstab2d(c, b, tol=0.0, maxit=8, tiles=tiles)
    assert np.allclose(t["hist"], g["hist"], rtol=1e-12, atol=0)
    assert np.allclose(t["alpha"], g["alpha"], rtol=1e-12) and np.allclose(t["omega"], g["omega"], rtol=1e-12)


def test_bicgstab2d_tiled_one_tile_is_the_gather(orc):
    """tiles (1, 1) is the gather solve bitwise, in both precisions (one tile: no output halo)."""
    nx, ny = 20, 13
    diag, offs, c = _cd2d(orc, nx, ny, 0.1, seed=5)
    import inputs
    b = inputs.rhs_uniform_2d(nx, ny, seed=5) / diag
    a = orc.bicgstab2d(c, b, tol=0.0, maxit=10)
    t = orc.bicgstab2d(c, b, tol=0.0, maxit=10, tiles=(1, 1))
    assert np.array_equal(a["x"], t["x"]) and np.array_equal(a["hist"], t["hist"])
    c16, b16 = orc.quantize_coeffs(c, "mixed"), orc.f16_from_double(b)
    a = orc.bicgstab2d(c16, b16, tol=0.0, maxit=10, prec="mixed")
    t = orc.bicgstab2d(c16, b16, tol=0.0, maxit=10, prec="mixed", tiles=(1, 1))
    assert np.array_equal(a["x"], t["x"]) and np.array_equal(a["hist"], t["hist"])


def test_bicgstab2d_tiled_mixed_first_step_composes_pinned_primitives(orc):
    """One binary16 iteration on tiles, recomputed here from the pinned pieces (the tiled fp16
    SpMV apply9_tiles, exact binary16 FMA, fp32 dots of exact products): x_1 and hist[1] equal."""
    nx, ny, tiles = 17, 11, (3, 2)
    diag, offs, c = _cd2d(orc, nx, ny, 0.1, seed=6)
    import inputs
    c16 = orc.quantize_coeffs(c, "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform_2d(nx, ny, seed=6))
    r = orc.bicgstab2d(c16, b16, tol=0.0, maxit=1, prec="mixed", tiles=tiles)
    f = lambda a: orc.f16_to_double(a).astype(np.float32)

    def dot(a, b):  # per row in fp32, then over rows (o2d.c dot16_9)
        tot = np.float32(0)
        for j in range(ny):
            row = np.float32(0)
            for i in range(nx):
                row = np.float32(row + f(a)[j, i] * f(b)[j, i])
            tot = np.float32(tot + row)
        return tot
    rho = dot(b16, b16)
    v = orc.apply9_tiles(c16, b16, tiles, "mixed")
    alpha = np.float32(rho / dot(b16, v))
    ah = orc.f16_from_double(np.float64(alpha))
    neg = lambda h: np.uint16(h ^ 0x8000)
    s = orc.fma16_array(np.full_like(v, neg(ah)), v, b16)
    t = orc.apply9_tiles(c16, s, tiles, "mixed")
    omega = np.float32(dot(t, s) / dot(t, t))
    wh = orc.f16_from_double(np.float64(omega))
    x = orc.fma16_array(np.full_like(s, wh), s, orc.fma16_array(np.full_like(b16, ah), b16, np.zeros_like(b16)))
    assert np.array_equal(r["x"], x)
    rr = orc.fma16_array(np.full_like(t, neg(wh)), t, s)
    assert r["hist"][1] == np.sqrt(np.float64(dot(rr, rr))) / np.sqrt(np.float64(rho))
