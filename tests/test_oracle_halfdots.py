"""Pins of the half-dot oracle (oracle/osr.c o16h_*, R22; SURVEY §8(f)
NEXT-4: the paper's "16-bit mode", where a PE's core-local
dot over its z pencil runs in fp16 and the AllReduce stays 32-bit).

  * the textbook case that separates half from mixed accumulation (SPEC.md:43-44:
    2048 + 1 is 2048 in fp16, 2049 with a 32-bit add);
  * an independent pencil built from numpy's float16 rounding of exact fp64
    values (inputs k/64, so every product and sum is exact in fp64 before the
    one fp16 rounding), on a mesh with several ragged segments;
  * exactness while every running sum stays an fp16 integer (<= 2048);
  * one-plane segments: each pencil is one rounded product;
  * the half-dot SR sweep: its vectors equal the mixed sweep's bitwise, its
    twelve sums are the half dots of the vectors it returns;
  * the half-dot SR solve: A = I stops after one iteration with x = b exactly.
"""
import numpy as np
import pytest

import oracle as orc

SEG = [0, 3, 4, 9]  # ragged: lengths 3, 1, 5, nz - 9


def _vec(rng, shape, lo=-64, hi=64):
    return rng.integers(lo, hi + 1, shape).astype(np.float64) / 64.0


def test_textbook_2048_plus_1():
    a = orc.f16_from_double(np.array([2048.0, 1.0]).reshape(2, 1, 1))
    one = orc.f16_from_double(np.ones((2, 1, 1)))
    assert orc.dot16h(a, one, [0]) == (2048.0, 2048.0)        # fp16 pencil: 2048 + 1 rounds to 2048
    assert orc.dot16h(a, one, [0, 1]) == (2049.0, 2049.0)     # two pencils, added 32-bit
    assert float(orc.dot16(a, one)) == 2049.0                 # the mixed instruction


def test_pencils_match_numpy_float16_rounding():
    rng = np.random.default_rng(3)
    nz, ny, nx = 13, 5, 7
    a64, b64 = _vec(rng, (nz, ny, nx)), _vec(rng, (nz, ny, nx))
    a16, b16 = orc.f16_from_double(a64), orc.f16_from_double(b64)
    want, want_abs = 0.0, 0.0
    bounds = SEG + [nz]
    for j in range(ny):
        for i in range(nx):
            for s in range(len(SEG)):
                acc = np.float16(0.0)
                for k in range(bounds[s], bounds[s + 1]):
                    acc = np.float16(a64[k, j, i] * b64[k, j, i] + np.float64(acc))  # exact, then one rounding
                want += float(acc)
                want_abs += abs(float(acc))
    got, got_abs = orc.dot16h(a16, b16, SEG)
    assert got == want and got_abs == want_abs


def test_exact_while_sums_are_small_integers():
    rng = np.random.default_rng(4)
    nz, ny, nx = 40, 3, 4
    a = rng.integers(-6, 7, (nz, ny, nx)).astype(np.float64)
    b = rng.integers(-6, 7, (nz, ny, nx)).astype(np.float64)  # |running sum| <= 40 * 36 < 2048
    got, _ = orc.dot16h(orc.f16_from_double(a), orc.f16_from_double(b), [0])
    assert got == float(np.sum(a * b))


def test_one_plane_segments_round_each_product():
    rng = np.random.default_rng(5)
    nz, ny, nx = 6, 4, 3
    a16 = orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    b16 = orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    prod = orc.f16_to_double(a16) * orc.f16_to_double(b16)  # exact in fp64 (22 significant bits)
    want = float(np.sum(orc.f16_to_double(orc.f16_from_double(prod))))
    got, _ = orc.dot16h(a16, b16, list(range(nz)))
    assert got == pytest.approx(want, rel=1e-15, abs=1e-15)


def test_bad_segments_rejected():
    z = np.zeros((4, 1, 1), np.uint16)
    for seg in ([], [1], [0, 0], [0, 2, 1], [0, 4]):
        with pytest.raises(ValueError):
            orc.dot16h(z, z, seg)


def test_half_dot_sweep_vectors_and_sums():
    rng = np.random.default_rng(6)
    nz, ny, nx = 11, 6, 5
    c16 = [orc.f16_from_double(rng.uniform(-0.16, 0.16, (nz, ny, nx))) for _ in range(6)]
    vec = lambda: orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    rh, x, r, p, v, q, y = (vec() for _ in range(7))
    sc = (0.61, 0.93, -0.27)
    mixed = orc.sr_sweep16(c16, sc, rh, x, r, p, v, q, y)
    half = orc.sr_sweep16(c16, sc, rh, x, r, p, v, q, y, segments=SEG)
    for m, h in zip(mixed[:6], half[:6]):
        assert np.array_equal(m, h)
    xn, rn, pn, vn, qn, yn, dots, dabs = half
    pairs = [(rh, vn), (rh, rn), (rh, qn), (rh, yn), (qn, rn), (qn, vn), (yn, rn), (yn, vn), (qn, qn), (qn, yn),
             (yn, yn), (rn, rn)]
    for d, (a, b) in enumerate(pairs):
        s, ab = orc.dot16h(a, b, SEG)
        assert dots[d] == np.float32(s) and dabs[d] == ab, d
    # the half sums differ from the mixed ones by at most the pencils' fp16 roundings:
    # gamma_L * sum|a_i b_i| with L = 5 (the longest segment) and u = 2^-11
    for d, (a, b) in enumerate(pairs):
        scale = float(np.vdot(np.abs(orc.f16_to_double(a)), np.abs(orc.f16_to_double(b))))
        assert abs(float(dots[d]) - float(mixed[6][d])) <= 5 * 2.0 ** -11 * scale + 1e-6 * scale, d


def test_half_dot_solve_identity_one_iteration():
    rng = np.random.default_rng(7)
    nz, ny, nx = 5, 4, 3
    z = [np.zeros((nz, ny, nx), np.uint16)] * 6
    b = orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    ref = orc.bicgstab16(z, b, tol=1e-6, maxit=10, schedule="sr", segments=[0, 2])
    assert ref["iters"] == 1 and ref["status"] == orc.ORC_CONVERGED
    assert np.array_equal(ref["x"], b)


def test_half_dot_solve_tracks_mixed_early():
    """On a well-conditioned system the half-dot iteration follows the mixed one for
    the first steps (the sums agree to the pencils' rounding)."""
    import inputs
    n = 8
    diag, offs = inputs.problem_fields(inputs.KIND_CD, n, n, n, seed=1, delta=0.1)
    c16 = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(n, n, n, seed=1))
    mixed = orc.bicgstab16(c16, b16, tol=0.0, maxit=12, schedule="sr")
    half = orc.bicgstab16(c16, b16, tol=0.0, maxit=12, schedule="sr", segments=[0])
    assert half["hist"][0] == pytest.approx(mixed["hist"][0], rel=1e-3)
    assert np.all(np.abs(half["hist"][:5] - mixed["hist"][:5]) <= 5e-2 * mixed["hist"][:5])


def test_half_dot_underflow_is_breakdown_not_convergence():
    """R23: once ||r|| is ~6e-4 the squares of r's entries fall below fp16's smallest
    subnormal and every half pencil of (r,r) is 0, while (rhat, r) - products of O(1)
    entries with r - stays representable.  (r,r) = 0 with (rhat, r) != 0 is impossible
    in exact arithmetic (r = 0 => (rhat, r) = 0), so the solve reports BREAKDOWN there,
    never CONVERGED: with tol > 0 it stops with status BREAKDOWN (not a false
    convergence); the mixed dots (fp32 sums of exact products) do not underflow."""
    import inputs
    n = 10
    diag, offs = inputs.problem_fields(inputs.KIND_CD, n, n, n, seed=2, delta=0.1)
    c16 = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(n, n, n, seed=2))
    half = orc.bicgstab16(c16, b16, tol=0.0, maxit=40, schedule="sr", segments=[0])
    zero = np.flatnonzero(half["hist"] == 0.0)
    assert zero.size > 0, "the half-dot (r,r) never underflowed"
    k = int(zero[0])
    assert half["status"] == orc.ORC_BREAKDOWN and half["event_it"] == k
    stop = orc.bicgstab16(c16, b16, tol=1e-9, maxit=40, schedule="sr", segments=[0])
    assert stop["status"] == orc.ORC_BREAKDOWN and stop["iters"] == k
    mixed = orc.bicgstab16(c16, b16, tol=0.0, maxit=k, schedule="sr")
    assert np.all(mixed["hist"] > 0.0)


# ---------------- half dots in the classic schedule (Alg. 1 as printed; R22, R28) ----------------
def test_classic_half_first_iteration_composes_pinned_primitives():
    """One iteration of the classic half-dot solve recomputed from pinned pieces: the fused fp16
    SpMV (apply16), exact binary16 FMA, the half pencils (o16h_dot, pinned above) rounded once to
    fp32 for sigma, (t,s), (t,t), (r,r), and the mixed setup dots (R28) - x_1 and hist[1] equal."""
    import inputs
    nx, ny, nz, seg = 7, 6, 9, [0, 4]
    diag, offs = inputs.problem_fields(inputs.KIND_CD, nx, ny, nz, seed=3, delta=0.1)
    c16 = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), "mixed")
    b = orc.f16_from_double(inputs.rhs_uniform(nx, ny, nz, seed=3))
    r = orc.bicgstab16(c16, b, tol=0.0, maxit=1, segments=seg)
    hd = lambda a, c: np.float32(orc.dot16h(a, c, seg)[0])
    rho = np.float32(orc.dot16(b, b))  # setup: mixed
    v = orc.apply16(c16, b)
    alpha = np.float32(rho / hd(b, v))
    ah = orc.f16_from_double(np.float64(alpha))
    neg = lambda h: np.uint16(h ^ 0x8000)
    s = orc.fma16_array(np.full_like(v, neg(ah)), v, b)
    t = orc.apply16(c16, s)
    omega = np.float32(hd(t, s) / hd(t, t))
    wh = orc.f16_from_double(np.float64(omega))
    x = orc.fma16_array(np.full_like(s, wh), s, orc.fma16_array(np.full_like(b, ah), b, np.zeros_like(b)))
    assert np.array_equal(r["x"], x)
    rr = orc.fma16_array(np.full_like(t, neg(wh)), t, s)
    assert r["hist"][1] == np.sqrt(np.float64(hd(rr, rr))) / np.sqrt(np.float64(rho))


def test_classic_half_identity_and_tracking():
    """A = I: one iteration, x = b; on a well-conditioned system the classic half-dot solve follows
    the classic mixed one for the first iterations; with no segments it is the mixed solve."""
    rng = np.random.default_rng(8)
    nz, ny, nx = 5, 4, 3
    z = [np.zeros((nz, ny, nx), np.uint16)] * 6
    b = orc.f16_from_double(rng.uniform(-1, 1, (nz, ny, nx)))
    ref = orc.bicgstab16(z, b, tol=1e-6, maxit=10, segments=[0, 2])
    assert ref["iters"] == 1 and ref["status"] == orc.ORC_CONVERGED and np.array_equal(ref["x"], b)
    import inputs
    n = 8
    diag, offs = inputs.problem_fields(inputs.KIND_CD, n, n, n, seed=1, delta=0.1)
    c16 = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(n, n, n, seed=1))
    mixed = orc.bicgstab16(c16, b16, tol=0.0, maxit=12)
    half = orc.bicgstab16(c16, b16, tol=0.0, maxit=12, segments=[0])
    assert half["hist"][0] == mixed["hist"][0]  # the setup stays mixed (R28)
    assert np.all(np.abs(half["hist"][:5] - mixed["hist"][:5]) <= 5e-2 * mixed["hist"][:5])


def test_classic_half_underflow_is_breakdown():
    """R23 in the classic schedule: the half pencils of (r,r) underflow before r is zero, and the
    solve reports BREAKDOWN there (never CONVERGED)."""
    import inputs
    n = 8
    diag, offs = inputs.problem_fields(inputs.KIND_CD, n, n, n, seed=1, delta=0.1)
    c16 = orc.quantize_coeffs(orc.jacobi_scale(diag, offs), "mixed")
    b16 = orc.f16_from_double(inputs.rhs_uniform(n, n, n, seed=1))
    half = orc.bicgstab16(c16, b16, tol=0.0, maxit=40, segments=[0])
    zero = np.flatnonzero(half["hist"] == 0.0)
    assert zero.size > 0 and half["status"] == orc.ORC_BREAKDOWN and half["event_it"] == int(zero[0])
    stop = orc.bicgstab16(c16, b16, tol=1e-9, maxit=40, segments=[0])
    assert stop["status"] == orc.ORC_BREAKDOWN and stop["iters"] == int(zero[0])
    mixed = orc.bicgstab16(c16, b16, tol=0.0, maxit=int(zero[0]))
    assert np.all(mixed["hist"] > 0.0)
