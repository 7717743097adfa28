"""Pins for the oracle's binary16 primitives (o16_*), independent of the oracle.

References used here, none of which is the oracle's own code:
  * numpy's float16 <-> float64 conversions (a library routine);
  * exact-in-fp64 sums/products of two fp16 values, then numpy's rounding
    (fp16+fp16 needs <= 41 significant bits, fp16*fp16 <= 22: both exact in
    fp64, so the only rounding is numpy's);
  * exact rational arithmetic (fractions.Fraction) with nearest-even chosen by
    brute-force comparison of the neighbouring fp16 candidates;
  * SPEC.md examples ("scalarmodel") and IEEE 754 zero-sign rules.
"""
from fractions import Fraction

import numpy as np
import pytest

F16_INF = 0x7C00


def _all_finite_f16():
    h = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16)
    e = (h >> 10) & 31
    return h[e != 31]


def test_roundtrip_all_finite(orc):
    h = _all_finite_f16()
    assert h.size == 63488  # SPEC.md:62 "for all 63488 finite fp16 bit patterns"
    d = orc.f16_to_double(h)
    assert np.array_equal(d, h.view(np.float16).astype(np.float64))
    assert np.array_equal(orc.f16_from_double(d), h)


def test_from_double_matches_numpy_random_and_ties(orc):
    rng = np.random.default_rng(0)
    # random fp32 bit patterns (all exponents), widened exactly to fp64
    bits = rng.integers(0, 2 ** 32, size=1 << 21, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32).astype(np.float64)
    x = x[np.isfinite(x)]
    assert np.array_equal(orc.f16_from_double(x), x.astype(np.float16).view(np.uint16))
    # random doubles concentrated in the fp16 range (incl. subnormal range)
    y = rng.uniform(-1, 1, 1 << 20) * np.exp2(rng.uniform(-30, 17, 1 << 20))
    assert np.array_equal(orc.f16_from_double(y), y.astype(np.float16).view(np.uint16))
    # every midpoint between consecutive positive finite fp16 values, and its
    # two double neighbours: the tie-to-even rule and the off-by-one-ulp cases
    h = np.arange(0, 0x7BFF, dtype=np.uint16)
    lo = h.view(np.float16).astype(np.float64)
    hi = (h + 1).view(np.float16).astype(np.float64)
    mid = (lo + hi) / 2
    for t in (mid, np.nextafter(mid, 0), np.nextafter(mid, np.inf), -mid, -np.nextafter(mid, np.inf)):
        assert np.array_equal(orc.f16_from_double(t), t.astype(np.float16).view(np.uint16))


def test_spec_examples(orc):
    one, two, three = 0x3C00, 0x4000, 0x4200
    assert orc.add16(one, two) == three
    assert orc.add16(0x6800, one) == 0x6800                      # 2048+1 -> 2048
    assert orc.f16_from_double(np.array([65520.0]))[0] == F16_INF
    assert orc.f16_from_double(np.array([65519.99]))[0] == 0x7BFF
    assert orc.f16_from_double(np.array([1.0]))[0] == one
    # Mixed: 2048 + 1 accumulated in fp32 is 2049 - the dot
    a = np.array([[[0x6800, one]]], dtype=np.uint16)
    b = np.array([[[one, one]]], dtype=np.uint16)
    # shape (nz=1, ny=1, nx=2): two pencils summed in fp32
    assert orc.dot16(a, b) == 2049.0
    # fmac(0, 3, 4) = 12; fmac(x, a, 0) = x
    assert orc.fma16(0x4200, 0x4400, 0) == 0x4A00
    assert orc.fma16(0x3555, 0, 0x4321) == 0x4321


def test_add_mul_match_exact_then_round(orc):
    rng = np.random.default_rng(1)
    a_all = _all_finite_f16()
    b_some = rng.choice(a_all, 160)
    a = np.repeat(a_all, b_some.size)
    b = np.tile(b_some, a_all.size)
    da = a.view(np.float16).astype(np.float64)
    db = b.view(np.float16).astype(np.float64)
    ref_add = (da + db).astype(np.float16).view(np.uint16)
    ref_mul = (da * db).astype(np.float16).view(np.uint16)
    got_add = orc.add16_array(a, b)
    got_mul = orc.mul16_array(a, b)
    # compare as values (numpy may produce a different NaN payload; none here: finite)
    assert np.array_equal(got_add, ref_add)
    assert np.array_equal(got_mul, ref_mul)


def _rn16_fraction(F: Fraction, sign_if_zero: int = 0) -> int:
    """nearest-even binary16 of an exact rational, by candidate comparison"""
    if F == 0:
        return 0x8000 if sign_if_zero else 0
    neg = F < 0
    A = -F if neg else F
    if A >= 65520:
        return (0x8000 if neg else 0) | F16_INF
    h = np.float16(float(A))
    cands = set()
    for c in (h, np.nextafter(h, np.float16(np.inf)), np.nextafter(h, np.float16(0))):
        if np.isfinite(c):
            cands.add(int(np.array(c, dtype=np.float16).view(np.uint16)))
    best = None
    for c in sorted(cands):
        dist = abs(Fraction(float(np.array(c, np.uint16).view(np.float16))) - A)
        key = (dist, c & 1)
        if best is None or key < best[0]:
            best = (key, c)
    return (0x8000 if neg else 0) | best[1]


def _val(h):
    return Fraction(float(np.array(h, np.uint16).view(np.float16)))


def test_fma_matches_exact_rational(orc):
    rng = np.random.default_rng(2)
    fin = _all_finite_f16()
    n = 4000
    a = rng.choice(fin, n)
    b = rng.choice(fin, n)
    c = rng.choice(fin, n)
    # bias half the cases toward comparable magnitudes (real cancellation / rounding)
    c[: n // 2] = np.array([x ^ 0x8000 for x in c[: n // 2]], dtype=np.uint16)
    got = orc.fma16_array(a, b, c)
    for i in range(n):
        F = _val(a[i]) * _val(b[i]) + _val(c[i])
        if F == 0:
            continue  # zero signs checked separately
        assert got[i] == _rn16_fraction(F), (hex(a[i]), hex(b[i]), hex(c[i]))


def test_fma_ties_and_subnormals(orc):
    cases = []
    rng = np.random.default_rng(3)
    fin = _all_finite_f16()
    pos = fin[(fin < 0x7C00) & (fin > 0)]
    for h in rng.choice(pos, 800):
        x = _val(h)
        e = ((int(h) >> 10) & 31)
        ulp = Fraction(2) ** ((e if e > 0 else 1) - 25)
        half = ulp / 2
        if half >= Fraction(2) ** -24:  # half-ulp representable -> exact tie via 1*h + half
            hb = _rn16_fraction(half)
            if _val(hb) == half:
                cases.append((0x3C00, int(h), hb))
                cases.append((0x3C00, int(h) ^ 0x8000, hb ^ 0x8000))
    # products landing in the subnormal range
    for _ in range(800):
        a = int(rng.choice(pos[pos < 0x2000]))
        b = int(rng.choice(pos[pos < 0x2400]))
        c = int(rng.choice(pos[pos < 0x0400]))
        cases.append((a, b, c))
        cases.append((a, b ^ 0x8000, c))
    A = np.array([x[0] for x in cases], np.uint16)
    B = np.array([x[1] for x in cases], np.uint16)
    C = np.array([x[2] for x in cases], np.uint16)
    got = orc.fma16_array(A, B, C)
    for i in range(len(cases)):
        F = _val(A[i]) * _val(B[i]) + _val(C[i])
        if F == 0:
            continue
        assert got[i] == _rn16_fraction(F), tuple(hex(x) for x in cases[i])


def test_fma_fused_differs_from_unfused_witness(orc):
    # a witness where fma != round(round(a*b)+c) must exist
    rng = np.random.default_rng(4)
    fin = _all_finite_f16()
    a = rng.choice(fin, 200000)
    b = rng.choice(fin, 200000)
    c = rng.choice(fin, 200000)
    fused = orc.fma16_array(a, b, c)
    unf = orc.add16_array(orc.mul16_array(a, b), c)
    diff = np.nonzero(fused != unf)[0]
    assert diff.size > 0
    i = diff[0]
    F = _val(a[i]) * _val(b[i]) + _val(c[i])
    assert fused[i] == _rn16_fraction(F)


def test_zero_signs_and_specials(orc):
    P0, N0, ONE, MONE, INF, NINF = 0x0000, 0x8000, 0x3C00, 0xBC00, 0x7C00, 0xFC00
    assert orc.fma16(P0, ONE, N0) == P0     # (+0)+(-0) = +0
    assert orc.fma16(N0, ONE, N0) == N0     # (-0)+(-0) = -0
    assert orc.fma16(ONE, ONE, MONE) == P0  # exact cancellation -> +0 (RNE)
    assert orc.fma16(MONE, P0, N0) == N0    # (-0) + (-0)
    assert orc.mul16(MONE, P0) == N0        # IEEE: -1 * +0 = -0
    assert orc.add16(N0, N0) == N0
    assert orc.fma16(INF, ONE, ONE) == INF
    assert orc.fma16(INF, P0, ONE) & 0x7C00 == 0x7C00 and orc.fma16(INF, P0, ONE) & 0x3FF  # NaN
    assert orc.add16(INF, NINF) & 0x3FF     # NaN
    assert orc.mul16(0x7BFF, 0x7BFF) == INF  # overflow
    assert orc.mul16(0x0001, 0x3800) == 0x0000  # 2^-24 * 0.5 -> tie -> even (0)
    assert orc.mul16(0x0003, 0x3800) == 0x0002  # 1.5 quanta -> tie -> even (2)


# ------------------------------------------------- fp32 fused multiply-add --
def _rn32_fraction(F):
    """Nearest-even fp32 to the rational F (finite, normal-range results here), by brute force over
    the neighbours of numpy's float32 of float(F)."""
    c = np.float32(float(F))
    cands = {c, np.nextafter(c, np.float32(np.inf)), np.nextafter(c, np.float32(-np.inf))}
    best = None
    for x in cands:
        d = abs(Fraction(float(x)) - F)
        key = (d, int(np.array(x, np.float32).view(np.uint32)) & 1)  # ties: even significand
        if best is None or key < best[0]:
            best = (key, x)
    return best[1]


def test_fma32_matches_exact_rational(orc):
    """o32_fma_array (the fp32 AXPY primitive of the classic-phase mirrors): one rounding of the
    exact a*b + c; a single-rounding witness differs from round(round(a*b) + c)."""
    rng = np.random.default_rng(5)
    n = 6000
    a = rng.uniform(-2, 2, n).astype(np.float32)
    b = rng.uniform(-2, 2, n).astype(np.float32)
    c = rng.uniform(-2, 2, n).astype(np.float32)
    c[: n // 3] = (-(a[: n // 3].astype(np.float64) * b[: n // 3])).astype(np.float32)  # cancellation
    got = orc.fma32_array(a, b, c)
    unfused_differs = 0
    for i in range(n):
        F = Fraction(float(a[i])) * Fraction(float(b[i])) + Fraction(float(c[i]))
        if F == 0:
            assert got[i] == 0
            continue
        assert got[i] == _rn32_fraction(F), (a[i], b[i], c[i])
        unfused_differs += got[i] != np.float32(np.float32(a[i] * b[i]) + c[i])
    assert unfused_differs > 0
    # scalar broadcasting, as the mirrors use it
    assert np.array_equal(orc.fma32_array(np.float32(0.5), b[:8], c[:8]), orc.fma32_array(np.full(8, 0.5), b[:8], c[:8]))
