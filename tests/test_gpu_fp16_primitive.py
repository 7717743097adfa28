"""The fp16 FMA the mixed kernels are built on, against the oracle's exact binary16
arithmetic (SURVEY §8(c) "fp16 primitives": the optional cross-check of fma16 against
the GPU's __hfma; it validates the primitive only).

A 1-row mesh nx x 1 x 2 whose only coupling is z (c_zp of plane 0; x couplings zero,
no diagonal scaling) makes the SpMV of plane 0 ONE fused multiply-add per point after
the zero terms: u[i, 0] = fma16(c[i], v[i, 1], v[i, 0]).  The expected values come
from the oracle's apply16 mirror of the same chain (which also fixes what the zero
terms do to a -0 accumulator) and, for a != -0, equal o16_fma directly.  Operands:
random bit patterns over all finite binary16 values (normals and subnormals), operands
biased to tiny exponents (subnormal and underflowing products), products near the
overflow threshold, and every finite b for a few (a, c) pairs."""
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


def _finite(bits):
    return (bits & 0x7C00) != 0x7C00


def _draw(rng, n, exp_lo=0, exp_hi=30):
    sign = rng.integers(0, 2, n).astype(np.uint16) << 15
    exp = rng.integers(exp_lo, exp_hi + 1, n).astype(np.uint16) << 10
    man = rng.integers(0, 1024, n).astype(np.uint16)
    return sign | exp | man


def _cases():
    rng = np.random.default_rng(2010)
    n = 1 << 18
    out = []
    out.append((_draw(rng, n), _draw(rng, n), _draw(rng, n)))                          # anything finite
    out.append((_draw(rng, n, 0, 8), _draw(rng, n, 0, 12), _draw(rng, n, 0, 12)))      # subnormal land
    out.append((_draw(rng, n, 20, 30), _draw(rng, n, 22, 30), _draw(rng, n, 22, 30)))  # overflow edge
    allb = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    allb = allb[_finite(allb)]
    for a, c in ((0x3C00, 0x3C00), (0x0001, 0x3800), (0x7BFF, 0x3C01), (0x8400, 0x0400), (0x1400, 0xB555)):
        out.append((np.full(allb.size, a, np.uint16), allb, np.full(allb.size, c, np.uint16)))
    return out


@pytest.mark.parametrize("case", range(8))
def test_hfma_matches_exact_binary16(sten, case):
    torch = torch_cuda()
    a, b, c = _cases()[case]
    nx = a.size
    v = np.zeros((2, 1, nx), np.uint16)
    v[0, 0] = a
    v[1, 0] = b
    zero = np.zeros((2, 1, nx))
    czp = zero.copy()
    czp[0, 0] = orc.f16_to_double(c)
    offs = [zero, zero, zero, zero, zero, czp]  # xm xp ym yp zm zp
    st = sten.stencil_create(nx, 1, 2, [None] + [torch.from_numpy(o).cuda() for o in offs])
    x = torch.from_numpy(v.view(np.int16)).cuda().view(torch.float16)
    y = torch.empty_like(x)
    sten.stencil_apply(st, sten.MIXED, x, y)
    got = y.view(torch.int16).cpu().numpy().view(np.uint16)[0, 0]
    c16 = [np.zeros((2, 1, nx), np.uint16) for _ in range(6)]
    c16[5][0, 0] = c
    want = orc.apply16(c16, v)[0, 0]
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    direct = orc.fma16_array(c, b, a)
    keep = a != 0x8000
    assert np.array_equal(got[keep], direct[keep])
    st.close()
