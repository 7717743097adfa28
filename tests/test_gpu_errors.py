"""Error behaviour of the C ABI (include/sten.h "Errors: ..."): invalid arguments are
refused with a negative code and a message (sten_last_error), never run, and a
handle stays usable after a refused call."""
import ctypes

import numpy as np
import pytest

import inputs
from gpu_util import fields, gpu_stencil, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sten():
    torch_cuda()
    import paper_2010_03660_b200 as s
    return s


def _raw_create(sten, nx, ny, nz, nslabs=1, dtype=0, null_at=None):
    torch = torch_cuda()
    n = max(nx * ny * nz, 1)
    keep = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in range(7)]
    arr = (ctypes.c_void_p * 7)(*[t.data_ptr() for t in keep])
    if null_at is not None:
        arr[null_at] = None
    h = ctypes.c_void_p()
    rc = sten.lib().stencil_create(nx, ny, nz, arr, dtype, nslabs, None, None, ctypes.byref(h))
    msg = sten.lib().sten_last_error().decode()
    if rc == 0:
        sten.lib().stencil_destroy(h)
    return rc, msg


@pytest.mark.parametrize("dims,nslabs,dtype,null_at,word", [
    ((0, 4, 4), 1, 0, None, "positive"),          # empty mesh
    ((4, -1, 4), 1, 0, None, "positive"),
    ((4, 4, 6), 4, 0, None, "nslabs"),            # nz not divisible into the slabs
    ((4, 4, 4), 0, 0, None, "nslabs"),
    ((4, 4, 4), 1, 7, None, "coeff_dtype"),
    ((4, 4, 4), 1, 0, 3, "coeffs[3]"),            # a NULL coupling array
    (((1 << 20) + 8, 1, 1), 1, 0, None, "too large"),
])
def test_create_refuses(sten, dims, nslabs, dtype, null_at, word):
    rc, msg = _raw_create(sten, *dims, nslabs=nslabs, dtype=dtype, null_at=null_at)
    assert rc == -1 and word in msg, (rc, msg)


def test_solve_and_apply_refuse_bad_arguments_and_stay_usable(sten):
    torch = torch_cuda()
    nx, ny, nz = 12, 10, 8
    diag, offs = fields(inputs.KIND_CD, nx, ny, nz)
    st = gpu_stencil(diag, offs)
    b = torch.from_numpy(inputs.rhs_uniform(nx, ny, nz)).float().cuda()
    x = torch.empty_like(b)
    for tol, maxit in ((-1.0, 10), (float("nan"), 10), (0.0, -1)):
        with pytest.raises(sten.StenError):
            sten.bicgstab_solve(st, sten.FP32, b, None, tol, maxit, x)
    with pytest.raises(sten.StenError):  # precision code
        sten._check(sten.lib().stencil_apply(st.handle, 7, b.data_ptr(), x.data_ptr(), None))
    with pytest.raises(sten.StenError):  # storage type does not match the precision
        sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, 3, x)
    with pytest.raises(sten.StenError):  # wrong size
        sten.stencil_apply(st, sten.FP32, b[:-1], x[:-1])
    with pytest.raises(sten.StenError):
        sten.set_schedule(st, 5)
    with pytest.raises(sten.StenError):
        sten.set_sr_tiling(st, sten.FP32, 12, 2, 2, 16, 16)  # no such tile height
    with pytest.raises(sten.StenError):
        sten.set_sr_exchange(st, 9)
    # still usable, and the refused calls left no state behind
    it, hist, status = sten.bicgstab_solve(st, sten.FP32, b, None, 1e-6, 200, x)
    assert status == sten.CONVERGED and hist[-1] <= 1e-6
    st.close()


def test_maximum_row_length_is_accepted(sten):
    """nx = 2^20 (the largest accepted row) on a 1 x 1 cross-section: one apply, exact."""
    torch = torch_cuda()
    nx = 1 << 20
    zero = torch.zeros((1, 1, nx), dtype=torch.float64, device="cuda")
    xm = torch.full((1, 1, nx), -0.25, dtype=torch.float64, device="cuda")
    xm[0, 0, 0] = 0.0
    st = sten.stencil_create(nx, 1, 1, [None, xm, zero, zero, zero, zero, zero])
    v = torch.ones((1, 1, nx), dtype=torch.float32, device="cuda")
    u = torch.empty_like(v)
    sten.stencil_apply(st, sten.FP32, v, u)
    want = np.full(nx, 0.75, np.float32)
    want[0] = 1.0
    assert np.array_equal(u.cpu().numpy().ravel(), want)
    st.close()
