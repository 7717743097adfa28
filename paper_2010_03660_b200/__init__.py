"""B200-native BiCGStab for Jacobi-scaled 7-point stencils (arXiv 2010.03660).

Thin ctypes binding of libsten.so (include/sten.h): the same entry points,
argument marshalling only - every step of the solve runs in the library's
CUDA kernels.  There is no CPU fallback: if libsten.so is missing or cannot be
loaded every call raises StenError.

Vectors may be torch tensors (CUDA or CPU) or numpy arrays; their element type
must match the precision: float32 for FP32, float16 (torch.float16, or numpy
float16/uint16 bit patterns) for MIXED.  Coefficients are float64 or float32.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import roofline  # noqa: F401  (work/traffic accounting)

FP32 = 0
MIXED = 1
SCHED_CLASSIC = 0
SCHED_SR = 1
DOTS_MIXED, DOTS_HALF = 0, 1
XCHG_SERIAL, XCHG_OVERLAP, XCHG_FUSED = 0, 1, 2
(OPT_TMA_L2_PROMOTION, OPT_EW_CTAS_PER_SM, OPT_COEF_PREFETCH, OPT_SR_L2_PREFETCH, OPT_SR_LIGHT_LAST,
 OPT_CLASSIC_OVERLAP, OPT_CLASSIC_FUSED, OPT_CLASSIC_CONST) = 1, 2, 3, 4, 5, 6, 7, 8
DT_F64 = 0
DT_F32 = 1

CONVERGED, MAXIT, BREAKDOWN, NONFINITE, TIMEOUT = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "converged", 1: "maxit", 2: "breakdown", 3: "nonfinite", 4: "timeout"}

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsten.so")


class StenError(RuntimeError):
    pass


_BARRIER_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p)


class _Stats(ctypes.Structure):
    _fields_ = [("phase_ms", ctypes.c_double * 3), ("phase_launches", ctypes.c_longlong * 3),
                ("solve_ms", ctypes.c_double), ("kernel_launches", ctypes.c_longlong),
                ("event_iter", ctypes.c_int), ("graph_chunk", ctypes.c_int), ("handover", ctypes.c_int)]


_lib = None


def lib():
    """Load libsten.so; raise StenError (never fall back) if it is unavailable."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise StenError(f"{LIB_PATH} not built - run `python -m paper_2010_03660_b200.build` "
                            "(or __graft_entry__.build())")
        try:
            L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        except OSError as e:  # pragma: no cover
            raise StenError(f"cannot load {LIB_PATH}: {e}") from e
        P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.sten_version.restype = I
        L.sten_last_error.restype = ctypes.c_char_p
        L.sten_comm_unique_id.argtypes = [P]
        L.sten_comm_create.argtypes = [P, I, I, I, ctypes.POINTER(P)]
        L.sten_comm_destroy.argtypes = [P]
        L.stencil_create.argtypes = [I, I, I, P, I, I, P, P, ctypes.POINTER(P)]
        L.stencil_destroy.argtypes = [P]
        L.stencil_create_const.argtypes = [I, I, I, P, I, P, P, ctypes.POINTER(P)]
        L.stencil2d_create.argtypes = [I, I, P, I, P, ctypes.POINTER(P)]
        L.stencil2d_apply.argtypes = [P, I, P, P, P]
        L.stencil2d_last_ms.argtypes = [P, ctypes.POINTER(D)]
        L.stencil2d_destroy.argtypes = [P]
        L.stencil2d_set_tiles.argtypes = [P, I, I]
        L.stencil2d_set_timing.argtypes = [P, I]
        L.stencil2d_phase_ms.argtypes = [P, P, ctypes.POINTER(ctypes.c_longlong)]
        L.bicgstab2d_solve.argtypes = [P, I, P, P, D, I, P, ctypes.POINTER(I), P, ctypes.POINTER(I), P]
        L.stencil_apply.argtypes = [P, I, P, P, P]
        L.bicgstab_solve.argtypes = [P, I, P, P, D, I, P, ctypes.POINTER(I), P, ctypes.POINTER(I), P]
        L.bicgstab_solve_batch.argtypes = [P, I, I, P, P, D, I, P, P, P, P]
        L.sten_scalar_history.argtypes = [P, I, P, P]
        L.sten_set_timing.argtypes = [P, I]
        L.sten_set_option.argtypes = [P, I, I]
        L.sten_set_host_barrier.argtypes = [P, _BARRIER_FN, P]
        L.sten_get_option.argtypes = [P, I, ctypes.POINTER(ctypes.c_int)]
        L.sten_get_stats.argtypes = [P, ctypes.POINTER(_Stats)]
        L.sten_iter_ms.argtypes = [P, I, ctypes.POINTER(ctypes.c_float), I, ctypes.POINTER(ctypes.c_int)]
        L.sten_set_tiling.argtypes = [P, I, I, I, I, I]
        L.sten_set_schedule.argtypes = [P, I]
        L.sten_set_dot_precision.argtypes = [P, I]
        L.sten_sr_segments.argtypes = [P, I, P, I, ctypes.POINTER(I)]
        L.sten_set_sr_tiling.argtypes = [P, I, I, I, I, I, I]
        L.sten_set_sr_exchange.argtypes = [P, I]
        L.sten_p2p_export.argtypes = [P, I, P, ctypes.POINTER(ctypes.c_size_t)]
        L.sten_p2p_import.argtypes = [P, I, P, ctypes.c_size_t]
        L.sten_classic_phase.argtypes = [P, I, I, D, D, D, P, P, P, P, P, P, P, P]
        L.sten_classic_segments.argtypes = [P, I, ctypes.POINTER(ctypes.c_int), I, ctypes.POINTER(ctypes.c_int)]
        L.sten_set_sr_chunks.argtypes = [P, I, I, I, I]
        L.sten_sr_sweep.argtypes = [P, I, D, D, D, P, P, P, P, P, P, P, P, P]
        L.bicgstab_refine.argtypes = [P, P, P, D, I, D, I, P, ctypes.POINTER(I), ctypes.POINTER(I), P,
                                      ctypes.POINTER(I), P]
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        msg = lib().sten_last_error().decode(errors="replace")
        raise StenError(f"libsten error {rc}: {msg}")


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise StenError("tensor must be contiguous")
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise StenError("array must be C-contiguous")
        return ctypes.c_void_p(a.ctypes.data)
    raise StenError(f"unsupported array type {type(a)}")


def _itemsize(a):
    if hasattr(a, "element_size"):
        return a.element_size()
    return a.itemsize


def _numel(a):
    return a.numel() if hasattr(a, "numel") else a.size


def _stream(stream):
    if stream is not None:
        return ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    try:
        import torch
        if torch.cuda.is_available():
            return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover
        pass
    return ctypes.c_void_p(0)


def _check_vec(a, precision, n, name):
    if a is None:
        raise StenError(f"{name} is required")
    want = 4 if precision == FP32 else 2
    if _itemsize(a) != want:
        raise StenError(f"{name}: element size {_itemsize(a)} does not match precision {precision}")
    if _numel(a) != n:
        raise StenError(f"{name}: {_numel(a)} elements, expected {n}")


def version() -> int:
    return lib().sten_version()


# ------------------------------------------------------------------ comm --
class Comm:
    def __init__(self, handle, nranks, rank):
        self.handle, self.nranks, self.rank = handle, nranks, rank

    def close(self):
        if self.handle:
            lib().sten_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().sten_comm_unique_id(buf))
    return buf.raw


def comm_create(unique_id: bytes | None, nranks: int, rank: int, cuda_device: int | None = None) -> Comm:
    """sten_comm_create on `cuda_device` (default: the current device).  unique_id None gives a
    peer-memory-only communicator (no NCCL; after p2p_setup, halos and all-reduces through CUDA IPC:
    the fused SR sweep, or the classic schedule in host lockstep)."""
    if cuda_device is None:
        import torch
        cuda_device = torch.cuda.current_device()
    h = ctypes.c_void_p()
    buf = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
    _check(lib().sten_comm_create(buf, nranks, rank, int(cuda_device), ctypes.byref(h)))
    return Comm(h, nranks, rank)


# --------------------------------------------------------------- stencil --
class Stencil:
    """Owner of a sten_stencil handle."""

    def __init__(self, handle, nx, ny, nz, comm):
        self.handle, self.nx, self.ny, self.nz, self.comm = handle, nx, ny, nz, comm

    @property
    def npoints(self) -> int:
        return self.nx * self.ny * self.nz

    def close(self):
        if self.handle:
            lib().stencil_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def stencil_create(nx: int, ny: int, nz_global: int, coeffs, nslabs: int = 1, comm: Comm | None = None,
                   stream=None) -> Stencil:
    """coeffs = [diag or None, A_xm, A_xp, A_ym, A_yp, A_zm, A_zp], dense (nz, ny, nx) each with
    nz = nz_global / comm.nranks: this rank's z-slab (sten.h slab convention)."""
    R = comm.nranks if comm else 1
    if nz_global % R:
        raise StenError(f"nz_global={nz_global} not divisible by {R} ranks")
    nz = nz_global // R
    if len(coeffs) != 7:
        raise StenError("coeffs must have 7 entries (diag, xm, xp, ym, yp, zm, zp)")
    ref = next(c for c in coeffs[1:] if c is not None)
    dt = DT_F64 if _itemsize(ref) == 8 else DT_F32
    n = nx * ny * nz
    keep = []
    arr = (ctypes.c_void_p * 7)()
    for i, c in enumerate(coeffs):
        if c is None:
            arr[i] = None
            continue
        if _itemsize(c) != _itemsize(ref) or _numel(c) != n:
            raise StenError(f"coeffs[{i}] has the wrong dtype or size")
        keep.append(c)
        arr[i] = _ptr(c).value
    h = ctypes.c_void_p()
    _check(lib().stencil_create(nx, ny, nz_global, arr, dt, nslabs, comm.handle if comm else None,
                                _stream(stream), ctypes.byref(h)))
    return Stencil(h, nx, ny, nz, comm)


def stencil_create_const(nx: int, ny: int, nz_global: int, coeffs, nslabs: int = 1, comm: Comm | None = None,
                         stream=None) -> Stencil:
    """Constant operator: coeffs = (a_P, A_xm, A_xp, A_ym, A_yp, A_zm, A_zp) as 7 floats."""
    R = comm.nranks if comm else 1
    if nz_global % R:
        raise StenError(f"nz_global={nz_global} not divisible by {R} ranks")
    if len(coeffs) != 7:
        raise StenError("coeffs must have 7 entries (diag, xm, xp, ym, yp, zm, zp)")
    arr = np.ascontiguousarray(coeffs, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib().stencil_create_const(nx, ny, nz_global, arr.ctypes.data_as(ctypes.c_void_p), nslabs,
                                      comm.handle if comm else None, _stream(stream), ctypes.byref(h)))
    return Stencil(h, nx, ny, nz_global // R, comm)


def stencil_destroy(st: Stencil):
    st.close()


def stencil_apply(st: Stencil, precision: int, x, y, stream=None):
    _check_vec(x, precision, st.npoints, "x")
    _check_vec(y, precision, st.npoints, "y")
    _check(lib().stencil_apply(st.handle, precision, _ptr(x), _ptr(y), _stream(stream)))
    return y


def bicgstab_solve(st: Stencil, precision: int, b, x0, tol: float, maxit: int, x_out, stream=None):
    """Returns (iters, res_hist[0..iters] as numpy fp64, status)."""
    _check_vec(b, precision, st.npoints, "b")
    _check_vec(x_out, precision, st.npoints, "x_out")
    if x0 is not None:
        _check_vec(x0, precision, st.npoints, "x0")
    hist = np.zeros(max(maxit, 0) + 1, dtype=np.float64)
    it = ctypes.c_int(0)
    status = ctypes.c_int(-1)
    _check(lib().bicgstab_solve(st.handle, precision, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(x_out),
                                ctypes.byref(it), hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(status),
                                _stream(stream)))
    return it.value, hist[: it.value + 1].copy(), status.value


def bicgstab_solve_batch(st: Stencil, precision: int, bs, xs, tol: float, maxit: int, stream=None):
    """n independent solves (x0 = 0) with pipelined host<->device copies (pinned host
    vectors overlap with the solves).  Returns [(iters, res_hist, status)] per system."""
    if len(bs) != len(xs):
        raise StenError("bs and xs must have the same length")
    n = len(bs)
    for i, (b, x) in enumerate(zip(bs, xs)):
        _check_vec(b, precision, st.npoints, f"b[{i}]")
        _check_vec(x, precision, st.npoints, f"x[{i}]")
    bp = (ctypes.c_void_p * max(n, 1))(*[_ptr(b) for b in bs])
    xp = (ctypes.c_void_p * max(n, 1))(*[_ptr(x) for x in xs])
    its = np.zeros(max(n, 1), np.int32)
    sts = np.zeros(max(n, 1), np.int32)
    hist = np.zeros((max(n, 1), max(maxit, 0) + 1), np.float64)
    _check(lib().bicgstab_solve_batch(st.handle, precision, n, bp, xp, float(tol), int(maxit),
                                      its.ctypes.data_as(ctypes.c_void_p), hist.ctypes.data_as(ctypes.c_void_p),
                                      sts.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
    return [(int(its[i]), hist[i, : its[i] + 1].copy(), int(sts[i])) for i in range(n)]


def scalar_history(st: Stencil, n: int):
    a = np.zeros(n, np.float64)
    w = np.zeros(n, np.float64)
    _check(lib().sten_scalar_history(st.handle, n, a.ctypes.data_as(ctypes.c_void_p),
                                     w.ctypes.data_as(ctypes.c_void_p)))
    return a, w


def set_option(st: Stencil, option: int, value: int):
    """sten_set_option: an explicit tuning knob of the handle (OPT_*)."""
    _check(lib().sten_set_option(st.handle, int(option), int(value)))


def get_option(st: Stencil, option: int) -> int:
    v = ctypes.c_int(0)
    _check(lib().sten_get_option(st.handle, int(option), ctypes.byref(v)))
    return v.value


def set_host_barrier(st: Stencil, fn):
    """sten_set_host_barrier: fn() (a Python callable, e.g. torch.distributed.barrier over gloo) is
    called before every peer-memory all-reduce's waiting kernel; None turns it off.  For several
    ranks sharing one GPU only."""
    cb = _BARRIER_FN(lambda _ctx: fn()) if fn is not None else _BARRIER_FN()
    st._barrier_cb = cb  # keep the trampoline alive as long as the handle may call it
    _check(lib().sten_set_host_barrier(st.handle, cb, None))


def set_timing(st: Stencil, enable: bool):
    _check(lib().sten_set_timing(st.handle, int(bool(enable))))


def get_stats(st: Stencil) -> dict:
    s = _Stats()
    _check(lib().sten_get_stats(st.handle, ctypes.byref(s)))
    return dict(phase_ms=list(s.phase_ms), phase_launches=list(s.phase_launches), solve_ms=s.solve_ms,
                kernel_launches=s.kernel_launches, event_iter=s.event_iter, graph_chunk=s.graph_chunk,
                handover=s.handover)


def iter_ms(st: Stencil, phase: int = -1) -> list:
    """Per-iteration device ms of the last timed solve (sten_iter_ms): phase 0-2 = H1/H2/H3
    (SR: 0 = the sweep), -1 = the sum."""
    n = ctypes.c_int(0)
    _check(lib().sten_iter_ms(st.handle, phase, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_float * max(n.value, 1))()
    _check(lib().sten_iter_ms(st.handle, phase, buf, n.value, ctypes.byref(n)))
    return [float(buf[i]) for i in range(n.value)]


def set_tiling(st: Stencil, precision: int, bx: int = 0, by: int = 0, zc: int = 0, stages: int = 0):
    _check(lib().sten_set_tiling(st.handle, precision, bx, by, zc, stages))


def set_schedule(st: Stencil, schedule: int):
    """SCHED_CLASSIC (Alg. 1 as printed) or SCHED_SR (single reduction, R19)."""
    _check(lib().sten_set_schedule(st.handle, int(schedule)))


def set_dot_precision(st: Stencil, dots: int):
    """DOTS_MIXED (fp16 products summed in fp32) or DOTS_HALF (fp16 column pencils, R22)
    for the MIXED SR sweeps of this handle."""
    _check(lib().sten_set_dot_precision(st.handle, int(dots)))


def classic_segments(st: Stencil, precision: int):
    """First planes of the classic kernels' z chunks on this rank (sten_classic_segments)."""
    n = ctypes.c_int(0)
    _check(lib().sten_classic_segments(st.handle, precision, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_int * max(n.value, 1))()
    _check(lib().sten_classic_segments(st.handle, precision, buf, n.value, ctypes.byref(n)))
    return [int(buf[i]) for i in range(n.value)]


def set_sr_chunks(st: Stencil, precision: int, zc: int, tail_planes: int = 0, zc_tail: int = 0):
    """sten_set_sr_chunks: zc-plane chunks, the last tail_planes planes in zc_tail-plane chunks."""
    _check(lib().sten_set_sr_chunks(st.handle, precision, zc, tail_planes, zc_tail))


def sr_segments(st: Stencil, precision: int):
    """First planes of the SR chunk plan's z segments on this rank (the pencils of DOTS_HALF)."""
    n = ctypes.c_int(0)
    _check(lib().sten_sr_segments(st.handle, precision, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_int * max(n.value, 1))()
    _check(lib().sten_sr_segments(st.handle, precision, buf, n.value, ctypes.byref(n)))
    return [int(buf[i]) for i in range(n.value)]


def set_sr_exchange(st: Stencil, mode: int):
    """XCHG_SERIAL / XCHG_OVERLAP / XCHG_FUSED (peer-memory halo stores + one-shot all-reduce)."""
    _check(lib().sten_set_sr_exchange(st.handle, int(mode)))


def set_sr_tiling(st: Stencil, precision: int, by: int = 0, stages: int = 0, cstages: int = 0, zc: int = 0,
                  pack: int = 0):
    _check(lib().sten_set_sr_tiling(st.handle, precision, by, stages, cstages, zc, pack))


def sr_sweep(st: Stencil, precision: int, scalars, rh, x, r, p, v, q, y, stream=None):
    """One SR sweep in place on (x, r, p, v, q, y); returns the 12 fp32 dot sums."""
    for name, a in (("rh", rh), ("x", x), ("r", r), ("p", p), ("v", v), ("q", q), ("y", y)):
        _check_vec(a, precision, st.npoints, name)
    dots = np.zeros(12, np.float32)
    al, om, be = (float(t) for t in scalars)
    _check(lib().sten_sr_sweep(st.handle, precision, al, om, be, _ptr(rh), _ptr(x), _ptr(r), _ptr(p), _ptr(v),
                               _ptr(q), _ptr(y), dots.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
    return dots


def classic_phase(st: Stencil, precision: int, phase: int, scalars, r, p, v, rh, out0, out1, stream=None):
    """sten_classic_phase: one H1 (phase 1: out0 = p', out1 = v' = A p', returns [(rh, v')]) or
    H2 (phase 2: out0 = s, out1 = t = A s, returns [(t, s), (t, t)]) on caller vectors.
    scalars = (alpha, omega, beta)."""
    for name, a in (("r", r), ("v", v), ("out0", out0), ("out1", out1)) + (
            (("p", p), ("rh", rh)) if phase == 1 else ()):
        _check_vec(a, precision, st.npoints, name)
    dots = np.zeros(2, np.float32)
    al, om, be = (float(t) for t in scalars)
    _check(lib().sten_classic_phase(st.handle, precision, int(phase), al, om, be, _ptr(r), _ptr(p), _ptr(v),
                                    _ptr(rh), _ptr(out0), _ptr(out1), dots.ctypes.data_as(ctypes.c_void_p),
                                    _stream(stream)))
    return dots[:1] if phase == 1 else dots


def bicgstab_refine(st: Stencil, b, x0, tol: float, outer_maxit: int, inner_tol: float, inner_maxit: int, x_out,
                    stream=None):
    """Mixed-precision iterative refinement (fp32 b, x0, x_out).
    Returns (outer_iters, inner_iters, res_hist[0..outer_iters], status)."""
    _check_vec(b, FP32, st.npoints, "b")
    _check_vec(x_out, FP32, st.npoints, "x_out")
    if x0 is not None:
        _check_vec(x0, FP32, st.npoints, "x0")
    hist = np.zeros(max(outer_maxit, 0) + 1, dtype=np.float64)
    ko, ki, status = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int(-1)
    _check(lib().bicgstab_refine(st.handle, _ptr(b), _ptr(x0), float(tol), int(outer_maxit), float(inner_tol),
                                 int(inner_maxit), _ptr(x_out), ctypes.byref(ko), ctypes.byref(ki),
                                 hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(status), _stream(stream)))
    return ko.value, ki.value, hist[: ko.value + 1].copy(), status.value


# ------------------------------------------------------- 2D 9-point SpMV --
class Stencil2D:
    def __init__(self, handle, nx, ny):
        self.handle, self.nx, self.ny = handle, nx, ny

    def close(self):
        if self.handle:
            lib().stencil2d_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def stencil2d_create(nx: int, ny: int, coeffs, stream=None) -> Stencil2D:
    """coeffs = [diag or None, 8 couplings in the order (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0)
    (-1,+1) (0,+1) (+1,+1)], dense (ny, nx) each, float64 or float32."""
    if len(coeffs) != 9:
        raise StenError("coeffs must have 9 entries (diag + 8 couplings)")
    ref = next(c for c in coeffs[1:] if c is not None)
    dt = DT_F64 if _itemsize(ref) == 8 else DT_F32
    arr = (ctypes.c_void_p * 9)()
    for i, c in enumerate(coeffs):
        if c is None:
            arr[i] = None
            continue
        if _itemsize(c) != _itemsize(ref) or _numel(c) != nx * ny:
            raise StenError(f"coeffs[{i}] has the wrong dtype or size")
        arr[i] = _ptr(c).value
    h = ctypes.c_void_p()
    _check(lib().stencil2d_create(nx, ny, arr, dt, _stream(stream), ctypes.byref(h)))
    return Stencil2D(h, nx, ny)


def stencil2d_apply(st: Stencil2D, precision: int, x, y, stream=None):
    _check_vec(x, precision, st.nx * st.ny, "x")
    _check_vec(y, precision, st.nx * st.ny, "y")
    _check(lib().stencil2d_apply(st.handle, precision, _ptr(x), _ptr(y), _stream(stream)))
    ms = ctypes.c_double(0.0)
    _check(lib().stencil2d_last_ms(st.handle, ctypes.byref(ms)))
    return ms.value


def stencil2d_set_tiles(st: Stencil2D, tiles_x: int, tiles_y: int):
    """The paper's tiled output-halo SpMV (R24) for stencil2d_apply; (1, 1) = gather."""
    _check(lib().stencil2d_set_tiles(st.handle, int(tiles_x), int(tiles_y)))


def stencil2d_set_timing(st: Stencil2D, enable: bool):
    _check(lib().stencil2d_set_timing(st.handle, 1 if enable else 0))


def stencil2d_phase_ms(st: Stencil2D):
    """(mean ms of H1, H2, H3 over the last timed 2D solve, iterations timed)"""
    ms = np.zeros(3, np.float64)
    n = ctypes.c_longlong(0)
    _check(lib().stencil2d_phase_ms(st.handle, ms.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
    return ms, n.value


def bicgstab2d_solve(st: Stencil2D, precision: int, b, x0, tol: float, maxit: int, x_out, stream=None):
    """BiCGStab on the 2D 9-point operator (R25).  Returns (iters, res_hist, status)."""
    n = st.nx * st.ny
    _check_vec(b, precision, n, "b")
    _check_vec(x_out, precision, n, "x_out")
    if x0 is not None:
        _check_vec(x0, precision, n, "x0")
    hist = np.zeros(max(maxit, 0) + 1, dtype=np.float64)
    it = ctypes.c_int(0)
    status = ctypes.c_int(-1)
    _check(lib().bicgstab2d_solve(st.handle, precision, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(x_out),
                                  ctypes.byref(it), hist.ctypes.data_as(ctypes.c_void_p), ctypes.byref(status),
                                  _stream(stream)))
    ms = ctypes.c_double(0.0)
    _check(lib().stencil2d_last_ms(st.handle, ctypes.byref(ms)))
    st.last_solve_ms = ms.value
    return it.value, hist[: it.value + 1].copy(), status.value


def p2p_export(st: Stencil, precision: int) -> bytes:
    n = ctypes.c_size_t(0)
    _check(lib().sten_p2p_export(st.handle, precision, None, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _check(lib().sten_p2p_export(st.handle, precision, buf, ctypes.byref(n)))
    return buf.raw[: n.value]


def p2p_import(st: Stencil, precision: int, records):
    """records: every rank's p2p_export() bytes, in rank order."""
    size = len(records[0])
    if any(len(r) != size for r in records):
        raise StenError("p2p records differ in size")
    blob = b"".join(records)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(lib().sten_p2p_import(st.handle, precision, buf, size))


def p2p_setup(st: Stencil, precision: int):
    """Exchange the IPC records over the default torch.distributed group and import them
    (selects the fused peer-memory halo + all-reduce path across ranks)."""
    import torch.distributed as dist
    mine = p2p_export(st, precision)
    allrec = [None] * dist.get_world_size()
    dist.all_gather_object(allrec, mine)
    p2p_import(st, precision, allrec)
