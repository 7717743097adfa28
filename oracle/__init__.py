"""ctypes binding of the CPU oracle (liboracle.so, plain C in this directory).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py - never by the product
package.  See oracle.h for what each function computes and which passage of
/root/reference/PAPER.md it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["o64.c", "o16.c", "osr.c", "o2d.c"]

ORC_CONVERGED, ORC_MAXIT, ORC_BREAKDOWN, ORC_NONFINITE = 0, 1, 2, 3


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, s) for s in _SOURCES]
    hdr = os.path.join(_HERE, "oracle.h")
    if not force and os.path.exists(_LIB_PATH):
        newest = max(os.path.getmtime(p) for p in srcs + [hdr])
        if os.path.getmtime(_LIB_PATH) >= newest:
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
           "-ffp-contract=off", "-fno-fast-math", "-Wall", "-o", _LIB_PATH + ".tmp"] + srcs + ["-lm"]
    subprocess.check_call(cmd, cwd=_HERE)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _declare(_lib)
    return _lib


_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_I64 = ctypes.c_int64
_U16 = ctypes.c_uint16


def _declare(L):
    L.o64_jacobi_scale.argtypes = [_I, _I, _I, _P, _P, _P]
    L.o64_apply.argtypes = [_I, _I, _I, _P, _P, _P]
    L.o64_apply_raw.argtypes = [_I, _I, _I, _P, _P, _P, _P]
    L.o64_dot.argtypes = [_I64, _P, _P]
    L.oracle_set_threads.argtypes = [_I]
    for f in ("o64_apply9_tiles", "o32_apply9_tiles", "o16_apply9_tiles"):
        getattr(L, f).argtypes = [_I, _I, _I, _I, _P, _P, _P]
    for f in ("o2d64_bicgstab", "o2d16_bicgstab"):
        getattr(L, f).argtypes = [_I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P]
        getattr(L, f).restype = _I
    for f in ("o2d64_bicgstab_tiles", "o2d16_bicgstab_tiles"):
        getattr(L, f).argtypes = [_I, _I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P]
        getattr(L, f).restype = _I
    L.o64_dot.restype = _D
    L.o64_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P]
    L.o64_bicgstab.restype = _I
    L.o64_true_residual.argtypes = [_I, _I, _I, _P, _P, _P]
    L.o64_true_residual.restype = _D
    L.o16_to_double.argtypes = [_U16]
    L.o16_to_double.restype = _D
    L.o16_from_double.argtypes = [_D]
    L.o16_from_double.restype = _U16
    for f in ("o16_fma",):
        getattr(L, f).argtypes = [_U16, _U16, _U16]
        getattr(L, f).restype = _U16
    for f in ("o16_add", "o16_mul"):
        getattr(L, f).argtypes = [_U16, _U16]
        getattr(L, f).restype = _U16
    L.o16_from_double_array.argtypes = [_I64, _P, _P]
    L.o16_to_double_array.argtypes = [_I64, _P, _P]
    L.o16_fma_array.argtypes = [_I64, _P, _P, _P, _P]
    L.o16_add_array.argtypes = [_I64, _P, _P, _P]
    L.o32_fma_array.argtypes = [_I64, _P, _P, _P, _P]
    L.o16_mul_array.argtypes = [_I64, _P, _P, _P]
    L.o16_apply_fused.argtypes = [_I, _I, _I, _P, _P, _P]
    L.o16_apply_unfused.argtypes = [_I, _I, _I, _P, _P, _P]
    L.o16_dot.argtypes = [_I, _I, _I, _P, _P]
    L.o16_dot.restype = ctypes.c_float
    L.o16_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _I, _P, _P, _P, _P, _P, _P]
    L.o16h_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]
    L.o16h_bicgstab.restype = _I
    L.o16_bicgstab.restype = _I
    L.o32_apply_fma.argtypes = [_I, _I, _I, _P, _P, _P]
    L.oracle_num_threads.restype = _I
    L.o64_jacobi_scale9.argtypes = [_I, _I, _P, _P, _P]
    L.o64_apply9.argtypes = [_I, _I, _P, _P, _P]
    L.o16_apply9.argtypes = [_I, _I, _P, _P, _P]
    L.o32_apply9.argtypes = [_I, _I, _P, _P, _P]
    L.o64_sr_sweep.argtypes = [_I, _I, _I, _P, _D, _D, _D, _P, _P, _P, _P, _P, _P, _P, _P]
    L.o16_sr_sweep.argtypes = [_I, _I, _I, _P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                               _P, _P, _P, _P, _P, _P, _P, _P]
    L.o32_sr_sweep.argtypes = [_I, _I, _I, _P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                               _P, _P, _P, _P, _P, _P, _P, _P]
    L.o64_sr_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P]
    L.o64_sr_bicgstab.restype = _I
    L.o16_sr_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _P, _P, _P, _P, _P, _P]
    L.o16_sr_bicgstab.restype = _I
    L.o16h_dot.argtypes = [_I, _I, _I, _P, _P, _I, _P, _P, _P]
    L.o16h_sr_sweep.argtypes = [_I, _I, _I, _P, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _P]
    L.o16h_sr_bicgstab.argtypes = [_I, _I, _I, _P, _P, _P, _D, _I, _I, _P, _P, _P, _P, _P, _P, _P]
    L.o16h_sr_bicgstab.restype = _I


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _arr6(arrs):
    t = (ctypes.c_void_p * 6)(*[a.ctypes.data for a in arrs])
    return t


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------- fp64 ----------------

def jacobi_scale(diag, offs):
    """Jacobi-scaled couplings c_d = off_d / diag (0 out of mesh). Shapes (nz,ny,nx)."""
    offs = [_c(o, np.float64) for o in offs]
    nz, ny, nx = offs[0].shape
    d = None if diag is None else _c(diag, np.float64)
    out = [np.empty((nz, ny, nx), np.float64) for _ in range(6)]
    lib().o64_jacobi_scale(nx, ny, nz, None if d is None else _ptr(d), _arr6(offs), _arr6(out))
    return out


def apply64(c, v):
    c = [_c(a, np.float64) for a in c]
    v = _c(v, np.float64)
    nz, ny, nx = v.shape
    u = np.empty_like(v)
    lib().o64_apply(nx, ny, nz, _arr6(c), _ptr(v), _ptr(u))
    return u


def apply_raw64(diag, offs, v):
    offs = [_c(a, np.float64) for a in offs]
    diag = _c(diag, np.float64)
    v = _c(v, np.float64)
    nz, ny, nx = v.shape
    u = np.empty_like(v)
    lib().o64_apply_raw(nx, ny, nz, _ptr(diag), _arr6(offs), _ptr(v), _ptr(u))
    return u


def dot64(a, b):
    a = _c(a, np.float64).ravel()
    b = _c(b, np.float64).ravel()
    return lib().o64_dot(a.size, _ptr(a), _ptr(b))


def bicgstab64(c, b, x0=None, tol=0.0, maxit=50, schedule="classic"):
    """Returns dict(x, hist, iters, status, event_it, alpha, omega).
    schedule "classic": Alg. 1 as printed; "sr": the single-reduction schedule (osr.c)."""
    c = [_c(a, np.float64) for a in c]
    b = _c(b, np.float64)
    nz, ny, nx = b.shape
    x = np.empty_like(b)
    hist = np.full(maxit + 1, np.nan)
    al = np.full(maxit + 1, np.nan)
    om = np.full(maxit + 1, np.nan)
    st = ctypes.c_int(-1)
    ev = ctypes.c_int(0)
    x0p = None if x0 is None else _ptr(_c(x0, np.float64))
    x0keep = None if x0 is None else _c(x0, np.float64)
    if x0keep is not None:
        x0p = _ptr(x0keep)
    fn = lib().o64_sr_bicgstab if schedule == "sr" else lib().o64_bicgstab
    it = fn(nx, ny, nz, _arr6(c), _ptr(b), x0p, float(tol), int(maxit),
                            _ptr(x), _ptr(hist), _ptr(al), _ptr(om), ctypes.byref(st), ctypes.byref(ev))
    return dict(x=x, hist=hist[: it + 1], iters=it, status=st.value, event_it=ev.value,
                alpha=al[1: it + 1], omega=om[1: it + 1])


def true_residual64(c, b, x):
    c = [_c(a, np.float64) for a in c]
    b = _c(b, np.float64)
    x = _c(x, np.float64)
    nz, ny, nx = b.shape
    return lib().o64_true_residual(nx, ny, nz, _arr6(c), _ptr(b), _ptr(x))


# ---------------- fp16 ----------------

def f16_from_double(x):
    """RNE rounding fp64 -> binary16 bit patterns (uint16)."""
    x = _c(x, np.float64)
    h = np.empty(x.shape, np.uint16)
    lib().o16_from_double_array(x.size, _ptr(x), _ptr(h))
    return h


def f16_to_double(h):
    h = _c(h, np.uint16)
    x = np.empty(h.shape, np.float64)
    lib().o16_to_double_array(h.size, _ptr(h), _ptr(x))
    return x


def fma16(a: int, b: int, c: int) -> int:
    return lib().o16_fma(a, b, c)


def add16(a: int, b: int) -> int:
    return lib().o16_add(a, b)


def mul16(a: int, b: int) -> int:
    return lib().o16_mul(a, b)


def fma16_array(a, b, c):
    a, b, c = (_c(t, np.uint16) for t in (a, b, c))
    out = np.empty(a.shape, np.uint16)
    lib().o16_fma_array(a.size, _ptr(a), _ptr(b), _ptr(c), _ptr(out))
    return out


def fma32_array(a, b, c):
    """a*b + c with ONE rounding to fp32 (C99 fmaf), element-wise; broadcasts scalars."""
    a, b, c = np.broadcast_arrays(*(np.asarray(t, np.float32) for t in (a, b, c)))
    a, b, c = (_c(t, np.float32) for t in (a, b, c))
    out = np.empty(a.shape, np.float32)
    lib().o32_fma_array(a.size, _ptr(a), _ptr(b), _ptr(c), _ptr(out))
    return out


def add16_array(a, b):
    a, b = (_c(t, np.uint16) for t in (a, b))
    out = np.empty(a.shape, np.uint16)
    lib().o16_add_array(a.size, _ptr(a), _ptr(b), _ptr(out))
    return out


def mul16_array(a, b):
    a, b = (_c(t, np.uint16) for t in (a, b))
    out = np.empty(a.shape, np.uint16)
    lib().o16_mul_array(a.size, _ptr(a), _ptr(b), _ptr(out))
    return out


def apply16(c16, v16, unfused: bool = False):
    c16 = [_c(a, np.uint16) for a in c16]
    v16 = _c(v16, np.uint16)
    nz, ny, nx = v16.shape
    u = np.empty_like(v16)
    f = lib().o16_apply_unfused if unfused else lib().o16_apply_fused
    f(nx, ny, nz, _arr6(c16), _ptr(v16), _ptr(u))
    return u


def dot16(a16, b16):
    a16 = _c(a16, np.uint16)
    b16 = _c(b16, np.uint16)
    nz, ny, nx = a16.shape
    return float(lib().o16_dot(nx, ny, nz, _ptr(a16), _ptr(b16)))


def _segments(segments, nz):
    seg = np.ascontiguousarray(np.asarray(segments, dtype=np.int32))
    if seg.ndim != 1 or len(seg) == 0 or seg[0] != 0 or np.any(np.diff(seg) <= 0) or seg[-1] >= max(nz, 1):
        raise ValueError(f"segments must start at 0 and ascend strictly below nz={nz}: {segments}")
    return seg


def dot16h(a16, b16, segments):
    """Half dot (R22): fp16 pencil per (x, y) column and z segment, exact sum of the
    segment sums.  Returns (sum, sum of |segment sums|)."""
    a16 = _c(a16, np.uint16)
    b16 = _c(b16, np.uint16)
    nz, ny, nx = a16.shape
    seg = _segments(segments, nz)
    sm, ab = ctypes.c_double(0.0), ctypes.c_double(0.0)
    lib().o16h_dot(nx, ny, nz, _ptr(a16), _ptr(b16), len(seg), _ptr(seg), ctypes.byref(sm), ctypes.byref(ab))
    return sm.value, ab.value


def bicgstab16(c16, b16, x0=None, tol=0.0, maxit=50, unfused=False, schedule="classic", segments=None):
    c16 = [_c(a, np.uint16) for a in c16]
    b16 = _c(b16, np.uint16)
    nz, ny, nx = b16.shape
    x = np.empty_like(b16)
    hist = np.full(maxit + 1, np.nan)
    al = np.full(maxit + 1, np.nan, np.float32)
    om = np.full(maxit + 1, np.nan, np.float32)
    st = ctypes.c_int(-1)
    ev = ctypes.c_int(0)
    x0keep = None if x0 is None else _c(x0, np.uint16)
    if schedule == "sr":
        if unfused:
            raise ValueError("the SR schedule has only the fused (GPU-mirroring) variant")
        seg = np.zeros(1, np.int32) if segments is None else _segments(segments, nz)
        it = lib().o16h_sr_bicgstab(nx, ny, nz, _arr6(c16), _ptr(b16),
                                    None if x0keep is None else _ptr(x0keep), float(tol), int(maxit),
                                    0 if segments is None else len(seg), _ptr(seg),
                                    _ptr(x), _ptr(hist), _ptr(al), _ptr(om),
                                    ctypes.byref(st), ctypes.byref(ev))
    else:  # Alg. 1; segments: the iteration's dots as half-mode pencils (R22, R28)
        seg = np.zeros(1, np.int32) if segments is None else _segments(segments, nz)
        it = lib().o16h_bicgstab(nx, ny, nz, _arr6(c16), _ptr(b16),
                                 None if x0keep is None else _ptr(x0keep), float(tol), int(maxit),
                                 int(bool(unfused)), 0 if segments is None else len(seg), _ptr(seg),
                                 _ptr(x), _ptr(hist), _ptr(al), _ptr(om), ctypes.byref(st), ctypes.byref(ev))
    return dict(x=x, hist=hist[: it + 1], iters=it, status=st.value, event_it=ev.value,
                alpha=al[1: it + 1], omega=om[1: it + 1])


# ---------------- single-reduction sweeps (osr.c) ----------------

def sr_sweep64(c, scalars, rh, x, r, p, v, q, y):
    """One SR sweep in fp64.  Returns (x, r, p, v, q, y, dots[12]) (new arrays)."""
    c = [_c(a, np.float64) for a in c]
    vecs = [_c(a, np.float64).copy() for a in (x, r, p, v, q, y)]
    rh = _c(rh, np.float64)
    nz, ny, nx = rh.shape
    dots = np.zeros(12, np.float64)
    a, w, b = (float(s) for s in scalars)
    lib().o64_sr_sweep(nx, ny, nz, _arr6(c), a, w, b, _ptr(rh), *[_ptr(t) for t in vecs], _ptr(dots))
    return (*vecs, dots)


def sr_sweep16(c16, scalars, rh, x, r, p, v, q, y, segments=None):
    """One SR sweep, fp16 mirror (uint16 bit patterns; fp32 scalars and dots).
    segments (list of first planes): half dots over those z segments (R22); then
    the result has a 9th element, the 12 scales (sums of |segment sums|)."""
    c16 = [_c(a, np.uint16) for a in c16]
    vecs = [_c(a, np.uint16).copy() for a in (x, r, p, v, q, y)]
    rh = _c(rh, np.uint16)
    nz, ny, nx = rh.shape
    dots = np.zeros(12, np.float32)
    a, w, b = (float(np.float32(s)) for s in scalars)
    if segments is None:
        lib().o16_sr_sweep(nx, ny, nz, _arr6(c16), a, w, b, _ptr(rh), *[_ptr(t) for t in vecs], _ptr(dots))
        return (*vecs, dots)
    seg = _segments(segments, nz)
    dabs = np.zeros(12, np.float64)
    lib().o16h_sr_sweep(nx, ny, nz, _arr6(c16), a, w, b, _ptr(rh), *[_ptr(t) for t in vecs], len(seg), _ptr(seg),
                        _ptr(dots), _ptr(dabs))
    return (*vecs, dots, dabs)


def sr_sweep32(c32, scalars, rh, x, r, p, v, q, y):
    """One SR sweep, fp32 mirror of the GPU's element-wise order (dots in fp64)."""
    c32 = [_c(a, np.float32) for a in c32]
    vecs = [_c(a, np.float32).copy() for a in (x, r, p, v, q, y)]
    rh = _c(rh, np.float32)
    nz, ny, nx = rh.shape
    dots = np.zeros(12, np.float64)
    a, w, b = (float(np.float32(s)) for s in scalars)
    lib().o32_sr_sweep(nx, ny, nz, _arr6(c32), a, w, b, _ptr(rh), *[_ptr(t) for t in vecs], _ptr(dots))
    return (*vecs, dots)


# ---------------- iterative refinement (R21) ----------------

def refine16(c64, bhat32, x0=None, tol=1e-6, outer_maxit=20, inner_tol=1e-3, inner_maxit=100, schedule="classic"):
    """Mixed-precision iterative refinement, step by step as R21 states it
    (PAPER.md:591, 598 name iterative refinement as the remedy for the fp16
    plateau).  Composes the pinned pieces: the fp32 FMA-chain SpMV mirror
    (apply32_fma), fp32 element-wise arithmetic (numpy float32), binary16
    rounding (f16_from_double) and the O16 solver (bicgstab16).
    bhat32: the scaled right-hand side b_hat (float32).  The first stagnation
    (three outer steps without a 1% gain) switches the inner solves to the
    other schedule (classic <-> sr: they round differently, and on weakly
    dominant systems either fp16 iteration can stall where the other still
    gains) instead of stopping; the second one stops (BREAKDOWN).  An inner
    solve that ends NONFINITE (fp16 overflow) adds no update to x and halves
    the inner iteration cap for the rest of the call.  Returns dict(x (float32), hist (outer
    residuals), outer, inner, status, handover (outer step of the switch, or -1))."""
    c32 = quantize_coeffs(c64, "fp32")
    c16 = quantize_coeffs(c64, "mixed")
    b = np.asarray(bhat32, np.float32)
    nb = float(np.sqrt(np.sum(b.astype(np.float64) ** 2)))
    x = np.zeros_like(b) if x0 is None else np.asarray(x0, np.float32).copy()
    if nb == 0.0:
        return dict(x=np.zeros_like(b), hist=np.array([0.0]), outer=0, inner=0, status=ORC_CONVERGED, handover=-1)
    hist, inner, status, best, stale, handover = [], 0, ORC_MAXIT, None, 0, -1
    for k in range(outer_maxit + 1):
        r = b - apply32_fma(c32, x)                      # fp32: one rounding per element
        res = float(np.sqrt(np.sum(r.astype(np.float64) ** 2))) / nb
        hist.append(res)
        if not np.isfinite(res):
            status = ORC_NONFINITE
            break
        if res <= tol:
            status = ORC_CONVERGED
            break
        if best is None or res < 0.99 * best:          # stagnation: 3 steps without a 1% gain
            best = res if best is None else min(best, res)
            stale = 0
        else:
            stale += 1
            if stale >= 3:
                if handover < 0:  # R21: the first stagnation switches the inner schedule
                    schedule, stale, handover = ("classic" if schedule == "sr" else "sr"), 0, k
                else:
                    status = ORC_BREAKDOWN
                    break
        if k == outer_maxit:
            break
        sigma = 2.0 ** np.frexp(float(np.max(np.abs(r))))[1]  # power of two >= max|r|
        r16 = f16_from_double(r.astype(np.float64) / sigma)
        d = bicgstab16(c16, r16, tol=inner_tol, maxit=inner_maxit, schedule=schedule)
        inner += d["iters"]
        if d["status"] == ORC_NONFINITE:  # R21: a diverged inner solve adds nothing; the cap halves
            inner_maxit = max(1, inner_maxit // 2)
            continue
        x = (x.astype(np.float64) + sigma * f16_to_double(d["x"])).astype(np.float32)
    return dict(x=x, hist=np.array(hist), outer=len(hist) - 1, inner=inner, status=status, handover=handover)


# ---------------- 2D 9-point SpMV (o2d.c) ----------------

def _arr8(arrs):
    return (ctypes.c_void_p * 8)(*[a.ctypes.data for a in arrs])


def jacobi_scale9(diag, offs):
    """Scaled couplings of the 2D 9-point operator; arrays (ny, nx), offs in the o2d.c order."""
    offs = [_c(o, np.float64) for o in offs]
    ny, nx = offs[0].shape
    d = None if diag is None else _c(diag, np.float64)
    out = [np.empty((ny, nx), np.float64) for _ in range(8)]
    lib().o64_jacobi_scale9(nx, ny, None if d is None else _ptr(d), _arr8(offs), _arr8(out))
    return out


def apply9_64(c, v):
    c = [_c(a, np.float64) for a in c]
    v = _c(v, np.float64)
    ny, nx = v.shape
    u = np.empty_like(v)
    lib().o64_apply9(nx, ny, _arr8(c), _ptr(v), _ptr(u))
    return u


def apply9_16(c16, v16):
    c16 = [_c(a, np.uint16) for a in c16]
    v16 = _c(v16, np.uint16)
    ny, nx = v16.shape
    u = np.empty_like(v16)
    lib().o16_apply9(nx, ny, _arr8(c16), _ptr(v16), _ptr(u))
    return u


def apply9_32(c32, v32):
    c32 = [_c(a, np.float32) for a in c32]
    v32 = _c(v32, np.float32)
    ny, nx = v32.shape
    u = np.empty_like(v32)
    lib().o32_apply9(nx, ny, _arr8(c32), _ptr(v32), _ptr(u))
    return u


def apply9_tiles(c, v, tiles, prec="fp64"):
    """The paper's tiled 2D SpMV (o2d.c): tiles = (TX, TY); prec fp64 / fp32 /
    mixed (binary16 bit patterns)."""
    TX, TY = tiles
    dt = {"fp64": np.float64, "fp32": np.float32, "mixed": np.uint16}[prec]
    c = [_c(a, dt) for a in c]
    v = _c(v, dt)
    ny, nx = v.shape
    u = np.empty_like(v)
    fn = {"fp64": lib().o64_apply9_tiles, "fp32": lib().o32_apply9_tiles, "mixed": lib().o16_apply9_tiles}[prec]
    fn(nx, ny, int(TX), int(TY), _arr8(c), _ptr(v), _ptr(u))
    return u


def bicgstab2d(c, b, x0=None, tol=0.0, maxit=50, prec="fp64", tiles=(1, 1)):
    """BiCGStab on the 2D 9-point operator: prec fp64 (float64 arrays) or mixed
    (binary16 bit patterns, the GPU's operation order); tiles = (TX, TY) > (1, 1): the paper's tiled
    output-halo SpMV (R24).  Returns dict(x, hist, iters, status, event_it, alpha, omega) like
    bicgstab64."""
    dt = np.float64 if prec == "fp64" else np.uint16
    c = [_c(a, dt) for a in c]
    b = _c(b, dt)
    ny, nx = b.shape
    x = np.empty_like(b)
    hist = np.zeros(maxit + 1)
    ad = np.float64 if prec == "fp64" else np.float32
    al, om = np.zeros(maxit + 1, ad), np.zeros(maxit + 1, ad)
    st, ev = ctypes.c_int(0), ctypes.c_int(0)
    x0c = None if x0 is None else _c(x0, dt)
    fn = lib().o2d64_bicgstab_tiles if prec == "fp64" else lib().o2d16_bicgstab_tiles
    it = fn(nx, ny, int(tiles[0]), int(tiles[1]), _arr8(c), _ptr(b), None if x0c is None else _ptr(x0c), float(tol),
            int(maxit), _ptr(x), _ptr(hist), _ptr(al), _ptr(om), ctypes.byref(st), ctypes.byref(ev))
    return dict(x=x, hist=hist[: it + 1], iters=it, status=st.value, event_it=ev.value, alpha=al[: it + 1],
                omega=om[: it + 1])


# ---------------- fp32 mirror ----------------

def apply32_fma(c32, v32):
    c32 = [_c(a, np.float32) for a in c32]
    v32 = _c(v32, np.float32)
    nz, ny, nx = v32.shape
    u = np.empty_like(v32)
    lib().o32_apply_fma(nx, ny, nz, _arr6(c32), _ptr(v32), _ptr(u))
    return u


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle's loops (timing only)."""
    lib().oracle_set_threads(int(n))


# ---------------- quantisation helpers (R3: RN from the fp64 scaled value) ----

def quantize_coeffs(c64, precision: str):
    """Round the fp64 Jacobi-scaled couplings to the working precision."""
    if precision == "fp32":
        return [np.asarray(a, np.float64).astype(np.float32) for a in c64]
    return [f16_from_double(a) for a in c64]


def scale_rhs(b_work, diag, precision: str):
    """b_hat = rn_w(b / diag) in fp64 (R3).  b_work holds working-precision values
    (float32 array or uint16 fp16 bit patterns)."""
    if precision == "fp32":
        bd = np.asarray(b_work, np.float32).astype(np.float64)
        return (bd / np.asarray(diag, np.float64)).astype(np.float32)
    bd = f16_to_double(b_work)
    return f16_from_double(bd / np.asarray(diag, np.float64))
