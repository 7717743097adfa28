"""ctypes binding of the device twin of the input generator (gen_cuda.cu).

Generates the same fields as gen.py directly into CUDA tensors - used for the
600x595x1536 configurations whose fp64 fields (7 x 4.4 GB) are impractical to
build in numpy and push over PCIe.  Bit-identity with gen.py is checked by
tests/test_gpu_parity.py::test_device_generator_matches_numpy.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .gen import SEED_DEFAULT, KIND_CD_WEAK, weak_kz_table

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libsten_inputs.so")
SRC = os.path.join(_HERE, "gen_cuda.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
           "-Xcompiler", "-fPIC", "-shared", SRC, "-o", LIB + ".tmp"]
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} not built (inputs.cuda.build())")
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        L.sten_inputs_fields.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong,
                                         ctypes.c_ulonglong, ctypes.c_double, P, P, P, P]
        L.sten_inputs_uniform.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_longlong,
                                          ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_int, P, P]
        L.sten_inputs_fields2d.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_double, P, P, P]
        _lib = L
    return _lib


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def fields_device(kind: int, nx: int, ny: int, nz: int, z0: int = 0, seed: int = SEED_DEFAULT,
                  delta: float = 0.1, kz_table=None, nz_global: int | None = None):
    """(diag, [off_xm..off_zp]) as fp64 CUDA tensors of shape (nz, ny, nx)."""
    import torch
    dev = torch.device("cuda")
    diag = torch.empty((nz, ny, nx), dtype=torch.float64, device=dev)
    offs = [torch.empty_like(diag) for _ in range(6)]
    kz = None
    if kind == KIND_CD_WEAK:
        if kz_table is None:
            kz_table = weak_kz_table(nz_global if nz_global is not None else z0 + nz)
        kz = torch.as_tensor(np.asarray(kz_table, np.float64), device=dev)
    arr = (ctypes.c_void_p * 6)(*[o.data_ptr() for o in offs])
    rc = lib().sten_inputs_fields(kind, nx, ny, nz, z0, seed, 1.0 + float(delta),
                                  None if kz is None else ctypes.c_void_p(kz.data_ptr()),
                                  ctypes.c_void_p(diag.data_ptr()), arr, _stream())
    if rc != 0:
        raise RuntimeError(f"sten_inputs_fields failed ({rc})")
    return diag, offs


def fields2d_device(nx: int, ny: int, seed: int = SEED_DEFAULT, delta: float = 0.1):
    """(diag, offs[8]) of the 2D 9-point stand-in as fp64 CUDA tensors (ny, nx) (gen.py problem_fields_2d)."""
    import torch
    diag = torch.empty((ny, nx), dtype=torch.float64, device="cuda")
    offs = [torch.empty_like(diag) for _ in range(8)]
    arr = (ctypes.c_void_p * 8)(*[o.data_ptr() for o in offs])
    rc = lib().sten_inputs_fields2d(nx, ny, seed, 1.0 + float(delta), ctypes.c_void_p(diag.data_ptr()), arr,
                                    _stream())
    if rc != 0:
        raise RuntimeError(f"sten_inputs_fields2d failed ({rc})")
    return diag, offs


def uniform_device(nx: int, ny: int, nz: int, z0: int = 0, seed: int = SEED_DEFAULT, stream: int = 0,
                   lo: float = -1.0, hi: float = 1.0, dtype: str = "f64"):
    import torch
    t = torch.empty((nz, ny, nx), dtype=torch.float64 if dtype == "f64" else torch.float32, device="cuda")
    rc = lib().sten_inputs_uniform(nx, ny, nz, z0, seed, stream, lo, hi, 0 if dtype == "f64" else 1,
                                   ctypes.c_void_p(t.data_ptr()), _stream())
    if rc != 0:
        raise RuntimeError(f"sten_inputs_uniform failed ({rc})")
    return t
