"""Helpers shared by the GPU parity tests: build the same problem for the CUDA
path (through the C ABI) and for the oracle, from the seeded input module."""
import numpy as np

import inputs
import oracle as orc


def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU test needs a CUDA device"
    return torch


def fields(kind, nx, ny, nz, delta=0.1, seed=1):
    return inputs.problem_fields(kind, nx, ny, nz, seed=seed, delta=delta)


def gpu_stencil(diag, offs, nslabs=1, unit_diag=False):
    torch = torch_cuda()
    import paper_2010_03660_b200 as sten
    nz, ny, nx = offs[0].shape
    coeffs = [None if unit_diag else torch.from_numpy(np.ascontiguousarray(diag)).cuda()]
    coeffs += [torch.from_numpy(np.ascontiguousarray(o)).cuda() for o in offs]
    st = sten.stencil_create(nx, ny, nz, coeffs, nslabs=nslabs)
    torch.cuda.synchronize()
    return st


def oracle_coeffs(diag, offs, prec, unit_diag=False):
    c64 = orc.jacobi_scale(None if unit_diag else diag, offs)
    return orc.quantize_coeffs(c64, prec)


def to_gpu_vec(a, prec):
    """numpy fp32 array, or fp16 bit patterns (uint16), -> CUDA tensor of the precision."""
    torch = torch_cuda()
    if prec == "fp32":
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint16).view(np.float16)).cuda()


def from_gpu_vec(t, prec):
    a = t.detach().cpu().numpy()
    return a.astype(np.float32) if prec == "fp32" else a.view(np.uint16)


def widen(a, prec):
    return a.astype(np.float64) if prec == "fp32" else orc.f16_to_double(a)


def quantize_vec(x64, prec):
    return x64.astype(np.float32) if prec == "fp32" else orc.f16_from_double(x64)


def rel_inf(a, ref):
    return float(np.max(np.abs(a - ref)) / max(np.max(np.abs(ref)), 1e-300))
