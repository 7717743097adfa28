"""Counter-based generator for the synthetic 7-point-stencil test problems.

Every random value is a pure function of (seed, stream, global linear index),
global index = i + nx*(j + ny*k_global), x fastest, z slowest.  The mixing
function is the SplitMix64 finalizer; a uniform in [0,1) takes the top 53
bits.  ``uniform(a, b) = a + (b - a) * u`` is evaluated with two separately
rounded fp64 operations (no FMA) - the CUDA twin (gen_cuda.cu) uses
__dmul_rn/__dadd_rn so both sides agree bit for bit.

Problem kinds (readings of BASELINE.json configs):

* KIND_POISSON  - constant 7-point Poisson matrix: diagonal 6, off-diagonals -1
  (config 1).  Dirichlet-zero boundary: the diagonal keeps all six
  neighbours' weight; entries that would couple to points outside the mesh are
  present in the fields but ignored by the solver's Jacobi-scaling step.
* KIND_CD       - first-order upwinded convection-diffusion (the MFIX scheme
  family): per point k~U(0.5,2) (stream 1), velocity
  (ux,uy,uz)~U(-1,1)^3 (streams 2-4); a_xm = k + max(ux,0),
  a_xp = k + max(-ux,0) (same for y, z); a_P = (1+delta) * sum(a_nb);
  A[P,P] = a_P, A[P,nb] = -a_nb (configs 2-4).
* KIND_CD_WEAK  - as KIND_CD but k = kz(z_global) * (1 + 0.1*xi), xi~U(-1,1)
  (stream 5), kz(z) = 1.25 + 0.75*sin(2*pi*z/512) (config 5).  The kz table is
  computed here once on the host and handed to the CUDA twin, so no
  transcendental is evaluated on two different math libraries.

* 2D (problem_fields_2d; the paper's 9-point SpMV / BiCG sketch, PAPER.md:362-373,
  gives no test matrix): first-order upwinded convection-diffusion on an nx*ny
  mesh with the 9-point Laplacian's corner couplings: per point k~U(0.5,2)
  (stream 1), (ux,uy)~U(-1,1)^2 (streams 2-3); faces a_xm = k + max(ux,0),
  a_xp = k + max(-ux,0), a_ym = k + max(uy,0), a_yp = k + max(-uy,0); corners
  a_c = k/4 (the 4:1 face:corner ratio of the "Mehrstellen" 9-point Laplacian);
  a_P = (1+delta) * sum(a_nb) summed in the o2d.c neighbour order; A[P,nb] = -a_nb.
  Index i + nx*j.

The right-hand side b ~ U(-1,1) (stream 0) is the right-hand side of the
ORIGINAL (un-scaled) system A x = b.
"""
from __future__ import annotations

import numpy as np

SEED_DEFAULT = 1

STREAM_B = 0
STREAM_K = 1
STREAM_UX = 2
STREAM_UY = 3
STREAM_UZ = 4
STREAM_NOISE = 5

KIND_POISSON = 0
KIND_CD = 1
KIND_CD_WEAK = 2

_C_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C_STREAM = np.uint64(0xD1B54A32D192ED03)
_C_OFF = np.uint64(0x632BE59BD9B4E019)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = float(2.0 ** -53)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k = np.array([np.uint64(seed) * _C_GOLD + np.uint64(stream) * _C_STREAM + _C_OFF],
                     dtype=np.uint64)
    return _mix(k)[0]


def hash_u64(seed: int, stream: int, idx) -> np.ndarray:
    """h = mix(key(seed,stream) + (idx+1)*GOLD)  (all mod 2^64)."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _key(seed, stream) + (idx + np.uint64(1)) * _C_GOLD
    return _mix(z)


def uniform01(seed: int, stream: int, idx) -> np.ndarray:
    return (hash_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * _TWO_M53


def uniform(seed: int, stream: int, idx, a: float, b: float) -> np.ndarray:
    u = uniform01(seed, stream, idx)
    w = np.float64(b) - np.float64(a)
    t = w * u            # rounded product
    return np.float64(a) + t   # rounded sum


def weak_kz_table(nz_global: int, period: int = 512) -> np.ndarray:
    z = np.arange(nz_global, dtype=np.float64)
    return 1.25 + 0.75 * np.sin(2.0 * np.pi * z / float(period))


def field_at(kind: int, nx: int, ny: int, i, j, kg, seed: int = SEED_DEFAULT,
             delta: float = 0.1, kz_table=None):
    """(diag, [off_xm, off_xp, off_ym, off_yp, off_zm, off_zp]) at global points.

    ``i, j, kg`` are integer arrays (kg = global z index).  Returns fp64 arrays.
    """
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    kg = np.asarray(kg, dtype=np.int64)
    shape = np.broadcast(i, j, kg).shape
    if kind == KIND_POISSON:
        diag = np.full(shape, 6.0)
        offs = [np.full(shape, -1.0) for _ in range(6)]
        return diag, offs
    idx = (np.broadcast_to(i, shape) + nx * (np.broadcast_to(j, shape) + ny * np.broadcast_to(kg, shape)))
    idx = idx.astype(np.uint64)
    if kind == KIND_CD:
        kd = uniform(seed, STREAM_K, idx, 0.5, 2.0)
    elif kind == KIND_CD_WEAK:
        if kz_table is None:
            raise ValueError("KIND_CD_WEAK needs kz_table")
        xi = uniform(seed, STREAM_NOISE, idx, -1.0, 1.0)
        kz = np.asarray(kz_table, dtype=np.float64)[np.broadcast_to(kg, shape)]
        kd = kz * (1.0 + 0.1 * xi)
    else:
        raise ValueError(f"unknown kind {kind}")
    ux = uniform(seed, STREAM_UX, idx, -1.0, 1.0)
    uy = uniform(seed, STREAM_UY, idx, -1.0, 1.0)
    uz = uniform(seed, STREAM_UZ, idx, -1.0, 1.0)
    a = [kd + np.maximum(ux, 0.0), kd + np.maximum(-ux, 0.0),
         kd + np.maximum(uy, 0.0), kd + np.maximum(-uy, 0.0),
         kd + np.maximum(uz, 0.0), kd + np.maximum(-uz, 0.0)]
    s = a[0] + a[1]
    s = s + a[2]
    s = s + a[3]
    s = s + a[4]
    s = s + a[5]
    diag = (1.0 + float(delta)) * s
    offs = [-ai for ai in a]
    return diag, offs


def problem_fields(kind: int, nx: int, ny: int, nz: int, z0: int = 0,
                   seed: int = SEED_DEFAULT, delta: float = 0.1, kz_table=None):
    """Fields of planes [z0, z0+nz) of the global mesh, each shaped (nz, ny, nx)."""
    kg, j, i = np.meshgrid(np.arange(z0, z0 + nz), np.arange(ny), np.arange(nx), indexing="ij")
    diag, offs = field_at(kind, nx, ny, i, j, kg, seed=seed, delta=delta, kz_table=kz_table)
    return np.ascontiguousarray(diag), [np.ascontiguousarray(o) for o in offs]


def rhs_uniform(nx: int, ny: int, nz: int, z0: int = 0, seed: int = SEED_DEFAULT,
                stream: int = STREAM_B) -> np.ndarray:
    """b ~ U(-1,1) (or x_true for config 1) on planes [z0, z0+nz), shape (nz,ny,nx)."""
    kg, j, i = np.meshgrid(np.arange(z0, z0 + nz), np.arange(ny), np.arange(nx), indexing="ij")
    idx = (i + nx * (j + ny * kg)).astype(np.uint64)
    return uniform(seed, stream, idx, -1.0, 1.0)


def field_at_2d(nx: int, i, j, seed: int = SEED_DEFAULT, delta: float = 0.1):
    """(diag, offs[8]) of the 2D 9-point stand-in at global points (i, j) of an nx-wide mesh
    (integer arrays), offs in the o2d.c order (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1)
    (0,+1) (+1,+1).  fp64."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    i, j = np.broadcast_arrays(i, j)
    idx = (i + nx * j).astype(np.uint64)
    kd = uniform(seed, STREAM_K, idx, 0.5, 2.0)
    ux = uniform(seed, STREAM_UX, idx, -1.0, 1.0)
    uy = uniform(seed, STREAM_UY, idx, -1.0, 1.0)
    corner = 0.25 * kd
    a = [corner, kd + np.maximum(uy, 0.0), corner, kd + np.maximum(ux, 0.0), kd + np.maximum(-ux, 0.0),
         corner, kd + np.maximum(-uy, 0.0), corner]
    s = a[0] + a[1]
    for d in range(2, 8):
        s = s + a[d]
    diag = (1.0 + float(delta)) * s
    return np.ascontiguousarray(diag), [np.ascontiguousarray(-ad) for ad in a]


def problem_fields_2d(nx: int, ny: int, seed: int = SEED_DEFAULT, delta: float = 0.1):
    """(diag, offs[8]) of the 2D 9-point stand-in, arrays (ny, nx), offs in the o2d.c order
    (-1,-1) (0,-1) (+1,-1) (-1,0) (+1,0) (-1,+1) (0,+1) (+1,+1)."""
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    return field_at_2d(nx, i, j, seed=seed, delta=delta)


def rhs_uniform_2d(nx: int, ny: int, seed: int = SEED_DEFAULT, stream: int = STREAM_B) -> np.ndarray:
    """b ~ U(-1,1) on the 2D mesh, shape (ny, nx)."""
    j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    return uniform(seed, stream, (i + nx * j).astype(np.uint64), -1.0, 1.0)
