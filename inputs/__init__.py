"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This package holds NO arithmetic of the method (no Jacobi scaling, no SpMV, no
BiCGStab step). It only draws the random fields that define a test problem
(the un-scaled 7-point matrix entries and the right-hand side) from a
counter-based generator, so that every consumer - numpy here, the CUDA twin in
``gen_cuda.cu`` - produces bit-identical values for any global mesh index,
independent of how the mesh is split into z-slabs.

See DESIGN.md "Input recipe" for the readings of the paper this follows
(PAPER.md:459-461 mesh shape; BASELINE.json configs 1-5).
"""
from .gen import (  # noqa: F401
    SEED_DEFAULT,
    STREAM_B,
    STREAM_K,
    STREAM_UX,
    STREAM_UY,
    STREAM_UZ,
    STREAM_NOISE,
    KIND_POISSON,
    KIND_CD,
    KIND_CD_WEAK,
    hash_u64,
    uniform01,
    uniform,
    weak_kz_table,
    problem_fields,
    rhs_uniform,
    field_at,
    problem_fields_2d,
    field_at_2d,
    rhs_uniform_2d,
)
