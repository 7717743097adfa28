"""Work and traffic accounting for the BiCGStab hot path (no arithmetic of the method).

Flops: the paper's count, 44 operations per meshpoint per iteration
(Table "Operations per meshpoint per iteration";
PAPER.md:462-464).  Split by fused phase:
  H1  p-update (2 AXPY = 4) + SpMV (12) + (rhat, v) dot (2)   = 18
  H2  s = r - alpha v (2) + SpMV (12) + (t,s), (t,t) dots (4) = 18
  H3  x += alpha p + omega s (4) + r = s - omega t (2) + (rhat, r) dot (2) = 8
The extra (r, r) dot used for stopping is not credited (as in the paper).

Bytes: ALGORITHMIC traffic of the fused schedule - one read or write of an
N-point array is one "pass":
  H1 reads r, p, v, rhat + 6 coefficients, writes p', v'     = 12 passes
  H2 reads r, v + 6 coefficients, writes s, t                = 10 passes
  H3 reads x, p, s, t, rhat, r... (r not read: r = s - w t), writes x, r = 7 passes
"""

FLOPS_PER_POINT_ITER = 44
PHASE_FLOPS = {"H1": 18, "H2": 18, "H3": 8}

PASSES = {"H1": 12, "H2": 10, "H3": 7}
PASSES_PER_ITER = sum(PASSES.values())  # 29

ELEM_BYTES = {"fp32": 4, "mixed": 2}

# Single-reduction schedule (R19): one sweep per iteration reads
# x, r, p, v, q, y, rhat + 6 coefficients and writes x, r, p, v, q, y.
PASSES_SR = 19


# constant-coefficient operator (stencil_create_const): no coefficient
# arrays are read - the SR sweep 13 passes, the classic phases H1 6, H2 4, H3 7 = 17
PASSES_SR_CONST = PASSES_SR - 6
PASSES_CONST = {"H1": PASSES["H1"] - 6, "H2": PASSES["H2"] - 6, "H3": PASSES["H3"]}
PASSES_PER_ITER_CONST = sum(PASSES_CONST.values())  # 17


def passes_per_iter(schedule: str = "classic", const_op: bool = False) -> int:
    if schedule == "sr":
        return PASSES_SR_CONST if const_op else PASSES_SR
    return PASSES_PER_ITER_CONST if const_op else PASSES_PER_ITER


def bytes_per_point_iter(precision: str, schedule: str = "classic", const_op: bool = False) -> int:
    return passes_per_iter(schedule, const_op) * ELEM_BYTES[precision]


def sweep_bytes(precision: str, npoints: int, const_op: bool = False) -> int:
    return (PASSES_SR_CONST if const_op else PASSES_SR) * ELEM_BYTES[precision] * npoints


def phase_bytes(phase: str, precision: str, npoints: int, const_op: bool = False) -> int:
    return (PASSES_CONST if const_op else PASSES)[phase] * ELEM_BYTES[precision] * npoints
