"""CPU oracle timing (SURVEY.md §8(d) "CPU oracle timing"): the oracle as it stands, on
the GPU box's host cores -- O64 (all cores and one thread) on configs 1 and 2 and a
600x595x192 slab of config 3, O16 on configs 1 and 2 and a 600x595x16 slab -- plus a
STREAM-like host copy bandwidth measured in the same run.  A baseline for context,
not a target.  Writes profiles/<tag>_cpu_oracle.md.

Each measurement runs in a subprocess so OMP_NUM_THREADS takes effect."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(kind, nx, ny, nz, prec, iters):
    """Child: build the scaled system, time `iters` BiCGStab iterations of the oracle."""
    import numpy as np

    import inputs
    import oracle as orc
    k = {"poisson": inputs.KIND_POISSON, "cd": inputs.KIND_CD}[kind]
    diag, offs = inputs.problem_fields(k, nx, ny, nz, seed=1, delta=0.1)
    b64 = inputs.rhs_uniform(nx, ny, nz, seed=1)
    c64 = orc.jacobi_scale(diag, offs)
    if prec == "O16":
        c16 = orc.quantize_coeffs(c64, "mixed")
        bh = orc.scale_rhs(orc.f16_from_double(b64), diag, "mixed")
        t0 = time.perf_counter()
        orc.bicgstab16(c16, bh, tol=0.0, maxit=iters)
    else:
        bh = b64 / diag
        t0 = time.perf_counter()
        orc.bicgstab64(c64, bh, tol=0.0, maxit=iters)
    dt = time.perf_counter() - t0
    pts = nx * ny * nz
    print(json.dumps({"s": dt, "gpts": pts * iters / dt / 1e9, "threads": orc.num_threads()}))
    del np


def host_copy_gbs():
    import numpy as np
    n = 1 << 28  # 2 GiB of float64
    a = np.ones(n)
    b = np.empty_like(a)
    np.copyto(b, a)
    best = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        np.copyto(b, a)
        best = max(best, 2 * a.nbytes / (time.perf_counter() - t0) / 1e9)
    return best


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def main(tag="r1"):
    cases = [("cfg 1 (32^3 Poisson)", "poisson", 32, 32, 32, 10),
             ("cfg 2 (128^3 cd)", "cd", 128, 128, 128, 10),
             ("cfg 3 slab 600x595x192", "cd", 600, 595, 192, 3),
             ("cfg 3 slab 600x595x16", "cd", 600, 595, 16, 3)]
    rows = []
    for label, kind, nx, ny, nz, iters in cases:
        for prec in ("O64", "O16"):
            if prec == "O16" and nz == 192:
                continue  # software fp16: the 16-plane slab stands for config 3
            if prec == "O64" and nz == 16:
                continue
            for threads in ("all", "1"):
                env = dict(os.environ)
                if threads == "1":
                    env["OMP_NUM_THREADS"] = "1"
                its = iters if threads == "all" or nz < 64 else 1
                out = subprocess.run([sys.executable, __file__, "--one", kind, str(nx), str(ny), str(nz), prec,
                                      str(its)], env=env, capture_output=True, text=True, timeout=1800)
                if out.returncode != 0:
                    rows.append(f"| {label} | {prec} | {threads} | failed: {out.stderr.strip()[-120:]} | | |")
                    continue
                r = json.loads(out.stdout.strip().splitlines()[-1])
                rows.append(f"| {label} | {prec} | {r['threads']} | {its} | {r['s']:.2f} | {r['gpts'] * 1e3:.2f} |")
                print(rows[-1], flush=True)
    bw = host_copy_gbs()
    text = [f"# {tag}: CPU oracle timing on the GPU box's host (`python tools/cpu_oracle_study.py`)\n",
            f"Host: {cpu_model()}, {os.cpu_count()} logical CPUs; STREAM-like copy (numpy, one thread, "
            f"2 GiB, read + write bytes): {bw:.1f} GB/s.\n",
            "The oracle as it stands (plain C, OpenMP over z-planes where it has loops to share; O16 is exact "
            "binary16 arithmetic in software). Inputs as in bench.py (seed 1, delta 0.1). Context only: the "
            "GPU/CPU ratio says nothing about kernel quality, the roofline fraction does.\n",
            "| case | oracle | threads | iterations | seconds | Mpoint-iter/s |", "|---|---|---|---|---|---|"]
    text += rows
    path = os.path.join(ROOT, "profiles", f"{tag}_cpu_oracle.md")
    with open(path, "w") as f:
        f.write("\n".join(text) + "\n")
    print("\n".join(text))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(sys.argv[2], *(int(v) for v in sys.argv[3:6]), sys.argv[6], int(sys.argv[7]))
    else:
        main(*(sys.argv[1:2] or ["r1"]))
