#!/usr/bin/env python
"""Benchmark: BiCGStab Gpoint-iter/s and % of the HBM roofline (BASELINE.json metric).

One "step" = one bicgstab_solve of the whole hot path (S1 init, then H1, H2, H3
for `maxit` iterations, tol = 0 so exactly maxit iterations run) on a synthetic
problem with the shape of the paper's run:
  N = 1 : config 3  - 600x595x1536, convection-diffusion (delta = 0.1), mixed fp16
  N > 1 : config 5  - weak scaling, 600x595x(1536*N), one 1536-plane z-slab per
          GPU, halo planes + fp32 scalar all-reduce over NCCL
  (`--workload` overrides; fp32 with --precision fp32).
Timing: W untimed warm-up steps, then K steps bracketed by barrier + device
sync, CUDA events on the solve's stream, max over ranks.  The working set
(16.5 GB) is > 100x the 126 MB L2, so no flush is needed between steps.

`--impl reference` times the CPU oracle (oracle/, O16 for mixed, O64 for fp32)
on a bounded z-slab sample of the same workload, on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NX, NY, NZ = 600, 595, 1536
PAPER_GPT_ITER_S = 548_352_000 / 28.1e-6 / 1e9  # CS-1: 19514 Gpt-iter/s
FALLBACK_HBM_GBS = 6650.0
METRIC = "BiCGStab Gpoint-iter/s & % HBM roofline, 600×595×1536 mixed fp16, 1–8 GPU"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="sten", choices=["sten", "reference"])
    p.add_argument("--precision", default="mixed", choices=["mixed", "fp32"])
    p.add_argument("--maxit", type=int, default=100)
    p.add_argument("--tol", type=float, default=0.0, help="0: exactly maxit iterations (config 3a)")
    p.add_argument("--workload", default="auto", choices=["auto", "cfg3", "cfg4", "cfg5"],
                   help="cfg3: 600x595x1536 on one GPU; cfg4: the same mesh split over the N GPUs (strong "
                        "scaling); cfg5: 600x595x(1536 N), one slab per GPU (weak scaling, default for N>1)")
    p.add_argument("--nz", type=int, default=NZ, help="planes per GPU (debug / profiling)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--schedule", default="sr", choices=["sr", "classic"],
                   help="sr: single-reduction sweep (19 passes, DESIGN.md R19); classic: Alg. 1 as printed (29)")
    p.add_argument("--dots", default="mixed", choices=["mixed", "half"],
                   help="mixed precision only: inner products as fp16 products summed in fp32 (the paper's "
                        "instruction), or half: fp16 column pencils (DESIGN.md R22, NEXT-4; SR schedule)")
    p.add_argument("--operator", default="fields", choices=["fields", "poisson-const"],
                   help="fields: the workload's per-point coefficient fields; poisson-const: the constant "
                        "7-point Poisson operator (config 1's) at the same mesh via stencil_create_const "
                        "(no coefficient streams in the SR sweep, NEXT-4)")
    p.add_argument("--tiling", default="", help="bx,by,zc,stages override (classic)")
    p.add_argument("--sr-tiling", default="", help="by,stages,cstages,zc override (sr)")
    p.add_argument("--cpu-planes", type=int, default=0, help="oracle sample planes (0 = auto)")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def measured_traffic(kernel_prefix: str):
    """DRAM bytes per launch of the dominant kernel from the latest committed ncu
    capture (profiles/<round>_traffic.json, full-size cfg3 launches)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for path in reversed(files):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        for k, launches in d.get("kernels", {}).items():
            if k.startswith(kernel_prefix) and launches:
                return (float(np.mean([x["traffic_bytes"] for x in launches])),
                        os.path.relpath(path, ROOT))
    return None, None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 6 and parts[0].isdigit():
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [int(r[0]) for r in rows]
        mx = max(int(r[1]) for r in rows)
        under = [s for s in sm if s > 0.5 * mx] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(statistics.median(under)), "sm_max_mhz": float(mx), "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------- oracle --
def oracle_sample(precision: str, workload: str, planes: int, iters: int, z0: int = 0):
    """Time the oracle as it stands on a z-slab sample [z0, z0+planes) of the workload."""
    import inputs
    import oracle as orc
    kind = inputs.KIND_CD_WEAK if workload == "cfg5" else inputs.KIND_CD
    kz = inputs.weak_kz_table(NZ) if kind == inputs.KIND_CD_WEAK else None
    diag, offs = inputs.problem_fields(kind, NX, NY, planes, z0=z0, seed=1, delta=0.1, kz_table=kz)
    b64 = inputs.rhs_uniform(NX, NY, planes, z0=z0, seed=1)
    c64 = orc.jacobi_scale(diag, offs)
    t0 = time.perf_counter()
    if precision == "mixed":
        c16 = orc.quantize_coeffs(c64, "mixed")
        bh = orc.scale_rhs(orc.f16_from_double(b64), diag, "mixed")
        t0 = time.perf_counter()
        orc.bicgstab16(c16, bh, tol=0.0, maxit=iters)
    else:
        c32 = [c.astype(np.float32).astype(np.float64) for c in c64]
        bh = orc.scale_rhs(b64.astype(np.float32), diag, "fp32").astype(np.float64)
        t0 = time.perf_counter()
        orc.bicgstab64(c32, bh, tol=0.0, maxit=iters)
    dt = time.perf_counter() - t0
    pts = NX * NY * planes
    return dict(value=pts * iters / dt / 1e9, unit="Gpoint-iter/s", cores=orc.num_threads(), kind="oracle",
                sample=f"{'O16' if precision == 'mixed' else 'O64'} BiCGStab, {iters} iterations on a "
                       f"{NX}x{NY}x{planes} z-slab of {workload} ({pts} points), {dt:.1f} s"), dt


def cpu_baseline_auto(precision, workload, planes_override=0):
    # size the sample to ~10-30 s of oracle work
    planes = planes_override or (16 if precision == "mixed" else 64)
    iters = 3
    res, dt = oracle_sample(precision, workload, planes, iters)
    return res


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    workload = args.workload if args.workload != "auto" else ("cfg3" if args.gpus == 1 else "cfg5")
    planes = args.cpu_planes or (2 if args.precision == "mixed" else 8)
    iters = 2
    for _ in range(args.warmup):
        oracle_sample(args.precision, workload, planes, 1)
    vals, dts = [], []
    for _ in range(args.steps):
        res, dt = oracle_sample(args.precision, workload, planes, iters)
        vals.append(res["value"])
        dts.append(dt)
    value = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "Gpoint-iter/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(dts)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": value / PAPER_GPT_ITER_S,
            "dtype": "f16" if args.precision == "mixed" else "f64", "data": "synthetic",
            "config": {"workload": workload, "mesh": [NX, NY, NZ], "precision": args.precision,
                       "sample_planes": planes, "iters_per_step": iters},
            "cpu_baseline": dict(res, value=value,
                                 sample=f"{args.steps} steps, each: " + res["sample"].rsplit(",", 1)[0]),
            "e2e": {"value": value, "unit": "Gpoint-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU --
def run_sten(args):
    import torch
    import torch.distributed as dist

    import inputs
    import inputs.cuda as icuda
    import paper_2010_03660_b200 as sten
    from paper_2010_03660_b200 import roofline

    rank, world, local = dist_env()
    n = world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    workload = args.workload if args.workload != "auto" else ("cfg3" if n == 1 else "cfg5")
    prec = sten.MIXED if args.precision == "mixed" else sten.FP32
    tdt = torch.float16 if prec == sten.MIXED else torch.float32
    from paper_2010_03660_b200 import dist as sdist
    # weak scaling (config 5): every rank owns one args.nz-plane slab of the global mesh;
    # strong scaling (config 4): the args.nz planes are split over the ranks
    strong = workload == "cfg4"
    z0, nzl = sdist.slab_of(rank, world, args.nz if strong else args.nz * world)

    comm = None
    if world > 1:
        comm = sdist.bootstrap_comm(sten, rank, world)

    # problem: fields of this rank's slab generated on the device (inputs/gen_cuda.cu)
    kind = inputs.KIND_CD_WEAK if workload == "cfg5" else inputs.KIND_CD
    kz = inputs.weak_kz_table(nzl * n) if kind == inputs.KIND_CD_WEAK else None
    if args.operator == "poisson-const":
        st = sten.stencil_create_const(NX, NY, nzl, (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0), nslabs=1, comm=comm)
    else:
        diag, offs = icuda.fields_device(kind, NX, NY, nzl, z0=z0, seed=1, delta=0.1, kz_table=kz)
        st = sten.stencil_create(NX, NY, nzl, [diag] + offs, nslabs=1, comm=comm)
        del diag, offs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if args.tiling:
        bx, by, zc, stg = (int(v) for v in args.tiling.split(","))
        sten.set_tiling(st, prec, bx, by, zc, stg)
    sr = args.schedule == "sr"
    sten.set_schedule(st, sten.SCHED_SR if sr else sten.SCHED_CLASSIC)
    if sr and world > 1 and os.environ.get("STEN_P2P", "0") == "1":
        sten.p2p_setup(st, prec)  # fused peer-memory halos + all-reduce across ranks (opt-in)
    if args.sr_tiling:
        sten.set_sr_tiling(st, prec, *(int(v) for v in args.sr_tiling.split(",")))
    if args.dots == "half":
        sten.set_dot_precision(st, sten.DOTS_HALF)
    b = icuda.uniform_device(NX, NY, nzl, z0=z0, seed=1, stream=0).to(tdt)
    x = torch.empty_like(b)
    maxit = args.maxit
    npts_local = NX * NY * nzl
    npts = npts_local * n

    def barrier():
        if world > 1:
            dist.barrier()

    tol = args.tol
    sten.set_timing(st, True)
    for _ in range(args.warmup):
        sten.bicgstab_solve(st, prec, b, None, tol, maxit, x)
    torch.cuda.synchronize()
    barrier()

    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    launches = 0
    h1_ms, h1_n = 0.0, 0
    ph_ms = [0.0, 0.0, 0.0]
    iters_done = 0
    barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    last = None
    for _ in range(args.steps):
        last = sten.bicgstab_solve(st, prec, b, None, tol, maxit, x)
        iters_done += last[0]
        s = sten.get_stats(st)
        launches += s["kernel_launches"]
        for p in range(3):
            ph_ms[p] += s["phase_ms"][p]
        h1_ms += s["phase_ms"][0]
        h1_n += s["phase_launches"][0]
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    t_ms = sdist.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    it, hist, status = last
    value = npts * iters_done / (t_ms / 1e3) / 1e9

    # end to end through the C ABI with pinned HOST buffers: one bicgstab_solve_batch call
    # solves the K steps' systems, every step's b uploaded and x downloaded (pipelined
    # with the neighbouring steps' solves on the library's copy stream)
    e2e = None
    if not args.no_e2e:
        bh = [b.cpu().pin_memory() for _ in range(2)]
        xh = [torch.empty_like(bh[0]).pin_memory() for _ in range(2)]
        sten.set_timing(st, False)
        sten.bicgstab_solve_batch(st, prec, bh, xh, tol, maxit)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sten.bicgstab_solve_batch(st, prec, [bh[i % 2] for i in range(args.steps)],
                                        [xh[i % 2] for i in range(args.steps)], tol, maxit)
        torch.cuda.synchronize()
        te = sdist.max_over_ranks(time.perf_counter() - t0, device="cuda")
        e_iters = sum(r[0] for r in res)
        esz = b.element_size()
        e2e = {"value": npts * e_iters / te / 1e9, "unit": "Gpoint-iter/s",
               "h2d_bytes_per_step": npts_local * esz,
               "d2h_bytes_per_step": npts_local * esz + 8 * (e_iters // max(args.steps, 1) + 1),
               "api": "bicgstab_solve_batch (pinned host b in, x out every step; copies overlap the "
                      "neighbouring steps' solves)", "clock": "host wall clock around the call"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_kind = measured_peak()
    pname = "mixed" if prec == sten.MIXED else "fp32"
    h1_avg_ms = h1_ms / max(h1_n, 1)
    # dominant kernel: the SR sweep (one per iteration) or the classic H1 stencil
    const_op = args.operator == "poisson-const"
    h1_bytes = (roofline.sweep_bytes(pname, npts_local, const_op) if sr
                else roofline.phase_bytes("H1", pname, npts_local))
    achieved = h1_bytes / (h1_avg_ms / 1e3) / 1e9
    bpi = roofline.bytes_per_point_iter(pname, args.schedule, const_op and sr)
    whole_gbs = npts_local * iters_done * bpi / (t_ms / 1e3) / 1e9
    tname = "half" if prec == sten.MIXED else "float"
    kname = f"k_sr<{tname}>" if sr else f"k_stencil<{tname},H1>"
    traffic, traffic_src = (None, None)
    if prec == sten.MIXED and nzl == NZ and not args.tiling and not args.sr_tiling and not const_op:
        traffic, traffic_src = measured_traffic("k_sr<__half" if sr else "k_stencil<__half, 1")
    line = {
        "metric": METRIC, "value": value, "unit": "Gpoint-iter/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": value / PAPER_GPT_ITER_S,
        "dtype": "f16" if prec == sten.MIXED else "f32", "data": "synthetic",
        "config": {"workload": workload, "mesh": [NX, NY, nzl * n], "mesh_per_gpu": [NX, NY, nzl],
                   "precision": pname, "schedule": args.schedule, "operator": args.operator,
                   **({"dots": "half"} if args.dots == "half" and prec == sten.MIXED else {}),
                   "maxit": maxit, "tol": tol,
                   "iters_per_solve": iters_done / args.steps,
                   "parallelism": f"zslab{n}",
                   "l2": "no flush: 16.5 GB working set per GPU >> 126 MB L2",
                   "gflops": value * roofline.FLOPS_PER_POINT_ITER,
                   "hbm_frac_whole_step": whole_gbs / peak, "bytes_per_point_iter": bpi,
                   "status": sten.STATUS_NAMES.get(status, status), "final_rel_residual": float(hist[-1])},
        "roofline": {"bound": "hbm", "kernel": kname,
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": h1_bytes, "avg_launch_ms": h1_avg_ms,
                     "phase_ms_per_iter": [p / max(h1_n, 1) for p in ph_ms][:1 if sr else 3]},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_auto(pname, workload, args.cpu_planes)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_sten(args)


if __name__ == "__main__":
    sys.exit(main())
