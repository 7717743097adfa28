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
    p.add_argument("--schedule", default="classic", choices=["sr", "classic"],
                   help="headline schedule. classic: Alg. 1 as printed (29 passes); sr: single-reduction sweep "
                        "(19 passes, DESIGN.md R19, NEXT-1). The other one is measured in the same run and "
                        "reported as a labelled field unless --no-other")
    p.add_argument("--no-other", action="store_true", help="do not measure the non-headline schedule")
    p.add_argument("--dots", default="mixed", choices=["mixed", "half"],
                   help="mixed precision only: inner products as fp16 products summed in fp32 (the paper's "
                        "instruction), or half: fp16 column pencils (DESIGN.md R22, R28, NEXT-4)")
    p.add_argument("--operator", default="fields", choices=["fields", "poisson-const"],
                   help="fields: the workload's per-point coefficient fields; poisson-const: the constant "
                        "7-point Poisson operator (config 1's) at the same mesh via stencil_create_const "
                        "(no coefficient streams in the SR sweep, NEXT-4)")
    p.add_argument("--tiling", default="", help="bx,by,zc,stages override (classic)")
    p.add_argument("--sr-tiling", default="", help="by,stages,cstages,zc override (sr)")
    p.add_argument("--sr-chunks", default="", help="zc,tail_planes,zc_tail: SR chunk plan override (experiments)")
    p.add_argument("--cpu-planes", type=int, default=0, help="oracle sample planes (0 = auto)")
    p.add_argument("--set-option", action="append", default=[], metavar="NAME=V",
                   help="sten_set_option before the run, e.g. TMA_L2_PROMOTION=0 (experiments)")
    p.add_argument("--no-tts", action="store_true", help="skip the labelled time-to-solution field (1e-6: fp32 "
                   "BiCGStab vs mixed refinement)")
    p.add_argument("--no-2d", action="store_true", help="skip the labelled NEXT-3 field (2D 9-point BiCGStab at "
                                                         "the paper's 22800 x 22800, PAPER.md:371-373)")
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
def _slab_system(workload: str, planes: int, z0: int = 0):
    import inputs
    import oracle as orc
    kind = inputs.KIND_CD_WEAK if workload == "cfg5" else inputs.KIND_CD
    kz = inputs.weak_kz_table(NZ) if kind == inputs.KIND_CD_WEAK else None
    diag, offs = inputs.problem_fields(kind, NX, NY, planes, z0=z0, seed=1, delta=0.1, kz_table=kz)
    b64 = inputs.rhs_uniform(NX, NY, planes, z0=z0, seed=1)
    c64 = orc.jacobi_scale(diag, offs)
    return diag, c64, b64


def oracle_sample(precision: str, workload: str, planes: int, iters: int, z0: int = 0, threads: int = 0,
                  system=None):
    """Time the oracle as it stands on a z-slab sample [z0, z0+planes) of the workload:
    O16 (the fp16-emulating oracle of the mixed path) or O64 (fp64; for fp32 runs on the
    fp32-quantised couplings)."""
    import oracle as orc
    diag, c64, b64 = system or _slab_system(workload, planes, z0)
    if threads:
        orc.set_threads(threads)
    if precision == "mixed":
        c16 = orc.quantize_coeffs(c64, "mixed")
        bh = orc.scale_rhs(orc.f16_from_double(b64), diag, "mixed")
        t0 = time.perf_counter()
        orc.bicgstab16(c16, bh, tol=0.0, maxit=iters)
        name = "O16"
    else:
        if precision == "fp32":
            c64 = [c.astype(np.float32).astype(np.float64) for c in c64]
            bh = orc.scale_rhs(b64.astype(np.float32), diag, "fp32").astype(np.float64)
        else:  # "fp64": the method in the host's native precision
            bh = b64 / diag
        t0 = time.perf_counter()
        orc.bicgstab64(c64, bh, tol=0.0, maxit=iters)
        name = "O64"
    dt = time.perf_counter() - t0
    pts = NX * NY * planes
    return dict(value=pts * iters / dt / 1e9, unit="Gpoint-iter/s", cores=orc.num_threads(), kind="oracle",
                sample=f"{name} BiCGStab, {iters} iterations on a {NX}x{NY}x{planes} z-slab of {workload} "
                       f"({pts} points), {dt:.1f} s"), dt


def host_copy_gbs():
    """STREAM-like host copy (numpy, one thread, 1 GiB, read + write bytes)."""
    n = 1 << 27
    a = np.ones(n)
    b_ = np.empty_like(a)
    np.copyto(b_, a)
    best = 0.0
    for _ in range(3):
        t0 = time.perf_counter()
        np.copyto(b_, a)
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


def cpu_baseline_auto(precision, workload, planes_override=0):
    """SURVEY.md 8(d) CPU oracle timing on this host: O64 on all cores and on one thread
    (10 iterations, 600x595x192 slab of the workload), next to O16 (the fp16-emulating
    oracle, software binary16: 3 iterations on a 600x595x16 slab), with nproc and the host
    copy bandwidth.  `value` = O64 on all cores: the fastest the oracle runs here."""
    import oracle as orc
    nproc = os.cpu_count()
    planes = planes_override or 192
    system = _slab_system(workload, planes)
    o64p = "fp32" if precision == "fp32" else "fp64"
    allc, _ = oracle_sample(o64p, workload, planes, 10, threads=nproc, system=system)
    one, _ = oracle_sample(o64p, workload, planes, 10, threads=1, system=system)
    del system
    orc.set_threads(nproc)
    o16 = None
    if precision == "mixed":
        o16, _ = oracle_sample("mixed", workload, 16, 3, threads=nproc)
    res = dict(allc)
    res.update({"nproc": nproc, "cpu_model": cpu_model(), "host_copy_gbs": host_copy_gbs(),
                "o64_all_cores": allc, "o64_1_thread": one,
                "note": "O64 = fp64 oracle (the method in the host's native precision)" +
                        ("" if precision == "fp32" else "; O16 = fp16-emulating oracle of the mixed path")})
    if o16:
        res["o16_all_cores"] = o16
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
def event_split(iter_ms, event_iter, schedule):
    """Per-iteration device ms before / after the first breakdown event of a solve.
    Classic: entry j is iteration j + 1; SR: entry j is sweep j (it produces r_j).
    Iterations up to and including the event iteration count as pre-event."""
    if not iter_ms:
        return None
    first = 0 if schedule == "sr" else 1
    its = list(range(first, first + len(iter_ms)))
    if event_iter <= 0:
        pre, post = iter_ms, []
    else:
        pre = [m for it, m in zip(its, iter_ms) if it <= event_iter]
        post = [m for it, m in zip(its, iter_ms) if it > event_iter]
    mean = lambda v: float(np.mean(v)) if v else None  # noqa: E731
    return {"event_iter": int(event_iter), "n_pre": len(pre), "n_post": len(post),
            "ms_per_iter_pre": mean(pre), "ms_per_iter_post": mean(post), "ms_per_iter_all": mean(iter_ms)}


def run_schedule(sten, st, prec, schedule, b, x, args, world, sdist, npts, clocks_gpu=None):
    """W warm-up solves, then K timed solves of `schedule` on handle `st` (CUDA events on the
    solve's stream, max over ranks).  Returns the timing record."""
    import torch
    import torch.distributed as dist

    sten.set_schedule(st, sten.SCHED_SR if schedule == "sr" else sten.SCHED_CLASSIC)
    sten.set_timing(st, True)
    for _ in range(args.warmup):
        sten.bicgstab_solve(st, prec, b, None, args.tol, args.maxit, x)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(clocks_gpu) if clocks_gpu is not None else None
    launches, iters_done = 0, 0
    ph_ms, ph_n = [0.0, 0.0, 0.0], [0, 0, 0]
    per_iter, events = [], []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0.record(stream)
    last = None
    for _ in range(args.steps):
        last = sten.bicgstab_solve(st, prec, b, None, args.tol, args.maxit, x)
        iters_done += last[0]
        s = sten.get_stats(st)
        launches += s["kernel_launches"]
        for p in range(3):
            ph_ms[p] += s["phase_ms"][p]
            ph_n[p] += s["phase_launches"][p]
        per_iter.append([sten.iter_ms(st, p) for p in range(3)])
        events.append(s["event_iter"])
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    t_ms = sdist.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    it, hist, status = last
    # first-event split, per step, from the per-launch events inside the solve graphs
    splits = [event_split([a + b_ + c for a, b_, c in zip(*pi)], ev, schedule) for pi, ev in zip(per_iter, events)]
    splits = [sp for sp in splits if sp]
    value_window = npts * iters_done / (t_ms / 1e3) / 1e9
    value, basis = value_window, "all timed iterations"
    ev_rec = None
    if splits:
        pre = float(np.mean([sp["ms_per_iter_pre"] for sp in splits]))
        allm = float(np.mean([sp["ms_per_iter_all"] for sp in splits]))
        posts = [sp["ms_per_iter_post"] for sp in splits if sp["ms_per_iter_post"] is not None]
        post = float(np.mean(posts)) if posts else None
        ev_rec = {"event_iter": int(events[-1]), "event_iters_all_steps": sorted(set(int(e) for e in events)),
                  "iters_pre_event": splits[-1]["n_pre"], "iters_post_event": splits[-1]["n_post"],
                  "ms_per_iter_pre_event": pre, "ms_per_iter_post_event": post, "ms_per_iter_all": allm}
        if post is not None and post < 0.99 * pre:
            # post-event iterations ran > 1% faster: rate the whole window as if every iteration
            # took the pre-event time (init and graph gaps stay in)
            value = value_window * allm / pre
            basis = "pre-event iterations (post-event ran %.1f%% faster)" % (100 * (1 - post / pre))
        ev_rec["value_basis"] = basis
        ev_rec["value_all_iterations"] = value_window
    # dominant kernel's per-launch time: pre-event launches when the rule above applied
    dom = 0
    if ev_rec and basis.startswith("pre-event"):
        dom_ms = float(np.mean([np.mean([m for k, m in enumerate(pi[dom]) if (k + (0 if schedule == "sr" else 1)) <= ev])
                                for pi, ev in zip(per_iter, events)]))
    else:
        dom_ms = ph_ms[dom] / max(ph_n[dom], 1)
    return {"t_ms": t_ms, "iters_done": iters_done, "value": value, "value_window": value_window,
            "launches": launches, "ph_ms": ph_ms, "ph_n": ph_n, "dom_ms": dom_ms, "events": ev_rec,
            "status": sten.STATUS_NAMES.get(status, status), "final_rel_residual": float(hist[-1]),
            "hist_10": float(hist[min(10, len(hist) - 1)]), "clocks": clk}


def _tts_one(sten, st, b, b32, x32, tol):
    """The three timed solves of one schedule (the handle's current one)."""
    import torch
    out = {}
    # BASELINE config 3's "tol 1e-3 run": the mixed solve to the mixed-mode target
    xm = torch.empty_like(b)
    sten.bicgstab_solve(st, sten.MIXED, b, None, 1e-3, 100, xm)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, hist, status = sten.bicgstab_solve(st, sten.MIXED, b, None, 1e-3, 100, xm)
    ms = (time.perf_counter() - t0) * 1e3
    out["mixed_tol_1e-3"] = {"ms": ms, "iters": it, "rel_residual": float(hist[-1]), "status": int(status)}
    del xm
    sten.bicgstab_solve(st, sten.FP32, b32, None, tol, 500, x32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    it, hist, status = sten.bicgstab_solve(st, sten.FP32, b32, None, tol, 500, x32)
    ms = (time.perf_counter() - t0) * 1e3
    out["fp32_bicgstab"] = {"ms": ms, "iters": it, "rel_residual": float(hist[-1]), "status": int(status)}
    sten.bicgstab_refine(st, b32, None, tol, 30, 1e-2, 200, x32)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, tol, 30, 1e-2, 200, x32)
    ms = (time.perf_counter() - t0) * 1e3
    out["mixed_refinement"] = {"ms": ms, "outer_steps": ko, "fp16_iters": ki, "true_rel_residual_fp32": float(rh[-1]),
                               "status": int(status), "inner_tol": 1e-2}
    out["speedup_vs_fp32"] = out["fp32_bicgstab"]["ms"] / ms
    return out


def run_tts(sten, st, b, tol=1e-6):
    """Labelled field: the mixed solve to 1e-3 (BASELINE config 3's tol run), and the time to
    ||r||/||b|| <= tol on the bench's system (cfg 3, delta = 0.1) - fp32
    BiCGStab (Alg. 1) against the mixed iterative refinement (R21: fp32 residual and update, fp16
    inner solves of Alg. 1 to 1e-2; NEXT-2): the fp16 bandwidth carried to an
    fp32-accurate answer.  One warm-up call each (graph capture), then one timed call; the library
    synchronises its stream before returning, so the host clock around the call is the device time
    plus the call overhead.  The same three solves again on the single-reduction schedule (NEXT-1,
    R19: fp32 solve and the refinement's fp16 inner solves as SR sweeps) in the "sr" sub-field; the
    handle is left on the classic schedule."""
    import torch
    b32 = b.float()
    x32 = torch.empty_like(b32)
    out = {"tol": tol, "schedule": "classic", "clock": "host wall clock around the (synchronising) call"}
    sten.set_schedule(st, sten.SCHED_CLASSIC)
    out.update(_tts_one(sten, st, b, b32, x32, tol))
    sten.set_schedule(st, sten.SCHED_SR)
    out["sr"] = dict(schedule="sr", **_tts_one(sten, st, b, b32, x32, tol))
    out["sr"]["speedup_vs_classic_fp32"] = out["fp32_bicgstab"]["ms"] / out["sr"]["mixed_refinement"]["ms"]
    sten.set_schedule(st, sten.SCHED_CLASSIC)
    del b32, x32
    torch.cuda.empty_cache()
    return out


def run_2d(sten, icuda, peak, n=22800, maxit=100):
    """The labelled NEXT-3 field: BiCGStab on the 2D 9-point operator at the paper's 22800 x 22800
    (R25), mixed fp16, `maxit` iterations at tol = 0, on the seeded 2D
    stand-in; per-phase CUDA events, roofline on its 33 passes (H1 14, H2 12, H3 7)."""
    import torch
    diag, offs = icuda.fields2d_device(n, n, seed=1, delta=0.1)
    s2 = sten.stencil2d_create(n, n, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    b = icuda.uniform_device(n, n, 1, seed=1, stream=0).view(n, n).half()
    x = torch.empty_like(b)
    sten.stencil2d_set_timing(s2, True)
    sten.bicgstab2d_solve(s2, sten.MIXED, b, None, 0.0, 4, x)
    runs = []
    for _ in range(3):
        it, hist, status = sten.bicgstab2d_solve(s2, sten.MIXED, b, None, 0.0, maxit, x)
        ph, nit = sten.stencil2d_phase_ms(s2)
        runs.append((float(sum(ph)), [float(v) for v in ph]))
    sten.stencil2d_set_timing(s2, False)
    tot = []
    for _ in range(3):
        sten.bicgstab2d_solve(s2, sten.MIXED, b, None, 0.0, maxit, x)
        tot.append(s2.last_solve_ms / maxit)
    s2.close()
    del b, x
    torch.cuda.empty_cache()
    per_it = float(np.median(tot))
    ph = sorted(runs)[1][1]
    npts = n * n
    h1_gbs = 14 * 2 * npts / (ph[0] * 1e-3) / 1e9
    return {"label": "2D 9-point BiCGStab (SURVEY 8(f) NEXT-3, PAPER.md:362-373), mixed fp16, 22800 x 22800, "
                     f"{maxit} iterations at tol 0, seeded stand-in (DESIGN.md R25)",
            "value": npts / (per_it * 1e-3) / 1e9, "unit": "Gpoint-iter/s", "ms_per_iter": per_it,
            "whole_iteration_frac": 33 * 2 * npts / (per_it * 1e-3) / 1e9 / peak, "passes_per_iter": 33,
            "phase_ms_per_iter": ph,
            "roofline": {"bound": "hbm", "kernel": "k_bicg9<half,H1>", "achieved": h1_gbs, "peak": peak,
                         "unit": "GB/s", "frac": h1_gbs / peak, "passes": 14}}


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
    nz_global = args.nz if strong else args.nz * world
    z0, nzl = sdist.slab_of(rank, world, nz_global)

    comm = None
    if world > 1:
        comm = sdist.bootstrap_comm(sten, rank, world)

    # problem: fields of this rank's slab generated on the device (inputs/gen_cuda.cu)
    kind = inputs.KIND_CD_WEAK if workload == "cfg5" else inputs.KIND_CD
    kz = inputs.weak_kz_table(nz_global) if kind == inputs.KIND_CD_WEAK else None
    const_op = args.operator == "poisson-const"
    if const_op:
        st = sten.stencil_create_const(NX, NY, nz_global, (6.0, -1.0, -1.0, -1.0, -1.0, -1.0, -1.0), nslabs=1, comm=comm)
    else:
        diag, offs = icuda.fields_device(kind, NX, NY, nzl, z0=z0, seed=1, delta=0.1, kz_table=kz)
        st = sten.stencil_create(NX, NY, nz_global, [diag] + offs, nslabs=1, comm=comm)
        del diag, offs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if args.tiling:
        bx, by, zc, stg = (int(v) for v in args.tiling.split(","))
        sten.set_tiling(st, prec, bx, by, zc, stg)
    if args.sr_tiling:
        sten.set_sr_tiling(st, prec, *(int(v) for v in args.sr_tiling.split(",")))
    if args.sr_chunks:
        sten.set_sr_chunks(st, prec, *(int(v) for v in args.sr_chunks.split(",")))
    if args.dots == "half":
        sten.set_dot_precision(st, sten.DOTS_HALF)
    for kv in args.set_option:
        name, val = kv.split("=")
        sten.set_option(st, getattr(sten, "OPT_" + name), int(val))
    if world > 1 and os.environ.get("STEN_P2P", "0") == "1":
        # fused compute + collective over peer memory across ranks (opt-in): the SR sweep's and the
        # classic phase kernels' own halo stores and inbox deposits (STEN_OPT_CLASSIC_FUSED)
        sten.set_option(st, sten.OPT_CLASSIC_FUSED, 1)
        sten.p2p_setup(st, prec)
    b = icuda.uniform_device(NX, NY, nzl, z0=z0, seed=1, stream=0).to(tdt)
    x = torch.empty_like(b)
    npts_local = NX * NY * nzl
    npts = npts_local * n
    pname = "mixed" if prec == sten.MIXED else "fp32"
    peak, peak_kind = measured_peak()

    # the headline schedule first, then (unless --no-sr / it is the headline) the SR schedule
    head = args.schedule
    scheds = [head] + ([] if args.no_other else [s_ for s_ in ("classic", "sr") if s_ != head])
    recs = {}
    for sch in scheds:
        recs[sch] = run_schedule(sten, st, prec, sch, b, x, args, world, sdist, npts,
                                 clocks_gpu=local if sch == head else None)
    # a headline window that saw a hardware / thermal slowdown, or SM clocks stuck far below the
    # maximum with no reason, is measured once more (the second window is the one reported)
    clk = recs[head]["clocks"]
    bad = clk and (set(clk["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
                   or (not clk["reasons"] and clk["sm_mhz"] < 0.7 * clk["sm_max_mhz"]))
    # (every rank takes the same decision: the flag is all-reduced, MAX over ranks)
    if sdist.max_over_ranks(1.0 if bad else 0.0, device="cuda") > 0.0:
        first = clk
        recs[head] = run_schedule(sten, st, prec, head, b, x, args, world, sdist, npts, clocks_gpu=local)
        if recs[head]["clocks"] is not None:
            recs[head]["clocks"]["remeasured_after"] = first

    def roofline_of(sch, r):
        sr = sch == "sr"
        kb = (roofline.sweep_bytes(pname, npts_local, const_op) if sr
              else roofline.phase_bytes("H1", pname, npts_local, const_op))
        achieved = kb / (r["dom_ms"] / 1e3) / 1e9
        tname = "half" if prec == sten.MIXED else "float"
        kname = f"k_sr<{tname}>" if sr else f"k_stencil<{tname},H1>"
        traffic, traffic_src = (None, None)
        if nzl == NZ and not args.tiling and not args.sr_tiling and not args.sr_chunks and args.dots != "half":
            # the exact instance the run launches (fields / constant couplings), from the latest capture
            # (ncu prints the defaulted template arguments of k_stencil either elided or in full)
            tn = "__half" if prec == sten.MIXED else "float"
            if sr:
                kpre = ([f"k_sr<{tn}, 8, 3, 2, 1"] if const_op and prec == sten.MIXED else
                        [f"k_sr<{tn}, 16, 2, 2, 1"] if const_op else [f"k_sr<{tn}, 16, 2, 2, 0"])
            else:
                kpre = ([f"k_stencil<{tn}, 1, 16, 2, 2, 0, 0, 1>"] if const_op else
                        [f"k_stencil<{tn}, 1, 16, 2, 2, 0>", f"k_stencil<{tn}, 1, 16, 2, 2, 0, 0, 0>"])
            for kp in kpre:
                traffic, traffic_src = measured_traffic(kp)
                if traffic is not None:
                    break
        passes = roofline.passes_per_iter(sch, const_op)
        bpi = roofline.bytes_per_point_iter(pname, sch, const_op)
        # whole step against the schedule's algorithmic bytes (classic: SURVEY 8(d)'s 29 passes)
        whole_gbs = npts_local * r["iters_done"] * bpi / (r["t_ms"] / 1e3) / 1e9
        whole_gbs_v = r["value"] / n * bpi  # Gpt-iter/s per GPU x B/pt-iter = GB/s
        phase_n = max(r["ph_n"][0], 1)
        return {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": kb, "avg_launch_ms": r["dom_ms"],
                "passes_per_iter": passes, "bytes_per_point_iter": bpi,
                "whole_step_frac": whole_gbs / peak, "whole_step_frac_value_basis": whole_gbs_v / peak,
                "phase_ms_per_iter": [p / phase_n for p in r["ph_ms"]][:1 if sr else 3]}

    # end to end through the C ABI with pinned HOST buffers: one bicgstab_solve_batch call
    # solves the K steps' systems, every step's b uploaded and x downloaded (pipelined
    # with the neighbouring steps' solves on the library's copy stream)
    def e2e_of(sch):
        sten.set_schedule(st, sten.SCHED_SR if sch == "sr" else sten.SCHED_CLASSIC)
        bh = [b.cpu().pin_memory() for _ in range(2)]
        xh = [torch.empty_like(bh[0]).pin_memory() for _ in range(2)]
        sten.set_timing(st, False)
        sten.bicgstab_solve_batch(st, prec, bh, xh, args.tol, args.maxit)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = sten.bicgstab_solve_batch(st, prec, [bh[i % 2] for i in range(args.steps)],
                                        [xh[i % 2] for i in range(args.steps)], args.tol, args.maxit)
        torch.cuda.synchronize()
        te = sdist.max_over_ranks(time.perf_counter() - t0, device="cuda")
        e_iters = sum(r_[0] for r_ in res)
        esz = b.element_size()
        return {"value": npts * e_iters / te / 1e9, "unit": "Gpoint-iter/s",
                "h2d_bytes_per_step": npts_local * esz,
                "d2h_bytes_per_step": npts_local * esz + 8 * (e_iters // max(args.steps, 1) + 1),
                "schedule": sch,
                "api": "bicgstab_solve_batch (pinned host b in, x out every step; copies overlap the "
                       "neighbouring steps' solves)", "clock": "host wall clock around the call"}

    e2e = {} if args.no_e2e else {sch: e2e_of(sch) for sch in scheds}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    h = recs[head]
    pc, ps = roofline.passes_per_iter("classic", const_op), roofline.passes_per_iter("sr", const_op)
    cnote = " (constant couplings as scalars, NEXT-4)" if const_op else ""
    sched_names = {"classic": f"Alg. 1 as printed (PAPER.md:172-186): H1, H2, H3, 3 reductions, {pc} passes{cnote}",
                   "sr": f"single-reduction sweep (DESIGN.md R19, SURVEY 8(f) NEXT-1): {ps} passes, 1 reduction{cnote}"}
    line = {
        "metric": METRIC, "value": h["value"], "unit": "Gpoint-iter/s", "n_gpus": n, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["t_ms"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": h["value"] / PAPER_GPT_ITER_S,
        "dtype": "f16" if prec == sten.MIXED else "f32", "data": "synthetic",
        "config": {"workload": workload, "mesh": [NX, NY, nz_global], "mesh_per_gpu": [NX, NY, nzl],
                   "precision": pname, "schedule": head, "schedule_is": sched_names[head],
                   "operator": args.operator,
                   **({"dots": "half"} if args.dots == "half" and prec == sten.MIXED else {}),
                   **({"options": args.set_option} if args.set_option else {}),
                   **({"sr_chunks": args.sr_chunks} if args.sr_chunks else {}),
                   "maxit": args.maxit, "tol": args.tol,
                   "iters_per_solve": h["iters_done"] / args.steps,
                   "parallelism": f"zslab{n}",
                   "l2": "no flush: 16.5 GB working set per GPU >> 126 MB L2",
                   "gflops": h["value"] * roofline.FLOPS_PER_POINT_ITER,
                   "status": h["status"], "final_rel_residual": h["final_rel_residual"],
                   "rel_residual_iter10": h["hist_10"],
                   "events": h["events"],
                   "paper_cs1_gpt_iter_s_context": PAPER_GPT_ITER_S},
        "roofline": roofline_of(head, h),
        "gpu_launches": int(h["launches"]),
        "clocks": h["clocks"],
    }
    if head in e2e:
        line["e2e"] = e2e[head]
    for sch in scheds:
        if sch == head:
            continue
        r = recs[sch]
        line[sch] = {"label": sched_names[sch], "value": r["value"], "unit": "Gpoint-iter/s",
                     "ms_per_step": r["t_ms"] / args.steps, "iters_per_solve": r["iters_done"] / args.steps,
                     "gflops_alg1_equivalent": r["value"] * roofline.FLOPS_PER_POINT_ITER,
                     "gflops_note": "Alg. 1's 44 flop per point-iteration (PAPER.md:399-417) credited per "
                                    "iteration; the SR sweep itself performs more (three SpMVs, 12 dots)"
                                    if sch == "sr" else "44 flop per point-iteration (PAPER.md:399-417)",
                     "status": r["status"], "final_rel_residual": r["final_rel_residual"],
                     "rel_residual_iter10": r["hist_10"], "events": r["events"],
                     "roofline": roofline_of(sch, r), "gpu_launches": int(r["launches"]),
                     **({"e2e": e2e[sch]} if sch in e2e else {})}
    if not args.no_tts and world == 1 and prec == sten.MIXED and not const_op and workload == "cfg3":
        line["time_to_solution"] = run_tts(sten, st, b)
    if not args.no_2d and world == 1 and prec == sten.MIXED:
        del st, b, x
        torch.cuda.empty_cache()
        line["next3_2d"] = run_2d(sten, icuda, peak)
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
