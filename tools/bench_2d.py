"""Measure the 2D 9-point path (NEXT-3) at the paper's 2D geometry, 22800 x 22800,
against the HBM roofline, on the seeded 2D stand-in (inputs.fields2d_device, R25):

  * stencil2d_apply, gather (10 arrays per point: 8 couplings, v, u) and the paper's tiled
    output-halo form (R24) at two tilings: 8 x 1 tiles (a multi-GPU-sized
    decomposition) and 600 x 600 tiles of 38 x 38 points (the paper's per-core sub-block,
    PAPER.md:371: "a sub-block up-to 38x38 in size, corresponding to geometries of 22800x22800");
  * bicgstab2d_solve (R25), mixed fp16 and fp32, 100 iterations at tol = 0, per-phase
    device times by CUDA events (stencil2d_set_timing), 33 passes per iteration (H1 14, H2 12, H3 7),
    and the mixed solve to tol 1e-3.

Kernel / phase times by CUDA events on the launching stream, median of repeats after warm-up;
every array is > L2 (1.04 GB per fp16 vector), so no flush is needed.  Writes
gpurun_out/<tag>_2d.md and .json (copied to profiles/)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

PASSES = {"H1": 14, "H2": 12, "H3": 7}


def tmo(ms):
    return round(float(ms), 4)


def main(tag="r2", n=22800, maxit=100):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    diag, offs = icuda.fields2d_device(n, n, seed=1, delta=0.1)
    st = sten.stencil2d_create(n, n, [diag] + offs)
    del offs
    torch.cuda.empty_cache()
    npts = n * n
    rec = {"mesh": [n, n], "points": npts, "peak_gbs": peak, "apply": [], "solve": []}
    lines = [f"# {tag}: 2D 9-point path at {n}x{n} (PAPER.md:362-373, 371), `python tools/bench_2d.py {tag}`\n",
             "Seeded 2D stand-in (inputs.fields2d_device, delta = 0.1, R25); b ~ U(-1,1) (stream 0); "
             f"roofline = measured copy peak {peak:.0f} GB/s (MEASURED_PEAKS.json).\n",
             "## SpMV (stencil2d_apply): 10 arrays per point\n",
             "| precision | form | tiles | ms (median of 10) | algorithmic GB/s | fraction of peak | Gpoint/s |",
             "|---|---|---|---|---|---|---|"]
    g = torch.Generator(device="cuda").manual_seed(1)
    for prec, dt, es in ((sten.MIXED, torch.float16, 2), (sten.FP32, torch.float32, 4)):
        x = (torch.rand((n, n), device="cuda", generator=g, dtype=torch.float32) * 2 - 1).to(dt)
        y = torch.empty_like(x)
        for tiles in ((1, 1), (1, 8), (600, 600)):
            sten.stencil2d_set_tiles(st, *tiles)
            for _ in range(3):
                sten.stencil2d_apply(st, prec, x, y)
            ms = statistics.median(sten.stencil2d_apply(st, prec, x, y) for _ in range(10))
            gbs = 10 * es * npts / (ms * 1e-3) / 1e9
            form = "gather" if tiles == (1, 1) else "tiled output halo"
            lines.append(f"| {'mixed fp16' if es == 2 else 'fp32'} | {form} | {tiles[0]}x{tiles[1]} | {ms:.3f} | "
                         f"{gbs:.0f} | {gbs / peak:.3f} | {npts / (ms * 1e-3) / 1e9:.1f} |")
            rec["apply"].append({"precision": "mixed" if es == 2 else "fp32", "tiles": list(tiles), "ms": ms,
                                 "gbs": gbs, "frac": gbs / peak})
        sten.stencil2d_set_tiles(st, 1, 1)
        del x, y
        torch.cuda.empty_cache()
    lines += ["", f"## BiCGStab (bicgstab2d_solve), {maxit} iterations at tol = 0: 33 passes per iteration\n",
              "| precision | ms / iteration | Gpoint-iter/s | whole-iteration GB/s (33 passes) | fraction | "
              "H1 ms (GB/s, frac) | H2 ms (GB/s, frac) | H3 ms (GB/s, frac) | status, event iter |",
              "|---|---|---|---|---|---|---|---|---|"]
    b64 = icuda.uniform_device(n, n, 1, seed=1, stream=0).view(n, n)  # = inputs.rhs_uniform_2d (R16)
    for prec, dt, es in ((sten.MIXED, torch.float16, 2), (sten.FP32, torch.float32, 4)):
        b = b64.to(dt)
        x = torch.empty_like(b)
        sten.stencil2d_set_timing(st, True)
        sten.bicgstab2d_solve(st, prec, b, None, 0.0, 4, x)  # warm-up (graph capture of its chunk)
        runs = []
        for _ in range(3):
            it, hist, status = sten.bicgstab2d_solve(st, prec, b, None, 0.0, maxit, x)
            ph, nit = sten.stencil2d_phase_ms(st)
            runs.append((sum(ph), ph, it, status, hist))
        runs.sort(key=lambda r: r[0])
        tot, ph, it, status, hist = runs[1]
        # the whole solve without the per-phase events (graph of maxit iterations, no polling)
        sten.stencil2d_set_timing(st, False)
        sten.bicgstab2d_solve(st, prec, b, None, 0.0, maxit, x)
        solve_ms = statistics.median([(sten.bicgstab2d_solve(st, prec, b, None, 0.0, maxit, x), st.last_solve_ms)[1]
                                      for _ in range(3)])
        per_it = solve_ms / maxit
        whole = 33 * es * npts / (per_it * 1e-3) / 1e9
        cells = []
        phrec = {}
        for k, name in enumerate(("H1", "H2", "H3")):
            gb = PASSES[name] * es * npts / (ph[k] * 1e-3) / 1e9
            cells.append(f"{ph[k]:.3f} ({gb:.0f}, {gb / peak:.3f})")
            phrec[name] = {"ms": ph[k], "gbs": gb, "frac": gb / peak, "passes": PASSES[name]}
        ev = next((i for i, h in enumerate(hist) if h == 0.0), None)
        lines.append(f"| {'mixed fp16' if es == 2 else 'fp32'} | {per_it:.3f} | {npts / (per_it * 1e-3) / 1e9:.1f} | "
                     f"{whole:.0f} | {whole / peak:.3f} | " + " | ".join(cells) +
                     f" | {status}, {ev if ev is not None else '-'} |")
        rec["solve"].append({"precision": "mixed" if es == 2 else "fp32", "maxit": maxit, "ms_per_iter": per_it,
                             "gpt_iter_s": npts / (per_it * 1e-3) / 1e9, "whole_gbs": whole, "whole_frac": whole / peak,
                             "phases": phrec, "status": status, "hist_last": float(hist[-1])})
        for tiles in ((1, 8), (600, 600)):  # BiCGStab on the paper's tiled output-halo SpMV (unfused)
            sten.stencil2d_set_tiles(st, *tiles)
            sten.bicgstab2d_solve(st, prec, b, None, 0.0, 4, x)
            runs = []
            for _ in range(3):
                sten.bicgstab2d_solve(st, prec, b, None, 0.0, 20, x)
                runs.append(st.last_solve_ms / 20)
            tms = sorted(runs)[1]
            rec.setdefault("tiled_solve", []).append({"precision": "mixed" if es == 2 else "fp32",
                                                      "tiles": list(tiles), "ms_per_iter": tmo(tms)})
            sten.stencil2d_set_tiles(st, 1, 1)
        if prec == sten.MIXED:
            it2, hist2, st2 = sten.bicgstab2d_solve(st, prec, b, None, 1e-3, 200, x)
            rec["mixed_tol_1e-3"] = {"iters": it2, "status": st2, "hist_last": float(hist2[-1]),
                                     "ms": st.last_solve_ms}
        del b, x
        torch.cuda.empty_cache()
    st.close()
    if rec.get("tiled_solve"):
        lines += ["", "## BiCGStab on the tiled output-halo SpMV (unfused phases; 20 iterations, tol = 0)\n",
                  "| precision | tiles | ms / iteration | vs the fused gather solve |", "|---|---|---|---|"]
        fused = {r["precision"]: r["ms_per_iter"] for r in rec["solve"]}
        for r in rec["tiled_solve"]:
            lines.append(f"| {r['precision']} | {r['tiles'][0]}x{r['tiles'][1]} | {r['ms_per_iter']:.3f} | "
                         f"{r['ms_per_iter'] / fused[r['precision']]:.2f}x |")
    t = rec.get("mixed_tol_1e-3")
    if t:
        lines.append(f"\nMixed solve to tol 1e-3: {t['iters']} iterations, status {t['status']}, final recurrence "
                     f"residual {t['hist_last']:.3e}, {t['ms']:.2f} ms.")
    lines.append("\nSpMV: one CTA per 256-B x 32-row tile, v through a TMA box with a one-point halo, the eight "
                 "couplings as streaming 16-B loads; the tiled form adds the output-halo ring (k_ring9) and the "
                 "x and y rounds (k_round9).  Solve: persistent k_bicg9<H1>, k_bicg9<H2> (one CTA per SM walking the tiles, TMA boxes of r, p, v / "
                 "r, v' into a 2-stage ring, the SpMV input formed once per box element in shared memory) and "
                 "k_h3_bulk; on tiles: k_upd9, the tiled SpMV, k_dot9 per phase.")
    out = "\n".join(lines) + "\n"
    print(out)
    outdir = os.path.join(ROOT, "gpurun_out")  # brought back by gpurun; copied into profiles/ by hand
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"{tag}_2d.md"), "w") as f:
        f.write(out)
    with open(os.path.join(outdir, f"{tag}_2d.json"), "w") as f:
        json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r2")
