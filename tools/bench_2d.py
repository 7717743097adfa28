"""Measure the 2D 9-point SpMV (NEXT-3) at the paper's 2D geometry, 22800 x 22800
(PAPER.md:371), against the HBM roofline: 10 arrays per point (8 couplings, v, u).
Kernel time by CUDA events around the launch (stencil2d_last_ms), median of 20
after 3 warm-ups; inputs are device-resident and larger than L2.  Writes
profiles/<tag>_2d.md."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2010_03660_b200 as sten  # noqa: E402


def main(tag="r1", n=22800):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    g = torch.Generator(device="cuda").manual_seed(1)
    diag = torch.rand((n, n), device="cuda", generator=g, dtype=torch.float32) + 8.0
    offs = [-(torch.rand((n, n), device="cuda", generator=g, dtype=torch.float32)) for _ in range(8)]
    st = sten.stencil2d_create(n, n, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    lines = [f"# {tag}: 2D 9-point SpMV at {n}x{n} (PAPER.md:362-373, 371), `python tools/bench_2d.py`\n",
             "| precision | kernel ms (median of 20) | algorithmic GB/s (10 arrays/pt) | fraction of measured "
             f"{peak:.0f} GB/s | Gpoint/s |", "|---|---|---|---|---|"]
    for prec, dt, es in ((sten.MIXED, torch.float16, 2), (sten.FP32, torch.float32, 4)):
        x = (torch.rand((n, n), device="cuda", generator=g, dtype=torch.float32) * 2 - 1).to(dt)
        y = torch.empty_like(x)
        for _ in range(3):
            sten.stencil2d_apply(st, prec, x, y)
        ms = statistics.median(sten.stencil2d_apply(st, prec, x, y) for _ in range(20))
        gbs = 10 * es * n * n / (ms * 1e-3) / 1e9
        lines.append(f"| {'mixed fp16' if es == 2 else 'fp32'} | {ms:.3f} | {gbs:.0f} | {gbs / peak:.3f} | "
                     f"{n * n / (ms * 1e-3) / 1e9:.1f} |")
        del x, y
    st.close()
    lines.append("\nOne CTA per 256-B x 32-row tile, v through a TMA box with a one-point halo, the eight "
                 "couplings as streaming 16-B loads; no output halo (gather form, DESIGN.md).")
    out = "\n".join(lines) + "\n"
    print(out)
    with open(os.path.join(ROOT, "profiles", f"{tag}_2d.md"), "w") as f:
        f.write(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1")
