"""Probe: SR sweep time on an arbitrary mesh and SR tiling (for ncu DRAM-traffic runs).

python tools/sr_wave_probe.py NX NY NZ [by,S,SC,zc,pack] -- runs a mixed SR solve of 6
iterations twice (graphs warm) and prints the device time per sweep.  Used to test
whether one wave of tiles per z chunk (tiles = SM count, all neighbours co-resident
and started together) removes the halo re-reads of the default launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import inputs.cuda as ic  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402


def main():
    nx, ny, nz = (int(v) for v in sys.argv[1:4])
    ic.build()
    diag, offs = ic.fields_device(inputs.KIND_CD, nx, ny, nz, seed=1, delta=0.1)
    st = sten.stencil_create(nx, ny, nz, [diag] + offs)
    del diag, offs
    torch.cuda.empty_cache()
    sten.set_schedule(st, sten.SCHED_SR)
    if len(sys.argv) > 4:
        sten.set_sr_tiling(st, sten.MIXED, *(int(v) for v in sys.argv[4].split(",")))
    b = ic.uniform_device(nx, ny, nz, seed=1, stream=0).half()
    x = torch.empty_like(b)
    its = 20
    for _ in range(2):
        sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, its, x)
    ms = sten.get_stats(st)["solve_ms"]
    per = ms / (its + 1)
    gpts = nx * ny * nz * its / (ms / 1e3) / 1e9
    print(f"mesh {nx}x{ny}x{nz} tiling {sys.argv[4] if len(sys.argv) > 4 else 'default'}: "
          f"{per:.4f} ms/sweep, {gpts:.1f} Gpoint-iter/s, {38 * nx * ny * nz / per / 1e6:.0f} GB/s algorithmic")
    st.close()


if __name__ == "__main__":
    main()
