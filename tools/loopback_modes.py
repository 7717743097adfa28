"""The classic and SR schedules on LOOPBACK z-slabs of config 3 (one GPU playing G ranks): device
ms per iteration for each exchange mode - the cost of the decomposition machinery itself (halo
copies or peer stores, per-slab reductions, the scalar step) against the undecomposed handle.
python tools/loopback_modes.py [maxit]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import inputs.cuda as icuda  # noqa: E402
import paper_2010_03660_b200 as sten  # noqa: E402

NX, NY, NZ = 600, 595, 1536
maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 40
diag, offs = icuda.fields_device(inputs.KIND_CD, NX, NY, NZ, seed=1, delta=0.1)
b = icuda.uniform_device(NX, NY, NZ, seed=1, stream=0).half()
x = torch.empty_like(b)
for nslabs in (1, 2, 4):
    st = sten.stencil_create(NX, NY, NZ, [diag] + offs, nslabs=nslabs)
    modes = [("classic", None)] if nslabs == 1 else [("classic serial", (0, 0)), ("classic overlap", (1, 0)),
                                                     ("classic fused", (0, 1))]
    modes += [("sr", "sr")] if nslabs == 1 else [("sr fused", "sr")]
    for name, m in modes:
        if m == "sr":
            sten.set_schedule(st, sten.SCHED_SR)
        else:
            sten.set_schedule(st, sten.SCHED_CLASSIC)
            if m:
                sten.set_option(st, sten.OPT_CLASSIC_OVERLAP, m[0])
                sten.set_option(st, sten.OPT_CLASSIC_FUSED, m[1])
        sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, maxit, x)
        ms = []
        for _ in range(3):
            sten.bicgstab_solve(st, sten.MIXED, b, None, 0.0, maxit, x)
            ms.append(sten.get_stats(st)["solve_ms"] / maxit)
        print(f"slabs {nslabs} {name:16s} {min(ms):.4f} ms/iteration  {NX * NY * NZ / (min(ms) * 1e-3) / 1e9:.1f} "
              f"Gpoint-iter/s", flush=True)
    st.close()
