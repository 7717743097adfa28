"""Where the time to 1e-6 goes (bench.py time_to_solution): one mixed iterative refinement
(bicgstab_refine) on config 3 per schedule, timed by the host clock around the call, and its
kernels summed by name from a torch.profiler (CUPTI) trace of a second call.
Run on the GPU box: python tools/tts_breakdown.py > gpurun_out/tts_breakdown.log"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import inputs
    import inputs.cuda as icuda
    import paper_2010_03660_b200 as sten

    NX, NY, NZ = 600, 595, 1536
    torch.cuda.set_device(0)
    diag, offs = icuda.fields_device(inputs.KIND_CD, NX, NY, NZ, z0=0, seed=1, delta=0.1)
    st = sten.stencil_create(NX, NY, NZ, [diag] + offs)
    del diag, offs
    b32 = icuda.uniform_device(NX, NY, NZ, z0=0, seed=1, stream=0).to(torch.float16).float()
    x32 = torch.empty_like(b32)
    inner_tol = float(os.environ.get("TTS_INNER_TOL", "1e-2"))
    for name, sch in (("classic", sten.SCHED_CLASSIC), ("sr", sten.SCHED_SR)):
        sten.set_schedule(st, sch)
        sten.bicgstab_refine(st, b32, None, 1e-6, 30, inner_tol, 200, x32)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ko, ki, rh, status = sten.bicgstab_refine(st, b32, None, 1e-6, 30, inner_tol, 200, x32)
        ms = (time.perf_counter() - t0) * 1e3
        print(f"[{name}] refine {ms:.2f} ms outer {ko} inner {ki} true res {rh[-1]:.3e} status {status}")
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            sten.bicgstab_refine(st, b32, None, 1e-6, 30, inner_tol, 200, x32)
            torch.cuda.synchronize()
        tot = {}
        for e in prof.events():
            if e.device_type == torch.autograd.DeviceType.CUDA:
                k = e.name.split("(")[0][:60]
                c, t = tot.get(k, (0, 0.0))
                tot[k] = (c + 1, t + e.time_range.elapsed_us() / 1e3)
        s = 0.0
        for k, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
            s += t
            print(f"   {t:9.3f} ms {c:5d}x  {k}")
        print(f"   {s:9.3f} ms total device")


if __name__ == "__main__":
    main()
