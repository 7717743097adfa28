import sys, os, statistics
sys.path.insert(0, '/root/repo')
import torch
import paper_2010_03660_b200 as sten
tag = sys.argv[1]
if tag != 'base':
    sten.LIB_PATH = f'/root/repo/paper_2010_03660_b200/libsten_{tag}.so'
import inputs.cuda as icuda
n = 22800
diag, offs = icuda.fields2d_device(n, n, seed=1, delta=0.1)
st = sten.stencil2d_create(n, n, [diag] + offs)
del diag, offs
for dt, P in ((torch.float16, sten.MIXED), (torch.float32, sten.FP32)):
    x = (torch.rand((n, n), device='cuda') * 2 - 1).to(dt); y = torch.empty_like(x)
    for tiles in ((1, 1), (1, 8), (600, 600)):
        sten.stencil2d_set_tiles(st, *tiles)
        for _ in range(3): sten.stencil2d_apply(st, P, x, y)
        ms = statistics.median(sten.stencil2d_apply(st, P, x, y) for _ in range(10))
        print(tag, dt, tiles, round(ms, 3), flush=True)
