import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, inputs
import paper_2010_03660_b200 as sten
nx,ny,nz=64,48,40
d,o = inputs.problem_fields(1,nx,ny,nz)
st = sten.stencil_create(nx,ny,nz,[torch.from_numpy(d).cuda()]+[torch.from_numpy(a).cuda() for a in o])
b = torch.rand(nz,ny,nx,device='cuda').half(); x = torch.empty_like(b)
print(sten.bicgstab_solve(st,1,b,None,0.0,10,x)[0])
sten.set_timing(st, True)
try:
    print(sten.bicgstab_solve(st,1,b,None,0.0,10,x)[0], sten.get_stats(st))
except Exception as e: print('ERR', e)
