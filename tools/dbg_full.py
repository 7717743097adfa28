import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch, inputs, inputs.cuda as ic
import paper_2010_03660_b200 as sten
nx,ny,nz = 600,595,int(sys.argv[1]) if len(sys.argv)>1 else 1536
d,o = ic.fields_device(1,nx,ny,nz,seed=1,delta=0.1)
st = sten.stencil_create(nx,ny,nz,[d]+o); del d,o
b = ic.uniform_device(nx,ny,nz,seed=1).half(); x = torch.empty_like(b)
for prec in (1, 0):
    bb = b if prec == 1 else b.float(); xx = torch.empty_like(bb)
    it,h,stt = sten.bicgstab_solve(st,prec,bb,None,0.0,100,xx)
    a,w = sten.scalar_history(st,100)
    print('prec',prec,'status',stt,'event',sten.get_stats(st)['event_iter'])
    for i in range(0,101,4): print(i,'%.3e'%h[i], '' if i==0 else 'a=%.3e w=%.3e'%(a[i-1],w[i-1]))
