#!/bin/bash
# tools/sweep.sh "<tilings...>" [extra bench args]: per-phase HBM rates for each tiling
for t in $1; do
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --tiling $t $2 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); n=600*595*d['config']['mesh_per_gpu'][2]; e=2 if d['dtype']=='f16' else 4
p=d['roofline']['phase_ms_per_iter']
print('$t', 'Gpt/s %.1f'%d['value'], 'TB/s H1 %.2f H2 %.2f H3 %.2f'%(12*e*n/p[0]/1e9, 10*e*n/p[1]/1e9, 7*e*n/p[2]/1e9), ['%.3f'%x for x in p], d['config']['status'])"
done
