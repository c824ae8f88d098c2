mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_srad.py -q -m gpu > gpurun_out/pytest_srad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_srad.log
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2107_05681_b200 as d
d.init()
n=16384
g=torch.Generator(device='cuda').manual_seed(5)
j0=torch.exp(torch.rand((n,n),generator=g,device='cuda'))
j=torch.empty_like(j0)
for fast in (False, True):
  r={}
  for v in (0,1):
    ts=[]
    for i in range(3):
      j.copy_(j0); st=d.srad(j,100,0.5,d.RODINIA_ROI,v,fast=fast)
      if i: ts.append(st['kernel_ms'])
    r[v]=min(ts)
  print('fast',fast,'unmelded %.1f ms melded %.1f ms speedup %.3f GB/s %.0f'%(r[0],r[1],r[0]/r[1], 8*n*n*100/(r[1]*1e-3)/1e9),flush=True)
" > gpurun_out/time_srad.log 2>&1
