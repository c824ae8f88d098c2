mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_nqueens.py -q -m gpu > gpurun_out/pytest_nq.log 2>&1; echo rc=$? >> gpurun_out/pytest_nq.log
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import paper_2107_05681_b200 as d
d.init()
for base in (6,7,8):
  for m in (False, True):
    r={}
    for v in (0,1):
      ts=[]
      for i in range(5):
        s,_,st=d.nqueens(16,base,v,mirror=m); assert s==14772512
        if i>=1: ts.append(st['kernel_ms'])
      r[v]=min(ts)
    print('base',base,'mirror',m,'unmelded %.3f melded %.3f speedup %.3f'%(r[0],r[1],r[0]/r[1]),flush=True)
" > gpurun_out/time_nq2.log 2>&1
