for l in 5 3 2; do
 echo LPR=$l; PCLAB_SPMV_LPR=$l python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2412_07127_b200 as P
w=P.workloads.CONFIGS[2]; a,b,m=P.workloads.build(w); pc=P.Precond(a,'ic0')
bt=torch.from_numpy(b).cuda(); xt=torch.zeros_like(bt)
print(pc.profile_device(bt.data_ptr(), xt.data_ptr(), 20))
x = torch.randn(a.n, dtype=torch.float64, device='cuda'); y=torch.empty_like(x)
a.spmv_device(x.data_ptr(), y.data_ptr()); torch.cuda.synchronize()
import time; t=time.perf_counter()
for _ in range(10): a.spmv_device(x.data_ptr(), y.data_ptr())
torch.cuda.synchronize(); print('plain spmv ms', (time.perf_counter()-t)/10*1e3)
"
done
