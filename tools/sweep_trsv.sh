for mb in 4 5 6 8; do
 cp build/lib_mb$mb.so paper_2412_07127_b200/libpclab_b200.so
 echo MINB=$mb; python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2412_07127_b200 as P
w=P.workloads.CONFIGS[2]; a,b,m=P.workloads.build(w); pc=P.Precond(a,'ic0')
bt=torch.from_numpy(b).cuda(); xt=torch.zeros_like(bt)
print(pc.profile_device(bt.data_ptr(), xt.data_ptr(), 20))
"
done
