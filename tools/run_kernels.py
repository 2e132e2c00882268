"""Developer driver for ncu: build one workload and launch the PCG-loop
kernels a few times (spmv, both sweeps, one short PCG)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_40"
m = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "0" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
kind = sys.argv[4] if len(sys.argv) > 4 else "ic0"
w = P.workloads.by_name(name)
if m:
    w = w.scaled(m)
a, b, model = P.workloads.build(w)
pc = P.Precond(a, kind, model if kind in ("nic", "gnnic") else None)
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    a.spmv_device(x.data_ptr(), y.data_ptr())
    pc.trsv_device(False, x.data_ptr(), y.data_ptr())
    pc.trsv_device(True, x.data_ptr(), y.data_ptr())
bt = torch.from_numpy(b).cuda()
xt = torch.zeros_like(bt)
try:
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=8)
except P.NumericError as e:  # gnnic on elasticity: the reference's own breakdown
    rep = {"iterations": str(e)}
torch.cuda.synchronize()
print("ok", a.n, a.nnz, rep["iterations"])
