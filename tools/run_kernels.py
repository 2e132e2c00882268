"""Developer driver for ncu: build one workload and launch the PCG-loop
kernels a few times (stand-alone SpMV and both sweeps, then a short IC(0)
PCG whose loop runs the padded sweeps and the product); with kind 'gnnic'
also build the GNN-corrected preconditioner once (the GNN kernels)."""
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
pc = P.Precond(a, "ic0")
if kind in ("nic", "gnnic"):
    P.Precond(a, kind, model)
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(reps):
    a.spmv_device(x.data_ptr(), y.data_ptr())
    pc.trsv_device(False, x.data_ptr(), y.data_ptr())
    pc.trsv_device(True, x.data_ptr(), y.data_ptr())
bt = torch.from_numpy(b).cuda()
xt = torch.zeros_like(bt)
rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=8)
torch.cuda.synchronize()
print("ok", a.n, a.nnz, rep["iterations"])
