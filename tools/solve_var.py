"""Developer probe: run-to-run spread of the PCG loop time on one workload."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
bt = torch.from_numpy(b).cuda()
for k in range(reps):
    pc = P.Precond(a, "ic0")
    xt = torch.zeros_like(bt)
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=w.rel_tol, max_iters=w.max_iters)
    print(f"run {k}: its {rep['iterations']} cg {rep['cg_time']*1e3:.1f} ms -> {rep['cg_time']/rep['iterations']*1e3:.3f} ms/it"
          f"  tri_solve {rep.get('tri_solve_time_per_iter', 0)*1e3:.3f} ms", flush=True)
prof = pc.profile_device(bt.data_ptr(), xt.data_ptr(), 40)
print(prof)
for k in range(reps):
    pc = P.Precond(a, "ic0")
    xt = torch.zeros_like(bt)
    prof = pc.profile_device(bt.data_ptr(), xt.data_ptr(), 60)
    tot = sum(v for kk, v in prof.items() if kk.endswith("_ms"))
    print(f"eager {k}: {tot:.3f} ms/it  L {prof['sweep_lower_ms']:.3f} U {prof['sweep_upper_ms']:.3f} spmv {prof['spmv_ms']:.3f}", flush=True)
