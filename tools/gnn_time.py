"""Developer probe: wall time of the IC(0) and gnnic preconditioner builds
(the difference is the GNN forward pass) on one workload."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
P.Precond(a, "ic0")
P.Precond(a, "gnnic", model)
for kind in ("ic0", "gnnic", "ic0", "gnnic"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.Precond(a, kind, model if kind == "gnnic" else None)
    torch.cuda.synchronize()
    print(kind, f"{(time.perf_counter() - t0) * 1e3:.1f} ms", flush=True)
