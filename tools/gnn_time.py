"""Developer probe: device time of the IC(0) and gnnic preconditioner
builds on one workload, with and without a fresh symbolic analysis, and
the per-phase split the library reports (Precond.timings())."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "elasticity_q1_118"
w = P.workloads.by_name(name)
a, b, model = P.workloads.build(w)
for drop in (False, True, False, True, True):
    for kind in ("ic0", "gnnic"):
        if drop:
            a.drop_analysis()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pc = P.Precond(a, kind, model if kind == "gnnic" else None)
        torch.cuda.synchronize()
        print(kind, "drop" if drop else "keep", f"{(time.perf_counter() - t0) * 1e3:.1f} ms", pc.timings(), flush=True)
        del pc
