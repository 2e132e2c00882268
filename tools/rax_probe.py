"""Developer probe: one small elasticity solve (iterations, time), for A/B
of PCG-loop variants under a short timeout."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10
w = P.workloads.by_name("elasticity_q1_40").scaled(m)
a, b, model = P.workloads.build(w)
t = time.time()
x, rep = P.pcg_solve(a, b, "ic0", rel_tol=1e-8, max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 3000)
print("n", a.n, "iters", rep["iterations"], "conv", rep["converged"], "rel", rep["final_rel_residual"],
      "true", rep["true_rel_residual"], "s", round(time.time() - t, 3), flush=True)
