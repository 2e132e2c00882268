"""Developer probe: run each stage of the device path against the oracle on
small systems and print the discrepancies (used while bringing up kernels)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))) if len(b) else 0.0


def probe(w):
    t = time.time()
    a, b, model = P.workloads.build(w)
    oa, ob, op = P.workloads.build_oracle(w)
    rp, cols, vals = a.csr()
    print(f"[{w.name}] n={a.n} nnz={a.nnz} build {time.time()-t:.2f}s")
    print("  pattern eq", np.array_equal(rp, oa.rp) and np.array_equal(cols, oa.cols),
          "vals bitexact", np.array_equal(vals.view(np.int64), oa.vals.view(np.int64)),
          "rhs eq", np.array_equal(b, ob))
    ic = P.Precond(a, "ic0")
    info = ic.info()
    print("  info", info, ic.timings())
    lo, up, nlo, nup = ic.levels()
    L = O.lower(oa)
    U, _ = O.transpose(L)
    olo, onlo = O.levels_lower(L)
    oup, onup = O.levels_upper(U)
    print("  levels lower eq", np.array_equal(lo, olo), nlo, onlo, " upper eq", np.array_equal(up, oup), nup, onup)
    lic = ic.factor()
    olic, att = O.ic0(oa)
    print("  ic0 bitexact", np.array_equal(lic.view(np.int64), olic.view(np.int64)), "maxrel", rel(lic, olic))
    g = P.Precond(a, "gnnic", model)
    lg = g.factor()
    olg = O.factor(oa, "gnnic", op)
    print("  gnnic maxrel", rel(lg, olg), "sigma", g.info()["sigma"], g.timings())
    for kind in ["none", "jacobi", "ic0", "gnnic", "nic"]:
        try:
            t = time.time()
            x, rep = P.pcg_solve(a, b, kind, model, rel_tol=w.rel_tol, max_iters=2000)
            dt = time.time() - t
            xo, ro = O.pcg(oa, ob, kind, op, rel_tol=w.rel_tol, max_iters=2000)
            print(f"  {kind:7s} its {rep['iterations']} vs {ro['iterations']} conv {rep['converged']} "
                  f"xrel {np.linalg.norm(x-xo)/max(np.linalg.norm(xo),1e-300):.2e} "
                  f"true_rel {rep['true_rel_residual']:.2e} cg {rep['cg_time']*1e3:.2f}ms wall {dt*1e3:.1f}ms")
        except Exception as e:
            print("  ", kind, "ERR", type(e).__name__, e)


if __name__ == "__main__":
    W = P.workloads.Workload
    probe(W("poisson8", "poisson", 8, seed=0, gnn_seed=0, rhs="uniform"))
    probe(W("diff12", "diffusion", 12, seed=3, gnn_seed=0, variable=True, rhs="uniform"))
    probe(P.workloads.CONFIGS[0])
    probe(W("elast6", "elasticity", 6, seed=1, gnn_seed=1))
    probe(W("elast16", "elasticity", 16, seed=1, gnn_seed=1))
