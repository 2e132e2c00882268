"""Developer check of the sweeps on a few systems: stand-alone sweeps against
the oracle, a short PCG, and a digest of the device results (compare the
digest across PCLAB_RANGE=0/1 runs: the range-pipelined sweep must be
bit-identical to the round-robin one)."""
import hashlib
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

W = P.workloads
cases = [W.by_name("elasticity_q1_40").scaled(m) for m in (3, 6, 11)] + \
        [W.CONFIGS[4].scaled(m) for m in (9, 24)] + [W.CONFIGS[0].scaled(10)]
h = hashlib.sha256()
for w in cases:
    a, b, model = W.build(w)
    oa, ob, op = W.build_oracle(w)
    pc = P.Precond(a, "ic0")
    L = O.lower(oa)
    L.vals = O.ic0(oa)[0]
    U, _ = O.transpose(L)
    r = np.random.default_rng(1).standard_normal(a.n)
    rt = torch.from_numpy(r).cuda()
    yt = torch.empty_like(rt)
    errs = []
    for upper, ref in ((False, O.trsv_lower(L, r)), (True, O.trsv_upper(U, r))):
        pc.trsv_device(upper, rt.data_ptr(), yt.data_ptr())
        y = yt.cpu().numpy()
        h.update(y.tobytes())
        errs.append(float(np.linalg.norm(y - ref) / np.linalg.norm(ref)))
    x, rep = P.pcg_solve(a, b, "ic0", rel_tol=1e-8, max_iters=3000)
    xo, ro = O.pcg(oa, ob, "ic0", rel_tol=1e-8, max_iters=3000)
    h.update(x.tobytes())
    print(f"{w.name} n={a.n} sweep err {errs[0]:.2e} {errs[1]:.2e} iters {rep['iterations']} vs {ro['iterations']}"
          f" x err {np.linalg.norm(x - xo) / np.linalg.norm(xo):.2e} layout {pc.layout()}", flush=True)
print("digest", h.hexdigest())

name = sys.argv[1] if len(sys.argv) > 1 else ""
if name:
    w = W.by_name(name)
    t0 = time.time()
    a, b, model = W.build(w)
    pc = P.Precond(a, "ic0")
    print("built", time.time() - t0, pc.info(), flush=True)
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    for _ in range(2):
        prof = pc.profile_device(bt.data_ptr(), xt.data_ptr(), 20)
    print("profile", prof, flush=True)
    xt.zero_()
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=w.rel_tol, max_iters=w.max_iters)
    print("solve", {k: rep[k] for k in ("iterations", "converged", "cg_time", "true_rel_residual")}, flush=True)
