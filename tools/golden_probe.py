"""Developer probe: device results against the committed full-size reference
goldens (tests/golden/fullsize_<cfg>.npz)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2412_07127_b200 as P  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                         f"fullsize_{which}.npz"))
w = P.workloads.CONFIGS[2 if which == "cfg2" else 4]
a, b, model = P.workloads.build(w)
print(which, "n", a.n, "golden n", g["n"], flush=True)
lidx = g["lidx"]
for kind in ("ic0", "gnnic"):
    if f"{kind}.vals" not in g:
        continue
    f = P.Precond(a, kind, model if kind == "gnnic" else None).factor()
    ref = g[f"{kind}.vals"]
    rel = np.abs(f[lidx] - ref) / np.maximum(np.abs(ref), 1e-300)
    print(kind, "factor max rel", rel.max(), "bit-equal frac", np.mean(f[lidx] == ref), flush=True)
for kind in ("ic0", "gnnic"):
    tag = f"pcg.{kind}"
    if f"{tag}.error" in g:
        try:
            x, rep = P.pcg_solve(a, b, kind, model if kind == "gnnic" else None, rel_tol=w.rel_tol,
                                 max_iters=w.max_iters)
            print(tag, "device converged?", rep["converged"], rep["iterations"], "ref error:", g[f"{tag}.error"][0])
        except P.PclabError as e:
            print(tag, "device error:", e, "| ref error:", g[f"{tag}.error"][0], flush=True)
        continue
    if f"{tag}.iters" not in g:
        continue
    import torch
    pc = P.Precond(a, kind, model if kind == "gnnic" else None)
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=w.rel_tol, max_iters=w.max_iters,
                          record_history=True)
    x = xt.cpu().numpy()
    hd = np.array(rep["residual_history"])
    hr = g[f"{tag}.hist"]
    m = min(len(hd), len(hr))
    rel = np.abs(hd[:m] - hr[:m]) / hr[:m]
    for k in (1, 10, 50, 100, 200, 400, 600, 800, 1000, 1200, m - 1):
        if k < m:
            print(f"  hist[{k}] dev {hd[k]:.6e} ref {hr[k]:.6e} rel diff {rel[k]:.2e}")
    print("  first iteration with rel diff > 1e-10:", int(np.argmax(rel > 1e-10)) if (rel > 1e-10).any() else None,
          " > 1e-6:", int(np.argmax(rel > 1e-6)) if (rel > 1e-6).any() else None)
    xi, xr = g[f"{tag}.xidx"], g[f"{tag}.x"]
    print(tag, "iters dev", rep["iterations"], "ref", g[f"{tag}.iters"],
          "x sample rel err", np.linalg.norm(x[xi] - xr) / np.linalg.norm(xr),
          "xnorm dev", np.linalg.norm(x), "ref", g[f"{tag}.xnorm"][0],
          "true res dev", rep["true_rel_residual"], "ref", g[f"{tag}.resid"], flush=True)
