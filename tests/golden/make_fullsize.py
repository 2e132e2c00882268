"""Full-size reference goldens for the BASELINE headline configs.

Runs the UNMODIFIED reference (oracle/_ref, built from /root/reference by
oracle/Makefile) on the full BASELINE systems and commits a compact record
of what it produced, so the GPU box (which has no reference) can check the
device at full size:

* configs[2] (Q1 elasticity 118^3, 5,012,994 dofs):
  - ic0 PCG to rtol 1e-8 (krylov.cpp:114-190 with precond.cpp:109-143):
    iteration count, converged flag, final / true relative residual, the
    whole residual history, ||x||_2, x at 4096 seeded indices, sha256 of x;
  - the IC(0) factor at 4096 seeded entries of L (reference);
  - the GNN-corrected factor (gnn_ic_predict, precond.cpp:155-168) at the
    same entries and the error PCG raises with it ("pcg: nonpositive
    curvature at iteration 1", krylov.cpp:151-154). These two come from the
    C oracle (oracle/pclab_oracle.c): the reference's own gnn_forward keeps
    every per-edge activation of the 202M-edge graph and was OOM-killed at
    54 GB in this 62 GB container; the oracle is pinned bit-for-bit to the
    reference's gnn_forward / gnn_ic_predict / pcg on the committed small
    fixtures (tests/test_oracle.py). Keys record which one produced what
    (`<tag>.source`).
* configs[3] (Q1 elasticity 149^3, 10,062,150 dofs, lognormal(0, 1.5)):
  IC(0) breaks down after the reference's three shifts, so ic0 and gnnic
  fail; the NIC factor (nic_predict, precond.cpp:145) at 4096 seeded
  entries and what PCG does with it, from the C oracle (the reference's
  gnn_forward does not fit the build container's memory at this size).
* configs[4] (7-point FV diffusion 256^3, 16,777,216 dofs): gnnic PCG to
  rtol 1e-8, max 5000 iterations: the same solve record, plus the GNN-
  corrected factor at 4096 seeded entries.

The systems themselves come from the C oracle (the reference has no Q1
generator; its gen_poisson with per-cell coefficients is the oracle's,
pinned bit-for-bit by tests/test_oracle.py), so everything downstream of
assembly is the reference's own arithmetic.

Usage (build container only, needs /root/reference and ~30 GB RAM; each
config takes 10-25 minutes on one core):
    python tests/golden/make_fullsize.py cfg2
    python tests/golden/make_fullsize.py cfg3
    python tests/golden/make_fullsize.py cfg4
Writes tests/golden/fullsize_<cfg>.npz.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2412_07127_b200.workloads import CONFIGS  # noqa: E402

NSAMPLE = 4096
SAMPLE_SEED = 20241209


def sample_idx(n: int, salt: int) -> np.ndarray:
    rng = np.random.default_rng(SAMPLE_SEED + salt)
    return np.sort(rng.choice(n, size=min(NSAMPLE, n), replace=False)).astype(np.int64)


def solve_record(d, tag, a, b, kind, params, max_iters, use_oracle=False):
    t0 = time.time()
    d[f"{tag}.source"] = np.array(["oracle" if use_oracle else "reference"])
    try:
        if use_oracle:
            x, rep, hist = O.pcg(a, b, kind, params, rel_tol=1e-8, max_iters=max_iters, history=True)
            rep = dict(rep, p_time=0.0, cg_time=0.0)
        else:
            x, rep, hist = O.ref_pcg(a, b, kind, params, rel_tol=1e-8, max_iters=max_iters, history=True)
    except O.OracleError as e:
        d[f"{tag}.error"] = np.array([str(e)])
        print(tag, "error:", e, f"({time.time() - t0:.0f} s)", flush=True)
        return
    xi = sample_idx(a.n, 1)
    d[f"{tag}.iters"] = np.array([rep["iterations"], rep["converged"]], np.int64)
    d[f"{tag}.resid"] = np.array([rep["final_rel_residual"], rep["true_rel_residual"]])
    d[f"{tag}.hist"] = hist
    d[f"{tag}.xnorm"] = np.array([np.linalg.norm(x)])
    d[f"{tag}.xidx"] = xi
    d[f"{tag}.x"] = x[xi]
    d[f"{tag}.xsha256"] = np.array([hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()])
    d[f"{tag}.times"] = np.array([rep["p_time"], rep["cg_time"]])
    print(tag, "iters", rep["iterations"], "conv", rep["converged"], "true", rep["true_rel_residual"],
          f"p {rep['p_time']:.1f} s cg {rep['cg_time']:.1f} s", flush=True)


def factor_record(d, tag, a, kind, params, lidx, use_oracle=False):
    t0 = time.time()
    d[f"{tag}.source"] = np.array(["oracle" if use_oracle else "reference"])
    try:
        if use_oracle:
            v, pt = O.factor(a, kind, params), 0.0
        else:
            v, pt = O.ref_factor(a, kind, params)
    except O.OracleError as e:
        d[f"{tag}.error"] = np.array([str(e)])
        print(tag, "error:", e, flush=True)
        return
    d[f"{tag}.vals"] = v[lidx]
    d[f"{tag}.p_time"] = np.array([pt])
    print(tag, f"factor {time.time() - t0:.1f} s (p_time {pt:.1f})", flush=True)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: make -C oracle")
    from paper_2412_07127_b200 import workloads as W

    cfg = {"cfg2": CONFIGS[2], "cfg3": CONFIGS[3], "cfg4": CONFIGS[4]}[which]
    t0 = time.time()
    a, b, params = W.build_oracle(cfg)
    print(which, "n", a.n, "nnz", a.nnz, f"built in {time.time() - t0:.0f} s", flush=True)
    d = {"n": np.array([a.n, a.nnz], np.int64)}
    nl = O.lib().or_lower_nnz(a.n, a.rp, a.cols)
    lidx = sample_idx(nl, 2)
    d["lidx"] = lidx
    d["nnz_lower"] = np.array([nl], np.int64)
    if which == "cfg2":
        factor_record(d, "gnnic", a, "gnnic", params, lidx, use_oracle=True)
        solve_record(d, "pcg.gnnic", a, b, "gnnic", params, -1, use_oracle=True)
        factor_record(d, "ic0", a, "ic0", None, lidx)
        solve_record(d, "pcg.ic0", a, b, "ic0", None, -1)
    elif which == "cfg3":
        factor_record(d, "ic0", a, "ic0", None, lidx, use_oracle=True)
        factor_record(d, "nic", a, "nic", params, lidx, use_oracle=True)
        solve_record(d, "pcg.nic", a, b, "nic", params, 20, use_oracle=True)
    else:
        factor_record(d, "gnnic", a, "gnnic", params, lidx)
        solve_record(d, "pcg.gnnic", a, b, "gnnic", params, cfg.max_iters)
    out = os.path.join(HERE, f"fullsize_{which}.npz")
    np.savez_compressed(out, **d)
    print("wrote", out, f"total {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
