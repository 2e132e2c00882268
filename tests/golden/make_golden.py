"""Regenerate tests/golden/reference_fixtures.npz from the REFERENCE itself.

Every array here is produced by the reference's own C++ code
(/root/reference/proj/src compiled unmodified into oracle/_ref by
oracle/Makefile), called through oracle/ref_shim.cpp. The Q1-elasticity
system is not a reference generator: its CSR comes from the C oracle and is
then pushed through the reference's ic0 / gnn_ic_predict / pcg, which pins
everything downstream of assembly.

Run in the build container (needs /root/reference):  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_fixtures.npz")


def put_csr(d, name, a):
    d[f"{name}.rp"] = a.rp
    d[f"{name}.cols"] = a.cols
    d[f"{name}.vals"] = a.vals


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref not built: make -C oracle")
    d = {}
    systems = {
        "p2_m8": O.ref_gen_poisson(2, 8, False, 0),
        "p2_m6_v19": O.ref_gen_poisson(2, 6, True, 19),
        "p3_m5_v5": O.ref_gen_poisson(3, 5, True, 5),
        "p3_m1": O.ref_gen_poisson(3, 1, False, 0),
    }
    systems["el_m3"] = O.gen_elasticity(3, O.lognormal_field(27, O.derive_seed(1, 0x4D4F44), 1.0))
    for name, a in systems.items():
        put_csr(d, name, a)
    params = O.ref_gnn_init(1)
    d["gnn_init_1"] = params
    d["gnn_init_0"] = O.ref_gnn_init(0)
    for name in ("p2_m6_v19", "p3_m5_v5", "el_m3"):
        a = systems[name]
        d[f"{name}.features"] = O.ref_node_features(a)
        out, sigma = O.ref_gnn_forward(a, params)
        d[f"{name}.gnn_out"] = out
        d[f"{name}.sigma"] = np.array([sigma])
        for kind in ("ic0", "gnnic", "nic"):
            try:
                d[f"{name}.{kind}"] = O.ref_factor(a, kind, params)[0]
            except O.OracleError as e:
                d[f"{name}.{kind}.error"] = np.array([str(e)])
        b = O.uniform_pm1_field(a.n, 7)
        d[f"{name}.b"] = b
        for kind in ("none", "jacobi", "ic0", "gnnic", "nic"):
            try:
                x, rep, hist = O.ref_pcg(a, b, kind, params, rel_tol=1e-8, max_iters=2000, history=True)
                d[f"{name}.pcg.{kind}.x"] = x
                d[f"{name}.pcg.{kind}.iters"] = np.array([rep["iterations"], rep["converged"]])
                d[f"{name}.pcg.{kind}.hist"] = hist
            except O.OracleError as e:
                d[f"{name}.pcg.{kind}.error"] = np.array([str(e)])
    # Kershaw's matrix: IC(0) breakdown after the shifts (test_precond.cpp)
    r = [0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3]
    c = [0, 1, 3, 0, 1, 2, 1, 2, 3, 0, 2, 3]
    v = [3, -2, 2, -2, 3, -2, -2, 3, -2, 2, -2, 3]
    rp = np.array([0, 3, 6, 9, 12], np.int64)
    kers = O.Csr(4, rp, np.array(c, np.int32), np.array(v, np.float64))
    try:
        O.ref_factor(kers, "ic0")
    except O.OracleError as e:
        d["kershaw.error"] = np.array([str(e)])
    np.savez_compressed(OUT, **d)
    print("wrote", OUT, len(d), "arrays")


if __name__ == "__main__":
    main()
