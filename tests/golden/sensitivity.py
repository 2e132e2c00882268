"""How sensitive is the reference's own iteration count to rounding?

The C oracle restates the reference's pcg / tri_solve / csr_matvec / ic0
bit-for-bit (tests/test_oracle.py pins it). This script rebuilds the same
source two more ways and runs the full BASELINE solves with each build:
  * fma_contracted: gcc -ffp-contract=fast -march=native -- a*b+c fused
    into one rounding in the dots, axpys, products and substitutions (the
    arithmetic the device uses); same algorithm, same order;
  * dot_strided_1024: the three dot products per iteration summed in 1024
    interleaved partials, then the partials in order (a parallel
    reduction's association; every other operation as the reference).
The iteration counts show how far apart correct implementations of the
same algorithm land at these sizes.

Usage (build container, ~15-25 minutes per config on one core):
    python tests/golden/sensitivity.py cfg2     # ic0, configs[2]
    python tests/golden/sensitivity.py cfg4     # gnnic, configs[4]
Writes tests/golden/sensitivity_<cfg>.json.
"""
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def run(which: str, lib: str) -> dict:
    code = f"""
import json, sys, time
sys.path.insert(0, {ROOT!r})
import numpy as np
from oracle import oracle as O
from paper_2412_07127_b200 import workloads as W
w = W.CONFIGS[{2 if which == 'cfg2' else 4}]
a, b, params = W.build_oracle(w)
kind = {'"ic0"' if which == 'cfg2' else '"gnnic"'}
t = time.time()
x, rep, hist = O.pcg(a, b, kind, params, rel_tol=w.rel_tol, max_iters=w.max_iters, history=True)
print(json.dumps({{"iterations": int(rep["iterations"]), "converged": int(rep["converged"]),
                  "final_rel_residual": rep["final_rel_residual"], "true_rel_residual": rep["true_rel_residual"],
                  "xnorm": float(np.linalg.norm(x)), "seconds": time.time() - t,
                  "hist_tail": [float(v) for v in hist[-12:]]}}))
"""
    env = dict(os.environ, ORACLE_LIB=lib)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    src = os.path.join(ROOT, "oracle", "pclab_oracle.c")
    fma = f"/tmp/liboracle_fma_{which}.so"
    strided = f"/tmp/liboracle_dot1024_{which}.so"
    subprocess.run(["gcc", "-O2", "-ffp-contract=fast", "-march=native", "-fPIC", "-shared", "-o", fma, src, "-lm"],
                   check=True)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-DOR_DOT_STRIDED=1024", "-fPIC", "-shared", "-o", strided,
                    src, "-lm"], check=True)
    from concurrent.futures import ThreadPoolExecutor
    libs = {"reference_rounding": os.path.join(ROOT, "oracle", "liboracle.so"), "fma_contracted": fma,
            "dot_strided_1024": strided}
    with ThreadPoolExecutor(max_workers=int(os.environ.get("SENS_JOBS", "2"))) as ex:
        futs = {k: ex.submit(run, which, lib) for k, lib in libs.items()}
        runs = {k: f.result() for k, f in futs.items()}
    res = {"config": which, "kind": "ic0" if which == "cfg2" else "gnnic",
           "note": "same oracle source (bit-identical to the reference when built as oracle/Makefile does) "
                   "built three ways; see the module docstring", **runs}
    with open(os.path.join(HERE, f"sensitivity_{which}.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v["iterations"] for k, v in res.items() if isinstance(v, dict)}))


if __name__ == "__main__":
    main()
