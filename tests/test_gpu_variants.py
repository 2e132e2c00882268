"""Opt-in kernel variants, each in a fresh process (their switches are read
once per process): the backward sweep fused with the product
(PCLAB_FUSE=1), the chain-segment sweep (PCLAB_CHAIN=1) and the entry-lane
sweep on a node-blocked matrix (PCLAB_BSR=0). Same parity bar as the
default path: PCG iterations +-1 and the solution within 1e-8 of the
oracle, sweeps within 1e-12."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2412_07127_b200 as P
from oracle import oracle as O
w = P.workloads.by_name("elasticity_q1_40").scaled(10)
a, b, model = P.workloads.build(w)
oa, ob, op = P.workloads.build_oracle(w)
x, rep = P.pcg_solve(a, b, "ic0", rel_tol=1e-8, max_iters=2000)
xo, ro = O.pcg(oa, ob, "ic0", rel_tol=1e-8, max_iters=2000)
assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 1, (rep["iterations"], ro["iterations"])
assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
pc = P.Precond(a, "ic0")
L = O.lower(oa)
L.vals = O.ic0(oa)[0]
U, _ = O.transpose(L)
r = np.random.default_rng(1).standard_normal(a.n)
rt = torch.from_numpy(r).cuda()
yt = torch.empty_like(rt)
for upper, ref in ((False, O.trsv_lower(L, r)), (True, O.trsv_upper(U, r))):
    pc.trsv_device(upper, rt.data_ptr(), yt.data_ptr())
    assert np.linalg.norm(yt.cpu().numpy() - ref) <= 1e-12 * np.linalg.norm(ref)
print("ok", rep["iterations"], ro["iterations"])
"""


@pytest.mark.parametrize("env", [{"PCLAB_FUSE": "1"}, {"PCLAB_CHAIN": "1"}, {"PCLAB_BSR": "0"},
                                 {"PCLAB_CHAIN": "1", "PCLAB_CHAIN_K": "3"}])
def test_variant_parity(env):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=e, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok")
