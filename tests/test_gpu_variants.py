"""Kernel variants, each in a fresh process (their switches are read once
per process): the entry-lane sweep on a node-blocked matrix (PCLAB_BSR=0)
and the cooperative Kahn levelling (PCLAB_LEVEL_QUEUE=0). Same parity bar
as the default path: PCG iterations +-1 and the solution within 1e-8 of the
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


@pytest.mark.parametrize("env", [{"PCLAB_BSR": "0"}, {"PCLAB_LEVEL_QUEUE": "0"}])
def test_variant_parity(env):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=e, cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("ok")


IC0 = r"""
import hashlib, sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2412_07127_b200 as P
h = hashlib.sha256()
for w in (P.workloads.by_name("elasticity_q1_40").scaled(9), P.workloads.CONFIGS[0].scaled(12),
          P.workloads.CONFIGS[4].scaled(14)):
    a, b, model = P.workloads.build(w)
    h.update(P.Precond(a, "ic0").factor().tobytes())
print(h.hexdigest())
"""


def test_ic0_mask_kernel_bit_identical_to_merge_walk():
    """The mask-driven IC(0) (symbolic masks from the block-column view or
    from scalar rows (PCLAB_IC0_BSR_MASKS=0) + the block / row mask kernels)
    and the merge-walk kernel (PCLAB_IC0_MASKS=0) produce the same factor
    bits."""
    outs = []
    for env in ({"PCLAB_IC0_MASKS": "0"}, {}, {"PCLAB_IC0_BSR_MASKS": "0"}):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, "-c", IC0.format(root=ROOT)], env=e, cwd=ROOT,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        outs.append(out.stdout.strip())
    assert len(set(outs)) == 1, outs


SWEEP_BITS = r"""
import hashlib, sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2412_07127_b200 as P
h = hashlib.sha256()
w = P.workloads.by_name("elasticity_q1_40").scaled(12)
a, b, model = P.workloads.build(w)
for kind in ("ic0", "gnnic"):
    pc = P.Precond(a, kind, model if kind == "gnnic" else None)
    r = torch.from_numpy(np.random.default_rng(2).standard_normal(a.n)).cuda()
    y = torch.empty_like(r)
    for upper in (False, True):
        pc.trsv_device(upper, r.data_ptr(), y.data_ptr())
        h.update(y.cpu().numpy().tobytes())
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=300)
    h.update(xt.cpu().numpy().tobytes())
print(h.hexdigest())
"""


def test_item_stream_sweep_bit_identical_to_csr_sweep():
    """bss_trsv_kernel (factor values re-laid per schedule slot, bss.cu) and
    bsr_trsv_kernel (values read from the L / U CSR, PCLAB_BSS=0) use the
    same lane mapping, FMA order, shuffle tree and diagonal solve: both
    sweeps and whole PCG solves are bit-identical."""
    outs = []
    for env in ({"PCLAB_BSS": "0"}, {}):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, "-c", SWEEP_BITS.format(root=ROOT)], env=e, cwd=ROOT,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        outs.append(out.stdout.strip())
    assert len(set(outs)) == 1, outs



REC_BITS = r"""
import hashlib, sys
import numpy as np
import torch
sys.path.insert(0, {root!r})
import paper_2412_07127_b200 as P
h = hashlib.sha256()
for m in (24, 33):
    w = P.workloads.by_name("diffusion_fv_256").scaled(m)
    a, b, model = P.workloads.build(w)
    for kind in ("ic0", "gnnic"):
        pc = P.Precond(a, kind, model if kind == "gnnic" else None)
        r = torch.from_numpy(np.random.default_rng(2).standard_normal(a.n)).cuda()
        y = torch.empty_like(r)
        for upper in (False, True):
            pc.trsv_device(upper, r.data_ptr(), y.data_ptr())
            h.update(y.cpu().numpy().tobytes())
        bt = torch.from_numpy(b).cuda()
        xt = torch.zeros_like(bt)
        rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=300)
        h.update(xt.cpu().numpy().tobytes())
        h.update(str(rep["iterations"]).encode())
print(h.hexdigest())
"""


def test_record_sweep_bit_identical_to_item_stream_sweep():
    """rec_trsv_kernel (one fixed 128-byte record per slot, everything
    requested ahead; 7-point diffusion, blocks of 2 rows) against
    rrs_trsv_kernel (PCLAB_REC=0): same lane / entry mapping, FMA order,
    shuffle tree and diagonal solve -- sweeps and whole PCG solves are
    bit-identical (even and odd mesh sizes: the odd one has idle slots)."""
    outs = []
    for env in ({"PCLAB_REC": "0"}, {}):
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, "-c", REC_BITS.format(root=ROOT)], env=e, cwd=ROOT,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        outs.append(out.stdout.strip())
    assert len(set(outs)) == 1, outs


def test_branch_free_tanh_matches_library():
    """tanh_nb (csrc/gnn_math.cuh, the GNN kernels' tanh) against the CUDA
    library's on 2^24 points of [-24, 24], 2^20 tiny arguments and the
    special values: absolute difference below 1e-14 (tools/tanh_check.cu,
    compiled by __graft_entry__.build())."""
    exe = os.path.join(ROOT, "build", "tanh_check")
    if not os.path.exists(exe):  # normally built by __graft_entry__.build()
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe,
                        os.path.join(ROOT, "tools", "tanh_check.cu")], check=True, timeout=300)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
