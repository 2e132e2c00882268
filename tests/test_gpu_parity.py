"""Parity of the device path (through the C-ABI) with the CPU oracle and the
reference's own fixtures.

Bars (BASELINE north star): CSR assembly, level sets and IC(0) factor
bit-exact; GNN-corrected factor within 1e-5 relative per entry (observed
~1e-11: the network runs in fp64); PCG iteration count within +-1 and the
solution within 1e-8 relative of the oracle's for well-conditioned solves.
The nic preconditioner with random-init weights is exponentially
ill-conditioned (its iteration count is a rounding lottery in the reference
too); it is held to a 3% iteration band instead.
"""
import numpy as np
import pytest

import paper_2412_07127_b200 as P
from conftest import bits, csr_from
from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = P.workloads.Workload
SMALL = [
    W("poisson2d_8", "poisson", 8, seed=0, gnn_seed=0, dim=2, rhs="uniform"),
    W("poisson3d_var_9", "diffusion", 9, seed=5, gnn_seed=0, variable=True, rhs="uniform"),
    W("diffusion_pm3_10", "diffusion", 10, seed=4, gnn_seed=1, variable=True, log10_lo=-3, log10_hi=3,
      rhs="uniform"),
    W("elasticity_4", "elasticity", 4, seed=1, gnn_seed=1),
    W("elasticity_7_s15", "elasticity", 7, seed=3, gnn_seed=1, sigma=1.5),
    P.workloads.CONFIGS[0],
]
IDS = [w.name for w in SMALL]
_cache = {}


def built(w):
    if w.name not in _cache:
        a, b, model = P.workloads.build(w)
        oa, ob, op = P.workloads.build_oracle(w)
        _cache[w.name] = (a, b, model, oa, ob, op)
    return _cache[w.name]


def max_rel(x, ref):
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1e-300))) if len(ref) else 0.0


@pytest.mark.parametrize("w", SMALL, ids=IDS)
def test_assembly_bit_exact(w):
    a, b, model, oa, ob, op = built(w)
    rp, cols, vals = a.csr()
    assert np.array_equal(rp, oa.rp) and np.array_equal(cols, oa.cols)
    assert np.array_equal(bits(vals), bits(oa.vals))
    assert np.array_equal(bits(b), bits(ob))
    assert np.array_equal(bits(model.params()), bits(op))


@pytest.mark.parametrize("w", SMALL, ids=IDS)
def test_level_sets_exact(w):
    a, _, _, oa, _, _ = built(w)
    lo, up, nlo, nup = P.Precond(a, "ic0").levels()
    L = O.lower(oa)
    U, _ = O.transpose(L)
    olo, onlo = O.levels_lower(L)
    oup, onup = O.levels_upper(U)
    assert np.array_equal(lo, olo) and nlo == onlo
    assert np.array_equal(up, oup) and nup == onup


@pytest.mark.parametrize("w", SMALL, ids=IDS)
def test_block_levels_exact(w):
    a, _, _, oa, _, _ = built(w)
    info = P.Precond(a, "ic0").info()
    bs = info["block_size"]
    L = O.lower(oa)
    U, _ = O.transpose(L)
    assert info["block_levels_lower"] == O.block_levels_lower(L, bs)[1]
    assert info["block_levels_upper"] == O.block_levels_upper(U, bs)[1]
    if w.family == "elasticity":
        assert bs == 3


@pytest.mark.parametrize("w", SMALL, ids=IDS)
def test_ic0_bit_exact(w):
    a, _, _, oa, _, _ = built(w)
    assert np.array_equal(bits(P.Precond(a, "ic0").factor()), bits(O.ic0(oa)[0]))


@pytest.mark.parametrize("w", SMALL, ids=IDS)
def test_gnn_corrected_factor(w):
    a, _, model, oa, _, op = built(w)
    for kind in ("gnnic", "nic"):
        pc = P.Precond(a, kind, model)
        ref = O.factor(oa, kind, op)
        assert max_rel(pc.factor(), ref) < 1e-5, kind
    _, sigma = O.gnn_forward(oa, op)
    # sd of the lower values: a deterministic tree sum on the device vs the
    # reference's sequential sum -- equal up to reassociation
    assert abs(P.Precond(a, "gnnic", model).info()["sigma"] - sigma) <= 1e-11 * sigma


def chaotic(w, kind):
    """Solves whose iteration count is a rounding lottery in any arithmetic
    order: random-init GNN corrections on elasticity (exponentially
    ill-conditioned L) and unpreconditioned / diagonal CG on high-contrast
    elasticity. They are held to a band, not to +-1."""
    if w.family == "elasticity":
        return kind in ("none", "jacobi", "gnnic", "nic")
    if w.log10_hi - w.log10_lo > 2:  # 10^6 coefficient contrast
        return kind in ("none", "nic")
    return kind == "nic"


def attempt(f):
    """(result, None) or (None, error message) -- both sides raise the
    reference's messages (krylov.cpp:151-154 etc.)."""
    try:
        return f(), None
    except (P.PclabError, O.OracleError) as e:
        return None, str(e)


@pytest.mark.parametrize("w", SMALL, ids=IDS)
@pytest.mark.parametrize("kind", ["none", "jacobi", "ic0", "gnnic"])
def test_pcg_parity(w, kind):
    a, b, model, oa, ob, op = built(w)
    cap = 3000
    dev, dev_err = attempt(lambda: P.pcg_solve(a, b, kind, model, rel_tol=w.rel_tol, max_iters=cap))
    ora, ora_err = attempt(lambda: O.pcg(oa, ob, kind, op, rel_tol=w.rel_tol, max_iters=cap))
    # a failing solve fails the same way on both sides
    assert dev_err == ora_err
    if dev_err:
        return
    (x, rep), (xo, ro) = dev, ora
    assert rep["converged"] == bool(ro["converged"])
    if chaotic(w, kind):
        if ro["converged"]:
            assert abs(rep["iterations"] - ro["iterations"]) <= max(2, 0.1 * ro["iterations"])
            assert np.linalg.norm(x - xo) <= 1e-6 * np.linalg.norm(xo)
        else:
            # both stalled at the cap: the final residuals agree to a factor 10
            assert rep["iterations"] == ro["iterations"] == cap
            assert abs(np.log10(rep["final_rel_residual"]) - np.log10(ro["final_rel_residual"])) <= 1.0
        return
    assert abs(rep["iterations"] - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    assert rep["true_rel_residual"] <= 10 * w.rel_tol and not rep["residual_mismatch"]


@pytest.mark.parametrize("w", SMALL[:2], ids=IDS[:2])
def test_nic_band(w):
    a, b, model, oa, ob, op = built(w)
    x, rep = P.pcg_solve(a, b, "nic", model, rel_tol=w.rel_tol, max_iters=3000)
    xo, ro = O.pcg(oa, ob, "nic", op, rel_tol=w.rel_tol, max_iters=3000)
    assert rep["converged"] and ro["converged"]
    assert abs(rep["iterations"] - ro["iterations"]) <= max(1, 0.03 * ro["iterations"])


def test_residual_history_tracks_oracle():
    w = SMALL[4]
    a, b, model, oa, ob, op = built(w)
    pc = P.Precond(a, "ic0")
    import torch
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=500, record_history=True)
    _, ro, hist = O.pcg(oa, ob, "ic0", rel_tol=1e-8, max_iters=500, history=True)
    h = np.array(rep["residual_history"])
    k = min(len(h), len(hist))
    assert abs(len(h) - len(hist)) <= 1
    assert max_rel(h[:10], hist[:10]) < 1e-10  # early iterates agree to rounding
    assert max_rel(h[:k], hist[:k]) < 1e-3  # and drift only slowly afterwards


@pytest.mark.parametrize("name", ["p2_m6_v19", "p3_m5_v5", "el_m3"])
def test_reference_fixtures_on_device(golden, name):
    g = csr_from(golden, name)
    a = P.Matrix.from_csr(g.rp, g.cols, g.vals)
    model = P.Model.from_params(golden["gnn_init_1"])
    assert np.array_equal(bits(P.Precond(a, "ic0").factor()), bits(golden[f"{name}.ic0"]))
    assert max_rel(P.Precond(a, "gnnic", model).factor(), golden[f"{name}.gnnic"]) < 1e-5
    b = golden[f"{name}.b"]
    for kind in ("none", "jacobi", "ic0", "gnnic"):
        x, rep = P.pcg_solve(a, b, kind, model, rel_tol=1e-8, max_iters=2000)
        it, conv = golden[f"{name}.pcg.{kind}.iters"]
        if name.startswith("el_") and kind == "gnnic":
            # more iterations than unknowns: a rounding lottery (see chaotic())
            assert rep["converged"] == bool(conv) and abs(rep["iterations"] - it) <= max(2, 0.1 * it), kind
            continue
        assert abs(rep["iterations"] - it) <= 1 and rep["converged"] == bool(conv), kind
        xr = golden[f"{name}.pcg.{kind}.x"]
        assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr), kind


def test_acceptance_c5_on_device():
    """Reference test_output.txt: none 432, diagonal 231, no-fill factor 70."""
    ms = P.derive_seed(2026, 5)
    a = P.Matrix.gen_poisson(2, 64, True, ms)
    b = P.field_uniform_pm1(a.n, P.derive_seed(ms, 14))
    its = [P.pcg_solve(a, b, k)[1]["iterations"] for k in ("none", "jacobi", "ic0")]
    # preconditioned counts are exact; plain CG at 432 iterations is within
    # the reduction-order band (device tree sums vs the reference's sequential)
    assert its[1:] == [231, 70] and abs(its[0] - 432) <= 3


def test_spmv_and_sweeps_match_oracle():
    import torch
    w = SMALL[3]
    a, _, _, oa, _, _ = built(w)
    x = np.random.default_rng(0).standard_normal(a.n)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty_like(xt)
    a.spmv_device(xt.data_ptr(), yt.data_ptr())
    y_ref = O.matvec(oa, x)
    assert np.linalg.norm(yt.cpu().numpy() - y_ref) <= 1e-14 * np.linalg.norm(y_ref)
    pc = P.Precond(a, "ic0")
    L = O.lower(oa)
    L.vals = O.ic0(oa)[0]
    U, _ = O.transpose(L)
    for upper, ref in ((False, O.trsv_lower(L, x)), (True, O.trsv_upper(U, x))):
        pc.trsv_device(upper, xt.data_ptr(), yt.data_ptr())
        assert np.linalg.norm(yt.cpu().numpy() - ref) <= 1e-12 * np.linalg.norm(ref)


def _seq_matvec(rp, cols, vals, x):
    y = np.empty(len(rp) - 1)
    for i in range(len(rp) - 1):
        acc = 0.0
        for k in range(rp[i], rp[i + 1]):
            acc = acc + vals[k] * x[cols[k]]
        y[i] = acc
    return y


def test_short_row_spmv_bit_exact():
    """Short scalar rows run the row-tile product (a warp per 32 rows,
    products staged, each row summed from 0 in CSR order, unfused): the
    reference's csr_matvec (sparse.cpp:121-135) bit for bit — also across
    empty rows and a row longer than one staging chunk."""
    import torch
    rng = np.random.default_rng(7)
    n = 3000
    lens = rng.integers(0, 9, n)
    lens[100], lens[2999] = 700, 300
    lens[2000:2040] = 0
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int32)
    cases = [P.Matrix.gen_poisson(2, 40), P.Matrix.gen_diffusion(3, 13, -3.0, 3.0, 4),
             P.Matrix.from_csr(rp, cols, rng.standard_normal(int(rp[-1])))]
    for a in cases:
        arp, acols, avals = a.csr()
        x = rng.standard_normal(a.n)
        xt = torch.from_numpy(x).cuda()
        yt = torch.empty_like(xt)
        a.spmv_device(xt.data_ptr(), yt.data_ptr())
        assert np.array_equal(bits(yt.cpu().numpy()), bits(_seq_matvec(arp, acols, avals, x)))


def test_deterministic_runs():
    w = SMALL[1]
    a, b, model, *_ = built(w)
    x1, r1 = P.pcg_solve(a, b, "gnnic", model, rel_tol=1e-8)
    x2, r2 = P.pcg_solve(a, b, "gnnic", model, rel_tol=1e-8)
    assert r1["iterations"] == r2["iterations"] and np.array_equal(bits(x1), bits(x2))


def test_edge_cases():
    a = P.Matrix.gen_poisson(2, 6)
    n = a.n
    x, rep = P.pcg_solve(a, np.zeros(n), "ic0")
    assert rep["converged"] and rep["iterations"] == 0 and not x.any()
    b = P.field_uniform_pm1(n, 3)
    x, rep = P.pcg_solve(a, b, "ic0", rel_tol=1e-12, max_iters=2)
    assert rep["iterations"] == 2 and not rep["converged"]
    one = P.Matrix.gen_poisson(3, 1)
    x, rep = P.pcg_solve(one, np.array([6.0]), "ic0")
    assert rep["iterations"] == 1 and abs(x[0] - 1.0) < 1e-15


@pytest.mark.parametrize("m", [2, 3, 4])
def test_tiny_2d_poisson_sweeps_and_pcg(m):
    """Systems whose dof blocks have <= 2 off-block entries (2-D 5-point
    stencils up to 4 x 4): the sweep schedule is cut for the narrowest lane
    group the kernels instantiate (round 1 built these for 2 lanes and ran
    them with 4: the PCG never finished)."""
    a = P.Matrix.gen_poisson(2, m)
    oa = O.gen_poisson(2, m)
    b = P.field_uniform_pm1(a.n, 11)
    x, rep = P.pcg_solve(a, b, "ic0", rel_tol=1e-10)
    xo, ro = O.pcg(oa, b, "ic0", rel_tol=1e-10)
    assert rep["converged"] and abs(rep["iterations"] - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)


def test_error_paths():
    b2 = np.ones(2)
    asym = P.Matrix.from_coo(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [2.0, 1.0, 0.5, 2.0])
    with pytest.raises(P.FormatError, match="not symmetric"):
        P.pcg_solve(asym, b2, "ic0")
    nodiag = P.Matrix.from_coo(2, 2, [0, 1], [0, 0], [1.0, 1.0])
    with pytest.raises(P.NumericError, match="jacobi: nonpositive diagonal at row 1"):
        P.pcg_solve(nodiag, b2, "jacobi")
    kers = P.Matrix.from_coo(4, 4, [0, 0, 0, 1, 1, 1, 2, 2, 2, 3, 3, 3], [0, 1, 3, 0, 1, 2, 1, 2, 3, 0, 2, 3],
                             [3, -2, 2, -2, 3, -2, -2, 3, -2, 2, -2, 3])
    with pytest.raises(P.NumericError, match="row 3"):
        P.Precond(kers, "ic0")
    a = P.Matrix.gen_poisson(2, 4)
    with pytest.raises(P.ArgumentError, match="needs a model"):
        P.pcg_solve(a, np.ones(16), "gnnic")
    with pytest.raises(P.ArgumentError, match="unknown preconditioner kind"):
        P.pcg_solve(a, np.ones(16), "ilu")
    with pytest.raises(P.FormatError, match="duplicate"):
        P.Matrix.from_coo(2, 2, [0, 0], [1, 1], [1.0, 2.0])
    with pytest.raises(P.FormatError, match="out of bounds"):
        P.Matrix.from_coo(2, 2, [0, 2], [0, 0], [1.0, 2.0])
    with pytest.raises(P.ArgumentError):
        P.Matrix.gen_poisson(4, 3)


def test_shift_rescues_singular_on_device():
    a = P.Matrix.from_coo(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0])
    l = P.Precond(a, "ic0").factor()
    assert np.array_equal(bits(l), bits(O.ic0(O.Csr(2, np.array([0, 2, 4]), np.array([0, 1, 0, 1], np.int32),
                                                    np.ones(4)))[0]))


def test_matrix_market_roundtrip(tmp_path):
    a = P.Matrix.gen_poisson(3, 5, True, 9)
    p = str(tmp_path / "a.mtx")
    a.write(p)
    assert open(p).readline().strip() == "%%MatrixMarket matrix coordinate real symmetric"
    b = P.Matrix.read(p)
    for u, v in zip(a.csr(), b.csr()):
        assert np.array_equal(u, v)


def test_from_coo_equals_generator():
    a = P.Matrix.gen_poisson(2, 7, True, 3)
    rp, cols, vals = a.csr()
    rows = np.repeat(np.arange(a.n), np.diff(rp))
    perm = np.random.default_rng(1).permutation(len(vals))
    b = P.Matrix.from_coo(a.n, a.n, rows[perm], cols[perm], vals[perm])
    for u, v in zip(a.csr(), b.csr()):
        assert np.array_equal(u, v)
