"""The CPU oracle is pinned to the reference: committed fixtures produced by
the reference itself (tests/golden), the reference's own committed test
output (acceptance criterion 5), and -- where oracle/_ref is built -- live
bit-for-bit comparison against the reference compiled from its sources."""
import numpy as np
import pytest

from conftest import bits, csr_from
from oracle import oracle as O

SYSTEMS = ["p2_m8", "p2_m6_v19", "p3_m5_v5", "p3_m1", "el_m3"]
ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_generators_match_reference_fixtures(golden):
    for name, (dim, m, k) in {"p2_m8": (2, 8, None), "p2_m6_v19": (2, 6, 19), "p3_m5_v5": (3, 5, 5),
                              "p3_m1": (3, 1, None)}.items():
        a = O.gen_poisson(dim, m, None if k is None else O.cell_coeffs(m ** dim, k, -1.0, 1.0))
        g = csr_from(golden, name)
        assert np.array_equal(a.rp, g.rp) and np.array_equal(a.cols, g.cols)
        assert np.array_equal(bits(a.vals), bits(g.vals)), name


def test_gnn_init_matches_reference(golden):
    assert np.array_equal(bits(O.gnn_init(1)), bits(golden["gnn_init_1"]))
    assert np.array_equal(bits(O.gnn_init(0)), bits(golden["gnn_init_0"]))
    assert O.gnn_init(1).size == 997  # test_gnn.cpp: "the documented 997"


@pytest.mark.parametrize("name", ["p2_m6_v19", "p3_m5_v5", "el_m3"])
def test_features_gnn_and_factors_bit_exact(golden, name):
    a = csr_from(golden, name)
    p = golden["gnn_init_1"]
    assert np.array_equal(bits(O.node_features(a)), bits(golden[f"{name}.features"]))
    out, sigma = O.gnn_forward(a, p)
    assert np.array_equal(bits(out), bits(golden[f"{name}.gnn_out"]))
    assert sigma == golden[f"{name}.sigma"][0]
    for kind in ("ic0", "gnnic", "nic"):
        if f"{name}.{kind}" in golden.files:
            assert np.array_equal(bits(O.factor(a, kind, p)), bits(golden[f"{name}.{kind}"])), kind


@pytest.mark.parametrize("name", ["p2_m6_v19", "p3_m5_v5", "el_m3"])
def test_pcg_bit_exact(golden, name):
    a = csr_from(golden, name)
    p = golden["gnn_init_1"]
    b = golden[f"{name}.b"]
    for kind in ("none", "jacobi", "ic0", "gnnic", "nic"):
        x, rep, hist = O.pcg(a, b, kind, p, rel_tol=1e-8, max_iters=2000, history=True)
        it, conv = golden[f"{name}.pcg.{kind}.iters"]
        assert rep["iterations"] == it and rep["converged"] == conv, kind
        assert np.array_equal(bits(x), bits(golden[f"{name}.pcg.{kind}.x"])), kind
        assert np.array_equal(bits(hist), bits(golden[f"{name}.pcg.{kind}.hist"])), kind


def test_acceptance_c5_iteration_counts():
    """The reference's committed acceptance output (test_output.txt):
    'iterations: none 432, diagonal 231, no-fill factor 70' on
    gen_poisson(2, 64, derive_seed(2026, 5)), rhs experiment_rhs, rtol 1e-6."""
    ms = O.derive_seed(2026, 5)
    a = O.gen_poisson(2, 64, O.cell_coeffs(64 * 64, ms, -1.0, 1.0))
    b = O.uniform_pm1_field(a.n, O.derive_seed(ms, 14))
    its = [O.pcg(a, b, k, rel_tol=1e-6)[1]["iterations"] for k in ("none", "jacobi", "ic0")]
    assert its == [432, 231, 70]


def test_kershaw_breakdown_names_row_3(golden):
    rp = np.array([0, 3, 6, 9, 12], np.int64)
    c = np.array([0, 1, 3, 0, 1, 2, 1, 2, 3, 0, 2, 3], np.int32)
    v = np.array([3, -2, 2, -2, 3, -2, -2, 3, -2, 2, -2, 3], np.float64)
    with pytest.raises(O.OracleError, match="row 3"):
        O.ic0(O.Csr(4, rp, c, v))
    assert "row 3" in str(golden["kershaw.error"][0])


def test_ic0_shift_rescues_singular():
    # test_precond.cpp: [[1,1],[1,1]] factors A + 1e-8 I on the first retry
    a = O.Csr(2, np.array([0, 2, 4], np.int64), np.array([0, 1, 0, 1], np.int32), np.ones(4))
    l, att = O.ic0(a)
    assert att == 1 and l[2] > 0
    assert abs(l[0] ** 2 - (1 + 1e-8)) < 1e-12


def test_ic0_tridiagonal_is_exact_cholesky():
    n = 50
    rows, cols, vals = [], [], []
    for i in range(n):
        for j, v in ((i - 1, -1.0), (i, 2.0), (i + 1, -1.0)):
            if 0 <= j < n:
                rows.append(i), cols.append(j), vals.append(v)
    rp = np.searchsorted(rows, np.arange(n + 1)).astype(np.int64)
    a = O.Csr(n, rp, np.array(cols, np.int32), np.array(vals))
    dense = np.zeros((n, n))
    for i in range(n):
        dense[i, cols[rp[i]:rp[i + 1]]] = vals[rp[i]:rp[i + 1]]
    ch = np.linalg.cholesky(dense)
    lo = O.lower(a)
    l, _ = O.ic0(a)
    for i in range(n):
        for k in range(lo.rp[i], lo.rp[i + 1]):
            assert abs(l[k] - ch[i, lo.cols[k]]) <= 1e-12 * abs(ch[i, lo.cols[k]])


def brute_levels(l):
    lv = np.zeros(l.n, np.int64)
    for i in range(l.n):
        deps = [j for j in l.cols[l.rp[i]:l.rp[i + 1]] if j < i]
        lv[i] = max((lv[j] + 1 for j in deps), default=0)
    return lv


@pytest.mark.parametrize("name", SYSTEMS)
def test_level_sets_match_definition(golden, name):
    a = csr_from(golden, name)
    lo = O.lower(a)
    lv, nl = O.levels_lower(lo)
    want = brute_levels(lo)
    assert np.array_equal(lv, want) and nl == want.max() + 1
    up, _ = O.transpose(lo)
    lu, _ = O.levels_upper(up)
    # backward sweep on U = L^T: row i waits for every j > i in its row
    want_u = np.zeros(a.n, np.int64)
    for i in range(a.n - 1, -1, -1):
        deps = [j for j in up.cols[up.rp[i]:up.rp[i + 1]] if j > i]
        want_u[i] = max((want_u[j] + 1 for j in deps), default=0)
    assert np.array_equal(lu, want_u)


def test_elasticity_generator_properties():
    ke = O.element_stiffness(1.0 / 7, 0.3)
    assert np.array_equal(ke, ke.T)
    ev = np.linalg.eigvalsh(ke)
    assert np.sum(np.abs(ev) < 1e-12 * ev.max()) == 6  # six rigid-body modes
    m = 4
    a = O.gen_elasticity(m, O.lognormal_field(m ** 3, 3, 1.0))
    n, nnz = O.elasticity_dims(m)
    assert (a.n, a.nnz) == (n, nnz) == (3 * (m + 1) ** 2 * m, a.rp[-1])
    import scipy.sparse as sp
    A = sp.csr_matrix((a.vals, a.cols, a.rp), shape=(a.n, a.n))
    assert (A != A.T).nnz == 0  # bitwise symmetric, as lower_triangle demands
    assert np.linalg.eigvalsh(A.toarray()).min() > 0  # clamped: SPD
    nnz_row = np.diff(a.rp)
    assert nnz_row.max() == 81


@ref_only
def test_live_reference_elasticity_and_diffusion():
    """Oracle == reference bit for bit on systems built by the oracle's own
    generators (elasticity, 10^u diffusion)."""
    p = O.gnn_init(1)
    e = O.gen_elasticity(3, O.lognormal_field(27, 11, 1.0))
    d = O.gen_poisson(3, 6, O.cell_coeffs(216, 4, -3.0, 3.0))
    for a in (e, d):
        for kind in ("ic0", "gnnic", "nic"):
            assert np.array_equal(bits(O.factor(a, kind, p)), bits(O.ref_factor(a, kind, p)[0]))
        b = O.normal_field(a.n, 5)
        for kind in ("none", "jacobi", "ic0", "gnnic"):
            x1, r1 = O.pcg(a, b, kind, p, rel_tol=1e-8, max_iters=3000)
            x2, r2 = O.ref_pcg(a, b, kind, p, rel_tol=1e-8, max_iters=3000)
            assert r1["iterations"] == r2["iterations"] and np.array_equal(bits(x1), bits(x2))


@ref_only
def test_live_reference_generator_seeds():
    for dim, m, seed in ((2, 9, 3), (3, 7, 101)):
        a = O.ref_gen_poisson(dim, m, True, seed)
        b = O.gen_poisson(dim, m, O.cell_coeffs(m ** dim, seed, -1.0, 1.0))
        assert np.array_equal(bits(a.vals), bits(b.vals)) and np.array_equal(a.cols, b.cols)
