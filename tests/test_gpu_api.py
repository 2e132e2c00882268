"""C-ABI behaviour the advisor flagged: a preconditioner
outlives pclab_matrix_drop_analysis; malformed row_ptr is a FormatError, not
a device fault; a per-call stream is not sticky; rectangular COO input is
accepted at construction and rejected by each solve with the reference's
own message (sparse.cpp:55-72 accepts it; precond.cpp:92, sparse.cpp:190,
features.cpp:13 and krylov.cpp:118 reject it)."""
import numpy as np
import pytest
import torch

import paper_2412_07127_b200 as P

pytestmark = pytest.mark.gpu


def test_precond_survives_drop_analysis():
    w = P.workloads.by_name("elasticity_q1_40").scaled(6)
    a, b, model = P.workloads.build(w)
    x_ref, r_ref = P.pcg_solve(a, b, "ic0", rel_tol=1e-8)
    for kind in ("ic0", "gnnic"):
        pc = P.Precond(a, kind, model if kind == "gnnic" else None)
        a.drop_analysis()
        bt = torch.from_numpy(b).cuda()
        xt = torch.zeros_like(bt)
        rep = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, max_iters=3000)
        if kind == "ic0":
            assert rep["iterations"] == r_ref["iterations"]
            assert np.array_equal(xt.cpu().numpy(), x_ref)
        yt = torch.empty_like(bt)
        pc.trsv_device(False, bt.data_ptr(), yt.data_ptr())
        assert np.isfinite(yt.cpu().numpy()).all()
        assert pc.info()["nnz_lower"] > 0
        del pc
    # jacobi / none after a drop: no analysis needed
    x, rep = P.pcg_solve(a, b, "jacobi", rel_tol=1e-6, max_iters=5000)
    assert rep["iterations"] > 0


@pytest.mark.parametrize("rp, msg", [
    ([1, 2, 3], "row_ptr\\[0\\] != 0"),
    ([0, 3, 2], "not monotone"),
    ([0, 1, 5], "row_ptr\\[n\\] != nnz"),
    ([0, 1, 1 << 40], "row_ptr"),
])
def test_from_csr_rejects_malformed_row_ptr(rp, msg):
    rp = np.array(rp, np.int64)
    cols = np.array([0, 1], np.int32)
    vals = np.array([1.0, 1.0])
    rpt = torch.from_numpy(rp).cuda()
    ct = torch.from_numpy(cols).cuda()
    vt = torch.from_numpy(vals).cuda()
    with pytest.raises(P.FormatError, match=msg):
        P.Matrix.from_csr_device(2, 2, rpt.data_ptr(), ct.data_ptr(), vt.data_ptr())
    # the CUDA context is still healthy
    a = P.Matrix.gen_poisson(2, 4)
    x, rep = P.pcg_solve(a, np.ones(16), "ic0", rel_tol=1e-8)
    assert rep["converged"]


def test_call_stream_is_not_sticky():
    a = P.Matrix.gen_poisson(3, 8)
    pc = P.Precond(a, "ic0")
    b = P.field_uniform_pm1(a.n, 2)
    bt = torch.from_numpy(b).cuda()
    xt = torch.zeros_like(bt)
    s = torch.cuda.Stream()
    rep1 = pc.solve_device(bt.data_ptr(), xt.data_ptr(), rel_tol=1e-8, stream=s.cuda_stream)
    torch.cuda.synchronize()
    del s  # the caller's stream is gone; later calls must not use it
    torch.cuda.synchronize()
    x2, rep2 = P.pcg_solve(a, b, "ic0", rel_tol=1e-8)
    yt = torch.empty_like(bt)
    a.spmv_device(bt.data_ptr(), yt.data_ptr())
    pc.trsv_device(True, bt.data_ptr(), yt.data_ptr())
    assert rep2["iterations"] == rep1["iterations"]
    assert np.array_equal(x2, xt.cpu().numpy())


def test_rectangular_coo_accepted_then_rejected_like_the_reference():
    # 2 x 3, a column >= n_rows: make_coo accepts it
    a = P.Matrix.from_coo(2, 3, [0, 0, 1, 1], [0, 2, 1, 2], [2.0, 1.0, 3.0, 1.0])
    assert a.shape() == (2, 3, 4)
    b = np.ones(2)
    with pytest.raises(P.ArgumentError, match="^pcg: shape mismatch$"):
        P.pcg_solve(a, b, "none")
    with pytest.raises(P.ArgumentError, match="^jacobi: matrix not square$"):
        P.pcg_solve(a, b, "jacobi")
    with pytest.raises(P.ArgumentError, match="^lower_triangle: matrix not square$"):
        P.pcg_solve(a, b, "ic0")
    model = P.Model.init(1)
    with pytest.raises(P.ArgumentError, match="^lower_triangle: matrix not square$"):
        P.pcg_solve(a, b, "gnnic", model)
    with pytest.raises(P.ArgumentError, match="^node_features: matrix not square$"):
        P.pcg_solve(a, b, "nic", model)
    with pytest.raises(P.FormatError, match="out of bounds"):
        P.Matrix.from_coo(2, 3, [0], [3], [1.0])


def test_device_coo_matches_make_coo_order_and_errors():
    """make_coo (sparse.cpp:55-72) on the device: the first offending entry
    in (row, col) order is the one reported, whether the input arrives
    sorted (fast path) or shuffled (radix sort), with or without an
    out-of-bounds entry (two stable passes on the raw signed pairs)."""
    a = P.Matrix.gen_poisson(3, 6, True, 4)
    rp, cols, vals = a.csr()
    rows = np.repeat(np.arange(a.n), np.diff(rp))
    for perm in (np.arange(len(vals)), np.random.default_rng(3).permutation(len(vals))):
        b = P.Matrix.from_coo(a.n, a.n, rows[perm], cols[perm], vals[perm])
        for u, v in zip(a.csr(), b.csr()):
            assert np.array_equal(u, v)
    r = [5, 2, 2, 0, 9]
    c = [1, 3, 3, 0, 0]
    with pytest.raises(P.FormatError, match=r"^coo: entries not sorted or duplicate at \(2, 3\)$"):
        P.Matrix.from_coo(6, 6, r, c, [1.0] * 5)  # (9, 0) is out of bounds but sorts last
    with pytest.raises(P.FormatError, match=r"^coo: entry \(-1, 4\) out of bounds$"):
        P.Matrix.from_coo(6, 6, r + [-1], c + [4], [1.0] * 6)  # (-1, 4) sorts first
    with pytest.raises(P.FormatError, match=r"^coo: entry \(1, 6\) out of bounds$"):
        P.Matrix.from_coo(6, 6, [0, 1, 1], [0, 2, 6], [1.0] * 3)
    e = P.Matrix.from_coo(3, 3, [], [], [])
    assert e.shape() == (3, 3, 0)
