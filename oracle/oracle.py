"""ctypes/numpy front end for the CPU checkers.

TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / ``--impl reference`` legs, never by the product
package. Two libraries are wrapped:

* ``C``   -- oracle/liboracle.so, the plain-C restatement (pclab_oracle.c)
* ``REF`` -- oracle/_ref/libpclab_ref.so, the unmodified reference sources
  compiled in place plus ref_shim.cpp (present wherever it was built)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

_lib = None
_ref = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        # ORACLE_LIB: another build of pclab_oracle.c (tests/golden/sensitivity.py)
        path = os.environ.get("ORACLE_LIB") or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run make -C oracle)")
        _lib = C.CDLL(path)
        L = _lib
        L.or_uniform_at.restype = C.c_double
        L.or_uniform_at.argtypes = [C.c_uint64, C.c_uint64]
        L.or_normal_at.restype = C.c_double
        L.or_normal_at.argtypes = [C.c_uint64, C.c_uint64]
        L.or_derive_seed.restype = C.c_uint64
        L.or_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.or_poisson_n.restype = C.c_int64
        L.or_poisson_n.argtypes = [C.c_int, C.c_int64]
        L.or_poisson_nnz.restype = C.c_int64
        L.or_poisson_nnz.argtypes = [C.c_int, C.c_int64]
        L.or_cell_coeffs.argtypes = [C.c_int64, C.c_uint64, C.c_double, C.c_double, _f64p]
        L.or_gen_poisson.argtypes = [C.c_int, C.c_int64, C.c_void_p, _i64p, _i32p, _f64p]
        L.or_element_stiffness.argtypes = [C.c_double, C.c_double, _f64p]
        L.or_elasticity_dims.argtypes = [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_lognormal_field.argtypes = [C.c_int64, C.c_uint64, C.c_double, _f64p]
        L.or_normal_field.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.or_uniform_pm1_field.argtypes = [C.c_int64, C.c_uint64, _f64p]
        L.or_gen_elasticity.argtypes = [C.c_int64, C.c_double, _f64p, _i64p, _i32p, _f64p]
        L.or_lower_nnz.restype = C.c_int64
        L.or_lower_nnz.argtypes = [C.c_int64, _i64p, _i32p]
        L.or_lower.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p]
        L.or_transpose.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _i64p, _i32p, _f64p, _i64p]
        for f in (L.or_levels_lower, L.or_levels_upper):
            f.restype = C.c_int64
            f.argtypes = [C.c_int64, _i64p, _i32p, _i32p]
        for f in (L.or_block_levels_lower, L.or_block_levels_upper):
            f.restype = C.c_int64
            f.argtypes = [C.c_int64, C.c_int, _i64p, _i32p, _i32p]
        L.or_csr_matvec.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p]
        for f in (L.or_trsv_lower, L.or_trsv_upper):
            f.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p, C.POINTER(C.c_int64)]
        L.or_ic0.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p,
                             C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.or_node_features.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p]
        L.or_scale_by_std.restype = C.c_double
        L.or_scale_by_std.argtypes = [C.c_int64, _f64p, _f64p]
        L.or_gnn_init.argtypes = [C.c_uint64, _f64p]
        L.or_gnn_zero.argtypes = [_f64p]
        L.or_gnn_forward.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p,
                                     C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.or_pcg.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, C.c_int,
                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int64,
                             _f64p, C.c_void_p, C.c_void_p]
    return _lib


class RefReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int32),
                ("residual_mismatch", C.c_int32), ("final_rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("p_time", C.c_double),
                ("cg_time", C.c_double), ("total_time", C.c_double),
                ("tri_solve_time_per_iter", C.c_double)]


class OrReport(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int),
                ("final_rel_residual", C.c_double), ("true_rel_residual", C.c_double),
                ("residual_mismatch", C.c_int)]


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libpclab_ref.so"))


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libpclab_ref.so")
        if not os.path.exists(path):
            raise RuntimeError(f"reference not built: {path}")
        _ref = C.CDLL(path)
        R = _ref
        R.ref_last_error.restype = C.c_char_p
        R.ref_gen_poisson_nnz.restype = C.c_int64
        R.ref_gen_poisson_nnz.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_uint64]
        R.ref_gen_poisson.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_uint64, _i64p, _i32p, _f64p]
        R.ref_gnn_init.argtypes = [C.c_uint64, _f64p]
        R.ref_node_features.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p]
        R.ref_gnn_forward.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p,
                                      C.POINTER(C.c_double)]
        R.ref_factor.argtypes = [C.c_int, C.c_int64, _i64p, _i32p, _f64p, C.c_void_p, _f64p,
                                 C.POINTER(C.c_double)]
        R.ref_pcg.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, C.c_char_p, C.c_void_p,
                              C.c_double, C.c_int64, _f64p, C.POINTER(RefReport), C.c_void_p]
        R.ref_pcg_factor.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p, _f64p, C.c_double,
                                     C.c_int64, _f64p, C.POINTER(RefReport)]
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


# --------------------------------------------------------------- matrices
@dataclass
class Csr:
    n: int
    rp: np.ndarray  # int64 [n+1]
    cols: np.ndarray  # int32 [nnz]
    vals: np.ndarray  # float64 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])


def uniform_at(seed: int, i: int) -> float:
    return lib().or_uniform_at(seed, i)


def derive_seed(seed: int, tag: int) -> int:
    return lib().or_derive_seed(seed, tag)


def cell_coeffs(n: int, seed: int, lo: float, hi: float) -> np.ndarray:
    k = np.empty(n, np.float64)
    lib().or_cell_coeffs(n, seed, lo, hi, k)
    return k


def gen_poisson(dim: int, m: int, cell_k: np.ndarray | None = None) -> Csr:
    L = lib()
    n = L.or_poisson_n(dim, m)
    nnz = L.or_poisson_nnz(dim, m)
    rp = np.empty(n + 1, np.int64)
    cols = np.empty(nnz, np.int32)
    vals = np.empty(nnz, np.float64)
    kp = None if cell_k is None else np.ascontiguousarray(cell_k, np.float64).ctypes.data
    keep = cell_k
    st = L.or_gen_poisson(dim, m, kp, rp, cols, vals)
    del keep
    if st:
        raise OracleError(st, "gen_poisson: bad arguments")
    return Csr(n, rp, cols, vals)


def element_stiffness(h: float, nu: float) -> np.ndarray:
    ke = np.empty(576, np.float64)
    lib().or_element_stiffness(h, nu, ke)
    return ke.reshape(24, 24)


def elasticity_dims(m: int) -> tuple[int, int]:
    n, nnz = C.c_int64(), C.c_int64()
    lib().or_elasticity_dims(m, C.byref(n), C.byref(nnz))
    return n.value, nnz.value


def lognormal_field(n: int, seed: int, sigma: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().or_lognormal_field(n, seed, sigma, out)
    return out


def normal_field(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().or_normal_field(n, seed, out)
    return out


def uniform_pm1_field(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().or_uniform_pm1_field(n, seed, out)
    return out


def gen_elasticity(m: int, moduli: np.ndarray, nu: float = 0.3) -> Csr:
    n, nnz = elasticity_dims(m)
    rp = np.empty(n + 1, np.int64)
    cols = np.empty(nnz, np.int32)
    vals = np.empty(nnz, np.float64)
    st = lib().or_gen_elasticity(m, nu, np.ascontiguousarray(moduli, np.float64), rp, cols, vals)
    if st:
        raise OracleError(st, "gen_elasticity: bad arguments")
    assert rp[-1] == nnz
    return Csr(n, rp, cols, vals)


# -------------------------------------------------------------- structure
def lower(a: Csr) -> Csr:
    L = lib()
    nnz = L.or_lower_nnz(a.n, a.rp, a.cols)
    rp = np.empty(a.n + 1, np.int64)
    cols = np.empty(max(nnz, 1), np.int32)
    vals = np.empty(max(nnz, 1), np.float64)
    L.or_lower(a.n, a.rp, a.cols, a.vals, rp, cols, vals)
    return Csr(a.n, rp, cols[:nnz].copy(), vals[:nnz].copy())


def transpose(l: Csr) -> tuple[Csr, np.ndarray]:
    nnz = l.nnz
    rp = np.empty(l.n + 1, np.int64)
    cols = np.empty(max(nnz, 1), np.int32)
    vals = np.empty(max(nnz, 1), np.float64)
    u2l = np.empty(max(nnz, 1), np.int64)
    lib().or_transpose(l.n, l.rp, l.cols, l.vals, rp, cols, vals, u2l)
    return Csr(l.n, rp, cols[:nnz].copy(), vals[:nnz].copy()), u2l[:nnz].copy()


def levels_lower(l: Csr) -> tuple[np.ndarray, int]:
    lv = np.empty(max(l.n, 1), np.int32)
    nl = lib().or_levels_lower(l.n, l.rp, l.cols, lv)
    return lv[: l.n], int(nl)


def levels_upper(u: Csr) -> tuple[np.ndarray, int]:
    lv = np.empty(max(u.n, 1), np.int32)
    nl = lib().or_levels_upper(u.n, u.rp, u.cols, lv)
    return lv[: u.n], int(nl)


def block_levels_lower(l: Csr, bs: int) -> tuple[np.ndarray, int]:
    lv = np.empty(max(l.n // bs, 1), np.int32)
    nl = lib().or_block_levels_lower(l.n, bs, l.rp, l.cols, lv)
    return lv[: l.n // bs], int(nl)


def block_levels_upper(u: Csr, bs: int) -> tuple[np.ndarray, int]:
    lv = np.empty(max(u.n // bs, 1), np.int32)
    nl = lib().or_block_levels_upper(u.n, bs, u.rp, u.cols, lv)
    return lv[: u.n // bs], int(nl)


# ---------------------------------------------------------------- kernels
def matvec(a: Csr, x: np.ndarray) -> np.ndarray:
    y = np.empty(a.n, np.float64)
    lib().or_csr_matvec(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(x, np.float64), y)
    return y


def trsv_lower(l: Csr, b: np.ndarray) -> np.ndarray:
    x = np.empty(l.n, np.float64)
    bad = C.c_int64(-1)
    st = lib().or_trsv_lower(l.n, l.rp, l.cols, l.vals, np.ascontiguousarray(b, np.float64), x,
                             C.byref(bad))
    if st:
        raise OracleError(st, f"tri_solve_lower: row {bad.value}")
    return x


def trsv_upper(u: Csr, b: np.ndarray) -> np.ndarray:
    x = np.empty(u.n, np.float64)
    bad = C.c_int64(-1)
    st = lib().or_trsv_upper(u.n, u.rp, u.cols, u.vals, np.ascontiguousarray(b, np.float64), x,
                             C.byref(bad))
    if st:
        raise OracleError(st, f"tri_solve_upper: row {bad.value}")
    return x


# -------------------------------------------------------- preconditioners
def ic0(a: Csr) -> tuple[np.ndarray, int]:
    """IC(0) factor values on lower(a)'s pattern and the shift attempts used."""
    lo = lower(a)
    out = np.empty(max(lo.nnz, 1), np.float64)
    fail = C.c_int64(-1)
    att = C.c_int(0)
    st = lib().or_ic0(a.n, lo.rp, lo.cols, lo.vals, out, C.byref(fail), C.byref(att))
    if st == 2:
        raise OracleError(st, f"ic0: missing diagonal at row {fail.value}")
    if st:
        raise OracleError(st, f"ic0: nonpositive pivot at row {fail.value}")
    return out[: lo.nnz], att.value


def node_features(a: Csr) -> np.ndarray:
    f = np.empty((max(a.n, 1), 9), np.float64)
    lib().or_node_features(a.n, a.rp, a.cols, a.vals, f)
    return f[: a.n]


def gnn_init(seed: int) -> np.ndarray:
    p = np.empty(997, np.float64)
    lib().or_gnn_init(seed, p)
    return p


def gnn_zero() -> np.ndarray:
    p = np.empty(997, np.float64)
    lib().or_gnn_zero(p)
    return p


def gnn_forward(a: Csr, params: np.ndarray) -> tuple[np.ndarray, float]:
    ne = lib().or_lower_nnz(a.n, a.rp, a.cols)
    out = np.empty(max(ne, 1), np.float64)
    sigma = C.c_double()
    bad = C.c_int(0)
    st = lib().or_gnn_forward(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(params), out,
                              C.byref(sigma), C.byref(bad))
    if st:
        raise OracleError(st, f"gnn forward: non-finite activation in block {bad.value}")
    return out[:ne], sigma.value


def factor(a: Csr, kind: str, params: np.ndarray | None = None) -> np.ndarray:
    """L values on lower(a)'s pattern for kind in {ic0, gnnic, nic}
    (precond.cpp:109, 155, 145)."""
    if kind == "ic0":
        return ic0(a)[0]
    out, sigma = gnn_forward(a, params)
    if kind == "nic":
        l = out * sigma
    else:
        l = ic0(a)[0] + out
    lo = lower(a)
    diag = l[lo.rp[1:] - 1]
    if not np.all(diag > 0.0):
        raise OracleError(3, "lower factor: nonpositive diagonal")
    return l


def pcg(a: Csr, b: np.ndarray, kind: str = "ic0", params: np.ndarray | None = None,
        rel_tol: float = 1e-6, max_iters: int = -1, lvals: np.ndarray | None = None,
        history: bool = False):
    """krylov.cpp:114 pcg. Returns (x, report dict[, history])."""
    L = lib()
    x = np.empty(a.n, np.float64)
    rep = OrReport()
    lo = None
    kcode = {"none": 0, "jacobi": 1}.get(kind, 2)
    if kcode == 2:
        lo = lower(a)
        lo.vals = np.ascontiguousarray(lvals if lvals is not None else factor(a, kind, params))
    hist = np.zeros(a.n * 10 + 2 if max_iters < 0 else max_iters + 2, np.float64) if history else None
    st = L.or_pcg(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(b, np.float64), kcode,
                  lo.rp.ctypes.data if lo else None, lo.cols.ctypes.data if lo else None,
                  lo.vals.ctypes.data if lo else None, rel_tol, max_iters, x, C.byref(rep),
                  hist.ctypes.data if hist is not None else None)
    if st == 6:  # OR_ERR_CURVATURE: the reference's message (krylov.cpp:151-154)
        raise OracleError(3, f"pcg: nonpositive curvature at iteration {rep.iterations} (matrix not SPD?)")
    if st:
        raise OracleError(st, "pcg: zero pivot in the triangular solve")
    r = {k: getattr(rep, k) for k, _ in OrReport._fields_}
    if history:
        return x, r, hist[: rep.iterations + 1]
    return x, r


# ------------------------------------------------------- reference (_ref)
def ref_check(st: int):
    if st:
        raise OracleError(st, ref().ref_last_error().decode())


def ref_gen_poisson(dim: int, m: int, variable: bool, seed: int) -> Csr:
    R = ref()
    n = m ** dim
    nnz = R.ref_gen_poisson_nnz(dim, m, int(variable), seed)
    rp = np.empty(n + 1, np.int64)
    cols = np.empty(nnz, np.int32)
    vals = np.empty(nnz, np.float64)
    ref_check(R.ref_gen_poisson(dim, m, int(variable), seed, rp, cols, vals))
    return Csr(n, rp, cols, vals)


def ref_gnn_init(seed: int) -> np.ndarray:
    p = np.empty(997, np.float64)
    ref().ref_gnn_init(seed, p)
    return p


def ref_node_features(a: Csr) -> np.ndarray:
    f = np.empty((max(a.n, 1), 9), np.float64)
    ref_check(ref().ref_node_features(a.n, a.rp, a.cols, a.vals, f))
    return f[: a.n]


def ref_gnn_forward(a: Csr, params: np.ndarray) -> tuple[np.ndarray, float]:
    ne = lib().or_lower_nnz(a.n, a.rp, a.cols)
    out = np.empty(max(ne, 1), np.float64)
    sigma = C.c_double()
    ref_check(ref().ref_gnn_forward(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(params),
                                    out, C.byref(sigma)))
    return out[:ne], sigma.value


def ref_factor(a: Csr, kind: str, params: np.ndarray | None = None) -> tuple[np.ndarray, float]:
    ne = lib().or_lower_nnz(a.n, a.rp, a.cols)
    out = np.empty(max(ne, 1), np.float64)
    pt = C.c_double()
    p = None if params is None else np.ascontiguousarray(params, np.float64)
    ref_check(ref().ref_factor({"ic0": 0, "gnnic": 1, "nic": 2}[kind], a.n, a.rp, a.cols,
                               a.vals, p.ctypes.data if p is not None else None, out,
                               C.byref(pt)))
    return out[:ne], pt.value


def ref_pcg(a: Csr, b: np.ndarray, kind: str = "ic0", params: np.ndarray | None = None,
            rel_tol: float = 1e-6, max_iters: int = -1, history: bool = False):
    x = np.empty(a.n, np.float64)
    rep = RefReport()
    p = None if params is None else np.ascontiguousarray(params, np.float64)
    hist = np.zeros(a.n * 10 + 2 if max_iters < 0 else max_iters + 2, np.float64) if history else None
    ref_check(ref().ref_pcg(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(b, np.float64),
                            kind.encode(), p.ctypes.data if p is not None else None, rel_tol,
                            max_iters, x, C.byref(rep),
                            hist.ctypes.data if hist is not None else None))
    r = {k: getattr(rep, k) for k, _ in RefReport._fields_}
    if history:
        return x, r, hist[: rep.iterations + 1]
    return x, r


class RefSession:
    """The reference's pcg() on a resident system + IC(0)-kind factor
    (ref_shim.cpp ref_pcg_session_*): one stock pcg() call per run()."""

    def __init__(self, a: Csr, lvals: np.ndarray):
        R = ref()
        R.ref_pcg_session_new.restype = C.c_void_p
        R.ref_pcg_session_new.argtypes = [C.c_int64, _i64p, _i32p, _f64p, _f64p]
        R.ref_pcg_session_run.argtypes = [C.c_void_p, _f64p, C.c_double, C.c_int64, _f64p,
                                          C.POINTER(RefReport)]
        R.ref_pcg_session_free.argtypes = [C.c_void_p]
        self.n = a.n
        self.h = R.ref_pcg_session_new(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(lvals))
        if not self.h:
            raise OracleError(1, R.ref_last_error().decode())

    def run(self, b: np.ndarray, rel_tol: float, max_iters: int):
        x = np.empty(self.n, np.float64)
        rep = RefReport()
        ref_check(ref().ref_pcg_session_run(self.h, np.ascontiguousarray(b, np.float64), rel_tol, max_iters, x,
                                            C.byref(rep)))
        return x, {k: getattr(rep, k) for k, _ in RefReport._fields_}

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_pcg_session_free(self.h)
            self.h = None


def ref_pcg_factor(a: Csr, lvals: np.ndarray, b: np.ndarray, rel_tol: float, max_iters: int):
    x = np.empty(a.n, np.float64)
    rep = RefReport()
    ref_check(ref().ref_pcg_factor(a.n, a.rp, a.cols, a.vals, np.ascontiguousarray(lvals),
                                   np.ascontiguousarray(b, np.float64), rel_tol, max_iters, x,
                                   C.byref(rep)))
    return x, {k: getattr(rep, k) for k, _ in RefReport._fields_}
