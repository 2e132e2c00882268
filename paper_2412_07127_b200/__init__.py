"""B200-native PCG + IC(0) + GNN-correction path (drop-in for the
reference's ``pclab_pcg_solve`` path, /root/reference/proj/include/pclab.h).

Host side mirror of the reference C API over ``libpclab_b200.so``: same
entry-point names, argument meaning, status codes and error messages
(capi.cpp:33-56), plus device-resident extensions. Every numerical step
runs in the hand-written sm_100a kernels under ``csrc/``; if the shared
library is missing this module raises on import of any entry point -- there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCLAB_LIB") or os.path.join(HERE, "libpclab_b200.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_vp = C.c_void_p

KINDS = ("none", "jacobi", "ic0", "nic", "gnnic")


class PclabError(RuntimeError):
    status = 5

    def __init__(self, msg: str):
        super().__init__(msg)


class ArgumentError(PclabError, ValueError):
    status = 1


class FormatError(PclabError):
    status = 2


class NumericError(PclabError, ArithmeticError):
    status = 3


class IoError(PclabError, OSError):
    status = 4


class InternalError(PclabError):
    status = 5


_ERRORS = {1: ArgumentError, 2: FormatError, 3: NumericError, 4: IoError, 5: InternalError}

_lib: Optional[C.CDLL] = None


def lib() -> C.CDLL:
    """The loaded extension; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    sig = {
        "pclab_version": (C.c_char_p, []),
        "pclab_status_name": (C.c_char_p, [C.c_int]),
        "pclab_last_error": (C.c_char_p, []),
        "pclab_matrix_from_coo": (st, [C.c_int64, C.c_int64, C.c_int64, _vp, _vp, _vp, C.POINTER(_vp)]),
        "pclab_matrix_from_csr": (st, [C.c_int64, C.c_int64, _vp, _vp, _vp, C.POINTER(_vp)]),
        "pclab_matrix_gen_poisson": (st, [C.c_int, C.c_int64, C.c_int, C.c_uint64, C.POINTER(_vp)]),
        "pclab_matrix_gen_diffusion": (st, [C.c_int, C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                            C.POINTER(_vp)]),
        "pclab_matrix_gen_elasticity": (st, [C.c_int64, C.c_double, _f64p, C.POINTER(_vp)]),
        "pclab_matrix_shape": (st, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "pclab_matrix_csr": (st, [_vp, _vp, _vp, _vp]),
        "pclab_matrix_device_csr": (st, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
        "pclab_matrix_free": (None, [_vp]),
        "pclab_matrix_read": (st, [C.c_char_p, C.POINTER(_vp)]),
        "pclab_matrix_write": (st, [_vp, C.c_char_p]),
        "pclab_model_init": (st, [C.c_uint64, C.POINTER(_vp)]),
        "pclab_model_load": (st, [C.c_char_p, C.POINTER(_vp)]),
        "pclab_model_save": (st, [_vp, C.c_char_p]),
        "pclab_model_param_count": (st, [_vp, C.POINTER(C.c_uint64)]),
        "pclab_model_from_params": (st, [_f64p, C.c_int64, C.POINTER(_vp)]),
        "pclab_model_params": (st, [_vp, _f64p]),
        "pclab_model_free": (None, [_vp]),
        "pclab_pcg_solve": (st, [_vp, _f64p, C.c_char_p, _vp, C.c_double, C.c_int64, _f64p,
                                 C.POINTER(C.c_void_p)]),
        "pclab_run": (st, [C.c_char_p, C.c_char_p, C.POINTER(C.c_void_p)]),
        "pclab_string_free": (None, [C.c_void_p]),
        "pclab_precond_build": (st, [_vp, C.c_char_p, _vp, C.POINTER(_vp)]),
        "pclab_precond_free": (None, [_vp]),
        "pclab_precond_info": (st, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                    C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
        "pclab_precond_factor": (st, [_vp, _vp]),
        "pclab_precond_levels": (st, [_vp, _vp, _vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
        "pclab_precond_timings": (st, [_vp, _f64p]),
        "pclab_pcg_solve_device": (st, [_vp, _vp, _vp, _vp, C.c_double, C.c_int64, C.c_int, _vp,
                                        C.POINTER(C.c_void_p)]),
        "pclab_spmv_device": (st, [_vp, _vp, _vp, _vp]),
        "pclab_pcg_profile": (st, [_vp, _vp, _vp, _vp, C.c_int64, _f64p]),
        "pclab_precond_layout": (st, [_vp, _i64p]),
        "pclab_set_stream": (None, [_vp]),
        "pclab_matrix_drop_analysis": (st, [_vp]),
        "pclab_launch_count": (C.c_longlong, []),
        "pclab_trsv_device": (st, [_vp, C.c_int, _vp, _vp, _vp]),
        "pclab_uniform_at": (C.c_double, [C.c_uint64, C.c_uint64]),
        "pclab_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
        "pclab_field_normal": (None, [C.c_int64, C.c_uint64, _f64p]),
        "pclab_field_lognormal": (None, [C.c_int64, C.c_uint64, C.c_double, _f64p]),
        "pclab_field_uniform_pm1": (None, [C.c_int64, C.c_uint64, _f64p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def exported_symbols() -> list[str]:
    """Every function include/pclab_b200.h declares (checked by the tests)."""
    import re
    hdr = os.path.join(HERE, "..", "include", "pclab_b200.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(pclab_[a-z0-9_]+)\s*\(", src)))


def _check(status: int):
    if status != 0:
        msg = lib().pclab_last_error().decode()
        raise _ERRORS.get(status, InternalError)(msg)


def _take_string(p: C.c_void_p) -> str:
    if not p.value:
        return ""
    s = C.string_at(p.value).decode()
    lib().pclab_string_free(p)
    return s


def version() -> str:
    return lib().pclab_version().decode()


# ------------------------------------------------------------------ matrix
class Matrix:
    """Device-resident CSR (int64 row_ptr, int32 cols, fp64 values)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pclab_matrix_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def from_coo(cls, n_rows: int, n_cols: int, rows, cols, values) -> "Matrix":
        r = np.ascontiguousarray(rows, np.int64)
        c = np.ascontiguousarray(cols, np.int64)
        v = np.ascontiguousarray(values, np.float64)
        h = _vp()
        _check(lib().pclab_matrix_from_coo(n_rows, n_cols, len(v), r.ctypes.data, c.ctypes.data,
                                           v.ctypes.data, C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, row_ptr, cols, vals) -> "Matrix":
        """Host numpy arrays or device pointers (ints) for all three."""
        h = _vp()
        if isinstance(row_ptr, int):
            raise ArgumentError("use from_csr_device for device pointers")
        rp = np.ascontiguousarray(row_ptr, np.int64)
        c = np.ascontiguousarray(cols, np.int32)
        v = np.ascontiguousarray(vals, np.float64)
        _check(lib().pclab_matrix_from_csr(len(rp) - 1, len(v), rp.ctypes.data, c.ctypes.data,
                                           v.ctypes.data, C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr_device(cls, n: int, nnz: int, rp_ptr: int, cols_ptr: int, vals_ptr: int) -> "Matrix":
        h = _vp()
        _check(lib().pclab_matrix_from_csr(n, nnz, rp_ptr, cols_ptr, vals_ptr, C.byref(h)))
        return cls(h)

    @classmethod
    def gen_poisson(cls, dim: int, m: int, variable_coeff: bool = False, coeff_seed: int = 0) -> "Matrix":
        h = _vp()
        _check(lib().pclab_matrix_gen_poisson(dim, m, int(variable_coeff), coeff_seed, C.byref(h)))
        return cls(h)

    @classmethod
    def gen_diffusion(cls, dim: int, m: int, log10_lo: float, log10_hi: float, seed: int) -> "Matrix":
        h = _vp()
        _check(lib().pclab_matrix_gen_diffusion(dim, m, log10_lo, log10_hi, seed, C.byref(h)))
        return cls(h)

    @classmethod
    def gen_elasticity(cls, m: int, moduli, nu: float = 0.3) -> "Matrix":
        mod = np.ascontiguousarray(moduli, np.float64)
        if mod.size != m ** 3:
            raise ArgumentError("gen_elasticity: need one modulus per element (m^3)")
        h = _vp()
        _check(lib().pclab_matrix_gen_elasticity(m, nu, mod, C.byref(h)))
        return cls(h)

    @classmethod
    def read(cls, path: str) -> "Matrix":
        h = _vp()
        _check(lib().pclab_matrix_read(path.encode(), C.byref(h)))
        return cls(h)

    def write(self, path: str):
        _check(lib().pclab_matrix_write(self._h, path.encode()))

    def shape(self) -> tuple[int, int, int]:
        n, m, z = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().pclab_matrix_shape(self._h, C.byref(n), C.byref(m), C.byref(z)))
        return n.value, m.value, z.value

    @property
    def n(self) -> int:
        return self.shape()[0]

    @property
    def nnz(self) -> int:
        return self.shape()[2]

    def csr(self):
        n, _, nnz = self.shape()
        rp = np.empty(n + 1, np.int64)
        c = np.empty(max(nnz, 1), np.int32)
        v = np.empty(max(nnz, 1), np.float64)
        _check(lib().pclab_matrix_csr(self._h, rp.ctypes.data, c.ctypes.data, v.ctypes.data))
        return rp, c[:nnz], v[:nnz]

    def device_csr(self) -> tuple[int, int, int]:
        a, b, c = _vp(), _vp(), _vp()
        _check(lib().pclab_matrix_device_csr(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value or 0, b.value or 0, c.value or 0

    def drop_analysis(self):
        _check(lib().pclab_matrix_drop_analysis(self._h))

    def spmv_device(self, x_ptr: int, y_ptr: int, stream: int = 0):
        _check(lib().pclab_spmv_device(self._h, x_ptr, y_ptr, stream or None))


# ------------------------------------------------------------------- model
class Model:
    """The 997-parameter message-passing network (gnn.hpp:18-27)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pclab_model_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @classmethod
    def init(cls, seed: int) -> "Model":
        h = _vp()
        _check(lib().pclab_model_init(seed, C.byref(h)))
        return cls(h)

    @classmethod
    def zero(cls) -> "Model":
        p = np.zeros(997)
        p[:9] = 1.0
        return cls.from_params(p)

    @classmethod
    def from_params(cls, params) -> "Model":
        p = np.ascontiguousarray(params, np.float64)
        h = _vp()
        _check(lib().pclab_model_from_params(p, p.size, C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path: str) -> "Model":
        h = _vp()
        _check(lib().pclab_model_load(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path: str):
        _check(lib().pclab_model_save(self._h, path.encode()))

    def param_count(self) -> int:
        c = C.c_uint64()
        _check(lib().pclab_model_param_count(self._h, C.byref(c)))
        return c.value

    def params(self) -> np.ndarray:
        p = np.empty(997)
        _check(lib().pclab_model_params(self._h, p))
        return p


# ---------------------------------------------------------- preconditioner
class Precond:
    """Preconditioner built on the device (precond.cpp:109-168)."""

    def __init__(self, matrix: Matrix, kind: str, model: Optional[Model] = None):
        self.matrix = matrix
        self.kind = kind
        self.model = model
        h = _vp()
        _check(lib().pclab_precond_build(matrix.handle, kind.encode(),
                                         model.handle if model is not None else None, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.pclab_precond_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        nl, bs, lo, up, sg = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_double()
        _check(lib().pclab_precond_info(self._h, C.byref(nl), C.byref(bs), C.byref(lo), C.byref(up),
                                        C.byref(sg)))
        return {"nnz_lower": nl.value, "block_size": bs.value, "block_levels_lower": lo.value,
                "block_levels_upper": up.value, "sigma": sg.value}

    def layout(self) -> dict:
        """Device layout of the sweeps and the product (pclab_precond_layout)."""
        t = np.zeros(8, dtype=np.int64)
        _check(lib().pclab_precond_layout(self._h, t))
        return {"node_blocked": bool(t[0]), "a_node_blocked": bool(t[1]), "block_cols_lower": int(t[2]),
                "block_cols_upper": int(t[3]), "block_cols_a": int(t[4]), "slots_lower": int(t[5]),
                "slots_upper": int(t[6]), "lanes": int(t[7]) % 1000, "slot_records": int(t[7]) >= 1000}

    def factor(self) -> np.ndarray:
        out = np.empty(max(self.info()["nnz_lower"], 1))
        _check(lib().pclab_precond_factor(self._h, out.ctypes.data))
        return out[: self.info()["nnz_lower"]]

    def levels(self):
        n = self.matrix.n
        lo = np.empty(max(n, 1), np.int32)
        up = np.empty(max(n, 1), np.int32)
        a, b = C.c_int32(), C.c_int32()
        _check(lib().pclab_precond_levels(self._h, lo.ctypes.data, up.ctypes.data, C.byref(a), C.byref(b)))
        return lo[:n], up[:n], a.value, b.value

    def timings(self) -> dict:
        t = np.zeros(4)
        _check(lib().pclab_precond_timings(self._h, t))
        return {"analysis_ms": t[0], "ic0_ms": t[1], "gnn_ms": t[2], "total_ms": t[3]}

    def trsv_device(self, upper: bool, b_ptr: int, x_ptr: int, stream: int = 0):
        _check(lib().pclab_trsv_device(self._h, int(upper), b_ptr, x_ptr, stream or None))

    def profile_device(self, b_ptr: int, x_ptr: int, iters: int) -> dict:
        """Per-kernel device ms of the PCG loop (eager iterations)."""
        t = np.zeros(8)
        _check(lib().pclab_pcg_profile(self.matrix.handle, self._h, b_ptr, x_ptr, iters, t))
        return {"spmv_ms": t[0], "axpy_ms": t[1], "sweep_lower_ms": t[2], "sweep_upper_ms": t[3],
                "dot_ms": t[4], "iterations": int(t[5])}

    def solve_device(self, b_ptr: int, x_ptr: int, rel_tol: float = 1e-6, max_iters: int = -1,
                     record_history: bool = False, stream: int = 0) -> dict:
        rep = C.c_void_p()
        _check(lib().pclab_pcg_solve_device(self.matrix.handle, self._h, b_ptr, x_ptr, rel_tol, max_iters,
                                            int(record_history), stream or None, C.byref(rep)))
        return json.loads(_take_string(rep))


# ------------------------------------------------------------------- solve
def pcg_solve(a: Matrix, b, kind: str = "ic0", model: Optional[Model] = None, rel_tol: float = -1.0,
              max_iters: int = -1):
    """pclab_pcg_solve (pclab.h:73): host b in, (x, report dict) out."""
    bb = np.ascontiguousarray(b, np.float64)
    x = np.empty_like(bb)
    rep = C.c_void_p()
    _check(lib().pclab_pcg_solve(a.handle, bb, kind.encode(), model.handle if model else None, rel_tol,
                                 max_iters, x, C.byref(rep)))
    return x, json.loads(_take_string(rep))


def set_stream(stream: int):
    """Run all library work on this cudaStream_t (0 = the library's own)."""
    lib().pclab_set_stream(stream or None)


def launch_count() -> int:
    return int(lib().pclab_launch_count())


def run(command: str, config: Optional[dict] = None) -> dict:
    out = C.c_void_p()
    _check(lib().pclab_run(command.encode(), json.dumps(config or {}).encode(), C.byref(out)))
    return json.loads(_take_string(out))


# ------------------------------------------------------------ seeded inputs
def uniform_at(seed: int, i: int) -> float:
    return lib().pclab_uniform_at(seed, i)


def derive_seed(seed: int, tag: int) -> int:
    return lib().pclab_derive_seed(seed, tag)


def field_normal(n: int, seed: int) -> np.ndarray:
    out = np.empty(n)
    lib().pclab_field_normal(n, seed, out)
    return out


def field_lognormal(n: int, seed: int, sigma: float) -> np.ndarray:
    out = np.empty(n)
    lib().pclab_field_lognormal(n, seed, sigma, out)
    return out


def field_uniform_pm1(n: int, seed: int) -> np.ndarray:
    out = np.empty(n)
    lib().pclab_field_uniform_pm1(n, seed, out)
    return out


from . import workloads  # noqa: E402,F401
