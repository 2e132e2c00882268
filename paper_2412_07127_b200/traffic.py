"""Algorithmic HBM bytes of the PCG-loop kernels (the roofline numerators).

Per launch, for the layout the kernels actually run on (Precond.layout()):

* node-blocked sweep (bss_trsv_kernel): every factor value once (8 B), one
  column index per 3x3 block (4 B), one 16-byte slot header per slot, and
  per row the right-hand side, 1/l_ii, the solution write and the re-arm
  write of the other sweep vector (4 x 8 B);
* entry-lane sweep (rec_trsv_kernel / rrs_trsv_kernel, not node-blocked):
  value + column index per entry (12 B), 16 B per slot, the same 32 B per
  row (the fixed 128-byte records of rec_trsv_kernel move 1.04x these bytes:
  profiles/ncu_traffic.json);
* product (k_pupdate + k_spmv_bsr_pap / k_spmv_pap): p <- z + beta p
  (24 B/row), A's values (8 B) + block or entry column indices, row / block
  pointers, p gathered once, q written;
* axpy (x += alpha p, r -= alpha q, ||r||): 48 B/row; dot (r.z): 16 B/row.

With 3x3 node blocks the PCG loop keeps p, y and z padded to 4 doubles per
node (32-byte gathers / polls / publications), so those vectors count
32/3 B per row where they are read or written.

The reference's own format (scalar CSR, int32 columns, int64 row pointers)
is reported beside it as `csr_equivalent_bytes`.
"""
from __future__ import annotations

V4 = 32.0 / 3.0  # bytes per row of a vector padded to 4 doubles per 3-dof node


def padded(lay: dict, bs: int) -> bool:
    """Mirror of pcg_solve's choice (pcg.cu): padded p / y / z for 3x3
    node-blocked A and L."""
    return bool(lay["a_node_blocked"] and lay["node_blocked"] and bs == 3)


def sweep_bytes(lay: dict, nnz_lower: int, n: int, upper: bool, pad: bool = False) -> int:
    slots = lay["slots_upper" if upper else "slots_lower"]
    if lay["node_blocked"]:
        bc = lay["block_cols_upper" if upper else "block_cols_lower"]
        # rhs (r plain / y padded), 1/l_ii, solution write, re-arm write
        per_row = (V4 if upper else 8) + 8 + V4 + 8 if pad else 32
        return int(8 * nnz_lower + 4 * bc + 16 * slots + per_row * n)
    # the backward sweep's re-arm of y is k_axpy's on the unpadded path
    return 12 * nnz_lower + 16 * slots + (24 if upper else 32) * n


def product_bytes(lay: dict, nnz: int, n: int, bs: int, pad: bool = False) -> int:
    if lay["a_node_blocked"]:
        v = V4 if pad else 8
        # p update (z, p read, p written), values, block columns, row and
        # block pointers, p gathered once, q written
        return int(3 * v * n + 8 * nnz + 4 * lay["block_cols_a"] + 8 * n + 8 * (n // bs + 1) + (v + 8) * n)
    return 24 * n + 12 * nnz + 8 * (n + 1) + 16 * n


def spmv_bytes(lay: dict, nnz: int, n: int, bs: int) -> int:
    """Stand-alone y = A x (no p update)."""
    return product_bytes(lay, nnz, n, bs) - 24 * n


def csr_iteration_bytes(nnz: int, nnz_lower: int, n: int) -> int:
    sweep = 12 * nnz_lower + 8 * (n + 1) + 32 * n
    return 2 * sweep + (24 * n + 12 * nnz + 8 * (n + 1) + 16 * n) + 48 * n + 16 * n


def iteration_kernels(pc, n: int, nnz: int, prof: dict) -> dict:
    """{kernel: {ms, bytes, gbs}} for one PCG iteration from a
    Precond.profile_device() result."""
    lay = pc.layout()
    info = pc.info()
    nl, bs = info["nnz_lower"], max(info["block_size"], 1)
    pad = padded(lay, bs)
    lo, up = sweep_bytes(lay, nl, n, False, pad), sweep_bytes(lay, nl, n, True, pad)
    prod = product_bytes(lay, nnz, n, bs, pad)
    kern = {
        "sweep_lower": {"ms": prof["sweep_lower_ms"], "bytes": lo},
        "sweep_upper": {"ms": prof["sweep_upper_ms"], "bytes": up},
        "spmv_p": {"ms": prof["spmv_ms"], "bytes": prod},
    }
    v = V4 if pad else 8
    # p, q, x r/w, r r/w (+ the re-arm of an unpadded y)
    rearm = 8 if (info["nnz_lower"] > 0 and not pad) else 0
    kern["axpy_norm"] = {"ms": prof["axpy_ms"], "bytes": int((v + 40 + rearm) * n)}
    kern["dot"] = {"ms": prof["dot_ms"], "bytes": int((8 + v) * n)}
    for k in kern.values():
        k["gbs"] = k["bytes"] / k["ms"] / 1e6 if k["ms"] > 0 else None
    return kern
