/* CPU oracle for the PCG + IC(0) + GNN-correction hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This is a plain-C restatement of the
 * reference's algorithm (reference: /root/reference/proj/src, cited per
 * function in pclab_oracle.c). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker or the timed CPU baseline. The product library
 * (paper_2412_07127_b200/libpclab_b200.so) never links or calls it.
 *
 * Pinning: the restatement is checked bit-for-bit against the reference
 * compiled from its own sources (oracle/_ref/libpclab_ref.so, built by
 * oracle/Makefile) and against the committed fixtures in tests/golden/.
 * The Q1-elasticity and 10^u-diffusion generators are NOT in the
 * reference (its generator is gen_poisson only); they are this repo's own
 * specification of BASELINE.json configs 1-4 and are "parity unpinned"
 * against the reference: the product's device assembly is checked against
 * them bit-for-bit, and everything downstream of assembly (IC(0), GNN,
 * PCG) is pinned against the reference by feeding the same CSR into
 * oracle/_ref.
 *
 * Storage: CSR with int64 row pointers and int32 column indices, columns
 * strictly increasing within each row, fp64 values. */
#ifndef PCLAB_ORACLE_H
#define PCLAB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_ERR_ARGUMENT = 1, OR_ERR_FORMAT = 2, OR_ERR_NUMERIC = 3,
       /* or_pcg: p^T A p <= 0 (krylov.cpp:151-154); rep->iterations = the failing k */
       OR_ERR_CURVATURE = 6 };

/* ---- counter-based RNG (reference rng.hpp) ---- */
uint64_t or_mix64(uint64_t x);
uint64_t or_bits_at(uint64_t seed, uint64_t i);
double or_uniform_at(uint64_t seed, uint64_t i);
uint64_t or_derive_seed(uint64_t seed, uint64_t tag);
double or_normal_at(uint64_t seed, uint64_t i);

/* ---- generators ---- */
int64_t or_poisson_n(int dim, int64_t m);
int64_t or_poisson_nnz(int dim, int64_t m);
/* k_log10_lo == k_log10_hi == 0 selects the constant stencil (k = 1);
 * otherwise k_c = 10^(lo + (hi - lo) * u_c), u_c = uniform_at(seed, c). */
void or_cell_coeffs(int64_t n, uint64_t seed, double lo, double hi, double* k);
int or_gen_poisson(int dim, int64_t m, const double* cell_k, int64_t* row_ptr,
                   int32_t* cols, double* vals);
void or_element_stiffness(double h, double nu, double* ke /* 24x24 */);
void or_elasticity_dims(int64_t m, int64_t* n, int64_t* nnz);
void or_lognormal_field(int64_t n, uint64_t seed, double sigma, double* out);
void or_normal_field(int64_t n, uint64_t seed, double* out);
void or_uniform_pm1_field(int64_t n, uint64_t seed, double* out);
int or_gen_elasticity(int64_t m, double nu, const double* moduli,
                      int64_t* row_ptr, int32_t* cols, double* vals);

/* ---- structure ---- */
int64_t or_lower_nnz(int64_t n, const int64_t* rp, const int32_t* cols);
void or_lower(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
              int64_t* lrp, int32_t* lcols, double* lvals);
/* U = L^T in CSR; u2l[k] = position in L of U entry k. */
void or_transpose(int64_t n, const int64_t* lrp, const int32_t* lcols,
                  const double* lvals, int64_t* urp, int32_t* ucols, double* uvals,
                  int64_t* u2l);
int64_t or_levels_lower(int64_t n, const int64_t* lrp, const int32_t* lcols,
                        int32_t* level);
int64_t or_levels_upper(int64_t n, const int64_t* urp, const int32_t* ucols,
                        int32_t* level);
/* Block-row DAG for consecutive blocks of bs rows (n % bs == 0). */
int64_t or_block_levels_lower(int64_t n, int bs, const int64_t* lrp,
                              const int32_t* lcols, int32_t* level);
int64_t or_block_levels_upper(int64_t n, int bs, const int64_t* urp,
                              const int32_t* ucols, int32_t* level);

/* ---- kernels ---- */
void or_csr_matvec(int64_t n, const int64_t* rp, const int32_t* cols,
                   const double* vals, const double* x, double* y);
int or_trsv_lower(int64_t n, const int64_t* lrp, const int32_t* lcols,
                  const double* lvals, const double* b, double* x, int64_t* bad_row);
int or_trsv_upper(int64_t n, const int64_t* urp, const int32_t* ucols,
                  const double* uvals, const double* b, double* x, int64_t* bad_row);

/* ---- preconditioners ---- */
/* IC(0) on the lower pattern (values = lower triangle of A). Returns
 * OR_OK, OR_ERR_NUMERIC (breakdown after shifts, *fail_row set) or
 * OR_ERR_FORMAT (missing diagonal, *fail_row set). *attempts = shifts used. */
int or_ic0(int64_t n, const int64_t* lrp, const int32_t* lcols, const double* avals,
           double* out, int64_t* fail_row, int* attempts);

enum { OR_NODE_FEATURES = 9, OR_HIDDEN = 8, OR_BLOCKS = 3, OR_PARAMS = 997 };
void or_node_features(int64_t n, const int64_t* rp, const int32_t* cols,
                      const double* vals, double* feat);
/* scale_by_std on the lower values; returns sigma (1 when constant). */
double or_scale_by_std(int64_t nnz, const double* v, double* out);
void or_gnn_init(uint64_t seed, double* params);
void or_gnn_zero(double* params);
/* Forward pass over the lower-triangle graph of full symmetric A.
 * out[k] aligned with the lower CSR order; *sigma receives the edge scale.
 * Returns OR_OK or OR_ERR_NUMERIC with *bad_block = 1-based block. */
int or_gnn_forward(int64_t n, const int64_t* rp, const int32_t* cols,
                   const double* vals, const double* params, double* out,
                   double* sigma, int* bad_block);

/* ---- solver ---- */
enum { OR_PC_NONE = 0, OR_PC_JACOBI = 1, OR_PC_FACTOR = 2 };
typedef struct {
    int64_t iterations;
    int converged;
    double final_rel_residual;
    double true_rel_residual;
    int residual_mismatch;
} or_report;
/* kind OR_PC_FACTOR uses (lrp, lcols, lvals) as L; OR_PC_JACOBI uses the
 * diagonal of A. history (optional) receives iterations+1 values. */
int or_pcg(int64_t n, const int64_t* rp, const int32_t* cols, const double* vals,
           const double* b, int kind, const int64_t* lrp, const int32_t* lcols,
           const double* lvals, double rel_tol, int64_t max_iters, double* x,
           or_report* rep, double* history);

#ifdef __cplusplus
}
#endif
#endif
