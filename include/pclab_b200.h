#ifndef PCLAB_B200_H
#define PCLAB_B200_H

/* B200-native drop-in for the reference's solve path.
 *
 * Part 1 declares, with identical names, argument meaning, status codes
 * and error messages, the entry points of the reference C API
 * (/root/reference/proj/include/pclab.h) that the PCG + IC(0) + GNN
 * correction path binds; a program linked against libpclab can relink
 * against libpclab_b200.so unchanged. Matrices and models are opaque
 * handles whose payload lives in HBM; host arrays are copied in and out.
 *
 * Part 2 adds device-resident entry points (plain pointers and sizes, no
 * framework types): CSR construction, the device generators of the
 * benchmark systems, the preconditioner object, the device-pointer solve
 * and the individual kernels, used by the parity tests and the benchmark.
 *
 * Index conventions: CSR row pointers int64, column indices int32 (sorted,
 * unique per row), values fp64. All device functions run on `stream`
 * (NULL selects the library's own stream) and are synchronous unless noted.
 */

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------
 * Part 1: the reference interface (pclab.h:16-89)
 * ------------------------------------------------------------------- */

/* pclab.h:16-23 */
typedef enum pclab_status {
    PCLAB_OK = 0,
    PCLAB_ERR_ARGUMENT = 1,
    PCLAB_ERR_FORMAT = 2,
    PCLAB_ERR_NUMERIC = 3,
    PCLAB_ERR_IO = 4,
    PCLAB_ERR_INTERNAL = 5
} pclab_status;

typedef struct pclab_matrix pclab_matrix; /* pclab.h:25, device CSR */
typedef struct pclab_model pclab_model;   /* pclab.h:26, 997 params */

const char* pclab_version(void);                       /* pclab.h:28 */
const char* pclab_status_name(pclab_status status);    /* pclab.h:29 */
const char* pclab_last_error(void);                    /* pclab.h:32 */

/* pclab.h:41-43: triplets, 0-based, sorted and validated like make_coo
 * (sparse.cpp:55-72), then uploaded as CSR. */
pclab_status pclab_matrix_from_coo(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                   const int64_t* rows, const int64_t* cols,
                                   const double* values, pclab_matrix** out);

/* pclab.h:49-50: assembled on the device, values bit-identical to
 * gen_poisson (sparse.cpp:285-305). */
pclab_status pclab_matrix_gen_poisson(int dim, int64_t m, int variable_coeff,
                                      uint64_t coeff_seed, pclab_matrix** out);

/* pclab.h:52-54 */
pclab_status pclab_matrix_shape(const pclab_matrix* a, int64_t* n_rows,
                                int64_t* n_cols, int64_t* nnz);
void pclab_matrix_free(pclab_matrix* a);

/* pclab.h:58-62: GnnModel::init (gnn.cpp:96) and the pclab-gnn JSON
 * checkpoint (gnn.cpp:226-249). */
pclab_status pclab_model_init(uint64_t seed, pclab_model** out);
pclab_status pclab_model_load(const char* path, pclab_model** out);
pclab_status pclab_model_save(const pclab_model* model, const char* path);
pclab_status pclab_model_param_count(const pclab_model* model, uint64_t* out);
void pclab_model_free(pclab_model* model);

/* pclab.h:73-76 (capi.cpp:197-216): host b in, host x out; kind one of
 * none, jacobi, ic0, nic, gnnic; rel_tol <= 0 -> 1e-6; max_iters <= 0 ->
 * 10 n. The report JSON carries the reference's keys plus device phase
 * timings. */
pclab_status pclab_pcg_solve(const pclab_matrix* a, const double* b,
                             const char* kind, const pclab_model* model,
                             double rel_tol, int64_t max_iters, double* x_out,
                             char** report_json_out);

/* pclab.h:37-38: Matrix Market coordinate real general/symmetric. */
pclab_status pclab_matrix_read(const char* path, pclab_matrix** out);
pclab_status pclab_matrix_write(const pclab_matrix* a, const char* path);

/* pclab.h:84-86: the experiment commands (gen/train/eval/...) are outside
 * the accelerated path; this returns PCLAB_ERR_ARGUMENT. */
pclab_status pclab_run(const char* command, const char* config_json,
                       char** summary_json_out);

void pclab_string_free(char* s); /* pclab.h:87 */

/* ---------------------------------------------------------------------
 * Part 2: B200 extensions
 * ------------------------------------------------------------------- */

typedef struct pclab_precond pclab_precond;

/* CSR from host or device memory (cudaMemcpyDefault decides). */
pclab_status pclab_matrix_from_csr(int64_t n, int64_t nnz, const int64_t* row_ptr,
                                   const int32_t* cols, const double* vals,
                                   pclab_matrix** out);
/* Variable-coefficient diffusion (BASELINE config 5): per-cell k =
 * 10^(lo + (hi - lo) u), u = uniform_at(seed, c); lo=-1, hi=1 is
 * gen_poisson's variable family bit for bit. */
pclab_status pclab_matrix_gen_diffusion(int dim, int64_t m, double log10_lo,
                                        double log10_hi, uint64_t seed,
                                        pclab_matrix** out);
/* Q1 hexahedral linear elasticity on m^3 elements of the unit cube,
 * z = 0 face clamped; moduli[m^3] (host) per element, Poisson ratio nu. */
pclab_status pclab_matrix_gen_elasticity(int64_t m, double nu, const double* moduli,
                                         pclab_matrix** out);
/* Copy the CSR back (host or device destinations). */
pclab_status pclab_matrix_csr(const pclab_matrix* a, int64_t* row_ptr, int32_t* cols,
                              double* vals);
/* Discard the cached symbolic analysis so the next preconditioner build
 * redoes it (benchmarks time the full path). */
pclab_status pclab_matrix_drop_analysis(pclab_matrix* a);
/* Device pointers of the CSR (no copy). */
pclab_status pclab_matrix_device_csr(const pclab_matrix* a, const int64_t** row_ptr,
                                     const int32_t** cols, const double** vals);

/* Model from 997 host parameters (layout gnn.hpp:18-27). */
pclab_status pclab_model_from_params(const double* params, int64_t count, pclab_model** out);
pclab_status pclab_model_params(const pclab_model* model, double* out);

/* Preconditioner: symbolic analysis (L/U patterns, level sets, sync-free
 * schedules), IC(0) and/or the GNN correction, all on the device. */
pclab_status pclab_precond_build(pclab_matrix* a, const char* kind,
                                 const pclab_model* model, pclab_precond** out);
void pclab_precond_free(pclab_precond* p);
/* nnz of L (= nnz of the lower triangle of A) and the detected dof block. */
pclab_status pclab_precond_info(const pclab_precond* p, int64_t* nnz_lower,
                                int32_t* block_size, int32_t* levels_lower,
                                int32_t* levels_upper, double* sigma);

/* Device data layout of the sweeps and product (for traffic accounting):
 * out8 = [node-blocked sweeps, node-blocked A, block columns of L, of U,
 * of A, sweep slots lower, upper, lanes per block (+ 1000 when the sweeps
 * run on fixed 128-byte slot records)]. Zeros before analysis. */
pclab_status pclab_precond_layout(const pclab_precond* p, int64_t* out8);
/* Factor values in lower-triangle (row, col) order, as the reference's
 * LowerFactor stores them. Host or device destination. */
pclab_status pclab_precond_factor(const pclab_precond* p, double* out);
/* Per-row level of the forward (L) and backward (L^T) substitution DAGs;
 * returns the level counts. Host or device destinations. */
pclab_status pclab_precond_levels(const pclab_precond* p, int32_t* level_lower,
                                  int32_t* level_upper, int32_t* nlevels_lower,
                                  int32_t* nlevels_upper);
/* Phase timings of the build (ms): analysis, ic0, gnn, total. */
pclab_status pclab_precond_timings(const pclab_precond* p, double* ms4);

/* PCG with a built preconditioner; b and x are DEVICE pointers. A non-NULL
 * `stream` (cudaStream_t) is used for this call only; NULL runs on the
 * library stream (pclab_set_stream). The preconditioner co-owns the matrix
 * analysis its factor lives on, so it stays usable after
 * pclab_matrix_drop_analysis. */
pclab_status pclab_pcg_solve_device(pclab_matrix* a, const pclab_precond* p,
                                    const double* b, double* x, double rel_tol,
                                    int64_t max_iters, int record_history,
                                    void* stream, char** report_json_out);

/* Per-kernel device times of the PCG loop: runs up to max_iters eager
 * iterations (rel_tol 1e-300) with a CUDA event between kernels and writes
 * ms8 = [p-update + A p (+ pAp), axpy + norm, sweep L, sweep L^T, dot,
 * iterations, 0, 0]. */
pclab_status pclab_pcg_profile(pclab_matrix* a, const pclab_precond* p, const double* b,
                               double* x, int64_t max_iters, double* ms8);

/* Run all subsequent library work on `stream` (a cudaStream_t; NULL
 * restores the library's private stream). This is the only sticky stream
 * setter: the `stream` argument of the *_device calls applies to that call
 * alone. */
void pclab_set_stream(void* stream);

/* Kernel launches issued by the library so far (graph nodes included). */
long long pclab_launch_count(void);

/* Individual kernels on device vectors (`stream`: this call only). */
pclab_status pclab_spmv_device(const pclab_matrix* a, const double* x, double* y,
                               void* stream);
/* upper != 0 solves L^T x = b, else L x = b, with p's factor. */
pclab_status pclab_trsv_device(const pclab_precond* p, int upper, const double* b,
                               double* x, void* stream);

/* Seeded host fields used by the benchmark inputs. */
double pclab_uniform_at(uint64_t seed, uint64_t i);
uint64_t pclab_derive_seed(uint64_t seed, uint64_t tag);
void pclab_field_normal(int64_t n, uint64_t seed, double* out);
void pclab_field_lognormal(int64_t n, uint64_t seed, double sigma, double* out);
void pclab_field_uniform_pm1(int64_t n, uint64_t seed, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PCLAB_B200_H */
