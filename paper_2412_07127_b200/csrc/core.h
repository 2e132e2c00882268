// Host-side objects of the B200 path. Everything large lives in HBM; the
// host keeps only shapes, device pointers and small scalars.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace pclab_b200 {


cudaStream_t lib_stream();
void* dev_alloc(size_t bytes);  // stream-ordered on lib_stream(), pooled
void dev_free(void* p);

// Owning device buffer. Allocation and release are stream-ordered on the
// library stream (cudaMallocAsync from a pool that keeps its memory), so
// temporaries never force a device-wide synchronisation.
template <class T>
struct DevBuf {
    T* p = nullptr;
    int64_t n = 0;
    DevBuf() = default;
    explicit DevBuf(int64_t count) { alloc(count); }
    void alloc(int64_t count) {
        reset();
        n = count;
        if (count > 0) p = static_cast<T*>(dev_alloc(sizeof(T) * static_cast<size_t>(count)));
    }
    void reset() {
        if (p) dev_free(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { reset(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    size_t bytes() const { return sizeof(T) * static_cast<size_t>(n); }
};

// CSR in HBM: int64 row pointers, int32 column indices (strictly
// increasing per row), fp64 values.
struct DevCsr {
    int64_t n = 0, nnz = 0;
    DevBuf<int64_t> rp;
    DevBuf<int32_t> cols;
    DevBuf<double> vals;
};

// Dependency schedule of a triangular sweep over blocks of `bs`
// consecutive rows: blocks sorted by (level, index) and cut into warp
// items of at most `per_item` blocks of one level.
struct Schedule {
    int bs = 1;
    int lanes = 32;     // lanes per block inside a warp (32 / per_item)
    int per_item = 1;   // blocks per warp item
    int64_t nblocks = 0;
    int32_t nlevels = 0;
    int64_t nitems = 0;
    DevBuf<int32_t> level;       // [nblocks] level of each block
    DevBuf<int32_t> crit;        // [nblocks] row polled first (-1: no dependency; filled if need_crit)
    bool need_crit = true;
    DevBuf<int32_t> order;       // [nblocks] blocks in schedule order
    DevBuf<int64_t> item_first;  // [nitems] first position in `order`
    DevBuf<int32_t> item_cnt;    // [nitems] blocks in the item
    DevBuf<int32_t> slots;       // [nitems * per_item] block per lane group, -1 idle
    DevBuf<int32_t> slot_rp;     // [nitems * per_item * 4] 16-byte slot records {block (-1 idle),
                                 //  first row pointer, first block column, row lengths 10 bits each}
    int64_t max_level_width = 0;
    // item-ordered value stream of the node-blocked sweep (bss.cu)
    bool bss = false;
    int64_t bss_nvals = 0;
    DevBuf<int4> bss_hdr;     // [slots] {block, neighbours, value offset, column offset}
    DevBuf<int32_t> bss_col;  // neighbour block ids, slot after slot
    // scalar blocks of 2 rows with <= 8 off-block entries: fixed 128-byte slot records (rec_trsv_kernel)
    bool rec = false;
};

// Block-column view of a node-blocked CSR matrix (Analysis::bsr): block
// row b's off-block neighbour blocks are bcol[bp[b] .. bp[b + 1]), each
// stored as its first column (a multiple of bs). One index per bs x bs
// block instead of one per entry: the sweeps and the product read a ninth
// of the column indices.
struct BlockCols {
    DevBuf<int64_t> bp;    // [nblocks + 1]
    DevBuf<int32_t> bcol;  // [bp[nblocks]]
};

// Symbolic analysis of a structurally symmetric matrix (the reference's
// lower_triangle + csr_transpose, sparse.cpp:137/189, done once on the
// device): L pattern with A's lower values, U = L^T pattern, the slot map
// U -> L, and the forward/backward schedules.
struct Analysis {
    DevCsr lower;            // pattern of L, values = lower triangle of A
    DevCsr upper;            // pattern of U = L^T (values unused)
    DevBuf<int64_t> u2l;     // [nnz(U)] position in L of each U entry
    int bs = 1;              // detected dof block size (3 for elasticity)
    bool bsr = false;        // off-block pattern made of whole bs x bs blocks
    bool rr = false;         // not node-blocked: round-robin entry-lane sweep (rr_trsv_kernel)
    BlockCols lbc, ubc;      // block columns of L / U (bsr)
    bool a_bsr = false;      // A itself node-blocked: product through abc
    BlockCols abc;
    Schedule row_lo;         // bs = 1, one row per warp (IC(0))
    Schedule blk_lo, blk_up; // bs-blocked sweeps (triangular solves)
    Schedule rowlev_up;      // bs = 1 upper levels (reported only)
    double ms = 0.0;         // wall time of the analysis (CUDA events)
    uint64_t id = 0;         // unique per analysis (IC(0) mask cache key)
};

struct Matrix {
    DevCsr a;                  // a.n rows
    int64_t n_cols = 0;        // columns (the reference's SparseCoo::n_cols; square for every solve)
    DevBuf<int64_t> diag_pos;  // [n] position of a_ii in row i, -1 if absent
    bool symmetric_known = false, symmetric = false;
    int64_t missing_diag_row = -1;  // first row without a diagonal
    std::shared_ptr<Analysis> an;  // co-owned by the preconditioners built on it
};

struct Model {
    std::vector<double> params;  // 997, layout of gnn.hpp:18-27
};

enum class Kind { None = 0, Jacobi = 1, IC0 = 2, NIC = 3, GnnIC = 4 };
const char* kind_name(Kind k);
Kind parse_kind(const std::string& s);

struct Precond {
    Kind kind = Kind::None;
    const Matrix* a = nullptr;  // the matrix it was built from (identity only; never dereferenced)
    std::shared_ptr<Analysis> an;  // factor kinds: the analysis its factor lives on
    DevBuf<double> lvals;       // factor values on L's pattern
    DevBuf<double> uvals;       // same values on U's pattern (gathered)
    DevBuf<double> invd;        // 1 / l_ii (both sweeps)
    DevBuf<double> bss_lo, bss_up;               // item-ordered sweep values (bss.cu)
    DevBuf<double> rec_lo, rec_up;               // 128-byte slot records (bss.cu, Schedule::rec)
    DevBuf<double> diag;        // Jacobi payload
    double sigma = 1.0;         // GNN edge scale
    int ic0_attempts = 0;
    double ms_analysis = 0, ms_ic0 = 0, ms_gnn = 0, ms_total = 0;
};

struct SolveReport {
    int64_t iterations = 0;
    bool converged = false;
    double final_rel_residual = 0, true_rel_residual = 0;
    bool residual_mismatch = false;
    double p_time = 0, cg_time = 0, total_time = 0, tri_solve_time_per_iter = 0;
    double analysis_time = 0, ic0_time = 0, gnn_time = 0;
    std::vector<double> residual_history;
    std::string to_json() const;
};

// ----------------------------------------------------------- entry points
cudaStream_t lib_stream();

// one value from device memory (synchronises the stream)
template <class T>
T dev_read(const T* d, cudaStream_t st) {
    T v;
    CK(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return v;
}
// devsort.cu: exclusive prefix sum in place; stable LSD radix sort of
// (key, value) pairs on the low `bits` bits of unsigned keys
void scan_inplace(int64_t* p, int64_t n, cudaStream_t st);
template <class K, class V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int bits, cudaStream_t st);

// matrices (gen.cu / capi.cpp)
std::unique_ptr<Matrix> matrix_from_csr_host(int64_t n, const int64_t* rp, const int32_t* cols,
                                             const double* vals, cudaStream_t st);
// rp / cols / vals may be host or device pointers; row_ptr is checked on
// the device (rp[0] = 0, monotone, rp[n] = nnz) before any column is read
std::unique_ptr<Matrix> matrix_from_csr_device(int64_t n, int64_t nnz, const int64_t* rp,
                                               const int32_t* cols, const double* vals,
                                               cudaStream_t st, int64_t n_cols = -1);
// coo.cu: make_coo (sparse.cpp:55-72) on the device; host or device pointers
std::unique_ptr<Matrix> matrix_from_coo_device(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                                               const int64_t* cols, const double* vals, cudaStream_t st);
std::unique_ptr<Matrix> gen_poisson_device(int dim, int64_t m, const double* cell_k_host,
                                           cudaStream_t st);
std::unique_ptr<Matrix> gen_elasticity_device(int64_t m, double nu, const double* moduli_host,
                                              cudaStream_t st);
void matrix_validate(Matrix& a, cudaStream_t st);  // diag positions, row order
bool matrix_symmetric(Matrix& a, cudaStream_t st);

// analysis.cu
Analysis& ensure_analysis(Matrix& a, cudaStream_t st);
// block-column view; mode 0: L (diagonal last), 1: U (diagonal first), 2: A
void build_block_cols(const DevCsr& M, int bs, int mode, BlockCols& bc, cudaStream_t st);
void compute_levels(const DevCsr& pred, const DevCsr& succ, int bs, bool upper, Schedule& s,
                    cudaStream_t st, const BlockCols* pbc = nullptr, const BlockCols* sbc = nullptr);

// ic0.cu: factor values on an.lower's pattern; returns shift attempts
int ic0_factor(const Matrix& a, const Analysis& an, double* out, cudaStream_t st);

// gnn.cu: GNN forward over the lower-triangle graph; out aligned with L.
void gnn_forward(const Matrix& a, const Analysis& an, const Model& m, double* out,
                 double* sigma_out, cudaStream_t st);

// kernels.cu
void spmv(const Matrix& a, const double* x, double* y, cudaStream_t st);
struct Precond;
void trsv(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, cudaStream_t st);
void launch_trsv(const Analysis& an, const double* vals, const double* invd, bool upper, const double* b,
                 double* x, double* reset, const int* done, unsigned* ctr, cudaStream_t st, bool pad = false);
// bss.cu: item-ordered value streams of the node-blocked sweeps
void build_bss(Analysis& an, cudaStream_t st);
void fill_bss(const Analysis& an, Precond& p, cudaStream_t st);
bool launch_bss(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                const int* done, cudaStream_t st, bool pad);
void launch_sweep(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                  const int* done, unsigned* ctr, cudaStream_t st, bool pad);
void reciprocal_diag(const Analysis& an, const double* lvals, double* invd, cudaStream_t st);
int spmv_lanes(const Matrix& a);
void gather_upper(const Analysis& an, const double* lvals, double* uvals, cudaStream_t st);
void fill_pending(double* p, int64_t n, cudaStream_t st);

// precond + pcg (pcg.cu)
std::unique_ptr<Precond> build_precond(Matrix& a, Kind k, const Model* m, cudaStream_t st);
SolveReport pcg_solve(Matrix& a, const Precond& p, const double* b_dev, double* x_dev,
                      double rel_tol, int64_t max_iters, bool record_history,
                      cudaStream_t st, double* prof_ms = nullptr);

// host helpers (host.cpp)
void element_stiffness(double h, double nu, double* ke);
uint64_t derive_seed(uint64_t seed, uint64_t tag);
double uniform_at(uint64_t seed, uint64_t i);
double normal_at(uint64_t seed, uint64_t i);
std::vector<double> gnn_init_params(uint64_t seed);

}  // namespace pclab_b200
