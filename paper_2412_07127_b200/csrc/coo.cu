// Device COO -> CSR for the reference's constructor pclab_matrix_from_coo
// (capi.cpp:120-137 -> make_coo, sparse.cpp:55-72 + SparseCoo::validate,
// sparse.cpp:25-43): the triplets are sorted by (row, column), then the
// first entry, in sorted order, that is out of bounds or repeats its
// predecessor raises the reference's message. The host sort of round 1
// (one core, 400M triplets for configs[2]) is replaced by:
//   * a bounds/sortedness pass; input already in (row, col) order -- every
//     CSR-ordered generator and Matrix Market file written by this library
//     -- skips the sort;
//   * otherwise a radix sort of the packed key row * n_cols + col (62 bits
//     when every entry is in bounds), or, with an out-of-bounds entry
//     present, two stable passes (column, then row) on the raw signed
//     int64 pairs so the reported entry is the reference's first one;
//   * row pointers by binary search over the sorted rows, int32 columns and
//     the values gathered through the permutation.
#include "core.h"

namespace pclab_b200 {

namespace {

inline unsigned gridn(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

// flags[0]: any out-of-bounds entry, flags[1]: any descent in (row, col)
__global__ void coo_scan_flags(int64_t nnz, int64_t nr, int64_t nc, const int64_t* __restrict__ r,
                               const int64_t* __restrict__ c, int* __restrict__ flags) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const int64_t i = r[k], j = c[k];
    if (i < 0 || i >= nr || j < 0 || j >= nc) flags[0] = 1;
    if (k > 0) {
        const int64_t pi = r[k - 1], pj = c[k - 1];
        if (pi > i || (pi == i && pj >= j)) flags[1] = 1;  // not strictly increasing (dup or descent)
    }
}

__global__ void coo_pack(int64_t nnz, int64_t nc, const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                         unsigned long long* __restrict__ key, int64_t* __restrict__ idx) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    key[k] = static_cast<unsigned long long>(r[k]) * static_cast<unsigned long long>(nc) +
             static_cast<unsigned long long>(c[k]);
    idx[k] = k;
}

// signed int64 -> order-preserving unsigned key
__global__ void coo_signed_key(int64_t nnz, const int64_t* __restrict__ v, const int64_t* __restrict__ perm,
                               unsigned long long* __restrict__ key) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const int64_t x = v[perm ? perm[k] : k];
    key[k] = static_cast<unsigned long long>(x) ^ 0x8000000000000000ULL;
}

__global__ void iota64(int64_t n, int64_t* __restrict__ p) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k < n) p[k] = k;
}

// first sorted position that is out of bounds or equal to its predecessor
__global__ void coo_first_bad(int64_t nnz, int64_t nr, int64_t nc, const int64_t* __restrict__ r,
                              const int64_t* __restrict__ c, const int64_t* __restrict__ perm,
                              unsigned long long* __restrict__ first) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const int64_t s = perm ? perm[k] : k;
    const int64_t i = r[s], j = c[s];
    bool bad = i < 0 || i >= nr || j < 0 || j >= nc;
    if (!bad && k > 0) {
        const int64_t ps = perm ? perm[k - 1] : k - 1;
        bad = r[ps] == i && c[ps] == j;
    }
    if (bad) atomicMin(first, static_cast<unsigned long long>(k));
}

// CSR of the sorted, valid triplets
__global__ void coo_row_ptr(int64_t nr, int64_t nnz, const int64_t* __restrict__ r, const int64_t* __restrict__ perm,
                            int64_t* __restrict__ rp) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nr) return;
    int64_t lo = 0, hi = nnz;  // first sorted position with row >= i
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (r[perm ? perm[mid] : mid] < i) lo = mid + 1; else hi = mid;
    }
    rp[i] = lo;
}

__global__ void coo_gather(int64_t nnz, const int64_t* __restrict__ c, const double* __restrict__ v,
                           const int64_t* __restrict__ perm, int32_t* __restrict__ cols, double* __restrict__ vals) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nnz) return;
    const int64_t s = perm ? perm[k] : k;
    cols[k] = static_cast<int32_t>(c[s]);
    vals[k] = v[s];
}


std::string entry_str(int64_t i, int64_t j) {
    return "(" + std::to_string(i) + ", " + std::to_string(j) + ")";
}

}  // namespace

std::unique_ptr<Matrix> matrix_from_coo_device(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* rows,
                                               const int64_t* cols, const double* vals, cudaStream_t st) {
    if (n_rows < 0 || n_cols < 0) throw FormatError("coo: negative dimensions");
    if (n_cols > INT32_MAX || n_rows > INT32_MAX)
        throw DimensionError("coo: dimensions exceed the int32 column index range");
    DevBuf<int64_t> r(nnz), c(nnz);
    DevBuf<double> v(nnz);
    if (nnz > 0) {
        CK(cudaMemcpyAsync(r.p, rows, sizeof(int64_t) * nnz, cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(c.p, cols, sizeof(int64_t) * nnz, cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(v.p, vals, sizeof(double) * nnz, cudaMemcpyDefault, st));
    }
    DevBuf<int> flags(2);
    CK(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), st));
    if (nnz > 0) {
        coo_scan_flags<<<gridn(nnz, 256), 256, 0, st>>>(nnz, n_rows, n_cols, r.p, c.p, flags.p);
        CK_LAUNCH();
    }
    int hf[2];
    CK(cudaMemcpyAsync(hf, flags.p, sizeof hf, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    DevBuf<int64_t> perm;
    if (hf[0] || hf[1]) {
        perm.alloc(nnz);
        DevBuf<unsigned long long> key(nnz), skey(nnz);
        DevBuf<int64_t> idx(nnz);
        if (!hf[0]) {
            // every entry in bounds: one radix sort on row * n_cols + col
            coo_pack<<<gridn(nnz, 256), 256, 0, st>>>(nnz, n_cols, r.p, c.p, key.p, idx.p);
            CK_LAUNCH();
            int bits = 1;
            while (bits < 64 && (1ULL << bits) < static_cast<unsigned long long>(n_rows) * n_cols) ++bits;
            radix_sort_pairs(key.p, skey.p, idx.p, perm.p, nnz, bits, st);
        } else {
            // raw signed pairs: stable by column, then stable by row
            iota64<<<gridn(nnz, 256), 256, 0, st>>>(nnz, idx.p);
            coo_signed_key<<<gridn(nnz, 256), 256, 0, st>>>(nnz, c.p, nullptr, key.p);
            CK_LAUNCH();
            radix_sort_pairs(key.p, skey.p, idx.p, perm.p, nnz, 64, st);
            coo_signed_key<<<gridn(nnz, 256), 256, 0, st>>>(nnz, r.p, perm.p, key.p);
            CK_LAUNCH();
            radix_sort_pairs(key.p, skey.p, perm.p, idx.p, nnz, 64, st);
            std::swap(perm, idx);
        }
        DevBuf<unsigned long long> first(1);
        CK(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), st));
        coo_first_bad<<<gridn(nnz, 256), 256, 0, st>>>(nnz, n_rows, n_cols, r.p, c.p, perm.p, first.p);
        CK_LAUNCH();
        const unsigned long long fb = dev_read(first.p, st);
        if (fb != ~0ULL) {
            int64_t s = 0, i = 0, j = 0;
            CK(cudaMemcpyAsync(&s, perm.p + fb, sizeof s, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemcpyAsync(&i, r.p + s, sizeof i, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(&j, c.p + s, sizeof j, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (i < 0 || i >= n_rows || j < 0 || j >= n_cols)
                throw FormatError("coo: entry " + entry_str(i, j) + " out of bounds");
            throw FormatError("coo: entries not sorted or duplicate at " + entry_str(i, j));
        }
    }
    auto mat = std::make_unique<Matrix>();
    DevCsr& a = mat->a;
    a.n = n_rows;
    a.nnz = nnz;
    mat->n_cols = n_cols;
    a.rp.alloc(n_rows + 1);
    coo_row_ptr<<<gridn(n_rows + 1, 256), 256, 0, st>>>(n_rows, nnz, r.p, perm.p, a.rp.p);
    CK_LAUNCH();
    a.cols.alloc(nnz);
    a.vals.alloc(nnz);
    if (nnz > 0) {
        coo_gather<<<gridn(nnz, 256), 256, 0, st>>>(nnz, c.p, v.p, perm.p, a.cols.p, a.vals.p);
        CK_LAUNCH();
    }
    matrix_validate(*mat, st);
    return mat;
}

}  // namespace pclab_b200
