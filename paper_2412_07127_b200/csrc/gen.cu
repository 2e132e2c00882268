// Device-resident CSR assembly and validation.
//
// The Poisson/diffusion assembly restates assemble_poisson
// (reference src/sparse.cpp:232-282) row by row on the device, with the
// diagonal accumulated in the reference's order and every operation
// explicitly rounded (__dadd_rn/__dmul_rn/__ddiv_rn: no FMA contraction), so
// the values are bit-identical to the reference's. The Q1 elasticity
// assembly has no reference counterpart; its order is specified by
// oracle/pclab_oracle.c (or_gen_elasticity) and matched bit for bit.

#include "core.h"

namespace pclab_b200 {

namespace {

__constant__ double c_ke[576];

__device__ __forceinline__ double face_k(double klo, double khi) {
    // 2.0 * klo * khi / (klo + khi), evaluated left to right
    return __ddiv_rn(__dmul_rn(__dmul_rn(2.0, klo), khi), __dadd_rn(klo, khi));
}

__device__ __forceinline__ double kval(const double* k, int64_t c) { return k ? k[c] : 1.0; }

template <bool FILL>
__global__ void poisson_rows(int dim, int64_t m, const double* __restrict__ k,
                             int64_t* __restrict__ rp, int32_t* __restrict__ cols,
                             double* __restrict__ vals, int64_t n) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c >= n) return;
    const int64_t crd[3] = {c % m, (c / m) % m, dim == 3 ? c / (m * m) : 0};
    const int64_t st[3] = {1, m, m * m};
    if (!FILL) {
        int cnt = 1;
        for (int ax = 0; ax < dim; ++ax) cnt += (crd[ax] > 0) + (crd[ax] + 1 < m);
        rp[c] = cnt;
        return;
    }
    const double kc = kval(k, c);
    double diag = 0.0;
    for (int ax = dim - 1; ax >= 0; --ax)
        if (crd[ax] > 0) diag = __dadd_rn(diag, face_k(kval(k, c - st[ax]), kc));
    for (int ax = 0; ax < dim; ++ax) {
        if (crd[ax] == 0) diag = __dadd_rn(diag, kc);
        if (crd[ax] + 1 < m)
            diag = __dadd_rn(diag, face_k(kc, kval(k, c + st[ax])));
        else
            diag = __dadd_rn(diag, kc);
    }
    int64_t pos = rp[c];
    for (int ax = dim - 1; ax >= 0; --ax)
        if (crd[ax] > 0) {
            cols[pos] = static_cast<int32_t>(c - st[ax]);
            vals[pos++] = -face_k(kval(k, c - st[ax]), kc);
        }
    cols[pos] = static_cast<int32_t>(c);
    vals[pos++] = diag;
    for (int ax = 0; ax < dim; ++ax)
        if (crd[ax] + 1 < m) {
            cols[pos] = static_cast<int32_t>(c + st[ax]);
            vals[pos++] = -face_k(kc, kval(k, c + st[ax]));
        }
}

// One thread per row of the clamped Q1 system; see or_gen_elasticity.
template <bool FILL>
__global__ void elasticity_rows(int64_t m, const double* __restrict__ moduli,
                                int64_t* __restrict__ rp, int32_t* __restrict__ cols,
                                double* __restrict__ vals, int64_t n) {
    const int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (row >= n) return;
    const int64_t p1 = m + 1;
    const int64_t off = 3 * p1 * p1;
    const int64_t node = row / 3 + p1 * p1;
    const int c = static_cast<int>(row % 3);
    const int64_t ix = node % p1, iy = (node / p1) % p1, iz = node / (p1 * p1);
    if (!FILL) {
        const int cx = (ix > 0) + 1 + (ix + 1 < p1);
        const int cy = (iy > 0) + 1 + (iy + 1 < p1);
        const int cz = (iz > 1) + 1 + (iz + 1 < p1);
        rp[row] = 3 * cx * cy * cz;
        return;
    }
    int64_t pos = rp[row];
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int64_t qx = ix + dx, qy = iy + dy, qz = iz + dz;
                if (qx < 0 || qx >= p1 || qy < 0 || qy >= p1 || qz < 1 || qz >= p1) continue;
                const int64_t q = qx + p1 * qy + p1 * p1 * qz;
                for (int d = 0; d < 3; ++d) {
                    double acc = 0.0;
                    for (int64_t ez = iz - 1; ez <= iz; ++ez) {
                        if (ez < 0 || ez >= m || ez < qz - 1 || ez > qz) continue;
                        for (int64_t ey = iy - 1; ey <= iy; ++ey) {
                            if (ey < 0 || ey >= m || ey < qy - 1 || ey > qy) continue;
                            for (int64_t ex = ix - 1; ex <= ix; ++ex) {
                                if (ex < 0 || ex >= m || ex < qx - 1 || ex > qx) continue;
                                const int64_t e = ex + m * ey + m * m * ez;
                                const int a = static_cast<int>((ix - ex) + 2 * (iy - ey) + 4 * (iz - ez));
                                const int b = static_cast<int>((qx - ex) + 2 * (qy - ey) + 4 * (qz - ez));
                                acc = __dadd_rn(acc, __dmul_rn(moduli[e], c_ke[(3 * a + c) * 24 + 3 * b + d]));
                            }
                        }
                    }
                    cols[pos] = static_cast<int32_t>(3 * q + d - off);
                    vals[pos++] = acc;
                }
            }
}

// Row structure checks (SparseCoo::validate, sparse.cpp:25-43, on CSR)
// plus the diagonal position of every row.
// row_ptr shape (checked before any column is read): rp[0] = 0, monotone,
// rp[n] = nnz; the first offending row (or n for a bad end) lands in *bad
__global__ void rowptr_check(int64_t n, int64_t nnz, const int64_t* __restrict__ rp,
                             unsigned long long* __restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > n) return;
    bool ok;
    if (i == 0) ok = rp[0] == 0;
    else ok = rp[i] >= rp[i - 1] && rp[i] <= nnz;
    if (i == n) ok = ok && rp[n] == nnz;
    if (!ok) atomicMin(bad, static_cast<unsigned long long>(i));
}

__global__ void validate_rows(int64_t n, int64_t n_cols, const int64_t* __restrict__ rp,
                              const int32_t* __restrict__ cols, int64_t* __restrict__ diag_pos,
                              unsigned long long* __restrict__ bad_row,
                              unsigned long long* __restrict__ missing_diag) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t b = rp[i], e = rp[i + 1];
    int64_t dp = -1;
    bool ok = e >= b;
    for (int64_t k = b; ok && k < e; ++k) {
        const int32_t j = cols[k];
        if (j < 0 || j >= n_cols || (k > b && cols[k - 1] >= j)) ok = false;
        if (j == i) dp = k;
    }
    diag_pos[i] = dp;
    if (!ok) atomicMin(bad_row, static_cast<unsigned long long>(i));
    if (dp < 0) atomicMin(missing_diag, static_cast<unsigned long long>(i));
}

// is_symmetric (sparse.cpp:178-187): every (i,j,v), i != j, has (j,i,v).
__global__ void symmetry_check(int64_t n, const int64_t* __restrict__ rp,
                               const int32_t* __restrict__ cols, const double* __restrict__ vals,
                               int* __restrict__ asym) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        const int32_t j = cols[k];
        if (j == i) continue;
        int64_t lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cols[mid] < i) lo = mid + 1; else hi = mid;
        }
        const bool found = lo < rp[j + 1] && cols[lo] == i;
        if (!found || __double_as_longlong(vals[lo]) != __double_as_longlong(vals[k])) {
            // +0.0 / -0.0 compare equal in the reference (operator!=)
            if (!(found && vals[lo] == vals[k])) *asym = 1;
        }
    }
}


int64_t read_i64(const int64_t* d, cudaStream_t st) {
    int64_t v;
    CK(cudaMemcpyAsync(&v, d, sizeof v, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return v;
}

}  // namespace

void matrix_validate(Matrix& a, cudaStream_t st) {
    const int64_t n = a.a.n;
    a.diag_pos.alloc(n);
    DevBuf<unsigned long long> flags(2);
    const unsigned long long init[2] = {~0ULL, ~0ULL};
    CK(cudaMemcpyAsync(flags.p, init, sizeof init, cudaMemcpyHostToDevice, st));
    if (n > 0) {
        validate_rows<<<(n + 255) / 256, 256, 0, st>>>(n, a.n_cols, a.a.rp.p, a.a.cols.p, a.diag_pos.p,
                                                       flags.p, flags.p + 1);
        CK_LAUNCH();
    }
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, flags.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h[0] != ~0ULL)
        throw FormatError("csr: row " + std::to_string(h[0]) +
                          " has unsorted, duplicate or out-of-range columns");
    a.missing_diag_row = h[1] == ~0ULL ? -1 : static_cast<int64_t>(h[1]);
}

bool matrix_symmetric(Matrix& a, cudaStream_t st) {
    if (a.symmetric_known) return a.symmetric;
    DevBuf<int> flag(1);
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
    if (a.a.n > 0) {
        symmetry_check<<<(a.a.n + 255) / 256, 256, 0, st>>>(a.a.n, a.a.rp.p, a.a.cols.p,
                                                           a.a.vals.p, flag.p);
        CK_LAUNCH();
    }
    int h = 0;
    CK(cudaMemcpyAsync(&h, flag.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    a.symmetric_known = true;
    a.symmetric = h == 0;
    return a.symmetric;
}

std::unique_ptr<Matrix> gen_poisson_device(int dim, int64_t m, const double* cell_k_host,
                                           cudaStream_t st) {
    if (dim != 2 && dim != 3) throw DimensionError("gen_poisson: dim must be 2 or 3");
    if (m < 1) throw DimensionError("gen_poisson: m must be >= 1");
    const int64_t n = dim == 2 ? m * m : m * m * m;
    auto mat = std::make_unique<Matrix>();
    DevCsr& a = mat->a;
    a.n = n;
    mat->n_cols = n;
    a.rp.alloc(n + 1);
    DevBuf<double> k;
    if (cell_k_host) {
        k.alloc(n);
        CK(cudaMemcpyAsync(k.p, cell_k_host, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    }
    const int T = 256;
    const unsigned g = static_cast<unsigned>((n + T - 1) / T);
    poisson_rows<false><<<g, T, 0, st>>>(dim, m, k.p, a.rp.p, nullptr, nullptr, n);
    CK_LAUNCH();
    CK(cudaMemsetAsync(a.rp.p + n, 0, sizeof(int64_t), st));
    scan_inplace(a.rp.p, n + 1, st);
    a.nnz = read_i64(a.rp.p + n, st);
    a.cols.alloc(a.nnz);
    a.vals.alloc(a.nnz);
    poisson_rows<true><<<g, T, 0, st>>>(dim, m, k.p, a.rp.p, a.cols.p, a.vals.p, n);
    CK_LAUNCH();
    matrix_validate(*mat, st);
    mat->symmetric_known = mat->symmetric = true;  // symmetric by construction
    return mat;
}

std::unique_ptr<Matrix> gen_elasticity_device(int64_t m, double nu, const double* moduli_host,
                                              cudaStream_t st) {
    if (m < 1) throw DimensionError("gen_elasticity: m must be >= 1");
    const int64_t p1 = m + 1;
    const int64_t n = 3 * p1 * p1 * m;
    double ke[576];
    element_stiffness(1.0 / static_cast<double>(m), nu, ke);
    CK(cudaMemcpyToSymbolAsync(c_ke, ke, sizeof ke, 0, cudaMemcpyHostToDevice, st));
    DevBuf<double> mod(m * m * m);
    CK(cudaMemcpyAsync(mod.p, moduli_host, sizeof(double) * m * m * m, cudaMemcpyHostToDevice, st));
    auto mat = std::make_unique<Matrix>();
    DevCsr& a = mat->a;
    a.n = n;
    mat->n_cols = n;
    a.rp.alloc(n + 1);
    const int T = 128;
    const unsigned g = static_cast<unsigned>((n + T - 1) / T);
    elasticity_rows<false><<<g, T, 0, st>>>(m, mod.p, a.rp.p, nullptr, nullptr, n);
    CK_LAUNCH();
    CK(cudaMemsetAsync(a.rp.p + n, 0, sizeof(int64_t), st));
    scan_inplace(a.rp.p, n + 1, st);
    a.nnz = read_i64(a.rp.p + n, st);
    a.cols.alloc(a.nnz);
    a.vals.alloc(a.nnz);
    elasticity_rows<true><<<g, T, 0, st>>>(m, mod.p, a.rp.p, a.cols.p, a.vals.p, n);
    CK_LAUNCH();
    matrix_validate(*mat, st);
    mat->symmetric_known = mat->symmetric = true;  // Ke mirrored: exactly symmetric
    return mat;
}

std::unique_ptr<Matrix> matrix_from_csr_device(int64_t n, int64_t nnz, const int64_t* rp,
                                               const int32_t* cols, const double* vals,
                                               cudaStream_t st, int64_t n_cols) {
    if (n < 0 || nnz < 0) throw FormatError("csr: negative dimension");
    if (n_cols < 0) n_cols = n;
    if (n > INT32_MAX || n_cols > INT32_MAX)
        throw FormatError("csr: dimensions exceed the int32 column index range");
    auto mat = std::make_unique<Matrix>();
    DevCsr& a = mat->a;
    a.n = n;
    a.nnz = nnz;
    mat->n_cols = n_cols;
    a.rp.alloc(n + 1);
    CK(cudaMemcpyAsync(a.rp.p, rp, sizeof(int64_t) * (n + 1), cudaMemcpyDefault, st));
    {
        DevBuf<unsigned long long> bad(1);
        CK(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
        rowptr_check<<<static_cast<unsigned>((n + 1 + 255) / 256), 256, 0, st>>>(n, nnz, a.rp.p, bad.p);
        CK_LAUNCH();
        const unsigned long long b = read_i64(reinterpret_cast<const int64_t*>(bad.p), st);
        if (b != ~0ULL) {
            if (b == 0) throw FormatError("csr: row_ptr[0] != 0");
            if (static_cast<int64_t>(b) == n) throw FormatError("csr: row_ptr[n] != nnz");
            throw FormatError("csr: row_ptr not monotone at row " + std::to_string(b - 1));
        }
    }
    a.cols.alloc(nnz);
    a.vals.alloc(nnz);
    if (nnz > 0) {
        CK(cudaMemcpyAsync(a.cols.p, cols, sizeof(int32_t) * nnz, cudaMemcpyDefault, st));
        CK(cudaMemcpyAsync(a.vals.p, vals, sizeof(double) * nnz, cudaMemcpyDefault, st));
    }
    matrix_validate(*mat, st);
    return mat;
}

std::unique_ptr<Matrix> matrix_from_csr_host(int64_t n, const int64_t* rp, const int32_t* cols,
                                             const double* vals, cudaStream_t st) {
    if (n < 0) throw FormatError("csr: negative dimension");
    if (rp[0] != 0) throw FormatError("csr: row_ptr[0] != 0");
    for (int64_t i = 0; i < n; ++i)
        if (rp[i + 1] < rp[i]) throw FormatError("csr: row_ptr not monotone at row " + std::to_string(i));
    return matrix_from_csr_device(n, rp[n], rp, cols, vals, st);
}

}  // namespace pclab_b200
