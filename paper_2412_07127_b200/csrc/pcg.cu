// Preconditioner construction and the PCG loop (reference: ic0 /
// nic_predict / gnn_ic_predict src/precond.cpp:109-168, pcg
// src/krylov.cpp:114-190).
//
// One PCG iteration is five kernels, all resident-data, no host round trip:
//   1. spmv_p : p <- z + beta p (on the fly, double-buffered), q = A p,
//               pAp (deterministic two-pass), alpha = rz / pAp
//   2. axpy   : x += alpha p, r -= alpha q, ||r|| -> convergence flag
//   3. sweep L: y = L^-1 r   (sync-free; also re-arms z)
//   4. sweep U: z = L^-T y   (sync-free; also re-arms y)
//   5. dot_rz : rz' = r.z, beta = rz'/rz
// Scalars live in device memory; the last CTA of each reduction finalises
// them in a fixed order, so runs are bit-reproducible. Iterations are
// captured in a CUDA graph (every kernel no-ops once `done` is set) and the
// host polls the flag once per graph launch; the iteration count is exact.
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstring>

#include "core.h"
#include "sweep.cuh"

namespace pclab_b200 {


namespace {

constexpr int kT = 256;

struct Scal {
    double rz, pap, alpha, beta, bnorm, rel, rel_tol, rr;
    long long iter, max_iters;
    int done, converged, error, pad;
    unsigned ticket[4];
    unsigned ctr[4];  // claim counters of the fallback sweeps (L, U)
};

// Last-CTA finalisation of a per-CTA partial: returns true in the CTA
// that must finish the reduction; *total is then valid in thread 0.
__device__ __forceinline__ bool finish_partial(double local, double* part, unsigned* ticket,
                                               double* total) {
    __shared__ double sm[kT / 32];
    __shared__ bool last;
    const double bs = block_sum<kT>(local, sm);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = bs;
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return false;
    double s = 0.0;
    for (unsigned b = threadIdx.x; b < gridDim.x; b += kT) s += __ldcg(part + b);
    s = block_sum<kT>(s, sm);
    if (threadIdx.x == 0) {
        *total = s;
        *ticket = 0;
    }
    return true;
}

// p <- z + beta p (beta from the previous dot; 0 on the first iteration)
__global__ void __launch_bounds__(kT)
k_pupdate(int64_t n, const double* __restrict__ z, double* __restrict__ p, const Scal* S) {
    if (S->done) return;
    const double beta = S->beta;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT)
        p[i] = fma(beta, p[i], z[i]);
}

// q = A p and pAp. Lane groups of LPR lanes per row; every index and value
// load of a row (up to 4 LPR entries) is issued before the first gather.
template <int LPR, int U>
__global__ void __launch_bounds__(kT)
k_spmv_pap(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
           const double* __restrict__ vals, const double* __restrict__ p, double* __restrict__ q,
           Scal* S, double* part) {
    if (S->done) return;
    const int gl = threadIdx.x % LPR;
    const int64_t g0 = (blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x) / LPR;
    const int64_t ng = static_cast<int64_t>(gridDim.x) * kT / LPR;
    const int64_t nround = (n + ng - 1) / ng;
    double loc = 0.0;
    for (int64_t r = 0; r < nround; ++r) {
        const int64_t row = g0 + r * ng;
        const bool active = row < n;
        double acc = 0.0;
        if (active) {
            const int64_t b = rp[row], e = rp[row + 1];
            for (int64_t k0 = b + gl; k0 < e; k0 += U * LPR) {
                int32_t j[U];
                double v[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t k = k0 + u * LPR;
                    j[u] = k < e ? __ldg(cols + k) : -1;
                    v[u] = k < e ? __ldg(vals + k) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (j[u] >= 0) acc = fma(v[u], __ldg(p + j[u]), acc);
            }
        }
        acc = group_sum<LPR>(acc);
        if (active && gl == 0) {
            q[row] = acc;
            loc = fma(p[row], acc, loc);
        }
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[0], &tot) && threadIdx.x == 0) {
        S->pap = tot;
        if (!(tot > 0.0)) {
            S->error = 1;
            S->done = 1;
        } else {
            S->alpha = S->rz / tot;
        }
        S->ctr[0] = 0;
        S->ctr[1] = 0;
        S->ctr[2] = 0;
        S->ctr[3] = 0;
    }
}

// q = A p and pAp for short scalar rows: a warp per 32 consecutive rows
// (tile_rows_dot), row pointers a tile ahead.
__global__ void TILE_LB(kT)
k_spmv_tile_pap(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                const double* __restrict__ vals, const double* __restrict__ p, double* __restrict__ q,
                Scal* S, double* part) {
    if (S->done) return;
    __shared__ double sh[kT / 32][kTileCh];
    const int lane = threadIdx.x & 31;
    const int64_t nt = (n + 31) / 32;
    const int64_t gw = (blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * kT) >> 5;
    double loc = 0.0;
    RowSpan s = row_span(rp, n, gw * 32 + lane);
    for (int64_t t = gw; t < nt; t += nw) {
        const RowSpan sn = row_span(rp, n, (t + nw) * 32 + lane);
        const double acc = tile_rows_dot(s, cols, vals, p, sh[threadIdx.x >> 5], lane);
        const int64_t row = t * 32 + lane;
        if (row < n) {
            q[row] = acc;
            loc = fma(p[row], acc, loc);
        }
        s = sn;
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[0], &tot) && threadIdx.x == 0) {
        S->pap = tot;
        if (!(tot > 0.0)) {
            S->error = 1;
            S->done = 1;
        } else {
            S->alpha = S->rz / tot;
        }
        S->ctr[0] = 0;
        S->ctr[1] = 0;
        S->ctr[2] = 0;
        S->ctr[3] = 0;
    }
}

// ---- padded p (node-blocked A, bs = 3): p stored as 4 doubles per node
// (32-byte aligned, pad = 0), so the product gathers a neighbour's three
// values with ONE 256-bit load instead of three 8-byte loads (a third of
// the gather wavefronts of the L1-bound product). Entry i lives at
// 4 (i / 3) + i % 3.
__device__ __forceinline__ int64_t p4_index(int64_t i) { return 4 * (i / 3) + i % 3; }

__device__ __forceinline__ void ldg256(const double* p, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// p <- z + beta p on the padded layout (ZPAD: z padded too, the sweeps'
// padded output)
template <bool ZPAD>
__global__ void __launch_bounds__(kT)
k_pupdate4(int64_t n, const double* __restrict__ z, double* __restrict__ p4, const Scal* S) {
    if (S->done) return;
    const double beta = S->beta;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT) {
        const int64_t k = p4_index(i);
        p4[k] = fma(beta, p4[k], z[ZPAD ? k : i]);
    }
}

// q = A p (padded p) and pAp: k_spmv_bsr_pap<3> with one 256-bit gather
// per neighbour block; same per-row summation order.
// 5 CTAs/SM (40 warps at 48 registers): configs[2] product 0.652 ms at 4,
// 0.644 at 5, 0.813 at 6
#ifndef PAP4_MINB
#define PAP4_MINB 5
#endif
__global__ void __launch_bounds__(kT, PAP4_MINB)
k_spmv_bsr_pap4(int64_t nb, const int64_t* __restrict__ rp, const int64_t* __restrict__ bp,
                const int32_t* __restrict__ bcol, const double* __restrict__ vals, const double* __restrict__ p4,
                double* __restrict__ q, Scal* S, double* part) {
    if (S->done) return;
    constexpr int BS = 3;
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * kT + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * kT) >> 5);
    double loc = 0.0;
    // 32-bit row / block-column offsets (nnz(A) < 2^32, checked by the
    // launcher): five registers per row record instead of nine
    struct Row32 {
        uint32_t r[BS];
        uint32_t c0;
        int cnt;
    };
    auto row32 = [&](int b) {
        Row32 o{};
        if (b < nb) {
#pragma unroll
            for (int t = 0; t < BS; ++t) o.r[t] = static_cast<uint32_t>(__ldg(rp + static_cast<int64_t>(b) * BS + t));
            const int64_t c0 = __ldg(bp + b);
            o.c0 = static_cast<uint32_t>(c0);
            o.cnt = static_cast<int>(__ldg(bp + b + 1) - c0);
        }
        return o;
    };
    Row32 m = row32(gw);
    for (int b = gw; b < nb; b += nw) {
        const Row32 mn = row32(b + nw);
        double acc[BS] = {0.0, 0.0, 0.0};
        for (int n = lane; n < m.cnt; n += 32) {
            const int32_t xc = __ldg(bcol + (m.c0 + n));
            double a[BS][BS];
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) a[t][c] = __ldg(vals + (m.r[t] + BS * n + c));
            double xv[4];
            ldg256(p4 + 4 * static_cast<uint32_t>(xc / 3), xv[0], xv[1], xv[2], xv[3]);
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) acc[t] = fma(a[t][c], xv[c], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<32>(acc[t]);
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < BS; ++t) {
                const int64_t row = static_cast<int64_t>(b) * BS + t;
                q[row] = acc[t];
                loc = fma(p4[4 * static_cast<int64_t>(b) + t], acc[t], loc);
            }
        }
        m = mn;
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[0], &tot) && threadIdx.x == 0) {
        S->pap = tot;
        if (!(tot > 0.0)) {
            S->error = 1;
            S->done = 1;
        } else {
            S->alpha = S->rz / tot;
        }
        S->ctr[0] = 0;
        S->ctr[1] = 0;
        S->ctr[2] = 0;
        S->ctr[3] = 0;
    }
}

// x += alpha p (padded p), r -= alpha q, ||r|| -> convergence
__global__ void __launch_bounds__(kT)
k_axpy4(int64_t n, const double* __restrict__ p4, const double* __restrict__ q, double* __restrict__ x,
        double* __restrict__ r, Scal* S, double* part, double* hist);

// q = A p and pAp for a node-blocked A (Analysis::a_bsr): warp per block
// row (grid-stride), the next row's pointers loaded while this one runs.
template <int BS>
__global__ void __launch_bounds__(kT)
k_spmv_bsr_pap(int64_t nb, const int64_t* __restrict__ rp, const int64_t* __restrict__ bp,
                const int32_t* __restrict__ bcol, const double* __restrict__ vals, const double* __restrict__ p,
                double* __restrict__ q, Scal* S, double* part) {
    if (S->done) return;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * kT) >> 5;
    double loc = 0.0;
    BsrRow<BS> m = bsr_row<BS>(gw, nb, rp, bp);
    for (int64_t b = gw; b < nb; b += nw) {
        const BsrRow<BS> mn = bsr_row<BS>(b + nw, nb, rp, bp);
        double acc[BS];
        bsr_row_dot<BS>(m, bcol, vals, p, acc);
        if (lane == 0) {
#pragma unroll
            for (int t = 0; t < BS; ++t) {
                const int64_t row = b * BS + t;
                q[row] = acc[t];
                loc = fma(p[row], acc[t], loc);
            }
        }
        m = mn;
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[0], &tot) && threadIdx.x == 0) {
        S->pap = tot;
        if (!(tot > 0.0)) {
            S->error = 1;
            S->done = 1;
        } else {
            S->alpha = S->rz / tot;
        }
        S->ctr[0] = 0;
        S->ctr[1] = 0;
        S->ctr[2] = 0;
        S->ctr[3] = 0;
    }
}

__global__ void __launch_bounds__(kT)
k_axpy(int64_t n, const double* __restrict__ p, const double* __restrict__ q, double* __restrict__ x,
       double* __restrict__ r, Scal* S, double* part, double* hist, double* __restrict__ rearm) {
    if (S->done) return;
    const double alpha = S->alpha;
    double loc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT) {
        // y of the unpadded sweeps is re-armed here, in a streaming kernel that
        // runs between the sweep that read it and the one that fills it: the
        // backward sweep re-arming its own right-hand side cost it 0.09 ms
        // on the 256^3 diffusion system (0.90 -> 0.81), this store 0.02
        if (rearm) rearm[i] = pending_value();
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        loc = fma(ri, ri, loc);
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[1], &tot) && threadIdx.x == 0) {
        S->rr = tot;
        const double rel = sqrt(tot) / S->bnorm;
        const long long it = S->iter + 1;
        S->iter = it;
        S->rel = rel;
        if (hist) hist[it] = rel;
        if (rel <= S->rel_tol) {
            S->converged = 1;
            S->done = 1;
        } else if (it >= S->max_iters) {
            S->done = 1;
        }
    }
}

__global__ void __launch_bounds__(kT)
k_axpy4(int64_t n, const double* __restrict__ p4, const double* __restrict__ q, double* __restrict__ x,
       double* __restrict__ r, Scal* S, double* part, double* hist) {
    if (S->done) return;
    const double alpha = S->alpha;
    double loc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT) {
        x[i] = fma(alpha, p4[p4_index(i)], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        loc = fma(ri, ri, loc);
    }
    double tot;
    if (finish_partial(loc, part, &S->ticket[1], &tot) && threadIdx.x == 0) {
        S->rr = tot;
        const double rel = sqrt(tot) / S->bnorm;
        const long long it = S->iter + 1;
        S->iter = it;
        S->rel = rel;
        if (hist) hist[it] = rel;
        if (rel <= S->rel_tol) {
            S->converged = 1;
            S->done = 1;
        } else if (it >= S->max_iters) {
            S->done = 1;
        }
    }
}

// mode 0: rz' -> beta, rz   mode 1: setup rz (beta = 0)   mode 2: bnorm
__global__ void __launch_bounds__(kT)
k_dot(int64_t n, const double* __restrict__ a, const double* __restrict__ b, Scal* S, double* part,
      int mode) {
    if (mode == 0 && S->done) return;
    double loc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT)
        loc = fma(a[i], b[i], loc);
    double tot;
    if (finish_partial(loc, part, &S->ticket[2], &tot) && threadIdx.x == 0) {
        if (mode == 0) {
            S->beta = tot / S->rz;
            S->rz = tot;
        } else if (mode == 1) {
            S->rz = tot;
            S->beta = 0.0;
        } else {
            S->bnorm = sqrt(tot);
        }
    }
}

// k_dot with b on the padded layout (r . z, z the sweeps' padded output)
// mode 0: rz' -> beta, rz   mode 1: setup rz (beta = 0)   mode 2: bnorm
__global__ void __launch_bounds__(kT)
k_dot_z4(int64_t n, const double* __restrict__ a, const double* __restrict__ b, Scal* S, double* part,
      int mode) {
    if (mode == 0 && S->done) return;
    double loc = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT)
        loc = fma(a[i], b[p4_index(i)], loc);
    double tot;
    if (finish_partial(loc, part, &S->ticket[2], &tot) && threadIdx.x == 0) {
        if (mode == 0) {
            S->beta = tot / S->rz;
            S->rz = tot;
        } else if (mode == 1) {
            S->rz = tot;
            S->beta = 0.0;
        } else {
            S->bnorm = sqrt(tot);
        }
    }
}

__global__ void k_jacobi(int64_t n, const double* __restrict__ r, const double* __restrict__ d,
                         double* __restrict__ z, const Scal* S) {
    if (S->done) return;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * kT)
        z[i] = r[i] / d[i];
}

__global__ void k_resid(int64_t n, const double* __restrict__ b, double* __restrict__ ax) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (i < n) ax[i] = b[i] - ax[i];
}

__global__ void k_combine(int64_t n, const int64_t* __restrict__ lrp, double* __restrict__ l,
                          const double* __restrict__ o, double sigma, int nic,
                          unsigned long long* bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (i >= n) return;
    for (int64_t k = lrp[i]; k < lrp[i + 1]; ++k) l[k] = nic ? o[k] * sigma : l[k] + o[k];
    if (!(l[lrp[i + 1] - 1] > 0.0)) atomicMin(bad, static_cast<unsigned long long>(i));
}

__global__ void k_jacobi_diag(int64_t n, const double* __restrict__ vals,
                              const int64_t* __restrict__ dpos, double* __restrict__ d,
                              unsigned long long* bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (i >= n) return;
    const double v = dpos[i] >= 0 ? vals[dpos[i]] : 0.0;
    d[i] = v;
    if (!(v > 0.0)) atomicMin(bad, static_cast<unsigned long long>(i));
}

inline unsigned gfor(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

struct Timer {
    cudaEvent_t a, b;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s) {
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st));
    }
    double ms() {
        CK(cudaEventRecord(b, st));
        CK(cudaEventSynchronize(b));
        float t = 0;
        CK(cudaEventElapsedTime(&t, a, b));
        return t;
    }
    ~Timer() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
};

unsigned long long read_flag(unsigned long long* d, cudaStream_t st) {
    unsigned long long h;
    CK(cudaMemcpyAsync(&h, d, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h;
}

}  // namespace

const char* kind_name(Kind k) {
    switch (k) {
        case Kind::None: return "none";
        case Kind::Jacobi: return "jacobi";
        case Kind::IC0: return "ic0";
        case Kind::NIC: return "nic";
        case Kind::GnnIC: return "gnnic";
    }
    return "unknown";
}

Kind parse_kind(const std::string& k) {
    if (k == "none") return Kind::None;
    if (k == "jacobi") return Kind::Jacobi;
    if (k == "ic0") return Kind::IC0;
    if (k == "nic") return Kind::NIC;
    if (k == "gnnic") return Kind::GnnIC;
    throw DimensionError("unknown preconditioner kind '" + k + "'");
}

std::unique_ptr<Precond> build_precond(Matrix& a, Kind kind, const Model* model, cudaStream_t st) {
    auto p = std::make_unique<Precond>();
    p->kind = kind;
    p->a = &a;
    const int64_t n = a.a.n;
    Timer total(st);
    if (kind == Kind::None) return p;
    // the reference's first failing check per kind (precond.cpp:92, sparse.cpp:190, features.cpp:13)
    const bool square = a.n_cols == a.a.n;
    DevBuf<unsigned long long> bad(1);
    CK(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
    if (kind == Kind::Jacobi) {
        if (!square) throw DimensionError("jacobi: matrix not square");
        p->diag.alloc(n);
        if (n) k_jacobi_diag<<<gfor(n), kT, 0, st>>>(n, a.a.vals.p, a.diag_pos.p, p->diag.p, bad.p);
        CK_LAUNCH();
        const auto f = read_flag(bad.p, st);
        if (f != ~0ULL) throw NumericError("jacobi: nonpositive diagonal at row " + std::to_string(f));
        p->ms_total = total.ms();
        return p;
    }
    if ((kind == Kind::NIC || kind == Kind::GnnIC) && model == nullptr)
        throw DimensionError(std::string("kind '") + kind_name(kind) + "' needs a model");
    if (!square)
        throw DimensionError(kind == Kind::NIC ? "node_features: matrix not square"
                                               : "lower_triangle: matrix not square");
    if (!matrix_symmetric(a, st)) throw FormatError("lower_triangle: matrix not symmetric");
    if (a.missing_diag_row >= 0) {
        if (kind == Kind::NIC)
            throw FormatError("lower factor: missing diagonal at row " + std::to_string(a.missing_diag_row));
        throw FormatError("ic0: missing diagonal at row " + std::to_string(a.missing_diag_row));
    }
    {
        const bool fresh = !a.an;
        Timer t(st);
        ensure_analysis(a, st);
        p->ms_analysis = fresh ? a.an->ms : 0.0;
        (void)t;
    }
    p->an = a.an;
    const Analysis& an = *a.an;
    p->lvals.alloc(an.lower.nnz);
    p->uvals.alloc(an.upper.nnz);
    if (kind == Kind::IC0 || kind == Kind::GnnIC) {
        Timer t(st);
        p->ic0_attempts = ic0_factor(a, an, p->lvals.p, st);
        p->ms_ic0 = t.ms();
    }
    if (kind == Kind::NIC || kind == Kind::GnnIC) {
        Timer t(st);
        DevBuf<double> out(an.lower.nnz);
        gnn_forward(a, an, *model, out.p, &p->sigma, st);
        if (n)
            k_combine<<<gfor(n), kT, 0, st>>>(n, an.lower.rp.p, p->lvals.p, out.p, p->sigma,
                                              kind == Kind::NIC, bad.p);
        CK_LAUNCH();
        const auto f = read_flag(bad.p, st);
        if (f != ~0ULL)
            throw NumericError("lower factor: nonpositive diagonal at row " + std::to_string(f));
        p->ms_gnn = t.ms();
    }
    gather_upper(an, p->lvals.p, p->uvals.p, st);
    p->invd.alloc(n);
    reciprocal_diag(an, p->lvals.p, p->invd.p, st);
    fill_bss(an, *p, st);
    p->ms_total = total.ms();  // the analysis ran inside this interval
    return p;
}

SolveReport pcg_solve(Matrix& a, const Precond& pc, const double* b, double* x, double rel_tol,
                      int64_t max_iters, bool record, cudaStream_t st, double* prof_ms) {
    if (a.n_cols != a.a.n) throw DimensionError("pcg: shape mismatch");
    if (!(rel_tol > 0.0)) throw DimensionError("pcg: rel_tol must be > 0");
    const int64_t n = a.a.n;
    if (max_iters < 0) max_iters = 10 * n;
    SolveReport rep;
    rep.p_time = pc.ms_total / 1e3;
    rep.analysis_time = pc.ms_analysis / 1e3;
    rep.ic0_time = pc.ms_ic0 / 1e3;
    rep.gnn_time = pc.ms_gnn / 1e3;
    const bool factor = pc.kind == Kind::IC0 || pc.kind == Kind::NIC || pc.kind == Kind::GnnIC;
    Timer cg(st);
    const auto h0 = std::chrono::steady_clock::now();
    static const bool gtrace = getenv("PCLAB_PCG_TRACE") != nullptr;
    auto trace = [&](const char* what) {
        if (gtrace)
            fprintf(stderr, "solve %s at %.3f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
    };
    CK(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
    const int parts_max = sm_count() * 8;
    DevBuf<Scal> S(1);
    DevBuf<double> part(parts_max), r(n), q(n), pa, y, zbuf, tmp(n);
    DevBuf<double> hist;
    if (record) hist.alloc(max_iters + 1);
    Scal h{};
    h.rel_tol = rel_tol;
    h.max_iters = max_iters;
    CK(cudaMemcpyAsync(S.p, &h, sizeof h, cudaMemcpyHostToDevice, st));
    // vector kernels: 8 CTAs per SM (axpy 58 -> 45 us, dot 26 -> 25 us on configs[2])
    const unsigned vgrid = static_cast<unsigned>(sm_count() * 8);
    const unsigned sgrid = static_cast<unsigned>(sm_count() * 8);
    if (n) k_dot<<<vgrid, kT, 0, st>>>(n, b, b, S.p, part.p, 2);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(&h, S.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.bnorm == 0.0 || n == 0) {
        rep.converged = true;
        if (record) rep.residual_history.push_back(0.0);
        rep.cg_time = cg.ms() / 1e3;
        rep.total_time = rep.p_time + rep.cg_time;
        return rep;
    }
    CK(cudaMemcpyAsync(r.p, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    // rel_0 = ||b|| / ||b|| (krylov.cpp:143): identical operands, exactly 1
    const double rel0 = 1.0;
    rep.final_rel_residual = rel0;
    if (record) {
        CK(cudaMemcpyAsync(hist.p, &rel0, sizeof rel0, cudaMemcpyHostToDevice, st));
    }
    if (rel0 <= rel_tol) {
        rep.converged = true;
        if (record) rep.residual_history.push_back(rel0);
        rep.cg_time = cg.ms() / 1e3;
        rep.total_time = rep.p_time + rep.cg_time;
        rep.true_rel_residual = 1.0;
        return rep;
    }
    trace("setup");
    // the sweeps run on the preconditioner's own analysis (co-owned: it
    // survives pclab_matrix_drop_analysis); the product's block view is A's
    const Analysis* an = factor ? pc.an.get() : nullptr;
    if (factor && (!an || an->lower.n != n)) throw DimensionError("tri_solve_lower: shape mismatch");
    const Analysis* aan = a.an ? a.an.get() : (pc.a == &a ? pc.an.get() : nullptr);
    const bool a_bsr = aan && aan->a_bsr;
    // padded p for the node-blocked 3x3 product (and sweeps of the same
    // node layout); k_spmv_bsr_pap4 indexes A with 32 bits
    const bool padp = a_bsr && aan->bs == 3 && a.a.nnz < (1LL << 32) && aan->abc.bcol.n < (1LL << 32) &&
                      (!factor || (an->bsr && an->bs == 3));
    pa.alloc(padp ? 4 * (n / 3) : n);
    // sweep vectors y, z padded too (node-blocked 3x3 sweeps): 256-bit polls
    // and publications (bsr_item PAD)
    const bool padz = padp && factor;
    double* z = r.p;  // kind none: z aliases r
    if (factor) {
        y.alloc(padz ? 4 * (n / 3) : n);
        zbuf.alloc(padz ? 4 * (n / 3) : n);
        z = zbuf.p;
        fill_pending(y.p, y.n, st);
        fill_pending(z, zbuf.n, st);
    } else if (pc.kind == Kind::Jacobi) {
        zbuf.alloc(n);
        z = zbuf.p;
    }
    // ---- z0 = M^-1 r0, rz, beta = 0, p = 0
    {
        Timer tt(st);
        if (factor) {
            CK(cudaMemsetAsync(S.p->ctr, 0, sizeof(unsigned) * 4, st));
            launch_sweep(*an, pc, false, r.p, y.p, z, nullptr, S.p->ctr, st, padz);
            launch_sweep(*an, pc, true, y.p, z, padz ? y.p : nullptr, nullptr, S.p->ctr + 1, st, padz);
        } else if (pc.kind == Kind::Jacobi) {
            k_jacobi<<<vgrid, kT, 0, st>>>(n, r.p, pc.diag.p, z, S.p);
        }
        CK_LAUNCH();
        rep.tri_solve_time_per_iter = factor ? tt.ms() / 1e3 : 0.0;
    }
    if (padz)
        k_dot_z4<<<vgrid, kT, 0, st>>>(n, r.p, z, S.p, part.p, 1);
    else
        k_dot<<<vgrid, kT, 0, st>>>(n, r.p, z, S.p, part.p, 1);
    CK(cudaMemsetAsync(pa.p, 0, pa.bytes(), st));
    CK_LAUNCH();
    const int lpr = spmv_lanes(a);
    static const unsigned tgrid = [] {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_spmv_tile_pap, kT, 0));
        return static_cast<unsigned>(std::min(std::max(per_sm, 1), 8) * sm_count());
    }();
    auto one_wave = [](auto kernel) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kT, 0));
        return static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
    };
    static const unsigned bsr_grid3 = one_wave(k_spmv_bsr_pap<3>);
    static const unsigned bsr_grid2 = one_wave(k_spmv_bsr_pap<2>);
    static const unsigned bsr_grid4 = one_wave(k_spmv_bsr_pap4);
    // one PCG iteration, five or six kernels; `mark` runs after each stage
    // (event hook for profiling): [product, axpy, sweep L, sweep U, dot]
    auto iteration_parts = [&](double* pp, auto&& mark) {
        if (padp) {
            if (padz)
                k_pupdate4<true><<<vgrid, kT, 0, st>>>(n, z, pp, S.p);
            else
                k_pupdate4<false><<<vgrid, kT, 0, st>>>(n, z, pp, S.p);
            const BlockCols& bc = aan->abc;
            k_spmv_bsr_pap4<<<bsr_grid4, kT, 0, st>>>(n / 3, a.a.rp.p, bc.bp.p, bc.bcol.p, a.a.vals.p, pp, q.p, S.p,
                                                     part.p);
            mark();
            k_axpy4<<<vgrid, kT, 0, st>>>(n, pp, q.p, x, r.p, S.p, part.p, record ? hist.p : nullptr);
            mark();
        } else {
            k_pupdate<<<vgrid, kT, 0, st>>>(n, z, pp, S.p);
            if (a_bsr) {
                // grid = one resident wave (grid-stride rows; a second partial
                // wave doubles the tail: measured 0.75 vs 0.93 ms at 1.5 waves)
                const BlockCols& bc = aan->abc;
                if (aan->bs == 3)
                    k_spmv_bsr_pap<3><<<bsr_grid3, kT, 0, st>>>(n / 3, a.a.rp.p, bc.bp.p, bc.bcol.p, a.a.vals.p, pp,
                                                               q.p, S.p, part.p);
                else
                    k_spmv_bsr_pap<2><<<bsr_grid2, kT, 0, st>>>(n / 2, a.a.rp.p, bc.bp.p, bc.bcol.p, a.a.vals.p, pp,
                                                               q.p, S.p, part.p);
            } else switch (lpr) {
                case 1: k_spmv_tile_pap<<<tgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 4: k_spmv_pap<4, 4><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 8: k_spmv_pap<8, 4><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 9: k_spmv_pap<8, 12><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 5: k_spmv_pap<4, 8><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 3: k_spmv_pap<4, 12><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 2: k_spmv_pap<2, 16><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 17: k_spmv_pap<16, 3><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                case 16: k_spmv_pap<16, 6><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
                default: k_spmv_pap<32, 4><<<sgrid, kT, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, pp, q.p, S.p, part.p); break;
            }
            mark();
            k_axpy<<<vgrid, kT, 0, st>>>(n, pp, q.p, x, r.p, S.p, part.p, record ? hist.p : nullptr,
                                         factor ? y.p : nullptr);
            mark();
        }
        if (factor) {
            launch_sweep(*an, pc, false, r.p, y.p, z, &S.p->done, S.p->ctr, st, padz);
            mark();
            // padded y is re-armed by the backward sweep itself, unpadded y by k_axpy
            launch_sweep(*an, pc, true, y.p, z, padz ? y.p : nullptr, &S.p->done, S.p->ctr + 1, st, padz);
            mark();
        } else {
            if (pc.kind == Kind::Jacobi) k_jacobi<<<vgrid, kT, 0, st>>>(n, r.p, pc.diag.p, z, S.p);
            mark();
            mark();
        }
        if (padz)
            k_dot_z4<<<vgrid, kT, 0, st>>>(n, r.p, z, S.p, part.p, 0);
        else
            k_dot<<<vgrid, kT, 0, st>>>(n, r.p, z, S.p, part.p, 0);
        mark();
    };
    auto iteration = [&](double* pp) { iteration_parts(pp, [] {}); };
    // pinned done flag, allocated once per host thread: a pinned allocation
    // inside the timed solve could stall the host (page pinning) while the
    // GPU idles
    thread_local int* hdone = [] {
        int* h = nullptr;
        CK(cudaMallocHost(&h, sizeof(int)));
        return h;
    }();
    if (prof_ms) {
        // eager iterations with an event between kernels: per-kernel device
        // times averaged over iterations, [spmv_p, axpy, sweep L, sweep U, dot]
        constexpr int kK = 5;
        cudaEvent_t ev[kK + 1];
        for (auto& e : ev) CK(cudaEventCreate(&e));
        double acc[kK] = {0, 0, 0, 0, 0};
        int done_iters = 0;
        for (;;) {
            int k = 0;
            CK(cudaEventRecord(ev[k++], st));
            iteration_parts(pa.p, [&] { CK(cudaEventRecord(ev[k++], st)); });
            CK(cudaMemcpyAsync(hdone, &S.p->done, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (*hdone) break;  // converged inside: the partial iteration is not counted
            for (int t = 0; t < kK; ++t) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, ev[t], ev[t + 1]));
                acc[t] += ms;
            }
            ++done_iters;
        }
        for (int t = 0; t < kK; ++t) prof_ms[t] = done_iters ? acc[t] / done_iters : 0.0;
        prof_ms[kK] = done_iters;
        prof_ms[kK + 1] = 0.0;
        prof_ms[kK + 2] = 0.0;
        for (auto& e : ev) cudaEventDestroy(e);
    } else {
        // iterations captured in a CUDA graph; the host reads the done flag
        // once per replay (every kernel no-ops after convergence)
        const int per_graph = n > 2000000 ? 8 : 16;
        cudaGraph_t graph;
        cudaGraphExec_t exec;
        const long long before = launch_count();
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int k = 0; k < per_graph; ++k) iteration(pa.p);
        CK(cudaStreamEndCapture(st, &graph));
        trace("captured");
        CK(cudaGraphInstantiate(&exec, graph, 0));
        trace("instantiated");
        size_t nodes = 0;
        CK(cudaGraphGetNodes(graph, nullptr, &nodes));
        g_launches = before;  // captured launches are counted per replay below
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            CK(cudaGraphLaunch(exec, st));
            count_launches(static_cast<long long>(nodes));
            CK(cudaMemcpyAsync(hdone, &S.p->done, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (gtrace)
                fprintf(stderr, "graph %.3f ms\n",
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            if (*hdone) break;
        }
        cudaGraphExecDestroy(exec);
        cudaGraphDestroy(graph);
    }
    trace("loop done");
    rep.cg_time = cg.ms() / 1e3;
    CK(cudaMemcpyAsync(&h, S.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.error)
        throw NumericError("pcg: nonpositive curvature at iteration " + std::to_string(h.iter + 1) +
                           " (matrix not SPD?)");
    rep.iterations = h.iter;
    rep.converged = h.converged != 0;
    rep.final_rel_residual = h.rel;
    if (record) {
        rep.residual_history.resize(h.iter + 1);
        CK(cudaMemcpyAsync(rep.residual_history.data(), hist.p, sizeof(double) * (h.iter + 1),
                           cudaMemcpyDeviceToHost, st));
    }
    // true residual ||b - A x|| / ||b|| (krylov.cpp:182-188); k_dot mode 2
    // writes its norm into the bnorm slot
    const double bnorm = h.bnorm;
    spmv(a, x, tmp.p, st);
    k_resid<<<gfor(n), kT, 0, st>>>(n, b, tmp.p);
    k_dot<<<vgrid, kT, 0, st>>>(n, tmp.p, tmp.p, S.p, part.p, 2);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(&h, S.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    rep.true_rel_residual = h.bnorm / bnorm;
    rep.residual_mismatch =
        std::fabs(rep.true_rel_residual - rep.final_rel_residual) > 10.0 * rel_tol;
    rep.total_time = rep.p_time + rep.cg_time;
    return rep;
}

}  // namespace pclab_b200
