// Host wrappers for the stand-alone sparse kernels (SpMV, the two sweeps,
// U value gather, pending fill). The PCG loop uses fused variants in
// pcg.cu; these are the building blocks exposed through the C-ABI.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "core.h"
#include "sweep.cuh"

namespace pclab_b200 {

namespace {

__global__ void fill_kernel(unsigned long long* p, int64_t n, unsigned long long v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

template <int LPR>
__global__ void __launch_bounds__(256)
spmv_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
            const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y) {
    const int gl = threadIdx.x % LPR;
    const int64_t g0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / LPR;
    const int64_t ng = static_cast<int64_t>(gridDim.x) * blockDim.x / LPR;
    const int64_t nround = (n + ng - 1) / ng;
    for (int64_t r = 0; r < nround; ++r) {
        const int64_t row = g0 + r * ng;
        const bool active = row < n;
        const double s = row_dot<LPR>(rp, cols, vals, x, row, gl, active);
        if (active && gl == 0) y[row] = s;
    }
}

// short scalar rows: a warp per 32 consecutive rows (tile_rows_dot), the
// next tile's row pointers loaded a tile ahead
__global__ void TILE_LB(256)
spmv_tile_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                 const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y) {
    __shared__ double sh[8][kTileCh];
    const int lane = threadIdx.x & 31;
    const int64_t nt = (n + 31) / 32;
    const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    RowSpan s = row_span(rp, n, gw * 32 + lane);
    for (int64_t t = gw; t < nt; t += nw) {
        const RowSpan sn = row_span(rp, n, (t + nw) * 32 + lane);
        const double acc = tile_rows_dot(s, cols, vals, x, sh[threadIdx.x >> 5], lane);
        const int64_t row = t * 32 + lane;
        if (row < n) y[row] = acc;
        s = sn;
    }
}

template <int BS>
__global__ void __launch_bounds__(256)
spmv_bsr_kernel(int64_t nb, const int64_t* __restrict__ rp, const int64_t* __restrict__ bp,
                const int32_t* __restrict__ bcol, const double* __restrict__ vals, const double* __restrict__ x,
                double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    BsrRow<BS> m = bsr_row<BS>(gw, nb, rp, bp);
    for (int64_t b = gw; b < nb; b += nw) {
        const BsrRow<BS> mn = bsr_row<BS>(b + nw, nb, rp, bp);
        double acc[BS];
        bsr_row_dot<BS>(m, bcol, vals, x, acc);
        if (lane < BS) {
            double v = acc[0];
#pragma unroll
            for (int t = 1; t < BS; ++t)
                if (lane == t) v = acc[t];
            y[b * BS + lane] = v;
        }
        m = mn;
    }
}

// y = A x for node-blocked A with 32-bit entry / block-column offsets
// (nnz < 2^32): the row records fit five registers, so five 256-thread CTAs
// per SM stay resident without spills (40 warps of loads in flight).
template <int BS>
__global__ void __launch_bounds__(256, 5)
spmv_bsr32_kernel(int nb, const int64_t* __restrict__ rp, const int64_t* __restrict__ bp,
                  const int32_t* __restrict__ bcol, const double* __restrict__ vals, const double* __restrict__ x,
                  double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
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
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        for (int n = lane; n < m.cnt; n += 32) {
            const int32_t xc = __ldg(bcol + (m.c0 + n));
            double a[BS][BS], xv[BS];
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) a[t][c] = __ldg(vals + (m.r[t] + BS * n + c));
#pragma unroll
            for (int c = 0; c < BS; ++c) xv[c] = __ldg(x + xc + c);
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) acc[t] = fma(a[t][c], xv[c], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<32>(acc[t]);
        if (lane < BS) {
            double v = acc[0];
#pragma unroll
            for (int t = 1; t < BS; ++t)
                if (lane == t) v = acc[t];
            y[static_cast<int64_t>(b) * BS + lane] = v;
        }
        m = mn;
    }
}

// plain <-> padded (4 doubles per 3-dof node) vector copies
__global__ void pad_copy_kernel(int64_t n, const double* __restrict__ src, double* __restrict__ dst, bool to_pad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int64_t k = 4 * (i / 3) + i % 3;
    if (to_pad) dst[k] = src[i];
    else dst[i] = src[k];
}

__global__ void gather_kernel(int64_t m, const int64_t* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k < m) dst[k] = src[idx[k]];
}

}  // namespace

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

// CTAs of `kernel` (256 threads) the whole GPU holds at once.
template <typename K>
static unsigned resident_ctas(K kernel) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0));
    return static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
}

void fill_pending(double* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    fill_kernel<<<sm_count() * 4, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(p), n, kPending);
    CK_LAUNCH();
}

int spmv_lanes(const Matrix& a) {
    const double avg = a.a.n ? static_cast<double>(a.a.nnz) / static_cast<double>(a.a.n) : 1.0;
    // Few lanes per row, many rows per warp: on the 81-entry elasticity rows
    // 4 lanes x 8 loads in flight beat 8/16/32 lanes (measured, configs[2]:
    // 1.04 vs 1.09/1.25/1.18 ms). Code 5 = 4 lanes with 8 loads per round.
    // Code 1 = a warp per 32 short rows (tile_rows_dot; 7-point stencils).
    int l = avg > 48 ? 5 : (avg <= 12 ? 1 : 4);
    if (avg > 200) l = 32;
    if (getenv("PCLAB_SPMV_LPR")) l = atoi(getenv("PCLAB_SPMV_LPR"));
    return l;
}

void spmv(const Matrix& a, const double* x, double* y, cudaStream_t st) {
    const int64_t n = a.a.n;
    if (n == 0) return;
    const unsigned grid = static_cast<unsigned>(sm_count() * 8);
    if (a.an && a.an->a_bsr) {  // node-blocked: one column index per block
        const BlockCols& bc = a.an->abc;
        static const unsigned g3 = resident_ctas(spmv_bsr_kernel<3>), g2 = resident_ctas(spmv_bsr_kernel<2>);
        static const unsigned g32 = resident_ctas(spmv_bsr32_kernel<3>);
        if (a.an->bs == 3 && a.a.nnz < (1LL << 32) && bc.bcol.n < (1LL << 32) && n / 3 < (1LL << 31))
            spmv_bsr32_kernel<3><<<g32, 256, 0, st>>>(static_cast<int>(n / 3), a.a.rp.p, bc.bp.p, bc.bcol.p,
                                                       a.a.vals.p, x, y);
        else if (a.an->bs == 3)
            spmv_bsr_kernel<3><<<g3, 256, 0, st>>>(n / 3, a.a.rp.p, bc.bp.p, bc.bcol.p, a.a.vals.p, x, y);
        else
            spmv_bsr_kernel<2><<<g2, 256, 0, st>>>(n / 2, a.a.rp.p, bc.bp.p, bc.bcol.p, a.a.vals.p, x, y);
        CK_LAUNCH();
        return;
    }
    switch (spmv_lanes(a)) {
        case 1: {
            static const unsigned gt = resident_ctas(spmv_tile_kernel);
            spmv_tile_kernel<<<gt, 256, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, x, y);
            break;
        }
        case 4:
        case 5: spmv_kernel<4><<<grid, 256, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, x, y); break;
        case 8: spmv_kernel<8><<<grid, 256, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, x, y); break;
        case 16: spmv_kernel<16><<<grid, 256, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, x, y); break;
        default: spmv_kernel<32><<<grid, 256, 0, st>>>(n, a.a.rp.p, a.a.cols.p, a.a.vals.p, x, y); break;
    }
    CK_LAUNCH();
}

void gather_upper(const Analysis& an, const double* lvals, double* uvals, cudaStream_t st) {
    const int64_t m = an.upper.nnz;
    if (m == 0) return;
    gather_kernel<<<static_cast<unsigned>((m + 255) / 256), 256, 0, st>>>(m, an.u2l.p, lvals, uvals);
    CK_LAUNCH();
}

// Resident warps for a sweep: enough to hold a few levels of items in
// flight (loads stream while the frontier advances) but not so many that
// idle pollers crowd L2.
// Measured on configs[2]: 4 levels for the entry-lane sweep, 2 for the
// node-blocked one (its pollers read BS values each, 1.40 vs 1.65 ms at 4).
static unsigned trsv_grid(const Schedule& s, double depth, int warps_per_cta = 8) {
    const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
    const int64_t warps = static_cast<int64_t>(depth * per_level) + 1;
    const int64_t blocks = (warps + warps_per_cta - 1) / warps_per_cta;
    return static_cast<unsigned>(
        std::min<int64_t>(std::max<int64_t>(blocks, sm_count()), sm_count() * (64 / warps_per_cta)));
}

// Claim-based entry-lane sweep: the fallback for rows longer than the
// round-robin sweeps' packed slot records allow (1023 entries).
template <int LG, int BS, bool UP>
static void launch_trsv_t(const Schedule& s, const DevCsr& M, const double* vals, const double* invd,
                          const double* b, double* x, double* reset, const int* done, unsigned* ctr,
                          cudaStream_t st) {
    trsv_kernel<LG, BS, UP><<<trsv_grid(s, 4.0), 256, 0, st>>>(s.nitems, s.slots.p, s.crit.p, M.rp.p, M.cols.p,
                                                                vals, invd, b, x, reset, done, ctr);
}

// Round-robin items need every warp resident: the grid is capped at what
// the GPU holds (measured best on configs[2]: as many warps as fit).
template <int LG, int BS, bool UP, bool PAD>
static void launch_bsr_d(const Schedule& s, const int32_t* bcol, const double* vals, const double* invd,
                         const double* b, double* x, double* reset, const int* done, cudaStream_t st) {
    static unsigned cap = 0;
    if (!cap) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsr_trsv_kernel<LG, BS, UP, PAD>, BSR_THREADS, 0));
        cap = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
    }
    if (s.nitems * s.per_item >= (1LL << 31)) throw DimensionError("node-blocked sweep: too many schedule slots");
    const unsigned grid = std::min(trsv_grid(s, 5.0, BSR_THREADS / 32), cap);  // ~all resident warps
    bsr_trsv_kernel<LG, BS, UP, PAD><<<grid, BSR_THREADS, 0, st>>>(s.nitems, s.slot_rp.p, bcol, vals, invd, b, x,
                                                                   reset, done);
}

// pad: output / re-arm vectors (and the upper sweep's right-hand side)
// stored 4 doubles per node (PCG loop, BS = 3)
template <int LG, int BS, bool UP>
static void launch_bsr_t(const Schedule& s, const int32_t* bcol, const double* vals, const double* invd,
                         const double* b, double* x, double* reset, const int* done, cudaStream_t st, bool pad) {
    if constexpr (BS == 3) {
        if (pad) {
            launch_bsr_d<LG, BS, UP, true>(s, bcol, vals, invd, b, x, reset, done, st);
            return;
        }
    }
    if (pad) throw DimensionError("padded sweeps need 3x3 node blocks");
    launch_bsr_d<LG, BS, UP, false>(s, bcol, vals, invd, b, x, reset, done, st);
}

template <int LG, int BS, bool UP, int CH>
static void launch_rr_t(const Schedule& s, const DevCsr& M, const double* vals, const double* invd, const double* b,
                        double* x, double* reset, const int* done, cudaStream_t st) {
    static unsigned cap = 0;
    if (!cap) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rr_trsv_kernel<LG, BS, UP, CH>, RR_THREADS, 0));
        cap = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
    }
    const unsigned grid = std::min(trsv_grid(s, 6.0, RR_THREADS / 32), cap);
    rr_trsv_kernel<LG, BS, UP, CH><<<grid, RR_THREADS, 0, st>>>(s.nitems, s.slot_rp.p, M.cols.p, vals, invd, b, x,
                                                                reset, done);
}

template <int BS, bool UP>
static void launch_trsv_bs(const Schedule& s, const DevCsr& M, bool rr, const BlockCols* bc, const double* vals,
                           const double* invd, const double* b, double* x, double* reset, const int* done,
                           unsigned* ctr, cudaStream_t st, bool pad) {
    if (pad && !bc) throw DimensionError("padded sweeps need the node-blocked sweep");
    if constexpr (BS > 1) {
        if (bc) {
            const int32_t* bcol = bc->bcol.p;
            switch (s.lanes) {
            case 4: launch_bsr_t<4, BS, UP>(s, bcol, vals, invd, b, x, reset, done, st, pad); break;
            case 8: launch_bsr_t<8, BS, UP>(s, bcol, vals, invd, b, x, reset, done, st, pad); break;
            case 16: launch_bsr_t<16, BS, UP>(s, bcol, vals, invd, b, x, reset, done, st, pad); break;
            default: launch_bsr_t<32, BS, UP>(s, bcol, vals, invd, b, x, reset, done, st, pad); break;
            }
            return;
        }
    }
    if (rr) {
        switch (s.lanes) {
            case 4: launch_rr_t<4, BS, UP, 2>(s, M, vals, invd, b, x, reset, done, st); break;
            case 8: launch_rr_t<8, BS, UP, 1>(s, M, vals, invd, b, x, reset, done, st); break;
            case 16: launch_rr_t<16, BS, UP, 2>(s, M, vals, invd, b, x, reset, done, st); break;
            default: launch_rr_t<32, BS, UP, 4>(s, M, vals, invd, b, x, reset, done, st); break;
        }
        return;
    }
    switch (s.lanes) {
        case 4: launch_trsv_t<4, BS, UP>(s, M, vals, invd, b, x, reset, done, ctr, st); break;
        case 8: launch_trsv_t<8, BS, UP>(s, M, vals, invd, b, x, reset, done, ctr, st); break;
        case 16: launch_trsv_t<16, BS, UP>(s, M, vals, invd, b, x, reset, done, ctr, st); break;
        default: launch_trsv_t<32, BS, UP>(s, M, vals, invd, b, x, reset, done, ctr, st); break;
    }
}

// Launch one sweep; `ctr` must be zero on entry. Caller owns x (filled
// with kPending) and the optional reset buffer.
void launch_trsv(const Analysis& an, const double* vals, const double* invd, bool upper, const double* b, double* x,
                 double* reset, const int* done, unsigned* ctr, cudaStream_t st, bool pad) {
    const Schedule& s = upper ? an.blk_up : an.blk_lo;
    const DevCsr& M = upper ? an.upper : an.lower;
    const BlockCols* bcol = an.bsr ? &(upper ? an.ubc : an.lbc) : nullptr;  // node-blocked sweep
    if (s.nitems == 0) return;
    if (s.lanes != 4 && s.lanes != 8 && s.lanes != 16 && s.lanes != 32)
        throw CudaError("sweep schedule built for " + std::to_string(s.lanes) + " lanes per block");
    if (upper) {
        if (an.bs == 3) launch_trsv_bs<3, true>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
        else if (an.bs == 2) launch_trsv_bs<2, true>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
        else launch_trsv_bs<1, true>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
    } else {
        if (an.bs == 3) launch_trsv_bs<3, false>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
        else if (an.bs == 2) launch_trsv_bs<2, false>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
        else launch_trsv_bs<1, false>(s, M, an.rr, bcol, vals, invd, b, x, reset, done, ctr, st, pad);
    }
    CK_LAUNCH();
}

// One sweep of a preconditioner: on the item-ordered streams / slot records
// (bss.cu) when they exist, else the round-robin sweeps above on the L / U CSR.
void launch_sweep(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                  const int* done, unsigned* ctr, cudaStream_t st, bool pad) {
    if (launch_bss(an, p, upper, b, x, reset, done, st, pad)) return;
    launch_trsv(an, upper ? p.uvals.p : p.lvals.p, p.invd.p, upper, b, x, reset, done, ctr, st, pad);
}

void trsv(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, cudaStream_t st) {
    DevBuf<unsigned> ctr(1);
    CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned), st));
    fill_pending(x, an.lower.n, st);
    // 3x3 node-blocked sweeps run on the padded layout of the PCG loop
    // (4 doubles per node: 256-bit polls / publications): the right-hand
    // side of the backward sweep and the output go through padded copies
    const bool pad = an.bsr && an.bs == 3;
    if (pad) {
        const int64_t n = an.lower.n, n4 = 4 * (n / 3);
        DevBuf<double> x4(n4), b4;
        fill_pending(x4.p, n4, st);
        if (upper) {
            b4.alloc(n4);
            CK(cudaMemsetAsync(b4.p, 0, b4.bytes(), st));
            pad_copy_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, b, b4.p, true);
            CK_LAUNCH();
        }
        launch_sweep(an, p, upper, upper ? b4.p : b, x4.p, nullptr, nullptr, ctr.p, st, true);
        pad_copy_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, x4.p, x, false);
        CK_LAUNCH();
        CK(cudaStreamSynchronize(st));
        return;
    }
    launch_sweep(an, p, upper, b, x, nullptr, nullptr, ctr.p, st, false);
    CK(cudaStreamSynchronize(st));
}

__global__ void invd_kernel(int64_t n, const int64_t* __restrict__ lrp, const double* __restrict__ l,
                            double* __restrict__ invd) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) invd[i] = 1.0 / l[lrp[i + 1] - 1];
}

void reciprocal_diag(const Analysis& an, const double* lvals, double* invd, cudaStream_t st) {
    const int64_t n = an.lower.n;
    if (n == 0) return;
    invd_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, an.lower.rp.p, lvals, invd);
    CK_LAUNCH();
}

}  // namespace pclab_b200
