// GNN forward pass over the lower-triangle graph of A (reference:
// build_graph src/features.cpp:74-84, node_features src/features.cpp:11-72,
// scale_by_std src/sparse.cpp:206-224, gnn_forward src/gnn.cpp:127-219).
//
// Node state and edge features live in HBM; the 997 parameters live in
// constant memory (every lane reads the same weight: broadcast). The
// hidden width is 8, so each MLP is a handful of CUDA-core fp64 FMAs per
// edge -- there is no dense contraction for the tensor cores. The
// message aggregation is a deterministic CSR-segmented sum: node v sums
// its L row (columns <= v) and then its U row (columns > v, through the
// U->L slot map), which is exactly the reference's accumulation order
// over the edge list; no atomics anywhere.
#include "core.h"
#include "gnn_math.cuh"

namespace pclab_b200 {

namespace {

constexpr int kF = 9, kH = 8;
__constant__ double c_p[997];

// ParamLayout (src/gnn.cpp:14-41) as compile-time offsets: block b holds
// the edge MLP (in -> kH -> 1) then the node MLP (in -> kH -> kH), each as
// W1 [kH x in], b1 [kH], W2 [out x kH], b2 [out], after 18 leading entries.
// With constant offsets every weight is a direct constant-bank operand of
// its FMA (no address arithmetic, no LDC per weight).
constexpr int edge_in(int b) { return b == 0 ? 1 + 2 * kF : 2 + 2 * kH; }
constexpr int node_in(int b) { return b == 0 ? kF + 2 : kH + 2; }
constexpr int mlp_size(int in, int out) { return kH * in + kH + out * kH + out; }
constexpr int edge_off(int b) {
    int off = 18;
    for (int i = 0; i < b; ++i) off += mlp_size(edge_in(i), 1) + mlp_size(node_in(i), kH);
    return off;
}
constexpr int node_off(int b) { return edge_off(b) + mlp_size(edge_in(b), 1); }
static_assert(node_off(2) + mlp_size(node_in(2), kH) == 997, "parameter layout");

// y = W2 tanh(W1 x + b1) + b2 (mlp_apply, src/gnn.cpp:43-57), same
// accumulation order as the reference (bias first, then inputs in order)
template <int OFF, int IN, int OUT>
__device__ __forceinline__ void mlp(const double* x, double* y) {
    constexpr int W1 = OFF, B1 = OFF + kH * IN, W2 = B1 + kH, B2 = W2 + OUT * kH;
    // inputs outer, hidden units inner: kH independent FMA chains (each in
    // the reference's order: bias, then inputs 0..IN-1), every input
    // consumed once -- no input vector kept live across the hidden units
    double hid[kH];
#pragma unroll
    for (int h = 0; h < kH; ++h) hid[h] = c_p[B1 + h];
#pragma unroll
    for (int i = 0; i < IN; ++i)
#pragma unroll
        for (int h = 0; h < kH; ++h) hid[h] = fma(c_p[W1 + h * IN + i], x[i], hid[h]);
#pragma unroll
    for (int h = 0; h < kH; ++h) hid[h] = tanh_nb(hid[h]);
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
        double acc = c_p[B2 + o];
#pragma unroll
        for (int h = 0; h < kH; ++h) acc = fma(c_p[W2 + o * kH + h], hid[h], acc);
        y[o] = acc;
    }
}

// ---------------------------------------------------------------- features
__global__ void degree_kernel(int64_t n, const int64_t* __restrict__ rp,
                              const int64_t* __restrict__ dpos, double* __restrict__ deg) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) deg[i] = static_cast<double>(rp[i + 1] - rp[i] - (dpos[i] >= 0 ? 1 : 0));
}

// FL lanes per row (lanes over the entries, coalesced; 32 / FL rows per
// warp): diagonal, |off| sum and max, neighbour-degree max / min / mean,
// then their variance from the row's entries again (L1-resident). Sums are
// fixed shuffle trees (the reference adds in entry order; the features
// differ from it by rounding only, and the degrees and their mean are
// exact integers / quotients). Measured on configs[2] (81 entries per row):
// 32 lanes per row 4.4 ms (issue-bound on the per-row reductions and tail).
constexpr int FL = 8;
__global__ void __launch_bounds__(256)
features_kernel(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                const double* __restrict__ vals, const double* __restrict__ deg, double* __restrict__ f) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / FL;
    const int gl = threadIdx.x % FL;
    const bool act = i < n;
    const int64_t b = act ? rp[i] : 0, e = act ? rp[i + 1] : 0;
    double diag = 0.0, osum = 0.0, omax = 0.0, mx = 0.0, mn = 1e300, dsum = 0.0;
    int cnt = 0;
    for (int64_t k = b + gl; k < e; k += FL) {
        const double av = fabs(vals[k]);
        const int32_t j = cols[k];
        if (j == i) {
            diag = av;
            continue;
        }
        osum += av;
        omax = fmax(omax, av);
        const double d = deg[j];
        mx = fmax(mx, d);
        mn = fmin(mn, d);
        dsum += d;
        ++cnt;
    }
#pragma unroll
    for (int o = FL / 2; o > 0; o >>= 1) {
        diag += __shfl_xor_sync(0xffffffffu, diag, o, FL);  // one lane holds it
        osum += __shfl_xor_sync(0xffffffffu, osum, o, FL);
        omax = fmax(omax, __shfl_xor_sync(0xffffffffu, omax, o, FL));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o, FL));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o, FL));
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o, FL);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o, FL);
    }
    const double mean = cnt > 0 ? dsum / static_cast<double>(cnt) : 0.0;
    double var = 0.0;
    if (cnt > 0)
        for (int64_t k = b + gl; k < e; k += FL) {
            const int32_t j = cols[k];
            if (j == i) continue;
            const double dd = deg[j] - mean;
            var += dd * dd;
        }
    var = group_sum<FL>(var);
    if (act && gl == 0) {
        double* row = f + i * kF;
        row[0] = deg[i];
        row[1] = cnt > 0 ? mx : 0.0;
        row[2] = cnt > 0 ? mn : 0.0;
        row[3] = mean;
        row[4] = cnt > 0 ? var / static_cast<double>(cnt) : 0.0;
        const double denom = diag + osum;
        row[5] = denom > 0.0 ? diag / denom : 0.0;
        row[6] = omax > 0.0 ? fmin(fmax(diag / omax, 0.0), 100.0) : 100.0;
        const double angle = 2.0 * 3.14159265358979323846 * static_cast<double>(i) / static_cast<double>(n);
        double sn, cs;
        sincos(angle, &sn, &cs);
        row[7] = sn;
        row[8] = cs;
    }
}

// Deterministic column sums of an n x W row-major array (fixed grid, fixed
// tree): stage 1 per-block partials, stage 2 one block sums them in order.
template <int W, bool SQDEV>
__global__ void colsum_partial(int64_t n, const double* __restrict__ a, const double* __restrict__ mu,
                               double* __restrict__ part) {
    __shared__ double sm[W][8];
    double acc[W];
#pragma unroll
    for (int c = 0; c < W; ++c) acc[c] = 0.0;
    for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
        for (int c = 0; c < W; ++c) {
            const double x = a[v * W + c];
            acc[c] += SQDEV ? (x - mu[c]) * (x - mu[c]) : x;
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int c = 0; c < W; ++c) {
        const double s = group_sum<32>(acc[c]);
        if (lane == 0) sm[c][wid] = s;
    }
    __syncthreads();
    if (threadIdx.x < W) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sm[threadIdx.x][w];
        part[blockIdx.x * W + threadIdx.x] = s;
    }
}

template <int W>
__global__ void colsum_final(int nparts, const double* __restrict__ part, double* __restrict__ out,
                             double scale) {
    if (threadIdx.x < W) {
        double s = 0.0;
        for (int b = 0; b < nparts; ++b) s += part[b * W + threadIdx.x];
        out[threadIdx.x] = s * scale;
    }
}

__global__ void normalize_kernel(int64_t n, const double* __restrict__ f, const double* __restrict__ mu,
                                 const double* __restrict__ var, double* __restrict__ x0) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n * kF) return;
    const int c = static_cast<int>(i % kF);
    const double inv = 1.0 / (sqrt(var[c]) + 1e-6);
    const double xh = (f[i] - mu[c]) * inv;
    x0[i] = c_p[c] * xh + c_p[kF + c];
}

// edge-feature scale: sd of the lower values and max|v|
__global__ void absmax_kernel(int64_t m, const double* __restrict__ v, unsigned long long* out) {
    unsigned long long best = 0;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < m;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        best = max(best, static_cast<unsigned long long>(__double_as_longlong(fabs(v[k]))));
    atomicMax(out, best);
}

__global__ void scale_kernel(int64_t m, const double* __restrict__ v, const double* __restrict__ sd,
                             double* __restrict__ out) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k < m) out[k] = v[k] / sd[0];
}

__global__ void count_kernel(int64_t n, const int64_t* __restrict__ lrp, const int64_t* __restrict__ urp,
                             double* __restrict__ cnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) cnt[i] = static_cast<double>((lrp[i + 1] - lrp[i]) + (urp[i + 1] - urp[i]) - 1);
}

// ------------------------------------------------------------ message passing
// Row index of every L entry (the edge's target node), for the flat edge
// kernel: one warp per row writes its entries.
__global__ void edge_rows_kernel(int64_t n, const int64_t* __restrict__ lrp, int32_t* __restrict__ erow) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (i >= n) return;
    for (int64_t k = lrp[i] + (threadIdx.x & 31); k < lrp[i + 1]; k += 32) erow[k] = static_cast<int32_t>(i);
}

// First layer of the edge MLP split by operand: the terms of the node
// states x_i and x_j depend on one node each, so every node gets its two
// projections once (16 values: pq[v] = {W1_i x_v, W1_j x_v}) and an edge
// adds them instead of redoing 2 x 8 x XW FMAs (the reference sums bias,
// then inputs in order; this is the same sum regrouped -- rounding-level
// differences, held to the 1e-5 bar).
template <int BLK>
__global__ void __launch_bounds__(256)
node_proj_kernel(int64_t n, const double* __restrict__ x, double* __restrict__ pq) {
    constexpr bool FIRST = BLK == 0;
    constexpr int XW = FIRST ? kF : kH;
    constexpr int IN = edge_in(BLK);
    constexpr int W1 = edge_off(BLK);
    constexpr int I0 = FIRST ? 1 : 2;  // first x_i input
    const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= n) return;
    double xv[XW];
#pragma unroll
    for (int c = 0; c < XW; ++c) xv[c] = x[v * XW + c];
    double p[kH], q[kH];
#pragma unroll
    for (int h = 0; h < kH; ++h) {
        p[h] = 0.0;
        q[h] = 0.0;
    }
#pragma unroll
    for (int c = 0; c < XW; ++c)
#pragma unroll
        for (int h = 0; h < kH; ++h) {
            p[h] = fma(c_p[W1 + h * IN + I0 + c], xv[c], p[h]);
            q[h] = fma(c_p[W1 + h * IN + I0 + XW + c], xv[c], q[h]);
        }
    double2* o = reinterpret_cast<double2*>(pq + v * 2 * kH);
#pragma unroll
    for (int h = 0; h < kH; h += 2) {
        o[h / 2] = make_double2(p[h], p[h + 1]);
        o[kH / 2 + h / 2] = make_double2(q[h], q[h + 1]);
    }
}

// Edge updater: one thread per edge of the flat L entry list (every lane
// busy whatever the row lengths), edge (i, j) = (erow[k], lcols[k]):
// hidden = b1 + w_prev e_prev + w_f f + (W1_i x_i) + (W1_j x_j), tanh, the
// output layer. Consecutive edges share their row, so the x_i projection
// is an L1 broadcast; the x_j projection is an L2-resident gather.
template <int BLK>
__global__ void __launch_bounds__(256)
edge_kernel(int64_t ne, const int32_t* __restrict__ erow, const int32_t* __restrict__ lcols,
            const double* __restrict__ pq, const double* __restrict__ ef, const double* __restrict__ eprev,
            double* __restrict__ eout, int* __restrict__ bad) {
    constexpr bool FIRST = BLK == 0;
    constexpr int IN = edge_in(BLK);
    constexpr int W1 = edge_off(BLK), B1 = W1 + kH * IN, W2 = B1 + kH, B2 = W2 + kH;
    bool nonfinite = false;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < ne;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = erow[k], j = lcols[k];
        const double fk = ef[k];
        const double pk = FIRST ? 0.0 : eprev[k];
        const double2* pi = reinterpret_cast<const double2*>(pq + i * 2 * kH);
        const double2* qj = reinterpret_cast<const double2*>(pq + j * 2 * kH) + kH / 2;
        double hid[kH];
#pragma unroll
        for (int h = 0; h < kH; h += 2) {
            const double2 a = pi[h / 2], b = qj[h / 2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                double t = c_p[B1 + h + u];
                if (!FIRST) t = fma(c_p[W1 + (h + u) * IN], pk, t);
                t = fma(c_p[W1 + (h + u) * IN + (FIRST ? 0 : 1)], fk, t);
                hid[h + u] = tanh_nb(t + (u ? a.y : a.x) + (u ? b.y : b.x));
            }
        }
        double y = c_p[B2];
#pragma unroll
        for (int h = 0; h < kH; ++h) y = fma(c_p[W2 + h], hid[h], y);
        eout[k] = y;
        nonfinite |= !isfinite(y);
    }
    if (nonfinite) *bad = 1;
}

// Node updater with the fused sum/mean aggregation.
template <int BLK>
__global__ void __launch_bounds__(256)
node_kernel(int64_t n, const int64_t* __restrict__ lrp, const int64_t* __restrict__ urp,
            const int64_t* __restrict__ u2l, const double* __restrict__ cnt,
            const double* __restrict__ x, const double* __restrict__ e, double* __restrict__ xo,
            int* __restrict__ bad) {
    constexpr int XW = BLK == 0 ? kF : kH;
    const int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (v >= n) return;
    double s = 0.0;
    for (int64_t k = lrp[v]; k < lrp[v + 1]; ++k) s += e[k];
    for (int64_t t = urp[v] + 1; t < urp[v + 1]; ++t) s += e[u2l[t]];
    double in[XW + 2];
#pragma unroll
    for (int c = 0; c < XW; ++c) in[c] = x[v * XW + c];
    in[XW] = s;
    in[XW + 1] = cnt[v] > 0.0 ? s / cnt[v] : 0.0;
    double y[kH];
    mlp<node_off(BLK), node_in(BLK), kH>(in, y);
    bool nonfinite = false;
#pragma unroll
    for (int h = 0; h < kH; ++h) {
        xo[v * kH + h] = y[h];
        nonfinite |= !isfinite(y[h]);
    }
    if (nonfinite) *bad = 1;
}

// Diagonal outputs pass through o -> exp(o / 2) (src/gnn.cpp:215-217).
__global__ void output_kernel(int64_t n, const int64_t* __restrict__ lrp, double* __restrict__ e) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) {
        const int64_t d = lrp[i + 1] - 1;
        e[d] = exp(e[d] / 2.0);
    }
}

inline unsigned gfor(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

template <int BLK>
void launch_edge(int64_t n, int64_t ne, const int32_t* erow, const int32_t* lcols, const double* x, double* pq,
                 const double* ef, const double* eprev, double* eout, int* bad, cudaStream_t st) {
    node_proj_kernel<BLK><<<gfor(n, 256), 256, 0, st>>>(n, x, pq);
    CK_LAUNCH();
    static unsigned grid = 0;
    if (!grid) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, edge_kernel<BLK>, 256, 0));
        grid = static_cast<unsigned>(std::max(per_sm, 1) * sm_count() * 4);
    }
    edge_kernel<BLK><<<grid, 256, 0, st>>>(ne, erow, lcols, pq, ef, eprev, eout, bad);
    CK_LAUNCH();
}

}  // namespace

void gnn_forward(const Matrix& A, const Analysis& an, const Model& model, double* out,
                 double* sigma_out, cudaStream_t st) {
    if (model.params.size() != 997) throw DimensionError("gnn: parameter vector has wrong length");
    CK(cudaMemcpyToSymbolAsync(c_p, model.params.data(), sizeof(double) * 997, 0,
                               cudaMemcpyHostToDevice, st));
    const int64_t n = A.a.n;
    const DevCsr& L = an.lower;
    const DevCsr& U = an.upper;
    const int64_t ne = L.nnz;
    if (n == 0) {
        *sigma_out = 1.0;
        return;
    }
    const int T = 256;
    // ---- node features (features.cpp:11-72)
    DevBuf<double> deg(n), feat(n * kF), x0(n * kF), cnt(n);
    degree_kernel<<<gfor(n, T), T, 0, st>>>(n, A.a.rp.p, A.diag_pos.p, deg.p);
    features_kernel<<<gfor(n * FL, T), T, 0, st>>>(n, A.a.rp.p, A.a.cols.p, A.a.vals.p, deg.p, feat.p);
    CK_LAUNCH();
    // ---- graph normalisation statistics (gnn.cpp:141-160)
    const int parts = sm_count() * 2;
    DevBuf<double> part(parts * kF), stats(2 * kF + 4);
    double* mu = stats.p;
    double* var = stats.p + kF;
    colsum_partial<kF, false><<<parts, T, 0, st>>>(n, feat.p, nullptr, part.p);
    colsum_final<kF><<<1, 32, 0, st>>>(parts, part.p, mu, 1.0 / static_cast<double>(n));
    colsum_partial<kF, true><<<parts, T, 0, st>>>(n, feat.p, mu, part.p);
    colsum_final<kF><<<1, 32, 0, st>>>(parts, part.p, var, 1.0 / static_cast<double>(n));
    normalize_kernel<<<gfor(n * kF, T), T, 0, st>>>(n, feat.p, mu, var, x0.p);
    CK_LAUNCH();
    // ---- edge features: lower values scaled by their population sd
    //      (scale_by_std, sparse.cpp:206-224)
    DevBuf<double> ef(ne);
    double* emean = stats.p + 2 * kF;
    double* evar = stats.p + 2 * kF + 1;
    DevBuf<double> epart(parts);
    colsum_partial<1, false><<<parts, T, 0, st>>>(ne, L.vals.p, nullptr, epart.p);
    colsum_final<1><<<1, 32, 0, st>>>(parts, epart.p, emean, 1.0 / static_cast<double>(ne));
    colsum_partial<1, true><<<parts, T, 0, st>>>(ne, L.vals.p, emean, epart.p);
    colsum_final<1><<<1, 32, 0, st>>>(parts, epart.p, evar, 1.0 / static_cast<double>(ne));
    DevBuf<unsigned long long> amax(1);
    CK(cudaMemsetAsync(amax.p, 0, sizeof(unsigned long long), st));
    absmax_kernel<<<parts, T, 0, st>>>(ne, L.vals.p, amax.p);
    CK_LAUNCH();
    double hv[2];
    unsigned long long am_bits = 0;
    CK(cudaMemcpyAsync(hv, emean, sizeof hv, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&am_bits, amax.p, sizeof am_bits, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double amx;
    memcpy(&amx, &am_bits, sizeof amx);
    const double sd = std::sqrt(hv[1]);
    double sigma = 1.0;
    if (sd <= 1e-13 * amx) {
        CK(cudaMemcpyAsync(ef.p, L.vals.p, sizeof(double) * ne, cudaMemcpyDeviceToDevice, st));
    } else {
        sigma = sd;
        CK(cudaMemcpyAsync(evar, &sigma, sizeof(double), cudaMemcpyHostToDevice, st));
        scale_kernel<<<gfor(ne, T), T, 0, st>>>(ne, L.vals.p, evar, ef.p);
        CK_LAUNCH();
    }
    *sigma_out = sigma;
    count_kernel<<<gfor(n, T), T, 0, st>>>(n, L.rp.p, U.rp.p, cnt.p);
    // ---- three message-passing blocks (gnn.cpp:162-205)
    DevBuf<int32_t> erow(ne);
    edge_rows_kernel<<<gfor(n * 32, T), T, 0, st>>>(n, L.rp.p, erow.p);
    CK_LAUNCH();
    DevBuf<double> e1(ne), e2(ne), xa(n * kH), xb(n * kH), pq(n * 2 * kH);
    DevBuf<int> bad(6);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int) * 6, st));
    launch_edge<0>(n, ne, erow.p, L.cols.p, x0.p, pq.p, ef.p, nullptr, e1.p, bad.p, st);
    node_kernel<0><<<gfor(n, T), T, 0, st>>>(n, L.rp.p, U.rp.p, an.u2l.p, cnt.p, x0.p, e1.p, xa.p, bad.p + 1);
    CK_LAUNCH();
    launch_edge<1>(n, ne, erow.p, L.cols.p, xa.p, pq.p, ef.p, e1.p, e2.p, bad.p + 2, st);
    node_kernel<1><<<gfor(n, T), T, 0, st>>>(n, L.rp.p, U.rp.p, an.u2l.p, cnt.p, xa.p, e2.p, xb.p, bad.p + 3);
    CK_LAUNCH();
    launch_edge<2>(n, ne, erow.p, L.cols.p, xb.p, pq.p, ef.p, e2.p, out, bad.p + 4, st);
    // the final node state feeds nothing (gnn.cpp:199-205 computes it and
    // checks it for finiteness)
    node_kernel<2><<<gfor(n, T), T, 0, st>>>(n, L.rp.p, U.rp.p, an.u2l.p, cnt.p, xb.p, out, xa.p, bad.p + 5);
    CK_LAUNCH();
    int hb[6];
    CK(cudaMemcpyAsync(hb, bad.p, sizeof hb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (int k = 0; k < 6; ++k)
        if (hb[k])
            throw NumericError(std::string("gnn forward: non-finite ") + (k % 2 ? "node" : "edge") +
                               " activation in block " + std::to_string(k / 2 + 1));
    output_kernel<<<gfor(n, T), T, 0, st>>>(n, L.rp.p, out);
    CK_LAUNCH();
}

}  // namespace pclab_b200
