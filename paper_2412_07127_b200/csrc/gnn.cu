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

namespace pclab_b200 {

namespace {

constexpr int kF = 9, kH = 8;
__constant__ double c_p[997];

struct MlpOff {
    int w1, b1, w2, b2, in, out;
};
// ParamLayout (src/gnn.cpp:14-41)
struct Layout {
    MlpOff edge[3], node[3];
};
Layout make_layout() {
    Layout L{};
    int off = 18;
    const int ein[3] = {1 + 2 * kF, 2 + 2 * kH, 2 + 2 * kH};
    const int nin[3] = {kF + 2, kH + 2, kH + 2};
    for (int b = 0; b < 3; ++b) {
        MlpOff* ms[2] = {&L.edge[b], &L.node[b]};
        const int ins[2] = {ein[b], nin[b]};
        const int outs[2] = {1, kH};
        for (int t = 0; t < 2; ++t) {
            ms[t]->in = ins[t];
            ms[t]->out = outs[t];
            ms[t]->w1 = off;
            off += kH * ins[t];
            ms[t]->b1 = off;
            off += kH;
            ms[t]->w2 = off;
            off += outs[t] * kH;
            ms[t]->b2 = off;
            off += outs[t];
        }
    }
    return L;
}

// y = W2 tanh(W1 x + b1) + b2 (mlp_apply, src/gnn.cpp:43-57)
template <int IN, int OUT>
__device__ __forceinline__ void mlp(const MlpOff m, const double* x, double* y) {
    double hid[kH];
#pragma unroll
    for (int h = 0; h < kH; ++h) {
        double acc = c_p[m.b1 + h];
#pragma unroll
        for (int i = 0; i < IN; ++i) acc = fma(c_p[m.w1 + h * IN + i], x[i], acc);
        hid[h] = tanh(acc);
    }
#pragma unroll
    for (int o = 0; o < OUT; ++o) {
        double acc = c_p[m.b2 + o];
#pragma unroll
        for (int h = 0; h < kH; ++h) acc = fma(c_p[m.w2 + o * kH + h], hid[h], acc);
        y[o] = acc;
    }
}

// ---------------------------------------------------------------- features
__global__ void degree_kernel(int64_t n, const int64_t* __restrict__ rp,
                              const int64_t* __restrict__ dpos, double* __restrict__ deg) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) deg[i] = static_cast<double>(rp[i + 1] - rp[i] - (dpos[i] >= 0 ? 1 : 0));
}

__global__ void features_kernel(int64_t n, const int64_t* __restrict__ rp,
                                const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                const double* __restrict__ deg, double* __restrict__ f) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double diag = 0.0, osum = 0.0, omax = 0.0, mx = 0.0, mn = 1e300, mean = 0.0;
    int cnt = 0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        const double av = fabs(vals[k]);
        if (cols[k] == i) {
            diag = av;
            continue;
        }
        osum += av;
        omax = fmax(omax, av);
        const double d = deg[cols[k]];
        mx = fmax(mx, d);
        mn = fmin(mn, d);
        mean += d;
        ++cnt;
    }
    double* row = f + i * kF;
    row[0] = deg[i];
    row[1] = row[2] = row[3] = row[4] = 0.0;
    if (cnt > 0) {
        mean /= static_cast<double>(cnt);
        double var = 0.0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (cols[k] == i) continue;
            const double dd = deg[cols[k]] - mean;
            var += dd * dd;
        }
        row[1] = mx;
        row[2] = mn;
        row[3] = mean;
        row[4] = var / static_cast<double>(cnt);
    }
    const double denom = diag + osum;
    row[5] = denom > 0.0 ? diag / denom : 0.0;
    row[6] = omax > 0.0 ? fmin(fmax(diag / omax, 0.0), 100.0) : 100.0;
    const double angle = 2.0 * 3.14159265358979323846 * static_cast<double>(i) / static_cast<double>(n);
    double sn, cs;
    sincos(angle, &sn, &cs);
    row[7] = sn;
    row[8] = cs;
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
// Edge updater: lane group of G lanes per row, lanes over the row's edges.
template <int XW, bool FIRST, int G>
__global__ void __launch_bounds__(256)
edge_kernel(int64_t n, MlpOff m, const int64_t* __restrict__ lrp, const int32_t* __restrict__ lcols,
            const double* __restrict__ x, const double* __restrict__ ef,
            const double* __restrict__ eprev, double* __restrict__ eout, int* __restrict__ bad) {
    constexpr int IN = (FIRST ? 1 : 2) + 2 * XW;
    const int64_t gid = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / G;
    const int gl = threadIdx.x % G;
    const int64_t ngroups = static_cast<int64_t>(gridDim.x) * blockDim.x / G;
    bool nonfinite = false;
    for (int64_t i = gid; i < n; i += ngroups) {
        double xi[XW];
#pragma unroll
        for (int c = 0; c < XW; ++c) xi[c] = x[i * XW + c];
        for (int64_t k = lrp[i] + gl; k < lrp[i + 1]; k += G) {
            const int32_t j = lcols[k];
            double in[IN];
            int w = 0;
            if (!FIRST) in[w++] = eprev[k];
            in[w++] = ef[k];
#pragma unroll
            for (int c = 0; c < XW; ++c) in[w + c] = xi[c];
#pragma unroll
            for (int c = 0; c < XW; ++c) in[w + XW + c] = x[static_cast<int64_t>(j) * XW + c];
            double y;
            mlp<IN, 1>(m, in, &y);
            eout[k] = y;
            nonfinite |= !isfinite(y);
        }
    }
    if (nonfinite) *bad = 1;
}

// Node updater with the fused sum/mean aggregation.
template <int XW>
__global__ void __launch_bounds__(256)
node_kernel(int64_t n, MlpOff m, const int64_t* __restrict__ lrp, const int64_t* __restrict__ urp,
            const int64_t* __restrict__ u2l, const double* __restrict__ cnt,
            const double* __restrict__ x, const double* __restrict__ e, double* __restrict__ xo,
            int* __restrict__ bad) {
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
    mlp<XW + 2, kH>(m, in, y);
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

template <int XW, bool FIRST>
void launch_edge(int G, unsigned grid, cudaStream_t st, int64_t n, MlpOff m, const int64_t* lrp,
                 const int32_t* lcols, const double* x, const double* ef, const double* eprev,
                 double* eout, int* bad) {
    switch (G) {
        case 4: edge_kernel<XW, FIRST, 4><<<grid, 256, 0, st>>>(n, m, lrp, lcols, x, ef, eprev, eout, bad); break;
        case 8: edge_kernel<XW, FIRST, 8><<<grid, 256, 0, st>>>(n, m, lrp, lcols, x, ef, eprev, eout, bad); break;
        case 16: edge_kernel<XW, FIRST, 16><<<grid, 256, 0, st>>>(n, m, lrp, lcols, x, ef, eprev, eout, bad); break;
        default: edge_kernel<XW, FIRST, 32><<<grid, 256, 0, st>>>(n, m, lrp, lcols, x, ef, eprev, eout, bad); break;
    }
    CK_LAUNCH();
}

}  // namespace

void gnn_forward(const Matrix& A, const Analysis& an, const Model& model, double* out,
                 double* sigma_out, cudaStream_t st) {
    const Layout ly = make_layout();
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
    features_kernel<<<gfor(n, T), T, 0, st>>>(n, A.a.rp.p, A.a.cols.p, A.a.vals.p, deg.p, feat.p);
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
    const double avg = static_cast<double>(ne) / static_cast<double>(n);
    int G = 4;
    while (G < 32 && G < avg) G *= 2;
    const unsigned egrid = static_cast<unsigned>(sm_count() * 16);
    DevBuf<double> e1(ne), e2(ne), xa(n * kH), xb(n * kH);
    DevBuf<int> bad(6);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int) * 6, st));
    launch_edge<kF, true>(G, egrid, st, n, ly.edge[0], L.rp.p, L.cols.p, x0.p, ef.p, nullptr, e1.p, bad.p);
    node_kernel<kF><<<gfor(n, T), T, 0, st>>>(n, ly.node[0], L.rp.p, U.rp.p, an.u2l.p, cnt.p, x0.p, e1.p,
                                               xa.p, bad.p + 1);
    CK_LAUNCH();
    launch_edge<kH, false>(G, egrid, st, n, ly.edge[1], L.rp.p, L.cols.p, xa.p, ef.p, e1.p, e2.p, bad.p + 2);
    node_kernel<kH><<<gfor(n, T), T, 0, st>>>(n, ly.node[1], L.rp.p, U.rp.p, an.u2l.p, cnt.p, xa.p, e2.p,
                                               xb.p, bad.p + 3);
    CK_LAUNCH();
    launch_edge<kH, false>(G, egrid, st, n, ly.edge[2], L.rp.p, L.cols.p, xb.p, ef.p, e2.p, out, bad.p + 4);
    // the final node state feeds nothing (gnn.cpp:199-205 computes it and
    // checks it for finiteness)
    node_kernel<kH><<<gfor(n, T), T, 0, st>>>(n, ly.node[2], L.rp.p, U.rp.p, an.u2l.p, cnt.p, xb.p, out,
                                               xa.p, bad.p + 5);
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
