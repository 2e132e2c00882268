// Item-ordered value streams of the node-blocked sweeps (bss_trsv_kernel,
// sweep.cuh): per slot of a sweep schedule (Schedule::slots, 2 blocks per
// warp item), a 16-byte header and the block's neighbour ids (per
// analysis), and the block's factor values re-laid block-major (per
// factor: a gather from the L / U values after every factor build).
#include "core.h"
#include "sweep.cuh"

namespace pclab_b200 {

#ifdef BSS_TRACE  // developer trace (tools/bss_trace.py): not in the product build
extern "C" int pclab_debug_bss_trace(void* p) {
    unsigned long long* q = static_cast<unsigned long long*>(p);
    return static_cast<int>(cudaMemcpyToSymbol(g_bss_trace, &q, sizeof(q)));
}
#endif

namespace {

inline unsigned gridn(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__global__ void bss_lengths(int64_t ns, const int32_t* __restrict__ slots, const int64_t* __restrict__ bp,
                            int64_t* __restrict__ lv, int64_t* __restrict__ lc) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s > ns) return;
    if (s == ns) {
        lv[s] = lc[s] = 0;
        return;
    }
    const int32_t b = slots[s];
    const int64_t nb = b >= 0 ? bp[b + 1] - bp[b] : 0;
    lv[s] = b >= 0 ? 9 * nb + 6 : 0;
    lc[s] = nb;
}

// headers and neighbour block ids (warp per slot)
__global__ void bss_headers(int64_t ns, const int32_t* __restrict__ slots, const int64_t* __restrict__ bp,
                            const int32_t* __restrict__ bcol, const int64_t* __restrict__ voff,
                            const int64_t* __restrict__ coff, int4* __restrict__ hdr, int32_t* __restrict__ scol) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int32_t b = slots[s];
    const int64_t nb = b >= 0 ? bp[b + 1] - bp[b] : 0;
    if (lane == 0)
        hdr[s] = make_int4(b, static_cast<int>(nb), static_cast<int>(static_cast<uint32_t>(voff[s])),
                           static_cast<int>(static_cast<uint32_t>(coff[s])));
    for (int64_t n = lane; n < nb; n += 32) scol[coff[s] + n] = bcol[bp[b] + n] / 3;
}

// values of one slot (warp per slot): entry (t, c) of neighbour n's 3x3
// block at (3t + c) * nb + n -- entry-major, so the sweep's 16 lanes (one
// neighbour each) read consecutive doubles with every load -- then the
// in-block entries in solve_diag_block's order, then 1 / l_tt
template <bool UPPER>
__global__ void bss_values(int64_t ns, const int4* __restrict__ hdr, const int64_t* __restrict__ rp,
                           const double* __restrict__ vals, const double* __restrict__ invd,
                           double* __restrict__ sval) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int4 h = hdr[s];
    if (h.x < 0) return;
    const int64_t b = h.x;
    const int nb = h.y;
    double* v = sval + static_cast<uint32_t>(h.z);
    for (int idx = lane; idx < 9 * nb; idx += 32) {
        const int n = idx / 9, w = idx % 9, t = w / 3, c = w % 3;
        v[w * nb + n] = vals[rp[3 * b + t] + (UPPER ? 3 - t : 0) + 3 * n + c];
    }
    if (lane == 0) {
        double* d = v + 9 * nb;
        int q = 0;
#pragma unroll
        for (int t = 0; t < 3; ++t)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (!UPPER && c < t) d[q++] = vals[rp[3 * b + t + 1] - (t + 1) + c];
                if (UPPER && c > t) d[q++] = vals[rp[3 * b + t] + (c - t)];
            }
#pragma unroll
        for (int t = 0; t < 3; ++t) d[3 + t] = invd[3 * b + t];
    }
}

// ---- scalar (entry-lane) slots: block rows r0 .. r0+bs-1 of L (diagonal
// last) or U (diagonal first); a slot's off-block entries in row order
__device__ __forceinline__ void slot_rows_of(const int64_t* rp, int64_t b, int bs, bool upper, int64_t* ob, int* oc) {
    for (int t = 0; t < bs; ++t) {
        const int64_t r = b * bs + t;
        ob[t] = upper ? rp[r] + (bs - t) : rp[r];
        oc[t] = static_cast<int>(upper ? rp[r + 1] - ob[t] : rp[r + 1] - (t + 1) - rp[r]);
    }
}

__global__ void rrs_lengths(int64_t ns, int bs, bool upper, const int32_t* __restrict__ slots,
                            const int64_t* __restrict__ rp, int64_t* __restrict__ lv, int64_t* __restrict__ lc) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s > ns) return;
    if (s == ns) {
        lv[s] = lc[s] = 0;
        return;
    }
    const int32_t b = slots[s];
    int64_t ob[3];
    int oc[3], tot = 0;
    if (b >= 0) {
        slot_rows_of(rp, b, bs, upper, ob, oc);
        for (int t = 0; t < bs; ++t) tot += oc[t];
    }
    lv[s] = b >= 0 ? tot + bs * (bs - 1) / 2 + bs : 0;
    lc[s] = tot;
}

__global__ void rrs_headers(int64_t ns, int bs, bool upper, const int32_t* __restrict__ slots,
                            const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                            const int64_t* __restrict__ voff, const int64_t* __restrict__ coff,
                            int4* __restrict__ hdr, int32_t* __restrict__ code) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int32_t b = slots[s];
    int64_t ob[3];
    int oc[3], tot = 0;
    if (b >= 0) {
        slot_rows_of(rp, b, bs, upper, ob, oc);
        for (int t = 0; t < bs; ++t) tot += oc[t];
    }
    if (lane == 0)
        hdr[s] = make_int4(b, tot, static_cast<int>(static_cast<uint32_t>(voff[s])),
                           static_cast<int>(static_cast<uint32_t>(coff[s])));
    int base = 0;
    for (int t = 0; t < bs && b >= 0; ++t) {
        for (int e = lane; e < oc[t]; e += 32) code[coff[s] + base + e] = (cols[ob[t] + e] << 2) | t;
        base += oc[t];
    }
}

template <bool UPPER>
__global__ void rrs_values(int64_t ns, int bs, const int4* __restrict__ hdr, const int64_t* __restrict__ rp,
                           const double* __restrict__ vals, const double* __restrict__ invd,
                           double* __restrict__ sval) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int4 h = hdr[s];
    if (h.x < 0) return;
    const int64_t b = h.x;
    int64_t ob[3];
    int oc[3];
    slot_rows_of(rp, b, bs, UPPER, ob, oc);
    double* v = sval + static_cast<uint32_t>(h.z);
    int base = 0;
    for (int t = 0; t < bs; ++t) {
        for (int e = lane; e < oc[t]; e += 32) v[base + e] = vals[ob[t] + e];
        base += oc[t];
    }
    if (lane == 0) {
        double* d = v + base;
        int q = 0;
        for (int t = 0; t < bs; ++t)
            for (int c = 0; c < bs; ++c) {
                if (!UPPER && c < t) d[q++] = vals[rp[b * bs + t + 1] - (t + 1) + c];
                if (UPPER && c > t) d[q++] = vals[rp[b * bs + t] + (c - t)];
            }
        for (int t = 0; t < bs; ++t) d[q + t] = invd[b * bs + t];
    }
}

__global__ void slot_max_entries(int64_t ns, const int4* __restrict__ hdr, int* __restrict__ mx) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    int v = s < ns && hdr[s].x >= 0 ? hdr[s].y : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0 && v > 0) atomicMax(mx, v);
}

// one 128-byte record per slot from the slot's header, codes and values
// (16 doubles: 8 values, 8 int32 codes, in-block entry, 2 reciprocal pivots, block id)
__global__ void rec_pack(int64_t ns, const int4* __restrict__ hdr, const int32_t* __restrict__ scode,
                         const double* __restrict__ sval, double* __restrict__ rec) {
    const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (idx >= 16 * ns) return;
    const int64_t s = idx >> 4;
    const int j = static_cast<int>(idx & 15);
    const int4 h = hdr[s];
    const int total = h.x >= 0 ? h.y : 0;
    const double* v = sval + static_cast<uint32_t>(h.z);
    const int32_t* cd = scode + static_cast<uint32_t>(h.w);
    double o = 0.0;
    if (j < 8) {
        o = j < total ? v[j] : 0.0;
    } else if (j < 12) {
        const int c0 = 2 * (j - 8), c1 = c0 + 1;
        // unused lanes repeat entry 0's column (a poll of the same sector) with the ignore bit
        const int32_t idle = total > 0 ? (cd[0] & ~3) | 2 : 2;
        const uint32_t a = static_cast<uint32_t>(c0 < total ? cd[c0] : idle);
        const uint32_t b = static_cast<uint32_t>(c1 < total ? cd[c1] : idle);
        o = __longlong_as_double(static_cast<long long>(a | (static_cast<uint64_t>(b) << 32)));
    } else if (j < 15) {
        o = h.x >= 0 ? v[total + (j - 12)] : 0.0;
    } else {
        o = __longlong_as_double(static_cast<long long>(h.x));
    }
    rec[idx] = o;
}

bool rec_enabled() {
    static const bool on = !(getenv("PCLAB_REC") && atoi(getenv("PCLAB_REC")) == 0);
    return on;
}

void build_one_scalar(Schedule& s, const DevCsr& M, int bs, bool upper, cudaStream_t st) {
    s.bss = false;
    s.rec = false;
    const int64_t ns = s.nitems * s.per_item;
    if (ns == 0 || ns >= (1LL << 31) || bs > 3) return;
    DevBuf<int64_t> voff(ns + 1), coff(ns + 1);
    rrs_lengths<<<gridn(ns + 1, 256), 256, 0, st>>>(ns, bs, upper, s.slots.p, M.rp.p, voff.p, coff.p);
    CK_LAUNCH();
    scan_inplace(voff.p, ns + 1, st);
    scan_inplace(coff.p, ns + 1, st);
    const int64_t nv = dev_read(voff.p + ns, st), nc = dev_read(coff.p + ns, st);
    if (nv >= (1LL << 32) || nc >= (1LL << 32) || M.n >= (1LL << 29)) return;
    s.bss_hdr.alloc(ns);
    s.bss_col.alloc(std::max<int64_t>(nc, 1));
    rrs_headers<<<gridn(ns * 32, 256), 256, 0, st>>>(ns, bs, upper, s.slots.p, M.rp.p, M.cols.p, voff.p, coff.p,
                                                    s.bss_hdr.p, s.bss_col.p);
    CK_LAUNCH();
    s.bss_nvals = nv;
    s.bss = true;
    if (rec_enabled() && bs == 2 && s.lanes == 8 && s.per_item == 4) {
        DevBuf<int> mx(1);
        CK(cudaMemsetAsync(mx.p, 0, sizeof(int), st));
        slot_max_entries<<<gridn(ns, 256), 256, 0, st>>>(ns, s.bss_hdr.p, mx.p);
        CK_LAUNCH();
        s.rec = dev_read(mx.p, st) <= 8 && ns < (1LL << 30);
    }
}

void build_one(Schedule& s, const BlockCols& bc, cudaStream_t st) {
    s.bss = false;
    if (s.lanes != 16 || s.per_item != 2) return;
    const int64_t ns = s.nitems * s.per_item;
    if (ns == 0 || ns >= (1LL << 31)) return;
    DevBuf<int64_t> voff(ns + 1), coff(ns + 1);
    bss_lengths<<<gridn(ns + 1, 256), 256, 0, st>>>(ns, s.slots.p, bc.bp.p, voff.p, coff.p);
    CK_LAUNCH();
    scan_inplace(voff.p, ns + 1, st);
    scan_inplace(coff.p, ns + 1, st);
    const int64_t nv = dev_read(voff.p + ns, st), nc = dev_read(coff.p + ns, st);
    if (nv >= (1LL << 32) || nc >= (1LL << 32)) return;
    s.bss_hdr.alloc(ns);
    s.bss_col.alloc(std::max<int64_t>(nc, 1));
    bss_headers<<<gridn(ns * 32, 256), 256, 0, st>>>(ns, s.slots.p, bc.bp.p, bc.bcol.p, voff.p, coff.p,
                                                    s.bss_hdr.p, s.bss_col.p);
    CK_LAUNCH();
    s.bss_nvals = nv;
    s.bss = true;
}

}  // namespace

bool bss_enabled() {
    static const bool on = !(getenv("PCLAB_BSS") && atoi(getenv("PCLAB_BSS")) == 0);
    return on;
}

void build_bss(Analysis& an, cudaStream_t st) {
    an.blk_lo.bss = an.blk_up.bss = false;
    if (!bss_enabled()) return;
    if (an.bsr && an.bs == 3) {
        build_one(an.blk_lo, an.lbc, st);
        build_one(an.blk_up, an.ubc, st);
    } else if (!an.bsr && an.rr) {
        build_one_scalar(an.blk_lo, an.lower, an.bs, false, st);
        build_one_scalar(an.blk_up, an.upper, an.bs, true, st);
    }
    if (!(an.blk_lo.bss && an.blk_up.bss)) an.blk_lo.bss = an.blk_up.bss = false;
    if (!(an.blk_lo.bss && an.blk_lo.rec && an.blk_up.rec)) an.blk_lo.rec = an.blk_up.rec = false;
}

void fill_bss(const Analysis& an, Precond& p, cudaStream_t st) {
    if (!an.blk_lo.bss) return;
    for (int up = 0; up < 2; ++up) {
        const Schedule& s = up ? an.blk_up : an.blk_lo;
        DevBuf<double>& out = up ? p.bss_up : p.bss_lo;
        out.alloc(std::max<int64_t>(s.bss_nvals, 1));
        const int64_t ns = s.nitems * s.per_item;
        if (!an.bsr) {
            if (up)
                rrs_values<true><<<gridn(ns * 32, 256), 256, 0, st>>>(ns, an.bs, s.bss_hdr.p, an.upper.rp.p,
                                                                     p.uvals.p, p.invd.p, out.p);
            else
                rrs_values<false><<<gridn(ns * 32, 256), 256, 0, st>>>(ns, an.bs, s.bss_hdr.p, an.lower.rp.p,
                                                                      p.lvals.p, p.invd.p, out.p);
            CK_LAUNCH();
            if (s.rec) {  // the sweeps read the records only
                DevBuf<double>& rec = up ? p.rec_up : p.rec_lo;
                rec.alloc(16 * ns);
                rec_pack<<<gridn(16 * ns, 256), 256, 0, st>>>(ns, s.bss_hdr.p, s.bss_col.p, out.p, rec.p);
                CK_LAUNCH();
                CK(cudaStreamSynchronize(st));
                out.reset();
            }
            continue;
        }
        if (up)
            bss_values<true><<<gridn(ns * 32, 256), 256, 0, st>>>(ns, s.bss_hdr.p, an.upper.rp.p, p.uvals.p,
                                                                 p.invd.p, out.p);
        else
            bss_values<false><<<gridn(ns * 32, 256), 256, 0, st>>>(ns, s.bss_hdr.p, an.lower.rp.p, p.lvals.p,
                                                                  p.invd.p, out.p);
        CK_LAUNCH();
    }
}

template <int LG, int BS, bool UP, int CH>
void launch_rrs_t(const Schedule& s, const double* sv, const double* b, double* x, double* reset, const int* done,
                  cudaStream_t st) {
    static unsigned cap = 0;
    if (!cap) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rrs_trsv_kernel<LG, BS, UP, CH>, RR_THREADS, 0));
        cap = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
    }
    const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
    const int64_t warps = static_cast<int64_t>(6.0 * per_level) + 1;
    const int64_t blocks = std::max<int64_t>((warps + RR_THREADS / 32 - 1) / (RR_THREADS / 32), sm_count());
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, cap));
    rrs_trsv_kernel<LG, BS, UP, CH><<<grid, RR_THREADS, 0, st>>>(s.nitems, s.bss_hdr.p, s.bss_col.p, sv, b, x,
                                                                 reset, done);
    CK_LAUNCH();
}

template <int BS, bool UP>
void launch_rrs_bs(const Schedule& s, const double* sv, const double* b, double* x, double* reset, const int* done,
                   cudaStream_t st) {
    switch (s.lanes) {
        case 4: launch_rrs_t<4, BS, UP, 2>(s, sv, b, x, reset, done, st); break;
        case 8: launch_rrs_t<8, BS, UP, 1>(s, sv, b, x, reset, done, st); break;
        case 16: launch_rrs_t<16, BS, UP, 2>(s, sv, b, x, reset, done, st); break;
        default: launch_rrs_t<32, BS, UP, 4>(s, sv, b, x, reset, done, st); break;
    }
}

bool launch_bss(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                const int* done, cudaStream_t st, bool pad) {
    const Schedule& s = upper ? an.blk_up : an.blk_lo;
    const double* sv = upper ? p.bss_up.p : p.bss_lo.p;
    if (!an.bsr && s.bss && s.rec && s.nitems > 0 && (upper ? p.rec_up.p : p.rec_lo.p)) {
        if (pad) return false;
        auto kern = upper ? rec_trsv_kernel<true> : rec_trsv_kernel<false>;
        static unsigned cap[2] = {0, 0};
        if (!cap[upper]) {
            int per_sm = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RR_THREADS, 0));
            if (const char* e = getenv("PCLAB_REC_CTAS")) per_sm = std::min(per_sm, std::max(atoi(e), 1));
            cap[upper] = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
        }
        const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
        const int64_t warps = static_cast<int64_t>(6.0 * per_level) + 1;
        const int64_t blocks = std::max<int64_t>((warps + RR_THREADS / 32 - 1) / (RR_THREADS / 32), sm_count());
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, cap[upper]));
        kern<<<grid, RR_THREADS, 0, st>>>(s.nitems, upper ? p.rec_up.p : p.rec_lo.p, b, x, reset, done);
        CK_LAUNCH();
        return true;
    }
    if (!s.bss || !sv || s.nitems == 0) return false;
    if (!an.bsr) {
        if (pad) return false;
        if (upper) {
            if (an.bs == 3) launch_rrs_bs<3, true>(s, sv, b, x, reset, done, st);
            else if (an.bs == 2) launch_rrs_bs<2, true>(s, sv, b, x, reset, done, st);
            else launch_rrs_bs<1, true>(s, sv, b, x, reset, done, st);
        } else {
            if (an.bs == 3) launch_rrs_bs<3, false>(s, sv, b, x, reset, done, st);
            else if (an.bs == 2) launch_rrs_bs<2, false>(s, sv, b, x, reset, done, st);
            else launch_rrs_bs<1, false>(s, sv, b, x, reset, done, st);
        }
        return true;
    }
    if (!pad) return false;
    auto kern = upper ? bss_trsv_kernel<true> : bss_trsv_kernel<false>;
    static unsigned cap[2] = {0, 0};
    if (!cap[upper]) {
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BSR_THREADS, 0));
        cap[upper] = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
    }
    // every warp resident (round-robin items), ~5 levels of items in flight
    const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
    const int64_t warps = static_cast<int64_t>(5.0 * per_level) + 1;
    const int64_t blocks = std::max<int64_t>((warps + BSR_THREADS / 32 - 1) / (BSR_THREADS / 32), sm_count());
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, cap[upper]));
    kern<<<grid, BSR_THREADS, 0, st>>>(static_cast<int>(s.nitems), s.bss_hdr.p, s.bss_col.p, sv, b, x, reset, done);
    CK_LAUNCH();
    return true;
}

}  // namespace pclab_b200
