// TMA-staged item streams of the node-blocked sweeps (bst_trsv_kernel).
//
// The round-robin sweep (sweep.cuh: warp w of W runs items w, w + W, ...)
// knows every item a warp will run, so nothing about an item's matrix data
// has to wait for the dependency chain -- only the polls of the neighbours'
// solution values do. Here each warp owns a ring of S shared-memory stages
// and keeps S items' records in flight with one bulk copy each
// (cp.async.bulk global -> shared, completion on a per-stage mbarrier): the
// whole record -- header, 3x3 neighbour blocks, in-block entries, reciprocal
// pivots, neighbour ids -- is one contiguous, 16-byte aligned piece of a
// per-factor byte stream laid out in item order. A warp's loop is then
//   wait(stage) -> 10 shared-memory loads per lane -> polls -> FMAs ->
//   shuffle tree -> 3x3 solve -> publish -> refill the stage (item + S*W)
// with no address arithmetic, no L1 prefetch and no global matrix loads in
// registers. Lane mapping, FMA order, shuffle tree and diagonal solve are
// bss_trsv_kernel's / bsr_item's: bit-identical results.
//
// Record of item i (slots 2i, 2i+1 of the schedule; bytes, all 16-aligned):
//   int4   {block0, block1, neighbours0, neighbours1}   (-1 / 0: idle slot)
//   double slot 0: 9 * nb0 block values (block-major, row-major inside),
//                  3 in-block entries, 3 reciprocal pivots
//   double slot 1: the same                      (+ one pad double if odd)
//   int32  neighbour block ids of slot 0, of slot 1     (padded to 16 bytes)
#include "core.h"
#include "sweep.cuh"
#include "bst.cuh"

namespace pclab_b200 {

namespace {

void build_one(Schedule& s, const BlockCols& bc, cudaStream_t st) {
    s.bst = false;
    if (s.lanes != 16 || s.per_item != 2 || s.nitems == 0 || s.nitems >= (1LL << 30)) return;
    DevBuf<int64_t> off(s.nitems + 1);
    DevBuf<int> mx(1);
    CK(cudaMemsetAsync(mx.p, 0, sizeof(int), st));
    bst_lengths<<<gridn(s.nitems + 1, 256), 256, 0, st>>>(s.nitems, s.slots.p, bc.bp.p, off.p, mx.p);
    CK_LAUNCH();
    scan_inplace(off.p, s.nitems + 1, st);
    const int64_t total16 = dev_read(off.p + s.nitems, st);
    const int max_bytes = dev_read(mx.p, st);
    if (total16 >= (1LL << 32) || max_bytes > kBstMaxStage) return;
    s.bst_loc.alloc(s.nitems);
    bst_locs<<<gridn(s.nitems, 256), 256, 0, st>>>(s.nitems, off.p, s.bst_loc.p);
    CK_LAUNCH();
    s.bst_bytes = 16 * total16;
    s.bst_stage = max_bytes;
    s.bst = true;
}


}  // namespace

// ------------------------------------------------------------ the sweep
#ifndef BST_CTAS
#define BST_CTAS 7
#endif
constexpr int kBstWarps = BSR_THREADS / 32;

template <bool UPPER, int S>
__global__ void __launch_bounds__(BSR_THREADS, BST_CTAS)
bst_trsv_kernel(int nitems, const uint2* __restrict__ loc, const unsigned char* __restrict__ stream,
                const double* rhs, double* out, double* reset, const int* __restrict__ done, int stage_bytes) {
    if (done && *done) return;
    constexpr int BS = 3, LG = 16, NIB = 3;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bars[kBstWarps * S];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int grp = lane / LG, gl = lane % LG;
    const uint32_t ring = smem_addr(smem) + static_cast<uint32_t>(wi * S * stage_bytes);
    const uint32_t bar0 = smem_addr(bars + wi * S);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    int it = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    uint64_t pol = 0;
    uint2 nl = make_uint2(0, 0);
    if (lane == 0) {
        pol = evict_first_policy();
        for (int j = 0; j < S; ++j)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8 * j) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int j = 0; j < S; ++j) {
            const int i = it + j * nw;
            if (i < nitems) {
                const uint2 l = __ldg(loc + i);
                mbar_expect_tx(bar0 + 8 * j, l.y);
                tma_bulk_g2s_hint(ring + j * stage_bytes, stream + 16 * static_cast<uint64_t>(l.x), l.y, bar0 + 8 * j,
                                  pol);
            }
        }
        if (it + S * nw < nitems) nl = __ldg(loc + it + S * nw);
    }
    __syncwarp();
    int j = 0;
    unsigned ph = 0;
    for (; it < nitems; it += nw) {
        const uint32_t rec = ring + j * stage_bytes;
        mbar_wait_addr(bar0 + 8 * j, ph);
        int4 hd;
        asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(hd.x), "=r"(hd.y), "=r"(hd.z), "=r"(hd.w) : "r"(rec));
        const int blk = grp ? hd.y : hd.x;
        const int nb = grp ? hd.w : hd.z;
        const bool active = blk >= 0;
        const int nv0 = hd.x >= 0 ? 9 * hd.z + 6 : 0, nv1 = hd.y >= 0 ? 9 * hd.w + 6 : 0;
        const uint32_t v = rec + 16 + (grp ? 8 * nv0 : 0);
        const uint32_t c = rec + 16 + 8 * ((nv0 + nv1 + 1) & ~1) + (grp ? 4 * hd.z : 0);
        double rc[BS] = {0.0, 0.0, 0.0}, bin[NIB], binv[BS];
        if (active && gl == 0) {
            if constexpr (UPPER) {  // padded y: one 256-bit load
                double d3;
                asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(rc[0]), "=d"(rc[1]), "=d"(rc[2]), "=d"(d3)
                             : "l"(rhs + 4 * static_cast<int64_t>(blk)));
                (void)d3;
            } else {
#pragma unroll
                for (int t = 0; t < BS; ++t) rc[t] = rhs[static_cast<int64_t>(blk) * BS + t];
            }
#pragma unroll
            for (int q = 0; q < NIB; ++q)
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bin[q]) : "r"(v + 8 * (9 * nb + q)));
#pragma unroll
            for (int t = 0; t < BS; ++t)
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(binv[t]) : "r"(v + 8 * (9 * nb + NIB + t)));
        }
        double acc[BS] = {0.0, 0.0, 0.0};
        const int nbmax = max(hd.z, hd.w);
        for (int n0 = 0; n0 < nbmax; n0 += LG) {
            const int n = n0 + gl;
            const bool own = n < nb;
            double a[BS][BS], xv[BS] = {0.0, 0.0, 0.0};
            int32_t xb = 0;
            if (own) {
                asm volatile("ld.shared.s32 %0, [%1];" : "=r"(xb) : "r"(c + 4 * n));
                const uint32_t vn = v + 72 * n;
#pragma unroll
                for (int t = 0; t < BS; ++t)
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc)
                        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[t][cc]) : "r"(vn + 8 * (BS * t + cc)));
                ld_relaxed_v4(out + 4 * static_cast<int64_t>(xb), xv);
            } else {
#pragma unroll
                for (int t = 0; t < BS; ++t)
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) a[t][cc] = 0.0;
            }
            bool pend = own && (is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]));
            while (__any_sync(0xffffffffu, pend)) {
                if (pend) {
                    ld_relaxed_v4(out + 4 * static_cast<int64_t>(xb), xv);
                    pend = is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]);
                }
            }
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int cc = 0; cc < BS; ++cc) acc[t] = fma(a[t][cc], xv[cc], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (active && gl == 0) {
            double x[BS];
            solve_diag_block<BS, UPPER>(rc, acc, bin, binv, x);
            st_relaxed_v4(out + 4 * static_cast<int64_t>(blk), x[0], x[1], x[2], 0.0);
        }
        // every lane's shared-memory reads of this stage were consumed by
        // the shuffle tree above: the stage can take item it + S * nw
        __syncwarp();
        if (reset && active && gl < BS) reset[4 * static_cast<int64_t>(blk) + gl] = pending_value();
        if (lane == 0) {
            if (it + S * nw < nitems) {
                mbar_expect_tx(bar0 + 8 * j, nl.y);
                tma_bulk_g2s_hint(rec, stream + 16 * static_cast<uint64_t>(nl.x), nl.y, bar0 + 8 * j, pol);
            }
            if (it + (S + 1) * nw < nitems) nl = __ldg(loc + it + (S + 1) * nw);
        }
        if (++j == S) {
            j = 0;
            ph ^= 1u;
        }
    }
}

bool bst_enabled() {
    static const bool on = env_int("PCLAB_BST", 1) != 0;
    return on;
}

void build_bst(Analysis& an, cudaStream_t st) {
    an.blk_lo.bst = an.blk_up.bst = false;
    if (!bst_enabled() || !(an.bsr && an.bs == 3)) return;
    build_one(an.blk_lo, an.lbc, st);
    build_one(an.blk_up, an.ubc, st);
    if (!(an.blk_lo.bst && an.blk_up.bst)) an.blk_lo.bst = an.blk_up.bst = false;
}

void fill_bst(const Analysis& an, Precond& p, cudaStream_t st) {
    if (!an.blk_lo.bst) return;
    for (int up = 0; up < 2; ++up) {
        const Schedule& s = up ? an.blk_up : an.blk_lo;
        DevBuf<unsigned char>& out = up ? p.bst_up : p.bst_lo;
        out.alloc(std::max<int64_t>(s.bst_bytes, 16));
        if (up)
            rec_fill<true, false><<<gridn(s.nitems * 32, 256), 256, 0, st>>>(
                s.nitems, 0, nullptr, s.bst_loc.p, s.slots.p, nullptr, nullptr, an.ubc.bp.p, an.ubc.bcol.p, an.upper.rp.p,
                p.uvals.p, p.invd.p, out.p);
        else
            rec_fill<false, false><<<gridn(s.nitems * 32, 256), 256, 0, st>>>(
                s.nitems, 0, nullptr, s.bst_loc.p, s.slots.p, nullptr, nullptr, an.lbc.bp.p, an.lbc.bcol.p, an.lower.rp.p,
                p.lvals.p, p.invd.p, out.p);
        CK_LAUNCH();
    }
}

template <bool UPPER, int S>
void launch_bst_t(const Schedule& s, const unsigned char* stream, const double* b, double* x, double* reset,
                  const int* done, cudaStream_t st) {
    auto kern = bst_trsv_kernel<UPPER, S>;
    const int stage = (s.bst_stage + 15) & ~15;
    const size_t dyn = static_cast<size_t>(kBstWarps) * S * stage;
    static size_t dyn_set = 0;
    static unsigned cap = 0;
    if (dyn != dyn_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BSR_THREADS, dyn));
        cap = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
        dyn_set = dyn;
    }
    // every warp resident (round-robin items), ~5 levels of items in flight
    const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
    const int64_t warps = static_cast<int64_t>(5.0 * per_level) + 1;
    const int64_t blocks = std::max<int64_t>((warps + kBstWarps - 1) / kBstWarps, sm_count());
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, cap));
    kern<<<grid, BSR_THREADS, dyn, st>>>(static_cast<int>(s.nitems), s.bst_loc.p, stream, b, x, reset, done, stage);
    CK_LAUNCH();
}

bool launch_bst(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                const int* done, cudaStream_t st, bool pad) {
    const Schedule& s = upper ? an.blk_up : an.blk_lo;
    const unsigned char* stream = upper ? p.bst_up.p : p.bst_lo.p;
    if (!pad || !s.bst || !stream || s.nitems == 0) return false;
    static const int stages = env_int("PCLAB_BST_STAGES", 3);
    switch (stages) {
        case 2:
            upper ? launch_bst_t<true, 2>(s, stream, b, x, reset, done, st)
                  : launch_bst_t<false, 2>(s, stream, b, x, reset, done, st);
            break;
        case 4:
            upper ? launch_bst_t<true, 4>(s, stream, b, x, reset, done, st)
                  : launch_bst_t<false, 4>(s, stream, b, x, reset, done, st);
            break;
        default:
            upper ? launch_bst_t<true, 3>(s, stream, b, x, reset, done, st)
                  : launch_bst_t<false, 3>(s, stream, b, x, reset, done, st);
            break;
    }
    return true;
}

}  // namespace pclab_b200
