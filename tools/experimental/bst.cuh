// Shared pieces of the TMA-staged item records (bst.cu, lts.cu): record
// sizes, the length / location kernels and the bulk-copy PTX wrappers.
#pragma once
#include "core.h"
#include "sweep.cuh"

namespace pclab_b200 {
namespace {

inline unsigned gridn(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__device__ __forceinline__ int slot_nvals(int32_t b, int nb) { return b >= 0 ? 9 * nb + 6 : 0; }
__device__ __forceinline__ int item_bytes(int32_t b0, int nb0, int32_t b1, int nb1) {
    const int nv = (slot_nvals(b0, nb0) + slot_nvals(b1, nb1) + 1) & ~1;
    const int cb = (4 * (nb0 + nb1) + 15) & ~15;
    return 16 + 8 * nv + cb;
}

// record length of every item in 16-byte units (one extra zero for the scan)
__global__ void bst_lengths(int64_t nitems, const int32_t* __restrict__ slots, const int64_t* __restrict__ bp,
                            int64_t* __restrict__ len16, int* __restrict__ max_bytes) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i > nitems) return;
    if (i == nitems) {
        len16[i] = 0;
        return;
    }
    const int32_t b0 = slots[2 * i], b1 = slots[2 * i + 1];
    const int nb0 = b0 >= 0 ? static_cast<int>(bp[b0 + 1] - bp[b0]) : 0;
    const int nb1 = b1 >= 0 ? static_cast<int>(bp[b1 + 1] - bp[b1]) : 0;
    const int bytes = item_bytes(b0, nb0, b1, nb1);
    len16[i] = bytes / 16;
    atomicMax(max_bytes, bytes);
}

__global__ void bst_locs(int64_t nitems, const int64_t* __restrict__ off16, uint2* __restrict__ loc) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= nitems) return;
    loc[i] = make_uint2(static_cast<uint32_t>(off16[i]), static_cast<uint32_t>(16 * (off16[i + 1] - off16[i])));
}

int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_bulk_g2s_hint(uint32_t dst, const void* src, unsigned bytes, uint32_t bar,
                                                  uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_addr(uint32_t bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}\n" ::"r"(bar), "r"(parity)
        : "memory");
}


// one item's record (warp per item). LOCAL (lts.cu): a neighbour inside the
// item's tile (sweep positions [tile_q.x, tile_q.x + tile_q.y) of `nbk`
// nodes) is stored as -(1 + position in the tile) instead of its node id, and a
// block's neighbours are reordered: the (at most kLtsCrit) neighbours at most
// two levels below the block first -- their count goes into the header's high
// half-words -- then the others, each group in column order.
constexpr int kLtsCrit = 7;
template <bool UPPER, bool LOCAL>
__global__ void rec_fill(int64_t nitems, int64_t nbk, const int32_t* __restrict__ level,
                         const uint2* __restrict__ loc,
                         const int32_t* __restrict__ slots, const int32_t* __restrict__ item_tile,
                         const int2* __restrict__ tile_q, const int64_t* __restrict__ bp,
                         const int32_t* __restrict__ bcol,
                         const int64_t* __restrict__ rp, const double* __restrict__ vals,
                         const double* __restrict__ invd, unsigned char* __restrict__ stream) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= nitems) return;
    unsigned char* rec = stream + 16 * static_cast<uint64_t>(loc[i].x);
    int32_t b[2] = {slots[2 * i], slots[2 * i + 1]};
    int nb[2];
    for (int g = 0; g < 2; ++g) nb[g] = b[g] >= 0 ? static_cast<int>(bp[b[g] + 1] - bp[b[g]]) : 0;
    int ncrit[2] = {0, 0};
    int2 tq = make_int2(0, 0);
    if constexpr (LOCAL) tq = tile_q[item_tile[i]];
    const int nv0 = slot_nvals(b[0], nb[0]), nv1 = slot_nvals(b[1], nb[1]);
    const int nvt = (nv0 + nv1 + 1) & ~1;
    double* vbase = reinterpret_cast<double*>(rec + 16);
    int32_t* cbase = reinterpret_cast<int32_t*>(rec + 16 + 8 * nvt);
    for (int g = 0; g < 2; ++g) {
        if (b[g] < 0) continue;
        const int64_t blk = b[g];
        double* v = vbase + (g ? nv0 : 0);
        int pos = lane;  // position of neighbour `lane` in the record
        if (LOCAL && nb[g] <= 32) {
            bool crit = false;
            if (lane < nb[g]) crit = level[bcol[bp[blk] + lane] / 3] >= level[blk] - 2;
            unsigned m = __ballot_sync(0xffffffffu, crit);
            crit = crit && __popc(m & ((1u << lane) - 1u)) < kLtsCrit;
            m = __ballot_sync(0xffffffffu, crit);
            ncrit[g] = __popc(m);
            const int before = __popc(m & ((1u << lane) - 1u));
            pos = crit ? before : ncrit[g] + (lane - before);
        }
        for (int base = 0; base < 9 * nb[g]; base += 32) {
            const int idx = base + lane;
            const int n = min(idx / 9, nb[g] - 1), w = idx % 9, t = w / 3, c = w % 3;
            const int pn = nb[g] <= 32 ? __shfl_sync(0xffffffffu, pos, n) : n;
            if (idx < 9 * nb[g]) v[9 * pn + w] = vals[rp[3 * blk + t] + (UPPER ? 3 - t : 0) + 3 * n + c];
        }
        if (lane == 0) {
            double* d = v + 9 * nb[g];
            int q = 0;
#pragma unroll
            for (int t = 0; t < 3; ++t)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (!UPPER && c < t) d[q++] = vals[rp[3 * blk + t + 1] - (t + 1) + c];
                    if (UPPER && c > t) d[q++] = vals[rp[3 * blk + t] + (c - t)];
                }
#pragma unroll
            for (int t = 0; t < 3; ++t) d[3 + t] = invd[3 * blk + t];
        }
        int32_t* c = cbase + (g ? nb[0] : 0);
        for (int n = lane; n < nb[g]; n += 32) {
            const int32_t id = bcol[bp[blk] + n] / 3;
            int32_t code = id;
            if constexpr (LOCAL) {
                const int64_t qn = UPPER ? nbk - 1 - id : id;
                if (qn >= tq.x && qn < static_cast<int64_t>(tq.x) + tq.y) code = -(1 + static_cast<int32_t>(qn - tq.x));
            }
            c[nb[g] <= 32 ? pos : n] = code;
        }
    }
    if (lane == 0)
        *reinterpret_cast<int4*>(rec) = make_int4(b[0], b[1], nb[0] | (ncrit[0] << 16), nb[1] | (ncrit[1] << 16));
    if (lane == 0 && ((nv0 + nv1) & 1)) vbase[nv0 + nv1] = 0.0;
    const int nc = nb[0] + nb[1], ncp = (nc + 3) & ~3;
    if (lane < ncp - nc) cbase[nc + lane] = 0;
}


}  // namespace
}  // namespace pclab_b200
