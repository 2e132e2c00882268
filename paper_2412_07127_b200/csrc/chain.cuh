// Chain sweep fed by bulk copies (node-blocked matrices with chain
// segments, Schedule::seg_first/seg_len).
//
// A segment is a run of consecutive blocks (in sweep order) where every
// block depends on the block before it -- on a structured mesh a pencil of
// nodes along the fastest index. One warp walks a segment block by block,
// lane n owning neighbour block n, and hands each block's solution to the
// next block in registers (the lane owning that neighbour takes it from a
// shuffle instead of polling L2). Only dependencies across segments pay the
// L2 publication round trip: on the 118^3 mesh 468 of the 819 hops of the
// longest level path are in-segment.
//
// Everything a step reads except the cross-segment dependencies is static
// and contiguous over the segment (factor entries, block columns, 1/l_ii,
// the right-hand side), so lane 0 streams it into a per-warp ring of NSLOT
// shared-memory slots with 1-D bulk copies (cp.async.bulk, completion on an
// mbarrier per slot), CB blocks per slot, NSLOT chunks ahead. The segment's
// row and block pointers are staged once when the warp takes it. The
// cross-segment dependency values are loaded CK steps early into a ring of
// registers (named statically by unrolling the step loop CK times) and
// re-polled only if still pending when their step comes.
//
// Segments are dealt round-robin to all resident warps in (level of the
// first block, index) order; the analysis checks that every dependency of
// a block in segment I lies in a segment < I + W (Schedule::chain_maxfwd),
// so the unfinished block of lowest level among the W segments in flight
// is always runnable (deadlock-free).
#pragma once

#include "sweep.cuh"

namespace pclab_b200 {

constexpr int kChainSlots = 4;  // bulk-copy ring depth (chunks)
constexpr int kChainCB = 2;     // blocks per chunk
constexpr int kChainCK = 4;     // dependency-poll lookahead (steps)
constexpr int kChainMaxSeg = 128;

// Per-warp shared-memory layout (bytes), computed on the host from the
// largest block (entries, neighbour blocks) of the sweep.
struct ChainLayout {
    int vals_cap;   // doubles per slot
    int bcol_cap;   // ints per slot
    int vec_cap;    // doubles per slot for 1/l_ii and for the rhs
    unsigned rps_off, bps_off, slot_off, slot_bytes, warp_bytes;
};

__host__ __device__ inline unsigned chain_align16(unsigned x) { return (x + 15u) & ~15u; }

__host__ inline ChainLayout chain_layout(int bs, int maxblk, int maxnb) {
    ChainLayout l;
    l.vals_cap = kChainCB * maxblk + 4;
    l.bcol_cap = kChainCB * maxnb + 8;
    l.vec_cap = kChainCB * bs + 4;
    l.rps_off = chain_align16(8 * kChainSlots);
    l.bps_off = l.rps_off + chain_align16(8 * (kChainMaxSeg * bs + 4));
    l.slot_off = l.bps_off + chain_align16(8 * (kChainMaxSeg + 4));
    l.slot_bytes = chain_align16(8 * l.vals_cap) + chain_align16(4 * l.bcol_cap) + 2 * chain_align16(8 * l.vec_cap);
    l.warp_bytes = l.slot_off + kChainSlots * l.slot_bytes;
    return l;
}

template <int BS, bool UPPER>
__global__ void __launch_bounds__(256, BSR_MINB)
chain_tma_kernel(int64_t nseg, const int32_t* __restrict__ sfirst, const int32_t* __restrict__ slen,
                 const int64_t* __restrict__ rp, const int64_t* __restrict__ bp, const int32_t* __restrict__ bcol,
                 const double* __restrict__ vals, const double* __restrict__ invd, const double* rhs, double* out,
                 double* reset, const int* __restrict__ done, ChainLayout L, long long* trace) {
    if (done && *done) return;
    extern __shared__ __align__(16) unsigned char chain_smem[];
    constexpr int NIB = BS * (BS - 1) / 2;
    constexpr int64_t dir = UPPER ? -1 : 1;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    unsigned char* base = chain_smem + static_cast<size_t>(wib) * L.warp_bytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(base);
    int64_t* rps = reinterpret_cast<int64_t*>(base + L.rps_off);
    int64_t* bps = reinterpret_cast<int64_t*>(base + L.bps_off);
    auto slot_vals = [&](int q) { return reinterpret_cast<double*>(base + L.slot_off + q * L.slot_bytes); };
    auto slot_bcol = [&](int q) {
        return reinterpret_cast<int32_t*>(base + L.slot_off + q * L.slot_bytes + chain_align16(8 * L.vals_cap));
    };
    auto slot_inv = [&](int q) {
        return reinterpret_cast<double*>(base + L.slot_off + q * L.slot_bytes + chain_align16(8 * L.vals_cap) +
                                         chain_align16(4 * L.bcol_cap));
    };
    auto slot_rhs = [&](int q) { return slot_inv(q) + chain_align16(8 * L.vec_cap) / 8; };
    if (lane == 0) {
        for (int q = 0; q < kChainSlots; ++q) mbar_init(bar + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int64_t W = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    unsigned long long chunk_seq = 0;  // chunks issued by this warp so far (slot = seq % NSLOT)
    for (int64_t I = warp; I < nseg; I += W) {
        const int64_t b0 = __ldg(sfirst + I);
        const int len = __ldg(slen + I);
        const int64_t lo = UPPER ? b0 - len + 1 : b0, hi = UPPER ? b0 : b0 + len - 1;
        // stage the segment's row pointers and block pointers
        const int64_t rp_base = (lo * BS) & ~1LL, bp_base = lo & ~1LL;
        for (int64_t e = rp_base + lane; e <= (hi + 1) * BS; e += 32) rps[e - rp_base] = __ldg(rp + e);
        for (int64_t e = bp_base + lane; e <= hi + 1; e += 32) bps[e - bp_base] = __ldg(bp + e);
        __syncwarp();
        auto RP = [&](int64_t e) { return rps[e - rp_base]; };
        auto BP = [&](int64_t e) { return bps[e - bp_base]; };
        const int nchunks = (len + kChainCB - 1) / kChainCB;
        const unsigned long long seq0 = chunk_seq;
        auto chunk_blocks = [&](int k, int64_t& blo, int64_t& bhi) {
            const int64_t s_a = static_cast<int64_t>(k) * kChainCB;
            const int64_t s_b = min(static_cast<int64_t>(len), s_a + kChainCB) - 1;
            const int64_t ba = b0 + dir * s_a, bb = b0 + dir * s_b;
            blo = min(ba, bb);
            bhi = max(ba, bb);
        };
        auto issue = [&](int k) {  // lane 0
            const int q = static_cast<int>((seq0 + k) % kChainSlots);
            int64_t blo, bhi;
            chunk_blocks(k, blo, bhi);
            const int64_t v0 = RP(blo * BS) & ~1LL, v1 = (RP((bhi + 1) * BS) + 1) & ~1LL;
            const int64_t c0 = BP(blo) & ~3LL, c1 = (BP(bhi + 1) + 3) & ~3LL;
            const int64_t i0 = (blo * BS) & ~1LL, i1 = ((bhi + 1) * BS + 1) & ~1LL;
            const unsigned vb = static_cast<unsigned>(8 * (v1 - v0)), cb = static_cast<unsigned>(4 * (c1 - c0)),
                           ib = static_cast<unsigned>(8 * (i1 - i0));
            mbar_arrive_expect_tx(bar + q, vb + cb + 2 * ib);
            tma_bulk_g2s(slot_vals(q), vals + v0, vb, bar + q);
            tma_bulk_g2s(slot_bcol(q), bcol + c0, cb, bar + q);
            tma_bulk_g2s(slot_inv(q), invd + i0, ib, bar + q);
            tma_bulk_g2s(slot_rhs(q), rhs + i0, ib, bar + q);
        };
        auto wait_chunk = [&](int k) {
            const unsigned long long g = seq0 + k;
            mbar_wait(bar + g % kChainSlots, static_cast<unsigned>((g / kChainSlots) & 1));
        };
        if (lane == 0)
            for (int k = 0; k < min(nchunks, kChainSlots); ++k) issue(k);
        chunk_seq += nchunks;
        // dependency-poll ring: lane's neighbour column and values, CK steps early
        int32_t pxc[kChainCK];
        double pxv[kChainCK][BS];
        auto poll_fill = [&](int j, int s) {
            pxc[j] = -1;
#pragma unroll
            for (int c = 0; c < BS; ++c) pxv[j][c] = 0.0;
            if (s >= len) return;
            const int k = s / kChainCB;
            if (s % kChainCB == 0 || s < kChainCK) wait_chunk(k);
            const int64_t b = b0 + dir * s;
            const int64_t c0 = BP(b);
            const int nb = static_cast<int>(BP(b + 1) - c0);
            const bool own = lane < nb;
            const bool chain = s > 0 && lane == (UPPER ? 0 : nb - 1);
            int64_t blo, bhi;
            chunk_blocks(k, blo, bhi);
            const int32_t* sb = slot_bcol(static_cast<int>((seq0 + k) % kChainSlots)) - (BP(blo) & ~3LL);
            if (own) {
                pxc[j] = sb[c0 + lane];
                if (!chain) {
#pragma unroll
                    for (int c = 0; c < BS; ++c) pxv[j][c] = ld_relaxed(out + pxc[j] + c);
                }
            }
        };
#pragma unroll
        for (int j = 0; j < kChainCK; ++j) poll_fill(j, j);
        double xprev[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) xprev[t] = 0.0;
        for (int s0 = 0; s0 < len; s0 += kChainCK) {
#pragma unroll
            for (int j = 0; j < kChainCK; ++j) {
                const int s = s0 + j;
                if (s >= len) break;
                long long t_start = 0;
                if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
                const int k = s / kChainCB;
                const int q = static_cast<int>((seq0 + k) % kChainSlots);
                int64_t blo, bhi;
                chunk_blocks(k, blo, bhi);
                const double* sv = slot_vals(q) - (RP(blo * BS) & ~1LL);
                const double* si = slot_inv(q) - ((blo * BS) & ~1LL);
                const double* sr = slot_rhs(q) - ((blo * BS) & ~1LL);
                const int64_t b = b0 + dir * s;
                int64_t r[BS + 1];
#pragma unroll
                for (int t = 0; t <= BS; ++t) r[t] = RP(b * BS + t);
                const int nb = static_cast<int>(BP(b + 1) - BP(b));
                const bool own = lane < nb;
                const bool chain = s > 0 && lane == (UPPER ? 0 : nb - 1);
                double a[BS][BS];
#pragma unroll
                for (int t = 0; t < BS; ++t) {
                    const int64_t ob = UPPER ? r[t] + (BS - t) : r[t];
#pragma unroll
                    for (int c = 0; c < BS; ++c) a[t][c] = own ? sv[ob + BS * lane + c] : 0.0;
                }
                // cross-segment dependencies: re-poll any still pending.
                // (Measured: 95 % of steps find a dependency that was pending
                // when loaded CK steps early -- the neighbour pencils run just
                // in time -- and pay one L2 round trip here; refreshing the
                // next step's values one step early halves that share but the
                // refresh itself is then waited on: 1.45 vs 1.34 ms.)
                bool pend = false;
#pragma unroll
                for (int c = 0; c < BS; ++c) pend |= own && !chain && is_pending(pxv[j][c]);
                int repolls = 0;
                while (__any_sync(0xffffffffu, pend)) {
                    ++repolls;
                    pend = false;
#pragma unroll
                    for (int c = 0; c < BS; ++c)
                        if (own && !chain && is_pending(pxv[j][c])) {
                            pxv[j][c] = ld_relaxed(out + pxc[j] + c);
                            pend |= is_pending(pxv[j][c]);
                        }
                }
                long long t_ready = 0;
                if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_ready));
                double acc[BS];
#pragma unroll
                for (int t = 0; t < BS; ++t) {
                    acc[t] = 0.0;
#pragma unroll
                    for (int c = 0; c < BS; ++c) acc[t] = fma(a[t][c], chain ? xprev[c] : pxv[j][c], acc[t]);
                }
#pragma unroll
                for (int t = 0; t < BS; ++t) acc[t] = group_sum<32>(acc[t]);
                double xb[BS];
#pragma unroll
                for (int t = 0; t < BS; ++t) xb[t] = 0.0;
                if (lane == 0) {
                    if (!UPPER) {
#pragma unroll
                        for (int t = 0; t < BS; ++t) {
                            double sacc = sr[b * BS + t] - acc[t];
#pragma unroll
                            for (int u = 0; u < t; ++u) sacc -= sv[r[t + 1] - (t + 1) + u] * xb[u];
                            xb[t] = sacc * si[b * BS + t];
                        }
                    } else {
#pragma unroll
                        for (int t = BS - 1; t >= 0; --t) {
                            double sacc = sr[b * BS + t] - acc[t];
#pragma unroll
                            for (int u = t + 1; u < BS; ++u) sacc -= sv[r[t] + (u - t)] * xb[u];
                            xb[t] = sacc * si[b * BS + t];
                        }
                    }
#pragma unroll
                    for (int t = 0; t < BS; ++t) st_relaxed(out + b * BS + t, xb[t]);
                    if (trace) {
                        long long t_pub;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_pub));
                        trace[4 * b + 0] = t_start;
                        trace[4 * b + 1] = t_pub;
                        trace[4 * b + 2] = t_ready;
                        trace[4 * b + 3] = (s > 0 ? 1 : 0) | (min(repolls, 1000) << 1);
                    }
                }
#pragma unroll
                for (int t = 0; t < BS; ++t) xprev[t] = __shfl_sync(0xffffffffu, xb[t], 0);
                if (reset && lane < BS) reset[b * BS + lane] = pending_value();
                // chunk k done: its slot takes chunk k + NSLOT
                if (s == len - 1 || s % kChainCB == kChainCB - 1) {
                    __syncwarp();
                    if (lane == 0 && k + kChainSlots < nchunks) issue(k + kChainSlots);
                }
                poll_fill(j, s + kChainCK);
            }
        }
    }
}

}  // namespace pclab_b200
