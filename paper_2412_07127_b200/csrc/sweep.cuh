// Device kernels for the sparse hot loop: CSR SpMV (lane group per row)
// and the sync-free dof-blocked triangular sweeps.
#pragma once

#include "common.cuh"

// minimum resident 256-thread blocks per SM for the warp sweep (register cap)
#ifndef TRSV_MINB
#define TRSV_MINB 4
#endif
// node-blocked sweep CTA: 128 threads, 7 resident per SM (28 warps at <= 72
// registers), entries prefetched into L1 one item ahead (slot records two
// ahead). Measured on configs[2] per sweep: 6/SM 0.868 ms, 7/SM 0.859, 7/SM
// with one-item prefetch 0.849, 8/SM 1.02 (spills)
#ifndef BSR_THREADS
#define BSR_THREADS 128
#endif
#ifndef BSR_CTAS
#define BSR_CTAS 7
#endif

namespace pclab_b200 {

// Rows per warp = 32 / LPR; each lane group of LPR lanes reduces one row
// with a fixed shuffle tree (deterministic).
template <int LPR>
__device__ __forceinline__ double row_dot(const int64_t* __restrict__ rp,
                                          const int32_t* __restrict__ cols,
                                          const double* __restrict__ vals,
                                          const double* __restrict__ x, int64_t row, int gl,
                                          bool active) {
    constexpr int U = LPR <= 4 ? 8 : (LPR == 16 ? 6 : 4);  // loads of a row batch issued before the gathers
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
                if (j[u] >= 0) acc = fma(v[u], __ldg(x + j[u]), acc);
        }
    }
    return group_sum<LPR>(acc);
}

// Short scalar rows (7-point stencils): a warp takes 32 consecutive rows,
// whose entries are one contiguous range. The lanes stream that range with
// coalesced index / value loads (kTileU per lane issued before the gathers),
// stage the products in shared memory, and then each lane adds up its own
// row in CSR order starting from 0 — the reference's csr_matvec
// (sparse.cpp:121-135: acc += v * x, unfused) bit for bit. Ranges longer
// than the stage run in chunks; the per-row order is unchanged.
// measured on the 256^3 7-point product (stand-alone, L2 flushed):
// U = 10 at 5 CTAs/SM 0.356 ms; U = 8: 0.371; U = 12 / 16 at 4 CTAs/SM
// 0.399 / 0.411; U = 6 at 6 CTAs/SM 0.558; lane 31's end pointer through a
// shuffle instead of a second load 0.494
#ifndef TILE_U
#define TILE_U 10
#endif
#ifndef TILE_MINB
#define TILE_MINB 5
#endif
#if TILE_MINB > 0
#define TILE_LB(t) __launch_bounds__(t, TILE_MINB)
#else
#define TILE_LB(t) __launch_bounds__(t)
#endif
constexpr int kTileU = TILE_U;
constexpr int kTileCh = 32 * kTileU;  // products staged per warp per chunk

struct RowSpan {
    int64_t b, e;
};

// lane l of a row tile: [rp[row], rp[row + 1]) (row = tile start + l)
__device__ __forceinline__ RowSpan row_span(const int64_t* __restrict__ rp, int64_t n, int64_t row) {
    return RowSpan{__ldg(rp + (row < n ? row : n)), __ldg(rp + (row + 1 < n ? row + 1 : n))};
}

__device__ __forceinline__ double tile_rows_dot(const RowSpan& s, const int32_t* __restrict__ cols,
                                                const double* __restrict__ vals, const double* __restrict__ x,
                                                double* sh, int lane) {
    const int64_t base = __shfl_sync(0xffffffffu, s.b, 0);
    const int64_t end = __shfl_sync(0xffffffffu, s.e, 31);
    double acc = 0.0;
    for (int64_t c0 = base; c0 < end; c0 += kTileCh) {
        const int cnt = static_cast<int>(end - c0 < kTileCh ? end - c0 : kTileCh);
        int32_t j[kTileU];
        double v[kTileU];
#pragma unroll
        for (int u = 0; u < kTileU; ++u) {
            const int k = lane + 32 * u;
            j[u] = k < cnt ? __ldg(cols + (c0 + k)) : 0;
            v[u] = k < cnt ? __ldg(vals + (c0 + k)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kTileU; ++u) {
            const int k = lane + 32 * u;
            if (k < cnt) sh[k] = __dmul_rn(v[u], __ldg(x + j[u]));
        }
        __syncwarp();
        const int64_t kb = s.b > c0 ? s.b : c0, ke = s.e < c0 + cnt ? s.e : c0 + cnt;
        for (int64_t k = kb; k < ke; ++k) acc = __dadd_rn(acc, sh[k - c0]);
        __syncwarp();
    }
    return acc;
}

// Row pointers of block row b (node-blocked product), loaded one row ahead.
template <int BS>
struct BsrRow {
    int64_t r[BS];
    int64_t c0;
    int cnt;
};

template <int BS>
__device__ __forceinline__ BsrRow<BS> bsr_row(int64_t b, int64_t nb, const int64_t* __restrict__ rp,
                                              const int64_t* __restrict__ bp) {
    BsrRow<BS> m;
    const bool ok = b < nb;
#pragma unroll
    for (int t = 0; t < BS; ++t) m.r[t] = ok ? __ldg(rp + b * BS + t) : 0;
    m.c0 = ok ? __ldg(bp + b) : 0;
    m.cnt = ok ? static_cast<int>(__ldg(bp + b + 1) - m.c0) : 0;
    return m;
}

// (A x) for one block row whose pointers are in hand; lane n owns
// neighbour block n (32-wide rounds). Result valid in every lane.
template <int BS>
__device__ __forceinline__ void bsr_row_dot(const BsrRow<BS>& m, const int32_t* __restrict__ bcol,
                                            const double* __restrict__ vals, const double* __restrict__ x,
                                            double (&acc)[BS]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < BS; ++t) acc[t] = 0.0;
    for (int n = lane; n < m.cnt; n += 32) {
        const int32_t xc = __ldg(bcol + m.c0 + n);
        double a[BS][BS];
#pragma unroll
        for (int t = 0; t < BS; ++t)
#pragma unroll
            for (int c = 0; c < BS; ++c) a[t][c] = __ldg(vals + m.r[t] + BS * n + c);
        double xv[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) xv[c] = __ldg(x + xc + c);
#pragma unroll
        for (int t = 0; t < BS; ++t)
#pragma unroll
            for (int c = 0; c < BS; ++c) acc[t] = fma(a[t][c], xv[c], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < BS; ++t) acc[t] = group_sum<32>(acc[t]);
}

// Dense BSxBS diagonal block of a sweep item: rows forward (L, in-block
// entries left of the diagonal in `bin`, row by row) or backward (U, right
// of the diagonal), each row s = rhs - acc - sum(bin * x), x = s / l_tt as
// s * (1 / l_tt).
template <int BS, bool UPPER>
__device__ __forceinline__ void solve_diag_block(const double (&rhs)[BS], const double (&acc)[BS],
                                                 const double* bin, const double (&binv)[BS], double (&xb)[BS]) {
    if (!UPPER) {
        int q = 0;
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            double s = rhs[t] - acc[t];
#pragma unroll
            for (int u = 0; u < t; ++u) s -= bin[q++] * xb[u];
            xb[t] = s * binv[t];
        }
    } else {
#pragma unroll
        for (int t = BS - 1; t >= 0; --t) {
            double s = rhs[t] - acc[t];
            // bin holds, row by row, U[t][s] for s > t
            int q = 0;
#pragma unroll
            for (int r = 0; r < t; ++r) q += BS - 1 - r;
#pragma unroll
            for (int u = t + 1; u < BS; ++u) s -= bin[q + (u - t - 1)] * xb[u];
            xb[t] = s * binv[t];
        }
    }
}

// Per-item state of a sweep, loaded one item ahead.
template <int BS>
struct SweepMeta {
    int64_t blk;  // -1: idle lane group
    int64_t rp[BS + 1];
    int32_t crit;
    double rhs[BS];  // right-hand side of the block (loaded one item ahead)
};

template <int BS>
__device__ __forceinline__ SweepMeta<BS> sweep_meta(unsigned it, int64_t nitems, int G, int grp,
                                                    const int32_t* __restrict__ slots,
                                                    const int32_t* __restrict__ crit,
                                                    const int64_t* __restrict__ rp, const double* rhs) {
    SweepMeta<BS> m;
    m.blk = it < nitems ? static_cast<int64_t>(__ldg(slots + static_cast<int64_t>(it) * G + grp)) : -1;
    m.crit = -1;
#pragma unroll
    for (int t = 0; t <= BS; ++t) m.rp[t] = 0;
#pragma unroll
    for (int t = 0; t < BS; ++t) m.rhs[t] = 0.0;
    if (m.blk >= 0) {
        m.crit = __ldg(crit + m.blk);
#pragma unroll
        for (int t = 0; t <= BS; ++t) m.rp[t] = __ldg(rp + m.blk * BS + t);
#pragma unroll
        for (int t = 0; t < BS; ++t) m.rhs[t] = rhs[m.blk * BS + t];
    }
    return m;
}

// Sync-free blocked triangular sweep.
//
// Work items (warp-sized) are claimed from a global counter in (level,
// index) order, so every dependency of an item was claimed earlier by a
// running warp. Each of the G = 32/LG lane groups owns one block of BS
// consecutive rows (slots[item*G + group], -1 = idle). Per item:
//   1. indices/values of the off-block entries, the right-hand side, the
//      in-block entries and the reciprocal pivots are loaded -- none of
//      them depends on the sweep's progress, so they stream while waiting;
//   2. lane 0 of the group spins on ONE address: the last-published row of
//      the predecessor block with the highest level (`crit`, from the
//      analysis). One poller per block instead of one per entry keeps L2
//      free for the streaming loads;
//   3. all dependency values are read (a value still pending is re-polled);
//   4. lane 0 solves the dense BSxBS diagonal block and publishes the BS
//      results (kPending -> value is the publication).
// The next item is claimed and its metadata loaded while this one runs.
//
//   lower (L, row-sorted, diagonal last):  rows r0..r0+BS-1 forward
//   upper (U = L^T, diagonal first):       rows r0+BS-1..r0 backward
template <int LG, int BS, bool UPPER>
__global__ void __launch_bounds__(256, TRSV_MINB)
trsv_kernel(int64_t nitems, const int32_t* __restrict__ slots, const int32_t* __restrict__ crit,
            const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
            const double* __restrict__ vals, const double* __restrict__ invd, const double* rhs,
            double* out, double* reset, const int* __restrict__ done, unsigned* counter) {
    if (done && *done) return;
    constexpr int G = 32 / LG;
    // entries per lane per round: one round covers a 3x3-blocked elasticity
    // node (<= 117 off-block entries) so every load is issued before any spin
    constexpr int CH = LG >= 32 ? 4 : (LG >= 16 ? 8 : 2);
    constexpr int NIB = BS * (BS - 1) / 2;  // strictly-triangular in-block entries
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    // two items in flight per warp: while item `it` waits on its
    // dependencies, the entries of `next` are already being pulled into L1
    unsigned it = 0, next = 0;
    if (lane == 0) {
        it = atomicAdd(counter, 1u);
        next = atomicAdd(counter, 1u);
    }
    it = __shfl_sync(0xffffffffu, it, 0);
    next = __shfl_sync(0xffffffffu, next, 0);
    SweepMeta<BS> m = sweep_meta<BS>(it, nitems, G, grp, slots, crit, rp, rhs);
    SweepMeta<BS> mn = sweep_meta<BS>(next, nitems, G, grp, slots, crit, rp, rhs);
    while (it < nitems) {
        if (mn.blk >= 0) {
            // prefetch the next item's rows: 128-byte lines of values and indices
            const int64_t e0 = mn.rp[0], e1 = mn.rp[BS];
            for (int64_t a = (e0 & ~15LL) + 16 * gl; a < e1; a += 16 * LG)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(vals + a));
            for (int64_t a = (e0 & ~31LL) + 32 * gl; a < e1; a += 32 * LG)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(cols + a));
            if (gl == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(invd + mn.blk * BS));
        }
        unsigned after = 0;
        if (lane == 0) after = atomicAdd(counter, 1u);
        const bool active = m.blk >= 0;
        const int64_t r0 = active ? m.blk * BS : 0;
        int64_t ob[BS], oc[BS];
        int total = 0;
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            ob[t] = UPPER ? m.rp[t] + (BS - t) : m.rp[t];
            oc[t] = active ? (UPPER ? m.rp[t + 1] - ob[t] : m.rp[t + 1] - (t + 1) - m.rp[t]) : 0;
            total += static_cast<int>(oc[t]);
        }
        // (1) stream: first chunk of entries + the diagonal-block data
        double v[CH];
        int32_t jj[CH];
        int tt[CH];
        auto load_chunk = [&](int base) {
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                int e = base + c * LG + gl;
                tt[c] = -1;
                jj[c] = 0;
                v[c] = 0.0;
                if (e < total) {
                    int t = 0;
#pragma unroll
                    for (int s = 0; s < BS - 1; ++s)
                        if (t == s && e >= oc[s]) {
                            e -= static_cast<int>(oc[s]);
                            t = s + 1;
                        }
                    tt[c] = t;
                    jj[c] = ld_stream(cols + ob[t] + e);
                    v[c] = ld_stream(vals + ob[t] + e);
                }
            }
        };
        load_chunk(0);
        double brhs[BS], binv[BS], bin[NIB > 0 ? NIB : 1];
        if (active && gl == 0) {
#pragma unroll
            for (int t = 0; t < BS; ++t) {
                brhs[t] = m.rhs[t];  // loaded with the metadata, one item ahead
                binv[t] = __ldg(invd + r0 + t);
            }
            int q = 0;
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int s = 0; s < BS; ++s) {
                    if (!UPPER && s < t) bin[q++] = ld_stream(vals + m.rp[t + 1] - (t + 1) + s);
                    if (UPPER && s > t) bin[q++] = ld_stream(vals + m.rp[t] + (s - t));
                }
        }
        // (2) one poller per block on the critical predecessor
        // warp-uniform spins (divergent per-lane spin loops let the scheduler
        // park the waiting half of the warp for microseconds); the group's
        // lanes poll the same address, so it is one request per group
        {
            const bool poll = active && m.crit >= 0;
            while (__any_sync(0xffffffffu, poll && is_pending(ld_relaxed(out + (poll ? m.crit : 0))))) {
            }
        }
        // (3) gather the dependencies
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        const int tmax = __reduce_max_sync(0xffffffffu, total);
        for (int base = 0; base < tmax; base += LG * CH) {
            if (base > 0) load_chunk(base);
            double xv[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) xv[c] = tt[c] >= 0 ? ld_relaxed(out + jj[c]) : 0.0;
            bool pend = false;
#pragma unroll
            for (int c = 0; c < CH; ++c) pend |= tt[c] >= 0 && is_pending(xv[c]);
            while (__any_sync(0xffffffffu, pend)) {
                pend = false;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (tt[c] >= 0 && is_pending(xv[c])) {
                        xv[c] = ld_relaxed(out + jj[c]);
                        pend |= is_pending(xv[c]);
                    }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int t = 0; t < BS; ++t)
                    if (tt[c] == t) acc[t] = fma(v[c], xv[c], acc[t]);
        }
        after = __shfl_sync(0xffffffffu, after, 0);
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        // (4) diagonal block
        if (active && gl == 0) {
            double xb[BS];
            solve_diag_block<BS, UPPER>(brhs, acc, bin, binv, xb);
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[r0 + gl] = pending_value();
        // the next item's metadata is fetched only after publication, so its
        // dependent loads never sit on this item's critical path
        it = next;
        m = mn;
        next = after;
        mn = sweep_meta<BS>(after, nitems, G, grp, slots, crit, rp, rhs);
    }
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Per-item state of the node-blocked sweep: one 16-byte slot record
// (Schedule::slot_rp) = {block (-1: idle lane group), first row pointer,
// first block column, the BS row lengths packed 10 bits each}.
struct BsrSlot {
    int32_t blk;
    uint32_t r0;
    uint32_t bp;
    uint32_t lens;
};

__device__ __forceinline__ BsrSlot bsr_slot(int64_t it, int64_t nitems, int G, int grp,
                                            const int32_t* __restrict__ srec) {
    const int4 v = it < nitems ? __ldg(reinterpret_cast<const int4*>(srec) + (it * G + grp)) : make_int4(-1, 0, 0, 0);
    return BsrSlot{v.x, static_cast<uint32_t>(v.y), static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
}

__device__ __forceinline__ BsrSlot bsr_slot32(int it, int nitems, int G, int grp, const int32_t* __restrict__ srec) {
    const int4 v = it < nitems ? __ldg(reinterpret_cast<const int4*>(srec) + (it * G + grp)) : make_int4(-1, 0, 0, 0);
    return BsrSlot{v.x, static_cast<uint32_t>(v.y), static_cast<uint32_t>(v.z), static_cast<uint32_t>(v.w)};
}

template <int BS>
__device__ __forceinline__ void slot_rows(const BsrSlot& m, int64_t (&rp)[BS + 1]) {
    rp[0] = m.r0;
#pragma unroll
    for (int t = 0; t < BS; ++t) rp[t + 1] = rp[t] + static_cast<int64_t>((m.lens >> (10 * t)) & 1023u);
}

// Neighbour blocks of a slot's block (node-blocked sweeps): row 0 holds
// them all plus the diagonal (L) or the whole diagonal block row (U).
template <int BS, bool UPPER>
__device__ __forceinline__ int slot_nb(const BsrSlot& m) {
    if (m.blk < 0) return 0;
    const int len0 = static_cast<int>(m.lens & 1023u);
    return (len0 - (UPPER ? BS : 1)) / BS;
}

// Node-blocked sweep (Analysis::bsr: the off-block pattern is made of
// whole BSxBS blocks shared by the block's BS rows -- elasticity, where the
// dofs of a node couple to every dof of each neighbour node). Lane n of the
// block's LG lanes owns neighbour block n: it streams the BSxBS values and
// polls the neighbour's BS solution values directly, so the load that
// observes a dependency's publication is also its gather (no critical-
// predecessor poll followed by a second L2 round trip), and a neighbour's
// values are read once instead of once per row.
//
// Items are dealt round-robin: warp w of W runs items w, w + W, w + 2W, ...
// (all W warps resident). Every dependency of an item has a smaller index,
// so the smallest unfinished item is always runnable: its warp has finished
// everything before it. With the sequence known, nothing waits on a claim
// and every load is issued a whole item before its value is needed:
//   item k+3: slot record        item k+2: entries prefetched into L1
//   item k+1: right-hand side    item k:   entries, dependency polls
// One item of the node-blocked sweep: this lane group's block `m` (rows
// r0..r0+BS-1, right-hand side rc), lane gl owning neighbour blocks gl,
// gl+LG, ...: stream the 3x3 values, poll the neighbours' values, reduce,
// solve the diagonal block, publish, re-arm `reset`.
//
// PAD (BS = 3, inside the PCG loop): the sweep's output / re-arm vectors are
// stored padded, 4 doubles per node, so a dependency poll is ONE 256-bit
// relaxed load of the neighbour's 3 values and the publication one 256-bit
// store (a third of the poll instructions and wavefronts); the upper
// sweep's right-hand side (y) is padded too.
__device__ __forceinline__ void ld_relaxed_v4(const double* p, double (&v)[3]) {
    double d;
    asm volatile("ld.relaxed.gpu.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(d)
                 : "l"(p)
                 : "memory");
    (void)d;  // the pad element
}
__device__ __forceinline__ void st_relaxed_v4(double* p, double a, double b, double c, double d) {
    asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
                 : "memory");
}

template <int LG, int BS, bool UPPER, bool PAD = false>
__device__ __forceinline__ void bsr_item(const BsrSlot& m, const double (&rc)[BS], const int32_t* __restrict__ bcol,
                                         const double* __restrict__ vals, const double* __restrict__ invd,
                                         double* out, double* reset) {
    static_assert(!PAD || BS == 3, "padded vectors hold 3-dof nodes");
    constexpr int NIB = BS * (BS - 1) / 2;
    const int lane = threadIdx.x & 31;
    const int gl = lane % LG;
    const bool active = m.blk >= 0;
    const int64_t r0 = active ? static_cast<int64_t>(m.blk) * BS : 0;
    // 32-bit entry offsets (slot records guarantee < 2^32): one wide
    // multiply-add per address instead of 64-bit add pairs
    uint32_t mrp[BS + 1];
    mrp[0] = m.r0;
#pragma unroll
    for (int t = 0; t < BS; ++t) mrp[t + 1] = mrp[t] + ((m.lens >> (10 * t)) & 1023u);
    // off-block entries of row t start at ob[t]; nb neighbour blocks
    uint32_t ob[BS];
#pragma unroll
    for (int t = 0; t < BS; ++t) ob[t] = UPPER ? mrp[t] + (BS - t) : mrp[t];
    const int nb = active ? static_cast<int>((UPPER ? mrp[1] - ob[0] : mrp[1] - 1 - mrp[0]) / BS) : 0;
    double binv[BS], bin[NIB > 0 ? NIB : 1];
    if (active && gl == 0) {
#pragma unroll
        for (int t = 0; t < BS; ++t) binv[t] = __ldg(invd + r0 + t);
        int q = 0;
#pragma unroll
        for (int t = 0; t < BS; ++t)
#pragma unroll
            for (int s = 0; s < BS; ++s) {
                if (!UPPER && s < t) bin[q++] = ld_stream(vals + mrp[t + 1] - (t + 1) + s);
                if (UPPER && s > t) bin[q++] = ld_stream(vals + mrp[t] + (s - t));
            }
    }
    double acc[BS];
#pragma unroll
    for (int t = 0; t < BS; ++t) acc[t] = 0.0;
    const int nbmax = __reduce_max_sync(0xffffffffu, nb);
    // RU neighbour rounds per pass with every load of the pass issued
    // before the first poll (LG = 8: a lane owns neighbours gl and gl + 8)
    constexpr int RU = LG <= 8 ? 2 : 1;
    for (int n0 = 0; n0 < nbmax; n0 += LG * RU) {
        double a[RU][BS][BS], xv[RU][BS];
        int32_t xc[RU];
        bool own[RU];
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            const int n = n0 + r * LG + gl;
            own[r] = n < nb;
            xc[r] = 0;
            if (own[r]) {
                xc[r] = ld_stream(bcol + m.bp + n);
#pragma unroll
                for (int t = 0; t < BS; ++t)
#pragma unroll
                    for (int c = 0; c < BS; ++c) a[r][t][c] = ld_stream(vals + ob[t] + BS * n + c);
            } else {
#pragma unroll
                for (int t = 0; t < BS; ++t)
#pragma unroll
                    for (int c = 0; c < BS; ++c) a[r][t][c] = 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < RU; ++r) {
            if (own[r]) {
                if constexpr (PAD) {
                    double w3[3];
                    ld_relaxed_v4(out + 4 * static_cast<int64_t>(xc[r] / 3), w3);
#pragma unroll
                    for (int c = 0; c < BS; ++c) xv[r][c] = w3[c];
                } else {
#pragma unroll
                    for (int c = 0; c < BS; ++c) xv[r][c] = ld_relaxed(out + xc[r] + c);
                }
            } else {
#pragma unroll
                for (int c = 0; c < BS; ++c) xv[r][c] = 0.0;
            }
        }
        bool pend = false;
#pragma unroll
        for (int r = 0; r < RU; ++r)
#pragma unroll
            for (int c = 0; c < BS; ++c) pend |= own[r] && is_pending(xv[r][c]);
        while (__any_sync(0xffffffffu, pend)) {
            pend = false;
#pragma unroll
            for (int r = 0; r < RU; ++r) {
                if constexpr (PAD) {
                    bool any = false;
#pragma unroll
                    for (int c = 0; c < BS; ++c) any |= is_pending(xv[r][c]);
                    if (own[r] && any) {
                        double w3[3];
                        ld_relaxed_v4(out + 4 * static_cast<int64_t>(xc[r] / 3), w3);
#pragma unroll
                        for (int c = 0; c < BS; ++c) {
                            xv[r][c] = w3[c];
                            pend |= is_pending(w3[c]);
                        }
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < BS; ++c)
                        if (own[r] && is_pending(xv[r][c])) {
                            xv[r][c] = ld_relaxed(out + xc[r] + c);
                            pend |= is_pending(xv[r][c]);
                        }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RU; ++r)
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) acc[t] = fma(a[r][t][c], xv[r][c], acc[t]);
    }
#pragma unroll
    for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
    if (active && gl == 0) {
        double xb[BS];
        solve_diag_block<BS, UPPER>(rc, acc, bin, binv, xb);
        if constexpr (PAD) {
            st_relaxed_v4(out + 4 * static_cast<int64_t>(m.blk), xb[0], xb[1], xb[2], 0.0);
        } else {
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
    }
    __syncwarp();
    if (reset && active && gl < BS) reset[(PAD ? 4 * static_cast<int64_t>(m.blk) : r0) + gl] = pending_value();
}

template <int LG, int BS, bool UPPER, bool PAD = false>
__device__ __forceinline__ void bsr_sweep(int64_t nitems, const int32_t* __restrict__ srec, const int32_t* __restrict__ bcol,
                                          const double* __restrict__ vals, const double* __restrict__ invd,
                                          const double* rhs, double* out, double* reset, int64_t warp,
                                          int64_t nwarps) {
    constexpr int G = 32 / LG;
    constexpr int RS = PAD && UPPER ? 4 : BS;  // right-hand side stride (padded y)
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    // 32-bit item indices (items * G < 2^31, checked by the launcher)
    const int nit = static_cast<int>(nitems), nw = static_cast<int>(nwarps);
    int it = static_cast<int>(warp);
    BsrSlot m = bsr_slot32(it, nit, G, grp, srec);
    BsrSlot m1 = bsr_slot32(it + nw, nit, G, grp, srec);
    BsrSlot m2 = bsr_slot32(it + 2 * nw, nit, G, grp, srec);
    // one 128-byte line per lane covers a block's rows up to 16 * LG
    // doubles (3 elasticity rows: ~125); longer rows take the loop
    auto prefetch = [&](const BsrSlot& q) {
        if (q.blk >= 0) {
            const uint32_t e0 = q.r0 & ~15u;
            uint32_t e1 = q.r0;
#pragma unroll
            for (int t = 0; t < BS; ++t) e1 += (q.lens >> (10 * t)) & 1023u;
            uint32_t a = e0 + 16u * gl;
            if (a < e1) asm volatile("prefetch.global.L1 [%0];" ::"l"(vals + a));
            for (a += 16u * LG; a < e1; a += 16u * LG) asm volatile("prefetch.global.L1 [%0];" ::"l"(vals + a));
            if (gl == 0) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(bcol + q.bp));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(invd + static_cast<int64_t>(q.blk) * BS));
            }
        }
    };
    prefetch(m);
    while (it < nit) {
        prefetch(m1);
        // loaded as the item starts: only the diagonal solve (after the
        // dependency polls) consumes it
        double rhs0[BS];
        if constexpr (RS == 4) {  // padded y: one 256-bit load
            double d3 = 0.0;
            rhs0[0] = rhs0[1] = rhs0[2] = 0.0;
            if (m.blk >= 0)
                asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(rhs0[0]), "=d"(rhs0[1]), "=d"(rhs0[2]), "=d"(d3)
                             : "l"(rhs + 4 * static_cast<int64_t>(m.blk)));
            (void)d3;
        } else {
#pragma unroll
            for (int t = 0; t < BS; ++t) rhs0[t] = m.blk >= 0 ? rhs[static_cast<int64_t>(m.blk) * BS + t] : 0.0;
        }
        bsr_item<LG, BS, UPPER, PAD>(m, rhs0, bcol, vals, invd, out, reset);
        it += nw;
        m = m1;
        m1 = m2;
        m2 = bsr_slot32(it + 2 * nw, nit, G, grp, srec);
    }
}

template <int LG, int BS, bool UPPER, bool PAD>
__global__ void __launch_bounds__(BSR_THREADS, BSR_CTAS)
bsr_trsv_kernel(int64_t nitems, const int32_t* __restrict__ srec,
                const int32_t* __restrict__ bcol, const double* __restrict__ vals,
                const double* __restrict__ invd, const double* rhs, double* out, double* reset,
                const int* __restrict__ done) {
    if (done && *done) return;
    bsr_sweep<LG, BS, UPPER, PAD>(nitems, srec, bcol, vals, invd, rhs, out, reset,
                                  (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5,
                                  (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5);
}

// ------------------------------------------------------------------------
// Node-blocked sweep on the item-ordered stream (bss.cu): the 3x3 node-
// blocked, padded PCG-loop case of bsr_trsv_kernel with the factor values
// re-laid per slot of the schedule -- a slot's block holds its neighbour
// blocks' values contiguously (entry-major: entry (t, c) of neighbour n at
// (3t + c) * nb + n, so the 16 lanes of a block read consecutive doubles),
// then the 3 strictly-lower / -upper in-block entries and the 3 reciprocal
// pivots -- and the neighbour block ids beside them. A slot is one 16-byte
// header {block, neighbours, value offset, column offset}; every address of
// an item is that header plus an immediate, and one L1 prefetch per lane
// covers the next item's values. Same lane mapping, FMA order, shuffle tree
// and diagonal solve as bsr_item: bit-identical results.
#ifndef BSS_CTAS
#define BSS_CTAS 7
#endif
#ifdef BSS_TRACE  // developer trace (tools/bss_trace.py): per node {item start, dependencies seen, published, last dependency}
static __device__ unsigned long long* g_bss_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif
template <bool UPPER>
__global__ void __launch_bounds__(BSR_THREADS, BSS_CTAS)
bss_trsv_kernel(int nitems, const int4* __restrict__ hdr, const int32_t* __restrict__ scol,
                const double* __restrict__ sval, const double* rhs, double* out, double* reset,
                const int* __restrict__ done) {
    if (done && *done) return;
    constexpr int BS = 3, LG = 16, G = 2, NIB = 3;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    int it = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    auto hdr_at = [&](int i) { return i < nitems ? __ldg(hdr + (i * G + grp)) : make_int4(-1, 0, 0, 0); };
    int4 h = hdr_at(it), h1 = hdr_at(it + nw), h2 = hdr_at(it + 2 * nw);
    // a block's values span <= 9 * 16 + 6 doubles: one 128-byte line per
    // lane (lines from the one holding the first value)
    auto prefetch = [&](const int4& q) {
        if (q.x >= 0) {
            const uintptr_t v0 = reinterpret_cast<uintptr_t>(sval + static_cast<uint32_t>(q.z));
            const uintptr_t v1 = v0 + 8 * static_cast<uintptr_t>(9 * q.y + 6);
            const uintptr_t a = (v0 & ~uintptr_t(127)) + 128 * static_cast<uintptr_t>(gl);
            if (a < v1) asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
            if (gl == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(scol + static_cast<uint32_t>(q.w)));
        }
    };
    prefetch(h);
    while (it < nitems) {
        prefetch(h1);
        const bool active = h.x >= 0;
        const int64_t blk = active ? h.x : 0;
        const int nb = active ? h.y : 0;
#ifdef BSS_TRACE
        const unsigned long long tr0 = gtime();
        int tr_cnt = 0, tr_dep = -1;
#endif
        const double* v = sval + static_cast<uint32_t>(h.z);
        const int32_t* c = scol + static_cast<uint32_t>(h.w);
        double rc[BS] = {0.0, 0.0, 0.0}, bin[NIB], binv[BS];
        if (active && gl == 0) {
            if constexpr (UPPER) {  // padded y: one 256-bit load
                double d3;
                asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                             : "=d"(rc[0]), "=d"(rc[1]), "=d"(rc[2]), "=d"(d3)
                             : "l"(rhs + 4 * blk));
                (void)d3;
            } else {
#pragma unroll
                for (int t = 0; t < BS; ++t) rc[t] = rhs[blk * BS + t];
            }
#pragma unroll
            for (int j = 0; j < NIB; ++j) bin[j] = __ldg(v + 9 * nb + j);
#pragma unroll
            for (int t = 0; t < BS; ++t) binv[t] = __ldg(v + 9 * nb + NIB + t);
        }
        double acc[BS] = {0.0, 0.0, 0.0};
        const int nbmax = __reduce_max_sync(0xffffffffu, nb);
        for (int n0 = 0; n0 < nbmax; n0 += LG) {
            const int n = n0 + gl;
            const bool own = n < nb;
            double a[BS][BS], xv[BS] = {0.0, 0.0, 0.0};
            int32_t xb = 0;
            if (own) {
                xb = __ldg(c + n);
                const double* vn = v + n;
#pragma unroll
                for (int t = 0; t < BS; ++t)
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) a[t][cc] = __ldg(vn + (BS * t + cc) * nb);
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
#ifdef BSS_TRACE
                    ++tr_cnt;
#endif
                }
            }
#ifdef BSS_TRACE
            {  // the lane that polled longest holds the last dependency
                int mx = tr_cnt;
#pragma unroll
                for (int o = LG / 2; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const unsigned who = __ballot_sync(0xffffffffu, own && tr_cnt == mx && mx > 0) >> (grp * LG) & 0xffffu;
                const int src = who ? grp * LG + __ffs(who) - 1 : lane;
                const int dep = __shfl_sync(0xffffffffu, xb, src);
                tr_dep = who ? dep : -1;
                tr_cnt = mx;
            }
#endif
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int cc = 0; cc < BS; ++cc) acc[t] = fma(a[t][cc], xv[cc], acc[t]);
        }
#ifdef BSS_TRACE
        const unsigned long long tr1 = gtime();
#endif
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (active && gl == 0) {
            double x[BS];
            solve_diag_block<BS, UPPER>(rc, acc, bin, binv, x);
            st_relaxed_v4(out + 4 * blk, x[0], x[1], x[2], 0.0);
#ifdef BSS_TRACE
            if (g_bss_trace) {
                const unsigned long long tr2 = gtime();
                g_bss_trace[4 * blk + 0] = tr0;
                g_bss_trace[4 * blk + 1] = tr1;
                g_bss_trace[4 * blk + 2] = tr2;
                g_bss_trace[4 * blk + 3] = (static_cast<unsigned long long>(static_cast<unsigned>(tr_cnt)) << 32) |
                                           static_cast<unsigned>(tr_dep);
            }
#endif
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[4 * blk + gl] = pending_value();
        it += nw;
        h = h1;
        h1 = h2;
        h2 = hdr_at(it + 2 * nw);
    }
}

// Round-robin sweep for matrices that are not node-blocked (Poisson, FV
// diffusion): the scheduling of bsr_sweep -- items dealt round-robin to all
// resident warps, slot records two items ahead, entries prefetched into L1
// one item ahead, dependency values polled directly -- with lanes over the
// block's off-block entries (lane gl takes entries gl, gl + LG, ... of the
// block's rows in order) instead of over neighbour blocks.
// RR_THREADS-thread CTAs, RR_CTAS resident per SM
// (diffusion 256^3, per sweep: 256 x 4/SM 1.18 ms, 128 x 9/SM 1.15, 128 x 12/SM 1.28)
#ifndef RR_THREADS
#define RR_THREADS 128
#endif
#ifndef RR_CTAS
#define RR_CTAS 9
#endif
template <int LG, int BS, bool UPPER, int CH>
__global__ void __launch_bounds__(RR_THREADS, RR_CTAS)
rr_trsv_kernel(int64_t nitems, const int32_t* __restrict__ srec,
               const int32_t* __restrict__ cols, const double* __restrict__ vals, const double* __restrict__ invd,
               const double* rhs, double* out, double* reset, const int* __restrict__ done) {
    if (done && *done) return;
    constexpr int G = 32 / LG;
    constexpr int NIB = BS * (BS - 1) / 2;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int64_t it = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    BsrSlot m = bsr_slot(it, nitems, G, grp, srec);
    BsrSlot m1 = bsr_slot(it + nwarps, nitems, G, grp, srec);
    BsrSlot m2 = bsr_slot(it + 2 * nwarps, nitems, G, grp, srec);
    BsrSlot m3 = bsr_slot(it + 3 * nwarps, nitems, G, grp, srec);
    double rhs0[BS], rhs1[BS];
#pragma unroll
    for (int t = 0; t < BS; ++t) {
        rhs0[t] = m.blk >= 0 ? rhs[static_cast<int64_t>(m.blk) * BS + t] : 0.0;
        rhs1[t] = m1.blk >= 0 ? rhs[static_cast<int64_t>(m1.blk) * BS + t] : 0.0;
    }
    auto prefetch = [&](const BsrSlot& q) {
        if (q.blk >= 0) {
            int64_t rq[BS + 1];
            slot_rows<BS>(q, rq);
            const int64_t e0 = rq[0], e1 = rq[BS];
            for (int64_t a = (e0 & ~15LL) + 16 * gl; a < e1; a += 16 * LG)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(vals + a));
            for (int64_t a = (e0 & ~31LL) + 32 * gl; a < e1; a += 32 * LG)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(cols + a));
            if (gl == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(invd + static_cast<int64_t>(q.blk) * BS));
        }
    };
    prefetch(m);
    prefetch(m1);
    while (it < nitems) {
        prefetch(m2);
        const bool active = m.blk >= 0;
        const int64_t r0 = active ? static_cast<int64_t>(m.blk) * BS : 0;
        int64_t mrp[BS + 1];
        slot_rows<BS>(m, mrp);
        int64_t ob[BS];
        int oc[BS];
        int total = 0;
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            ob[t] = UPPER ? mrp[t] + (BS - t) : mrp[t];
            oc[t] = active ? static_cast<int>(UPPER ? mrp[t + 1] - ob[t] : mrp[t + 1] - (t + 1) - mrp[t]) : 0;
            total += oc[t];
        }
        double binv[BS], bin[NIB > 0 ? NIB : 1];
        if (active && gl == 0) {
#pragma unroll
            for (int t = 0; t < BS; ++t) binv[t] = __ldg(invd + r0 + t);
            int q = 0;
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int s = 0; s < BS; ++s) {
                    if (!UPPER && s < t) bin[q++] = ld_stream(vals + mrp[t + 1] - (t + 1) + s);
                    if (UPPER && s > t) bin[q++] = ld_stream(vals + mrp[t] + (s - t));
                }
        }
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        const int tmax = __reduce_max_sync(0xffffffffu, total);
        for (int base = 0; base < tmax; base += LG * CH) {
            double v[CH], xv[CH];
            int32_t jj[CH];
            int tt[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                int e = base + c * LG + gl;
                tt[c] = -1;
                jj[c] = 0;
                v[c] = 0.0;
                xv[c] = 0.0;
                if (e < total) {
                    // row of entry e (selects, not a dynamically indexed array)
                    int t = 0;
                    int64_t obt = ob[0];
#pragma unroll
                    for (int s = 0; s < BS - 1; ++s)
                        if (t == s && e >= oc[s]) {
                            e -= oc[s];
                            t = s + 1;
                            obt = ob[s + 1];
                        }
                    tt[c] = t;
                    jj[c] = ld_stream(cols + obt + e);
                    v[c] = ld_stream(vals + obt + e);
                    xv[c] = ld_relaxed(out + jj[c]);
                }
            }
            bool pend = false;
#pragma unroll
            for (int c = 0; c < CH; ++c) pend |= tt[c] >= 0 && is_pending(xv[c]);
            while (__any_sync(0xffffffffu, pend)) {
                pend = false;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (tt[c] >= 0 && is_pending(xv[c])) {
                        xv[c] = ld_relaxed(out + jj[c]);
                        pend |= is_pending(xv[c]);
                    }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int t = 0; t < BS; ++t)
                    if (tt[c] == t) acc[t] = fma(v[c], xv[c], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (active && gl == 0) {
            double xb[BS];
            solve_diag_block<BS, UPPER>(rhs0, acc, bin, binv, xb);
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[r0 + gl] = pending_value();
        it += nwarps;
        m = m1;
        m1 = m2;
        m2 = m3;
        m3 = bsr_slot(it + 3 * nwarps, nitems, G, grp, srec);
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            rhs0[t] = rhs1[t];
            rhs1[t] = m1.blk >= 0 ? rhs[static_cast<int64_t>(m1.blk) * BS + t] : 0.0;
        }
    }
}

// Entry-lane sweep on the item-ordered stream (bss.cu, scalar / not node-
// blocked matrices): rr_trsv_kernel with each slot's off-block entries
// re-laid contiguously -- values, then the in-block entries and reciprocal
// pivots -- and each entry's column with its block row in the low two bits
// (code = col << 2 | t). The lane / entry mapping, FMA order, shuffle tree
// and diagonal solve are rr_trsv_kernel's: bit-identical results.
template <int LG, int BS, bool UPPER, int CH>
__global__ void __launch_bounds__(RR_THREADS, RR_CTAS)
rrs_trsv_kernel(int64_t nitems, const int4* __restrict__ hdr, const int32_t* __restrict__ scode,
                const double* __restrict__ sval, const double* rhs, double* out, double* reset,
                const int* __restrict__ done) {
    if (done && *done) return;
    constexpr int G = 32 / LG;
    constexpr int NIB = BS * (BS - 1) / 2;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    int64_t it = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    auto hdr_at = [&](int64_t i) { return i < nitems ? __ldg(hdr + (i * G + grp)) : make_int4(-1, 0, 0, 0); };
    int4 m = hdr_at(it), m1 = hdr_at(it + nwarps), m2 = hdr_at(it + 2 * nwarps), m3 = hdr_at(it + 3 * nwarps);
    double rhs0[BS], rhs1[BS];
#pragma unroll
    for (int t = 0; t < BS; ++t) {
        rhs0[t] = m.x >= 0 ? rhs[static_cast<int64_t>(m.x) * BS + t] : 0.0;
        rhs1[t] = m1.x >= 0 ? rhs[static_cast<int64_t>(m1.x) * BS + t] : 0.0;
    }
    auto prefetch = [&](const int4& q) {
        if (q.x >= 0) {
            const uintptr_t v0 = reinterpret_cast<uintptr_t>(sval + static_cast<uint32_t>(q.z));
            const uintptr_t v1 = v0 + 8 * static_cast<uintptr_t>(q.y + NIB + BS);
            for (uintptr_t a = (v0 & ~uintptr_t(127)) + 128 * static_cast<uintptr_t>(gl); a < v1; a += 128 * LG)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
            if (gl == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(scode + static_cast<uint32_t>(q.w)));
        }
    };
    prefetch(m);
    prefetch(m1);
    while (it < nitems) {
        prefetch(m2);
        const bool active = m.x >= 0;
        const int64_t r0 = active ? static_cast<int64_t>(m.x) * BS : 0;
        const int total = active ? m.y : 0;
        const double* v = sval + static_cast<uint32_t>(m.z);
        const int32_t* cd = scode + static_cast<uint32_t>(m.w);
        double binv[BS], bin[NIB > 0 ? NIB : 1];
        if (active && gl == 0) {
#pragma unroll
            for (int j = 0; j < NIB; ++j) bin[j] = __ldg(v + total + j);
#pragma unroll
            for (int t = 0; t < BS; ++t) binv[t] = __ldg(v + total + NIB + t);
        }
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        const int tmax = __reduce_max_sync(0xffffffffu, total);
        for (int base = 0; base < tmax; base += LG * CH) {
            double vv[CH], xv[CH];
            int32_t jj[CH];
            int tt[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int e = base + c * LG + gl;
                tt[c] = -1;
                jj[c] = 0;
                vv[c] = 0.0;
                xv[c] = 0.0;
                if (e < total) {
                    const int32_t code = __ldg(cd + e);
                    tt[c] = code & 3;
                    jj[c] = code >> 2;
                    vv[c] = __ldg(v + e);
                    xv[c] = ld_relaxed(out + jj[c]);
                }
            }
            bool pend = false;
#pragma unroll
            for (int c = 0; c < CH; ++c) pend |= tt[c] >= 0 && is_pending(xv[c]);
#ifdef RRS_PROBE_NODEP
            pend = false;
#endif
            while (__any_sync(0xffffffffu, pend)) {
                pend = false;
#pragma unroll
                for (int c = 0; c < CH; ++c)
                    if (tt[c] >= 0 && is_pending(xv[c])) {
                        xv[c] = ld_relaxed(out + jj[c]);
                        pend |= is_pending(xv[c]);
                    }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c)
#pragma unroll
                for (int t = 0; t < BS; ++t)
                    if (tt[c] == t) acc[t] = fma(vv[c], xv[c], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (active && gl == 0) {
            double xb[BS];
            solve_diag_block<BS, UPPER>(rhs0, acc, bin, binv, xb);
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[r0 + gl] = pending_value();
        it += nwarps;
        m = m1;
        m1 = m2;
        m2 = m3;
        m3 = hdr_at(it + 3 * nwarps);
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            rhs0[t] = rhs1[t];
            rhs1[t] = m1.x >= 0 ? rhs[static_cast<int64_t>(m1.x) * BS + t] : 0.0;
        }
    }
}

// ------------------------------------------------------------------------
// Slot-record sweep (bss.cu: Schedule::rec) for scalar matrices whose blocks
// of 2 rows have at most 8 off-block entries (5- / 7-point stencils): the
// entry-lane sweep of rrs_trsv_kernel<8, 2> on ONE fixed 128-byte record per
// slot -- 8 values, 8 entry codes (col << 2 | row in block; unused lanes
// repeat entry 0's column with bit 1 set: a poll of the same sector, ignored),
// the in-block entry, the two reciprocal pivots and the block id -- at
// rec + 16 * (item * 4 + group). No header or offset stands between an item
// and its data, so everything is requested before it is needed: the entry
// codes three items ahead, the values and the dependencies' sectors (an L2
// prefetch) two, the right-hand side and the FIRST dependency poll one item
// ahead (an item usually starts with its dependencies already in registers
// and re-polls only the pending ones). Lane / entry mapping, FMA order,
// shuffle tree and diagonal solve are rrs_trsv_kernel's: bit-identical.
// 56 registers, 9 CTAs (36 warps) per SM: a whole level of a 256^3 mesh is
// resident (10 CTAs spill, 8 leave late warps: 0.81 / 0.84 / 0.91 ms).
#ifndef REC_CTAS
#define REC_CTAS 9
#endif
template <bool UPPER>
__global__ void __launch_bounds__(RR_THREADS, REC_CTAS)
rec_trsv_kernel(int64_t nitems, const double* __restrict__ rec, const double* rhs, double* out, double* reset,
                const int* __restrict__ done) {
    if (done && *done) return;
    constexpr int LG = 8, G = 4, BS = 2;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    // 32-bit item and slot indices (the launcher checks items * 4 < 2^31)
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5), nit = static_cast<int>(nitems);
    int it = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    // a slot's record: value of lane gl at q[gl], its code at q[8] + 4 gl, diagonal data at q[12..15]
    auto rec_of = [&](int i) { return rec + 16 * static_cast<int64_t>(i * G + grp); };
    // Per-lane item state: the lane's entry (value, code), ONE of the four
    // diagonal doubles (lane 0 in-block entry, 1 and 2 the reciprocal pivots,
    // 3 the block id; lane 0 collects them by shuffles once the dependencies
    // are in -- 2 registers instead of 8 per item in flight), the right-hand
    // side (lane t holds row t's) and the first poll's result.
    struct Item {
        double val;
        int32_t code;
        double dg;
        double rh;
        double xv;
    };
    // Every load below writes its destination register directly: a default
    // value overwritten under a per-lane condition compiles to a load into a
    // temporary and a predicated move that waits for the load on the spot
    // (measured: a quarter of the sweep's time). Lanes without a use load a
    // harmless duplicate instead.
    // stage 3 of an item (three items ahead): its entry codes; its four
    // records (512 bytes) reach L2 two items before that
    auto stage3 = [&](Item& m, int i) {
        if (i < nit)  // warp-uniform
            m.code = __ldg(reinterpret_cast<const int32_t*>(rec_of(i) + 8) + gl);
        else
            m.code = 2;
        if (i + 2 * nw < nit && lane < 4)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rec + 16 * static_cast<int64_t>((i + 2 * nw) * G + lane)));
    };
    // stage 2 (two items ahead): the dependencies' sectors are asked into L2
    // -- a first poll of a value not yet published would otherwise wait for
    // the pending marker to come back from DRAM (x does not fit in L2 beside
    // the record stream) -- and the value and diagonal data are loaded
    auto stage2 = [&](Item& m, int i) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(out + (m.code >> 2)));
        if (i < nit) {
            const double* q = rec_of(i);
            m.val = __ldg(q + gl);
            m.dg = __ldg(q + 12 + (gl & 3));
        } else {
            m.val = 0.0;
            m.dg = __longlong_as_double(-1LL);
        }
    };
    // stage 1 (one item ahead): right-hand side and first poll
    auto stage1 = [&](Item& m) {
        m.xv = ld_relaxed(out + (m.code >> 2));  // unused lanes repeat entry 0's column: same sector, ignored
        const long long blk = __double_as_longlong(__shfl_sync(0xffffffffu, m.dg, 3, LG));
        m.rh = rhs[blk >= 0 ? blk * BS + (gl & 1) : 0];
    };
#ifdef BSS_TRACE
    unsigned long long tr_prev = gtime();
#endif
    // one item: `a` is solved while `b`, `c` and `d` (the next three) go
    // through stages 1, 2 and 3
    auto step = [&](Item& a, Item& b, Item& c, Item& d) {
        stage3(d, it + 3 * nw);
        stage2(c, it + 2 * nw);
#ifdef BSS_TRACE
        const unsigned long long trf = gtime();
#endif
        stage1(b);
        const bool has = (a.code & 2) == 0;
        const int col = a.code >> 2;
#ifdef BSS_TRACE
        const unsigned long long tr0 = gtime();
        int tr_cnt = 0;
#endif
        // wait for the pending dependencies only
        double xv = a.xv;
        bool pend = has && is_pending(xv);
        while (__any_sync(0xffffffffu, pend)) {
            if (pend) {
                xv = ld_relaxed(out + col);
                pend = is_pending(xv);
#ifdef BSS_TRACE
                ++tr_cnt;
#endif
            }
        }
#ifdef BSS_TRACE
        int tr_dep = -1;
        {
            int mx = tr_cnt;
#pragma unroll
            for (int o = LG / 2; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const unsigned who = __ballot_sync(0xffffffffu, has && tr_cnt == mx && mx > 0) >> (grp * LG) & 0xffu;
            const int src = who ? grp * LG + __ffs(who) - 1 : lane;
            const int dep = __shfl_sync(0xffffffffu, col, src);
            tr_dep = who ? dep / BS : -1;
            tr_cnt = mx;
        }
        const unsigned long long tr1 = gtime();
#endif
        const int t = a.code & 1;
        double acc[BS];
        acc[0] = has && t == 0 ? fma(a.val, xv, 0.0) : 0.0;
        acc[1] = has && t == 1 ? fma(a.val, xv, 0.0) : 0.0;
        const double rhs1 = __shfl_sync(0xffffffffu, a.rh, 1, LG);
        const double binv0 = __shfl_sync(0xffffffffu, a.dg, 1, LG);
        const double binv1 = __shfl_sync(0xffffffffu, a.dg, 2, LG);
        const long long blk = __double_as_longlong(__shfl_sync(0xffffffffu, a.dg, 3, LG));
        acc[0] = group_sum<LG>(acc[0]);
        acc[1] = group_sum<LG>(acc[1]);
        if (gl == 0 && blk >= 0) {
            const double rhv[BS] = {a.rh, rhs1}, bin[1] = {a.dg}, binv[BS] = {binv0, binv1};
            double xb[BS];
            solve_diag_block<BS, UPPER>(rhv, acc, bin, binv, xb);
            // rows 2 blk and 2 blk + 1: one 16-byte publication (readers poll their own 8 bytes)
            asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1,%2};" ::"l"(out + blk * BS), "d"(xb[0]), "d"(xb[1])
                         : "memory");
#ifdef BSS_TRACE
            if (g_bss_trace) {
                g_bss_trace[4 * blk + 0] = tr0;
                g_bss_trace[4 * blk + 1] = tr1;
                g_bss_trace[4 * blk + 2] = gtime();
                const unsigned long long gap = min(tr0 - tr_prev, 65535ULL);  // loop top: from the last item's end
                const unsigned long long gapf = min(trf - tr_prev, 65535ULL);  // ... of which up to the fetch
                g_bss_trace[4 * blk + 3] = (gap << 48) | (gapf << 32) | static_cast<unsigned>(tr_dep);
                (void)tr_cnt;
            }
#endif
        }
#ifdef BSS_TRACE
        tr_prev = gtime();
#endif
        __syncwarp();
        if (reset && gl < BS && blk >= 0) reset[blk * BS + gl] = pending_value();
        it += nw;
    };
    // the four items in flight trade roles instead of moving through
    // registers: a move of a value still being loaded would stall the warp for
    // the rest of the load's latency
    Item m0, m1, m2, m3;
    stage3(m0, it);
    stage3(m1, it + nw);
    stage3(m2, it + 2 * nw);
    stage2(m0, it);
    stage2(m1, it + nw);
    stage1(m0);
    while (true) {
        if (it >= nit) break;
        step(m0, m1, m2, m3);
        if (it >= nit) break;
        step(m1, m2, m3, m0);
        if (it >= nit) break;
        step(m2, m3, m0, m1);
        if (it >= nit) break;
        step(m3, m0, m1, m2);
    }
}

}  // namespace pclab_b200
