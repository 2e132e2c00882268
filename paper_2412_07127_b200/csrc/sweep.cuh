// Device kernels for the sparse hot loop: CSR SpMV (lane group per row)
// and the sync-free dof-blocked triangular sweeps.
#pragma once

#include "common.cuh"

namespace pclab_b200 {

// Rows per warp = 32 / LPR; each lane group of LPR lanes reduces one row
// with a fixed shuffle tree (deterministic).
template <int LPR>
__device__ __forceinline__ double row_dot(const int64_t* __restrict__ rp,
                                          const int32_t* __restrict__ cols,
                                          const double* __restrict__ vals,
                                          const double* __restrict__ x, int64_t row, int gl,
                                          bool active) {
    double acc = 0.0;
    if (active) {
        const int64_t b = rp[row], e = rp[row + 1];
        int64_t k = b + gl;
        // 4 independent loads in flight per lane per round
        for (; k + 3 * LPR < e; k += 4 * LPR) {
            const int32_t j0 = __ldg(cols + k), j1 = __ldg(cols + k + LPR),
                          j2 = __ldg(cols + k + 2 * LPR), j3 = __ldg(cols + k + 3 * LPR);
            const double v0 = __ldg(vals + k), v1 = __ldg(vals + k + LPR),
                         v2 = __ldg(vals + k + 2 * LPR), v3 = __ldg(vals + k + 3 * LPR);
            acc = fma(v0, __ldg(x + j0), acc);
            acc = fma(v1, __ldg(x + j1), acc);
            acc = fma(v2, __ldg(x + j2), acc);
            acc = fma(v3, __ldg(x + j3), acc);
        }
        for (; k < e; k += LPR) acc = fma(__ldg(vals + k), __ldg(x + __ldg(cols + k)), acc);
    }
    return group_sum<LPR>(acc);
}

// Per-item state of a sweep, loaded one item ahead.
template <int BS>
struct SweepMeta {
    int64_t blk;  // -1: idle lane group
    int64_t rp[BS + 1];
    int32_t crit;
};

template <int BS>
__device__ __forceinline__ SweepMeta<BS> sweep_meta(unsigned it, int64_t nitems, int G, int grp,
                                                    const int32_t* __restrict__ slots,
                                                    const int32_t* __restrict__ crit,
                                                    const int64_t* __restrict__ rp) {
    SweepMeta<BS> m;
    m.blk = it < nitems ? static_cast<int64_t>(__ldg(slots + static_cast<int64_t>(it) * G + grp)) : -1;
    m.crit = -1;
#pragma unroll
    for (int t = 0; t <= BS; ++t) m.rp[t] = 0;
    if (m.blk >= 0) {
        m.crit = __ldg(crit + m.blk);
#pragma unroll
        for (int t = 0; t <= BS; ++t) m.rp[t] = __ldg(rp + m.blk * BS + t);
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
__global__ void __launch_bounds__(256)
trsv_kernel(int64_t nitems, const int32_t* __restrict__ slots, const int32_t* __restrict__ crit,
            const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
            const double* __restrict__ vals, const double* __restrict__ invd, const double* rhs,
            double* out, double* reset, const int* __restrict__ done, unsigned* counter,
            int tune, long long* trace) {
    if (done && *done) return;
    const bool use_crit = (tune & 0xff) == 0;
    const unsigned sleep_ns = static_cast<unsigned>(tune >> 8);
    constexpr int G = 32 / LG;
    constexpr int CH = (LG >= 16) ? 4 : 2;
    constexpr int NIB = BS * (BS - 1) / 2;  // strictly-triangular in-block entries
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    unsigned it = 0;
    if (lane == 0) it = atomicAdd(counter, 1u);
    it = __shfl_sync(0xffffffffu, it, 0);
    SweepMeta<BS> m = sweep_meta<BS>(it, nitems, G, grp, slots, crit, rp);
    while (it < nitems) {
        unsigned next = 0;
        if (lane == 0) next = atomicAdd(counter, 1u);
        long long tr0 = 0;
        if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr0));
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
                    jj[c] = __ldg(cols + ob[t] + e);
                    v[c] = __ldg(vals + ob[t] + e);
                }
            }
        };
        load_chunk(0);
        double brhs[BS], binv[BS], bin[NIB > 0 ? NIB : 1];
        if (active && gl == 0) {
#pragma unroll
            for (int t = 0; t < BS; ++t) {
                brhs[t] = rhs[r0 + t];
                binv[t] = __ldg(invd + r0 + t);
            }
            int q = 0;
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int s = 0; s < BS; ++s) {
                    if (!UPPER && s < t) bin[q++] = __ldg(vals + m.rp[t + 1] - (t + 1) + s);
                    if (UPPER && s > t) bin[q++] = __ldg(vals + m.rp[t] + (s - t));
                }
        }
        // (2) one poller per block on the critical predecessor
        if (use_crit && active && gl == 0 && m.crit >= 0)
            while (is_pending(ld_relaxed(out + m.crit))) {
                if (sleep_ns) __nanosleep(sleep_ns);
            }
        __syncwarp();
        long long tr1 = 0;
        if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr1));
        // (3) gather the dependencies
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        for (int base = 0; base < total; base += LG * CH) {
            if (base > 0) load_chunk(base);
            double xv[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) xv[c] = tt[c] >= 0 ? ld_relaxed(out + jj[c]) : 0.0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (tt[c] < 0) continue;
                while (is_pending(xv[c])) {
                    if (sleep_ns) __nanosleep(sleep_ns);
                    xv[c] = ld_relaxed(out + jj[c]);
                }
#pragma unroll
                for (int t = 0; t < BS; ++t)
                    if (tt[c] == t) acc[t] = fma(v[c], xv[c], acc[t]);
            }
        }
        next = __shfl_sync(0xffffffffu, next, 0);
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        // (4) diagonal block
        if (active && gl == 0) {
            double xb[BS];
            if (!UPPER) {
                int q = 0;
#pragma unroll
                for (int t = 0; t < BS; ++t) {
                    double s = brhs[t] - acc[t];
#pragma unroll
                    for (int u = 0; u < t; ++u) s -= bin[q++] * xb[u];
                    xb[t] = s * binv[t];
                }
            } else {
#pragma unroll
                for (int t = BS - 1; t >= 0; --t) {
                    double s = brhs[t] - acc[t];
                    // bin holds, row by row, U[t][s] for s > t
                    int q = 0;
#pragma unroll
                    for (int r = 0; r < t; ++r) q += BS - 1 - r;
#pragma unroll
                    for (int u = t + 1; u < BS; ++u) s -= bin[q + (u - t - 1)] * xb[u];
                    xb[t] = s * binv[t];
                }
            }
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
        if (trace && lane == 0) {
            long long tr2;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tr2));
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            trace[4LL * it + 0] = tr0;
            trace[4LL * it + 1] = tr1;
            trace[4LL * it + 2] = tr2;
            trace[4LL * it + 3] = smid;
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[r0 + gl] = pending_value();
        // the next item's metadata is fetched only after publication, so its
        // dependent loads never sit on this item's critical path
        it = next;
        m = sweep_meta<BS>(next, nitems, G, grp, slots, crit, rp);
    }
}

}  // namespace pclab_b200
