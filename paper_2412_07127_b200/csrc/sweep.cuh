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

// Sync-free blocked triangular sweep.
//
// Work items (warp-sized) come from a global counter in (level, index)
// order, so every dependency of an item was claimed earlier by a running
// warp. Each of the 32/LG lane groups owns one block of BS consecutive
// rows: the off-block products are accumulated in parallel (values and
// indices are loaded before the dependency spin), then lane 0 of the
// group solves the dense BSxBS diagonal block sequentially and publishes
// the BS results; publication is the store itself (kPending -> value).
//
//   lower (L, row-sorted, diagonal last):  rows r0..r0+BS-1 forward
//   upper (U = L^T, diagonal first):       rows r0+BS-1..r0 backward
template <int LG, int BS, bool UPPER>
__global__ void __launch_bounds__(256)
trsv_kernel(int64_t nitems, const int32_t* __restrict__ order,
            const int64_t* __restrict__ item_first, const int32_t* __restrict__ item_cnt,
            const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
            const double* __restrict__ vals, const double* rhs, double* out,
            double* reset, const int* __restrict__ done, unsigned* counter) {
    if (done && *done) return;
    constexpr int CH = 4;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LG, gl = lane % LG;
    for (;;) {
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(counter, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems) return;
        const int64_t first = item_first[it];
        const bool active = grp < item_cnt[it];
        const int64_t r0 = active ? static_cast<int64_t>(order[first + grp]) * BS : 0;
        int64_t ob[BS], oc[BS], beg[BS], end[BS];
        int total = 0;
#pragma unroll
        for (int t = 0; t < BS; ++t) {
            beg[t] = active ? rp[r0 + t] : 0;
            end[t] = active ? rp[r0 + t + 1] : 0;
            ob[t] = UPPER ? beg[t] + (BS - t) : beg[t];
            oc[t] = active ? (UPPER ? end[t] - ob[t] : end[t] - (t + 1) - beg[t]) : 0;
            total += static_cast<int>(oc[t]);
        }
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
        for (int base = 0; base < total; base += LG * CH) {
            double v[CH], xv[CH];
            int32_t jj[CH];
            int tt[CH];
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
                    const int64_t k = ob[t] + e;
                    tt[c] = t;
                    jj[c] = __ldg(cols + k);
                    v[c] = __ldg(vals + k);
                }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) xv[c] = tt[c] >= 0 ? ld_relaxed(out + jj[c]) : 0.0;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (tt[c] < 0) continue;
                while (is_pending(xv[c])) {
                    __nanosleep(32);
                    xv[c] = ld_relaxed(out + jj[c]);
                }
#pragma unroll
                for (int t = 0; t < BS; ++t)
                    if (tt[c] == t) acc[t] = fma(v[c], xv[c], acc[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (active && gl == 0) {
            double xb[BS];
            if (!UPPER) {
#pragma unroll
                for (int t = 0; t < BS; ++t) {
                    double s = rhs[r0 + t] - acc[t];
#pragma unroll
                    for (int q = 0; q < t; ++q) s -= vals[end[t] - (t + 1) + q] * xb[q];
                    xb[t] = s / vals[end[t] - 1];
                }
            } else {
#pragma unroll
                for (int t = BS - 1; t >= 0; --t) {
                    double s = rhs[r0 + t] - acc[t];
#pragma unroll
                    for (int q = t + 1; q < BS; ++q) s -= vals[beg[t] + (q - t)] * xb[q];
                    xb[t] = s / vals[beg[t]];
                }
            }
#pragma unroll
            for (int t = 0; t < BS; ++t) st_relaxed(out + r0 + t, xb[t]);
        }
        __syncwarp();
        if (reset && active && gl < BS) reset[r0 + gl] = pending_value();
    }
}

}  // namespace pclab_b200
