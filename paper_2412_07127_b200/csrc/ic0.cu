// Level-scheduled, sync-free IC(0) numeric factorisation, bit-identical to
// the reference's up-looking ic0_attempt (src/precond.cpp:23-75) and
// driven by its shift policy (src/precond.cpp:109-143).
//
// Reference order per row i: for each off-diagonal entry (i, j) in column
// order, s = a_ij; s -= l_ic * l_jc for every shared column c < j in
// ascending c; l_ij = s / l_jj; diag_acc += l_ij^2; finally
// l_ii = sqrt(a_ii + shift - diag_acc).
//
// Device mapping: one warp per row, rows claimed in (level, index) order.
// Lane t owns entry t of the row and keeps its running s_t in a register.
// Step u finalises entry u (owner lane divides by l_{c_u c_u}) and
// broadcasts l_{i c_u}; every later lane t whose row c_t contains column
// c_u subtracts l_{i c_u} * l_{c_t c_u}. Entry t therefore receives its
// subtractions in ascending column order, exactly the reference's merge
// order, and every product/difference/quotient is explicitly rounded
// (no FMA), so the factor is bit-identical. Each entry of L starts as
// kPending and is published by its final store; dependants poll only the
// entries they read, so rows pipeline across levels without barriers.
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "core.h"

namespace pclab_b200 {

namespace {

template <int C>
__global__ void __launch_bounds__(256)
ic0_kernel(int64_t nitems, int per_item, int bs, const int32_t* __restrict__ slots,
           const int64_t* __restrict__ lrp, const int32_t* __restrict__ lcols,
           const double* __restrict__ avals, double shift, double* v, unsigned long long* fail_row,
           unsigned* counter) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(counter, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems * bs) return;
        // claim v = item * bs + t: row t of every block of the item. Rows t of
        // a block are claimed right after rows 0..t-1 (a topological order),
        // by different warps, so the in-block chain pipelines entry by entry.
        const int64_t item = it / bs;
        const int t_row = static_cast<int>(it % bs);
    for (int g = 0; g < per_item; ++g) {
        const int32_t blk = slots[item * per_item + g];
        if (blk < 0) continue;
        const int64_t i = static_cast<int64_t>(blk) * bs + t_row;
        const int64_t beg = lrp[i];
        const int nd = static_cast<int>(lrp[i + 1] - beg) - 1;  // off-diagonals
        double s[C], qval[C], dj[C];
        int32_t jc[C], qcol[C];
        int64_t q[C], qend[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int t = lane + 32 * c;
            jc[c] = -1;
            qcol[c] = INT_MAX;
            q[c] = qend[c] = 0;
            s[c] = qval[c] = dj[c] = 0.0;
            if (t < nd) {
                jc[c] = lcols[beg + t];
                s[c] = avals[beg + t];
                q[c] = lrp[jc[c]];
                qend[c] = lrp[jc[c] + 1] - 1;  // position of l_jj
                dj[c] = ld_relaxed(v + qend[c]);
                if (q[c] < qend[c]) {
                    qcol[c] = lcols[q[c]];
                    qval[c] = ld_relaxed(v + q[c]);
                }
            }
        }
        double diag_acc = 0.0;
        for (int u = 0; u < nd; ++u) {
            const int owner = u & 31, oc = u >> 5;
            double l = 0.0;
            int32_t cu = 0;
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (c == oc && lane == owner) {
                    double d = dj[c];
                    while (is_pending(d)) d = ld_relaxed(v + qend[c]);
                    l = __ddiv_rn(s[c], d);
                    st_relaxed(v + beg + u, l);
                    cu = jc[c];
                }
            l = __shfl_sync(0xffffffffu, l, owner);
            cu = __shfl_sync(0xffffffffu, cu, owner);
            diag_acc = __dadd_rn(diag_acc, __dmul_rn(l, l));
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int t = lane + 32 * c;
                if (t <= u || t >= nd) continue;
                while (qcol[c] < cu) {
                    ++q[c];
                    if (q[c] < qend[c]) {
                        qcol[c] = lcols[q[c]];
                        qval[c] = ld_relaxed(v + q[c]);
                    } else {
                        qcol[c] = INT_MAX;
                    }
                }
                if (qcol[c] == cu) {
                    double w = qval[c];
                    while (is_pending(w)) w = ld_relaxed(v + q[c]);
                    s[c] = __dsub_rn(s[c], __dmul_rn(l, w));
                    ++q[c];
                    if (q[c] < qend[c]) {
                        qcol[c] = lcols[q[c]];
                        qval[c] = ld_relaxed(v + q[c]);
                    } else {
                        qcol[c] = INT_MAX;
                    }
                }
            }
        }
        if (lane == 0) {
            const double sd = __dsub_rn(__dadd_rn(avals[beg + nd], shift), diag_acc);
            if (!(sd > 0.0)) {
                st_relaxed(v + beg + nd, __longlong_as_double(static_cast<long long>(kBroken)));
                atomicMin(fail_row, static_cast<unsigned long long>(i));
            } else {
                st_relaxed(v + beg + nd, __dsqrt_rn(sd));
            }
        }
        __syncwarp();
    }  // rows of the item
    }
}

// ---------------------------------------------------------------- masks
// Symbolic half of the mask factorisation (rows of <= 64 entries). For
// off-diagonal entry t of row i (column j): bit u of mu[k] is set when
// column c_u (u < t) of row i also occurs in row j, and bit p of mj[k]
// marks that occurrence's position p in row j -- the k-th set bit of mu
// pairs with the k-th set bit of mj. This is the reference's merge
// (precond.cpp:40-60) done once, without dependencies: warp per row, row
// i's columns in shared memory, lane t walks row j.
//
// Node-blocked L (Analysis::bsr, bs > 1): the bs rows of a block share their
// off-block columns, so row bs*b + t's masks for its first nd0 entries
// equal row bs*b's, and its in-block entry s (column bs*b + s) meets every
// earlier entry of both rows: mu = mj = (1 << p) - 1 at position p. One warp
// per block then merges only row bs*b.
__global__ void __launch_bounds__(256)
ic0_masks(int64_t nunits, int bs, const int64_t* __restrict__ lrp, const int32_t* __restrict__ lcols,
          unsigned long long* __restrict__ mu, unsigned long long* __restrict__ mj) {
    __shared__ int32_t rowc[8][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t unit = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (unit >= nunits) return;
    const int64_t i = unit * bs;  // bs = 1: every row is a unit
    const int64_t beg = lrp[i];
    const int nd = static_cast<int>(lrp[i + 1] - beg) - 1;
    for (int t = lane; t < nd; t += 32) rowc[w][t] = lcols[beg + t];
    __syncwarp();
    for (int t = lane; t < nd; t += 32) {
        const int32_t j = rowc[w][t];
        const int64_t rj = lrp[j];
        const int nj = static_cast<int>(lrp[j + 1] - rj) - 1;
        unsigned long long bu = 0, bj = 0;
        int u = 0, q = 0;
        int32_t cq = q < nj ? lcols[rj] : INT_MAX;
        while (u < t && q < nj) {
            const int32_t cu = rowc[w][u];
            if (cu < cq) {
                ++u;
            } else if (cq < cu) {
                ++q;
                cq = q < nj ? lcols[rj + q] : INT_MAX;
            } else {
                bu |= 1ULL << u;
                bj |= 1ULL << q;
                ++u;
                ++q;
                cq = q < nj ? lcols[rj + q] : INT_MAX;
            }
        }
        for (int r = 0; r < bs; ++r) {  // rows of the block share these entries
            const int64_t br = lrp[i + r];
            mu[br + t] = bu;
            mj[br + t] = bj;
        }
    }
    // in-block entries of rows t >= 1 (position p = nd + s, column i + s)
    for (int r = 1; r < bs; ++r) {
        const int64_t br = lrp[i + r];
        for (int sidx = lane; sidx < r; sidx += 32) {
            const int p = nd + sidx;
            const unsigned long long m = p >= 64 ? ~0ULL : (1ULL << p) - 1;
            mu[br + p] = m;
            mj[br + p] = m;
        }
    }
}

// The same masks from the block-column view (node-blocked L, bs = 3):
// row 3I+r's off-block entry p = 3k + c is column 3K + c, K = N_I[k]. Its
// row (3K + c) holds the off-block blocks N_K and in-block columns 3K..3K+c-1,
// so the matches are every component of each K' in N_I[0..k) that is also
// in N_K (row j position 3m' + c', m' = index of K' in N_K), plus columns
// 3K + c' < 3K + c (row j position 3|N_K| + c'). One lane per neighbour
// block merges two lists of <= 32 blocks instead of two rows of scalars.
__global__ void __launch_bounds__(256)
ic0_masks_bsr(int64_t nbk, const int64_t* __restrict__ lrp, const int64_t* __restrict__ bp,
              const int32_t* __restrict__ bcol, unsigned long long* __restrict__ mu,
              unsigned long long* __restrict__ mj) {
    constexpr int BS = 3;
    __shared__ int32_t nbr[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t I = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (I >= nbk) return;
    const int64_t b0 = bp[I];
    const int ni = static_cast<int>(bp[I + 1] - b0);  // <= 21 (checked by the caller: 3 ni + 2 < 64)
    if (lane < ni) nbr[w][lane] = bcol[b0 + lane] / BS;
    __syncwarp();
    int64_t beg[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) beg[r] = lrp[I * BS + r];
    if (lane < ni) {
        const int k = lane;
        const int32_t K = nbr[w][k];
        const int64_t c0 = bp[K];
        const int nk = static_cast<int>(bp[K + 1] - c0);
        unsigned long long bu = 0, bj = 0;
        int u = 0, q = 0;
        int32_t cq = q < nk ? bcol[c0] / BS : INT_MAX;
        while (u < k && q < nk) {
            const int32_t cu = nbr[w][u];
            if (cu < cq) {
                ++u;
            } else if (cq < cu) {
                ++q;
                cq = q < nk ? bcol[c0 + q] / BS : INT_MAX;
            } else {
                bu |= 7ULL << (BS * u);
                bj |= 7ULL << (BS * q);
                ++u;
                ++q;
                cq = q < nk ? bcol[c0 + q] / BS : INT_MAX;
            }
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            // components c' < c of block K itself
            const unsigned long long own_u = ((1ULL << c) - 1) << (BS * k);
            const unsigned long long own_j = ((1ULL << c) - 1) << (BS * nk);
#pragma unroll
            for (int r = 0; r < BS; ++r) {
                mu[beg[r] + BS * k + c] = bu | own_u;
                mj[beg[r] + BS * k + c] = bj | own_j;
            }
        }
    }
    // in-block entries of rows r >= 1 (position p = 3 ni + s, column 3I + s)
    for (int r = 1; r < BS; ++r)
        for (int sidx = lane; sidx < r; sidx += 32) {
            const int p = BS * ni + sidx;
            const unsigned long long m = (1ULL << p) - 1;
            mu[beg[r] + p] = m;
            mj[beg[r] + p] = m;
        }
}

// Numeric half: the ic0_kernel schedule (warp per row, rows in (level,
// index) order, lane t owns entry t, step u finalises entry u and
// broadcasts l_{i c_u}), but a lane learns from its masks whether step u
// touches it and where l_{j c_u} sits in row j -- no merge walk. The value
// of the next match is loaded one match ahead. Same per-entry operation
// order as the reference, explicitly rounded: bit-identical.
template <int C>
__global__ void __launch_bounds__(256)
ic0_mask_kernel(int64_t nitems, int per_item, int bs, const int32_t* __restrict__ slots,
                const int64_t* __restrict__ lrp, const int32_t* __restrict__ lcols,
                const double* __restrict__ avals, const unsigned long long* __restrict__ mu,
                const unsigned long long* __restrict__ mj, double shift, double* v,
                unsigned long long* fail_row, unsigned* counter) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(counter, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nitems * bs) return;
        const int64_t item = it / bs;
        const int t_row = static_cast<int>(it % bs);
        for (int g = 0; g < per_item; ++g) {
            const int32_t blk = slots[item * per_item + g];
            if (blk < 0) continue;
            const int64_t i = static_cast<int64_t>(blk) * bs + t_row;
            const int64_t beg = lrp[i];
            const int nd = static_cast<int>(lrp[i + 1] - beg) - 1;
            double s[C], dj[C], wn[C];
            unsigned long long bu[C], bj[C];
            int64_t rj[C], dpos[C];
            int32_t jc[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int t = lane + 32 * c;
                bu[c] = bj[c] = 0;
                s[c] = dj[c] = wn[c] = 0.0;
                rj[c] = dpos[c] = 0;
                jc[c] = 0;
                if (t < nd) {
                    jc[c] = lcols[beg + t];
                    s[c] = avals[beg + t];
                    bu[c] = mu[beg + t];
                    bj[c] = mj[beg + t];
                    rj[c] = lrp[jc[c]];
                    dpos[c] = lrp[jc[c] + 1] - 1;  // l_jj
                    dj[c] = ld_relaxed(v + dpos[c]);
                    if (bj[c]) wn[c] = ld_relaxed(v + rj[c] + (__ffsll(static_cast<long long>(bj[c])) - 1));
                }
            }
            double diag_acc = 0.0;
            for (int u = 0; u < nd; ++u) {
                const int owner = u & 31, oc = u >> 5;
                double l = 0.0;
                int32_t cu = 0;
#pragma unroll
                for (int c = 0; c < C; ++c)
                    if (c == oc && lane == owner) {
                        double d = dj[c];
                        while (is_pending(d)) d = ld_relaxed(v + dpos[c]);
                        l = __ddiv_rn(s[c], d);
                        st_relaxed(v + beg + u, l);
                        cu = jc[c];
                    }
                l = __shfl_sync(0xffffffffu, l, owner);
                (void)cu;
                diag_acc = __dadd_rn(diag_acc, __dmul_rn(l, l));
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    if ((bu[c] >> u) & 1ULL) {
                        const int pos = __ffsll(static_cast<long long>(bj[c])) - 1;
                        double w = wn[c];
                        while (is_pending(w)) w = ld_relaxed(v + rj[c] + pos);
                        s[c] = __dsub_rn(s[c], __dmul_rn(l, w));
                        bj[c] &= bj[c] - 1;
                        if (bj[c]) wn[c] = ld_relaxed(v + rj[c] + (__ffsll(static_cast<long long>(bj[c])) - 1));
                    }
                }
            }
            if (lane == 0) {
                const double sd = __dsub_rn(__dadd_rn(avals[beg + nd], shift), diag_acc);
                if (!(sd > 0.0)) {
                    st_relaxed(v + beg + nd, __longlong_as_double(static_cast<long long>(kBroken)));
                    atomicMin(fail_row, static_cast<unsigned long long>(i));
                } else {
                    st_relaxed(v + beg + nd, __dsqrt_rn(sd));
                }
            }
            __syncwarp();
        }
    }
}

// Node-blocked numeric IC(0) (Analysis::bsr): one warp per node block
// factors its BS rows together. The rows share their off-block columns,
// their masks and every l_{j c_u} they subtract, so lane p carries entry p
// of all BS rows and step u divides, publishes and broadcasts the BS
// values l_{r c_u} at once; the in-block entries (r, q), q < r, accumulate
// l_{r c_u} l_{q c_u} from those broadcasts and are finished after the
// off-block steps, followed by the diagonals. Per entry the reference's
// order (ascending shared column, explicitly rounded), so bit-identical;
// ~BS x fewer instructions per row than ic0_mask_kernel and no polling
// between the rows of a block.
template <int BS, int C>
__global__ void __launch_bounds__(256)
ic0_block_kernel(int64_t nslots, const int32_t* __restrict__ slots, const int64_t* __restrict__ lrp,
                 const int32_t* __restrict__ lcols, const double* __restrict__ avals,
                 const unsigned long long* __restrict__ mu, const unsigned long long* __restrict__ mj, double shift,
                 double* v, unsigned long long* fail_row, unsigned* counter) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned it = 0;
        if (lane == 0) it = atomicAdd(counter, 1u);
        it = __shfl_sync(0xffffffffu, it, 0);
        if (it >= nslots) return;
        const int32_t blk = slots[it];
        if (blk < 0) continue;
        const int64_t i0 = static_cast<int64_t>(blk) * BS;
        int64_t beg[BS];
#pragma unroll
        for (int r = 0; r < BS; ++r) beg[r] = lrp[i0 + r];
        const int nd0 = static_cast<int>(lrp[i0 + 1] - beg[0]) - 1;  // off-block entries
        double s[C][BS], dj[C], wn[C];
        unsigned long long bu[C], bj[C];
        int64_t rj[C], dpos[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            const int t = lane + 32 * c;
            bu[c] = bj[c] = 0;
            dj[c] = wn[c] = 0.0;
            rj[c] = dpos[c] = 0;
#pragma unroll
            for (int r = 0; r < BS; ++r) s[c][r] = 0.0;
            if (t < nd0) {
                const int32_t j = lcols[beg[0] + t];
#pragma unroll
                for (int r = 0; r < BS; ++r) s[c][r] = avals[beg[r] + t];
                bu[c] = mu[beg[0] + t];
                bj[c] = mj[beg[0] + t];
                rj[c] = lrp[j];
                dpos[c] = lrp[j + 1] - 1;
                dj[c] = ld_relaxed(v + dpos[c]);
                if (bj[c]) wn[c] = ld_relaxed(v + rj[c] + (__ffsll(static_cast<long long>(bj[c])) - 1));
            }
        }
        // in-block entries (r, q), q < r: running sums (every lane keeps a copy)
        double sin[BS][BS];
#pragma unroll
        for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int q = 0; q < BS; ++q) sin[r][q] = q < r ? avals[beg[r] + nd0 + q] : 0.0;
        double dacc[BS];
#pragma unroll
        for (int r = 0; r < BS; ++r) dacc[r] = 0.0;
        for (int u = 0; u < nd0; ++u) {
            const int owner = u & 31, oc = u >> 5;
            double l[BS];
#pragma unroll
            for (int r = 0; r < BS; ++r) l[r] = 0.0;
#pragma unroll
            for (int c = 0; c < C; ++c)
                if (c == oc && lane == owner) {
                    double d = dj[c];
                    while (is_pending(d)) d = ld_relaxed(v + dpos[c]);
#pragma unroll
                    for (int r = 0; r < BS; ++r) {
                        l[r] = __ddiv_rn(s[c][r], d);
                        st_relaxed(v + beg[r] + u, l[r]);
                    }
                }
#pragma unroll
            for (int r = 0; r < BS; ++r) {
                l[r] = __shfl_sync(0xffffffffu, l[r], owner);
                dacc[r] = __dadd_rn(dacc[r], __dmul_rn(l[r], l[r]));
            }
#pragma unroll
            for (int r = 1; r < BS; ++r)
#pragma unroll
                for (int q = 0; q < r; ++q) sin[r][q] = __dsub_rn(sin[r][q], __dmul_rn(l[r], l[q]));
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if ((bu[c] >> u) & 1ULL) {
                    const int pos = __ffsll(static_cast<long long>(bj[c])) - 1;
                    double w = wn[c];
                    while (is_pending(w)) w = ld_relaxed(v + rj[c] + pos);
#pragma unroll
                    for (int r = 0; r < BS; ++r) s[c][r] = __dsub_rn(s[c][r], __dmul_rn(l[r], w));
                    bj[c] &= bj[c] - 1;
                    if (bj[c]) wn[c] = ld_relaxed(v + rj[c] + (__ffsll(static_cast<long long>(bj[c])) - 1));
                }
            }
        }
        if (lane == 0) {
            // rows in order: in-block entries (column order), then the diagonal
            double dg[BS], lin[BS][BS];
#pragma unroll
            for (int r = 0; r < BS; ++r) {
#pragma unroll
                for (int q = 0; q < r; ++q) {
                    double sq = sin[r][q];
#pragma unroll
                    for (int q2 = 0; q2 < q; ++q2) sq = __dsub_rn(sq, __dmul_rn(lin[r][q2], lin[q][q2]));
                    lin[r][q] = __ddiv_rn(sq, dg[q]);
                    st_relaxed(v + beg[r] + nd0 + q, lin[r][q]);
                    dacc[r] = __dadd_rn(dacc[r], __dmul_rn(lin[r][q], lin[r][q]));
                }
                const double sd = __dsub_rn(__dadd_rn(avals[beg[r] + nd0 + r], shift), dacc[r]);
                if (!(sd > 0.0)) {
                    dg[r] = __longlong_as_double(static_cast<long long>(kBroken));
                    atomicMin(fail_row, static_cast<unsigned long long>(i0 + r));
                } else {
                    dg[r] = __dsqrt_rn(sd);
                }
                st_relaxed(v + beg[r] + nd0 + r, dg[r]);
            }
        }
        __syncwarp();
    }
}

__global__ void row_stats(int64_t n, const int64_t* __restrict__ rp, const double* __restrict__ lv,
                          unsigned* maxlen, unsigned long long* maxdiag) {
    unsigned ml = 0;
    unsigned long long md = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        ml = max(ml, static_cast<unsigned>(rp[i + 1] - rp[i]));
        // |a_ii| >= 0: its IEEE bit pattern orders like an unsigned integer
        md = max(md, static_cast<unsigned long long>(__double_as_longlong(fabs(lv[rp[i + 1] - 1]))));
    }
    ml = __reduce_max_sync(0xffffffffu, ml);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) md = max(md, __shfl_xor_sync(0xffffffffu, md, o));
    if ((threadIdx.x & 31) == 0) {
        atomicMax(maxlen, ml);
        atomicMax(maxdiag, md);
    }
}

}  // namespace

int ic0_factor(const Matrix& a, const Analysis& an, double* out, cudaStream_t st) {
    const int64_t n = a.a.n;
    const DevCsr& L = an.lower;
    if (n == 0) return 0;
    // max|a_ii| over the diagonal (precond.cpp:114-118) sets the shift scale
    DevBuf<unsigned> mx(1);
    DevBuf<unsigned long long> md(1);
    CK(cudaMemsetAsync(mx.p, 0, sizeof(unsigned), st));
    CK(cudaMemsetAsync(md.p, 0, sizeof(unsigned long long), st));
    row_stats<<<static_cast<unsigned>(sm_count() * 4), 256, 0, st>>>(n, L.rp.p, L.vals.p, mx.p, md.p);
    CK_LAUNCH();
    unsigned maxlen = 0;
    unsigned long long mdbits = 0;
    CK(cudaMemcpyAsync(&maxlen, mx.p, sizeof maxlen, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&mdbits, md.p, sizeof mdbits, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    double max_diag;
    std::memcpy(&max_diag, &mdbits, sizeof max_diag);
    if (maxlen > 256)
        throw DimensionError("ic0: a row of L has " + std::to_string(maxlen) +
                             " entries; the device kernel supports up to 256");
    const double alpha0 = 1e-8 * max_diag;
    DevBuf<unsigned long long> fail(1);
    DevBuf<unsigned> ctr(1);
    // a few levels of rows resident: enough to pipeline, few idle pollers
    // the forward-sweep block schedule: a warp per item, rows in order
    const Schedule& s = an.blk_lo;
    const double per_level = s.nlevels ? static_cast<double>(s.nitems) / s.nlevels : 1.0;
    static const double depth = getenv("PCLAB_IC0_DEPTH") ? atof(getenv("PCLAB_IC0_DEPTH")) : 6.0;
    const int64_t blocks = (static_cast<int64_t>(depth * per_level) + 8) / 8;
    const unsigned grid = static_cast<unsigned>(
        std::min<int64_t>(std::max<int64_t>(blocks, sm_count()), sm_count() * 8));
    // rows of <= 64 entries: symbolic masks once, then the mask kernel
    // (PCLAB_IC0_MASKS=0 keeps the merge-walk kernel)
    static const bool masks_env = !(getenv("PCLAB_IC0_MASKS") && atoi(getenv("PCLAB_IC0_MASKS")) == 0);
    const bool use_masks = masks_env && maxlen <= 64;
    // masks live in a grow-only process scratch (3.2 GB on configs[2]):
    // re-allocating them per analysis fragments the stream-ordered pool
    // (measured: IC(0) 0.06 -> 0.33 s when allocated per call); recomputed
    // only when the pattern (analysis) changes
    static DevBuf<unsigned long long>& mu = *new DevBuf<unsigned long long>();  // never freed
    static DevBuf<unsigned long long>& mj = *new DevBuf<unsigned long long>();
    static uint64_t mask_id = 0;
    if (use_masks && (mask_id != an.id || mu.n < L.nnz)) {
        if (mu.n < L.nnz) {
            mu.alloc(L.nnz);
            mj.alloc(L.nnz);
        }
        mask_id = an.id;
        static const bool bsr_masks = !(getenv("PCLAB_IC0_BSR_MASKS") && atoi(getenv("PCLAB_IC0_BSR_MASKS")) == 0);
        if (bsr_masks && an.bsr && an.bs == 3 && maxlen <= 64) {
            // (maxlen <= 64 bounds 3 |N| + 2 for every block row, so all
            // bit positions fit)
            const int64_t nbk = n / 3;
            ic0_masks_bsr<<<static_cast<unsigned>((nbk * 32 + 255) / 256), 256, 0, st>>>(nbk, L.rp.p, an.lbc.bp.p,
                                                                                          an.lbc.bcol.p, mu.p, mj.p);
        } else {
            const int mbs = an.bsr ? an.bs : 1;
            const int64_t units = n / mbs;
            ic0_masks<<<static_cast<unsigned>((units * 32 + 255) / 256), 256, 0, st>>>(units, mbs, L.rp.p, L.cols.p,
                                                                                       mu.p, mj.p);
        }
        CK_LAUNCH();
    }
    for (int attempt = 0;; ++attempt) {
        const double shift = attempt == 0 ? 0.0 : alpha0 * static_cast<double>(1 << (attempt - 1));
        fill_pending(out, L.nnz, st);
        CK(cudaMemsetAsync(fail.p, 0xff, sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(ctr.p, 0, sizeof(unsigned), st));
        if (use_masks && an.bsr && an.bs == 3 && s.per_item > 0)
            ic0_block_kernel<3, 2><<<grid, 256, 0, st>>>(s.nitems * s.per_item, s.slots.p, L.rp.p, L.cols.p,
                                                          L.vals.p, mu.p, mj.p, shift, out, fail.p, ctr.p);
        else if (use_masks && an.bsr && an.bs == 2 && s.per_item > 0)
            ic0_block_kernel<2, 2><<<grid, 256, 0, st>>>(s.nitems * s.per_item, s.slots.p, L.rp.p, L.cols.p,
                                                          L.vals.p, mu.p, mj.p, shift, out, fail.p, ctr.p);
        else if (use_masks)
            ic0_mask_kernel<2><<<grid, 256, 0, st>>>(s.nitems, s.per_item, s.bs, s.slots.p, L.rp.p, L.cols.p,
                                                      L.vals.p, mu.p, mj.p, shift, out, fail.p, ctr.p);
        else if (maxlen <= 64)
            ic0_kernel<2><<<grid, 256, 0, st>>>(s.nitems, s.per_item, s.bs, s.slots.p, L.rp.p, L.cols.p,
                                                 L.vals.p, shift, out, fail.p, ctr.p);
        else if (maxlen <= 128)
            ic0_kernel<4><<<grid, 256, 0, st>>>(s.nitems, s.per_item, s.bs, s.slots.p, L.rp.p, L.cols.p,
                                                 L.vals.p, shift, out, fail.p, ctr.p);
        else
            ic0_kernel<8><<<grid, 256, 0, st>>>(s.nitems, s.per_item, s.bs, s.slots.p, L.rp.p, L.cols.p,
                                                 L.vals.p, shift, out, fail.p, ctr.p);
        CK_LAUNCH();
        unsigned long long f = 0;
        CK(cudaMemcpyAsync(&f, fail.p, sizeof f, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (f == ~0ULL) return attempt;
        if (attempt == 3)
            throw NumericError("ic0: nonpositive pivot at row " + std::to_string(f));
    }
}

}  // namespace pclab_b200
