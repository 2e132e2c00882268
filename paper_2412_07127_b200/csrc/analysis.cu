// Device symbolic analysis: L/U patterns, the U->L slot map, dof-block
// detection, level sets of both triangular sweeps and their warp schedules.
//
// The reference performs lower_triangle (src/sparse.cpp:189-204) and
// csr_transpose (src/sparse.cpp:137-157) on the host on every solve and has
// no level analysis at all (its substitution is sequential,
// src/krylov.cpp:60-112). Here the patterns are built once in HBM and the
// dependency DAG of each sweep is levelled so that warps can run it
// sync-free in topological order.
#include <cstdlib>

#include <cooperative_groups.h>

#include "core.h"

namespace pclab_b200 {

namespace cg = cooperative_groups;

namespace {

__global__ void lu_counts(int64_t n, const int64_t* __restrict__ rp,
                          const int64_t* __restrict__ dpos, int64_t* __restrict__ lcnt,
                          int64_t* __restrict__ ucnt) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    lcnt[i] = dpos[i] - rp[i] + 1;
    ucnt[i] = rp[i + 1] - dpos[i];
}

__global__ void lu_fill(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ cols,
                        const double* __restrict__ vals, const int64_t* __restrict__ dpos,
                        const int64_t* __restrict__ lrp, int32_t* __restrict__ lcols,
                        double* __restrict__ lvals, const int64_t* __restrict__ urp,
                        int32_t* __restrict__ ucols) {
    // warp per row, lanes over the entries (coalesced copies)
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t b = rp[i], d = dpos[i], e = rp[i + 1], lo = lrp[i], uo = urp[i];
    for (int64_t k = b + lane; k <= d; k += 32) {
        lcols[lo + (k - b)] = cols[k];
        lvals[lo + (k - b)] = vals[k];
    }
    for (int64_t k = d + lane; k < e; k += 32) ucols[uo + (k - d)] = cols[k];
}

// u2l[t]: U entry (i, j), j >= i, is L entry (j, i) in row j.
__global__ void u2l_fill(int64_t n, const int64_t* __restrict__ urp,
                         const int32_t* __restrict__ ucols, const int64_t* __restrict__ lrp,
                         const int32_t* __restrict__ lcols, int64_t* __restrict__ u2l) {
    const int64_t i = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    for (int64_t t = urp[i] + lane; t < urp[i + 1]; t += 32) {
        const int32_t j = ucols[t];
        int64_t lo = lrp[j], hi = lrp[j + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (lcols[mid] < i) lo = mid + 1; else hi = mid;
        }
        u2l[t] = lo;
    }
}

// Row i of block b = i / bs is "dense-diagonal" if its last (i % bs) + 1
// entries are exactly columns b*bs .. i.
__global__ void block_check(int64_t n, int bs, const int64_t* __restrict__ lrp,
                            const int32_t* __restrict__ lcols, int* __restrict__ bad) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int t = static_cast<int>(i % bs);
    const int64_t e = lrp[i + 1];
    if (e - lrp[i] < t + 1) { *bad = 1; return; }
    for (int s = 0; s <= t; ++s)
        if (lcols[e - 1 - s] != i - s) { *bad = 1; return; }
}

// Node-blocked off-block pattern: the BS rows of every block reference the
// same set of whole BS-wide column blocks (row t of block b holds, past its
// in-block entries, columns BS*k .. BS*k+BS-1 for each neighbour k, in
// order). Checked on L; U = L^T inherits it.
__global__ void bsr_check(int64_t nb, int bs, const int64_t* __restrict__ lrp,
                          const int32_t* __restrict__ lcols, int* __restrict__ bad) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t r0 = b * bs;
    const int64_t cnt = lrp[r0 + 1] - 1 - lrp[r0];  // off-block entries of row 0
    if (cnt % bs) { *bad = 1; return; }
    for (int t = 0; t < bs; ++t) {
        const int64_t beg = lrp[r0 + t];
        if (lrp[r0 + t + 1] - (t + 1) - beg != cnt) { *bad = 1; return; }
        for (int64_t k = 0; k < cnt; k += bs) {
            const int32_t c0 = lcols[lrp[r0] + k];
            if (c0 % bs) { *bad = 1; return; }
            for (int c = 0; c < bs; ++c)
                if (lcols[beg + k + c] != c0 + c) { *bad = 1; return; }
        }
    }
}

// Same property on the full matrix A (every row of block b holds whole
// BS-wide column blocks, the same set for its BS rows).
__global__ void bsr_check_full(int64_t nb, int bs, const int64_t* __restrict__ arp,
                               const int32_t* __restrict__ acols, int* __restrict__ bad) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t r0 = b * bs;
    const int64_t cnt = arp[r0 + 1] - arp[r0];
    if (cnt % bs) { *bad = 1; return; }
    for (int t = 0; t < bs; ++t) {
        const int64_t beg = arp[r0 + t];
        if (arp[r0 + t + 1] - beg != cnt) { *bad = 1; return; }
        for (int64_t k = 0; k < cnt; k += bs) {
            const int32_t c0 = acols[arp[r0] + k];
            if (c0 % bs) { *bad = 1; return; }
            for (int c = 0; c < bs; ++c)
                if (acols[beg + k + c] != c0 + c) { *bad = 1; return; }
        }
    }
}

// Level sets by Kahn layering on the block DAG: a block's level is one
// more than the largest level among its predecessors, so releasing a block
// when its last predecessor is processed assigns exactly that level (the
// frontier order is irrelevant; the schedule is sorted afterwards). One
// launch per level, replayed from a CUDA graph.
struct KState {
    unsigned long long beg, end, tail;
    int lvl, pad;
};

__device__ __forceinline__ bool is_pred(int64_t jb, int64_t b, bool upper) {
    return upper ? jb > b : jb < b;
}

__global__ void kahn_init(int64_t nb, int bs, const int64_t* __restrict__ prp,
                          const int32_t* __restrict__ pcols, bool upper, int32_t* __restrict__ indeg,
                          int32_t* __restrict__ level, int32_t* __restrict__ fr, KState* ks) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    int cnt = 0;
    for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
        for (int64_t k = prp[i]; k < prp[i + 1]; ++k) cnt += is_pred(pcols[k] / bs, b, upper);
    indeg[b] = cnt;
    level[b] = -1;
    if (cnt == 0) {
        level[b] = 0;
        fr[atomicAdd(&ks->tail, 1ULL)] = static_cast<int32_t>(b);
    }
}

// Node-blocked variant: predecessors / successors are the block columns
// (one entry per neighbour block instead of bs x bs scalar entries).
__global__ void kahn_init_bc(int64_t nb, const int64_t* __restrict__ pbp, int32_t* __restrict__ indeg,
                             int32_t* __restrict__ level, int32_t* __restrict__ fr, KState* ks) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int cnt = static_cast<int>(pbp[b + 1] - pbp[b]);
    indeg[b] = cnt;
    level[b] = -1;
    if (cnt == 0) {
        level[b] = 0;
        fr[atomicAdd(&ks->tail, 1ULL)] = static_cast<int32_t>(b);
    }
}

// warp per frontier block, lanes over the successor entries
__global__ void kahn_step(int bs, const int64_t* __restrict__ srp, const int32_t* __restrict__ scols,
                          bool upper, int32_t* __restrict__ indeg, int32_t* __restrict__ level,
                          int32_t* __restrict__ fr, KState* ks) {
    const unsigned long long beg = ks->beg, end = ks->end;
    const int nl = ks->lvl + 1;
    const int lane = threadIdx.x & 31;
    const unsigned long long w0 = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) >> 5;
    const unsigned long long nw = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    for (unsigned long long p = beg + w0; p < end; p += nw) {
        const int64_t b = fr[p];
        for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
            for (int64_t k = srp[i] + lane; k < srp[i + 1]; k += 32) {
                const int64_t jb = scols[k] / bs;
                if (!is_pred(b, jb, upper)) continue;  // b precedes jb
                if (atomicSub(&indeg[jb], 1) == 1) {
                    level[jb] = nl;
                    fr[atomicAdd(&ks->tail, 1ULL)] = static_cast<int32_t>(jb);
                }
            }
    }
}

// All levels in one cooperative launch: process the frontier, grid barrier,
// thread 0 advances the frontier window, grid barrier. BC: successors from
// a block-column view (sbp/sbcol), one atomic per neighbour block -- a
// frontier block's successors fit one warp round, so a level costs one
// atomic round trip instead of one per 32 scalar entries.
template <bool BC>
__global__ void kahn_persistent(int bs, const int64_t* __restrict__ srp,
                                const int32_t* __restrict__ scols, bool upper,
                                int32_t* __restrict__ indeg, int32_t* __restrict__ level,
                                int32_t* __restrict__ fr, KState* ks) {
    cg::grid_group g = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const unsigned long long w0 = (blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x) >> 5;
    const unsigned long long nw = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
    volatile KState* vk = ks;
    for (;;) {
        const unsigned long long beg = vk->beg, end = vk->end;
        if (beg == end) return;
        const int nl = vk->lvl + 1;
        for (unsigned long long p = beg + w0; p < end; p += nw) {
            const int64_t b = __ldcg(fr + p);  // appended by other CTAs: bypass L1
            if (BC) {
                for (int64_t k = srp[b] + lane; k < srp[b + 1]; k += 32) {
                    const int64_t jb = scols[k] / bs;
                    if (atomicSub(&indeg[jb], 1) == 1) {
                        level[jb] = nl;
                        fr[atomicAdd(&ks->tail, 1ULL)] = static_cast<int32_t>(jb);
                    }
                }
            } else {
                for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
                    for (int64_t k = srp[i] + lane; k < srp[i + 1]; k += 32) {
                        const int64_t jb = scols[k] / bs;
                        if (!is_pred(b, jb, upper)) continue;
                        if (atomicSub(&indeg[jb], 1) == 1) {
                            level[jb] = nl;
                            fr[atomicAdd(&ks->tail, 1ULL)] = static_cast<int32_t>(jb);
                        }
                    }
            }
        }
        g.sync();
        if (g.thread_rank() == 0) {
            const unsigned long long t = vk->tail;
            vk->beg = end;
            if (t != end) {
                vk->end = t;
                vk->lvl = nl;
            }
        }
        g.sync();
    }
}

// Sync-free levelling over block columns (no grid barrier per level): a
// work queue of released blocks. A warp pops the next queue slot (waits
// until it is written), sets level(b) = 1 + max level of its predecessors
// (all final: a predecessor writes its level, fences, and only then
// decrements b's counter), fences, and releases the successors whose
// counters reach zero by appending them. Levels equal Kahn's (longest path
// from a root). Deadlock-free with every warp resident: slots are written
// in claim order by running warps, and a popped slot below the number of
// blocks is always eventually written.
__global__ void __launch_bounds__(256)
level_queue_kernel(int64_t nb, int bs, const int64_t* __restrict__ pbp, const int32_t* __restrict__ pbcol,
                   const int64_t* __restrict__ sbp, const int32_t* __restrict__ sbcol, int32_t* __restrict__ indeg,
                   int32_t* level, int32_t* queue, unsigned long long* cnt /* [0] head, [1] tail */) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long h = 0;
        if (lane == 0) h = atomicAdd(cnt, 1ULL);
        h = __shfl_sync(0xffffffffu, h, 0);
        if (h >= static_cast<unsigned long long>(nb)) return;
        int32_t b = -1;
        if (lane == 0) {
            volatile int32_t* vq = queue + h;
            while ((b = *vq) < 0) __nanosleep(32);
        }
        b = __shfl_sync(0xffffffffu, b, 0);
        int lv = 0;
        for (int64_t k = pbp[b] + lane; k < pbp[b + 1]; k += 32)
            lv = max(lv, 1 + *reinterpret_cast<volatile int32_t*>(level + pbcol[k] / bs));
        lv = __reduce_max_sync(0xffffffffu, lv);
        if (lane == 0) level[b] = lv;
        __threadfence();
        __syncwarp();
        for (int64_t k = sbp[b] + lane; k < sbp[b + 1]; k += 32) {
            const int64_t jb = sbcol[k] / bs;
            if (atomicSub(&indeg[jb], 1) == 1) {
                const unsigned long long t = atomicAdd(cnt + 1, 1ULL);
                *reinterpret_cast<volatile int32_t*>(queue + t) = static_cast<int32_t>(jb);
            }
        }
    }
}

__global__ void level_queue_init(int64_t nb, const int64_t* __restrict__ pbp, int32_t* __restrict__ indeg,
                                 int32_t* __restrict__ queue, unsigned long long* cnt) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int c = static_cast<int>(pbp[b + 1] - pbp[b]);
    indeg[b] = c;
    if (c == 0) queue[atomicAdd(cnt + 1, 1ULL)] = static_cast<int32_t>(b);
}

__global__ void kahn_start(KState* ks) {
    ks->beg = 0;
    ks->end = ks->tail;
    ks->lvl = 0;
}

__global__ void kahn_advance(KState* ks) {
    if (ks->end == ks->tail) {
        ks->beg = ks->end;  // frontier exhausted: stays empty
        return;
    }
    ks->beg = ks->end;
    ks->end = ks->tail;
    ks->lvl += 1;
}

// The dependency a sweep polls first: the predecessor block of highest
// (level, index); its last-published row is bs - 1.
__global__ void crit_kernel(int64_t nb, int bs, const int64_t* __restrict__ prp,
                            const int32_t* __restrict__ pcols, bool upper,
                            const int32_t* __restrict__ level, int32_t* __restrict__ crit) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    int64_t best = -1;
    int bl = -1;
    for (int64_t i = b * bs; i < (b + 1) * bs; ++i)
        for (int64_t k = prp[i]; k < prp[i + 1]; ++k) {
            const int64_t jb = pcols[k] / bs;
            if (!is_pred(jb, b, upper)) continue;
            const int l = level[jb];
            if (l > bl || (l == bl && jb > best)) {
                bl = l;
                best = jb;
            }
        }
    crit[b] = best < 0 ? -1 : static_cast<int32_t>(best * bs + bs - 1);
}

__global__ void iota32(int32_t* p, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) p[i] = static_cast<int32_t>(i);
}

__global__ void level_starts(int64_t nb, const int32_t* __restrict__ sorted_level,
                             int64_t* __restrict__ start) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p >= nb) return;
    if (p == 0 || sorted_level[p] != sorted_level[p - 1]) start[sorted_level[p]] = p;
}

__global__ void items_per_level(int32_t nl, int64_t nb, int per_item,
                                const int64_t* __restrict__ start, int64_t* __restrict__ nit) {
    const int64_t l = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (l >= nl) return;
    const int64_t end = l + 1 < nl ? start[l + 1] : nb;
    nit[l] = (end - start[l] + per_item - 1) / per_item;
}

__global__ void slots_fill(int64_t nitems, int per_item, const int32_t* __restrict__ order,
                           const int64_t* __restrict__ first, const int32_t* __restrict__ cnt,
                           int32_t* __restrict__ slots) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nitems * per_item) return;
    const int64_t it = k / per_item;
    const int g = static_cast<int>(k % per_item);
    slots[k] = g < cnt[it] ? order[first[it] + g] : -1;
}

// Slot records (BsrSlot, 16 bytes): k = {block, rp[first row], bp[block],
// row lengths packed 10 bits per row}, so an item's first dependent load is
// its entries. Flags rows longer than 1023 entries or offsets beyond 32 bits.
__global__ void slot_rp_fill(int64_t nslots, int bs, const int32_t* __restrict__ slots,
                             const int64_t* __restrict__ rp, const int64_t* __restrict__ bp,
                             int32_t* __restrict__ srec, int* __restrict__ bad) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= nslots) return;
    const int32_t b = slots[k];
    int64_t r0 = 0, c0 = 0;
    uint32_t lens = 0;
    if (b >= 0) {
        const int64_t i = static_cast<int64_t>(b) * bs;
        r0 = rp[i];
        c0 = bp ? bp[b] : 0;
        if (bs > 3 || r0 > 0xffffffffLL || c0 > 0xffffffffLL) *bad = 1;
        for (int t = 0; t < bs && t < 3; ++t) {
            const int64_t len = rp[i + t + 1] - rp[i + t];
            if (len > 1023) *bad = 1;
            lens |= static_cast<uint32_t>(len & 1023) << (10 * t);
        }
    }
    srec[4 * k] = b;
    srec[4 * k + 1] = static_cast<int32_t>(static_cast<uint32_t>(r0));
    srec[4 * k + 2] = static_cast<int32_t>(static_cast<uint32_t>(c0));
    srec[4 * k + 3] = static_cast<int32_t>(lens);
}

// Block-column view (BlockCols). mode 0: L (off-block entries first),
// 1: U (bs in-block entries first in the block's first row), 2: A (all).
__global__ void bc_count(int64_t nb, int bs, int mode, const int64_t* __restrict__ rp, int64_t* __restrict__ cnt) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t len = rp[b * bs + 1] - rp[b * bs];
    cnt[b] = (len - (mode == 0 ? 1 : mode == 1 ? bs : 0)) / bs;
}

__global__ void bc_fill(int64_t nb, int bs, int mode, const int64_t* __restrict__ rp,
                        const int32_t* __restrict__ cols, const int64_t* __restrict__ bp,
                        int32_t* __restrict__ bcol) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t first = rp[b * bs] + (mode == 1 ? bs : 0);
    for (int64_t k = bp[b]; k < bp[b + 1]; ++k) bcol[k] = cols[first + (k - bp[b]) * bs];
}

__global__ void items_fill(int32_t nl, int64_t nb, int per_item, const int64_t* __restrict__ start,
                           const int64_t* __restrict__ item_start, int64_t* __restrict__ first,
                           int32_t* __restrict__ cnt) {
    const int64_t l = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (l >= nl) return;
    const int64_t s = start[l], e = l + 1 < nl ? start[l + 1] : nb;
    int64_t it = item_start[l];
    for (int64_t p = s; p < e; p += per_item, ++it) {
        first[it] = p;
        cnt[it] = static_cast<int32_t>(min(static_cast<int64_t>(per_item), e - p));
    }
}

inline unsigned grid_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace



void compute_levels(const DevCsr& pred, const DevCsr& succ, int bs, bool upper, Schedule& s,
                    cudaStream_t st, const BlockCols* pbc, const BlockCols* sbc) {
    const int64_t n = pred.n;
    s.bs = bs;
    s.nblocks = n / bs;
    s.level.alloc(std::max<int64_t>(s.nblocks, 1));
    s.crit.alloc(std::max<int64_t>(s.nblocks, 1));
    if (s.nblocks == 0) return;
    const int64_t nb = s.nblocks;
    const bool bc = pbc && sbc && pbc->bp.p && sbc->bp.p;
    static const bool queue_on = !(getenv("PCLAB_LEVEL_QUEUE") && atoi(getenv("PCLAB_LEVEL_QUEUE")) == 0);
    if (bc && queue_on) {
        DevBuf<int32_t> indeg(nb), queue(nb);
        DevBuf<unsigned long long> cnt(2);
        CK(cudaMemsetAsync(cnt.p, 0, 2 * sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(queue.p, 0xff, sizeof(int32_t) * nb, st));
        level_queue_init<<<grid_for(nb, 256), 256, 0, st>>>(nb, pbc->bp.p, indeg.p, queue.p, cnt.p);
        CK_LAUNCH();
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, level_queue_kernel, 256, 0));
        const unsigned grid = static_cast<unsigned>(sm_count() * std::max(1, std::min(per_sm, 4)));
        level_queue_kernel<<<grid, 256, 0, st>>>(nb, bs, pbc->bp.p, pbc->bcol.p, sbc->bp.p, sbc->bcol.p, indeg.p,
                                                 s.level.p, queue.p, cnt.p);
        CK_LAUNCH();
        unsigned long long hc[2];
        CK(cudaMemcpyAsync(hc, cnt.p, sizeof hc, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (hc[1] != static_cast<unsigned long long>(nb))
            throw FormatError("level analysis: dependency graph has a cycle");
        if (s.need_crit) {
            crit_kernel<<<grid_for(nb, 256), 256, 0, st>>>(nb, bs, pred.rp.p, pred.cols.p, upper, s.level.p,
                                                           s.crit.p);
            CK_LAUNCH();
        }
        return;
    }
    DevBuf<int32_t> indeg(nb), fr(nb);
    DevBuf<KState> ks(1);
    CK(cudaMemsetAsync(ks.p, 0, sizeof(KState), st));
    if (bc)
        kahn_init_bc<<<grid_for(nb, 256), 256, 0, st>>>(nb, pbc->bp.p, indeg.p, s.level.p, fr.p, ks.p);
    else
        kahn_init<<<grid_for(nb, 256), 256, 0, st>>>(nb, bs, pred.rp.p, pred.cols.p, upper, indeg.p, s.level.p,
                                                     fr.p, ks.p);
    CK_LAUNCH();
    kahn_start<<<1, 1, 0, st>>>(ks.p);  // frontier of level 0 = the seeds
    CK_LAUNCH();
    // one cooperative persistent launch: a grid barrier per level instead
    // of a kernel launch per level
    auto kern = bc ? kahn_persistent<true> : kahn_persistent<false>;
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0));
    const unsigned grid = static_cast<unsigned>(sm_count() * std::max(1, std::min(per_sm, 4)));
    {
        int bs_ = bs;
        const int64_t* srp = bc ? sbc->bp.p : succ.rp.p;
        const int32_t* scols = bc ? sbc->bcol.p : succ.cols.p;
        bool up = upper;
        int32_t* ind = indeg.p;
        int32_t* lev = s.level.p;
        int32_t* frp = fr.p;
        KState* ksp = ks.p;
        void* args[] = {&bs_, &srp, &scols, &up, &ind, &lev, &frp, &ksp};
        CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(kern), grid, 256, args, 0, st));
        CK_LAUNCH();
    }
    KState h{};
    CK(cudaMemcpyAsync(&h, ks.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.tail != static_cast<unsigned long long>(nb))
        throw FormatError("level analysis: dependency graph has a cycle");
    if (s.need_crit) {
        crit_kernel<<<grid_for(nb, 256), 256, 0, st>>>(nb, bs, pred.rp.p, pred.cols.p, upper, s.level.p,
                                                       s.crit.p);
        CK_LAUNCH();
    }
}

static void build_schedule(const DevCsr& pred, const DevCsr& succ, int bs, bool upper, int lanes,
                           Schedule& s, cudaStream_t st, const BlockCols* pbc = nullptr,
                           const BlockCols* sbc = nullptr) {
    compute_levels(pred, succ, bs, upper, s, st, pbc, sbc);
    s.lanes = lanes;
    s.per_item = 32 / lanes;
    const int64_t nb = s.nblocks;
    if (nb == 0) return;
    DevBuf<int32_t> idx(nb), sorted_lv(nb);
    s.order.alloc(nb);
    iota32<<<grid_for(nb, 256), 256, 0, st>>>(idx.p, nb);
    CK_LAUNCH();
    // levels are non-negative: sort them as unsigned keys
    radix_sort_pairs(reinterpret_cast<const uint32_t*>(s.level.p), reinterpret_cast<uint32_t*>(sorted_lv.p), idx.p,
                     s.order.p, nb, 32, st);
    s.nlevels = dev_read(sorted_lv.p + nb - 1, st) + 1;
    DevBuf<int64_t> start(s.nlevels), nit(s.nlevels + 1);
    level_starts<<<grid_for(nb, 256), 256, 0, st>>>(nb, sorted_lv.p, start.p);
    items_per_level<<<grid_for(s.nlevels, 256), 256, 0, st>>>(s.nlevels, nb, s.per_item, start.p,
                                                             nit.p);
    CK(cudaMemsetAsync(nit.p + s.nlevels, 0, sizeof(int64_t), st));
    CK_LAUNCH();
    // widest level (for reporting)
    {
        std::vector<int64_t> hs(s.nlevels);
        CK(cudaMemcpyAsync(hs.data(), start.p, sizeof(int64_t) * s.nlevels, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        s.max_level_width = 0;
        for (int32_t l = 0; l < s.nlevels; ++l) {
            const int64_t e = l + 1 < s.nlevels ? hs[l + 1] : nb;
            s.max_level_width = std::max(s.max_level_width, e - hs[l]);
        }
    }
    scan_inplace(nit.p, s.nlevels + 1, st);
    s.nitems = dev_read(nit.p + s.nlevels, st);
    s.item_first.alloc(s.nitems);
    s.item_cnt.alloc(s.nitems);
    items_fill<<<grid_for(s.nlevels, 128), 128, 0, st>>>(s.nlevels, nb, s.per_item, start.p, nit.p,
                                                        s.item_first.p, s.item_cnt.p);
    CK_LAUNCH();
    s.slots.alloc(s.nitems * s.per_item);
    slots_fill<<<grid_for(s.nitems * s.per_item, 256), 256, 0, st>>>(s.nitems, s.per_item, s.order.p,
                                                                     s.item_first.p, s.item_cnt.p, s.slots.p);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(st));
}

void build_block_cols(const DevCsr& M, int bs, int mode, BlockCols& bc, cudaStream_t st) {
    const int64_t nb = M.n / bs;
    bc.bp.alloc(nb + 1);
    if (nb > 0) {
        bc_count<<<grid_for(nb, 256), 256, 0, st>>>(nb, bs, mode, M.rp.p, bc.bp.p);
        CK_LAUNCH();
    }
    CK(cudaMemsetAsync(bc.bp.p + nb, 0, sizeof(int64_t), st));
    scan_inplace(bc.bp.p, nb + 1, st);
    const int64_t tot = dev_read(bc.bp.p + nb, st);
    bc.bcol.alloc(std::max<int64_t>(tot, 1));
    if (nb > 0) {
        bc_fill<<<grid_for(nb, 256), 256, 0, st>>>(nb, bs, mode, M.rp.p, M.cols.p, bc.bp.p, bc.bcol.p);
        CK_LAUNCH();
    }
}


Analysis& ensure_analysis(Matrix& m, cudaStream_t st) {
    if (m.an) return *m.an;
    const DevCsr& a = m.a;
    const int64_t n = a.n;
    if (m.missing_diag_row >= 0)
        throw FormatError("missing diagonal at row " + std::to_string(m.missing_diag_row));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    auto an = std::make_unique<Analysis>();
    static std::atomic<uint64_t> next_id{1};
    an->id = next_id++;
    DevCsr& L = an->lower;
    DevCsr& U = an->upper;
    L.n = U.n = n;
    L.rp.alloc(n + 1);
    U.rp.alloc(n + 1);
    if (n > 0) {
        lu_counts<<<grid_for(n, 256), 256, 0, st>>>(n, a.rp.p, m.diag_pos.p, L.rp.p, U.rp.p);
        CK_LAUNCH();
    }
    CK(cudaMemsetAsync(L.rp.p + n, 0, sizeof(int64_t), st));
    CK(cudaMemsetAsync(U.rp.p + n, 0, sizeof(int64_t), st));
    scan_inplace(L.rp.p, n + 1, st);
    scan_inplace(U.rp.p, n + 1, st);
    L.nnz = dev_read(L.rp.p + n, st);
    U.nnz = dev_read(U.rp.p + n, st);
    L.cols.alloc(L.nnz);
    L.vals.alloc(L.nnz);
    U.cols.alloc(U.nnz);
    an->u2l.alloc(U.nnz);
    if (n > 0) {
        lu_fill<<<grid_for(n * 32, 256), 256, 0, st>>>(n, a.rp.p, a.cols.p, a.vals.p, m.diag_pos.p,
                                                       L.rp.p, L.cols.p, L.vals.p, U.rp.p, U.cols.p);
        CK_LAUNCH();
        u2l_fill<<<grid_for(n * 32, 256), 256, 0, st>>>(n, U.rp.p, U.cols.p, L.rp.p, L.cols.p,
                                                        an->u2l.p);
        CK_LAUNCH();
    }
    // dof block size: the largest bs in {3, 2} whose diagonal blocks are
    // dense, else 1
    an->bs = 1;
    for (int bs : {3, 2}) {
        if (n == 0 || n % bs) continue;
        DevBuf<int> bad(1);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        block_check<<<grid_for(n, 256), 256, 0, st>>>(n, bs, L.rp.p, L.cols.p, bad.p);
        CK_LAUNCH();
        if (dev_read(bad.p, st) == 0) {
            an->bs = bs;
            break;
        }
    }
    // lanes per block from the mean off-block entry count
    const int bs = an->bs;
    const double off_per_block =
        n ? (static_cast<double>(L.nnz) - static_cast<double>(n / bs) * bs * (bs + 1) / 2.0) /
                static_cast<double>(n / bs)
          : 0.0;
    an->bsr = false;
    if (bs > 1 && !(getenv("PCLAB_BSR") && atoi(getenv("PCLAB_BSR")) == 0)) {
        DevBuf<int> bad(1);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        bsr_check<<<grid_for(n / bs, 256), 256, 0, st>>>(n / bs, bs, L.rp.p, L.cols.p, bad.p);
        CK_LAUNCH();
        an->bsr = dev_read(bad.p, st) == 0;
    }
    // node-blocked: one lane per neighbour block; else one per entry
    const double work = an->bsr ? off_per_block / (bs * bs) : off_per_block;
    // (4 = the narrowest lane group the sweeps instantiate: the schedule's
    // items must hold exactly 32 / lanes blocks of the kernel that runs them)
    int lanes = 4;
    while (lanes < 32 && lanes < work) lanes *= 2;
    if (getenv("PCLAB_LANES")) lanes = atoi(getenv("PCLAB_LANES"));
    // (row-granular level sets are computed on request only: pclab_precond_levels;
    // the critical-predecessor index is needed by the claim-based fallback
    // sweep only, filled below when the round-robin slot records do not fit)
    an->blk_lo.need_crit = an->blk_up.need_crit = false;
    if (an->bsr) {  // block columns first: the levelling walks them
        build_block_cols(L, bs, 0, an->lbc, st);
        build_block_cols(U, bs, 1, an->ubc, st);
    }
    build_schedule(L, U, bs, false, lanes, an->blk_lo, st, an->bsr ? &an->lbc : nullptr,
                   an->bsr ? &an->ubc : nullptr);
    build_schedule(U, L, bs, true, lanes, an->blk_up, st, an->bsr ? &an->ubc : nullptr,
                   an->bsr ? &an->lbc : nullptr);
    an->rr = false;
    DevBuf<int> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    {
        for (Schedule* sc : {&an->blk_lo, &an->blk_up}) {
            const bool lo = sc == &an->blk_lo;
            const DevCsr& M = lo ? L : U;
            const int64_t ns = sc->nitems * sc->per_item;
            sc->slot_rp.alloc(std::max<int64_t>(4 * ns, 1));
            if (ns > 0) {
                slot_rp_fill<<<grid_for(ns, 256), 256, 0, st>>>(
                    ns, bs, sc->slots.p, M.rp.p, an->bsr ? (lo ? an->lbc : an->ubc).bp.p : nullptr, sc->slot_rp.p,
                    bad.p);
                CK_LAUNCH();
            }
        }
        an->rr = !an->bsr && dev_read(bad.p, st) == 0;
        if (!an->bsr && !an->rr) {
            for (Schedule* sc : {&an->blk_lo, &an->blk_up}) {
                if (sc->need_crit || sc->nblocks == 0) continue;
                const bool up = sc == &an->blk_up;
                const DevCsr& P = up ? U : L;
                crit_kernel<<<grid_for(sc->nblocks, 256), 256, 0, st>>>(sc->nblocks, bs, P.rp.p, P.cols.p, up,
                                                                        sc->level.p, sc->crit.p);
                CK_LAUNCH();
                sc->need_crit = true;
            }
        }
    }
    if (an->bsr) {
        if (dev_read(bad.p, st) != 0) {  // a row too long for the packed record: entry-lane sweep
            an->bsr = false;
            for (Schedule* sc : {&an->blk_lo, &an->blk_up}) {
                if (sc->need_crit || sc->nblocks == 0) continue;
                const bool up = sc == &an->blk_up;
                const DevCsr& P = up ? U : L;
                crit_kernel<<<grid_for(sc->nblocks, 256), 256, 0, st>>>(sc->nblocks, bs, P.rp.p, P.cols.p, up,
                                                                        sc->level.p, sc->crit.p);
                CK_LAUNCH();
                sc->need_crit = true;
            }
        }
    }
    // the item-ordered value streams / slot records (bss.cu) on the final sweep layout
    build_bss(*an, st);
    // node-blocked A: the PCG product reads one column index per block
    an->a_bsr = false;
    if (an->bsr) {
        DevBuf<int> bad(1);
        CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        bsr_check_full<<<grid_for(n / bs, 256), 256, 0, st>>>(n / bs, bs, a.rp.p, a.cols.p, bad.p);
        CK_LAUNCH();
        if (dev_read(bad.p, st) == 0) {
            build_block_cols(a, bs, 2, an->abc, st);
            an->a_bsr = true;
        }
    }
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    an->ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    m.an = std::move(an);
    return *m.an;
}

}  // namespace pclab_b200
