// Line-tile sweep (lts_trsv_kernel) for node-blocked factors.
//
// The substitution DAG of a mesh numbered line by line is made of long
// chains: node b depends on node b - 1 one level below it (a grid line along
// x on the 118^3 elasticity mesh: 119 nodes), and a node's other critical
// (level - 1) dependencies sit on the neighbouring lines. The round-robin
// sweeps (sweep.cuh, bst.cu) pay one L2 round trip per level for every such
// dependency -- 823 levels x ~1 us. Here the chain structure is read off the
// matrix and kept on chip:
//
//  * chain   = maximal run of consecutive sweep positions q (lower sweep:
//              q = node, upper: q = nodes - 1 - node) in which each node
//              depends on its predecessor and sits one level above it;
//  * unit    = two consecutive chains, run by ONE warp (16 lanes per chain,
//              lane n owning neighbour block n as in bsr_item): the unit's
//              items pair the two chains' nodes of equal level, in level
//              order, so an item's two nodes never depend on each other;
//  * tile    = kLtsWarps consecutive units = one CTA. Every node of the tile
//              publishes its solution to a shared-memory slot as well as to
//              the global vector; dependencies inside the tile are polled in
//              shared memory (tens of cycles), the others in L2 as before,
//              and those of the NEXT item are issued before the current item
//              is processed (they are mostly final by then).
//
// Tiles are taken in sweep order with a ticket (ctr, zero on entry), so every
// dependency of a running tile lies in a tile that is resident or finished;
// a warp runs its items in level order, so the unfinished node of the lowest
// level among the taken tiles is always runnable: deadlock-free without any
// barrier between levels. The item records are bst.cu's (one bulk copy per
// item into a per-warp ring of S stages), a warp's items being consecutive in
// the stream. Per lane the FMA order, the shuffle tree and the diagonal solve
// are bsr_item's: results are bit-identical to the other node-blocked sweeps.
#include "core.h"
#include "sweep.cuh"
#include "bst.cuh"

#include <cstdio>

namespace pclab_b200 {

namespace {

constexpr int kLtsWarps = BSR_THREADS / 32;  // units per tile
constexpr int kLtsChains = 2 * kLtsWarps;    // chains per tile
constexpr int kLtsMaxTileNodes = 2048;

__device__ __forceinline__ int64_t blk_at(int64_t q, int64_t nb, bool upper) { return upper ? nb - 1 - q : q; }

// 1 where a chain starts (one extra zero for the scan)
__global__ void lts_flags(int64_t nb, bool upper, const int32_t* __restrict__ level,
                          const int64_t* __restrict__ bp, const int32_t* __restrict__ bcol,
                          int64_t* __restrict__ f) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q > nb) return;
    if (q == nb) {
        f[q] = 0;
        return;
    }
    const int64_t b = blk_at(q, nb, upper);
    int start = 1;
    if (q > 0 && bp[b + 1] > bp[b]) {
        const int64_t prev = upper ? b + 1 : b - 1;
        const int64_t adj = upper ? bcol[bp[b]] / 3 : bcol[bp[b + 1] - 1] / 3;
        if (adj == prev && level[b] == level[prev] + 1) start = 0;
    }
    f[q] = start;
}

__global__ void lts_chain_first(int64_t nb, const int64_t* __restrict__ f, int64_t* __restrict__ first) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q > nb) return;
    if (q == nb)
        first[f[nb]] = nb;
    else if (f[q + 1] != f[q])
        first[f[q]] = q;
}

struct UnitSpan {
    int64_t q0, q1;    // first sweep position of each chain
    int len0, len1;    // nodes (0: chain absent)
    int l0, l1, lmin, lmax;
};

// unit u = warp u % kLtsWarps of tile u / kLtsWarps: chains 2w, 2w + 1 of the tile's run
__device__ __forceinline__ UnitSpan unit_span(int64_t u, const int2* __restrict__ tile_ch, int64_t nb, bool upper,
                                              const int64_t* __restrict__ first,
                                              const int32_t* __restrict__ level) {
    UnitSpan s;
    const int2 tc = tile_ch[u / kLtsWarps];
    const int w = static_cast<int>(u % kLtsWarps);
    const int have = tc.y - 2 * w;
    const int64_t c0 = tc.x + 2 * w;
    s.q0 = s.q1 = 0;
    s.len0 = s.len1 = 0;
    s.l0 = s.l1 = s.lmin = s.lmax = 0;
    if (have >= 1) {
        s.q0 = first[c0];
        s.len0 = static_cast<int>(first[c0 + 1] - s.q0);
        s.l0 = level[blk_at(s.q0, nb, upper)];
        s.lmin = s.l0;
        s.lmax = s.l0 + s.len0;
    }
    if (have >= 2) {
        s.q1 = first[c0 + 1];
        s.len1 = static_cast<int>(first[c0 + 2] - s.q1);
        s.l1 = level[blk_at(s.q1, nb, upper)];
        s.lmin = min(s.lmin, s.l1);
        s.lmax = max(s.lmax, s.l1 + s.len1);
    }
    return s;
}

__global__ void lts_chain_levels(int64_t nchains, int64_t nb, bool upper, const int64_t* __restrict__ first,
                                 const int32_t* __restrict__ level, int32_t* __restrict__ l0) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (c < nchains) l0[c] = level[blk_at(first[c], nb, upper)];
}

__global__ void lts_unit_lengths(int64_t nunits, const int2* __restrict__ tile_ch, int64_t nb, bool upper,
                                 const int64_t* __restrict__ first, const int32_t* __restrict__ level,
                                 int64_t* __restrict__ ulen) {
    const int64_t u = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (u > nunits) return;
    if (u == nunits) {
        ulen[u] = 0;
        return;
    }
    const UnitSpan s = unit_span(u, tile_ch, nb, upper, first, level);
    ulen[u] = s.lmax - s.lmin;
}

// the nodes of every item (warp per unit) and the item's tile
__global__ void lts_items(int64_t nunits, const int2* __restrict__ tile_ch, int64_t nb, bool upper,
                          const int64_t* __restrict__ first, const int32_t* __restrict__ level,
                          const int64_t* __restrict__ uitem, int32_t* __restrict__ slots,
                          int32_t* __restrict__ item_tile, int32_t* __restrict__ unit_item) {
    const int64_t u = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (u > nunits) return;
    if (lane == 0) unit_item[u] = static_cast<int32_t>(uitem[u]);
    if (u == nunits) return;
    const UnitSpan s = unit_span(u, tile_ch, nb, upper, first, level);
    for (int k = lane; k < s.lmax - s.lmin; k += 32) {
        const int lev = s.lmin + k;
        const int64_t i = uitem[u] + k;
        const int p0 = lev - s.l0, p1 = lev - s.l1;
        slots[2 * i] = p0 >= 0 && p0 < s.len0 ? static_cast<int32_t>(blk_at(s.q0 + p0, nb, upper)) : -1;
        slots[2 * i + 1] = p1 >= 0 && p1 < s.len1 ? static_cast<int32_t>(blk_at(s.q1 + p1, nb, upper)) : -1;
        item_tile[i] = static_cast<int32_t>(u / kLtsWarps);
    }
}

// sweep-position range of every tile, the tile of every node
__global__ void lts_tiles(int64_t ntiles, const int2* __restrict__ tile_ch, const int64_t* __restrict__ first,
                          int2* __restrict__ tile_q, int* __restrict__ max_nodes) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= ntiles) return;
    const int2 tc = tile_ch[t];
    const int64_t q0 = first[tc.x], q1 = first[tc.x + tc.y];
    tile_q[t] = make_int2(static_cast<int>(q0), static_cast<int>(q1 - q0));
    atomicMax(max_nodes, static_cast<int>(q1 - q0));
}
__global__ void lts_node_tiles(int64_t ntiles, const int2* __restrict__ tile_q, int32_t* __restrict__ node_tile) {
    const int64_t t = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    if (t >= ntiles) return;
    const int2 tq = tile_q[t];
    for (int k = threadIdx.x & 31; k < tq.y; k += 32) node_tile[tq.x + k] = static_cast<int32_t>(t);
}
// the ticket order must be a topological order of the tiles: every
// neighbour of a node lies in the node's tile or in an earlier one
__global__ void lts_check_order(int64_t nb, bool upper, const int64_t* __restrict__ bp,
                                const int32_t* __restrict__ bcol, const int32_t* __restrict__ node_tile,
                                int* __restrict__ bad) {
    const int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (q >= nb) return;
    const int64_t b = blk_at(q, nb, upper);
    const int32_t mine = node_tile[q];
    for (int64_t e = bp[b]; e < bp[b + 1]; ++e) {
        const int64_t qn = blk_at(bcol[e] / 3, nb, upper);
        if (node_tile[qn] > mine) *bad = 1;
    }
}

void build_one(LineTiles& lt, const Schedule& s, const BlockCols& bc, bool upper, cudaStream_t st) {
    lt.ok = false;
    lt.upper = upper;
    const int64_t nb = s.nblocks;
    lt.nb = nb;
    if (nb < 16 || nb >= (1LL << 30) || s.level.n < nb) return;
    DevBuf<int64_t> f(nb + 1);
    lts_flags<<<gridn(nb + 1, 256), 256, 0, st>>>(nb, upper, s.level.p, bc.bp.p, bc.bcol.p, f.p);
    CK_LAUNCH();
    scan_inplace(f.p, nb + 1, st);
    const int64_t nchains = dev_read(f.p + nb, st);
    // short chains: nothing to keep on chip
    if (nchains * 4 > nb) return;
    DevBuf<int64_t> first(nchains + 1);
    lts_chain_first<<<gridn(nb + 1, 256), 256, 0, st>>>(nb, f.p, first.p);
    CK_LAUNCH();
    // Ticket order: chains by window of their start level, sweep order
    // inside a window (the wavefront crosses the windows one after the
    // other, so the resident tiles are the active ones); a tile is a run of
    // up to kLtsChains consecutive chains of one window. The chain start
    // levels are few (one per grid line): ordered on the host.
    DevBuf<int32_t> l0(nchains);
    lts_chain_levels<<<gridn(nchains, 256), 256, 0, st>>>(nchains, nb, upper, first.p, s.level.p, l0.p);
    CK_LAUNCH();
    std::vector<int32_t> hl0(static_cast<size_t>(nchains));
    CK(cudaMemcpyAsync(hl0.data(), l0.p, sizeof(int32_t) * hl0.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int stride = nchains > 1 ? hl0[1] - hl0[0] : 1;
    stride = std::min(std::max(stride, 1), 64);
    const int window = std::max(env_int("PCLAB_LTS_WINDOW", kLtsChains * stride), 1);
    int32_t maxl = 0;
    for (int32_t v : hl0) maxl = std::max(maxl, v);
    const int nwin = maxl / window + 1;
    std::vector<int64_t> wfirst(static_cast<size_t>(nwin) + 1, 0);
    for (int32_t v : hl0) ++wfirst[static_cast<size_t>(v / window) + 1];
    for (int w = 0; w < nwin; ++w) wfirst[w + 1] += wfirst[w];
    std::vector<int32_t> perm(hl0.size());
    {
        std::vector<int64_t> pos(wfirst.begin(), wfirst.end() - 1);
        for (int64_t c = 0; c < nchains; ++c) perm[static_cast<size_t>(pos[hl0[c] / window]++)] = static_cast<int32_t>(c);
    }
    std::vector<int2> htile;
    for (int64_t r = 0; r < nchains; ++r) {
        const int32_t c = perm[r];
        const bool cut = r == 0 || hl0[c] / window != hl0[perm[r - 1]] / window || c != perm[r - 1] + 1 ||
                         htile.back().y == kLtsChains;
        if (cut)
            htile.push_back(make_int2(c, 1));
        else
            ++htile.back().y;
    }
    const int64_t ntiles = static_cast<int64_t>(htile.size()), nunits = ntiles * kLtsWarps;
    lt.tile_ch.alloc(ntiles);
    CK(cudaMemcpyAsync(lt.tile_ch.p, htile.data(), sizeof(int2) * htile.size(), cudaMemcpyHostToDevice, st));
    DevBuf<int64_t> uitem(nunits + 1);
    lts_unit_lengths<<<gridn(nunits + 1, 256), 256, 0, st>>>(nunits, lt.tile_ch.p, nb, upper, first.p, s.level.p,
                                                            uitem.p);
    CK_LAUNCH();
    scan_inplace(uitem.p, nunits + 1, st);
    const int64_t nitems = dev_read(uitem.p + nunits, st);  // (also orders the host tile list before it dies)
    if (nitems == 0 || nitems >= (1LL << 30)) return;
    lt.tile_q.alloc(ntiles);
    DevBuf<int> mx(3);
    CK(cudaMemsetAsync(mx.p, 0, 3 * sizeof(int), st));
    lts_tiles<<<gridn(ntiles, 256), 256, 0, st>>>(ntiles, lt.tile_ch.p, first.p, lt.tile_q.p, mx.p);
    CK_LAUNCH();
    {
        DevBuf<int32_t> node_tile(nb);
        lts_node_tiles<<<gridn(ntiles * 32, 256), 256, 0, st>>>(ntiles, lt.tile_q.p, node_tile.p);
        CK_LAUNCH();
        lts_check_order<<<gridn(nb, 256), 256, 0, st>>>(nb, upper, bc.bp.p, bc.bcol.p, node_tile.p, mx.p + 2);
        CK_LAUNCH();
    }
    lt.slots.alloc(2 * nitems);
    lt.item_tile.alloc(nitems);
    lt.unit_item.alloc(nunits + 1);
    lts_items<<<gridn((nunits + 1) * 32, 256), 256, 0, st>>>(nunits, lt.tile_ch.p, nb, upper, first.p, s.level.p,
                                                            uitem.p, lt.slots.p, lt.item_tile.p, lt.unit_item.p);
    CK_LAUNCH();
    DevBuf<int64_t> off(nitems + 1);
    bst_lengths<<<gridn(nitems + 1, 256), 256, 0, st>>>(nitems, lt.slots.p, bc.bp.p, off.p, mx.p + 1);
    CK_LAUNCH();
    scan_inplace(off.p, nitems + 1, st);
    const int64_t total16 = dev_read(off.p + nitems, st);
    int h[3];
    CK(cudaMemcpyAsync(h, mx.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    lt.nchains = nchains;
    lt.ntiles = ntiles;
    lt.nitems = nitems;
    lt.stage = h[1];
    lt.max_tile_nodes = h[0];
    if (h[2] != 0 || total16 >= (1LL << 32) || h[1] > kBstMaxStage || h[0] > kLtsMaxTileNodes) return;
    lt.loc.alloc(nitems);
    bst_locs<<<gridn(nitems, 256), 256, 0, st>>>(nitems, off.p, lt.loc.p);
    CK_LAUNCH();
    lt.nchains = nchains;
    lt.nunits = nunits;
    lt.ntiles = ntiles;
    lt.nitems = nitems;
    lt.stream_bytes = 16 * total16;
    lt.stage = h[1];
    lt.max_tile_nodes = h[0];
    lt.ok = true;
}

// ------------------------------------------------------------ the sweep

// ---- warp roles of a tile (CTA):
//   warps 0 .. kLtsWarps-1     solver of unit w: the critical chain only
//   warp kLtsWarps             copy warp: keeps every unit's stage ring full
//   then K helper warps per unit (helper h of unit w takes the unit's items
//   h, h + K, ...)
// A node's neighbours come in two groups (rec_fill): the critical ones, at
// most two levels below it -- they become final just before the node can be
// solved -- and the rest, final long before. A helper warp reduces the rest
// ahead of time: q = sum(A_n x_n) - rhs over the non-critical neighbours,
// published in the node's shared-memory q slot. The solver's item is then
//   critical lanes: poll neighbour (shared memory / L2, the L2 ones issued an
//   item ahead), 9 FMAs;   lane ncrit: q;   8-lane shuffle tree;   3x3 solve;
//   publish (shared-memory slot + global vector)
// -- the only work left on the level-to-level dependency chain.
struct LtsDec {
    uint32_t v, c;  // shared-memory addresses of the lane group's values / neighbour codes
    int blk, nb, ncrit;
};

__device__ __forceinline__ LtsDec lts_decode(uint32_t rec, int grp, int& other_rest) {
    int4 hd;
    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(hd.x), "=r"(hd.y), "=r"(hd.z), "=r"(hd.w) : "r"(rec));
    const int nb0 = hd.z & 0xffff, nb1 = hd.w & 0xffff, nc0 = hd.z >> 16, nc1 = hd.w >> 16;
    LtsDec d;
    d.blk = grp ? hd.y : hd.x;
    d.nb = grp ? nb1 : nb0;
    d.ncrit = grp ? nc1 : nc0;
    const int nv0 = hd.x >= 0 ? 9 * nb0 + 6 : 0, nv1 = hd.y >= 0 ? 9 * nb1 + 6 : 0;
    d.v = rec + 16 + (grp ? 8 * nv0 : 0);
    d.c = rec + 16 + 8 * ((nv0 + nv1 + 1) & ~1) + (grp ? 4 * nb0 : 0);
    other_rest = max(nb0 - nc0, nb1 - nc1);
    return d;
}

__device__ __forceinline__ void lts_poll(int xb, uint32_t res, const double* out, double (&xv)[3]) {
    if (xb < 0) {
        const uint32_t a = res + 32u * static_cast<uint32_t>(-xb - 1);
        asm volatile("ld.volatile.shared.v2.f64 {%0,%1}, [%2];" : "=d"(xv[0]), "=d"(xv[1]) : "r"(a) : "memory");
        asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(xv[2]) : "r"(a + 16) : "memory");
    } else {
        ld_relaxed_v4(out + 4 * static_cast<int64_t>(xb), xv);
    }
}

__device__ __forceinline__ void lts_load9(uint32_t vn, double (&a)[3][3]) {
#pragma unroll
    for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int c = 0; c < 3; ++c) asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[t][c]) : "r"(vn + 8 * (3 * t + c)));
}

__device__ __forceinline__ bool mbar_test(uint32_t bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// solver state of an item whose record has landed
struct LtsSol {
    LtsDec d;
    int xb;        // critical neighbour of this lane (>= 0 node id: L2 poll, < 0: tile slot)
    int role;      // 0 idle lane, 1 critical neighbour, 2 the q lane
    double xv[3];  // neighbour values / q (pending until read)
};

__device__ __forceinline__ void lts_sol_load(LtsSol& s, uint32_t rec, int grp, int gl, const double* out) {
    int rest;
    s.d = lts_decode(rec, grp, rest);
    s.role = s.d.blk < 0 ? 0 : (gl < s.d.ncrit ? 1 : (gl == s.d.ncrit ? 2 : 0));
    s.xb = 0;
    s.xv[0] = pending_value();
    s.xv[1] = s.xv[2] = 0.0;
    if (s.role == 1) {
        asm volatile("ld.shared.s32 %0, [%1];" : "=r"(s.xb) : "r"(s.d.c + 4 * gl));
        if (s.xb >= 0) ld_relaxed_v4(out + 4 * static_cast<int64_t>(s.xb), s.xv);
    }
}

constexpr int lts_threads(int helpers) { return (kLtsWarps * (1 + helpers) + 1) * 32; }

template <bool UPPER, int S, int K, bool TRACE = false>
__global__ void __launch_bounds__(lts_threads(K), 2)
lts_trsv_kernel(int ntiles, int nunits, int nbk, const int2* __restrict__ tile_q,
                const int32_t* __restrict__ unit_item, const uint2* __restrict__ loc,
                const unsigned char* __restrict__ stream, const double* rhs, double* out, double* reset,
                const int* __restrict__ done, unsigned* ticket, int stage_bytes, int res_bytes,
                long long* trace, int opt) {
    if (done && *done) return;
    constexpr int BS = 3, LG = 16, NIB = 3;
    constexpr int NT = lts_threads(K);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t full[kLtsWarps * S], empty[kLtsWarps * S];
    __shared__ int s_tile;
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int grp = lane / LG, gl = lane % LG;
    const uint32_t res = smem_addr(smem);                   // solutions of the tile's nodes
    const uint32_t qs = res + static_cast<uint32_t>(res_bytes);  // helpers' partial sums
    const uint32_t rings = qs + static_cast<uint32_t>(res_bytes);
    if (threadIdx.x == 0) {
        for (int j = 0; j < kLtsWarps * S; ++j) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(full + j)) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_addr(empty + j)) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // unit slot of this warp and its role
    const bool is_copy = wi == kLtsWarps;
    const bool is_solver = wi < kLtsWarps;
    const int w = is_solver ? wi : (wi - kLtsWarps - 1) % kLtsWarps;  // (copy warp: per lane)
    const int h = is_solver || is_copy ? 0 : (wi - kLtsWarps - 1) / kLtsWarps;
    unsigned cnt = 0;  // items of unit slot w (copy warp: slot `lane`) before this tile
    const double pend_v = pending_value();
    uint64_t pol = 0;
    if (is_copy) pol = evict_first_policy();
    for (;;) {
        if (threadIdx.x == 0) s_tile = static_cast<int>(atomicAdd(ticket, 1u));
        __syncthreads();
        const int t = s_tile;
        if (t >= ntiles) break;
        const int2 tq = __ldg(tile_q + t);
        if (TRACE && threadIdx.x == 0) {
            long long now;
            unsigned sm;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
            asm volatile("mov.u32 %0, %smid;" : "=r"(sm));
            trace[4 * t] = now;
            trace[4 * t + 3] = sm;
        }
        for (int idx = threadIdx.x; idx < 2 * tq.y; idx += NT) {
            asm volatile("st.shared.v2.f64 [%0], {%1,%1};" ::"r"(res + 16u * idx), "d"(pend_v) : "memory");
            asm volatile("st.shared.v2.f64 [%0], {%1,%1};" ::"r"(qs + 16u * idx), "d"(pend_v) : "memory");
        }
        __syncthreads();
        if (is_copy) {
            // ---- copy warp: lane w feeds unit w, round-robin, never blocking
            if (lane < kLtsWarps) {
                const int u = t * kLtsWarps + lane;
                int i = u < nunits ? __ldg(unit_item + u) : 0;
                const int i1 = u < nunits ? __ldg(unit_item + u + 1) : 0;
                const uint32_t ring = rings + static_cast<uint32_t>(lane * S * stage_bytes);
                const uint32_t fb = smem_addr(full + lane * S), eb = smem_addr(empty + lane * S);
                uint2 l = i < i1 ? __ldg(loc + i) : make_uint2(0, 0);
                while (i < i1) {
                    const unsigned st = cnt % S, use = cnt / S;
                    if (use == 0 || mbar_test(eb + 8 * st, (use - 1) & 1u)) {
                        mbar_expect_tx(fb + 8 * st, l.y);
                        tma_bulk_g2s_hint(ring + st * stage_bytes, stream + 16 * static_cast<uint64_t>(l.x), l.y,
                                          fb + 8 * st, pol);
                        ++cnt;
                        ++i;
                        if (i < i1) l = __ldg(loc + i);
                    }
                }
            }
        } else {
            const int u = t * kLtsWarps + w;
            const int i0 = u < nunits ? __ldg(unit_item + u) : 0, i1 = u < nunits ? __ldg(unit_item + u + 1) : 0;
            const uint32_t ring = rings + static_cast<uint32_t>(w * S * stage_bytes);
            const uint32_t fb = smem_addr(full + w * S), eb = smem_addr(empty + w * S);
            if (is_solver && i0 < i1) {
                // ---- solver: the critical chain
                LtsSol nx;
                mbar_wait_addr(fb + 8 * (cnt % S), (cnt / S) & 1u);
                lts_sol_load(nx, ring + (cnt % S) * stage_bytes, grp, gl, out);
                for (int i = i0; i < i1; ++i) {
                    const LtsSol cur = nx;
                    const unsigned ca = cnt + static_cast<unsigned>(i - i0);
                    if (i + 1 < i1) {
                        mbar_wait_addr(fb + 8 * ((ca + 1) % S), ((ca + 1) / S) & 1u);
                        lts_sol_load(nx, ring + ((ca + 1) % S) * stage_bytes, grp, gl, out);
                    }
                    const bool active = cur.d.blk >= 0;
                    const uint32_t slot =
                        32u * static_cast<uint32_t>(active ? (UPPER ? nbk - 1 - cur.d.blk : cur.d.blk) - tq.x : 0);
                    double bin[NIB], binv[BS], a[BS][BS], xv[BS];
                    if (active && gl == 0) {
#pragma unroll
                        for (int q = 0; q < NIB; ++q)
                            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(bin[q]) : "r"(cur.d.v + 8 * (9 * cur.d.nb + q)));
#pragma unroll
                        for (int tt = 0; tt < BS; ++tt)
                            asm volatile("ld.shared.f64 %0, [%1];"
                                         : "=d"(binv[tt])
                                         : "r"(cur.d.v + 8 * (9 * cur.d.nb + NIB + tt)));
                    }
                    if (cur.role == 1) {
                        lts_load9(cur.d.v + 72 * gl, a);
                    } else {
#pragma unroll
                        for (int tt = 0; tt < BS; ++tt)
#pragma unroll
                            for (int cc = 0; cc < BS; ++cc) a[tt][cc] = 0.0;
                    }
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) xv[cc] = cur.xv[cc];
                    bool pend = cur.role != 0 && (is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]));
                    while (__any_sync(0xffffffffu, pend)) {
                        if (pend) {
                            lts_poll(cur.role == 2 ? -1 - static_cast<int>(slot / 32u) : cur.xb, cur.role == 2 ? qs : res,
                                     out, xv);
                            pend = is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]);
                        }
                    }
                    double acc[BS];
#pragma unroll
                    for (int tt = 0; tt < BS; ++tt) {
                        acc[tt] = cur.role == 2 ? xv[tt] : 0.0;
#pragma unroll
                        for (int cc = 0; cc < BS; ++cc) acc[tt] = fma(a[tt][cc], xv[cc], acc[tt]);
                    }
#pragma unroll
                    for (int tt = 0; tt < BS; ++tt) acc[tt] = group_sum<8>(acc[tt]);
                    if (active && gl == 0) {
                        const double zero[BS] = {0.0, 0.0, 0.0};
                        double x[BS];
                        solve_diag_block<BS, UPPER>(zero, acc, bin, binv, x);
                        asm volatile("st.volatile.shared.v2.f64 [%0], {%1,%2};" ::"r"(res + slot), "d"(x[0]), "d"(x[1])
                                     : "memory");
                        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(res + slot + 16), "d"(x[2]) : "memory");
                        st_relaxed_v4(out + 4 * static_cast<int64_t>(cur.d.blk), x[0], x[1], x[2], 0.0);
                    }
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(eb + 8 * (ca % S)) : "memory");
                    if (TRACE && i == i0 && lane == 0 && wi == 0) {
                        long long now;
                        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
                        trace[4 * t + 1] = now;
                    }
                }
            } else if (!is_solver) {
                // ---- helper h of unit w: q = sum over the non-critical neighbours - rhs
                for (int i = i0 + h; i < i1; i += K) {
                    const unsigned ca = cnt + static_cast<unsigned>(i - i0);
                    mbar_wait_addr(fb + 8 * (ca % S), (ca / S) & 1u);
                    int rest;
                    const LtsDec d = lts_decode(ring + (ca % S) * stage_bytes, grp, rest);
                    const bool active = d.blk >= 0;
                    double rc[BS] = {0.0, 0.0, 0.0};
                    if (active && gl == 0) {
                        if constexpr (UPPER) {  // padded y: one 256-bit load
                            double d3;
                            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                                         : "=d"(rc[0]), "=d"(rc[1]), "=d"(rc[2]), "=d"(d3)
                                         : "l"(rhs + 4 * static_cast<int64_t>(d.blk)));
                            (void)d3;
                        } else {
#pragma unroll
                            for (int tt = 0; tt < BS; ++tt) rc[tt] = rhs[static_cast<int64_t>(d.blk) * 3 + tt];
                        }
                    }
                    double acc[BS] = {0.0, 0.0, 0.0};
                    for (int n0 = 0; n0 < rest; n0 += LG) {
                        const int n = d.ncrit + n0 + gl;
                        const bool own = active && n < d.nb;
                        double a[BS][BS], xv[BS] = {0.0, 0.0, 0.0};
                        int32_t xb = 0;
                        if (own) {
                            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(xb) : "r"(d.c + 4 * n));
                            lts_load9(d.v + 72 * n, a);
                            lts_poll(xb, res, out, xv);
                        } else {
#pragma unroll
                            for (int tt = 0; tt < BS; ++tt)
#pragma unroll
                                for (int cc = 0; cc < BS; ++cc) a[tt][cc] = 0.0;
                        }
                        bool pend = own && (is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]));
                        while (__any_sync(0xffffffffu, pend)) {
                            if (opt & 4) __nanosleep(40);
                            if (pend) {
                                lts_poll(xb, res, out, xv);
                                pend = is_pending(xv[0]) || is_pending(xv[1]) || is_pending(xv[2]);
                            }
                        }
#pragma unroll
                        for (int tt = 0; tt < BS; ++tt)
#pragma unroll
                            for (int cc = 0; cc < BS; ++cc) acc[tt] = fma(a[tt][cc], xv[cc], acc[tt]);
                    }
#pragma unroll
                    for (int tt = 0; tt < BS; ++tt) acc[tt] = group_sum<LG>(acc[tt]);
                    if (active && gl == 0) {
                        const uint32_t slot = qs + 32u * static_cast<uint32_t>((UPPER ? nbk - 1 - d.blk : d.blk) - tq.x);
                        asm volatile("st.volatile.shared.v2.f64 [%0], {%1,%2};" ::"r"(slot), "d"(acc[0] - rc[0]),
                                     "d"(acc[1] - rc[1])
                                     : "memory");
                        asm volatile("st.volatile.shared.f64 [%0], %1;" ::"r"(slot + 16), "d"(acc[2] - rc[2]) : "memory");
                    }
                    __syncwarp();
                    if (lane == 0)
                        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(eb + 8 * (ca % S)) : "memory");
                    if (reset && active && gl < BS) reset[4 * static_cast<int64_t>(d.blk) + gl] = pend_v;
                }
            }
            cnt += static_cast<unsigned>(i1 - i0);
        }
        __syncthreads();  // the tile's slots are re-armed for the next tile
        if (TRACE && threadIdx.x == 0) {
            long long now;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
            trace[4 * t + 2] = now;
        }
    }
}

int lts_stages() {
    static const int s = env_int("PCLAB_LTS_STAGES", 4);
    return s;
}

template <bool UPPER, int S, int K>
void launch_lts_t(const LineTiles& lt, const unsigned char* stream, const double* b, double* x, double* reset,
                  const int* done, unsigned* ctr, cudaStream_t st) {
    auto kern = lts_trsv_kernel<UPPER, S, K>;
    constexpr int NT = lts_threads(K);
    const int stage = (lt.stage + 15) & ~15;
    const int res_bytes = (32 * lt.max_tile_nodes + 127) & ~127;
    const size_t dyn = 2 * static_cast<size_t>(res_bytes) + static_cast<size_t>(kLtsWarps) * S * stage;
    static size_t dyn_set = 0;
    static unsigned cap = 0;
    if (dyn != dyn_set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, dyn));
        cap = static_cast<unsigned>(std::max(per_sm, 1) * sm_count());
        dyn_set = dyn;
    }
    static const int opt = env_int("PCLAB_LTS_OPT", 0);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(lt.ntiles, cap));
    kern<<<grid, NT, dyn, st>>>(static_cast<int>(lt.ntiles), static_cast<int>(lt.nunits), static_cast<int>(lt.nb),
                               lt.tile_q.p, lt.unit_item.p, lt.loc.p, stream, b, x, reset, done, ctr, stage, res_bytes,
                               nullptr, opt);
    CK_LAUNCH();
    if (const char* path = getenv("PCLAB_LTS_TRACE")) {  // developer probe: per-tile timestamps of a second run
        CK(cudaStreamSynchronize(st));
        auto tkern = lts_trsv_kernel<UPPER, S, K, true>;
        CK(cudaFuncSetAttribute(tkern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
        CK(cudaFuncSetAttribute(tkern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        DevBuf<long long> tr(4 * lt.ntiles);
        CK(cudaMemsetAsync(tr.p, 0, tr.bytes(), st));
        CK(cudaMemsetAsync(ctr, 0, sizeof(unsigned), st));
        fill_pending(x, 4 * lt.nb, st);
        tkern<<<grid, NT, dyn, st>>>(static_cast<int>(lt.ntiles), static_cast<int>(lt.nunits),
                                    static_cast<int>(lt.nb), lt.tile_q.p, lt.unit_item.p, lt.loc.p, stream, b, x,
                                    nullptr, done, ctr, stage, res_bytes, tr.p, opt);
        CK_LAUNCH();
        std::vector<long long> h(static_cast<size_t>(4 * lt.ntiles));
        CK(cudaMemcpyAsync(h.data(), tr.p, tr.bytes(), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (FILE* fp = fopen((std::string(path) + (UPPER ? ".up" : ".lo")).c_str(), "w")) {
            std::vector<int2> tc(static_cast<size_t>(lt.ntiles));
            CK(cudaMemcpy(tc.data(), lt.tile_ch.p, sizeof(int2) * tc.size(), cudaMemcpyDeviceToHost));
            for (int64_t t = 0; t < lt.ntiles; ++t)
                fprintf(fp, "%lld %d %d %lld %lld %lld %lld\n", (long long)t, tc[t].x, tc[t].y, h[4 * t], h[4 * t + 1],
                        h[4 * t + 2], h[4 * t + 3]);
            fclose(fp);
        }
    }
}

template <bool UPPER>
void launch_lts_s(const LineTiles& lt, const unsigned char* stream, const double* b, double* x, double* reset,
                  const int* done, unsigned* ctr, cudaStream_t st) {
    static const int helpers = env_int("PCLAB_LTS_HELPERS", 2);
    const int s = lts_stages();
    if (helpers <= 1) {
        launch_lts_t<UPPER, 4, 1>(lt, stream, b, x, reset, done, ctr, st);
    } else if (helpers >= 3) {
        launch_lts_t<UPPER, 5, 3>(lt, stream, b, x, reset, done, ctr, st);
    } else if (s <= 3) {
        launch_lts_t<UPPER, 3, 2>(lt, stream, b, x, reset, done, ctr, st);
    } else if (s >= 6) {
        launch_lts_t<UPPER, 6, 2>(lt, stream, b, x, reset, done, ctr, st);
    } else {
        launch_lts_t<UPPER, 4, 2>(lt, stream, b, x, reset, done, ctr, st);
    }
}

}  // namespace

bool lts_enabled() {
    static const bool on = env_int("PCLAB_LTS", 1) != 0;
    return on;
}

void build_lts(Analysis& an, cudaStream_t st) {
    an.lt_lo.ok = an.lt_up.ok = false;
    if (!lts_enabled() || !(an.bsr && an.bs == 3)) return;
    if (an.blk_lo.lanes != 16 || an.blk_up.lanes != 16) return;
    build_one(an.lt_lo, an.blk_lo, an.lbc, false, st);
    if (an.lt_lo.ok) build_one(an.lt_up, an.blk_up, an.ubc, true, st);
    if (env_int("PCLAB_LTS_VERBOSE", 0))
        for (const LineTiles* lt : {&an.lt_lo, &an.lt_up})
            fprintf(stderr, "lts %s: ok %d nodes %lld chains %lld tiles %lld items %lld stage %d tile nodes %d stream %.1f MB\n",
                    lt->upper ? "upper" : "lower", int(lt->ok), (long long)lt->nb, (long long)lt->nchains,
                    (long long)lt->ntiles, (long long)lt->nitems, lt->stage, lt->max_tile_nodes,
                    lt->stream_bytes / 1e6);
    if (!(an.lt_lo.ok && an.lt_up.ok)) an.lt_lo.ok = an.lt_up.ok = false;
}

void fill_lts(const Analysis& an, Precond& p, cudaStream_t st) {
    if (!an.lt_lo.ok) return;
    for (int up = 0; up < 2; ++up) {
        const LineTiles& lt = up ? an.lt_up : an.lt_lo;
        DevBuf<unsigned char>& out = up ? p.lts_up : p.lts_lo;
        out.alloc(std::max<int64_t>(lt.stream_bytes, 16));
        if (up)
            rec_fill<true, true><<<gridn(lt.nitems * 32, 256), 256, 0, st>>>(
                lt.nitems, lt.nb, (up ? an.blk_up : an.blk_lo).level.p, lt.loc.p, lt.slots.p, lt.item_tile.p, lt.tile_q.p, an.ubc.bp.p, an.ubc.bcol.p,
                an.upper.rp.p, p.uvals.p, p.invd.p, out.p);
        else
            rec_fill<false, true><<<gridn(lt.nitems * 32, 256), 256, 0, st>>>(
                lt.nitems, lt.nb, (up ? an.blk_up : an.blk_lo).level.p, lt.loc.p, lt.slots.p, lt.item_tile.p, lt.tile_q.p, an.lbc.bp.p, an.lbc.bcol.p,
                an.lower.rp.p, p.lvals.p, p.invd.p, out.p);
        CK_LAUNCH();
    }
}

bool launch_lts(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                const int* done, unsigned* ctr, cudaStream_t st, bool pad) {
    const LineTiles& lt = upper ? an.lt_up : an.lt_lo;
    const unsigned char* stream = upper ? p.lts_up.p : p.lts_lo.p;
    if (!pad || !lt.ok || !stream || !ctr) return false;
    if (upper)
        launch_lts_s<true>(lt, stream, b, x, reset, done, ctr, st);
    else
        launch_lts_s<false>(lt, stream, b, x, reset, done, ctr, st);
    return true;
}

}  // namespace pclab_b200
