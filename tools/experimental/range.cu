// Range-pipelined triangular sweeps (y = L^-1 r, z = L^-T y) for the PCG
// loop -- the reference's tri_solve_lower / tri_solve_upper
// (src/krylov.cpp:60-112), sequential there, as a pipelined wavefront here.
//
// Why: a sync-free sweep over the whole GPU pays one L2 round trip per
// level of the dependency DAG (823 node levels on configs[2]), and every
// warp waits on its own item's loads. Here the nodes are cut, in sweep
// order, into contiguous ranges; a persistent CTA owns a range and walks it
// level by level ("steps"):
//   * a producer warp streams each step's data -- node headers, encoded
//     neighbour columns, the factor values of the step's nodes, laid out
//     contiguously in sweep order (the per-factor stream) -- into a ring of
//     shared-memory stages with one bulk copy (TMA, cp.async.bulk) per
//     step, several steps ahead, completion on per-stage mbarriers;
//   * consumer warps take a step's nodes (LG lanes per node, lane n = the
//     node's n-th neighbour block), read the values from shared memory, read
//     each dependency from the CTA's ring of recent results (shared memory,
//     when the analysis proved the slot still holds it) or poll it in global
//     memory (another range, NaN-marker protocol of the sync-free sweeps),
//     reduce, solve the dense diagonal block, and publish to the ring and to
//     global memory; a named barrier closes the step.
// A dependency inside the range costs a barrier instead of an L2 round
// trip; only dependencies across ranges go through L2, and the matrix
// stream arrives ahead of need instead of on each item's critical path.
//
// Deadlock freedom: dependencies of range r lie in ranges < r (sweep order),
// CTA c runs ranges c, c + G, ... in order, and the grid (one CTA per SM) is
// co-resident, so the lowest unfinished range always runs.
//
// Arithmetic: per node, lane n accumulates its neighbour block's BS x BS
// products in the order of bsr_item, the LG lanes reduce with the same
// shuffle tree and the diagonal block is solved by solve_diag_block -- for
// the same LG the results are bit-identical to the round-robin sweep's.
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "core.h"
#include "sweep.cuh"

namespace pclab_b200 {

namespace {

constexpr int kRing = 512;     // ring slots (power of two): results of recent nodes
constexpr int kStages = 8;     // mbarrier slots = most steps in flight

inline unsigned gridn(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

__host__ __device__ inline int64_t logical_of(int64_t b, int64_t nb, bool upper) { return upper ? nb - 1 - b : b; }

// node-blocked (BS = 3): neighbours from the block-column view; scalar (BS =
// 1): from the CSR rows (L: diagonal last, U: diagonal first)
template <int BS, bool UPPER>
__device__ __forceinline__ int node_nb(const int64_t* __restrict__ bp, int64_t b) {
    return static_cast<int>(bp[b + 1] - bp[b]) - (BS == 1 ? 1 : 0);
}
template <int BS, bool UPPER>
__device__ __forceinline__ int64_t node_col0(const int64_t* __restrict__ bp, int64_t b) {
    return bp[b] + ((BS == 1 && UPPER) ? 1 : 0);
}

template <int BS>
__host__ __device__ constexpr int node_vals(int nb) {
    return BS * BS * nb + BS * (BS + 1) / 2;
}
__host__ __device__ inline int64_t al16(int64_t x) { return (x + 15) & ~int64_t(15); }
__host__ __device__ inline int64_t step_bytes(int64_t cnt, int64_t snb, int64_t svals) {
    return 16 * cnt + al16(4 * snb) + al16(8 * svals);
}

// ------------------------------------------------------------ schedule build
__global__ void rs_keys(int64_t nb, bool upper, int64_t R, const int32_t* __restrict__ level,
                        unsigned long long* __restrict__ key, int32_t* __restrict__ val) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const unsigned long long r = static_cast<unsigned long long>(logical_of(b, nb, upper) / R);
    key[b] = (r << 32) | static_cast<unsigned>(level[b]);
    val[b] = static_cast<int32_t>(b);
}

__global__ void rs_group_flags(int64_t nb, const unsigned long long* __restrict__ skey, int64_t* __restrict__ flag) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p < nb) flag[p] = (p == 0 || skey[p] != skey[p - 1]) ? 1 : 0;
    if (p == nb) flag[p] = 0;
}

__global__ void rs_group_first(int64_t nb, const unsigned long long* __restrict__ skey,
                               const int64_t* __restrict__ gid, int64_t* __restrict__ gfirst) {
    const int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (p < nb && (p == 0 || skey[p] != skey[p - 1])) gfirst[gid[p]] = p;
    if (p == nb) gfirst[gid[nb]] = nb;
}

// Greedy split of each (range, level) group into steps of at most `maxb`
// staged bytes. pass 0 counts the steps of each group, pass 1 writes them
// ({0, bytes / 16, nodes, first position}).
template <int BS, bool UPPER>
__global__ void rs_split(int64_t ng, const int64_t* __restrict__ gfirst, const int32_t* __restrict__ order,
                         const int64_t* __restrict__ bp, int64_t maxb, int pass, int64_t* __restrict__ gsteps,
                         int4* __restrict__ steps, int* __restrict__ bad) {
    const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (g >= ng) return;
    int64_t ns = 0, first = gfirst[g], cnt = 0, snb = 0, sv = 0;
    int64_t out = pass ? gsteps[g] : 0;
    auto emit = [&]() {
        if (pass) steps[out + ns] = make_int4(0, static_cast<int>(step_bytes(cnt, snb, sv) / 16),
                                              static_cast<int>(cnt), static_cast<int>(first));
        ++ns;
    };
    for (int64_t p = gfirst[g]; p < gfirst[g + 1]; ++p) {
        const int k = node_nb<BS, UPPER>(bp, order[p]);
        if (step_bytes(1, k, node_vals<BS>(k)) > maxb) *bad = 1;
        if (cnt > 0 && step_bytes(cnt + 1, snb + k, sv + node_vals<BS>(k)) > maxb) {
            emit();
            first = p;
            cnt = snb = sv = 0;
        }
        ++cnt;
        snb += k;
        sv += node_vals<BS>(k);
    }
    if (cnt > 0) emit();
    if (!pass) gsteps[g] = ns;
}

__global__ void rs_len_copy(int64_t ns, const int4* __restrict__ steps, int64_t* __restrict__ len) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s < ns) len[s] = steps[s].y;
    if (s == ns) len[s] = 0;
}

__global__ void rs_offsets(int64_t ns, const int64_t* __restrict__ off16, int4* __restrict__ steps) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s < ns) steps[s].x = static_cast<int>(static_cast<uint32_t>(off16[s]));
}

// first step of each range; step of each node
__global__ void rs_ranges(int64_t ns, int64_t nb, bool upper, int64_t R, int64_t nranges,
                          const int4* __restrict__ steps, const int32_t* __restrict__ order,
                          int64_t* __restrict__ range_step, int32_t* __restrict__ step_of) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s > ns) return;
    if (s == ns) {
        range_step[nranges] = ns;
        return;
    }
    const int4 st = steps[s];
    const int64_t r = logical_of(order[st.w], nb, upper) / R;
    const int64_t rp = s ? logical_of(order[steps[s - 1].w], nb, upper) / R : -1;
    if (r != rp) range_step[r] = s;
    for (int k = 0; k < st.z; ++k) step_of[order[st.w + k]] = static_cast<int32_t>(s);
}

// nxt[m]: the first step >= step_of[m] at which another node of m's range
// writes m's ring slot (m mod kRing); INT_MAX if none. A dependant d of m in
// the same range reads the ring iff step_of[d] < nxt[m].
__global__ void rs_next_writer(int64_t nb, bool upper, int64_t R, const int32_t* __restrict__ step_of,
                               int32_t* __restrict__ nxt) {
    const int64_t m = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (m >= nb) return;
    const int64_t r = logical_of(m, nb, upper) / R;
    const int64_t l0 = r * R, l1 = l0 + R < nb ? l0 + R : nb;
    const int64_t b0 = upper ? nb - l1 : l0, b1 = upper ? nb - l0 : l1;  // block interval of the range
    const int32_t sm = step_of[m];
    int32_t best = INT_MAX;
    const int64_t slot = m & (kRing - 1);
    int64_t m2 = b0 + ((slot - (b0 & (kRing - 1))) & (kRing - 1));
    for (; m2 < b1; m2 += kRing) {
        if (m2 == m) continue;
        const int32_t s2 = step_of[m2];
        if (s2 >= sm && s2 < best) best = s2;
    }
    nxt[m] = best;
}

// ------------------------------------------------------------ stream fill
// One warp per step: node headers {node, neighbours, first column (int32
// units from the step base), first value (double units)}, the encoded
// neighbour columns ((node << 1) | ring bit), then per node its BS x BS
// neighbour blocks (block-major, row-major inside a block), the NIB
// strictly-triangular diagonal-block entries (solve_diag_block order) and
// the BS reciprocal pivots.
template <int BS, bool UPPER>
__global__ void __launch_bounds__(256)
rs_fill(int64_t ns, int64_t nb_total, int64_t R, const int4* __restrict__ steps, const int32_t* __restrict__ order,
        const int32_t* __restrict__ step_of, const int32_t* __restrict__ nxt, const int64_t* __restrict__ bp,
        const int32_t* __restrict__ bcol, const int64_t* __restrict__ rp, const double* __restrict__ vals,
        const double* __restrict__ invd, unsigned char* __restrict__ stream) {
    constexpr int NIB = BS * (BS - 1) / 2;
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= ns) return;
    const int4 st = steps[s];
    unsigned char* base = stream + static_cast<int64_t>(static_cast<uint32_t>(st.x)) * 16;
    const int cnt = st.z;
    const int64_t p0 = st.w;
    int tot_nb = 0;
    for (int k = lane; k < cnt; k += 32) tot_nb += node_nb<BS, UPPER>(bp, order[p0 + k]);
    tot_nb = __reduce_add_sync(0xffffffffu, tot_nb);
    const int col0 = 4 * cnt;                                            // int32 units
    const int val0 = static_cast<int>((16 * cnt + al16(4 * static_cast<int64_t>(tot_nb))) / 8);  // double units
    int4* hdr = reinterpret_cast<int4*>(base);
    int32_t* ccol = reinterpret_cast<int32_t*>(base);
    double* cval = reinterpret_cast<double*>(base);
    // headers (chunks of 32 nodes, running offsets)
    int run_c = 0, run_v = 0;
    for (int k0 = 0; k0 < cnt; k0 += 32) {
        const int k = k0 + lane;
        const int nbk = k < cnt ? node_nb<BS, UPPER>(bp, order[p0 + k]) : 0;
        const int vk = k < cnt ? node_vals<BS>(nbk) : 0;
        int ic = nbk, iv = vk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, ic, o), b = __shfl_up_sync(0xffffffffu, iv, o);
            if (lane >= o) {
                ic += a;
                iv += b;
            }
        }
        if (k < cnt) hdr[k] = make_int4(order[p0 + k], nbk, col0 + run_c + ic - nbk, val0 + run_v + iv - vk);
        run_c += __shfl_sync(0xffffffffu, ic, 31);
        run_v += __shfl_sync(0xffffffffu, iv, 31);
    }
    __syncwarp();
    // per node: columns and values
    for (int k = 0; k < cnt; ++k) {
        const int4 h = hdr[k];
        const int64_t b = h.x;
        const int nbk = h.y;
        const int32_t sb = step_of[b];
        const int64_t rb = logical_of(b, nb_total, UPPER) / R;
        const int64_t c0 = node_col0<BS, UPPER>(bp, b);
        for (int n = lane; n < nbk; n += 32) {
            const int64_t nbr = bcol[c0 + n] / BS;
            const bool ring = logical_of(nbr, nb_total, UPPER) / R == rb && sb < nxt[nbr];
            const bool fresh = ring && step_of[nbr] == sb - 1;  // produced in the step just before
            ccol[h.z + n] = static_cast<int32_t>((nbr << 2) | (ring ? 1 : 0) | (fresh ? 2 : 0));
        }
        double* v = cval + h.w;
        for (int idx = lane; idx < BS * BS * nbk; idx += 32) {
            const int n = idx / (BS * BS), w = idx % (BS * BS), t = w / BS, c = w % BS;
            const int64_t row = b * BS + t;
            int64_t src;
            if (BS == 1) src = rp[row] + (UPPER ? 1 : 0) + n;
            else src = rp[row] + (UPPER ? (BS - t) : 0) + BS * n + c;
            v[idx] = vals[src];
        }
        if (lane == 0) {
            double* d = v + BS * BS * nbk;
            int q = 0;
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    if (!UPPER && c < t) d[q++] = vals[rp[b * BS + t + 1] - (t + 1) + c];
                    if (UPPER && c > t) d[q++] = vals[rp[b * BS + t] + (c - t)];
                }
#pragma unroll
            for (int t = 0; t < BS; ++t) d[NIB + t] = invd[b * BS + t];
        }
    }
}

// ------------------------------------------------------------ the sweep
__device__ __forceinline__ void bar_consumers(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_bulk_g2s_evict_first(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n\t}"
        ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

template <int BS>
constexpr int ring_slot_doubles() { return BS == 1 ? 1 : 4; }

// NCW consumer warps + 1 producer warp; LG lanes per node, lane gl owning
// neighbour blocks gl, gl + LG, ... (UR rounds held in registers; a node
// with more neighbours takes the extra rounds from the stage at use).
//
// Consumer pipeline: while step k's barrier is pending, each warp already
// holds step k+1's item in registers -- header, encoded columns, values,
// right-hand side, the diagonal block, every dependency finished two or
// more steps earlier (ring) and every dependency of another range (global,
// possibly still pending). After the barrier only the dependencies
// produced in step k (ring, "new" bit) remain to be read, so a step's
// critical path is: ring reads -> FMAs -> reduce -> solve -> publish.
template <int BS, int LG, int NCW, bool UPPER, bool PAD, bool TRACE = false>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
range_trsv_kernel(int64_t nranges, const int64_t* __restrict__ range_step, const int4* __restrict__ steps,
                  const unsigned char* __restrict__ stream, const double* rhs, double* out, double* reset,
                  const int* __restrict__ done, int buf_bytes, long long* trace, int exp) {
    static_assert(!PAD || BS == 3, "padded vectors hold 3-dof nodes");
    if (done && *done) return;
    constexpr int NW = NCW + 1, G = 32 / LG;
    constexpr int UR = LG >= 16 ? 1 : (LG >= 8 ? 2 : 4);
    constexpr int RS = PAD && UPPER ? 4 : BS;  // right-hand side stride per node
    constexpr int OS = PAD ? 4 : BS;           // output stride per node
    constexpr int NIB = BS * (BS - 1) / 2;
    constexpr int RSD = ring_slot_doubles<BS>();
    extern __shared__ __align__(128) unsigned char smem[];
    double* ring = reinterpret_cast<double*>(smem);
    unsigned char* buf = smem + kRing * RSD * sizeof(double);
    __shared__ uint64_t full[kStages], empty[kStages];
    __shared__ int spos[kStages], scnt[kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int j = 0; j < kStages; ++j) {
            mbar_init(&full[j], 1);
            mbar_init(&empty[j], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == NW - 1) {
        // ---- producer: one bulk copy per step, as far ahead as the stage
        // ring (bytes and mbarrier slots) allows
        if (lane != 0) return;
        int64_t k = 0, freed = 0;
        int head = 0;
        for (int64_t r = blockIdx.x; r < nranges; r += gridDim.x) {
            const int64_t s1 = range_step[r + 1];
            for (int64_t s = range_step[r]; s < s1; ++s, ++k) {
                const int4 st = steps[s];
                const int len = st.y * 16;
                int pos = 0;
                for (;;) {
                    const int64_t inflight = k - freed;
                    if (inflight < kStages) {
                        if (inflight == 0) {
                            pos = 0;
                            break;
                        }
                        const int tail = spos[freed % kStages];
                        if (head >= tail) {
                            if (head + len <= buf_bytes) {
                                pos = head;
                                break;
                            }
                            if (len < tail) {
                                pos = 0;
                                break;
                            }
                        } else if (head + len < tail) {
                            pos = head;
                            break;
                        }
                    }
                    mbar_wait(&empty[freed % kStages], static_cast<unsigned>((freed / kStages) & 1));
                    ++freed;
                }
                const int slot = static_cast<int>(k % kStages);
                spos[slot] = pos;
                scnt[slot] = st.z;
                head = pos + len;
                mbar_arrive_expect_tx(&full[slot], static_cast<unsigned>(len));
                tma_bulk_g2s_evict_first(buf + pos, stream + static_cast<int64_t>(static_cast<uint32_t>(st.x)) * 16,
                                         static_cast<unsigned>(len), &full[slot]);
            }
        }
        return;
    }
    // ---- consumers
    const int grp = lane / LG, gl = lane % LG;
    int64_t K = 0;
    for (int64_t r = blockIdx.x; r < nranges; r += gridDim.x) K += range_step[r + 1] - range_step[r];
    if (K == 0) return;
    // the warp's item of a step (node q = warp * G + grp)
    bool act = false;
    int64_t blk = 0;
    int nb = 0, cnt = 0;
    const unsigned char* base = nullptr;
    const uint32_t* cc = nullptr;
    const double* cv = nullptr;
    uint32_t code[UR];
    double a[UR][BS][BS], xv[UR][BS], rc[BS], bin[NIB > 0 ? NIB : 1], binv[BS];
    auto load_dep = [&](int64_t nbr, double (&v)[BS]) {
        if constexpr (PAD) {
            ld_relaxed_v4(out + 4 * nbr, v);
        } else {
#pragma unroll
            for (int c = 0; c < BS; ++c) v[c] = ld_relaxed(out + nbr * BS + c);
        }
    };
    auto ring_dep = [&](int64_t nbr, double (&v)[BS]) {
        const double* rs = ring + RSD * (nbr & (kRing - 1));
#pragma unroll
        for (int c = 0; c < BS; ++c) v[c] = rs[c];
    };
    auto load_rhs = [&](int64_t b, double (&v)[BS]) {
        if constexpr (RS == 4) {
            double d3 = 0.0;
            asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                         : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(d3)
                         : "l"(rhs + 4 * b));
            (void)d3;
        } else {
#pragma unroll
            for (int t = 0; t < BS; ++t) v[t] = rhs[b * BS + t];
        }
    };
    // item q of step kk into registers; the step's stage must have landed
    auto load_item = [&](int q) {
        act = q < cnt;
        const int4 h = act ? reinterpret_cast<const int4*>(base)[q] : make_int4(0, 0, 0, 0);
        blk = h.x;
        nb = h.y;
        cc = reinterpret_cast<const uint32_t*>(base) + h.z;
        cv = reinterpret_cast<const double*>(base) + h.w;
#pragma unroll
        for (int u = 0; u < UR; ++u) {
            const int n = u * LG + gl;
            const bool own = n < nb;
            code[u] = own ? cc[n] : 0u;
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) a[u][t][c] = own ? cv[BS * BS * n + BS * t + c] : 0.0;
#pragma unroll
            for (int c = 0; c < BS; ++c) xv[u][c] = 0.0;
            if (own) {
                if (!(code[u] & 1u)) {
                    if (TRACE && (exp & 2)) ring_dep(code[u] >> 2, xv[u]);
                    else load_dep(code[u] >> 2, xv[u]);
                }
                else if (!(code[u] & 2u)) ring_dep(code[u] >> 2, xv[u]);
            }
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) rc[t] = 0.0;
        if (act && gl == 0) {
            if (!(TRACE && (exp & 1))) load_rhs(blk, rc);
            const double* d = cv + BS * BS * nb;
#pragma unroll
            for (int j = 0; j < NIB; ++j) bin[j] = d[j];
#pragma unroll
            for (int t = 0; t < BS; ++t) binv[t] = d[NIB + t];
        }
    };
    auto wait_stage = [&](int64_t kk) {
        const int slot = static_cast<int>(kk % kStages);
        mbar_wait(&full[slot], static_cast<unsigned>((kk / kStages) & 1));
        cnt = scnt[slot];
        base = buf + spos[slot];
    };
    // finish the item in registers: new ring deps, pending polls, FMAs,
    // extra rounds, reduce, solve, publish
    auto finish_item = [&]() {
#pragma unroll
        for (int u = 0; u < UR; ++u)
            if (u * LG + gl < nb && (code[u] & 3u) == 3u) ring_dep(code[u] >> 2, xv[u]);
        bool pend = false;
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
            for (int c = 0; c < BS; ++c) pend |= u * LG + gl < nb && !(code[u] & 1u) && is_pending(xv[u][c]);
        if (TRACE && (exp & 2)) pend = false;
        while (__any_sync(0xffffffffu, pend)) {
            pend = false;
#pragma unroll
            for (int u = 0; u < UR; ++u) {
                bool pu = false;
#pragma unroll
                for (int c = 0; c < BS; ++c) pu |= u * LG + gl < nb && !(code[u] & 1u) && is_pending(xv[u][c]);
                if (pu) {
                    load_dep(code[u] >> 2, xv[u]);
#pragma unroll
                    for (int c = 0; c < BS; ++c) pend |= is_pending(xv[u][c]);
                }
            }
        }
        double acc[BS];
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = 0.0;
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) acc[t] = fma(a[u][t][c], xv[u][c], acc[t]);
        // neighbours beyond the register rounds, straight from the stage
        const int nbmax = __reduce_max_sync(0xffffffffu, nb);
        for (int n0 = LG * UR; n0 < nbmax; n0 += LG) {
            const int n = n0 + gl;
            const bool own = n < nb;
            const uint32_t cd = own ? cc[n] : 0u;
            double v[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) v[c] = 0.0;
            if (own) {
                if (cd & 1u) ring_dep(cd >> 2, v);
                else load_dep(cd >> 2, v);
            }
            bool pp = own && !(cd & 1u) && (is_pending(v[0]) || (BS > 1 && is_pending(v[BS - 1])) ||
                                             (BS > 2 && is_pending(v[1])));
            while (__any_sync(0xffffffffu, pp)) {
                if (pp) {
                    load_dep(cd >> 2, v);
                    pp = false;
#pragma unroll
                    for (int c = 0; c < BS; ++c) pp |= is_pending(v[c]);
                }
            }
#pragma unroll
            for (int t = 0; t < BS; ++t)
#pragma unroll
                for (int c = 0; c < BS; ++c) acc[t] = fma(own ? cv[BS * BS * n + BS * t + c] : 0.0, v[c], acc[t]);
        }
#pragma unroll
        for (int t = 0; t < BS; ++t) acc[t] = group_sum<LG>(acc[t]);
        if (act && gl == 0) {
            double xb[BS];
            solve_diag_block<BS, UPPER>(rc, acc, bin, binv, xb);
            double* rs = ring + RSD * (blk & (kRing - 1));
#pragma unroll
            for (int t = 0; t < BS; ++t) rs[t] = xb[t];
            if constexpr (PAD) {
                st_relaxed_v4(out + 4 * blk, xb[0], xb[1], xb[2], 0.0);
            } else {
#pragma unroll
                for (int t = 0; t < BS; ++t) st_relaxed(out + blk * BS + t, xb[t]);
            }
        }
        if (reset && act && gl < BS) reset[OS * blk + gl] = pending_value();
    };
    const int q0 = warp * G + grp;
    int64_t tr_r = blockIdx.x, ts = TRACE ? range_step[blockIdx.x] : 0;  // trace: global step of kk
    wait_stage(0);
    load_item(q0);
    for (int64_t kk = 0; kk < K; ++kk) {
        long long t0 = 0, t1 = 0;
        if (TRACE && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        finish_item();
        // items beyond one per lane group (steps wider than NCW * G nodes)
        for (int q = q0 + NCW * G; q - grp < cnt; q += NCW * G) {
            load_item(q);
#pragma unroll
            for (int u = 0; u < UR; ++u)  // every dependency of this step is visible: no "new" split
                if (u * LG + gl < nb && (code[u] & 3u) == 3u) ring_dep(code[u] >> 2, xv[u]);
            finish_item();
        }
        if (TRACE && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (kk + 1 < K) {
            wait_stage(kk + 1);
            load_item(q0);
        }
        bar_consumers(NCW * 32);
        if (threadIdx.x == 0) mbar_arrive(&empty[kk % kStages]);
        if (TRACE && threadIdx.x == 0) {
            long long t2;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
            long long* tr = trace + 8 * ts;
            tr[0] = t0;
            tr[1] = t1;
            tr[2] = t2;
        }
        if (TRACE && ++ts == range_step[tr_r + 1]) {
            tr_r += gridDim.x;
            if (tr_r < nranges) ts = range_step[tr_r];
        }
    }
}

// ------------------------------------------------------------ host side
int64_t max_dyn_smem() {
    static int v = 0;
    if (!v) {
        int dev = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    }
    return v;
}

template <int BS>
int64_t stage_bytes() {
    // dynamic shared memory = ring + stages; 1 KB left for the static part
    const int64_t ring = static_cast<int64_t>(kRing) * ring_slot_doubles<BS>() * 8;
    return ((max_dyn_smem() - 1024 - ring) / 16) * 16;
}

int64_t range_nodes_for(int64_t nb) {
    static const int64_t env = getenv("PCLAB_RANGE_NODES") ? atoll(getenv("PCLAB_RANGE_NODES")) : 0;
    if (env > 0) return env;
    const int64_t g = sm_count();
    return std::max<int64_t>(64, (nb + g - 1) / g);
}

template <int BS, bool UPPER>
void build_one(const Analysis& an, const Schedule& s, RangeSched& rs, cudaStream_t st) {
    const int64_t nb = s.nblocks;
    rs = RangeSched{};
    rs.upper = UPPER;
    rs.bs = BS;
    rs.nb = nb;
    if (nb == 0 || nb >= (1LL << 30)) return;
    const int64_t* bp = BS == 1 ? (UPPER ? an.upper.rp.p : an.lower.rp.p) : (UPPER ? an.ubc.bp.p : an.lbc.bp.p);
    const int64_t R = range_nodes_for(nb);
    rs.range_nodes = R;
    rs.nranges = (nb + R - 1) / R;
    // stream order: (range, level, node)
    DevBuf<unsigned long long> key(nb), skey(nb);
    DevBuf<int32_t> val(nb);
    rs.order.alloc(nb);
    rs_keys<<<gridn(nb, 256), 256, 0, st>>>(nb, UPPER, R, s.level.p, key.p, val.p);
    CK_LAUNCH();
    {
        int bits = 32;
        while (bits < 64 && (1LL << (bits - 32)) < rs.nranges) ++bits;
        radix_sort_pairs(key.p, skey.p, val.p, rs.order.p, nb, bits, st);
    }
    // groups
    DevBuf<int64_t> gid(nb + 1);
    rs_group_flags<<<gridn(nb + 1, 256), 256, 0, st>>>(nb, skey.p, gid.p);
    CK_LAUNCH();
    scan_inplace(gid.p, nb + 1, st);
    const int64_t ng = dev_read(gid.p + nb, st);
    DevBuf<int64_t> gfirst(ng + 1);
    rs_group_first<<<gridn(nb + 1, 256), 256, 0, st>>>(nb, skey.p, gid.p, gfirst.p);
    CK_LAUNCH();
    // steps
    const int64_t maxb = std::min<int64_t>(stage_bytes<BS>() / 3, 96 * 1024);
    DevBuf<int64_t> gsteps(ng + 1);
    DevBuf<int> bad(1);
    CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    CK(cudaMemsetAsync(gsteps.p + ng, 0, sizeof(int64_t), st));
    rs_split<BS, UPPER><<<gridn(ng, 128), 128, 0, st>>>(ng, gfirst.p, rs.order.p, bp, maxb, 0, gsteps.p, nullptr,
                                                        bad.p);
    CK_LAUNCH();
    if (dev_read(bad.p, st)) return;  // a node larger than a stage: round-robin sweep
    if (nb >= (1LL << 29)) return;     // node ids in 30-bit codes
    scan_inplace(gsteps.p, ng + 1, st);
    rs.nsteps = dev_read(gsteps.p + ng, st);
    rs.steps.alloc(rs.nsteps);
    rs_split<BS, UPPER><<<gridn(ng, 128), 128, 0, st>>>(ng, gfirst.p, rs.order.p, bp, maxb, 1, gsteps.p, rs.steps.p,
                                                        bad.p);
    CK_LAUNCH();
    DevBuf<int64_t> off(rs.nsteps + 1);
    rs_len_copy<<<gridn(rs.nsteps + 1, 256), 256, 0, st>>>(rs.nsteps, rs.steps.p, off.p);
    CK_LAUNCH();
    scan_inplace(off.p, rs.nsteps + 1, st);
    const int64_t tot16 = dev_read(off.p + rs.nsteps, st);
    if (tot16 >= (1LL << 32)) return;
    rs.stream_bytes = tot16 * 16;
    rs.max_step_bytes = maxb;
    rs_offsets<<<gridn(rs.nsteps, 256), 256, 0, st>>>(rs.nsteps, off.p, rs.steps.p);
    CK_LAUNCH();
    rs.range_step.alloc(rs.nranges + 1);
    rs.step_of.alloc(nb);
    rs_ranges<<<gridn(rs.nsteps + 1, 256), 256, 0, st>>>(rs.nsteps, nb, UPPER, R, rs.nranges, rs.steps.p,
                                                        rs.order.p, rs.range_step.p, rs.step_of.p);
    CK_LAUNCH();
    rs.nxt.alloc(nb);
    rs_next_writer<<<gridn(nb, 256), 256, 0, st>>>(nb, UPPER, R, rs.step_of.p, rs.nxt.p);
    CK_LAUNCH();
    rs.ok = true;
}

template <int BS, bool UPPER>
void fill_one(const Analysis& an, const RangeSched& rs, const double* vals, const double* invd,
              DevBuf<unsigned char>& stream, cudaStream_t st) {
    stream.alloc(rs.stream_bytes);
    const int64_t* bp = BS == 1 ? (UPPER ? an.upper.rp.p : an.lower.rp.p) : (UPPER ? an.ubc.bp.p : an.lbc.bp.p);
    const int32_t* bcol = BS == 1 ? (UPPER ? an.upper.cols.p : an.lower.cols.p)
                                  : (UPPER ? an.ubc.bcol.p : an.lbc.bcol.p);
    const int64_t* rp = UPPER ? an.upper.rp.p : an.lower.rp.p;
    rs_fill<BS, UPPER><<<gridn(rs.nsteps * 32, 256), 256, 0, st>>>(rs.nsteps, rs.nb, rs.range_nodes, rs.steps.p,
                                                                  rs.order.p, rs.step_of.p, rs.nxt.p, bp, bcol, rp,
                                                                  vals, invd, stream.p);
    CK_LAUNCH();
}

// developer trace (PCLAB_RANGE_TRACE=<file>): per step {wait start, stage
// ready, step done} globaltimer stamps of the stand-alone sweeps
long long* g_rtrace = nullptr;

template <int BS, int LG, int NCW, bool UPPER, bool PAD, bool TRACE>
void launch_tt(const RangeSched& rs, const unsigned char* stream, const double* b, double* x, double* reset,
               const int* done, cudaStream_t st) {
    const int64_t buf = stage_bytes<BS>();
    const int64_t smem = static_cast<int64_t>(kRing) * ring_slot_doubles<BS>() * 8 + buf;
    static bool set = false;
    auto kern = range_trsv_kernel<BS, LG, NCW, UPPER, PAD, TRACE>;
    if (!set) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        set = true;
    }
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(rs.nranges, sm_count()));
    kern<<<grid, (NCW + 1) * 32, smem, st>>>(rs.nranges, rs.range_step.p, rs.steps.p, stream, b, x, reset, done,
                                            static_cast<int>(buf), g_rtrace,
                                            getenv("PCLAB_RANGE_EXP") ? atoi(getenv("PCLAB_RANGE_EXP")) : 0);
    CK_LAUNCH();
}

template <int BS, int LG, int NCW, bool UPPER, bool PAD>
void launch_t(const RangeSched& rs, const unsigned char* stream, const double* b, double* x, double* reset,
              const int* done, cudaStream_t st) {
    if (g_rtrace) launch_tt<BS, LG, NCW, UPPER, PAD, true>(rs, stream, b, x, reset, done, st);
    else launch_tt<BS, LG, NCW, UPPER, PAD, false>(rs, stream, b, x, reset, done, st);
}

int range_lanes(int bs) {
    static const int env = getenv("PCLAB_RANGE_LG") ? atoi(getenv("PCLAB_RANGE_LG")) : 0;
    if (env > 0) return env;
    return bs == 3 ? 4 : 1;
}

template <int BS, bool UPPER, bool PAD>
void launch_bs(const RangeSched& rs, const unsigned char* stream, const double* b, double* x, double* reset,
               const int* done, cudaStream_t st) {
    if constexpr (BS == 3) {
        switch (range_lanes(3)) {
            case 16: launch_t<3, 16, 23, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
            case 17: launch_t<3, 16, 31, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
            case 8: launch_t<3, 8, 15, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
            default: launch_t<3, 4, 8, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
        }
    } else {
        switch (range_lanes(1)) {
            case 4: launch_t<1, 4, 15, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
            case 2: launch_t<1, 2, 8, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
            default: launch_t<1, 1, 8, UPPER, PAD>(rs, stream, b, x, reset, done, st); break;
        }
    }
}

}  // namespace

// Opt-in (PCLAB_RANGE=1): measured slower than the round-robin sweep on
// configs[2] (1.5 vs 0.82 ms per sweep; see DESIGN.md "Range-pipelined
// sweep"), kept for the measurements and its parity test.
bool range_sweeps_enabled() {
    static const bool on = getenv("PCLAB_RANGE") && atoi(getenv("PCLAB_RANGE")) != 0;
    return on;
}

void build_range_scheds(Analysis& an, cudaStream_t st) {
    an.rs_lo = RangeSched{};
    an.rs_up = RangeSched{};
    if (!range_sweeps_enabled()) return;
    if (an.bsr && an.bs == 3) {
        build_one<3, false>(an, an.blk_lo, an.rs_lo, st);
        build_one<3, true>(an, an.blk_up, an.rs_up, st);
    } else if (!an.bsr && an.bs == 1) {
        build_one<1, false>(an, an.blk_lo, an.rs_lo, st);
        build_one<1, true>(an, an.blk_up, an.rs_up, st);
    } else if (!an.bsr) {
        // scalar rows grouped in dense bs-row diagonal blocks (7-point
        // stencils detect bs = 2): the range sweep works on single rows, so
        // level the row DAG (level queue over one-row block columns)
        BlockCols lbc1, ubc1;
        build_block_cols(an.lower, 1, 0, lbc1, st);
        build_block_cols(an.upper, 1, 1, ubc1, st);
        Schedule lo1, up1;
        lo1.need_crit = up1.need_crit = false;
        compute_levels(an.lower, an.upper, 1, false, lo1, st, &lbc1, &ubc1);
        compute_levels(an.upper, an.lower, 1, true, up1, st, &ubc1, &lbc1);
        build_one<1, false>(an, lo1, an.rs_lo, st);
        build_one<1, true>(an, up1, an.rs_up, st);
    }
    if (!(an.rs_lo.ok && an.rs_up.ok)) {
        an.rs_lo = RangeSched{};
        an.rs_up = RangeSched{};
    }
}

void fill_range_streams(const Analysis& an, Precond& p, cudaStream_t st) {
    if (!an.rs_lo.ok) return;
    if (an.rs_lo.bs == 3) {
        fill_one<3, false>(an, an.rs_lo, p.lvals.p, p.invd.p, p.stream_lo, st);
        fill_one<3, true>(an, an.rs_up, p.uvals.p, p.invd.p, p.stream_up, st);
    } else {
        fill_one<1, false>(an, an.rs_lo, p.lvals.p, p.invd.p, p.stream_lo, st);
        fill_one<1, true>(an, an.rs_up, p.uvals.p, p.invd.p, p.stream_up, st);
    }
}

void range_trace_begin(const Analysis& an, bool upper, cudaStream_t st) {
    const RangeSched& rs = upper ? an.rs_up : an.rs_lo;
    if (!getenv("PCLAB_RANGE_TRACE") || !rs.ok) return;
    CK(cudaMallocAsync(&g_rtrace, sizeof(long long) * 8 * rs.nsteps, st));
}

void range_trace_end(const Analysis& an, bool upper, cudaStream_t st) {
    const RangeSched& rs = upper ? an.rs_up : an.rs_lo;
    if (!g_rtrace) return;
    std::vector<long long> t(8 * rs.nsteps);
    std::vector<int4> sv(rs.nsteps);
    std::vector<int64_t> rsx(rs.nranges + 1);
    CK(cudaMemcpyAsync(t.data(), g_rtrace, sizeof(long long) * t.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(sv.data(), rs.steps.p, sizeof(int4) * sv.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rsx.data(), rs.range_step.p, sizeof(int64_t) * rsx.size(), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaFree(g_rtrace));
    g_rtrace = nullptr;
    const std::string path = std::string(getenv("PCLAB_RANGE_TRACE")) + (upper ? ".up" : ".lo");
    FILE* f = fopen(path.c_str(), "wb");
    if (!f) return;
    const int64_t hdr[3] = {rs.nsteps, rs.nranges, rs.range_nodes};
    fwrite(hdr, sizeof hdr, 1, f);
    fwrite(t.data(), sizeof(long long), t.size(), f);
    fwrite(sv.data(), sizeof(int4), sv.size(), f);
    fwrite(rsx.data(), sizeof(int64_t), rsx.size(), f);
    fclose(f);
}

bool launch_range_trsv(const Analysis& an, const Precond& p, bool upper, const double* b, double* x, double* reset,
                       const int* done, cudaStream_t st, bool pad) {
    const RangeSched& rs = upper ? an.rs_up : an.rs_lo;
    const unsigned char* stream = upper ? p.stream_up.p : p.stream_lo.p;
    if (!rs.ok || !stream) return false;
    if (rs.bs == 3) {
        if (!pad) return false;
        if (upper) launch_bs<3, true, true>(rs, stream, b, x, reset, done, st);
        else launch_bs<3, false, true>(rs, stream, b, x, reset, done, st);
    } else {
        if (pad) return false;
        if (upper) launch_bs<1, true, false>(rs, stream, b, x, reset, done, st);
        else launch_bs<1, false, false>(rs, stream, b, x, reset, done, st);
    }
    return true;
}

}  // namespace pclab_b200
