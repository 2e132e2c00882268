// Hand-written device scan and radix sort for the set-up path (symbolic
// analysis, level schedules, COO -> CSR): the building blocks CUB supplied
// in round 1.
//
// scan_inplace: exclusive prefix sum of int64, three phases (tile sums ->
// scan of the tile sums, recursive -> tile-local scans plus offsets), one
// 1024-element tile per 256-thread CTA.
//
// radix_sort_pairs: stable LSD radix sort, 8-bit digits. Per pass:
//   1. per-tile digit histograms, stored digit-major (hist[d * ntiles + t]),
//   2. one exclusive scan over them -> every (digit, tile) output base,
//   3. scatter: a tile's items are ranked in tile order (8 striped rounds of
//      256; inside a round, warps rank by __match_any_sync and the warps of
//      the CTA add up in warp order), so equal digits keep their order.
#include <cstdint>

#include "core.h"

namespace pclab_b200 {

namespace {

constexpr int kScanT = 256, kScanItems = 4, kScanTile = kScanT * kScanItems;
constexpr int kSortT = 256, kSortItems = 8, kSortTile = kSortT * kSortItems, kRadix = 256;

inline unsigned gridn(int64_t n, int64_t t) { return static_cast<unsigned>((n + t - 1) / t); }

// inclusive scan of one value per thread across the CTA (256 threads)
__device__ __forceinline__ int64_t block_inclusive_scan(int64_t v, int64_t* warp_sums /* 8 */, int64_t& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    int64_t off = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kScanT / 32; ++w) {
        const int64_t s = warp_sums[w];
        if (w < wid) off += s;
        tot += s;
    }
    __syncthreads();
    total = tot;
    return v + off;
}

__global__ void __launch_bounds__(kScanT) scan_tile_sums(const int64_t* __restrict__ p, int64_t n,
                                                         int64_t* __restrict__ sums) {
    __shared__ int64_t ws[kScanT / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
    int64_t s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        const int64_t i = base + j * kScanT + threadIdx.x;
        if (i < n) s += p[i];
    }
    int64_t tot;
    block_inclusive_scan(s, ws, tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_tile_apply(int64_t* __restrict__ p, int64_t n,
                                                          const int64_t* __restrict__ offs) {
    __shared__ int64_t ws[kScanT / 32];
    // blocked items: thread t owns tile positions t*4 .. t*4+3
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
    int64_t v[kScanItems], s = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = base + j < n ? p[base + j] : 0;
        s += v[j];
    }
    int64_t tot;
    const int64_t incl = block_inclusive_scan(s, ws, tot);
    int64_t run = incl - s + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n) p[base + j] = run;
        run += v[j];
    }
}

// ---------------------------------------------------------------- radix
template <class K>
__device__ __forceinline__ unsigned digit_of(K k, int shift) {
    return static_cast<unsigned>((k >> shift) & static_cast<K>(kRadix - 1));
}

template <class K>
__global__ void __launch_bounds__(kSortT) radix_hist(const K* __restrict__ keys, int64_t n, int shift,
                                                     int64_t ntiles, int64_t* __restrict__ hist) {
    __shared__ int h[kRadix];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSortTile;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int64_t i = base + j * kSortT + threadIdx.x;
        if (i < n) atomicAdd(&h[digit_of(keys[i], shift)], 1);
    }
    __syncthreads();
    hist[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <class K, class V>
__global__ void __launch_bounds__(kSortT) radix_scatter(const K* __restrict__ kin, K* __restrict__ kout,
                                                        const V* __restrict__ vin, V* __restrict__ vout, int64_t n,
                                                        int shift, int64_t ntiles,
                                                        const int64_t* __restrict__ offs) {
    constexpr int NW = kSortT / 32;
    __shared__ int cnt[NW][kRadix];
    __shared__ int64_t run[kRadix];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    run[threadIdx.x] = offs[static_cast<int64_t>(threadIdx.x) * ntiles + blockIdx.x];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kSortTile;
    const unsigned lt = (1u << lane) - 1u;
    for (int j = 0; j < kSortItems; ++j) {
#pragma unroll
        for (int w = 0; w < NW; ++w) cnt[w][threadIdx.x] = 0;
        __syncthreads();
        const int64_t i = base + j * kSortT + threadIdx.x;
        const bool ok = i < n;
        K k{};
        V v{};
        unsigned d = kRadix;  // out-of-range items take a digit no one else has
        if (ok) {
            k = kin[i];
            v = vin[i];
            d = digit_of(k, shift);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt);
        if (ok && rank == 0) cnt[wid][d] = __popc(peers);
        __syncthreads();
        if (ok) {
            int before = 0;
            for (int w = 0; w < wid; ++w) before += cnt[w][d];
            const int64_t pos = run[d] + before + rank;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncthreads();
        int tot = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) tot += cnt[w][threadIdx.x];
        run[threadIdx.x] += tot;
        __syncthreads();
    }
}

}  // namespace

void scan_inplace(int64_t* p, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles == 1) {
        scan_tile_apply<<<1, kScanT, 0, st>>>(p, n, nullptr);
        CK_LAUNCH();
        return;
    }
    DevBuf<int64_t> sums(tiles);
    scan_tile_sums<<<static_cast<unsigned>(tiles), kScanT, 0, st>>>(p, n, sums.p);
    CK_LAUNCH();
    scan_inplace(sums.p, tiles, st);
    scan_tile_apply<<<static_cast<unsigned>(tiles), kScanT, 0, st>>>(p, n, sums.p);
    CK_LAUNCH();
}

template <class K, class V>
void radix_sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, int bits, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t ntiles = (n + kSortTile - 1) / kSortTile;
    DevBuf<int64_t> hist(ntiles * kRadix);
    DevBuf<K> kt(n);
    DevBuf<V> vt(n);
    const int passes = (bits + 7) / 8;
    // ping-pong so the last pass lands in (kout, vout)
    const K* ks = kin;
    const V* vs = vin;
    for (int pass = 0; pass < passes; ++pass) {
        const bool to_out = ((passes - 1 - pass) % 2) == 0;
        K* kd = to_out ? kout : kt.p;
        V* vd = to_out ? vout : vt.p;
        radix_hist<K><<<static_cast<unsigned>(ntiles), kSortT, 0, st>>>(ks, n, 8 * pass, ntiles, hist.p);
        CK_LAUNCH();
        scan_inplace(hist.p, ntiles * kRadix, st);
        radix_scatter<K, V><<<static_cast<unsigned>(ntiles), kSortT, 0, st>>>(ks, kd, vs, vd, n, 8 * pass, ntiles,
                                                                            hist.p);
        CK_LAUNCH();
        ks = kd;
        vs = vd;
    }
    if (passes == 0) {
        CK(cudaMemcpyAsync(kout, kin, sizeof(K) * n, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(vout, vin, sizeof(V) * n, cudaMemcpyDeviceToDevice, st));
    }
}

template void radix_sort_pairs<uint32_t, int32_t>(const uint32_t*, uint32_t*, const int32_t*, int32_t*, int64_t, int,
                                                  cudaStream_t);
template void radix_sort_pairs<unsigned long long, int32_t>(const unsigned long long*, unsigned long long*,
                                                            const int32_t*, int32_t*, int64_t, int, cudaStream_t);
template void radix_sort_pairs<unsigned long long, int64_t>(const unsigned long long*, unsigned long long*,
                                                            const int64_t*, int64_t*, int64_t, int, cudaStream_t);

}  // namespace pclab_b200
