// Shared device/host plumbing for the B200 PCG + IC(0) + GNN-correction path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

namespace pclab_b200 {

// ---------------------------------------------------------------- errors
// Mirrors the reference's exception taxonomy (error.hpp:8-29); the C-ABI
// folds these onto pclab_status exactly like capi.cpp:33-56.
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DimensionError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error in ") + what + " (" + file + ":" +
                        std::to_string(line) + "): " + cudaGetErrorString(e));
}
// Count of kernel launches issued by the library (CK_LAUNCH after each
// launch; graph replays add their node counts explicitly).
inline std::atomic<long long> g_launches{0};
inline void count_launches(long long k) { g_launches += k; }
inline long long launch_count() { return g_launches.load(); }

#define CK(x) ::pclab_b200::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH()                                                                         \
    do {                                                                                    \
        ::pclab_b200::count_launches(1);                                                    \
        ::pclab_b200::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
    } while (0)

// Number of SMs on the current device (148 on B200).
int sm_count();

// ------------------------------------------------------------ device bits
// "Not yet computed" marker for the sync-free solves and the IC(0)
// factorisation: a NaN whose two 32-bit halves are equal, so a plain
// 32-bit fill writes it. Real results never carry this payload (arithmetic
// NaNs are canonical 0x7ff8...).
constexpr unsigned long long kPending = 0x7FFA5A5A7FFA5A5AULL;
// Tiled sweep: bits of a packed block column that hold the distance back
// to a same-CTA dependency (TileSched::tcol).
constexpr int kTileDistBits = 10;
// Row broke down during IC(0): dependants consume it and produce NaN.
constexpr unsigned long long kBroken = 0x7FF8000000000000ULL;

#ifdef __CUDACC__
__device__ __forceinline__ double ld_relaxed(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double(static_cast<long long>(v));
}
__device__ __forceinline__ void st_relaxed(double* p, double x) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p),
                 "l"(static_cast<unsigned long long>(__double_as_longlong(x)))
                 : "memory");
}
// Streaming loads of matrix data (read once per sweep/SpMV): evict-first in
// L2 so the solution vectors the dependency gathers read stay resident.
#ifdef PCLAB_NO_EVICT_HINT
__device__ __forceinline__ double ld_stream(const double* p) { return __ldg(p); }
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldg(p); }
#else
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile(
        "{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "ld.global.nc.L2::cache_hint.f64 %0, [%1], pol;\n\t}"
        : "=d"(v)
        : "l"(p));
    return v;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
    int32_t v;
    asm volatile(
        "{\n\t.reg .b64 pol;\n\tcreatepolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "ld.global.nc.L2::cache_hint.s32 %0, [%1], pol;\n\t}"
        : "=r"(v)
        : "l"(p));
    return v;
}
#endif
// The high word alone identifies the marker: 0x7FFA5A5A is a NaN exponent
// with a payload arithmetic never produces (its NaNs are canonical 0x7FF8...),
// so one 32-bit compare per value instead of a 64-bit one.
__device__ __forceinline__ bool is_pending(double v) {
    return static_cast<unsigned>(__double2hiint(v)) == static_cast<unsigned>(kPending >> 32);
}
// Spin until the slot holds a computed value.
__device__ __forceinline__ double wait_value(const double* p) {
    double v = ld_relaxed(p);
    while (is_pending(v)) {
        __nanosleep(20);
        v = ld_relaxed(p);
    }
    return v;
}
__device__ __forceinline__ double pending_value() {
    return __longlong_as_double(static_cast<long long>(kPending));
}

template <int W>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, W);
    return v;
}

// Deterministic block reduction (fixed tree) of one double per thread.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* smem /* BLOCK/32 */) {
    v = group_sum<32>(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) smem[wid] = v;
    __syncthreads();
    double t = 0.0;
    if (wid == 0) {
        t = lane < BLOCK / 32 ? smem[lane] : 0.0;
        t = group_sum<32>(t);
    }
    __syncthreads();
    return t;  // valid in thread 0
}
#endif

}  // namespace pclab_b200
