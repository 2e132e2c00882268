// Developer microbenchmark: one-way latency of a 256-bit relaxed publication
// observed by a 256-bit relaxed poll on another SM (the sweeps' hop), and
// the post-arrival chain of a sweep item (9 FMAs, a 16-lane shuffle tree of
// three sums, the 3x3 diagonal solve, the store).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/pingpong tools/pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st4(double* p, double a) {
    asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(p), "d"(a) : "memory");
}
__device__ __forceinline__ double ld4(const double* p) {
    double a, b, c, d;
    asm volatile("ld.relaxed.gpu.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
    return a + b + c + d;
}

// CTA 0 and CTA 1 (lane 0 each) bounce a counter through two 32-byte slots
__global__ void pingpong(double* slots, int rounds, long long* out) {
    if (threadIdx.x != 0) return;
    double* mine = slots + 4 * 8 * blockIdx.x;          // 256 B apart
    double* theirs = slots + 4 * 8 * (1 - blockIdx.x);
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    long long t0 = clock64();
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    for (int r = 1; r <= rounds; ++r) {
        if (blockIdx.x == 0) {
            st4(mine, static_cast<double>(r));
            while (ld4(theirs) != 4.0 * r) {}
        } else {
            while (ld4(theirs) != 4.0 * r) {}
            st4(mine, static_cast<double>(r));
        }
    }
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    out[3 * blockIdx.x] = clock64() - t0;
    out[3 * blockIdx.x + 1] = g1 - g0;
    out[3 * blockIdx.x + 2] = smid;
}

template <int LG>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
    for (int o = LG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o, LG);
    return v;
}

// the post-arrival chain, repeated dependently
__global__ void chain(const double* in, double* out, int reps, long long* cyc) {
    const int lane = threadIdx.x & 31;
    double a[9];
    for (int j = 0; j < 9; ++j) a[j] = in[lane * 9 + j];
    double x[3] = {in[300], in[301], in[302]};
    const double b0 = in[303], b1 = in[304], b2 = in[305], i0 = in[306], i1 = in[307], i2 = in[308];
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        double acc[3] = {0.0, 0.0, 0.0};
        for (int t = 0; t < 3; ++t)
            for (int c = 0; c < 3; ++c) acc[t] = fma(a[3 * t + c], x[c], acc[t]);
        for (int t = 0; t < 3; ++t) acc[t] = gsum<16>(acc[t]);
        const double s0 = (1.0 - acc[0]) * i0;
        const double s1 = (1.0 - acc[1] - b0 * s0) * i1;
        const double s2 = (1.0 - acc[2] - b1 * s0 - b2 * s1) * i2;
        x[0] = s0 * 1e-3;
        x[1] = s1 * 1e-3;
        x[2] = s2 * 1e-3;
    }
    cyc[threadIdx.x] = clock64() - t0;
    out[threadIdx.x] = x[0] + x[1] + x[2];
}

int main() {
    double* slots;
    long long* out;
    cudaMalloc(&slots, 4096);
    cudaMemset(slots, 0, 4096);
    cudaMallocManaged(&out, 64 * sizeof(long long));
    const int rounds = 20000;
    for (int trial = 0; trial < 3; ++trial) {
        cudaMemset(slots, 0, 4096);
        pingpong<<<2, 32>>>(slots, rounds, out);
        cudaDeviceSynchronize();
        printf("pingpong: round trip %.1f cycles, %.1f ns (SMs %lld, %lld)\n", double(out[0]) / rounds,
               double(out[1]) / rounds, out[2], out[5]);
    }
    double* in;
    double* o;
    cudaMallocManaged(&in, 512 * sizeof(double));
    cudaMalloc(&o, 64 * sizeof(double));
    for (int i = 0; i < 512; ++i) in[i] = 0.001 * (i % 17);
    chain<<<1, 32>>>(in, o, 10000, out);
    cudaDeviceSynchronize();
    printf("item chain: %.1f cycles per dependent repetition\n", double(out[0]) / 10000);
    return 0;
}
