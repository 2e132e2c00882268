// Developer microbenchmark: the sweeps' hop (256-bit relaxed publication seen by
// a 256-bit relaxed poll on another SM) measured on 74 SM pairs at once, idle
// and while the other warps of every SM stream a buffer larger than L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/pingpong2 tools/pingpong2.cu
//   build/pingpong2 [streaming warps per SM = 0,4,8,15]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void st4(double* p, double a) {
    asm volatile("st.relaxed.gpu.global.v4.f64 [%0], {%1,%1,%1,%1};" ::"l"(p), "d"(a) : "memory");
}
__device__ __forceinline__ double ld4(const double* p) {
    double a, b, c, d;
    asm volatile("ld.relaxed.gpu.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p) : "memory");
    return a + b + c + d;
}

// CTA b and CTA b ^ 1 bounce a counter (warp 0, lane 0); warps 1..nstream stream `buf`
__global__ void __launch_bounds__(512, 1)
pp(double* slots, int rounds, long long* out, const int4* buf, long long nvec, int nstream, int* sink, int stride) {
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane != 0) return;
        const int me = blockIdx.x, other = blockIdx.x ^ 1;
        double* mine = slots + static_cast<long long>(stride) * me;
        double* theirs = slots + static_cast<long long>(stride) * other;
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        long long g0, g1;
        // handshake so both sides are running
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        for (int r = 1; r <= rounds; ++r) {
            if (r == 11) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
            if ((me & 1) == 0) {
                st4(mine, static_cast<double>(r));
                while (ld4(theirs) != 4.0 * r) {}
            } else {
                while (ld4(theirs) != 4.0 * r) {}
                st4(mine, static_cast<double>(r));
            }
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
        out[2 * me] = g1 - g0;
        out[2 * me + 1] = smid;
        done = 1;
        return;
    }
    if (warp > nstream) return;
    int acc = 0;
    const long long per = nvec / (gridDim.x * nstream);
    const int4* p = buf + (static_cast<long long>(blockIdx.x) * nstream + (warp - 1)) * per;
    while (!done) {
        for (long long i = lane; i + 7 * 32 < per && !done; i += 8 * 32) {
            int4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].w;
        }
    }
    if (acc == 0x12345678) *sink = acc;
}

int main(int argc, char** argv) {
    const int rounds = 3010;
    double* slots;
    long long* out;
    int* sink;
    int4* buf;
    const long long bytes = 4LL << 30, nvec = bytes / 16;
    cudaMalloc(&slots, 1 << 22);
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    cudaMalloc(&sink, 4);
    cudaMallocManaged(&out, 512 * sizeof(long long));
    for (int stride : {32, 4096 + 32}) {
        for (int ns : {0, 2, 4, 8, 15}) {
            cudaMemset(slots, 0, 1 << 22);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            pp<<<148, 512>>>(slots, rounds, out, buf, nvec, ns, sink, stride);
            cudaEventRecord(e1);
            if (cudaDeviceSynchronize() != cudaSuccess) {
                printf("kernel failed\n");
                return 1;
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<double> hop;
            for (int b = 0; b < 148; b += 2) hop.push_back(double(out[2 * b]) / (rounds - 10) / 2.0);
            std::sort(hop.begin(), hop.end());
            printf("slot stride %4d doubles, %2d streaming warps/SM: hop ns min %.0f p25 %.0f median %.0f p75 %.0f max %.0f (kernel %.2f ms)\n",
                   stride, ns, hop.front(), hop[hop.size() / 4], hop[hop.size() / 2], hop[3 * hop.size() / 4], hop.back(), ms);
            if (ns == 0 && stride == 32) {
                printf("  pairs (sm, sm, hop ns):");
                for (int b = 0; b < 148; b += 2) printf(" (%lld,%lld,%.0f)", out[2 * b + 1], out[2 * b + 3], double(out[2 * b]) / (rounds - 10) / 2.0);
                printf("\n");
            }
        }
    }
    return 0;
}
