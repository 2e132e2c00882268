// Developer microbenchmark: one-way handoff latency between two warps
// (a) on different SMs through L2 (st/ld .relaxed.gpu), (b) in one CTA
// through shared memory (volatile). Prints ns per one-way hop.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pp_global(volatile unsigned long long* flag, int iters, long long* out) {
    const int me = blockIdx.x;  // 0 or 1, different SMs (grid 2 x 32 threads, 1 block/SM forced by smem)
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (int i = 0; i < iters; ++i) {
        if (me == 0) {
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            } while (v != 2ULL * i);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(2ULL * i + 1) : "memory");
        } else {
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            } while (v != 2ULL * i + 1);
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(flag), "l"(2ULL * i + 2) : "memory");
        }
    }
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    if (me == 0) out[0] = t_end - t_start, out[1] = clock64() - t0;
}

__global__ void pp_shared(int iters, long long* out) {
    __shared__ volatile unsigned long long flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) != 0 || w > 1) return;
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    for (int i = 0; i < iters; ++i) {
        if (w == 0) {
            while (flag != 2ULL * i) {
            }
            flag = 2ULL * i + 1;
        } else {
            while (flag != 2ULL * i + 1) {
            }
            flag = 2ULL * i + 2;
        }
    }
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    if (w == 0) out[2] = t_end - t_start;
}

int main() {
    unsigned long long* flag;
    long long* out;
    cudaMalloc(&flag, 8);
    cudaMalloc(&out, 64);
    const int iters = 20000;
    long long h[4];
    cudaFuncSetAttribute(pp_global, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(flag, 0, 8);
        pp_global<<<2, 32, 200 * 1024>>>(flag, iters, out);
        pp_shared<<<1, 64>>>(iters, out);
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("global one-way hop: %.1f ns (%.0f cycles); shared one-way hop: %.1f ns\n",
               h[0] / (2.0 * iters), h[1] / (2.0 * iters), h[2] / (2.0 * iters));
    }
    return 0;
}
