// Accuracy of the GNN kernels' branch-free tanh (csrc/gnn_math.cuh) against
// the CUDA library's, on the device: 2^24 points of [-24, 24], 2^20 tiny
// arguments and the special values. Prints the largest absolute difference;
// exit status 1 above 1e-14.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tanh_check tools/tanh_check.cu
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2412_07127_b200/csrc/gnn_math.cuh"

__global__ void check(long long n, double* maxerr, int* bad) {
    double worst = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double x;
        if (i < (1LL << 24)) x = -24.0 + 48.0 * (double)i / (double)(1LL << 24);
        else x = ((i & 1) ? -1.0 : 1.0) * exp2(-60.0 + 58.0 * (double)(i - (1LL << 24)) / (double)(1LL << 20));
        const double e = fabs(pclab_b200::tanh_nb(x) - tanh(x));
        worst = fmax(worst, e);
    }
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)maxerr, (unsigned long long)__double_as_longlong(worst));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const double inf = __longlong_as_double(0x7ff0000000000000LL);
        const double nan = __longlong_as_double(0x7ff8000000000000LL);
        int b = 0;
        b |= pclab_b200::tanh_nb(inf) != 1.0;
        b |= pclab_b200::tanh_nb(-inf) != -1.0;
        b |= !(pclab_b200::tanh_nb(nan) != pclab_b200::tanh_nb(nan));
        b |= pclab_b200::tanh_nb(0.0) != 0.0;
        b |= pclab_b200::tanh_nb(700.0) != 1.0;
        *bad = b;
    }
}

int main() {
    double* d;
    int* bad;
    cudaMallocManaged(&d, sizeof(double));
    cudaMallocManaged(&bad, sizeof(int));
    *d = 0.0;
    *bad = 0;
    check<<<1184, 256>>>((1LL << 24) + (1LL << 20), d, bad);
    if (cudaDeviceSynchronize() != cudaSuccess) {
        printf("kernel failed\n");
        return 2;
    }
    printf("tanh_nb vs tanh: max abs difference %.3e, special values %s\n", *d, *bad ? "WRONG" : "ok");
    return (*d < 1e-14 && !*bad) ? 0 : 1;
}
