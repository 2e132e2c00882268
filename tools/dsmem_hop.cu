// Developer microbenchmark for DESIGN's next step: the publication -> observation
// hop when the consumer polls its OWN shared memory and the producer writes it
// through the cluster's distributed shared memory (st.shared::cluster), against
// the L2 hop of tools/pingpong2.cu (289 ns idle, 350-560 ns under load). CTA
// pairs (rank 0 <-> rank `far`) of every cluster bounce a counter; optionally
// the other warps of every CTA stream a buffer larger than L2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dsmem_hop tools/dsmem_hop.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned cluster_addr(const void* smem_ptr, unsigned rank) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem_ptr)), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_remote4(unsigned addr, double v) {
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1,%1};" ::"r"(addr), "d"(v) : "memory");
    asm volatile("st.shared::cluster.v2.f64 [%0], {%1,%1};" ::"r"(addr + 16), "d"(v) : "memory");
}
__device__ __forceinline__ double ld_local(const volatile double* p) { return p[3]; }  // the last word written

template <int CS>
__global__ void __launch_bounds__(512, 1)
hop(int rounds, long long* out, const int4* buf, long long nvec, int nstream, int far, int* sink,
    volatile int* finished, int npairs) {
    __shared__ double box[4];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    if (threadIdx.x == 0) box[0] = box[1] = box[2] = box[3] = 0.0;
    cl.sync();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        if (lane == 0 && (rank == 0 || rank == static_cast<unsigned>(far))) {
            const unsigned peer = rank == 0 ? far : 0;
            const unsigned remote = cluster_addr(box, peer);
            long long g0 = 0, g1;
            for (int r = 1; r <= rounds; ++r) {
                if (r == 11) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
                if (rank == 0) {
                    st_remote4(remote, static_cast<double>(r));
                    while (ld_local(box) != static_cast<double>(r)) {}
                } else {
                    while (ld_local(box) != static_cast<double>(r)) {}
                    st_remote4(remote, static_cast<double>(r));
                }
            }
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            if (rank == 0) {
                out[blockIdx.x / CS] = g1 - g0;
                atomicAdd(const_cast<int*>(finished), 1);
            }
        }
    } else if (warp <= nstream) {  // every SM streams until every pair is through
        int acc = 0;
        const long long per = nvec / (static_cast<long long>(gridDim.x) * nstream);
        const int4* p = buf + (static_cast<long long>(blockIdx.x) * nstream + (warp - 1)) * per;
        while (*finished < npairs) {
            for (long long i = lane; i + 7 * 32 < per && *finished < npairs; i += 8 * 32) {
                int4 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + 32 * u);
#pragma unroll
                for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].w;
            }
        }
        if (acc == 0x12345678) *sink = acc;
    }
    cl.sync();  // nobody leaves while a peer may still write its shared memory
}

template <int CS>
void run(int rounds, long long* out, const int4* buf, long long nvec, int* sink, int* finished) {
    const int grid = (148 / CS) * CS;
    for (int far : {1, CS - 1}) {
        if (far == 1 && CS == 2 && false) continue;
        for (int ns : {0, 4, 15}) {
            cudaMemset(finished, 0, sizeof(int));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(512);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = CS;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (CS > 8) cudaFuncSetAttribute(hop<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaError_t e = cudaLaunchKernelEx(&cfg, hop<CS>, rounds, out, buf, nvec, ns, far, sink,
                                               static_cast<volatile int*>(finished), grid / CS);
            if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
                printf("cluster %d: launch failed (%s)\n", CS, cudaGetErrorString(cudaGetLastError()));
                return;
            }
            std::vector<double> h;
            for (int c = 0; c < grid / CS; ++c) h.push_back(double(out[c]) / (rounds - 10) / 2.0);
            std::sort(h.begin(), h.end());
            printf("cluster of %2d, ranks 0 <-> %2d, %2d streaming warps/SM: hop ns min %.0f median %.0f max %.0f (%zu pairs)\n", CS,
                   far, ns, h.front(), h[h.size() / 2], h.back(), h.size());
        }
        if (CS == 2) break;
    }
}

int main() {
    const int rounds = 3010;
    long long* out;
    int* sink;
    int4* buf;
    const long long bytes = 4LL << 30, nvec = bytes / 16;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    cudaMalloc(&sink, 4);
    cudaMallocManaged(&out, 512 * sizeof(long long));
    int* finished;
    cudaMalloc(&finished, sizeof(int));
    run<2>(rounds, out, buf, nvec, sink, finished);
    run<8>(rounds, out, buf, nvec, sink, finished);
    run<16>(rounds, out, buf, nvec, sink, finished);
    return 0;
}
