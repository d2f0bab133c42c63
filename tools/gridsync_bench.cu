// Grid-barrier cost on one GPU: cooperative_groups grid.sync() vs a
// sense-reversing barrier (one atomic per CTA + one spinning thread), each
// followed by the fixed-order read of per-CTA partials that MGS does.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gsb tools/gridsync_bench.cu && /tmp/gsb
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* part) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        g.sync();
    }
}

__device__ __forceinline__ void bar_arrive_wait(unsigned* count, volatile unsigned* gen, unsigned nb,
                                                unsigned& mygen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = mygen;
        __threadfence();
        if (atomicAdd(count, 1u) == nb - 1) {
            *count = 0;
            __threadfence();
            atomicExch(const_cast<unsigned*>(gen), g0 + 1);
        } else {
            while (*gen == g0) {
            }
        }
        __threadfence();
    }
    ++mygen;
    __syncthreads();
}

__global__ void k_custom(int iters, double* part, unsigned* count, unsigned* gen) {
    unsigned mygen = *reinterpret_cast<volatile unsigned*>(gen);
    __syncthreads();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0) part[blockIdx.x] = i;
        bar_arrive_wait(count, gen, gridDim.x, mygen);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* part;
    unsigned *count, *gen;
    cudaMalloc(&part, 8 * 4096);
    cudaMalloc(&count, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(count, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {256, 1024}) {
        for (int iters : {1, 1001}) {
            void* args[] = {&iters, &part};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, sms, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("cg grid.sync   threads=%4d iters=%5d  %.3f ms  (%.2f us/iter)\n", threads, iters, ms,
                   1e3 * ms / iters);
            void* args2[] = {&iters, &part, &count, &gen};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_custom, sms, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("custom barrier threads=%4d iters=%5d  %.3f ms  (%.2f us/iter)  err=%s\n", threads, iters,
                   ms, 1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
