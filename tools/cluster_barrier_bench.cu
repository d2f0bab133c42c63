// Per-level cost of a cluster-wide sweep step (ILU apply): cluster barrier
// alone, + cluster-scope fence, + one L2 gather/store round per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cluster_barrier_bench tools/cluster_barrier_bench.cu
#include <cstdio>

template <int MODE>
__global__ void k(double* z, int levels, int n) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int nthr = gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int l = 0; l < levels; ++l) {
        if (MODE >= 2) {
            const int i = (g * 7 + l * 131) % n;
            acc += __ldcg(z + i);
            __stcg(z + (g + l * nthr) % n, acc);
        }
        if (MODE >= 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (acc == 12345.0) z[0] = acc;
}

template <int MODE>
float run(int cs, int threads, double* z, int levels, int n) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k<MODE>, z, levels, n);
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k<MODE>, z, levels, n);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return 1e3f * ms / levels;
}

int main() {
    const int n = 1 << 21, levels = 2000;
    double* z;
    cudaMalloc(&z, 8 * n);
    cudaMemset(z, 0, 8 * n);
    for (int cs : {1, 4, 8, 16})
        for (int th : {256, 1024}) {
            const float t0 = run<0>(cs, th, z, levels, n);
            const float t1 = run<1>(cs, th, z, levels, n);
            const float t2 = run<2>(cs, th, z, levels, n);
            printf("cluster %2d x %4d threads: barrier %.2f us, +fence %.2f us, +gather/store %.2f us (%s)\n",
                   cs, th, t0, t1, t2, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
