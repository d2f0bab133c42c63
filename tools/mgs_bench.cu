// Per-column cost of the resident-w MGS kernel (k_mgs_res) split into its
// parts: the full kernel, the reduction + grid barrier chain alone, and the
// column stream alone (no grid barrier). n = config 5 (2,097,152).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -Ipaper_2405_01599_b200/csrc -o tools/mgs_bench tools/mgs_bench.cu \
//     -Lpaper_2405_01599_b200/_lib -lktb -Xlinker -rpath=paper_2405_01599_b200/_lib
#include "../paper_2405_01599_b200/csrc/ktb_gmres.cu"

#include <cstdio>

namespace ktb {
template <int E>
__global__ void __launch_bounds__(kRThreads, 1) k_sync_only(int k, double2* slots, double* h,
                                                            long long tag0) {
    __shared__ double red[2 * kRThreads / 32];
    __shared__ double bc[2];
    const int nb = gridDim.x, tid = threadIdx.x;
    double c = tid;
    for (int q = 0; q < k; ++q) {
        double p = c * 1e-9, dummy = 0.0;
        block_sum_w0(p, dummy, red);
        double2* sl = slots + static_cast<int64_t>(q) * nb;
        if (tid == 0) publish(sl + blockIdx.x, p, tag0 + q);
        if (tid < 32) {
            const double t = poll_total(sl, nb, tag0 + q);
            if (tid == 0) bc[0] = t;
        }
        __syncthreads();
        c = bc[0];
    }
    if (blockIdx.x == 0 && tid == 0) h[0] = c;
}

template <int E>
__global__ void __launch_bounds__(kRThreads, 1) k_stream_only(const double* __restrict__ V,
                                                              int64_t n, int k, double* h) {
    extern __shared__ double s_v[];
    const int tid = threadIdx.x;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * E * kRThreads + tid;
    double wr[E], p = 0.0;
    for (int e = 0; e < E; ++e) wr[e] = 1.0, s_v[e * kRThreads + tid] = 0.0;
    for (int q = 1; q < k; ++q) {
        const double* Vc = V + static_cast<int64_t>(q) * n;
        double vn[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
            vn[e] = i < n ? __ldcg(Vc + i) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
            wr[e] = __dadd_rn(wr[e], __dmul_rn(-1e-9, s_v[e * kRThreads + tid]));
            s_v[e * kRThreads + tid] = vn[e];
            p += vn[e] * wr[e];
        }
        __syncthreads();
    }
    if (p == 12345.0) h[0] = p;
}
}  // namespace ktb

int main() {
    using namespace ktb;
    const int64_t n = 2097152;
    constexpr int E = 14;
    const int m = 31;
    double *V, *w, *vn, *h;
    double2* part;
    int* brk;
    cudaMalloc(&V, 8 * n * m);
    cudaMalloc(&w, 8 * n);
    cudaMalloc(&vn, 8 * n);
    cudaMalloc(&h, 8 * 64);
    cudaMalloc(&part, 16 * 64 * 256);
    cudaMemset(part, 0, 16 * 64 * 256);
    long long tag = 64;
    cudaMalloc(&brk, 4);
    cudaMemset(V, 0, 8 * n * m);
    cudaMemset(w, 0, 8 * n);
    const int nb = static_cast<int>((n + E * kRThreads - 1) / (E * kRThreads));
    const size_t smem = E * kRThreads * 8;
    cudaFuncSetAttribute(k_mgs_res<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * smem));
    cudaFuncSetAttribute(k_stream_only<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int k : {1, 16, 30}) {
        float t[3];
        for (int rep = 0; rep < 2; ++rep) {
            int kk = k;
            int64_t nn = n;
            void* args[] = {&V, &nn, &kk, &w, &vn, &h, &part, &brk, &tag};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_mgs_res<E>, nb, kRThreads, args, 2 * smem, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[0], a, b);
            tag += 64;
            void* args2[] = {&kk, &part, &h, &tag};
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_sync_only<E>, nb, kRThreads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[1], a, b);
            tag += 64;
            cudaEventRecord(a);
            k_stream_only<E><<<nb, kRThreads, smem>>>(V, n, k, h);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[2], a, b);
        }
        printf("k=%2d  full %.1f us   sync-chain only %.1f us   column stream only %.1f us  (%s)\n", k,
               1e3 * t[0], 1e3 * t[1], 1e3 * t[2], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
