// Random-gather ceiling for config 3 (tool, not product): how fast can the
// B200 serve uniformly random 8-byte x[col] gathers when x (32 MB, config 3's
// 4M doubles) is L2-resident, and what does an SpMV-shaped stream (int32
// column + fp64 value per nonzero, x gathered at the column, one sum per 8
// nonzeros) reach with the same random columns? The second number is the
// ceiling an SpMV kernel over config 3's uniform columns can approach; the
// U1/U2/U3 kernels are judged against it next to the HBM roofline.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_bench tools/gather_bench.cu
//   tools/gather_bench [n_x=4000000] [nnz=39552727]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t mix(uint64_t z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return static_cast<uint32_t>(z ^ (z >> 31));
}

__global__ void k_fill_cols(int32_t* col, int64_t nnz, uint32_t nx) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz;
         i += int64_t(gridDim.x) * blockDim.x)
        col[i] = static_cast<int32_t>(mix(i) % nx);
}

// (1) pure gathers: G independent random loads per thread in flight
template <int G>
__global__ void k_gather(const double* __restrict__ x, uint32_t nx, int64_t total, double* out) {
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x * G;
    for (int64_t base = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * G; base < total;
         base += stride) {
        double v[G];
#pragma unroll
        for (int g = 0; g < G; ++g) v[g] = __ldg(x + mix(base + g) % nx);
#pragma unroll
        for (int g = 0; g < G; ++g) acc += v[g];
    }
    if (acc == 12345.678) out[0] = acc;
}

// (2) SpMV-shaped: coalesced int32 col + fp64 val stream, x gathered at col,
// each thread sums 8 consecutive nonzeros (a row of config 3's mean length)
__global__ void k_spmv_like(const int32_t* __restrict__ col, const double* __restrict__ val,
                            const double* __restrict__ x, int64_t nnz, double* __restrict__ y) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t b = t * 8;
    if (b >= nnz) return;
    int32_t c[8];
    double v[8], xv[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        c[k] = b + k < nnz ? __ldcs(col + b + k) : 0;
        v[k] = b + k < nnz ? __ldcs(val + b + k) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) xv[k] = __ldg(x + c[k]);
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k] * xv[k];
    y[t] = s;
}

int main(int argc, char** argv) {
    const uint32_t nx = argc > 1 ? static_cast<uint32_t>(atoll(argv[1])) : 4000000u;
    const int64_t nnz = argc > 2 ? atoll(argv[2]) : 39552727;
    double *x, *val, *y, *out;
    int32_t* col;
    cudaMalloc(&x, 8ull * nx);
    cudaMalloc(&val, 8ull * nnz);
    cudaMalloc(&col, 4ull * nnz);
    cudaMalloc(&y, 8ull * (nnz / 8 + 1));
    cudaMalloc(&out, 8);
    cudaMemset(x, 0, 8ull * nx);
    cudaMemset(val, 0, 8ull * nnz);
    k_fill_cols<<<2048, 256>>>(col, nnz, nx);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto launch, int reps) {
        launch();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        return best;
    };
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int occ : {4, 8, 16}) {
        const int grid = sms * occ;
        const float ms = time([&] { k_gather<8><<<grid, 256>>>(x, nx, nnz, out); }, 20);
        printf("pure random gathers (x %u doubles, L2-resident), %d CTAs x 256, 8 in flight: "
               "%.1f us for %lld gathers = %.1f G gathers/s (%.0f GB/s of 32-B sectors)\n",
               nx, grid, ms * 1e3, (long long)nnz, nnz / (ms * 1e-3) / 1e9,
               nnz * 32.0 / (ms * 1e-3) / 1e9);
    }
    const int64_t threads = (nnz + 7) / 8;
    const float ms = time([&] {
        k_spmv_like<<<static_cast<int>((threads + 255) / 256), 256>>>(col, val, x, nnz, y);
    }, 20);
    const double bytes = 12.0 * nnz + 8.0 * nx + 8.0 * threads;
    printf("SpMV-shaped stream (col+val coalesced, random x gather, 8 nnz per thread): %.1f us "
           "for %lld nnz = %.1f G nnz/s, %.0f GB/s of streamed+x+y bytes\n",
           ms * 1e3, (long long)nnz, nnz / (ms * 1e-3) / 1e9, bytes / (ms * 1e-3) / 1e9);
    return 0;
}
