// ktb_vec.cu -- device BLAS-1 building blocks of the distributed Krylov loop
// (GMRES over row-sharded vectors, NCCL all-reduce of
// the local partial dots). Reference arithmetic: dot / axpy / scal in
// common.hpp:33-56, the orthogonalisation passes of ortho.hpp:55-111.
//
// Every reduction is deterministic: a fixed grid of kVecBlocks blocks, each
// thread striding over its elements, a fixed-shape block tree, and one
// ordered pass over the block partials. The multi-vector forms work on a
// column-major basis V (column j at V + j*ldv).
#include "ktb_internal.cuh"
#include "ktb_ptx.cuh"

namespace ktb {

namespace {

constexpr int kVecThreads = 256;
constexpr int kVecBlocks = 2 * kNumSMs;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    KTB_SYNC();  // sh reused across calls
    if (lane == 0) sh[warp] = v;
    KTB_SYNC();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < kVecThreads / 32; ++k) s += sh[k];
    return s;  // valid in thread 0
}

// partial[j * gridDim.x + b] = sum over block b's elements of V_j[i] * w[i]
__global__ void __launch_bounds__(kVecThreads) k_mdot_partial(int64_t n, int k,
                                                              const double* __restrict__ V,
                                                              int64_t ldv,
                                                              const double* __restrict__ w,
                                                              double* __restrict__ partial) {
    __shared__ double sh[kVecThreads / 32];
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kVecThreads;
    for (int j = 0; j < k; ++j) {
        const double* q = V + j * ldv;
        double s = 0.0;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(kVecThreads) + threadIdx.x; i < n;
             i += stride)
            s += q[i] * w[i];
        s = block_sum(s, sh);
        if (threadIdx.x == 0) partial[static_cast<int64_t>(j) * gridDim.x + blockIdx.x] = s;
    }
}

__global__ void k_mdot_final(int k, int nb, const double* __restrict__ partial,
                             double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= k) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[static_cast<int64_t>(j) * nb + b];
    out[j] = s;
}

// w[i] += alpha * coef[j] * V_j[i], j ascending (= k successive axpy calls)
__global__ void k_maxpy(int64_t n, int k, const double* __restrict__ V, int64_t ldv,
                        const double* __restrict__ coef, double alpha, double* __restrict__ w) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride) {
        double acc = w[i];
        for (int j = 0; j < k; ++j) acc += (alpha * coef[j]) * V[j * ldv + i];
        w[i] = acc;
    }
}

__global__ void k_axpby(int64_t n, double a, const double* x, double b, double* y) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride)
        y[i] = a * x[i] + b * y[i];
}

// x[i] *= s (scal, common.hpp) or x[i] /= s (gmres.hpp:85 basis[i] = r[i] / beta)
__global__ void k_scale(int64_t n, double s, int divide, double* __restrict__ x) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += stride)
        x[i] = divide ? x[i] / s : x[i] * s;
}

int grid_for(int64_t n) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ceil_div64(n, 256), 8 * kNumSMs)));
}

}  // namespace

int64_t vec_mdot_scratch(int k) { return static_cast<int64_t>(k) * kVecBlocks; }

void vec_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* out,
              double* scratch, cudaStream_t s) {
    require(n >= 0 && k >= 0 && ldv >= n, "vec: bad dimensions");
    require(k == 0 || scratch != nullptr, "vec: mdot needs scratch");
    if (k == 0) return;
    k_mdot_partial<<<kVecBlocks, kVecThreads, 0, s>>>(n, k, V, ldv, w, scratch);
    KTB_LAUNCH();
    k_mdot_final<<<ceil_div(k, 32), 32, 0, s>>>(k, kVecBlocks, scratch, out);
    KTB_LAUNCH();
}

void vec_maxpy(int64_t n, int k, const double* V, int64_t ldv, const double* coef, double alpha,
               double* w, cudaStream_t s) {
    require(n >= 0 && k >= 0 && ldv >= n, "vec: bad dimensions");
    if (k == 0 || n == 0) return;
    k_maxpy<<<grid_for(n), 256, 0, s>>>(n, k, V, ldv, coef, alpha, w);
    KTB_LAUNCH();
}

void vec_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s) {
    require(n >= 0, "vec: bad dimensions");
    if (n == 0) return;
    k_axpby<<<grid_for(n), 256, 0, s>>>(n, a, x, b, y);
    KTB_LAUNCH();
}

void vec_scale(int64_t n, double sc, int divide, double* x, cudaStream_t s) {
    require(n >= 0, "vec: bad dimensions");
    if (n == 0) return;
    k_scale<<<grid_for(n), 256, 0, s>>>(n, sc, divide, x);
    KTB_LAUNCH();
}

}  // namespace ktb
