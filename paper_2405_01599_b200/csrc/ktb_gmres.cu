// ktb_gmres.cu -- device-resident restarted GMRES(m) with modified
// Gram-Schmidt (config 5 consumer; reference gmres.hpp:16-173 with
// OrthoKind::mgs, ortho.hpp:69-111, identity preconditioner, x0 = 0).
//
// Vectors (basis V of m+1 columns, w, r, x, b) live in HBM; the SpMV is the
// caller's plan. The scalar recurrence (Givens rotations, residual estimate,
// back-substitution) runs on the host exactly as the reference writes it,
// fed by device-computed projections. Orthogonalisation is one cooperative
// kernel per Arnoldi step: per column q it applies w -= h_q V_q and, in the
// same pass, accumulates the next projection <V_{q+1}, w> (or |w|^2 after the
// last column), with a deterministic fixed-order grid reduction between
// passes. Element-wise updates use explicitly rounded mul/add so each element
// follows the reference's arithmetic; only the dot-product summation order
// differs (parallel tree instead of serial), hence the iteration count can
// move by a step or two.
#include <cooperative_groups.h>

#include <chrono>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "ktb_internal.cuh"
#include "ktb_ptx.cuh"

namespace cg = cooperative_groups;

namespace ktb {

constexpr int kGThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    KTB_SYNC();
    if (l == 0) red[w] = v;
    KTB_SYNC();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < kGThreads / 32; ++k) s += red[k];
    return s;  // valid in thread 0
}

// Fixed-order sum of the per-block partials (every thread gets the same).
__device__ __forceinline__ double grid_total(const double* partials, int nb) {
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partials[b];
    return s;
}

__global__ void __launch_bounds__(kGThreads) k_mgs(const double* __restrict__ V, int64_t n,
                                                   int k, double* __restrict__ w,
                                                   double* __restrict__ vnext,
                                                   double* __restrict__ h,
                                                   double* __restrict__ partials,
                                                   int* __restrict__ breakdown) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double red[kGThreads / 32];
    const int nb = gridDim.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    volatile double* vp = partials;
    // input norm^2 and the first projection <V_0, w>
    double a = 0.0, b = 0.0;
    for (int64_t i = t0; i < n; i += stride) {
        const double wi = w[i];
        a += wi * wi;
        b += V[i] * wi;
    }
    a = block_sum(a, red);
    b = block_sum(b, red);
    if (threadIdx.x == 0) {
        vp[blockIdx.x] = a;
        vp[nb + blockIdx.x] = b;
    }
    grid.sync();
    const double in2 = grid_total(partials, nb);
    double c = grid_total(partials + nb, nb);
    int slot = 0;  // alternate partial buffers between passes
    for (int q = 0; q < k; ++q) {
        if (blockIdx.x == 0 && threadIdx.x == 0) h[q] = c;
        const double* Vq = V + static_cast<int64_t>(q) * n;
        const bool last = q + 1 == k;
        const double* Vn = last ? nullptr : V + static_cast<int64_t>(q + 1) * n;
        const double mc = -c;
        double p = 0.0;
        for (int64_t i = t0; i < n; i += stride) {
            const double wi = __dadd_rn(w[i], __dmul_rn(mc, Vq[i]));  // axpy(-c, q, v)
            w[i] = wi;
            p += last ? wi * wi : Vn[i] * wi;
        }
        p = block_sum(p, red);
        if (threadIdx.x == 0) vp[(slot ^ 1) * nb * 2 + blockIdx.x] = p;
        grid.sync();
        slot ^= 1;
        c = grid_total(partials + slot * nb * 2, nb);
    }
    // c = |w|^2 after the last column
    const double nrm = sqrt(c);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        h[k] = nrm;
        *breakdown = nrm <= 1e-14 * sqrt(in2) ? 1 : 0;
    }
    if (!(nrm <= 1e-14 * sqrt(in2))) {
        const double inv = 1.0 / nrm;  // scal(1.0 / r.norm, v)
        for (int64_t i = t0; i < n; i += stride) vnext[i] = __dmul_rn(w[i], inv);
    }
}

// ---- MGS with w resident on chip --------------------------------------------
// The same projections, update arithmetic and breakdown test as k_mgs, but
// w never goes back to HBM inside the step: one CTA of kRThreads per SM owns
// a contiguous slice of E * kRThreads elements, w's slice lives in registers
// (E per thread) and the slice of the next column in shared memory. Per
// column q the pass is: w_i -= h_q * V_q,i (V_q from shared memory, loaded by
// the previous pass), load V_{q+1} (the only HBM traffic: one basis column
// per projection) into the same shared slot, accumulate <V_{q+1}, w>. The grid
// reduction is fixed-order and computed identically by every CTA (one warp
// reads the per-CTA partials in order + a fixed shuffle tree), so every CTA
// sees the same h_q bit for bit.
#ifndef KTB_MGS_THREADS
#define KTB_MGS_THREADS 1024  // 512 (E up to 32) measured equal
#endif
constexpr int kRThreads = KTB_MGS_THREADS;

// Cross-CTA exchange without a grid barrier: CTA b publishes its partial of
// reduction r as one 16-byte (value, tag) store into slot[r * nb + b], the
// tag being unique to this launch and reduction; warp 0 of every CTA polls
// the nb slots until each carries the expected tag (16-byte stores and loads
// of one aligned pair are seen whole, the property CUB's decoupled look-back
// relies on), then sums them in a fixed order + a fixed shuffle tree, so
// every CTA obtains the same total bit for bit. One L2 round trip after the
// last CTA's store replaces barrier + re-read.
constexpr int kMaxPart = 8;  // nb <= 256

__device__ __forceinline__ void publish(double2* slot, double v, long long tag) {
    KTB_CHAOS_DELAY(0x7075);
    __stcg(slot, make_double2(v, __longlong_as_double(tag)));
}

// warp 0 only; returns the total in every lane of warp 0
__device__ __forceinline__ double poll_total(const double2* slot, int nb, long long tag) {
    const int lane = threadIdx.x & 31;
    double acc[kMaxPart];
    unsigned pending = 0;
#pragma unroll
    for (int m = 0; m < kMaxPart; ++m) {
        acc[m] = 0.0;
        if (lane + 32 * m < nb) pending |= 1u << m;
    }
    while (pending) {
        KTB_CHAOS_DELAY(0x706f);
#pragma unroll
        for (int m = 0; m < kMaxPart; ++m) {
            if ((pending >> m) & 1u) {
                const double2 v = __ldcv(slot + lane + 32 * m);
                if (__double_as_longlong(v.y) == tag) {
                    acc[m] = v.x;
                    pending &= ~(1u << m);
                }
            }
        }
    }
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < kMaxPart; ++m) t += acc[m];
    __syncwarp();
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

// block sum of a (and b) into warp 0 (every lane of warp 0 holds the sums)
__device__ __forceinline__ void block_sum_w0(double& a, double& b, double* red) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[2 * w] = a;
        red[2 * w + 1] = b;
    }
    KTB_SYNC();
    if (threadIdx.x < 32) {
        a = l < blockDim.x / 32 ? red[2 * l] : 0.0;
        b = l < blockDim.x / 32 ? red[2 * l + 1] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
    }
}

// slots: (k + 2) * nb pairs; tag0: unique per launch (the host advances it
// by 64 each launch), tags tag0 + r for reductions r = 0..k+1
// issue point pinned (volatile asm is not moved across the exchange below)
__device__ __forceinline__ double ld_cg_pinned(const double* p) {
    double r;
    asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

template <int E>
__global__ void __launch_bounds__(kRThreads, 1) k_mgs_res(const double* __restrict__ V, int64_t n,
                                                          int k, const double* __restrict__ w,
                                                          double* __restrict__ vnext,
                                                          double* __restrict__ h,
                                                          double2* __restrict__ slots,
                                                          int* __restrict__ breakdown,
                                                          long long tag0) {
    // this CTA's slices: w and the current column (E * kRThreads each)
    extern __shared__ double smem_d[];
    double* s_w = smem_d;
    double* s_v = smem_d + E * kRThreads;
    __shared__ double red[2 * kRThreads / 32];
    __shared__ double bc[2];
    const int nb = gridDim.x, tid = threadIdx.x;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * E * kRThreads + tid;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
        const double wi = i < n ? w[i] : 0.0;
        const double v = i < n ? V[i] : 0.0;
        s_w[e * kRThreads + tid] = wi;
        s_v[e * kRThreads + tid] = v;
        a += wi * wi;
        b += v * wi;
    }
    // V_{q+1} is loaded one pass ahead into registers (its latency overlaps
    // the exchange of the previous projection) and pulled into L2 two passes
    // ahead
    double vn[E];
    auto load_col = [&](int col) {
        const double* Vc = V + static_cast<int64_t>(col) * n;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
            vn[e] = i < n ? ld_cg_pinned(Vc + i) : 0.0;
        }
    };
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * E * kRThreads;
    const int64_t s1 = min(n, s0 + static_cast<int64_t>(E) * kRThreads);
    auto prefetch_col = [&](int col) {  // column starts are only 8-byte aligned for odd n
        const double* c0 = V + static_cast<int64_t>(col) * n;
        if (tid == 0 && s1 > s0) prefetch_l2_range(c0 + s0, c0 + s1);
    };
    if (k > 1) load_col(1);
    if (k > 2) prefetch_col(2);
    if (k > 3) prefetch_col(3);
    block_sum_w0(a, b, red);
    if (tid == 0) {
        publish(slots + blockIdx.x, a, tag0);
        publish(slots + nb + blockIdx.x, b, tag0 + 1);
    }
    if (tid < 32) {
        const double t0 = poll_total(slots, nb, tag0);
        const double t1 = poll_total(slots + nb, nb, tag0 + 1);
        if (tid == 0) {
            bc[0] = t0;
            bc[1] = t1;
        }
    }
    KTB_SYNC();
    const double in2 = bc[0];
    double c = bc[1];
    for (int q = 0; q < k; ++q) {
        if (blockIdx.x == 0 && tid == 0) h[q] = c;
        const bool last = q + 1 == k;
        const double mc = -c;
        double p = 0.0, dummy = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int o = e * kRThreads + tid;
            const double wi = __dadd_rn(s_w[o], __dmul_rn(mc, s_v[o]));  // axpy(-c, q, v)
            s_w[o] = wi;
            if (last) {
                p += wi * wi;
            } else {
                s_v[o] = vn[e];
                p += vn[e] * wi;
            }
        }
        if (q + 2 < k) load_col(q + 2);
        if (q + 4 < k) prefetch_col(q + 4);
        block_sum_w0(p, dummy, red);
        double2* sl = slots + static_cast<int64_t>(q + 2) * nb;
        if (tid == 0) publish(sl + blockIdx.x, p, tag0 + q + 2);
        if (tid < 32) {
            const double t = poll_total(sl, nb, tag0 + q + 2);
            if (tid == 0) bc[0] = t;
        }
        KTB_SYNC();
        c = bc[0];
    }
    const double nrm = sqrt(c);
    const bool brk = nrm <= 1e-14 * sqrt(in2);
    if (blockIdx.x == 0 && tid == 0) {
        h[k] = nrm;
        *breakdown = brk ? 1 : 0;
    }
    if (!brk) {
        const double inv = 1.0 / nrm;  // scal(1.0 / r.norm, v)
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
            if (i < n) vnext[i] = __dmul_rn(s_w[e * kRThreads + tid], inv);
        }
    }
}

// Exchange of k_mgs_dma (tools/exchange_bench.cu, 148 CTAs: 1.6 us per
// exchange instead of 2.7 us for the layout above): one slot per 128-byte line
// (stores of different SMs into one line serialise in L2), the <= 8 slot loads
// of a lane's poll round in flight together, and three rows of slots reused
// by every reduction of every launch -- row 2 for the input norm, rows 0 / 1
// alternating for the projections (a CTA rewrites a row for reduction r + 2
// only after its poll of r + 1 completed, i.e. after every CTA finished
// reading r). Same summation order as poll_total.
constexpr int kLineSlots = 8;  // double2 per 128-byte line
constexpr int kPollParts = 5;  // nb <= 160 (one CTA per SM)
__device__ __forceinline__ double2 ld_relaxed_pair(const double2* p) {
    double2 v;
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
// warp 0 only; returns the total in every lane of warp 0
__device__ __forceinline__ double poll_total_lines(const double2* row, int nb, long long tag) {
    const int lane = threadIdx.x & 31;
    double2 v[kPollParts];
    bool ok;
    do {
        KTB_CHAOS_DELAY(0x706c);
#pragma unroll
        for (int m = 0; m < kPollParts; ++m)
            if (32 * m < nb) v[m] = ld_relaxed_pair(row + min(lane + 32 * m, nb - 1) * kLineSlots);
        ok = true;
#pragma unroll
        for (int m = 0; m < kPollParts; ++m)
            if (32 * m < nb) ok = ok && __double_as_longlong(v[m].y) == tag;
    } while (!__all_sync(0xffffffffu, ok));
    double t = 0.0;
#pragma unroll
    for (int m = 0; m < kPollParts; ++m)
        if (32 * m < nb) t += lane + 32 * m < nb ? v[m].x : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

// ---- MGS with w in registers and the basis columns fed by bulk copies --------
// The same slices, element-to-thread mapping, update arithmetic, reduction
// trees and exchange as k_mgs_res (bit-identical projections), but w's slice
// stays in registers (E per thread) and the basis columns arrive in two
// shared-memory buffers by one bulk copy each (cp.async.bulk + mbarrier):
// column q+1 is requested as soon as the pass over column q-1's buffer is
// done, i.e. before this CTA publishes projection q, so its HBM time overlaps
// the cross-CTA exchange instead of following it, and a pass is two
// shared-memory reads per element (update from column q, product with column
// q+1) with no shared-memory stores. Needs even n (16-byte aligned column
// slices) and 2 * E * kRThreads * 8 bytes of shared memory (E <= 14).
template <int E>
__global__ void __launch_bounds__(kRThreads, 1) k_mgs_dma(const double* __restrict__ V, int64_t n,
                                                          int k, const double* __restrict__ w,
                                                          double* __restrict__ vnext,
                                                          double* __restrict__ h,
                                                          double2* __restrict__ slots,
                                                          int* __restrict__ breakdown,
                                                          long long tag0) {
    extern __shared__ __align__(128) double smem_d[];
    constexpr int kSlice = E * kRThreads;
    double* buf0 = smem_d;
    double* buf1 = smem_d + kSlice;
    __shared__ double red[2 * kRThreads / 32];
    __shared__ double bc[2];
    __shared__ __align__(8) uint64_t full[2];
    const int nb = gridDim.x, tid = threadIdx.x;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * kSlice;
    const int len = static_cast<int>(max(int64_t(0), min(n - s0, static_cast<int64_t>(kSlice))));
    const int64_t base = s0 + tid;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int col) {  // thread 0: column col's slice into buffer col & 1
        if (len > 0) {
            mbar_arrive_expect_tx(&full[col & 1], static_cast<uint32_t>(len) * 8u);
            tma_load_1d((col & 1) ? buf1 : buf0, V + static_cast<int64_t>(col) * n + s0,
                        static_cast<uint32_t>(len) * 8u, &full[col & 1], pol);
        }
    };
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        fence_mbar_init();
    }
    // the slice's tail past n (last CTA) reads as zero in both buffers
    for (int o = len + tid; o < kSlice; o += kRThreads) buf0[o] = buf1[o] = 0.0;
    KTB_SYNC();
    if (tid == 0) {
        fence_proxy_async_smem();
        issue(0);
        if (k > 1) issue(1);
    }
    double wr[E];
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
        wr[e] = i < n ? w[i] : 0.0;
    }
    if (len > 0) mbar_wait(&full[0], 0);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        a += wr[e] * wr[e];
        b += buf0[e * kRThreads + tid] * wr[e];
    }
    block_sum_w0(a, b, red);
    const int rowlen = nb * kLineSlots;  // rows 0 / 1: projections, row 2: the input norm
    if (tid == 0) {
        publish(slots + 2 * rowlen + blockIdx.x * kLineSlots, a, tag0);
        publish(slots + rowlen + blockIdx.x * kLineSlots, b, tag0 + 1);
    }
    if (tid < 32) {
        const double t0 = poll_total_lines(slots + 2 * rowlen, nb, tag0);
        const double t1 = poll_total_lines(slots + rowlen, nb, tag0 + 1);
        if (tid == 0) {
            bc[0] = t0;
            bc[1] = t1;
        }
    }
    KTB_SYNC();
    const double in2 = bc[0];
    double c = bc[1];
    for (int q = 0; q < k; ++q) {
        if (blockIdx.x == 0 && tid == 0) h[q] = c;
        const bool last = q + 1 == k;
        const double mc = -c;
        const double* cur = (q & 1) ? buf1 : buf0;
        const double* nxt = (q & 1) ? buf0 : buf1;
        // column q+1 is the ((q+1) >> 1)-th fill of its buffer
        if (!last && len > 0) mbar_wait(&full[(q + 1) & 1], ((q + 1) >> 1) & 1);
        double p = 0.0, dummy = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int o = e * kRThreads + tid;
            const double wi = __dadd_rn(wr[e], __dmul_rn(mc, cur[o]));  // axpy(-c, q, v)
            wr[e] = wi;
            p += last ? wi * wi : nxt[o] * wi;
        }
        // block_sum_w0, split: after its barrier every thread has read column
        // q's buffer, which thread 0 then refills with column q+2
        for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
        if ((tid & 31) == 0) {
            red[2 * (tid >> 5)] = p;
            red[2 * (tid >> 5) + 1] = dummy;
        }
        KTB_SYNC();
        if (tid == 0 && q + 2 < k) {
            fence_proxy_async_smem();
            issue(q + 2);
        }
        double2* sl = slots + (q & 1) * rowlen;
        if (tid < 32) {
            p = tid < kRThreads / 32 ? red[2 * tid] : 0.0;
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            if (tid == 0) publish(sl + blockIdx.x * kLineSlots, p, tag0 + q + 2);
            const double t = poll_total_lines(sl, nb, tag0 + q + 2);
            if (tid == 0) bc[0] = t;
        }
        KTB_SYNC();
        c = bc[0];
    }
    const double nrm = sqrt(c);
    const bool brk = nrm <= 1e-14 * sqrt(in2);
    if (blockIdx.x == 0 && tid == 0) {
        h[k] = nrm;
        *breakdown = brk ? 1 : 0;
    }
    if (!brk) {
        const double inv = 1.0 / nrm;  // scal(1.0 / r.norm, v)
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int64_t i = base + static_cast<int64_t>(e) * kRThreads;
            if (i < n) vnext[i] = __dmul_rn(wr[e], inv);
        }
    }
}

__global__ void k_sub_from(const double* __restrict__ b, double* __restrict__ r, int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) r[i] = __dsub_rn(b[i], r[i]);
}

__global__ void k_div(const double* __restrict__ r, double beta, double* __restrict__ v,
                      int64_t n) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) v[i] = __ddiv_rn(r[i], beta);
}

__global__ void __launch_bounds__(kGThreads) k_sumsq(const double* __restrict__ r, int64_t n,
                                                     double* __restrict__ partials) {
    __shared__ double red[kGThreads / 32];
    double a = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = r[i];
        a += v * v;
    }
    a = block_sum(a, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = a;
}

// x += sum_l y_l V_l with the reference's per-element order (w = 0; w += y_l
// V_l for l ascending; x += 1.0 * w), gmres.hpp:138-143.
__global__ void k_update_x(const double* __restrict__ V, const double* __restrict__ y, int j,
                           int64_t n, double* __restrict__ x) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int l = 0; l < j; ++l) acc = __dadd_rn(acc, __dmul_rn(y[l], V[static_cast<int64_t>(l) * n + i]));
    x[i] = __dadd_rn(x[i], __dmul_rn(1.0, acc));
}

// x += 1.0 * z (gmres.hpp:142 axpy(1.0, z, res.x))
__global__ void k_add_z(const double* __restrict__ z, int64_t n, double* __restrict__ x) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) x[i] = __dadd_rn(x[i], __dmul_rn(1.0, z[i]));
}

}  // namespace ktb

namespace ktb {

struct GmresWork {
    int64_t n, m;
    bool prec;
    int nb, res_nb;
    DBuf<double> b, x, r, w, V, zp, partials, dy;
    DBuf<double2> slots;  // k_mgs_res exchange: (m + 2) reductions x CTAs
    long long tag = 64;
    PinnedBuf<double> h_pin;
    PinnedBuf<int> brk_pin;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> ev_s, ev_e, ev_step;
    GmresWork(int64_t n_, int64_t m_, bool prec_, int nb_, int res_nb_)
        : n(n_), m(m_), prec(prec_), nb(nb_), res_nb(res_nb_), b(n_), x(n_), r(n_), w(n_),
          V(static_cast<size_t>(n_) * (m_ + 1)), zp(prec_ ? n_ : 1), partials(4 * nb_),
          dy(m_ + 1),
          slots(std::max(static_cast<size_t>(m_ + 3), static_cast<size_t>(3 * kLineSlots)) *
                std::max(res_nb_, 1)),
          h_pin(static_cast<size_t>(m_ + 1) * (m_ + 2)), brk_pin(m_ + 1), ev_s(m_ + 1),
          ev_e(m_ + 1), ev_step(m_ + 1) {
        KTB_CUDA(cudaEventCreate(&ev0));
        KTB_CUDA(cudaEventCreate(&ev1));
        for (int64_t q = 0; q <= m_; ++q) {
            KTB_CUDA(cudaEventCreate(&ev_s[q]));
            KTB_CUDA(cudaEventCreate(&ev_e[q]));
            KTB_CUDA(cudaEventCreateWithFlags(&ev_step[q], cudaEventDisableTiming));
        }
    }
    ~GmresWork() {
        for (auto e : {ev0, ev1})
            if (e) cudaEventDestroy(e);
        for (auto* v : {&ev_s, &ev_e, &ev_step})
            for (auto e : *v)
                if (e) cudaEventDestroy(e);
    }
    GmresWork(const GmresWork&) = delete;
    GmresWork& operator=(const GmresWork&) = delete;
};

// Restarted GMRES(m), MGS, x0 = 0 (gmres.hpp:16-173); host b/x spans. P:
// optional ILU(0) right preconditioner (Precond, solver_types.hpp:22-27).
void gmres_run(ktb_plan* A, ktb_ilu* P, const double* b_host, double* x_host, int64_t m,
               double tol, int64_t max_iters, double* history, ktb_gmres_result* res) {
        require(A != nullptr && res != nullptr, "gmres: null argument");
        require(m >= 1, "gmres: need 1 <= m <= m_max");  // gmres.hpp:20
        require(tol > 0.0, "gmres: tol must be positive");  // gmres.hpp:21
        const ktb_matrix* M = A->m;
        require(M->n == M->ncols, "gmres: dimension mismatch");
        DeviceGuard g(M->device);
        const auto t_start = std::chrono::steady_clock::now();
        const int64_t n = M->n;
        cudaStream_t st = A->stream;
        *res = ktb_gmres_result{};
        int dev = 0, sms = 0, per_sm = 0;
        KTB_CUDA(cudaGetDevice(&dev));
        KTB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mgs, kGThreads, 0));
        require(per_sm >= 1, "gmres: cooperative MGS kernel does not fit");
        const int nb = sms * std::min(per_sm, 2);
        // resident-w MGS: one CTA per SM holds E * kRThreads elements
        const int64_t per_cta = ceil_div64(n, static_cast<int64_t>(sms) * kRThreads);
        int E = 0;
        for (int e : {1, 2, 4, 8, 12, 14, 16, 24, 28, 32})
            if (e >= per_cta) {
                E = e;
                break;
            }
        const void* res_fn = nullptr;
        switch (E) {
            case 1: res_fn = reinterpret_cast<const void*>(&k_mgs_res<1>); break;
            case 2: res_fn = reinterpret_cast<const void*>(&k_mgs_res<2>); break;
            case 4: res_fn = reinterpret_cast<const void*>(&k_mgs_res<4>); break;
            case 8: res_fn = reinterpret_cast<const void*>(&k_mgs_res<8>); break;
            case 12: res_fn = reinterpret_cast<const void*>(&k_mgs_res<12>); break;
            case 14: res_fn = reinterpret_cast<const void*>(&k_mgs_res<14>); break;
            case 16: res_fn = reinterpret_cast<const void*>(&k_mgs_res<16>); break;
            case 24: res_fn = reinterpret_cast<const void*>(&k_mgs_res<24>); break;
            case 28: res_fn = reinterpret_cast<const void*>(&k_mgs_res<28>); break;
            case 32: res_fn = reinterpret_cast<const void*>(&k_mgs_res<32>); break;
            default: break;
        }
        const size_t res_smem = static_cast<size_t>(E) * kRThreads * 16;  // two slices
        // even n and E <= 14: w in registers, columns double-buffered by bulk copies
        if ((n & 1) == 0 && sms <= 32 * kPollParts && !std::getenv("KTB_GMRES_NO_DMA_MGS")) {
            switch (E) {
                case 1: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<1>); break;
                case 2: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<2>); break;
                case 4: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<4>); break;
                case 8: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<8>); break;
                case 12: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<12>); break;
                case 14: res_fn = reinterpret_cast<const void*>(&k_mgs_dma<14>); break;
                default: break;
            }
        }
        int res_nb = 0;
        if (res_fn && !std::getenv("KTB_GMRES_STREAM_MGS")) {
            allow_max_dynamic_smem(res_fn);
            int occ = 0;
            KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, res_fn, kRThreads,
                                                                   res_smem));
            // E * kRThreads * grid must cover n with one CTA per SM
            if (occ >= 1) res_nb = static_cast<int>(ceil_div64(n, static_cast<int64_t>(E) * kRThreads));
            if (res_nb > sms) res_nb = 0;
        }
        if (P) {
            int64_t pn = 0;
            ilu0_info(P, &pn, nullptr, nullptr, nullptr);
            require(pn == n, "gmres: dimension mismatch");
        }
        // workspace cached on the plan (device vectors, basis, exchange slots,
        // pinned step outputs, events): repeated solves allocate nothing --
        // per-solve cudaMalloc/cudaMallocHost of ~0.5 GB showed up as
        // occasional 0.3-0.5 s outliers in the solve time
        auto* Wk = static_cast<GmresWork*>(A->gmres_ws.get());
        if (!Wk || Wk->n != n || Wk->m != m || Wk->prec != (P != nullptr) || Wk->nb != nb ||
            Wk->res_nb != res_nb) {
            A->gmres_ws.reset();
            A->gmres_ws = std::shared_ptr<void>(new GmresWork(n, m, P != nullptr, nb, res_nb),
                                                [](void* q) { delete static_cast<GmresWork*>(q); });
            Wk = static_cast<GmresWork*>(A->gmres_ws.get());
            KTB_CUDA(cudaMemsetAsync(Wk->slots.p, 0, Wk->slots.bytes(), st));
        }
        DBuf<double>& b = Wk->b;
        DBuf<double>& x = Wk->x;
        DBuf<double>& r = Wk->r;
        DBuf<double>& w = Wk->w;
        DBuf<double>& V = Wk->V;
        DBuf<double>& zp = Wk->zp;
        DBuf<double>& partials = Wk->partials;
        DBuf<double>& dy = Wk->dy;
        DBuf<double2>& slots = Wk->slots;
        long long& tag = Wk->tag;  // exchange tags never repeat across solves
        KTB_CUDA(cudaMemcpyAsync(b.p, b_host, 8 * n, cudaMemcpyHostToDevice, st));
        KTB_CUDA(cudaMemsetAsync(x.p, 0, 8 * n, st));
        const int eb = ceil_div(n, 256);
        cudaEvent_t ev0 = Wk->ev0, ev1 = Wk->ev1;
        bool pending = false;
        auto settle = [&]() {  // after a stream sync: account the last SpMV
            if (pending) {
                float ms = 0.f;
                KTB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
                res->spmv_seconds += ms * 1e-3;
                pending = false;
            }
        };
        auto spmv_timed = [&](const double* in, double* out) {
            KTB_CUDA(cudaEventRecord(ev0, st));
            plan_run(A, in, out, 0, n);
            KTB_CUDA(cudaEventRecord(ev1, st));
            pending = true;
            res->spmv_calls++;
        };
        auto norm2 = [&](const double* v) {
            k_sumsq<<<nb, kGThreads, 0, st>>>(v, n, partials.p);
            KTB_LAUNCH();
            std::vector<double> hp(nb);
            KTB_CUDA(cudaMemcpyAsync(hp.data(), partials.p, 8 * nb, cudaMemcpyDeviceToHost, st));
            KTB_CUDA(cudaStreamSynchronize(st));
            settle();
            double s = 0.0;
            for (double v : hp) s += v;
            return std::sqrt(s);
        };
        const double nb2 = norm2(b.p);
        if (nb2 == 0.0) {
            res->converged = 1;
            KTB_CUDA(cudaMemcpyAsync(x_host, x.p, 8 * n, cudaMemcpyDeviceToHost, st));
            KTB_CUDA(cudaStreamSynchronize(st));
            return;
        }
        // per-step outputs of the pipelined Arnoldi loop (pinned host memory
        // the MGS kernel writes directly); per-step SpMV and completion events
        auto& h_pin = Wk->h_pin;
        auto& brk_pin = Wk->brk_pin;
        auto &ev_s = Wk->ev_s, &ev_e = Wk->ev_e, &ev_step = Wk->ev_step;
        auto launch_step = [&](int64_t jj) {
            const double* src = V.p + jj * n;
            if (P) {  // gmres.hpp:91-92: z = M^{-1} v_j, w = A z
                ilu0_apply(P, src, zp.p, st);
                src = zp.p;
            }
            KTB_CUDA(cudaEventRecord(ev_s[jj], st));
            plan_run(A, src, w.p, 0, n);
            KTB_CUDA(cudaEventRecord(ev_e[jj], st));
            // orthogonalise against columns 0..jj; V_{jj+1} = w / |w|
            int kk = static_cast<int>(jj + 1);
            const double* Vp = V.p;
            double* wp = w.p;
            double* vn = V.p + (jj + 1) * n;
            // projections and the breakdown flag go straight to pinned host
            // memory (mapped under UVA): no copy nodes between the steps
            double* hp = h_pin.p + jj * (m + 2);
            double* pp = partials.p;
            int* bp = brk_pin.p + jj;
            int64_t nn = n;
            if (res_nb > 0) {
                // cooperative launch: all CTAs co-resident (they poll each other)
                double2* sp = slots.p;
                void* rargs[] = {&Vp, &nn, &kk, &wp, &vn, &hp, &sp, &bp, &tag};
                KTB_CUDA(cudaLaunchCooperativeKernel(res_fn, dim3(res_nb), dim3(kRThreads),
                                                     rargs, res_smem, st));
                tag += 64;
            } else {
                void* args[] = {&Vp, &nn, &kk, &wp, &vn, &hp, &pp, &bp};
                KTB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_mgs),
                                                     dim3(nb), dim3(kGThreads), args, 0, st));
            }
            KTB_CUDA(cudaEventRecord(ev_step[jj], st));
        };
        auto account_step = [&](int64_t jj) {  // a step the recurrence takes
            float ms = 0.f;
            KTB_CUDA(cudaEventElapsedTime(&ms, ev_s[jj], ev_e[jj]));
            res->spmv_seconds += ms * 1e-3;
            res->spmv_calls++;
        };
        const int64_t r_stride = m + 1;
        std::vector<double> h(m + 2), cs(m + 1), sn(m + 1), gv(m + 2), r_cols(r_stride * m),
            yv(m + 1);
        double rr = 1.0;
        bool stop = false;
        while (!stop) {
            spmv_timed(x.p, r.p);
            k_sub_from<<<eb, 256, 0, st>>>(b.p, r.p, n);
            KTB_LAUNCH();
            const double beta = norm2(r.p);
            rr = beta / nb2;
            if (rr < tol) {
                res->converged = 1;
                break;
            }
            k_div<<<eb, 256, 0, st>>>(r.p, beta, V.p, n);
            KTB_LAUNCH();
            std::fill(gv.begin(), gv.end(), 0.0);
            gv[0] = beta;
            int64_t j = 0;
            bool lucky = false;
            int64_t launched = -1;
            while (j < m) {
                if (res->iterations >= max_iters) {
                    stop = true;
                    break;
                }
                // the device runs one Arnoldi step ahead of the host recurrence:
                // step j+1 only needs V_{j+1} (written by step j's MGS), so it is
                // enqueued before step j's projections are read back; a step the
                // host then does not take (convergence, breakdown, iteration cap)
                // is discarded (not counted; it only wrote V_{j+2} and w)
                if (launched < j) launch_step(j);
                launched = j;
                if (j + 1 < m) {
                    launch_step(j + 1);
                    launched = j + 1;
                }
                // spin on the step's event (a blocking sync lets the OS park the
                // host thread: measured 2-3x outliers in the solve time)
                for (;;) {
                    const cudaError_t q = cudaEventQuery(ev_step[j]);
                    if (q == cudaSuccess) break;
                    if (q != cudaErrorNotReady) KTB_CUDA(q);
                }
                account_step(j);
                const double* hj = h_pin.p + j * (m + 2);
                for (int64_t q = 0; q <= j + 1; ++q) h[q] = hj[q];
                if (brk_pin.p[j]) {
                    h[j + 1] = 0.0;
                    lucky = true;
                }
                // gmres.hpp:100-116, verbatim scalar recurrence
                for (int64_t i = 0; i < j; ++i) {
                    const double t1 = h[i], t2 = h[i + 1];
                    h[i] = cs[i] * t1 + sn[i] * t2;
                    h[i + 1] = -sn[i] * t1 + cs[i] * t2;
                }
                const double denom = std::hypot(h[j], h[j + 1]);
                if (denom == 0.0) {
                    cs[j] = 1.0;
                    sn[j] = 0.0;
                } else {
                    cs[j] = h[j] / denom;
                    sn[j] = h[j + 1] / denom;
                }
                h[j] = denom;
                gv[j + 1] = -sn[j] * gv[j];
                gv[j] *= cs[j];
                for (int64_t q = 0; q <= j; ++q) r_cols[j * r_stride + q] = h[q];
                res->iterations++;
                rr = std::abs(gv[j + 1]) / nb2;
                if (history) history[res->iterations - 1] = rr;
                ++j;
                if (lucky || rr < tol) break;
            }
            if (j > 0) {  // gmres.hpp:125-143
                for (int64_t i = j - 1; i >= 0; --i) {
                    double s = gv[i];
                    for (int64_t l = i + 1; l < j; ++l) s -= r_cols[l * r_stride + i] * yv[l];
                    const double rii = r_cols[i * r_stride + i];
                    yv[i] = rii != 0.0 ? s / rii : 0.0;
                }
                KTB_CUDA(cudaMemcpyAsync(dy.p, yv.data(), 8 * j, cudaMemcpyHostToDevice, st));
                if (P) {  // w = Q y; z = M^{-1} w; x += z (gmres.hpp:138-143)
                    KTB_CUDA(cudaMemsetAsync(w.p, 0, 8 * n, st));
                    k_update_x<<<eb, 256, 0, st>>>(V.p, dy.p, static_cast<int>(j), n, w.p);
                    KTB_LAUNCH();
                    ilu0_apply(P, w.p, zp.p, st);
                    k_add_z<<<eb, 256, 0, st>>>(zp.p, n, x.p);
                } else {
                    k_update_x<<<eb, 256, 0, st>>>(V.p, dy.p, static_cast<int>(j), n, x.p);
                }
                KTB_LAUNCH();
            }
            if (rr < tol) {
                res->converged = 1;
                break;
            }
            if (lucky) {
                res->breakdown = 1;
                break;
            }
            if (stop) break;
            res->restarts++;
        }
        res->recurrence_residual = rr;
        spmv_timed(x.p, r.p);
        k_sub_from<<<eb, 256, 0, st>>>(b.p, r.p, n);
        KTB_LAUNCH();
        res->true_residual = norm2(r.p) / nb2;
        res->fault_convergence = res->converged && res->true_residual > tol;
        KTB_CUDA(cudaMemcpyAsync(x_host, x.p, 8 * n, cudaMemcpyDeviceToHost, st));
        KTB_CUDA(cudaStreamSynchronize(st));
        settle();
        res->seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

}  // namespace ktb
