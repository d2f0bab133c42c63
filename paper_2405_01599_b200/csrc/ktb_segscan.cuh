// ktb_segscan.cuh -- warp/block segmented scans over (flag, value) pairs.
//
// A pair (f, v) is "a run of products; f = a segment (row) boundary occurs
// inside it; v = the sum since the last boundary". The associative combine
// of an earlier pair a with a later pair b is
//     (a.f | b.f,  b.f ? b.v : a.v + b.v)
// which is the carry propagation of the reference's segmented-scan kernels
// (spmv.hpp:148-165 U4 flag scan, spmv.hpp:91-101 ordered slice combine).
#pragma once

#include <cuda_runtime.h>

namespace ktb {

struct SegPair {
    int f;
    double v;
};

__device__ __forceinline__ SegPair seg_combine(SegPair a, SegPair b) {
    return {a.f | b.f, b.f ? b.v : a.v + b.v};
}

// Inclusive warp scan.
__device__ __forceinline__ SegPair warp_seg_scan_incl(SegPair x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int f = __shfl_up_sync(0xffffffffu, x.f, o);
        const double v = __shfl_up_sync(0xffffffffu, x.v, o);
        if (lane >= o) {
            if (!x.f) x.v += v;
            x.f |= f;
        }
    }
    return x;
}

// Block-wide exclusive segmented scan for NT threads (multiple of 32).
// Returns the exclusive prefix; *total receives the block aggregate.
template <int NT>
__device__ __forceinline__ SegPair block_seg_scan_excl(SegPair x, SegPair* total) {
    constexpr int NW = NT / 32;
    __shared__ int s_f[NW];
    __shared__ double s_v[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const SegPair incl = warp_seg_scan_incl(x);
    SegPair excl;
    excl.f = __shfl_up_sync(0xffffffffu, incl.f, 1);
    excl.v = __shfl_up_sync(0xffffffffu, incl.v, 1);
    if (lane == 0) excl = {0, 0.0};
    if (lane == 31) {
        s_f[warp] = incl.f;
        s_v[warp] = incl.v;
    }
    __syncthreads();
    SegPair wp = {0, 0.0};
    SegPair agg = {0, 0.0};
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        const SegPair a = {s_f[w], s_v[w]};
        if (w < warp) wp = seg_combine(wp, a);
        agg = seg_combine(agg, a);
    }
    *total = agg;
    __syncthreads();  // s_f/s_v reusable after return
    return seg_combine(wp, excl);
}

}  // namespace ktb
