// ktb_unsym.cu -- unsymmetric CRS SpMV kernels for sm_100a.
//
//   U1  row-parallel CRS  (spmv.hpp:74-86 with ROW_BASED partition.hpp:38-41)
//       -> V lanes per row (V = 1..32, from the mean row length), shuffle
//          reduction; rows are assigned to lane groups in order.
//   U2  nnz-balanced CRS  (spmv.hpp:74-86 with NNZ_BALANCED partition.hpp:42-52)
//       -> merge-path tiles: every CTA consumes the same number of
//          (row-end + nonzero) items; products staged in smem with coalesced
//          loads; block-wide segmented scan; per-tile carry fixed up after.
//   U3  branchless segmented scan (spmv.hpp:127-146, bss.hpp:34-69)
//       -> one GPU thread = one BSS lane; lane chunks follow the reference rule
//          [nnz*p/jl, nnz*(p+1)/jl) with jl = ceil(nnz / E); row starts come
//          from the bit-packed row_start_flag array; lane carries are combined
//          by a block segmented scan, tile carries by the fixup kernel.
//   U4  original segmented scan (spmv.hpp:148-165): U3 with the per-element
//       flag branch left in (correctness reference, never a tuning candidate).
#include <cub/cub.cuh>

#include <utility>

#include "ktb_internal.cuh"
#include "ktb_ptx.cuh"
#include "ktb_segscan.cuh"

namespace ktb {

__device__ __forceinline__ double ldg_f64(const double* p) { return __ldg(p); }
__device__ __forceinline__ int32_t ldg_i32(const int32_t* p) { return __ldg(p); }

// Streaming loads for the matrix arrays: read once, do not keep in L1, evict
// first from L2 (so x, gathered repeatedly, stays resident).
__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(r) : "l"(p), "l"(pol_first()));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
        : "=r"(r) : "l"(p), "l"(pol_first()));
    return r;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(r) : "l"(p), "l"(pol_first()));
    return r;
}
__device__ __forceinline__ double ld_plain_f64(const double* p) {
    double r;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int32_t ld_plain_i32(const int32_t* p) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
// x gathers: keep in L2
__device__ __forceinline__ double ld_x(const double* p) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol_last()));
    return r;
}

// =============================================================== U1
// V lanes per row, R consecutive rows per lane group: the row bounds, then
// the first V entries of all R rows, then their x gathers are issued before
// any use (R-fold memory-level parallelism); rows longer than V finish in a
// lane-strided tail loop.
template <int V, int R>
__global__ void __launch_bounds__(256) k_u1(const int32_t* __restrict__ rp,
                                            const int32_t* __restrict__ col,
                                            const double* __restrict__ val,
                                            const double* __restrict__ x, double* __restrict__ y,
                                            int32_t row_begin, int32_t row_end) {
    const int sub = threadIdx.x & (V - 1);
    const int64_t group = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / V;
    const int64_t row0 = row_begin + group * R;
    int32_t b[R], e[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t row = row0 + r;
        b[r] = row < row_end ? ldg_i32(rp + row) : 0;
        e[r] = row < row_end ? ldg_i32(rp + row + 1) : 0;
    }
    int32_t c[R];
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int32_t k = b[r] + sub;
        c[r] = k < e[r] ? ld_stream_i32(col + k) : -1;
        v[r] = k < e[r] ? ld_stream_f64(val + k) : 0.0;
    }
    double s[R];
#pragma unroll
    for (int r = 0; r < R; ++r) s[r] = c[r] >= 0 ? v[r] * ld_x(x + c[r]) : 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r)
        for (int32_t k = b[r] + sub + V; k < e[r]; k += V)
            s[r] += ld_stream_f64(val + k) * ld_x(x + ld_stream_i32(col + k));
    if (V > 1) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int o = V / 2; o > 0; o >>= 1) s[r] += __shfl_xor_sync(0xffffffffu, s[r], o, V);
    }
    if (sub == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (row0 + r < row_end) y[row0 + r] = s[r];
    }
}

// ---- U1, thread per row over a warp-sliced copy (param 100) ---------------
// The reference's U1 worker sums each of its rows serially, left to right
// (spmv.hpp:74-86), bitwise equal to spmv_ref (csr.hpp:69-84). Here one
// thread does exactly that for one row, with the same non-contracted
// multiply-then-add (so y is bitwise equal to the reference), over a copy of
// the matrix laid out for the warp: rows in slices of 32, slice s of width
// W_s = its longest row, entry k of row 32s + l at sell_off[s] + 32k + l
// (SELL-32, column-major inside the slice; padding col -1). Every column and
// value load of a warp is one coalesced 128/256-byte line, there is no
// cross-lane reduction, and the whole row's loads then gathers are in flight
// at once. The plan builds the copy on the device (k_sell_*); it is refused
// when padding would more than triple the matrix (power-law rows).
constexpr int kSellUnroll = 8;
#ifndef KTB_U1S_THREADS
#define KTB_U1S_THREADS 128  // 4 slices per CTA: vs 256, config 4 2.13-2.15 vs 2.33 ms, config 5 39.5 vs 42 us
#endif
constexpr int kU1sThreads = KTB_U1S_THREADS;
#ifndef KTB_U1S_MINB
#define KTB_U1S_MINB 1  // 7 (config 1's 8192 slices in one wave) caps registers at 32 and
                        // spills: slower on configs 1, 4 and 5
#endif
// CTA shape: 64, 128 (default) or 256 threads, all instantiated; the
// selector times them as launch-shape candidates (p->cta_threads)
//
// kDict (U1 param 102): the same slices with the columns coded, not stored:
// each slice keeps a dictionary of at most 15 column deltas (col - row; a
// stencil row has 7) and every slot a 4-bit code (15 = padding), 8 codes per
// 32-bit word, so a slot streams 8 B of value + 0.5 B of code instead of
// 8 + 4 B; the column is row + dict[code] (one warp shuffle). Same entries,
// same order, same arithmetic: y stays bitwise equal to spmv_ref.
template <int kThreads, bool kDict>
__global__ void __launch_bounds__(kThreads, KTB_U1S_MINB) k_u1s(const int64_t* __restrict__ soff,
                                             const int32_t* __restrict__ scol,
                                             const double* __restrict__ sval,
                                             const double* __restrict__ x, double* __restrict__ y,
                                             int32_t row_begin, int32_t row_end, int ell,
                                             const int32_t* __restrict__ perm, int64_t xpf,
                                             int64_t xlen, const uint32_t* __restrict__ codes,
                                             const int32_t* __restrict__ dict) {
    const int lane = threadIdx.x & 31;
    if (xpf >= 0 && threadIdx.x == 0) {
        // x entries of this CTA's own rows into L2 while the first column /
        // value loads are in flight: the gathers (own rows and the rows of the
        // CTAs running beside it) then find x in L2 instead of making a
        // second DRAM round trip (xpf = the rows' column shift; -1 = off)
        const int64_t r0 = static_cast<int64_t>(row_begin & ~31) + blockIdx.x * int64_t(kThreads);
        const int64_t lo = max(r0 + xpf, int64_t(0)), hi = min(r0 + kThreads + xpf, xlen);
        if (hi > lo) prefetch_l2_range(x + lo, x + hi);
    }
    const int64_t s = (row_begin >> 5) + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32;
    int64_t row = s * 32 + lane;
    if (s * 32 >= row_end) return;
    if (perm) row = __ldg(perm + row);  // sorted slices: slot -> row (-1: padding)
    int64_t o;
    int W;
    if (ell) {  // uniform width: offsets implicit
        o = s * 32 * ell;
        W = ell;
    } else {
        o = __ldg(soff + s);
        W = static_cast<int>((__ldg(soff + s + 1) - o) >> 5);
    }
    const int32_t* sc = scol + o + lane;
    const double* sv = sval + o + lane;
    int32_t dv = 0;
    const uint32_t* cw = nullptr;
    if constexpr (kDict) {
        dv = __ldg(dict + s * 16 + (lane & 15));  // lane j < 15 holds delta j
        cw = codes + (o >> 3) + (lane >> 3);      // 4 words per 32 slots
    }
    double sum = 0.0;
    for (int k0 = 0; k0 < W; k0 += kSellUnroll) {
        int32_t c[kSellUnroll];
        double v[kSellUnroll], xv[kSellUnroll];
        if constexpr (kDict) {
            // every code and value load of the batch first, the decode
            // shuffles after them (a shuffle between loads would serialise
            // the batch into one round trip per slot)
            uint32_t wd[kSellUnroll];
#pragma unroll
            for (int u = 0; u < kSellUnroll; ++u) {
                const bool ok = k0 + u < W;  // warp-uniform
                wd[u] = ok ? ld_stream_u32(cw + (k0 + u) * 4) : 0xffffffffu;
                v[u] = ok ? ld_stream_f64(sv + (k0 + u) * 32) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < kSellUnroll; ++u) {
                const int code = static_cast<int>((wd[u] >> ((lane & 7) * 4)) & 15u);
                const int32_t d = __shfl_sync(0xffffffffu, dv, code);
                c[u] = code != 15 ? static_cast<int32_t>(row) + d : -1;
            }
        } else {
#pragma unroll
            for (int u = 0; u < kSellUnroll; ++u) {
                const bool ok = k0 + u < W;  // warp-uniform
                c[u] = ok ? ld_stream_i32(sc + (k0 + u) * 32) : -1;
                v[u] = ok ? ld_stream_f64(sv + (k0 + u) * 32) : 0.0;
            }
        }
#pragma unroll
        for (int u = 0; u < kSellUnroll; ++u) xv[u] = c[u] >= 0 ? ld_x(x + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < kSellUnroll; ++u)
            if (c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
    }
    if (perm ? row >= 0 : (row >= row_begin && row < row_end)) y[row] = sum;
}

// ---- U1 params 103 / 104: persistent, software-pipelined warp slices ---------
// The warp-sliced kernel above runs one slice per warp and one wave of CTAs
// after another: each warp's column/value loads and then its x gathers are
// two serial round trips, and with ~31 resident warps per SM that is what
// bounds it (ncu, config 4: 6.24 TB/s, eligible warps 0.75 per scheduler).
// Here a grid of resident CTAs walks the slices (warp g takes g, g+G, ...)
// two deep: the loads of the next slice are issued before the gathers of the
// current one, so a warp always has one slice's stream and another's gathers
// in flight. Uniform slice width W <= 8 (ELL; the stencils), int32 columns
// (103) or the coded columns of 102 (104). Row sums unchanged: bitwise
// spmv_ref.
template <bool kDict>
struct SliceRegs {
    uint32_t cw[8];  // int32 column or code word per slot
    double v[8];
    int32_t dv;      // dictionary entry (kDict)
};

template <bool kDict>
__device__ __forceinline__ void slice_load(SliceRegs<kDict>& R, int64_t s, int64_t s_end, int W,
                                           const int32_t* __restrict__ scol,
                                           const double* __restrict__ sval,
                                           const uint32_t* __restrict__ codes,
                                           const int32_t* __restrict__ dict, int lane) {
    const bool live = s < s_end;  // warp-uniform
    const int64_t o = s * 32 * W;
    if (kDict) R.dv = live ? __ldg(dict + s * 16 + (lane & 15)) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const bool ok = live && u < W;
        if (kDict)
            R.cw[u] = ok ? ld_stream_u32(codes + (o >> 3) + u * 4 + (lane >> 3)) : 0xffffffffu;
        else
            R.cw[u] = ok ? static_cast<uint32_t>(ld_stream_i32(scol + o + u * 32 + lane))
                         : 0xffffffffu;
        R.v[u] = ok ? ld_stream_f64(sval + o + u * 32 + lane) : 0.0;
    }
}

template <bool kDict>
__device__ __forceinline__ void slice_finish(const SliceRegs<kDict>& R, int64_t s, int32_t r0,
                                             int32_t r1, const double* __restrict__ x,
                                             double* __restrict__ y, int lane) {
    const int64_t row = s * 32 + lane;
    int32_t c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        if (kDict) {
            const int code = static_cast<int>((R.cw[u] >> ((lane & 7) * 4)) & 15u);
            const int32_t d = __shfl_sync(0xffffffffu, R.dv, code);
            c[u] = code != 15 ? static_cast<int32_t>(row) + d : -1;
        } else {
            c[u] = static_cast<int32_t>(R.cw[u]);
        }
    }
    double xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) xv[u] = c[u] >= 0 ? ld_x(x + c[u]) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
        if (c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(R.v[u], xv[u]));
    if (row >= r0 && row < r1) y[row] = sum;
}

// 80 registers = 3 CTAs (24 warps) per SM for both forms; the int32-column
// form needs the 3-CTA bound to get there (82 registers otherwise: 2 CTAs,
// 33 % slower), the coded form gets 80 unconstrained (an explicit bound of 1
// gives 95 registers and half the speed)
template <bool kDict>
__global__ void __launch_bounds__(256, kDict ? 0 : 3) k_u1p(const int32_t* __restrict__ scol,
                                             const double* __restrict__ sval,
                                             const uint32_t* __restrict__ codes,
                                             const int32_t* __restrict__ dict,
                                             const double* __restrict__ x, double* __restrict__ y,
                                             int32_t row_begin, int32_t row_end, int W) {
    const int lane = threadIdx.x & 31;
    const int64_t G = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    const int64_t s0 = row_begin >> 5, s_end = (static_cast<int64_t>(row_end) + 31) >> 5;
    int64_t s = s0 + blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5);
    SliceRegs<kDict> A, B;
    slice_load(A, s, s_end, W, scol, sval, codes, dict, lane);
    // two slices per trip so that the register sets alternate without copies
    for (; s < s_end; s += 2 * G) {
        slice_load(B, s + G, s_end, W, scol, sval, codes, dict, lane);
        slice_finish(A, s, row_begin, row_end, x, y, lane);
        if (s + G >= s_end) break;
        slice_load(A, s + 2 * G, s_end, W, scol, sval, codes, dict, lane);
        slice_finish(B, s + G, row_begin, row_end, x, y, lane);
    }
}

// ---- U1 param 105: persistent coded slices staged by per-warp bulk copies ----
// 104 keeps the next slice in registers, which caps it at two slices per warp
// in flight and 24 warps per SM (80 registers). Here every warp owns a ring
// of kU1tStages shared-memory stages; lane 0 fills a stage with one slice's
// values (32 W doubles, contiguous in the ELL copy), its code words and its
// dictionary by three bulk copies (cp.async.bulk, completion on the stage's
// mbarrier) kU1tStages slices ahead, so a warp keeps that many slices of the
// stream in flight without registers. Lanes read their values / codes from
// the stage (conflict-free), decode through the staged dictionary, gather x,
// sum left to right (bitwise spmv_ref) and hand the stage back.
#ifndef KTB_U1T_STAGES
#define KTB_U1T_STAGES 2
#endif
#ifndef KTB_U1T_WARPS
#define KTB_U1T_WARPS 8
#endif
#ifndef KTB_U1T_MINB
#define KTB_U1T_MINB 1
#endif
constexpr int kU1tStages = KTB_U1T_STAGES;
constexpr int kU1tWarps = KTB_U1T_WARPS;
// stage = one slice's values (32 W doubles), code words (4 W) and dictionary (16)
inline int u1t_stage_bytes(int W) { return (32 * 8 * W + 16 * W + 64 + 15) & ~15; }
inline int u1t_smem(int W) { return kU1tWarps * kU1tStages * (u1t_stage_bytes(W) + 8); }

__global__ void __launch_bounds__(kU1tWarps * 32, KTB_U1T_MINB) k_u1t(const double* __restrict__ sval,
                                                         const uint32_t* __restrict__ codes,
                                                         const int32_t* __restrict__ dict,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ y, int32_t row_begin,
                                                         int32_t row_end, int W, int stage_bytes) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* ring = smem + warp * (kU1tStages * stage_bytes);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kU1tWarps * kU1tStages * stage_bytes) +
                     warp * kU1tStages;
    const int coff = 32 * 8 * W, doff = coff + 16 * W;  // codes, dictionary within a stage
    const int64_t G = static_cast<int64_t>(gridDim.x) * kU1tWarps;
    const int64_t s0 = (row_begin >> 5) + blockIdx.x * static_cast<int64_t>(kU1tWarps) + warp;
    const int64_t s_end = (static_cast<int64_t>(row_end) + 31) >> 5;
    const uint32_t vbytes = 32u * 8u * W, cbytes = 16u * W;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int64_t s, int st) {  // lane 0
        unsigned char* b = ring + st * stage_bytes;
        mbar_arrive_expect_tx(&bars[st], vbytes + cbytes + 64);
        tma_load_1d(b, sval + s * 32 * W, vbytes, &bars[st], pol);
        tma_load_1d(b + coff, codes + s * 4 * W, cbytes, &bars[st], pol);
        tma_load_1d(b + doff, dict + s * 16, 64, &bars[st], pol);
    };
    if (lane == 0) {
        for (int st = 0; st < kU1tStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
        for (int st = 0; st < kU1tStages; ++st)
            if (s0 + st * G < s_end) issue(s0 + st * G, st);
    }
    __syncwarp();
    int it = 0;
    for (int64_t s = s0; s < s_end; s += G, ++it) {
        const int st = it % kU1tStages;
        const uint32_t ph = (it / kU1tStages) & 1;
        mbar_wait(&bars[st], ph);
        const unsigned char* b = ring + st * stage_bytes;
        const double* sv = reinterpret_cast<const double*>(b);
        const uint32_t* sc = reinterpret_cast<const uint32_t*>(b + coff);
        const int32_t* sd = reinterpret_cast<const int32_t*>(b + doff);
        const int64_t row = s * 32 + lane;
        int32_t c[8];
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool ok = u < W;  // warp-uniform
            const uint32_t wd = ok ? sc[u * 4 + (lane >> 3)] : 0xffffffffu;
            const int code = static_cast<int>((wd >> ((lane & 7) * 4)) & 15u);
            c[u] = code != 15 ? static_cast<int32_t>(row) + sd[code] : -1;
            v[u] = ok ? sv[u * 32 + lane] : 0.0;
        }
        __syncwarp();  // every lane has its slots: the stage may be refilled
        if (lane == 0 && s + kU1tStages * G < s_end) {
            fence_proxy_async_smem();
            issue(s + kU1tStages * G, st);
        }
        double xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = c[u] >= 0 ? ld_x(x + c[u]) : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c[u] >= 0) sum = __dadd_rn(sum, __dmul_rn(v[u], xv[u]));
        if (row >= row_begin && row < row_end) y[row] = sum;
    }
}

// ---- U1 param 106: persistent slices with coded (column, value) pairs ----
// Many matrices (every constant-coefficient stencil, graph Laplacians,
// adjacency matrices) hold only a handful of distinct (column - row, value)
// pairs per block of rows. 106 stores one record per 64 rows: a dictionary of
// the block's pairs (16 bytes each: the fp64 bit pattern, the int32 column
// delta, a "real" word; the last entry is the padding pair) and per row
// ceil(W/4) 32-bit words of 8-bit pair codes (word k of rows l and l + 32
// side by side at 64 k + 2 l). With D dictionary entries (the plan's maximum
// + padding, <= 64) and slice width W <= 32 a record is 16 D + 256 ceil(W/4)
// bytes: 640 for the 7-point stencils (10 B per row instead of 8.5 B per
// slot), 2,240 for a 27-point stencil. The values the kernel multiplies are
// the stored bit patterns and the sum runs left to right with unfused
// multiply-add: bitwise spmv_ref. More pairs or wider rows refuse the layout
// (the selector and the halo operator fall back to 105). One bulk copy per
// record fills a stage of the warp's ring. A lane owns rows l and l + 32; a
// batch is two code words (8 slots) of both rows: the 4-byte delta lookups and
// the 16 gathers go out first, the 8-byte value lookups follow when the
// products are formed, so an in-flight slot holds its gathered x and nothing
// else (64 registers, 32 warps per SM). When the two rows' code words are
// equal in every lane (always, away from a boundary) one lookup serves both
// rows. The kernel is bound by the L1TEX data pipe (ncu: ~3 wavefronts per
// 256-byte gather, ~1 per lookup; 73 % busy), not by HBM. Measured and
// dropped: an L2 prefetch of x at the sweep's front (+40 % time on config 4),
// one code word per batch (+11 %), 80 registers / 24 warps (+28 %), CTAs of 4
// warps (+12 %); 2, 4 or 6 stages make no difference on config 4.
constexpr int kU1vMaxDict = 64;  // dictionary entries per record incl. padding
#ifndef KTB_U1V_WARPS
#define KTB_U1V_WARPS 8
#endif
#ifndef KTB_U1V_MINB
#define KTB_U1V_MINB 4  // 64 registers, 32 warps per SM
#endif
constexpr int kU1vWarps = KTB_U1V_WARPS;

struct U1vLayout {
    int dict = 0;    // dictionary entries incl. the padding pair
    int words = 0;   // code words per row
    int rec = 0;     // record bytes (global stride)
    int stride = 0;  // stage stride in shared memory (dictionary aligned for the OR lookup)
    int stages = 0;
};
static U1vLayout u1v_layout(int max_pairs, int W) {
    U1vLayout L;
    L.dict = max_pairs + 1;
    L.words = (W + 3) / 4;
    L.rec = 16 * L.dict + 256 * L.words;
    int a = 256;
    while (a < 16 * L.dict) a <<= 1;
    L.stride = (L.rec + a - 1) / a * a;
#ifdef KTB_U1V_STAGES
    L.stages = KTB_U1V_STAGES;
#else
    L.stages = L.stride <= 1024 ? 4 : L.stride <= 1536 ? 3 : 2;
#endif
    return L;
}
static int u1v_smem(const U1vLayout& L) { return kU1vWarps * L.stages * (L.stride + 8) + 1024; }

// One warp per 64-row record of the ELL copy (32-row slices 2 s and 2 s + 1).
// Pass 1 (rec == nullptr): the record's pair count into the plan-wide
// maximum. Pass 2: the record -- the pair dictionary by ballot matching
// (first-occurrence order; lane j holds pairs j and 32 + j), then the code
// bytes; the padding code is dict - 1.
__global__ void k_vrec_build(const int32_t* __restrict__ scol, const double* __restrict__ sval,
                             int64_t slices32, int64_t recs, int W, int dict, int rec_bytes,
                             unsigned char* __restrict__ rec, int* __restrict__ max_pairs) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= recs) return;  // whole warps
    int32_t dc[2] = {0, 0};
    unsigned long long dv[2] = {0, 0};
    int np = 0;
    const int pad = dict - 1;
    uint32_t word[2] = {0, 0};
    unsigned char* r = rec ? rec + s * rec_bytes : nullptr;
    for (int k = 0; k < 4 * ((W + 3) / 4); ++k) {
        for (int h = 0; h < 2; ++h) {
            int code = pad;
            const int64_t s32 = 2 * s + h;
            if (k < W && s32 < slices32) {
                const int64_t at = (s32 * W + k) * 32 + lane;
                const int32_t c = scol[at];
                const unsigned long long vb =
                    static_cast<unsigned long long>(__double_as_longlong(sval[at]));
                const int32_t d = c - static_cast<int32_t>(s32 * 32 + lane);
                unsigned pending = __ballot_sync(0xffffffffu, c >= 0);
                while (pending) {
                    const int src = __ffs(pending) - 1;
                    const int32_t wd = __shfl_sync(0xffffffffu, d, src);
                    const unsigned long long wv = __shfl_sync(0xffffffffu, vb, src);
                    const unsigned same =
                        __ballot_sync(0xffffffffu, c >= 0 && d == wd && vb == wv);
                    const unsigned hit0 =
                        __ballot_sync(0xffffffffu, lane < np && dc[0] == wd && dv[0] == wv);
                    const unsigned hit1 =
                        __ballot_sync(0xffffffffu, lane + 32 < np && dc[1] == wd && dv[1] == wv);
                    int j;
                    if (hit0) {
                        j = __ffs(hit0) - 1;
                    } else if (hit1) {
                        j = 32 + __ffs(hit1) - 1;
                    } else {
                        j = np < 64 ? np : 63;  // past 63 pairs only the count matters (refused)
                        if (np < 64 && lane == (j & 31)) {
                            dc[j >> 5] = wd;
                            dv[j >> 5] = wv;
                        }
                        ++np;
                    }
                    if ((same >> lane) & 1u) code = j;
                    pending &= ~same;
                }
            }
            word[h] |= static_cast<uint32_t>(code & 255) << (8 * (k & 3));
        }
        if ((k & 3) == 3) {
            if (r)
                reinterpret_cast<uint2*>(r + 16 * dict)[(k >> 2) * 32 + lane] =
                    make_uint2(word[0], word[1]);
            word[0] = word[1] = 0;
        }
    }
    if (!r) {
        if (lane == 0) atomicMax(max_pairs, np);
        return;
    }
    for (int h = 0; h < 2; ++h) {
        const int j = 32 * h + lane;
        if (j < dict) {
            const bool real = j < np;
            uint4 e;
            e.x = real ? static_cast<uint32_t>(dv[h]) : 0u;
            e.y = real ? static_cast<uint32_t>(dv[h] >> 32) : 0u;
            e.z = real ? static_cast<uint32_t>(dc[h]) : 0u;
            e.w = real ? 1u : 0u;
            reinterpret_cast<uint4*>(r)[j] = e;
        }
    }
}

// dictionary entry at byte offset `off` of the stage: the fp64 bit pattern at
// +0, the int32 column delta at +8. The delta is read when the gather is
// issued and the value when its product is formed, so that an in-flight slot
// holds two registers (the gathered x) and nothing else.
__device__ __forceinline__ int32_t u1v_delta(uint32_t sb, uint32_t off) {
    int32_t d;
    asm volatile("ld.shared.s32 %0, [%1+8];" : "=r"(d) : "r"(sb | off));
    return d;
}
__device__ __forceinline__ double u1v_value(uint32_t sb, uint32_t off) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(sb | off));
    return v;
}
// byte offset (code << 4) of slot b of a code word
__device__ __forceinline__ uint32_t u1v_off(uint32_t ww, int b) {
    return (b == 0 ? (ww << 4) : (ww >> (8 * b - 4))) & 0xff0u;
}
__device__ __forceinline__ double u1v_gather(const double* xr, int32_t delta) {
    const double* px;
    asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(px) : "r"(delta), "l"(xr));
    return ld_x(px);
}

#ifndef KTB_U1V_BATCH
#define KTB_U1V_BATCH 2  // code words (4 slots each) per batch of gathers
#endif

// kW = the plan's slice width (slots kW.. of the last code word are padding in
// every row and cost nothing). Per-warp state is kept small (the kernel runs
// at 64 registers, 32 warps per SM): the current stage and barrier address,
// the global address of the next record to fetch, the record's first row.
template <int kW>
__global__ void __launch_bounds__(kU1vWarps * 32, KTB_U1V_MINB)
    k_u1v(const unsigned char* __restrict__ rec, const double* __restrict__ x,
          double* __restrict__ y, int32_t row_begin, int32_t row_end, int32_t nrows,
          int32_t xlen, int dict_bytes, int rec_bytes, int stride, int stages) {
    constexpr int kWords = (kW + 3) / 4;
    constexpr int kB = KTB_U1V_BATCH;
    extern __shared__ unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // stages aligned to the dictionary's power-of-two size in the shared
    // window: an entry's address is then (stage | code << 4), one logic op
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t ring = base + warp * (stages * stride);
    const uint32_t bars = base + kU1vWarps * stages * stride + warp * stages * 8;
    const int G = static_cast<int>(gridDim.x) * kU1vWarps;
    const int first = (row_begin >> 6) + blockIdx.x * kU1vWarps + warp;
    const int last = static_cast<int>((static_cast<int64_t>(row_end) + 63) >> 6);
    int left = first < last ? (last - first + G - 1) / G : 0;  // this warp's records
    const uint64_t pol = policy_evict_first();
    const int64_t gstep = static_cast<int64_t>(G) * rec_bytes;
    const unsigned char* src = rec + static_cast<int64_t>(first) * rec_bytes;  // next record
    const uint32_t pad = static_cast<uint32_t>(dict_bytes - 16);  // the padding pair's offset
    auto issue = [&](uint32_t dst, uint32_t bar) {  // lane 0: one bulk copy per record
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(rec_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
            "l"(src), "r"(rec_bytes), "r"(bar), "l"(pol)
            : "memory");
        src += gstep;
    };
    const uint32_t rstep = static_cast<uint32_t>(G) * 64u;
    if (lane == 0) {
        for (int st = 0; st < stages; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bars + st * 8), "r"(1)
                         : "memory");
        fence_mbar_init();
        for (int st = 0; st < stages && st < left; ++st) issue(ring + st * stride, bars + st * 8);
    }
    __syncwarp();
    int st = 0;
    uint32_t ph = 0, sb = ring, bar = bars;
    uint32_t row = static_cast<uint32_t>(first) * 64u + lane;  // rows row and row + 32
    for (; left > 0; --left, row += rstep) {
        {
            KTB_CHAOS_DELAY(0x7531);
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "WAITV_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra WAITV_%=;\n"
                "}\n" ::"r"(bar),
                "r"(ph)
                : "memory");
        }
        // rows past the end of the matrix (last record) hold padding only: their
        // unconditional gathers read x at the last row instead
        const double* xa = x + min(row, static_cast<uint32_t>(nrows - 1));
        const double* xb = x + min(row + 32u, static_cast<uint32_t>(nrows - 1));
        const uint32_t cb = sb + dict_bytes + lane * 8;
        double sa = 0.0, sb2 = 0.0;
        // kB code words (4 slots each) of both rows at a time: all their
        // gathers in flight, then the products in slot order
#pragma unroll
        for (int g = 0; g < kWords; g += kB) {
            uint32_t wa[kB], wb[kB];
            bool same = true;
#pragma unroll
            for (int j = 0; j < kB; ++j)
                if (g + j < kWords) {
                    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];"
                                 : "=r"(wa[j]), "=r"(wb[j])
                                 : "r"(cb + (g + j) * 256));
                    same = same && wa[j] == wb[j];
                }
            double xva[4 * kB], xvb[4 * kB];
            if (__all_sync(0xffffffffu, same)) {  // one lookup serves both rows
#pragma unroll
                for (int j = 0; j < kB; ++j)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * (g + j) + u < kW) {
                            const int32_t d = u1v_delta(sb, u1v_off(wa[j], u));
                            xva[4 * j + u] = u1v_gather(xa, d);
                            xvb[4 * j + u] = u1v_gather(xb, d);
                        }
#pragma unroll
                for (int j = 0; j < kB; ++j)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * (g + j) + u < kW) {
                            const uint32_t off = u1v_off(wa[j], u);
                            const double v = u1v_value(sb, off);
                            const double ta = __dadd_rn(sa, __dmul_rn(v, xva[4 * j + u]));
                            const double tb = __dadd_rn(sb2, __dmul_rn(v, xvb[4 * j + u]));
                            sa = off != pad ? ta : sa;
                            sb2 = off != pad ? tb : sb2;
                        }
            } else {
#pragma unroll
                for (int j = 0; j < kB; ++j)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * (g + j) + u < kW) {
                            xva[4 * j + u] = u1v_gather(xa, u1v_delta(sb, u1v_off(wa[j], u)));
                            xvb[4 * j + u] = u1v_gather(xb, u1v_delta(sb, u1v_off(wb[j], u)));
                        }
#pragma unroll
                for (int j = 0; j < kB; ++j)
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (4 * (g + j) + u < kW) {
                            const uint32_t oa = u1v_off(wa[j], u), ob = u1v_off(wb[j], u);
                            const double ta =
                                __dadd_rn(sa, __dmul_rn(u1v_value(sb, oa), xva[4 * j + u]));
                            const double tb =
                                __dadd_rn(sb2, __dmul_rn(u1v_value(sb, ob), xvb[4 * j + u]));
                            sa = oa != pad ? ta : sa;
                            sb2 = ob != pad ? tb : sb2;
                        }
            }
        }
        __syncwarp();  // every lane has read its last entries: the stage may be refilled
        if (lane == 0 && left > stages) {
            fence_proxy_async_smem();
            issue(sb, bar);
        }
        if (row >= static_cast<uint32_t>(row_begin) && row < static_cast<uint32_t>(row_end))
            y[row] = sa;
        if (row + 32u >= static_cast<uint32_t>(row_begin) &&
            row + 32u < static_cast<uint32_t>(row_end))
            y[row + 32u] = sb2;
        sb += stride;
        bar += 8;
        if (++st == stages) {
            st = 0;
            ph ^= 1u;
            sb = ring;
            bar = bars;
        }
    }
}

using U1vFn = void (*)(const unsigned char*, const double*, double*, int32_t, int32_t, int32_t,
                       int32_t, int, int, int, int);
template <int... kWs>
static U1vFn u1v_pick(int W, std::integer_sequence<int, kWs...>) {
    U1vFn fn = nullptr;
    ((W == kWs + 1 ? (fn = k_u1v<kWs + 1>, 0) : 0), ...);
    return fn;
}
static U1vFn u1v_kernel(int W) {
    U1vFn fn = u1v_pick(W, std::make_integer_sequence<int, 32>{});
    if (!fn) throw Invalid("u1: coded slices need one slice width <= 32");
    return fn;
}

// ---- U1 param 101 setup helpers: rows sorted by length ----------------------
__global__ void k_sort_keys(const int32_t* __restrict__ rp, int64_t n, int32_t cap,
                            int32_t* __restrict__ key, int32_t* __restrict__ row) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int32_t len = rp[i + 1] - rp[i];
    key[i] = len <= cap ? len : -1;  // long rows sort last
    row[i] = static_cast<int32_t>(i);
}

// keys sorted descending: the number of keys >= 0
__global__ void k_count_nonneg_sorted(const int32_t* __restrict__ key, int64_t n,
                                      int64_t* __restrict__ out) {
    int64_t lo = 0, hi = n;  // first index with key < 0
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (key[mid] >= 0)
            lo = mid + 1;
        else
            hi = mid;
    }
    *out = lo;
}

// slice widths from the sorted keys (slot 32s holds the slice's longest row)
__global__ void k_sorted_width(const int32_t* __restrict__ key, int64_t ns, int64_t slices,
                               int64_t* __restrict__ w32) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s > slices) return;
    w32[s] = s == slices ? 0 : static_cast<int64_t>(key[s * 32]) * 32;
}

__global__ void k_sorted_fill(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ val, const int32_t* __restrict__ srow,
                              int64_t ns, int64_t slices, const int64_t* __restrict__ soff,
                              int32_t* __restrict__ perm, int32_t* __restrict__ scol,
                              double* __restrict__ sval) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t s = t >> 5;
    if (s >= slices) return;
    const int lane = static_cast<int>(t & 31);
    const int32_t r = t < ns ? srow[t] : -1;
    perm[t] = r;
    const int64_t o = soff[s];
    const int W = static_cast<int>((soff[s + 1] - o) >> 5);
    const int32_t b = r >= 0 ? rp[r] : 0, len = r >= 0 ? rp[r + 1] - b : 0;
    for (int k = 0; k < W; ++k) {
        const int64_t d = o + static_cast<int64_t>(k) * 32 + lane;
        scol[d] = k < len ? col[b + k] : -1;
        sval[d] = k < len ? val[b + k] : 0.0;
    }
}

__global__ void k_long_counts(const int32_t* __restrict__ rp, const int32_t* __restrict__ lrow,
                              int64_t nl, int32_t* __restrict__ lrp) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i <= nl) lrp[i] = i < nl ? rp[lrow[i] + 1] - rp[lrow[i]] : 0;
}

// one block per long row: copy its entries into the compact sub-matrix
__global__ void k_long_copy(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int32_t* __restrict__ lrow,
                            const int32_t* __restrict__ lrp, int32_t* __restrict__ lcol,
                            double* __restrict__ lval) {
    const int32_t r = lrow[blockIdx.x];
    const int32_t b = rp[r], len = rp[r + 1] - b, d = lrp[blockIdx.x];
    for (int32_t k = threadIdx.x; k < len; k += blockDim.x) {
        lcol[d + k] = col[b + k];
        lval[d + k] = val[b + k];
    }
}

__global__ void k_scatter_rows(const double* __restrict__ src, const int32_t* __restrict__ rows,
                               int64_t nl, double* __restrict__ y) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < nl) y[rows[i]] = src[i];
}

__global__ void k_sell_width(const int32_t* __restrict__ rp, int64_t n, int64_t slices,
                             int64_t* __restrict__ w32) {
    const int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s > slices) return;
    if (s == slices) {
        w32[s] = 0;  // scan sentinel
        return;
    }
    int32_t w = 0;
    for (int64_t r = s * 32; r < min(n, s * 32 + 32); ++r) w = max(w, rp[r + 1] - rp[r]);
    w32[s] = static_cast<int64_t>(w) * 32;
}

__global__ void k_fill_i64(int64_t* __restrict__ a, int64_t count, int64_t v) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < count) a[i] = v;
}

__global__ void k_sell_fill(const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, int64_t n,
                            const int64_t* __restrict__ soff, int32_t* __restrict__ scol,
                            double* __restrict__ sval) {
    const int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t s = r >> 5;
    if (s * 32 >= n) return;
    const int lane = static_cast<int>(r & 31);
    const int64_t o = soff[s];
    const int W = static_cast<int>((soff[s + 1] - o) >> 5);
    const int32_t b = r < n ? rp[r] : 0, len = r < n ? rp[r + 1] - b : 0;
    for (int k = 0; k < W; ++k) {
        const int64_t d = o + static_cast<int64_t>(k) * 32 + lane;
        scol[d] = k < len ? col[b + k] : -1;
        sval[d] = k < len ? val[b + k] : 0.0;
    }
}

static void u1_sell_setup(ktb_plan* p, bool force_uniform = false) {
    const ktb_matrix* m = p->m;
    const int64_t slices = ceil_div64(m->n, 32);
    p->sell_off.alloc(slices + 1);
    k_sell_width<<<ceil_div(slices + 1, 256), 256, 0, p->stream>>>(m->row_ptr.p, m->n, slices,
                                                                     p->sell_off.p);
    KTB_LAUNCH();
    // uniform width (ELL: slice offsets implicit, one dependent load fewer per
    // warp) when it costs at most 1/16 more than the per-slice widths
    DBuf<int64_t> stats(2);
    size_t tmp = 0, tmp2 = 0;
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, p->sell_off.p, p->sell_off.p,
                                           slices + 1, p->stream));
    KTB_CUDA(cub::DeviceReduce::Max(nullptr, tmp2, p->sell_off.p, stats.p, slices, p->stream));
    DBuf<unsigned char> scratch(std::max(tmp, tmp2));
    KTB_CUDA(cub::DeviceReduce::Max(scratch.p, tmp2, p->sell_off.p, stats.p, slices, p->stream));
    KTB_CUDA(cub::DeviceReduce::Sum(nullptr, tmp2, p->sell_off.p, stats.p + 1, slices, p->stream));
    if (tmp2 > scratch.n) scratch.alloc(tmp2);
    KTB_CUDA(cub::DeviceReduce::Sum(scratch.p, tmp2, p->sell_off.p, stats.p + 1, slices, p->stream));
    int64_t st[2] = {0, 0};
    KTB_CUDA(cudaMemcpyAsync(st, stats.p, sizeof(st), cudaMemcpyDeviceToHost, p->stream));
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    p->ell_width = 0;
    if (force_uniform && st[0] > 32 * 32)
        throw Invalid("u1: coded slices need one slice width <= 32");
    // (the pair-coded records take one width whatever it costs: a padding
    // slot is one byte there)
    if (st[0] > 0 && (force_uniform || st[0] * slices <= st[1] + st[1] / 16)) {
        p->ell_width = static_cast<int>(st[0] / 32);
        k_fill_i64<<<ceil_div(slices, 256), 256, 0, p->stream>>>(p->sell_off.p, slices, st[0]);
        KTB_LAUNCH();
    }
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, p->sell_off.p, p->sell_off.p,
                                           slices + 1, p->stream));
    int64_t padded = 0;
    KTB_CUDA(cudaMemcpyAsync(&padded, p->sell_off.p + slices, sizeof(int64_t),
                             cudaMemcpyDeviceToHost, p->stream));
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    if (padded > 3 * m->nnz + 256 * slices)
        throw Invalid("u1: warp-sliced layout would more than triple the matrix");
    p->sell_col.alloc(padded);
    p->sell_val.alloc(padded);
    k_sell_fill<<<ceil_div(slices * 32, 256), 256, 0, p->stream>>>(
        m->row_ptr.p, m->col.p, m->val.p, m->n, p->sell_off.p, p->sell_col.p, p->sell_val.p);
    KTB_LAUNCH();
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    p->extra_bytes = (p->ell_width ? 0 : 8 * (slices + 1)) + 12 * (padded - m->nnz) - 4 * (m->n + 1);
}

// U1 param 102: per slice, the dictionary of column deltas and the 4-bit
// codes, from the warp-sliced copy (one warp per slice). A slice needing more
// than 15 distinct deltas refuses the whole layout (the selector then skips
// the candidate; random-column matrices such as config 3).
__global__ void k_dict_build(const int64_t* __restrict__ soff, const int32_t* __restrict__ scol,
                             int64_t slices, int ell, uint32_t* __restrict__ codes,
                             int32_t* __restrict__ dict, int* __restrict__ overflow) {
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= slices) return;  // whole warps
    int64_t o;
    int W;
    if (ell) {
        o = s * 32 * ell;
        W = ell;
    } else {
        o = soff[s];
        W = static_cast<int>((soff[s + 1] - o) >> 5);
    }
    const int32_t row = static_cast<int32_t>(s * 32 + lane);
    int32_t dv = 0;  // lane j < count: delta j
    int count = 0;
    bool ok = true;
    for (int k = 0; k < W; ++k) {
        const int32_t c = scol[o + static_cast<int64_t>(k) * 32 + lane];
        const int32_t d = c - row;
        int code = 15;
        unsigned pending = __ballot_sync(0xffffffffu, c >= 0);
        while (pending) {
            const int src = __ffs(pending) - 1;
            const int32_t want = __shfl_sync(0xffffffffu, d, src);
            const unsigned same = __ballot_sync(0xffffffffu, c >= 0 && d == want);
            const unsigned hit = __ballot_sync(0xffffffffu, lane < count && dv == want);
            int j;
            if (hit) {
                j = __ffs(hit) - 1;
            } else if (count < 15) {
                j = count++;
                if (lane == j) dv = want;
            } else {
                j = 15;
                ok = false;
            }
            if ((same >> lane) & 1u) code = j;
            pending &= ~same;
        }
        // 8 codes per word: lane 8g+i contributes bits 4i..4i+3 of word g
        uint32_t part = static_cast<uint32_t>(code & 15) << ((lane & 7) * 4);
        for (int sh = 1; sh < 8; sh <<= 1) part |= __shfl_xor_sync(0xffffffffu, part, sh);
        if ((lane & 7) == 0) codes[(o >> 3) + static_cast<int64_t>(k) * 4 + (lane >> 3)] = part;
    }
    if (lane < 16) dict[s * 16 + lane] = lane < count ? dv : 0;
    if (!ok && lane == 0) atomicOr(overflow, 1);
}

static void u1_dict_setup(ktb_plan* p) {
    const int64_t slices = ceil_div64(p->m->n, 32);
    const int64_t padded = static_cast<int64_t>(p->sell_col.n);
    p->sell_codes.alloc(std::max<int64_t>(padded / 8, 1));
    p->sell_dict.alloc(std::max<int64_t>(slices * 16, 1));
    DBuf<int> overflow(1);
    KTB_CUDA(cudaMemsetAsync(overflow.p, 0, sizeof(int), p->stream));
    k_dict_build<<<ceil_div(slices * 32, 256), 256, 0, p->stream>>>(
        p->sell_off.p, p->sell_col.p, slices, p->ell_width, p->sell_codes.p, p->sell_dict.p,
        overflow.p);
    KTB_LAUNCH();
    int ov = 0;
    KTB_CUDA(cudaMemcpyAsync(&ov, overflow.p, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    if (ov) throw Invalid("u1: a warp slice needs more than 15 distinct column deltas");
    p->sell_col.release();  // the codes replace the columns
    // 0.5 B of code per slot + 64 B of dictionary per slice instead of 4 B columns
    p->extra_bytes += static_cast<int64_t>(padded / 2 + 64 * slices) - 4 * padded;
}

// U1 param 106: the slice records (pair dictionary + code words) from the
// ELL copy; they replace both the columns and the values.
static void u1_vrec_setup(ktb_plan* p) {
    const int64_t slices32 = ceil_div64(p->m->n, 32), recs = ceil_div64(p->m->n, 64);
    const int W = p->ell_width;
    DBuf<int> maxp(1);
    KTB_CUDA(cudaMemsetAsync(maxp.p, 0, sizeof(int), p->stream));
    const int grid = ceil_div(recs * 32, 256);
    k_vrec_build<<<grid, 256, 0, p->stream>>>(p->sell_col.p, p->sell_val.p, slices32, recs, W, 0,
                                              0, nullptr, maxp.p);
    KTB_LAUNCH();
    int mp = 0;
    KTB_CUDA(cudaMemcpyAsync(&mp, maxp.p, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    if (mp + 1 > kU1vMaxDict)
        throw Invalid("u1: 64 rows need more than 63 distinct (column delta, value) pairs");
    const U1vLayout L = u1v_layout(mp, W);
    p->rec_dict = L.dict;
    p->rec_words = L.words;
    p->rec_bytes = L.rec;
    p->rec_stride = L.stride;
    p->rec_stages = L.stages;
    p->sell_rec.alloc(std::max<int64_t>(recs, 1) * L.rec);
    k_vrec_build<<<grid, 256, 0, p->stream>>>(p->sell_col.p, p->sell_val.p, slices32, recs, W,
                                              L.dict, L.rec, p->sell_rec.p, maxp.p);
    KTB_LAUNCH();
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    const int64_t padded = static_cast<int64_t>(p->sell_col.n);
    p->sell_col.release();
    p->sell_val.release();
    // one record per 64 rows instead of the warp-sliced copy's 12 B per slot
    p->extra_bytes += recs * L.rec - 12 * padded;
}

// U1 param 101: rows of length <= kSortedCap sorted by length (descending,
// stable) into warp slices -- near-uniform slice widths for any row-length
// distribution; longer rows go to a compact sub-matrix reduced by U2 warp
// tiles into long_y and scattered into y. Row sums of the sliced rows keep
// the reference's left-to-right order; the long rows' carry the tiles' order.
constexpr int32_t kSortedCap = 256;
static void u1_sorted_setup(ktb_plan* p) {
    const ktb_matrix* m = p->m;
    const int64_t n = m->n;
    cudaStream_t st = p->stream;
    DBuf<int32_t> key(n), row(n), skey(n), srow(n);
    k_sort_keys<<<ceil_div(n, 256), 256, 0, st>>>(m->row_ptr.p, n, kSortedCap, key.p, row.p);
    KTB_LAUNCH();
    size_t tmp = 0;
    KTB_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, key.p, skey.p, row.p,
                                                       srow.p, n, 0, 32, st));
    DBuf<unsigned char> scratch(tmp);
    KTB_CUDA(cub::DeviceRadixSort::SortPairsDescending(scratch.p, tmp, key.p, skey.p, row.p,
                                                       srow.p, n, 0, 32, st));
    // short rows: the sorted prefix with key >= 0 (binary search on the device)
    DBuf<int64_t> d_ns(1);
    k_count_nonneg_sorted<<<1, 1, 0, st>>>(skey.p, n, d_ns.p);
    KTB_LAUNCH();
    int64_t ns = 0;
    KTB_CUDA(cudaMemcpyAsync(&ns, d_ns.p, 8, cudaMemcpyDeviceToHost, st));
    KTB_CUDA(cudaStreamSynchronize(st));
    const int64_t nl = n - ns;
    const int64_t slices = std::max<int64_t>(1, ceil_div64(ns, 32));
    p->sell_off.alloc(slices + 1);
    k_sorted_width<<<ceil_div(slices + 1, 256), 256, 0, st>>>(skey.p, ns, slices, p->sell_off.p);
    KTB_LAUNCH();
    if (ns == 0) KTB_CUDA(cudaMemsetAsync(p->sell_off.p, 0, 8 * (slices + 1), st));
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, p->sell_off.p, p->sell_off.p,
                                           slices + 1, st));
    if (tmp > scratch.n) scratch.alloc(tmp);
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, p->sell_off.p, p->sell_off.p,
                                           slices + 1, st));
    int64_t padded = 0;
    KTB_CUDA(cudaMemcpyAsync(&padded, p->sell_off.p + slices, 8, cudaMemcpyDeviceToHost, st));
    KTB_CUDA(cudaStreamSynchronize(st));
    p->sell_col.alloc(std::max<int64_t>(padded, 1));
    p->sell_val.alloc(std::max<int64_t>(padded, 1));
    p->sell_perm.alloc(slices * 32);
    k_sorted_fill<<<ceil_div(slices * 32, 256), 256, 0, st>>>(
        m->row_ptr.p, m->col.p, m->val.p, srow.p, ns, slices, p->sell_off.p, p->sell_perm.p,
        p->sell_col.p, p->sell_val.p);
    KTB_LAUNCH();
    p->ell_width = 0;
    int64_t long_nnz = 0;
    if (nl > 0) {
        p->long_rows.alloc(nl);
        KTB_CUDA(cudaMemcpyAsync(p->long_rows.p, srow.p + ns, 4 * nl, cudaMemcpyDeviceToDevice, st));
        auto* lm = new ktb_matrix();
        p->long_m = lm;
        lm->device = m->device;
        lm->n = nl;
        lm->ncols = m->ncols;
        lm->kind = KTB_GENERAL;
        lm->sm_count = m->sm_count;
        lm->row_ptr.alloc(nl + 1);
        k_long_counts<<<ceil_div(nl + 1, 256), 256, 0, st>>>(m->row_ptr.p, p->long_rows.p, nl,
                                                             lm->row_ptr.p);
        KTB_LAUNCH();
        KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, lm->row_ptr.p, lm->row_ptr.p, nl + 1,
                                               st));
        if (tmp > scratch.n) scratch.alloc(tmp);
        KTB_CUDA(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, lm->row_ptr.p, lm->row_ptr.p,
                                               nl + 1, st));
        int32_t lnnz = 0;
        KTB_CUDA(cudaMemcpyAsync(&lnnz, lm->row_ptr.p + nl, 4, cudaMemcpyDeviceToHost, st));
        KTB_CUDA(cudaStreamSynchronize(st));
        lm->nnz = long_nnz = lnnz;
        lm->col.alloc(lnnz);
        lm->val.alloc(lnnz);
        k_long_copy<<<static_cast<int>(nl), 256, 0, st>>>(m->row_ptr.p, m->col.p, m->val.p,
                                                          p->long_rows.p, lm->row_ptr.p, lm->col.p,
                                                          lm->val.p);
        KTB_LAUNCH();
        KTB_CUDA(cudaStreamSynchronize(st));
        auto* lp = new ktb_plan();
        p->long_plan = lp;
        lp->m = lm;
        lp->kernel = KTB_U2;
        lp->param = 8;
        lp->workers = p->workers;
        lp->stream = st;
        plan_setup(lp);
        p->long_y.alloc(nl);
        KTB_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
        KTB_CUDA(cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming));
        KTB_CUDA(cudaEventCreateWithFlags(&p->join, cudaEventDisableTiming));
    }
    KTB_CUDA(cudaStreamSynchronize(st));
    // vs the model: padding slots, perm (4 B/slot) instead of row_ptr, the
    // long rows' tile bookkeeping and their y round trip
    p->extra_bytes = 12 * (padded + long_nnz - m->nnz) + 4 * (slices * 32) - 4 * (m->n + 1) +
                     (p->long_plan ? p->long_plan->extra_bytes + 16 * nl : 0);
}

static int pick_lanes(const ktb_matrix* m) {
    const double mean = m->n ? static_cast<double>(m->nnz) / static_cast<double>(m->n) : 1.0;
    int v = 1;
    while (v < 32 && v < mean) v <<= 1;
    return v;
}

void u1_setup(ktb_plan* p) {
    require(p->cta_threads == 0 ||
                ((p->param == 100 || p->param == 101 || p->param == 102) &&
                 (p->cta_threads == 64 || p->cta_threads == 128 || p->cta_threads == 256)),
            "u1: only the warp-sliced forms (params 100, 101) take a CTA shape: 64, 128 or 256 "
            "threads");
    {  // KTB_U1S_XPF=0 turns the x prefetch off (A/B measurements)
        const char* e = std::getenv("KTB_U1S_XPF");
        p->x_prefetch = !(e && e[0] == '0');
    }
    if (p->param == 100) {
        u1_sell_setup(p);
        p->launches = 1;
        return;
    }
    if (p->param == 102) {
        u1_sell_setup(p);
        u1_dict_setup(p);
        p->launches = 1;
        return;
    }
    if (p->param == 106) {  // persistent slices, coded (column delta, value) pairs
        require(p->cta_threads == 0, "u1: the staged slices run 256-thread CTAs");
        u1_sell_setup(p, true);
        if (p->ell_width < 1 || p->ell_width > 32)
            throw Invalid("u1: coded slices need one slice width <= 32");
        u1_vrec_setup(p);
        const U1vLayout L = u1v_layout(p->rec_dict - 1, p->ell_width);
        const int smem = u1v_smem(L);
        const U1vFn fn = u1v_kernel(p->ell_width);
        allow_max_dynamic_smem(fn);
        int occ = 0;
        KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kU1vWarps * 32, smem));
        p->ctas = static_cast<int64_t>(std::max(occ, 1)) * p->m->sm_count;
        p->launches = 1;
        return;
    }
    if (p->param == 105) {  // persistent coded slices staged by per-warp bulk copies
        require(p->cta_threads == 0, "u1: the staged slices run 256-thread CTAs");
        u1_sell_setup(p);
        if (p->ell_width < 1 || p->ell_width > 8)
            throw Invalid("u1: staged slices need one slice width <= 8");
        if ((reinterpret_cast<uintptr_t>(p->sell_val.p) & 15) != 0)
            throw Invalid("u1: staged slices need 16-byte aligned values");
        u1_dict_setup(p);
        const int smem = u1t_smem(p->ell_width);
        allow_max_dynamic_smem(k_u1t);
        int occ = 0;
        KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_u1t, kU1tWarps * 32, smem));
        p->ctas = static_cast<int64_t>(std::max(occ, 1)) * p->m->sm_count;
        p->launches = 1;
        return;
    }
    if (p->param == 103 || p->param == 104) {  // persistent pipelined slices (ELL, W <= 8)
        require(p->cta_threads == 0, "u1: the persistent slices run 256-thread CTAs");
        u1_sell_setup(p);
        if (p->ell_width < 1 || p->ell_width > 8)
            throw Invalid("u1: persistent slices need one slice width <= 8");
        if (p->param == 104) u1_dict_setup(p);
        int occ = 0;
        if (p->param == 104)
            KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_u1p<true>, 256, 0));
        else
            KTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_u1p<false>, 256, 0));
        p->ctas = static_cast<int64_t>(std::max(occ, 1)) * p->m->sm_count;
        p->launches = 1;
        return;
    }
    if (p->param == 101) {
        u1_sorted_setup(p);
        p->launches = 1 + (p->long_plan ? p->long_plan->launches + 1 : 0);
        return;
    }
    if (p->param <= 0) p->param = pick_lanes(p->m);
    int v = 1;
    while (v < p->param && v < 32) v <<= 1;
    p->param = v;
    p->launches = 1;
}

// k_u1s over `threads` slice lanes in the plan's CTA shape
static void launch_u1s(ktb_plan* p, int64_t threads, const int64_t* soff, const double* x,
                       double* y, int32_t r0, int32_t r1, int ell, const int32_t* perm) {
    const int t = p->cta_threads ? p->cta_threads : kU1sThreads;
    // x prefetch: row-ordered slices only (the sorted form permutes rows)
    const int64_t xpf = (!perm && p->x_prefetch) ? p->m->col_shift : -1;
    const int64_t xlen = p->m->ncols;
    const int grid = ceil_div(threads, t);
    p->ctas = grid;
    const bool dict = p->param == 102;
#define KTB_U1S_LAUNCH(T, D)                                                                   \
    k_u1s<T, D><<<grid, T, 0, p->stream>>>(soff, p->sell_col.p, p->sell_val.p, x, y, r0, r1,    \
                                           ell, perm, xpf, xlen, p->sell_codes.p,             \
                                           p->sell_dict.p)
    switch (t * 2 + (dict ? 1 : 0)) {
        case 128: KTB_U1S_LAUNCH(64, false); break;
        case 129: KTB_U1S_LAUNCH(64, true); break;
        case 256: KTB_U1S_LAUNCH(128, false); break;
        case 257: KTB_U1S_LAUNCH(128, true); break;
        case 512: KTB_U1S_LAUNCH(256, false); break;
        case 513: KTB_U1S_LAUNCH(256, true); break;
        default: throw Invalid("u1: warp-sliced CTAs are 64, 128 or 256 threads");
    }
#undef KTB_U1S_LAUNCH
    KTB_LAUNCH();
}

void u1_run(ktb_plan* p, const double* x, double* y, int64_t r0, int64_t r1) {
    const int64_t rows = r1 - r0;
    if (rows <= 0) return;
    if (p->param == 101) {  // whole matrix (spmv_rows refuses 101)
        // the long rows (U2 tiles on the sub-matrix, then a scatter into y) run
        // on a side stream forked from and joined back to the plan's stream:
        // they overlap the slice kernel (disjoint rows of y, x read-only)
        if (p->long_plan) {
            KTB_CUDA(cudaEventRecord(p->fork, p->stream));
            KTB_CUDA(cudaStreamWaitEvent(p->side, p->fork, 0));
            p->long_plan->stream = p->side;
            plan_run(p->long_plan, x, p->long_y.p, 0, p->long_plan->m->n);
            const int64_t nl = p->long_plan->m->n;
            k_scatter_rows<<<ceil_div(nl, 256), 256, 0, p->side>>>(p->long_y.p, p->long_rows.p,
                                                                    nl, y);
            KTB_LAUNCH();
            KTB_CUDA(cudaEventRecord(p->join, p->side));
        }
        const int64_t slices = static_cast<int64_t>(p->sell_off.n) - 1;
        launch_u1s(p, slices * 32, p->sell_off.p, x, y, 0, static_cast<int32_t>(slices * 32), 0,
                   p->sell_perm.p);
        if (p->long_plan) KTB_CUDA(cudaStreamWaitEvent(p->stream, p->join, 0));
        return;
    }
    if (p->param == 106) {
        const int64_t recs = ceil_div64(r1, 64) - (r0 >> 6);
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(p->ctas, ceil_div64(recs, kU1vWarps))));
        const U1vLayout L = u1v_layout(p->rec_dict - 1, p->ell_width);
        u1v_kernel(p->ell_width)<<<grid, kU1vWarps * 32, u1v_smem(L), p->stream>>>(
            p->sell_rec.p, x, y, static_cast<int32_t>(r0), static_cast<int32_t>(r1),
            static_cast<int32_t>(p->m->n), static_cast<int32_t>(p->m->ncols), 16 * L.dict, L.rec,
            L.stride, L.stages);
        KTB_LAUNCH();
        return;
    }
    if (p->param == 105) {
        const int64_t slices = ceil_div64(r1, 32) - (r0 >> 5);
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(p->ctas, ceil_div64(slices, kU1tWarps))));
        k_u1t<<<grid, kU1tWarps * 32, u1t_smem(p->ell_width), p->stream>>>(
            p->sell_val.p, p->sell_codes.p, p->sell_dict.p, x, y, static_cast<int32_t>(r0),
            static_cast<int32_t>(r1), p->ell_width, u1t_stage_bytes(p->ell_width));
        KTB_LAUNCH();
        return;
    }
    if (p->param == 103 || p->param == 104) {
        const int64_t slices = ceil_div64(r1, 32) - (r0 >> 5);
        const int grid = static_cast<int>(std::max<int64_t>(
            1, std::min<int64_t>(p->ctas, ceil_div64(slices, 8))));
        if (p->param == 104)
            k_u1p<true><<<grid, 256, 0, p->stream>>>(nullptr, p->sell_val.p, p->sell_codes.p,
                                                     p->sell_dict.p, x, y, static_cast<int32_t>(r0),
                                                     static_cast<int32_t>(r1), p->ell_width);
        else
            k_u1p<false><<<grid, 256, 0, p->stream>>>(p->sell_col.p, p->sell_val.p, nullptr,
                                                      nullptr, x, y, static_cast<int32_t>(r0),
                                                      static_cast<int32_t>(r1), p->ell_width);
        KTB_LAUNCH();
        return;
    }
    if (p->param == 100 || p->param == 102) {
        const int64_t s0 = r0 >> 5, s1 = ceil_div64(r1, 32);
        launch_u1s(p, (s1 - s0) * 32, p->sell_off.p, x, y, static_cast<int32_t>(r0),
                   static_cast<int32_t>(r1), p->ell_width, nullptr);
        return;
    }
    const int V = static_cast<int>(p->param);
#ifndef KTB_U1_R
#define KTB_U1_R 4
#endif
    constexpr int R = KTB_U1_R;
    const int64_t threads = ceil_div64(rows, R) * V;
    const int grid = ceil_div(threads, 256);
    p->ctas = grid;
    const ktb_matrix* m = p->m;
#define KTB_U1_CASE(VV)                                                                        \
    case VV:                                                                                    \
        k_u1<VV, R><<<grid, 256, 0, p->stream>>>(m->row_ptr.p, m->col.p, m->val.p, x, y,       \
                                                 static_cast<int32_t>(r0),                      \
                                                 static_cast<int32_t>(r1));                     \
        break;
    switch (V) {
        KTB_U1_CASE(1)
        KTB_U1_CASE(2)
        KTB_U1_CASE(4)
        KTB_U1_CASE(8)
        KTB_U1_CASE(16)
        KTB_U1_CASE(32)
        default: throw Invalid("u1: bad lane count");
    }
#undef KTB_U1_CASE
    KTB_LAUNCH();
}

// =============================================================== carries
// Tile carries (row, value) in tile order; the rows are non-decreasing, so
// the tiles carrying one row form a run. One thread per tile: the tile's row
// and its neighbours' go out in one round trip; a tile that is a run by itself
// (almost all of them: a run of L tiles needs a row of > 256 (L - 1)
// nonzeros) adds its carry to y at once. The longer runs starting in a warp
// are then summed by the whole warp one after the other, 32 carries at a time
// (lane-strided partial sums, then a fixed shuffle tree: deterministic), and
// added to y once: a run of L tiles costs L/32 dependent rounds (a
// 65,536-long row spans 256 tiles: 8), where a serial walk cost L.
__global__ void __launch_bounds__(256) k_fixup_carries(const int32_t* __restrict__ crow,
                                                       const double* __restrict__ cval,
                                                       int64_t tiles, int64_t n,
                                                       double* __restrict__ y) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool in = t < tiles;
    const int32_t r = in ? __ldg(crow + t) : -1;
    const int32_t prev = in && t > 0 ? __ldg(crow + t - 1) : -1;
    const int32_t next = in && t + 1 < tiles ? __ldg(crow + t + 1) : -1;
    const double cv = in ? __ldg(cval + t) : 0.0;
    const bool start = r >= 0 && r < n && prev != r;  // the run's first tile
    if (start && next != r) y[r] += cv;
    unsigned longer = __ballot_sync(0xffffffffu, start && next == r);
    while (longer) {
        const int src = __ffs(longer) - 1;
        longer &= longer - 1;
        const int64_t t0 = __shfl_sync(0xffffffffu, t, src);
        const int32_t rr = __shfl_sync(0xffffffffu, r, src);
        double acc = 0.0;
        for (int64_t u0 = t0;; u0 += 32) {
            const int64_t u = u0 + lane;
            const bool same = u < tiles && __ldg(crow + u) == rr;
            if (same) acc += __ldg(cval + u);
            if (__ballot_sync(0xffffffffu, same) != 0xffffffffu) break;
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[rr] += acc;
    }
}

static void fixup_run(ktb_plan* p, double* y) {
    k_fixup_carries<<<ceil_div(p->tiles, 256), 256, 0, p->stream>>>(
        p->carry_row.p, p->carry_val.p, p->tiles, p->m->n, y);
    KTB_LAUNCH();
}

// =============================================================== U2
constexpr int kU2Threads = 256;

// Merge-path search along the diagonal `diag` of the (row ends, nz indices)
// merge: returns the number of row ends consumed.
__device__ __forceinline__ int64_t merge_search(const int32_t* __restrict__ row_end, int64_t n,
                                                int64_t nnz, int64_t diag) {
    int64_t lo = diag > nnz ? diag - nnz : 0;
    int64_t hi = diag < n ? diag : n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(row_end[mid]) <= diag - mid - 1)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

__global__ void k_u2_coords(const int32_t* __restrict__ rp, int64_t n, int64_t nnz,
                            int64_t tile_items, int64_t tiles, MergeCoord* coords) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t > tiles) return;
    const int64_t diag = min(t * tile_items, n + nnz);
    const int64_t r = merge_search(rp + 1, n, nnz, diag);
    coords[t].row = static_cast<int32_t>(r);
    coords[t].nz = static_cast<int32_t>(diag - r);
}

template <int IPT>
__global__ void __launch_bounds__(kU2Threads) k_u2(const int32_t* __restrict__ rp,
                                                   const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y,
                                                   const MergeCoord* __restrict__ coords,
                                                   int32_t* __restrict__ carry_row,
                                                   double* __restrict__ carry_val) {
    constexpr int TILE = kU2Threads * IPT;
    __shared__ double s_prod[TILE];
    __shared__ int32_t s_end[TILE + 1];
    const int tid = threadIdx.x;
    const MergeCoord c0 = coords[blockIdx.x], c1 = coords[blockIdx.x + 1];
    const int nrows = c1.row - c0.row;
    const int nnzs = c1.nz - c0.nz;
    // stage products (coalesced): all column/value loads of the thread first,
    // then all x gathers, then the products -> IPT independent chains per thread
    {
        int32_t cc[IPT];
        double vv[IPT];
#pragma unroll
        for (int u = 0; u < IPT; ++u) {
            const int i = u * kU2Threads + tid;
            cc[u] = i < nnzs ? ld_stream_i32(col + c0.nz + i) : -1;
            vv[u] = i < nnzs ? ld_stream_f64(val + c0.nz + i) : 0.0;
        }
        double xv[IPT];
#pragma unroll
        for (int u = 0; u < IPT; ++u) xv[u] = cc[u] >= 0 ? ld_x(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < IPT; ++u) {
            const int i = u * kU2Threads + tid;
            if (i < nnzs) s_prod[i] = vv[u] * xv[u];
        }
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int i = u * kU2Threads + tid;
        if (i < nrows) s_end[i] = ldg_i32(rp + c0.row + 1 + i);
    }
    if (tid == 0) s_end[nrows] = 0x7fffffff;  // the open row at tile end never closes here
    KTB_SYNC();

    // this thread's merge-path start inside the tile
    const int diag = min(tid * IPT, nrows + nnzs);
    int lo = max(diag - nnzs, 0), hi = min(diag, nrows);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s_end[mid] - c0.nz <= diag - mid - 1)
            lo = mid + 1;
        else
            hi = mid;
    }
    int xr = lo, yz = diag - lo;
    const int end_items = nrows + nnzs;
    double run = 0.0;
    double emit_v[IPT];
    int emit_r[IPT];
    int nemit = 0;
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        emit_r[it] = -1;
        emit_v[it] = 0.0;
        if (xr + yz < end_items) {
            if (c0.nz + yz < s_end[xr]) {
                run += s_prod[yz];
                ++yz;
            } else {
                emit_r[it] = xr;
                emit_v[it] = run;
                ++nemit;
                run = 0.0;
                ++xr;
            }
        }
    }
    SegPair agg;
    const SegPair pre = block_seg_scan_excl<kU2Threads>(SegPair{nemit > 0, run}, &agg);
    KTB_SYNC();  // s_prod is reused for row outputs below
    bool first = true;
#pragma unroll
    for (int it = 0; it < IPT; ++it) {
        if (emit_r[it] >= 0) {
            s_prod[emit_r[it]] = emit_v[it] + (first ? pre.v : 0.0);
            first = false;
        }
    }
    KTB_SYNC();
    for (int i = tid; i < nrows; i += kU2Threads) y[c0.row + i] = s_prod[i];
    if (tid == 0) {
        carry_row[blockIdx.x] = c1.row;
        carry_val[blockIdx.x] = agg.v;
    }
}

// ---- U2, warp tiles --------------------------------------------------------
// Each warp owns T = 32*IPT consecutive nonzeros [z0, z0+T) (nnz-balanced)
// and the rows whose end falls in (z0, z0+T] (wrow[w] .. wrow[w+1]). No
// block-level synchronisation: the 8 warps of a CTA are independent.
//   1. striped, coalesced col/val loads; x gathers (all IPT in flight);
//   2. meanwhile the row ends of the tile become a T-bit mask (smem, one
//      atomicOr per row) plus the ordinal -> row list; empty rows get y = 0;
//   3. products go to a padded per-warp smem buffer (stride IPT+2 doubles,
//      so the blocked 16-byte reads below are bank-conflict free) and each
//      thread sums its IPT consecutive products, emitting every row that
//      ends inside them;
//   4. the head segment of each thread takes the carry of the lanes before
//      it: one flag-aware warp scan (the flags are the ballot of "has an
//      end", so only the value is shuffled);
//   5. the open row at the tile end is the tile carry (k_fixup_carries).
#ifndef KTB_U2W_MINB
#define KTB_U2W_MINB 5
#endif
// CTA shape: 4 warps by default (8: 4 % slower on config 3); both shapes are
// instantiated and the selector times them (launch-shape candidates).
template <int IPT, int kTileWarps>
__global__ void __launch_bounds__(32 * kTileWarps, KTB_U2W_MINB * 8 / kTileWarps) k_u2w(const int32_t* __restrict__ rp,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ x,
                                                          double* __restrict__ y,
                                                          const int32_t* __restrict__ wrow,
                                                          int64_t nnz, int64_t tiles,
                                                          int32_t* __restrict__ carry_row,
                                                          double* __restrict__ carry_val) {
    constexpr int T = 32 * IPT;
    static_assert(IPT == 4 || IPT == 8, "u2w: IPT");
    // thread b's IPT products are b's row of the buffer; its 16-byte chunks
    // are XOR-swizzled by the row's position among the rows sharing a 128-byte
    // line (b >> SH), so the striped 8-byte stores and the blocked 16-byte
    // loads are both bank-conflict free
    constexpr int SH = IPT == 8 ? 1 : 2;
    // s_end: 16-byte chunks of 4 ints, IPT/4 per thread row, 32/IPT rows per
    // 128-byte line -> chunk swizzle by (b >> ESH)
    constexpr int ESH = IPT == 8 ? 2 : 3;
    constexpr int EMASK = IPT / 4 - 1;
    __shared__ __align__(16) double s_prod[kTileWarps][T];
    // s_end[i] = 1 + row ending at item i of the tile, 0 = no row ends there
    __shared__ __align__(16) int32_t s_end[kTileWarps][T];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kTileWarps + warp;
    if (w >= tiles) return;
    const int64_t z0 = w * T;
    const int cnt = static_cast<int>(nnz - z0 < T ? nnz - z0 : T);
    const int32_t ra = __ldg(wrow + w), rb = __ldg(wrow + w + 1);
#pragma unroll
    for (int q = 0; q < IPT; q += 4) {  // own row, in the swizzled chunk order (conflict-free)
        const int phys = ((q >> 2) ^ ((lane >> ESH) & EMASK)) << 2;
        *reinterpret_cast<int4*>(&s_end[warp][lane * IPT + phys]) = make_int4(0, 0, 0, 0);
    }

    int32_t c[IPT];
    double v[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int i = u * 32 + lane;
        c[u] = i < cnt ? ld_stream_i32(col + z0 + i) : -1;
        v[u] = i < cnt ? ld_stream_f64(val + z0 + i) : 0.0;
    }
    // first 32 row bounds in flight together with the gathers
    bool in = ra + lane < rb;
    int32_t rb_ = in ? __ldg(rp + ra + lane) : 0;
    int32_t re_ = in ? __ldg(rp + ra + lane + 1) : 0;
    double xv[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) xv[u] = c[u] >= 0 ? ld_x(x + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const int i = u * 32 + lane;
        const int b = i / IPT, j = i % IPT;
        s_prod[warp][b * IPT + ((((j >> 1) ^ ((b >> SH) & (IPT / 2 - 1))) << 1) | (j & 1))] =
            v[u] * xv[u];
    }
    __syncwarp();  // s_end zeroed before the scatter below
    for (int32_t r0 = ra;;) {
        const int32_t r = r0 + lane;
        if (in) {
            if (re_ > rb_) {
                const int i = static_cast<int>(re_ - 1 - z0);
                const int b = i / IPT, j = i % IPT;
                s_end[warp][b * IPT + ((((j >> 2) ^ ((b >> ESH) & EMASK)) << 2) | (j & 3))] = r + 1;
            }
            else
                y[r] = 0.0;  // empty row
        }
        r0 += 32;
        if (r0 >= rb) break;
        in = r0 + lane < rb;
        rb_ = in ? __ldg(rp + r0 + lane) : 0;
        re_ = in ? __ldg(rp + r0 + lane + 1) : 0;
    }
    __syncwarp();

    double p[IPT];
#pragma unroll
    for (int cc = 0; cc < IPT / 2; ++cc) {
        const int phys = (cc ^ ((lane >> SH) & (IPT / 2 - 1))) << 1;
        const double2 q = *reinterpret_cast<const double2*>(&s_prod[warp][lane * IPT + phys]);
        p[2 * cc] = q.x;
        p[2 * cc + 1] = q.y;
    }
    int32_t er[IPT];
#pragma unroll
    for (int q = 0; q < IPT; q += 4) {
        const int phys = ((q >> 2) ^ ((lane >> ESH) & EMASK)) << 2;
        const int4 e4 = *reinterpret_cast<const int4*>(&s_end[warp][lane * IPT + phys]);
        er[q] = e4.x;
        er[q + 1] = e4.y;
        er[q + 2] = e4.z;
        er[q + 3] = e4.w;
    }
    double run = 0.0, head = 0.0;
    int32_t head_row = 0;
    bool has = false;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        run += p[j];
        if (er[j]) {
            if (has) {
                y[er[j] - 1] = run;
            } else {
                head = run;
                head_row = er[j] - 1;
            }
            has = true;
            run = 0.0;
        }
    }
    // S(t) = tail_t + (has_t ? 0 : S(t-1)) over the lanes
    const uint32_t F = __ballot_sync(0xffffffffu, has);
    double S = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double up = __shfl_up_sync(0xffffffffu, S, d);
        if (lane >= d && ((F >> (lane - d + 1)) & ((1u << d) - 1u)) == 0u) S += up;
    }
    double cin = __shfl_up_sync(0xffffffffu, S, 1);
    if (lane == 0) cin = 0.0;
    if (has) y[head_row] = head + cin;
    if (lane == 31) {
        carry_row[w] = rb;
        carry_val[w] = S;
    }
}

// 32-byte streaming loads (sm_100 LDG.256): a lane's load is one whole sector,
// where two 16-byte loads of a lane-blocked layout fetch every sector twice
__device__ __forceinline__ void ld_stream_v8i32(const int32_t* p, int32_t* r) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.s32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p), "l"(pol_first()));
}
__device__ __forceinline__ void ld_stream_v4f64(const double* p, double* r) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
        : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3])
        : "l"(p), "l"(pol_first()));
}

// first row whose end lies beyond z = w*T (w = 0: row 0)
__global__ void k_u2w_rows(const int32_t* __restrict__ rp, int64_t n, int64_t nnz, int64_t T,
                           int64_t tiles, int32_t* __restrict__ wrow) {
    const int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (w > tiles) return;
    if (w == 0) {
        wrow[0] = 0;
        return;
    }
    const int64_t z = min(w * T, nnz);
    int64_t lo = 0, hi = n;  // first r in [0, n) with rp[r+1] > z, else n
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (static_cast<int64_t>(rp[mid + 1]) > z)
            hi = mid;
        else
            lo = mid + 1;
    }
    wrow[w] = static_cast<int32_t>(lo);
}

// param: 4 / 8 = warp tiles with that many items per thread (default 8);
// 104 / 108 / 112 = the merge-path kernel with IPT = param - 100.
// p->cta_threads: warp tiles in CTAs of 128 (default) or 256 threads.
void u2_setup(ktb_plan* p) {
    if (p->param <= 0) p->param = 8;
    const int prm = static_cast<int>(p->param);
    const ktb_matrix* m = p->m;
    if (prm == 4 || prm == 8) {
        require(p->cta_threads == 0 || p->cta_threads == 128 || p->cta_threads == 256,
                "u2: warp tiles run in CTAs of 128 or 256 threads");
        const int64_t T = 32 * prm;
        p->tiles = std::max<int64_t>(1, ceil_div64(m->nnz, T));
        p->wrow.alloc(p->tiles + 1);
        p->carry_row.alloc(p->tiles);
        p->carry_val.alloc(p->tiles);
        k_u2w_rows<<<ceil_div(p->tiles + 1, 256), 256, 0, p->stream>>>(
            m->row_ptr.p, m->n, m->nnz, T, p->tiles, p->wrow.p);
        KTB_LAUNCH();
        KTB_CUDA(cudaStreamSynchronize(p->stream));
        p->ctas = ceil_div64(p->tiles, p->cta_threads == 256 ? 8 : 4);
        p->launches = 2;
        p->extra_bytes = p->tiles * (4 + 4 + 8) * 2;
        return;
    }
    require(p->cta_threads == 0, "u2: the merge-path tiles have one CTA shape");
    int ipt = prm - 100;
    if (ipt != 4 && ipt != 8 && ipt != 12) ipt = 8;
    p->param = 100 + ipt;
    const int64_t tile_items = static_cast<int64_t>(kU2Threads) * ipt;
    p->tiles = std::max<int64_t>(1, ceil_div64(m->n + m->nnz, tile_items));
    p->coords.alloc(p->tiles + 1);
    p->carry_row.alloc(p->tiles);
    p->carry_val.alloc(p->tiles);
    k_u2_coords<<<ceil_div(p->tiles + 1, 256), 256, 0, p->stream>>>(
        m->row_ptr.p, m->n, m->nnz, tile_items, p->tiles, p->coords.p);
    KTB_LAUNCH();
    KTB_CUDA(cudaStreamSynchronize(p->stream));
    p->ctas = p->tiles;
    p->launches = 2;
    p->extra_bytes = p->tiles * (8 + 4 + 8) * 2;
}

void u2_run(ktb_plan* p, const double* x, double* y) {
    const ktb_matrix* m = p->m;
    const int prm = static_cast<int>(p->param);
    if (prm < 100) {
        const int warps = p->cta_threads == 256 ? 8 : 4;
        const int grid = static_cast<int>(ceil_div64(p->tiles, warps));
#define KTB_U2W_CASE(I, WW)                                                                   \
    if (prm == I && warps == WW)                                                               \
        k_u2w<I, WW><<<grid, 32 * WW, 0, p->stream>>>(m->row_ptr.p, m->col.p, m->val.p, x, y,  \
                                                      p->wrow.p, m->nnz, p->tiles,             \
                                                      p->carry_row.p, p->carry_val.p);
        KTB_U2W_CASE(4, 4)
        KTB_U2W_CASE(8, 4)
        KTB_U2W_CASE(4, 8)
        KTB_U2W_CASE(8, 8)
#undef KTB_U2W_CASE
        KTB_LAUNCH();
        fixup_run(p, y);
        return;
    }
    const int grid = static_cast<int>(p->tiles);
#define KTB_U2_CASE(I)                                                                       \
    case I:                                                                                   \
        k_u2<I><<<grid, kU2Threads, 0, p->stream>>>(m->row_ptr.p, m->col.p, m->val.p, x, y,   \
                                                    p->coords.p, p->carry_row.p,              \
                                                    p->carry_val.p);                          \
        break;
    switch (prm - 100) {
        KTB_U2_CASE(4)
        KTB_U2_CASE(8)
        KTB_U2_CASE(12)
        default: throw Invalid("u2: bad items per thread");
    }
#undef KTB_U2_CASE
    KTB_LAUNCH();
    fixup_run(p, y);
}

// =============================================================== U3 / U4
constexpr int kU3Threads = 256;

__global__ void k_flag_bits(const int32_t* __restrict__ rp, int64_t n, uint32_t* bits) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) {
        const int32_t s = rp[i];
        if (s < rp[i + 1]) atomicOr(&bits[s >> 5], 1u << (s & 31));
    }
}

__global__ void k_nonempty_mark(const int32_t* __restrict__ rp, int64_t n, int32_t* mark) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n) mark[i] = rp[i] < rp[i + 1];
}

__global__ void k_nonempty_scatter(const int32_t* __restrict__ rp, int64_t n,
                                   const int32_t* ord, int32_t* seg_row) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n && rp[i] < rp[i + 1]) seg_row[ord[i]] = static_cast<int32_t>(i);
}

// tile_q[t] = number of row starts before the tile's first nonzero
__global__ void k_tile_q(const uint32_t* __restrict__ bits, int64_t nnz, int64_t jl,
                         int64_t tiles, int32_t* tile_q) {
    // one block per tile; count set bits in [0, K0) with a strided popc reduction
    const int64_t t = blockIdx.x;
    if (t >= tiles) return;
    const int64_t K0 = nnz * (t * kU3Threads) / jl;
    const int64_t words = K0 >> 5;
    long long c = 0;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) c += __popc(bits[w]);
    if (threadIdx.x == 0 && (K0 & 31)) c += __popc(bits[words] & ((1u << (K0 & 31)) - 1u));
    using BR = cub::BlockReduce<long long, 256>;
    __shared__ typename BR::TempStorage tmp;
    const long long tot = BR(tmp).Sum(c);
    if (threadIdx.x == 0) tile_q[t] = static_cast<int32_t>(tot);
}

// ---- U3, warp-level BSS (param 1008) ---------------------------------------
// The branchless segmented scan as a flag-driven warp-level scan: a warp owns
// 256 consecutive nonzeros, lane b the 8 at [z0 + 8b, z0 + 8b + 8) (16-byte
// vector loads), whose row-start flags are one byte of the reference's
// row_start_flag bit array (bss.hpp:34-69). Segment ids come from the tile's
// flag prefix + a warp prefix of the lanes' popcounts; a flag closes the
// previous segment, whose row is seg_row[q] (the nonempty-row map). The run
// before a lane's first flag takes the carry of the lanes before it (one
// flag-aware warp scan, as k_u2w), the run open at the tile end is the tile
// carry (k_fixup_carries). Empty rows and the last nonempty row (never closed
// by a flag) are zeroed first by k_zero_rows (fused into the warps' work it
// measured 2-10 us slower on config 3).
__global__ void k_tile_pop(const uint32_t* __restrict__ bits, int64_t tiles,
                           int32_t* __restrict__ pop) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t > tiles) return;
    int c = 0;
    if (t < tiles)
        for (int k = 0; k < 8; ++k) c += __popc(bits[t * 8 + k]);
    pop[t] = c;
}

__global__ void k_zero_rows(const int32_t* __restrict__ rows, int64_t cnt, double* __restrict__ y) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < cnt) y[rows[i]] = 0.0;
}

__global__ void k_empty_list(const int32_t* __restrict__ rp, int64_t n,
                             const int32_t* __restrict__ ord, int32_t* __restrict__ out) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i < n && rp[i] == rp[i + 1]) out[i - ord[i]] = static_cast<int32_t>(i);  // ord = nonempty before i
}

template <int kTileWarps>
__global__ void __launch_bounds__(32 * kTileWarps, 32 / kTileWarps) k_u3w(const int32_t* __restrict__ col,
                                                 const double* __restrict__ val,
                                                 const double* __restrict__ x,
                                                 double* __restrict__ y, int64_t nnz,
                                                 int64_t tiles,
                                                 const uint32_t* __restrict__ bits,
                                                 const int32_t* __restrict__ seg_row,
                                                 const int32_t* __restrict__ wq,
                                                 int32_t* __restrict__ carry_row,
                                                 double* __restrict__ carry_val) {
    constexpr int IPT = 8, NS = 4;  // NS: segment rows fetched ahead per lane
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t w = static_cast<int64_t>(blockIdx.x) * kTileWarps + warp;
    if (w >= tiles) return;
    const int64_t z0 = w * 256, k0 = z0 + lane * IPT;
    int32_t c[IPT];
    double v[IPT];
    if (z0 + 256 <= nnz) {
        // 8 columns = one 32-byte sector, 8 values = two
        ld_stream_v8i32(col + k0, c);
        ld_stream_v4f64(val + k0, v);
        ld_stream_v4f64(val + k0 + 4, v + 4);
    } else {
#pragma unroll
        for (int j = 0; j < IPT; ++j) {
            const bool ok = k0 + j < nnz;
            c[j] = ok ? ld_stream_i32(col + k0 + j) : -1;
            v[j] = ok ? ld_stream_f64(val + k0 + j) : 0.0;
        }
    }
    // the tile's 8 flag words (one sector; every lane reads all of them, so
    // the lane's prefix is local popcounts instead of a shuffle scan) and the
    // tile prefix go out with the column/value loads; the x gathers are issued
    // before anything waits on them
    const uint4 fa = __ldg(reinterpret_cast<const uint4*>(bits + (z0 >> 5)));
    const uint4 fb = __ldg(reinterpret_cast<const uint4*>(bits + (z0 >> 5)) + 1);
    const int wq0 = __ldg(wq + w);
    double xv[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) xv[j] = c[j] >= 0 ? ld_x(x + c[j]) : 0.0;
    // this lane's 8 flags: byte (lane & 3) of word lane >> 2
    const uint32_t fw8[8] = {fa.x, fa.y, fa.z, fa.w, fb.x, fb.y, fb.z, fb.w};
    const int wi = lane >> 2, sh = (lane & 3) * 8;
    uint32_t fw = 0;
    int before = 0;  // flags of the tile before this lane's first element
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        if (k < wi) before += __popc(fw8[k]);
        if (k == wi) fw = fw8[k];
    }
    before += __popc(fw & ((1u << sh) - 1u));
    const uint32_t m = (fw >> sh) & 0xffu;
    const int nf = __popc(m);
    const int qb = wq0 + before;  // flags before this lane's first element
    // rows of the segments this lane closes (qb-1 .. qb+nf-2) and the one it
    // leaves open (qb+nf-1), fetched with the gathers
    int32_t sr[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const int q = qb - 1 + i;
        sr[i] = (i <= nf && q >= 0) ? __ldg(seg_row + q) : 0;
    }
    double run = 0.0, head = 0.0;
    bool has = false;
    int closed = 0;  // segments closed so far in this lane
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        if ((m >> j) & 1u) {  // a row starts here: the open segment closes
            if (has) {
                const int32_t r = closed < NS ? sr[closed] : __ldg(seg_row + qb - 1 + closed);
                y[r] = run;
            } else {
                head = run;
            }
            has = true;
            ++closed;
            run = 0.0;
        }
        run += __dmul_rn(v[j], xv[j]);
    }
    const uint32_t F = __ballot_sync(0xffffffffu, has);
    double S = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double up = __shfl_up_sync(0xffffffffu, S, d);
        if (lane >= d && ((F >> (lane - d + 1)) & ((1u << d) - 1u)) == 0u) S += up;
    }
    double cin = __shfl_up_sync(0xffffffffu, S, 1);
    if (lane == 0) cin = 0.0;
    if (has && qb >= 1) y[sr[0]] = head + cin;
    if (lane == 31) {
        const int q = qb + nf - 1;  // the segment open at the tile end
        carry_row[w] = q >= 0 ? (nf < NS ? sr[nf] : __ldg(seg_row + q)) : -1;
        carry_val[w] = S;
    }
}

// E = nominal nonzeros per lane; actual chunk lengths are floor/ceil of
// nnz/jl, at most E (jl = ceil(nnz/E)), so the per-lane loop is unrolled to E.
template <int E, bool BRANCHY>
__global__ void __launch_bounds__(kU3Threads) k_u3(const int32_t* __restrict__ col,
                                                   const double* __restrict__ val,
                                                   const double* __restrict__ x,
                                                   double* __restrict__ y, int64_t n,
                                                   int64_t nnz, int64_t jl,
                                                   const uint32_t* __restrict__ bits,
                                                   const int32_t* __restrict__ seg_row,
                                                   int64_t nq,
                                                   const int32_t* __restrict__ tile_q,
                                                   int32_t* __restrict__ carry_row,
                                                   double* __restrict__ carry_val) {
    constexpr int TILE = kU3Threads * E;
    constexpr int PAD = TILE + TILE / E + 1;
    __shared__ double s_prod[PAD];
    const int tid = threadIdx.x;
    const int64_t t = blockIdx.x;
    const int64_t p0 = t * kU3Threads;
    const int64_t p1 = min(p0 + kU3Threads, jl);
    const int64_t K0 = nnz * p0 / jl, K1 = nnz * p1 / jl;
    const int span = static_cast<int>(K1 - K0);
    {
        int32_t cc[E];
        double vv[E], xv[E];
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int i = u * kU3Threads + tid;
            cc[u] = i < span ? ld_plain_i32(col + K0 + i) : -1;
            vv[u] = i < span ? ld_plain_f64(val + K0 + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < E; ++u) xv[u] = cc[u] >= 0 ? ldg_f64(x + cc[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int i = u * kU3Threads + tid;
            if (i < span) s_prod[i + i / E] = vv[u] * xv[u];
        }
    }
    // this lane's chunk (reference rule, bss.hpp:49-50)
    const int64_t p = p0 + tid;
    const bool lane_ok = p < jl;
    const int64_t a = lane_ok ? nnz * p / jl : K1;
    const int64_t b = lane_ok ? nnz * (p + 1) / jl : K1;
    const int len = static_cast<int>(b - a);
    // flag bits of [a, b): at most E+1 <= 33 bits, from two words
    uint32_t m = 0;
    if (len > 0) {
        const int64_t w = a >> 5;
        const int sh = static_cast<int>(a & 31);
        uint64_t pair = bits[w];
        if (((b - 1) >> 5) != w) pair |= static_cast<uint64_t>(bits[w + 1]) << 32;
        m = static_cast<uint32_t>(pair >> sh);
        if (len < 32) m &= (1u << len) - 1u;
    }
    const int nf = __popc(m);
    // q of the lane's first element = flags before a = tile_q + block prefix of nf
    using BS = cub::BlockScan<int, kU3Threads>;
    __shared__ typename BS::TempStorage scan_tmp;
    int qpre = 0, qtot = 0;
    BS(scan_tmp).ExclusiveSum(nf, qpre, qtot);
    KTB_SYNC();
    int64_t q = static_cast<int64_t>(tile_q[t]) + qpre;  // flags strictly before a

    // walk: close the open segment at each row start (flag), emit complete rows
    double run = 0.0;
    int first_row = -1;
    double first_val = 0.0;
    const int base = static_cast<int>(a - K0);
#pragma unroll
    for (int e = 0; e < E; ++e) {
        if (e < len) {
            const int li = base + e;
            const double prod = s_prod[li + li / E];
            bool f;
            if (BRANCHY) {
                // original scan (spmv.hpp:157): fetch and test the element's flag
                const int64_t k = a + e;
                f = (__ldg(bits + (k >> 5)) >> (k & 31)) & 1u;
            } else {
                f = (m >> e) & 1u;  // BSS: flags of the whole chunk in one register
            }
            if (f) {
                if (q > 0) {
                    const int32_t r = seg_row[q - 1];
                    const int32_t rn = seg_row[q];
                    if (first_row < 0) {
                        first_row = r;
                        first_val = run;
                    } else {
                        y[r] = run;
                    }
                    for (int32_t z = r + 1; z < rn; ++z) y[z] = 0.0;  // empty rows between
                } else {
                    for (int32_t z = 0; z < seg_row[0]; ++z) y[z] = 0.0;  // leading empties
                }
                run = 0.0;
                ++q;
            }
            run += prod;
        }
    }
    SegPair agg;
    const SegPair pre = block_seg_scan_excl<kU3Threads>(SegPair{nf > 0, run}, &agg);
    if (first_row >= 0) y[first_row] = first_val + pre.v;
    if (lane_ok && p == jl - 1) {
        // the last nonempty row is never closed by a flag: seed it with 0 and
        // let the carry fixup add the open segment; trailing empty rows are 0
        const int32_t last = seg_row[nq - 1];
        y[last] = 0.0;
        for (int64_t z = last + 1; z < n; ++z) y[z] = 0.0;
    }
    if (tid == 0) {
        const int64_t qe = static_cast<int64_t>(tile_q[t]) + qtot;  // flags before K1
        carry_row[t] = qe > 0 ? seg_row[qe - 1] : -1;
        carry_val[t] = agg.v;
    }
}

void u3_setup(ktb_plan* p) {
    const ktb_matrix* m = p->m;
    require(m->nnz > 0, "bss plan: empty matrix");
    const bool warp_tiles = p->param == 1008 && p->kernel == KTB_U3;
    require(p->cta_threads == 0 || (warp_tiles && (p->cta_threads == 128 || p->cta_threads == 256)),
            "u3: only the warp tiles (param 1008) take a CTA shape: 128 or 256 threads");
    int E = p->param > 0 ? static_cast<int>(p->param) : 8;
    if (warp_tiles) E = 8;
    if (E != 4 && E != 8 && E != 16) E = 8;
    p->param = warp_tiles ? 1008 : E;
    p->jl = ceil_div64(m->nnz, E);
    p->tiles = warp_tiles ? ceil_div64(m->nnz, 256) : ceil_div64(p->jl, kU3Threads);
    cudaStream_t s = p->stream;
    const int64_t words = ceil_div64(m->nnz, 32) + 1;
    p->flag_bits.alloc(words);
    KTB_CUDA(cudaMemsetAsync(p->flag_bits.p, 0, 4 * words, s));
    k_flag_bits<<<ceil_div(m->n, 256), 256, 0, s>>>(m->row_ptr.p, m->n, p->flag_bits.p);
    KTB_LAUNCH();
    DBuf<int32_t> mark(m->n), ord(m->n);
    k_nonempty_mark<<<ceil_div(m->n, 256), 256, 0, s>>>(m->row_ptr.p, m->n, mark.p);
    KTB_LAUNCH();
    size_t tmp = 0;
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, mark.p, ord.p, m->n, s));
    DBuf<uint8_t> tb(tmp ? tmp : 1);
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, mark.p, ord.p, m->n, s));
    int32_t lo = 0, lm = 0;
    KTB_CUDA(cudaMemcpyAsync(&lo, ord.p + m->n - 1, 4, cudaMemcpyDeviceToHost, s));
    KTB_CUDA(cudaMemcpyAsync(&lm, mark.p + m->n - 1, 4, cudaMemcpyDeviceToHost, s));
    KTB_CUDA(cudaStreamSynchronize(s));
    p->nq = static_cast<int64_t>(lo) + lm;
    p->seg_row.alloc(p->nq + 1);
    k_nonempty_scatter<<<ceil_div(m->n, 256), 256, 0, s>>>(m->row_ptr.p, m->n, ord.p,
                                                           p->seg_row.p);
    KTB_LAUNCH();
    const int32_t nrow = static_cast<int32_t>(m->n);
    KTB_CUDA(cudaMemcpyAsync(p->seg_row.p + p->nq, &nrow, 4, cudaMemcpyHostToDevice, s));
    if (warp_tiles) {
        // flags before each 256-nonzero tile: per-tile popcounts + a scan
        p->tile_q.alloc(p->tiles + 1);
        if (ceil_div64(m->nnz, 32) + 1 < p->tiles * 8) {
            // the bit array covers whole tiles (zero padded)
            DBuf<uint32_t> nb(p->tiles * 8);
            KTB_CUDA(cudaMemsetAsync(nb.p, 0, 4 * p->tiles * 8, s));
            KTB_CUDA(cudaMemcpyAsync(nb.p, p->flag_bits.p, 4 * words, cudaMemcpyDeviceToDevice, s));
            p->flag_bits = std::move(nb);
        }
        k_tile_pop<<<ceil_div(p->tiles + 1, 256), 256, 0, s>>>(p->flag_bits.p, p->tiles,
                                                              p->tile_q.p);
        KTB_LAUNCH();
        size_t t2 = 0;
        KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, p->tile_q.p, p->tile_q.p,
                                               p->tiles + 1, s));
        DBuf<uint8_t> tb2(t2 ? t2 : 1);
        KTB_CUDA(cub::DeviceScan::ExclusiveSum(tb2.p, t2, p->tile_q.p, p->tile_q.p, p->tiles + 1,
                                               s));
        // rows no flag closes: the empty ones and the last nonempty row
        p->nzero = m->n - p->nq + 1;
        p->zero_rows.alloc(p->nzero);
        k_empty_list<<<ceil_div(m->n, 256), 256, 0, s>>>(m->row_ptr.p, m->n, ord.p,
                                                         p->zero_rows.p);
        KTB_LAUNCH();
        KTB_CUDA(cudaMemcpyAsync(p->zero_rows.p + p->nzero - 1, p->seg_row.p + p->nq - 1, 4,
                                 cudaMemcpyDeviceToDevice, s));
        p->ctas = ceil_div64(p->tiles, 8);
    } else {
        p->tile_q.alloc(p->tiles);
        k_tile_q<<<static_cast<int>(p->tiles), 256, 0, s>>>(p->flag_bits.p, m->nnz, p->jl,
                                                            p->tiles, p->tile_q.p);
        KTB_LAUNCH();
    }
    p->carry_row.alloc(p->tiles);
    p->carry_val.alloc(p->tiles);
    KTB_CUDA(cudaStreamSynchronize(s));
    if (!warp_tiles) p->ctas = p->tiles;
    p->launches = warp_tiles ? 3 : 2;
    // flag bits + nonempty-row map replace row_ptr; tile carries
    p->extra_bytes = 4 * words + 4 * (p->nq - (m->n + 1)) + p->tiles * (4 + 8) * 2 +
                     (warp_tiles ? 12 * p->nzero : 0);
}

void u3_run(ktb_plan* p, const double* x, double* y) {
    const ktb_matrix* m = p->m;
    if (p->param == 1008 && p->kernel == KTB_U3) {
        k_zero_rows<<<ceil_div(p->nzero, 256), 256, 0, p->stream>>>(p->zero_rows.p, p->nzero, y);
        KTB_LAUNCH();
        if (p->cta_threads == 256)
            k_u3w<8><<<static_cast<int>(ceil_div64(p->tiles, 8)), 256, 0, p->stream>>>(
                m->col.p, m->val.p, x, y, m->nnz, p->tiles, p->flag_bits.p, p->seg_row.p,
                p->tile_q.p, p->carry_row.p, p->carry_val.p);
        else
            k_u3w<4><<<static_cast<int>(ceil_div64(p->tiles, 4)), 128, 0, p->stream>>>(
                m->col.p, m->val.p, x, y, m->nnz, p->tiles, p->flag_bits.p, p->seg_row.p,
                p->tile_q.p, p->carry_row.p, p->carry_val.p);
        KTB_LAUNCH();
        fixup_run(p, y);
        return;
    }
    const int grid = static_cast<int>(p->tiles);
    const bool br = p->kernel == KTB_U4;
#define KTB_U3_CASE(EE)                                                                        \
    case EE:                                                                                    \
        if (br)                                                                                 \
            k_u3<EE, true><<<grid, kU3Threads, 0, p->stream>>>(                                 \
                m->col.p, m->val.p, x, y, m->n, m->nnz, p->jl, p->flag_bits.p, p->seg_row.p,    \
                p->nq, p->tile_q.p, p->carry_row.p, p->carry_val.p);                            \
        else                                                                                    \
            k_u3<EE, false><<<grid, kU3Threads, 0, p->stream>>>(                                \
                m->col.p, m->val.p, x, y, m->n, m->nnz, p->jl, p->flag_bits.p, p->seg_row.p,    \
                p->nq, p->tile_q.p, p->carry_row.p, p->carry_val.p);                            \
        break;
    switch (p->param) {
        KTB_U3_CASE(4)
        KTB_U3_CASE(8)
        KTB_U3_CASE(16)
        default: throw Invalid("u3: bad lane length");
    }
#undef KTB_U3_CASE
    KTB_LAUNCH();
    fixup_run(p, y);
}

}  // namespace ktb
