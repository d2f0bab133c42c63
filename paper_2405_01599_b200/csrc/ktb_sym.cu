// ktb_sym.cu -- symmetric (diagonal + strict upper) CRS SpMV for sm_100a.
//
// Reference: spmv_sym (spmv.hpp:180-234). Each worker writes row-direction
// sums y_i = sum_j U_ij x_j for its rows and scatters transposed products
// U_ij x_i (j != i) into a private n-vector; a cross-worker reduction then
// adds the scratch vectors into y over [0,n) (S1/S2) or only over the
// worker's nonzero region [lo,hi) (S3, partition.hpp:73-96).
//
// GPU mapping:
//   S1/S2  "full-range reduction": the transposed products go straight to y
//          with fp64 red.global (L2 atomics) after a memset; rows are split
//          row-based (S1) or into NNZ_BALANCED CTA blocks (S2). Not
//          deterministic (atomic order), tolerance-checked.
//   S3     "zero-omission window": one persistent CTA per SM owns an
//          NNZ_BALANCED row block (bit-exact boundaries, P = #SMs). Its
//          transposed products accumulate in a shared-memory ring that covers
//          exactly the CTA's reduction region [lo, hi); rows are finalised
//          from the ring as soon as no later row of the block can reach them,
//          and only the part of the region beyond the block (the spill) is
//          reduced across CTAs, in fixed ascending-CTA order. Shared-memory
//          fp64 atomics are a CAS loop on sm_100a (ATOMS.CAST.SPIN.64), so
//          the ring is updated with plain ld/st in ROUNDS: the plan assigns
//          every entry of a sub-tile of S rows to a round such that no two
//          entries of one round target the same window slot (greedy bipartite
//          edge colouring, done once on the host), stores the sub-tile in
//          round-major SELL order (coalesced), and the kernel separates rounds
//          with a CTA barrier. The result is deterministic.
#include <algorithm>
#include <type_traits>
#include <cstring>
#include <vector>

#include <atomic>
#include <cstdlib>
#include <thread>

#include "ktb_internal.cuh"
#include "ktb_ptx.cuh"

namespace ktb {

__device__ __forceinline__ double ld_stream_f64s(const double* p) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ int32_t ld_stream_i32s(const int32_t* p) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// ================================================================ S1 / S2
template <int V>
__global__ void __launch_bounds__(256) k_sym_atomic(const int32_t* __restrict__ rp,
                                                    const int32_t* __restrict__ col,
                                                    const double* __restrict__ val,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y, int64_t n,
                                                    const int32_t* __restrict__ blocks) {
    const int sub = threadIdx.x & (V - 1);
    int64_t first, stride, last;
    if (blocks) {  // S2: CTA b owns rows [blocks[b], blocks[b+1])
        first = blocks[blockIdx.x] + threadIdx.x / V;
        last = blocks[blockIdx.x + 1];
        stride = blockDim.x / V;
    } else {  // S1: contiguous rows in launch order
        first = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / V;
        last = n;
        stride = static_cast<int64_t>(gridDim.x) * blockDim.x / V;
    }
    const int64_t trips = first < last ? (last - first + stride - 1) / stride : 0;
    // all lanes of a group run the same number of trips (shuffle safety)
    for (int64_t t = 0; t < trips; ++t) {
        const int64_t i = first + t * stride;
        const bool active = i < last;
        int32_t b = 0, e = 0;
        double xi = 0.0;
        if (active) {
            b = __ldg(rp + i);
            e = __ldg(rp + i + 1);
            xi = __ldg(x + i);
        }
        double s = 0.0;
        for (int32_t k = b + sub; k < e; k += V) {
            const int32_t j = ld_stream_i32s(col + k);
            const double v = ld_stream_f64s(val + k);
            s += v * __ldg(x + j);
            if (j != i) atomicAdd(y + j, v * xi);
        }
        if (V > 1) {
#pragma unroll
            for (int o = V / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, V);
        }
        if (active && sub == 0) atomicAdd(y + i, s);
    }
}

void s12_setup(ktb_plan* p) {
    ktb_matrix* m = p->m;
    require(m->kind == KTB_SYM_UPPER, "spmv: symmetric kernel on a general matrix");
    if (p->kernel == KTB_S1 && p->param == 106) {
        // S1 with gathered transposed products: row-based, and the "reduction"
        // disappears -- every row reads its lower entries from the expanded
        // matrix's pair-coded warp slices (U1 106: a 27-point stencil row is
        // 27 one-byte codes + its share of a 28-pair dictionary, less than
        // the upper triangle's CRS). Deterministic, bitwise equal to
        // spmv_ref(expand_symmetric(A)); refused (Invalid) when a slice of the
        // expanded matrix has too many distinct (column delta, value) pairs.
        {
            std::lock_guard<std::mutex> lk(m->lazy_mu);
            if (!m->expanded) m->expanded = expand_symmetric_dev(m, p->stream);
        }
        p->long_plan = plan_create_internal(m->expanded, KTB_U1, 106, 0, p->stream);
        p->launches = 1;
        p->ctas = p->long_plan->ctas;
        // the records instead of the upper triangle's CRS
        p->extra_bytes = static_cast<int64_t>(p->long_plan->sell_rec.n) - 12 * m->nnz -
                         4 * (m->n + 1);
        return;
    }
    if (p->param <= 0) {
        const double mean = m->n ? double(m->nnz) / double(m->n) : 1.0;
        int v = 1;
        while (v < 32 && v < mean) v <<= 1;
        p->param = v;
    }
    int v = 1;
    while (v < p->param && v < 32) v <<= 1;
    p->param = v;
    if (p->kernel == KTB_S2) {
        const int P = m->sm_count * 8;
        p->blocks.alloc(P + 1);
        build_row_partition_dev(m, P, KTB_NNZ_BALANCED, p->blocks.p, p->stream);
        p->ctas = P;
    } else {
        p->ctas = std::max<int64_t>(1, std::min<int64_t>(ceil_div64(m->n * v, 256),
                                                         int64_t(m->sm_count) * 64));
    }
    p->launches = 2;
    p->extra_bytes = 8 * m->n;  // y memset
}

void s12_run(ktb_plan* p, const double* x, double* y) {
    const ktb_matrix* m = p->m;
    if (p->long_plan) {  // S1 106: the expanded coded slices
        p->long_plan->stream = p->stream;
        plan_run(p->long_plan, x, y, 0, m->n);
        return;
    }
    KTB_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * m->n, p->stream));
    const int grid = static_cast<int>(p->ctas);
    const int32_t* blocks = p->kernel == KTB_S2 ? p->blocks.p : nullptr;
#define KTB_S_CASE(VV)                                                                       \
    case VV:                                                                                  \
        k_sym_atomic<VV><<<grid, 256, 0, p->stream>>>(m->row_ptr.p, m->col.p, m->val.p, x, y, \
                                                      m->n, blocks);                          \
        break;
    switch (p->param) {
        KTB_S_CASE(1)
        KTB_S_CASE(2)
        KTB_S_CASE(4)
        KTB_S_CASE(8)
        KTB_S_CASE(16)
        KTB_S_CASE(32)
        default: throw Invalid("s1/s2: bad lane count");
    }
#undef KTB_S_CASE
    KTB_LAUNCH();
}

// ================================================================ S3
// Zero-omission window kernel (see the file header). One block per SM owns
// its NNZ_BALANCED row block; sub-tiles of kRows rows are processed in
// rounds from a TMA-fed shared-memory ring (one round of one sub-tile per
// stage, copied to registers on arrival), x is gathered kGD rounds ahead,
// and each round's scatter is a plain ld/add/st on the window ring followed
// by one block barrier. The part of each block's region beyond the block
// (the spill) goes to a global buffer; k_s3_fixup adds it into the next
// blocks' head rows in ascending source order (deterministic).
constexpr int kRows = 2048;  // rows per sub-tile; CTA shape 256 x 8 (77.5-77.7 us on config
                             // 2) or 512 x 4 (79.1-79.4 us), a template parameter of k_s3
#ifndef KTB_S3_GD
#define KTB_S3_GD 1
#endif
constexpr int kStages = 4;  // TMA ring depth = register ring depth (one round-chunk each)
constexpr int kGD = KTB_S3_GD;  // chunks gathered ahead (copied to registers, x gathers issued)
// stage = one round of a sub-tile: fp64 values then int16 sub-tile-relative
// columns, in a thread-swizzled order so each thread reads its 4 values with
// two conflict-free LDS.128 (chunk k*512+t holds rows t+1024k, t+1024k+512)
// and its 4 columns with one LDS.64 (chunk t holds rows t+512u, u = 0..3)
constexpr int kStageBytes = kRows * (8 + 2);  // 20480
constexpr int kS3RoundCap = 64;  // max rounds per sub-tile (colour classes)
constexpr int kS3SmemFixed = kStages * kStageBytes + kStages * 8 + 128;
#ifndef KTB_S3_FIXROWS
#define KTB_S3_FIXROWS 1024
#endif
constexpr int kFixRows = KTB_S3_FIXROWS;  // rows per fixup block (kFixRows / 256 per thread)

// host-side positions of sub-tile row t in a round's value / column arrays
// for a CTA of T threads (T rows per u, 2048 / T rows per thread)
inline int64_t s3_val_pos(int t, int T) {
    const int th = t % T, u = t / T;
    return (static_cast<int64_t>(u / 2) * T + th) * 2 + (u % 2);
}
inline int64_t s3_col_pos(int t, int T) {
    const int th = t % T, u = t / T;
    return static_cast<int64_t>(th) * (kRows / T) + u;
}

// column u (sign-extended int16) from its packed word
__device__ __forceinline__ int col_of(uint32_t w, int u) {
    return (u & 1) ? static_cast<int>(w) >> 16 : static_cast<int>(w << 16) >> 16;
}

// unsigned wrap into [0, W) for s in [0, 2W)
__device__ __forceinline__ int wrap(int s, int W) {
    return static_cast<int>(min(static_cast<unsigned>(s), static_cast<unsigned>(s - W)));
}

// chunk metadata (one int per round-chunk): bits 0-6 round, bit 7 last round
// of its sub-tile, bit 8 "no barrier after" (this round and the next target
// disjoint window slots), bits 9.. sub-tile index local to the block
#ifndef KTB_S3_ABL
#define KTB_S3_ABL 0  // timing ablations (wrong results): 1 no gathers, 2 no window, 4 no barrier
#endif
#ifndef KTB_S3_PAIRS
#define KTB_S3_PAIRS 0
#endif
constexpr bool kS3Pairs = KTB_S3_PAIRS;
__device__ __forceinline__ int meta_round(int m) { return m & 127; }
__device__ __forceinline__ bool meta_last(int m) { return (m >> 7) & 1; }
__device__ __forceinline__ bool meta_nobar(int m) { return (m >> 8) & 1; }
__device__ __forceinline__ int meta_sub(int m) { return (m >> 9) & 0x1fffff; }
// padding chunk (the loop runs a multiple of kStages chunks): no data, no work
constexpr int kMetaEmpty = 1 << 30;
__device__ __forceinline__ bool meta_empty(int m) { return m & kMetaEmpty; }

// One block of kS3Threads threads per SM. Thread 0 drives the TMA ring: it
// issues the first kStages chunks, waits for chunk q+kGD+1 before the round
// barrier of chunk q (the barrier then publishes the landed stage to every
// thread), and refills a stage with chunk +kStages right after the barrier
// that follows the stage's copy into registers. Register ring slot and smem
// stage of chunk q are both q % kStages, so every shared-memory offset below
// is a compile-time constant of the unrolled loop.
// Launch shapes: 256 threads x 8 rows (default) or 512 x 4 (the selector
// times both; plan param bits 16.., the SELL positions follow the shape).
template <int kS3T>
__global__ void __launch_bounds__(kS3T, 1)
    k_s3(const int32_t* __restrict__ cta_row, const int32_t* __restrict__ cta_chunk,
         const int32_t* __restrict__ chunk_meta, const int32_t* __restrict__ cta_qreal,
         const unsigned char* __restrict__ sell,
         const int64_t* __restrict__ cta_base, const double* __restrict__ diag,
         const double* __restrict__ x, double* __restrict__ y, int W, int reach, int n,
         const int32_t* __restrict__ spill_hi, const int64_t* __restrict__ spill_off,
         double* __restrict__ spill) {
    constexpr int kS3Threads = kS3T;           // this instantiation's shape
    constexpr int kRPT = kRows / kS3T;         // rows per thread: t + kS3Threads*u
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
    double* win = reinterpret_cast<double*>(smem + kS3SmemFixed);

    const int tid = threadIdx.x;
    const int c = blockIdx.x;
    const int32_t R0 = cta_row[c], R1 = cta_row[c + 1];
    const int q0 = cta_chunk[c];
    const int QP = cta_chunk[c + 1] - q0 - kGD - 1;  // chunks incl. padding (multiple of kStages)
    const int Q = cta_qreal[c];                   // real round-chunks of this block
    const int32_t* meta = chunk_meta + q0;        // QP + kGD + 1 entries
    const unsigned char* gchunk = sell + cta_base[c] * kStageBytes;
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int qq, int st) {  // thread 0 only
        mbar_arrive_expect_tx(&full[st], kStageBytes);
        tma_load_1d(smem + st * kStageBytes, gchunk + int64_t(qq) * kStageBytes, kStageBytes,
                    &full[st], pol);
    };
    // x is first touched by the far reach of the window: pull the initial
    // window and then each sub-tile's new front into L2 ahead of the gathers
    // (the bench flushes L2 between steps).
#ifndef KTB_S3_AHEAD
#define KTB_S3_AHEAD 2
#endif
    constexpr int kAhead = KTB_S3_AHEAD;  // sub-tiles of look-ahead
    auto pf = [&](int64_t lo, int64_t hi) {  // x may be only 8-byte aligned (basis columns)
        lo = max(lo, int64_t(0));
        hi = min(hi, int64_t(n));
        if (hi > lo) prefetch_l2_range(x + lo, x + hi);
    };
    if (tid == 0) {
        for (int st = 0; st < kStages; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
        if (Q > 0) {
            for (int k = 0; k < kStages && k < Q; ++k) issue(k, k);
            pf(R0, int64_t(R0) + kRows * (kAhead + 1) + reach);
        }
    }
    for (int k = tid; k < W; k += kS3Threads) win[k] = 0.0;
    KTB_SYNC();
    // let the fixup grid launch early (programmatic dependent launch): its
    // blocks take SMs as these retire and wait for this grid's completion
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (Q > 0) {
        const uint64_t keep = policy_evict_last();  // y head rows are re-read by the fixup
        uint32_t cr[kStages][kRPT / 2];  // packed int16 sub-tile-relative columns (-1: pad)
        double vr[kStages][kRPT], xr[kStages][kRPT];
        int mr[kStages];
        // copy chunk qq (stage ST) to registers and issue its x gathers
        int mnext = __ldg(meta + 0);  // metadata of the next chunk to gather
        auto gather = [&](int qq, auto stc) {
            constexpr int ST = decltype(stc)::value;
            const int mm = mnext;
            mnext = __ldg(meta + qq + 1);  // one chunk ahead: never on the gather's critical path
            mr[ST] = mm;
            const bool live = !meta_empty(mm);  // padding chunk: its stage holds no data
            const unsigned char* sb = smem + ST * kStageBytes;
            if constexpr (kRPT == 8) {
                const uint4 cp = reinterpret_cast<const uint4*>(sb + kRows * 8)[tid];
                cr[ST][0] = cp.x;
                cr[ST][1] = cp.y;
                cr[ST][2] = cp.z;
                cr[ST][3] = cp.w;
            } else if constexpr (kRPT == 4) {
                const uint2 cp = reinterpret_cast<const uint2*>(sb + kRows * 8)[tid];
                cr[ST][0] = cp.x;
                cr[ST][1] = cp.y;
            } else {  // kRPT == 2
                cr[ST][0] = reinterpret_cast<const uint32_t*>(sb + kRows * 8)[tid];
            }
#pragma unroll
            for (int k2 = 0; k2 < kRPT / 2; ++k2) {
                const double2 vp = reinterpret_cast<const double2*>(sb)[k2 * kS3Threads + tid];
                vr[ST][2 * k2] = vp.x;
                vr[ST][2 * k2 + 1] = vp.y;
            }
            const double* xa = x + R0 + meta_sub(mm) * kRows;  // x at the chunk's row 0
            // opaque to the optimiser: the gathers below then form their
            // addresses as xa + 8*off (one wide multiply-add) instead of
            // re-associating into 64-bit index arithmetic per gather
#ifndef KTB_S3_OPAQUE_XA
#define KTB_S3_OPAQUE_XA 1
#endif
#if KTB_S3_OPAQUE_XA
            asm("mov.b64 %0, %0;" : "+l"(xa));
#endif
#pragma unroll
            for (int u = 0; u < kRPT; ++u) {
                const int cu = col_of(cr[ST][u >> 1], u);
                // always a valid address; the padding select happens at use
#if KTB_S3_ABL & 1
                xr[ST][u] = 1.0 + cu;  // ablation: no x gathers
#else
                // unsigned 32-bit offset from the chunk's base pointer: one
                // wide multiply-add per address instead of 64-bit index math
                xr[ST][u] = __ldg(xa + static_cast<uint32_t>(live ? max(cu, 0) : 0));
#endif
            }
        };
        // prologue: chunks 0..kGD landed and visible; gather 0..kGD-1
        if (tid == 0)
            for (int k = 0; k <= kGD && k < Q; ++k) mbar_wait(&full[k], 0);
        KTB_SYNC();
        static_assert(kGD >= 1 && kGD <= 2, "prologue gathers kGD chunks");
        gather(0, std::integral_constant<int, 0>{});
        if (kGD > 1) gather(1, std::integral_constant<int, 1>{});
        KTB_SYNC();
        if (tid == 0)
            for (int k = 0; k < kGD && k + kStages < Q; ++k) {
                fence_proxy_async_smem();
                issue(k + kStages, k);
            }
        int off = 0;  // ring slot of the current sub-tile's row 0
        int32_t a = R0;
        double rowsum[kRPT], xi[kRPT], di[kRPT], xin[kRPT];
#pragma unroll
        for (int u = 0; u < kRPT; ++u) {
            rowsum[u] = 0.0;
            const int32_t i = a + u * kS3Threads + tid;
            xi[u] = i < R1 ? __ldg(x + i) : 0.0;
            xin[u] = di[u] = 0.0;
        }
        int wph = 0;  // parity of the stage waited for (flips every kStages chunks)
        int pend = -1;  // thread 0: chunk whose refill waits for the next barrier
        auto body = [&](int q, auto kc) {
            constexpr int K = decltype(kc)::value;          // stage / slot of chunk q
            constexpr int KG = (K + kGD) % kStages;         // stage / slot of chunk q+kGD
            constexpr int KW = (K + kGD + 1) % kStages;     // stage of chunk q+kGD+1
            gather(q + kGD, std::integral_constant<int, KG>{});  // padded meta: always valid
            const int m = mr[K];
            if (meta_empty(m)) {  // padding chunk: keep the barrier cadence only
                KTB_SYNC();
                return;
            }
            if (meta_round(m) == 0) {  // this sub-tile's diagonal, next one's x_i, the x front
#pragma unroll
                for (int u = 0; u < kRPT; ++u) {
                    const int32_t i = a + u * kS3Threads + tid;
                    di[u] = i < R1 ? __ldg(diag + i) : 0.0;
                    xin[u] = i + kRows < R1 ? __ldg(x + i + kRows) : 0.0;
                }
                if (tid == 0) {
                    const int64_t front = int64_t(a) + int64_t(kAhead + 1) * kRows + reach;
                    pf(front, front + kRows);
                }
            }
            double wv[kRPT];
            int sl[kRPT];
            bool sc[kRPT];
#pragma unroll
            for (int u = 0; u < kRPT; ++u) {
                const int cu = col_of(cr[K][u >> 1], u);
                sc[u] = cu >= 0;
                rowsum[u] += sc[u] ? vr[K][u] * xr[K][u] : 0.0;
                sl[u] = wrap(cu + off, W);
                KTB_DCHECK(!sc[u] || (sl[u] >= 0 && sl[u] < W));
                KTB_DCHECK(!sc[u] || a + cu < n);
#if !(KTB_S3_ABL & 2)
                if (sc[u]) wv[u] = win[sl[u]];
#endif
            }
#if !(KTB_S3_ABL & 2)
#pragma unroll
            for (int u = 0; u < kRPT; ++u)
                if (sc[u]) win[sl[u]] = wv[u] + vr[K][u] * xi[u];
#else
            rowsum[0] += xi[1] * vr[K][2];  // ablation: no window RMW
#endif
            if (meta_nobar(m)) {
                // next round targets other slots: no barrier; every thread
                // checks the stage it gathers next itself, and the refill of
                // stage KG waits for the next barrier
                if (q + kGD + 1 < Q) mbar_wait(&full[KW], wph ^ (KW <= K ? 1 : 0));
                if (tid == 0 && q + kGD < Q && q + kGD + kStages < Q) pend = q + kGD + kStages;
                return;
            }
            if (tid == 0 && q + kGD + 1 < Q) mbar_wait(&full[KW], wph ^ (KW <= K ? 1 : 0));
#if KTB_S3_ABL & 4
            if (q + kGD + 1 < Q) mbar_wait(&full[KW], wph ^ (KW <= K ? 1 : 0));  // ablation: no barrier
#else
            KTB_SYNC();
#endif
            if (tid == 0) {
                if (pend >= 0) {  // the refill deferred by the previous round
                    fence_proxy_async_smem();
                    issue(pend, (KG + kStages - 1) % kStages);
                    pend = -1;
                }
                if (q + kGD < Q && q + kGD + kStages < Q) {
                    fence_proxy_async_smem();  // stage KG was copied out before the barrier
                    issue(q + kGD + kStages, KG);
                }
            }
            if (meta_last(m)) {  // sub-tile complete: finalise its rows
#pragma unroll
                for (int u = 0; u < kRPT; ++u) {
                    const int32_t i = a + u * kS3Threads + tid;
                    if (i < R1) {
                        const int slot = wrap(u * kS3Threads + tid + off, W);
                        st_hint_f64(y + i, di[u] * xi[u] + rowsum[u] + win[slot], keep);
                        win[slot] = 0.0;
                    }
                    rowsum[u] = 0.0;
                    xi[u] = xin[u];
                }
                KTB_SYNC();
                off = wrap(off + kRows, W);
                a += kRows;
            }
        };
        static_assert(kStages == 4, "the unrolled body covers four stages");
        for (int q = 0; q < QP; q += kStages) {
            body(q, std::integral_constant<int, 0>{});
            body(q + 1, std::integral_constant<int, 1>{});
            body(q + 2, std::integral_constant<int, 2>{});
            body(q + 3, std::integral_constant<int, 3>{});
            wph ^= 1;
        }
    }
    // spill: the region beyond the block, [R1, spill_hi)
    const int32_t hi = spill_hi[c];
    if (hi > R1) {
        const int64_t so = spill_off[c];
        const uint64_t keep = policy_evict_last();
        for (int32_t j = R1 + tid; j < hi; j += kS3Threads)
            st_hint_f64(spill + so + (j - R1), win[(j - R0) % W], keep);
    }
}

// Head rows of block d receive the spills of earlier blocks, summed in
// ascending source order and added once (deterministic). One block per
// segment of <= kFixRows head rows of one destination, 4 rows per thread; the
// segment's source metadata is plan data loaded before griddepcontrol.wait,
// so after it every y and spill load of the thread goes out at once.
#ifndef KTB_S3_FIXUP_MINB
#define KTB_S3_FIXUP_MINB 5  // <= 51 registers, 5 blocks/SM: measured best of 1, 5, 6
#endif
__global__ void __launch_bounds__(256, KTB_S3_FIXUP_MINB) k_s3_fixup(const int4* __restrict__ desc,
                                                  const int32_t* __restrict__ seg_src,
                                                  const int32_t* __restrict__ cta_row,
                                                  const int32_t* __restrict__ spill_hi,
                                                  const int64_t* __restrict__ spill_off,
                                                  const double* __restrict__ spill,
                                                  double* __restrict__ y) {
    constexpr int U = kFixRows / 256;
    // plan data, readable before the dependency resolves: rows [j0, j1), the
    // number of sources spilling into them (ascending), the first two
    // sources' ranges and spill bases inline
    const int4 a = desc[3 * blockIdx.x], b = desc[3 * blockIdx.x + 1], c = desc[3 * blockIdx.x + 2];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // k_s3 complete and visible
    const int32_t j0 = a.x, j1 = a.y, ns = a.z;
    const int64_t base0 = static_cast<int64_t>(
        static_cast<uint64_t>(static_cast<uint32_t>(c.x)) | (static_cast<uint64_t>(c.y) << 32));
    const int64_t base1 = static_cast<int64_t>(
        static_cast<uint64_t>(static_cast<uint32_t>(c.z)) | (static_cast<uint64_t>(c.w) << 32));
    double yv[U], v0[U], v1[U];
    bool touched[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {  // every load of the block in one round trip
        const int32_t j = j0 + u * 256 + threadIdx.x;
        const bool in = j < j1;
        const bool i0 = in && ns > 0 && j >= b.x && j < b.y;
        const bool i1 = in && ns > 1 && j >= b.z && j < b.w;
        yv[u] = in ? __ldcg(y + j) : 0.0;
        v0[u] = i0 ? __ldcg(spill + base0 + j) : 0.0;
        v1[u] = i1 ? __ldcg(spill + base1 + j) : 0.0;
        touched[u] = i0 || i1;
    }
    double acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = v0[u] + v1[u];  // ascending source order
    for (int k = 2; k < ns; ++k) {  // more than two sources: rare (tiny blocks)
        const int src = seg_src[a.w + k];
        const int32_t s0 = cta_row[src + 1], hi = spill_hi[src];
        const double* sp = spill + spill_off[src] - s0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t j = j0 + u * 256 + threadIdx.x;
            if (j < j1 && j >= s0 && j < hi) {
                acc[u] += __ldcg(sp + j);
                touched[u] = true;
            }
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int32_t j = j0 + u * 256 + threadIdx.x;
        if (touched[u]) y[j] = yv[u] + acc[u];
    }
}

// Entries the window pass leaves out (far from the window, congested slots)
// and rows too long for the round layout, as per-target contribution lists:
// one warp per target row sums its contributions lane-strided, reduces with
// a fixed butterfly and adds once into y[t] (after the window pass and the
// fixup): deterministic for any input.
__global__ void __launch_bounds__(256) k_s3_patch(const int32_t* __restrict__ rows,
                                                  const int32_t* __restrict__ rp,
                                                  const int32_t* __restrict__ src,
                                                  const double* __restrict__ val, int64_t m,
                                                  const double* __restrict__ x,
                                                  double* __restrict__ y) {
    const int64_t g = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (g >= m) return;  // whole warps exit together
    double s = 0.0;
    for (int32_t k = __ldg(rp + g) + lane; k < __ldg(rp + g + 1); k += 32)
        s += __ldg(val + k) * __ldg(x + __ldg(src + k));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        const int32_t t = __ldg(rows + g);
        y[t] = y[t] + s;
    }
}

void s3_setup(ktb_plan* p) {
    ktb_matrix* m = p->m;
    require(m->kind == KTB_SYM_UPPER, "spmv: symmetric kernel on a general matrix");
    auto& L = p->sw;
    cudaStream_t st = p->stream;
    const int S = kRows;
    require(p->cta_threads == 0 || p->cta_threads == 256 || p->cta_threads == 512,
            "s3: CTAs of 256 or 512 threads");
    const int T3 = p->cta_threads == 512 ? 512 : 256;
    const int64_t n = m->n, nnz = m->nnz;
    const int P = std::max(1, m->sm_count);
    L.ctas = P;
    L.rows_per_sub = S;
    // bit-exact NNZ_BALANCED boundaries with P = #SMs (partition.hpp:42-52)
    L.cta_row.alloc(P + 1);
    build_row_partition_dev(m, P, KTB_NNZ_BALANCED, L.cta_row.p, st);
    std::vector<int32_t> bnd(P + 1), rp(n + 1), col(nnz);
    std::vector<double> val(nnz);
    KTB_CUDA(cudaMemcpyAsync(bnd.data(), L.cta_row.p, 4 * (P + 1), cudaMemcpyDeviceToHost, st));
    KTB_CUDA(cudaMemcpyAsync(rp.data(), m->row_ptr.p, 4 * (n + 1), cudaMemcpyDeviceToHost, st));
    if (nnz) {
        KTB_CUDA(cudaMemcpyAsync(col.data(), m->col.p, 4 * nnz, cudaMemcpyDeviceToHost, st));
        KTB_CUDA(cudaMemcpyAsync(val.data(), m->val.p, 8 * nnz, cudaMemcpyDeviceToHost, st));
    }
    KTB_CUDA(cudaStreamSynchronize(st));

    // window: S rows + the largest reach of any row, capped by shared memory
    int max_smem = 0;
    KTB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                                    m->device));
    const int64_t cap = std::min<int64_t>(32767,  // int16 relative columns
                                          std::max<int64_t>(S + 32, (max_smem - kS3SmemFixed) / 8));
    int64_t reach = 0;
    for (int64_t i = 0; i < n; ++i)
        if (rp[i + 1] > rp[i]) reach = std::max<int64_t>(reach, col[rp[i + 1] - 1] - i);
    int64_t W = std::min<int64_t>(cap, ((S + reach + 1 + 31) / 32) * 32);
    W = std::max<int64_t>(W, S + 32);
    L.window = static_cast<int>(W);
    L.reach = static_cast<int>(std::min<int64_t>(reach, W));

    // Per block (independent given the bit-exact boundaries): colour each
    // sub-tile's entries into rounds and lay out its round-chunks. Blocks run
    // on all host cores; the merge below concatenates them in block order, so
    // the layout is identical for any thread count.
    struct BlockOut {
        std::vector<int32_t> rounds;      // per sub-tile
        std::vector<char> nobar;          // per chunk: no barrier after it
        std::vector<unsigned char> sell;  // the block's round-chunks
        std::vector<int32_t> far_i, far_j, long_rows;
        std::vector<double> far_v;
        int32_t spill_hi = 0;
        int64_t slots = 0;
    };
    std::vector<double> sdiag(n, 0.0);  // dense diagonal stream (rows disjoint per block)
    std::vector<BlockOut> outs(P);
    // rows longer than this go to the long-row path
    const double mean = n ? double(nnz) / double(n) : 1.0;
    const int64_t long_len = std::max<int64_t>(32, std::min<int64_t>(kS3RoundCap, 4 * mean + 8));
    auto do_block = [&](int c, std::vector<uint64_t>& colmask, std::vector<int32_t>& touched) {
        BlockOut& o = outs[c];
        const int32_t R0 = bnd[c], R1 = bnd[c + 1];
        int32_t hi = R1;
        for (int32_t a = R0; a < R1; a += S) {
            const int32_t rows = std::min<int32_t>(S, R1 - a);
            // greedy colouring: entry -> lowest round free in its row and in
            // its target slot; a congested slot turns the entry "far"
            std::vector<std::vector<std::pair<int, int64_t>>> assign(rows);  // (round, k)
            int R = 0;
            touched.clear();
            for (int32_t t = 0; t < rows; ++t) {
                const int32_t i = a + t;
                if (rp[i + 1] - rp[i] > long_len) {
                    o.long_rows.push_back(i);
                    continue;
                }
                uint64_t rowmask = 0;
                for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
                    const int32_t j = col[k];
                    if (j == i) {  // the diagonal goes to the dense d stream
                        sdiag[i] = val[k];
                        continue;
                    }
                    bool far = static_cast<int64_t>(j) - a >= W;
                    uint64_t* cm = !far ? &colmask[static_cast<size_t>(j - a)] : nullptr;
                    uint64_t busy = rowmask | (cm ? *cm : 0);
                    if (!~busy) {  // slot congested: scatter through the far path
                        far = true;
                        cm = nullptr;
                    }
                    if (far) {  // handled entirely by the patch pass (row and transposed)
                        o.far_i.push_back(i);
                        o.far_j.push_back(j);
                        o.far_v.push_back(val[k]);
                        continue;
                    }
                    const int r = __builtin_ctzll(~busy);
                    rowmask |= 1ull << r;
                    if (!*cm) touched.push_back(j - a);
                    *cm |= 1ull << r;
                    hi = std::max<int32_t>(hi, j + 1);
                    assign[t].push_back({r, k});
                    R = std::max(R, r + 1);
                }
            }
            // rounds whose window targets are disjoint may run back to back
            // without a block barrier between them: conflict[r] = rounds
            // sharing a target slot with round r; execution order = pairs of
            // disjoint rounds (greedy) then singles, never two elided
            // barriers in a row, the sub-tile's last chunk always barriered
            std::vector<uint64_t> conflict(kS3RoundCap, 0);
            for (int32_t sl : touched) {
                uint64_t mm = colmask[static_cast<size_t>(sl)];
                const uint64_t all = mm;
                while (mm) {
                    const int r = __builtin_ctzll(mm);
                    mm &= mm - 1;
                    conflict[r] |= all;
                }
            }
            for (int32_t sl : touched) colmask[static_cast<size_t>(sl)] = 0;
            R = std::max(R, 1);  // every sub-tile is one pipeline item at least
            std::vector<int> order, pos_of(R, -1);
            for (int r = 0; r < R; ++r) {
                if (pos_of[r] >= 0) continue;
                int mate = -1;
                if (kS3Pairs)
                    for (int t2 = r + 1; t2 < R; ++t2)
                        if (pos_of[t2] < 0 && !((conflict[r] >> t2) & 1)) {
                            mate = t2;
                            break;
                        }
                pos_of[r] = static_cast<int>(order.size());
                order.push_back(r);
                o.nobar.push_back(mate >= 0 ? 1 : 0);
                if (mate >= 0) {
                    pos_of[mate] = static_cast<int>(order.size());
                    order.push_back(mate);
                    o.nobar.push_back(0);
                }
            }
            const size_t basei = o.sell.size() / kStageBytes;  // in chunks, block-local
            o.rounds.push_back(R);
            o.sell.resize((basei + R) * kStageBytes);
            for (size_t ch = basei; ch < basei + R; ++ch) {  // values 0.0, columns -1 (padding)
                std::memset(&o.sell[ch * kStageBytes], 0, kRows * 8);
                std::memset(&o.sell[ch * kStageBytes + kRows * 8], 0xff, kRows * 2);
            }
            for (int32_t t = 0; t < rows; ++t)
                for (auto [r, k] : assign[t]) {
                    unsigned char* ch = &o.sell[(basei + pos_of[r]) * kStageBytes];
                    reinterpret_cast<double*>(ch)[s3_val_pos(t, T3)] = val[k];
                    reinterpret_cast<int16_t*>(ch + kRows * 8)[s3_col_pos(t, T3)] =
                        static_cast<int16_t>(col[k] - a);  // < W <= 32767
                }
            o.slots += static_cast<int64_t>(R) * S;
        }
        o.spill_hi = hi;
    };
    {
        const int T = std::max(1, std::min<int>(P, static_cast<int>(std::thread::hardware_concurrency())));
        std::atomic<int> next{0};
        auto worker = [&] {
            std::vector<uint64_t> colmask(static_cast<size_t>(W), 0);
            std::vector<int32_t> touched;
            for (int c; (c = next.fetch_add(1)) < P;) do_block(c, colmask, touched);
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
    }
    // merge in block order
    std::vector<int32_t> cta_sub(P + 1, 0), sub_rounds;
    std::vector<char> sub_nobar;  // per chunk in SELL order: no barrier after it
    std::vector<int64_t> sub_base;
    std::vector<int32_t> spill_hi(P), far_i, far_j, long_rows;
    std::vector<double> far_v;
    int64_t nchunks = 0, total_slots = 0;
    for (int c = 0; c < P; ++c) {
        const BlockOut& o = outs[c];
        cta_sub[c] = static_cast<int32_t>(sub_rounds.size());
        for (int32_t R : o.rounds) {
            sub_base.push_back(nchunks);
            sub_rounds.push_back(R);
            nchunks += R;
        }
        sub_nobar.insert(sub_nobar.end(), o.nobar.begin(), o.nobar.end());
        far_i.insert(far_i.end(), o.far_i.begin(), o.far_i.end());
        far_j.insert(far_j.end(), o.far_j.begin(), o.far_j.end());
        far_v.insert(far_v.end(), o.far_v.begin(), o.far_v.end());
        long_rows.insert(long_rows.end(), o.long_rows.begin(), o.long_rows.end());
        spill_hi[c] = o.spill_hi;
        total_slots += o.slots;
    }
    std::vector<unsigned char> sell(static_cast<size_t>(nchunks) * kStageBytes);
    {
        size_t pos = 0;
        for (auto& o : outs) {
            if (!o.sell.empty()) std::memcpy(&sell[pos], o.sell.data(), o.sell.size());
            pos += o.sell.size();
            std::vector<unsigned char>().swap(o.sell);
        }
    }
    cta_sub[P] = static_cast<int32_t>(sub_rounds.size());
    // per-block chunk table: one entry per (sub-tile, round), in SELL order
    // per block: real chunks, padded to a multiple of kStages, + kGD + 1 look-ahead
    std::vector<int32_t> cta_chunk(P + 1, 0), chunk_meta, cta_qreal(P, 0);
    std::vector<int64_t> cta_base(P, 0);
    for (int c = 0; c < P; ++c) {
        cta_chunk[c] = static_cast<int32_t>(chunk_meta.size());
        cta_base[c] = cta_sub[c] < cta_sub[c + 1] ? sub_base[cta_sub[c]] : 0;
        int q = 0;
        for (int sidx = cta_sub[c]; sidx < cta_sub[c + 1]; ++sidx) {
            const int R = sub_rounds[sidx];
            const int64_t q0g = sub_base[sidx];
            for (int r = 0; r < R; ++r, ++q)
                chunk_meta.push_back(((sidx - cta_sub[c]) << 9) | r | (r == R - 1 ? 128 : 0) |
                                     (sub_nobar[q0g + r] ? 256 : 0));
        }
        cta_qreal[c] = q;
        const int qp = (q + kStages - 1) / kStages * kStages;
        for (; q < qp + kGD + 1; ++q) chunk_meta.push_back(kMetaEmpty);
    }
    cta_chunk[P] = static_cast<int32_t>(chunk_meta.size());
    L.padded = total_slots;
    L.far = static_cast<int64_t>(far_i.size());

    // spill layout and head ranges
    std::vector<int64_t> spill_off(P);
    int64_t so = 0;
    for (int c = 0; c < P; ++c) {
        spill_off[c] = so;
        so += std::max<int32_t>(0, spill_hi[c] - bnd[c + 1]);
    }
    L.spill_total = so;
    std::vector<int32_t> head_end(P), first_src(P);
    for (int d = 0; d < P; ++d) {
        int32_t he = bnd[d];
        int32_t fs = d;
        for (int c = 0; c < d; ++c)
            if (spill_hi[c] > bnd[d]) {
                he = std::max<int32_t>(he, std::min<int32_t>(spill_hi[c], bnd[d + 1]));
                fs = std::min(fs, c);
            }
        head_end[d] = he;
        first_src[d] = fs;
    }
    // fixup blocks: <= kFixRows head rows of one destination each, with the
    // sources whose spill range meets them (ascending) -- 3 int4 per block:
    // (j0, j1, nsrc, list offset), (s0, hi) x 2, spill base (off - s0) x 2
    std::vector<int32_t> segs, seg_src;
    for (int d = 0; d < P; ++d)
        for (int32_t j = bnd[d]; j < head_end[d]; j += kFixRows) {
            const int32_t j1 = std::min<int32_t>(head_end[d], j + kFixRows);
            const int32_t list = static_cast<int32_t>(seg_src.size());
            for (int c = first_src[d]; c < d; ++c)
                if (spill_hi[c] > j && bnd[c + 1] < j1) seg_src.push_back(c);
            const int32_t ns = static_cast<int32_t>(seg_src.size()) - list;
            int32_t rng[4] = {0, 0, 0, 0};
            int64_t base[2] = {0, 0};
            for (int k = 0; k < std::min(ns, 2); ++k) {
                const int c = seg_src[list + k];
                rng[2 * k] = bnd[c + 1];
                rng[2 * k + 1] = spill_hi[c];
                base[k] = spill_off[c] - bnd[c + 1];
            }
            const int32_t v[12] = {j, j1, ns, list, rng[0], rng[1], rng[2], rng[3],
                                   static_cast<int32_t>(base[0] & 0xffffffff),
                                   static_cast<int32_t>(base[0] >> 32),
                                   static_cast<int32_t>(base[1] & 0xffffffff),
                                   static_cast<int32_t>(base[1] >> 32)};
            segs.insert(segs.end(), v, v + 12);
        }
    L.nsegs = static_cast<int64_t>(segs.size() / 12);

    auto up32 = [&](DBuf<int32_t>& d, const std::vector<int32_t>& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        if (!h.empty())
            KTB_CUDA(cudaMemcpyAsync(d.p, h.data(), 4 * h.size(), cudaMemcpyHostToDevice, st));
    };
    auto up64 = [&](DBuf<int64_t>& d, const std::vector<int64_t>& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        if (!h.empty())
            KTB_CUDA(cudaMemcpyAsync(d.p, h.data(), 8 * h.size(), cudaMemcpyHostToDevice, st));
    };
    auto upd = [&](DBuf<double>& d, const std::vector<double>& h) {
        d.alloc(std::max<size_t>(h.size(), 1));
        if (!h.empty())
            KTB_CUDA(cudaMemcpyAsync(d.p, h.data(), 8 * h.size(), cudaMemcpyHostToDevice, st));
    };
    up32(L.cta_chunk, cta_chunk);
    up32(L.chunk_meta, chunk_meta);
    up32(L.cta_qreal, cta_qreal);
    up64(L.cta_base, cta_base);
    L.sell.alloc(std::max<int64_t>(nchunks, 1) * kStageBytes);
    if (nchunks)
        KTB_CUDA(cudaMemcpyAsync(L.sell.p, sell.data(), nchunks * kStageBytes,
                                 cudaMemcpyHostToDevice, st));
    up32(L.spill_hi, spill_hi);
    up64(L.spill_off, spill_off);
    L.spill.alloc(std::max<int64_t>(so, 1));
    up32(L.segs, segs);
    up32(L.seg_src, seg_src);
    // far entries (both products) and long rows (row sum incl. diagonal and
    // transposed products) as contributions grouped by target row; the
    // stable sort keeps each target's contributions in a fixed order
    L.nlong = static_cast<int64_t>(long_rows.size());
    {
        struct Contrib {
            int32_t t, s;
            double v;
        };
        std::vector<Contrib> cs;
        for (size_t e = 0; e < far_i.size(); ++e) {
            cs.push_back({far_i[e], far_j[e], far_v[e]});
            cs.push_back({far_j[e], far_i[e], far_v[e]});
        }
        for (int32_t i : long_rows)
            for (int32_t k = rp[i]; k < rp[i + 1]; ++k) {
                cs.push_back({i, col[k], val[k]});
                if (col[k] != i) cs.push_back({col[k], i, val[k]});
            }
        std::stable_sort(cs.begin(), cs.end(),
                         [](const Contrib& a, const Contrib& b) { return a.t < b.t; });
        std::vector<int32_t> prow, prp(1, 0), psrc(cs.size());
        std::vector<double> pval(cs.size());
        for (size_t e = 0; e < cs.size(); ++e) {
            if (e == 0 || cs[e].t != cs[e - 1].t) {
                if (e) prp.push_back(static_cast<int32_t>(e));
                prow.push_back(cs[e].t);
            }
            psrc[e] = cs[e].s;
            pval[e] = cs[e].v;
        }
        if (!cs.empty()) prp.push_back(static_cast<int32_t>(cs.size()));
        L.npatch = static_cast<int64_t>(prow.size());
        up32(L.patch_row, prow);
        up32(L.patch_rp, prp);
        up32(L.patch_src, psrc);
        upd(L.patch_val, pval);
    }
    upd(L.diag, sdiag);
    KTB_CUDA(cudaStreamSynchronize(st));
    if (T3 == 512)
        allow_max_dynamic_smem(k_s3<512>);
    else
        allow_max_dynamic_smem(k_s3<256>);
    p->ctas = P;
    // (round 1 also carried an in-kernel cooperative merge, 85.2 vs 82.9 us,
    // and a persistent two-deep fixup, 82.3 vs 80.3-80.9 us on config 2; both
    // slower than this PDL-launched per-segment fixup and removed)
    p->launches = 1 + (L.nsegs ? 1 : 0) + (L.npatch ? 1 : 0);
    // padding slots (12 B each) + spill write/read + head-row read-modify-write
    // SELL stream (10 B/slot incl. padding) vs the 12 B/nnz model, + spill
    // write/read + head-row read-modify-write in the fixup; row_ptr unused
    p->extra_bytes = total_slots * 10 + 8 * n - nnz * 12 - 4 * (n + 1) + so * 8 * 2 + so * 8 * 2;
}

void s3_run(ktb_plan* p, const double* x, double* y) {
    auto& L = p->sw;
    const size_t smem = kS3SmemFixed + static_cast<size_t>(L.window) * 8;
    auto kern = p->cta_threads == 512 ? k_s3<512> : k_s3<256>;
    kern<<<L.ctas, p->cta_threads == 512 ? 512 : 256, smem, p->stream>>>(
        L.cta_row.p, L.cta_chunk.p, L.chunk_meta.p, L.cta_qreal.p, L.sell.p, L.cta_base.p,
        L.diag.p, x, y, L.window, L.reach, static_cast<int>(p->m->n), L.spill_hi.p,
        L.spill_off.p, L.spill.p);
    KTB_LAUNCH();
    if (L.nsegs) {  // the fixup's blocks launch early and wait for k_s3 (PDL)
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(L.nsegs));
        cfg.blockDim = dim3(256);
        cfg.stream = p->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        KTB_CUDA(cudaLaunchKernelEx(&cfg, k_s3_fixup, reinterpret_cast<const int4*>(L.segs.p),
                                    static_cast<const int32_t*>(L.seg_src.p),
                                    static_cast<const int32_t*>(L.cta_row.p),
                                    static_cast<const int32_t*>(L.spill_hi.p),
                                    static_cast<const int64_t*>(L.spill_off.p),
                                    static_cast<const double*>(L.spill.p), y));
    }
    if (L.npatch) {
        k_s3_patch<<<ceil_div(L.npatch, 8), 256, 0, p->stream>>>(
            L.patch_row.p, L.patch_rp.p, L.patch_src.p, L.patch_val.p, L.npatch, x, y);
        KTB_LAUNCH();
    }
}

}  // namespace ktb
