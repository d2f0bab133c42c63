// ktb_ptx.cuh -- sm_100a PTX helpers: mbarriers, TMA bulk copies, cache
// policies, named barriers.
#pragma once

#include <cstdint>

namespace ktb {

// ---- race stress build (KTB_CHAOS, libktb_chaos.so) ------------------------
// compute-sanitizer is unavailable on the GPU pool, so the hand-synchronised
// kernels (S3's TMA/mbarrier ring and window rounds, the MGS tag exchange, the
// ILU cluster sweep, the warp-tile carries) are stressed instead: every
// barrier, mbarrier wait and cross-CTA publish/poll is preceded by a
// pseudo-random per-thread sleep (0-2 us on 1 call in 4), which reorders
// warps, lanes and CTAs far beyond normal jitter, and KTB_DCHECK bounds
// checks trap. tests/test_chaos_gpu.py runs this build and requires results
// bitwise equal to the normal build's (a missing barrier or fence shows up
// as a wrong or non-reproducible y). Compiled out otherwise.
#ifdef KTB_CHAOS
__device__ __forceinline__ void chaos_delay(uint32_t salt) {
    uint32_t h = static_cast<uint32_t>(clock64()) ^ (salt * 0x9e3779b9u) ^
                 (blockIdx.x * 0x85ebca6bu) ^ (threadIdx.x * 0xc2b2ae35u);
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    if ((h & 3) == 0) __nanosleep((h >> 16) & 2047);
}
#define KTB_CHAOS_DELAY(salt) ::ktb::chaos_delay(static_cast<uint32_t>(salt))
#define KTB_DCHECK(c)        \
    do {                     \
        if (!(c)) __trap();  \
    } while (0)
// a block-wide barrier reached by every thread: delay, reconverge, sync
#define KTB_SYNC()                     \
    do {                               \
        KTB_CHAOS_DELAY(__LINE__);     \
        __syncwarp();                  \
        __syncthreads();               \
    } while (0)
#else
#define KTB_CHAOS_DELAY(salt) \
    do {                      \
    } while (0)
#define KTB_DCHECK(c) \
    do {              \
    } while (0)
#define KTB_SYNC() __syncthreads()
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order earlier generic-proxy accesses of shared memory before subsequent
// async-proxy (TMA) writes to it
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    KTB_CHAOS_DELAY(0x6d62);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 1-D TMA bulk copy global -> shared, completion counted on `bar` in bytes.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Bring [src, src+bytes) into L2 ahead of use (no completion tracking).
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Bring the bytes [begin, end) into L2 for ANY addresses: the range is widened
// to 16-byte boundaries (the bulk-prefetch alignment rule); the widened bytes
// stay inside the allocation's 256-byte granule, so nothing unmapped is named.
__device__ __forceinline__ void prefetch_l2_range(const void* begin, const void* end) {
    const uintptr_t lo = reinterpret_cast<uintptr_t>(begin) & ~uintptr_t(15);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(end) + 15) & ~uintptr_t(15);
    if (hi > lo)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
                     "r"(static_cast<uint32_t>(hi - lo))
                     : "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ double ldg_hint_f64(const double* p, uint64_t policy) {
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(policy));
    return r;
}

__device__ __forceinline__ void st_hint_f64(double* p, double v, uint64_t policy) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(policy)
                 : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace ktb
