// ktb_ilu.cu -- ILU(0) factorisation and its triangular solves on the device
// (SURVEY.md §8f row 4; ilu0.hpp:23-69 ilu0_factorize, :73-87 ilu0_apply).
//
// Every row keeps the reference's exact operation sequence -- the same loop,
// in the same order, one thread per row -- and the rows run in level
// order: level(i) = 1 + max level of the rows it reads. For the
// factorisation and the forward sweep those are the row's lower-pattern
// columns; for the backward sweep its upper-pattern columns. Products and
// sums are written with __dmul_rn / __dsub_rn / __ddiv_rn so nothing is
// contracted into an FMA: the factors and the solve are bitwise equal to the
// reference (built without FMA contraction, as the oracle is).
//
// Scheduling: a level with many rows is one launch across the GPU; a run of
// consecutive small levels is one single-CTA launch that walks the levels
// with a barrier between them (chains of one-row levels cost a barrier, not
// a launch). The apply's launch sequence (forward then backward) is captured
// once in a CUDA graph over internal buffers.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "ktb_internal.cuh"
#include "ktb_ptx.cuh"

namespace ktb {

namespace {

constexpr int kRunThreads = 1024;   // single-CTA level runs
constexpr int kSmallLevel = 2048;   // levels up to this many rows go into a run

enum { kFactor = 0, kForward = 1, kBackward = 2 };

template <int OP>
__device__ __forceinline__ void ilu_row(int32_t i, const int32_t* __restrict__ rp,
                                        const int32_t* __restrict__ col, double* val,
                                        const int32_t* __restrict__ diag,
                                        const double* __restrict__ r, double* z, int* err) {
    if (OP == kFactor) {  // ilu0.hpp:42-66
        const int32_t e = rp[i + 1];
        for (int32_t kp = rp[i]; kp < e; ++kp) {
            const int32_t k = col[kp];
            if (k >= i) break;
            const double pivot = val[diag[k]];
            const double lik = __ddiv_rn(val[kp], pivot);
            val[kp] = lik;
            int32_t pi = kp + 1, pk = diag[k] + 1;
            const int32_t ek = rp[k + 1];
            while (pi < e && pk < ek) {
                const int32_t ci = col[pi], ck = col[pk];
                if (ci == ck) {
                    val[pi] = __dsub_rn(val[pi], __dmul_rn(lik, val[pk]));
                    ++pi;
                    ++pk;
                } else if (ci < ck) {
                    ++pi;
                } else {
                    ++pk;
                }
            }
        }
        if (val[diag[i]] == 0.0) atomicMin(err, i);  // the reference's first raise
    } else if (OP == kForward) {  // ilu0.hpp:76-80 (unit L)
        double s = r[i];
        const int32_t d = diag[i];
        for (int32_t k = rp[i]; k < d; ++k) s = __dsub_rn(s, __dmul_rn(val[k], z[col[k]]));
        z[i] = s;
    } else {  // ilu0.hpp:81-86
        double s = z[i];
        const int32_t d = diag[i], e = rp[i + 1];
        for (int32_t k = d + 1; k < e; ++k) s = __dsub_rn(s, __dmul_rn(val[k], z[col[k]]));
        z[i] = __ddiv_rn(s, val[d]);
    }
}

template <int OP>
__global__ void __launch_bounds__(256) k_ilu_level(const int32_t* __restrict__ rows, int32_t cnt,
                                                   const int32_t* __restrict__ rp,
                                                   const int32_t* __restrict__ col, double* val,
                                                   const int32_t* __restrict__ diag,
                                                   const double* __restrict__ r, double* z,
                                                   int* err) {
    const int32_t t = blockIdx.x * 256 + threadIdx.x;
    if (t < cnt) ilu_row<OP>(rows[t], rp, col, val, diag, r, z, err);
}

template <int OP>
__global__ void __launch_bounds__(kRunThreads) k_ilu_run(const int32_t* __restrict__ rows,
                                                         const int32_t* __restrict__ lev_ptr,
                                                         int32_t lev0, int32_t lev1,
                                                         const int32_t* __restrict__ rp,
                                                         const int32_t* __restrict__ col,
                                                         double* val,
                                                         const int32_t* __restrict__ diag,
                                                         const double* __restrict__ r, double* z,
                                                         int* err) {
    for (int32_t l = lev0; l < lev1; ++l) {
        const int32_t b = lev_ptr[l], e = lev_ptr[l + 1];
        for (int32_t t = b + threadIdx.x; t < e; t += kRunThreads)
            ilu_row<OP>(rows[t], rp, col, val, diag, r, z, err);
        KTB_SYNC();  // this level's rows are final for the next
    }
}

// ---- the apply as one cluster launch per sweep ----------------------------
// The triangular sweeps are latency chains (levels x dependent round trips).
// A level-ordered packed copy of each triangle lets one thread-block cluster
// walk all levels of a sweep in one launch: the rows of a level are spread
// over the cluster's threads and a cluster barrier separates levels. Each
// row's record -- row id, entry count and its first kPre entries (the
// reference's order) -- sits at fixed-stride slots, so it is one round of
// independent loads, issued for the next level before the barrier; z is
// read through L2 (other SMs of the cluster wrote it); the z stores are
// fenced at cluster scope before those prefetch loads and the barrier
// arrival itself is relaxed, so the barrier does not wait for the prefetch.
// A level then costs one round of z gathers + the store fence + the barrier.
#ifndef KTB_ILU_CL_THREADS
#define KTB_ILU_CL_THREADS 512  // per CTA of the 16-CTA cluster: 2.46 ms per apply vs 3.0 ms at 1024
#endif
constexpr int kClThreads = KTB_ILU_CL_THREADS;
constexpr int kPre = 4;
#ifndef KTB_ILU_SPLIT_BARRIER
#define KTB_ILU_SPLIT_BARRIER 1
#endif

struct Packed {  // one sweep, rows in level order
    DBuf<int32_t> row, cnt;   // row id, strict-triangle entries of the row
    DBuf<int32_t> col;        // kPre x count (slot u of record t at u * count + t)
    DBuf<double> val;
    DBuf<double> dval;        // the factor's diagonal of the record's row (backward)
    DBuf<int32_t> xptr, xcol; // entries beyond kPre: CSR over records
    DBuf<double> xval;
    DBuf<int32_t> lev;        // levels+1 boundaries into the records
    int32_t nlev = 0;
    int64_t count = 0;
    int cluster = 0;          // CTAs per cluster (0: not used)
};

template <bool BACK>
__global__ void __launch_bounds__(kClThreads, 1)
    k_ilu_sweep_cluster(const int32_t* __restrict__ prow, const int32_t* __restrict__ pcnt,
                        const int32_t* __restrict__ pcol, const double* __restrict__ pval,
                        const double* __restrict__ pdiag,
                        const int32_t* __restrict__ xptr, const int32_t* __restrict__ xcol,
                        const double* __restrict__ xval, int64_t count,
                        const int32_t* __restrict__ lev, int32_t nlev,
                        const double* __restrict__ r, double* z) {
    const int nthr = kClThreads * static_cast<int>(gridDim.x);  // one cluster = the grid
    const int g = blockIdx.x * kClThreads + threadIdx.x;
    struct Rec {
        int32_t i, m;
        int32_t c[kPre];
        double v[kPre], d;
    };
    // a row's record: independent loads of setup data only (one round trip;
    // the fence before each barrier waits for it, so it must stay one trip)
    // records stream through once per apply: evict-first, so they do not
    // push z (re-read every level) out of L2
    uint64_t ef;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(ef));
    auto ldi = [&](const int32_t* p) {
        int32_t v;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
            : "=r"(v) : "l"(p), "l"(ef));
        return v;
    };
    auto ldd = [&](const double* p) {
        double v;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
            : "=d"(v) : "l"(p), "l"(ef));
        return v;
    };
    auto load = [&](int64_t t, Rec& R) {
        R.i = ldi(prow + t);
        R.m = ldi(pcnt + t);
#pragma unroll
        for (int u = 0; u < kPre; ++u) {
            R.c[u] = ldi(pcol + u * count + t);
            R.v[u] = ldd(pval + u * count + t);
        }
        R.d = BACK ? ldd(pdiag + t) : 1.0;
    };
    auto finish = [&](int64_t t, const Rec& R) {
        // the reference's order: s = r_i (z_i backward), s -= l_ik z_k in entry
        // order; the starting value goes out with the gathers (one round trip)
        double zk[kPre];
#pragma unroll
        for (int u = 0; u < kPre; ++u) zk[u] = u < R.m ? __ldcg(z + R.c[u]) : 0.0;
        double sacc = BACK ? __ldcg(z + R.i) : __ldg(r + R.i);
#pragma unroll
        for (int u = 0; u < kPre; ++u)
            if (u < R.m) sacc = __dsub_rn(sacc, __dmul_rn(R.v[u], zk[u]));
        if (R.m > kPre)
            for (int32_t k = __ldg(xptr + t); k < __ldg(xptr + t + 1); ++k)
                sacc = __dsub_rn(sacc, __dmul_rn(__ldg(xval + k), __ldcg(z + __ldg(xcol + k))));
        if (BACK) sacc = __ddiv_rn(sacc, R.d);
        __stcg(z + R.i, sacc);
    };
    Rec cur{}, nxt{};
    int32_t lb = nlev > 0 ? __ldg(lev) : 0, le = nlev > 0 ? __ldg(lev + 1) : 0;
    if (nlev > 0 && lb + g < le) load(lb + g, cur);
    for (int32_t l = 0; l < nlev; ++l) {
        const int32_t nb = l + 1 < nlev ? __ldg(lev + l + 1) : 0;
        const int32_t ne = l + 1 < nlev ? __ldg(lev + l + 2) : 0;
        // the records two levels ahead are pulled into L2 (bulk prefetch: no
        // completion to wait for, so the fence below does not wait for it)
        if (l + 2 < nlev && threadIdx.x < 11) {
            const int64_t b2 = __ldg(lev + l + 2), e2 = __ldg(lev + l + 3);
            const int a = threadIdx.x;  // one array per thread: row, cnt, col x kPre, val x kPre, d
            const char* base;
            int es;
            if (a == 0) {
                base = reinterpret_cast<const char*>(prow);
                es = 4;
            } else if (a == 1) {
                base = reinterpret_cast<const char*>(pcnt);
                es = 4;
            } else if (a < 2 + kPre) {
                base = reinterpret_cast<const char*>(pcol + (a - 2) * count);
                es = 4;
            } else if (a < 2 + 2 * kPre) {
                base = reinterpret_cast<const char*>(pval + (a - 2 - kPre) * count);
                es = 8;
            } else {
                base = reinterpret_cast<const char*>(pdiag);
                es = 8;
            }
            if (blockIdx.x == static_cast<unsigned>(a) % gridDim.x && (BACK || a != 2 + 2 * kPre)) {
                const uintptr_t lo = reinterpret_cast<uintptr_t>(base + b2 * es) & ~uintptr_t(15);
                const uintptr_t hi = (reinterpret_cast<uintptr_t>(base + e2 * es) + 15) & ~uintptr_t(15);
                if (hi > lo)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo),
                                 "r"(static_cast<uint32_t>(hi - lo))
                                 : "memory");
            }
        }
        if (lb + g < le) finish(lb + g, cur);
        for (int32_t t = lb + g + nthr; t < le; t += nthr) {
            Rec R;
            load(t, R);
            finish(t, R);
        }
        // z stores ordered before the barrier; the next level's first record
        // (L2-resident: bulk-prefetched two levels ago) is loaded after the
        // fence, so the fence does not wait for it, and lands during the
        // barrier
#if KTB_ILU_SPLIT_BARRIER
        // split-phase: the arrive releases this level's z stores, the next
        // record's loads go out between arrive and wait
        KTB_CHAOS_DELAY(0x696c);
        __syncwarp();
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        if (l + 1 < nlev && nb + g < ne) load(nb + g, nxt);
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#else
        KTB_CHAOS_DELAY(0x696d);
        __syncwarp();
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        if (l + 1 < nlev && nb + g < ne) load(nb + g, nxt);
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;" ::: "memory");
#endif
        cur = nxt;
        lb = nb;
        le = ne;
    }
}

struct Schedule {
    std::vector<int32_t> ptr;  // level boundaries into rows
    DBuf<int32_t> rows, dptr;
    struct Seg {
        bool run;
        int32_t l0, l1;
    };
    std::vector<Seg> segs;
};

// rows grouped by level (ascending rows within a level) + launch segments
void build_schedule(const std::vector<int32_t>& level, int32_t nlev, Schedule& S) {
    const int64_t n = static_cast<int64_t>(level.size());
    S.ptr.assign(nlev + 1, 0);
    for (int32_t l : level) ++S.ptr[l + 1];
    for (int32_t l = 0; l < nlev; ++l) S.ptr[l + 1] += S.ptr[l];
    std::vector<int32_t> next(S.ptr.begin(), S.ptr.end() - 1), rows(n);
    for (int64_t i = 0; i < n; ++i) rows[next[level[i]]++] = static_cast<int32_t>(i);
    S.rows.alloc(std::max<int64_t>(n, 1));
    S.dptr.alloc(nlev + 1);
    if (n) KTB_CUDA(cudaMemcpy(S.rows.p, rows.data(), 4 * n, cudaMemcpyHostToDevice));
    KTB_CUDA(cudaMemcpy(S.dptr.p, S.ptr.data(), 4 * (nlev + 1), cudaMemcpyHostToDevice));
    S.segs.clear();
    for (int32_t l = 0; l < nlev;) {
        if (S.ptr[l + 1] - S.ptr[l] > kSmallLevel) {
            S.segs.push_back({false, l, l + 1});
            ++l;
            continue;
        }
        int32_t e = l;
        while (e < nlev && S.ptr[e + 1] - S.ptr[e] <= kSmallLevel) ++e;
        S.segs.push_back({true, l, e});
        l = e;
    }
}

template <int OP>
void run_schedule(const Schedule& S, const ktb_ilu* f, const double* r, double* z, int* err,
                  cudaStream_t s);

}  // namespace

}  // namespace ktb

struct ktb_ilu {
    int device = 0;
    int64_t n = 0, nnz = 0;
    ktb::DBuf<int32_t> rp, col, diag;
    ktb::DBuf<double> val;
    ktb::Schedule lower, upper;
    ktb::Packed plow, pup;  // cluster apply (when the device supports the cluster)
    ktb::DBuf<double> rbuf, zbuf;
    ktb::DBuf<int> err;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t apply_graph = nullptr;
    int64_t launches = 0;  // per apply
    // the applies share rbuf/zbuf: each apply's stream waits for the previous
    // apply (on whatever stream it ran), so applies of one factor on several
    // streams serialise instead of racing on the buffers
    cudaEvent_t done = nullptr;
    ~ktb_ilu() {
        if (apply_graph) cudaGraphExecDestroy(apply_graph);
        if (done) cudaEventDestroy(done);
        if (stream) cudaStreamDestroy(stream);
    }
};

namespace ktb {
namespace {

template <int OP>
void run_schedule(const Schedule& S, const ktb_ilu* f, const double* r, double* z, int* err,
                  cudaStream_t s) {
    for (const auto& g : S.segs) {
        if (g.run) {
            k_ilu_run<OP><<<1, kRunThreads, 0, s>>>(S.rows.p, S.dptr.p, g.l0, g.l1, f->rp.p,
                                                    f->col.p, f->val.p, f->diag.p, r, z, err);
        } else {
            const int32_t b = S.ptr[g.l0], cnt = S.ptr[g.l0 + 1] - b;
            k_ilu_level<OP><<<ceil_div(cnt, 256), 256, 0, s>>>(S.rows.p + b, cnt, f->rp.p,
                                                               f->col.p, f->val.p, f->diag.p, r,
                                                               z, err);
        }
        KTB_LAUNCH();
    }
}

// largest cluster (16 non-portable, else 8) the sweep kernel can run as;
// 0 = use the per-level launches (KTB_ILU_LEVEL_LAUNCHES=1 forces that)
int cluster_size_for_sweeps(int device) {
    const char* env = std::getenv("KTB_ILU_LEVEL_LAUNCHES");
    if (env && env[0] == '1') return 0;
    int supported = 0;
    cudaDeviceGetAttribute(&supported, cudaDevAttrClusterLaunch, device);
    if (!supported) return 0;
    for (const void* fn : {reinterpret_cast<const void*>(&k_ilu_sweep_cluster<false>),
                           reinterpret_cast<const void*>(&k_ilu_sweep_cluster<true>)})
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess) {
            cudaGetLastError();
            return 0;
        }
    for (int cs : {16, 8}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(kClThreads);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, &k_ilu_sweep_cluster<false>, &cfg) ==
                cudaSuccess &&
            nclusters >= 1)
            return cs;
        cudaGetLastError();
    }
    return 0;
}

__global__ void k_pack_counts(const int32_t* __restrict__ rows, int64_t n,
                              const int32_t* __restrict__ rp, const int32_t* __restrict__ diag,
                              bool upper, int32_t* __restrict__ cnt, int32_t* __restrict__ xcnt) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const int32_t i = rows[t];
    const int32_t b = upper ? diag[i] + 1 : rp[i], e = upper ? rp[i + 1] : diag[i];
    cnt[t] = e - b;
    xcnt[t] = max(0, e - b - kPre);
}

__global__ void k_pack_fill(const int32_t* __restrict__ rows, int64_t n,
                            const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const double* __restrict__ val, const int32_t* __restrict__ diag,
                            bool upper, int32_t* __restrict__ pc, double* __restrict__ pv,
                            double* __restrict__ pd, const int32_t* __restrict__ xptr,
                            int32_t* __restrict__ xc, double* __restrict__ xv) {
    const int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const int32_t i = rows[t];
    const int32_t b = upper ? diag[i] + 1 : rp[i], e = upper ? rp[i + 1] : diag[i];
    for (int u = 0; u < kPre; ++u) {
        const bool ok = b + u < e;
        pc[u * n + t] = ok ? col[b + u] : 0;
        pv[u * n + t] = ok ? val[b + u] : 0.0;
    }
    pd[t] = val[diag[i]];
    for (int32_t k = b + kPre; k < e; ++k) {
        xc[xptr[t] + k - b - kPre] = col[k];
        xv[xptr[t] + k - b - kPre] = val[k];
    }
}

// rows in schedule (level) order with their strict-triangle entries, values
// from the factors (lower: unit L below the diagonal; upper: above it); built
// on the device from the factors in place
void build_packed(const Schedule& S, const ktb_ilu* f, bool upper, Packed& P, cudaStream_t s) {
    const int64_t n = f->n;
    P.nlev = static_cast<int32_t>(S.ptr.size()) - 1;
    P.count = n;
    P.row.alloc(std::max<int64_t>(n, 1));
    P.cnt.alloc(std::max<int64_t>(n, 1));
    P.xptr.alloc(n + 1);
    KTB_CUDA(cudaMemcpyAsync(P.row.p, S.rows.p, 4 * n, cudaMemcpyDeviceToDevice, s));
    k_pack_counts<<<ceil_div(n, 256), 256, 0, s>>>(S.rows.p, n, f->rp.p, f->diag.p, upper,
                                                   P.cnt.p, P.xptr.p);
    KTB_LAUNCH();
    size_t tmp = 0;
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, P.xptr.p, P.xptr.p, n + 1, s));
    DBuf<unsigned char> scratch(tmp);
    KTB_CUDA(cudaMemsetAsync(P.xptr.p + n, 0, 4, s));
    KTB_CUDA(cub::DeviceScan::ExclusiveSum(scratch.p, tmp, P.xptr.p, P.xptr.p, n + 1, s));
    int32_t nx = 0;
    KTB_CUDA(cudaMemcpyAsync(&nx, P.xptr.p + n, 4, cudaMemcpyDeviceToHost, s));
    KTB_CUDA(cudaStreamSynchronize(s));
    P.col.alloc(static_cast<size_t>(kPre) * std::max<int64_t>(n, 1));
    P.val.alloc(static_cast<size_t>(kPre) * std::max<int64_t>(n, 1));
    P.dval.alloc(std::max<int64_t>(n, 1));
    P.xcol.alloc(std::max(nx, 1));
    P.xval.alloc(std::max(nx, 1));
    k_pack_fill<<<ceil_div(n, 256), 256, 0, s>>>(S.rows.p, n, f->rp.p, f->col.p, f->val.p,
                                                 f->diag.p, upper, P.col.p, P.val.p, P.dval.p,
                                                 P.xptr.p, P.xcol.p, P.xval.p);
    KTB_LAUNCH();
    P.lev.alloc(S.ptr.size());
    KTB_CUDA(cudaMemcpyAsync(P.lev.p, S.ptr.data(), 4 * S.ptr.size(), cudaMemcpyHostToDevice, s));
    KTB_CUDA(cudaStreamSynchronize(s));
}

template <bool BACK>
void launch_cluster_sweep(const Packed& P, const ktb_ilu* f, const double* r, double* z,
                          cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(P.cluster);
    cfg.blockDim = dim3(kClThreads);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = P.cluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    KTB_CUDA(cudaLaunchKernelEx(&cfg, k_ilu_sweep_cluster<BACK>,
                                static_cast<const int32_t*>(P.row.p),
                                static_cast<const int32_t*>(P.cnt.p),
                                static_cast<const int32_t*>(P.col.p),
                                static_cast<const double*>(P.val.p),
                                static_cast<const double*>(P.dval.p),
                                static_cast<const int32_t*>(P.xptr.p),
                                static_cast<const int32_t*>(P.xcol.p),
                                static_cast<const double*>(P.xval.p), P.count,
                                static_cast<const int32_t*>(P.lev.p), P.nlev, r, z));
}

}  // namespace

ktb_ilu* ilu0_create(const ktb_matrix* m, cudaStream_t user_stream) {
    require(m != nullptr, "matrix: null handle");
    require(m->kind == KTB_GENERAL, "ilu0: general matrices only");
    DeviceGuard g(m->device);
    auto f = std::make_unique<ktb_ilu>();
    f->device = m->device;
    f->n = m->n;
    f->nnz = m->nnz;
    const int64_t n = m->n, nnz = m->nnz;
    KTB_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
    cudaStream_t s = f->stream;
    if (user_stream) {  // order after the caller's producer of the matrix
        cudaEvent_t ev;
        KTB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        KTB_CUDA(cudaEventRecord(ev, user_stream));
        KTB_CUDA(cudaStreamWaitEvent(s, ev, 0));
        KTB_CUDA(cudaEventDestroy(ev));
    }
    // host analysis: diagonal positions (ilu0.hpp:31-40) and the two level maps
    std::vector<int32_t> rp(n + 1), col(nnz), diag(n, -1);
    KTB_CUDA(cudaMemcpy(rp.data(), m->row_ptr.p, 4 * (n + 1), cudaMemcpyDeviceToHost));
    if (nnz) KTB_CUDA(cudaMemcpy(col.data(), m->col.p, 4 * nnz, cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < n; ++i) {
        for (int32_t k = rp[i]; k < rp[i + 1]; ++k)
            if (col[k] == i) {
                diag[i] = k;
                break;
            }
        if (diag[i] < 0)
            throw Invalid("ilu0: structurally missing diagonal in row " + std::to_string(i));
    }
    std::vector<int32_t> lev(n, 0), ulev(n, 0);
    int32_t nl = n ? 1 : 0, nu = n ? 1 : 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t l = 0;
        for (int32_t k = rp[i]; k < diag[i]; ++k) l = std::max(l, lev[col[k]] + 1);
        lev[i] = l;
        nl = std::max(nl, l + 1);
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        int32_t l = 0;
        for (int32_t k = diag[i] + 1; k < rp[i + 1]; ++k) l = std::max(l, ulev[col[k]] + 1);
        ulev[i] = l;
        nu = std::max(nu, l + 1);
    }
    build_schedule(lev, nl, f->lower);
    build_schedule(ulev, nu, f->upper);
    // device copies of the pattern; factors start as A's values
    f->rp.alloc(n + 1);
    f->col.alloc(std::max<int64_t>(nnz, 1));
    f->val.alloc(std::max<int64_t>(nnz, 1));
    f->diag.alloc(std::max<int64_t>(n, 1));
    f->err.alloc(1);
    f->rbuf.alloc(std::max<int64_t>(n, 1));
    f->zbuf.alloc(std::max<int64_t>(n, 1));
    KTB_CUDA(cudaMemcpyAsync(f->rp.p, m->row_ptr.p, 4 * (n + 1), cudaMemcpyDeviceToDevice, s));
    if (nnz) {
        KTB_CUDA(cudaMemcpyAsync(f->col.p, m->col.p, 4 * nnz, cudaMemcpyDeviceToDevice, s));
        KTB_CUDA(cudaMemcpyAsync(f->val.p, m->val.p, 8 * nnz, cudaMemcpyDeviceToDevice, s));
    }
    if (n) KTB_CUDA(cudaMemcpyAsync(f->diag.p, diag.data(), 4 * n, cudaMemcpyHostToDevice, s));
    const int big = 0x7fffffff;
    KTB_CUDA(cudaMemcpyAsync(f->err.p, &big, 4, cudaMemcpyHostToDevice, s));
    run_schedule<kFactor>(f->lower, f.get(), nullptr, nullptr, f->err.p, s);
    int first_zero = big;
    KTB_CUDA(cudaMemcpyAsync(&first_zero, f->err.p, 4, cudaMemcpyDeviceToHost, s));
    KTB_CUDA(cudaStreamSynchronize(s));
    if (first_zero != big)
        throw Invalid("ilu0: zero pivot at row " + std::to_string(first_zero));
    // packed, level-ordered triangles for the cluster sweeps (factor values)
    const int cs = cluster_size_for_sweeps(m->device);
    if (cs > 0 && n > 0) {
        build_packed(f->lower, f.get(), false, f->plow, s);
        build_packed(f->upper, f.get(), true, f->pup, s);
        f->plow.cluster = f->pup.cluster = cs;
    }
    // the apply: forward then backward sweep over rbuf -> zbuf, as one graph
    cudaGraph_t graph;
    KTB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    if (f->plow.cluster) {
        launch_cluster_sweep<false>(f->plow, f.get(), f->rbuf.p, f->zbuf.p, s);
        launch_cluster_sweep<true>(f->pup, f.get(), f->rbuf.p, f->zbuf.p, s);
    } else {
        run_schedule<kForward>(f->lower, f.get(), f->rbuf.p, f->zbuf.p, f->err.p, s);
        run_schedule<kBackward>(f->upper, f.get(), f->rbuf.p, f->zbuf.p, f->err.p, s);
    }
    KTB_CUDA(cudaStreamEndCapture(s, &graph));
    const cudaError_t ie = cudaGraphInstantiate(&f->apply_graph, graph, 0);
    cudaGraphDestroy(graph);
    KTB_CUDA(ie);
    f->launches = f->plow.cluster ? 2
                                  : static_cast<int64_t>(f->lower.segs.size() +
                                                         f->upper.segs.size());
    return f.release();
}

void ilu0_info(const ktb_ilu* f, int64_t* n, int64_t* nl, int64_t* nu, int64_t* launches) {
    if (n) *n = f->n;
    if (nl) *nl = static_cast<int64_t>(f->lower.ptr.size()) - 1;
    if (nu) *nu = static_cast<int64_t>(f->upper.ptr.size()) - 1;
    if (launches) *launches = f->launches;
}

void ilu0_download(const ktb_ilu* f, int32_t* diag, double* val) {
    DeviceGuard g(f->device);
    KTB_CUDA(cudaStreamSynchronize(f->stream));
    if (diag && f->n) KTB_CUDA(cudaMemcpy(diag, f->diag.p, 4 * f->n, cudaMemcpyDeviceToHost));
    if (val && f->nnz) KTB_CUDA(cudaMemcpy(val, f->val.p, 8 * f->nnz, cudaMemcpyDeviceToHost));
}

void ilu0_destroy(ktb_ilu* f) {
    if (!f) return;
    DeviceGuard g(f->device);
    delete f;
}

// Runs on stream `s` exactly as given (NULL = the legacy default stream, the
// one a caller on torch's default stream is ordered with).
void ilu0_apply(ktb_ilu* f, const double* r, double* z, cudaStream_t s) {
    DeviceGuard g(f->device);
    const int64_t n = f->n;
    if (n == 0) return;
    if (!f->done) {
        KTB_CUDA(cudaEventCreateWithFlags(&f->done, cudaEventDisableTiming));
    } else {
        KTB_CUDA(cudaStreamWaitEvent(s, f->done, 0));
    }
    KTB_CUDA(cudaMemcpyAsync(f->rbuf.p, r, 8 * n, cudaMemcpyDeviceToDevice, s));
    KTB_CUDA(cudaGraphLaunch(f->apply_graph, s));
    KTB_CUDA(cudaMemcpyAsync(z, f->zbuf.p, 8 * n, cudaMemcpyDeviceToDevice, s));
    KTB_CUDA(cudaEventRecord(f->done, s));
}

}  // namespace ktb
