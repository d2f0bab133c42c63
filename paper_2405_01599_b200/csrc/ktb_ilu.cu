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
#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "ktb_internal.cuh"

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
        __syncthreads();  // this level's rows are final for the next
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
    ktb::DBuf<double> rbuf, zbuf;
    ktb::DBuf<int> err;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t apply_graph = nullptr;
    int64_t launches = 0;  // per apply
    ~ktb_ilu() {
        if (apply_graph) cudaGraphExecDestroy(apply_graph);
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
    // the apply: forward then backward sweep over rbuf -> zbuf, as one graph
    cudaGraph_t graph;
    KTB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    run_schedule<kForward>(f->lower, f.get(), f->rbuf.p, f->zbuf.p, f->err.p, s);
    run_schedule<kBackward>(f->upper, f.get(), f->rbuf.p, f->zbuf.p, f->err.p, s);
    KTB_CUDA(cudaStreamEndCapture(s, &graph));
    const cudaError_t ie = cudaGraphInstantiate(&f->apply_graph, graph, 0);
    cudaGraphDestroy(graph);
    KTB_CUDA(ie);
    f->launches = static_cast<int64_t>(f->lower.segs.size() + f->upper.segs.size());
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
    KTB_CUDA(cudaMemcpyAsync(f->rbuf.p, r, 8 * n, cudaMemcpyDeviceToDevice, s));
    KTB_CUDA(cudaGraphLaunch(f->apply_graph, s));
    KTB_CUDA(cudaMemcpyAsync(z, f->zbuf.p, 8 * n, cudaMemcpyDeviceToDevice, s));
}

}  // namespace ktb
