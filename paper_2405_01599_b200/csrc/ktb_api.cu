// ktb_api.cu -- the extern "C" boundary of libktb (include/ktb.h), plan
// dispatch and the device-time kernel selector.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <limits>
#include <string>
#include <tuple>
#include <vector>

#include <functional>

#include "ktb_internal.cuh"

namespace ktb {
// defined in the kernel translation units
void u1_setup(ktb_plan* p);
void u1_run(ktb_plan* p, const double* x, double* y, int64_t r0, int64_t r1);
void u2_setup(ktb_plan* p);
void u2_run(ktb_plan* p, const double* x, double* y);
void u3_setup(ktb_plan* p);
void u3_run(ktb_plan* p, const double* x, double* y);
void s12_setup(ktb_plan* p);
void s12_run(ktb_plan* p, const double* x, double* y);
void s3_setup(ktb_plan* p);
void s3_run(ktb_plan* p, const double* x, double* y);
void reduction_regions_dev(const ktb_matrix* m, int P, const int32_t* d_bnd, int64_t* d_lo,
                           int64_t* d_hi, cudaStream_t s);
void bss_plan_size(const ktb_matrix* m, int64_t jl, int64_t* jl_eff, int64_t* total,
                   cudaStream_t s);
void bss_plan_copy(const ktb_matrix* m, int64_t jl, int64_t* h_start, int64_t* h_len,
                   int64_t* h_row, int64_t* h_lane, int64_t* h_rowptr, uint8_t* h_flag,
                   cudaStream_t s);
ktb_matrix* gen_stencil7(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1, bool slab,
                         double diag, double off, double cxm, double cxp, int device);
ktb_matrix* gen_stencil27_upper(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                                int device);
void seeded_vector_dev(int64_t n, uint64_t seed, int64_t offset, double* d_out, cudaStream_t s);
void gmres_run(ktb_plan* A, ktb_ilu* P, const double* b_host, double* x_host, int64_t m,
               double tol, int64_t max_iters, double* history, ktb_gmres_result* res);
ktb_matrix* gen_powerlaw(int64_t n, uint64_t seed, int64_t target, double empty_frac,
                         int64_t max_len, int device);
ktb_matrix* matrix_slice(const ktb_matrix* m, int64_t r0, int64_t r1);
void build_row_partition_rowptr(const int64_t* h_rp, int64_t n, int P, int scheme, int device,
                                int64_t* h_out);
void powerlaw_host(int64_t n, uint64_t seed, int64_t target, double empty_frac,
                   int64_t max_len, std::vector<int64_t>& rp, std::vector<int32_t>* col,
                   std::vector<double>* val);

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    // a launch check (cudaGetLastError) must only see this call's launches:
    // drop any non-sticky error an earlier call (or a caller's own runtime
    // use) left behind -- those were reported where they happened
    (void)cudaGetLastError();
    try {
        f();
        return KTB_OK;
    } catch (const Invalid& e) {
        g_err = e.what();
        return KTB_ERR_INVALID;
    } catch (const SelectError& e) {
        g_err = e.what();
        return KTB_ERR_SELECT;
    } catch (const CudaError& e) {
        g_err = e.what();
        return KTB_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return KTB_ERR_CUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return KTB_ERR_CUDA;
    }
}

bool is_sym_kernel(int k) { return k == KTB_S1 || k == KTB_S2 || k == KTB_S3; }
bool is_unsym_kernel(int k) { return k >= KTB_U1 && k <= KTB_U4; }

// csr.hpp:38-54, same checks and messages, on the caller's host arrays.
template <typename I>
void validate_host(int64_t n, const I* rp, const I* ci, bool upper, int64_t* max_row,
                   int64_t* bw, int64_t ncols = -1) {
    if (ncols < 0) ncols = n;
    require(n >= 0, "csr: negative dimension");
    require(rp != nullptr, "csr: row_ptr length != n+1");
    require(rp[0] == 0, "csr: row_ptr[0] != 0");
    const int64_t nnz = rp[n];
    require(nnz >= 0, "csr: row_ptr[n] != nnz");
    int64_t ml = 0, b = 0;
    for (int64_t i = 0; i < n; ++i) {
        require(rp[i] <= rp[i + 1], "csr: row_ptr not nondecreasing");
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            require(ci[k] >= 0 && ci[k] < ncols, "csr: column index out of range");
            if (k > rp[i]) require(ci[k - 1] < ci[k], "csr: columns not strictly increasing");
            if (upper) require(ci[k] >= i, "sym csr: entry below the diagonal");
        }
        ml = std::max<int64_t>(ml, rp[i + 1] - rp[i]);
        if (rp[i + 1] > rp[i]) b = std::max<int64_t>(b, static_cast<int64_t>(ci[rp[i + 1] - 1]) - i);
    }
    *max_row = ml;
    *bw = b;
}

template <typename I>
ktb_matrix* create_matrix(int64_t n, const I* rp, const I* ci, const double* v, int kind,
                          int device, int64_t ncols = -1) {
    require(kind == KTB_GENERAL || kind == KTB_SYM_UPPER, "csr: bad matrix kind");
    if (ncols < 0) ncols = n;
    require(ncols < (int64_t(1) << 31) - 1, "csr: n or nnz >= 2^31 does not fit the int32 device layout");
    int64_t ml = 0, bw = 0;
    validate_host(n, rp, ci, kind == KTB_SYM_UPPER, &ml, &bw, ncols);
    const int64_t nnz = rp[n];
    require(n < (int64_t(1) << 31) - 1 && nnz < (int64_t(1) << 31) - 1,
            "csr: n or nnz >= 2^31 does not fit the int32 device layout");
    DeviceGuard g(device);
    auto* m = new ktb_matrix();
    try {
        m->device = device;
        KTB_CUDA(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
        m->n = n;
        m->ncols = ncols;
        m->nnz = nnz;
        m->kind = kind;
        m->max_row_nnz = ml;
        m->bandwidth = bw;
        std::vector<int32_t> rp32(n + 1), ci32(nnz);
        for (int64_t i = 0; i <= n; ++i) rp32[i] = static_cast<int32_t>(rp[i]);
        for (int64_t k = 0; k < nnz; ++k) ci32[k] = static_cast<int32_t>(ci[k]);
        m->row_ptr.alloc(n + 1);
        m->col.alloc(nnz);
        m->val.alloc(nnz);
        KTB_CUDA(cudaMemcpy(m->row_ptr.p, rp32.data(), 4 * (n + 1), cudaMemcpyHostToDevice));
        if (nnz) {
            KTB_CUDA(cudaMemcpy(m->col.p, ci32.data(), 4 * nnz, cudaMemcpyHostToDevice));
            KTB_CUDA(cudaMemcpy(m->val.p, v, 8 * nnz, cudaMemcpyHostToDevice));
        }
    } catch (...) {
        delete m;
        throw;
    }
    return m;
}

}  // namespace

int guarded_call(const std::function<void()>& f) { return guarded(f); }

// read a buffer larger than L2 (evicts the dirty lines a preceding memset
// left, so a timed kernel starts with a cold and clean L2)
__global__ void k_flush_read(const double* __restrict__ a, int64_t n, double* sink) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        s += __ldcg(a + i);
    if (s == 1.2345e300) *sink = s;
}

void flush_read(const double* a, int64_t n, double* sink, cudaStream_t s) {
    k_flush_read<<<4 * kNumSMs, 512, 0, s>>>(a, n, sink);
    KTB_LAUNCH();
}

// A GENERAL n x ncols device matrix from int64 host CRS (halo row blocks).
ktb_matrix* matrix_create_rect(int64_t n, int64_t ncols, const int64_t* rp, const int64_t* ci,
                               const double* v, int device) {
    return create_matrix(n, rp, ci, v, KTB_GENERAL, device, ncols);
}

// ---------------------------------------------------------------- dispatch
void plan_setup(ktb_plan* p) {
    // param = variant | (CTA threads << 16): the launch shape rides in the
    // high bits so that a shape is an ordinary selector candidate
    if (p->param >= (int64_t(1) << 16)) {
        p->cta_threads = static_cast<int>((p->param >> 16) & 0xffff);
        p->param &= 0xffff;
    }
    switch (p->kernel) {
        case KTB_U1: u1_setup(p); break;
        case KTB_U2: u2_setup(p); break;
        case KTB_U3:
        case KTB_U4: u3_setup(p); break;
        case KTB_S1:
        case KTB_S2: s12_setup(p); break;
        case KTB_S3: s3_setup(p); break;
        default: throw Invalid("spmv: unknown kernel");
    }
}

ktb_plan* plan_create_internal(ktb_matrix* m, int kernel, int64_t param, int workers,
                               cudaStream_t stream) {
    DeviceGuard g(m->device);
    std::unique_ptr<ktb_plan> p(new ktb_plan());
    p->m = m;
    p->kernel = kernel;
    p->param = param;
    p->workers = workers > 0 ? workers : m->sm_count;
    if (stream) {
        p->stream = stream;
    } else {
        KTB_CUDA(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        p->own_stream = true;
    }
    if (m->n > 0) plan_setup(p.get());
    return p.release();
}

void plan_run(ktb_plan* p, const double* x, double* y, int64_t r0, int64_t r1) {
    if (p->m->n == 0) return;
    switch (p->kernel) {
        case KTB_U1: u1_run(p, x, y, r0, r1); break;
        case KTB_U2: u2_run(p, x, y); break;
        case KTB_U3:
        case KTB_U4: u3_run(p, x, y); break;
        case KTB_S1:
        case KTB_S2: s12_run(p, x, y); break;
        case KTB_S3: s3_run(p, x, y); break;
        default: throw Invalid("spmv: unknown kernel");
    }
}

}  // namespace ktb

ktb_matrix::~ktb_matrix() { delete expanded; }

ktb_plan::~ktb_plan() {
    if (own_stream && stream) cudaStreamDestroy(stream);
    delete long_plan;
    delete long_m;
    for (int b = 0; b < 2; ++b) {
        if (ev_in[b]) cudaEventDestroy(ev_in[b]);
        if (ev_comp[b]) cudaEventDestroy(ev_comp[b]);
        if (ev_out[b]) cudaEventDestroy(ev_out[b]);
    }
    if (cin) cudaStreamDestroy(cin);
    if (cout) cudaStreamDestroy(cout);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (side) cudaStreamDestroy(side);
}

using namespace ktb;

extern "C" {

const char* ktb_last_error(void) { return g_err.c_str(); }
int ktb_version(void) { return 1; }

int ktb_device_count(int* count) {
    return guarded([&] { KTB_CUDA(cudaGetDeviceCount(count)); });
}

int ktb_matrix_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                      const double* values, int kind, int device, ktb_matrix** out) {
    return guarded([&] { *out = create_matrix(n, row_ptr, col_idx, values, kind, device); });
}

int ktb_matrix_create_i32(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                          const double* values, int kind, int device, ktb_matrix** out) {
    return guarded([&] { *out = create_matrix(n, row_ptr, col_idx, values, kind, device); });
}

int ktb_matrix_destroy(ktb_matrix* m) {
    return guarded([&] {
        if (m) {
            DeviceGuard g(m->device);
            delete m;
        }
    });
}

int ktb_matrix_info(const ktb_matrix* m, int64_t* n, int64_t* nnz, int* kind,
                    int64_t* max_row_nnz, int64_t* bandwidth) {
    return guarded([&] {
        require(m != nullptr, "matrix: null handle");
        if (n) *n = m->n;
        if (nnz) *nnz = m->nnz;
        if (kind) *kind = m->kind;
        if (max_row_nnz) *max_row_nnz = m->max_row_nnz;
        if (bandwidth) *bandwidth = m->bandwidth;
    });
}

int ktb_matrix_download(const ktb_matrix* m, int32_t* row_ptr, int32_t* col_idx,
                        double* values) {
    return guarded([&] {
        DeviceGuard g(m->device);
        if (row_ptr)
            KTB_CUDA(cudaMemcpy(row_ptr, m->row_ptr.p, 4 * (m->n + 1), cudaMemcpyDeviceToHost));
        if (col_idx && m->nnz)
            KTB_CUDA(cudaMemcpy(col_idx, m->col.p, 4 * m->nnz, cudaMemcpyDeviceToHost));
        if (values && m->nnz)
            KTB_CUDA(cudaMemcpy(values, m->val.p, 8 * m->nnz, cudaMemcpyDeviceToHost));
    });
}

int ktb_matrix_slice(const ktb_matrix* m, int64_t row_begin, int64_t row_end,
                     ktb_matrix** out) {
    return guarded([&] { *out = matrix_slice(m, row_begin, row_end); });
}

int ktb_ilu0_create(const ktb_matrix* m, void* stream, ktb_ilu** out) {
    return guarded([&] { *out = ilu0_create(m, static_cast<cudaStream_t>(stream)); });
}

int ktb_ilu0_info(const ktb_ilu* f, int64_t* n, int64_t* lower_levels, int64_t* upper_levels,
                  int64_t* launches_per_apply) {
    return guarded([&] {
        require(f != nullptr, "ilu0: null handle");
        ilu0_info(f, n, lower_levels, upper_levels, launches_per_apply);
    });
}

int ktb_ilu0_download(const ktb_ilu* f, int32_t* diag_ptr, double* values) {
    return guarded([&] {
        require(f != nullptr, "ilu0: null handle");
        ilu0_download(f, diag_ptr, values);
    });
}

int ktb_ilu0_apply(ktb_ilu* f, const double* r, double* z, int ptr_kind, void* stream) {
    return guarded([&] {
        require(f != nullptr, "ilu0: null handle");
        require(ptr_kind == KTB_PTR_HOST || ptr_kind == KTB_PTR_DEVICE, "ilu0: bad pointer kind");
        int64_t n = 0;
        ilu0_info(f, &n, nullptr, nullptr, nullptr);
        if (ptr_kind == KTB_PTR_DEVICE) {
            ilu0_apply(f, r, z, static_cast<cudaStream_t>(stream));
            return;
        }
        DBuf<double> dr(std::max<int64_t>(n, 1)), dz(std::max<int64_t>(n, 1));
        if (n) KTB_CUDA(cudaMemcpy(dr.p, r, 8 * n, cudaMemcpyHostToDevice));
        ilu0_apply(f, dr.p, dz.p, nullptr);  // legacy default stream, then synchronous
        KTB_CUDA(cudaStreamSynchronize(nullptr));
        if (n) KTB_CUDA(cudaMemcpy(z, dz.p, 8 * n, cudaMemcpyDeviceToHost));
    });
}

int ktb_ilu0_destroy(ktb_ilu* f) {
    return guarded([&] { ilu0_destroy(f); });
}

int64_t ktb_vec_mdot_scratch(int k) { return vec_mdot_scratch(k); }

int ktb_vec_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* out,
                 double* scratch, void* stream) {
    return guarded(
        [&] { vec_mdot(n, k, V, ldv, w, out, scratch, static_cast<cudaStream_t>(stream)); });
}

int ktb_vec_maxpy(int64_t n, int k, const double* V, int64_t ldv, const double* coef,
                  double alpha, double* w, void* stream) {
    return guarded(
        [&] { vec_maxpy(n, k, V, ldv, coef, alpha, w, static_cast<cudaStream_t>(stream)); });
}

int ktb_vec_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream) {
    return guarded([&] { vec_axpby(n, a, x, b, y, static_cast<cudaStream_t>(stream)); });
}

int ktb_vec_scale(int64_t n, double s, int divide, double* x, void* stream) {
    return guarded([&] { vec_scale(n, s, divide, x, static_cast<cudaStream_t>(stream)); });
}

int ktb_mm_probe(const char* path, int64_t* n, int64_t* entries, int* symmetric) {
    return guarded([&] {
        require(path != nullptr, "matrix market: null path");
        const MmHeader h = mm_probe(path);
        if (n) *n = h.n;
        if (entries) *entries = h.entries;
        if (symmetric) *symmetric = h.symmetric ? 1 : 0;
    });
}

int ktb_mm_read(const char* path, int want_symmetric, ktb_csr_host** out) {
    return guarded([&] {
        require(path != nullptr && out != nullptr, "matrix market: null path");
        *out = mm_read(path, want_symmetric != 0);
    });
}

int ktb_csr_host_info(const ktb_csr_host* h, int64_t* n, int64_t* nnz, int* kind) {
    return guarded([&] {
        require(h != nullptr, "matrix: null handle");
        if (n) *n = h->n;
        if (nnz) *nnz = static_cast<int64_t>(h->col.size());
        if (kind) *kind = h->kind;
    });
}

int ktb_csr_host_copy(const ktb_csr_host* h, int64_t* row_ptr, int64_t* col_idx,
                      double* values) {
    return guarded([&] {
        require(h != nullptr, "matrix: null handle");
        if (row_ptr) std::memcpy(row_ptr, h->row_ptr.data(), 8 * h->row_ptr.size());
        if (col_idx && !h->col.empty()) std::memcpy(col_idx, h->col.data(), 8 * h->col.size());
        if (values && !h->val.empty()) std::memcpy(values, h->val.data(), 8 * h->val.size());
    });
}

int ktb_csr_host_upload(const ktb_csr_host* h, int device, ktb_matrix** out) {
    return guarded([&] {
        require(h != nullptr, "matrix: null handle");
        *out = mm_upload(*h, device);
    });
}

int ktb_csr_host_destroy(ktb_csr_host* h) {
    return guarded([&] { delete h; });
}

int ktb_mm_write(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, int kind) {
    return guarded([&] {
        require(path != nullptr, "matrix market: null path");
        require(kind == KTB_GENERAL || kind == KTB_SYM_UPPER, "matrix: unknown kind");
        int64_t mr = 0, bw = 0;
        validate_host(n, row_ptr, col_idx, kind == KTB_SYM_UPPER, &mr, &bw);
        mm_write(path, n, row_ptr, col_idx, values, kind);
    });
}

int ktb_dist_create(int64_t n_global, int world, const int64_t* boundaries, int rank,
                    const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                    ktb_dist** out) {
    return guarded(
        [&] { *out = dist_create(n_global, world, boundaries, rank, row_ptr, col_idx, values); });
}

int ktb_dist_destroy(ktb_dist* d) {
    return guarded([&] {
        if (d) {
            if (d->device >= 0) {
                DeviceGuard g(d->device);
                delete d;
            } else {
                delete d;
            }
        }
    });
}

int ktb_dist_info(const ktb_dist* d, int64_t* n_local, int64_t* n_ghost, int64_t* nnz_local,
                  int64_t* nnz_ghost, int64_t* ghost_rows) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        if (n_local) *n_local = d->n_loc;
        if (n_ghost) *n_ghost = static_cast<int64_t>(d->ghosts.size());
        if (nnz_local) *nnz_local = static_cast<int64_t>(d->d_v.size());
        if (nnz_ghost) *nnz_ghost = static_cast<int64_t>(d->o_v.size());
        if (ghost_rows) *ghost_rows = static_cast<int64_t>(d->o_rows.size());
    });
}

int ktb_dist_ghosts(const ktb_dist* d, int64_t* ghost_cols, int64_t* recv_counts) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        if (ghost_cols) std::copy(d->ghosts.begin(), d->ghosts.end(), ghost_cols);
        if (recv_counts) std::copy(d->recv_counts.begin(), d->recv_counts.end(), recv_counts);
    });
}

int ktb_dist_set_sends(ktb_dist* d, const int64_t* send_counts, const int64_t* send_cols) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        dist_set_sends(d, send_counts, send_cols);
    });
}

int ktb_dist_local_csr(const ktb_dist* d, int32_t* row_ptr, int32_t* col_idx, double* values) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        if (row_ptr) std::copy(d->d_rp.begin(), d->d_rp.end(), row_ptr);
        if (col_idx) std::copy(d->d_ci.begin(), d->d_ci.end(), col_idx);
        if (values) std::copy(d->d_v.begin(), d->d_v.end(), values);
    });
}

int ktb_dist_ghost_csr(const ktb_dist* d, int32_t* rows, int32_t* row_ptr, int32_t* col_idx,
                       double* values) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        if (rows) std::copy(d->o_rows.begin(), d->o_rows.end(), rows);
        if (row_ptr) std::copy(d->o_rp.begin(), d->o_rp.end(), row_ptr);
        if (col_idx) std::copy(d->o_ci.begin(), d->o_ci.end(), col_idx);
        if (values) std::copy(d->o_v.begin(), d->o_v.end(), values);
    });
}

int ktb_dist_upload(ktb_dist* d, int device) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        dist_upload(d, device);
    });
}

int ktb_dist_local_matrix(ktb_dist* d, ktb_matrix** local) {
    return guarded([&] {
        require(d != nullptr && d->local != nullptr, "dist: not uploaded");
        *local = d->local;
    });
}

int ktb_dist_pack(const ktb_dist* d, const double* x_owned, double* send_buf, void* stream) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        dist_pack(d, x_owned, send_buf, static_cast<cudaStream_t>(stream));
    });
}

int ktb_dist_ghost_spmv(const ktb_dist* d, const double* x_ghost, double* y, void* stream) {
    return guarded([&] {
        require(d != nullptr, "dist: null handle");
        dist_ghost_spmv(d, x_ghost, y, static_cast<cudaStream_t>(stream));
    });
}

int ktb_gen_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, double off, double c_xm,
                     double c_xp, int device, ktb_matrix** out) {
    return guarded(
        [&] { *out = gen_stencil7(nx, ny, nz, 0, nz, false, diag, off, c_xm, c_xp, device); });
}

int ktb_gen_stencil27_upper(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                            int device, ktb_matrix** out) {
    return guarded([&] { *out = gen_stencil27_upper(nx, ny, nz, diag, off, device); });
}

int ktb_gen_stencil7_slab(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1,
                          double diag, double off, int device, ktb_matrix** out) {
    return guarded(
        [&] { *out = gen_stencil7(nx, ny, nz, z0, z1, true, diag, off, off, off, device); });
}

int ktb_gen_powerlaw(int64_t n, uint64_t seed, int64_t target_nnz, double empty_frac,
                     int64_t max_len, int device, ktb_matrix** out) {
    return guarded([&] { *out = gen_powerlaw(n, seed, target_nnz, empty_frac, max_len, device); });
}

int ktb_gen_powerlaw_host(int64_t n, uint64_t seed, int64_t target_nnz, double empty_frac,
                          int64_t max_len, int64_t* row_ptr, int32_t* col, double* val) {
    return guarded([&] {
        std::vector<int64_t> rp;
        std::vector<int32_t> c;
        std::vector<double> v;
        powerlaw_host(n, seed, target_nnz, empty_frac, max_len, rp, col ? &c : nullptr,
                      col ? &v : nullptr);
        std::copy(rp.begin(), rp.end(), row_ptr);
        if (col) {
            std::copy(c.begin(), c.end(), col);
            std::copy(v.begin(), v.end(), val);
        }
    });
}

int ktb_seeded_vector(int64_t n, uint64_t seed, int64_t offset, double* d_out, void* stream) {
    return guarded([&] {
        seeded_vector_dev(n, seed, offset, d_out, static_cast<cudaStream_t>(stream));
    });
}

int ktb_row_partition(const ktb_matrix* m, int num_workers, int scheme, int64_t* boundaries) {
    return guarded([&] {
        require(num_workers >= 1, "row partition: num_workers must be >= 1");
        require(scheme == KTB_ROW_BASED || scheme == KTB_NNZ_BALANCED,
                "row partition: bad scheme");
        DeviceGuard g(m->device);
        DBuf<int32_t> d(num_workers + 1);
        build_row_partition_dev(m, num_workers, scheme, d.p, 0);
        std::vector<int32_t> h(num_workers + 1);
        KTB_CUDA(cudaMemcpy(h.data(), d.p, 4 * (num_workers + 1), cudaMemcpyDeviceToHost));
        for (int p = 0; p <= num_workers; ++p) boundaries[p] = h[p];
    });
}

int ktb_row_partition_rowptr(const int64_t* row_ptr, int64_t n, int num_workers, int scheme,
                             int device, int64_t* boundaries) {
    return guarded([&] {
        require(num_workers >= 1, "row partition: num_workers must be >= 1");
        require(scheme == KTB_ROW_BASED || scheme == KTB_NNZ_BALANCED,
                "row partition: bad scheme");
        require(n >= 0 && row_ptr != nullptr, "csr: row_ptr length != n+1");
        build_row_partition_rowptr(row_ptr, n, num_workers, scheme, device, boundaries);
    });
}

int ktb_reduction_regions(const ktb_matrix* m, int num_workers, const int64_t* boundaries,
                          int64_t* lo, int64_t* hi) {
    return guarded([&] {
        require(m->kind == KTB_SYM_UPPER, "reduction regions: matrix is not symmetric storage");
        require(num_workers >= 1 && boundaries[num_workers] == m->n,
                "reduction regions: partition/matrix dimension mismatch");
        DeviceGuard g(m->device);
        std::vector<int32_t> b32(num_workers + 1);
        for (int p = 0; p <= num_workers; ++p) b32[p] = static_cast<int32_t>(boundaries[p]);
        DBuf<int32_t> db(num_workers + 1);
        DBuf<int64_t> dlo(num_workers), dhi(num_workers);
        KTB_CUDA(cudaMemcpy(db.p, b32.data(), 4 * (num_workers + 1), cudaMemcpyHostToDevice));
        reduction_regions_dev(m, num_workers, db.p, dlo.p, dhi.p, 0);
        KTB_CUDA(cudaMemcpy(lo, dlo.p, 8 * num_workers, cudaMemcpyDeviceToHost));
        KTB_CUDA(cudaMemcpy(hi, dhi.p, 8 * num_workers, cudaMemcpyDeviceToHost));
    });
}

int ktb_bss_plan_size(const ktb_matrix* m, int64_t jl, int64_t* jl_eff, int64_t* total_slices) {
    return guarded([&] {
        DeviceGuard g(m->device);
        bss_plan_size(m, jl, jl_eff, total_slices, 0);
    });
}

int ktb_bss_plan_copy(const ktb_matrix* m, int64_t jl, int64_t* slice_start, int64_t* slice_len,
                      int64_t* slice_row, int64_t* lane_slice_ptr, int64_t* row_slice_ptr,
                      uint8_t* row_start_flag) {
    return guarded([&] {
        DeviceGuard g(m->device);
        bss_plan_copy(m, jl, slice_start, slice_len, slice_row, lane_slice_ptr, row_slice_ptr,
                      row_start_flag, 0);
    });
}

int ktb_expand_symmetric(const ktb_matrix* m, ktb_matrix** out) {
    return guarded([&] { *out = expand_symmetric_dev(m, 0); });
}

int ktb_plan_create(ktb_matrix* m, int kernel, int64_t param, int workers, void* stream,
                    ktb_plan** out) {
    return guarded([&] {
        require(m != nullptr, "plan: null matrix");
        if (is_sym_kernel(kernel))
            require(m->kind == KTB_SYM_UPPER, "spmv: symmetric kernel on a general matrix");
        else
            require(is_unsym_kernel(kernel), "spmv: unknown kernel");
        if (is_unsym_kernel(kernel))
            require(m->kind == KTB_GENERAL, "spmv: unsymmetric kernel on symmetric storage");
        *out = plan_create_internal(m, kernel, param, workers, static_cast<cudaStream_t>(stream));
    });
}

int ktb_plan_destroy(ktb_plan* p) {
    return guarded([&] {
        if (p) {
            DeviceGuard g(p->m->device);
            delete p;
        }
    });
}

int ktb_plan_info(const ktb_plan* p, int* kernel, int64_t* param, int64_t* ctas,
                  int* launches_per_apply, int64_t* extra_bytes) {
    return guarded([&] {
        if (kernel) *kernel = p->kernel;
        if (param)
            *param = p->kernel == KTB_U3 || p->kernel == KTB_U4
                         ? p->jl
                         : p->param | (static_cast<int64_t>(p->cta_threads) << 16);
        if (ctas) *ctas = p->ctas;
        if (launches_per_apply) *launches_per_apply = p->launches;
        if (extra_bytes) *extra_bytes = p->extra_bytes;
    });
}

int ktb_plan_s3_info(const ktb_plan* p, int64_t* far_entries, int64_t* long_rows,
                     int64_t* patch_rows, int64_t* spill_doubles, int* window, int64_t* slots) {
    return guarded([&] {
        require(p != nullptr && p->kernel == KTB_S3, "plan: not an S3 plan");
        const auto& L = p->sw;
        if (far_entries) *far_entries = L.far;
        if (long_rows) *long_rows = L.nlong;
        if (patch_rows) *patch_rows = L.npatch;
        if (spill_doubles) *spill_doubles = L.spill_total;
        if (window) *window = L.window;
        if (slots) *slots = L.padded;
    });
}

int ktb_plan_set_stream(ktb_plan* p, void* stream) {
    return guarded([&] {
        if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
        p->own_stream = false;
        p->stream = static_cast<cudaStream_t>(stream);
    });
}

int ktb_spmv(ktb_plan* p, const double* x, double* y, int ptr_kind) {
    return guarded([&] {
        require(p != nullptr, "spmv: null plan");
        require(x != nullptr && y != nullptr, "spmv: dimension mismatch");
        const ktb_matrix* m = p->m;
        DeviceGuard g(m->device);
        if (ptr_kind == KTB_PTR_DEVICE) {
            plan_run(p, x, y, 0, m->n);
            return;
        }
        require(ptr_kind == KTB_PTR_HOST, "spmv: bad pointer kind");
        if (p->dx.n < static_cast<size_t>(m->ncols)) p->dx.alloc(std::max<int64_t>(m->ncols, 1));
        if (p->dy.n < static_cast<size_t>(m->n)) p->dy.alloc(std::max<int64_t>(m->n, 1));
        KTB_CUDA(cudaMemcpyAsync(p->dx.p, x, 8 * m->ncols, cudaMemcpyHostToDevice, p->stream));
        plan_run(p, p->dx.p, p->dy.p, 0, m->n);
        KTB_CUDA(cudaMemcpyAsync(y, p->dy.p, 8 * m->n, cudaMemcpyDeviceToHost, p->stream));
        KTB_CUDA(cudaStreamSynchronize(p->stream));
    });
}

int ktb_spmv_host_pipelined(ktb_plan* p, int64_t count, const double* x, int64_t ldx,
                            double* y, int64_t ldy) {
    return guarded([&] {
        require(p != nullptr, "spmv: null plan");
        require(x != nullptr && y != nullptr && count >= 0 && ldx >= 0 && ldy >= 0,
                "spmv: dimension mismatch");
        const ktb_matrix* m = p->m;
        DeviceGuard g(m->device);
        const int64_t nx = std::max<int64_t>(m->ncols, 1), ny = std::max<int64_t>(m->n, 1);
        if (p->dx.n < static_cast<size_t>(nx)) p->dx.alloc(nx);
        if (p->dy.n < static_cast<size_t>(ny)) p->dy.alloc(ny);
        if (p->dx2.n < static_cast<size_t>(nx)) p->dx2.alloc(nx);
        if (p->dy2.n < static_cast<size_t>(ny)) p->dy2.alloc(ny);
        if (!p->cin) {
            KTB_CUDA(cudaStreamCreateWithFlags(&p->cin, cudaStreamNonBlocking));
            KTB_CUDA(cudaStreamCreateWithFlags(&p->cout, cudaStreamNonBlocking));
            for (int b = 0; b < 2; ++b) {
                KTB_CUDA(cudaEventCreateWithFlags(&p->ev_in[b], cudaEventDisableTiming));
                KTB_CUDA(cudaEventCreateWithFlags(&p->ev_comp[b], cudaEventDisableTiming));
                KTB_CUDA(cudaEventCreateWithFlags(&p->ev_out[b], cudaEventDisableTiming));
            }
        }
        double* bx[2] = {p->dx.p, p->dx2.p};
        double* by[2] = {p->dy.p, p->dy2.p};
        // both copy streams start after whatever the plan's stream holds
        KTB_CUDA(cudaEventRecord(p->ev_comp[0], p->stream));
        KTB_CUDA(cudaStreamWaitEvent(p->cin, p->ev_comp[0], 0));
        KTB_CUDA(cudaStreamWaitEvent(p->cout, p->ev_comp[0], 0));
        for (int64_t k = 0; k < count; ++k) {
            const int b = static_cast<int>(k & 1);
            if (k >= 2) KTB_CUDA(cudaStreamWaitEvent(p->cin, p->ev_comp[b], 0));  // bx[b] free
            KTB_CUDA(cudaMemcpyAsync(bx[b], x + k * ldx, 8 * m->ncols, cudaMemcpyHostToDevice,
                                     p->cin));
            KTB_CUDA(cudaEventRecord(p->ev_in[b], p->cin));
            KTB_CUDA(cudaStreamWaitEvent(p->stream, p->ev_in[b], 0));
            if (k >= 2) KTB_CUDA(cudaStreamWaitEvent(p->stream, p->ev_out[b], 0));  // by[b] free
            plan_run(p, bx[b], by[b], 0, m->n);
            KTB_CUDA(cudaEventRecord(p->ev_comp[b], p->stream));
            KTB_CUDA(cudaStreamWaitEvent(p->cout, p->ev_comp[b], 0));
            KTB_CUDA(cudaMemcpyAsync(y + k * ldy, by[b], 8 * m->n, cudaMemcpyDeviceToHost,
                                     p->cout));
            KTB_CUDA(cudaEventRecord(p->ev_out[b], p->cout));
        }
        KTB_CUDA(cudaStreamSynchronize(p->cout));
        KTB_CUDA(cudaStreamSynchronize(p->stream));
    });
}

int ktb_spmv_rows(ktb_plan* p, int64_t row_begin, int64_t row_end, const double* x, double* y) {
    return guarded([&] {
        require(p->kernel == KTB_U1 && p->param != 101,
                "spmv_rows: row sub-ranges need the U1 plan");
        require(row_begin >= 0 && row_begin <= row_end && row_end <= p->m->n,
                "spmv_rows: bad row range");
        DeviceGuard g(p->m->device);
        u1_run(p, x, y, row_begin, row_end);
    });
}

int ktb_gmres(ktb_plan* A, const double* b, double* x, int64_t m, double tol, int64_t max_iters,
              double* history, ktb_gmres_result* res) {
    return guarded([&] { gmres_run(A, nullptr, b, x, m, tol, max_iters, history, res); });
}

int ktb_gmres_ilu0(ktb_plan* A, ktb_ilu* P, const double* b, double* x, int64_t m, double tol,
                   int64_t max_iters, double* history, ktb_gmres_result* res) {
    return guarded([&] {
        require(P != nullptr, "ilu0: null handle");
        gmres_run(A, P, b, x, m, tol, max_iters, history, res);
    });
}

int ktb_stream_sync(void* stream) {
    return guarded([&] { KTB_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
}

int ktb_host_alloc(size_t bytes, void** out) {
    return guarded([&] { KTB_CUDA(cudaMallocHost(out, bytes)); });
}
int ktb_host_free(void* p) {
    return guarded([&] { KTB_CUDA(cudaFreeHost(p)); });
}
int ktb_device_alloc(int device, size_t bytes, void** out) {
    return guarded([&] {
        DeviceGuard g(device);
        KTB_CUDA(cudaMalloc(out, bytes));
    });
}
int ktb_device_free(void* p) {
    return guarded([&] { KTB_CUDA(cudaFree(p)); });
}
int ktb_memcpy(void* dst, const void* src, size_t bytes, int kind, void* stream) {
    return guarded([&] {
        KTB_CUDA(cudaMemcpyAsync(dst, src, bytes, static_cast<cudaMemcpyKind>(kind),
                                 static_cast<cudaStream_t>(stream)));
    });
}

int ktb_time_spmv(ktb_plan* p, const double* x, double* y, int reps, size_t flush_bytes,
                  double* avg_ms, double* min_ms) {
    return guarded([&] {
        require(reps >= 1, "time: reps must be >= 1");
        DeviceGuard g(p->m->device);
        DBuf<uint8_t> flush;
        if (flush_bytes) flush.alloc(flush_bytes);
        std::vector<cudaEvent_t> ev(2 * reps);
        for (auto& e : ev) KTB_CUDA(cudaEventCreate(&e));
        for (int r = 0; r < reps; ++r) {
            if (flush_bytes)
                KTB_CUDA(cudaMemsetAsync(flush.p, r & 0xff, flush_bytes, p->stream));
            KTB_CUDA(cudaEventRecord(ev[2 * r], p->stream));
            plan_run(p, x, y, 0, p->m->n);
            KTB_CUDA(cudaEventRecord(ev[2 * r + 1], p->stream));
        }
        KTB_CUDA(cudaStreamSynchronize(p->stream));
        double tot = 0.0, mn = std::numeric_limits<double>::infinity();
        for (int r = 0; r < reps; ++r) {
            float ms = 0.f;
            KTB_CUDA(cudaEventElapsedTime(&ms, ev[2 * r], ev[2 * r + 1]));
            tot += ms;
            mn = std::min(mn, static_cast<double>(ms));
        }
        for (auto& e : ev) cudaEventDestroy(e);
        *avg_ms = tot / reps;
        if (min_ms) *min_ms = mn;
    });
}

// ---------------------------------------------------------------- selector
// autotune.hpp:216-259 (time_candidate / pick_winner) and :267-377.
int ktb_select(ktb_matrix* m, const ktb_select_opts* opts_in, void* stream, ktb_plan** winner,
               ktb_candidate* cands, int max_cands, int* n_cands, int* selected) {
    return guarded([&] {
        require(m != nullptr && m->n > 0 && m->nnz > 0, "kernel selection: empty matrix");
        DeviceGuard g(m->device);
        ktb_select_opts opts{};
        if (opts_in) opts = *opts_in;
        const int trials = opts.timed_trials > 0 ? std::min(opts.timed_trials, 8) : 3;
        // RAII for everything this call creates: a throw anywhere below
        // (CUDA error, bad_alloc) leaks no plan, event or stream
        struct StreamGuard {
            cudaStream_t s = nullptr;
            ~StreamGuard() {
                if (s) cudaStreamDestroy(s);
            }
        } own;
        struct EventGuard {
            cudaEvent_t e = nullptr;
            ~EventGuard() {
                if (e) cudaEventDestroy(e);
            }
        } e0, e1;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (!st) {
            KTB_CUDA(cudaStreamCreateWithFlags(&own.s, cudaStreamNonBlocking));
            st = own.s;
        }
        const int64_t n = m->n;
        DBuf<double> x(n), ref(n), y(n);
        probe_vector_dev(n, x.p, st);
        // the check: serial-order spmv_ref on the stored (GENERAL) or
        // expanded (SYM_UPPER, csr.hpp:88-123) matrix
        if (m->kind == KTB_SYM_UPPER) {
            {
                std::lock_guard<std::mutex> lk(m->lazy_mu);
                if (!m->expanded) m->expanded = expand_symmetric_dev(m, st);
            }
            check_spmv_ref_order(m->expanded, x.p, ref.p, st);
        } else {
            check_spmv_ref_order(m, x.p, ref.p, st);
        }
        struct Cand {
            int kernel;
            int64_t param;
            ktb_candidate rep;
        };
        std::vector<Cand> list;
        auto add = [&](int k, int64_t prm, const char* name, int ordinal, int threads = 0) {
            Cand c{k, prm | (static_cast<int64_t>(threads) << 16), {}};
            std::strncpy(c.rep.name, name, 7);
            c.rep.ordinal = ordinal;
            c.rep.param = prm;  // replaced by the plan's resolved value once set up
            c.rep.workers = opts.workers > 0 ? opts.workers : m->sm_count;
            c.rep.best_seconds = std::numeric_limits<double>::infinity();
            c.rep.cta_threads = threads;
            list.push_back(c);
        };
        // the reference's candidate set (autotune.hpp:283-313: U1, U2, U3 x
        // lane counts / S1, S2, S3) crossed with the GPU variants of each and
        // their launch shapes -- the GPU form of the worker-count sweep
        // (autotune.hpp:163, 206-212): CTA threads instead of OpenMP threads
        if (m->kind == KTB_SYM_UPPER) {
            add(KTB_S1, 0, "s1", 0);
            add(KTB_S1, 106, "s1", 0);  // transposed products gathered: expanded coded slices
            add(KTB_S2, 0, "s2", 1);
            for (int t : {256, 512}) add(KTB_S3, 0, "s3", 2, t);
        } else {
            add(KTB_U1, 0, "u1", 0);
            for (int t : {128, 64, 256}) add(KTB_U1, 100, "u1", 0, t);  // warp-sliced copy
            for (int t : {128, 64, 256}) add(KTB_U1, 102, "u1", 0, t);  // + coded columns
            add(KTB_U1, 106, "u1", 0);  // persistent slices, coded columns and values
            add(KTB_U1, 105, "u1", 0);  // persistent coded slices, bulk-copy staged
            add(KTB_U1, 104, "u1", 0);  // persistent pipelined slices, coded columns
            add(KTB_U1, 103, "u1", 0);  // the same with int32 columns
            for (int t : {128, 64, 256}) add(KTB_U1, 101, "u1", 0, t);  // rows sorted by length
            for (int t : {128, 256}) add(KTB_U2, 8, "u2", 1, t);         // warp tiles
            add(KTB_U2, 108, "u2", 1);                                   // merge-path tiles
            std::vector<int64_t> ept = {4, 8, 16};
            if (opts.params && opts.n_params > 0) ept.assign(opts.params, opts.params + opts.n_params);
            for (int64_t e : ept)
                if (m->nnz >= 4 * e) add(KTB_U3, e, "u3", 2);
            for (int t : {128, 256}) add(KTB_U3, 1008, "u3", 2, t);  // warp-level BSS tiles
        }
        KTB_CUDA(cudaEventCreate(&e0.e));
        KTB_CUDA(cudaEventCreate(&e1.e));
        // cold-L2 trials (default): the warm back-to-back timing of the
        // reference protocol ranks candidates by how they run with x, y and
        // part of the matrix left in the 126 MB L2 -- on config 2 it picked
        // S3's 512-thread shape (71.8 vs 73.7 us warm), 7 % slower cold
        DBuf<unsigned char> fl_w, fl_r;
        DBuf<double> fl_sink(1);
        if (!opts.warm_trials) {
            int l2 = 0;
            KTB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, m->device));
            const size_t fb = 2 * static_cast<size_t>(std::max(l2, 64 << 20));
            fl_w.alloc(fb);
            fl_r.alloc(fb);
            KTB_CUDA(cudaMemsetAsync(fl_r.p, 0, fb, st));
        }
        auto flush = [&] {
            if (opts.warm_trials) return;
            KTB_CUDA(cudaMemsetAsync(fl_w.p, 0x5a, fl_w.bytes(), st));
            flush_read(reinterpret_cast<const double*>(fl_r.p), fl_r.bytes() / 8, fl_sink.p, st);
        };
        // only the incumbent winner stays alive: candidates are timed one at
        // a time and a loser's device copy is released at once, so selection
        // holds at most two plans (pick_winner, autotune.hpp:242-259, applied
        // incrementally -- the same lexicographic (best, ordinal, param,
        // workers) order, earlier candidate kept on a full tie)
        std::unique_ptr<ktb_plan> best_plan;
        int best = -1;
        auto better = [&](const ktb_candidate& c, const ktb_candidate& b) {
            return std::make_tuple(c.best_seconds, c.ordinal, c.param, c.workers) <
                   std::make_tuple(b.best_seconds, b.ordinal, b.param, b.workers);
        };
        for (size_t ci = 0; ci < list.size(); ++ci) {
            auto& c = list[ci];
            std::unique_ptr<ktb_plan> p(new ktb_plan());
            const auto t_setup = std::chrono::steady_clock::now();
            try {
                p->m = m;
                p->kernel = c.kernel;
                p->param = c.param;
                p->workers = c.rep.workers;
                p->stream = st;
                plan_setup(p.get());
            } catch (const Invalid&) {
                c.rep.correct = 0;  // layout not applicable: reported as failing the check
                continue;
            }
            c.rep.setup_seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t_setup).count();
            c.rep.param = (c.kernel == KTB_U3) ? p->jl : p->param;
            // warm-up doubles as the correctness cross-check (autotune.hpp:226-229)
            plan_run(p.get(), x.p, y.p, 0, n);
            c.rep.executions = 1;
            c.rep.correct = outputs_match_dev(n, y.p, ref.p, st);
            if (!c.rep.correct) continue;
            for (int t = 0; t < trials; ++t) {
                double sec;
                flush();
                if (opts.now) {
                    KTB_CUDA(cudaStreamSynchronize(st));
                    const double tic = opts.now(opts.now_ctx);
                    plan_run(p.get(), x.p, y.p, 0, n);
                    KTB_CUDA(cudaStreamSynchronize(st));
                    sec = opts.now(opts.now_ctx) - tic;
                } else {
                    KTB_CUDA(cudaEventRecord(e0.e, st));
                    plan_run(p.get(), x.p, y.p, 0, n);
                    KTB_CUDA(cudaEventRecord(e1.e, st));
                    KTB_CUDA(cudaEventSynchronize(e1.e));
                    float ms = 0.f;
                    KTB_CUDA(cudaEventElapsedTime(&ms, e0.e, e1.e));
                    sec = ms * 1e-3;
                }
                ++c.rep.executions;
                c.rep.trial_seconds[c.rep.n_trials++] = sec;
                c.rep.best_seconds = std::min(c.rep.best_seconds, sec);
            }
            if (best < 0 || better(c.rep, list[best].rep)) {
                KTB_CUDA(cudaStreamSynchronize(st));
                best = static_cast<int>(ci);
                best_plan = std::move(p);  // the previous incumbent is released here
            }
        }
        if (n_cands) *n_cands = static_cast<int>(list.size());
        if (cands)
            for (int i = 0; i < static_cast<int>(list.size()) && i < max_cands; ++i)
                cands[i] = list[i].rep;
        if (best < 0) throw SelectError("kernel selection: every candidate failed the oracle check");
        if (selected) *selected = best;
        if (own.s) {  // hand the private stream to the winner
            best_plan->stream = own.s;
            best_plan->own_stream = true;
            own.s = nullptr;
        }
        *winner = best_plan.release();
    });
}

}  // extern "C"
