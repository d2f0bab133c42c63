// ktb_internal.cuh -- shared internals of libktb (not part of the ABI).
#pragma once

#include <functional>
#include <memory>
#include <mutex>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ktb.h"

namespace ktb {

// Contract violation (maps to KTB_ERR_INVALID; message = reference wording).
struct Invalid : std::runtime_error {
    explicit Invalid(const std::string& m) : std::runtime_error(m) {}
};
struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};
struct SelectError : std::runtime_error {
    explicit SelectError(const std::string& m) : std::runtime_error(m) {}
};

inline void require(bool cond, const char* msg) {
    if (!cond) throw Invalid(msg);
}

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        (void)cudaGetLastError();  // reported here: do not leak into a later launch check
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                        std::to_string(line) + ")");
    }
}
#define KTB_CUDA(x) ::ktb::cuda_check((x), #x, __FILE__, __LINE__)
#define KTB_LAUNCH() ::ktb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

constexpr int kNumSMs = 148;  // B200; queried at runtime, this is the default

// RAII device buffer.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) KTB_CUDA(cudaMalloc(&p, sizeof(T) * count));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        release();
        p = o.p;
        n = o.n;
        o.p = nullptr;
        o.n = 0;
        return *this;
    }
    size_t bytes() const { return sizeof(T) * n; }
};

// RAII pinned host buffer (async device->host copies).
template <typename T>
struct PinnedBuf {
    T* p = nullptr;
    explicit PinnedBuf(size_t count) {
        if (count) KTB_CUDA(cudaMallocHost(&p, sizeof(T) * count));
    }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) KTB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace ktb

// Device-resident CRS. int32 indices (nnz < 2^31), fp64 values.
struct ktb_matrix {
    int device = 0;
    int64_t n = 0, nnz = 0;
    int64_t ncols = 0;  // == n except for halo slabs (config 4 sharding)
    int64_t col_shift = 0;  // x index of row r's own entry is r + col_shift (halo slabs, slices)
    int kind = KTB_GENERAL;
    int64_t max_row_nnz = 0;
    int64_t bandwidth = 0;  // max(col - row) over stored entries (>= 0 for sym upper)
    int sm_count = ktb::kNumSMs;
    ktb::DBuf<int32_t> row_ptr;  // n+1
    ktb::DBuf<int32_t> col;      // nnz
    ktb::DBuf<double> val;       // nnz
    // Lazily built (under lazy_mu: plans of one matrix may be set up from
    // several host threads): expanded full matrix (sym) for the selector's
    // check and S1 106.
    ktb_matrix* expanded = nullptr;
    std::mutex lazy_mu;
    ~ktb_matrix();
};

// Host CRS as loaded from a Matrix Market file (reference index width).
struct ktb_csr_host {
    int64_t n = 0;
    int kind = KTB_GENERAL;
    std::vector<int64_t> row_ptr, col;
    std::vector<double> val;
};

namespace ktb {
void dist_comm_free(ktb_dist* d);  // ktb_comm.cu: the attached exchange state
}

// One rank's share of a row-block sharded CRS (ktb_dist.cu).
struct ktb_dist {
    int64_t n_global = 0, row0 = 0, n_loc = 0;
    int world = 1, rank = 0;
    std::vector<int64_t> bnd;
    // host split
    std::vector<int32_t> d_rp, d_ci, o_rows, o_rp, o_ci;
    std::vector<double> d_v, o_v;
    std::vector<int64_t> ghosts, recv_counts;
    std::vector<int32_t> send_idx;
    std::vector<int64_t> send_counts;
    bool sends_set = false;
    // device
    int device = -1;
    ktb_matrix* local = nullptr;  // A_d
    ktb::DBuf<int32_t> dev_orows, dev_orp, dev_oci, dev_send;
    ktb::DBuf<double> dev_ov;
    int lanes = 1;
    // ktb_dist_connect: communicator, ghost / send buffers, A_d plan, streams
    void* comm_state = nullptr;
    ~ktb_dist() {
        ktb::dist_comm_free(this);
        delete local;
    }
};

namespace ktb {

// ---- Matrix Market ingest (ktb_mm.cu) --------------------------------------
struct MmHeader {  // ktune::MmInfo (matrix_market.hpp:18-22)
    int64_t n = 0, entries = 0;
    bool symmetric = false;
};
MmHeader mm_probe(const std::string& path);
ktb_csr_host* mm_read(const std::string& path, bool want_symmetric);
ktb_matrix* mm_upload(const ktb_csr_host& h, int device);
void mm_write(const std::string& path, int64_t n, const int64_t* rp, const int64_t* ci,
              const double* v, int kind);

// ---- general row-block sharding (ktb_dist.cu) -----------------------------
ktb_dist* dist_create(int64_t n_global, int world, const int64_t* bnd, int rank,
                      const int64_t* rp, const int64_t* ci, const double* v);
void dist_set_sends(ktb_dist* d, const int64_t* counts, const int64_t* cols);
void dist_upload(ktb_dist* d, int device);
void dist_pack(const ktb_dist* d, const double* x_owned, double* send_buf, cudaStream_t s);
void dist_ghost_spmv(const ktb_dist* d, const double* x_ghost, double* y, cudaStream_t s);

// ---- ILU(0) (ktb_ilu.cu) ---------------------------------------------------
ktb_ilu* ilu0_create(const ktb_matrix* m, cudaStream_t user_stream);
void ilu0_apply(ktb_ilu* f, const double* r, double* z, cudaStream_t s);
void ilu0_info(const ktb_ilu* f, int64_t* n, int64_t* nl, int64_t* nu, int64_t* launches);
void ilu0_download(const ktb_ilu* f, int32_t* diag, double* val);
void ilu0_destroy(ktb_ilu* f);

// ---- device BLAS-1 of the distributed Krylov loop (ktb_vec.cu) -----------
int64_t vec_mdot_scratch(int k);
void vec_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* out,
              double* scratch, cudaStream_t s);
void vec_maxpy(int64_t n, int k, const double* V, int64_t ldv, const double* coef, double alpha,
               double* w, cudaStream_t s);
void vec_axpby(int64_t n, double a, const double* x, double b, double* y, cudaStream_t s);
void vec_scale(int64_t n, double sc, int divide, double* x, cudaStream_t s);

// ---- plans ---------------------------------------------------------------
struct MergeCoord {
    int32_t row;
    int32_t nz;
};

// S3 (zero-omission window) execution layout: see ktb_sym.cu.
struct SymWindowLayout {
    int ctas = 0;          // persistent CTAs = P of the NNZ_BALANCED partition
    int rows_per_sub = 0;  // rows per sub-tile (= threads per CTA)
    int window = 0;        // smem ring length in doubles
    int64_t padded = 0;    // total SELL slots (entries + padding)
    int64_t far = 0;       // entries scattered outside the window (atomic path)
    int64_t spill_total = 0;
    DBuf<int32_t> cta_row;     // ctas+1 (bit-exact NNZ_BALANCED boundaries)
    DBuf<int32_t> cta_chunk;   // ctas+1: round-chunk ranges per block
    DBuf<int32_t> chunk_meta;  // per chunk: sub-tile | last | round (padded, see k_s3)
    DBuf<int32_t> cta_qreal;   // per block: real chunk count
    DBuf<int64_t> cta_base;    // per block: SELL offset of its first chunk
    DBuf<unsigned char> sell;  // per round-chunk: fp64 values then int16 relative columns
    DBuf<double> diag;         // dense diagonal (0 for long rows: the long path adds it)
    DBuf<int32_t> spill_hi;    // per CTA: end of its spill range (start = cta_row[c+1])
    DBuf<int64_t> spill_off;   // per CTA: offset into spill
    DBuf<double> spill;
    DBuf<int32_t> segs;        // fixup block descriptors (3 int4 each, see s3_setup)
    DBuf<int32_t> seg_src;     // per fixup block: its spilling sources, ascending
    int64_t nsegs = 0;
    int reach = 0;             // max(col - row), clipped to the window
    int64_t nlong = 0;         // rows too long for the round layout
    // entries outside the window (far) and the long rows, as per-target
    // contribution lists: y[t] += sum_k v_k x[src_k] in a fixed order, one
    // warp per target row after the window pass (deterministic)
    int64_t npatch = 0;        // target rows
    DBuf<int32_t> patch_row, patch_rp, patch_src;
    DBuf<double> patch_val;
};

}  // namespace ktb

struct ktb_plan {
    ktb_matrix* m = nullptr;
    int kernel = KTB_U1;
    int64_t param = 0;
    int cta_threads = 0;  // launch shape (param bits 16..31); 0 = the kernel's default
    bool x_prefetch = true;  // U1 warp-sliced: pull each CTA's own x rows into L2 first
    int workers = 1;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int64_t ctas = 0;
    int launches = 1;
    int64_t extra_bytes = 0;
    // U2 merge-path tiles / U3 BSS lanes
    ktb::DBuf<ktb::MergeCoord> coords;  // U2 merge path: tiles+1 merge coordinates
    ktb::DBuf<int32_t> wrow;            // U2 warp tiles: first row of each tile (+ n)
    int64_t jl = 0;                     // U3: lane count (reference BssPlan jl)
    int64_t nq = 0;                     // U3: nonempty rows
    ktb::DBuf<uint32_t> flag_bits;      // U3: row_start_flag, 1 bit per nonzero
    ktb::DBuf<int32_t> seg_row;         // U3: q-th nonempty row (+ sentinel n)
    ktb::DBuf<int32_t> tile_q;          // U3: flags before each tile
    ktb::DBuf<int32_t> zero_rows;       // U3 warp tiles: empty rows + the last nonempty row
    int64_t nzero = 0;
    ktb::DBuf<double> carry_val;        // per tile carry-out
    ktb::DBuf<int32_t> carry_row;
    int64_t tiles = 0;
    // U1 param 100: warp-sliced (SELL-32) copy of the matrix, see ktb_unsym.cu
    ktb::DBuf<int64_t> sell_off;        // slices+1 element offsets (slice width = diff / 32)
    ktb::DBuf<int32_t> sell_col;        // -1 = padding
    ktb::DBuf<double> sell_val;
    int ell_width = 0;                  // > 0: every slice has this width (offsets implicit)
    // U1 param 102: column-delta dictionary (16 int32 per slice) and 4-bit codes
    ktb::DBuf<uint32_t> sell_codes;
    ktb::DBuf<int32_t> sell_dict;
    ktb::DBuf<unsigned char> sell_rec;  // U1 106: slice records (pair dictionary + code words)
    int rec_dict = 0, rec_words = 0, rec_bytes = 0, rec_stride = 0, rec_stages = 0;
    // U1 param 101: rows sorted by length into the slices (slot -> row), rows
    // longer than the slice cap in a compact sub-matrix run by U2 warp tiles
    ktb::DBuf<int32_t> sell_perm;
    ktb::DBuf<int32_t> long_rows;
    ktb::DBuf<double> long_y;
    ktb_matrix* long_m = nullptr;
    ktb_plan* long_plan = nullptr;
    cudaStream_t side = nullptr;        // the long rows run beside the slices
    cudaEvent_t fork = nullptr, join = nullptr;
    // S1/S2 row blocks
    ktb::DBuf<int32_t> blocks;          // P+1 row boundaries
    // S3
    ktb::SymWindowLayout sw;
    // host staging for KTB_PTR_HOST
    ktb::DBuf<double> dx, dy;
    // GMRES workspace reused across solves with this plan (ktb_gmres.cu)
    std::shared_ptr<void> gmres_ws;
    // ktb_spmv_host_pipelined: second buffer pair, copy streams, events
    ktb::DBuf<double> dx2, dy2;
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr},
                ev_out[2] = {nullptr, nullptr};
    ~ktb_plan();
};

namespace ktb {

// ---- internal entry points (implemented across the .cu files) -------------
void build_row_partition_dev(const ktb_matrix* m, int P, int scheme, int32_t* d_out,
                             cudaStream_t s);
void plan_setup(ktb_plan* p);
ktb_plan* plan_create_internal(ktb_matrix* m, int kernel, int64_t param, int workers,
                               cudaStream_t stream);
void plan_run(ktb_plan* p, const double* dx, double* dy, int64_t row_begin, int64_t row_end);
void check_spmv_ref_order(const ktb_matrix* m, const double* dx, double* dy, cudaStream_t s);
ktb_matrix* expand_symmetric_dev(const ktb_matrix* m, cudaStream_t s);
void probe_vector_dev(int64_t n, double* d_out, cudaStream_t s);
int outputs_match_dev(int64_t n, const double* dy, const double* dref, cudaStream_t s);
void compute_matrix_stats(ktb_matrix* m, cudaStream_t s);

// Runs f, mapping the exception types above to KTB_ERR_* and the thread's
// ktb_last_error() message (ktb_api.cu).
int guarded_call(const std::function<void()>& f);

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Opt a kernel into the device's full dynamic shared memory. The attribute is
// per function, not per plan: setting it to one plan's need lets a later plan
// with a smaller need lower it under an earlier plan's launches (seen as
// "invalid argument" with two U1 105 plans of different widths, and with
// ranks building plans concurrently). Every caller sets the same value, so
// the order and concurrency of plan setups no longer matter.
template <class F>
inline void allow_max_dynamic_smem(F fn) {
    int dev = 0, optin = 0;
    KTB_CUDA(cudaGetDevice(&dev));
    KTB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    KTB_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(fn)));
    KTB_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
}

}  // namespace ktb
