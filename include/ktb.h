/*
 * ktb.h -- C ABI of libktb, the B200-native (sm_100a) SpMV engine that drops
 * in under the reference's OpenATLib-style entry points (ktune).
 *
 * Plain C: opaque handles, plain pointers and sizes, int status codes
 * (0 = OK), thread-local ktb_last_error(). No torch or C++ types cross it.
 * Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj/include/ktune/).
 *
 * Threading (the reference: one caller thread per WorkerPool, spmv.hpp:37-40):
 * a matrix may be shared by plans set up and applied from several host
 * threads at once (its lazily built members are created under a lock); one
 * plan is used by one thread at a time (it owns scratch, staging buffers and
 * a stream, like a WorkerPool). tools/fuzz_threads.py exercises both.
 *
 * Index width: the reference's index_t is int64 (common.hpp:13); the host
 * side of this ABI takes int64 arrays unchanged and narrows to int32 on the
 * device, failing with KTB_ERR_INVALID if n or nnz >= 2^31.
 */
#ifndef KTB_H
#define KTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
#define KTB_OK 0
#define KTB_ERR_INVALID 1  /* contract violation: the ktune::Error cases (common.hpp:18-25) */
#define KTB_ERR_CUDA 2     /* CUDA runtime failure (no device, launch error, OOM) */
#define KTB_ERR_SELECT 3   /* every candidate failed the oracle check (autotune.hpp:257) */

/* Message of the last failing call on this thread; reference wording where
 * the reference has one (e.g. "spmv: dimension mismatch", spmv.hpp:115). */
const char* ktb_last_error(void);
int ktb_version(void);
int ktb_device_count(int* count);

/* ---------------------------------------------------------------- enums */
/* Kernel tags: ktune::UnsymKernel {u1_row,u2_nnz,u3_bss,u4_ss} and
 * ktune::SymKernel {s1_row,s2_nnz,s3_nnz_zero_omit} (spmv.hpp:15-16). */
enum {
    KTB_U1 = 0, /* row-parallel CRS: warp/vector-per-row          */
    KTB_U2 = 1, /* nnz-balanced: merge-path tiles                 */
    KTB_U3 = 2, /* branchless segmented scan (flag-driven)        */
    KTB_U4 = 3, /* original segmented scan (per-element branch)   */
    KTB_S1 = 16, /* symmetric, row-based, full-range reduction    */
    KTB_S2 = 17, /* symmetric, nnz-balanced, full-range reduction */
    KTB_S3 = 18  /* symmetric, nnz-balanced, zero-omission window */
};
enum { KTB_ROW_BASED = 0, KTB_NNZ_BALANCED = 1 }; /* ktune::PartitionScheme (partition.hpp:12) */
enum { KTB_GENERAL = 0, KTB_SYM_UPPER = 1 };      /* CsrMatrix / SymCsrMatrix (csr.hpp:13,59) */
enum { KTB_PTR_HOST = 0, KTB_PTR_DEVICE = 1 };

typedef struct ktb_matrix ktb_matrix;
typedef struct ktb_plan ktb_plan;

/* --------------------------------------------------------------- matrix */
/* Replaces CsrMatrix / SymCsrMatrix construction + validate()
 * (csr.hpp:13-65). Validates exactly like csr.hpp:38-54 (same messages),
 * uploads once to `device` and narrows indices to int32. */
int ktb_matrix_create(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                      const double* values, int kind, int device, ktb_matrix** out);
/* Same, from int32 HOST arrays (no narrowing step). */
int ktb_matrix_create_i32(int64_t n, const int32_t* row_ptr, const int32_t* col_idx,
                          const double* values, int kind, int device, ktb_matrix** out);
int ktb_matrix_destroy(ktb_matrix* m);
/* n, nnz, kind, max_row_nnz (csr.hpp:23-28), bandwidth = max(col - row). */
int ktb_matrix_info(const ktb_matrix* m, int64_t* n, int64_t* nnz, int* kind,
                    int64_t* max_row_nnz, int64_t* bandwidth);
/* Device copies of the stored arrays (int32 row_ptr/col, fp64 values) for
 * parity tests; any output may be NULL. Host destination pointers. */
int ktb_matrix_download(const ktb_matrix* m, int32_t* row_ptr, int32_t* col_idx, double* values);
/* Rows [row_begin, row_end) of a GENERAL device matrix as a new device matrix
 * over the same column space (row_ptr rebased; used to give the interior and
 * boundary rows of a halo slab their own plans). */
int ktb_matrix_slice(const ktb_matrix* m, int64_t row_begin, int64_t row_end, ktb_matrix** out);

/* ------------------------------------------------------- Matrix Market */
/* Coordinate real general/symmetric files (matrix_market.hpp). Same
 * accept/reject rules and messages as the reference; parsed in parallel. */
typedef struct ktb_csr_host ktb_csr_host; /* host CRS, int64 indices */
/* probe_matrix_market (matrix_market.hpp:154-158): header only. */
int ktb_mm_probe(const char* path, int64_t* n, int64_t* entries, int* symmetric);
/* load_matrix_market(path, want_symmetric) (matrix_market.hpp:165-194):
 * *kind = KTB_SYM_UPPER for the SymCsrMatrix alternative, else KTB_GENERAL. */
int ktb_mm_read(const char* path, int want_symmetric, ktb_csr_host** out);
int ktb_csr_host_info(const ktb_csr_host* h, int64_t* n, int64_t* nnz, int* kind);
/* Copies row_ptr (n+1), col_idx (nnz), values (nnz); NULL skips an array. */
int ktb_csr_host_copy(const ktb_csr_host* h, int64_t* row_ptr, int64_t* col_idx,
                      double* values);
/* Uploads as a device matrix (int32 indices): parallel narrowing through a
 * pinned staging ring; the CRS was already validated by ktb_mm_read. */
int ktb_csr_host_upload(const ktb_csr_host* h, int device, ktb_matrix** out);
int ktb_csr_host_destroy(ktb_csr_host* h);
/* write_matrix_market (matrix_market.hpp:223-239): KTB_GENERAL writes
 * "i j v"; KTB_SYM_UPPER writes the stored upper triangle transposed
 * (lower form, "symmetric" banner); values "%.17g". */
int ktb_mm_write(const char* path, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, int kind);

/* Generators (SURVEY.md §8d recipes), built directly on the device.
 * 3-D 7-point stencil on nx*ny*nz, x fastest, columns sorted
 * (-z,-y,-x,diag,+x,+y,+z); c_xm/c_xp are the -x/+x coefficients
 * (configs 1, 4, 5). */
int ktb_gen_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, double off, double c_xm,
                     double c_xp, int device, ktb_matrix** out);
/* 3-D 27-point stencil, diagonal + strict upper triangle (config 2). */
int ktb_gen_stencil27_upper(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                            int device, ktb_matrix** out);
/* Row-block slab of the 7-point stencil for z-planes [z0, z1) with a one-plane
 * halo: local columns index [halo_lo plane | owned planes | halo_hi plane]
 * (config 4 sharding). has_lo/has_hi are 0 on end ranks. */
int ktb_gen_stencil7_slab(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1,
                          double diag, double off, int device, ktb_matrix** out);
/* Irregular power-law matrix of config 3 (recipe in DESIGN.md, counter-based
 * splitmix64 streams: bit-identical for any thread count and in
 * tests/matgen.py): n rows, empty_frac empty rows, Pareto(1.5) row lengths
 * scaled to ~target_nnz, capped at max_len, distinct sorted uniform columns,
 * values U[-1,1). Built on the host with all cores, uploaded to `device`. */
int ktb_gen_powerlaw(int64_t n, uint64_t seed, int64_t target_nnz, double empty_frac,
                     int64_t max_len, int device, ktb_matrix** out);
/* Host-only form (no GPU needed). row_ptr has n+1 entries; when col/val are
 * NULL only row_ptr is produced (size query: nnz = row_ptr[n]). */
int ktb_gen_powerlaw_host(int64_t n, uint64_t seed, int64_t target_nnz, double empty_frac,
                          int64_t max_len, int64_t* row_ptr, int32_t* col, double* val);
/* lanczos.hpp:17-29 detail::seeded_vector (splitmix64 -> U[-1,1)), written
 * to a device buffer, element i = value of stream position offset+i. */
int ktb_seeded_vector(int64_t n, uint64_t seed, int64_t offset, double* d_out, void* stream);

/* ------------------------------------------------ plan artefacts (bit-exact) */
/* partition.hpp:28-55 build_row_partition, computed on the device.
 * boundaries: host, num_workers+1 entries. */
int ktb_row_partition(const ktb_matrix* m, int num_workers, int scheme, int64_t* boundaries);
/* The same from a HOST int64 row_ptr (n+1 entries) -- the reference's
 * build_row_partition(std::span<const index_t> row_ptr, P, scheme) form --
 * computed on `device`. */
int ktb_row_partition_rowptr(const int64_t* row_ptr, int64_t n, int num_workers, int scheme,
                             int device, int64_t* boundaries);
/* partition.hpp:73-96 build_reduction_regions for a SYM_UPPER matrix on the
 * given partition (host arrays, P = num_workers). */
int ktb_reduction_regions(const ktb_matrix* m, int num_workers, const int64_t* boundaries,
                          int64_t* lo, int64_t* hi);
/* bss.hpp:34-69 build_bss_plan on the device. Two calls: sizes first
 * (jl_eff = min(jl, nnz), total_slices), then the arrays (host, caller-sized;
 * any may be NULL). */
int ktb_bss_plan_size(const ktb_matrix* m, int64_t jl, int64_t* jl_eff, int64_t* total_slices);
int ktb_bss_plan_copy(const ktb_matrix* m, int64_t jl, int64_t* slice_start, int64_t* slice_len,
                      int64_t* slice_row, int64_t* lane_slice_ptr, int64_t* row_slice_ptr,
                      uint8_t* row_start_flag);
/* csr.hpp:88-123 expand_symmetric on the device; out is a new GENERAL matrix
 * with the reference's exact entry order. */
int ktb_expand_symmetric(const ktb_matrix* m, ktb_matrix** out);

/* -------------------------------------------------------------- plans */
/* An execution plan: kernel + its device-side decomposition + stream.
 * Replaces the (UnsymChoice|SymChoice) value (autotune.hpp:168-183).
 *   param:   U1: lanes per row V in {0=auto,1,2,4,...,32}; 100 = one thread
 *                per row over a warp-sliced (SELL-32/ELL) copy, bitwise equal
 *                to spmv_ref; 101 = the same over rows sorted by length (rows
 *                > 256 through U2 tiles on a side stream); 102 = the warp
 *                slices with each slice's columns coded as 4-bit indices into
 *                a <= 15-entry dictionary of column deltas (8.5 B per slot
 *                instead of 12); 103 / 104 = persistent, two-deep pipelined
 *                warp slices (uniform width <= 8) with int32 / coded columns;
 *                105 = persistent coded slices staged through per-warp
 *                bulk-copy (TMA) rings; 106 = persistent warps over pair-coded
 *                records (per 64 rows a dictionary of <= 63 distinct (column
 *                delta, fp64 bit pattern) pairs and one 8-bit code per slot,
 *                slice width <= 32: 10 B per 7-point row; refused otherwise)
 *                -- the halo operator's default, falling back to 105;
 *                100-106 are all bitwise equal to spmv_ref;
 *            U2: 0/4/8 = warp tiles of 32*IPT nonzeros (0 = 8);
 *                104/108/112 = merge-path tiles;
 *            U3/U4: nonzeros per segment lane E in {4,8,16} (0 = 8); U3 1008
 *                = flag-driven warp-level BSS over 256-nonzero tiles;
 *            S1/S2: lanes per row (0 = auto); S1 106 = the transposed products
 *                gathered from the expanded matrix's pair-coded records (U1
 *                106 over expand_symmetric(A); bitwise equal to
 *                spmv_ref(expand_symmetric(A)); refused like U1 106);
 *                S3: 0 (2048-row sub-tiles).
 *            The selector (ktb_select) sweeps these; see INTEGRATION.md.
 *            Bits 16..31 of param carry a launch shape (CTA threads; 0 =
 *            default): U1 100/101 take 64/128/256, U2 warp tiles and U3 1008
 *            take 128/256; the selector times each shape as a candidate.
 *   workers: the reference worker count P whose partition/regions the plan
 *            also materialises as artefacts (0 = engine default).
 *   stream:  cudaStream_t to run on (NULL = the plan creates its own). */
int ktb_plan_create(ktb_matrix* m, int kernel, int64_t param, int workers, void* stream,
                    ktb_plan** out);
int ktb_plan_destroy(ktb_plan* p);
/* kernel, param actually used, #CTAs of the main kernel, launches per apply,
 * extra device bytes read/written per apply beyond the minimum-traffic model. */
int ktb_plan_info(const ktb_plan* p, int* kernel, int64_t* param, int64_t* ctas,
                  int* launches_per_apply, int64_t* extra_bytes);
int ktb_plan_set_stream(ktb_plan* p, void* stream);
/* S3 layout facts: entries outside the shared-memory window (or on a
 * congested slot), rows too long for the round layout -- both applied by the
 * deterministic per-target patch pass (patch_rows targets) -- the spill
 * doubles merged by the fixup, the window length and the SELL slots. */
int ktb_plan_s3_info(const ktb_plan* p, int64_t* far_entries, int64_t* long_rows,
                     int64_t* patch_rows, int64_t* spill_doubles, int* window, int64_t* slots);

/* y = A*x. Replaces spmv_unsym (spmv.hpp:111-170) and spmv_sym
 * (spmv.hpp:180-234). ptr_kind KTB_PTR_DEVICE: x,y are device pointers, the
 * call is asynchronous on the plan's stream. KTB_PTR_HOST: x,y are host
 * pointers (pinned for full speed); the call copies x in, runs, copies y out
 * and synchronises (the LinOp::apply contract, solver_types.hpp:17-20). */
int ktb_spmv(ktb_plan* p, const double* x, double* y, int ptr_kind);
/* y_k = A*x_k for k < count, host vectors x + k*ldx, y + k*ldy (ldx/ldy in
 * doubles; 0 = the same vector every time, still copied every time): the
 * LinOp::apply contract of ktb_spmv(KTB_PTR_HOST) applied count times, with
 * the host->device copy of vector k+1 and the device->host copy of result
 * k-1 overlapping the SpMV of k (two device buffer pairs, copy-in / compute
 * / copy-out streams). Host memory should be pinned for the overlap.
 * Returns after the last result is in y. */
int ktb_spmv_host_pipelined(ktb_plan* p, int64_t count, const double* x, int64_t ldx,
                            double* y, int64_t ldy);
/* Same on a row sub-range [row_begin, row_end) of the plan's matrix (the
 * halo-overlap split of config 4). Only y[row_begin, row_end) is written. */
int ktb_spmv_rows(ktb_plan* p, int64_t row_begin, int64_t row_end, const double* x, double* y);

/* ------------------------------------------------------------ selector */
typedef double (*ktb_now_fn)(void* ctx);

typedef struct {
    const int64_t* params; /* per-kernel parameter sweep for U3 (NULL = default) */
    int n_params;
    int timed_trials;      /* default 3 (autotune.hpp:162) */
    int workers;           /* reference worker count for artefacts (0 = default) */
    ktb_now_fn now;        /* injected host timer (autotune.hpp:164); NULL = CUDA events */
    void* now_ctx;
    int warm_trials;       /* 0 (default): before every timed trial L2 is flushed (2x its
                              size written, then another 2x read), so each candidate is timed
                              the way it runs on a matrix streamed from HBM; 1: back to back
                              with a warm L2, the reference's protocol (autotune.hpp:216-240) */
} ktb_select_opts;

typedef struct {
    char name[8];          /* "u1".."u3", "s1".."s3" */
    int ordinal;           /* first tie-break key (autotune.hpp:248-259) */
    int64_t param;         /* second key (jl analogue) */
    int workers;
    int correct;           /* warm-up output matched the check (autotune.hpp:226-229) */
    int executions;        /* warm-up + timed runs, <= 4 */
    int n_trials;
    double best_seconds;
    double trial_seconds[8];
    int cta_threads;       /* launch shape (CTA threads; 0 = the kernel's default) */
    double setup_seconds;  /* plan build (host + device) before the warm-up */
} ktb_candidate;

/* select_spmv_unsym / select_spmv_sym (autotune.hpp:267-377) on device
 * time: probe_vector x (autotune.hpp:188-196), a serial-order device check
 * (spmv_ref order, bitwise equal to csr.hpp:69-78; for symmetric storage on
 * the device expand_symmetric), one warm-up = correctness check with
 * outputs_match tolerance, timed trials, min, lexicographic tie-break
 * (best, ordinal, param, workers). Returns the winning plan (caller
 * destroys) and the report. */
int ktb_select(ktb_matrix* m, const ktb_select_opts* opts, void* stream, ktb_plan** winner,
               ktb_candidate* cands, int max_cands, int* n_cands, int* selected);

/* ---------------------------------------------------------- consumer */
typedef struct {
    int64_t iterations;  /* Arnoldi steps (gmres.hpp:119) */
    int64_t restarts;
    int64_t spmv_calls;
    int converged;
    int breakdown;
    int fault_convergence;  /* recurrence met tol, true residual did not (gmres.hpp:169) */
    double recurrence_residual;
    double true_residual;
    double seconds;         /* wall time of the solve */
    double spmv_seconds;    /* device time inside the SpMV applies (CUDA events) */
} ktb_gmres_result;

/* gmres_m (gmres.hpp:16-173): restarted GMRES(m) with modified Gram-Schmidt
 * (ortho.hpp:88-94), x0 = 0, no preconditioner, stop at relative recurrence
 * residual < tol or max_iters; true residual recomputed at exit. All vectors
 * device-resident; A is any GENERAL-matrix plan. b, x, history: HOST arrays
 * (history: max_iters doubles or NULL). */
int ktb_gmres(ktb_plan* A, const double* b, double* x, int64_t m, double tol, int64_t max_iters,
              double* history, ktb_gmres_result* res);

/* ------------------------------------------- general row-block sharding */
/* SURVEY.md §8f row 3 (no reference counterpart: the reference is single
 * process). Rank `rank` of `world` owns rows and x entries
 * [boundaries[rank], boundaries[rank+1]) of an n_global-row CRS; row_ptr /
 * col_idx / values are ITS rows (local row_ptr, GLOBAL column ids). The
 * rows split into A_d (owned columns, square, a regular ktb_matrix: any
 * kernel, any plan, the selector) and A_o (rows touching other ranks'
 * columns, over the ghost index space). Ghost columns are sorted ascending,
 * so they arrive grouped by owner rank: one receive buffer = the ghost
 * vector. create/info/ghosts/set_sends are host-only (no device calls). */
typedef struct ktb_dist ktb_dist;
int ktb_dist_create(int64_t n_global, int world, const int64_t* boundaries, int rank,
                    const int64_t* row_ptr, const int64_t* col_idx, const double* values,
                    ktb_dist** out);
int ktb_dist_destroy(ktb_dist* d);
/* n_local rows; n_ghost columns; stored entries of A_d / A_o; rows of A_o. */
int ktb_dist_info(const ktb_dist* d, int64_t* n_local, int64_t* n_ghost, int64_t* nnz_local,
                  int64_t* nnz_ghost, int64_t* ghost_rows);
/* Ghost column ids (global, ascending; n_ghost) and per-owner counts (world). */
int ktb_dist_ghosts(const ktb_dist* d, int64_t* ghost_cols, int64_t* recv_counts);
/* What this rank sends: per-peer counts (world) and the owned global column
 * ids concatenated in peer order (each peer's ghost list for this rank). */
int ktb_dist_set_sends(ktb_dist* d, const int64_t* send_counts, const int64_t* send_cols);
/* Host copies of the split (CPU tests): A_d as CRS (n_local+1, nnz_local);
 * A_o as (row ids, row_ptr ghost_rows+1, ghost-space columns, values). */
int ktb_dist_local_csr(const ktb_dist* d, int32_t* row_ptr, int32_t* col_idx, double* values);
int ktb_dist_ghost_csr(const ktb_dist* d, int32_t* rows, int32_t* row_ptr, int32_t* col_idx,
                       double* values);
/* Upload both blocks to `device`; the A_d handle stays owned by d. */
int ktb_dist_upload(ktb_dist* d, int device);
int ktb_dist_local_matrix(ktb_dist* d, ktb_matrix** local);
/* send_buf[k] = x_owned[send_idx[k]] (device pointers). */
int ktb_dist_pack(const ktb_dist* d, const double* x_owned, double* send_buf, void* stream);
/* y += A_o x_ghost (device pointers); run after A_d x_owned -> y. */
int ktb_dist_ghost_spmv(const ktb_dist* d, const double* x_ghost, double* y, void* stream);

/* ------------------------------------------ communicator (native NCCL) */
/* The multi-GPU data plane: one process per GPU, one
 * communicator per process. No reference counterpart (the reference is a
 * single-process OpenMP library). */
typedef struct ktb_comm ktb_comm;
typedef struct ktb_loopback_world ktb_loopback_world;
#define KTB_COMM_ID_BYTES 128 /* sizeof(ncclUniqueId) */
enum { KTB_SUM = 0, KTB_MAX = 1 };
/* ncclGetUniqueId: rank 0 calls it and hands the bytes to every rank out of
 * band (MPI, a TCP store, torch.distributed.broadcast_object_list). */
int ktb_comm_id(uint8_t* id /* KTB_COMM_ID_BYTES */);
/* ncclCommInitRank on `device` (collective over the world). */
int ktb_comm_create(const uint8_t* id, int world, int rank, int device, ktb_comm** out);
/* Borrow a caller's ncclComm_t (e.g. torch's ProcessGroupNCCL::_comm_ptr());
 * it is not destroyed by ktb_comm_destroy. device < 0: take the comm's. */
int ktb_comm_wrap(void* nccl_comm, int device, ktb_comm** out);
/* Test transport: `world` ranks inside ONE process, each rank driven by its
 * own host thread; messages are matched on the host and moved by device
 * copies (no kernel ever waits on another rank). Same semantics as NCCL's
 * grouped send/recv, all-reduce and all-gather, host-synchronous. */
int ktb_loopback_world_create(int world, ktb_loopback_world** out);
int ktb_loopback_world_destroy(ktb_loopback_world* w);
int ktb_comm_create_loopback(ktb_loopback_world* w, int rank, int device, ktb_comm** out);
int ktb_comm_info(const ktb_comm* c, int* world, int* rank, int* device, int* nccl_version,
                  int* is_nccl);
int ktb_comm_destroy(ktb_comm* c);
/* In place over device doubles (KTB_SUM / KTB_MAX), enqueued on stream. */
int ktb_comm_allreduce(ktb_comm* c, double* buf, int64_t count, int op, void* stream);
/* recv[r*bytes, (r+1)*bytes) = rank r's `send` (device buffers). */
int ktb_comm_allgather(ktb_comm* c, const void* send, void* recv, size_t bytes, void* stream);
/* One grouped send + receive (peer < 0 or 0 bytes skips that half). */
int ktb_comm_sendrecv(ktb_comm* c, const void* send, size_t send_bytes, int send_peer, void* recv,
                      size_t recv_bytes, int recv_peer, void* stream);

/* ------------------------------------- halo row-block operator (config 4) */
/* spmv_unsym (spmv.hpp:111-126) over a row block with a banded halo: `local`
 * holds this rank's n rows with LOCAL columns over [halo_lo | owned n |
 * halo_hi] (ncols = halo_lo + n + halo_hi); rank r-1 owns the rows just
 * below, r+1 just above. Collective: the ranks exchange their shapes, so
 * each learns how many owned entries its neighbours read. The rows split into
 * the interior (no halo column) and the boundary rows, each a row slice with
 * its own plan (kernel/param as ktb_plan_create; the matrix may be destroyed
 * after this call). */
typedef struct ktb_halo ktb_halo;
int ktb_halo_create(ktb_matrix* local, int64_t halo_lo, int64_t halo_hi, ktb_comm* comm,
                    int kernel, int64_t param, ktb_halo** out);
/* Config 4's shard: z-planes [r*nz/W, (r+1)*nz/W) of the 3-D 7-point stencil
 * with one-plane halos, generated on the communicator's device. */
int ktb_halo_create_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                             ktb_comm* comm, int kernel, int64_t param, ktb_halo** out);
/* The same from this rank's rows in the caller's global numbering (rows
 * [row0, row0+n_local) of an n_global-row matrix, int64 row_ptr local, GLOBAL
 * columns): the halos are the column ranges below row0 and above the block
 * (a banded row block; columns in between are read from the owned x). */
int ktb_halo_create_csr(int64_t n_global, int64_t row0, int64_t n_local, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, ktb_comm* comm, int kernel,
                        int64_t param, ktb_halo** out);
int ktb_halo_info(const ktb_halo* h, int64_t* n_local, int64_t* x_len, int64_t* owned_offset,
                  int64_t* interior_begin, int64_t* interior_end, int64_t* nnz, int* launches);
/* Rows and stored entries of the interior and boundary parts. */
/* The U1 variant (plan param) the interior / first boundary rows resolved to
 * after the create call's fallbacks (106 -> 105 -> 104 -> 100); -1 = no rows. */
int ktb_halo_plan_params(const ktb_halo* h, int64_t* interior_param, int64_t* boundary_param);
int ktb_halo_parts(const ktb_halo* h, int64_t* interior_rows, int64_t* interior_nnz,
                   int64_t* boundary_rows, int64_t* boundary_nnz);
/* y = A x (device pointers, asynchronous on stream). x has x_len entries with
 * the owned ones at owned_offset; the halo entries are written by the
 * exchange: one NCCL group (send owned edges, receive halos in place) on a
 * high-priority communication stream, overlapped with the interior rows on
 * `stream`; the boundary rows follow an event wait. */
int ktb_halo_spmv(ktb_halo* h, double* x, double* y, void* stream);
/* The exchange alone (stream waits for it). */
int ktb_halo_exchange(ktb_halo* h, double* x, void* stream);
/* y = A x from HOST memory (LinOp::apply contract, solver_types.hpp:17-20):
 * x_owned (n_local, pinned for overlap) in, y (n_local) out, synchronous.
 * The copies overlap inside the call: x goes host->device in `chunks` row
 * chunks, each interior row chunk runs once the x chunks its columns reach
 * have landed, and its y rows go device->host while later chunks compute;
 * the halo exchange follows the last x chunk, the boundary rows run last. */
int ktb_halo_spmv_host(ktb_halo* h, const double* x_owned, double* y, int chunks);
/* Per-apply kernel timing (CUDA events on the apply's stream): after
 * ktb_halo_set_timing(h, 1), ktb_halo_timing returns the device time of the
 * last apply's interior rows and boundary rows (waits for them). */
int ktb_halo_set_timing(ktb_halo* h, int on);
int ktb_halo_timing(ktb_halo* h, double* interior_ms, double* boundary_ms);
int ktb_halo_destroy(ktb_halo* h);

/* ------------------------------- general split over a communicator */
/* Attach a ktb_dist split to a communicator (collective): uploads to the
 * comm's device, exchanges the ghost lists (all-gather of counts, grouped
 * send/recv of the lists; replaces ktb_dist_set_sends) and builds the A_d
 * plan (kernel/param; U1 param 100 falls back to U2 tiles when the
 * warp-sliced copy is refused). */
int ktb_dist_connect(ktb_dist* d, ktb_comm* comm, int kernel, int64_t param);
/* Use a caller-owned plan for A_d (built on ktb_dist_local_matrix, e.g. by
 * ktb_select); NULL restores zero-fill for an empty A_d. */
int ktb_dist_set_plan(ktb_dist* d, ktb_plan* plan);
/* y = A x over the row block (device pointers, asynchronous on stream):
 * pack -> NCCL ghost exchange on the communication stream, overlapped with
 * A_d x_owned -> y on `stream` -> y += A_o x_ghost after an event wait. */
int ktb_dist_spmv(ktb_dist* d, const double* x_owned, double* y, void* stream);
/* Pack + ghost exchange alone (stream waits for it). */
int ktb_dist_exchange(ktb_dist* d, const double* x_owned, void* stream);
int ktb_dist_launches(const ktb_dist* d, int* launches);
/* The send lists in force (after ktb_dist_connect or ktb_dist_set_sends):
 * per-peer counts (world) and the owned GLOBAL column ids in peer order. */
int ktb_dist_sends(const ktb_dist* d, int64_t* send_counts, int64_t* send_cols);

/* ------------------------------- distributed Krylov building blocks */
/* Device BLAS-1 for GMRES over row-sharded vectors (dot / axpy / scal of
 * common.hpp:33-56 and the passes of ortho.hpp:55-111); the caller
 * all-reduces the local partial dots (NCCL). Deterministic reductions.
 * V: column-major basis, column j at V + j*ldv. All pointers device. */
/* scratch doubles needed by ktb_vec_mdot for k columns */
int64_t ktb_vec_mdot_scratch(int k);
/* out[j] = <V_j, w>, j < k (local partial dot products) */
int ktb_vec_mdot(int64_t n, int k, const double* V, int64_t ldv, const double* w, double* out,
                 double* scratch, void* stream);
/* w += alpha * coef[j] * V_j for j = 0..k-1 in order (k axpy calls fused) */
int ktb_vec_maxpy(int64_t n, int k, const double* V, int64_t ldv, const double* coef,
                  double alpha, double* w, void* stream);
/* y = a*x + b*y */
int ktb_vec_axpby(int64_t n, double a, const double* x, double b, double* y, void* stream);
/* x[i] *= s (divide = 0, scal) or x[i] /= s (divide = 1) */
int ktb_vec_scale(int64_t n, double s, int divide, double* x, void* stream);

/* -------------------------------------------------------------- ILU(0) */
typedef struct ktb_ilu ktb_ilu;
/* gmres_m with ILU(0) right preconditioning (gmres.hpp:16-173 with
 * Precond{ilu0_apply}, the pairing meta.hpp:195-201 makes): each Arnoldi
 * step applies z = M^{-1} v_j before the SpMV, the correction is
 * x += M^{-1}(Q y). Same arguments as ktb_gmres plus the factors. */
int ktb_gmres_ilu0(ktb_plan* A, ktb_ilu* P, const double* b, double* x, int64_t m, double tol,
                   int64_t max_iters, double* history, ktb_gmres_result* res);
/* ilu0.hpp: incomplete LU on the pattern of a GENERAL matrix (unit L, U on
 * the stored pattern). Factors and solves are bitwise equal to the
 * reference's (level-scheduled rows, reference operation order, no FMA). */
/* ilu0_factorize (ilu0.hpp:23-69); same messages ("ilu0: structurally
 * missing diagonal in row i", "ilu0: zero pivot at row i"). stream may be
 * NULL. */
int ktb_ilu0_create(const ktb_matrix* m, void* stream, ktb_ilu** out);
/* n, dependency levels of the lower / upper sweeps, kernel launches per apply */
int ktb_ilu0_info(const ktb_ilu* f, int64_t* n, int64_t* lower_levels, int64_t* upper_levels,
                  int64_t* launches_per_apply);
/* IluFactors::diag_ptr (n) and ::values (nnz) to host; either may be NULL */
int ktb_ilu0_download(const ktb_ilu* f, int32_t* diag_ptr, double* values);
/* ilu0_apply (ilu0.hpp:73-87): z = (LU)^{-1} r. ptr_kind KTB_PTR_DEVICE: device
 * pointers, enqueued on `stream` (NULL = the legacy default stream);
 * KTB_PTR_HOST: host arrays, synchronous. Applies of one factor on different
 * streams are serialised (they share the factor's solve buffers). */
int ktb_ilu0_apply(ktb_ilu* f, const double* r, double* z, int ptr_kind, void* stream);
int ktb_ilu0_destroy(ktb_ilu* f);

/* ---------------------------------------------------------- host memory */
int ktb_host_alloc(size_t bytes, void** out);  /* pinned */
int ktb_host_free(void* p);
int ktb_device_alloc(int device, size_t bytes, void** out);
int ktb_device_free(void* p);
int ktb_memcpy(void* dst, const void* src, size_t bytes, int kind /*cudaMemcpyKind*/, void* stream);
int ktb_stream_sync(void* stream);

/* ---------------------------------------------------------- timing */
/* Average device time in ms of `reps` back-to-back applies on the plan's
 * stream, measured with CUDA events on that stream; when flush_bytes > 0 an
 * L2-flushing write of that size runs before each apply and is excluded by
 * per-apply event pairs. x,y device pointers. */
int ktb_time_spmv(ktb_plan* p, const double* x, double* y, int reps, size_t flush_bytes,
                  double* avg_ms, double* min_ms);

#ifdef __cplusplus
}
#endif

#endif /* KTB_H */
