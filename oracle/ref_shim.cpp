// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers around the UNMODIFIED reference headers
// (/root/reference/proj/include/ktune/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libktune_ref.so. Nothing here re-implements an algorithm: every
// function forwards to the reference symbol it names. Used to (1) generate the
// golden fixtures in tests/golden/, (2) pin the C restatement in
// oracle/ktune_oracle.c bitwise, and (3) time the reference's own CPU path
// (bench.py --impl reference / cpu_baseline, kind "reference").
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <variant>
#include <vector>

#include "ktune/ktune.hpp"

using namespace ktune;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ktune::Error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

CsrMatrix make_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
    CsrMatrix a;
    a.n = n;
    a.row_ptr.assign(rp, rp + n + 1);
    a.col_idx.assign(ci, ci + rp[n]);
    a.values.assign(v, v + rp[n]);
    return a;
}

SymCsrMatrix make_sym(int64_t n, const int64_t* rp, const int64_t* ci, const double* v) {
    SymCsrMatrix a;
    a.n = n;
    a.row_ptr.assign(rp, rp + n + 1);
    a.col_idx.assign(ci, ci + rp[n]);
    a.values.assign(v, v + rp[n]);
    return a;
}

}  // namespace

extern "C" {

const char* kr_last_error() { return g_err.c_str(); }

int kr_max_threads() { return omp_get_max_threads(); }

// csr.hpp:38-54
int kr_validate(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int upper) {
    return guarded([&] {
        if (upper)
            make_sym(n, rp, ci, v).validate();
        else
            make_csr(n, rp, ci, v).validate();
    });
}

// csr.hpp:69-78
int kr_spmv_ref(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* x,
                double* y) {
    return guarded([&] {
        const auto a = make_csr(n, rp, ci, v);
        spmv_ref(a, std::span<const double>(x, n), std::span<double>(y, n));
    });
}

// csr.hpp:88-123 (caller sizes the outputs with the full nnz)
int kr_expand_symmetric(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                        int64_t nnz_full, int64_t* orp, int64_t* oci, double* ov) {
    return guarded([&] {
        const auto full = expand_symmetric(make_sym(n, rp, ci, v));
        require(full.nnz() == nnz_full, "shim: nnz_full mismatch");
        std::memcpy(orp, full.row_ptr.data(), sizeof(int64_t) * (n + 1));
        std::memcpy(oci, full.col_idx.data(), sizeof(int64_t) * nnz_full);
        std::memcpy(ov, full.values.data(), sizeof(double) * nnz_full);
    });
}

// partition.hpp:28-55
int kr_build_row_partition(int64_t n, const int64_t* rp, int workers, int scheme, int64_t* out) {
    return guarded([&] {
        const auto part = build_row_partition(std::span<const index_t>(rp, n + 1), workers,
                                              scheme ? PartitionScheme::nnz_balanced
                                                     : PartitionScheme::row_based);
        std::memcpy(out, part.boundaries.data(), sizeof(int64_t) * (workers + 1));
    });
}

// partition.hpp:73-96, on the partition built by partition.hpp:28 with `scheme`.
int kr_build_reduction_regions(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                               int workers, int scheme, int64_t* lo, int64_t* hi) {
    return guarded([&] {
        const auto a = make_sym(n, rp, ci, v);
        const auto part = build_row_partition(a.row_ptr, workers,
                                              scheme ? PartitionScheme::nnz_balanced
                                                     : PartitionScheme::row_based);
        const auto r = build_reduction_regions(a, part);
        std::memcpy(lo, r.lo.data(), sizeof(int64_t) * workers);
        std::memcpy(hi, r.hi.data(), sizeof(int64_t) * workers);
    });
}

// bss.hpp:34-69
struct kr_bss {
    BssPlan plan;
};

int kr_bss_create(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t jl,
                  kr_bss** out) {
    return guarded([&] {
        auto h = std::make_unique<kr_bss>();
        h->plan = build_bss_plan(make_csr(n, rp, ci, v), jl);
        *out = h.release();
    });
}

void kr_bss_info(const kr_bss* h, int64_t* jl, int64_t* total_slices) {
    *jl = h->plan.jl;
    *total_slices = h->plan.total_slices();
}

void kr_bss_copy(const kr_bss* h, int64_t* slice_start, int64_t* slice_len, int64_t* slice_row,
                 int64_t* lane_slice_ptr, int64_t* row_slice_ptr, uint8_t* row_start_flag) {
    const auto& p = h->plan;
    std::memcpy(slice_start, p.slice_start.data(), sizeof(int64_t) * p.slice_start.size());
    std::memcpy(slice_len, p.slice_len.data(), sizeof(int64_t) * p.slice_len.size());
    std::memcpy(slice_row, p.slice_row.data(), sizeof(int64_t) * p.slice_row.size());
    std::memcpy(lane_slice_ptr, p.lane_slice_ptr.data(), sizeof(int64_t) * p.lane_slice_ptr.size());
    std::memcpy(row_slice_ptr, p.row_slice_ptr.data(), sizeof(int64_t) * p.row_slice_ptr.size());
    std::memcpy(row_start_flag, p.row_start_flag.data(), p.row_start_flag.size());
}

void kr_bss_destroy(kr_bss* h) { delete h; }

// spmv.hpp:111-170 with the plans the reference builders produce for
// `workers` (U1/U2) or `jl` (U3/U4). kernel: 0=u1 1=u2 2=u3 3=u4.
int kr_spmv_unsym(int kernel, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  int workers, int64_t jl, const double* x, double* y) {
    return guarded([&] {
        const auto a = make_csr(n, rp, ci, v);
        WorkerPool pool(workers);
        const std::span<const double> xs(x, n);
        const std::span<double> ys(y, n);
        if (kernel <= 1) {
            const auto part = build_row_partition(a.row_ptr, workers,
                                                  kernel == 0 ? PartitionScheme::row_based
                                                              : PartitionScheme::nnz_balanced);
            spmv_unsym(kernel == 0 ? UnsymKernel::u1_row : UnsymKernel::u2_nnz, a, &part,
                       nullptr, xs, ys, pool);
        } else {
            const auto plan = build_bss_plan(a, jl);
            spmv_unsym(kernel == 2 ? UnsymKernel::u3_bss : UnsymKernel::u4_ss, a, nullptr, &plan,
                       xs, ys, pool);
        }
    });
}

// spmv.hpp:180-234. kernel: 0=s1 1=s2 2=s3.
int kr_spmv_sym(int kernel, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                int workers, const double* x, double* y) {
    return guarded([&] {
        const auto a = make_sym(n, rp, ci, v);
        WorkerPool pool(workers);
        const auto part = build_row_partition(a.row_ptr, workers,
                                              kernel == 0 ? PartitionScheme::row_based
                                                          : PartitionScheme::nnz_balanced);
        ReductionRegions regions;
        if (kernel == 2) regions = build_reduction_regions(a, part);
        spmv_sym(kernel == 0   ? SymKernel::s1_row
                 : kernel == 1 ? SymKernel::s2_nnz
                               : SymKernel::s3_nnz_zero_omit,
                 a, part, kernel == 2 ? &regions : nullptr, std::span<const double>(x, n),
                 std::span<double>(y, n), pool);
    });
}

// lanczos.hpp:17-29 and autotune.hpp:188-196
void kr_seeded_vector(int64_t n, uint64_t seed, double* out) {
    const auto v = detail::seeded_vector(n, seed);
    std::memcpy(out, v.data(), sizeof(double) * n);
}

void kr_probe_vector(int64_t n, double* out) {
    const auto v = detail::probe_vector(n);
    std::memcpy(out, v.data(), sizeof(double) * n);
}

// autotune.hpp:267-377 with an optional injected timer (autotune.hpp:164).
typedef double (*kr_now_fn)(void*);

struct kr_cand {
    char name[8];
    int ordinal;
    int64_t jl;
    int workers;
    int correct;
    int executions;
    int n_trials;
    double best_seconds;
    double trial_seconds[8];
};

static void export_report(const TuningReport& rep, kr_cand* out, int max_out, int* n_out,
                          int* selected) {
    *n_out = static_cast<int>(rep.candidates.size());
    *selected = rep.selected;
    for (int i = 0; i < *n_out && i < max_out; ++i) {
        const auto& c = rep.candidates[i];
        std::memset(&out[i], 0, sizeof(kr_cand));
        std::strncpy(out[i].name, c.name.c_str(), 7);
        out[i].ordinal = c.ordinal;
        out[i].jl = c.jl;
        out[i].workers = c.workers;
        out[i].correct = c.correct;
        out[i].executions = c.executions;
        out[i].n_trials = static_cast<int>(c.trial_seconds.size());
        out[i].best_seconds = c.best_seconds;
        for (int t = 0; t < out[i].n_trials && t < 8; ++t) out[i].trial_seconds[t] = c.trial_seconds[t];
    }
}

int kr_select(int sym, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
              int pool_size, int timed_trials, const int64_t* jl_cands, int n_jl, int sweep,
              kr_now_fn now, void* now_ctx, kr_cand* out, int max_out, int* n_out, int* selected) {
    return guarded([&] {
        WorkerPool pool(pool_size);
        SelectOptions opts;
        opts.timed_trials = timed_trials;
        opts.sweep_workers = sweep != 0;
        if (jl_cands) opts.jl_candidates.assign(jl_cands, jl_cands + n_jl);
        if (now) opts.now = [now, now_ctx]() { return now(now_ctx); };
        if (sym) {
            const auto a = make_sym(n, rp, ci, v);
            auto [choice, rep] = select_spmv_sym(a, pool, opts);
            export_report(rep, out, max_out, n_out, selected);
        } else {
            const auto a = make_csr(n, rp, ci, v);
            auto [choice, rep] = select_spmv_unsym(a, pool, opts);
            export_report(rep, out, max_out, n_out, selected);
        }
    });
}

// A tuned reference engine (meta.hpp:20-82): select once, then run the
// selected kernel through the engine's LinOp. Used by bench.py's reference arm.
struct kr_engine {
    bool sym = false;
    CsrMatrix a;
    SymCsrMatrix s;
    std::unique_ptr<UnsymEngine> ue;
    std::unique_ptr<SymEngine> se;
    LinOp op;
    TuningReport rep;
};

int kr_engine_create(int sym, int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                     int pool_size, kr_engine** out) {
    return guarded([&] {
        auto e = std::make_unique<kr_engine>();
        e->sym = sym != 0;
        WorkerPool pool(pool_size);
        if (e->sym) {
            e->s = make_sym(n, rp, ci, v);
            auto [choice, rep] = select_spmv_sym(e->s, pool);
            e->rep = rep;
            e->se = std::make_unique<SymEngine>(e->s, choice);
            e->op = e->se->op();
        } else {
            e->a = make_csr(n, rp, ci, v);
            auto [choice, rep] = select_spmv_unsym(e->a, pool);
            e->rep = rep;
            e->ue = std::make_unique<UnsymEngine>(e->a, choice);
            e->op = e->ue->op();
        }
        *out = e.release();
    });
}

// The same engine over the 3-D 7-point stencil (configs 1 and 4) built in
// place as a ktune::CsrMatrix by all threads: no host copy of a 16 GB int64
// CRS through Python (bench.py's full 512^3 reference arm). Input recipe
// index (z*ny + y)*nx + x, columns sorted -z,-y,-x,diag,+x,+y,+z.
int kr_engine_create_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                              int pool_size, kr_engine** out) {
    return guarded([&] {
        auto e = std::make_unique<kr_engine>();
        const int64_t n = nx * ny * nz, plane = nx * ny;
        CsrMatrix& a = e->a;
        a.n = n;
        a.row_ptr.assign(n + 1, 0);
        auto count = [&](int64_t i) {
            const int64_t z = i / plane, r = i % plane, y = r / nx, x = r % nx;
            return int64_t(1) + (z > 0) + (y > 0) + (x > 0) + (x < nx - 1) + (y < ny - 1) +
                   (z < nz - 1);
        };
        const int T = std::max(1, pool_size);  // OMP_NUM_THREADS may be 1 (torchrun)
        std::vector<int64_t> part(T + 1, 0);
#pragma omp parallel num_threads(T)
        {
            const int t = omp_get_thread_num();
            const int64_t lo = n * t / T, hi = n * (t + 1) / T;
            int64_t acc = 0;
            for (int64_t i = lo; i < hi; ++i) acc += count(i);
            part[t + 1] = acc;
#pragma omp barrier
#pragma omp single
            for (int k = 0; k < T; ++k) part[k + 1] += part[k];
            acc = part[t];
            for (int64_t i = lo; i < hi; ++i) {
                a.row_ptr[i] = acc;
                acc += count(i);
            }
        }
        a.row_ptr[n] = part[T];
        a.col_idx.resize(a.row_ptr[n]);
        a.values.resize(a.row_ptr[n]);
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t i = 0; i < n; ++i) {
            const int64_t z = i / plane, r = i % plane, y = r / nx, x = r % nx;
            int64_t k = a.row_ptr[i];
            auto put = [&](int64_t c, double val) {
                a.col_idx[k] = c;
                a.values[k++] = val;
            };
            if (z > 0) put(i - plane, off);
            if (y > 0) put(i - nx, off);
            if (x > 0) put(i - 1, off);
            put(i, diag);
            if (x < nx - 1) put(i + 1, off);
            if (y < ny - 1) put(i + nx, off);
            if (z < nz - 1) put(i + plane, off);
        }
        a.validate();
        WorkerPool pool(pool_size);
        auto [choice, rep] = select_spmv_unsym(e->a, pool);
        e->rep = rep;
        e->ue = std::make_unique<UnsymEngine>(e->a, choice);
        e->op = e->ue->op();
        *out = e.release();
    });
}

void kr_engine_report(const kr_engine* e, kr_cand* out, int max_out, int* n_out, int* selected) {
    export_report(e->rep, out, max_out, n_out, selected);
}

void kr_engine_selected(const kr_engine* e, char* name, int64_t* jl, int* workers,
                        double* best_seconds) {
    const auto& c = e->rep.selected_candidate();
    std::strncpy(name, c.name.c_str(), 7);
    name[7] = 0;
    *jl = c.jl;
    *workers = c.workers;
    *best_seconds = c.best_seconds;
}

int kr_engine_apply(kr_engine* e, const double* x, double* y) {
    return guarded([&] {
        e->op.apply(std::span<const double>(x, e->op.n), std::span<double>(y, e->op.n));
    });
}

void kr_engine_destroy(kr_engine* e) { delete e; }

// gmres.hpp:16-173 through make_ref_op (gmres.hpp:176-180) or a tuned U1 engine.
int kr_gmres(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, const double* b,
             int64_t m, double tol, int64_t max_iters, int ortho_kind, int engine_workers,
             double* x, double* history, int64_t* iterations, int64_t* restarts,
             int64_t* spmv_calls, int* converged, double* rec_res, double* true_res,
             double* seconds, double* spmv_seconds) {
    return guarded([&] {
        const auto a = make_csr(n, rp, ci, v);
        KrylovConfig cfg;
        cfg.restart_m = m;
        cfg.m_max = m;
        cfg.tol = tol;
        cfg.max_iters = max_iters;
        cfg.max_time = 1e30;
        cfg.ortho.kind = static_cast<OrthoKind>(ortho_kind);
        SolverResult r;
        int64_t calls = 0;
        double spmv_s = 0.0;
        if (engine_workers > 0) {
            UnsymChoice ch;
            ch.kernel = UnsymKernel::u1_row;
            ch.workers = engine_workers;
            ch.row_part = build_row_partition(a.row_ptr, engine_workers, PartitionScheme::row_based);
            ch.nnz_part = build_row_partition(a.row_ptr, engine_workers, PartitionScheme::nnz_balanced);
            UnsymEngine eng(a, ch);
            r = gmres_m(eng.op(), std::span<const double>(b, n), cfg);
            calls = eng.calls();
            spmv_s = eng.kernel_seconds();
        } else {
            const LinOp base = make_ref_op(a);
            LinOp counted{n, [&](std::span<const double> xx, std::span<double> yy) {
                              const double t0 = steady_seconds();
                              base.apply(xx, yy);
                              spmv_s += steady_seconds() - t0;
                              ++calls;
                          }};
            r = gmres_m(counted, std::span<const double>(b, n), cfg);
        }
        std::memcpy(x, r.x.data(), sizeof(double) * n);
        if (history)
            std::memcpy(history, r.residual_history.data(),
                        sizeof(double) * r.residual_history.size());
        *iterations = r.iterations;
        *restarts = static_cast<int64_t>(r.restarts.size());
        *spmv_calls = calls;
        *converged = r.converged ? 1 : 0;
        *rec_res = r.recurrence_residual;
        *true_res = r.true_residual;
        *seconds = r.elapsed_seconds;
        *spmv_seconds = spmv_s;
    });
}

// matrix_market.hpp:154-158
int kr_mm_probe(const char* path, int64_t* n, int64_t* entries, int* symmetric) {
    return guarded([&] {
        const MmInfo h = probe_matrix_market(path);
        *n = h.n;
        *entries = h.entries;
        *symmetric = h.symmetric ? 1 : 0;
    });
}

// matrix_market.hpp:165-194; the result is held in a CsrMatrix (kind 1 =
// the SymCsrMatrix alternative) until kr_mm_copy/kr_mm_destroy.
struct kr_mm {
    CsrMatrix a;
    int kind = 0;
};

int kr_mm_load(const char* path, int want_symmetric, kr_mm** out) {
    return guarded([&] {
        auto r = load_matrix_market(path, want_symmetric != 0);
        auto* h = new kr_mm();
        if (std::holds_alternative<SymCsrMatrix>(r)) {
            h->a = static_cast<CsrMatrix&&>(std::get<SymCsrMatrix>(std::move(r)));
            h->kind = 1;
        } else {
            h->a = std::get<CsrMatrix>(std::move(r));
        }
        *out = h;
    });
}

void kr_mm_info(const kr_mm* h, int64_t* n, int64_t* nnz, int* kind) {
    *n = h->a.n;
    *nnz = h->a.nnz();
    *kind = h->kind;
}

void kr_mm_copy(const kr_mm* h, int64_t* rp, int64_t* ci, double* v) {
    std::memcpy(rp, h->a.row_ptr.data(), sizeof(int64_t) * h->a.row_ptr.size());
    std::memcpy(ci, h->a.col_idx.data(), sizeof(int64_t) * h->a.col_idx.size());
    std::memcpy(v, h->a.values.data(), sizeof(double) * h->a.values.size());
}

void kr_mm_destroy(kr_mm* h) { delete h; }

// matrix_market.hpp:223-239
int kr_mm_write(const char* path, int64_t n, const int64_t* rp, const int64_t* ci,
                const double* v, int kind) {
    return guarded([&] {
        if (kind == 1)
            write_matrix_market(path, make_sym(n, rp, ci, v));
        else
            write_matrix_market(path, make_csr(n, rp, ci, v));
    });
}


// ilu0.hpp:23-69 (+ messages) and :73-87
int kr_ilu0_factorize(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                      double* values_out, int64_t* diag_out) {
    return guarded([&] {
        const auto f = ilu0_factorize(make_csr(n, rp, ci, v));
        std::memcpy(values_out, f.values.data(), sizeof(double) * f.values.size());
        std::memcpy(diag_out, f.diag_ptr.data(), sizeof(int64_t) * f.diag_ptr.size());
    });
}

int kr_ilu0_apply(int64_t n, const int64_t* rp, const int64_t* ci, const double* fv,
                  const int64_t* diag, const double* r, double* z) {
    return guarded([&] {
        IluFactors f;
        f.n = n;
        f.row_ptr.assign(rp, rp + n + 1);
        f.col_idx.assign(ci, ci + rp[n]);
        f.values.assign(fv, fv + rp[n]);
        f.diag_ptr.assign(diag, diag + n);
        ilu0_apply(f, std::span<const double>(r, n), std::span<double>(z, n));
    });
}


// gmres_m with the ILU(0) right preconditioner (gmres.hpp:16-173 with
// Precond{ilu0_apply}, as meta.hpp:195-201 wires it), sequential operator.
int kr_gmres_ilu0(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                  const double* b, int64_t m, double tol, int64_t max_iters, int ortho_kind,
                  double* x, int64_t* iterations, int64_t* restarts, int* converged,
                  double* true_res) {
    return guarded([&] {
        const auto a = make_csr(n, rp, ci, v);
        const IluFactors f = ilu0_factorize(a);
        Precond pc;
        pc.apply = [&f](std::span<const double> r, std::span<double> z) { ilu0_apply(f, r, z); };
        KrylovConfig cfg;
        cfg.restart_m = m;
        cfg.m_max = m;
        cfg.tol = tol;
        cfg.max_iters = max_iters;
        cfg.max_time = 1e30;
        cfg.ortho.kind = static_cast<OrthoKind>(ortho_kind);
        const SolverResult r = gmres_m(make_ref_op(a), std::span<const double>(b, n), cfg, pc);
        std::memcpy(x, r.x.data(), sizeof(double) * n);
        *iterations = r.iterations;
        *restarts = static_cast<int64_t>(r.restarts.size());
        *converged = r.converged ? 1 : 0;
        *true_res = r.true_residual;
    });
}

}  // extern "C"
