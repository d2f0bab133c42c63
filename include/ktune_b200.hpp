// ktune_b200.hpp -- C++ drop-in shim over the libktb C ABI (ktb.h).
//
// Re-exposes the reference's SpMV operator interface (namespace ktune,
// /root/reference/proj/include/ktune/) on the B200 engine:
//
//   reference (file:line)                         here
//   spmv_unsym(kernel, A, part, plan, x, y, pool) ktb_cpp::spmv_unsym(kernel, A, x, y)
//     (spmv.hpp:111-170)
//   spmv_sym(kernel, A, part, regions, x, y, pool) ktb_cpp::spmv_sym(kernel, A, x, y)
//     (spmv.hpp:180-234)
//   select_spmv_unsym / select_spmv_sym           ktb_cpp::select_spmv_unsym / _sym
//     (autotune.hpp:267-377)                        -> {Choice, TuningReport}
//   UnsymEngine / SymEngine (meta.hpp:20-82)      ktb_cpp::UnsymEngine / SymEngine
//   LinOp (solver_types.hpp:17-20)                ktb_cpp::LinOp (same two members)
//   build_row_partition (partition.hpp:28-55)     ktb_cpp::build_row_partition
//   build_reduction_regions (partition.hpp:73-96) ktb_cpp::build_reduction_regions
//   build_bss_plan (bss.hpp:34-69)                ktb_cpp::bss_plan_arrays
//   ktune::Error (common.hpp:18-21)               ktb_cpp::Error (same messages)
//   ilu0_factorize / ilu0_apply (ilu0.hpp)        ktb_cpp::Ilu0 (.apply, .factors,
//     + Precond (solver_types.hpp:22-27)            .precond() -> ktune::Precond)
//   load_matrix_market / write_matrix_market      ktb_cpp::load_matrix_market<Csr, Sym>,
//     (matrix_market.hpp:165-239)                   ktb_cpp::write_matrix_market
//
// Matrices are taken by duck typing (any type with members n, row_ptr,
// col_idx, values holding int64 / double contiguous storage), so the
// reference's own ktune::CsrMatrix / SymCsrMatrix bind directly. The engine's
// op() returns a LinOp whose apply has the reference's host-span signature;
// it converts implicitly to ktune::LinOp, so reference solvers
// (gmres_m, bicgstab, lanczos_restarted, ...) run unchanged on the GPU SpMV.
#pragma once

#include <chrono>
#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "ktb.h"

namespace ktb_cpp {

using index_t = std::int64_t;

class Error : public std::runtime_error {  // mirrors ktune::Error
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

inline void check(int rc) {
    if (rc != KTB_OK) throw Error(ktb_last_error());
}

enum class UnsymKernel { u1_row = KTB_U1, u2_nnz = KTB_U2, u3_bss = KTB_U3, u4_ss = KTB_U4 };
enum class SymKernel { s1_row = KTB_S1, s2_nnz = KTB_S2, s3_nnz_zero_omit = KTB_S3 };
enum class PartitionScheme { row_based = KTB_ROW_BASED, nnz_balanced = KTB_NNZ_BALANCED };

// Owner of a device-resident matrix (uploaded once, int32 indices).
class DeviceMatrix {
public:
    template <typename M>
    DeviceMatrix(const M& a, bool symmetric_upper, int device = 0) {
        require_shapes(a);
        check(ktb_matrix_create(a.n, a.row_ptr.data(), a.col_idx.data(), a.values.data(),
                                symmetric_upper ? KTB_SYM_UPPER : KTB_GENERAL, device, &h_));
        n_ = a.n;
    }
    explicit DeviceMatrix(ktb_matrix* adopt) : h_(adopt) {
        int64_t n = 0;
        check(ktb_matrix_info(h_, &n, nullptr, nullptr, nullptr, nullptr));
        n_ = n;
    }
    ~DeviceMatrix() {
        if (h_) ktb_matrix_destroy(h_);
    }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    ktb_matrix* get() const { return h_; }
    index_t n() const { return n_; }

private:
    template <typename M>
    static void require_shapes(const M& a) {  // csr.hpp:39-43 length checks
        if (a.n < 0) throw Error("csr: negative dimension");
        if (static_cast<index_t>(a.row_ptr.size()) != a.n + 1)
            throw Error("csr: row_ptr length != n+1");
        if (a.col_idx.size() != a.values.size())
            throw Error("csr: col_idx/values length mismatch");
    }
    ktb_matrix* h_ = nullptr;
    index_t n_ = 0;
};

// An execution plan (kernel + device decomposition + stream).
class Plan {
public:
    Plan(std::shared_ptr<DeviceMatrix> m, int kernel, int64_t param = 0, int workers = 0,
         void* stream = nullptr)
        : m_(std::move(m)) {
        check(ktb_plan_create(m_->get(), kernel, param, workers, stream, &h_));
    }
    Plan(std::shared_ptr<DeviceMatrix> m, ktb_plan* adopt) : m_(std::move(m)), h_(adopt) {}
    ~Plan() {
        if (h_) ktb_plan_destroy(h_);
    }
    Plan(Plan&& o) noexcept : m_(std::move(o.m_)), h_(o.h_) { o.h_ = nullptr; }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;

    // host spans: y = A x with H2D/D2H inside (LinOp::apply contract)
    void apply(std::span<const double> x, std::span<double> y) const {
        if (static_cast<index_t>(x.size()) != m_->n() || static_cast<index_t>(y.size()) != m_->n())
            throw Error("spmv: dimension mismatch");  // spmv.hpp:114-115
        check(ktb_spmv(h_, x.data(), y.data(), KTB_PTR_HOST));
    }
    // count host vectors back to back (x_k = x[k*n ...], y_k likewise; one
    // vector reused when x.size() == n): the copies of neighbouring vectors
    // overlap the SpMV (ktb_spmv_host_pipelined; pinned memory for overlap)
    void apply_batch(std::span<const double> x, std::span<double> y, index_t count) const {
        const index_t n = m_->n();
        const bool x1 = static_cast<index_t>(x.size()) == n;
        const bool y1 = static_cast<index_t>(y.size()) == n;
        if (count < 0 || (!x1 && static_cast<index_t>(x.size()) != n * count) ||
            (!y1 && static_cast<index_t>(y.size()) != n * count))
            throw Error("spmv: dimension mismatch");
        check(ktb_spmv_host_pipelined(h_, count, x.data(), x1 ? 0 : n, y.data(), y1 ? 0 : n));
    }
    // device pointers, asynchronous on the plan's stream
    void apply_device(const double* x, double* y) const {
        check(ktb_spmv(h_, x, y, KTB_PTR_DEVICE));
    }
    int kernel() const {
        int k = 0;
        check(ktb_plan_info(h_, &k, nullptr, nullptr, nullptr, nullptr));
        return k;
    }
    ktb_plan* get() const { return h_; }
    const std::shared_ptr<DeviceMatrix>& matrix() const { return m_; }

private:
    std::shared_ptr<DeviceMatrix> m_;
    ktb_plan* h_ = nullptr;
};

struct TuningCandidate {  // autotune.hpp:130-139
    std::string name;
    int ordinal = 0;
    index_t jl = 0;
    int workers = 1;
    std::vector<double> trial_seconds;
    double best_seconds = 0;
    bool correct = false;
    int executions = 0;
};

struct TuningReport {  // autotune.hpp:141-158
    std::vector<TuningCandidate> candidates;
    int selected = -1;
    int trials_per_candidate = 3;
    const TuningCandidate& selected_candidate() const {
        if (selected < 0 || selected >= static_cast<int>(candidates.size()))
            throw Error("tuning report: nothing selected");
        return candidates[selected];
    }
    int max_executions() const {
        int m = 0;
        for (const auto& c : candidates) m = std::max(m, c.executions);
        return m;
    }
};

struct SelectOptions {  // autotune.hpp:160-165
    std::vector<index_t> jl_candidates;  // GPU: nonzeros per BSS lane (jl = nnz / E)
    int timed_trials = 3;
    std::function<double()> now;  // injectable timer; empty = CUDA events
    bool warm_trials = false;     // true: back-to-back trials (the reference's protocol)
};

struct Choice {  // UnsymChoice / SymChoice (autotune.hpp:168-183)
    std::shared_ptr<Plan> plan;
    int kernel = 0;
    index_t jl = 0;
    int workers = 1;
};

namespace detail {
inline double call_now(void* ctx) { return (*static_cast<std::function<double()>*>(ctx))(); }

inline std::pair<Choice, TuningReport> select(std::shared_ptr<DeviceMatrix> m,
                                              const SelectOptions& opts) {
    ktb_select_opts o{};
    o.params = opts.jl_candidates.empty() ? nullptr : opts.jl_candidates.data();
    o.n_params = static_cast<int>(opts.jl_candidates.size());
    o.timed_trials = opts.timed_trials;
    o.warm_trials = opts.warm_trials ? 1 : 0;
    std::function<double()> now = opts.now;
    if (now) {
        o.now = &call_now;
        o.now_ctx = &now;
    }
    std::vector<ktb_candidate> c(64);
    int nc = 0, sel = -1;
    ktb_plan* w = nullptr;
    check(ktb_select(m->get(), &o, nullptr, &w, c.data(), 64, &nc, &sel));
    TuningReport rep;
    rep.selected = sel;
    rep.trials_per_candidate = opts.timed_trials;
    for (int i = 0; i < nc && i < 64; ++i) {
        TuningCandidate t;
        t.name = c[i].name;
        t.ordinal = c[i].ordinal;
        t.jl = c[i].param;
        t.workers = c[i].workers;
        t.trial_seconds.assign(c[i].trial_seconds, c[i].trial_seconds + c[i].n_trials);
        t.best_seconds = c[i].best_seconds;
        t.correct = c[i].correct != 0;
        t.executions = c[i].executions;
        rep.candidates.push_back(t);
    }
    Choice ch;
    ch.plan = std::make_shared<Plan>(m, w);
    ch.kernel = ch.plan->kernel();
    ch.jl = rep.selected_candidate().jl;
    ch.workers = rep.selected_candidate().workers;
    return {ch, rep};
}
}  // namespace detail

template <typename M>
std::pair<Choice, TuningReport> select_spmv_unsym(const M& a, const SelectOptions& opts = {},
                                                  int device = 0) {
    if (a.n <= 0 || a.values.empty()) throw Error("kernel selection: empty matrix");
    return detail::select(std::make_shared<DeviceMatrix>(a, false, device), opts);
}

template <typename M>
std::pair<Choice, TuningReport> select_spmv_sym(const M& a, const SelectOptions& opts = {},
                                                int device = 0) {
    if (a.n <= 0 || a.values.empty()) throw Error("kernel selection: empty matrix");
    return detail::select(std::make_shared<DeviceMatrix>(a, true, device), opts);
}

// Same two members as ktune::LinOp; converts to any type constructible from
// {n, apply} (ktune::LinOp included).
struct LinOp {
    index_t n = 0;
    std::function<void(std::span<const double>, std::span<double>)> apply;
    template <typename L>
    operator L() const {
        return L{n, apply};
    }
};

// meta.hpp:20-82: the tuned kernel bound to its matrix; op() counts calls and
// in-call seconds like the reference engines.
class Engine {
public:
    explicit Engine(Choice choice) : choice_(std::move(choice)) {}
    LinOp op() {
        return {choice_.plan->matrix()->n(),
                [this](std::span<const double> x, std::span<double> y) {
                    const auto t0 = std::chrono::steady_clock::now();
                    choice_.plan->apply(x, y);
                    seconds_ += std::chrono::duration<double>(
                                    std::chrono::steady_clock::now() - t0)
                                    .count();
                    ++calls_;
                }};
    }
    index_t calls() const { return calls_; }
    double kernel_seconds() const { return seconds_; }
    int workers() const { return choice_.workers; }
    const Choice& choice() const { return choice_; }

private:
    Choice choice_;
    index_t calls_ = 0;
    double seconds_ = 0.0;
};
using UnsymEngine = Engine;
using SymEngine = Engine;

// spmv.hpp:111-234 one-shot forms (plan built and cached by the caller if hot)
template <typename M>
void spmv_unsym(UnsymKernel k, const M& a, std::span<const double> x, std::span<double> y,
                int device = 0) {
    Plan p(std::make_shared<DeviceMatrix>(a, false, device), static_cast<int>(k));
    p.apply(x, y);
}

template <typename M>
void spmv_sym(SymKernel k, const M& a, std::span<const double> x, std::span<double> y,
              int device = 0) {
    Plan p(std::make_shared<DeviceMatrix>(a, true, device), static_cast<int>(k));
    p.apply(x, y);
}

// Integer plan artefacts, computed on the device, bit-exact with the
// reference builders.
inline std::vector<index_t> build_row_partition(const DeviceMatrix& m, int workers,
                                                PartitionScheme s) {
    if (workers < 1) throw Error("row partition: num_workers must be >= 1");
    std::vector<index_t> b(workers + 1);
    check(ktb_row_partition(m.get(), workers, static_cast<int>(s), b.data()));
    return b;
}

inline std::pair<std::vector<index_t>, std::vector<index_t>> build_reduction_regions(
    const DeviceMatrix& m, const std::vector<index_t>& boundaries) {
    const int P = static_cast<int>(boundaries.size()) - 1;
    std::vector<index_t> lo(P), hi(P);
    check(ktb_reduction_regions(m.get(), P, boundaries.data(), lo.data(), hi.data()));
    return {lo, hi};
}

// ---------------------------------------------------------------- ILU(0)
// ilu0_factorize on the device (bit-exact factors); precond() plugs the
// device solve into the reference's solvers as their Precond.
struct PrecondView {
    std::function<void(std::span<const double>, std::span<double>)> apply;
    template <typename P>
    operator P() const {
        P p;
        p.apply = apply;
        return p;
    }
};

class Ilu0 {
public:
    explicit Ilu0(std::shared_ptr<DeviceMatrix> m) : m_(std::move(m)) {
        check(ktb_ilu0_create(m_->get(), nullptr, &h_));
    }
    template <typename M>
    explicit Ilu0(const M& a, int device = 0)
        : Ilu0(std::make_shared<DeviceMatrix>(a, false, device)) {}
    ~Ilu0() {
        if (h_) ktb_ilu0_destroy(h_);
    }
    Ilu0(const Ilu0&) = delete;
    Ilu0& operator=(const Ilu0&) = delete;
    // ilu0.hpp:73-87 on host spans (z = (LU)^{-1} r)
    void apply(std::span<const double> r, std::span<double> z) const {
        if (static_cast<index_t>(r.size()) != m_->n() || static_cast<index_t>(z.size()) != m_->n())
            throw Error("ilu0: dimension mismatch");
        check(ktb_ilu0_apply(h_, r.data(), z.data(), KTB_PTR_HOST, nullptr));
    }
    // device pointers, enqueued on `stream` (nullptr = legacy default stream)
    void apply_device(const double* r, double* z, void* stream = nullptr) const {
        check(ktb_ilu0_apply(h_, r, z, KTB_PTR_DEVICE, stream));
    }
    // IluFactors::diag_ptr and ::values (ilu0.hpp:14-18)
    std::pair<std::vector<index_t>, std::vector<double>> factors() const {
        int64_t nnz = 0;
        check(ktb_matrix_info(m_->get(), nullptr, &nnz, nullptr, nullptr, nullptr));
        std::vector<int32_t> d(static_cast<std::size_t>(m_->n()));
        std::vector<double> v(static_cast<std::size_t>(nnz));
        check(ktb_ilu0_download(h_, d.data(), v.data()));
        return {std::vector<index_t>(d.begin(), d.end()), std::move(v)};
    }
    PrecondView precond() const {
        return {[this](std::span<const double> r, std::span<double> z) { apply(r, z); }};
    }
    ktb_ilu* get() const { return h_; }

private:
    std::shared_ptr<DeviceMatrix> m_;
    ktb_ilu* h_ = nullptr;
};

// ------------------------------------------------------- Matrix Market
// load_matrix_market (matrix_market.hpp:165-194): the same variant shape --
// Sym when want_symmetric, Csr otherwise -- for any duck-typed Csr / Sym.
template <typename Csr, typename Sym>
std::variant<Csr, Sym> load_matrix_market(const std::string& path, bool want_symmetric) {
    ktb_csr_host* h = nullptr;
    check(ktb_mm_read(path.c_str(), want_symmetric ? 1 : 0, &h));
    int64_t n = 0, nnz = 0;
    int kind = 0;
    const int rc = ktb_csr_host_info(h, &n, &nnz, &kind);
    if (rc != KTB_OK) {
        ktb_csr_host_destroy(h);
        check(rc);
    }
    auto fill = [&](auto& a) {
        a.n = n;
        a.row_ptr.resize(static_cast<std::size_t>(n + 1));
        a.col_idx.resize(static_cast<std::size_t>(nnz));
        a.values.resize(static_cast<std::size_t>(nnz));
        const int r2 = ktb_csr_host_copy(h, a.row_ptr.data(), a.col_idx.data(), a.values.data());
        ktb_csr_host_destroy(h);
        check(r2);
    };
    if (kind == KTB_SYM_UPPER) {
        Sym s;
        fill(s);
        return s;
    }
    Csr a;
    fill(a);
    return a;
}

// write_matrix_market (matrix_market.hpp:223-239); symmetric_upper selects the
// SymCsrMatrix form (stored upper triangle written as the lower form)
template <typename M>
void write_matrix_market(const std::string& path, const M& a, bool symmetric_upper) {
    check(ktb_mm_write(path.c_str(), a.n, a.row_ptr.data(), a.col_idx.data(), a.values.data(),
                       symmetric_upper ? KTB_SYM_UPPER : KTB_GENERAL));
}

}  // namespace ktb_cpp
