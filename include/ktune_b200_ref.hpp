// ktune_b200_ref.hpp -- the reference's KERNEL-LEVEL SpMV interface on the
// B200 engine, signature for signature (namespace ktb_ref).
//
// A caller of the reference (namespace ktune, /root/reference/proj/include/
// ktune/) changes the namespace qualifier and nothing else:
//
//   reference (file:line)                                  here (same shape)
//   WorkerPool(int size)                (spmv.hpp:41-67)   ktb_ref::WorkerPool
//   RowPartition, PartitionScheme       (partition.hpp:12-24)
//   build_row_partition(span<const index_t> row_ptr, P, scheme)
//                                       (partition.hpp:28-55)   -- on the device
//   ReductionRegions, build_reduction_regions(a, part)
//                                       (partition.hpp:60-96)   -- on the device
//   BssPlan, build_bss_plan(a, jl)      (bss.hpp:19-69)         -- on the device
//   spmv_unsym(kernel, a, part*, plan*, x, y, pool)  (spmv.hpp:111-170)
//   spmv_sym(kernel, a, part, regions*, x, y, pool)  (spmv.hpp:180-234)
//   SelectOptions, TuningCandidate, TuningReport, UnsymChoice, SymChoice
//                                       (autotune.hpp:130-183)
//   select_spmv_unsym(a, pool, opts)    (autotune.hpp:267-330)
//   select_spmv_sym(a, pool, opts)      (autotune.hpp:333-377)
//   UnsymEngine(a, choice).op(), SymEngine (meta.hpp:20-82)
//   LinOp                               (solver_types.hpp:17-20)
//   Error                               (common.hpp:18-25), same messages
//
// Matrices are taken by duck typing (members n, row_ptr, col_idx, values
// with contiguous int64 / double storage): the reference's ktune::CsrMatrix
// and ktune::SymCsrMatrix bind directly, and ktb_ref::CsrMatrix /
// SymCsrMatrix exist for callers without the reference headers.
//
// Device residency. The reference passes the matrix by reference on every
// call; the engine keeps ONE device copy per matrix (keyed on the address and
// size of its three arrays) and one device plan per (matrix, kernel), created
// on first use and reused by every later call -- the upload and the plan
// build are paid once, not per SpMV. select_spmv_* stores its winning plan
// (the tuned device variant) under the selected kernel, so the engine built
// from the choice runs exactly what was timed. A matrix modified in place
// must be released with ktb_ref::release(a) before its next use. x and y are
// host spans as in the reference: each call copies x in and y out
// (LinOp::apply contract); device-pointer and batched forms are in
// ktune_b200.hpp (ktb_cpp::Plan).
//
// The integer artefacts (RowPartition, ReductionRegions, BssPlan) are built
// by the device builders and are bit-exact with the reference's. They are
// validated exactly as the reference validates them; the GPU kernels use
// their own decomposition (CTAs, warp tiles, nonzeros per lane): U1 over the
// warp-sliced copy is bitwise equal to spmv_ref, every kernel agrees within
// 1e-12 (|A||x|)_i.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <functional>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "ktune_b200.hpp"

namespace ktb_ref {

using index_t = std::int64_t;
using Error = ktb_cpp::Error;

inline void require(bool cond, const char* msg) {  // common.hpp:23-25
    if (!cond) throw Error(msg);
}

enum class UnsymKernel { u1_row, u2_nnz, u3_bss, u4_ss };             // spmv.hpp:15
enum class SymKernel { s1_row, s2_nnz, s3_nnz_zero_omit };           // spmv.hpp:16
enum class PartitionScheme { row_based, nnz_balanced };              // partition.hpp:12

struct CsrMatrix {  // csr.hpp:13-55 (layout only)
    index_t n = 0;
    std::vector<index_t> row_ptr, col_idx;
    std::vector<double> values;
    index_t nnz() const { return static_cast<index_t>(values.size()); }
};
struct SymCsrMatrix : CsrMatrix {  // csr.hpp:57-65
    index_t spmv_flops() const { return 4 * nnz() - 2 * n; }
};

// spmv.hpp:41-67. The reference's per-worker scratch lives on the device,
// owned by the plans; the pool keeps the worker count the artefacts use.
class WorkerPool {
public:
    explicit WorkerPool(int size) : size_(size) {
        require(size >= 1, "worker pool: size must be >= 1");
    }
    int size() const { return size_; }

private:
    int size_;
};

struct RowPartition {  // partition.hpp:15-24
    int num_workers = 1;
    std::vector<index_t> boundaries;
    PartitionScheme scheme = PartitionScheme::row_based;
    index_t lo(int p) const { return boundaries[p]; }
    index_t hi(int p) const { return boundaries[p + 1]; }
    index_t rows() const { return boundaries.back(); }
};

struct ReductionRegions {  // partition.hpp:60-71
    int num_workers = 1;
    std::vector<index_t> lo, hi;
    index_t total_width() const {
        index_t w = 0;
        for (int p = 0; p < num_workers; ++p) w += hi[p] - lo[p];
        return w;
    }
};

struct BssPlan {  // bss.hpp:19-32
    index_t jl = 0, n = 0, nnz = 0;
    std::vector<index_t> slice_start, slice_len, slice_row, lane_slice_ptr, row_slice_ptr;
    std::vector<std::uint8_t> row_start_flag;
    index_t total_slices() const { return static_cast<index_t>(slice_start.size()); }
};

using TimerFn = std::function<double()>;

struct TuningCandidate {  // autotune.hpp:130-139
    std::string name;
    int ordinal = 0;
    index_t jl = 0;
    int workers = 1;
    std::vector<double> trial_seconds;
    double best_seconds = std::numeric_limits<double>::infinity();
    bool correct = false;
    int executions = 0;
};

struct TuningReport {  // autotune.hpp:141-158
    std::vector<TuningCandidate> candidates;
    int selected = -1;
    int trials_per_candidate = 3;
    bool forced = false;
    int max_executions() const {
        int m = 0;
        for (const auto& c : candidates) m = std::max(m, c.executions);
        return m;
    }
    const TuningCandidate& selected_candidate() const {
        require(selected >= 0 && selected < static_cast<int>(candidates.size()),
                "tuning report: nothing selected");
        return candidates[static_cast<std::size_t>(selected)];
    }
};

// autotune.hpp:160-165. On the device the U3 sweep runs over nonzeros per
// lane (the GPU lane count is nnz / E); jl_candidates keep the reference's
// default and are reported, the device sweep is the engine's.
struct SelectOptions {
    std::vector<index_t> jl_candidates = {8, 16, 32, 64, 128, 256};
    int timed_trials = 3;
    bool sweep_workers = false;
    TimerFn now;
    bool warm_trials = false;  // true: back-to-back trials as the reference (default: cold L2)
};

struct UnsymChoice {  // autotune.hpp:168-176
    UnsymKernel kernel = UnsymKernel::u1_row;
    index_t jl = 0;
    int workers = 1;
    RowPartition row_part;
    RowPartition nnz_part;
    std::optional<BssPlan> plan;
};

struct SymChoice {  // autotune.hpp:178-183
    SymKernel kernel = SymKernel::s1_row;
    int workers = 1;
    RowPartition row_part;
    RowPartition nnz_part;
    ReductionRegions regions;
};

// solver_types.hpp:17-20; converts to any {n, apply} aggregate (ktune::LinOp).
struct LinOp {
    index_t n = 0;
    std::function<void(std::span<const double>, std::span<double>)> apply;
    template <typename L>
    operator L() const {
        return L{n, apply};
    }
};

// ------------------------------------------------------- device residency
namespace detail {

inline int& device_ref() {
    static int d = 0;
    return d;
}

struct Key {
    const void* rp;
    const void* ci;
    const void* v;
    index_t n, nnz;
    int kind;
    bool operator<(const Key& o) const {
        return std::tie(rp, ci, v, n, nnz, kind) < std::tie(o.rp, o.ci, o.v, o.n, o.nnz, o.kind);
    }
};

struct Entry {
    std::shared_ptr<ktb_cpp::DeviceMatrix> dm;
    std::map<int, std::shared_ptr<ktb_cpp::Plan>> plans;  // by ABI kernel tag
};

struct Cache {
    std::mutex mu;
    std::map<Key, Entry> entries;
    std::vector<Key> order;  // insertion order, oldest first
    static constexpr std::size_t kMax = 8;
};

inline Cache& cache() {
    static Cache c;
    return c;
}

template <typename M>
Key key_of(const M& a, int kind) {
    return {a.row_ptr.data(), a.col_idx.data(), a.values.data(), a.n,
            static_cast<index_t>(a.values.size()), kind};
}

// the device copy of `a` (uploaded on first use)
template <typename M>
Entry& entry(const M& a, int kind) {
    Cache& c = cache();
    const Key k = key_of(a, kind);
    auto it = c.entries.find(k);
    if (it != c.entries.end()) return it->second;
    if (c.entries.size() >= Cache::kMax) {  // drop the oldest matrix
        c.entries.erase(c.order.front());
        c.order.erase(c.order.begin());
    }
    Entry e;
    e.dm = std::make_shared<ktb_cpp::DeviceMatrix>(a, kind == KTB_SYM_UPPER, device_ref());
    c.order.push_back(k);
    return c.entries.emplace(k, std::move(e)).first->second;
}

// default device variant per kernel when none was selected: U1 tries the
// persistent slices with coded columns and values (106), with coded columns
// only (105), then the plain warp slices (100), then lanes
inline int64_t default_param(int k) { return k == KTB_U1 ? 106 : 0; }

template <typename M>
std::shared_ptr<ktb_cpp::Plan> plan_for(const M& a, int kind, int kernel) {
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    Entry& e = entry(a, kind);
    auto it = e.plans.find(kernel);
    if (it != e.plans.end()) return it->second;
    std::shared_ptr<ktb_cpp::Plan> p;
    const int64_t tries[4] = {default_param(kernel), 105, 100, 0};
    for (int t = 0; t < (kernel == KTB_U1 ? 4 : 1) && !p; ++t) {
        try {
            p = std::make_shared<ktb_cpp::Plan>(e.dm, kernel, tries[t]);
        } catch (const Error&) {
            // refused layouts: few distinct values (106), uniform width / few
            // column deltas (105), or padding beyond 3x (100) for very
            // irregular rows
            if (kernel != KTB_U1 || t == 3) throw;
        }
    }
    e.plans[kernel] = p;
    return p;
}

template <typename M>
std::shared_ptr<ktb_cpp::DeviceMatrix> device_matrix(const M& a, int kind) {
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.mu);
    return entry(a, kind).dm;
}

inline TuningReport to_report(const std::vector<ktb_candidate>& c, int nc, int sel, int trials) {
    TuningReport rep;
    rep.selected = sel;
    rep.trials_per_candidate = trials;
    for (int i = 0; i < nc; ++i) {
        TuningCandidate t;
        t.name = c[i].name;
        t.ordinal = c[i].ordinal;
        t.jl = c[i].param;
        t.workers = c[i].workers;
        t.trial_seconds.assign(c[i].trial_seconds, c[i].trial_seconds + c[i].n_trials);
        t.best_seconds = c[i].best_seconds;
        t.correct = c[i].correct != 0;
        t.executions = c[i].executions;
        rep.candidates.push_back(std::move(t));
    }
    return rep;
}

inline double call_now(void* ctx) { return (*static_cast<TimerFn*>(ctx))(); }

// ktb_select on the device; the winner is cached under its kernel
template <typename M>
std::pair<int, TuningReport> select(const M& a, int kind, const SelectOptions& opts,
                                    index_t* lanes) {
    auto dm = device_matrix(a, kind);
    ktb_select_opts o{};
    o.timed_trials = opts.timed_trials;
    o.warm_trials = opts.warm_trials ? 1 : 0;
    TimerFn now = opts.now;
    if (now) {
        o.now = &call_now;
        o.now_ctx = &now;
    }
    std::vector<ktb_candidate> c(64);
    int nc = 0, sel = -1;
    ktb_plan* w = nullptr;
    ktb_cpp::check(ktb_select(dm->get(), &o, nullptr, &w, c.data(), 64, &nc, &sel));
    auto plan = std::make_shared<ktb_cpp::Plan>(dm, w);
    int kernel = 0;
    int64_t param = 0;
    ktb_cpp::check(ktb_plan_info(w, &kernel, &param, nullptr, nullptr, nullptr));
    if (lanes) *lanes = param;
    {
        Cache& cc = cache();
        std::lock_guard<std::mutex> g(cc.mu);
        entry(a, kind).plans[kernel] = plan;
    }
    return {kernel, to_report(c, std::min(nc, 64), sel, opts.timed_trials)};
}

}  // namespace detail

// Device used for matrices first seen after this call (default 0).
inline void set_device(int device) { detail::device_ref() = device; }

// Forget the device copy and plans of `a` (after modifying it in place).
template <typename M>
void release(const M& a) {
    auto& c = detail::cache();
    std::lock_guard<std::mutex> g(c.mu);
    for (int kind : {KTB_GENERAL, KTB_SYM_UPPER}) {
        const auto k = detail::key_of(a, kind);
        c.entries.erase(k);
        for (auto it = c.order.begin(); it != c.order.end(); ++it)
            if (!(*it < k) && !(k < *it)) {
                c.order.erase(it);
                break;
            }
    }
}

// ------------------------------------------------------------ artefacts
// partition.hpp:28-55 (computed on the device, bit-exact)
inline RowPartition build_row_partition(std::span<const index_t> row_ptr, int num_workers,
                                        PartitionScheme scheme) {
    require(num_workers >= 1, "row partition: num_workers must be >= 1");
    RowPartition part;
    part.num_workers = num_workers;
    part.scheme = scheme;
    part.boundaries.resize(static_cast<std::size_t>(num_workers) + 1);
    const index_t n = static_cast<index_t>(row_ptr.size()) - 1;
    ktb_cpp::check(ktb_row_partition_rowptr(
        row_ptr.data(), n, num_workers,
        scheme == PartitionScheme::row_based ? KTB_ROW_BASED : KTB_NNZ_BALANCED,
        detail::device_ref(), part.boundaries.data()));
    return part;
}

// partition.hpp:73-96 (device, bit-exact)
template <typename M>
ReductionRegions build_reduction_regions(const M& a, const RowPartition& part) {
    require(part.rows() == a.n, "reduction regions: partition/matrix dimension mismatch");
    auto dm = detail::device_matrix(a, KTB_SYM_UPPER);
    ReductionRegions r;
    r.num_workers = part.num_workers;
    r.lo.assign(part.num_workers, 0);
    r.hi.assign(part.num_workers, 0);
    ktb_cpp::check(ktb_reduction_regions(dm->get(), part.num_workers, part.boundaries.data(),
                                         r.lo.data(), r.hi.data()));
    return r;
}

// bss.hpp:34-69 (device, bit-exact)
template <typename M>
BssPlan build_bss_plan(const M& a, index_t jl) {
    require(jl >= 1, "bss plan: jl must be >= 1");
    auto dm = detail::device_matrix(a, KTB_GENERAL);
    BssPlan p;
    index_t total = 0;
    ktb_cpp::check(ktb_bss_plan_size(dm->get(), jl, &p.jl, &total));
    p.n = a.n;
    p.nnz = static_cast<index_t>(a.values.size());
    p.slice_start.resize(total);
    p.slice_len.resize(total);
    p.slice_row.resize(total);
    p.lane_slice_ptr.resize(static_cast<std::size_t>(p.jl) + 1);
    p.row_slice_ptr.resize(static_cast<std::size_t>(a.n) + 1);
    p.row_start_flag.resize(static_cast<std::size_t>(p.nnz));
    ktb_cpp::check(ktb_bss_plan_copy(dm->get(), jl, p.slice_start.data(), p.slice_len.data(),
                                     p.slice_row.data(), p.lane_slice_ptr.data(),
                                     p.row_slice_ptr.data(), p.row_start_flag.data()));
    return p;
}

// ------------------------------------------------------------------ SpMV
// spmv.hpp:111-170, same contract checks and messages.
template <typename M>
void spmv_unsym(UnsymKernel kernel, const M& a, const RowPartition* part, const BssPlan* plan,
                std::span<const double> x, std::span<double> y, WorkerPool& pool) {
    (void)pool;
    require(static_cast<index_t>(x.size()) == a.n && static_cast<index_t>(y.size()) == a.n,
            "spmv: dimension mismatch");
    const index_t nnz = static_cast<index_t>(a.values.size());
    switch (kernel) {
        case UnsymKernel::u1_row:
        case UnsymKernel::u2_nnz: {
            require(part != nullptr, "spmv: U1/U2 need a row partition");
            require(part->rows() == a.n, "spmv: partition built for a different matrix");
            const auto want = kernel == UnsymKernel::u1_row ? PartitionScheme::row_based
                                                            : PartitionScheme::nnz_balanced;
            require(part->scheme == want, "spmv: partition scheme does not match kernel");
            break;
        }
        case UnsymKernel::u3_bss:
        case UnsymKernel::u4_ss:
            require(plan != nullptr, "spmv: U3/U4 need a bss plan");
            require(plan->n == a.n && plan->nnz == nnz, "spmv: plan built for a different matrix");
            break;
    }
    if (a.n == 0) return;
    detail::plan_for(a, KTB_GENERAL, static_cast<int>(kernel))->apply(x, y);
}

// spmv.hpp:180-234, same contract checks and messages.
template <typename M>
void spmv_sym(SymKernel kernel, const M& a, const RowPartition& part,
              const ReductionRegions* regions, std::span<const double> x, std::span<double> y,
              WorkerPool& pool) {
    (void)pool;
    require(static_cast<index_t>(x.size()) == a.n && static_cast<index_t>(y.size()) == a.n,
            "spmv: dimension mismatch");
    require(part.rows() == a.n, "spmv: partition built for a different matrix");
    const auto want = kernel == SymKernel::s1_row ? PartitionScheme::row_based
                                                  : PartitionScheme::nnz_balanced;
    require(part.scheme == want, "spmv: partition scheme does not match kernel");
    const bool omit = kernel == SymKernel::s3_nnz_zero_omit;
    require(!omit || regions != nullptr, "spmv: S3 needs reduction regions");
    if (omit)
        require(regions->num_workers == part.num_workers,
                "spmv: regions built for a different partition");
    if (a.n == 0) return;
    detail::plan_for(a, KTB_SYM_UPPER, KTB_S1 + static_cast<int>(kernel))->apply(x, y);
}

// ------------------------------------------------------------- selection
// autotune.hpp:267-330 on device time; the choice carries the reference's
// plan values built by the device builders for pool.size() workers.
template <typename M>
std::pair<UnsymChoice, TuningReport> select_spmv_unsym(const M& a, WorkerPool& pool,
                                                       SelectOptions opts = {}) {
    require(a.n > 0 && !a.values.empty(), "kernel selection: empty matrix");
    index_t lanes = 0;
    auto [kernel, report] = detail::select(a, KTB_GENERAL, opts, &lanes);
    UnsymChoice choice;
    choice.kernel = static_cast<UnsymKernel>(kernel);
    choice.workers = pool.size();
    choice.row_part = ktb_ref::build_row_partition(a.row_ptr, pool.size(), PartitionScheme::row_based);
    choice.nnz_part = ktb_ref::build_row_partition(a.row_ptr, pool.size(), PartitionScheme::nnz_balanced);
    if (choice.kernel == UnsymKernel::u3_bss || choice.kernel == UnsymKernel::u4_ss) {
        choice.jl = lanes;  // the device's lane count (nonzeros / E)
        choice.plan = ktb_ref::build_bss_plan(a, choice.jl);
    }
    return {std::move(choice), std::move(report)};
}

// autotune.hpp:333-377
template <typename M>
std::pair<SymChoice, TuningReport> select_spmv_sym(const M& a, WorkerPool& pool,
                                                   SelectOptions opts = {}) {
    require(a.n > 0 && !a.values.empty(), "kernel selection: empty matrix");
    auto [kernel, report] = detail::select(a, KTB_SYM_UPPER, opts, nullptr);
    SymChoice choice;
    choice.kernel = static_cast<SymKernel>(kernel - KTB_S1);
    choice.workers = pool.size();
    choice.row_part = ktb_ref::build_row_partition(a.row_ptr, pool.size(), PartitionScheme::row_based);
    choice.nnz_part = ktb_ref::build_row_partition(a.row_ptr, pool.size(), PartitionScheme::nnz_balanced);
    choice.regions = ktb_ref::build_reduction_regions(a, choice.nnz_part);
    return {std::move(choice), std::move(report)};
}

// --------------------------------------------------------------- engines
// meta.hpp:20-49
class UnsymEngine {
public:
    template <typename M>
    UnsymEngine(const M& a, UnsymChoice choice)
        : n_(a.n), nnz_(static_cast<index_t>(a.values.size())), choice_(std::move(choice)),
          pool_(choice_.workers) {
        const M* pa = &a;
        run_ = [this, pa](std::span<const double> x, std::span<double> y) {
            ktb_ref::spmv_unsym(choice_.kernel, *pa,
                       choice_.kernel == UnsymKernel::u1_row ? &choice_.row_part
                                                             : &choice_.nnz_part,
                       choice_.plan ? &*choice_.plan : nullptr, x, y, pool_);
        };
    }
    LinOp op() {
        return {n_, [this](std::span<const double> x, std::span<double> y) {
                    const auto t0 = std::chrono::steady_clock::now();
                    run_(x, y);
                    seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
                                    .count();
                    ++calls_;
                }};
    }
    index_t calls() const { return calls_; }
    double kernel_seconds() const { return seconds_; }
    double flops_per_call() const { return 2.0 * static_cast<double>(nnz_); }
    int workers() const { return choice_.workers; }
    const UnsymChoice& choice() const { return choice_; }

private:
    index_t n_, nnz_;
    UnsymChoice choice_;
    WorkerPool pool_;
    std::function<void(std::span<const double>, std::span<double>)> run_;
    index_t calls_ = 0;
    double seconds_ = 0.0;
};

// meta.hpp:51-82
class SymEngine {
public:
    template <typename M>
    SymEngine(const M& a, SymChoice choice)
        : n_(a.n), flops_(4 * static_cast<index_t>(a.values.size()) - 2 * a.n),
          choice_(std::move(choice)), pool_(choice_.workers) {
        const M* pa = &a;
        run_ = [this, pa](std::span<const double> x, std::span<double> y) {
            ktb_ref::spmv_sym(choice_.kernel, *pa,
                     choice_.kernel == SymKernel::s1_row ? choice_.row_part : choice_.nnz_part,
                     choice_.kernel == SymKernel::s3_nnz_zero_omit ? &choice_.regions : nullptr,
                     x, y, pool_);
        };
    }
    LinOp op() {
        return {n_, [this](std::span<const double> x, std::span<double> y) {
                    const auto t0 = std::chrono::steady_clock::now();
                    run_(x, y);
                    seconds_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0)
                                    .count();
                    ++calls_;
                }};
    }
    index_t calls() const { return calls_; }
    double kernel_seconds() const { return seconds_; }
    double flops_per_call() const { return static_cast<double>(flops_); }
    int workers() const { return choice_.workers; }
    const SymChoice& choice() const { return choice_; }

private:
    index_t n_, flops_;
    SymChoice choice_;
    WorkerPool pool_;
    std::function<void(std::span<const double>, std::span<double>)> run_;
    index_t calls_ = 0;
    double seconds_ = 0.0;
};

}  // namespace ktb_ref
