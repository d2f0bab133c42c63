// Kernel-level drop-in (TEST): the reference's own call sequences, with the
// namespace qualifier ktune:: changed to ktb_ref:: and nothing else, run on
// the B200 engine through include/ktune_b200_ref.hpp, against the unmodified
// reference (compiled from /root/reference headers by tests/cpp/Makefile).
//
// 1. meta.hpp:171-190 (linear_solve_meta's choice + engine set-up), both
//    branches (the fixed STABLE arguments and select_spmv_unsym), then the
//    reference's ktune::gmres_m on the resulting LinOp vs the same sequence in
//    namespace ktune -> same iteration count (+-2), true residual < tol.
// 2. spmv_unsym / spmv_sym (spmv.hpp:111-113, 180-182) for every kernel with
//    the artefacts from ktb_ref's builders: U1 on the stencil (warp-sliced
//    copy) bitwise = ktune::spmv_ref, every kernel within 1e-12 (|A||x|)_i.
// 3. build_row_partition / build_reduction_regions / build_bss_plan:
//    bit-exact vs the reference builders.
// 4. Contract errors: the same messages as the reference.
// 5. Residency: 200 calls on one matrix keep one device copy.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "ktune/ktune.hpp"
#include "ktune_b200_ref.hpp"

static ktune::CsrMatrix convdiff(ktune::index_t N) {
    ktune::CsrMatrix a;
    a.n = N * N * N;
    a.row_ptr.assign(a.n + 1, 0);
    for (ktune::index_t z = 0; z < N; ++z)
        for (ktune::index_t y = 0; y < N; ++y)
            for (ktune::index_t x = 0; x < N; ++x) {
                const ktune::index_t i = (z * N + y) * N + x;
                auto put = [&](ktune::index_t j, double v) {
                    a.col_idx.push_back(j);
                    a.values.push_back(v);
                };
                if (z > 0) put(i - N * N, -1.0);
                if (y > 0) put(i - N, -1.0);
                if (x > 0) put(i - 1, -1.3);
                put(i, 6.0);
                if (x < N - 1) put(i + 1, -0.7);
                if (y < N - 1) put(i + N, -1.0);
                if (z < N - 1) put(i + N * N, -1.0);
                a.row_ptr[i + 1] = static_cast<ktune::index_t>(a.col_idx.size());
            }
    return a;
}

// ---- meta.hpp:171-190, namespace ktune -> NS (the only change) ----------
#define META_CHOICE_SEQUENCE(NS, a, workers, stable, force_kernel, force_jl, tuning_opts,     \
                             out_forced, out_op, out_engine)                                  \
    NS::WorkerPool pool(workers);                                                             \
    NS::UnsymChoice choice;                                                                   \
    if (stable) {                                                                             \
        /* Fixed arguments, no measurements. */                                               \
        choice.kernel = force_kernel;                                                         \
        choice.workers = workers;                                                             \
        choice.row_part =                                                                     \
            NS::build_row_partition(a.row_ptr, workers, NS::PartitionScheme::row_based);      \
        choice.nnz_part =                                                                     \
            NS::build_row_partition(a.row_ptr, workers, NS::PartitionScheme::nnz_balanced);   \
        if (choice.kernel == NS::UnsymKernel::u3_bss || choice.kernel == NS::UnsymKernel::u4_ss) { \
            choice.jl = force_jl;                                                             \
            choice.plan = NS::build_bss_plan(a, choice.jl);                                   \
        }                                                                                     \
        out_forced = true;                                                                    \
    } else {                                                                                  \
        auto [c, report] = NS::select_spmv_unsym(a, pool, tuning_opts);                       \
        choice = std::move(c);                                                                \
        out_forced = report.forced;                                                           \
    }                                                                                         \
    NS::UnsymEngine out_engine(a, std::move(choice));                                         \
    const NS::LinOp out_op = out_engine.op();

static double worst_rel(const ktune::CsrMatrix& a, const std::vector<double>& x,
                        const std::vector<double>& y, const std::vector<double>& yref) {
    double w = 0.0;
    for (ktune::index_t i = 0; i < a.n; ++i) {
        double absax = 0.0;
        for (auto k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
            absax += std::abs(a.values[k] * x[a.col_idx[k]]);
        const double e = std::abs(y[i] - yref[i]);
        w = std::max(w, absax > 0 ? e / absax : (e > 0 ? 1.0 : 0.0));
    }
    return w;
}

template <typename F>
static std::string message_of(F&& f) {
    try {
        f();
    } catch (const std::exception& e) {
        return e.what();
    }
    return "<no error>";
}

int main(int argc, char** argv) {
    const ktune::index_t N = argc > 1 ? std::atoll(argv[1]) : 24;
    int fail = 0;
    // ---- 1: the meta.hpp choice sequence, both branches, then gmres_m
    const auto a = convdiff(N);
    std::vector<double> ones(a.n, 1.0), b(a.n);
    ktune::spmv_ref(a, ones, b);
    ktune::KrylovConfig cfg;
    cfg.restart_m = 30;
    cfg.m_max = 30;
    cfg.tol = 1e-8;
    cfg.max_iters = 3000;
    for (int stable = 1; stable >= 0; --stable) {
        const int workers = 8;
        bool forced_ref = false, forced_gpu = false;
        ktune::SelectOptions topt_ref;
        ktb_ref::SelectOptions topt_gpu;
        long long ref_its = 0, gpu_its = 0, gpu_calls = 0;
        double gpu_res = 1.0;
        {
            META_CHOICE_SEQUENCE(ktune, a, workers, stable, ktune::UnsymKernel::u1_row, 0,
                                 topt_ref, forced_ref, op, engine)
            ref_its = ktune::gmres_m(op, b, cfg).iterations;
        }
        {
            META_CHOICE_SEQUENCE(ktb_ref, a, workers, stable, ktb_ref::UnsymKernel::u1_row, 0,
                                 topt_gpu, forced_gpu, op, engine)
            const ktune::LinOp kop = op;
            const auto r = ktune::gmres_m(kop, b, cfg);
            gpu_its = r.iterations;
            gpu_res = ktune::true_residual_linear(a, r.x, b);
            gpu_calls = engine.calls();
            if (!r.converged || gpu_res >= cfg.tol) fail |= 1;
        }
        if (std::llabs(gpu_its - ref_its) > 2) fail |= 1;
        std::printf("{\"meta_%s\": {\"ref_iterations\": %lld, \"gpu_iterations\": %lld, "
                    "\"gpu_true_residual\": %.3e, \"engine_calls\": %lld}}\n",
                    stable ? "stable" : "select", ref_its, gpu_its, gpu_res, gpu_calls);
    }

    // ---- 2 + 3: every kernel and artefact on the reference's own generators
    const auto sk = ktune::gen_skewed_rows(3000, 5);
    const std::vector<const ktune::CsrMatrix*> mats = {&a, &sk};
    for (const auto* mp : mats) {
        const auto& m = *mp;
        std::vector<double> x = ktune::detail::seeded_vector(m.n, 3), y(m.n), yref(m.n);
        ktune::spmv_ref(m, x, yref);
        ktb_ref::WorkerPool gpool(4);
        ktune::WorkerPool rpool(4);
        for (int P : {1, 3, 8, 148})
            for (auto s : {0, 1}) {
                const auto g = ktb_ref::build_row_partition(
                    m.row_ptr, P, s ? ktb_ref::PartitionScheme::nnz_balanced
                                    : ktb_ref::PartitionScheme::row_based);
                const auto r = ktune::build_row_partition(
                    m.row_ptr, P, s ? ktune::PartitionScheme::nnz_balanced
                                    : ktune::PartitionScheme::row_based);
                if (g.boundaries != r.boundaries || g.num_workers != r.num_workers) fail |= 4;
            }
        for (ktune::index_t jl : {1, 8, 64, 256}) {
            const auto g = ktb_ref::build_bss_plan(m, jl);
            const auto r = ktune::build_bss_plan(m, jl);
            if (g.jl != r.jl || g.slice_start != r.slice_start || g.slice_len != r.slice_len ||
                g.slice_row != r.slice_row || g.lane_slice_ptr != r.lane_slice_ptr ||
                g.row_slice_ptr != r.row_slice_ptr || g.row_start_flag != r.row_start_flag)
                fail |= 4;
        }
        const auto rowp = ktb_ref::build_row_partition(m.row_ptr, 4, ktb_ref::PartitionScheme::row_based);
        const auto nnzp = ktb_ref::build_row_partition(m.row_ptr, 4, ktb_ref::PartitionScheme::nnz_balanced);
        const auto bss = ktb_ref::build_bss_plan(m, 32);
        double w[4];
        for (int k = 0; k < 4; ++k) {
            const auto kern = static_cast<ktb_ref::UnsymKernel>(k);
            std::fill(y.begin(), y.end(), NAN);
            ktb_ref::spmv_unsym(kern, m, k == 0 ? &rowp : &nnzp, k >= 2 ? &bss : nullptr, x, y,
                                gpool);
            w[k] = worst_rel(m, x, y, yref);
            // U1 over the warp-sliced copy (regular rows): bitwise = spmv_ref
            if (k == 0 && mp == &a && y != yref) fail |= 8;
            if (w[k] > 1e-12) fail |= 8;
        }
        std::printf("{\"unsym_n%lld\": {\"u1\": %.3g, \"u2\": %.3g, \"u3\": %.3g, \"u4\": %.3g}}\n",
                    static_cast<long long>(m.n), w[0], w[1], w[2], w[3]);
    }
    {
        const auto s = ktune::gen_poisson2d(150, 120);
        const auto full = ktune::expand_symmetric(s);
        std::vector<double> x = ktune::detail::seeded_vector(s.n, 4), y(s.n), yref(s.n);
        ktune::spmv_ref(full, x, yref);
        ktb_ref::WorkerPool pool(6);
        const auto rowp = ktb_ref::build_row_partition(s.row_ptr, 6, ktb_ref::PartitionScheme::row_based);
        const auto nnzp = ktb_ref::build_row_partition(s.row_ptr, 6, ktb_ref::PartitionScheme::nnz_balanced);
        const auto reg = ktb_ref::build_reduction_regions(s, nnzp);
        const auto rreg = ktune::build_reduction_regions(
            s, ktune::build_row_partition(s.row_ptr, 6, ktune::PartitionScheme::nnz_balanced));
        if (reg.lo != rreg.lo || reg.hi != rreg.hi) fail |= 4;
        double w[3];
        for (int k = 0; k < 3; ++k) {
            const auto kern = static_cast<ktb_ref::SymKernel>(k);
            ktb_ref::spmv_sym(kern, s, k == 0 ? rowp : nnzp, k == 2 ? &reg : nullptr, x, y, pool);
            w[k] = worst_rel(full, x, y, yref);
            if (w[k] > 1e-12) fail |= 16;
        }
        // select_spmv_sym + SymEngine, the reference's lanczos on its op
        auto [sc, srep] = ktb_ref::select_spmv_sym(s, pool);
        ktb_ref::SymEngine se(s, sc);
        const ktune::LinOp sop = se.op();
        sop.apply(x, y);
        const double ws = worst_rel(full, x, y, yref);
        if (ws > 1e-12 || sc.regions.num_workers != 6) fail |= 16;
        std::printf("{\"sym\": {\"s1\": %.3g, \"s2\": %.3g, \"s3\": %.3g, \"selected\": \"%s\", "
                    "\"engine\": %.3g}}\n",
                    w[0], w[1], w[2], srep.selected_candidate().name.c_str(), ws);
    }

    // ---- 4: contract errors, same messages as the reference
    {
        std::vector<double> x(a.n), y(a.n), bad(3);
        ktune::WorkerPool rp(2);
        ktb_ref::WorkerPool gp(2);
        const auto r_row = ktune::build_row_partition(a.row_ptr, 2, ktune::PartitionScheme::row_based);
        const auto g_row = ktb_ref::build_row_partition(a.row_ptr, 2, ktb_ref::PartitionScheme::row_based);
        const auto r_other = ktune::build_row_partition(sk.row_ptr, 2, ktune::PartitionScheme::row_based);
        const auto g_other = ktb_ref::build_row_partition(sk.row_ptr, 2, ktb_ref::PartitionScheme::row_based);
        struct Case {
            std::string ref, gpu;
        };
        std::vector<Case> cases = {
            {message_of([&] { ktune::spmv_unsym(ktune::UnsymKernel::u1_row, a, &r_row, nullptr, bad, y, rp); }),
             message_of([&] { ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u1_row, a, &g_row, nullptr, bad, y, gp); })},
            {message_of([&] { ktune::spmv_unsym(ktune::UnsymKernel::u1_row, a, nullptr, nullptr, x, y, rp); }),
             message_of([&] { ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u1_row, a, nullptr, nullptr, x, y, gp); })},
            {message_of([&] { ktune::spmv_unsym(ktune::UnsymKernel::u2_nnz, a, &r_row, nullptr, x, y, rp); }),
             message_of([&] { ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u2_nnz, a, &g_row, nullptr, x, y, gp); })},
            {message_of([&] { ktune::spmv_unsym(ktune::UnsymKernel::u1_row, a, &r_other, nullptr, x, y, rp); }),
             message_of([&] { ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u1_row, a, &g_other, nullptr, x, y, gp); })},
            {message_of([&] { ktune::spmv_unsym(ktune::UnsymKernel::u3_bss, a, nullptr, nullptr, x, y, rp); }),
             message_of([&] { ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u3_bss, a, nullptr, nullptr, x, y, gp); })},
            {message_of([&] { ktune::WorkerPool p(0); }), message_of([&] { ktb_ref::WorkerPool p(0); })},
            {message_of([&] { ktune::build_row_partition(a.row_ptr, 0, ktune::PartitionScheme::row_based); }),
             message_of([&] { ktb_ref::build_row_partition(a.row_ptr, 0, ktb_ref::PartitionScheme::row_based); })},
            {message_of([&] { ktune::CsrMatrix e; e.row_ptr = {0}; ktune::select_spmv_unsym(e, rp); }),
             message_of([&] { ktune::CsrMatrix e; e.row_ptr = {0}; ktb_ref::select_spmv_unsym(e, gp); })},
        };
        int same = 0;
        for (const auto& c : cases) {
            if (c.ref == c.gpu && c.ref != "<no error>") ++same;
            else std::printf("{\"message_mismatch\": [\"%s\", \"%s\"]}\n", c.ref.c_str(), c.gpu.c_str());
        }
        if (same != static_cast<int>(cases.size())) fail |= 32;
        std::printf("{\"messages\": {\"same\": %d, \"cases\": %zu}}\n", same, cases.size());
    }

    // ---- 5: residency -- repeated calls reuse one device copy and plan
    {
        ktb_ref::WorkerPool gp(4);
        const auto part = ktb_ref::build_row_partition(a.row_ptr, 4, ktb_ref::PartitionScheme::row_based);
        std::vector<double> x = ktune::detail::seeded_vector(a.n, 9), y(a.n);
        const std::size_t before = ktb_ref::detail::cache().entries.size();
        for (int k = 0; k < 200; ++k)
            ktb_ref::spmv_unsym(ktb_ref::UnsymKernel::u1_row, a, &part, nullptr, x, y, gp);
        const std::size_t after = ktb_ref::detail::cache().entries.size();
        if (after != before) fail |= 64;
        std::printf("{\"residency\": {\"device_matrices_before\": %zu, \"after_200_calls\": %zu}}\n",
                    before, after);
    }
    std::printf("{\"ok\": %s, \"fail_mask\": %d}\n", fail ? "false" : "true", fail);
    return fail ? 1 : 0;
}
