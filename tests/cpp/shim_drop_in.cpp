// Drop-in demonstration (TEST): the reference's own solvers and SpMV entry
// points, compiled from the unmodified reference headers, running on the
// B200 engine through include/ktune_b200.hpp. Built by tests/cpp/Makefile
// where /root/reference exists; run by tests/test_cpp_shim.py on a GPU.
//
// 1. config-5 recipe (7-pt convection-diffusion) at N^3: ktune::gmres_m with
//    the reference operator (make_ref_op) vs. with ktb_cpp::UnsymEngine::op()
//    -> same iteration count (+-2) and converged true residual < tol.
// 2. ktune::gen_poisson2d (SymCsrMatrix): ktb_cpp::select_spmv_sym winner vs
//    ktune::spmv_ref(ktune::expand_symmetric(A)).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "ktune/ktune.hpp"
#include "ktune_b200.hpp"

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

int main(int argc, char** argv) {
    const ktune::index_t N = argc > 1 ? std::atoll(argv[1]) : 32;
    int fail = 0;
    // ---- 1: GMRES(30) through the engine's LinOp
    const auto a = convdiff(N);
    std::vector<double> ones(a.n, 1.0), b(a.n);
    ktune::spmv_ref(a, ones, b);
    ktune::KrylovConfig cfg;
    cfg.restart_m = 30;
    cfg.m_max = 30;
    cfg.tol = 1e-8;
    cfg.max_iters = 3000;
    const auto ref = ktune::gmres_m(a, b, cfg);
    auto [choice, report] = ktb_cpp::select_spmv_unsym(a);
    ktb_cpp::UnsymEngine eng(choice);
    const ktune::LinOp op = eng.op();
    const auto gpu = ktune::gmres_m(op, b, cfg);
    const double true_res = ktune::true_residual_linear(a, gpu.x, b);
    std::printf("{\"gmres\": {\"n\": %lld, \"kernel\": \"%s\", \"ref_iterations\": %lld, "
                "\"gpu_iterations\": %lld, \"ref_residual\": %.17g, \"gpu_true_residual\": %.17g, "
                "\"gpu_converged\": %d, \"spmv_calls\": %lld, \"max_executions\": %d}}\n",
                static_cast<long long>(a.n), report.selected_candidate().name.c_str(),
                static_cast<long long>(ref.iterations), static_cast<long long>(gpu.iterations),
                ref.true_residual, true_res, gpu.converged ? 1 : 0,
                static_cast<long long>(eng.calls()), report.max_executions());
    if (!gpu.converged || true_res >= cfg.tol || std::llabs(gpu.iterations - ref.iterations) > 2)
        fail = 1;
    if (report.max_executions() > 4) fail = 1;

    // ---- 2: symmetric selection on a reference SymCsrMatrix
    const auto s = ktune::gen_poisson2d(300, 200);
    auto [schoice, srep] = ktb_cpp::select_spmv_sym(s);
    std::vector<double> x = ktune::detail::seeded_vector(s.n, 7), y(s.n), yref(s.n);
    schoice.plan->apply(x, y);
    const auto full = ktune::expand_symmetric(s);
    ktune::spmv_ref(full, x, yref);
    double worst = 0.0;
    for (ktune::index_t i = 0; i < s.n; ++i) {
        double absax = 0.0;
        for (auto k = full.row_ptr[i]; k < full.row_ptr[i + 1]; ++k)
            absax += std::abs(full.values[k] * x[full.col_idx[k]]);
        const double e = std::abs(y[i] - yref[i]);
        if (e > 1e-12 * absax) fail = 1;
        worst = std::max(worst, absax > 0 ? e / absax : e);
    }
    std::printf("{\"sym\": {\"n\": %lld, \"kernel\": \"%s\", \"worst_rel\": %.3g}}\n",
                static_cast<long long>(s.n), srep.selected_candidate().name.c_str(), worst);
    // ---- 3: contract errors keep the reference wording
    try {
        std::vector<double> bad(3);
        choice.plan->apply(bad, bad);
        fail = 1;
    } catch (const ktb_cpp::Error& e) {
        if (std::string(e.what()) != "spmv: dimension mismatch") fail = 1;
    }
    std::printf("{\"ok\": %s}\n", fail ? "false" : "true");
    return fail;
}
