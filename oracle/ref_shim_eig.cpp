// TEST INFRASTRUCTURE: extern "C" wrapper around the UNMODIFIED reference's
// restarted Lanczos (lanczos.hpp:54-199) for the parity tests of
// paper_2405_01599_b200.krylov.lanczos_restarted_dist. Separate library
// because it needs a real LAPACKE_dsteqr (dense_eig.hpp:22-35): linked by
// oracle/Makefile against the OpenBLAS the python env bundles.
#include <cstdint>
#include <cstring>
#include <string>

#include "ktune/lanczos.hpp"

using namespace ktune;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* kre_last_error() { return g_err.c_str(); }

// Sym storage (diag + upper, SymCsrMatrix) -> the reference's overload on
// symmetric storage (expand + sequential operator, lanczos.hpp:195-199).
int kre_lanczos(int64_t n, const int64_t* rp, const int64_t* ci, const double* v, int64_t k,
                int64_t m, double tol, int64_t max_iters, int ortho_kind, uint64_t seed,
                double* eigenvalues, double* residuals, int64_t* nfound, int64_t* iterations,
                int64_t* restarts, int* converged) {
    try {
        SymCsrMatrix a;
        a.n = n;
        a.row_ptr.assign(rp, rp + n + 1);
        a.col_idx.assign(ci, ci + rp[n]);
        a.values.assign(v, v + rp[n]);
        a.validate();
        KrylovConfig cfg;
        cfg.restart_m = m;
        cfg.m_max = m;
        cfg.tol = tol;
        cfg.max_iters = max_iters;
        cfg.max_time = 1e30;
        cfg.ortho.kind = static_cast<OrthoKind>(ortho_kind);
        cfg.seed = seed;
        const EigenResult r = lanczos_restarted(a, k, cfg);
        *nfound = static_cast<int64_t>(r.eigenvalues_re.size());
        for (std::size_t i = 0; i < r.eigenvalues_re.size(); ++i) {
            eigenvalues[i] = r.eigenvalues_re[i];
            residuals[i] = r.residuals[i];
        }
        *iterations = r.iterations;
        *restarts = static_cast<int64_t>(r.restarts.size());
        *converged = r.converged ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
