// ktb_gen.cu -- config-3 generator: irregular power-law CRS (BASELINE.json
// configs[2]; recipe fixed in DESIGN.md "config 3 recipe").
//
// Counter-based so that every implementation (this one, tests/matgen.py)
// produces identical bytes:
//   mix(z)      splitmix64 finalizer (lanczos.hpp:21-25)
//   U(s, k)     (mix(s + (k+1)*G) >> 11) * 2^-53            in [0, 1)
//   s_i         mix(seed + (i+1) * H)                         per-row stream
//   empty       U(s_i, 0) < empty_frac
//   L           largest integer with L^(1/alpha') ... i.e. floor((1-u)^(-1/alpha))
//               with u = U(s_i, 1), computed exactly: L^3 * (1-u)^2 <= 1
//               for alpha = 1.5, capped at max_len
//   L'          clamp(floor(L * target / sum(L) + 0.5), 1, max_len)
//   columns     candidates c_k = ((mix(s_i + (k+3)*G) >> 32) * n) >> 32,
//               k = 0, 1, ...; the first L' distinct, sorted ascending
//   values      2 * U(s_i ^ V, p) - 1 for sorted position p
#include <algorithm>
#include <cmath>
#include <thread>
#include <vector>

#include "ktb_internal.cuh"

namespace ktb {

namespace {
constexpr uint64_t kG = 0x9e3779b97f4a7c15ull;
constexpr uint64_t kH = 0xd1b54a32d192ed03ull;
constexpr uint64_t kV = 0xa5a5a5a5a5a5a5a5ull;

inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
inline double unif(uint64_t s, uint64_t k) {
    return static_cast<double>(mix(s + (k + 1) * kG) >> 11) * (1.0 / 9007199254740992.0);
}
// floor((1-u)^(-2/3)) exactly: largest L >= 1 with L^3 * (1-u)^2 <= 1
inline int64_t pareto15(double u, int64_t cap) {
    const volatile double w1 = 1.0 - u;  // exact
    const volatile double w = w1 * w1;    // one rounding, no contraction
    int64_t L = static_cast<int64_t>(std::floor(std::pow(w1, -2.0 / 3.0)));
    L = std::max<int64_t>(1, std::min<int64_t>(L, cap + 1));
    auto le1 = [&](int64_t l) {
        const volatile double l3 = static_cast<double>(l) * static_cast<double>(l) *
                                   static_cast<double>(l);  // exact below 2^53
        const volatile double p = l3 * w;
        return p <= 1.0;
    };
    while (L <= cap && le1(L + 1)) ++L;
    while (L > 1 && !le1(L)) --L;
    return std::min<int64_t>(L, cap);
}
}  // namespace

template <typename F>
static void parallel_rows(int64_t n, F&& f) {
    const int T = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) f(i);
        });
    for (auto& x : th) x.join();
}

// Host part: row_ptr (n+1), then columns / values. Deterministic for any
// thread count (every row has its own counter-based stream).
void powerlaw_host(int64_t n, uint64_t seed, int64_t target, double empty_frac,
                   int64_t max_len, std::vector<int64_t>& rp, std::vector<int32_t>* col,
                   std::vector<double>* val) {
    require(n >= 1 && n < (int64_t(1) << 31) - 1, "powerlaw: bad n");
    require(target >= 1 && max_len >= 1, "powerlaw: bad target/max_len");
    std::vector<int64_t> L(n);
    parallel_rows(n, [&](int64_t i) {
        const uint64_t s = mix(seed + static_cast<uint64_t>(i + 1) * kH);
        L[i] = unif(s, 0) < empty_frac ? 0 : pareto15(unif(s, 1), max_len);
    });
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) total += L[i];
    require(total > 0, "powerlaw: every row is empty");
    rp.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
        int64_t l = 0;
        if (L[i] > 0) {
            const volatile double t = static_cast<double>(L[i]) * static_cast<double>(target);
            const volatile double q = t / static_cast<double>(total);
            l = static_cast<int64_t>(std::floor(q + 0.5));
            l = std::max<int64_t>(1, std::min<int64_t>(l, std::min(max_len, n)));
        }
        rp[i + 1] = rp[i] + l;
    }
    if (!col) return;
    const int64_t nnz = rp[n];
    col->resize(nnz);
    val->resize(nnz);
    parallel_rows(n, [&](int64_t i) {
        const int64_t l = rp[i + 1] - rp[i];
        if (!l) return;
        const uint64_t s = mix(seed + static_cast<uint64_t>(i + 1) * kH);
        // first l distinct candidates in k order: the distinct values among
        // k < l, then further candidates k = l, l+1, ... not yet taken
        auto cand = [&](uint64_t k) {
            const uint64_t z = mix(s + (k + 3) * kG);
            return static_cast<int32_t>(((z >> 32) * static_cast<uint64_t>(n)) >> 32);
        };
        std::vector<int32_t> buf(l);
        for (int64_t t = 0; t < l; ++t) buf[t] = cand(static_cast<uint64_t>(t));
        std::sort(buf.begin(), buf.end());
        buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
        for (uint64_t k = static_cast<uint64_t>(l); static_cast<int64_t>(buf.size()) < l; ++k) {
            const int32_t cnd = cand(k);
            auto it = std::lower_bound(buf.begin(), buf.end(), cnd);
            if (it == buf.end() || *it != cnd) buf.insert(it, cnd);
        }
        const uint64_t sv = s ^ kV;
        for (int64_t p = 0; p < l; ++p) {
            (*col)[rp[i] + p] = buf[p];
            (*val)[rp[i] + p] = 2.0 * unif(sv, static_cast<uint64_t>(p)) - 1.0;
        }
    });
}

ktb_matrix* gen_powerlaw(int64_t n, uint64_t seed, int64_t target, double empty_frac,
                         int64_t max_len, int device) {
    std::vector<int64_t> rp;
    std::vector<int32_t> col;
    std::vector<double> val;
    powerlaw_host(n, seed, target, empty_frac, max_len, rp, &col, &val);
    const int64_t nnz = rp[n];
    require(nnz < (int64_t(1) << 31) - 1, "powerlaw: nnz >= 2^31");
    DeviceGuard guard(device);
    auto* m = new ktb_matrix();
    try {
        m->device = device;
        KTB_CUDA(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
        m->n = n;
        m->ncols = n;
        m->nnz = nnz;
        m->kind = KTB_GENERAL;
        std::vector<int32_t> rp32(n + 1);
        for (int64_t i = 0; i <= n; ++i) rp32[i] = static_cast<int32_t>(rp[i]);
        m->row_ptr.alloc(n + 1);
        m->col.alloc(nnz);
        m->val.alloc(nnz);
        KTB_CUDA(cudaMemcpy(m->row_ptr.p, rp32.data(), 4 * (n + 1), cudaMemcpyHostToDevice));
        KTB_CUDA(cudaMemcpy(m->col.p, col.data(), 4 * nnz, cudaMemcpyHostToDevice));
        KTB_CUDA(cudaMemcpy(m->val.p, val.data(), 8 * nnz, cudaMemcpyHostToDevice));
        compute_matrix_stats(m, 0);
    } catch (...) {
        delete m;
        throw;
    }
    return m;
}

}  // namespace ktb
