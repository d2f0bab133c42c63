// Multi-GPU data plane from C++ through the C ABI only (TEST): no Python, no
// torch, no reference headers -- ktb.h + libktb (which loads NCCL itself).
//
// 1. The real NCCL communicator at world 1 (ktb_comm_id / ktb_comm_create):
//    the config-4-shaped halo operator on a 64x48x40 stencil against a host
//    CRS product, device-pointer and host-chunked forms.
// 2. Three ranks in one process over the loopback transport (one std::thread
//    per rank, the exchange matched on the host): ktb_halo_create_stencil7
//    and ktb_dist_connect / ktb_dist_spmv on a banded matrix, every row
//    against the host product.
// Prints one JSON line per part; exit code 0 when every row matches.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "ktb.h"

#define CHECK(x)                                                                   \
    do {                                                                           \
        if ((x) != KTB_OK) {                                                       \
            std::printf("{\"error\": \"%s: %s\"}\n", #x, ktb_last_error());      \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

struct Csr {
    int64_t n = 0;
    std::vector<int64_t> rp{0}, ci;
    std::vector<double> v;
};

static Csr stencil7(int64_t nx, int64_t ny, int64_t nz) {
    Csr a;
    a.n = nx * ny * nz;
    for (int64_t z = 0; z < nz; ++z)
        for (int64_t y = 0; y < ny; ++y)
            for (int64_t x = 0; x < nx; ++x) {
                const int64_t i = (z * ny + y) * nx + x;
                auto put = [&](int64_t j, double val) {
                    a.ci.push_back(j);
                    a.v.push_back(val);
                };
                if (z > 0) put(i - nx * ny, -1.0);
                if (y > 0) put(i - nx, -1.0);
                if (x > 0) put(i - 1, -1.0);
                put(i, 6.0);
                if (x < nx - 1) put(i + 1, -1.0);
                if (y < ny - 1) put(i + nx, -1.0);
                if (z < nz - 1) put(i + nx * ny, -1.0);
                a.rp.push_back(static_cast<int64_t>(a.ci.size()));
            }
    return a;
}

static std::vector<double> seeded(int64_t n, uint64_t seed) {  // any fixed vector
    std::vector<double> x(n);
    uint64_t s = seed * 0x9e3779b97f4a7c15ull + 1;
    for (auto& e : x) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        e = static_cast<double>(s >> 11) / 9007199254740992.0 - 0.5;
    }
    return x;
}

static std::vector<double> host_spmv(const Csr& a, const std::vector<double>& x) {
    std::vector<double> y(a.n);
    for (int64_t i = 0; i < a.n; ++i) {
        double s = 0.0;
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) s += a.v[k] * x[a.ci[k]];
        y[i] = s;
    }
    return y;
}

static bool close_rows(const Csr& a, const std::vector<double>& x, const double* y,
                       const std::vector<double>& ref, int64_t r0, int64_t r1) {
    for (int64_t i = r0; i < r1; ++i) {
        double absax = 0.0;
        for (int64_t k = a.rp[i]; k < a.rp[i + 1]; ++k) absax += std::fabs(a.v[k] * x[a.ci[k]]);
        if (std::fabs(y[i - r0] - ref[i]) > 1e-12 * absax) return false;
    }
    return true;
}

int main() {
    int fails = 0;
    // ---- 1: NCCL at world 1
    {
        const int64_t nx = 64, ny = 48, nz = 40;
        const Csr a = stencil7(nx, ny, nz);
        const auto x = seeded(a.n, 4);
        const auto ref = host_spmv(a, x);
        uint8_t id[KTB_COMM_ID_BYTES];
        CHECK(ktb_comm_id(id));
        ktb_comm* comm = nullptr;
        CHECK(ktb_comm_create(id, 1, 0, 0, &comm));
        int world = 0, rank = -1, dev = -1, ver = 0, nccl = 0;
        CHECK(ktb_comm_info(comm, &world, &rank, &dev, &ver, &nccl));
        ktb_halo* h = nullptr;
        CHECK(ktb_halo_create_stencil7(nx, ny, nz, 6.0, -1.0, comm, KTB_U1, 104, &h));
        int64_t n_loc = 0, x_len = 0, off = 0;
        CHECK(ktb_halo_info(h, &n_loc, &x_len, &off, nullptr, nullptr, nullptr, nullptr));
        double *dx = nullptr, *dy = nullptr;
        cudaMalloc(&dx, 8 * x_len);
        cudaMalloc(&dy, 8 * n_loc);
        cudaMemcpy(dx + off, x.data(), 8 * n_loc, cudaMemcpyHostToDevice);
        CHECK(ktb_halo_spmv(h, dx, dy, nullptr));
        std::vector<double> y(n_loc), yh(n_loc);
        cudaMemcpy(y.data(), dy, 8 * n_loc, cudaMemcpyDeviceToHost);
        CHECK(ktb_halo_spmv_host(h, x.data(), yh.data(), 8));
        const bool ok = close_rows(a, x, y.data(), ref, 0, a.n) && y == yh;
        fails += !ok;
        std::printf("{\"nccl_world1\": {\"nccl\": %d, \"version\": %d, \"world\": %d, \"ok\": %s}}\n",
                    nccl, ver, world, ok ? "true" : "false");
        cudaFree(dx);
        cudaFree(dy);
        CHECK(ktb_halo_destroy(h));
        CHECK(ktb_comm_destroy(comm));
    }
    // ---- 2: three ranks over the loopback transport, one thread each
    {
        const int W = 3;
        const int64_t nx = 40, ny = 36, nz = 30;
        const Csr a = stencil7(nx, ny, nz);
        const auto x = seeded(a.n, 7);
        const auto ref = host_spmv(a, x);
        ktb_loopback_world* lw = nullptr;
        CHECK(ktb_loopback_world_create(W, &lw));
        std::vector<int> ok(W, 0), ok2(W, 0);
        std::vector<int64_t> bnd(W + 1);
        for (int r = 0; r <= W; ++r) bnd[r] = a.n * r / W;
        auto rank_main = [&](int r) {
            cudaSetDevice(0);
            ktb_comm* comm = nullptr;
            CHECK(ktb_comm_create_loopback(lw, r, 0, &comm));
            // halo operator: z-slabs
            ktb_halo* h = nullptr;
            CHECK(ktb_halo_create_stencil7(nx, ny, nz, 6.0, -1.0, comm, KTB_U1, 104, &h));
            int64_t n_loc = 0, x_len = 0, off = 0;
            CHECK(ktb_halo_info(h, &n_loc, &x_len, &off, nullptr, nullptr, nullptr, nullptr));
            const int64_t row0 = (r * nz / W) * nx * ny;
            std::vector<double> yh(n_loc);
            CHECK(ktb_halo_spmv_host(h, x.data() + row0, yh.data(), 4));
            ok[r] = close_rows(a, x, yh.data(), ref, row0, row0 + n_loc);
            CHECK(ktb_halo_destroy(h));
            // general split: equal row blocks (not plane-aligned), ghost exchange
            const int64_t r0 = bnd[r], r1 = bnd[r + 1];
            std::vector<int64_t> rp(a.rp.begin() + r0, a.rp.begin() + r1 + 1);
            for (auto& e : rp) e -= a.rp[r0];
            ktb_dist* d = nullptr;
            CHECK(ktb_dist_create(a.n, W, bnd.data(), r, rp.data(), a.ci.data() + a.rp[r0],
                                  a.v.data() + a.rp[r0], &d));
            CHECK(ktb_dist_connect(d, comm, KTB_U1, 104));
            double *dx = nullptr, *dy = nullptr;
            cudaMalloc(&dx, 8 * (r1 - r0));
            cudaMalloc(&dy, 8 * (r1 - r0));
            cudaMemcpy(dx, x.data() + r0, 8 * (r1 - r0), cudaMemcpyHostToDevice);
            cudaStream_t s;
            cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
            CHECK(ktb_dist_spmv(d, dx, dy, s));
            cudaStreamSynchronize(s);
            std::vector<double> y(r1 - r0);
            cudaMemcpy(y.data(), dy, 8 * (r1 - r0), cudaMemcpyDeviceToHost);
            ok2[r] = close_rows(a, x, y.data(), ref, r0, r1);
            cudaFree(dx);
            cudaFree(dy);
            cudaStreamDestroy(s);
            CHECK(ktb_dist_destroy(d));
            CHECK(ktb_comm_destroy(comm));
        };
        std::vector<std::thread> ts;
        for (int r = 0; r < W; ++r) ts.emplace_back(rank_main, r);
        for (auto& t : ts) t.join();
        CHECK(ktb_loopback_world_destroy(lw));
        bool all = true;
        for (int r = 0; r < W; ++r) all = all && ok[r] && ok2[r];
        fails += !all;
        std::printf("{\"loopback_world3\": {\"halo\": [%d, %d, %d], \"dist\": [%d, %d, %d], \"ok\": %s}}\n",
                    ok[0], ok[1], ok[2], ok2[0], ok2[1], ok2[2], all ? "true" : "false");
    }
    std::printf("{\"ok\": %s}\n", fails ? "false" : "true");
    return fails ? 1 : 0;
}
