// ktb_dist.cu -- general row-block sharding of an arbitrary CRS across ranks
// (the reference has no distributed path).
//
// Rank r of P owns rows [b_r, b_{r+1}) (any boundaries; the framework uses
// the reference's NNZ_BALANCED build_row_partition, partition.hpp:28-55) and
// the x entries with the same indices. Its rows split into
//   A_d  n_loc x n_loc, the owned columns renumbered c - b_r: a plain square
//        ktb_matrix, so every unsymmetric kernel and the selector apply;
//   A_o  the rows that touch other ranks' columns, compressed: row ids,
//        CRS over the ghost index space [0, n_ghost).
// Ghost columns are sorted ascending, hence grouped by owner rank in rank
// order: the receive buffer of one exchange IS the ghost vector. Per apply:
//   pack   send_buf[k] = x_owned[send_idx[k]]        (k_pack)
//   A_d x  on the compute stream while the exchange runs
//   y += A_o x_ghost                                  (k_ghost_acc)
// All host logic (ghost discovery, owner grouping, renumbering, send lists)
// is plain C++ with no device calls until ktb_dist_upload, so the protocol
// is testable on CPU ranks (gloo).
#include <algorithm>
#include <memory>
#include <vector>

#include "ktb_internal.cuh"

namespace ktb {

namespace {

__global__ void k_pack(int64_t count, const int32_t* __restrict__ idx,
                       const double* __restrict__ x, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __ldg(x + __ldg(idx + i));
}

// y[rows[g]] += sum_k A_o[g, k] * xg[k]; V lanes per compressed row.
template <int V>
__global__ void __launch_bounds__(256) k_ghost_acc(int32_t m, const int32_t* __restrict__ rows,
                                                   const int32_t* __restrict__ rp,
                                                   const int32_t* __restrict__ ci,
                                                   const double* __restrict__ v,
                                                   const double* __restrict__ xg,
                                                   double* __restrict__ y) {
    const int sub = threadIdx.x & (V - 1);
    const int64_t g = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / V;
    double s = 0.0;
    if (g < m) {
        const int32_t e = __ldg(rp + g + 1);
        for (int32_t k = __ldg(rp + g) + sub; k < e; k += V) s += __ldg(v + k) * __ldg(xg + __ldg(ci + k));
    }
    if (V > 1) {
#pragma unroll
        for (int o = V / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, V);
    }
    if (sub == 0 && g < m) y[__ldg(rows + g)] += s;
}

template <typename T>
void upload(DBuf<T>& d, const std::vector<T>& h) {
    d.alloc(h.size());
    if (!h.empty()) KTB_CUDA(cudaMemcpy(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice));
}

}  // namespace

ktb_dist* dist_create(int64_t n_global, int world, const int64_t* bnd, int rank,
                      const int64_t* rp, const int64_t* ci, const double* v) {
    require(world >= 1 && rank >= 0 && rank < world, "dist: bad rank/world");
    require(bnd != nullptr && bnd[0] == 0 && bnd[world] == n_global,
            "dist: boundaries must span [0, n)");
    for (int p = 0; p < world; ++p) require(bnd[p] <= bnd[p + 1], "dist: boundaries not nondecreasing");
    require(n_global < (int64_t(1) << 31) - 1, "dist: n >= 2^31 does not fit the int32 layout");
    auto d = std::make_unique<ktb_dist>();
    d->n_global = n_global;
    d->world = world;
    d->rank = rank;
    d->bnd.assign(bnd, bnd + world + 1);
    d->row0 = bnd[rank];
    d->n_loc = bnd[rank + 1] - bnd[rank];
    const int64_t n = d->n_loc, r0 = d->row0, r1 = r0 + n;
    require(rp != nullptr && rp[0] == 0, "csr: row_ptr[0] != 0");
    const int64_t nnz = rp[n];
    require(nnz < (int64_t(1) << 31) - 1, "dist: local nnz >= 2^31");
    for (int64_t i = 0; i < n; ++i) {  // csr.hpp:38-54 on the local rows
        require(rp[i] <= rp[i + 1], "csr: row_ptr not nondecreasing");
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            require(ci[k] >= 0 && ci[k] < n_global, "csr: column index out of range");
            if (k > rp[i]) require(ci[k - 1] < ci[k], "csr: columns not strictly increasing");
        }
    }
    // ghost columns: sorted, unique, hence grouped by owner in rank order
    for (int64_t k = 0; k < nnz; ++k)
        if (ci[k] < r0 || ci[k] >= r1) d->ghosts.push_back(ci[k]);
    std::sort(d->ghosts.begin(), d->ghosts.end());
    d->ghosts.erase(std::unique(d->ghosts.begin(), d->ghosts.end()), d->ghosts.end());
    d->recv_counts.assign(world, 0);
    for (int64_t c : d->ghosts) {
        const int owner =
            static_cast<int>(std::upper_bound(d->bnd.begin(), d->bnd.end(), c) - d->bnd.begin()) - 1;
        ++d->recv_counts[owner];
    }
    d->d_rp.assign(n + 1, 0);
    d->o_rp.push_back(0);
    for (int64_t i = 0; i < n; ++i) {
        int64_t nd = 0, no = 0;
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t c = ci[k];
            if (c >= r0 && c < r1) {
                d->d_ci.push_back(static_cast<int32_t>(c - r0));
                d->d_v.push_back(v[k]);
                ++nd;
            } else {
                const int64_t gi =
                    std::lower_bound(d->ghosts.begin(), d->ghosts.end(), c) - d->ghosts.begin();
                d->o_ci.push_back(static_cast<int32_t>(gi));
                d->o_v.push_back(v[k]);
                ++no;
            }
        }
        d->d_rp[i + 1] = d->d_rp[i] + static_cast<int32_t>(nd);
        if (no) {
            d->o_rows.push_back(static_cast<int32_t>(i));
            d->o_rp.push_back(d->o_rp.back() + static_cast<int32_t>(no));
        }
    }
    return d.release();
}

void dist_set_sends(ktb_dist* d, const int64_t* counts, const int64_t* cols) {
    int64_t total = 0;
    for (int p = 0; p < d->world; ++p) {
        require(counts[p] >= 0, "dist: negative send count");
        require(p != d->rank || counts[p] == 0, "dist: a rank does not send to itself");
        total += counts[p];
    }
    d->send_counts.assign(counts, counts + d->world);
    d->send_idx.resize(total);
    for (int64_t k = 0; k < total; ++k) {
        require(cols[k] >= d->row0 && cols[k] < d->row0 + d->n_loc,
                "dist: send column not owned by this rank");
        d->send_idx[k] = static_cast<int32_t>(cols[k] - d->row0);
    }
    d->sends_set = true;
    if (d->device >= 0) {
        DeviceGuard g(d->device);
        upload(d->dev_send, d->send_idx);
    }
}

ktb_matrix* make_device_matrix(int64_t n, int64_t ncols, const std::vector<int32_t>& rp,
                               const std::vector<int32_t>& ci, const std::vector<double>& v,
                               int kind, int device) {
    DeviceGuard g(device);
    auto m = std::make_unique<ktb_matrix>();
    m->device = device;
    KTB_CUDA(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
    m->n = n;
    m->ncols = ncols;
    m->nnz = rp[n];
    m->kind = kind;
    for (int64_t i = 0; i < n; ++i) {
        m->max_row_nnz = std::max<int64_t>(m->max_row_nnz, rp[i + 1] - rp[i]);
        if (rp[i + 1] > rp[i]) m->bandwidth = std::max<int64_t>(m->bandwidth, ci[rp[i + 1] - 1] - i);
    }
    upload(m->row_ptr, rp);
    upload(m->col, ci);
    upload(m->val, v);
    return m.release();
}

void dist_upload(ktb_dist* d, int device) {
    DeviceGuard g(device);
    delete d->local;
    d->local = nullptr;
    d->device = device;
    d->local = make_device_matrix(d->n_loc, d->n_loc, d->d_rp, d->d_ci, d->d_v, KTB_GENERAL, device);
    upload(d->dev_orows, d->o_rows);
    upload(d->dev_orp, d->o_rp);
    upload(d->dev_oci, d->o_ci);
    upload(d->dev_ov, d->o_v);
    if (d->sends_set) upload(d->dev_send, d->send_idx);
    const double mean =
        d->o_rows.empty() ? 1.0 : static_cast<double>(d->o_v.size()) / d->o_rows.size();
    int lanes = 1;
    while (lanes < 32 && lanes < mean) lanes <<= 1;
    d->lanes = lanes;
}

void dist_pack(const ktb_dist* d, const double* x_owned, double* send_buf, cudaStream_t s) {
    require(d->device >= 0, "dist: not uploaded");
    require(d->sends_set, "dist: send lists not set");
    const int64_t count = static_cast<int64_t>(d->send_idx.size());
    if (!count) return;
    DeviceGuard g(d->device);
    const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(count, 256), 4 * kNumSMs));
    k_pack<<<grid, 256, 0, s>>>(count, d->dev_send.p, x_owned, send_buf);
    KTB_LAUNCH();
}

void dist_ghost_spmv(const ktb_dist* d, const double* x_ghost, double* y, cudaStream_t s) {
    require(d->device >= 0, "dist: not uploaded");
    const int64_t m = static_cast<int64_t>(d->o_rows.size());
    if (!m) return;
    DeviceGuard g(d->device);
    const int grid = ceil_div(m * d->lanes, 256);
    const int32_t mm = static_cast<int32_t>(m);
    switch (d->lanes) {
#define KTB_GA(V)                                                                              \
    case V:                                                                                    \
        k_ghost_acc<V><<<grid, 256, 0, s>>>(mm, d->dev_orows.p, d->dev_orp.p, d->dev_oci.p,    \
                                            d->dev_ov.p, x_ghost, y);                          \
        break;
        KTB_GA(1)
        KTB_GA(2)
        KTB_GA(4)
        KTB_GA(8)
        KTB_GA(16)
        KTB_GA(32)
#undef KTB_GA
        default: throw Invalid("dist: bad lane count");
    }
    KTB_LAUNCH();
}

}  // namespace ktb
