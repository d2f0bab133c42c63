// ktb_comm.cu -- native multi-GPU data plane of libktb: the communicator
// (NCCL over NVLink/NVSwitch), the halo row-block operator of config 4 and the
// ghost exchange of the general row-block split.
//
// The reference is a single-process OpenMP library: nothing here
// replaces reference code; this is the B200 framework's scale-out of
// spmv_unsym (spmv.hpp:111-126). Each rank owns a contiguous row block of A
// and the same entries of x and y; y stays row-sharded, so the only data-plane
// traffic per SpMV is the x entries other ranks' rows read:
//   * halo operator (ktb_halo_*): the local matrix's columns are
//     [halo_lo | owned | halo_hi] (config 4's z-slab: one plane each side).
//     One NCCL group per apply sends the owned edges to the neighbours and
//     receives the halos straight into the caller's x buffer (no packing),
//     on a communication stream, while the interior rows (no halo columns)
//     run on the caller's stream; the boundary rows run after an event wait.
//   * general split (ktb_dist_connect / ktb_dist_spmv): ghost lists are
//     exchanged once (all-gather of counts, point-to-point lists); per apply
//     pack -> NCCL send/recv of the ghosts -> A_d x (overlapped) -> y += A_o xg.
//
// Transports. ktb_comm is an interface with two implementations:
//   * NCCL (ktb_comm_create / ktb_comm_wrap): the product path.
//   * loopback (ktb_comm_create_loopback): W ranks inside ONE process, each
//     driven by its own host thread, messages matched on the host and moved
//     with device-to-device copies. It exists so the exact offsets, peers and
//     ordering of the code above can be checked against the oracle on a
//     single GPU: the ranks never wait on each other inside a kernel (the
//     rendezvous is a host condition variable), so this is not the "ranks on
//     one GPU spinning on each other" anti-pattern.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "ktb_internal.cuh"

namespace ktb {
void plan_run(ktb_plan* p, const double* x, double* y, int64_t r0, int64_t r1);
ktb_matrix* matrix_slice(const ktb_matrix* m, int64_t r0, int64_t r1);
ktb_matrix* gen_stencil7(int64_t nx, int64_t ny, int64_t nz, int64_t z0, int64_t z1, bool slab,
                         double diag, double off_z, double c_xm, double c_xp, int device);
ktb_plan* plan_create_internal(ktb_matrix* m, int kernel, int64_t param, int workers,
                               cudaStream_t stream);
void dist_pack(const ktb_dist* d, const double* x_owned, double* send_buf, cudaStream_t s);
void dist_ghost_spmv(const ktb_dist* d, const double* x_ghost, double* y, cudaStream_t s);
void dist_set_sends(ktb_dist* d, const int64_t* counts, const int64_t* cols);
void dist_upload(ktb_dist* d, int device);
ktb_matrix* matrix_create_rect(int64_t n, int64_t ncols, const int64_t* rp, const int64_t* ci,
                               const double* v, int device);
}  // namespace ktb

// --------------------------------------------------------------- transport
struct ktb_comm {
    int world = 1, rank = 0, device = 0;
    virtual ~ktb_comm() = default;
    virtual const char* kind() const = 0;
    // point-to-point, grouped: every op between group_start and group_end is
    // matched as one unit (ncclGroupStart/End semantics); byte counts
    virtual void group_start() = 0;
    virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
    virtual void group_end() = 0;
    // in place, fp64 (KTB_SUM / KTB_MAX)
    virtual void allreduce(double* buf, int64_t count, int op, cudaStream_t s) = 0;
    // recv[r*bytes .. (r+1)*bytes) = rank r's send (device buffers)
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
};

namespace ktb {
namespace {


// ------------------------------------------------------------ NCCL loader
// libnccl is resolved at the first communicator call, not linked: a process
// that already loaded an NCCL (torch ships its own libnccl.so.2) keeps using
// that copy -- dlopen by soname returns the loaded object -- instead of a
// second, older copy shadowing the symbols torch expects. KTB_NCCL_LIB names
// an explicit library.
struct NcclApi {
#define KTB_NCCL_FN(name) decltype(&::name) name = nullptr;
    KTB_NCCL_FN(ncclGetUniqueId)
    KTB_NCCL_FN(ncclCommInitRank)
    KTB_NCCL_FN(ncclCommDestroy)
    KTB_NCCL_FN(ncclCommCount)
    KTB_NCCL_FN(ncclCommUserRank)
    KTB_NCCL_FN(ncclCommCuDevice)
    KTB_NCCL_FN(ncclGroupStart)
    KTB_NCCL_FN(ncclGroupEnd)
    KTB_NCCL_FN(ncclSend)
    KTB_NCCL_FN(ncclRecv)
    KTB_NCCL_FN(ncclAllReduce)
    KTB_NCCL_FN(ncclAllGather)
    KTB_NCCL_FN(ncclGetErrorString)
    KTB_NCCL_FN(ncclGetLastError)
    KTB_NCCL_FN(ncclGetVersion)
#undef KTB_NCCL_FN
};

const NcclApi& nccl_api() {
    static std::once_flag once;
    static NcclApi api;
    static std::string err;
    std::call_once(once, [] {
        const char* env = std::getenv("KTB_NCCL_LIB");
        void* h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            err = std::string("comm: cannot load NCCL: ") + (e ? e : "libnccl.so.2");
            return;
        }
        bool ok = true;
        auto get = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            ok &= fp != nullptr;
        };
#define KTB_NCCL_GET(name) get(api.name, #name);
        KTB_NCCL_GET(ncclGetUniqueId)
        KTB_NCCL_GET(ncclCommInitRank)
        KTB_NCCL_GET(ncclCommDestroy)
        KTB_NCCL_GET(ncclCommCount)
        KTB_NCCL_GET(ncclCommUserRank)
        KTB_NCCL_GET(ncclCommCuDevice)
        KTB_NCCL_GET(ncclGroupStart)
        KTB_NCCL_GET(ncclGroupEnd)
        KTB_NCCL_GET(ncclSend)
        KTB_NCCL_GET(ncclRecv)
        KTB_NCCL_GET(ncclAllReduce)
        KTB_NCCL_GET(ncclAllGather)
        KTB_NCCL_GET(ncclGetErrorString)
        KTB_NCCL_GET(ncclGetLastError)
        KTB_NCCL_GET(ncclGetVersion)
#undef KTB_NCCL_GET
        if (!ok) {
            err = "comm: libnccl.so.2 lacks a required symbol";
            api = NcclApi{};
        }
    });
    if (!api.ncclSend) throw CudaError(err);
    return api;
}

// ---------------------------------------------------------------- NCCL
void nccl_check(ncclResult_t r, ncclComm_t c, const char* what) {
    if (r == ncclSuccess || r == ncclInProgress) return;
    std::string m = std::string(what) + ": " + nccl_api().ncclGetErrorString(r);
    if (c) {
        const char* last = nccl_api().ncclGetLastError(c);
        if (last && *last) m += std::string(" (") + last + ")";
    }
    throw CudaError(m);
}
#define KTB_NCCL(x, c) ::ktb::nccl_check((x), (c), #x)

struct NcclComm final : ktb_comm {
    ncclComm_t c = nullptr;
    bool own = true;
    const char* kind() const override { return "nccl"; }
    ~NcclComm() override {
        if (own && c) nccl_api().ncclCommDestroy(c);
    }
    void group_start() override { KTB_NCCL(nccl_api().ncclGroupStart(), c); }
    void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
        KTB_NCCL(nccl_api().ncclSend(buf, bytes, ncclInt8, peer, c, s), c);
    }
    void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
        KTB_NCCL(nccl_api().ncclRecv(buf, bytes, ncclInt8, peer, c, s), c);
    }
    void group_end() override { KTB_NCCL(nccl_api().ncclGroupEnd(), c); }
    void allreduce(double* buf, int64_t count, int op, cudaStream_t s) override {
        KTB_NCCL(nccl_api().ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclDouble,
                               op == KTB_MAX ? ncclMax : ncclSum, c, s),
                 c);
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        KTB_NCCL(nccl_api().ncclAllGather(send, recv, bytes, ncclInt8, c, s), c);
    }
};

// ------------------------------------------------------------- loopback
struct LoopWorld {
    int W = 1;
    std::mutex mu;
    std::condition_variable cv;
    struct Msg {
        const void* p;
        size_t bytes;
        uint64_t id;
    };
    std::map<std::pair<int, int>, std::deque<Msg>> box;  // (src, dst) -> FIFO
    std::map<uint64_t, bool> consumed;
    uint64_t next_id = 1;
    // collectives: a generation barrier over W ranks plus per-rank slots
    std::vector<const void*> slot;
    int arrived = 0;
    uint64_t gen = 0;
    explicit LoopWorld(int w) : W(w), slot(w, nullptr) {}
    void barrier(std::unique_lock<std::mutex>& lk) {
        const uint64_t g = gen;
        if (++arrived == W) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct LoopComm final : ktb_comm {
    std::shared_ptr<LoopWorld> w;
    struct Op {
        bool is_send;
        void* p;
        size_t bytes;
        int peer;
        cudaStream_t s;
    };
    std::vector<Op> ops;
    bool in_group = false;
    const char* kind() const override { return "loopback"; }
    void group_start() override {
        ops.clear();
        in_group = true;
    }
    void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
        ops.push_back({true, const_cast<void*>(buf), bytes, peer, s});
        if (!in_group) group_end();
    }
    void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
        ops.push_back({false, buf, bytes, peer, s});
        if (!in_group) group_end();
    }
    void group_end() override {
        in_group = false;
        DeviceGuard g(device);
        // everything enqueued before the ops (x ready, halos free) has finished
        for (const Op& o : ops) KTB_CUDA(cudaStreamSynchronize(o.s));
        std::vector<uint64_t> mine;
        std::unique_lock<std::mutex> lk(w->mu);
        for (const Op& o : ops)
            if (o.is_send) {
                const uint64_t id = w->next_id++;
                w->box[{rank, o.peer}].push_back({o.p, o.bytes, id});
                w->consumed[id] = false;
                mine.push_back(id);
            }
        w->cv.notify_all();
        for (const Op& o : ops) {
            if (o.is_send) continue;
            auto& q = w->box[{o.peer, rank}];
            w->cv.wait(lk, [&] { return !q.empty(); });
            const LoopWorld::Msg m = q.front();
            q.pop_front();
            lk.unlock();
            require(m.bytes == o.bytes, "comm: send/recv size mismatch");
            if (m.bytes) {  // on the op's (non-blocking) stream: never the legacy stream
                KTB_CUDA(cudaMemcpyAsync(o.p, m.p, m.bytes, cudaMemcpyDeviceToDevice, o.s));
                KTB_CUDA(cudaStreamSynchronize(o.s));
            }
            lk.lock();
            w->consumed[m.id] = true;
            w->cv.notify_all();
        }
        // a sender's buffer stays untouched until its receiver has copied it
        w->cv.wait(lk, [&] {
            for (uint64_t id : mine)
                if (!w->consumed[id]) return false;
            return true;
        });
        for (uint64_t id : mine) w->consumed.erase(id);
        ops.clear();
    }
    void allreduce(double* buf, int64_t count, int op, cudaStream_t s) override {
        DeviceGuard g(device);
        KTB_CUDA(cudaStreamSynchronize(s));
        std::unique_lock<std::mutex> lk(w->mu);
        w->slot[rank] = buf;
        w->barrier(lk);
        std::vector<const void*> src = w->slot;
        lk.unlock();
        std::vector<double> acc(count), tmp(count);
        for (int r = 0; r < w->W; ++r) {  // fixed rank order: deterministic
            if (count) {
                KTB_CUDA(cudaMemcpyAsync(tmp.data(), src[r], 8 * count, cudaMemcpyDeviceToHost, s));
                KTB_CUDA(cudaStreamSynchronize(s));
            }
            for (int64_t i = 0; i < count; ++i)
                acc[i] = r == 0 ? tmp[i]
                                : (op == KTB_MAX ? std::max(acc[i], tmp[i]) : acc[i] + tmp[i]);
        }
        lk.lock();
        w->barrier(lk);  // every rank has read every buffer before any is overwritten
        lk.unlock();
        if (count) {
            KTB_CUDA(cudaMemcpyAsync(buf, acc.data(), 8 * count, cudaMemcpyHostToDevice, s));
            KTB_CUDA(cudaStreamSynchronize(s));
        }
    }
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        DeviceGuard g(device);
        KTB_CUDA(cudaStreamSynchronize(s));
        std::unique_lock<std::mutex> lk(w->mu);
        w->slot[rank] = send;
        w->barrier(lk);
        std::vector<const void*> src = w->slot;
        lk.unlock();
        for (int r = 0; r < w->W; ++r)
            if (bytes)
                KTB_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + r * bytes, src[r], bytes,
                                         cudaMemcpyDeviceToDevice, s));
        KTB_CUDA(cudaStreamSynchronize(s));
        lk.lock();
        w->barrier(lk);
    }
};

}  // namespace
}  // namespace ktb

struct ktb_loopback_world {
    std::shared_ptr<ktb::LoopWorld> w;
};

// ------------------------------------------------------------ halo operator
struct ktb_halo {
    ktb_comm* comm = nullptr;
    int device = 0;
    int64_t n = 0, halo_lo = 0, halo_hi = 0, nnz = 0;
    int64_t send_down = 0, send_up = 0;  // owned entries sent to rank-1 / rank+1
    int64_t ib = 0, ie = 0;              // interior rows [ib, ie)
    struct Part {
        int64_t r0, r1;
        ktb_matrix* m;
        ktb_plan* p;
    };
    std::vector<Part> interior, boundary;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    // ktb_halo_spmv_host: device x/y, copy streams, per-chunk events, and per
    // interior row chunk the last x chunk its columns reach
    ktb::DBuf<double> dx, dy;
    cudaStream_t cin = nullptr, cout = nullptr, comp = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_comp;
    cudaEvent_t ev_start = nullptr, ev_bnd = nullptr;
    int chunks = 0;
    // optional per-apply kernel timing on the compute stream (bench roofline):
    // [0,1] around the interior rows, [2,3] around the boundary rows
    bool timing = false;
    cudaEvent_t te[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<int64_t> cb;    // chunk c = owned rows [cb[c], cb[c+1])
    std::vector<int> need;      // interior rows of chunk c need x chunks <= need[c]
    ~ktb_halo() {
        for (auto* v : {&interior, &boundary})
            for (Part& q : *v) {
                delete q.p;
                delete q.m;
            }
        for (auto* v : {&ev_in, &ev_comp})
            for (cudaEvent_t e : *v) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_ready, ev_done, ev_start, ev_bnd, te[0], te[1], te[2], te[3]})
            if (e) cudaEventDestroy(e);
        for (cudaStream_t t : {cs, cin, cout, comp})
            if (t) cudaStreamDestroy(t);
    }
};

namespace ktb {
namespace {

// last row touching the low halo (-1 if none), first row touching the high
// halo (n if none); columns are sorted per row, so a row's extremes are its
// first and last entries
__global__ void k_halo_rows(int64_t n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ col, int64_t lo_end, int64_t hi_begin,
                            long long* last_lo, long long* first_hi) {
    long long ll = -1, fh = n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t a = rp[i], b = rp[i + 1];
        if (b > a) {
            if (col[a] < lo_end) ll = max(ll, static_cast<long long>(i));
            if (col[b - 1] >= hi_begin) fh = min(fh, static_cast<long long>(i));
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        ll = max(ll, __shfl_xor_sync(0xffffffffu, ll, o));
        fh = min(fh, __shfl_xor_sync(0xffffffffu, fh, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(last_lo, ll);
        atomicMin(first_hi, fh);
    }
}

void make_events(cudaStream_t* cs, cudaEvent_t* a, cudaEvent_t* b) {
    int lo = 0, hi = 0;
    KTB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // the exchange is latency-critical: highest priority so its copies are
    // scheduled ahead of the interior rows' CTAs
    KTB_CUDA(cudaStreamCreateWithPriority(cs, cudaStreamNonBlocking, hi));
    KTB_CUDA(cudaEventCreateWithFlags(a, cudaEventDisableTiming));
    KTB_CUDA(cudaEventCreateWithFlags(b, cudaEventDisableTiming));
}

void run_part(ktb_halo::Part& q, const double* x, double* y, cudaStream_t s) {
    q.p->stream = s;
    plan_run(q.p, x, y + q.r0, 0, q.m->n);
}

}  // namespace

ktb_halo* halo_create(ktb_matrix* local, int64_t halo_lo, int64_t halo_hi, ktb_comm* comm,
                      int kernel, int64_t param) {
    require(local != nullptr && comm != nullptr, "halo: null handle");
    require(local->kind == KTB_GENERAL, "halo: general matrices only");
    require(halo_lo >= 0 && halo_hi >= 0 && local->ncols == halo_lo + local->n + halo_hi,
            "halo: columns must be [halo_lo | owned | halo_hi]");
    require(local->device == comm->device, "halo: matrix and communicator on different devices");
    require(kernel >= KTB_U1 && kernel <= KTB_U4, "halo: unsymmetric kernels only");
    require(comm->rank > 0 || halo_lo == 0, "halo: rank 0 has no lower neighbour");
    require(comm->rank < comm->world - 1 || halo_hi == 0, "halo: last rank has no upper neighbour");
    DeviceGuard g(local->device);
    auto h = std::make_unique<ktb_halo>();
    h->comm = comm;
    h->device = local->device;
    h->n = local->n;
    h->halo_lo = halo_lo;
    h->halo_hi = halo_hi;
    h->nnz = local->nnz;
    make_events(&h->cs, &h->ev_ready, &h->ev_done);
    // (collective) neighbours' shapes: how much of my owned x each one reads
    const int W = comm->world, r = comm->rank;
    DBuf<int64_t> mine(3), all(3 * static_cast<size_t>(W));
    const int64_t me[3] = {local->n, halo_lo, halo_hi};
    KTB_CUDA(cudaMemcpyAsync(mine.p, me, sizeof me, cudaMemcpyHostToDevice, h->cs));
    comm->allgather(mine.p, all.p, sizeof me, h->cs);
    std::vector<int64_t> info(3 * static_cast<size_t>(W));
    KTB_CUDA(cudaMemcpyAsync(info.data(), all.p, 24 * W, cudaMemcpyDeviceToHost, h->cs));
    KTB_CUDA(cudaStreamSynchronize(h->cs));
    if (r > 0) h->send_down = info[3 * (r - 1) + 2];
    if (r < W - 1) h->send_up = info[3 * (r + 1) + 1];
    require(h->send_down <= h->n && h->send_up <= h->n,
            "halo: a neighbour's halo is wider than this rank's rows");
    if (r > 0) require(halo_lo <= info[3 * (r - 1)], "halo: halo_lo wider than the lower rank");
    if (r < W - 1) require(halo_hi <= info[3 * (r + 1)], "halo: halo_hi wider than the upper rank");
    // interior rows: no column in either halo
    int64_t last_lo = -1, first_hi = h->n;
    if (h->n > 0 && local->nnz > 0) {
        DBuf<long long> red(2);
        const long long init[2] = {-1, static_cast<long long>(h->n)};
        KTB_CUDA(cudaMemcpyAsync(red.p, init, sizeof init, cudaMemcpyHostToDevice, h->cs));
        const int grid = static_cast<int>(std::min<int64_t>(ceil_div64(h->n, 256), 4 * 148));
        k_halo_rows<<<grid, 256, 0, h->cs>>>(h->n, local->row_ptr.p, local->col.p, halo_lo,
                                             halo_lo + h->n, red.p, red.p + 1);
        KTB_LAUNCH();
        long long out[2];
        KTB_CUDA(cudaMemcpyAsync(out, red.p, sizeof out, cudaMemcpyDeviceToHost, h->cs));
        KTB_CUDA(cudaStreamSynchronize(h->cs));
        last_lo = out[0];
        first_hi = out[1];
    }
    h->ib = last_lo + 1;
    h->ie = std::max<int64_t>(first_hi, h->ib);
    auto add = [&](std::vector<ktb_halo::Part>& v, int64_t r0, int64_t r1) {
        if (r1 <= r0) return;
        ktb_halo::Part q{r0, r1, nullptr, nullptr};
        q.m = matrix_slice(local, r0, r1);
        try {
            // the persistent / coded slice forms need a uniform width and few
            // column deltas (a thin boundary part may not have them): fall
            // back 106 -> 105 -> 104 -> 100 (106 also needs few distinct values)
            const int64_t tries[4] = {param, param == 106 ? 105 : param == 105 ? 104 : 100,
                                      param == 106 ? 104 : 100, 100};
            for (int t = 0; t < 4 && !q.p; ++t) {
                try {
                    q.p = plan_create_internal(q.m, kernel, tries[t], 0, h->cs);
                } catch (const Invalid&) {
                    if (kernel != KTB_U1 || param < 102 || param > 106 || t == 3) throw;
                }
            }
        } catch (...) {
            delete q.m;
            throw;
        }
        v.push_back(q);
    };
    add(h->interior, h->ib, h->ie);
    add(h->boundary, 0, h->ib);
    add(h->boundary, h->ie, h->n);
    return h.release();
}

void halo_exchange(ktb_halo* h, double* x, cudaStream_t s) {
    ktb_comm* c = h->comm;
    const int r = c->rank;
    KTB_CUDA(cudaEventRecord(h->ev_ready, s));
    KTB_CUDA(cudaStreamWaitEvent(h->cs, h->ev_ready, 0));
    double* owned = x + h->halo_lo;
    c->group_start();
    if (r > 0) {
        if (h->send_down) c->send(owned, 8 * h->send_down, r - 1, h->cs);
        if (h->halo_lo) c->recv(x, 8 * h->halo_lo, r - 1, h->cs);
    }
    if (r < c->world - 1) {
        if (h->send_up) c->send(owned + h->n - h->send_up, 8 * h->send_up, r + 1, h->cs);
        if (h->halo_hi) c->recv(owned + h->n, 8 * h->halo_hi, r + 1, h->cs);
    }
    c->group_end();
    KTB_CUDA(cudaEventRecord(h->ev_done, h->cs));
}

void halo_spmv(ktb_halo* h, double* x, double* y, cudaStream_t s) {
    DeviceGuard g(h->device);
    halo_exchange(h, x, s);
    if (h->timing) KTB_CUDA(cudaEventRecord(h->te[0], s));
    for (auto& q : h->interior) run_part(q, x, y, s);  // overlaps the exchange
    if (h->timing) KTB_CUDA(cudaEventRecord(h->te[1], s));
    KTB_CUDA(cudaStreamWaitEvent(s, h->ev_done, 0));
    if (h->timing) KTB_CUDA(cudaEventRecord(h->te[2], s));
    for (auto& q : h->boundary) run_part(q, x, y, s);
    if (h->timing) KTB_CUDA(cudaEventRecord(h->te[3], s));
}

namespace {
// per row chunk c: max over its interior rows of the last column (local x
// coordinates) -> the x chunk the rows need before they can run
__global__ void k_chunk_reach(int64_t ib, int64_t ie, const int64_t* __restrict__ cb, int nchunks,
                              const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              long long* reach) {
    for (int64_t i = ib + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < ie;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t a = rp[i - ib], b = rp[i - ib + 1];
        if (b <= a) continue;
        int lo = 0, hi = nchunks - 1;  // chunk of row i
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cb[mid] <= i) lo = mid; else hi = mid - 1;
        }
        atomicMax(reach + lo, static_cast<long long>(col[b - 1]));
    }
}
}  // namespace

// y_host = A x_host through the halo operator with the copies overlapped
// inside the call: owned x in `chunks` row chunks host->device on one copy
// stream; each interior row chunk starts once the x chunks its columns reach
// have landed and its y rows go device->host on a second copy stream while
// the next chunks compute; the halo exchange starts after the last x chunk
// and the boundary rows run last. U1 plans only (row sub-ranges); other
// kernels use one chunk.
void halo_spmv_host(ktb_halo* h, const double* xh, double* yh, int chunks) {
    DeviceGuard g(h->device);
    const int64_t n = h->n, xlen = h->halo_lo + h->n + h->halo_hi;
    bool rows_ok = true;
    for (auto& q : h->interior) rows_ok &= q.p->kernel == KTB_U1 && q.p->param != 101;
    chunks = std::max(1, std::min<int>(rows_ok ? chunks : 1, static_cast<int>(std::max<int64_t>(n / 32, 1))));
    if (h->dx.n < static_cast<size_t>(std::max<int64_t>(xlen, 1))) h->dx.alloc(std::max<int64_t>(xlen, 1));
    if (h->dy.n < static_cast<size_t>(std::max<int64_t>(n, 1))) h->dy.alloc(std::max<int64_t>(n, 1));
    if (!h->cin) {
        KTB_CUDA(cudaStreamCreateWithFlags(&h->cin, cudaStreamNonBlocking));
        KTB_CUDA(cudaStreamCreateWithFlags(&h->cout, cudaStreamNonBlocking));
        KTB_CUDA(cudaStreamCreateWithFlags(&h->comp, cudaStreamNonBlocking));
        KTB_CUDA(cudaEventCreateWithFlags(&h->ev_start, cudaEventDisableTiming));
        KTB_CUDA(cudaEventCreateWithFlags(&h->ev_bnd, cudaEventDisableTiming));
    }
    if (chunks != h->chunks) {
        for (auto* v : {&h->ev_in, &h->ev_comp})
            for (cudaEvent_t e : *v) cudaEventDestroy(e);
        h->ev_in.assign(chunks, nullptr);
        h->ev_comp.assign(chunks, nullptr);
        for (int c = 0; c < chunks; ++c) {
            KTB_CUDA(cudaEventCreateWithFlags(&h->ev_in[c], cudaEventDisableTiming));
            KTB_CUDA(cudaEventCreateWithFlags(&h->ev_comp[c], cudaEventDisableTiming));
        }
        h->cb.assign(chunks + 1, 0);
        for (int c = 0; c <= chunks; ++c) h->cb[c] = (n * c / chunks) & ~int64_t(31);
        h->cb[chunks] = n;
        h->need.assign(chunks, chunks - 1);
        if (chunks > 1 && !h->interior.empty()) {
            const ktb_matrix* m = h->interior[0].m;
            DBuf<int64_t> dcb(chunks + 1);
            DBuf<long long> red(chunks);
            KTB_CUDA(cudaMemcpyAsync(dcb.p, h->cb.data(), 8 * (chunks + 1), cudaMemcpyHostToDevice, h->cin));
            KTB_CUDA(cudaMemsetAsync(red.p, 0, 8 * chunks, h->cin));
            k_chunk_reach<<<4 * 148, 256, 0, h->cin>>>(h->ib, h->ie, dcb.p, chunks, m->row_ptr.p,
                                                       m->col.p, red.p);
            KTB_LAUNCH();
            std::vector<long long> reach(chunks);
            KTB_CUDA(cudaMemcpyAsync(reach.data(), red.p, 8 * chunks, cudaMemcpyDeviceToHost, h->cin));
            KTB_CUDA(cudaStreamSynchronize(h->cin));
            for (int c = 0; c < chunks; ++c) {
                const int64_t last = std::max<long long>(reach[c] - h->halo_lo, 0);  // owned index
                int k = c;
                while (k + 1 < chunks && h->cb[k + 1] <= last) ++k;
                h->need[c] = std::max(k, c);
            }
        }
        h->chunks = chunks;
    }
    cudaStream_t s = h->comp;  // the call is synchronous: private compute stream
    double* dx = h->dx.p;
    double* dy = h->dy.p;
    double* owned = dx + h->halo_lo;
    // previous call fully drained (synchronous API), so buffers are free
    for (int c = 0; c < chunks; ++c) {
        const int64_t a = h->cb[c], b = h->cb[c + 1];
        if (b > a)
            KTB_CUDA(cudaMemcpyAsync(owned + a, xh + a, 8 * (b - a), cudaMemcpyHostToDevice, h->cin));
        KTB_CUDA(cudaEventRecord(h->ev_in[c], h->cin));
    }
    // the exchange needs the owned edges: after the last x chunk
    halo_exchange(h, dx, h->cin);
    for (int c = 0; c < chunks; ++c) {
        const int64_t a = std::max(h->cb[c], h->ib), b = std::min(h->cb[c + 1], h->ie);
        KTB_CUDA(cudaStreamWaitEvent(s, h->ev_in[h->need[c]], 0));
        if (b > a)
            for (auto& q : h->interior) {
                q.p->stream = s;
                plan_run(q.p, dx, dy + q.r0, a - q.r0, b - q.r0);
            }
        KTB_CUDA(cudaEventRecord(h->ev_comp[c], s));
        KTB_CUDA(cudaStreamWaitEvent(h->cout, h->ev_comp[c], 0));
        if (b > a)
            KTB_CUDA(cudaMemcpyAsync(yh + a, dy + a, 8 * (b - a), cudaMemcpyDeviceToHost, h->cout));
    }
    KTB_CUDA(cudaStreamWaitEvent(s, h->ev_done, 0));
    for (auto& q : h->boundary) run_part(q, dx, dy, s);
    KTB_CUDA(cudaEventRecord(h->ev_bnd, s));
    KTB_CUDA(cudaStreamWaitEvent(h->cout, h->ev_bnd, 0));
    for (auto& q : h->boundary)
        KTB_CUDA(cudaMemcpyAsync(yh + q.r0, dy + q.r0, 8 * (q.r1 - q.r0), cudaMemcpyDeviceToHost,
                                 h->cout));
    KTB_CUDA(cudaStreamSynchronize(h->cout));
    KTB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace ktb

// ---------------------------------------------------- general split: state
namespace ktb {

struct DistComm {  // attached to a ktb_dist by ktb_dist_connect
    ktb_comm* comm = nullptr;
    DBuf<double> xg, sendbuf;
    ktb_plan* plan = nullptr;  // A_d plan
    bool own_plan = true;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    std::vector<int64_t> ro, so;  // receive / send offsets per peer
    ~DistComm() {
        if (own_plan) delete plan;
        if (ev_ready) cudaEventDestroy(ev_ready);
        if (ev_done) cudaEventDestroy(ev_done);
        if (cs) cudaStreamDestroy(cs);
    }
};

void dist_comm_free(ktb_dist* d) {
    delete static_cast<DistComm*>(d->comm_state);
    d->comm_state = nullptr;
}

void dist_connect(ktb_dist* d, ktb_comm* comm, int kernel, int64_t param) {
    require(comm != nullptr, "dist: null communicator");
    require(comm->world == d->world && comm->rank == d->rank,
            "dist: communicator rank/world differ from the split's");
    DeviceGuard g(comm->device);
    dist_comm_free(d);
    if (d->device != comm->device) dist_upload(d, comm->device);
    auto st = std::make_unique<DistComm>();
    st->comm = comm;
    make_events(&st->cs, &st->ev_ready, &st->ev_done);
    const int W = d->world, r = d->rank;
    // (collective) every rank's per-owner ghost counts -> what each peer needs
    DBuf<int64_t> mine(W), all(static_cast<size_t>(W) * W);
    KTB_CUDA(cudaMemcpyAsync(mine.p, d->recv_counts.data(), 8 * W, cudaMemcpyHostToDevice, st->cs));
    comm->allgather(mine.p, all.p, 8 * W, st->cs);
    std::vector<int64_t> cnt(static_cast<size_t>(W) * W);
    KTB_CUDA(cudaMemcpyAsync(cnt.data(), all.p, 8 * W * W, cudaMemcpyDeviceToHost, st->cs));
    KTB_CUDA(cudaStreamSynchronize(st->cs));
    std::vector<int64_t> send_counts(W, 0);
    for (int p = 0; p < W; ++p) send_counts[p] = p == r ? 0 : cnt[static_cast<size_t>(p) * W + r];
    st->ro.assign(W + 1, 0);
    st->so.assign(W + 1, 0);
    for (int p = 0; p < W; ++p) {
        st->ro[p + 1] = st->ro[p] + d->recv_counts[p];
        st->so[p + 1] = st->so[p] + send_counts[p];
    }
    // (collective) the lists themselves: my ghost ids owned by p go to p
    DBuf<int64_t> gh(std::max<int64_t>(st->ro[W], 1)), want(std::max<int64_t>(st->so[W], 1));
    if (st->ro[W])
        KTB_CUDA(cudaMemcpyAsync(gh.p, d->ghosts.data(), 8 * st->ro[W], cudaMemcpyHostToDevice,
                                 st->cs));
    comm->group_start();
    for (int p = 0; p < W; ++p) {
        if (p == r) continue;
        if (d->recv_counts[p]) comm->send(gh.p + st->ro[p], 8 * d->recv_counts[p], p, st->cs);
        if (send_counts[p]) comm->recv(want.p + st->so[p], 8 * send_counts[p], p, st->cs);
    }
    comm->group_end();
    std::vector<int64_t> cols(st->so[W]);
    if (st->so[W])
        KTB_CUDA(cudaMemcpyAsync(cols.data(), want.p, 8 * st->so[W], cudaMemcpyDeviceToHost,
                                 st->cs));
    KTB_CUDA(cudaStreamSynchronize(st->cs));
    dist_set_sends(d, send_counts.data(), cols.data());
    st->xg.alloc(std::max<int64_t>(d->ghosts.size(), 1));
    st->sendbuf.alloc(std::max<int64_t>(st->so[W], 1));
    if (d->local->n > 0 && d->local->nnz > 0) {
        try {
            st->plan = plan_create_internal(d->local, kernel, param, 0, st->cs);
        } catch (const Invalid&) {
            if (kernel != KTB_U1 || param < 100 || param > 106) throw;
            // the warp-sliced / coded forms refuse irregular rows: nnz-balanced tiles
            st->plan = plan_create_internal(d->local, KTB_U2, 0, 0, st->cs);
        }
    }
    d->comm_state = st.release();
}

void dist_set_plan(ktb_dist* d, ktb_plan* plan) {
    auto* st = static_cast<DistComm*>(d->comm_state);
    require(st != nullptr, "dist: not connected");
    require(plan == nullptr || plan->m == d->local, "dist: plan built for a different matrix");
    if (st->own_plan) delete st->plan;
    st->plan = plan;
    st->own_plan = false;
}

void dist_exchange(ktb_dist* d, const double* x_owned, cudaStream_t s) {
    auto* st = static_cast<DistComm*>(d->comm_state);
    require(st != nullptr, "dist: not connected");
    const int W = d->world, r = d->rank;
    dist_pack(d, x_owned, st->sendbuf.p, s);
    KTB_CUDA(cudaEventRecord(st->ev_ready, s));
    KTB_CUDA(cudaStreamWaitEvent(st->cs, st->ev_ready, 0));
    ktb_comm* c = st->comm;
    c->group_start();
    for (int p = 0; p < W; ++p) {
        if (p == r) continue;
        if (st->so[p + 1] > st->so[p])
            c->send(st->sendbuf.p + st->so[p], 8 * (st->so[p + 1] - st->so[p]), p, st->cs);
        if (st->ro[p + 1] > st->ro[p])
            c->recv(st->xg.p + st->ro[p], 8 * (st->ro[p + 1] - st->ro[p]), p, st->cs);
    }
    c->group_end();
    KTB_CUDA(cudaEventRecord(st->ev_done, st->cs));
}

void dist_spmv(ktb_dist* d, const double* x_owned, double* y, cudaStream_t s) {
    auto* st = static_cast<DistComm*>(d->comm_state);
    require(st != nullptr, "dist: not connected");
    DeviceGuard g(d->device);
    dist_exchange(d, x_owned, s);
    if (st->plan) {
        st->plan->stream = s;
        plan_run(st->plan, x_owned, y, 0, d->local->n);
    } else if (d->n_loc) {
        KTB_CUDA(cudaMemsetAsync(y, 0, 8 * d->n_loc, s));
    }
    KTB_CUDA(cudaStreamWaitEvent(s, st->ev_done, 0));
    dist_ghost_spmv(d, st->xg.p, y, s);
}

int dist_launches(const ktb_dist* d) {
    auto* st = static_cast<const DistComm*>(d->comm_state);
    if (!st) return 0;
    return int(!d->send_idx.empty()) + (st->plan ? st->plan->launches : 1) +
           int(!d->o_rows.empty());
}

}  // namespace ktb

// ------------------------------------------------------------------ C ABI
using namespace ktb;

extern "C" {

int ktb_comm_id(uint8_t* id) {
    return guarded_call([&] {
        static_assert(sizeof(ncclUniqueId) == KTB_COMM_ID_BYTES, "ncclUniqueId size");
        ncclUniqueId u;
        KTB_NCCL(nccl_api().ncclGetUniqueId(&u), nullptr);
        std::memcpy(id, &u, sizeof u);
    });
}

int ktb_comm_create(const uint8_t* id, int world, int rank, int device, ktb_comm** out) {
    return guarded_call([&] {
        require(world >= 1 && rank >= 0 && rank < world, "comm: bad rank/world");
        DeviceGuard g(device);
        auto c = std::make_unique<NcclComm>();
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        KTB_NCCL(nccl_api().ncclCommInitRank(&c->c, world, u, rank), nullptr);
        c->world = world;
        c->rank = rank;
        c->device = device;
        *out = c.release();
    });
}

int ktb_comm_wrap(void* nccl_comm, int device, ktb_comm** out) {
    return guarded_call([&] {
        require(nccl_comm != nullptr, "comm: null ncclComm_t");
        auto c = std::make_unique<NcclComm>();
        c->c = static_cast<ncclComm_t>(nccl_comm);
        c->own = false;
        KTB_NCCL(nccl_api().ncclCommCount(c->c, &c->world), c->c);
        KTB_NCCL(nccl_api().ncclCommUserRank(c->c, &c->rank), c->c);
        int dev = -1;
        KTB_NCCL(nccl_api().ncclCommCuDevice(c->c, &dev), c->c);
        require(device < 0 || dev == device, "comm: ncclComm_t lives on another device");
        c->device = dev;
        *out = c.release();
    });
}

int ktb_loopback_world_create(int world, ktb_loopback_world** out) {
    return guarded_call([&] {
        require(world >= 1, "comm: bad rank/world");
        auto* w = new ktb_loopback_world();
        w->w = std::make_shared<LoopWorld>(world);
        *out = w;
    });
}

int ktb_loopback_world_destroy(ktb_loopback_world* w) {
    return guarded_call([&] { delete w; });
}

int ktb_comm_create_loopback(ktb_loopback_world* w, int rank, int device, ktb_comm** out) {
    return guarded_call([&] {
        require(w != nullptr && rank >= 0 && rank < w->w->W, "comm: bad rank/world");
        auto c = std::make_unique<LoopComm>();
        c->w = w->w;
        c->world = w->w->W;
        c->rank = rank;
        c->device = device;
        *out = c.release();
    });
}

int ktb_comm_info(const ktb_comm* c, int* world, int* rank, int* device, int* nccl_version,
                  int* is_nccl) {
    return guarded_call([&] {
        require(c != nullptr, "comm: null handle");
        if (world) *world = c->world;
        if (rank) *rank = c->rank;
        if (device) *device = c->device;
        if (nccl_version) {
            int v = 0;
            try {
                nccl_api().ncclGetVersion(&v);
            } catch (const CudaError&) {  // a loopback comm needs no NCCL
            }
            *nccl_version = v;
        }
        if (is_nccl) *is_nccl = std::strcmp(c->kind(), "nccl") == 0;
    });
}

int ktb_comm_destroy(ktb_comm* c) {
    return guarded_call([&] {
        if (c) {
            DeviceGuard g(c->device);
            delete c;
        }
    });
}

int ktb_comm_allreduce(ktb_comm* c, double* buf, int64_t count, int op, void* stream) {
    return guarded_call([&] {
        require(c != nullptr && count >= 0, "comm: bad all-reduce");
        require(op == KTB_SUM || op == KTB_MAX, "comm: bad reduction op");
        DeviceGuard g(c->device);
        c->allreduce(buf, count, op, static_cast<cudaStream_t>(stream));
    });
}

int ktb_comm_allgather(ktb_comm* c, const void* send, void* recv, size_t bytes, void* stream) {
    return guarded_call([&] {
        require(c != nullptr, "comm: null handle");
        DeviceGuard g(c->device);
        c->allgather(send, recv, bytes, static_cast<cudaStream_t>(stream));
    });
}

int ktb_comm_sendrecv(ktb_comm* c, const void* send, size_t send_bytes, int send_peer, void* recv,
                      size_t recv_bytes, int recv_peer, void* stream) {
    return guarded_call([&] {
        require(c != nullptr, "comm: null handle");
        DeviceGuard g(c->device);
        auto s = static_cast<cudaStream_t>(stream);
        c->group_start();
        if (send_peer >= 0 && send_bytes) c->send(send, send_bytes, send_peer, s);
        if (recv_peer >= 0 && recv_bytes) c->recv(recv, recv_bytes, recv_peer, s);
        c->group_end();
    });
}

int ktb_halo_create(ktb_matrix* local, int64_t halo_lo, int64_t halo_hi, ktb_comm* comm,
                    int kernel, int64_t param, ktb_halo** out) {
    return guarded_call([&] { *out = halo_create(local, halo_lo, halo_hi, comm, kernel, param); });
}

int ktb_halo_create_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, double off,
                             ktb_comm* comm, int kernel, int64_t param, ktb_halo** out) {
    return guarded_call([&] {
        require(comm != nullptr, "halo: null handle");
        const int W = comm->world, r = comm->rank;
        require(W >= 1 && W <= nz, "slab: need 1 <= world <= nz");
        const int64_t z0 = r * nz / W, z1 = (r + 1) * nz / W, plane = nx * ny;
        std::unique_ptr<ktb_matrix> slab(
            gen_stencil7(nx, ny, nz, z0, z1, true, diag, off, off, off, comm->device));
        *out = halo_create(slab.get(), z0 > 0 ? plane : 0, z1 < nz ? plane : 0, comm, kernel,
                           param);
    });
}

int ktb_halo_create_csr(int64_t n_global, int64_t row0, int64_t n_local, const int64_t* row_ptr,
                        const int64_t* col_idx, const double* values, ktb_comm* comm, int kernel,
                        int64_t param, ktb_halo** out) {
    return guarded_call([&] {
        require(comm != nullptr, "halo: null handle");
        require(n_local >= 0 && row0 >= 0 && row0 + n_local <= n_global,
                "halo: rows outside [0, n)");
        require(row_ptr != nullptr && row_ptr[0] == 0, "csr: row_ptr[0] != 0");
        const int64_t nnz = row_ptr[n_local];
        int64_t lo = row0, hi = row0 + n_local;
        for (int64_t k = 0; k < nnz; ++k) {
            require(col_idx[k] >= 0 && col_idx[k] < n_global, "csr: column index out of range");
            lo = std::min(lo, col_idx[k]);
            hi = std::max(hi, col_idx[k] + 1);
        }
        std::vector<int64_t> loc(col_idx, col_idx + nnz);
        for (auto& c : loc) c -= lo;
        std::unique_ptr<ktb_matrix> m(
            matrix_create_rect(n_local, hi - lo, row_ptr, loc.data(), values, comm->device));
        m->col_shift = row0 - lo;
        *out = halo_create(m.get(), row0 - lo, hi - row0 - n_local, comm, kernel, param);
    });
}

int ktb_halo_info(const ktb_halo* h, int64_t* n_local, int64_t* x_len, int64_t* owned_offset,
                  int64_t* interior_begin, int64_t* interior_end, int64_t* nnz, int* launches) {
    return guarded_call([&] {
        require(h != nullptr, "halo: null handle");
        if (n_local) *n_local = h->n;
        if (x_len) *x_len = h->halo_lo + h->n + h->halo_hi;
        if (owned_offset) *owned_offset = h->halo_lo;
        if (interior_begin) *interior_begin = h->ib;
        if (interior_end) *interior_end = h->ie;
        if (nnz) *nnz = h->nnz;
        if (launches) {
            int l = 0;
            for (auto* v : {&h->interior, &h->boundary})
                for (auto& q : *v) l += q.p->launches;
            *launches = l;
        }
    });
}

int ktb_halo_plan_params(const ktb_halo* h, int64_t* interior_param, int64_t* boundary_param) {
    return guarded_call([&] {
        require(h != nullptr, "halo: null handle");
        if (interior_param) *interior_param = h->interior.empty() ? -1 : h->interior[0].p->param;
        if (boundary_param) *boundary_param = h->boundary.empty() ? -1 : h->boundary[0].p->param;
    });
}

int ktb_halo_parts(const ktb_halo* h, int64_t* interior_rows, int64_t* interior_nnz,
                   int64_t* boundary_rows, int64_t* boundary_nnz) {
    return guarded_call([&] {
        require(h != nullptr, "halo: null handle");
        int64_t ir = 0, in = 0, br = 0, bn = 0;
        for (auto& q : h->interior) ir += q.m->n, in += q.m->nnz;
        for (auto& q : h->boundary) br += q.m->n, bn += q.m->nnz;
        if (interior_rows) *interior_rows = ir;
        if (interior_nnz) *interior_nnz = in;
        if (boundary_rows) *boundary_rows = br;
        if (boundary_nnz) *boundary_nnz = bn;
    });
}

int ktb_halo_spmv(ktb_halo* h, double* x, double* y, void* stream) {
    return guarded_call([&] {
        require(h != nullptr && x != nullptr && y != nullptr, "spmv: dimension mismatch");
        halo_spmv(h, x, y, static_cast<cudaStream_t>(stream));
    });
}

int ktb_halo_spmv_host(ktb_halo* h, const double* x_owned, double* y, int chunks) {
    return guarded_call([&] {
        require(h != nullptr && x_owned != nullptr && y != nullptr, "spmv: dimension mismatch");
        halo_spmv_host(h, x_owned, y, chunks);
    });
}

int ktb_halo_exchange(ktb_halo* h, double* x, void* stream) {
    return guarded_call([&] {
        require(h != nullptr && x != nullptr, "spmv: dimension mismatch");
        DeviceGuard g(h->device);
        auto s = static_cast<cudaStream_t>(stream);
        halo_exchange(h, x, s);
        KTB_CUDA(cudaStreamWaitEvent(s, h->ev_done, 0));
    });
}

int ktb_halo_set_timing(ktb_halo* h, int on) {
    return guarded_call([&] {
        require(h != nullptr, "halo: null handle");
        DeviceGuard g(h->device);
        if (on && !h->te[0])
            for (auto& e : h->te) KTB_CUDA(cudaEventCreate(&e));
        h->timing = on != 0;
    });
}

int ktb_halo_timing(ktb_halo* h, double* interior_ms, double* boundary_ms) {
    return guarded_call([&] {
        require(h != nullptr && h->timing, "halo: timing not enabled");
        DeviceGuard g(h->device);
        float a = 0.f, b = 0.f;
        KTB_CUDA(cudaEventSynchronize(h->te[3]));
        KTB_CUDA(cudaEventElapsedTime(&a, h->te[0], h->te[1]));
        KTB_CUDA(cudaEventElapsedTime(&b, h->te[2], h->te[3]));
        if (interior_ms) *interior_ms = a;
        if (boundary_ms) *boundary_ms = b;
    });
}

int ktb_halo_destroy(ktb_halo* h) {
    return guarded_call([&] {
        if (h) {
            DeviceGuard g(h->device);
            delete h;
        }
    });
}

int ktb_dist_connect(ktb_dist* d, ktb_comm* comm, int kernel, int64_t param) {
    return guarded_call([&] {
        require(d != nullptr, "dist: null handle");
        dist_connect(d, comm, kernel, param);
    });
}

int ktb_dist_set_plan(ktb_dist* d, ktb_plan* plan) {
    return guarded_call([&] {
        require(d != nullptr, "dist: null handle");
        dist_set_plan(d, plan);
    });
}

int ktb_dist_spmv(ktb_dist* d, const double* x_owned, double* y, void* stream) {
    return guarded_call([&] {
        // (a rank that owns no rows has nothing to point at)
        require(d != nullptr && ((x_owned != nullptr && y != nullptr) || d->n_loc == 0),
                "spmv: dimension mismatch");
        dist_spmv(d, x_owned, y, static_cast<cudaStream_t>(stream));
    });
}

int ktb_dist_exchange(ktb_dist* d, const double* x_owned, void* stream) {
    return guarded_call([&] {
        require(d != nullptr && (x_owned != nullptr || d->n_loc == 0), "spmv: dimension mismatch");
        DeviceGuard g(d->device);
        auto s = static_cast<cudaStream_t>(stream);
        dist_exchange(d, x_owned, s);
        KTB_CUDA(cudaStreamWaitEvent(s, static_cast<DistComm*>(d->comm_state)->ev_done, 0));
    });
}

int ktb_dist_launches(const ktb_dist* d, int* launches) {
    return guarded_call([&] { *launches = dist_launches(d); });
}

}  // extern "C"

extern "C" int ktb_dist_sends(const ktb_dist* d, int64_t* send_counts, int64_t* send_cols) {
    return guarded_call([&] {
        require(d != nullptr, "dist: null handle");
        require(d->sends_set, "dist: send lists not set");
        if (send_counts) std::copy(d->send_counts.begin(), d->send_counts.end(), send_counts);
        if (send_cols)
            for (size_t k = 0; k < d->send_idx.size(); ++k) send_cols[k] = d->row0 + d->send_idx[k];
    });
}
