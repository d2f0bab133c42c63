// ktb_mm.cu -- Matrix Market ingest, host side.
//
// Same accept/reject behaviour, results and messages as the reference's
// proj/include/ktune/matrix_market.hpp (parse_mm_header :37-65,
// read_mm_entries :67-86, coo_to_csr :89-108, load_matrix_market :165-194,
// writers :206-239), rebuilt for throughput: the file is mapped once, the
// entry section is cut into line-aligned ranges parsed by one thread each;
// when the entries arrive in (row, col) order (any file a Matrix Market
// writer produced, the reference's included) the CRS is assembled from the
// thread parts in parallel, otherwise by a stable counting sort. Entry
// tokens follow the
// `istream >> int64 >> int64 >> double` rules of libstdc++'s num_get (any
// isspace skipped, '+' or '-' sign, decimal digits; the double token is
// [sign] digits [. digits] [e [sign] digits] and must convert completely,
// +-inf results reject), so a line the reference rejects is rejected here
// with the same message, first bad line first.
//
// Duplicates: the reference orders the whole COO with std::sort, whose order
// among equal (row, col) keys is unspecified, and sums each run in that
// order. With two copies the sum is the same in any order (fp addition
// commutes), so the fast paths sum in file order; when some coordinate
// occurs three or more times the CRS is rebuilt exactly the reference's way
// (the file-order COO through the same std::sort and comparator, the same
// libstdc++), so the loaded matrix is bit-identical in every case.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "ktb_internal.cuh"

namespace ktb {

namespace {

struct Mapped {
    const char* p = nullptr;
    size_t len = 0;
    int fd = -1;
    explicit Mapped(const std::string& path) {
        fd = ::open(path.c_str(), O_RDONLY);
        struct stat st {};
        if (fd < 0 || ::fstat(fd, &st) != 0 || S_ISDIR(st.st_mode))
            throw Invalid("matrix market: cannot open " + path);
        len = static_cast<size_t>(st.st_size);
        if (len) {
            void* m = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
            if (m == MAP_FAILED) throw Invalid("matrix market: cannot open " + path);
            p = static_cast<const char*>(m);
            ::madvise(m, len, MADV_SEQUENTIAL);
        }
    }
    ~Mapped() {
        if (p) ::munmap(const_cast<char*>(p), len);
        if (fd >= 0) ::close(fd);
    }
    Mapped(const Mapped&) = delete;
    Mapped& operator=(const Mapped&) = delete;
};

std::string lower(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// std::getline over the mapping: the line without its '\n'; false at EOF
// with nothing extracted.
bool getline_at(const char* end, const char*& s, std::string& line) {
    if (s >= end) {
        line.clear();
        return false;
    }
    const char* e = static_cast<const char*>(std::memchr(s, '\n', end - s));
    if (!e) e = end;
    line.assign(s, e);
    s = e < end ? e + 1 : end;
    return true;
}

void check(bool cond, const std::string& msg) {
    if (!cond) throw Invalid(msg);
}

// matrix_market.hpp:37-65, with the same istringstream extraction.
MmHeader parse_header(const Mapped& f, const std::string& name, size_t* body) {
    const char* p = f.p;
    const char* end = f.p + f.len;
    std::string line;
    check(getline_at(end, p, line), "matrix market: empty file: " + name);
    std::istringstream hs(line);
    std::string banner, object, format, field, symmetry;
    hs >> banner >> object >> format >> field >> symmetry;
    check(banner == "%%MatrixMarket", "matrix market: malformed header line: " + name);
    check(lower(object) == "matrix" && lower(format) == "coordinate",
          "matrix market: only coordinate matrices are supported: " + name);
    const std::string fl = lower(field);
    check(fl != "pattern" && fl != "complex",
          "matrix market: unsupported field type '" + fl + "': " + name);
    check(fl == "real", "matrix market: only real matrices are supported: " + name);
    const std::string sym = lower(symmetry);
    check(sym == "general" || sym == "symmetric",
          "matrix market: unsupported symmetry '" + sym + "': " + name);
    while (getline_at(end, p, line)) {
        if (line.empty() || line[0] == '%') continue;
        break;
    }
    std::istringstream ss(line);
    int64_t rows = -1, cols = -1, entries = -1;
    ss >> rows >> cols >> entries;
    check(rows > 0 && cols > 0 && entries >= 0, "matrix market: malformed size line: " + name);
    check(rows == cols, "matrix market: matrix is not square: " + name);
    *body = static_cast<size_t>(p - f.p);
    return MmHeader{rows, entries, sym == "symmetric"};
}

inline bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}
inline bool is_digit(char c) { return c >= '0' && c <= '9'; }

// `>> int64` on [q, le): skip whitespace, optional sign, >= 1 digit.
inline bool get_int(const char*& q, const char* le, int64_t& out) {
    while (q < le && is_space(*q)) ++q;
    const char* s = q;
    bool neg = false;
    if (s < le && (*s == '+' || *s == '-')) neg = *s++ == '-';
    if (s >= le || !is_digit(*s)) return false;
    const char* d = s;
    while (s < le && is_digit(*s)) ++s;
    uint64_t mag = 0;
    auto r = std::from_chars(d, s, mag);
    if (r.ec != std::errc()) return false;  // overflow: failbit
    if (neg ? mag > uint64_t(1) << 63 : mag > uint64_t(std::numeric_limits<int64_t>::max()))
        return false;
    out = neg ? static_cast<int64_t>(0 - mag) : static_cast<int64_t>(mag);
    q = s;
    return true;
}

// `>> double`: the num_get token, converted completely, finite.
inline bool get_double(const char*& q, const char* le, double& out) {
    while (q < le && is_space(*q)) ++q;
    const char* s = q;
    if (s < le && (*s == '+' || *s == '-')) ++s;
    const char* m0 = s;
    while (s < le && is_digit(*s)) ++s;
    bool mant = s > m0;
    if (s < le && *s == '.') {
        ++s;
        const char* f0 = s;
        while (s < le && is_digit(*s)) ++s;
        mant = mant || s > f0;
    }
    if (!mant) return false;
    if (s < le && (*s == 'e' || *s == 'E')) {
        ++s;  // num_get accumulates the 'e' and any sign even if no digit follows,
        if (s < le && (*s == '+' || *s == '-')) ++s;  // then strtod stops short
        const char* e0 = s;
        while (s < le && is_digit(*s)) ++s;
        if (s == e0) return false;
    }
    const char* t = *q == '+' ? q + 1 : q;  // from_chars takes no '+'
    double v = 0;
    auto r = std::from_chars(t, s, v);
    if (r.ec == std::errc::result_out_of_range) {  // strtod: under/overflow
        std::string tok(q, s);
        v = std::strtod(tok.c_str(), nullptr);
    } else if (r.ec != std::errc() || r.ptr != s) {
        return false;
    }
    if (std::isinf(v)) return false;
    out = v;
    q = s;
    return true;
}

// KTB_HOST_THREADS overrides the host thread count (default: all cores).
size_t host_threads() {
    if (const char* e = std::getenv("KTB_HOST_THREADS")) {
        const long v = std::strtol(e, nullptr, 10);
        if (v >= 1) return static_cast<size_t>(v);
    }
    return std::max(1u, std::thread::hardware_concurrency());
}

template <typename F>
void parallel_for(int T, F&& f) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(f, t);
    f(0);
    for (auto& x : th) x.join();
}

// One parser thread's slice of the entry section, in file order; symmetric
// files are mirrored into the upper triangle as they are read
// (matrix_market.hpp:176-177). `sorted`: (row, col) strictly increasing.
struct Part {
    std::vector<int64_t> r, c;
    std::vector<double> v;
    std::string err;
    bool sorted = true;
};

// matrix_market.hpp:67-86, one thread per line-aligned range.
std::vector<Part> parse_entries(const Mapped& f, size_t body, const MmHeader& h,
                                const std::string& name) {
    const char* base = f.p + body;
    const size_t len = f.len - body;
    const size_t per = size_t(2) << 20;  // >= 2 MB of text per thread
    const int T = static_cast<int>(
        std::max<size_t>(1, std::min<size_t>(host_threads(), len / per)));
    std::vector<size_t> cut(T + 1, 0);
    cut[T] = len;
    for (int t = 1; t < T; ++t) {
        size_t s = std::max(len * t / T, cut[t - 1]);
        while (s < len && s > 0 && base[s - 1] != '\n') ++s;
        cut[t] = s;
    }
    std::vector<Part> part(T);
    parallel_for(T, [&](int t) {
        const char* s = base + cut[t];
        const char* e = base + cut[t + 1];
        Part& P = part[t];
        const size_t guess = (e - s) / 12 + 16;
        P.r.reserve(guess);
        P.c.reserve(guess);
        P.v.reserve(guess);
        int64_t pr = -1, pc = -1;
        while (s < e) {
            const char* nl = static_cast<const char*>(std::memchr(s, '\n', e - s));
            const char* le = nl ? nl : e;
            if (le == s || *s == '%') {
                s = nl ? nl + 1 : e;
                continue;
            }
            const char* q = s;
            int64_t i = 0, j = 0;
            double v = 0;
            if (!(get_int(q, le, i) && get_int(q, le, j) && get_double(q, le, v))) {
                P.err = "matrix market: malformed entry line: " + name;
                return;
            }
            if (!(i >= 1 && i <= h.n && j >= 1 && j <= h.n)) {
                P.err = "matrix market: index out of range: " + name;
                return;
            }
            --i;
            --j;
            if (h.symmetric && i > j) std::swap(i, j);
            P.sorted = P.sorted && (i > pr || (i == pr && j > pc));
            pr = i;
            pc = j;
            P.r.push_back(i);
            P.c.push_back(j);
            P.v.push_back(v);
            s = nl ? nl + 1 : e;
        }
    });
    for (auto& P : part) check(P.err.empty(), P.err);  // earliest bad line wins
    size_t total = 0;
    for (auto& P : part) total += P.r.size();
    check(static_cast<int64_t>(total) == h.entries,
          "matrix market: entry count does not match size line: " + name);
    return part;
}

// Entries already in strictly increasing (row, col) order across all parts:
// the CRS is their concatenation (no reordering, no duplicates, which is
// exactly what coo_to_csr yields), assembled in parallel.
bool assemble_sorted(int64_t n, std::vector<Part>& part, ktb_csr_host& a) {
    const int T = static_cast<int>(part.size());
    int64_t pr = -1, pc = -1;
    for (auto& P : part) {
        if (!P.sorted) return false;
        if (P.r.empty()) continue;
        if (!(P.r[0] > pr || (P.r[0] == pr && P.c[0] > pc))) return false;
        pr = P.r.back();
        pc = P.c.back();
    }
    std::vector<size_t> off(T + 1, 0);
    for (int t = 0; t < T; ++t) off[t + 1] = off[t] + part[t].r.size();
    a.n = n;
    a.row_ptr.assign(n + 1, 0);
    a.col.resize(off[T]);
    a.val.resize(off[T]);
    int64_t* cnt = a.row_ptr.data() + 1;
    parallel_for(T, [&](int t) {
        Part& P = part[t];
        const size_t m = P.r.size();
        if (m) {  // a part's first and last rows may be shared with a neighbour
            const int64_t r0 = P.r[0], r1 = P.r[m - 1];
            int64_t c0 = 0, c1 = 0;
            for (size_t k = 0; k < m; ++k) {
                const int64_t r = P.r[k];
                if (r == r0) ++c0;
                else if (r == r1) ++c1;
                else ++cnt[r];
            }
            __atomic_fetch_add(&cnt[r0], c0, __ATOMIC_RELAXED);
            if (c1) __atomic_fetch_add(&cnt[r1], c1, __ATOMIC_RELAXED);
            std::memcpy(a.col.data() + off[t], P.c.data(), 8 * m);
            std::memcpy(a.val.data() + off[t], P.v.data(), 8 * m);
        }
        std::vector<int64_t>().swap(P.r);
        std::vector<int64_t>().swap(P.c);
        std::vector<double>().swap(P.v);
    });
    for (int64_t i = 0; i < n; ++i) a.row_ptr[i + 1] += a.row_ptr[i];
    return true;
}

// matrix_market.hpp:89-108 verbatim in its ordering: the file-order COO
// through std::sort on (row, col), runs summed front to back. Used only when
// a coordinate occurs 3+ times (the order of such a run is std::sort's).
void coo_to_csr_reference_order(int64_t n, const std::vector<Part>& part, ktb_csr_host& a) {
    struct Entry {
        int64_t row, col;
        double value;
    };
    std::vector<Entry> coo;
    for (auto& P : part)
        for (size_t k = 0; k < P.r.size(); ++k) coo.push_back({P.r[k], P.c[k], P.v[k]});
    std::sort(coo.begin(), coo.end(), [](const Entry& x, const Entry& y) {
        return x.row < y.row || (x.row == y.row && x.col < y.col);
    });
    a.n = n;
    a.row_ptr.assign(n + 1, 0);
    a.col.clear();
    a.val.clear();
    for (size_t k = 0; k < coo.size();) {
        size_t e = k + 1;
        double v = coo[k].value;
        while (e < coo.size() && coo[e].row == coo[k].row && coo[e].col == coo[k].col)
            v += coo[e++].value;
        a.col.push_back(coo[k].col);
        a.val.push_back(v);
        ++a.row_ptr[coo[k].row + 1];
        k = e;
    }
    for (int64_t i = 0; i < n; ++i) a.row_ptr[i + 1] += a.row_ptr[i];
}

// matrix_market.hpp:89-108. Counting sort by row (stable), then a stable
// sort of each row by column: file order among duplicates (exact for runs
// of at most two; longer runs switch to coo_to_csr_reference_order).
void coo_to_csr(int64_t n, const std::vector<Part>& part, ktb_csr_host& a) {
    size_t m = 0;
    for (auto& P : part) m += P.r.size();
    std::vector<int64_t> start(n + 1, 0);
    for (auto& P : part)
        for (int64_t r : P.r) ++start[r + 1];
    for (int64_t i = 0; i < n; ++i) start[i + 1] += start[i];
    std::vector<int64_t> next(start.begin(), start.end() - 1);
    std::vector<int64_t> bc(m);
    std::vector<double> bv(m);
    for (auto& P : part)
        for (size_t k = 0; k < P.r.size(); ++k) {
            const int64_t p = next[P.r[k]]++;
            bc[p] = P.c[k];
            bv[p] = P.v[k];
        }
    a.n = n;
    a.row_ptr.assign(n + 1, 0);
    a.col.clear();
    a.val.clear();
    a.col.reserve(m);
    a.val.reserve(m);
    std::vector<uint32_t> ord;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t b = start[i], e = start[i + 1];
        bool sorted = true;
        for (int64_t k = b + 1; k < e && sorted; ++k) sorted = bc[k - 1] < bc[k];
        if (sorted) {  // the common case: no reordering, no duplicates
            a.col.insert(a.col.end(), bc.begin() + b, bc.begin() + e);
            a.val.insert(a.val.end(), bv.begin() + b, bv.begin() + e);
            a.row_ptr[i + 1] = a.row_ptr[i] + (e - b);
            continue;
        }
        ord.resize(e - b);
        for (int64_t k = 0; k < e - b; ++k) ord[k] = static_cast<uint32_t>(k);
        std::stable_sort(ord.begin(), ord.end(),
                         [&](uint32_t x, uint32_t y) { return bc[b + x] < bc[b + y]; });
        int64_t cnt = 0;
        for (size_t k = 0; k < ord.size();) {
            size_t q = k + 1;
            double v = bv[b + ord[k]];
            while (q < ord.size() && bc[b + ord[q]] == bc[b + ord[k]]) v += bv[b + ord[q++]];
            if (q - k >= 3) {  // a run whose sum depends on std::sort's order
                coo_to_csr_reference_order(n, part, a);
                return;
            }
            a.col.push_back(bc[b + ord[k]]);
            a.val.push_back(v);
            ++cnt;
            k = q;
        }
        a.row_ptr[i + 1] = a.row_ptr[i] + cnt;
    }
}

// csr.hpp:38-54 (checks that can fail on loaded data)
void validate(const ktb_csr_host& a, bool upper) {
    for (int64_t i = 0; i < a.n; ++i)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            require(a.col[k] >= 0 && a.col[k] < a.n, "csr: column index out of range");
            if (k > a.row_ptr[i])
                require(a.col[k - 1] < a.col[k], "csr: columns not strictly increasing");
            if (upper) require(a.col[k] >= i, "sym csr: entry below the diagonal");
        }
}

// csr.hpp:88-123 (expand_symmetric) on host arrays
void expand(const ktb_csr_host& s, ktb_csr_host& a) {
    const int64_t n = s.n;
    a.n = n;
    a.kind = KTB_GENERAL;
    a.row_ptr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = s.row_ptr[i]; k < s.row_ptr[i + 1]; ++k) {
            ++a.row_ptr[i + 1];
            if (s.col[k] != i) ++a.row_ptr[s.col[k] + 1];
        }
    for (int64_t i = 0; i < n; ++i) a.row_ptr[i + 1] += a.row_ptr[i];
    a.col.resize(a.row_ptr[n]);
    a.val.resize(a.row_ptr[n]);
    std::vector<int64_t> next(a.row_ptr.begin(), a.row_ptr.end() - 1);
    for (int64_t i = 0; i < n; ++i)  // mirrored lower entries (columns < row) first
        for (int64_t k = s.row_ptr[i]; k < s.row_ptr[i + 1]; ++k) {
            const int64_t j = s.col[k];
            if (j == i) continue;
            a.col[next[j]] = i;
            a.val[next[j]] = s.val[k];
            ++next[j];
        }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = s.row_ptr[i]; k < s.row_ptr[i + 1]; ++k) {
            a.col[next[i]] = s.col[k];
            a.val[next[i]] = s.val[k];
            ++next[i];
        }
}

// matrix_market.hpp:110-133
bool exactly_symmetric(const ktb_csr_host& a) {
    const int64_t n = a.n;
    std::vector<int64_t> trp(n + 1, 0);
    for (int64_t c : a.col) ++trp[c + 1];
    for (int64_t i = 0; i < n; ++i) trp[i + 1] += trp[i];
    if (trp != a.row_ptr) return false;
    std::vector<int64_t> next(trp.begin(), trp.end() - 1), tc(a.col.size());
    std::vector<double> tv(a.val.size());
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            const int64_t j = a.col[k];
            tc[next[j]] = i;
            tv[next[j]] = a.val[k];
            ++next[j];
        }
    return tc == a.col && tv == a.val;
}

// matrix_market.hpp:135-149
void fold_upper(const ktb_csr_host& a, ktb_csr_host& s) {
    s.n = a.n;
    s.kind = KTB_SYM_UPPER;
    s.row_ptr.assign(a.n + 1, 0);
    s.col.clear();
    s.val.clear();
    for (int64_t i = 0; i < a.n; ++i)
        for (int64_t k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k) {
            if (a.col[k] < i) continue;
            s.col.push_back(a.col[k]);
            s.val.push_back(a.val[k]);
            ++s.row_ptr[i + 1];
        }
    for (int64_t i = 0; i < a.n; ++i) s.row_ptr[i + 1] += s.row_ptr[i];
}

}  // namespace

MmHeader mm_probe(const std::string& path) {  // matrix_market.hpp:154-158
    Mapped f(path);
    size_t body = 0;
    return parse_header(f, path, &body);
}

ktb_csr_host* mm_read(const std::string& path, bool want_symmetric) {  // :165-194
    auto out = std::make_unique<ktb_csr_host>();
    MmHeader h;
    std::vector<Part> part;
    {
        Mapped f(path);
        size_t body = 0;
        h = parse_header(f, path, &body);
        part = parse_entries(f, body, h, path);
    }
    ktb_csr_host a;  // coo_to_csr (:89-108), upper triangle for symmetric files
    if (!assemble_sorted(h.n, part, a)) coo_to_csr(h.n, part, a);
    part.clear();
    if (h.symmetric) {
        validate(a, true);
        if (want_symmetric) {
            *out = std::move(a);
            out->kind = KTB_SYM_UPPER;
        } else {
            expand(a, *out);
        }
        return out.release();
    }
    a.kind = KTB_GENERAL;
    validate(a, false);
    if (!want_symmetric) {
        *out = std::move(a);
        return out.release();
    }
    check(exactly_symmetric(a),
          "matrix market: general file is not numerically symmetric: " + path);
    fold_upper(a, *out);
    return out.release();
}

// Loaded CRS -> device matrix. The arrays were validated by mm_read, so
// this pass only narrows the indices to the device's int32 layout and
// gathers the row statistics, in parallel, through a pinned staging ring
// (two 32 MB halves) so the DMA of one chunk overlaps the narrowing of the
// next.
ktb_matrix* mm_upload(const ktb_csr_host& h, int device) {
    const int64_t n = h.n;
    const int64_t nnz = static_cast<int64_t>(h.col.size());
    require(n < (int64_t(1) << 31) - 1 && nnz < (int64_t(1) << 31) - 1,
            "csr: n or nnz >= 2^31 does not fit the int32 device layout");
    DeviceGuard g(device);
    auto m = std::make_unique<ktb_matrix>();
    m->device = device;
    KTB_CUDA(cudaDeviceGetAttribute(&m->sm_count, cudaDevAttrMultiProcessorCount, device));
    m->n = n;
    m->ncols = n;
    m->nnz = nnz;
    m->kind = h.kind;
    m->row_ptr.alloc(n + 1);
    m->col.alloc(nnz);
    m->val.alloc(nnz);
    const int T = static_cast<int>(std::max<size_t>(1, std::min<size_t>(host_threads(), 64)));
    std::vector<int64_t> mx(T, 0), bw(T, 0);
    parallel_for(T, [&](int t) {  // row statistics (csr.hpp max_row_nnz, bandwidth)
        for (int64_t i = n * t / T; i < n * (t + 1) / T; ++i) {
            const int64_t b = h.row_ptr[i], e = h.row_ptr[i + 1];
            mx[t] = std::max(mx[t], e - b);
            if (e > b) bw[t] = std::max(bw[t], h.col[e - 1] - i);
        }
    });
    m->max_row_nnz = *std::max_element(mx.begin(), mx.end());
    m->bandwidth = *std::max_element(bw.begin(), bw.end());

    constexpr size_t kHalf = size_t(32) << 20;
    char* stage = nullptr;
    KTB_CUDA(cudaHostAlloc(&stage, 2 * kHalf, cudaHostAllocDefault));
    cudaStream_t st = nullptr;
    cudaEvent_t done[2] = {nullptr, nullptr};
    auto cleanup = [&] {
        if (st) cudaStreamSynchronize(st);
        for (auto& e : done)
            if (e) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
        cudaFreeHost(stage);
    };
    try {
        KTB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        for (auto& e : done) KTB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        int half = 0;
        bool used[2] = {false, false};
        // fill(dst, k0, k1): writes elements [k0, k1) of one array into dst
        auto pump = [&](void* dev, size_t elem, int64_t count, auto&& fill) {
            const int64_t per = static_cast<int64_t>(kHalf / elem);
            for (int64_t k0 = 0; k0 < count; k0 += per) {
                const int64_t k1 = std::min(count, k0 + per);
                char* buf = stage + half * kHalf;
                if (used[half]) KTB_CUDA(cudaEventSynchronize(done[half]));
                parallel_for(T, [&](int t) {
                    const int64_t a = k0 + (k1 - k0) * t / T, b = k0 + (k1 - k0) * (t + 1) / T;
                    fill(buf, k0, a, b);
                });
                KTB_CUDA(cudaMemcpyAsync(static_cast<char*>(dev) + k0 * elem, buf,
                                         (k1 - k0) * elem, cudaMemcpyHostToDevice, st));
                KTB_CUDA(cudaEventRecord(done[half], st));
                used[half] = true;
                half ^= 1;
            }
        };
        pump(m->row_ptr.p, 4, n + 1, [&](char* buf, int64_t k0, int64_t a, int64_t b) {
            auto* d = reinterpret_cast<int32_t*>(buf) - k0;
            for (int64_t k = a; k < b; ++k) d[k] = static_cast<int32_t>(h.row_ptr[k]);
        });
        pump(m->col.p, 4, nnz, [&](char* buf, int64_t k0, int64_t a, int64_t b) {
            auto* d = reinterpret_cast<int32_t*>(buf) - k0;
            for (int64_t k = a; k < b; ++k) d[k] = static_cast<int32_t>(h.col[k]);
        });
        pump(m->val.p, 8, nnz, [&](char* buf, int64_t k0, int64_t a, int64_t b) {
            std::memcpy(buf + (a - k0) * 8, h.val.data() + a, (b - a) * 8);
        });
        KTB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
    return m.release();
}

// matrix_market.hpp:206-239: general as "i j v", symmetric storage (upper)
// transposed to the conventional lower form; values "%.17g".
void mm_write(const std::string& path, int64_t n, const int64_t* rp, const int64_t* ci,
              const double* v, int kind) {
    std::FILE* out = std::fopen(path.c_str(), "w");
    check(out != nullptr, "matrix market: cannot write " + path);
    std::string buf;
    buf.reserve(size_t(1) << 20);
    buf += kind == KTB_SYM_UPPER ? "%%MatrixMarket matrix coordinate real symmetric\n"
                                 : "%%MatrixMarket matrix coordinate real general\n";
    buf += std::to_string(n) + ' ' + std::to_string(n) + ' ' + std::to_string(rp[n]) + '\n';
    bool ok = true;
    char num[64];
    for (int64_t i = 0; i < n && ok; ++i)
        for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t a = kind == KTB_SYM_UPPER ? ci[k] + 1 : i + 1;
            const int64_t b = kind == KTB_SYM_UPPER ? i + 1 : ci[k] + 1;
            std::snprintf(num, sizeof num, "%.17g", v[k]);
            buf += std::to_string(a);
            buf += ' ';
            buf += std::to_string(b);
            buf += ' ';
            buf += num;
            buf += '\n';
            if (buf.size() > (size_t(1) << 20)) {
                ok = std::fwrite(buf.data(), 1, buf.size(), out) == buf.size();
                buf.clear();
                if (!ok) break;
            }
        }
    if (ok && !buf.empty()) ok = std::fwrite(buf.data(), 1, buf.size(), out) == buf.size();
    ok = std::fclose(out) == 0 && ok;
    check(ok, "matrix market: write failed: " + path);
}

}  // namespace ktb
