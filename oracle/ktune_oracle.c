/*
 * ktune_oracle.c -- TEST INFRASTRUCTURE ONLY (see ktune_oracle.h).
 *
 * Plain-C restatement of the reference's CPU SpMV path. Each function cites
 * the reference file:line it restates (paths relative to
 * /root/reference/proj/include/ktune/). The OpenMP worker loops of the
 * reference are executed serially here: every worker's computation is
 * independent and the cross-worker reductions have a fixed order, so the
 * serial execution is bitwise identical to the parallel one.
 */
#include "ktune_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static const char* const k_messages[] = {
    "ok",
    "csr: negative dimension",                 /* csr.hpp:39 */
    "csr: row_ptr[0] != 0",                    /* csr.hpp:42 */
    "csr: row_ptr[n] != nnz",                  /* csr.hpp:43 */
    "csr: row_ptr not nondecreasing",          /* csr.hpp:45 */
    "csr: column index out of range",          /* csr.hpp:47 */
    "csr: columns not strictly increasing",    /* csr.hpp:49 */
    "sym csr: entry below the diagonal",       /* csr.hpp:51 */
    "row partition: num_workers must be >= 1", /* partition.hpp:30 */
    "bss plan: jl must be >= 1",               /* bss.hpp:35 */
    "bss plan: empty matrix",                  /* bss.hpp:36 */
    "gmres: dimension mismatch",               /* gmres.hpp:19 */
    "gmres: need 1 <= m <= m_max",             /* gmres.hpp:20 */
    "gmres: tol must be positive",             /* gmres.hpp:21 */
};

const char* ko_error_message(int code) {
    if (code < 0 || code >= (int)(sizeof(k_messages) / sizeof(k_messages[0]))) return "?";
    return k_messages[code];
}

/* csr.hpp:38-54 */
int ko_validate(int64_t n, const int64_t* row_ptr, int64_t nnz, const int64_t* col_idx,
                int upper_only) {
    if (n < 0) return 1;
    if (row_ptr[0] != 0) return 2;
    if (row_ptr[n] != nnz) return 3;
    for (int64_t i = 0; i < n; ++i) {
        if (row_ptr[i] > row_ptr[i + 1]) return 4;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            if (col_idx[k] < 0 || col_idx[k] >= n) return 5;
            if (k > row_ptr[i] && !(col_idx[k - 1] < col_idx[k])) return 6;
            if (upper_only && col_idx[k] < i) return 7;
        }
    }
    return 0;
}

/* csr.hpp:69-78: strictly left-to-right row sums. */
void ko_spmv_ref(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += values[k] * x[col_idx[k]];
        y[i] = s;
    }
}

/* csr.hpp:88-96 count pass */
int64_t ko_expand_symmetric_nnz(int64_t n, const int64_t* row_ptr, const int64_t* col_idx) {
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) total += (col_idx[k] != i) ? 2 : 1;
    return total;
}

/* csr.hpp:88-123: mirrored (lower) entries first in ascending source row,
 * then the native upper entries, giving sorted rows. */
void ko_expand_symmetric(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const double* values, int64_t* out_row_ptr, int64_t* out_col_idx,
                         double* out_values) {
    int64_t* count = (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            ++count[i];
            if (col_idx[k] != i) ++count[col_idx[k]];
        }
    out_row_ptr[0] = 0;
    for (int64_t i = 0; i < n; ++i) out_row_ptr[i + 1] = out_row_ptr[i] + count[i];
    int64_t* next = count; /* reuse */
    for (int64_t i = 0; i < n; ++i) next[i] = out_row_ptr[i];
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            const int64_t j = col_idx[k];
            if (j == i) continue;
            out_col_idx[next[j]] = i;
            out_values[next[j]] = values[k];
            ++next[j];
        }
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            out_col_idx[next[i]] = col_idx[k];
            out_values[next[i]] = values[k];
            ++next[i];
        }
    free(count);
}

/* partition.hpp:28-55. NNZ_BALANCED: smallest r in [0, n) with
 * row_ptr[r] * P >= p * nnz (std::lower_bound over row_ptr[0..n)); n if none. */
int ko_build_row_partition(const int64_t* row_ptr, int64_t n, int num_workers, int scheme,
                           int64_t* boundaries) {
    if (num_workers < 1) return 8;
    boundaries[0] = 0;
    boundaries[num_workers] = n;
    if (scheme == 0) {
        for (int p = 1; p < num_workers; ++p) boundaries[p] = n * p / num_workers;
    } else {
        const int64_t nnz = row_ptr[n];
        for (int p = 1; p < num_workers; ++p) {
            const int64_t target = (int64_t)p * nnz;
            int64_t lo = 0, len = n; /* search range [0, n) */
            while (len > 0) {
                const int64_t half = len / 2;
                const int64_t mid = lo + half;
                if (row_ptr[mid] * num_workers < target) {
                    lo = mid + 1;
                    len -= half + 1;
                } else {
                    len = half;
                }
            }
            boundaries[p] = lo;
        }
    }
    return 0;
}

/* partition.hpp:73-96 */
void ko_build_reduction_regions(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                                int num_workers, const int64_t* boundaries, int64_t* lo_out,
                                int64_t* hi_out) {
    for (int p = 0; p < num_workers; ++p) {
        int64_t lo = n, hi = 0;
        for (int64_t i = boundaries[p]; i < boundaries[p + 1]; ++i)
            for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
                const int64_t j = col_idx[k];
                if (j == i) continue;
                if (j < lo) lo = j;
                if (j + 1 > hi) hi = j + 1;
            }
        lo_out[p] = 0;
        hi_out[p] = 0;
        if (hi > lo) {
            lo_out[p] = lo;
            hi_out[p] = hi;
        }
    }
}

/* bss.hpp:34-61 slice walk, shared by the count and fill passes. */
static int64_t bss_walk(int64_t n, const int64_t* row_ptr, int64_t jl, int64_t* slice_start,
                        int64_t* slice_len, int64_t* slice_row, int64_t* lane_slice_ptr) {
    const int64_t nnz = row_ptr[n];
    int64_t row = 0, t = 0;
    if (lane_slice_ptr) lane_slice_ptr[0] = 0;
    for (int64_t p = 0; p < jl; ++p) {
        const int64_t chunk_lo = nnz * p / jl;
        const int64_t chunk_hi = nnz * (p + 1) / jl;
        int64_t pos = chunk_lo;
        while (pos < chunk_hi) {
            while (row_ptr[row + 1] <= pos) ++row;
            const int64_t cut = chunk_hi < row_ptr[row + 1] ? chunk_hi : row_ptr[row + 1];
            if (slice_start) {
                slice_start[t] = pos;
                slice_len[t] = cut - pos;
                slice_row[t] = row;
            }
            ++t;
            pos = cut;
        }
        if (lane_slice_ptr) lane_slice_ptr[p + 1] = t;
    }
    return t;
}

int ko_bss_count(int64_t n, const int64_t* row_ptr, int64_t jl, int64_t* jl_eff,
                 int64_t* total_slices) {
    if (jl < 1) return 9;
    const int64_t nnz = row_ptr[n];
    if (nnz <= 0) return 10;
    *jl_eff = jl < nnz ? jl : nnz;
    *total_slices = bss_walk(n, row_ptr, *jl_eff, NULL, NULL, NULL, NULL);
    return 0;
}

/* bss.hpp:38-69 */
void ko_bss_fill(int64_t n, const int64_t* row_ptr, int64_t jl_eff, int64_t* slice_start,
                 int64_t* slice_len, int64_t* slice_row, int64_t* lane_slice_ptr,
                 int64_t* row_slice_ptr, uint8_t* row_start_flag) {
    const int64_t nnz = row_ptr[n];
    memset(row_start_flag, 0, (size_t)nnz);
    for (int64_t i = 0; i < n; ++i)
        if (row_ptr[i] < row_ptr[i + 1]) row_start_flag[row_ptr[i]] = 1;
    const int64_t total = bss_walk(n, row_ptr, jl_eff, slice_start, slice_len, slice_row,
                                   lane_slice_ptr);
    for (int64_t i = 0; i <= n; ++i) row_slice_ptr[i] = 0;
    for (int64_t t = 0; t < total; ++t) ++row_slice_ptr[slice_row[t] + 1];
    for (int64_t i = 0; i < n; ++i) row_slice_ptr[i + 1] += row_slice_ptr[i];
}

/* spmv.hpp:74-86 */
void ko_spmv_row_blocks(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                        const double* values, int num_workers, const int64_t* boundaries,
                        const double* x, double* y) {
    (void)n;
    for (int p = 0; p < num_workers; ++p)
        for (int64_t i = boundaries[p]; i < boundaries[p + 1]; ++i) {
            double s = 0.0;
            for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) s += values[k] * x[col_idx[k]];
            y[i] = s;
        }
}

/* spmv.hpp:127-166 slice phase, then spmv.hpp:91-101 ordered combine. */
void ko_spmv_bss(int u4, int64_t n, const int64_t* col_idx, const double* values, int64_t jl,
                 const int64_t* slice_start, const int64_t* slice_len,
                 const int64_t* lane_slice_ptr, const int64_t* row_slice_ptr,
                 const uint8_t* row_start_flag, const double* x, double* sums, double* y) {
    if (!u4) {
        for (int64_t p = 0; p < jl; ++p)
            for (int64_t t = lane_slice_ptr[p]; t < lane_slice_ptr[p + 1]; ++t) {
                const int64_t lo = slice_start[t], hi = lo + slice_len[t];
                double s = 0.0;
                for (int64_t k = lo; k < hi; ++k) s += values[k] * x[col_idx[k]];
                sums[t] = s;
            }
    } else {
        for (int64_t p = 0; p < jl; ++p) {
            int64_t t = lane_slice_ptr[p];
            const int64_t lo = slice_start[t];
            const int64_t last = lane_slice_ptr[p + 1] - 1;
            const int64_t hi = slice_start[last] + slice_len[last];
            double s = 0.0;
            for (int64_t k = lo; k < hi; ++k) {
                if (k != lo && row_start_flag[k]) {
                    sums[t++] = s;
                    s = 0.0;
                }
                s += values[k] * x[col_idx[k]];
            }
            sums[t] = s;
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t t = row_slice_ptr[i]; t < row_slice_ptr[i + 1]; ++t) s += sums[t];
        y[i] = s;
    }
}

/* spmv.hpp:180-234 */
void ko_spmv_sym(int kernel, int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, int num_workers, const int64_t* boundaries,
                 const int64_t* lo, const int64_t* hi, int pool_size, const double* x,
                 double* y, double* scratch) {
    const int omit = (kernel == 2);
    for (int p = 0; p < num_workers; ++p) {
        double* sp = scratch + (size_t)p * (size_t)n;
        if (omit) {
            for (int64_t j = lo[p]; j < hi[p]; ++j) sp[j] = 0.0;
        } else {
            for (int64_t j = 0; j < n; ++j) sp[j] = 0.0;
        }
        for (int64_t i = boundaries[p]; i < boundaries[p + 1]; ++i) {
            const double xi = x[i];
            double s = 0.0;
            for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
                const int64_t j = col_idx[k];
                const double v = values[k];
                s += v * x[j];
                if (j != i) sp[j] += v * xi;
            }
            y[i] = s;
        }
    }
    const int red_chunks = pool_size;
    for (int c = 0; c < red_chunks; ++c) {
        const int64_t c_lo = n * c / red_chunks;
        const int64_t c_hi = n * (c + 1) / red_chunks;
        for (int p = 0; p < num_workers; ++p) {
            const double* sp = scratch + (size_t)p * (size_t)n;
            const int64_t l = omit ? (lo[p] > c_lo ? lo[p] : c_lo) : c_lo;
            const int64_t h = omit ? (hi[p] < c_hi ? hi[p] : c_hi) : c_hi;
            for (int64_t j = l; j < h; ++j) y[j] += sp[j];
        }
    }
}

/* lanczos.hpp:17-29 */
void ko_seeded_vector(int64_t n, uint64_t seed, double* out) {
    uint64_t state = seed;
    for (int64_t i = 0; i < n; ++i) {
        state += 0x9e3779b97f4a7c15ull;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        out[i] = (double)(z >> 11) / 4503599627370496.0 - 1.0;
    }
}

/* autotune.hpp:188-196 */
void ko_probe_vector(int64_t n, double* out) {
    uint64_t state = 0x9e3779b97f4a7c15ull;
    for (int64_t i = 0; i < n; ++i) {
        state = state * 6364136223846793005ull + 1442695040888963407ull;
        out[i] = 0.5 + (double)(state >> 11) / 9007199254740992.0;
    }
}

/* autotune.hpp:198-204 */
int ko_outputs_match(int64_t n, const double* y, const double* ref) {
    double scale = 1.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs(ref[i]);
        scale = (scale < a) ? a : scale; /* std::max(scale, |r|), NaN-faithful */
    }
    for (int64_t i = 0; i < n; ++i)
        if (fabs(y[i] - ref[i]) > 1e-10 * scale) return 0;
    return 1;
}

/* common.hpp:33-41 */
double ko_dot(int64_t n, const double* a, const double* b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

double ko_norm2(int64_t n, const double* a) { return sqrt(ko_dot(n, a, a)); }

/* common.hpp:50-52 */
static void axpy(int64_t n, double alpha, const double* x, double* y) {
    for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}

/* gmres.hpp:16-173 with OrthoKind::mgs (ortho.hpp:69-111), identity
 * preconditioner (copy, gmres.hpp:53-58), adapt_restart = false. */
int ko_gmres_mgs(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                 const double* values, const double* b, int64_t m, double tol,
                 int64_t max_iters, double* x, double* history, ko_gmres_result* res) {
    if (m < 1) return 12;
    if (!(tol > 0.0)) return 13;
    memset(res, 0, sizeof(*res));
    for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
    const double nb = ko_norm2(n, b);
    if (nb == 0.0) {
        res->converged = 1;
        return 0;
    }
    const int64_t r_stride = m + 1;
    double* basis = (double*)malloc(sizeof(double) * (size_t)n * (size_t)(m + 1));
    double* r_cols = (double*)malloc(sizeof(double) * (size_t)(r_stride * m));
    double* h = (double*)calloc((size_t)(m + 2), sizeof(double));
    double* cs = (double*)calloc((size_t)(m + 1), sizeof(double));
    double* sn = (double*)calloc((size_t)(m + 1), sizeof(double));
    double* g = (double*)calloc((size_t)(m + 2), sizeof(double));
    double* yv = (double*)calloc((size_t)(m + 1), sizeof(double));
    double* r = (double*)malloc(sizeof(double) * (size_t)n);
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    double* w = (double*)malloc(sizeof(double) * (size_t)n);

    double rr = 1.0;
    int stop = 0;
    while (!stop) {
        ko_spmv_ref(n, row_ptr, col_idx, values, x, r);
        res->spmv_calls++;
        for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
        const double beta = ko_norm2(n, r);
        rr = beta / nb;
        if (rr < tol) {
            res->converged = 1;
            break;
        }
        for (int64_t i = 0; i < n; ++i) basis[i] = r[i] / beta;
        for (int64_t i = 0; i < m + 2; ++i) g[i] = 0.0;
        g[0] = beta;

        int64_t j = 0;
        int lucky = 0;
        while (j < m) {
            if (res->iterations >= max_iters) {
                stop = 1;
                break;
            }
            memcpy(z, basis + j * n, sizeof(double) * (size_t)n);
            ko_spmv_ref(n, row_ptr, col_idx, values, z, w);
            res->spmv_calls++;

            /* ortho.hpp:69-111, MGS over k = j+1 columns */
            const int64_t k = j + 1;
            const double input_norm = ko_norm2(n, w);
            for (int64_t q = 0; q <= k; ++q) h[q] = 0.0;
            for (int64_t q = 0; q < k; ++q) {
                const double c = ko_dot(n, basis + q * n, w);
                axpy(n, -c, basis + q * n, w);
                h[q] += c;
            }
            const double nrm = ko_norm2(n, w);
            h[k] = nrm;
            if (nrm <= 1e-14 * input_norm) {
                h[j + 1] = 0.0;
                lucky = 1;
            } else {
                const double inv = 1.0 / nrm;
                for (int64_t i = 0; i < n; ++i) w[i] *= inv;
                memcpy(basis + (j + 1) * n, w, sizeof(double) * (size_t)n);
            }

            for (int64_t i = 0; i < j; ++i) {
                const double t1 = h[i], t2 = h[i + 1];
                h[i] = cs[i] * t1 + sn[i] * t2;
                h[i + 1] = -sn[i] * t1 + cs[i] * t2;
            }
            const double denom = hypot(h[j], h[j + 1]);
            if (denom == 0.0) {
                cs[j] = 1.0;
                sn[j] = 0.0;
            } else {
                cs[j] = h[j] / denom;
                sn[j] = h[j + 1] / denom;
            }
            h[j] = denom;
            g[j + 1] = -sn[j] * g[j];
            g[j] *= cs[j];
            for (int64_t q = 0; q <= j; ++q) r_cols[j * r_stride + q] = h[q];

            res->iterations++;
            rr = fabs(g[j + 1]) / nb;
            if (history) history[res->iterations - 1] = rr;
            ++j;
            if (lucky || rr < tol) break;
        }

        if (j > 0) {
            for (int64_t i = j - 1; i >= 0; --i) {
                double s = g[i];
                for (int64_t l = i + 1; l < j; ++l) s -= r_cols[l * r_stride + i] * yv[l];
                const double rii = r_cols[i * r_stride + i];
                yv[i] = rii != 0.0 ? s / rii : 0.0;
            }
            for (int64_t i = 0; i < n; ++i) w[i] = 0.0;
            for (int64_t l = 0; l < j; ++l) axpy(n, yv[l], basis + l * n, w);
            memcpy(z, w, sizeof(double) * (size_t)n);
            axpy(n, 1.0, z, x);
        }
        if (rr < tol) {
            res->converged = 1;
            break;
        }
        if (lucky) {
            res->breakdown = 1;
            break;
        }
        if (stop) break;
        res->restarts++;
    }

    res->recurrence_residual = rr;
    ko_spmv_ref(n, row_ptr, col_idx, values, x, r);
    res->spmv_calls++;
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    res->true_residual = ko_norm2(n, r) / nb;
    res->fault_convergence = res->converged && res->true_residual > tol;

    free(basis); free(r_cols); free(h); free(cs); free(sn); free(g); free(yv);
    free(r); free(z); free(w);
    return 0;
}

/* ilu0.hpp:23-69 */
int64_t ko_ilu0_factorize(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                          double* values, int64_t* diag_ptr) {
    for (int64_t i = 0; i < n; ++i) {
        diag_ptr[i] = -1;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
            if (col_idx[k] == i) {
                diag_ptr[i] = k;
                break;
            }
        if (diag_ptr[i] < 0) return -(1 + i);
    }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t kp = row_ptr[i]; kp < row_ptr[i + 1]; ++kp) {
            const int64_t k = col_idx[kp];
            if (k >= i) break;
            const double pivot = values[diag_ptr[k]];
            if (pivot == 0.0) return 1 + k;
            const double lik = values[kp] / pivot;
            values[kp] = lik;
            int64_t pi = kp + 1, pk = diag_ptr[k] + 1;
            while (pi < row_ptr[i + 1] && pk < row_ptr[k + 1]) {
                if (col_idx[pi] == col_idx[pk]) {
                    values[pi] -= lik * values[pk];
                    ++pi;
                    ++pk;
                } else if (col_idx[pi] < col_idx[pk]) {
                    ++pi;
                } else {
                    ++pk;
                }
            }
        }
        if (values[diag_ptr[i]] == 0.0) return 1 + i;
    }
    return 0;
}

/* ilu0.hpp:73-87 */
void ko_ilu0_apply(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                   const double* values, const int64_t* diag_ptr, const double* r, double* z) {
    for (int64_t i = 0; i < n; ++i) {
        double s = r[i];
        for (int64_t k = row_ptr[i]; col_idx[k] < i; ++k) s -= values[k] * z[col_idx[k]];
        z[i] = s;
    }
    for (int64_t i = n - 1; i >= 0; --i) {
        double s = z[i];
        for (int64_t k = diag_ptr[i] + 1; k < row_ptr[i + 1]; ++k) s -= values[k] * z[col_idx[k]];
        z[i] = s / values[diag_ptr[i]];
    }
}
