/*
 * rkfac_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C, FP64, single-threaded restatement of the reference's randomized K-FAC hot path
 * (arXiv 2206.15397 desk implementation under /root/reference/proj/include/rkfac).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this library.  The CUDA product path never links or calls it.
 *
 * Every function names the reference file:line it restates.  Loop orders follow the reference so
 * that, on the same inputs, results are bitwise identical to the reference build in oracle/_ref
 * (pinned by tests/test_oracle.py against tests/golden/ fixtures generated from oracle/_ref).
 *
 * Layout: row-major double, element (i,j) of an m x n matrix at [i*n + j] (matrix.hpp:47-48).
 * Status codes mirror include/rkfac_b200.h (errors.hpp:8-34).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_DIMENSION_MISMATCH 1
#define ORC_RANK_DEFICIENT 2
#define ORC_NO_CONVERGENCE 3
#define ORC_DAMPING_NONPOSITIVE 4
#define ORC_ALLOC 7

/* ------------------------------------------------------------------ rng.hpp */

/* rng.hpp:13-18 */
uint64_t orc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* rng.hpp:32-36  RngState(seed).substream(a, b).seed */
uint64_t orc_substream(uint64_t seed, uint64_t a, uint64_t b) {
    return orc_splitmix64(seed ^ orc_splitmix64(a ^ orc_splitmix64(b)));
}

/* rng.hpp:38-45 */
static double uniform_at(uint64_t seed, uint64_t ctr) {
    const uint64_t u = orc_splitmix64(seed ^ orc_splitmix64(ctr));
    return ((double)(u >> 11) + 1.0) * 0x1.0p-53;
}

/* rng.hpp:51-55: Box-Muller, cos branch only, two counters per normal. */
double orc_gaussian_at(uint64_t seed, uint64_t ctr) {
    const double u1 = uniform_at(seed, ctr);
    const double u2 = uniform_at(seed, ctr + 1);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793238462643383279502884 * u2);
}

/* rng.hpp:59-63: m x n row-major fill; draw k uses counters counter0 + 2k, +2k+1.
 * Returns the advanced counter (counter0 + 2*m*n). */
uint64_t orc_sample_gaussian(uint64_t seed, uint64_t counter0, size_t m, size_t n, double* out) {
    const size_t total = m * n;
    for (size_t k = 0; k < total; ++k) out[k] = orc_gaussian_at(seed, counter0 + 2 * (uint64_t)k);
    return counter0 + 2 * (uint64_t)total;
}

/* --------------------------------------------------------------- matrix.hpp */

/* matrix.hpp:75-89  C(m x n) = A(m x k) B(k x n), ikj, skipping a_ik == 0. */
static void mm(const double* a, const double* b, double* c, size_t m, size_t k, size_t n) {
    memset(c, 0, sizeof(double) * m * n);
    for (size_t i = 0; i < m; ++i) {
        double* crow = c + i * n;
        for (size_t kk = 0; kk < k; ++kk) {
            const double aik = a[i * k + kk];
            if (aik == 0.0) continue;
            const double* brow = b + kk * n;
            for (size_t j = 0; j < n; ++j) crow[j] += aik * brow[j];
        }
    }
}

/* matrix.hpp:92-107  C(ac x bc) = A^T B, A is r x ac, B is r x bc. */
static void mm_at_b(const double* a, const double* b, double* c, size_t r, size_t ac, size_t bc) {
    memset(c, 0, sizeof(double) * ac * bc);
    for (size_t k = 0; k < r; ++k) {
        const double* arow = a + k * ac;
        const double* brow = b + k * bc;
        for (size_t i = 0; i < ac; ++i) {
            const double aki = arow[i];
            if (aki == 0.0) continue;
            double* crow = c + i * bc;
            for (size_t j = 0; j < bc; ++j) crow[j] += aki * brow[j];
        }
    }
}

/* matrix.hpp:110-124  C(ar x br) = A B^T, A is ar x k, B is br x k. */
static void mm_a_bt(const double* a, const double* b, double* c, size_t ar, size_t k, size_t br) {
    for (size_t i = 0; i < ar; ++i) {
        const double* arow = a + i * k;
        for (size_t j = 0; j < br; ++j) {
            const double* brow = b + j * k;
            double s = 0.0;
            for (size_t kk = 0; kk < k; ++kk) s += arow[kk] * brow[kk];
            c[i * br + j] = s;
        }
    }
}

/* matrix.hpp:189-196 */
static void symmetrize(double* a, size_t n) {
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j) {
            const double v = 0.5 * (a[i * n + j] + a[j * n + i]);
            a[i * n + j] = v;
            a[j * n + i] = v;
        }
}

static double max_abs_of(const double* a, size_t len) {
    double m = 0.0;
    for (size_t i = 0; i < len; ++i) m = fmax(m, fabs(a[i]));
    return m;
}

/* ------------------------------------------------------------------- qr.hpp */

/* qr.hpp:23-87  Householder thin QR, diag(R) >= 0; numerically-zero pivots are skipped
 * (or RankDeficient when strict).  q: m x n, r: n x n (r may be NULL). */
int orc_qr_thin(const double* x, size_t m, size_t n, int strict, double* q, double* r) {
    if (m < n) return ORC_DIMENSION_MISMATCH;
    double* a = (double*)malloc(sizeof(double) * m * n);
    double* vs = (double*)malloc(sizeof(double) * m * (n ? n : 1)); /* v_k stored at vs + k*m */
    size_t* vlen = (size_t*)calloc(n ? n : 1, sizeof(size_t));
    double* betas = (double*)calloc(n ? n : 1, sizeof(double));
    double* rr = (double*)calloc(n * n ? n * n : 1, sizeof(double));
    if (!a || !vs || !vlen || !betas || !rr) return ORC_ALLOC;
    memcpy(a, x, sizeof(double) * m * n);
    int status = ORC_OK;

    for (size_t k = 0; k < n; ++k) {
        double norm = 0.0;
        for (size_t i = k; i < m; ++i) norm += a[i * n + k] * a[i * n + k];
        norm = sqrt(norm);
        if (norm < 1e-300) {
            if (strict) { status = ORC_RANK_DEFICIENT; goto done; }
            continue;
        }
        double* v = vs + k * m;
        const size_t len = m - k;
        for (size_t i = k; i < m; ++i) v[i - k] = a[i * n + k];
        const double alpha = (v[0] >= 0.0) ? -norm : norm;
        v[0] -= alpha;
        double vtv = 0.0;
        for (size_t i = 0; i < len; ++i) vtv += v[i] * v[i];
        if (vtv < 1e-300) continue;
        const double beta = 2.0 / vtv;
        for (size_t j = k; j < n; ++j) {
            double s = 0.0;
            for (size_t i = k; i < m; ++i) s += v[i - k] * a[i * n + j];
            s *= beta;
            for (size_t i = k; i < m; ++i) a[i * n + j] -= s * v[i - k];
        }
        a[k * n + k] = alpha;
        for (size_t i = k + 1; i < m; ++i) a[i * n + k] = 0.0;
        vlen[k] = len;
        betas[k] = beta;
    }

    memset(q, 0, sizeof(double) * m * n);
    for (size_t j = 0; j < n; ++j) q[j * n + j] = 1.0;
    for (size_t k = n; k-- > 0;) {
        if (vlen[k] == 0) continue;
        const double* v = vs + k * m;
        const double beta = betas[k];
        for (size_t j = 0; j < n; ++j) {
            double s = 0.0;
            for (size_t i = k; i < m; ++i) s += v[i - k] * q[i * n + j];
            s *= beta;
            for (size_t i = k; i < m; ++i) q[i * n + j] -= s * v[i - k];
        }
    }
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i; j < n; ++j) rr[i * n + j] = a[i * n + j];
    for (size_t k = 0; k < n; ++k) {
        if (rr[k * n + k] >= 0.0) continue;
        for (size_t j = k; j < n; ++j) rr[k * n + j] = -rr[k * n + j];
        for (size_t i = 0; i < m; ++i) q[i * n + k] = -q[i * n + k];
    }
    if (r) memcpy(r, rr, sizeof(double) * n * n);
done:
    free(a); free(vs); free(vlen); free(betas); free(rr);
    return status;
}

/* ------------------------------------------------------------------ eig.hpp */

/* eig.hpp:33-124  Householder tridiagonalisation, transposed accumulation (row i of v is
 * eigenvector i on exit of tql2). */
static void tred2(double* v, size_t n, double* d, double* e) {
    for (size_t j = 0; j < n; ++j) d[j] = v[(n - 1) * n + j];
    for (size_t i = n - 1; i > 0; --i) {
        double scale = 0.0, h = 0.0;
        for (size_t k = 0; k < i; ++k) scale += fabs(d[k]);
        if (scale == 0.0) {
            e[i] = d[i - 1];
            for (size_t j = 0; j < i; ++j) {
                d[j] = v[(i - 1) * n + j];
                v[i * n + j] = 0.0;
                v[j * n + i] = 0.0;
            }
        } else {
            for (size_t k = 0; k < i; ++k) {
                d[k] /= scale;
                h += d[k] * d[k];
            }
            double f = d[i - 1];
            double g = sqrt(h);
            if (f > 0.0) g = -g;
            e[i] = scale * g;
            h -= f * g;
            d[i - 1] = f - g;
            for (size_t j = 0; j < i; ++j) {
                v[j * n + i] = d[j];
                const double* row = v + j * n;
                double s = 0.0;
                for (size_t k = 0; k < i; ++k) s += row[k] * d[k];
                e[j] = s;
            }
            f = 0.0;
            for (size_t j = 0; j < i; ++j) {
                e[j] /= h;
                f += e[j] * d[j];
            }
            const double hh = f / (h + h);
            for (size_t j = 0; j < i; ++j) e[j] -= hh * d[j];
            for (size_t r = 0; r < i; ++r) {
                const double dr = d[r], er = e[r];
                double* row = v + r * n;
                for (size_t c = 0; c < i; ++c) row[c] -= dr * e[c] + er * d[c];
            }
            for (size_t j = 0; j < i; ++j) {
                d[j] = v[(i - 1) * n + j];
                v[i * n + j] = 0.0;
            }
        }
        d[i] = h;
    }
    double* w = (double*)malloc(sizeof(double) * n * n);
    double* diag = (double*)malloc(sizeof(double) * n);
    for (size_t r = 0; r < n; ++r)
        for (size_t c = 0; c < n; ++c) w[r * n + c] = v[c * n + r];
    for (size_t i = 0; i + 1 < n; ++i) {
        diag[i] = w[i * n + i];
        w[i * n + i] = 1.0;
        const double h = d[i + 1];
        if (h != 0.0) {
            const double* hv = w + (i + 1) * n;
            for (size_t k = 0; k <= i; ++k) d[k] = hv[k] / h;
            for (size_t j = 0; j <= i; ++j) {
                double* row = w + j * n;
                double g = 0.0;
                for (size_t k = 0; k <= i; ++k) g += hv[k] * row[k];
                for (size_t k = 0; k <= i; ++k) row[k] -= g * d[k];
            }
        }
        double* next = w + (i + 1) * n;
        for (size_t k = 0; k <= i; ++k) next[k] = 0.0;
    }
    diag[n - 1] = w[(n - 1) * n + (n - 1)];
    for (size_t j = 0; j < n; ++j) {
        d[j] = diag[j];
        w[j * n + (n - 1)] = 0.0;
    }
    w[(n - 1) * n + (n - 1)] = 1.0;
    e[0] = 0.0;
    memcpy(v, w, sizeof(double) * n * n);
    free(w);
    free(diag);
}

/* eig.hpp:131-193  implicit-shift QL; throws NoConvergence past 60 iterations per eigenvalue. */
static int tql2(double* v, size_t n, double* d, double* e, int max_iter) {
    for (size_t i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    double f = 0.0, tst1 = 0.0;
    const double eps = pow(2.0, -52.0);
    for (size_t l = 0; l < n; ++l) {
        tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
        size_t m = l;
        while (m < n && fabs(e[m]) > eps * tst1) ++m;
        if (m > l) {
            int iter = 0;
            do {
                if (++iter > max_iter) return ORC_NO_CONVERGENCE;
                double g = d[l];
                double p = (d[l + 1] - g) / (2.0 * e[l]);
                double r = hypot(p, 1.0);
                if (p < 0.0) r = -r;
                d[l] = e[l] / (p + r);
                d[l + 1] = e[l] * (p + r);
                const double dl1 = d[l + 1];
                double h = g - d[l];
                for (size_t i = l + 2; i < n; ++i) d[i] -= h;
                f += h;
                p = d[m];
                double c = 1.0, c2 = c, c3 = c;
                const double el1 = e[l + 1];
                double s = 0.0, s2 = 0.0;
                for (size_t i = m; i-- > l;) {
                    c3 = c2;
                    c2 = c;
                    s2 = s;
                    g = c * e[i];
                    h = c * p;
                    r = hypot(p, e[i]);
                    e[i + 1] = s * r;
                    s = e[i] / r;
                    c = p / r;
                    p = c * d[i] - s * g;
                    d[i + 1] = h + s * (c * g + s * d[i]);
                    double* vi = v + i * n;
                    double* vi1 = v + (i + 1) * n;
                    for (size_t k = 0; k < n; ++k) {
                        h = vi1[k];
                        vi1[k] = s * vi[k] + c * h;
                        vi[k] = c * vi[k] - s * h;
                    }
                }
                p = -s * s2 * c3 * el1 * e[l] / dl1;
                e[l] = s * p;
                d[l] = c * p;
            } while (fabs(e[l]) > eps * tst1);
        }
        d[l] += f;
        e[l] = 0.0;
    }
    return ORC_OK;
}

/* eig.hpp:210-237  S = P diag(d) P^T, d descending (stable), eigenvectors as columns of P. */
int orc_sym_eig(const double* s, size_t n, double* p, double* dout) {
    const double scale_ref = fmax(1.0, max_abs_of(s, n * n));
    double asym = 0.0;
    for (size_t i = 0; i < n; ++i)
        for (size_t j = i + 1; j < n; ++j) asym = fmax(asym, fabs(s[i * n + j] - s[j * n + i]));
    if (asym > 1e-8 * scale_ref) return ORC_DIMENSION_MISMATCH;
    if (n == 0) return ORC_OK;
    double* v = (double*)malloc(sizeof(double) * n * n);
    double* d = (double*)malloc(sizeof(double) * n);
    double* e = (double*)calloc(n, sizeof(double));
    size_t* idx = (size_t*)malloc(sizeof(size_t) * n);
    if (!v || !d || !e || !idx) return ORC_ALLOC;
    memcpy(v, s, sizeof(double) * n * n);
    symmetrize(v, n);
    int st = ORC_OK;
    if (n == 1) {
        p[0] = 1.0;
        dout[0] = v[0];
        goto out;
    }
    tred2(v, n, d, e);
    st = tql2(v, n, d, e, 60);
    if (st) goto out;
    /* eig.hpp:197-203 stable descending sort (insertion sort is stable). */
    for (size_t i = 0; i < n; ++i) idx[i] = i;
    for (size_t i = 1; i < n; ++i) {
        const size_t key = idx[i];
        size_t j = i;
        while (j > 0 && d[idx[j - 1]] < d[key]) {
            idx[j] = idx[j - 1];
            --j;
        }
        idx[j] = key;
    }
    for (size_t j = 0; j < n; ++j) {
        dout[j] = d[idx[j]];
        const double* row = v + idx[j] * n;
        for (size_t i = 0; i < n; ++i) p[i * n + j] = row[i];
    }
out:
    free(v); free(d); free(e); free(idx);
    return st;
}

/* ----------------------------------------------------------------- rnla.hpp */

/* rnla.hpp:35-43 */
void orc_clamp_sketch(size_t dim, size_t* r, size_t* p) {
    if (*r > dim) {
        *r = dim;
        *p = 0;
    } else if (*r + *p > dim) {
        *p = dim - *r;
    }
}

/* rnla.hpp:47-56  Q (d x w) spans X Omega after q power iterations; re-orthonormalised every
 * half step.  X is square (d x d) on the hot path. */
static int randomized_range(const double* x, size_t d, size_t w, size_t q_iters, uint64_t seed,
                            uint64_t* counter, double* q) {
    double* omega = (double*)malloc(sizeof(double) * d * w);
    double* y = (double*)malloc(sizeof(double) * d * w);
    double* z = (double*)malloc(sizeof(double) * d * w);
    if (!omega || !y || !z) return ORC_ALLOC;
    *counter = orc_sample_gaussian(seed, *counter, d, w, omega);
    mm(x, omega, y, d, d, w);
    int st = orc_qr_thin(y, d, w, 0, q, NULL);
    for (size_t t = 0; t < q_iters && !st; ++t) {
        mm_at_b(x, q, y, d, d, w);          /* X^T Q  (rnla.hpp:52) */
        st = orc_qr_thin(y, d, w, 0, z, NULL);
        if (st) break;
        mm(x, z, y, d, d, w);                /* X Z    (rnla.hpp:53) */
        st = orc_qr_thin(y, d, w, 0, q, NULL);
    }
    free(omega); free(y); free(z);
    return st;
}

/* rnla.hpp:90-105  srevd.  u: d x r_eff, dv: r_eff, with r_eff = clamped rank (written to *r_out).
 * (seed, *counter) is the RngState; the counter is advanced by 2*d*w like the reference. */
int orc_srevd(const double* x, size_t d, size_t r_in, size_t p_in, size_t q_iters, uint64_t seed,
              uint64_t* counter, double* u, double* dv, size_t* r_out) {
    size_t r = r_in, p = p_in;
    orc_clamp_sketch(d, &r, &p);
    const size_t w = r + p;
    double* q = (double*)malloc(sizeof(double) * d * w);
    double* xq = (double*)malloc(sizeof(double) * d * w);
    double* c = (double*)malloc(sizeof(double) * w * w);
    double* pm = (double*)malloc(sizeof(double) * w * w);
    double* ev = (double*)malloc(sizeof(double) * w);
    double* pr = (double*)malloc(sizeof(double) * w * (r ? r : 1));
    if (!q || !xq || !c || !pm || !ev || !pr) return ORC_ALLOC;
    int st = randomized_range(x, d, w, q_iters, seed, counter, q);
    if (!st) {
        mm(x, q, xq, d, d, w);
        mm_at_b(q, xq, c, d, w, w);
        symmetrize(c, w);
        st = orc_sym_eig(c, w, pm, ev);
    }
    if (!st) {
        for (size_t i = 0; i < w; ++i)
            for (size_t j = 0; j < r; ++j) pr[i * r + j] = pm[i * w + j];
        mm(q, pr, u, d, w, r);
        for (size_t j = 0; j < r; ++j) dv[j] = fmax(0.0, ev[j]);
        *r_out = r;
    }
    free(q); free(xq); free(c); free(pm); free(ev); free(pr);
    return st;
}

/* eig.hpp:243-299  svd_small for an m x n input with m >= n (the only case on the hot path:
 * svd_small(transpose(B)) with B = Q^T X of shape w x d, rnla.hpp:72).  Outputs the thin
 * u (m x n), s (n), v (n x n). */
static int svd_small_tall(const double* x, size_t m, size_t n, double* u, double* s, double* v) {
    double* gram = (double*)malloc(sizeof(double) * n * n);
    double* xv = (double*)malloc(sizeof(double) * m * n);
    double* wv = (double*)malloc(sizeof(double) * m);
    size_t* zero_modes = (size_t*)malloc(sizeof(size_t) * (n ? n : 1));
    if (!gram || !xv || !wv || !zero_modes) return ORC_ALLOC;
    mm_at_b(x, x, gram, m, n, n);
    symmetrize(gram, n);
    int st = orc_sym_eig(gram, n, v, s);
    if (st) goto out;
    for (size_t i = 0; i < n; ++i) s[i] = sqrt(fmax(0.0, s[i]));
    {
        const double smax = n ? s[0] : 0.0;
        const double tiny = fmax(smax * 1e-13, 1e-300);
        mm(x, v, xv, m, n, n);
        memset(u, 0, sizeof(double) * m * n);
        size_t nz = 0;
        for (size_t j = 0; j < n; ++j) {
            if (s[j] > tiny) {
                for (size_t i = 0; i < m; ++i) u[i * n + j] = xv[i * n + j] / s[j];
            } else {
                s[j] = 0.0;
                zero_modes[nz++] = j;
            }
        }
        /* eig.hpp:272-296 orthonormal completion of zero modes with canonical vectors. */
        size_t cand = 0;
        for (size_t zi = 0; zi < nz; ++zi) {
            const size_t j = zero_modes[zi];
            for (; cand < m; ++cand) {
                memset(wv, 0, sizeof(double) * m);
                wv[cand] = 1.0;
                for (int pass = 0; pass < 2; ++pass) {
                    for (size_t jj = 0; jj < n; ++jj) {
                        if (s[jj] == 0.0 && jj >= j) continue;
                        double dot = 0.0;
                        for (size_t i = 0; i < m; ++i) dot += wv[i] * u[i * n + jj];
                        for (size_t i = 0; i < m; ++i) wv[i] -= dot * u[i * n + jj];
                    }
                }
                double norm = 0.0;
                for (size_t i = 0; i < m; ++i) norm += wv[i] * wv[i];
                norm = sqrt(norm);
                if (norm > 1e-8) {
                    for (size_t i = 0; i < m; ++i) u[i * n + j] = wv[i] / norm;
                    ++cand;
                    break;
                }
            }
        }
    }
out:
    free(gram); free(xv); free(wv); free(zero_modes);
    return st;
}

/* rnla.hpp:62-77 + 81-85  rsvd_psd: keeps the V-side basis B^T P_r / s_r and s_r. */
int orc_rsvd_psd(const double* x, size_t d, size_t r_in, size_t p_in, size_t q_iters, uint64_t seed,
                 uint64_t* counter, double* u, double* dv, size_t* r_out) {
    size_t r = r_in, p = p_in;
    orc_clamp_sketch(d, &r, &p);
    const size_t w = r + p;
    double* q = (double*)malloc(sizeof(double) * d * w);
    double* b = (double*)malloc(sizeof(double) * w * d);
    double* bt = (double*)malloc(sizeof(double) * d * w);
    double* cu = (double*)malloc(sizeof(double) * d * w);
    double* cs = (double*)malloc(sizeof(double) * w);
    double* cv = (double*)malloc(sizeof(double) * w * w);
    if (!q || !b || !bt || !cu || !cs || !cv) return ORC_ALLOC;
    int st = randomized_range(x, d, w, q_iters, seed, counter, q);
    if (!st) {
        mm_at_b(q, x, b, d, w, d); /* B = Q^T X, w x d (rnla.hpp:69) */
        for (size_t i = 0; i < w; ++i)
            for (size_t j = 0; j < d; ++j) bt[j * w + i] = b[i * d + j];
        st = svd_small_tall(bt, d, w, cu, cs, cv);
    }
    if (!st) {
        for (size_t i = 0; i < d; ++i)
            for (size_t j = 0; j < r; ++j) u[i * r + j] = cu[i * w + j];
        for (size_t j = 0; j < r; ++j) dv[j] = cs[j];
        *r_out = r;
    }
    free(q); free(b); free(bt); free(cu); free(cs); free(cv);
    return st;
}

/* -------------------------------------------------------------- kfactor.hpp */

/* kfactor.hpp:33-41  mbar <- rho*mbar + (1-rho) m m^T, then symmetrize.  m is d x n. */
int orc_ea_update(double* mbar, size_t d, const double* m, size_t rows_m, size_t n, double rho) {
    if (rows_m != d) return ORC_DIMENSION_MISMATCH;
    double* outer = (double*)malloc(sizeof(double) * (d * d ? d * d : 1));
    if (!outer) return ORC_ALLOC;
    mm_a_bt(m, m, outer, d, n, d);
    for (size_t i = 0; i < d * d; ++i) mbar[i] = rho * mbar[i] + (1.0 - rho) * outer[i];
    symmetrize(mbar, d);
    free(outer);
    return ORC_OK;
}

/* kfactor.hpp:134-161  side 0 = LEFT: (U D U^T + l I)^{-1} V;  side 1 = RIGHT: V (U D U^T + l I)^{-1}.
 * u is dim x r, v is rows x cols, out has v's shape. */
int orc_apply_lowrank_damped_inverse(const double* u, const double* dv, size_t dim, size_t r,
                                     double lambda, const double* v, size_t rows, size_t cols,
                                     int side, double* out) {
    if (lambda <= 0.0) return ORC_DAMPING_NONPOSITIVE;
    double* bracket = (double*)malloc(sizeof(double) * (r ? r : 1));
    if (!bracket) return ORC_ALLOC;
    for (size_t i = 0; i < r; ++i) bracket[i] = 1.0 / (dv[i] + lambda) - 1.0 / lambda;
    if (side == 0) {
        if (rows != dim) { free(bracket); return ORC_DIMENSION_MISMATCH; }
        double* w = (double*)malloc(sizeof(double) * (r * cols ? r * cols : 1));
        mm_at_b(u, v, w, dim, r, cols);
        for (size_t i = 0; i < r; ++i)
            for (size_t j = 0; j < cols; ++j) w[i * cols + j] *= bracket[i];
        mm(u, w, out, dim, r, cols);
        for (size_t i = 0; i < rows * cols; ++i) out[i] += v[i] / lambda;
        free(w);
    } else {
        if (cols != dim) { free(bracket); return ORC_DIMENSION_MISMATCH; }
        double* w = (double*)malloc(sizeof(double) * (rows * r ? rows * r : 1));
        mm(v, u, w, rows, dim, r);
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < r; ++j) w[i * r + j] *= bracket[j];
        mm_a_bt(w, u, out, rows, r, dim);
        for (size_t i = 0; i < rows * cols; ++i) out[i] += v[i] / lambda;
        free(w);
    }
    free(bracket);
    return ORC_OK;
}

/* kfactor.hpp:165-186  exact damped inverse through a full eigenbasis (the exact K-FAC comparator). */
int orc_apply_eig_damped_inverse(const double* u, const double* dv, size_t dim, size_t r,
                                 double lambda, const double* v, size_t rows, size_t cols,
                                 int side, double* out) {
    if (lambda <= 0.0) return ORC_DAMPING_NONPOSITIVE;
    double* inv = (double*)malloc(sizeof(double) * (r ? r : 1));
    for (size_t i = 0; i < r; ++i) inv[i] = 1.0 / (dv[i] + lambda);
    if (side == 0) {
        double* w = (double*)malloc(sizeof(double) * (r * cols ? r * cols : 1));
        mm_at_b(u, v, w, dim, r, cols);
        for (size_t i = 0; i < r; ++i)
            for (size_t j = 0; j < cols; ++j) w[i * cols + j] *= inv[i];
        mm(u, w, out, dim, r, cols);
        free(w);
    } else {
        double* w = (double*)malloc(sizeof(double) * (rows * r ? rows * r : 1));
        mm(v, u, w, rows, dim, r);
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < r; ++j) w[i * r + j] *= inv[j];
        mm_a_bt(w, u, out, rows, r, dim);
        free(w);
    }
    free(inv);
    return ORC_OK;
}

/* optimizer.hpp:159-162: S = LEFT_G(RIGHT_A(J)).  ua: dA x rA, ug: dG x rG, j: dG x dA. */
int orc_precondition(const double* ua, const double* da, size_t dA, size_t rA, const double* ug,
                     const double* dg, size_t dG, size_t rG, double lambda, const double* j,
                     double* out) {
    double* mid = (double*)malloc(sizeof(double) * (dG * dA ? dG * dA : 1));
    if (!mid) return ORC_ALLOC;
    int st = orc_apply_lowrank_damped_inverse(ua, da, dA, rA, lambda, j, dG, dA, 1, mid);
    if (!st) st = orc_apply_lowrank_damped_inverse(ug, dg, dG, rG, lambda, mid, dG, dA, 0, out);
    free(mid);
    return st;
}

/* Synthetic factor statistics of SURVEY.md 8(d): M = X^T / sqrt(n), X = Z diag(s), s_i = i^-e (1-based),
 * Z = sample_gaussian(RngState(root).substream(step, f), n, d).  Writes M as d x n row-major. */
void orc_synthetic_m(uint64_t root, uint64_t step, uint64_t f, size_t n, size_t d, double e, double* m) {
    const uint64_t seed = orc_substream(root, step, f);
    const double inv_sqrt_n = 1.0 / sqrt((double)n);
    for (size_t k = 0; k < n; ++k)
        for (size_t i = 0; i < d; ++i) {
            const double z = orc_gaussian_at(seed, 2 * (uint64_t)(k * d + i));
            m[i * n + k] = z * pow((double)(i + 1), -e) * inv_sqrt_n;
        }
}
