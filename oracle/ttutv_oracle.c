/*
 * TEST INFRASTRUCTURE ONLY -- see ttutv_oracle.h.
 *
 * Plain-C restatement of the reference TT-UTV path. Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/src). Floating-point
 * operations are issued in the reference's order and the file is compiled with
 * -ffp-contract=off, so results are bitwise equal to the reference library.
 */
#include "ttutv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

#define AT(M, rows, i, j) ((M)[(i) + (int64_t)(j) * (rows)])

static double* dalloc(int64_t n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }
static int64_t* ialloc(int64_t n) { return (int64_t*)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t)); }
static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }

/* ---- generators.cpp:13-48 (splitmix64, 53-bit uniform, Box-Muller with a spare) ---- */
void orc_rng_init(orc_rng* r, uint64_t seed) {
    r->state = seed;
    r->has_spare = 0;
    r->spare = 0.0;
}
uint64_t orc_rng_u64(orc_rng* r) {
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_u64(r) >> 11) * 0x1.0p-53; }
double orc_rng_normal(orc_rng* r) {
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    const double u1 = 1.0 - orc_rng_uniform(r);
    const double u2 = orc_rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double ang = 2.0 * 3.141592653589793 * u2;
    r->spare = rad * sin(ang);
    r->has_spare = 1;
    return rad * cos(ang);
}
int64_t orc_rng_uniform_int(orc_rng* r, int64_t lo, int64_t hi) {
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
    uint64_t x = orc_rng_u64(r);
    while (x >= limit) x = orc_rng_u64(r);
    return lo + (int64_t)(x % span);
}
void orc_gen_gaussian(int64_t count, uint64_t seed, double* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    for (int64_t i = 0; i < count; ++i) out[i] = orc_rng_normal(&r);
}
void orc_gen_hilbert(const int64_t* dims, int d, double shift, double* out) {
    int64_t idx[64];
    int64_t n = 1;
    for (int k = 0; k < d; ++k) {
        idx[k] = 1;
        n *= dims[k];
    }
    for (int64_t e = 0; e < n; ++e) {
        int64_t s = 0;
        for (int k = 0; k < d; ++k) s += idx[k];
        out[e] = 1.0 / ((double)s - shift);
        for (int k = 0; k < d; ++k) { /* odometer, first index fastest (shape.cpp:94-105) */
            if (idx[k] < dims[k]) { ++idx[k]; break; }
            idx[k] = 1;
        }
    }
}
void orc_gen_planted_cores(const int64_t* dims, int d, const int64_t* ranks, uint64_t seed, double* out) {
    orc_rng r;
    orc_rng_init(&r, seed);
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
        const int64_t n = ranks[k] * dims[k] * ranks[k + 1];
        for (int64_t i = 0; i < n; ++i) out[off + i] = orc_rng_normal(&r);
        off += n;
    }
}

/* ---- kernels.cpp ---- */
double orc_sum_squares_serial(const double* x, int64_t n) { /* kernels.cpp:78-82 */
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}
double orc_sum_squares(const double* x, int64_t n) { /* kernels.cpp:84-102 */
    const int64_t blk = 4096, nb = (n + blk - 1) / blk;
    if (nb <= 1) return orc_sum_squares_serial(x, n);
    double tot = 0.0;
    for (int64_t b = 0; b < nb; ++b) {
        const int64_t lo = b * blk, hi = imin(n, lo + blk);
        tot += orc_sum_squares_serial(x + lo, hi - lo);
    }
    return tot;
}
/* C = op(A) op(B), one sequential dot per entry (kernels.cpp:28-46). */
void orc_matmul(const double* a, int64_t ar, int64_t ac, int ta, const double* b, int64_t br, int64_t bc, int tb,
                double* c) {
    const int64_t m = ta ? ac : ar, k = ta ? ar : ac, n = tb ? br : bc;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            double s = 0.0;
            for (int64_t l = 0; l < k; ++l) {
                const double av = ta ? AT(a, ar, l, i) : AT(a, ar, i, l);
                const double bv = tb ? AT(b, br, j, l) : AT(b, br, l, j);
                s += av * bv;
            }
            AT(c, m, i, j) = s;
        }
}
static double* transposed(const double* a, int64_t m, int64_t n) { /* kernels.cpp:71-76 */
    double* t = dalloc(m * n);
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) AT(t, n, j, i) = AT(a, m, i, j);
    return t;
}

/* ---- factor.cpp:17-135: Householder QR with column pivoting ---- */
/* dlarfg-style reflector on w(k:m, k); returns beta (factor.cpp:24-38). */
static double householder(double* w, int64_t m, int64_t k) {
    double* x = w + k * m + k;
    const int64_t len = m - k;
    if (len <= 1) return 0.0;
    double sigma = 0.0;
    for (int64_t i = 1; i < len; ++i) sigma += x[i] * x[i];
    const double alpha = x[0];
    if (sigma == 0.0) return 0.0;
    const double mu = sqrt(alpha * alpha + sigma);
    const double v0 = alpha + copysign(mu, alpha);
    const double beta = v0 * v0 / (copysign(mu, alpha) * v0);
    for (int64_t i = 1; i < len; ++i) x[i] /= v0;
    x[0] = -copysign(mu, alpha);
    return beta;
}
/* H = I - beta v v^T (v[0] = 1 implicit) on columns [from, to) (factor.cpp:43-58). */
static void reflect(double* w, int64_t m, int64_t k, double beta, int64_t from, int64_t to) {
    if (beta == 0.0 || from >= to) return;
    const double* v = w + k * m + k;
    const int64_t len = m - k;
    for (int64_t j = from; j < to; ++j) {
        double* c = w + j * m + k;
        double t = c[0];
        for (int64_t i = 1; i < len; ++i) t += v[i] * c[i];
        t *= beta;
        c[0] -= t;
        for (int64_t i = 1; i < len; ++i) c[i] -= t * v[i];
    }
}

int orc_qr_col_pivot(const double* a, int64_t m, int64_t n, double* q, double* r, int64_t* perm) {
    if (m <= 0 || n <= 0) return fail(1, "qr_col_pivot: empty matrix");
    const int64_t p = imin(m, n);
    double* w = dalloc(m * n);
    memcpy(w, a, sizeof(double) * (size_t)(m * n));
    double* beta = dalloc(p);
    double* nrm = dalloc(n);
    double* ref = dalloc(n);
    for (int64_t j = 0; j < n; ++j) {
        perm[j] = j;
        nrm[j] = ref[j] = orc_sum_squares_serial(w + j * m, m);
    }
    for (int64_t k = 0; k < p; ++k) {
        int64_t piv = k;
        for (int64_t j = k + 1; j < n; ++j)
            if (nrm[j] > nrm[piv]) piv = j;
        if (piv != k) {
            for (int64_t i = 0; i < m; ++i) {
                const double x = AT(w, m, i, k);
                AT(w, m, i, k) = AT(w, m, i, piv);
                AT(w, m, i, piv) = x;
            }
            int64_t ti = perm[k]; perm[k] = perm[piv]; perm[piv] = ti;
            double td = nrm[k]; nrm[k] = nrm[piv]; nrm[piv] = td;
            td = ref[k]; ref[k] = ref[piv]; ref[piv] = td;
        }
        beta[k] = householder(w, m, k);
        reflect(w, m, k, beta[k], k + 1, n);
        for (int64_t j = k + 1; j < n; ++j) {
            const double rkj = AT(w, m, k, j);
            nrm[j] -= rkj * rkj;
            if (nrm[j] < 1e-16 * ref[j] || nrm[j] < 0.0) {
                nrm[j] = orc_sum_squares_serial(w + j * m + k + 1, m - k - 1);
                ref[j] = nrm[j];
            }
        }
    }
    if (r) {
        memset(r, 0, sizeof(double) * (size_t)(p * n));
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i <= imin(j, p - 1); ++i) AT(r, p, i, j) = AT(w, m, i, j);
    }
    if (q) { /* economy Q by backward accumulation (factor.cpp:114-133) */
        memset(q, 0, sizeof(double) * (size_t)(m * p));
        for (int64_t j = 0; j < p; ++j) AT(q, m, j, j) = 1.0;
        for (int64_t k = p - 1; k >= 0; --k) {
            const double bk = beta[k];
            if (bk == 0.0) continue;
            const double* v = w + k * m + k;
            const int64_t len = m - k;
            for (int64_t j = k; j < p; ++j) {
                double* c = q + j * m + k;
                double t = c[0];
                for (int64_t i = 1; i < len; ++i) t += v[i] * c[i];
                t *= bk;
                c[0] -= t;
                for (int64_t i = 1; i < len; ++i) c[i] -= t * v[i];
            }
        }
    }
    free(w); free(beta); free(nrm); free(ref);
    return 0;
}

/* ---- factor.cpp:263-448: UTV by alternating pivoted QR passes ---- */
typedef struct {
    double* u; int64_t ur, uc;   /* dense U, or NULL while pu is the pending permutation */
    int64_t* pu; int64_t npu;
    double* v; int64_t vr, vc;
    int64_t* pv; int64_t npv;
    double* mid; int64_t mr, mc;
    int lower;
} Utv;

/* out(perm[j], :) = q(j, :) (factor.cpp:280-289) */
static double* rows_from(const double* q, int64_t qr, int64_t qc, const int64_t* perm) {
    double* o = dalloc(qr * qc);
    for (int64_t j = 0; j < qr; ++j)
        for (int64_t c = 0; c < qc; ++c) AT(o, qr, perm[j], c) = AT(q, qr, j, c);
    return o;
}
static double* pick_cols(const double* u, int64_t ur, const int64_t* perm, int64_t count) { /* :291-298 */
    double* o = dalloc(ur * count);
    for (int64_t j = 0; j < count; ++j) memcpy(o + j * ur, u + perm[j] * ur, sizeof(double) * (size_t)ur);
    return o;
}
/* side 0 = U, 1 = V: compose with a dense Q (:307-314, :327-334) */
static void with_q(Utv* s, int side, const double* q, int64_t qr, int64_t qc) {
    double** d = side ? &s->v : &s->u;
    int64_t *dr = side ? &s->vr : &s->ur, *dc = side ? &s->vc : &s->uc;
    int64_t** pp = side ? &s->pv : &s->pu;
    if (*pp) {
        double* o = rows_from(q, qr, qc, *pp);
        free(*pp);
        *pp = NULL;
        free(*d);
        *d = o;
        *dr = qr;
        *dc = qc;
    } else {
        double* o = dalloc(*dr * qc);
        orc_matmul(*d, *dr, *dc, 0, q, qr, qc, 0, o);
        free(*d);
        *d = o;
        *dc = qc;
    }
}
/* compose with a column selection (:316-325, :336-345) */
static void with_perm(Utv* s, int side, const int64_t* perm, int64_t count) {
    int64_t** pp = side ? &s->pv : &s->pu;
    int64_t* np = side ? &s->npv : &s->npu;
    if (*pp) {
        int64_t* c = ialloc(count);
        for (int64_t j = 0; j < count; ++j) c[j] = (*pp)[perm[j]];
        free(*pp);
        *pp = c;
        *np = count;
    } else {
        double** d = side ? &s->v : &s->u;
        int64_t *dr = side ? &s->vr : &s->ur, *dc = side ? &s->vc : &s->uc;
        double* o = pick_cols(*d, *dr, perm, count);
        free(*d);
        *d = o;
        *dc = count;
    }
}
static void flip(Utv* s, int to_lower) { /* flip_to_upper / flip_to_lower (:347-372) */
    const double* src = s->mid;
    int64_t m = s->mr, n = s->mc;
    double* tr = NULL;
    if (to_lower) {
        tr = transposed(s->mid, s->mr, s->mc);
        src = tr;
        m = s->mc;
        n = s->mr;
    }
    const int64_t p = imin(m, n);
    double* q = dalloc(m * p);
    double* r = dalloc(p * n);
    int64_t* perm = ialloc(n);
    orc_qr_col_pivot(src, m, n, q, r, perm);
    free(tr);
    if (to_lower) {
        with_perm(s, 0, perm, p);
        with_q(s, 1, q, m, p);
    } else {
        with_q(s, 0, q, m, p);
        with_perm(s, 1, perm, p);
    }
    double* sq = dalloc(p * p);
    for (int64_t j = 0; j < p; ++j)
        for (int64_t i = 0; i <= j; ++i) {
            if (to_lower) AT(sq, p, j, i) = AT(r, p, i, j);
            else AT(sq, p, i, j) = AT(r, p, i, j);
        }
    free(s->mid);
    s->mid = sq;
    s->mr = s->mc = p;
    s->lower = to_lower;
    free(q); free(r); free(perm);
}
static double* perm_matrix(const int64_t* perm, int64_t rows, int64_t cols) { /* :300-305 */
    double* o = dalloc(rows * cols);
    for (int64_t j = 0; j < cols; ++j) AT(o, rows, perm[j], j) = 1.0;
    return o;
}

int orc_utv(const double* a, int64_t m, int64_t n, int lower, int refine, double* u, double* t, double* v) {
    if (refine < 0) return fail(1, "refine_passes must be >= 0");
    if (refine > 64) return fail(1, "refine_passes is unreasonably large");
    if (m <= 0 || n <= 0) return fail(1, "utv: empty matrix");
    int passes = refine + 1;
    const int64_t p = imin(m, n);
    int direct = lower ? (passes % 2 == 0) : (passes % 2 == 1); /* utv_engine (:376-395) */
    if (passes == 1) {
        if (direct && m < n) { passes = 2; direct = 0; }
        else if (!direct && m > n) { passes = 2; direct = 1; }
    }
    Utv s;
    memset(&s, 0, sizeof s);
    if (direct) {
        s.u = dalloc(m * p); s.ur = m; s.uc = p;
        s.pv = ialloc(n); s.npv = n;
        s.mid = dalloc(p * n); s.mr = p; s.mc = n;
        orc_qr_col_pivot(a, m, n, s.u, s.mid, s.pv);
        s.lower = 0;
    } else {
        double* at = transposed(a, m, n);
        double* r = dalloc(p * m);
        s.v = dalloc(n * p); s.vr = n; s.vc = p;
        s.pu = ialloc(m); s.npu = m;
        orc_qr_col_pivot(at, n, m, s.v, r, s.pu);
        s.mid = transposed(r, p, m); s.mr = m; s.mc = p;
        s.lower = 1;
        free(at); free(r);
    }
    for (int pass = 1; pass < passes; ++pass) flip(&s, !s.lower);
    if (s.pu) { s.u = perm_matrix(s.pu, m, p); s.ur = m; s.uc = p; free(s.pu); s.pu = NULL; }
    if (s.pv) { s.v = perm_matrix(s.pv, n, p); s.vr = n; s.vc = p; free(s.pv); s.pv = NULL; }
    if (u) memcpy(u, s.u, sizeof(double) * (size_t)(m * p));
    if (t) memcpy(t, s.mid, sizeof(double) * (size_t)(p * p));
    if (v) memcpy(v, s.v, sizeof(double) * (size_t)(n * p));
    free(s.u); free(s.v); free(s.mid);
    return 0;
}

/* ---- factor.cpp:137-261: one-sided Jacobi SVD ---- */
static int complete_basis(double* u, int64_t m, int64_t j) { /* :143-162 */
    double* r = dalloc(m);
    for (int64_t cand = 0; cand < m; ++cand) {
        memset(r, 0, sizeof(double) * (size_t)m);
        r[cand] = 1.0;
        for (int pass = 0; pass < 2; ++pass)
            for (int64_t c = 0; c < j; ++c) {
                double proj = 0.0;
                for (int64_t i = 0; i < m; ++i) proj += AT(u, m, i, c) * r[i];
                for (int64_t i = 0; i < m; ++i) r[i] -= proj * AT(u, m, i, c);
            }
        const double nrm = sqrt(orc_sum_squares_serial(r, m));
        if (nrm > 0.5) {
            for (int64_t i = 0; i < m; ++i) AT(u, m, i, j) = r[i] / nrm;
            free(r);
            return 0;
        }
    }
    free(r);
    return fail(4, "svd: failed to complete an orthonormal basis");
}
static int svd_tall(const double* a, int64_t m, int64_t n, int max_sweeps, double tol, double* uo, double* so,
                    double* vo) { /* :164-252 */
    double* w = dalloc(m * n);
    memcpy(w, a, sizeof(double) * (size_t)(m * n));
    double* v = dalloc(n * n);
    for (int64_t i = 0; i < n; ++i) AT(v, n, i, i) = 1.0;
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
        int rotated = 0;
        for (int64_t i = 0; i + 1 < n; ++i)
            for (int64_t j = i + 1; j < n; ++j) {
                double* wi = w + i * m;
                double* wj = w + j * m;
                double aii = 0.0, ajj = 0.0, aij = 0.0;
                for (int64_t r = 0; r < m; ++r) {
                    aii += wi[r] * wi[r];
                    ajj += wj[r] * wj[r];
                    aij += wi[r] * wj[r];
                }
                if (aii == 0.0 || ajj == 0.0) continue;
                if (fabs(aij) <= tol * sqrt(aii * ajj)) continue;
                rotated = 1;
                const double zeta = (ajj - aii) / (2.0 * aij);
                const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + tt * tt);
                const double sn = cs * tt;
                for (int64_t r = 0; r < m; ++r) {
                    const double x = wi[r], y = wj[r];
                    wi[r] = cs * x - sn * y;
                    wj[r] = sn * x + cs * y;
                }
                double* vi = v + i * n;
                double* vj = v + j * n;
                for (int64_t r = 0; r < n; ++r) {
                    const double x = vi[r], y = vj[r];
                    vi[r] = cs * x - sn * y;
                    vj[r] = sn * x + cs * y;
                }
            }
        if (!rotated) break;
    }
    if (sweep == max_sweeps) {
        free(w); free(v);
        return fail(4, "svd: one-sided Jacobi did not converge");
    }
    double* s = dalloc(n);
    int64_t* order = ialloc(n);
    for (int64_t j = 0; j < n; ++j) {
        s[j] = sqrt(orc_sum_squares_serial(w + j * m, m));
        order[j] = j;
    }
    for (int64_t i = 1; i < n; ++i) { /* stable insertion sort, descending */
        const int64_t x = order[i];
        int64_t k = i;
        while (k > 0 && s[order[k - 1]] < s[x]) { order[k] = order[k - 1]; --k; }
        order[k] = x;
    }
    int rc = 0;
    memset(uo, 0, sizeof(double) * (size_t)(m * n));
    for (int64_t j = 0; j < n && rc == 0; ++j) {
        const int64_t src = order[j];
        const double sj = s[src];
        so[j] = sj;
        for (int64_t i = 0; i < n; ++i) AT(vo, n, i, j) = AT(v, n, i, src);
        if (sj > 0.0) for (int64_t i = 0; i < m; ++i) AT(uo, m, i, j) = AT(w, m, i, src) / sj;
        else rc = complete_basis(uo, m, j);
    }
    free(w); free(v); free(s); free(order);
    return rc;
}
int orc_svd(const double* a, int64_t m, int64_t n, int max_sweeps, double pair_tol, double* u, double* s, double* v) {
    if (m <= 0 || n <= 0) return fail(1, "svd: empty matrix");
    if (m >= n) return svd_tall(a, m, n, max_sweeps, pair_tol, u, s, v);
    double* at = transposed(a, m, n);
    const int rc = svd_tall(at, n, m, max_sweeps, pair_tol, v, s, u); /* roles swap (:256-261) */
    free(at);
    return rc;
}

/* ---- factor.cpp:450-562: truncation ---- */
static void kept_mass(int kind, const double* t, int64_t p, double* kept) { /* :476-505 */
    kept[0] = 0.0;
    for (int64_t r = 1; r <= p; ++r) {
        double add = 0.0;
        if (kind == 0) add = t[r - 1] * t[r - 1];
        else
            for (int64_t j = 0; j < r; ++j) {
                const double x = kind == 1 ? AT(t, p, r - 1, j) : AT(t, p, j, r - 1);
                add += x * x;
            }
        kept[r] = kept[r - 1] + add;
    }
}
static int64_t choose_rank(const double* kept, int64_t p, double eps) { /* pick_rank :512-520 */
    if (eps == 0.0) return p;
    const double target = kept[p] - eps * eps;
    for (int64_t r = 1; r < p; ++r)
        if (kept[r] >= target) return r;
    return p;
}
int orc_truncate(int kind, const double* u, const double* t, const double* v, int64_t m, int64_t n, int64_t p,
                 int64_t rank, double eps, int64_t* rank_out, double* residual, double* u1, double* t11, double* v1) {
    double* kept = dalloc(p + 1);
    kept_mass(kind, t, p, kept);
    int64_t r = rank;
    if (rank <= 0) {
        if (eps < 0.0) { free(kept); return fail(1, "tolerance must be >= 0"); }
        r = choose_rank(kept, p, eps);
    } else if (rank > p) {
        free(kept);
        return fail(1, "rank out of range");
    }
    *rank_out = r;
    const double disc = kept[p] - kept[r];
    *residual = sqrt(disc > 0.0 ? disc : 0.0);
    if (u1) memcpy(u1, u, sizeof(double) * (size_t)(m * r));
    if (v1) memcpy(v1, v, sizeof(double) * (size_t)(n * r));
    if (t11) {
        memset(t11, 0, sizeof(double) * (size_t)(r * r));
        for (int64_t j = 0; j < r; ++j)
            for (int64_t i = 0; i < r; ++i) AT(t11, r, i, j) = kind == 0 ? (i == j ? t[i] : 0.0) : AT(t, p, i, j);
    }
    free(kept);
    return 0;
}

/* ---- tt.cpp:52-73 / tensor_ops.cpp:101-111 ---- */
int orc_reconstruct(const double* cores, const int64_t* dims, const int64_t* ranks, int d, double* out) {
    int64_t left = dims[0], off = ranks[0] * dims[0] * ranks[1];
    double* b = dalloc(left * ranks[1]);
    memcpy(b, cores, sizeof(double) * (size_t)(left * ranks[1]));
    for (int k = 1; k < d; ++k) {
        const double* g = cores + off;
        const int64_t cols = dims[k] * ranks[k + 1];
        double* nx = dalloc(left * cols);
        orc_matmul(b, left, ranks[k], 0, g, ranks[k], cols, 0, nx);
        free(b);
        b = nx;
        left *= dims[k];
        off += ranks[k] * dims[k] * ranks[k + 1];
    }
    memcpy(out, b, sizeof(double) * (size_t)left);
    free(b);
    return 0;
}
double orc_rse(const double* est, const double* truth, int64_t n) {
    const double den = sqrt(orc_sum_squares(truth, n));
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double x = est[i] - truth[i];
        s += x * x;
    }
    return sqrt(s) / den;
}

/* ---- tt_decomp.cpp: sweeps ---- */
typedef struct {
    double* data; int64_t r0, n, r1;
} Core;

typedef struct {
    int method, retain, refine, fixed;
    const int64_t* ranks;
    double* budgets;
} Mode;

/* One factorisation + truncation of cut matrix c (m x n). Returns rank, residual and the
 * pieces each sweep needs (left kept factor l1 m x r, middle t11 r x r, right v1 n x r).
 * kind: 0 svd, 1 ulv, 2 urv. */
typedef struct { int64_t r; double res; double *u1, *t11, *v1, *fullu, *fullt; int64_t p; } Cut;

static int factor_cut(int kind, const double* c, int64_t m, int64_t n, int refine, int fixed, int64_t want,
                      double budget, Cut* out) {
    const int64_t p = imin(m, n);
    double* u = dalloc(m * p);
    double* t = dalloc(kind == 0 ? p : p * p);
    double* v = dalloc(n * p);
    int rc = kind == 0 ? orc_svd(c, m, n, 60, 1e-14, u, t, v) : orc_utv(c, m, n, kind == 1, refine, u, t, v);
    if (rc) { free(u); free(t); free(v); return rc; }
    int64_t r = fixed ? want : 0;
    out->u1 = dalloc(m * p); out->v1 = dalloc(n * p); out->t11 = dalloc(p * p);
    rc = orc_truncate(kind, u, t, v, m, n, p, r, budget, &out->r, &out->res, out->u1, out->t11, out->v1);
    out->fullu = u;
    out->fullt = t;
    out->p = p;
    free(v);
    return rc;
}
static void free_cut(Cut* c) { free(c->u1); free(c->t11); free(c->v1); free(c->fullu); free(c->fullt); }

static int put_core(double* cores_out, int64_t cap, int64_t* used, int64_t* core_dims, int k, const double* data,
                    int64_t r0, int64_t n, int64_t r1) {
    const int64_t sz = r0 * n * r1;
    if (*used + sz > cap) return fail(1, "oracle core buffer too small");
    memcpy(cores_out + *used, data, sizeof(double) * (size_t)sz);
    *used += sz;
    core_dims[3 * k] = r0;
    core_dims[3 * k + 1] = n;
    core_dims[3 * k + 2] = r1;
    return 0;
}

int orc_decompose(const double* a, const int64_t* dims, int d, int method, int sweep, int fixed_rank,
                  const int64_t* ranks, double eps, const double* weights, int nweights, int refine, int retain,
                  double* cores_out, int64_t cap, int64_t* core_dims, double* step_errors, int64_t* ranks_chosen,
                  double* bound, int* bound_kind, double* input_norm) {
    int64_t total = 1;
    for (int k = 0; k < d; ++k) total *= dims[k];
    /* bound_kind_for (tt_decomp.cpp:341-346) */
    const int plain = method == 1 && sweep == 1 && retain == 0;
    const double nrm = sqrt(orc_sum_squares(a, total));
    *input_norm = nrm;
    *bound_kind = plain;
    const int64_t cuts = d - 1;
    double* budgets = dalloc(cuts);
    if (fixed_rank) { /* resolve_mode (tt_decomp.cpp:32-71) */
        if (ranks[0] != 1 || ranks[d] != 1) { free(budgets); return fail(1, "boundary ranks must both be 1"); }
        for (int k = 0; k <= d; ++k)
            if (ranks[k] < 1) { free(budgets); return fail(1, "ranks must be >= 1"); }
    } else {
        if (eps < 0.0) { free(budgets); return fail(1, "tolerance must be >= 0"); }
        for (int64_t k = 0; k < cuts; ++k) {
            double w;
            if (nweights == 0) {
                const double c = (double)(cuts > 1 ? cuts : 1);
                w = plain ? 1.0 / c : 1.0 / sqrt(c);
            } else {
                w = weights[k];
            }
            budgets[k] = w * eps * nrm;
        }
    }
    for (int k = 0; k <= d; ++k) ranks_chosen[k] = 1;
    for (int64_t k = 0; k < cuts; ++k) step_errors[k] = 0.0;
    int64_t used = 0;
    int rc = 0;
    if (nrm == 0.0 || d == 1) { /* zero_input_result / order_one_result (:126-151) */
        for (int k = 0; k < d; ++k) {
            double* z = dalloc(dims[k]);
            if (d == 1 && nrm != 0.0) memcpy(z, a, sizeof(double) * (size_t)dims[0]);
            rc = put_core(cores_out, cap, &used, core_dims, k, z, 1, dims[k], 1);
            free(z);
        }
        *bound = 0.0;
        free(budgets);
        return rc;
    }
    const int kind = method == 0 ? 0 : method == 1 ? 1 : 2;
    if (method == 2 && sweep == 0) { /* left_orthogonal_via_urv: reverse, URV r2l, reverse back */
        free(budgets);
        return fail(1, "oracle: URV left-to-right is exercised through the reference library only");
    }
    double berr = 0.0;
    if (sweep == 0) { /* sweep_l2r (tt_decomp.cpp:156-211) */
        int64_t m = dims[0], n = total / dims[0], rprev = 1;
        double* c = dalloc(m * n);
        memcpy(c, a, sizeof(double) * (size_t)(m * n));
        for (int k = 1; k <= d - 1 && rc == 0; ++k) {
            const int64_t p = imin(m, n);
            int64_t want = fixed_rank ? imin(ranks[k], p) : 0;
            Cut cut;
            memset(&cut, 0, sizeof cut);
            rc = factor_cut(kind, c, m, n, refine, fixed_rank, want, fixed_rank ? 0.0 : budgets[k - 1], &cut);
            if (rc) break;
            const int64_t r = cut.r;
            step_errors[k - 1] = cut.res;
            ranks_chosen[k] = r;
            double* carry = dalloc(r * n);
            orc_matmul(cut.t11, r, r, 0, cut.v1, n, r, 1, carry); /* T11 V1^T (:192) */
            rc = put_core(cores_out, cap, &used, core_dims, k - 1, cut.u1, rprev, dims[k - 1], r);
            rprev = r;
            free_cut(&cut);
            free(c);
            c = carry;
            if (k < d - 1) {
                m = r * dims[k];
                n = n / dims[k];
            } else {
                rc = rc ? rc : put_core(cores_out, cap, &used, core_dims, d - 1, carry, r, dims[d - 1], 1);
            }
        }
        free(c);
    } else { /* sweep_r2l (tt_decomp.cpp:216-339); cores emitted in reverse then reordered */
        int64_t M = total / dims[d - 1], n = dims[d - 1], rnext = 1;
        double* c = dalloc(M * n);
        memcpy(c, a, sizeof(double) * (size_t)(M * n));
        double** held = (double**)calloc((size_t)d, sizeof(double*));
        int64_t* hd = ialloc(3 * d);
        for (int k = d; k >= 2 && rc == 0; --k) {
            const int64_t p = imin(M, n);
            const int64_t want = fixed_rank ? imin(ranks[k - 1], p) : 0;
            const int full_column = method == 1 && retain == 1;
            Cut cut;
            memset(&cut, 0, sizeof cut);
            int64_t r;
            double* carry;
            double* v1;
            if (full_column) { /* Alg. 4 full column: carry = U L(:, :r) (:241-270) */
                rc = factor_cut(1, c, M, n, refine, 1, p, 0.0, &cut); /* full factors */
                if (rc) break;
                const double* L = cut.fullt;
                double* kept = dalloc(p + 1);
                kept[0] = 0.0;
                for (int64_t j = 0; j < p; ++j) kept[j + 1] = kept[j] + orc_sum_squares_serial(L + j * p, p);
                if (fixed_rank) r = want;
                else {
                    const double bd = budgets[k - 2];
                    r = p;
                    if (bd > 0.0) {
                        const double target = kept[p] - bd * bd;
                        for (int64_t cand = 1; cand < p; ++cand)
                            if (kept[cand] >= target) { r = cand; break; }
                    }
                }
                const double disc = kept[p] - kept[r];
                cut.res = sqrt(disc > 0.0 ? disc : 0.0);
                carry = dalloc(M * r);
                orc_matmul(cut.fullu, M, p, 0, L, p, r, 0, carry);
                v1 = dalloc(n * r);
                memcpy(v1, cut.v1, sizeof(double) * (size_t)(n * r));
                free(kept);
            } else {
                rc = factor_cut(kind, c, M, n, refine, fixed_rank, want, fixed_rank ? 0.0 : budgets[k - 2], &cut);
                if (rc) break;
                r = cut.r;
                carry = dalloc(M * r);
                orc_matmul(cut.u1, M, r, 0, cut.t11, r, r, 0, carry); /* U1 T11 (:302) */
                v1 = dalloc(n * r);
                memcpy(v1, cut.v1, sizeof(double) * (size_t)(n * r));
            }
            step_errors[k - 2] = cut.res;
            ranks_chosen[k - 1] = r;
            held[k - 1] = transposed(v1, n, r); /* core_from_left_unfolding (:77-80) */
            hd[3 * (k - 1)] = r;
            hd[3 * (k - 1) + 1] = dims[k - 1];
            hd[3 * (k - 1) + 2] = rnext;
            rnext = r;
            free(v1);
            free_cut(&cut);
            free(c);
            c = carry;
            if (k > 2) {
                const int64_t rows = M / dims[k - 2];
                n = dims[k - 2] * r;
                M = rows;
            } else {
                held[0] = c;
                c = NULL;
                hd[0] = 1;
                hd[1] = dims[0];
                hd[2] = r;
            }
        }
        for (int k = 0; k < d && rc == 0; ++k)
            rc = put_core(cores_out, cap, &used, core_dims, k, held[k], hd[3 * k], hd[3 * k + 1], hd[3 * k + 2]);
        for (int k = 0; k < d; ++k) free(held[k]);
        free(held);
        free(hd);
        free(c);
    }
    for (int64_t k = 0; k < cuts; ++k) berr += plain ? step_errors[k] : step_errors[k] * step_errors[k];
    *bound = plain ? berr : sqrt(berr); /* finish (:116-124) */
    free(budgets);
    return rc;
}
