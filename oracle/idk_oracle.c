/*
 * idk_oracle.c -- TEST INFRASTRUCTURE ONLY (see idk_oracle.h).
 *
 * CPU restatement of the reference ID path.  Each function names the
 * reference file:line it follows; the operation order is kept so that, built
 * with -ffp-contract=off, results are bit-identical to the reference build.
 */
#include "idk_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* idko_last_error(void) { return g_err; }

#define IDX(i, j, ld) ((size_t)(j) * (size_t)(ld) + (size_t)(i))

/* ------------------------------------------------------------------------ */
/* mt19937_64 (std::mt19937_64; random.hpp:13) -- the published algorithm.   */
/* ------------------------------------------------------------------------ */
void idko_mt64_seed(idko_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

uint64_t idko_mt64_next(idko_mt64* g) {
    static const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UPPER) | (g->mt[(i + 1) % 312] & LOWER);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

/* random.hpp:18-20 */
double idko_next_uniform(idko_mt64* g) { return (double)(idko_mt64_next(g) >> 11) * 0x1.0p-53; }

/* random.cpp:10-15: Box-Muller, u1 in (0, 1]. */
static const double kPi = 3.141592653589793238462643383279502884;
double idko_next_normal(idko_mt64* g) {
    const double u1 = (double)((idko_mt64_next(g) >> 11) + 1) * 0x1.0p-53;
    const double u2 = idko_next_uniform(g);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2);
}

/* random.cpp:17-27 */
uint64_t idko_next_below(idko_mt64* g, uint64_t bound) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
        x = idko_mt64_next(g);
    } while (x >= limit);
    return x % bound;
}

/* random.cpp:29-41 (engine seeded as seeded_engine(seed), random.hpp:15) */
static int swr_engine(int64_t population, int64_t count, idko_mt64* g, int64_t* out) {
    if (count > population) return fail(IDKO_INVALID_ARG, "sample_without_replacement: count exceeds population");
    int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)(population > 0 ? population : 1));
    if (!pool) return fail(IDKO_NO_MEMORY, "out of memory");
    for (int64_t i = 0; i < population; ++i) pool[i] = i;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t j = i + (int64_t)idko_next_below(g, (uint64_t)(population - i));
        int64_t t = pool[i];
        pool[i] = pool[j];
        pool[j] = t;
    }
    memcpy(out, pool, sizeof(int64_t) * (size_t)count);
    free(pool);
    return IDKO_OK;
}

int idko_sample_without_replacement(int64_t population, int64_t count, uint64_t seed, int64_t* out) {
    idko_mt64 g;
    idko_mt64_seed(&g, seed);
    return swr_engine(population, count, &g, out);
}

/* random.cpp:43-55 */
uint64_t idko_mix_seed(uint64_t base, const char* label) {
    uint64_t h = 1469598103934665603ULL;
    for (const unsigned char* c = (const unsigned char*)label; *c; ++c) {
        h ^= *c;
        h *= 1099511628211ULL;
    }
    uint64_t z = base ^ h;
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* datasets.cpp:15-33 */
int idko_generate(int kind, int64_t rows, int64_t cols, uint64_t seed, double* out) {
    if (rows < 1 || cols < 1) return fail(IDKO_INVALID_ARG, "generate: dimensions must be positive");
    idko_mt64 g;
    idko_mt64_seed(&g, seed);
    const int64_t total = rows * cols;
    for (int64_t i = 0; i < total; ++i) {
        if (kind == 0) out[i] = (double)(idko_mt64_next(&g) >> 63);
        else if (kind == 1) out[i] = idko_next_normal(&g);
        else out[i] = idko_next_uniform(&g);
    }
    return IDKO_OK;
}

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 Omega (mirror of csrc/rng.cuh).                             */
/* ------------------------------------------------------------------------ */
void idko_philox4x32_10(uint32_t c[4], const uint32_t key[2]) {
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n1 = (uint32_t)p1;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        const uint32_t n3 = (uint32_t)p0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

void idko_omega_philox(int64_t l, int64_t m, uint64_t seed, double* out) {
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    const int64_t total = l * m;
    /* element pair (2j, 2j+1) <- Philox block j: the Box-Muller (cos, sin) pair */
    for (int64_t j = 0; 2 * j < total; ++j) {
        uint32_t c[4] = {(uint32_t)j, (uint32_t)((uint64_t)j >> 32), 0u, 0u};
        idko_philox4x32_10(c, key);
        const uint64_t r1 = ((uint64_t)c[1] << 32) | c[0];
        const uint64_t r2 = ((uint64_t)c[3] << 32) | c[2];
        const double u1 = (double)((r1 >> 11) + 1) * 0x1.0p-53;
        const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
        const double r = sqrt(-2.0 * log(u1)), th = 2.0 * kPi * u2;
        out[2 * j] = r * cos(th);
        if (2 * j + 1 < total) out[2 * j + 1] = r * sin(th);
    }
}

/* ------------------------------------------------------------------------ */
/* Dense core (matrix.cpp).                                                  */
/* ------------------------------------------------------------------------ */
/* matrix.cpp:28-48: saxpy order, b == 0 entries skipped. */
int idko_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* out) {
    memset(out, 0, sizeof(double) * (size_t)(m * n));
    for (int64_t j = 0; j < n; ++j) {
        double* oj = out + IDX(0, j, m);
        const double* bj = b + IDX(0, j, k);
        for (int64_t l = 0; l < k; ++l) {
            const double blj = bj[l];
            if (blj == 0.0) continue;
            const double* al = a + IDX(0, l, m);
            for (int64_t i = 0; i < m; ++i) oj[i] += al[i] * blj;
        }
    }
    return IDKO_OK;
}

/* matrix.cpp:50-66: a is k x m, b is k x n, out = a^T b (m x n). */
int idko_matmul_transpose_a(const double* a, int64_t k, int64_t m, const double* b, int64_t n,
                            double* out) {
    for (int64_t j = 0; j < n; ++j) {
        const double* bj = b + IDX(0, j, k);
        double* oj = out + IDX(0, j, m);
        for (int64_t i = 0; i < m; ++i) {
            const double* ai = a + IDX(0, i, k);
            double acc = 0.0;
            for (int64_t l = 0; l < k; ++l) acc += ai[l] * bj[l];
            oj[i] = acc;
        }
    }
    return IDKO_OK;
}

/* matrix.cpp:68-73 */
void idko_transpose(const double* a, int64_t m, int64_t n, double* out) {
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) out[IDX(j, i, n)] = a[IDX(i, j, m)];
}

/* matrix.cpp:121-130 */
int idko_select_columns(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t ncols,
                        double* out) {
    for (int64_t j = 0; j < ncols; ++j) {
        if (cols[j] < 0 || cols[j] >= n) return fail(IDKO_INVALID_ARG, "select_columns: index out of range");
        memcpy(out + IDX(0, j, m), a + IDX(0, cols[j], m), sizeof(double) * (size_t)m);
    }
    return IDKO_OK;
}

/* matrix.cpp:96-119 */
double idko_frobenius_norm(const double* a, int64_t total) {
    double sum = 0.0;
    for (int64_t i = 0; i < total; ++i) sum += a[i] * a[i];
    return sqrt(sum);
}

double idko_frobenius_distance(const double* a, const double* b, int64_t total) {
    double sum = 0.0;
    for (int64_t i = 0; i < total; ++i) {
        const double d = a[i] - b[i];
        sum += d * d;
    }
    return sqrt(sum);
}

double idko_max_abs(const double* a, int64_t total) {
    double best = 0.0;
    for (int64_t i = 0; i < total; ++i) {
        const double v = fabs(a[i]);
        best = best > v ? best : v; /* std::max(best, v) keeps best on ties/NaN */
    }
    return best;
}

/* ------------------------------------------------------------------------ */
/* Column-pivoted Householder QR (qr.cpp:16-126).                            */
/* ------------------------------------------------------------------------ */
/* qr.cpp:16-28 */
static double make_householder(double* x, int64_t len) {
    if (len <= 1) return 0.0;
    double tail = 0.0;
    for (int64_t i = 1; i < len; ++i) tail += x[i] * x[i];
    if (tail == 0.0) return 0.0;
    const double alpha = x[0];
    const double beta = -copysign(sqrt(alpha * alpha + tail), alpha);
    const double tau = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    for (int64_t i = 1; i < len; ++i) x[i] *= scale;
    x[0] = beta;
    return tau;
}

/* qr.cpp:31-38 */
static void apply_householder(const double* x, double tau, double* y, int64_t len) {
    if (tau == 0.0) return;
    double w = y[0];
    for (int64_t i = 1; i < len; ++i) w += x[i] * y[i];
    w *= tau;
    y[0] -= w;
    for (int64_t i = 1; i < len; ++i) y[i] -= w * x[i];
}

int idko_qr_column_pivoted(const double* a, int64_t m, int64_t n, int64_t steps, double* q,
                           double* r, int64_t* perm, double* taus_out, double* work_out) {
    const int64_t mn = m < n ? m : n;
    if (steps < 1 || steps > mn)
        return fail(IDKO_INVALID_ARG, "qr_column_pivoted: max_steps must lie in [1, min(rows, cols)]");
    double* work = (double*)malloc(sizeof(double) * (size_t)(m * n));
    double* live = (double*)malloc(sizeof(double) * (size_t)n);
    double* anchor = (double*)malloc(sizeof(double) * (size_t)n);
    double* taus = (double*)calloc((size_t)steps, sizeof(double));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)m);
    if (!work || !live || !anchor || !taus || !tmp) {
        free(work); free(live); free(anchor); free(taus); free(tmp);
        return fail(IDKO_NO_MEMORY, "out of memory");
    }
    memcpy(work, a, sizeof(double) * (size_t)(m * n));
    for (int64_t j = 0; j < n; ++j) perm[j] = j;

    /* qr.cpp:56-62 */
    for (int64_t j = 0; j < n; ++j) {
        double s = 0.0;
        const double* col = work + IDX(0, j, m);
        for (int64_t i = 0; i < m; ++i) s += col[i] * col[i];
        live[j] = anchor[j] = s;
    }

    for (int64_t step = 0; step < steps; ++step) {
        /* qr.cpp:66-78 */
        double vmax = 0.0;
        for (int64_t l = step; l < n; ++l) vmax = vmax < live[l] ? live[l] : vmax;
        int64_t pivot = step;
        if (vmax > 0.0) {
            const double threshold = (1.0 - 1e-14) * sqrt(vmax);
            for (int64_t l = step; l < n; ++l) {
                if (sqrt(live[l]) >= threshold) {
                    pivot = l;
                    break;
                }
            }
        }
        /* qr.cpp:79-86 */
        if (pivot != step) {
            double* cs = work + IDX(0, step, m);
            double* cp = work + IDX(0, pivot, m);
            memcpy(tmp, cs, sizeof(double) * (size_t)m);
            memcpy(cs, cp, sizeof(double) * (size_t)m);
            memcpy(cp, tmp, sizeof(double) * (size_t)m);
            int64_t tp = perm[step]; perm[step] = perm[pivot]; perm[pivot] = tp;
            double t = live[step]; live[step] = live[pivot]; live[pivot] = t;
            t = anchor[step]; anchor[step] = anchor[pivot]; anchor[pivot] = t;
        }
        /* qr.cpp:88-94 */
        double* pivot_col = work + IDX(step, step, m);
        const int64_t len = m - step;
        const double tau = make_householder(pivot_col, len);
        taus[step] = tau;
        for (int64_t l = step + 1; l < n; ++l)
            apply_householder(pivot_col, tau, work + IDX(step, l, m), len);
        /* qr.cpp:96-106 */
        for (int64_t l = step + 1; l < n; ++l) {
            const double head = work[IDX(step, l, m)];
            live[l] -= head * head;
            if (live[l] < 0.0) live[l] = 0.0;
            if (live[l] <= 1e-6 * anchor[l]) {
                double fresh = 0.0;
                const double* col = work + IDX(0, l, m);
                for (int64_t i = step + 1; i < m; ++i) fresh += col[i] * col[i];
                live[l] = anchor[l] = fresh;
            }
        }
    }

    /* qr.cpp:109-117 */
    if (q) {
        memset(q, 0, sizeof(double) * (size_t)(m * steps));
        for (int64_t j = 0; j < steps; ++j) q[IDX(j, j, m)] = 1.0;
        for (int64_t step = steps; step-- > 0;) {
            const double* v = work + IDX(step, step, m);
            const int64_t len = m - step;
            for (int64_t j = step; j < steps; ++j)
                apply_householder(v, taus[step], q + IDX(step, j, m), len);
        }
    }
    /* qr.cpp:119-123 */
    memset(r, 0, sizeof(double) * (size_t)(steps * n));
    for (int64_t j = 0; j < n; ++j) {
        const int64_t top = (j + 1) < steps ? (j + 1) : steps;
        for (int64_t i = 0; i < top; ++i) r[IDX(i, j, steps)] = work[IDX(i, j, m)];
    }
    if (taus_out) memcpy(taus_out, taus, sizeof(double) * (size_t)steps);
    if (work_out) memcpy(work_out, work, sizeof(double) * (size_t)(m * n));
    free(work); free(live); free(anchor); free(taus); free(tmp);
    return IDKO_OK;
}

/* ------------------------------------------------------------------------ */
/* Solvers (solve.cpp).                                                      */
/* ------------------------------------------------------------------------ */
/* solve.cpp:23-53; t is k x k, b (k x nrhs) is overwritten with x. */
int idko_solve_triangular(const double* t, int64_t k, double* x, int64_t nrhs, int upper) {
    for (int64_t i = 0; i < k; ++i) {
        if (fabs(t[IDX(i, i, k)]) <= 1e-300) {
            snprintf(g_err, sizeof g_err, "solve_triangular: zero diagonal at index %lld", (long long)i);
            return IDKO_SINGULAR;
        }
    }
    if (!upper) {
        for (int64_t j = 0; j < nrhs; ++j) {
            double* xj = x + IDX(0, j, k);
            for (int64_t i = 0; i < k; ++i) {
                double acc = xj[i];
                for (int64_t l = 0; l < i; ++l) acc -= t[IDX(i, l, k)] * xj[l];
                xj[i] = acc / t[IDX(i, i, k)];
            }
        }
    } else {
        for (int64_t j = 0; j < nrhs; ++j) {
            double* xj = x + IDX(0, j, k);
            for (int64_t i = k; i-- > 0;) {
                double acc = xj[i];
                for (int64_t l = i + 1; l < k; ++l) acc -= t[IDX(i, l, k)] * xj[l];
                xj[i] = acc / t[IDX(i, i, k)];
            }
        }
    }
    return IDKO_OK;
}

/* solve.cpp:55-78 */
int idko_solve_posdef(const double* s, int64_t k, double* b, int64_t nrhs) {
    double* l = (double*)calloc((size_t)(k * k), sizeof(double));
    double* lt = (double*)calloc((size_t)(k * k), sizeof(double));
    if (!l || !lt) { free(l); free(lt); return fail(IDKO_NO_MEMORY, "out of memory"); }
    for (int64_t i = 0; i < k; ++i) {
        for (int64_t j = 0; j <= i; ++j) {
            double acc = s[IDX(i, j, k)];
            for (int64_t p = 0; p < j; ++p) acc -= l[IDX(i, p, k)] * l[IDX(j, p, k)];
            if (i == j) {
                if (acc <= 0.0) {
                    snprintf(g_err, sizeof g_err, "solve_posdef: non-positive pivot at index %lld", (long long)i);
                    free(l); free(lt);
                    return IDKO_NOT_POSDEF;
                }
                l[IDX(i, i, k)] = sqrt(acc);
            } else {
                l[IDX(i, j, k)] = acc / l[IDX(j, j, k)];
            }
        }
    }
    int rc = idko_solve_triangular(l, k, b, nrhs, 0);
    if (rc == IDKO_OK) {
        idko_transpose(l, k, k, lt);
        rc = idko_solve_triangular(lt, k, b, nrhs, 1);
    }
    free(l); free(lt);
    return rc;
}

/* solve.cpp:97-258: Bunch-Kaufman LDL^T, lower storage. */
typedef struct { int64_t start, size, swap; } pivot_block;

static void swap_symmetric_lower(double* a, int64_t n, int64_t r, int64_t p) {
    double t;
    for (int64_t i = p + 1; i < n; ++i) { t = a[IDX(i, r, n)]; a[IDX(i, r, n)] = a[IDX(i, p, n)]; a[IDX(i, p, n)] = t; }
    for (int64_t j = r + 1; j < p; ++j) { t = a[IDX(j, r, n)]; a[IDX(j, r, n)] = a[IDX(p, j, n)]; a[IDX(p, j, n)] = t; }
    t = a[IDX(r, r, n)]; a[IDX(r, r, n)] = a[IDX(p, p, n)]; a[IDX(p, p, n)] = t;
}

static int ldlt_bunch_kaufman(double* a, int64_t n, pivot_block* blocks, int64_t* nblocks) {
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int64_t k = 0, nb = 0;
    while (k < n) {
        int64_t kstep = 1;
        const double absakk = fabs(a[IDX(k, k, n)]);
        int64_t imax = k;
        double colmax = 0.0;
        for (int64_t i = k + 1; i < n; ++i) {
            const double v = fabs(a[IDX(i, k, n)]);
            if (v > colmax) { colmax = v; imax = i; }
        }
        if ((absakk > colmax ? absakk : colmax) == 0.0) {
            snprintf(g_err, sizeof g_err, "solve_symmetric_indefinite: zero pivot block at index %lld", (long long)k);
            return IDKO_SINGULAR;
        }
        int64_t kp = k;
        if (absakk < alpha * colmax) {
            double rowmax = 0.0;
            for (int64_t j = k; j < imax; ++j) { const double v = fabs(a[IDX(imax, j, n)]); rowmax = rowmax < v ? v : rowmax; }
            for (int64_t i = imax + 1; i < n; ++i) { const double v = fabs(a[IDX(i, imax, n)]); rowmax = rowmax < v ? v : rowmax; }
            if (absakk >= alpha * colmax * (colmax / rowmax)) {
                kp = k;
            } else if (fabs(a[IDX(imax, imax, n)]) >= alpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int64_t kk = k + kstep - 1;
        if (kp != kk) {
            swap_symmetric_lower(a, n, kk, kp);
            if (kstep == 2) { double t = a[IDX(kk, k, n)]; a[IDX(kk, k, n)] = a[IDX(kp, k, n)]; a[IDX(kp, k, n)] = t; }
        }
        if (kstep == 1) {
            const double d = a[IDX(k, k, n)];
            if (d == 0.0) {
                snprintf(g_err, sizeof g_err, "solve_symmetric_indefinite: singular 1x1 pivot at index %lld", (long long)k);
                return IDKO_SINGULAR;
            }
            const double inv = 1.0 / d;
            for (int64_t j = k + 1; j < n; ++j) {
                const double w = a[IDX(j, k, n)] * inv;
                for (int64_t i = j; i < n; ++i) a[IDX(i, j, n)] -= a[IDX(i, k, n)] * w;
            }
            for (int64_t i = k + 1; i < n; ++i) a[IDX(i, k, n)] *= inv;
        } else {
            const double d21 = a[IDX(k + 1, k, n)];
            if (d21 == 0.0) {
                snprintf(g_err, sizeof g_err, "solve_symmetric_indefinite: singular 2x2 pivot at index %lld", (long long)k);
                return IDKO_SINGULAR;
            }
            const double d11 = a[IDX(k + 1, k + 1, n)] / d21;
            const double d22 = a[IDX(k, k, n)] / d21;
            const double det = d11 * d22 - 1.0;
            if (det == 0.0) {
                snprintf(g_err, sizeof g_err, "solve_symmetric_indefinite: singular 2x2 pivot at index %lld", (long long)k);
                return IDKO_SINGULAR;
            }
            const double t = 1.0 / det / d21;
            for (int64_t j = k + 2; j < n; ++j) {
                const double wk = t * (d11 * a[IDX(j, k, n)] - a[IDX(j, k + 1, n)]);
                const double wk1 = t * (d22 * a[IDX(j, k + 1, n)] - a[IDX(j, k, n)]);
                for (int64_t i = j; i < n; ++i)
                    a[IDX(i, j, n)] -= a[IDX(i, k, n)] * wk + a[IDX(i, k + 1, n)] * wk1;
                a[IDX(j, k, n)] = wk;
                a[IDX(j, k + 1, n)] = wk1;
            }
        }
        blocks[nb].start = k; blocks[nb].size = kstep; blocks[nb].swap = kp; ++nb;
        k += kstep;
    }
    *nblocks = nb;
    return IDKO_OK;
}

static void swap_rows(double* b, int64_t n, int64_t nrhs, int64_t r, int64_t p) {
    if (r == p) return;
    for (int64_t j = 0; j < nrhs; ++j) { double t = b[IDX(r, j, n)]; b[IDX(r, j, n)] = b[IDX(p, j, n)]; b[IDX(p, j, n)] = t; }
}

static void ldlt_solve(const double* a, int64_t n, const pivot_block* blocks, int64_t nb, double* b, int64_t nrhs) {
    for (int64_t bi = 0; bi < nb; ++bi) {
        const pivot_block* blk = &blocks[bi];
        const int64_t k = blk->start;
        swap_rows(b, n, nrhs, k + blk->size - 1, blk->swap);
        for (int64_t j = 0; j < nrhs; ++j) {
            double* bj = b + IDX(0, j, n);
            if (blk->size == 1) {
                const double bk = bj[k];
                for (int64_t i = k + 1; i < n; ++i) bj[i] -= a[IDX(i, k, n)] * bk;
            } else {
                const double bk = bj[k], bk1 = bj[k + 1];
                for (int64_t i = k + 2; i < n; ++i) bj[i] -= a[IDX(i, k, n)] * bk + a[IDX(i, k + 1, n)] * bk1;
            }
        }
    }
    for (int64_t bi = 0; bi < nb; ++bi) {
        const pivot_block* blk = &blocks[bi];
        const int64_t k = blk->start;
        if (blk->size == 1) {
            const double d = a[IDX(k, k, n)];
            for (int64_t j = 0; j < nrhs; ++j) b[IDX(k, j, n)] /= d;
        } else {
            const double akm1k = a[IDX(k + 1, k, n)];
            const double akm1 = a[IDX(k, k, n)] / akm1k;
            const double ak = a[IDX(k + 1, k + 1, n)] / akm1k;
            const double denom = akm1 * ak - 1.0;
            for (int64_t j = 0; j < nrhs; ++j) {
                const double bkm1 = b[IDX(k, j, n)] / akm1k;
                const double bk = b[IDX(k + 1, j, n)] / akm1k;
                b[IDX(k, j, n)] = (ak * bkm1 - bk) / denom;
                b[IDX(k + 1, j, n)] = (akm1 * bk - bkm1) / denom;
            }
        }
    }
    for (int64_t bi = nb; bi-- > 0;) {
        const pivot_block* blk = &blocks[bi];
        const int64_t k = blk->start;
        const int64_t below = k + blk->size;
        for (int64_t j = 0; j < nrhs; ++j) {
            double* bj = b + IDX(0, j, n);
            for (int64_t c = k; c < below; ++c) {
                double acc = 0.0;
                for (int64_t i = below; i < n; ++i) acc += a[IDX(i, c, n)] * bj[i];
                bj[c] -= acc;
            }
        }
        swap_rows(b, n, nrhs, k + blk->size - 1, blk->swap);
    }
}

/* solve.cpp:262-274 */
int idko_solve_symmetric_indefinite(const double* s, int64_t k, double* b, int64_t nrhs) {
    double* sym = (double*)malloc(sizeof(double) * (size_t)(k * k));
    pivot_block* blocks = (pivot_block*)malloc(sizeof(pivot_block) * (size_t)(k > 0 ? k : 1));
    if (!sym || !blocks) { free(sym); free(blocks); return fail(IDKO_NO_MEMORY, "out of memory"); }
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i < k; ++i) sym[IDX(i, j, k)] = 0.5 * (s[IDX(i, j, k)] + s[IDX(j, i, k)]);
    int64_t nb = 0;
    int rc = ldlt_bunch_kaufman(sym, k, blocks, &nb);
    if (rc == IDKO_OK) ldlt_solve(sym, k, blocks, nb, b, nrhs);
    free(sym); free(blocks);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* ID algorithms (id.cpp).                                                   */
/* ------------------------------------------------------------------------ */
static int require_rank_in_range(int64_t m, int64_t n, int64_t k, const char* op) {
    if (m == 0 || n == 0) { snprintf(g_err, sizeof g_err, "%s: empty matrix", op); return IDKO_INVALID_ARG; }
    const int64_t mn = m < n ? m : n;
    if (k < 1 || k > mn) { snprintf(g_err, sizeof g_err, "%s: k must lie in [1, min(rows, cols)]", op); return IDKO_INVALID_ARG; }
    return IDKO_OK;
}

/* id.cpp:20-25 */
static void leading_block(const double* r, int64_t k, double* out) {
    memset(out, 0, sizeof(double) * (size_t)(k * k));
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = 0; i <= j; ++i) out[IDX(i, j, k)] = r[IDX(i, j, k)];
}

/* Shared tail of optim_id / optim_rid (id.cpp:33-44, 65-75). */
static int normal_equation_tail(const double* a, int64_t m, int64_t n, int64_t k, const double* c,
                                const double* r, int indefinite, double* z, double* approx) {
    double* rk = (double*)malloc(sizeof(double) * (size_t)(k * k));
    double* gram = (double*)malloc(sizeof(double) * (size_t)(k * k));
    if (!rk || !gram) { free(rk); free(gram); return fail(IDKO_NO_MEMORY, "out of memory"); }
    leading_block(r, k, rk);
    idko_matmul_transpose_a(rk, k, k, rk, k, gram);
    idko_matmul_transpose_a(c, m, k, a, n, z); /* rhs = C^T A */
    int rc = indefinite ? idko_solve_symmetric_indefinite(gram, k, z, n) : idko_solve_posdef(gram, k, z, n);
    if (rc == IDKO_OK && approx) idko_matmul(c, m, k, z, n, approx);
    free(rk); free(gram);
    return rc;
}

/* id.cpp:29-45 */
int idko_optim_id(const double* a, int64_t m, int64_t n, int64_t k, int64_t* cols, double* z, double* approx) {
    int rc = require_rank_in_range(m, n, k, "optim_id");
    if (rc) return rc;
    double* r = (double*)malloc(sizeof(double) * (size_t)(k * n));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    double* c = (double*)malloc(sizeof(double) * (size_t)(m * k));
    if (!r || !perm || !c) { free(r); free(perm); free(c); return fail(IDKO_NO_MEMORY, "out of memory"); }
    rc = idko_qr_column_pivoted(a, m, n, k, NULL, r, perm, NULL, NULL);
    if (rc == IDKO_OK) {
        memcpy(cols, perm, sizeof(int64_t) * (size_t)k);
        idko_select_columns(a, m, n, cols, k, c);
        rc = normal_equation_tail(a, m, n, k, c, r, 0, z, approx);
    }
    free(r); free(perm); free(c);
    return rc;
}

/* id.cpp:47-76 */
int idko_optim_rid(const double* a, int64_t m, int64_t n, int64_t k, double frac, uint64_t seed,
                   int64_t* cols, double* z, double* approx) {
    int rc = require_rank_in_range(m, n, k, "optim_rid");
    if (rc) return rc;
    if (!(frac >= 0.0)) return fail(IDKO_INVALID_ARG, "optim_rid: oversampling_fraction must be non-negative");
    int64_t p = k + (int64_t)(uint64_t)(frac * (double)k);
    if (p > n) p = n;
    int64_t* sampled = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    double* as = (double*)malloc(sizeof(double) * (size_t)(m * p));
    double* r = (double*)malloc(sizeof(double) * (size_t)(k * p));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    double* c = (double*)malloc(sizeof(double) * (size_t)(m * k));
    if (!sampled || !as || !r || !perm || !c) {
        free(sampled); free(as); free(r); free(perm); free(c);
        return fail(IDKO_NO_MEMORY, "out of memory");
    }
    rc = idko_sample_without_replacement(n, p, seed, sampled);
    if (rc == IDKO_OK) {
        idko_select_columns(a, m, n, sampled, p, as);
        rc = idko_qr_column_pivoted(as, m, p, k, NULL, r, perm, NULL, NULL);
    }
    if (rc == IDKO_OK) {
        for (int64_t i = 0; i < k; ++i) cols[i] = sampled[perm[i]];
        idko_select_columns(as, m, p, perm, k, c);
        rc = normal_equation_tail(a, m, n, k, c, r, 1, z, approx);
    }
    free(sampled); free(as); free(r); free(perm); free(c);
    return rc;
}

int idko_interp_decomp(const double* a, int64_t m, int64_t n, int64_t k, const double* omega,
                       int64_t l, int64_t* cols, double* z, double* c, double* approx) {
    int rc = require_rank_in_range(m, n, k, omega ? "sketch_id" : "interp_decomp");
    if (rc) return rc;
    const int64_t mp = omega ? l : m; /* rows of the pivoted matrix */
    if (omega && (l < k)) return fail(IDKO_INVALID_ARG, "sketch_id: sketch rows must be >= k");
    double* y = NULL;
    if (omega) {
        y = (double*)malloc(sizeof(double) * (size_t)(l * n));
        if (!y) return fail(IDKO_NO_MEMORY, "out of memory");
        idko_matmul(omega, l, m, a, n, y); /* Y = Omega A, matrix.cpp:28-48 */
    }
    double* r = (double*)malloc(sizeof(double) * (size_t)(k * n));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    double* r11 = (double*)malloc(sizeof(double) * (size_t)(k * k));
    double* t = (double*)malloc(sizeof(double) * (size_t)(k * (n - k > 0 ? n - k : 1)));
    if (!r || !perm || !r11 || !t) {
        free(y); free(r); free(perm); free(r11); free(t);
        return fail(IDKO_NO_MEMORY, "out of memory");
    }
    rc = idko_qr_column_pivoted(omega ? y : a, mp, n, k, NULL, r, perm, NULL, NULL);
    if (rc == IDKO_OK) {
        leading_block(r, k, r11);
        memcpy(t, r + IDX(0, k, k), sizeof(double) * (size_t)(k * (n - k)));
        rc = idko_solve_triangular(r11, k, t, n - k, 1);
        if (rc == IDKO_SINGULAR && !omega) {
            /* optim_id surfaces rank deficiency through Cholesky (solve.cpp:66). */
            rc = IDKO_NOT_POSDEF;
        }
    }
    if (rc == IDKO_OK) {
        memcpy(cols, perm, sizeof(int64_t) * (size_t)k);
        for (int64_t j = 0; j < k; ++j) {
            double* zj = z + IDX(0, perm[j], k);
            memset(zj, 0, sizeof(double) * (size_t)k);
            zj[j] = 1.0;
        }
        for (int64_t j = k; j < n; ++j)
            memcpy(z + IDX(0, perm[j], k), t + IDX(0, j - k, k), sizeof(double) * (size_t)k);
        double* cc = c;
        if (!cc && approx) cc = (double*)malloc(sizeof(double) * (size_t)(m * k));
        if (cc) idko_select_columns(a, m, n, cols, k, cc);
        if (approx && cc) idko_matmul(cc, m, k, z, n, approx);
        if (cc != c) free(cc);
    }
    free(y); free(r); free(perm); free(r11); free(t);
    return rc;
}

/* id.cpp:78-95 */
int idko_id_auto(const double* a, int64_t m, int64_t n, int64_t k, int method, uint64_t seed,
                 double frac, int64_t p, int omega_mode, int64_t* cols, double* z, double* approx,
                 int* transposed) {
    int rc = require_rank_in_range(m, n, k, "id_auto");
    if (rc) return rc;
    const int tall = m > n;
    const double* src = a;
    double* at = NULL;
    int64_t mm = m, nn = n;
    if (tall) {
        at = (double*)malloc(sizeof(double) * (size_t)(m * n));
        if (!at) return fail(IDKO_NO_MEMORY, "out of memory");
        idko_transpose(a, m, n, at);
        src = at; mm = n; nn = m;
    }
    double* dual_approx = NULL;
    if (approx) {
        dual_approx = tall ? (double*)malloc(sizeof(double) * (size_t)(m * n)) : approx;
        if (!dual_approx) { free(at); return fail(IDKO_NO_MEMORY, "out of memory"); }
    }
    if (method == 0) {
        rc = idko_optim_id(src, mm, nn, k, cols, z, dual_approx);
    } else if (method == 1) {
        rc = idko_optim_rid(src, mm, nn, k, frac, seed, cols, z, dual_approx);
    } else {
        const int64_t l = k + p;
        double* omega = (double*)malloc(sizeof(double) * (size_t)(l * mm));
        if (!omega) rc = fail(IDKO_NO_MEMORY, "out of memory");
        else {
            if (omega_mode == 0) idko_omega_philox(l, mm, seed, omega);
            else idko_generate(1, l, mm, seed, omega);
            rc = idko_interp_decomp(src, mm, nn, k, omega, l, cols, z, NULL, dual_approx);
        }
        free(omega);
    }
    if (rc == IDKO_OK && approx && tall) idko_transpose(dual_approx, mm, nn, approx);
    if (tall && dual_approx) free(dual_approx);
    free(at);
    if (transposed) *transposed = tall;
    return rc;
}

/* id.cpp:97-122 */
int idko_diagnostics(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t k,
                     const double* z, int64_t zcols, const double* approx, double out[4]) {
    const double denom = idko_frobenius_norm(a, m * n);
    const double dist = idko_frobenius_distance(a, approx, m * n);
    out[0] = denom > 0.0 ? dist / denom : (dist > 0.0 ? INFINITY : 0.0);
    out[1] = idko_max_abs(z, k * zcols);
    double dev = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        const int64_t col = cols[j];
        if (col < 0 || col >= zcols) return fail(IDKO_INVALID_ARG, "diagnostics: column index outside coefficient matrix");
        for (int64_t i = 0; i < k; ++i) {
            const double want = i == j ? 1.0 : 0.0;
            const double d = fabs(z[IDX(i, col, k)] - want);
            dev = dev < d ? d : dev;
        }
    }
    out[2] = dev;
    out[3] = out[1] <= 2.0 + 1e-12 ? 1.0 : 0.0;
    return IDKO_OK;
}
