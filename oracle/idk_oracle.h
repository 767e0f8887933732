/*
 * idk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference (idkit, /root/reference/proj) ID
 * path, used as the parity checker for the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product library (paper_2105_07076_b200) never links it.
 *
 * Every function follows the reference's operation order (no FMA contraction:
 * build with -ffp-contract=off, as the reference's CMake Release build has no
 * -march and therefore no FMA).  Parity of this restatement against the
 * reference itself is pinned by tests/test_oracle_golden.py, which compares
 * bit-for-bit with oracle/_ref (the reference sources compiled as-is) and with
 * the committed fixtures under tests/golden/.
 *
 * Matrices are column-major fp64 with an explicit leading dimension, like
 * idkit::Matrix ((i,j) at data[j*rows+i], matrix.hpp:34-35).
 */
#ifndef IDK_ORACLE_H
#define IDK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    IDKO_OK = 0,
    IDKO_INVALID_ARG = 1,  /* std::invalid_argument */
    IDKO_SINGULAR = 2,     /* SingularMatrixError   (errors.hpp:9-13)  */
    IDKO_NOT_POSDEF = 3,   /* NotPositiveDefiniteError (errors.hpp:15-19) */
    IDKO_NO_MEMORY = 4
};

/* Message of the last failing call (thread-local). */
const char* idko_last_error(void);

/* ---- RNG: random.hpp:13-20, random.cpp:10-55 ---- */
typedef struct { uint64_t mt[312]; int idx; } idko_mt64;
void idko_mt64_seed(idko_mt64* g, uint64_t seed);
uint64_t idko_mt64_next(idko_mt64* g);
double idko_next_uniform(idko_mt64* g);
double idko_next_normal(idko_mt64* g);
uint64_t idko_next_below(idko_mt64* g, uint64_t bound);
int idko_sample_without_replacement(int64_t population, int64_t count, uint64_t seed, int64_t* out);
uint64_t idko_mix_seed(uint64_t base, const char* label);
/* datasets.cpp:15-33 generate(); kind 0 = boolean, 1 = gaussian, 2 = uniform. */
int idko_generate(int kind, int64_t rows, int64_t cols, uint64_t seed, double* out);

/* Counter-based Gaussian sketch Omega (l x m, column-major): Philox4x32-10
 * keyed by seed, counter = linear element index, Box-Muller with the
 * reference's u1/u2 conventions (random.cpp:10-15).  Mirrors the device
 * generator in paper_2105_07076_b200/csrc/rng.cuh. */
void idko_philox4x32_10(uint32_t ctr[4], const uint32_t key[2]);
void idko_omega_philox(int64_t l, int64_t m, uint64_t seed, double* out);

/* ---- dense core: matrix.cpp:28-130 ---- */
int idko_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* out);
int idko_matmul_transpose_a(const double* a, int64_t k, int64_t m, const double* b, int64_t n,
                            double* out);
void idko_transpose(const double* a, int64_t m, int64_t n, double* out);
int idko_select_columns(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t ncols,
                        double* out);
double idko_frobenius_norm(const double* a, int64_t total);
double idko_frobenius_distance(const double* a, const double* b, int64_t total);
double idko_max_abs(const double* a, int64_t total);

/* ---- qr.cpp:42-126 ----
 * q (m x steps) may be NULL; r is steps x n; perm has n entries.  taus
 * (steps) and work (m x n, the final in-place factor) may be NULL. */
int idko_qr_column_pivoted(const double* a, int64_t m, int64_t n, int64_t steps, double* q,
                           double* r, int64_t* perm, double* taus, double* work);

/* ---- solve.cpp:23-274 ---- (b is overwritten by the solution) */
int idko_solve_triangular(const double* t, int64_t k, double* b, int64_t nrhs, int upper);
int idko_solve_posdef(const double* s, int64_t k, double* b, int64_t nrhs);
int idko_solve_symmetric_indefinite(const double* s, int64_t k, double* b, int64_t nrhs);

/* ---- id.cpp:29-122 ----
 * cols: k entries; z: k x n (k x m when *transposed); approx: m x n (may be NULL). */
int idko_optim_id(const double* a, int64_t m, int64_t n, int64_t k, int64_t* cols, double* z,
                  double* approx);
int idko_optim_rid(const double* a, int64_t m, int64_t n, int64_t k, double frac, uint64_t seed,
                   int64_t* cols, double* z, double* approx);

/* North-star ID composed from the reference primitives:
 *   Y = Omega*A (omega != NULL, l rows) or Y = A (omega == NULL, det),
 *   CPQR(Y, k) -> perm, R;  T = solve_triangular(R11, R12, upper);
 *   Z[:, perm[j]] = e_j (j<k), T[:, j-k] (j>=k);  C = A[:, perm[:k]].
 * c (m x k) and approx (m x n) may be NULL.  Rank deficiency surfaces as
 * IDKO_SINGULAR (sketch) or IDKO_NOT_POSDEF (det, mirroring optim_id). */
int idko_interp_decomp(const double* a, int64_t m, int64_t n, int64_t k, const double* omega,
                       int64_t l, int64_t* cols, double* z, double* c, double* approx);

/* id.cpp:78-95 orientation dispatch.  method 0 = optim_id, 1 = optim_rid,
 * 2 = sketch (omega_mode 0 = Philox(seed) of l = k+p rows, 1 = mt19937
 * generate(gaussian, l, rows, seed)).  z must hold k x max(m, n). */
int idko_id_auto(const double* a, int64_t m, int64_t n, int64_t k, int method, uint64_t seed,
                 double frac, int64_t p, int omega_mode, int64_t* cols, double* z, double* approx,
                 int* transposed);

/* id.cpp:97-122.  out[0] = relative_error, out[1] = max_abs_z,
 * out[2] = identity_deviation, out[3] = entry_bound_satisfied. */
int idko_diagnostics(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t k,
                     const double* z, int64_t zcols, const double* approx, double out[4]);

#ifdef __cplusplus
}
#endif
#endif
