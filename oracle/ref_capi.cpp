// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libidkit_ref.so).  It lets the Python tests and bench.py's
// reference arm call the reference's own public API (id.hpp, qr.hpp,
// solve.hpp, matrix.hpp, datasets.hpp, tests/support/oracles.hpp) with plain
// pointers.  Nothing here re-implements reference arithmetic: every entry
// copies into an idkit::Matrix, calls the reference function, copies out.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "idkit/datasets.hpp"
#include "idkit/errors.hpp"
#include "idkit/id.hpp"
#include "idkit/matrix.hpp"
#include "idkit/qr.hpp"
#include "idkit/random.hpp"
#include "idkit/solve.hpp"
#include "idkit/svd.hpp"
#include "support/oracles.hpp"

using idkit::Matrix;

namespace {
thread_local std::string g_err;

Matrix from_ptr(const double* p, int64_t m, int64_t n) {
    Matrix a(static_cast<std::size_t>(m), static_cast<std::size_t>(n));
    if (m * n > 0) std::memcpy(a.data(), p, sizeof(double) * static_cast<std::size_t>(m * n));
    return a;
}

void to_ptr(const Matrix& a, double* p) {
    if (p && !a.empty()) std::memcpy(p, a.data(), sizeof(double) * a.rows() * a.cols());
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const idkit::SingularMatrixError& e) {
        g_err = e.what();
        return 2;
    } catch (const idkit::NotPositiveDefiniteError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

void put_result(const idkit::IdResult& r, int64_t* cols, double* z, double* approx, int* transposed) {
    for (std::size_t i = 0; i < r.cols.size(); ++i) cols[i] = static_cast<int64_t>(r.cols[i]);
    to_ptr(r.z, z);
    to_ptr(r.approx, approx);
    if (transposed) *transposed = r.transposed ? 1 : 0;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_optim_id(const double* a, int64_t m, int64_t n, int64_t k, int64_t* cols, double* z,
                 double* approx) {
    return guarded([&] {
        put_result(idkit::optim_id(from_ptr(a, m, n), static_cast<std::size_t>(k)), cols, z, approx,
                   nullptr);
    });
}

int ref_optim_rid(const double* a, int64_t m, int64_t n, int64_t k, double frac, uint64_t seed,
                  int64_t* cols, double* z, double* approx) {
    return guarded([&] {
        put_result(idkit::optim_rid(from_ptr(a, m, n), static_cast<std::size_t>(k), frac, seed), cols,
                   z, approx, nullptr);
    });
}

int ref_id_auto(const double* a, int64_t m, int64_t n, int64_t k, int randomized, uint64_t seed,
                double frac, int64_t* cols, double* z, double* approx, int* transposed) {
    return guarded([&] {
        put_result(idkit::id_auto(from_ptr(a, m, n), static_cast<std::size_t>(k),
                                  randomized ? idkit::IdMethod::randomized
                                             : idkit::IdMethod::deterministic,
                                  seed, frac),
                   cols, z, approx, transposed);
    });
}

int ref_qr_column_pivoted(const double* a, int64_t m, int64_t n, int64_t steps, double* q,
                          double* r, int64_t* perm) {
    return guarded([&] {
        const idkit::PivotedQr f =
            idkit::qr_column_pivoted(from_ptr(a, m, n), static_cast<std::size_t>(steps));
        to_ptr(f.q, q);
        to_ptr(f.r, r);
        for (std::size_t i = 0; i < f.perm.size(); ++i) perm[i] = static_cast<int64_t>(f.perm[i]);
    });
}

int ref_solve_triangular(const double* t, int64_t k, const double* b, int64_t nrhs, int upper,
                         double* x) {
    return guarded([&] {
        to_ptr(idkit::solve_triangular(from_ptr(t, k, k), from_ptr(b, k, nrhs),
                                       upper ? idkit::Triangle::upper : idkit::Triangle::lower),
               x);
    });
}

int ref_solve_posdef(const double* s, int64_t k, const double* b, int64_t nrhs, double* x) {
    return guarded([&] { to_ptr(idkit::solve_posdef(from_ptr(s, k, k), from_ptr(b, k, nrhs)), x); });
}

int ref_solve_symmetric_indefinite(const double* s, int64_t k, const double* b, int64_t nrhs,
                                   double* x) {
    return guarded([&] {
        to_ptr(idkit::solve_symmetric_indefinite(from_ptr(s, k, k), from_ptr(b, k, nrhs)), x);
    });
}

int ref_matmul(const double* a, int64_t m, int64_t k, const double* b, int64_t n, double* out) {
    return guarded([&] { to_ptr(idkit::matmul(from_ptr(a, m, k), from_ptr(b, k, n)), out); });
}

int ref_select_columns(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t ncols,
                       double* out) {
    return guarded([&] {
        std::vector<std::size_t> c(cols, cols + ncols);
        to_ptr(idkit::select_columns(from_ptr(a, m, n), std::span<const std::size_t>(c)), out);
    });
}

int ref_transpose(const double* a, int64_t m, int64_t n, double* out) {
    return guarded([&] { to_ptr(idkit::transpose(from_ptr(a, m, n)), out); });
}

int ref_diagnostics(const double* a, int64_t m, int64_t n, const int64_t* cols, int64_t k,
                    const double* z, int64_t zcols, const double* approx, double* out4) {
    return guarded([&] {
        idkit::IdResult r;
        r.cols.assign(cols, cols + k);
        r.z = from_ptr(z, k, zcols);
        r.approx = from_ptr(approx, m, n);
        const idkit::IdDiagnostics d = idkit::diagnostics(from_ptr(a, m, n), r);
        out4[0] = d.relative_error;
        out4[1] = d.max_abs_z;
        out4[2] = d.identity_deviation;
        out4[3] = d.entry_bound_satisfied ? 1.0 : 0.0;
    });
}

// datasets.cpp:15-33; kind 0 boolean, 1 gaussian, 2 uniform.
int ref_generate(int kind, int64_t rows, int64_t cols, uint64_t seed, double* out) {
    return guarded([&] {
        const idkit::GeneratorKind g = kind == 0   ? idkit::GeneratorKind::boolean
                                       : kind == 1 ? idkit::GeneratorKind::gaussian
                                                   : idkit::GeneratorKind::uniform;
        to_ptr(idkit::generate(g, static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), seed),
               out);
    });
}

uint64_t ref_mix_seed(uint64_t base, const char* label) { return idkit::mix_seed(base, label); }

int ref_sample_without_replacement(int64_t population, int64_t count, uint64_t seed, int64_t* out) {
    return guarded([&] {
        idkit::RandomEngine rng = idkit::seeded_engine(seed);
        const auto s = idkit::sample_without_replacement(static_cast<std::size_t>(population),
                                                         static_cast<std::size_t>(count), rng);
        for (std::size_t i = 0; i < s.size(); ++i) out[i] = static_cast<int64_t>(s[i]);
    });
}

// tests/support/oracles.hpp:40-46
int ref_gaussian_matrix(int64_t m, int64_t n, uint64_t seed, double* out) {
    return guarded([&] {
        to_ptr(oracles::gaussian_matrix(static_cast<std::size_t>(m), static_cast<std::size_t>(n), seed),
               out);
    });
}

// tests/support/oracles.hpp:83-138 (pivot-order oracle independent of qr.cpp)
int ref_gram_schmidt_pivoted(const double* a, int64_t m, int64_t n, int64_t steps, int64_t* order,
                             double* norms) {
    return guarded([&] {
        const auto g = oracles::gram_schmidt_pivoted(from_ptr(a, m, n), static_cast<std::size_t>(steps));
        for (std::size_t i = 0; i < g.order.size(); ++i) {
            order[i] = static_cast<int64_t>(g.order[i]);
            norms[i] = g.pivot_norms[i];
        }
    });
}

int ref_truncated_svd_error(const double* a, int64_t m, int64_t n, int64_t k, double* out) {
    return guarded([&] { *out = idkit::truncated_svd_error(from_ptr(a, m, n), static_cast<std::size_t>(k)); });
}

// The north-star ID composed from the reference's public primitives
// (SURVEY.md §3(5)): Y = matmul(Omega, A) (omega may be null -> Y = A),
// qr_column_pivoted(Y, k), solve_triangular(R11, R12, upper), scatter by perm,
// select_columns.  Pure calls into the reference; only the glue is ours.
int ref_sketch_id(const double* a, int64_t m, int64_t n, int64_t k, const double* omega, int64_t l,
                  int64_t* cols, double* z, double* c) {
    return guarded([&] {
        const Matrix A = from_ptr(a, m, n);
        const Matrix Y = omega ? idkit::matmul(from_ptr(omega, l, m), A) : A;
        const idkit::PivotedQr f = idkit::qr_column_pivoted(Y, static_cast<std::size_t>(k));
        const std::size_t kk = static_cast<std::size_t>(k), nn = static_cast<std::size_t>(n);
        Matrix r11(kk, kk), r12(kk, nn - kk);
        for (std::size_t j = 0; j < kk; ++j)
            for (std::size_t i = 0; i <= j; ++i) r11(i, j) = f.r(i, j);
        for (std::size_t j = kk; j < nn; ++j)
            for (std::size_t i = 0; i < kk; ++i) r12(i, j - kk) = f.r(i, j);
        const Matrix t = nn > kk ? idkit::solve_triangular(r11, r12, idkit::Triangle::upper) : r12;
        if (nn == kk) {
            // still validate the diagonal like solve_triangular would
            (void)idkit::solve_triangular(r11, Matrix(kk, 1), idkit::Triangle::upper);
        }
        Matrix zz(kk, nn);
        for (std::size_t j = 0; j < kk; ++j) zz(j, f.perm[j]) = 1.0;
        for (std::size_t j = kk; j < nn; ++j)
            for (std::size_t i = 0; i < kk; ++i) zz(i, f.perm[j]) = t(i, j - kk);
        std::vector<std::size_t> cc(f.perm.begin(), f.perm.begin() + static_cast<std::ptrdiff_t>(kk));
        for (std::size_t i = 0; i < kk; ++i) cols[i] = static_cast<int64_t>(cc[i]);
        to_ptr(zz, z);
        if (c) to_ptr(idkit::select_columns(A, cc), c);
    });
}

// The same composition at BASELINE scale on `threads` host threads, for the
// full-size parity tests (cfg4 / cfg5) and bench.py's reference arm.
//
// Bit-identical to ref_sketch_id with one thread: the reference's matmul
// computes output column j from input column j only (matrix.cpp:28-48), and
// solve_triangular solves each right-hand-side column on its own
// (solve.cpp:23-53), so splitting both by column blocks and calling the
// reference on each block changes no arithmetic.  qr_column_pivoted runs once,
// single-threaded, on the assembled Y.  select_columns runs per block on the
// columns that block owns (a pure copy).
//
// M (m x n) is the matrix decomposed: A itself (stored m x n, lda >= m) or,
// with trans != 0, A^T for the stored n x m matrix A (lda >= n) -- id_auto's
// dual (id.cpp:85), where every thread applies the reference's transpose to
// its own row block of A before the matmul.  Omega: verbatim (l x m) or, when
// omega == NULL, generate(gaussian, l, m, seed) inside the timed region.
// c (m x k) receives M[:, cols].  times5 (optional) = wall seconds of
// {omega, transpose + matmul, qr_column_pivoted, solve_triangular,
// select_columns}; copying A into per-thread idkit::Matrix blocks and
// assembling Y / Z from the blocks is harness work and is not timed.
int ref_sketch_id_mt(const double* a, int64_t lda, int64_t m, int64_t n, int trans, int64_t k,
                     const double* omega, int64_t l, uint64_t seed, int threads, int64_t* cols, double* z,
                     double* c, double* times5) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto secs = [](clk::time_point t0) { return std::chrono::duration<double>(clk::now() - t0).count(); };
        const std::size_t mm = static_cast<std::size_t>(m), nn = static_cast<std::size_t>(n);
        const std::size_t kk = static_cast<std::size_t>(k), ll = static_cast<std::size_t>(l);
        if (k < 1 || k > std::min(m, n) || l < k) throw std::invalid_argument("ref_sketch_id_mt: bad k / l");
        const int T = std::max(1, std::min<int>(threads, static_cast<int>(n)));
        std::vector<std::size_t> lo(T + 1);
        for (int t = 0; t <= T; ++t) lo[t] = nn * static_cast<std::size_t>(t) / static_cast<std::size_t>(T);
        auto parallel = [&](auto&& body) {
            std::vector<std::thread> pool;
            std::vector<std::exception_ptr> errs(T);
            for (int t = 0; t < T; ++t)
                pool.emplace_back([&, t] {
                    try {
                        body(t);
                    } catch (...) {
                        errs[t] = std::current_exception();
                    }
                });
            for (auto& th : pool) th.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        };
        double tm[5] = {0, 0, 0, 0, 0};
        // harness: each thread's block of the stored matrix as an idkit::Matrix
        std::vector<Matrix> blk(T);
        parallel([&](int t) {
            const std::size_t w = lo[t + 1] - lo[t];
            if (!trans) {
                blk[t] = Matrix(mm, w);
                for (std::size_t j = 0; j < w; ++j)
                    std::memcpy(blk[t].col_data(j), a + (lo[t] + j) * static_cast<std::size_t>(lda), sizeof(double) * mm);
            } else {  // rows [lo, hi) of the stored n x m matrix A
                blk[t] = Matrix(w, mm);
                for (std::size_t j = 0; j < mm; ++j)
                    std::memcpy(blk[t].col_data(j), a + j * static_cast<std::size_t>(lda) + lo[t], sizeof(double) * w);
            }
        });
        auto t0 = clk::now();
        const Matrix Om = omega ? from_ptr(omega, l, m) : idkit::generate(idkit::GeneratorKind::gaussian, ll, mm, seed);
        if (!omega) tm[0] = secs(t0);
        // Y = Omega * M, column block by column block
        std::vector<Matrix> yb(T);
        t0 = clk::now();
        parallel([&](int t) {
            if (trans) blk[t] = idkit::transpose(blk[t]);  // M's columns [lo, hi) = A^T's
            yb[t] = idkit::matmul(Om, blk[t]);
        });
        tm[1] = secs(t0);
        Matrix Y(ll, nn);
        for (int t = 0; t < T; ++t)
            if (!yb[t].empty()) std::memcpy(Y.col_data(lo[t]), yb[t].data(), sizeof(double) * ll * (lo[t + 1] - lo[t]));
        yb.clear();
        t0 = clk::now();
        const idkit::PivotedQr f = idkit::qr_column_pivoted(Y, kk);
        tm[2] = secs(t0);
        Matrix r11(kk, kk);
        for (std::size_t j = 0; j < kk; ++j)
            for (std::size_t i = 0; i <= j; ++i) r11(i, j) = f.r(i, j);
        // T = R11^-1 R12 by blocks of R12's columns
        const std::size_t nr = nn - kk;
        const int T2 = std::max(1, std::min<int>(T, static_cast<int>(std::max<std::size_t>(nr, 1))));
        std::vector<Matrix> tb(T2);
        t0 = clk::now();
        {
            std::vector<std::thread> pool;
            std::vector<std::exception_ptr> errs(T2);
            for (int t = 0; t < T2; ++t)
                pool.emplace_back([&, t] {
                    try {
                        const std::size_t b0 = nr * t / T2, b1 = nr * (t + 1) / T2;
                        Matrix r12(kk, b1 - b0);
                        for (std::size_t j = b0; j < b1; ++j)
                            for (std::size_t i = 0; i < kk; ++i) r12(i, j - b0) = f.r(i, kk + j);
                        if (b1 > b0 || nr == 0)
                            tb[t] = idkit::solve_triangular(r11, nr == 0 ? Matrix(kk, 1) : r12, idkit::Triangle::upper);
                    } catch (...) {
                        errs[t] = std::current_exception();
                    }
                });
            for (auto& th : pool) th.join();
            for (auto& e : errs)
                if (e) std::rethrow_exception(e);
        }
        tm[3] = secs(t0);
        Matrix zz(kk, nn);
        for (std::size_t j = 0; j < kk; ++j) zz(j, f.perm[j]) = 1.0;
        for (int t = 0; t < T2 && nr > 0; ++t) {
            const std::size_t b0 = nr * t / T2;
            for (std::size_t j = 0; j < tb[t].cols(); ++j)
                for (std::size_t i = 0; i < kk; ++i) zz(i, f.perm[kk + b0 + j]) = tb[t](i, j);
        }
        for (std::size_t i = 0; i < kk; ++i) cols[i] = static_cast<int64_t>(f.perm[i]);
        to_ptr(zz, z);
        if (c) {
            t0 = clk::now();
            parallel([&](int t) {
                std::vector<std::size_t> loc, at;
                for (std::size_t i = 0; i < kk; ++i)
                    if (f.perm[i] >= lo[t] && f.perm[i] < lo[t + 1]) {
                        loc.push_back(f.perm[i] - lo[t]);
                        at.push_back(i);
                    }
                if (loc.empty()) return;
                const Matrix cb = idkit::select_columns(blk[t], std::span<const std::size_t>(loc));
                for (std::size_t q = 0; q < at.size(); ++q)
                    std::memcpy(c + at[q] * mm, cb.col_data(q), sizeof(double) * mm);
            });
            tm[4] = secs(t0);
        }
        if (times5)
            for (int i = 0; i < 5; ++i) times5[i] = tm[i];
    });
}

// Threads over a batch of independent optim_id calls (cfg3; the
// calls are pure).  a holds `batch` m x n matrices at stride m*n.
int ref_optim_id_batch_mt(const double* a, int64_t batch, int64_t m, int64_t n, int64_t k, int threads,
                          int64_t* cols, double* z, double* approx) {
    return guarded([&] {
        const int T = std::max(1, std::min<int>(threads, static_cast<int>(std::max<int64_t>(batch, 1))));
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(T);
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                try {
                    for (int64_t b = t; b < batch; b += T) {
                        const idkit::IdResult r =
                            idkit::optim_id(from_ptr(a + b * m * n, m, n), static_cast<std::size_t>(k));
                        for (int64_t i = 0; i < k; ++i) cols[b * k + i] = static_cast<int64_t>(r.cols[i]);
                        to_ptr(r.z, z + b * k * n);
                        if (approx) to_ptr(r.approx, approx + b * m * n);
                    }
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

} // extern "C"
