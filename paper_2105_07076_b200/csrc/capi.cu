// capi.cu -- the extern "C" boundary (include/idkit_b200.h) and the host-side
// orchestration of the ID path on one B200.
//
// Stage order per call (all on the handle's stream):
//   sketch RID : [Omega] -> DMMA GEMM Y = Omega M -> persistent CPQR(Y, k)
//                -> R11 gather + blocked TRSM writing Z -> C gather -> status
//   det ID     : copy (or transpose) A -> persistent CPQR(A, k) -> same tail
//   batched    : one fused kernel, one CTA per matrix
#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/idkit_b200.h"
#include "kernels.h"
#include "nccl_api.h"

struct idk_context {
    int device = 0;
    int num_sms = 0;
    size_t smem_optin = 0;
    cudaStream_t stream = nullptr;
    std::string err;
    // compute workspace (bump-allocated per call, grow-only)
    char* ws = nullptr;
    size_t ws_cap = 0;
    size_t ws_off = 0;
    // host-entry staging (device copies of host inputs/outputs)
    char* io = nullptr;
    size_t io_cap = 0;
    int* h_status = nullptr;  // pinned
    double* h_omega = nullptr;  // pinned staging for IDK_OMEGA_MT19937
    size_t h_omega_cap = 0;
    long long* h_idx = nullptr;  // pinned staging for optim_rid's sampled columns
    size_t h_idx_cap = 0;
    int64_t launches = 0;
    int cpqr_mode = IDK_CPQR_AUTO;
    bool batched_exact = false;
    int sketch_order = IDK_SKETCH_DMMA;
    // pipelined host entry: status words land here (pinned) instead of a sync per ID
    int* async_status = nullptr;
    int* batched_status = nullptr;  // idk_optim_id_batched_host: device status words of the current chunk
    cudaStream_t s_in = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> ev_io;  // pipelined host entry: in / done / out per buffer set
    int* h_status_many = nullptr;
    int64_t h_status_many_cap = 0;
    // concurrent batch entry: child contexts, one stream + workspace each
    int lanes = 8;
    std::vector<idk_context*> kids;
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    // grouped sketch of the batch entry: a low-priority stream feeding the lanes
    cudaStream_t s_sketch = nullptr;
    std::vector<cudaEvent_t> ev_chunk;   // chunk c's Y ready
    std::vector<cudaEvent_t> ev_gprof;   // profiling: 3 per chunk (start, Omega done, GEMM done)
    // per-stage CUDA events on the launching stream (idk_set_profiling)
    bool profiling = false;
    cudaEvent_t ev[6] = {};
    float stage_ms[5] = {};
    // multi-GPU: the NCCL communicator of idk_id_sharded (idk_comm_init / idk_set_nccl_comm)
    idk::ncclComm_t nccl_comm = nullptr;
    bool nccl_owned = false;
    int nranks = 1, rank = 0;
    // peer mode of idk_id_sharded: every rank's Y buffer mapped into every other
    // rank (CUDA IPC over NVLink); the sketch writes its block straight into all of them
    double* ybuf = nullptr;  // this rank's Y (its own cudaMalloc: IPC exports whole allocations)
    size_t ybuf_cap = 0;
    double* peer_y[idk::kFanMax] = {};
    int* d_flag = nullptr;   // 1-int scratch of the stream-ordered barrier / agreement
    int p2p_state = 0;       // 0 untried, 1 on, -1 off (IPC unavailable: the NCCL all-gather runs)
    // caller-supplied host collectives (idk_set_host_collectives), used when no NCCL communicator is set
    idk_host_collectives hc = {};
    bool has_hc = false;
};

namespace {

int ensure_lanes(idk_context* h, int L);  // lane contexts of the concurrent entries (defined below)

constexpr size_t kAlign = 256;

size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

int set_err(idk_context* h, int code, const std::string& msg) {
    if (h) h->err = msg;
    return code;
}

int cuda_fail(idk_context* h, cudaError_t e, const char* where) {
    return set_err(h, IDK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define IDK_CUDA(call)                                      \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(h, _e, #call); \
    } while (0)

// Stage boundaries: 0 input prep (Omega / copy), 1 sketch GEMM, 2 CPQR,
// 3 R11 gather + TRSM (Z), 4 C gather.  mark(h, i) closes stage i-1.
void mark(idk_context* h, int i) {
    if (h->profiling) cudaEventRecord(h->ev[i], h->stream);
}

void collect_stage_times(idk_context* h) {
    if (!h->profiling) return;
    for (int i = 0; i < 5; ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]) != cudaSuccess) {
            cudaGetLastError();
            ms = 0.f;
        }
        h->stage_ms[i] = ms;
    }
}

// Grow-only buffer; growing synchronises the stream first (callers never
// hold pointers across calls: every entry synchronises before returning).
int ensure(idk_context* h, char** buf, size_t* cap, size_t bytes) {
    if (bytes <= *cap) return IDK_OK;
    cudaStreamSynchronize(h->stream);
    if (*buf) cudaFree(*buf);
    *buf = nullptr;
    *cap = 0;
    size_t want = std::max(bytes, static_cast<size_t>(1) << 20);
    if (cudaMalloc(reinterpret_cast<void**>(buf), want) != cudaSuccess) {
        cudaGetLastError();
        return set_err(h, IDK_ERR_NO_MEMORY, "cudaMalloc of " + std::to_string(want) + " bytes failed");
    }
    *cap = want;
    return IDK_OK;
}

struct Carve {
    size_t total = 0;
    size_t take(size_t bytes) {
        const size_t off = total;
        total += align_up(bytes);
        return off;
    }
};

int check_k(idk_context* h, int64_t m, int64_t n, int64_t k, const char* op) {
    if (m <= 0 || n <= 0) return set_err(h, IDK_ERR_INVALID_ARG, std::string(op) + ": empty matrix");
    if (k < 1 || k > std::min(m, n))
        return set_err(h, IDK_ERR_INVALID_ARG, std::string(op) + ": k must lie in [1, min(rows, cols)]");
    if (k > INT_MAX || m > INT_MAX) return set_err(h, IDK_ERR_INVALID_ARG, std::string(op) + ": dimension too large");
    return IDK_OK;
}

// Largest co-resident grid for the streaming CPQR kernel.
int cpqr_ctas(idk_context* h) { return h->num_sms; }

// Which CPQR kernel runs an m' x n factorisation (see idk_set_cpqr_mode).
struct CpqrChoice {
    bool resident = false;
    idk::ResidentPlan plan;
};

CpqrChoice choose_cpqr(idk_context* h, int64_t mrows, int64_t n, int64_t k) {
    CpqrChoice c;
    if (h->cpqr_mode == IDK_CPQR_STREAMING) return c;
    const int pref = h->cpqr_mode == IDK_CPQR_RESIDENT_GRID ? 1 : (h->cpqr_mode == IDK_CPQR_CLUSTER_PULL ? 2 : 0);
    c.plan = idk::cpqr_resident_plan(static_cast<int>(mrows), n, static_cast<int>(k), h->num_sms, pref);
    cudaGetLastError();
    c.resident = c.plan.ok;
    return c;
}

// Work buffers of one CPQR + Z solve on an m' x n matrix.
struct CpqrWs {
    size_t pos, pivots, taus, pub, barrier, r11, status;
    size_t xg = 0;  // streaming CPQR of a tall matrix: the shared, double-buffered reflector in L2
    bool has_xg = false;
};

// The streaming kernel keeps the reflector (m doubles) in shared memory when
// it fits; taller matrices keep one L2-resident copy (double-buffered) shared by all CTAs.
bool cpqr_needs_xglobal(int64_t mrows, int64_t n, int num_sms) {
    const int64_t G = std::min<int64_t>(n, num_sms);
    const int cols = static_cast<int>((n + G - 1) / G);
    return idk::cpqr_smem_bytes(static_cast<int>(mrows), cols) > 200 * 1024;
}

CpqrWs carve_cpqr(Carve& cv, int64_t mrows, int64_t n, int64_t k, int num_sms, const CpqrChoice& ch) {
    CpqrWs w;
    if (!ch.resident && cpqr_needs_xglobal(mrows, n, num_sms)) {
        w.has_xg = true;
        w.xg = cv.take(sizeof(double) * 2 * static_cast<size_t>(idk::cpqr_xglobal_ld(static_cast<int>(mrows))));
    }
    w.pos = cv.take(sizeof(long long) * n);
    w.pivots = cv.take(sizeof(long long) * k);
    w.taus = cv.take(sizeof(double) * k);
    size_t pub = idk::kCpqrPubBytes * 3 * static_cast<size_t>(num_sms + 1);
    if (ch.resident) pub = std::max(pub, idk::cpqr_resident_exchange_bytes(ch.plan, static_cast<int>(mrows)));
    w.pub = cv.take(pub);
    w.barrier = cv.take(sizeof(unsigned));
    w.r11 = cv.take(idk::id_solve_z_scratch(static_cast<int>(k)));
    w.status = cv.take(sizeof(int));
    return w;
}

int check_cpqr_fits(idk_context* h, int64_t mrows, int64_t n, const CpqrChoice& ch) {
    if (ch.resident) return IDK_OK;
    const int64_t G = std::min<int64_t>(n, h->num_sms);
    const int cols = static_cast<int>((n + G - 1) / G);
    if (idk::cpqr_smem_bytes(0, cols) > 200 * 1024)  // the per-column state (the reflector can live in L2)
        return set_err(h, IDK_ERR_INVALID_ARG,
                       "qr_column_pivoted: " + std::to_string(mrows) + " rows x " + std::to_string(n) +
                           " columns exceeds the persistent CPQR shared-memory budget");
    return IDK_OK;
}

cudaError_t run_cpqr(idk_context* h, const CpqrChoice& ch, double* W, int64_t mrows, int64_t n, int64_t k, char* base,
                     const CpqrWs& w, int64_t ldw = 0, const double* Win = nullptr, int64_t ldin = 0) {
    if (ldw < mrows) ldw = mrows;
    long long* pos = reinterpret_cast<long long*>(base + w.pos);
    long long* piv = reinterpret_cast<long long*>(base + w.pivots);
    double* taus = reinterpret_cast<double*>(base + w.taus);
    if (ch.resident)
        return idk::cpqr_resident_launch(ch.plan, W, ldw, static_cast<int>(mrows), n, static_cast<int>(k), pos, piv,
                                         taus, base + w.pub, reinterpret_cast<unsigned*>(base + w.barrier), h->stream,
                                         Win, ldin);
    return idk::cpqr_launch(W, ldw, static_cast<int>(mrows), n, static_cast<int>(k), pos, piv, taus, base + w.pub,
                            reinterpret_cast<unsigned*>(base + w.barrier), h->num_sms, cpqr_ctas(h), h->stream,
                            w.has_xg ? reinterpret_cast<double*>(base + w.xg) : nullptr, Win, ldin);
}

// CPQR(W) -> Z, C, cols; W is m' x n (ld m'), already resident and mutable.
int factor_and_solve(idk_context* h, const CpqrChoice& ch, double* W, int64_t mrows, int64_t n, int64_t k, char* base,
                     const CpqrWs& w, const double* d_a, int64_t lda, int64_t m_out, bool rows_of_a, int64_t* d_cols,
                     double* d_z, double* d_c, bool det, const double* Win = nullptr, int64_t ldin = 0) {
    long long* pos = reinterpret_cast<long long*>(base + w.pos);
    long long* piv = reinterpret_cast<long long*>(base + w.pivots);
    int* status = reinterpret_cast<int*>(base + w.status);
    IDK_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int), h->stream));
    mark(h, 2);
    IDK_CUDA(run_cpqr(h, ch, W, mrows, n, k, base, w, mrows, Win, ldin));
    mark(h, 3);
    IDK_CUDA(idk::id_solve_z(W, mrows, static_cast<int>(k), 0, n, piv, pos, reinterpret_cast<double*>(base + w.r11),
                             status, d_z, h->stream));
    mark(h, 4);
    h->launches += 3;
    if (d_c) {
        IDK_CUDA(idk::gather_columns(d_a, lda, m_out, piv, static_cast<int>(k), rows_of_a, d_c, h->stream));
        h->launches += 1;
    }
    mark(h, 5);
    IDK_CUDA(cudaMemcpyAsync(d_cols, piv, sizeof(long long) * k, cudaMemcpyDeviceToDevice, h->stream));
    if (h->async_status) {  // pipelined entry: the caller checks the status word later
        IDK_CUDA(cudaMemcpyAsync(h->async_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        return IDK_OK;
    }
    IDK_CUDA(cudaMemcpyAsync(h->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    collect_stage_times(h);
    const int bad = *h->h_status;
    if (bad != 0x7f7f7f7f) {
        if (det)
            return set_err(h, IDK_ERR_NOT_POSDEF,
                           "optim_id: rank-deficient input (R11 diagonal " + std::to_string(bad) +
                               " is zero; reference: solve_posdef non-positive pivot)");
        return set_err(h, IDK_ERR_SINGULAR, "solve_triangular: zero diagonal at index " + std::to_string(bad));
    }
    return IDK_OK;
}

// Deterministic ID of M (m x n).  M = A (lda >= m) or A^T (A stored n x m, lda >= n).
int det_id(idk_context* h, const double* d_a, int64_t m, int64_t n, int64_t lda, bool trans, int64_t k,
           int64_t* d_cols, double* d_z, double* d_c) {
    int rc = check_k(h, m, n, k, "optim_id");
    if (rc) return rc;
    if (!d_a || !d_cols || !d_z) return set_err(h, IDK_ERR_INVALID_ARG, "optim_id: null pointer");
    if (lda < (trans ? n : m)) return set_err(h, IDK_ERR_INVALID_ARG, "optim_id: lda too small");
    const CpqrChoice ch = choose_cpqr(h, m, n, k);
    if ((rc = check_cpqr_fits(h, m, n, ch))) return rc;
    Carve cv;
    const size_t wofs = cv.take(sizeof(double) * m * n);
    const CpqrWs w = carve_cpqr(cv, m, n, k, h->num_sms, ch);
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    double* W = reinterpret_cast<double*>(h->ws + wofs);
    mark(h, 0);
    // both CPQR kernels read A itself once and write the factor / the working copy to W
    // (the streaming kernel during its norm pass): no separate copy of A
    const bool direct = !trans;
    if (trans) {
        IDK_CUDA(idk::transpose_copy(d_a, lda, n, m, W, m, h->stream));
        h->launches += 1;
    }
    mark(h, 1);
    return factor_and_solve(h, ch, W, m, n, k, h->ws, w, d_a, lda, m, trans, d_cols, d_z, d_c, true,
                            direct ? d_a : nullptr, lda);
}

// Reference Box-Muller over mt19937_64 (random.cpp:10-15), column-major fill
// like generate(gaussian, l, m, seed) (datasets.cpp:15-33).
void host_generate_gaussian(double* out, int64_t total, uint64_t seed) {
    std::mt19937_64 rng(seed);
    const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
    for (int64_t e = 0; e < total; ++e) {
        const double u1 = static_cast<double>((rng() >> 11) + 1) * 0x1.0p-53;
        const double u2 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        out[e] = std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
    }
}

int sketch_rid(idk_context* h, const double* d_a, int64_t m, int64_t n, int64_t lda, bool trans, int64_t k,
               int64_t p, uint64_t seed, int omega_mode, const double* d_omega, int64_t* d_cols, double* d_z,
               double* d_c) {
    int rc = check_k(h, m, n, k, "sketch_rid");
    if (rc) return rc;
    if (p < 0) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: oversampling p must be non-negative");
    if (!d_a || !d_cols || !d_z) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: null pointer");
    if (lda < (trans ? n : m)) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: lda too small");
    if (omega_mode < 0 || omega_mode > 2) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: bad omega mode");
    if (omega_mode == IDK_OMEGA_VERBATIM && !d_omega)
        return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: verbatim omega requires d_omega");
    const int64_t l = k + p;
    const CpqrChoice ch = choose_cpqr(h, l, n, k);
    if ((rc = check_cpqr_fits(h, l, n, ch))) return rc;
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(l), n, m, h->num_sms);
    Carve cv;
    const size_t oofs = omega_mode == IDK_OMEGA_VERBATIM ? 0 : cv.take(sizeof(double) * l * m);
    const size_t yofs = cv.take(sizeof(double) * l * n);
    const size_t pofs = splits > 1 ? cv.take(sizeof(double) * l * n * splits) : 0;
    const CpqrWs w = carve_cpqr(cv, l, n, k, h->num_sms, ch);
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    const double* omega = d_omega;
    mark(h, 0);
    if (omega_mode != IDK_OMEGA_VERBATIM) {
        double* om = reinterpret_cast<double*>(h->ws + oofs);
        if (omega_mode == IDK_OMEGA_PHILOX) {
            IDK_CUDA(idk::omega_philox(om, l, m, seed, h->stream));
            h->launches += 1;
        } else {
            const size_t bytes = sizeof(double) * l * m;
            if (bytes > h->h_omega_cap) {
                cudaStreamSynchronize(h->stream);
                if (h->h_omega) cudaFreeHost(h->h_omega);
                h->h_omega = nullptr;
                h->h_omega_cap = 0;
                IDK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->h_omega), bytes));
                h->h_omega_cap = bytes;
            }
            IDK_CUDA(cudaStreamSynchronize(h->stream));  // staging buffer may still be in flight
            host_generate_gaussian(h->h_omega, l * m, seed);
            IDK_CUDA(cudaMemcpyAsync(om, h->h_omega, bytes, cudaMemcpyHostToDevice, h->stream));
        }
        omega = om;
    }
    mark(h, 1);
    double* Y = reinterpret_cast<double*>(h->ws + yofs);
    if (h->sketch_order == IDK_SKETCH_REFERENCE_ORDER) {  // matrix.cpp:28-48 arithmetic: Y bit-identical to matmul
        IDK_CUDA(idk::matmul_ref_order(omega, l, d_a, lda, l, n, static_cast<int>(m), Y, l, h->stream, trans));
        h->launches += 1;
    } else {
        IDK_CUDA(idk::sketch_gemm(omega, l, d_a, lda, trans, Y, l, static_cast<int>(l), n, m, splits,
                                  splits > 1 ? reinterpret_cast<double*>(h->ws + pofs) : nullptr, h->stream));
        h->launches += splits > 1 ? 2 : 1;
    }
    return factor_and_solve(h, ch, Y, l, n, k, h->ws, w, d_a, lda, m, trans, d_cols, d_z, d_c, false);
}

// sample_without_replacement(population, count, seeded_engine(seed))
// (random.cpp:17-41): partial Fisher-Yates over mt19937_64 with the
// reference's rejection rule for next_below.  O(count) engine draws on the
// host -- the column indices, not the matrix, are what crosses PCIe.
void host_sample_columns(long long* out, int64_t population, int64_t count, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::vector<long long> pool(static_cast<size_t>(population));
    for (int64_t i = 0; i < population; ++i) pool[static_cast<size_t>(i)] = i;
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t bound = static_cast<uint64_t>(population - i);
        const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
        uint64_t x;
        do {
            x = rng();
        } while (x >= limit);
        std::swap(pool[static_cast<size_t>(i)], pool[static_cast<size_t>(i + static_cast<int64_t>(x % bound))]);
    }
    std::memcpy(out, pool.data(), sizeof(long long) * static_cast<size_t>(count));
}

// The reference's own randomized ID, idkit::optim_rid (id.cpp:47-76):
// sample p = min(k + extra, n) columns of M, CPQR(M[:, S], k),
// cols = S[perm[:k]], C = M[:, cols], Z = solve_symmetric_indefinite(
// R_k^T R_k, C^T M) (Bunch-Kaufman LDL^T).  M = A or A^T as in sketch_rid.
int sampled_rid(idk_context* h, const double* d_a, int64_t m, int64_t n, int64_t lda, bool trans, int64_t k,
                int64_t extra, uint64_t seed, int64_t* d_cols, double* d_z, double* d_c) {
    int rc = check_k(h, m, n, k, "optim_rid");
    if (rc) return rc;
    if (extra < 0) return set_err(h, IDK_ERR_INVALID_ARG, "optim_rid: oversampling_fraction must be non-negative");
    if (!d_a || !d_cols || !d_z) return set_err(h, IDK_ERR_INVALID_ARG, "optim_rid: null pointer");
    if (lda < (trans ? n : m)) return set_err(h, IDK_ERR_INVALID_ARG, "optim_rid: lda too small");
    const int64_t p = std::min(k + extra, n);
    const CpqrChoice ch = choose_cpqr(h, m, p, k);
    // Tall samples: pivoted QR of the p x p factor R0 of A_S (shifted
    // CholeskyQR3, tsqr.cu) instead of the m x p sample itself.
    const bool tallq = m >= 8 * p && m >= 512 && p <= 1024;  // measured break-even is near m = 4p
    // the m x p sample itself is factored only without the R0 route (or when
    // that route falls back below): check its fit only then
    const bool sample_fits = check_cpqr_fits(h, m, p, ch) == IDK_OK;
    if (!tallq && !sample_fits) return IDK_ERR_INVALID_ARG;
    const CpqrChoice ch2 = tallq ? choose_cpqr(h, p, p, k) : ch;
    if (tallq && (rc = check_cpqr_fits(h, p, p, ch2))) return rc;
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(k), n, m, h->num_sms);
    const int gsplits = tallq ? idk::sketch_gemm_pick_splits(static_cast<int>(p), p, m, h->num_sms) : 1;
    Carve cv;
    const size_t sofs = cv.take(sizeof(long long) * p);
    const size_t wofs = cv.take(sizeof(double) * m * p);
    const CpqrWs w = carve_cpqr(cv, m, p, k, h->num_sms, ch);
    CpqrWs w2 = w;
    size_t wtofs = 0, gmofs = 0, l1ofs = 0, l2ofs = 0, l3ofs = 0, p1ofs = 0, r0ofs = 0, trofs = 0, stofs = 0, gpofs = 0;
    if (tallq) {
        w2 = carve_cpqr(cv, p, p, k, h->num_sms, ch2);
        wtofs = cv.take(sizeof(double) * m * p);
        gmofs = cv.take(sizeof(double) * p * p);
        l1ofs = cv.take(sizeof(double) * p * p);
        l2ofs = cv.take(sizeof(double) * p * p);
        l3ofs = cv.take(sizeof(double) * p * p);
        p1ofs = cv.take(sizeof(double) * p * p);
        r0ofs = cv.take(sizeof(double) * p * p);
        trofs = cv.take(sizeof(double));
        stofs = cv.take(sizeof(int) * 4);
        gpofs = gsplits > 1 ? cv.take(sizeof(double) * p * p * gsplits) : 0;
    }
    const size_t cofs = d_c ? 0 : cv.take(sizeof(double) * m * k);
    const size_t ctofs = cv.take(sizeof(double) * m * k);
    const size_t rtofs = cv.take(sizeof(double) * k * k);
    const size_t gofs = cv.take(sizeof(double) * k * k);
    const size_t fofs = cv.take(sizeof(double) * k * k);
    const size_t lofs = cv.take(idk::ldlt_scratch_bytes(static_cast<int>(k)));
    const size_t pofs = splits > 1 ? cv.take(sizeof(double) * k * n * splits) : 0;
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    char* base = h->ws;
    long long* sampled = reinterpret_cast<long long*>(base + sofs);
    double* W = reinterpret_cast<double*>(base + wofs);
    double* C = d_c ? d_c : reinterpret_cast<double*>(base + cofs);
    double* Ct = reinterpret_cast<double*>(base + ctofs);
    double* R11t = reinterpret_cast<double*>(base + rtofs);
    double* gram = reinterpret_cast<double*>(base + gofs);
    double* F = reinterpret_cast<double*>(base + fofs);
    const int ki = static_cast<int>(k), pi = static_cast<int>(p);

    const size_t idx_bytes = sizeof(long long) * p;
    if (idx_bytes > h->h_idx_cap) {
        cudaStreamSynchronize(h->stream);
        if (h->h_idx) cudaFreeHost(h->h_idx);
        h->h_idx = nullptr;
        h->h_idx_cap = 0;
        IDK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->h_idx), idx_bytes));
        h->h_idx_cap = idx_bytes;
    }
    IDK_CUDA(cudaStreamSynchronize(h->stream));  // the staging buffer may still be in flight
    host_sample_columns(h->h_idx, n, p, seed);
    mark(h, 0);
    IDK_CUDA(cudaMemcpyAsync(sampled, h->h_idx, idx_bytes, cudaMemcpyHostToDevice, h->stream));
    IDK_CUDA(idk::gather_columns(d_a, lda, m, sampled, static_cast<int>(p), trans, W, h->stream));
    h->launches += 1;
    mark(h, 1);
    // the matrix the pivoted QR runs on: the sample, or its R factor
    double* Wc = W;
    int64_t mc = m;
    CpqrChoice chc = ch;
    CpqrWs wc = w;
    if (tallq) {
        double* Wt = reinterpret_cast<double*>(base + wtofs);
        double* Gm = reinterpret_cast<double*>(base + gmofs);
        double* L1 = reinterpret_cast<double*>(base + l1ofs);
        double* L2 = reinterpret_cast<double*>(base + l2ofs);
        double* L3 = reinterpret_cast<double*>(base + l3ofs);
        double* P1 = reinterpret_cast<double*>(base + p1ofs);
        double* R0 = reinterpret_cast<double*>(base + r0ofs);
        double* tr = reinterpret_cast<double*>(base + trofs);
        int* st = reinterpret_cast<int*>(base + stofs);
        double* gpart = gsplits > 1 ? reinterpret_cast<double*>(base + gpofs) : nullptr;
        IDK_CUDA(cudaMemsetAsync(st, 0x7f, sizeof(int) * 3, h->stream));
        IDK_CUDA(cudaMemsetAsync(st + 3, 0, sizeof(int), h->stream));
        IDK_CUDA(idk::transpose_copy(W, m, m, p, Wt, p, h->stream));
        // G1 = A_S^T A_S (+ shift 11 (mp + p(p+1)) u ||A_S||_F^2), Cholesky, Q1^T = L1^-1 A_S^T
        IDK_CUDA(idk::sketch_gemm(Wt, p, W, m, false, Gm, p, pi, p, m, gsplits, gpart, h->stream));
        IDK_CUDA(idk::gram_trace(Gm, pi, tr, st + 3, h->stream));
        const double shift_factor = 11.0 * (static_cast<double>(m) * p + static_cast<double>(p) * (p + 1)) * 0x1.0p-53;
        IDK_CUDA(idk::cholesky_lower(Gm, pi, tr, shift_factor, L1, st, h->stream));
        IDK_CUDA(idk::trsv_lower_many(L1, pi, m, Wt, h->stream));
        // two plain Cholesky QR steps on Q1
        IDK_CUDA(idk::sketch_gemm(Wt, p, Wt, p, true, Gm, p, pi, p, m, gsplits, gpart, h->stream));
        IDK_CUDA(idk::cholesky_lower(Gm, pi, nullptr, 0.0, L2, st + 1, h->stream));
        IDK_CUDA(idk::trsv_lower_many(L2, pi, m, Wt, h->stream));
        IDK_CUDA(idk::sketch_gemm(Wt, p, Wt, p, true, Gm, p, pi, p, m, gsplits, gpart, h->stream));
        IDK_CUDA(idk::cholesky_lower(Gm, pi, nullptr, 0.0, L3, st + 2, h->stream));
        // R0 = L3^T L2^T L1^T = (L1 L2 L3)^T
        IDK_CUDA(idk::sketch_gemm(L1, p, L2, p, false, P1, p, pi, p, p, 1, nullptr, h->stream));
        IDK_CUDA(idk::sketch_gemm(P1, p, L3, p, false, Gm, p, pi, p, p, 1, nullptr, h->stream));
        IDK_CUDA(idk::transpose_copy(Gm, p, p, p, R0, p, h->stream));
        h->launches += 16 + (gsplits > 1 ? 3 : 0);
        int hst[4];
        IDK_CUDA(cudaMemcpyAsync(hst, st, sizeof(hst), cudaMemcpyDeviceToHost, h->stream));
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        // an exactly zero sampled column (the reference's rank-deficiency case) or a
        // failed Cholesky: keep the reference's own route, the pivoted QR of A_S
        if (hst[0] == 0x7f7f7f7f && hst[1] == 0x7f7f7f7f && hst[2] == 0x7f7f7f7f && hst[3] == 0) {
            Wc = R0;
            mc = p;
            chc = ch2;
            wc = w2;
        } else if (!sample_fits) {
            return set_err(h, IDK_ERR_INVALID_ARG,
                           "optim_rid: the sample needs the m x p pivoted QR, which exceeds the on-chip CPQR budget");
        }
    }
    long long* piv = reinterpret_cast<long long*>(base + wc.pivots);
    int* status = reinterpret_cast<int*>(base + wc.status);
    double* R11 = reinterpret_cast<double*>(base + wc.r11);
    IDK_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int), h->stream));
    mark(h, 2);
    IDK_CUDA(run_cpqr(h, chc, Wc, mc, p, k, base, wc));
    mark(h, 3);
    IDK_CUDA(idk::map_cols(sampled, piv, ki, reinterpret_cast<long long*>(d_cols), h->stream));
    IDK_CUDA(idk::gather_columns(d_a, lda, m, reinterpret_cast<const long long*>(d_cols), ki, trans, C, h->stream));
    // gram = R_k^T R_k, rhs = C^T M (written straight into Z), both on the DMMA pipe
    IDK_CUDA(idk::gather_r11(Wc, mc, piv, ki, R11, h->stream));
    IDK_CUDA(idk::transpose_copy(R11, k, k, k, R11t, k, h->stream));
    IDK_CUDA(idk::sketch_gemm(R11t, k, R11, k, false, gram, k, ki, k, k, 1, nullptr, h->stream));
    IDK_CUDA(idk::transpose_copy(C, m, m, k, Ct, k, h->stream));
    IDK_CUDA(idk::sketch_gemm(Ct, k, d_a, lda, trans, d_z, k, ki, n, m, splits,
                              splits > 1 ? reinterpret_cast<double*>(base + pofs) : nullptr, h->stream));
    IDK_CUDA(idk::ldlt_factor(gram, ki, F, base + lofs, status, h->stream));
    IDK_CUDA(idk::ldlt_solve(F, base + lofs, ki, n, d_z, h->stream));
    mark(h, 4);
    mark(h, 5);
    h->launches += 10 + (splits > 1 ? 1 : 0);
    if (h->async_status) {
        IDK_CUDA(cudaMemcpyAsync(h->async_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        return IDK_OK;
    }
    IDK_CUDA(cudaMemcpyAsync(h->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    collect_stage_times(h);
    const int bad = *h->h_status;
    if (bad != 0x7f7f7f7f)
        return set_err(h, IDK_ERR_SINGULAR,
                       "solve_symmetric_indefinite: zero pivot block at index " + std::to_string(bad));
    return IDK_OK;
}

int id_auto_dev(idk_context* h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t k, int method,
                uint64_t seed, int64_t p, int omega_mode, const double* d_omega, int64_t* d_cols, double* d_z,
                double* d_c, int* transposed) {
    int rc = check_k(h, m, n, k, "id_auto");
    if (rc) return rc;
    if (method < 0 || method > 2) return set_err(h, IDK_ERR_INVALID_ARG, "id_auto: method must be 0, 1 or 2");
    const bool tall = m > n;
    if (transposed) *transposed = tall ? 1 : 0;
    if (method == 2)  // the reference's column-sampling optim_rid, extra = floor(fraction * k) columns
        return tall ? sampled_rid(h, d_a, n, m, lda, true, k, p, seed, d_cols, d_z, d_c)
                    : sampled_rid(h, d_a, m, n, lda, false, k, p, seed, d_cols, d_z, d_c);
    if (!tall) {
        return method == 0 ? det_id(h, d_a, m, n, lda, false, k, d_cols, d_z, d_c)
                           : sketch_rid(h, d_a, m, n, lda, false, k, p, seed, omega_mode, d_omega, d_cols, d_z, d_c);
    }
    // Dual: decompose M = A^T (n x m), stored as A (m x n, lda >= m).
    return method == 0 ? det_id(h, d_a, n, m, lda, true, k, d_cols, d_z, d_c)
                       : sketch_rid(h, d_a, n, m, lda, true, k, p, seed, omega_mode, d_omega, d_cols, d_z, d_c);
}

}  // namespace

extern "C" {

int idk_abi_version(void) { return IDK_ABI_VERSION; }

const char* idk_status_string(int status) {
    switch (status) {
        case IDK_OK: return "ok";
        case IDK_ERR_INVALID_ARG: return "invalid argument";
        case IDK_ERR_SINGULAR: return "singular matrix";
        case IDK_ERR_NOT_POSDEF: return "not positive definite";
        case IDK_ERR_CUDA: return "cuda error";
        case IDK_ERR_NO_MEMORY: return "out of device memory";
        case IDK_ERR_NCCL: return "nccl error";
        default: return "unknown status";
    }
}

int idk_create(idk_handle* out, int device) {
    if (!out) return IDK_ERR_INVALID_ARG;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
        cudaGetLastError();
        return IDK_ERR_CUDA;
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) return IDK_ERR_CUDA;
    if (cudaSetDevice(device) != cudaSuccess) return IDK_ERR_CUDA;
    idk_context* h = new idk_context();
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    h->smem_optin = prop.sharedMemPerBlockOptin;
    if (cudaMallocHost(reinterpret_cast<void**>(&h->h_status), sizeof(int) * 4) != cudaSuccess) {
        delete h;
        return IDK_ERR_CUDA;
    }
    *out = h;
    return IDK_OK;
}

int idk_destroy(idk_handle h) {
    if (!h) return IDK_OK;
    cudaStreamSynchronize(h->stream);
    for (idk_context* kid : h->kids) {
        cudaStream_t ks = kid->stream;
        idk_destroy(kid);
        cudaStreamDestroy(ks);
    }
    for (cudaEvent_t e : h->ev_join) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_chunk) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_gprof) cudaEventDestroy(e);
    if (h->s_sketch) cudaStreamDestroy(h->s_sketch);
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->ws) cudaFree(h->ws);
    if (h->io) cudaFree(h->io);
    if (h->h_status) cudaFreeHost(h->h_status);
    if (h->h_omega) cudaFreeHost(h->h_omega);
    if (h->h_idx) cudaFreeHost(h->h_idx);
    if (h->h_status_many) cudaFreeHost(h->h_status_many);
    for (auto& e : h->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : h->ev_io) cudaEventDestroy(e);
    if (h->s_in) cudaStreamDestroy(h->s_in);
    if (h->s_out) cudaStreamDestroy(h->s_out);
    for (int g = 0; g < idk::kFanMax; ++g)
        if (h->peer_y[g] && h->peer_y[g] != h->ybuf) cudaIpcCloseMemHandle(h->peer_y[g]);
    if (h->ybuf) cudaFree(h->ybuf);
    if (h->d_flag) cudaFree(h->d_flag);
    if (h->nccl_comm && h->nccl_owned) {
        if (const idk::NcclApi* api = idk::nccl_api(nullptr)) api->CommDestroy(h->nccl_comm);
    }
    delete h;
    return IDK_OK;
}

int idk_set_stream(idk_handle h, void* stream) {
    if (!h) return IDK_ERR_INVALID_ARG;
    h->stream = static_cast<cudaStream_t>(stream);
    return IDK_OK;
}

const char* idk_last_error(idk_handle h) { return h ? h->err.c_str() : "null handle"; }

int64_t idk_kernel_launches(idk_handle h) { return h ? h->launches : 0; }

int idk_set_cpqr_mode(idk_handle h, int mode) {
    if (!h || mode < IDK_CPQR_AUTO || mode > IDK_CPQR_CLUSTER_PULL) return IDK_ERR_INVALID_ARG;
    h->cpqr_mode = mode;
    return IDK_OK;
}

int idk_set_sketch_order(idk_handle h, int order) {
    if (!h || (order != IDK_SKETCH_DMMA && order != IDK_SKETCH_REFERENCE_ORDER)) return IDK_ERR_INVALID_ARG;
    h->sketch_order = order;
    return IDK_OK;
}

int idk_set_batched_exact(idk_handle h, int exact) {
    if (!h) return IDK_ERR_INVALID_ARG;
    h->batched_exact = exact != 0;
    return IDK_OK;
}

int idk_cpqr_plan(idk_handle h, int64_t m, int64_t n, int64_t k, int64_t* out8) {
    if (!h || !out8) return IDK_ERR_INVALID_ARG;
    const CpqrChoice c = choose_cpqr(h, m, n, k);
    out8[0] = c.resident ? (c.plan.cluster ? (c.plan.push ? 1 : 4) : 2) : 3;
    out8[1] = c.plan.G;
    out8[2] = c.plan.nc;
    out8[3] = c.plan.S;
    out8[4] = c.plan.R;
    out8[5] = c.plan.l0;
    out8[6] = c.plan.threads;
    out8[7] = static_cast<int64_t>(c.plan.smem);
    return IDK_OK;
}

// Debug: per-step phase clocks of the resident CPQR (CTA 0), k*8 int64 on device.
int idk_debug_cpqr_trace(idk_handle h, int64_t* d_buf) {
    if (!h) return IDK_ERR_INVALID_ARG;
    idk::cpqr_resident_set_trace(reinterpret_cast<long long*>(d_buf));
    return IDK_OK;
}

int idk_set_profiling(idk_handle h, int enable) {
    if (!h) return IDK_ERR_INVALID_ARG;
    if (enable && !h->ev[0]) {
        for (auto& e : h->ev) IDK_CUDA(cudaEventCreate(&e));
    }
    h->profiling = enable != 0;
    return IDK_OK;
}

int idk_stage_times(idk_handle h, double* ms_out, int max_stages) {
    if (!h || !ms_out) return 0;
    const int n = max_stages < 5 ? max_stages : 5;
    for (int i = 0; i < n; ++i) ms_out[i] = h->stage_ms[i];
    return n;
}

int idk_optim_id(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t k, int64_t* d_cols,
                 double* d_z, double* d_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    return det_id(h, d_a, m, n, lda, false, k, d_cols, d_z, d_c);
}

int idk_sketch_rid(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int a_transposed, int64_t k,
                   int64_t p, uint64_t seed, int omega_mode, const double* d_omega, int64_t* d_cols, double* d_z,
                   double* d_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    return sketch_rid(h, d_a, m, n, lda, a_transposed != 0, k, p, seed, omega_mode, d_omega, d_cols, d_z, d_c);
}

int idk_optim_rid(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int a_transposed, int64_t k,
                  double oversampling_fraction, uint64_t seed, int64_t* d_cols, double* d_z, double* d_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (!(oversampling_fraction >= 0.0))
        return set_err(h, IDK_ERR_INVALID_ARG, "optim_rid: oversampling_fraction must be non-negative");
    // p = k + size_t(fraction * k) (id.cpp:54); the clamp to n happens inside
    const double extra = oversampling_fraction * static_cast<double>(k);
    const int64_t e = extra >= 9.0e18 ? INT64_MAX / 2 : static_cast<int64_t>(static_cast<uint64_t>(extra));
    return sampled_rid(h, d_a, m, n, lda, a_transposed != 0, k, e, seed, d_cols, d_z, d_c);
}

int idk_id_auto(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t k, int method,
                uint64_t seed, int64_t p, int omega_mode, const double* d_omega, int64_t* d_cols, double* d_z,
                double* d_c, int* transposed) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    return id_auto_dev(h, d_a, m, n, lda, k, method, seed, p, omega_mode, d_omega, d_cols, d_z, d_c, transposed);
}

int idk_optim_id_batched(idk_handle h, const double* d_a, int64_t batch, int64_t m, int64_t n, int64_t lda,
                         int64_t stride, int64_t k, int64_t* d_cols, double* d_z, double* d_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (batch < 0) return set_err(h, IDK_ERR_INVALID_ARG, "optim_id_batched: negative batch");
    int rc = check_k(h, m, n, k, "optim_id_batched");
    if (rc) return rc;
    if (lda < m || stride < lda * n) return set_err(h, IDK_ERR_INVALID_ARG, "optim_id_batched: bad lda/stride");
    const bool fast = !h->batched_exact && idk::batched_fast_ok(d_a, lda, stride, static_cast<int>(m),
                                                                 static_cast<int>(n), static_cast<int>(k), h->smem_optin);
    if (!fast && idk::batched_id_smem_bytes(static_cast<int>(m), static_cast<int>(n)) > h->smem_optin)
        return set_err(h, IDK_ERR_INVALID_ARG, "optim_id_batched: m x n too large for one CTA's shared memory");
    if (batch == 0) return IDK_OK;
    int* status = h->batched_status;  // device status words supplied by idk_optim_id_batched_host
    if (!status) {
        Carve cv;
        const size_t sofs = cv.take(sizeof(int) * batch);
        if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
        status = reinterpret_cast<int*>(h->ws + sofs);
    }
    // two threads per column (batched_group.cu) by default: 3 % faster than one thread per column
    // on cfg3 (profiles/batched_group_r02.txt); IDK_BATCHED_GROUP=0 selects batched_fast.cu
    static const int group = [] {
        const char* e = getenv("IDK_BATCHED_GROUP");
        return e ? atoi(e) : 2;
    }();
    if (fast && group > 0 && idk::batched_group_ok(d_a, lda, stride, static_cast<int>(m), static_cast<int>(n),
                                                   static_cast<int>(k), h->smem_optin))
        IDK_CUDA(idk::batched_id_group(d_a, lda, stride, batch, static_cast<int>(m), static_cast<int>(n),
                                       static_cast<int>(k), reinterpret_cast<long long*>(d_cols), d_z, d_c, status,
                                       h->num_sms, group, h->stream));
    else if (fast)
        IDK_CUDA(idk::batched_id_fast(d_a, lda, stride, batch, static_cast<int>(m), static_cast<int>(n),
                                      static_cast<int>(k), reinterpret_cast<long long*>(d_cols), d_z, d_c, status,
                                      h->num_sms, h->stream));
    else
        IDK_CUDA(idk::batched_id(d_a, lda, stride, batch, static_cast<int>(m), static_cast<int>(n),
                                 static_cast<int>(k), reinterpret_cast<long long*>(d_cols), d_z, d_c, status,
                                 h->stream));
    h->launches += 1;
    if (h->batched_status) return IDK_OK;  // idk_optim_id_batched_host checks the statuses itself
    std::vector<int> st(static_cast<size_t>(batch));
    IDK_CUDA(cudaMemcpyAsync(st.data(), status, sizeof(int) * batch, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    for (int64_t b = 0; b < batch; ++b)
        if (st[b] >= 0)
            return set_err(h, IDK_ERR_NOT_POSDEF, "optim_id_batched: matrix " + std::to_string(b) +
                                                      " is rank deficient (R11 diagonal " + std::to_string(st[b]) +
                                                      " is zero)");
    return IDK_OK;
}

int idk_optim_id_batched_host(idk_handle h, const double* h_a, int64_t batch, int64_t m, int64_t n, int64_t k,
                              int64_t* h_cols, double* h_z, double* h_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (batch < 0 || (batch > 0 && (!h_a || !h_cols || !h_z)))
        return set_err(h, IDK_ERR_INVALID_ARG, "optim_id_batched_host: bad arguments");
    int rc = check_k(h, m, n, k, "optim_id_batched");
    if (rc) return rc;
    if (batch == 0) return IDK_OK;
    // chunks of 2 x num_sms matrices through 3 buffer sets: chunk c+1 uploads
    // while chunk c factors and chunk c-1 downloads
    const int64_t chunk = std::min<int64_t>(batch, 2LL * h->num_sms);
    const int64_t nchunks = (batch + chunk - 1) / chunk;
    constexpr int S = 3;
    const int64_t mn = m * n;
    Carve cv;
    size_t aofs[S], cofs[S], zofs[S], ccofs[S];
    for (int b = 0; b < S; ++b) {
        aofs[b] = cv.take(sizeof(double) * mn * chunk);
        cofs[b] = cv.take(sizeof(int64_t) * k * chunk);
        zofs[b] = cv.take(sizeof(double) * k * n * chunk);
        ccofs[b] = cv.take(sizeof(double) * m * k * chunk);
    }
    const size_t sofs = cv.take(sizeof(int) * batch);
    if ((rc = ensure(h, &h->io, &h->io_cap, cv.total))) return rc;
    if (!h->s_in) {
        IDK_CUDA(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
        IDK_CUDA(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    }
    while (static_cast<int>(h->ev_io.size()) < 3 * S) {
        cudaEvent_t e;
        IDK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_io.push_back(e);
    }
    cudaEvent_t* ev_in = h->ev_io.data();
    cudaEvent_t* ev_done = ev_in + S;
    cudaEvent_t* ev_out = ev_done + S;
    if (!h->ev_fork) IDK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    IDK_CUDA(cudaEventRecord(h->ev_fork, h->stream));
    IDK_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_fork, 0));
    int* status = reinterpret_cast<int*>(h->io + sofs);
    const bool want_c = h_c != nullptr;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int b = static_cast<int>(c % S);
        const int64_t b0 = c * chunk, cnt = std::min<int64_t>(chunk, batch - b0);
        double* d_a = reinterpret_cast<double*>(h->io + aofs[b]);
        int64_t* d_cols = reinterpret_cast<int64_t*>(h->io + cofs[b]);
        double* d_z = reinterpret_cast<double*>(h->io + zofs[b]);
        double* d_c = want_c ? reinterpret_cast<double*>(h->io + ccofs[b]) : nullptr;
        if (c >= S) IDK_CUDA(cudaStreamWaitEvent(h->s_in, ev_out[b], 0));
        IDK_CUDA(cudaMemcpyAsync(d_a, h_a + b0 * mn, sizeof(double) * mn * cnt, cudaMemcpyHostToDevice, h->s_in));
        IDK_CUDA(cudaEventRecord(ev_in[b], h->s_in));
        IDK_CUDA(cudaStreamWaitEvent(h->stream, ev_in[b], 0));
        h->batched_status = status + b0;
        rc = idk_optim_id_batched(h, d_a, cnt, m, n, m, mn, k, d_cols, d_z, d_c);
        h->batched_status = nullptr;
        if (rc) {
            cudaStreamSynchronize(h->stream);
            cudaStreamSynchronize(h->s_in);
            cudaStreamSynchronize(h->s_out);
            return rc;
        }
        IDK_CUDA(cudaEventRecord(ev_done[b], h->stream));
        IDK_CUDA(cudaStreamWaitEvent(h->s_out, ev_done[b], 0));
        IDK_CUDA(cudaMemcpyAsync(h_cols + b0 * k, d_cols, sizeof(int64_t) * k * cnt, cudaMemcpyDeviceToHost, h->s_out));
        IDK_CUDA(cudaMemcpyAsync(h_z + b0 * k * n, d_z, sizeof(double) * k * n * cnt, cudaMemcpyDeviceToHost, h->s_out));
        if (want_c)
            IDK_CUDA(cudaMemcpyAsync(h_c + b0 * m * k, d_c, sizeof(double) * m * k * cnt, cudaMemcpyDeviceToHost,
                                     h->s_out));
        IDK_CUDA(cudaEventRecord(ev_out[b], h->s_out));
    }
    IDK_CUDA(cudaStreamWaitEvent(h->stream, ev_out[(nchunks - 1) % S], 0));
    std::vector<int> st(static_cast<size_t>(batch));
    IDK_CUDA(cudaMemcpyAsync(st.data(), status, sizeof(int) * batch, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    for (int64_t b = 0; b < batch; ++b)
        if (st[b] >= 0)
            return set_err(h, IDK_ERR_NOT_POSDEF, "optim_id_batched: matrix " + std::to_string(b) +
                                                      " is rank deficient (R11 diagonal " + std::to_string(st[b]) +
                                                      " is zero)");
    return IDK_OK;
}

int idk_sketch_omega(idk_handle h, int64_t l, int64_t m, uint64_t seed, double* d_omega) {
    if (!h) return IDK_ERR_INVALID_ARG;
    if (l < 0 || m < 0 || (!d_omega && l * m > 0)) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_omega: bad args");
    cudaSetDevice(h->device);
    IDK_CUDA(idk::omega_philox(d_omega, l, m, seed, h->stream));
    h->launches += 1;
    return IDK_OK;
}

int idk_sketch(idk_handle h, const double* d_omega, int64_t l, const double* d_a, int64_t m, int64_t n, int64_t lda,
               int a_transposed, double* d_y, int64_t ldy) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (l <= 0 || m <= 0 || n <= 0 || l > INT_MAX) return set_err(h, IDK_ERR_INVALID_ARG, "sketch: bad dimensions");
    if (lda < (a_transposed ? n : m) || ldy < l) return set_err(h, IDK_ERR_INVALID_ARG, "sketch: bad leading dimension");
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(l), n, m, h->num_sms);
    int rc;
    if (splits > 1 && (rc = ensure(h, &h->ws, &h->ws_cap, sizeof(double) * ldy * n * splits))) return rc;
    IDK_CUDA(idk::sketch_gemm(d_omega, l, d_a, lda, a_transposed != 0, d_y, ldy, static_cast<int>(l), n, m, splits,
                              reinterpret_cast<double*>(h->ws), h->stream));
    h->launches += splits > 1 ? 2 : 1;
    return IDK_OK;
}

int idk_qr_column_pivoted(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t steps,
                          double* d_q, double* d_r, int64_t* d_perm) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (m <= 0 || n <= 0 || steps < 1 || steps > std::min(m, n))
        return set_err(h, IDK_ERR_INVALID_ARG, "qr_column_pivoted: max_steps must lie in [1, min(rows, cols)]");
    if (lda < m) return set_err(h, IDK_ERR_INVALID_ARG, "qr_column_pivoted: lda too small");
    const CpqrChoice ch = choose_cpqr(h, m, n, steps);
    int rc = check_cpqr_fits(h, m, n, ch);
    if (rc) return rc;
    Carve cv;
    const size_t wofs = cv.take(sizeof(double) * m * n);
    const size_t permofs = cv.take(sizeof(long long) * n);
    const CpqrWs w = carve_cpqr(cv, m, n, steps, h->num_sms, ch);
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    char* base = h->ws;
    double* W = reinterpret_cast<double*>(base + wofs);
    // both CPQR kernels read A directly (the streaming one writes its working copy during the norm pass)
    long long* pos = reinterpret_cast<long long*>(base + w.pos);
    long long* piv = reinterpret_cast<long long*>(base + w.pivots);
    double* taus = reinterpret_cast<double*>(base + w.taus);
    IDK_CUDA(run_cpqr(h, ch, W, m, n, steps, base, w, m, d_a, lda));
    long long* perm = d_perm ? reinterpret_cast<long long*>(d_perm) : reinterpret_cast<long long*>(base + permofs);
    IDK_CUDA(idk::cpqr_finish(W, m, static_cast<int>(m), n, static_cast<int>(steps), pos, piv, taus, perm, d_r, d_q,
                              h->stream));
    h->launches += 1 + 1 + (d_r ? 1 : 0) + (d_q ? 1 : 0);
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

int idk_qr_column_pivoted_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t steps, double* h_q,
                               double* h_r, int64_t* h_perm) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (!h_a) return set_err(h, IDK_ERR_INVALID_ARG, "qr_column_pivoted: null pointer");
    if (m <= 0 || n <= 0 || steps < 1 || steps > std::min(m, n))
        return set_err(h, IDK_ERR_INVALID_ARG, "qr_column_pivoted: max_steps must lie in [1, min(rows, cols)]");
    Carve cv;
    const size_t aofs = cv.take(sizeof(double) * m * n);
    const size_t qofs = cv.take(sizeof(double) * m * steps);
    const size_t rofs = cv.take(sizeof(double) * steps * n);
    const size_t pofs = cv.take(sizeof(int64_t) * n);
    int rc = ensure(h, &h->io, &h->io_cap, cv.total);
    if (rc) return rc;
    double* d_a = reinterpret_cast<double*>(h->io + aofs);
    double* d_q = h_q ? reinterpret_cast<double*>(h->io + qofs) : nullptr;
    double* d_r = h_r ? reinterpret_cast<double*>(h->io + rofs) : nullptr;
    int64_t* d_perm = reinterpret_cast<int64_t*>(h->io + pofs);
    IDK_CUDA(cudaMemcpyAsync(d_a, h_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, h->stream));
    if ((rc = idk_qr_column_pivoted(h, d_a, m, n, m, steps, d_q, d_r, d_perm))) return rc;
    if (h_q) IDK_CUDA(cudaMemcpyAsync(h_q, d_q, sizeof(double) * m * steps, cudaMemcpyDeviceToHost, h->stream));
    if (h_r) IDK_CUDA(cudaMemcpyAsync(h_r, d_r, sizeof(double) * steps * n, cudaMemcpyDeviceToHost, h->stream));
    if (h_perm) IDK_CUDA(cudaMemcpyAsync(h_perm, d_perm, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

int idk_select_columns(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, const int64_t* d_cols,
                       int64_t ncols, int rows_of_a, double* d_out) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (m < 0 || n < 0 || ncols < 0 || lda < m) return set_err(h, IDK_ERR_INVALID_ARG, "select_columns: bad dimensions");
    if (ncols == 0) return IDK_OK;
    std::vector<int64_t> cols(static_cast<size_t>(ncols));
    IDK_CUDA(cudaMemcpyAsync(cols.data(), d_cols, sizeof(int64_t) * ncols, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    const int64_t limit = rows_of_a ? m : n;
    for (int64_t c : cols)
        if (c < 0 || c >= limit) return set_err(h, IDK_ERR_INVALID_ARG, "select_columns: index out of range");
    IDK_CUDA(idk::gather_columns(d_a, lda, rows_of_a ? n : m, reinterpret_cast<const long long*>(d_cols),
                                 static_cast<int>(ncols), rows_of_a != 0, d_out, h->stream));
    h->launches += 1;
    return IDK_OK;
}

int idk_id_from_sketch(idk_handle h, double* d_y, int64_t l, int64_t n, int64_t ldy, int64_t k, int64_t c_begin,
                       int64_t c_end, int64_t* d_cols, double* d_z_local) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    int rc = check_k(h, l, n, k, "id_from_sketch");
    if (rc) return rc;
    if (!d_y || !d_cols || (c_end > c_begin && !d_z_local) || ldy < l)
        return set_err(h, IDK_ERR_INVALID_ARG, "id_from_sketch: bad pointer or leading dimension");
    if (c_begin < 0 || c_end < c_begin || c_end > n)
        return set_err(h, IDK_ERR_INVALID_ARG, "id_from_sketch: column range outside [0, n]");
    const CpqrChoice ch = choose_cpqr(h, l, n, k);
    if ((rc = check_cpqr_fits(h, l, n, ch))) return rc;
    Carve cv;
    const CpqrWs w = carve_cpqr(cv, l, n, k, h->num_sms, ch);
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    char* base = h->ws;
    long long* pos = reinterpret_cast<long long*>(base + w.pos);
    long long* piv = reinterpret_cast<long long*>(base + w.pivots);
    int* status = reinterpret_cast<int*>(base + w.status);
    IDK_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int), h->stream));
    IDK_CUDA(run_cpqr(h, ch, d_y, l, n, k, base, w, ldy));
    h->launches += 1;
    // R11 + the local column range of Z only (columns are independent).
    IDK_CUDA(idk::id_solve_z(d_y, ldy, static_cast<int>(k), c_begin, c_end - c_begin, piv, pos,
                             reinterpret_cast<double*>(base + w.r11), status, d_z_local, h->stream));
    h->launches += 2;
    IDK_CUDA(cudaMemcpyAsync(d_cols, piv, sizeof(long long) * k, cudaMemcpyDeviceToDevice, h->stream));
    IDK_CUDA(cudaMemcpyAsync(h->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    if (*h->h_status != 0x7f7f7f7f)
        return set_err(h, IDK_ERR_SINGULAR, "solve_triangular: zero diagonal at index " + std::to_string(*h->h_status));
    return IDK_OK;
}

int idk_approx(idk_handle h, const double* d_c, int64_t m, int64_t k, const double* d_z, int64_t n, double* d_out,
               int64_t ldo) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (m <= 0 || n <= 0 || k <= 0 || m > INT_MAX || ldo < m || !d_c || !d_z || !d_out)
        return set_err(h, IDK_ERR_INVALID_ARG, "approx: bad arguments");
    IDK_CUDA(idk::sketch_gemm(d_c, m, d_z, k, false, d_out, ldo, static_cast<int>(m), n, k, 1, nullptr, h->stream));
    h->launches += 1;
    return IDK_OK;
}

int idk_diagnostics(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int transposed,
                    const int64_t* d_cols, int64_t k, const double* d_z, const double* d_c, double* h_out4) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (m <= 0 || n <= 0 || k <= 0 || lda < m || !d_a || !d_cols || !d_z || !h_out4)
        return set_err(h, IDK_ERR_INVALID_ARG, "diagnostics: bad arguments");
    // M: the decomposed matrix (A, or A^T for the dual); C is M's column subset.
    const int64_t mr = transposed ? n : m, mc = transposed ? m : n;
    if (mr > INT_MAX) return set_err(h, IDK_ERR_INVALID_ARG, "diagnostics: dimension too large");
    {  // id.cpp:108-111: an index outside the coefficient matrix is invalid_argument
        std::vector<int64_t> hc(static_cast<size_t>(k));
        IDK_CUDA(cudaMemcpyAsync(hc.data(), d_cols, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->stream));
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        for (int64_t c : hc)
            if (c < 0 || c >= mc)
                return set_err(h, IDK_ERR_INVALID_ARG, "diagnostics: column index outside coefficient matrix");
    }
    Carve cv;
    const size_t cofs = d_c ? 0 : cv.take(sizeof(double) * mr * k);
    const size_t pofs = cv.take(sizeof(double) * idk::resid_partials(static_cast<int>(mr), mc));
    const size_t oofs = cv.take(sizeof(double) * 4);
    int rc;
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    const double* c = d_c;
    if (!c) {
        double* cc = reinterpret_cast<double*>(h->ws + cofs);
        IDK_CUDA(idk::gather_columns(d_a, lda, mr, reinterpret_cast<const long long*>(d_cols), static_cast<int>(k),
                                     transposed != 0, cc, h->stream));
        h->launches += 1;
        c = cc;
    }
    double* out = reinterpret_cast<double*>(h->ws + oofs);
    // ||A - C Z||_F without materialising approx (fused into the DMMA GEMM epilogue);
    // for the dual, C Z is A^T's approximation: compare against A read transposed.
    IDK_CUDA(idk::gemm_residual(c, mr, d_z, k, static_cast<int>(mr), mc, k, d_a, lda, transposed != 0,
                                reinterpret_cast<double*>(h->ws + pofs), out, h->stream));
    IDK_CUDA(idk::z_stats(d_z, static_cast<int>(k), mc, reinterpret_cast<const long long*>(d_cols), out + 2,
                          h->stream));
    h->launches += 3;
    double hv[4];
    IDK_CUDA(cudaMemcpyAsync(hv, out, sizeof(hv), cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    const double dist = std::sqrt(hv[0]), denom = std::sqrt(hv[1]);
    h_out4[0] = denom > 0.0 ? dist / denom : (dist > 0.0 ? INFINITY : 0.0);  // id.cpp:104-106
    h_out4[1] = hv[2];
    h_out4[2] = hv[3];
    h_out4[3] = hv[2] <= 2.0 + 1e-12 ? 1.0 : 0.0;
    return IDK_OK;
}

int idk_id_auto_host_many(idk_handle h, int64_t count, const double* const* h_a, int64_t m, int64_t n, int64_t k,
                          int method, uint64_t seed, int64_t p, int omega_mode, int64_t* const* h_cols,
                          double* const* h_z, double* const* h_c, int* transposed) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (count < 0 || (count > 0 && (!h_a || !h_cols || !h_z)))
        return set_err(h, IDK_ERR_INVALID_ARG, "id_auto_host_many: bad arguments");
    int rc = check_k(h, m, n, k, "id_auto");
    if (rc) return rc;
    if (omega_mode == IDK_OMEGA_VERBATIM)
        return set_err(h, IDK_ERR_INVALID_ARG, "id_auto_host_many: verbatim omega needs the device entry");
    if (count == 0) return IDK_OK;
    const bool tall = m > n;
    const int64_t zc = tall ? m : n, crow = tall ? n : m;
    const bool want_c = h_c != nullptr;
    // Computes run on L lane contexts (one stream each, as idk_id_auto_batch),
    // so IDs whose device time exceeds their transfer time (small matrices:
    // cfg1) overlap on the GPU; uploads stay in order on s_in and downloads on
    // s_out.  S = 2L buffer sets: ID i+L's upload overlaps ID i's compute.
    int L = static_cast<int>(std::min<int64_t>({h->lanes, 8, count}));
    if (const char* e = getenv("IDK_HOST_LANES")) L = std::max(1, std::min(L, atoi(e)));  // tuning only
    const int S = 2 * L;
    if ((rc = ensure_lanes(h, L))) return rc;
    Carve cv;
    std::vector<size_t> aofs(S), cofs(S), zofs(S), ccofs(S);
    for (int b = 0; b < S; ++b) {
        aofs[b] = cv.take(sizeof(double) * m * n);
        cofs[b] = cv.take(sizeof(int64_t) * k);
        zofs[b] = cv.take(sizeof(double) * k * zc);
        ccofs[b] = cv.take(sizeof(double) * crow * k);
    }
    if ((rc = ensure(h, &h->io, &h->io_cap, cv.total))) return rc;
    if (!h->s_in) {
        IDK_CUDA(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
        IDK_CUDA(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
    }
    while (static_cast<int>(h->ev_io.size()) < 3 * S) {
        cudaEvent_t e;
        IDK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_io.push_back(e);
    }
    cudaEvent_t* ev_in = h->ev_io.data();
    cudaEvent_t* ev_done = ev_in + S;
    cudaEvent_t* ev_out = ev_done + S;
    if (count > h->h_status_many_cap) {
        if (h->h_status_many) cudaFreeHost(h->h_status_many);
        h->h_status_many = nullptr;
        h->h_status_many_cap = 0;
        IDK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->h_status_many), sizeof(int) * count));
        h->h_status_many_cap = count;
    }
    // work already queued on the handle's stream precedes every lane and copy
    if (!h->ev_fork) IDK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    IDK_CUDA(cudaEventRecord(h->ev_fork, h->stream));
    IDK_CUDA(cudaStreamWaitEvent(h->s_in, h->ev_fork, 0));
    for (int l = 0; l < L; ++l) {
        idk_context* kid = h->kids[static_cast<size_t>(l)];
        kid->cpqr_mode = h->cpqr_mode;
        kid->batched_exact = h->batched_exact;
        kid->profiling = false;
        IDK_CUDA(cudaStreamWaitEvent(kid->stream, h->ev_fork, 0));
    }
    int64_t launched = 0;
    for (int64_t i = 0; i < count; ++i) {
        const int b = static_cast<int>(i % S);
        idk_context* kid = h->kids[static_cast<size_t>(i % L)];
        double* d_a = reinterpret_cast<double*>(h->io + aofs[b]);
        int64_t* d_cols = reinterpret_cast<int64_t*>(h->io + cofs[b]);
        double* d_z = reinterpret_cast<double*>(h->io + zofs[b]);
        double* d_c = want_c ? reinterpret_cast<double*>(h->io + ccofs[b]) : nullptr;
        if (i >= S) IDK_CUDA(cudaStreamWaitEvent(h->s_in, ev_out[b], 0));  // set b fully drained
        IDK_CUDA(cudaMemcpyAsync(d_a, h_a[i], sizeof(double) * m * n, cudaMemcpyHostToDevice, h->s_in));
        IDK_CUDA(cudaEventRecord(ev_in[b], h->s_in));
        IDK_CUDA(cudaStreamWaitEvent(kid->stream, ev_in[b], 0));
        h->h_status_many[i] = 0x7f7f7f7f;
        kid->async_status = h->h_status_many + i;
        const int64_t before = kid->launches;
        rc = id_auto_dev(kid, d_a, m, n, m, k, method, seed, p, omega_mode, nullptr, d_cols, d_z, d_c, transposed);
        kid->async_status = nullptr;
        launched += kid->launches - before;
        if (rc) {
            rc = set_err(h, rc, kid->err);
            for (int l = 0; l < L; ++l) cudaStreamSynchronize(h->kids[static_cast<size_t>(l)]->stream);
            cudaStreamSynchronize(h->s_in);
            cudaStreamSynchronize(h->s_out);
            h->launches += launched;
            return rc;
        }
        IDK_CUDA(cudaEventRecord(ev_done[b], kid->stream));
        IDK_CUDA(cudaStreamWaitEvent(h->s_out, ev_done[b], 0));
        IDK_CUDA(cudaMemcpyAsync(h_cols[i], d_cols, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->s_out));
        IDK_CUDA(cudaMemcpyAsync(h_z[i], d_z, sizeof(double) * k * zc, cudaMemcpyDeviceToHost, h->s_out));
        if (want_c) IDK_CUDA(cudaMemcpyAsync(h_c[i], d_c, sizeof(double) * crow * k, cudaMemcpyDeviceToHost, h->s_out));
        IDK_CUDA(cudaEventRecord(ev_out[b], h->s_out));
    }
    h->launches += launched;
    // the handle's stream waits for everything (callers time on it)
    IDK_CUDA(cudaEventRecord(ev_out[(count - 1) % S], h->s_out));
    IDK_CUDA(cudaStreamWaitEvent(h->stream, ev_out[(count - 1) % S], 0));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    for (int64_t i = 0; i < count; ++i) {
        const int bad = h->h_status_many[i];
        if (bad != 0x7f7f7f7f) {
            const bool det = method == 0;
            return set_err(h, det ? IDK_ERR_NOT_POSDEF : IDK_ERR_SINGULAR,
                           "id_auto_host_many: matrix " + std::to_string(i) + ": R11 diagonal " +
                               std::to_string(bad) + " is zero");
        }
    }
    return IDK_OK;
}

}  // extern "C"

namespace {

// Lane contexts of the concurrent entries: one non-blocking, highest-priority
// stream and one grow-only workspace each (created on first use, kept).
int ensure_lanes(idk_context* h, int L) {
    while (static_cast<int>(h->kids.size()) < L) {
        idk_context* kid = nullptr;
        int rc = idk_create(&kid, h->device);
        if (rc) return set_err(h, rc, "lane context creation failed");
        cudaStream_t ks;
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        const char* pe = getenv("IDK_LANE_PRIO");
        if (pe && atoi(pe) == 0) hi = 0;
        // lanes run the latency-bound CPQRs: highest priority, so their clusters
        // are dispatched ahead of the (low-priority) grouped sketch CTAs
        if (cudaStreamCreateWithPriority(&ks, cudaStreamNonBlocking, hi) != cudaSuccess) {
            idk_destroy(kid);
            return set_err(h, IDK_ERR_CUDA, "lane stream creation failed");
        }
        kid->stream = ks;
        h->kids.push_back(kid);
        cudaEvent_t e;
        IDK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_join.push_back(e);
    }
    return IDK_OK;
}

// Grouped batch of sketch RIDs (idk_id_auto_batch, method 1, Philox Omega):
// the Omegas and sketches of `chunk` IDs at a time run as ONE Omega launch and
// ONE grouped DMMA GEMM on a low-priority stream (small sketches fill the GPU
// together instead of each running a split-K launch at half the DMMA rate),
// and lane i % L -- a high-priority stream -- factors Y_i (CPQR, Z, C) as soon
// as its chunk's sketch is done, overlapping the next chunk's GEMM.  Results
// are those of idk_id_auto on each ID: the grouped GEMM uses the same tile
// order and fixed split-K order as the single sketch for the same splits.
int batch_grouped(idk_context* h, int L, int64_t count, const double* const* d_a, int64_t m, int64_t n, int64_t lda,
                  int64_t k, const uint64_t* seeds, int64_t p, int64_t* const* d_cols, double* const* d_z,
                  double* const* d_c, int* transposed, int64_t* issued) {
    if (p < 0) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: oversampling p must be non-negative");
    if (lda < m) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: lda too small");
    const bool tall = m > n;
    if (transposed) *transposed = tall ? 1 : 0;
    const int64_t mm = tall ? n : m, nn = tall ? m : n;  // M = A or A^T: mm x nn
    const int64_t l = k + p;
    for (int64_t i = 0; i < count; ++i)
        if (!d_a[i] || !d_cols[i] || !d_z[i]) return set_err(h, IDK_ERR_INVALID_ARG, "sketch_rid: null pointer");
    const CpqrChoice ch = choose_cpqr(h, l, nn, k);
    int rc = check_cpqr_fits(h, l, nn, ch);
    if (rc) return rc;
    int chunk = 4;
    if (const char* e = getenv("IDK_BATCH_CHUNK")) chunk = std::max(1, atoi(e));
    chunk = static_cast<int>(std::min<int64_t>({chunk, count, idk::kGemmGroupMax}));
    // the single sketch's split count, so each Y_i is bit-identical to idk_id_auto's
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(l), nn, mm, h->num_sms);
    const int64_t nchunks = (count + chunk - 1) / chunk;
    Carve cv;
    const size_t oofs = cv.take(sizeof(double) * l * mm * chunk * 2);  // double-buffered by chunk parity
    const size_t yofs = cv.take(sizeof(double) * l * nn * count);
    const size_t pofs = splits > 1 ? cv.take(sizeof(double) * l * nn * splits * chunk * 2) : 0;
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    if (!h->s_sketch) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        IDK_CUDA(cudaStreamCreateWithPriority(&h->s_sketch, cudaStreamNonBlocking, lo));
    }
    while (static_cast<int64_t>(h->ev_chunk.size()) < nchunks) {
        cudaEvent_t e;
        IDK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->ev_chunk.push_back(e);
    }
    if (h->profiling) {
        while (static_cast<int64_t>(h->ev_gprof.size()) < 3 * nchunks) {
            cudaEvent_t e;
            IDK_CUDA(cudaEventCreate(&e));
            h->ev_gprof.push_back(e);
        }
    }
    IDK_CUDA(cudaStreamWaitEvent(h->s_sketch, h->ev_fork, 0));
    double* Ybase = reinterpret_cast<double*>(h->ws + yofs);
    for (int64_t c = 0; c < nchunks; ++c) {
        const int64_t i0 = c * chunk;
        const int cnt = static_cast<int>(std::min<int64_t>(chunk, count - i0));
        double* om = reinterpret_cast<double*>(h->ws + oofs) + (c & 1) * l * mm * chunk;
        double* part = splits > 1 ? reinterpret_cast<double*>(h->ws + pofs) + (c & 1) * l * nn * splits * chunk
                                  : nullptr;
        // Omega / partial buffers are double-buffered: chunk c reuses chunk c-2's, which
        // the stream order already finished (the GEMM of c-2 precedes this launch)
        idk::GroupSeeds sd{};
        idk::GemmGroup g{};
        g.count = cnt;
        g.a_stride = l * mm;
        for (int t = 0; t < cnt; ++t) {
            sd.s[t] = seeds ? seeds[i0 + t] : 0;
            g.b[t] = d_a[i0 + t];
            g.y[t] = Ybase + (i0 + t) * l * nn;
        }
        if (h->profiling) IDK_CUDA(cudaEventRecord(h->ev_gprof[3 * c], h->s_sketch));
        IDK_CUDA(idk::omega_philox_group(om, l, mm, sd, cnt, h->s_sketch));
        if (h->profiling) IDK_CUDA(cudaEventRecord(h->ev_gprof[3 * c + 1], h->s_sketch));
        IDK_CUDA(idk::sketch_gemm_group(om, lda, tall, g, l, static_cast<int>(l), nn, mm, splits, part,
                                        h->s_sketch));
        if (h->profiling) IDK_CUDA(cudaEventRecord(h->ev_gprof[3 * c + 2], h->s_sketch));
        IDK_CUDA(cudaEventRecord(h->ev_chunk[static_cast<size_t>(c)], h->s_sketch));
        h->launches += splits > 1 ? 3 : 2;
        for (int t = 0; t < cnt; ++t) {
            const int64_t i = i0 + t;
            idk_context* kid = h->kids[static_cast<size_t>(i % L)];
            IDK_CUDA(cudaStreamWaitEvent(kid->stream, h->ev_chunk[static_cast<size_t>(c)], 0));
            Carve kc;
            const CpqrWs w = carve_cpqr(kc, l, nn, k, kid->num_sms, ch);
            if ((rc = ensure(kid, &kid->ws, &kid->ws_cap, kc.total)))
                return set_err(h, rc, "id_auto_batch: matrix " + std::to_string(i) + ": " + kid->err);
            h->h_status_many[i] = 0x7f7f7f7f;
            kid->async_status = h->h_status_many + i;
            mark(kid, 0);
            mark(kid, 1);
            rc = factor_and_solve(kid, ch, g.y[t], l, nn, k, kid->ws, w, d_a[i], lda, mm, tall, d_cols[i], d_z[i],
                                  d_c ? d_c[i] : nullptr, false);
            kid->async_status = nullptr;
            if (rc) return set_err(h, rc, "id_auto_batch: matrix " + std::to_string(i) + ": " + kid->err);
            ++*issued;
        }
    }
    return IDK_OK;
}

}  // namespace

extern "C" {

int idk_set_concurrency(idk_handle h, int lanes) {
    if (!h || lanes < 1 || lanes > 64) return IDK_ERR_INVALID_ARG;
    h->lanes = lanes;
    return IDK_OK;
}

int idk_id_auto_batch(idk_handle h, int64_t count, const double* const* d_a, int64_t m, int64_t n, int64_t lda,
                      int64_t k, int method, const uint64_t* seeds, int64_t p, int omega_mode,
                      int64_t* const* d_cols, double* const* d_z, double* const* d_c, int* transposed) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (count < 0 || (count > 0 && (!d_a || !d_cols || !d_z)))
        return set_err(h, IDK_ERR_INVALID_ARG, "id_auto_batch: bad arguments");
    int rc = check_k(h, m, n, k, "id_auto");
    if (rc) return rc;
    if (omega_mode == IDK_OMEGA_VERBATIM)
        return set_err(h, IDK_ERR_INVALID_ARG, "id_auto_batch: verbatim omega needs idk_id_auto");
    if (count == 0) return IDK_OK;
    // child contexts: one non-blocking stream and one workspace per lane
    const int L = static_cast<int>(std::min<int64_t>(h->lanes, count));
    if ((rc = ensure_lanes(h, L))) return rc;
    if (!h->ev_fork) IDK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    if (!h->ev_fork) IDK_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    if (count > h->h_status_many_cap) {
        if (h->h_status_many) cudaFreeHost(h->h_status_many);
        h->h_status_many = nullptr;
        h->h_status_many_cap = 0;
        IDK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h->h_status_many), sizeof(int) * count));
        h->h_status_many_cap = count;
    }
    // inputs written on the caller's stream are visible to every lane
    IDK_CUDA(cudaEventRecord(h->ev_fork, h->stream));
    std::vector<int64_t> before(static_cast<size_t>(L));
    for (int l = 0; l < L; ++l) {
        idk_context* kid = h->kids[static_cast<size_t>(l)];
        kid->cpqr_mode = h->cpqr_mode;
        kid->batched_exact = h->batched_exact;
        if (h->profiling && !kid->ev[0])
            for (auto& e : kid->ev) IDK_CUDA(cudaEventCreate(&e));
        kid->profiling = h->profiling;
        before[static_cast<size_t>(l)] = kid->launches;
        IDK_CUDA(cudaStreamWaitEvent(kid->stream, h->ev_fork, 0));
    }
    int first_rc = IDK_OK;
    int64_t issued = 0;
    const auto t_enqueue0 = std::chrono::steady_clock::now();
    const char* ge = getenv("IDK_BATCH_GROUPED");
    // opt-in (IDK_BATCH_GROUPED=1): measured at cfg2 with 16 IDs it ties the per-lane
    // schedule (5681 vs 5632 IDs/s at chunk 4) -- the CPQR clusters (at most 7
    // co-resident 16-CTA clusters, profiles/probe_clusters_r01.txt) bound both
    const bool grouped = method == 1 && omega_mode == IDK_OMEGA_PHILOX && count >= 2 && ge && atoi(ge) == 1;
    if (grouped) {
        rc = batch_grouped(h, L, count, d_a, m, n, lda, k, seeds, p, d_cols, d_z, d_c, transposed, &issued);
        if (rc) first_rc = rc;
    }
    for (int64_t i = 0; !grouped && i < count && first_rc == IDK_OK; ++i, ++issued) {
        idk_context* kid = h->kids[static_cast<size_t>(i % L)];
        h->h_status_many[i] = 0x7f7f7f7f;
        kid->async_status = h->h_status_many + i;
        int tr = 0;
        rc = id_auto_dev(kid, d_a[i], m, n, lda, k, method, seeds ? seeds[i] : 0, p, omega_mode, nullptr, d_cols[i],
                         d_z[i], d_c ? d_c[i] : nullptr, &tr);
        kid->async_status = nullptr;
        if (transposed) *transposed = tr;
        if (rc) {
            first_rc = set_err(h, rc, "id_auto_batch: matrix " + std::to_string(i) + ": " + kid->err);
        }
    }
    for (int l = 0; l < L; ++l) {
        idk_context* kid = h->kids[static_cast<size_t>(l)];
        if (l == 0 && getenv("IDK_DEBUG_HOST_TIME"))
            fprintf(stderr, "id_auto_batch: host enqueue of %lld IDs took %.1f us\n", static_cast<long long>(issued),
                    std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t_enqueue0).count());
        IDK_CUDA(cudaEventRecord(h->ev_join[static_cast<size_t>(l)], kid->stream));
        IDK_CUDA(cudaStreamWaitEvent(h->stream, h->ev_join[static_cast<size_t>(l)], 0));
        h->launches += kid->launches - before[static_cast<size_t>(l)];
    }
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    if (h->profiling) {  // stage times of each lane's last ID, averaged over the lanes
        for (float& v : h->stage_ms) v = 0.f;
        for (int l = 0; l < L; ++l) {
            idk_context* kid = h->kids[static_cast<size_t>(l)];
            collect_stage_times(kid);
            for (int j = 0; j < 5; ++j) h->stage_ms[j] += kid->stage_ms[j] / static_cast<float>(L);
        }
        if (grouped && issued > 0) {  // Omega / sketch: the grouped launches' device time per ID
            float om = 0.f, gm = 0.f;
            const size_t chunks = h->ev_gprof.size() / 3;
            for (size_t c = 0; c < chunks; ++c) {
                float a = 0.f, b = 0.f;
                if (cudaEventElapsedTime(&a, h->ev_gprof[3 * c], h->ev_gprof[3 * c + 1]) != cudaSuccess) a = 0.f;
                if (cudaEventElapsedTime(&b, h->ev_gprof[3 * c + 1], h->ev_gprof[3 * c + 2]) != cudaSuccess) b = 0.f;
                cudaGetLastError();
                om += a;
                gm += b;
            }
            h->stage_ms[0] = om / static_cast<float>(issued);
            h->stage_ms[1] = gm / static_cast<float>(issued);
        }
    }
    if (first_rc) return first_rc;
    for (int64_t i = 0; i < issued; ++i) {
        const int bad = h->h_status_many[i];
        if (bad != 0x7f7f7f7f) {
            const bool det = method == 0;
            return set_err(h, det ? IDK_ERR_NOT_POSDEF : IDK_ERR_SINGULAR,
                           "id_auto_batch: matrix " + std::to_string(i) + ": zero pivot at index " +
                               std::to_string(bad));
        }
    }
    return IDK_OK;
}

// Host-buffer forms of idk_optim_id / idk_optim_rid (value semantics of
// id.hpp:40,47-48): A uploaded, the ID computed on the handle's stream, cols /
// Z / C downloaded.  `rid` selects the column-sampling estimator.
// Host-buffer ID with the reference's value semantics, IdResult included:
// method 0 optim_id, 1 optim_rid (oversampling fraction), 2 the Gaussian-sketch
// RID (p).  dual = true decomposes M = A^T of the tall host matrix A (m x n)
// with the device reading A transposed -- id_auto's dual (id.cpp:78-95)
// without the host transpose of id.cpp:85 -- and returns approx (m x n) =
// transpose(matmul(C, Z)) as id.cpp:92 does; approx is always formed on the
// device in matmul's exact arithmetic (matrix.cpp:28-48), so it is
// bit-identical to the reference's product of the same C and Z.
static int host_id(idk_handle h, int method, bool dual, const double* h_a, int64_t m, int64_t n, int64_t k,
                   double frac, int64_t p, uint64_t seed, int64_t* h_cols, double* h_z, double* h_c,
                   double* h_approx) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    static const char* names[3] = {"optim_id", "optim_rid", "sketch_rid"};
    if (method < 0 || method > 2) return set_err(h, IDK_ERR_INVALID_ARG, "id: method must be 0, 1 or 2");
    int rc = check_k(h, m, n, k, names[method]);
    if (rc) return rc;
    if (!h_a || !h_cols || !h_z) return set_err(h, IDK_ERR_INVALID_ARG, "optim: null pointer");
    if (method == 1 && !(frac >= 0.0))
        return set_err(h, IDK_ERR_INVALID_ARG, "optim_rid: oversampling_fraction must be non-negative");
    // M (mr x mc) is A, or A^T for the dual
    const int64_t mr = dual ? n : m, mc = dual ? m : n;
    Carve cv;
    const size_t aofs = cv.take(sizeof(double) * m * n);
    const size_t cofs = cv.take(sizeof(int64_t) * k);
    const size_t zofs = cv.take(sizeof(double) * k * mc);
    const size_t ccofs = cv.take(sizeof(double) * mr * k);
    const size_t apofs = h_approx ? cv.take(sizeof(double) * m * n) : 0;
    const size_t tpofs = h_approx && dual ? cv.take(sizeof(double) * m * n) : 0;
    if ((rc = ensure(h, &h->io, &h->io_cap, cv.total))) return rc;
    double* d_a = reinterpret_cast<double*>(h->io + aofs);
    int64_t* d_cols = reinterpret_cast<int64_t*>(h->io + cofs);
    double* d_z = reinterpret_cast<double*>(h->io + zofs);
    double* d_c = (h_c || h_approx) ? reinterpret_cast<double*>(h->io + ccofs) : nullptr;
    IDK_CUDA(cudaMemcpyAsync(d_a, h_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, h->stream));
    if (method == 1) {
        const double extra = frac * static_cast<double>(k);
        const int64_t e = extra >= 9.0e18 ? INT64_MAX / 2 : static_cast<int64_t>(static_cast<uint64_t>(extra));
        rc = sampled_rid(h, d_a, mr, mc, m, dual, k, e, seed, d_cols, d_z, d_c);
    } else if (method == 2) {
        rc = sketch_rid(h, d_a, mr, mc, m, dual, k, p, seed, IDK_OMEGA_PHILOX, nullptr, d_cols, d_z, d_c);
    } else {
        rc = det_id(h, d_a, mr, mc, m, dual, k, d_cols, d_z, d_c);
    }
    if (rc) return rc;
    IDK_CUDA(cudaMemcpyAsync(h_cols, d_cols, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaMemcpyAsync(h_z, d_z, sizeof(double) * k * mc, cudaMemcpyDeviceToHost, h->stream));
    if (h_c) IDK_CUDA(cudaMemcpyAsync(h_c, d_c, sizeof(double) * mr * k, cudaMemcpyDeviceToHost, h->stream));
    if (h_approx) {  // id.cpp:42,73 (and :92 for the dual): approx = matmul(C, Z), exact arithmetic
        double* d_ap = reinterpret_cast<double*>(h->io + apofs);
        double* d_prod = dual ? reinterpret_cast<double*>(h->io + tpofs) : d_ap;
        IDK_CUDA(idk::matmul_ref_order(d_c, mr, d_z, k, mr, mc, static_cast<int>(k), d_prod, mr, h->stream));
        h->launches += 1;
        if (dual) {
            IDK_CUDA(idk::transpose_copy(d_prod, mr, mr, mc, d_ap, m, h->stream));
            h->launches += 1;
        }
        IDK_CUDA(cudaMemcpyAsync(h_approx, d_ap, sizeof(double) * m * n, cudaMemcpyDeviceToHost, h->stream));
    }
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

int idk_optim_id_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int64_t* h_cols, double* h_z,
                      double* h_c, double* h_approx) {
    return host_id(h, 0, false, h_a, m, n, k, 0.0, 0, 0, h_cols, h_z, h_c, h_approx);
}

int idk_optim_rid_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, double oversampling_fraction,
                       uint64_t seed, int64_t* h_cols, double* h_z, double* h_c, double* h_approx) {
    return host_id(h, 1, false, h_a, m, n, k, oversampling_fraction, 0, seed, h_cols, h_z, h_c, h_approx);
}

int idk_id_auto_ref_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int method, uint64_t seed,
                         double oversampling_fraction, int64_t p, int64_t* h_cols, double* h_z, double* h_c,
                         double* h_approx, int* transposed) {
    const bool dual = m > n;  // id.cpp:84
    if (transposed) *transposed = dual ? 1 : 0;
    return host_id(h, method, dual, h_a, m, n, k, oversampling_fraction, p, seed, h_cols, h_z, h_c, h_approx);
}

int idk_matmul_ref(idk_handle h, const double* d_a, int64_t m, int64_t k, int64_t lda, const double* d_b, int64_t n,
                   int64_t ldb, double* d_c, int64_t ldc) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (m < 0 || n < 0 || k < 0 || k > INT_MAX || !d_a || !d_b || !d_c || lda < m || ldb < k || ldc < m)
        return set_err(h, IDK_ERR_INVALID_ARG, "matmul: bad arguments");
    IDK_CUDA(idk::matmul_ref_order(d_a, lda, d_b, ldb, m, n, static_cast<int>(k), d_c, ldc, h->stream));
    h->launches += 1;
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

int idk_id_auto_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int method, uint64_t seed,
                     int64_t p, int omega_mode, int64_t* h_cols, double* h_z, double* h_c, int* transposed) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    int rc = check_k(h, m, n, k, "id_auto");
    if (rc) return rc;
    if (!h_a || !h_cols || !h_z) return set_err(h, IDK_ERR_INVALID_ARG, "id_auto: null pointer");
    if (omega_mode == IDK_OMEGA_VERBATIM)
        return set_err(h, IDK_ERR_INVALID_ARG, "id_auto_host: verbatim omega needs the device entry");
    const bool tall = m > n;
    const int64_t zc = tall ? m : n;
    const int64_t crow = tall ? n : m;
    Carve cv;
    const size_t aofs = cv.take(sizeof(double) * m * n);
    const size_t cofs = cv.take(sizeof(int64_t) * k);
    const size_t zofs = cv.take(sizeof(double) * k * zc);
    const size_t ccofs = cv.take(sizeof(double) * crow * k);
    if ((rc = ensure(h, &h->io, &h->io_cap, cv.total))) return rc;
    double* d_a = reinterpret_cast<double*>(h->io + aofs);
    int64_t* d_cols = reinterpret_cast<int64_t*>(h->io + cofs);
    double* d_z = reinterpret_cast<double*>(h->io + zofs);
    double* d_c = h_c ? reinterpret_cast<double*>(h->io + ccofs) : nullptr;
    IDK_CUDA(cudaMemcpyAsync(d_a, h_a, sizeof(double) * m * n, cudaMemcpyHostToDevice, h->stream));
    rc = id_auto_dev(h, d_a, m, n, m, k, method, seed, p, omega_mode, nullptr, d_cols, d_z, d_c, transposed);
    if (rc) return rc;
    IDK_CUDA(cudaMemcpyAsync(h_cols, d_cols, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaMemcpyAsync(h_z, d_z, sizeof(double) * k * zc, cudaMemcpyDeviceToHost, h->stream));
    if (h_c) IDK_CUDA(cudaMemcpyAsync(h_c, d_c, sizeof(double) * crow * k, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

// ---- multi-GPU: column-sharded ID over NCCL ----------

// A new communicator / transport invalidates the peer mappings of the old one.
static void reset_peers(idk_handle h) {
    cudaStreamSynchronize(h->stream);
    for (int g = 0; g < idk::kFanMax; ++g) {
        if (h->peer_y[g] && h->peer_y[g] != h->ybuf) cudaIpcCloseMemHandle(h->peer_y[g]);
        h->peer_y[g] = nullptr;
    }
    if (h->ybuf) cudaFree(h->ybuf);
    h->ybuf = nullptr;
    h->ybuf_cap = 0;
    h->p2p_state = 0;
    h->has_hc = false;
}

int idk_shard_range(int64_t n, int nranks, int rank, int64_t* begin, int64_t* end) {
    if (n < 0 || nranks < 1 || rank < 0 || rank >= nranks || !begin || !end) return IDK_ERR_INVALID_ARG;
    const int64_t w = (n + nranks - 1) / nranks;
    *begin = std::min<int64_t>(static_cast<int64_t>(rank) * w, n);
    *end = std::min<int64_t>(*begin + w, n);
    return IDK_OK;
}

int idk_nccl_unique_id(void* out128) {
    if (!out128) return IDK_ERR_INVALID_ARG;
    std::string e;
    const idk::NcclApi* api = idk::nccl_api(&e);
    if (!api) return IDK_ERR_NCCL;
    idk::ncclUniqueId id;
    if (api->GetUniqueId(&id) != 0) return IDK_ERR_NCCL;
    std::memcpy(out128, id.internal, sizeof(id.internal));
    return IDK_OK;
}

int idk_comm_init(idk_handle h, int nranks, int rank, const void* id128) {
    if (!h || !id128 || nranks < 1 || rank < 0 || rank >= nranks) return IDK_ERR_INVALID_ARG;
    std::string e;
    const idk::NcclApi* api = idk::nccl_api(&e);
    if (!api) return set_err(h, IDK_ERR_NCCL, "comm_init: " + e);
    cudaSetDevice(h->device);
    reset_peers(h);
    if (h->nccl_comm && h->nccl_owned) api->CommDestroy(h->nccl_comm);
    h->nccl_comm = nullptr;
    idk::ncclUniqueId id;
    std::memcpy(id.internal, id128, sizeof(id.internal));
    idk::ncclComm_t c = nullptr;
    const idk::ncclResult_t r = api->CommInitRank(&c, nranks, id, rank);
    if (r != 0) return set_err(h, IDK_ERR_NCCL, std::string("ncclCommInitRank: ") + api->GetErrorString(r));
    h->nccl_comm = c;
    h->nccl_owned = true;
    h->nranks = nranks;
    h->rank = rank;
    return IDK_OK;
}

int idk_set_nccl_comm(idk_handle h, void* nccl_comm) {
    if (!h) return IDK_ERR_INVALID_ARG;
    std::string e;
    const idk::NcclApi* api = idk::nccl_api(&e);
    if (!api) return set_err(h, IDK_ERR_NCCL, "set_nccl_comm: " + e);
    reset_peers(h);
    if (h->nccl_comm && h->nccl_owned) api->CommDestroy(h->nccl_comm);
    h->nccl_comm = static_cast<idk::ncclComm_t>(nccl_comm);
    h->nccl_owned = false;
    h->nranks = 1;
    h->rank = 0;
    if (h->nccl_comm) {
        int cnt = 0, rk = 0;
        if (api->CommCount(h->nccl_comm, &cnt) != 0 || api->CommUserRank(h->nccl_comm, &rk) != 0)
            return set_err(h, IDK_ERR_NCCL, "set_nccl_comm: communicator query failed");
        h->nranks = cnt;
        h->rank = rk;
    }
    return IDK_OK;
}

int idk_comm_destroy(idk_handle h) {
    if (!h) return IDK_ERR_INVALID_ARG;
    reset_peers(h);
    if (h->nccl_comm && h->nccl_owned) {
        if (const idk::NcclApi* api = idk::nccl_api(nullptr)) api->CommDestroy(h->nccl_comm);
    }
    h->nccl_comm = nullptr;
    h->nccl_owned = false;
    h->nranks = 1;
    h->rank = 0;
    return IDK_OK;
}

int idk_sketch_fanout(idk_handle h, const double* d_omega, int64_t l, const double* d_a, int64_t m, int64_t n,
                      int64_t lda, int a_transposed, double* const* d_dst, int ndst, int64_t ldy, int64_t n_total) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    if (l <= 0 || m <= 0 || n < 0 || l > INT_MAX || n_total < n || ndst < 1 || ndst > idk::kFanMax || !d_dst ||
        ldy < l || lda < (a_transposed ? n : m))
        return set_err(h, IDK_ERR_INVALID_ARG, "sketch_fanout: bad arguments");
    if (n == 0) return IDK_OK;
    idk::FanOut f;
    f.count = ndst;
    for (int g = 0; g < ndst; ++g) f.y[g] = d_dst[g];
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(l), n_total, m, h->num_sms);
    int rc;
    if (splits > 1 && (rc = ensure(h, &h->ws, &h->ws_cap, sizeof(double) * ldy * n * splits))) return rc;
    IDK_CUDA(idk::sketch_gemm_fanout(d_omega, l, d_a, lda, a_transposed != 0, f, ldy, static_cast<int>(l), n, m, splits,
                                     reinterpret_cast<double*>(h->ws), h->stream));
    h->launches += 2;
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    return IDK_OK;
}

// The collectives of idk_id_sharded: NCCL on the handle's stream (stream-ordered),
// or the caller's host collectives (idk_set_host_collectives: the stream is
// synchronised and buffers staged through host memory around each call).
struct Coll {
    idk_context* h;
    const idk::NcclApi* api;  // null: host collectives
    int fail(const char* what, int r) {
        return set_err(h, IDK_ERR_NCCL, std::string(what) + ": " + (api ? api->GetErrorString(r) : "host collective failed"));
    }
    // every rank's `bytes` at d_send, concatenated in rank order into d_recv (device)
    int allgather(const void* d_send, void* d_recv, size_t bytes) {
        if (api) {
            const idk::ncclResult_t r = api->AllGather(d_send, d_recv, bytes, idk::kNcclUint8, h->nccl_comm, h->stream);
            return r ? fail("ncclAllGather", r) : IDK_OK;
        }
        std::vector<char> snd(bytes), rcv(bytes * static_cast<size_t>(h->nranks));
        IDK_CUDA(cudaMemcpyAsync(snd.data(), d_send, bytes, cudaMemcpyDeviceToHost, h->stream));
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        if (h->hc.allgather(h->hc.ctx, snd.data(), rcv.data(), bytes)) return fail("allgather", 0);
        IDK_CUDA(cudaMemcpyAsync(d_recv, rcv.data(), rcv.size(), cudaMemcpyHostToDevice, h->stream));
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        return IDK_OK;
    }
    // every rank sees the minimum of `v` over the ranks (host ints)
    int agree_min(int v, int* out) {
        if (api) {
            IDK_CUDA(cudaMemcpyAsync(h->d_flag, &v, sizeof(int), cudaMemcpyHostToDevice, h->stream));
            const idk::ncclResult_t r =
                api->AllReduce(h->d_flag, h->d_flag, 1, idk::kNcclInt32, idk::kNcclMin, h->nccl_comm, h->stream);
            if (r) return fail("ncclAllReduce", r);
            IDK_CUDA(cudaMemcpyAsync(out, h->d_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
            IDK_CUDA(cudaStreamSynchronize(h->stream));
            return IDK_OK;
        }
        std::vector<int> all(static_cast<size_t>(h->nranks));
        if (h->hc.allgather(h->hc.ctx, &v, all.data(), sizeof(int))) return fail("allgather", 0);
        *out = *std::min_element(all.begin(), all.end());
        return IDK_OK;
    }
    // every rank's work queued so far has finished before any rank's later work starts
    int barrier() {
        if (api) {
            const idk::ncclResult_t r =
                api->AllReduce(h->d_flag, h->d_flag + 1, 1, idk::kNcclInt32, idk::kNcclMin, h->nccl_comm, h->stream);
            return r ? fail("ncclAllReduce (barrier)", r) : IDK_OK;
        }
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        return h->hc.barrier(h->hc.ctx) ? fail("barrier", 0) : IDK_OK;
    }
    // C's columns from their owners (column j from rank owner[j]); d_c is m x k on every rank
    int columns_from_owners(double* d_c, int64_t m, int64_t k, const std::vector<int>& owner) {
        if (api) {
            for (int64_t j0 = 0; j0 < k; j0 += 512) {
                api->GroupStart();
                for (int64_t j = j0; j < std::min<int64_t>(k, j0 + 512); ++j)
                    api->Broadcast(d_c + j * m, d_c + j * m, static_cast<size_t>(m), idk::kNcclFloat64, owner[j],
                                   h->nccl_comm, h->stream);
                const idk::ncclResult_t r = api->GroupEnd();
                if (r) return fail("ncclBroadcast", r);
            }
            return IDK_OK;
        }
        std::vector<double> hc(static_cast<size_t>(m * k));
        IDK_CUDA(cudaMemcpyAsync(hc.data(), d_c, sizeof(double) * m * k, cudaMemcpyDeviceToHost, h->stream));
        IDK_CUDA(cudaStreamSynchronize(h->stream));
        for (int64_t j = 0; j < k; ++j)
            if (h->hc.broadcast(h->hc.ctx, hc.data() + j * m, sizeof(double) * m, owner[j])) return fail("broadcast", 0);
        IDK_CUDA(cudaMemcpyAsync(d_c, hc.data(), sizeof(double) * m * k, cudaMemcpyHostToDevice, h->stream));
        return IDK_OK;
    }
};

// Peer mode setup (collective): (re)allocate this rank's Y buffer, all-gather
// the CUDA IPC handles, open the peers' buffers, and agree (min over ranks)
// that every rank succeeded -- otherwise every rank falls back to the
// all-gather of Y together.
static int peer_setup(idk_handle h, Coll& co, size_t bytes) {
    const int G = h->nranks;
    if (h->p2p_state == -1) return IDK_OK;
    if (h->p2p_state == 1 && bytes <= h->ybuf_cap) return IDK_OK;
    const char* env = getenv("IDK_SHARD_P2P");
    if (G > idk::kFanMax || (env && atoi(env) == 0)) {
        h->p2p_state = -1;
        return IDK_OK;
    }
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    for (int g = 0; g < idk::kFanMax; ++g) {
        if (h->peer_y[g] && h->peer_y[g] != h->ybuf) cudaIpcCloseMemHandle(h->peer_y[g]);
        h->peer_y[g] = nullptr;
    }
    if (h->ybuf) cudaFree(h->ybuf);
    h->ybuf = nullptr;
    h->ybuf_cap = 0;
    int ok = 1;
    cudaIpcMemHandle_t mine;
    std::memset(&mine, 0, sizeof(mine));
    if (cudaMalloc(reinterpret_cast<void**>(&h->ybuf), bytes) != cudaSuccess ||
        cudaIpcGetMemHandle(&mine, h->ybuf) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
    }
    std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(G));
    char* d_h = nullptr;
    IDK_CUDA(cudaMalloc(reinterpret_cast<void**>(&d_h), sizeof(cudaIpcMemHandle_t) * (G + 1)));
    IDK_CUDA(cudaMemcpyAsync(d_h + sizeof(cudaIpcMemHandle_t) * h->rank, &mine, sizeof(mine), cudaMemcpyHostToDevice,
                             h->stream));
    int rc = co.allgather(d_h + sizeof(cudaIpcMemHandle_t) * h->rank, d_h, sizeof(cudaIpcMemHandle_t));
    if (rc) {
        cudaFree(d_h);
        return rc;
    }
    IDK_CUDA(cudaMemcpyAsync(all.data(), d_h, sizeof(cudaIpcMemHandle_t) * G, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    cudaFree(d_h);
    for (int g = 0; g < G && ok; ++g) {
        if (g == h->rank) {
            h->peer_y[g] = h->ybuf;
            continue;
        }
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, all[g], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            cudaGetLastError();
            ok = 0;
        } else {
            h->peer_y[g] = static_cast<double*>(p);
        }
    }
    int all_ok = 0;
    if ((rc = co.agree_min(ok, &all_ok))) return rc;  // every rank must take the same path
    if (!all_ok) {
        for (int g = 0; g < idk::kFanMax; ++g) {
            if (h->peer_y[g] && h->peer_y[g] != h->ybuf) cudaIpcCloseMemHandle(h->peer_y[g]);
            h->peer_y[g] = nullptr;
        }
        if (h->ybuf) cudaFree(h->ybuf);
        h->ybuf = nullptr;
        h->p2p_state = -1;
        return IDK_OK;
    }
    h->ybuf_cap = bytes;
    h->p2p_state = 1;
    return IDK_OK;
}

int idk_shard_peer_mode(idk_handle h) { return h ? h->p2p_state : 0; }

int idk_set_host_collectives(idk_handle h, int nranks, int rank, const idk_host_collectives* c) {
    if (!h || nranks < 1 || rank < 0 || rank >= nranks) return IDK_ERR_INVALID_ARG;
    if (c && (!c->allgather || !c->broadcast || !c->barrier))
        return set_err(h, IDK_ERR_INVALID_ARG, "set_host_collectives: every callback is required");
    reset_peers(h);
    if (h->nccl_comm && h->nccl_owned) {
        if (const idk::NcclApi* api = idk::nccl_api(nullptr)) api->CommDestroy(h->nccl_comm);
    }
    h->nccl_comm = nullptr;
    h->nccl_owned = false;
    h->has_hc = c != nullptr;
    if (c) h->hc = *c;
    h->nranks = c ? nranks : 1;
    h->rank = c ? rank : 0;
    h->p2p_state = 0;
    return IDK_OK;
}

int idk_id_sharded(idk_handle h, const double* d_a_local, int64_t m, int64_t n, int64_t lda, int a_transposed,
                   int64_t k, int64_t p, uint64_t seed, int omega_mode, const double* d_omega, int64_t* d_cols,
                   double* d_z_local, double* d_c) {
    if (!h) return IDK_ERR_INVALID_ARG;
    cudaSetDevice(h->device);
    int rc = check_k(h, m, n, k, "id_sharded");
    if (rc) return rc;
    if (p < 0) return set_err(h, IDK_ERR_INVALID_ARG, "id_sharded: oversampling p must be non-negative");
    if (omega_mode < 0 || omega_mode > 2 || (omega_mode == IDK_OMEGA_VERBATIM && !d_omega))
        return set_err(h, IDK_ERR_INVALID_ARG, "id_sharded: bad omega mode");
    const int G = h->nranks, r = h->rank;
    const idk::NcclApi* api = nullptr;
    if (G > 1 && h->nccl_comm) {
        std::string e;
        if (!(api = idk::nccl_api(&e))) return set_err(h, IDK_ERR_NCCL, "id_sharded: " + e);
    } else if (G > 1 && !h->has_hc) {
        return set_err(h, IDK_ERR_NCCL, "id_sharded: no communicator (idk_comm_init / idk_set_host_collectives)");
    }
    if (G > 1 && !h->d_flag) IDK_CUDA(cudaMalloc(reinterpret_cast<void**>(&h->d_flag), 2 * sizeof(int)));
    Coll co{h, api};
    int64_t b = 0, e_ = 0;
    idk_shard_range(n, G, r, &b, &e_);
    const int64_t w = (n + G - 1) / G, nr = e_ - b;
    const bool trans = a_transposed != 0;
    if (nr > 0 && (!d_a_local || lda < (trans ? nr : m)))
        return set_err(h, IDK_ERR_INVALID_ARG, "id_sharded: bad local block or leading dimension");
    if (!d_cols || (nr > 0 && !d_z_local)) return set_err(h, IDK_ERR_INVALID_ARG, "id_sharded: null output");
    const int64_t l = k + p;
    const CpqrChoice ch = choose_cpqr(h, l, n, k);
    if ((rc = check_cpqr_fits(h, l, n, ch))) return rc;
    // the split-K count of the unsharded sketch: every element of Y is summed in
    // the same order as on one GPU, so the sharded result is bit-identical
    const int splits = idk::sketch_gemm_pick_splits(static_cast<int>(l), n, m, h->num_sms);
    const size_t ybytes = sizeof(double) * l * w * G;  // rank q's block at column q*w
    if (G > 1 && (rc = peer_setup(h, co, ybytes))) return rc;
    const bool p2p = G > 1 && h->p2p_state == 1;
    Carve cv;
    const size_t oofs = omega_mode == IDK_OMEGA_VERBATIM ? 0 : cv.take(sizeof(double) * l * m);
    const size_t yofs = p2p ? 0 : cv.take(ybytes);  // NCCL mode: one in-place all-gather
    const size_t pofs = splits > 1 ? cv.take(sizeof(double) * l * nr * splits) : 0;
    const CpqrWs ws = carve_cpqr(cv, l, n, k, h->num_sms, ch);
    if ((rc = ensure(h, &h->ws, &h->ws_cap, cv.total))) return rc;
    const double* omega = d_omega;
    if (omega_mode != IDK_OMEGA_VERBATIM) {
        double* om = reinterpret_cast<double*>(h->ws + oofs);
        if (omega_mode == IDK_OMEGA_PHILOX) {
            IDK_CUDA(idk::omega_philox(om, l, m, seed, h->stream));
        } else {  // the reference's generate(gaussian) stream on the host (same on every rank)
            std::vector<double> hv(static_cast<size_t>(l * m));
            host_generate_gaussian(hv.data(), l * m, seed);
            IDK_CUDA(cudaMemcpyAsync(om, hv.data(), sizeof(double) * l * m, cudaMemcpyHostToDevice, h->stream));
            IDK_CUDA(cudaStreamSynchronize(h->stream));
        }
        h->launches += omega_mode == IDK_OMEGA_PHILOX ? 1 : 0;
        omega = om;
    }
    double* Y = p2p ? h->ybuf : reinterpret_cast<double*>(h->ws + yofs);
    if (p2p) {
        // the all-gather fused into the sketch: the split-K reduction stores this
        // rank's block into every rank's Y over NVLink, then a stream-ordered
        // barrier (a one-int NCCL all-reduce) tells each rank its Y is complete.  A
        // first barrier keeps this call's stores out of a peer's Y until that
        // peer's previous call (whose CPQR factors its Y in place) is done.
        if ((rc = co.barrier())) return rc;
        if (nr > 0) {
            idk::FanOut f;
            f.count = G;
            f.y[0] = Y + b * l;
            for (int g = 0, t = 1; g < G; ++g)
                if (g != r) f.y[t++] = h->peer_y[g] + b * l;
            IDK_CUDA(idk::sketch_gemm_fanout(omega, l, d_a_local, lda, trans, f, l, static_cast<int>(l), nr, m, splits,
                                             splits > 1 ? reinterpret_cast<double*>(h->ws + pofs) : nullptr,
                                             h->stream));
            h->launches += 2;
        }
        if ((rc = co.barrier())) return rc;
    } else if (nr > 0) {  // this rank's columns of Y = Omega M, straight into its slot of the gathered Y
        IDK_CUDA(idk::sketch_gemm(omega, l, d_a_local, lda, trans, Y + b * l, l, static_cast<int>(l), nr, m, splits,
                                  splits > 1 ? reinterpret_cast<double*>(h->ws + pofs) : nullptr, h->stream));
        h->launches += splits > 1 ? 2 : 1;
    }
    if (G > 1 && !p2p && (rc = co.allgather(Y + static_cast<int64_t>(r) * w * l, Y, sizeof(double) * w * l)))
        return rc;
    // replicated deterministic CPQR: bit-identical on every rank, so no broadcast of the pivots
    long long* pos = reinterpret_cast<long long*>(h->ws + ws.pos);
    long long* piv = reinterpret_cast<long long*>(h->ws + ws.pivots);
    int* status = reinterpret_cast<int*>(h->ws + ws.status);
    IDK_CUDA(cudaMemsetAsync(status, 0x7f, sizeof(int), h->stream));
    IDK_CUDA(run_cpqr(h, ch, Y, l, n, k, h->ws, ws));
    IDK_CUDA(idk::id_solve_z(Y, l, static_cast<int>(k), b, nr, piv, pos, reinterpret_cast<double*>(h->ws + ws.r11),
                             status, d_z_local, h->stream));
    h->launches += nr > 0 ? 3 : 2;
    IDK_CUDA(cudaMemcpyAsync(d_cols, piv, sizeof(long long) * k, cudaMemcpyDeviceToDevice, h->stream));
    std::vector<int64_t> hcols(static_cast<size_t>(k));
    IDK_CUDA(cudaMemcpyAsync(hcols.data(), piv, sizeof(int64_t) * k, cudaMemcpyDeviceToHost, h->stream));
    IDK_CUDA(cudaMemcpyAsync(h->h_status, status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    if (d_c && nr > 0) {  // the selected columns this rank owns
        IDK_CUDA(idk::gather_owned(d_a_local, lda, m, piv, static_cast<int>(k), b, e_, trans, d_c, h->stream));
        h->launches += 1;
    }
    IDK_CUDA(cudaStreamSynchronize(h->stream));
    if (*h->h_status != 0x7f7f7f7f)
        return set_err(h, IDK_ERR_SINGULAR, "solve_triangular: zero diagonal at index " + std::to_string(*h->h_status));
    if (d_c && G > 1) {  // each column of C comes from its one owner: exact, no reduction
        std::vector<int> owner(static_cast<size_t>(k));
        for (int64_t j = 0; j < k; ++j) owner[j] = static_cast<int>(hcols[j] / w);
        if ((rc = co.columns_from_owners(d_c, m, k, owner))) return rc;
        IDK_CUDA(cudaStreamSynchronize(h->stream));
    }
    return IDK_OK;
}

}  // extern "C"
