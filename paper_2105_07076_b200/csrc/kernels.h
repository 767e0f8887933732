// kernels.h -- host-side launchers of the sm_100a kernels (internal to the C-ABI library).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace idk {

// sketch_gemm.cu
constexpr int kGemmGroupMax = 32;
struct GemmGroup {  // grouped sketch members (kernel parameter, by value)
    int count = 0, splits = 1;
    int64_t a_stride = 0, c_stride = 0;
    const double* b[kGemmGroupMax];
    double* y[kGemmGroupMax];
};
constexpr int kFanMax = 8;
struct FanOut {  // destinations of a sharded sketch block (kernel parameter, by value)
    double* y[kFanMax];
    int count = 0;
};
cudaError_t sketch_gemm_fanout(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans, const FanOut& f,
                               int64_t ldc, int M, int64_t N, int64_t K, int splits, double* partial,
                               cudaStream_t stream);
struct GroupSeeds {
    uint64_t s[kGemmGroupMax];
};
cudaError_t sketch_gemm_group(const double* omega, int64_t ldb, bool b_trans, const GemmGroup& grp, int64_t ldc,
                              int M, int64_t N, int64_t K, int splits, double* partial, cudaStream_t stream);
cudaError_t sketch_gemm_tma(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans, double* out,
                            int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K, int splits, int wm,
                            cudaStream_t stream);
cudaError_t omega_philox_group(double* out, int64_t l, int64_t m, const GroupSeeds& seeds, int count,
                               cudaStream_t stream);
int sketch_gemm_pick_wm(int M, int64_t K = (1LL << 40));
int sketch_gemm_pick_splits(int M, int64_t N, int64_t K, int num_sms);
cudaError_t sketch_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans, double* Y,
                        int64_t ldc, int M, int64_t N, int64_t K, int splits, double* partial, cudaStream_t stream);
cudaError_t omega_philox(double* out, int64_t l, int64_t m, uint64_t seed, cudaStream_t stream);
int64_t resid_partials(int M, int64_t N);
cudaError_t gemm_residual(const double* A, int64_t lda, const double* B, int64_t ldb, int M, int64_t N, int64_t K,
                          const double* Ref, int64_t ldr, bool ref_trans, double* part, double* out2,
                          cudaStream_t stream);

// diag.cu
cudaError_t z_stats(const double* Z, int k, int64_t zc, const long long* cols, double* out2, cudaStream_t stream);

// cpqr.cu
constexpr size_t kCpqrPubBytes = 32;
size_t cpqr_smem_bytes(int m, int cols_per_cta);
cudaError_t cpqr_launch(double* W, int64_t ldw, int m, int64_t n, int k, long long* pos_out, long long* pivots,
                        double* taus, void* ws_pub, unsigned* barrier, int num_sms, int max_ctas,
                        cudaStream_t stream, double* xglobal = nullptr, const double* Win = nullptr,
                        int64_t ldin = 0);  // Win: read A in place, the working copy W is written by the norm pass
int64_t cpqr_xglobal_ld(int m);
cudaError_t cpqr_finish(const double* W, int64_t ldw, int m, int64_t n, int k, const long long* pos,
                        const long long* pivots, const double* taus, long long* perm, double* R, double* Q,
                        cudaStream_t stream);

// cpqr_resident.cu
struct ResidentPlan {
    bool ok = false;
    bool cluster = false;
    bool push = false;  // cluster exchange: every CTA holds every candidate column
    int G = 0, nc = 0, S = 0, R = 0, l0 = 0, lds = 0, threads = 0;
    size_t smem = 0;
    double cost = 0;
};
// cluster_pref: 0 = cluster (push, else pull) when it fits, else grid; 1 = grid only; 2 = cluster pull only
ResidentPlan cpqr_resident_plan(int m, int64_t n, int k, int num_sms, int cluster_pref);
void cpqr_resident_set_trace(long long* device_buf);  // debug phase timing (nullptr = off)
size_t cpqr_resident_exchange_bytes(const ResidentPlan& p, int m);
// Win (optional): read the input from here (ld = ldin) instead of W, so W need
// not hold a working copy first; the factor is written to W.
cudaError_t cpqr_resident_launch(const ResidentPlan& p, double* W, int64_t ldw, int m, int64_t n, int k,
                                 long long* pos_out, long long* pivots, double* taus, void* exch, unsigned* barrier,
                                 cudaStream_t stream, const double* Win = nullptr, int64_t ldin = 0);

// trsm.cu
int id_trsm_nb(int k);
size_t id_solve_z_scratch(int k);  // bytes of the R11 buffer id_solve_z needs
size_t id_trsm_smem_bytes(int k);
cudaError_t id_solve_z(const double* W, int64_t ldw, int k, int64_t c_begin, int64_t n, const long long* pivots,
                       const long long* pos, double* R11, int* status, double* Z, cudaStream_t stream);
cudaError_t gather_columns(const double* A, int64_t lda, int64_t rows, const long long* cols, int k, bool rows_of_a,
                           double* C, cudaStream_t stream);
cudaError_t gather_r11(const double* W, int64_t ldw, const long long* pivots, int k, double* R11,
                       cudaStream_t stream);
cudaError_t gather_owned(const double* A, int64_t lda, int64_t rows, const long long* cols, int k, int64_t c_begin,
                         int64_t c_end, bool rows_of_a, double* C, cudaStream_t stream);
cudaError_t copy_pivots(const long long* src, int k, long long* dst, cudaStream_t stream);

// batched.cu
size_t batched_id_smem_bytes(int m, int n);
cudaError_t batched_id(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                       long long* cols, double* Z, double* C, int* status, cudaStream_t stream);

// batched_fast.cu
size_t batched_fast_smem_bytes(int n, int k);
bool batched_fast_ok(const double* A, int64_t lda, int64_t stride, int m, int n, int k, size_t smem_optin);
cudaError_t batched_id_fast(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                            long long* cols, double* Z, double* C, int* status, int num_sms, cudaStream_t stream);

// batched_group.cu (S threads per column; group = 2 or 4)
size_t batched_group_smem_bytes(int n, int k);
bool batched_group_ok(const double* A, int64_t lda, int64_t stride, int m, int n, int k, size_t smem_optin);
cudaError_t batched_id_group(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                             long long* cols, double* Z, double* C, int* status, int num_sms, int group,
                             cudaStream_t stream);

// ldlt.cu (optim_rid's symmetric-indefinite solve)
size_t ldlt_scratch_bytes(int k);
cudaError_t ldlt_factor(const double* S, int k, double* F, void* scratch, int* status, cudaStream_t stream);
cudaError_t ldlt_solve(const double* F, const void* scratch, int k, int64_t n, double* B, cudaStream_t stream);
cudaError_t map_cols(const long long* sampled, const long long* piv, int k, long long* cols, cudaStream_t stream);

// tsqr.cu (shifted CholeskyQR3 R factor of a tall sample, for optim_rid)
cudaError_t cholesky_lower(const double* G, int p, const double* trace, double shift_factor, double* L, int* status,
                           cudaStream_t stream);
cudaError_t trsv_lower_many(const double* L, int p, int64_t n, double* X, cudaStream_t stream);
cudaError_t gram_trace(const double* G, int p, double* out, int* zero_col, cudaStream_t stream);

// util.cu
cudaError_t matmul_ref_order(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t M, int64_t N, int K,
                             double* C, int64_t ldc, cudaStream_t stream, bool b_trans = false);
cudaError_t transpose_copy(const double* A, int64_t lda, int64_t rows, int64_t cols, double* B, int64_t ldb,
                           cudaStream_t stream);

}  // namespace idk
