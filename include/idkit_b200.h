/*
 * idkit_b200.h -- C ABI of the B200-native interpolative-decomposition path.
 *
 * Drop-in boundary for the reference library idkit (/root/reference/proj).
 * The reference's boundary is a C++ API (include/idkit/*.hpp) with value
 * semantics and exceptions; this header is the extern "C" layer beneath a
 * C++ shim that keeps those signatures.  Every entry
 * names the reference interface it replaces.
 *
 * Conventions
 *   - Matrices are column-major fp64 with an explicit leading dimension, the
 *     idkit::Matrix storage contract ((i,j) at data[j*ld+i], matrix.hpp:34-35).
 *   - Indices are int64_t (the reference uses std::size_t).
 *   - `d_` pointers are device memory (cudaMalloc / torch CUDA tensors);
 *     `h_` pointers are host memory (pinned or pageable).
 *   - Every call is stream-ordered on the handle's stream.  Entries that
 *     must report a data-dependent error (singular R11) synchronise that
 *     stream before returning, exactly like the reference returns or throws.
 *   - Status codes map one-to-one to the reference's exception types
 *     (errors.hpp:9-41, std::invalid_argument); the message of the last
 *     failure is kept per handle.  Handles are not shared between threads;
 *     concurrent calls on distinct handles are safe.
 *   - There is no CPU fallback: without a usable sm_100 device every call
 *     returns IDK_ERR_CUDA.
 */
#ifndef IDKIT_B200_H
#define IDKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IDK_ABI_VERSION 1

#if defined(__GNUC__)
#define IDK_API __attribute__((visibility("default")))
#else
#define IDK_API
#endif

typedef struct idk_context* idk_handle;

typedef enum {
    IDK_OK = 0,
    IDK_ERR_INVALID_ARG = 1,  /* std::invalid_argument (id.cpp:14-18, 50-51; qr.cpp:45-46) */
    IDK_ERR_SINGULAR = 2,     /* idkit::SingularMatrixError (solve.cpp:27-30)              */
    IDK_ERR_NOT_POSDEF = 3,   /* idkit::NotPositiveDefiniteError (solve.cpp:66-68)         */
    IDK_ERR_CUDA = 4,         /* CUDA runtime failure / no sm_100 device                   */
    IDK_ERR_NO_MEMORY = 5,    /* device allocation failed                                  */
    IDK_ERR_NCCL = 6          /* NCCL missing or a collective failed (idk_id_sharded)     */
} idk_status;

/* How the Gaussian sketch Omega (l x m) is produced. */
typedef enum {
    IDK_OMEGA_PHILOX = 0,   /* on device: Philox4x32-10(seed, element index) + Box-Muller */
    IDK_OMEGA_MT19937 = 1,  /* on host: the reference's generate(gaussian, l, m, seed)
                               stream (datasets.cpp:15-33, mt19937_64), then uploaded      */
    IDK_OMEGA_VERBATIM = 2  /* caller-provided d_omega (l x m, ld = l)                     */
} idk_omega_mode;

/* Which CPQR kernel factors the pivoted matrix. */
typedef enum {
    IDK_CPQR_AUTO = 0,           /* resident, single cluster when it fits, else resident grid, else streaming */
    IDK_CPQR_RESIDENT_GRID = 1,  /* resident in registers + shared memory, one CTA per SM, grid exchange      */
    IDK_CPQR_STREAMING = 2,      /* trailing matrix streamed through L2 every step (any shape)               */
    IDK_CPQR_CLUSTER_PULL = 3    /* single cluster, winner column pulled over DSMEM (the large-m fallback
                                    of AUTO's cluster push exchange; selectable for testing)                 */
} idk_cpqr_mode;

/* Arithmetic of the sketch Y = Omega M. */
typedef enum {
    IDK_SKETCH_DMMA = 0,            /* default: FP64 tensor cores (DMMA), fixed-order split-K; deterministic */
    IDK_SKETCH_REFERENCE_ORDER = 1  /* the reference matmul's arithmetic (matrix.cpp:28-48: sequential sum,
                                       unfused multiply and add): Y bit-identical to idkit::matmul(Omega, M);
                                       SIMT, an order of magnitude slower -- for bit-compatibility checks   */
} idk_sketch_order;

/* ---- handle ---------------------------------------------------------------- */
IDK_API int idk_abi_version(void);
IDK_API int idk_create(idk_handle* out, int device);
IDK_API int idk_destroy(idk_handle h);
/* cudaStream_t passed as void*; NULL = the legacy default stream. */
IDK_API int idk_set_stream(idk_handle h, void* stream);
IDK_API const char* idk_last_error(idk_handle h);
IDK_API const char* idk_status_string(int status);
/* Number of kernels this handle launched since creation (bench evidence). */
IDK_API int64_t idk_kernel_launches(idk_handle h);
/* Select the CPQR kernel (idk_cpqr_mode); default IDK_CPQR_AUTO. */
IDK_API int idk_set_cpqr_mode(idk_handle h, int mode);
/* Select the sketch arithmetic (idk_sketch_order) of idk_sketch_rid / idk_id_auto; default DMMA. */
IDK_API int idk_set_sketch_order(idk_handle h, int order);
/* Batched entry: 1 = the bit-identical kernel (reference summation order,
 * unfused IEEE ops); 0 (default) = the throughput kernel (registers + TMA
 * prefetch + FMA), which matches within rounding. */
IDK_API int idk_set_batched_exact(idk_handle h, int exact);
/* The CPQR plan for an m x n, k-step factorisation: out8 = {kind (1 cluster push,
 * 2 resident grid, 3 streaming, 4 cluster pull), CTAs, columns per CTA, threads per column,
 * register rows per thread, shared-memory rows, threads per CTA, smem bytes}. */
IDK_API int idk_cpqr_plan(idk_handle h, int64_t m, int64_t n, int64_t k, int64_t* out8);
/* Debug: record %globaltimer at up to 16 phase marks per CPQR step (CTA 0) into d_buf
 * (k*16 int64 per CTA, device); NULL turns it off.  Process-wide. */
IDK_API int idk_debug_cpqr_trace(idk_handle h, int64_t* d_buf);
/* Record CUDA events at stage boundaries on the handle's stream. */
IDK_API int idk_set_profiling(idk_handle h, int enable);
/* Device time (ms) of the last ID call's stages: [0] input prep (Omega or the
 * working copy of A), [1] sketch GEMM, [2] CPQR, [3] R11 gather + TRSM (Z),
 * [4] C gather.  Returns the number of entries written (<= 5). */
IDK_API int idk_stage_times(idk_handle h, double* ms_out, int max_stages);

/* ---- the ID path (device pointers) ----------------------------------------- */

/* Deterministic rank-k ID of A (m x n, lda).  Replaces idkit::optim_id
 * (id.hpp:40, id.cpp:29-45): cols = first k pivots of qr_column_pivoted(A, k);
 * Z = [I | R11^-1 R12] P^T (k x n, ld = k) -- equal to the reference's
 * normal-equation Z in exact arithmetic; C = A[:, cols] (m x k, ld = m) if
 * d_c != NULL.  Rank deficiency (zero |r_ii|) -> IDK_ERR_NOT_POSDEF, as the
 * reference's Cholesky raises (test_id.cpp:120-129). */
IDK_API int idk_optim_id(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t k,
                 int64_t* d_cols, double* d_z, double* d_c);

/* Gaussian-sketch randomized ID (the north-star RID): Y = Omega * M with
 * Omega (k+p) x m, CPQR(Y, k), Z = [I | R11^-1 R12] P^T, C = M[:, cols].
 * M is A (m x n, lda >= m) or, when a_transposed != 0, the transpose of the
 * stored n x m matrix A (lda >= n) -- the id_auto dual (id.cpp:78-95) without
 * materialising A^T.  Then C (m x k) holds rows of the stored matrix.
 * Composed reference: generate -> matmul -> qr_column_pivoted ->
 * solve_triangular -> select_columns.  A zero |r_ii| ->
 * IDK_ERR_SINGULAR (solve.cpp:27-30). */
IDK_API int idk_sketch_rid(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int a_transposed,
                   int64_t k, int64_t p, uint64_t seed, int omega_mode, const double* d_omega,
                   int64_t* d_cols, double* d_z, double* d_c);

/* The reference's randomized ID, idkit::optim_rid (id.hpp:47-50, id.cpp:47-76):
 * sample p = min(k + floor(fraction * k), n) columns of M without replacement
 * (mt19937_64(seed), partial Fisher-Yates, random.cpp:29-41 -- bit-identical
 * to the reference's sample), CPQR of M[:, S] (k steps), cols = S[perm[:k]],
 * C = M[:, cols], Z = (R_k^T R_k)^-1 C^T M by Bunch-Kaufman LDL^T
 * (solve_symmetric_indefinite, solve.cpp:262-274).  M = A or A^T as in
 * idk_sketch_rid.  A singular pivot block -> IDK_ERR_SINGULAR (the
 * reference's SingularMatrixError, test_id.cpp:109-118); fraction < 0 ->
 * IDK_ERR_INVALID_ARG. */
IDK_API int idk_optim_rid(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int a_transposed,
                          int64_t k, double oversampling_fraction, uint64_t seed, int64_t* d_cols, double* d_z,
                          double* d_c);

/* Orientation dispatch, idkit::id_auto (id.hpp:55-56, id.cpp:78-95): A is
 * m x n; if m <= n the ID runs on A, else on A^T with *transposed = 1, cols
 * indexing rows of A and Z being k x m.  method 0 = deterministic
 * (idk_optim_id), 1 = Gaussian-sketch RID (idk_sketch_rid), 2 = the
 * reference's column-sampling RID (idk_optim_rid) with p = floor(fraction * k)
 * extra sampled columns (id.cpp:54).  d_z must hold
 * k * max(m, n) doubles; d_c (optional) m x k or n x k accordingly. */
IDK_API int idk_id_auto(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t k, int method,
                uint64_t seed, int64_t p, int omega_mode, const double* d_omega, int64_t* d_cols,
                double* d_z, double* d_c, int* transposed);

/* Batched deterministic ID (BASELINE cfg3): batch independent m x n
 * matrices at d_a + b*stride (lda each), one CTA per matrix, outputs packed:
 * cols b*k, Z b*k*n, C b*m*k.  Default kernel: persistent CTAs, one thread
 * per column in registers, next matrix prefetched by TMA bulk copies (m <= 64,
 * n <= 256, k <= 32); with idk_set_batched_exact(h, 1) (or other shapes)
 * the kernel that is bit-identical to the reference composition
 * qr_column_pivoted -> solve_triangular -> select_columns per matrix runs
 * (needs m*n in shared memory: 64 x 256 uses 139 KB).  A zero
 * |r_ii| in any matrix -> IDK_ERR_NOT_POSDEF (first failing batch index in
 * the message). */
IDK_API int idk_optim_id_batched(idk_handle h, const double* d_a, int64_t batch, int64_t m, int64_t n, int64_t lda,
                         int64_t stride, int64_t k, int64_t* d_cols, double* d_z, double* d_c);

/* Host-buffer form of idk_optim_id_batched (value semantics of optim_id,
 * id.hpp:40, per matrix): h_a holds batch packed column-major m x n matrices
 * (stride m*n), outputs packed as in the device entry.  Chunks of
 * 2 x num_SMs matrices are uploaded, factored and downloaded in a pipeline
 * (upload of chunk c+1 and download of chunk c-1 overlap the kernel of chunk
 * c); pinned host buffers make the copies asynchronous (with pageable buffers
 * every copy is synchronous and the three stages run one after another). */
IDK_API int idk_optim_id_batched_host(idk_handle h, const double* h_a, int64_t batch, int64_t m, int64_t n, int64_t k,
                                      int64_t* h_cols, double* h_z, double* h_c);

/* Sharded entry: the caller all-gathered the sketch Y
 * (l x n, ldy) of a column-sharded A; factor it (CPQR, identical on every
 * rank: deterministic) and solve Z only for its own columns [c_begin, c_end)
 * into d_z_local (k x (c_end - c_begin), ld = k).  Y is overwritten with the
 * factor.  cols = the k pivots (global column ids).  Collectives stay in the
 * host layer (paper_2105_07076_b200/sharded.py, torch.distributed/NCCL). */
IDK_API int idk_id_from_sketch(idk_handle h, double* d_y, int64_t l, int64_t n, int64_t ldy, int64_t k,
                               int64_t c_begin, int64_t c_end, int64_t* d_cols, double* d_z_local);

/* ---- multi-GPU: one process per GPU, column-sharded --
 * The reference has no distributed layer; its sharded operation is matmul
 * (matrix.cpp:28-48), whose output columns follow the input's.  These entries
 * shard the decomposed matrix M by column blocks over the ranks of an NCCL
 * communicator.  NCCL is bound at run time (the process's libnccl.so.2, e.g.
 * torch's); the library does not link it. */

/* Columns [*begin, *end) of an n-column M owned by `rank` of `nranks`: blocks
 * of w = ceil(n / nranks) columns, rank r owning [min(r w, n), min((r+1) w, n)),
 * so rank r's sketch block sits at column r*w of Y and a single in-place
 * ncclAllGather assembles Y. */
IDK_API int idk_shard_range(int64_t n, int nranks, int rank, int64_t* begin, int64_t* end);
/* NCCL bootstrap: rank 0 calls idk_nccl_unique_id (128 bytes, ncclUniqueId) and
 * distributes it through the caller's own channel; every rank then calls
 * idk_comm_init on its handle (device = the handle's).  idk_set_nccl_comm
 * attaches a caller-owned ncclComm_t instead (never destroyed here). */
IDK_API int idk_nccl_unique_id(void* out128);
IDK_API int idk_comm_init(idk_handle h, int nranks, int rank, const void* id128);
IDK_API int idk_set_nccl_comm(idk_handle h, void* nccl_comm);
IDK_API int idk_comm_destroy(idk_handle h);

/* A caller-supplied transport instead of NCCL (MPI, a test harness, ...):
 * host-memory collectives over the ranks, each returning 0 on success.
 * allgather: every rank's `bytes` from send, concatenated in rank order into
 * recv; broadcast: root's `bytes` of buf to every rank; barrier.  The library
 * synchronises its stream and stages device buffers through host memory
 * around each call.  NULL removes them.  An NCCL communicator, when set,
 * takes precedence. */
typedef struct {
    void* ctx;
    int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes);
    int (*broadcast)(void* ctx, void* buf, uint64_t bytes, int root);
    int (*barrier)(void* ctx);
} idk_host_collectives;
IDK_API int idk_set_host_collectives(idk_handle h, int nranks, int rank, const idk_host_collectives* c);
/* How idk_id_sharded exchanged Y on this handle: 1 = peer mode (fused into the
 * sketch over CUDA IPC mappings), -1 = all-gather (IPC unavailable or
 * IDK_SHARD_P2P=0), 0 = not yet decided (no multi-rank call so far). */
IDK_API int idk_shard_peer_mode(idk_handle h);

/* Sharded Gaussian-sketch RID (the north-star path over nranks GPUs; cfg4 /
 * cfg5).  Every rank passes its block of M's columns [begin, end) from
 * idk_shard_range: d_a_local is m x (end-begin) (lda >= m), or with
 * a_transposed != 0 the same columns of M = A^T as the stored row block of the
 * tall A, (end-begin) x m (lda >= end-begin) -- the id_auto dual (id.cpp:78-95).
 * Per rank: Omega (identical everywhere: Philox keyed by seed, the reference's
 * mt19937 stream, or verbatim) -> local DMMA sketch written into its slot of
 * Y -> one in-place ncclAllGather of Y ((k+p) x n) -> the deterministic CPQR
 * of Y, replicated (bit-identical on every rank, so no pivot broadcast) ->
 * Z for the local columns into d_z_local (k x (end-begin), ld = k) -> the
 * pivot columns this rank owns gathered into d_c and one grouped
 * ncclBroadcast per column from its owner, so C (m x k, ld = m) is complete
 * and bit-exact on every rank (optional).  Peer mode (default when every rank
 * can map the others' memory by CUDA IPC; IDK_SHARD_P2P=0 turns it off): the
 * all-gather is fused into the sketch -- its split-K reduction stores each
 * finished Y element into every rank's Y buffer over NVLink
 * (idk_sketch_fanout), bracketed by two stream-ordered one-int barriers.  d_cols (k) = global column ids of
 * M (row ids of A for the dual).  Results equal idk_sketch_rid's on the
 * unsharded matrix bit for bit (the split-K count is the unsharded one).
 * Without a communicator the call runs as one rank. */
IDK_API int idk_id_sharded(idk_handle h, const double* d_a_local, int64_t m, int64_t n, int64_t lda, int a_transposed,
                           int64_t k, int64_t p, uint64_t seed, int omega_mode, const double* d_omega,
                           int64_t* d_cols, double* d_z_local, double* d_c);

/* The sharded sketch with its all-gather fused in (what idk_id_sharded runs in
 * peer mode, where d_dst are the ranks' Y buffers mapped over NVLink by CUDA
 * IPC): Y_block (l x n) = Omega (l x m, ld = l) * M_block, M_block = A
 * (m x n, lda) or the transpose of the stored n x m block (a_transposed), and
 * the split-K reduction stores every finished element to all ndst (<= 8)
 * destinations d_dst[g] (ld = ldy).  The split-K count is the one of an
 * n_total-column sketch, so the block is bit-identical to the same columns of
 * idk_sketch on the whole matrix.  d_dst is a host array of device pointers. */
IDK_API int idk_sketch_fanout(idk_handle h, const double* d_omega, int64_t l, const double* d_a, int64_t m, int64_t n,
                              int64_t lda, int a_transposed, double* const* d_dst, int ndst, int64_t ldy,
                              int64_t n_total);

/* Concurrent entry for a stream of independent IDs (serving): `count` m x n
 * matrices d_a[i] (device, lda), results into d_cols[i], d_z[i] (k * max(m, n))
 * and, if d_c != NULL, d_c[i].  ID i runs on lane i % L (L = min(count,
 * idk_set_concurrency), default 8), each lane a non-blocking stream with its own
 * workspace, so one ID's CPQR (a 16-SM cluster at cfg2) overlaps other IDs'
 * sketch GEMMs and CPQRs.  Lanes start after the work already queued on the
 * handle's stream; the call returns after all IDs finished.  seeds[i] (host
 * array) or 0 when seeds == NULL.  Statuses are checked at the end; the first
 * failure is reported with its index. */
IDK_API int idk_id_auto_batch(idk_handle h, int64_t count, const double* const* d_a, int64_t m, int64_t n,
                              int64_t lda, int64_t k, int method, const uint64_t* seeds, int64_t p, int omega_mode,
                              int64_t* const* d_cols, double* const* d_z, double* const* d_c, int* transposed);
/* Number of concurrent lanes of idk_id_auto_batch (1..64, default 8). */
IDK_API int idk_set_concurrency(idk_handle h, int lanes);

/* ---- stages / primitives (device pointers) ---------------------------------- */

/* Omega (l x m, ld = l) = Philox Gaussian, keyed by seed (mirrors idko_omega_philox). */
IDK_API int idk_sketch_omega(idk_handle h, int64_t l, int64_t m, uint64_t seed, double* d_omega);

/* Y (l x n, ldy) = Omega (l x m, ld = l) * M, M = A or A^T as in idk_sketch_rid.
 * Replaces matmul(Omega, A) (matrix.cpp:28-48) on the DMMA pipe. */
IDK_API int idk_sketch(idk_handle h, const double* d_omega, int64_t l, const double* d_a, int64_t m, int64_t n,
               int64_t lda, int a_transposed, double* d_y, int64_t ldy);

/* idkit::qr_column_pivoted (qr.hpp:34, qr.cpp:42-126): q (m x steps, may be
 * NULL), r (steps x n, may be NULL), perm (n, may be NULL). */
IDK_API int idk_qr_column_pivoted(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int64_t steps,
                          double* d_q, double* d_r, int64_t* d_perm);

/* Host-buffer form of idk_qr_column_pivoted (qr.hpp:34): h_a m x n (ld = m);
 * h_q m x steps, h_r steps x n, h_perm n (each may be NULL). */
IDK_API int idk_qr_column_pivoted_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t steps,
                                       double* h_q, double* h_r, int64_t* h_perm);

/* idkit::select_columns (matrix.hpp:76, matrix.cpp:121-130): out (m x ncols)
 * = A[:, cols]; rows_of_a != 0 gathers rows instead (out is n x ncols). */
IDK_API int idk_select_columns(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, const int64_t* d_cols,
                       int64_t ncols, int rows_of_a, double* d_out);

/* IdResult::approx (id.hpp:17-22, id.cpp:42,73): out (m x n, ldo) = C (m x k,
 * ld = m) * Z (k x n, ld = k) on the DMMA pipe. */
IDK_API int idk_approx(idk_handle h, const double* d_c, int64_t m, int64_t k, const double* d_z, int64_t n,
                       double* d_out, int64_t ldo);

/* idkit::diagnostics (id.hpp:60, id.cpp:97-122) of a device result for the
 * stored m x n matrix A: h_out4 = {relative_error, max_abs_z,
 * identity_deviation, entry_bound_satisfied (0/1)}.  ||A - approx||_F is
 * computed inside the C*Z GEMM epilogue, so approx is never materialised.
 * transposed != 0: the dual result of id_auto (cols index rows, Z is k x m).
 * d_c may be NULL (gathered here). */
IDK_API int idk_diagnostics(idk_handle h, const double* d_a, int64_t m, int64_t n, int64_t lda, int transposed,
                            const int64_t* d_cols, int64_t k, const double* d_z, const double* d_c, double* h_out4);

/* ---- host-buffer entries (the reference's value-semantics calls) ------------ */

/* Same as idk_id_auto, host pointers in and out; host<->device copies are
 * part of the call.  h_a is m x n (ld = m); h_z holds k * max(m, n). */
IDK_API int idk_id_auto_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int method, uint64_t seed,
                     int64_t p, int omega_mode, int64_t* h_cols, double* h_z, double* h_c, int* transposed);

/* optim_id / optim_rid with host buffers (the reference's value semantics,
 * id.hpp:40 and :47-48): h_a is m x n (ld = m); h_z is k x n; h_c (optional)
 * m x k; h_approx (optional) m x n = IdResult::approx (id.cpp:42,73) computed
 * on the device by idk_matmul_ref, i.e. bit-identical to the reference's
 * matmul(select_columns(a, cols), z).  No orientation dispatch -- that is
 * idk_id_auto_host. */
IDK_API int idk_optim_id_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int64_t* h_cols,
                              double* h_z, double* h_c, double* h_approx);
IDK_API int idk_optim_rid_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k,
                               double oversampling_fraction, uint64_t seed, int64_t* h_cols, double* h_z,
                               double* h_c, double* h_approx);
/* idkit::id_auto with the reference's full value semantics (id.hpp:55-56,
 * id.cpp:78-95), IdResult::approx included: method 0 = optim_id, 1 = the
 * reference's randomized ID optim_rid (oversampling_fraction), 2 = the
 * Gaussian-sketch RID (oversampling p, Philox Omega keyed by seed).  h_a is
 * m x n (ld = m).  When m > n the ID runs on A^T with the device reading A
 * transposed (no host transpose, unlike id.cpp:85): *transposed = 1, cols
 * index rows of A, h_z is k x m, h_c (optional) n x k, and h_approx (optional,
 * m x n) = transpose(matmul(C, Z)) as id.cpp:92 forms it.  approx is computed
 * on the device in matmul's exact arithmetic (bit-identical to the
 * reference's matmul of the same C and Z). */
IDK_API int idk_id_auto_ref_host(idk_handle h, const double* h_a, int64_t m, int64_t n, int64_t k, int method,
                                 uint64_t seed, double oversampling_fraction, int64_t p, int64_t* h_cols, double* h_z,
                                 double* h_c, double* h_approx, int* transposed);

/* idkit::matmul (matrix.hpp:56, matrix.cpp:28-48) in the reference's exact
 * arithmetic (same summation order, zero skipping, unfused IEEE ops):
 * C (m x n, ldc) = A (m x k, lda) * B (k x n, ldb), bit-identical to the CPU
 * reference.  Device pointers. */
IDK_API int idk_matmul_ref(idk_handle h, const double* d_a, int64_t m, int64_t k, int64_t lda, const double* d_b,
                           int64_t n, int64_t ldb, double* d_c, int64_t ldc);

/* Pipelined host entry: `count` independent IDs of m x n matrices h_a[i]
 * (host, ld = m), results into h_cols[i], h_z[i] (k * max(m, n)) and, if
 * h_c != NULL, h_c[i].  The upload of matrix i+1 and the download of result
 * i-1 overlap the compute of ID i on separate streams (pinned host buffers
 * make the copies asynchronous; pageable ones serialise the pipeline); statuses are checked once at the end, the
 * first failure is reported with its index. */
IDK_API int idk_id_auto_host_many(idk_handle h, int64_t count, const double* const* h_a, int64_t m, int64_t n,
                                  int64_t k, int method, uint64_t seed, int64_t p, int omega_mode,
                                  int64_t* const* h_cols, double* const* h_z, double* const* h_c, int* transposed);

#ifdef __cplusplus
}
#endif
#endif
