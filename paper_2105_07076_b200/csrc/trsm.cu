// trsm.cu -- coefficient solve Z = [I | R11^-1 R12] P^T and the column gather.
//
// Reference: the north-star Z replaces optim_id's normal-equation solve
// (id.cpp:37-41) by the interpolation form built from the reference's own
// solve_triangular (solve.cpp:23-53, upper, back substitution) on
// R11 = leading_block(R, k) (id.cpp:20-25) and R12 = R[:, k:].  The scatter
// by perm needs no permutation pass: column c of Z depends only on column c
// of the factored matrix W, so each CTA solves a block of *physical* columns
// and writes e_pos(c) for the k pivot columns.
//
// The singular-diagonal floor |r_ii| <= 1e-300 (solve.cpp:19,27-30) is
// checked while R11 is gathered; the host maps it to SingularMatrixError
// (sketch) or NotPositiveDefiniteError (deterministic, solve.cpp:66-68).
#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kTrsmNB = 32;      // right-hand sides per CTA
constexpr int kTrsmThreads = 256;

__global__ void gather_r11_kernel(const double* __restrict__ W, int64_t ldw, const long long* __restrict__ pivots,
                                  int k, double* __restrict__ R11, int* __restrict__ status) {
    const int64_t total = static_cast<int64_t>(k) * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(e / k), i = static_cast<int>(e % k);
        const double v = (i <= j) ? W[pivots[j] * ldw + i] : 0.0;
        R11[e] = v;
        if (status && i == j && fabs(v) <= 1e-300) atomicMin(status, j);
    }
}

// X (k x nb tile of W's top k rows) <- R11^-1 X, blocked back substitution:
// 32-row diagonal blocks are solved warp-synchronously (lane = row, one warp
// per right-hand side), the rows above are updated by all threads.
__global__ void __launch_bounds__(kTrsmThreads)
id_trsm_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
               const long long* __restrict__ pos, double* __restrict__ Z, int NB) {
    extern __shared__ double X[];
    const int ldx = k | 1;  // odd stride: lane-per-column accesses are bank-conflict free
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NB;
    const int nb = static_cast<int>(min(static_cast<long long>(NB), static_cast<long long>(n - c0)));

    for (int e = tid; e < nb * k; e += blockDim.x) {
        const int c = e / k, i = e - c * k;
        X[c * ldx + i] = W[(c0 + c) * ldw + i];
    }
    __syncthreads();

    for (int hi = k; hi > 0;) {
        const int lo = hi > 32 ? hi - 32 : 0;
        const int bs = hi - lo;
        for (int c = warp; c < nb; c += nwarps) {
            double x = lane < bs ? X[c * ldx + lo + lane] : 0.0;
            for (int i = bs - 1; i >= 0; --i) {
                double xi = __shfl_sync(0xffffffffu, x, i);
                xi = xi / R11[static_cast<int64_t>(lo + i) * k + lo + i];
                if (lane == i) x = xi;
                if (lane < i) x = sub_rn(x, mul_rn(R11[static_cast<int64_t>(lo + i) * k + lo + lane], xi));
            }
            if (lane < bs) X[c * ldx + lo + lane] = x;
        }
        __syncthreads();
        for (int e = tid; e < lo * nb; e += blockDim.x) {
            const int c = e / lo, r = e - c * lo;
            const double* xc = X + c * ldx;
            double acc = 0.0;
            for (int l = lo; l < hi; ++l) acc += R11[static_cast<int64_t>(l) * k + r] * xc[l];
            X[c * ldx + r] = xc[r] - acc;
        }
        __syncthreads();
        hi = lo;
    }

    for (int e = tid; e < nb * k; e += blockDim.x) {
        const int c = e / k, i = e - c * k;
        const int64_t col = c0 + c;
        const long long p = pos[col];
        Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : X[c * ldx + i];
    }
}

// Blocked back substitution on the DMMA pipe (solve.cpp:43-51 restated for
// many right-hand sides): a CTA takes kDmmaNB columns of W's top k rows into
// shared memory with R11 (k padded to 32*NBLK with an identity block), then
// bottom-up per 32-row block b:
//   X_b   <- R_bb^-1 X_b       substitution, one thread per right-hand side
//                              (reciprocal diagonal, R_bb read by broadcast)
//   X_top <- X_top - R_{top,b} X_b   m8n8k4 DMMA tiles over the rows above
// The update carries the (k^2/2)(n) flops of the solve on the tensor pipe; the
// diagonal solves are 32 dependent steps per block.
constexpr int kDmmaNB = 64;       // right-hand sides per CTA
constexpr int kDmmaThreads = 128;

__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(smem))),
                 "l"(gmem)
                 : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

// PAIRS: k and ldw even and 16-byte aligned bases -- operands move as 16-byte
// pairs (cp.async.cg 16) and Z leaves as double2 stores: half the load/store
// instructions, which at k <= 128 are half of the kernel's (ncu, cfg5).
template <int NBLK, bool PAIRS>
__global__ void __launch_bounds__(kDmmaThreads)
id_trsm_dmma_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
                    const long long* __restrict__ pos, double* __restrict__ Z) {
    constexpr int KP = 32 * NBLK;
    constexpr int LD = KP + 4;  // = 4 (mod 16) doubles: fragment loads are bank-conflict free
    extern __shared__ __align__(16) double smem[];
    double* Rs = smem;                    // KP x KP, column-major, stride LD
    double* Xs = Rs + KP * LD;            // kDmmaNB right-hand sides, stride LD
    double* rinv = Xs + kDmmaNB * LD;     // KP
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kDmmaNB;
    const int nb = static_cast<int>(min(static_cast<long long>(kDmmaNB), static_cast<long long>(n - c0)));

    // operands land by cp.async (all loads in flight at once); padding is written directly
    if constexpr (PAIRS) {
        constexpr int KH = KP / 2;  // row pairs per column
        for (int e = tid; e < KP * KH; e += kDmmaThreads) {
            const int col = e / KH, row = 2 * (e - col * KH);
            double* dst = Rs + col * LD + row;
            if (row < k && col < k) {
                cp_async_16(dst, R11 + static_cast<int64_t>(col) * k + row);
            } else {
                dst[0] = row == col ? 1.0 : 0.0;
                dst[1] = row + 1 == col ? 1.0 : 0.0;
            }
        }
        for (int e = tid; e < kDmmaNB * KH; e += kDmmaThreads) {
            const int c = e / KH, row = 2 * (e - c * KH);
            double* dst = Xs + c * LD + row;
            if (c < nb && row < k) {
                cp_async_16(dst, W + (c0 + c) * ldw + row);
            } else {
                dst[0] = 0.0;
                dst[1] = 0.0;
            }
        }
    } else {
        for (int e = tid; e < KP * KP; e += kDmmaThreads) {
            const int col = e / KP, row = e - col * KP;
            double* dst = Rs + col * LD + row;
            if (row < k && col < k) cp_async_8(dst, R11 + static_cast<int64_t>(col) * k + row);
            else *dst = row == col ? 1.0 : 0.0;
        }
        for (int e = tid; e < kDmmaNB * KP; e += kDmmaThreads) {
            const int c = e / KP, row = e - c * KP;
            double* dst = Xs + c * LD + row;
            if (c < nb && row < k) cp_async_8(dst, W + (c0 + c) * ldw + row);
            else *dst = 0.0;
        }
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    for (int row = tid; row < KP; row += kDmmaThreads) rinv[row] = 1.0 / Rs[row * LD + row];
    __syncthreads();

#pragma unroll 1
    for (int b = NBLK - 1; b >= 0; --b) {
        const int r0 = 32 * b;
        if (tid < kDmmaNB) {  // X_b <- R_bb^-1 X_b for right-hand side tid
            double x[32];
            double* xc = Xs + tid * LD + r0;
#pragma unroll
            for (int r = 0; r < 32; ++r) x[r] = xc[r];
            const double* rb = Rs + r0 * LD + r0;
#pragma unroll
            for (int i = 31; i >= 0; --i) {
                x[i] *= rinv[r0 + i];
#pragma unroll
                for (int l = 0; l < i; ++l) x[l] = fma(-rb[i * LD + l], x[i], x[l]);
            }
#pragma unroll
            for (int r = 0; r < 32; ++r) xc[r] = x[r];
        }
        __syncthreads();
        // rows [0, r0): a warp takes one 8-row tile across all 8 column tiles
        // (8 independent accumulators share each A fragment), k-depth 32
        for (int rt = warp; rt < 4 * b; rt += kDmmaThreads / 32) {
            const int row = rt * 8 + fr;
            double acc[kDmmaNB / 8][2];
#pragma unroll
            for (int ct = 0; ct < kDmmaNB / 8; ++ct) {
                acc[ct][0] = Xs[(ct * 8 + 2 * fc) * LD + row];
                acc[ct][1] = Xs[(ct * 8 + 2 * fc + 1) * LD + row];
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = r0 + ks * 4 + fc;
                const double a = -Rs[kk * LD + row];
#pragma unroll
                for (int ct = 0; ct < kDmmaNB / 8; ++ct) dmma_8x8x4(acc[ct], a, Xs[(ct * 8 + fr) * LD + kk]);
            }
#pragma unroll
            for (int ct = 0; ct < kDmmaNB / 8; ++ct) {
                Xs[(ct * 8 + 2 * fc) * LD + row] = acc[ct][0];
                Xs[(ct * 8 + 2 * fc + 1) * LD + row] = acc[ct][1];
            }
        }
        __syncthreads();
    }

    // Z columns: the warp's positions are loaded up front (one round trip), then
    // coalesced stores along each column
    constexpr int kPer = kDmmaNB / (kDmmaThreads / 32);  // columns per warp (16)
    const long long mp = (lane < kPer && warp + (kDmmaThreads / 32) * lane < nb)
                             ? pos[c0 + warp + (kDmmaThreads / 32) * lane] : 0;
#pragma unroll 4
    for (int t = 0; t < kPer; ++t) {
        const int c = warp + (kDmmaThreads / 32) * t;
        const long long p = __shfl_sync(0xffffffffu, mp, t);
        if (c < nb) {
            const int64_t col = c0 + c;
            if constexpr (PAIRS) {
                double2* zc = reinterpret_cast<double2*>(Z + col * k);
                const double2* xc = reinterpret_cast<const double2*>(Xs + c * LD);
                for (int i2 = lane; i2 < k / 2; i2 += 32)
                    zc[i2] = p < k ? make_double2(2 * i2 == p ? 1.0 : 0.0, 2 * i2 + 1 == p ? 1.0 : 0.0) : xc[i2];
            } else {
                for (int i = lane; i < k; i += 32) Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : Xs[c * LD + i];
            }
        }
    }
}

// k in (128, 256]: R11 (up to 512 KB) stays in global memory (L2-resident):
// the DMMA A fragments are read from it directly (all 8 k-steps of a row
// tile issued before the first DMMA) and each 32x32 diagonal block is staged
// in shared memory for its substitution.  X (64 right-hand sides) and the
// reciprocal diagonal live in shared memory.
template <int NBLK, int NB, int THR>
__global__ void __launch_bounds__(THR)
id_trsm_dmma_big_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
                        const long long* __restrict__ pos, double* __restrict__ Z) {
    constexpr int KP = 32 * NBLK;
    constexpr int LD = KP + 4;
    constexpr int LDB = 32 + 1;  // diagonal block, column-major
    extern __shared__ __align__(16) double smem[];
    double* Xs = smem;                     // NB right-hand sides, stride LD
    double* Db = Xs + NB * LD;        // 32 x 32 diagonal block
    double* rinv = Db + 32 * LDB;          // KP
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NB;
    const int nb = static_cast<int>(min(static_cast<long long>(NB), static_cast<long long>(n - c0)));
    // R[row, col] with the identity padding beyond k
    auto rget = [&](int row, int col) -> double {
        return (row < k && col < k) ? __ldg(R11 + static_cast<int64_t>(col) * k + row) : (row == col ? 1.0 : 0.0);
    };

    for (int e = tid; e < NB * KP; e += THR) {
        const int c = e / KP, row = e - c * KP;
        double* dst = Xs + c * LD + row;
        if (c < nb && row < k) cp_async_8(dst, W + (c0 + c) * ldw + row);
        else *dst = 0.0;
    }
    for (int row = tid; row < KP; row += THR) rinv[row] = 1.0 / rget(row, row);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();

#pragma unroll 1
    for (int b = NBLK - 1; b >= 0; --b) {
        const int r0 = 32 * b;
        for (int e = tid; e < 32 * 32; e += THR) {
            const int col = e >> 5, row = e & 31;
            Db[col * LDB + row] = rget(r0 + row, r0 + col);
        }
        __syncthreads();
        if (tid < NB) {
            double x[32];
            double* xc = Xs + tid * LD + r0;
#pragma unroll
            for (int r = 0; r < 32; ++r) x[r] = xc[r];
#pragma unroll
            for (int i = 31; i >= 0; --i) {
                x[i] *= rinv[r0 + i];
#pragma unroll
                for (int l = 0; l < i; ++l) x[l] = fma(-Db[i * LDB + l], x[i], x[l]);
            }
#pragma unroll
            for (int r = 0; r < 32; ++r) xc[r] = x[r];
        }
        __syncthreads();
        for (int rt = warp; rt < 4 * b; rt += THR / 32) {
            const int row = rt * 8 + fr;
            double af[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) af[ks] = -rget(row, r0 + ks * 4 + fc);
            double acc[NB / 8][2];
#pragma unroll
            for (int ct = 0; ct < NB / 8; ++ct) {
                acc[ct][0] = Xs[(ct * 8 + 2 * fc) * LD + row];
                acc[ct][1] = Xs[(ct * 8 + 2 * fc + 1) * LD + row];
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = r0 + ks * 4 + fc;
#pragma unroll
                for (int ct = 0; ct < NB / 8; ++ct) dmma_8x8x4(acc[ct], af[ks], Xs[(ct * 8 + fr) * LD + kk]);
            }
#pragma unroll
            for (int ct = 0; ct < NB / 8; ++ct) {
                Xs[(ct * 8 + 2 * fc) * LD + row] = acc[ct][0];
                Xs[(ct * 8 + 2 * fc + 1) * LD + row] = acc[ct][1];
            }
        }
        __syncthreads();
    }

    constexpr int kPer = NB / (THR / 32);
    const long long mp = (lane < kPer && warp + (THR / 32) * lane < nb)
                             ? pos[c0 + warp + (THR / 32) * lane] : 0;
#pragma unroll 4
    for (int t = 0; t < kPer; ++t) {
        const int c = warp + (THR / 32) * t;
        const long long p = __shfl_sync(0xffffffffu, mp, t);
        if (c < nb) {
            const int64_t col = c0 + c;
            for (int i = lane; i < k; i += 32) Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : Xs[c * LD + i];
        }
    }
}

template <int NBLK, int NB, int THR>
cudaError_t launch_trsm_dmma_big_nb(const double* W, int64_t ldw, const double* R11, int k, int64_t n,
                                    const long long* pos, double* Z, cudaStream_t stream) {
    constexpr int KP = 32 * NBLK, LD = KP + 4;
    const size_t smem = sizeof(double) * (static_cast<size_t>(NB) * LD + 32 * 33 + KP);
    cudaError_t e = cudaFuncSetAttribute(id_trsm_dmma_big_kernel<NBLK, NB, THR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t blocks = (n + NB - 1) / NB;
    id_trsm_dmma_big_kernel<NBLK, NB, THR><<<static_cast<unsigned>(blocks), THR, smem, stream>>>(W, ldw, R11, k, n,
                                                                                                 pos, Z);
    return cudaGetLastError();
}

// Right-hand sides per CTA and threads: NB = 56 makes the 16384-column cfg4
// solve two nearly full waves of one CTA per SM (293 CTAs; 64 leaves the second
// wave 73 % full), and 8 warps share the DMMA row tiles of each block column
// (profiles/trsm_r02.txt).  IDK_TRSM_BIG=<nb> selects 64 / 56 / 48 / 32 for A/B.
template <int NBLK>
cudaError_t launch_trsm_dmma_big(const double* W, int64_t ldw, const double* R11, int k, int64_t n,
                                 const long long* pos, double* Z, cudaStream_t stream) {
    const char* ev = getenv("IDK_TRSM_BIG");
    const int sel = ev ? atoi(ev) : 56;
    switch (sel) {
        case 64: return launch_trsm_dmma_big_nb<NBLK, 64, 128>(W, ldw, R11, k, n, pos, Z, stream);
        case 65: return launch_trsm_dmma_big_nb<NBLK, 64, 256>(W, ldw, R11, k, n, pos, Z, stream);
        case 48: return launch_trsm_dmma_big_nb<NBLK, 48, 192>(W, ldw, R11, k, n, pos, Z, stream);
        case 32: return launch_trsm_dmma_big_nb<NBLK, 32, 128>(W, ldw, R11, k, n, pos, Z, stream);
        default: return launch_trsm_dmma_big_nb<NBLK, 56, 256>(W, ldw, R11, k, n, pos, Z, stream);
    }
}

// Inverses of the 32 x 32 diagonal blocks of R11 (identity beyond k), one CTA
// of 32 threads per block: thread j solves D x = e_j by back substitution
// (solve.cpp:43-51's order and divisions).  Dinv[b] is column-major, ld 32.
__global__ void __launch_bounds__(32) invert_diag_blocks_kernel(const double* __restrict__ R11, int k,
                                                                 double* __restrict__ Dinv) {
    const int b = blockIdx.x, j = threadIdx.x, r0 = 32 * b;
    __shared__ double D[32][33];
    for (int c = 0; c < 32; ++c) {
        const int row = r0 + j, col = r0 + c;
        D[j][c] = (row < k && col < k) ? R11[static_cast<int64_t>(col) * k + row] : (row == col ? 1.0 : 0.0);
    }
    __syncthreads();
    double x[32];
#pragma unroll
    for (int i = 31; i >= 0; --i) {
        double acc = i == j ? 1.0 : 0.0;
#pragma unroll
        for (int l = i + 1; l < 32; ++l) acc -= D[i][l] * x[l];
        x[i] = acc / D[i][i];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) Dinv[static_cast<int64_t>(b) * 1024 + j * 32 + i] = x[i];
}

// k in (128, 256] without the serial substitution: per 32-row block
// (bottom-up) X_b <- Dinv_b X_b and X_above -= R_above,b X_b, both on the DMMA
// pipe, so every warp works in every phase (the substitution kept one or two
// warps busy while the others waited at the barrier).
template <int NBLK, int NB, int THR>
__global__ void __launch_bounds__(THR)
id_trsm_dinv_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11,
                    const double* __restrict__ Dinv, int k, int64_t n, const long long* __restrict__ pos,
                    double* __restrict__ Z) {
    constexpr int KP = 32 * NBLK;
    constexpr int LD = KP + 4;
    constexpr int LDB = 32 + 4;  // Dinv block, column-major: fragment loads bank-conflict free
    constexpr int NW = THR / 32;
    constexpr int CT = NB / 8;    // 8-column tiles
    extern __shared__ __align__(16) double smem[];
    double* Xs = smem;            // NB right-hand sides, stride LD
    double* Db = Xs + NB * LD;    // 32 x 32 inverse diagonal block
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int fr = lane >> 2, fc = lane & 3;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NB;
    const int nb = static_cast<int>(min(static_cast<long long>(NB), static_cast<long long>(n - c0)));
    auto rget = [&](int row, int col) -> double {
        return (row < k && col < k) ? __ldg(R11 + static_cast<int64_t>(col) * k + row) : (row == col ? 1.0 : 0.0);
    };
    for (int e = tid; e < NB * KP; e += THR) {
        const int c = e / KP, row = e - c * KP;
        double* dst = Xs + c * LD + row;
        if (c < nb && row < k) cp_async_8(dst, W + (c0 + c) * ldw + row);
        else *dst = 0.0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();

#pragma unroll 1
    for (int b = NBLK - 1; b >= 0; --b) {
        const int r0 = 32 * b;
        for (int e = tid; e < 32 * 32; e += THR) Db[(e >> 5) * LDB + (e & 31)] = __ldg(Dinv + b * 1024 + e);
        __syncthreads();
        // X_b <- Dinv_b X_b: 4 row tiles x CT column tiles, k-depth 32
        constexpr int kTiles = 4 * CT;
        double acc[(kTiles + NW - 1) / NW][2];
#pragma unroll
        for (int t = 0; t < (kTiles + NW - 1) / NW; ++t) {
            acc[t][0] = acc[t][1] = 0.0;
            const int tile = warp + NW * t;
            if (tile < kTiles) {
                const int rt = tile / CT, ct = tile - rt * CT;
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const int kk = ks * 4 + fc;
                    dmma_8x8x4(acc[t], Db[kk * LDB + rt * 8 + fr], Xs[(ct * 8 + fr) * LD + r0 + kk]);
                }
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < (kTiles + NW - 1) / NW; ++t) {
            const int tile = warp + NW * t;
            if (tile < kTiles) {
                const int rt = tile / CT, ct = tile - rt * CT;
                const int row = r0 + rt * 8 + fr;
                Xs[(ct * 8 + 2 * fc) * LD + row] = acc[t][0];
                Xs[(ct * 8 + 2 * fc + 1) * LD + row] = acc[t][1];
            }
        }
        __syncthreads();
        // rows [0, r0) -= R[0:r0, block b] X_b
        for (int rt = warp; rt < 4 * b; rt += NW) {
            const int row = rt * 8 + fr;
            double af[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) af[ks] = -rget(row, r0 + ks * 4 + fc);
            double ac[CT][2];
#pragma unroll
            for (int ct = 0; ct < CT; ++ct) {
                ac[ct][0] = Xs[(ct * 8 + 2 * fc) * LD + row];
                ac[ct][1] = Xs[(ct * 8 + 2 * fc + 1) * LD + row];
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int kk = r0 + ks * 4 + fc;
#pragma unroll
                for (int ct = 0; ct < CT; ++ct) dmma_8x8x4(ac[ct], af[ks], Xs[(ct * 8 + fr) * LD + kk]);
            }
#pragma unroll
            for (int ct = 0; ct < CT; ++ct) {
                Xs[(ct * 8 + 2 * fc) * LD + row] = ac[ct][0];
                Xs[(ct * 8 + 2 * fc + 1) * LD + row] = ac[ct][1];
            }
        }
        __syncthreads();
    }

    constexpr int kPer = NB / NW;
    const long long mp = (lane < kPer && warp + NW * lane < nb) ? pos[c0 + warp + NW * lane] : 0;
#pragma unroll 4
    for (int t = 0; t < kPer; ++t) {
        const int c = warp + NW * t;
        const long long p = __shfl_sync(0xffffffffu, mp, t);
        if (c < nb) {
            const int64_t col = c0 + c;
            for (int i = lane; i < k; i += 32) Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : Xs[c * LD + i];
        }
    }
}

template <int NBLK, int NB, int THR>
cudaError_t launch_trsm_dinv(const double* W, int64_t ldw, const double* R11, double* Dinv, int k, int64_t n,
                             const long long* pos, double* Z, cudaStream_t stream) {
    invert_diag_blocks_kernel<<<NBLK, 32, 0, stream>>>(R11, k, Dinv);
    constexpr int KP = 32 * NBLK, LD = KP + 4;
    const size_t smem = sizeof(double) * (static_cast<size_t>(NB) * LD + 32 * 36);
    cudaError_t e = cudaFuncSetAttribute(id_trsm_dinv_kernel<NBLK, NB, THR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int64_t blocks = (n + NB - 1) / NB;
    id_trsm_dinv_kernel<NBLK, NB, THR><<<static_cast<unsigned>(blocks), THR, smem, stream>>>(W, ldw, R11, Dinv, k, n,
                                                                                             pos, Z);
    return cudaGetLastError();
}

template <int NBLK>
size_t trsm_dmma_smem() {
    constexpr int KP = 32 * NBLK, LD = KP + 4;
    return sizeof(double) * (static_cast<size_t>(KP) * LD + static_cast<size_t>(kDmmaNB) * LD + KP);
}

template <int NBLK>
cudaError_t launch_trsm_dmma(const double* W, int64_t ldw, const double* R11, int k, int64_t n,
                             const long long* pos, double* Z, cudaStream_t stream) {
    const size_t smem = trsm_dmma_smem<NBLK>();
    const int64_t blocks = (n + kDmmaNB - 1) / kDmmaNB;
    const char* pv = getenv("IDK_TRSM_PAIRS");
    const bool pairs = !(pv && atoi(pv) == 0) && k % 2 == 0 && ldw % 2 == 0 &&
                       (reinterpret_cast<uintptr_t>(W) & 15) == 0 && (reinterpret_cast<uintptr_t>(R11) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(Z) & 15) == 0;
    auto kern = pairs ? id_trsm_dmma_kernel<NBLK, true> : id_trsm_dmma_kernel<NBLK, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(blocks), kDmmaThreads, smem, stream>>>(W, ldw, R11, k, n, pos, Z);
    return cudaGetLastError();
}

// Warp-independent back substitution (solve.cpp:43-51 restated): each warp
// owns kCW right-hand sides with all k <= 32*KJ rows in registers (lane owns
// rows lane + 32 j).  Step i broadcasts the finished x_i by shuffle, every lane
// applies r_{.,i} x_i to its rows above i, and the owner of row i-1 finishes it
// (multiplying by 1/r_{i-1,i-1}, computed once).  R11 column i-1 is loaded
// while step i runs.  No block-level barrier anywhere.
constexpr int kCW = 4;

template <int KJ>
__global__ void __launch_bounds__(128)
id_trsm_warp_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
                    const long long* __restrict__ pos, double* __restrict__ Z) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t cbase = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wid) * kCW;
    if (cbase >= n) return;
    double x[kCW][KJ], rinv[KJ], rc[KJ], rn[KJ];
#pragma unroll
    for (int c = 0; c < kCW; ++c) {
        const bool ok = cbase + c < n;
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            const int row = lane + 32 * j;
            x[c][j] = (ok && row < k) ? W[(cbase + c) * ldw + row] : 0.0;
        }
    }
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        const int row = lane + 32 * j;
        rinv[j] = row < k ? 1.0 / R11[static_cast<int64_t>(row) * k + row] : 0.0;
    }
    // row k-1 has no updates: finish it
    {
        const int jl = (k - 1) >> 5, tl = (k - 1) & 31;
#pragma unroll
        for (int j = 0; j < KJ; ++j)
            if (j == jl && lane == tl)
#pragma unroll
                for (int c = 0; c < kCW; ++c) x[c][j] *= rinv[j];
    }
    // column k-1 of R11
#pragma unroll
    for (int j = 0; j < KJ; ++j) {
        const int row = lane + 32 * j;
        rc[j] = row < k - 1 ? __ldg(R11 + static_cast<int64_t>(k - 1) * k + row) : 0.0;
    }
#pragma unroll
    for (int j = KJ - 1; j >= 0; --j) {
        const int tmax = min(31, k - 1 - 32 * j);
        for (int t = tmax; t >= 0; --t) {
            const int i = 32 * j + t;
            if (i == 0) break;
            // prefetch column i-1 (rows < i-1)
#pragma unroll
            for (int jr = 0; jr < KJ; ++jr) {
                const int row = lane + 32 * jr;
                rn[jr] = (jr <= j && row < i - 1) ? __ldg(R11 + static_cast<int64_t>(i - 1) * k + row) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < kCW; ++c) {
                const double xi = __shfl_sync(0xffffffffu, x[c][j], t);
#pragma unroll
                for (int jr = 0; jr < j; ++jr) x[c][jr] = fma(-rc[jr], xi, x[c][jr]);
                if (lane < t) x[c][j] = fma(-rc[j], xi, x[c][j]);
            }
            // row i-1 is final now
            if (t > 0) {
                if (lane == t - 1)
#pragma unroll
                    for (int c = 0; c < kCW; ++c) x[c][j] *= rinv[j];
            } else if (j > 0) {
                if (lane == 31)
#pragma unroll
                    for (int c = 0; c < kCW; ++c) x[c][j - 1] *= rinv[j - 1];
            }
#pragma unroll
            for (int jr = 0; jr < KJ; ++jr) rc[jr] = rn[jr];
        }
    }
#pragma unroll
    for (int c = 0; c < kCW; ++c) {
        const int64_t col = cbase + c;
        if (col >= n) break;
        const long long p = pos[col];
#pragma unroll
        for (int j = 0; j < KJ; ++j) {
            const int row = lane + 32 * j;
            if (row < k) Z[col * k + row] = p < k ? (row == p ? 1.0 : 0.0) : x[c][j];
        }
    }
}

template <int KJ>
cudaError_t launch_trsm_warp(const double* W, int64_t ldw, const double* R11, int k, int64_t n, const long long* pos,
                             double* Z, cudaStream_t stream) {
    const int64_t warps = (n + kCW - 1) / kCW;
    const int64_t blocks = (warps + 3) / 4;
    id_trsm_warp_kernel<KJ><<<static_cast<unsigned>(blocks), 128, 0, stream>>>(W, ldw, R11, k, n, pos, Z);
    return cudaGetLastError();
}

// Right-looking back substitution over a k x NB tile of right-hand sides kept
// in shared memory (solve.cpp:43-51 restated column-parallel): step i finishes
// row i (the thread that applies the last update to x_i also divides by
// r_ii), then every thread subtracts r_{.,i} x_i from the rows above.  One
// __syncthreads per row; column i-1 of R11 is prefetched into shared memory
// while step i runs.
__global__ void __launch_bounds__(256)
id_trsm_rl_kernel(const double* __restrict__ W, int64_t ldw, const double* __restrict__ R11, int k, int64_t n,
                  const long long* __restrict__ pos, double* __restrict__ Z, int NB) {
    extern __shared__ double sm[];
    const int ldx = k | 1;
    double* X = sm;                                   // NB columns, stride ldx
    double* rcol = X + static_cast<size_t>(NB) * ldx;  // 2 x k: column i of R11 (double buffer)
    double* rdiag = rcol + 2 * k;                     // k
    const int tid = threadIdx.x, T = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * NB;
    const int nb = static_cast<int>(min(static_cast<long long>(NB), static_cast<long long>(n - c0)));

    for (int c = wid; c < nb; c += nw)
        for (int i = lane; i < k; i += 32) X[c * ldx + i] = W[(c0 + c) * ldw + i];
    for (int i = tid; i < k; i += T) {
        rdiag[i] = R11[static_cast<int64_t>(i) * k + i];
        rcol[((k - 1) & 1) * k + i] = R11[static_cast<int64_t>(k - 1) * k + i];
    }
    __syncthreads();
    // row k-1 has no updates: divide it
    for (int c = tid; c < nb; c += T) X[c * ldx + k - 1] = X[c * ldx + k - 1] / rdiag[k - 1];
    __syncthreads();
    for (int i = k - 1; i > 0; --i) {
        const double* rc = rcol + (i & 1) * k;  // R11[0:i, i]
        // prefetch column i-1 for the next step (async copy: no stall on L2 latency)
        double* rn = rcol + ((i - 1) & 1) * k;
        for (int r = tid; r < i - 1; r += T) {
            const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(rn + r));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst),
                         "l"(R11 + static_cast<int64_t>(i - 1) * k + r));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        // warp w owns columns w, w+nw, ...; lane owns rows lane, lane+32, ... (< i)
        for (int c = wid; c < nb; c += nw) {
            double* xc = X + c * ldx;
            const double xi = xc[i];
            for (int r = lane; r < i; r += 32) {
                double v = fma(-rc[r], xi, xc[r]);
                if (r == i - 1) v = v / rdiag[r];  // x_{i-1} is final now
                xc[r] = v;
            }
        }
        asm volatile("cp.async.wait_all;\n" ::);
        __syncthreads();
    }
    for (int c = wid; c < nb; c += nw) {
        const int64_t col = c0 + c;
        const long long p = pos[col];
        for (int i = lane; i < k; i += 32) Z[col * k + i] = p < k ? (i == p ? 1.0 : 0.0) : X[c * ldx + i];
    }
}

// C[:, j] = A[:, cols[j]]  (matrix.cpp:121-130), or for the id_auto dual
// C[:, j] = A[cols[j], :]^T (a row of the tall A is a column of A^T).
__global__ void gather_columns_kernel(const double* __restrict__ A, int64_t lda, int64_t rows,
                                      const long long* __restrict__ cols, int k, bool rows_of_a,
                                      double* __restrict__ C) {
    const int64_t total = rows * k;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / rows, i = e - j * rows;
        C[e] = rows_of_a ? A[cols[j] + i * lda] : A[cols[j] * lda + i];
    }
}

// C[:, j] = A[:, cols[j]] (matrix.cpp:121-130): blockIdx.y = j, each thread
// moves kGatherVec 16-byte pairs with streaming loads/stores (both columns
// 16-byte aligned: A, C aligned, lda and rows even).
constexpr int kGatherVec = 4;
__global__ void gather_columns_vec_kernel(const double* __restrict__ A, int64_t lda, int64_t rows,
                                          const long long* __restrict__ cols, double* __restrict__ C) {
    const int j = blockIdx.y;
    const double2* src = reinterpret_cast<const double2*>(A + cols[j] * lda);
    double2* dst = reinterpret_cast<double2*>(C + j * rows);
    const int64_t pairs = rows >> 1;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x * kGatherVec + threadIdx.x;
    double2 v[kGatherVec];
#pragma unroll
    for (int u = 0; u < kGatherVec; ++u) {
        const int64_t p = base + static_cast<int64_t>(u) * blockDim.x;
        if (p < pairs) v[u] = __ldcs(src + p);
    }
#pragma unroll
    for (int u = 0; u < kGatherVec; ++u) {
        const int64_t p = base + static_cast<int64_t>(u) * blockDim.x;
        if (p < pairs) __stcs(dst + p, v[u]);
    }
}

// Rows of A for the dual (id.cpp:85-92): C[i, j] = A[cols[j], i], C is n x k.
// A CTA takes 32 values of i: warp w reads A[cols[j], i0 + lane] for its j's
// (32 consecutive i of one row: 32 strided sectors), stages a 32 x k tile in
// shared memory, and writes C coalesced along i.
template <int LV>
__device__ __forceinline__ double ld_row_elem(const double* p) {
    if constexpr (LV == 1) return __ldg(p);
    if constexpr (LV == 2) {
        double v;
        asm volatile("ld.global.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
        return v;
    }
    if constexpr (LV == 3) {
        double v;
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
        return v;
    }
    return __ldcs(p);
}

template <int LV>
__global__ void gather_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t n,
                                   const long long* __restrict__ cols, int k, double* __restrict__ C) {
    extern __shared__ double tile[];  // k x 33
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int64_t i = i0 + lane;
    int j = wid;
    for (; j + 3 * nw < k; j += 4 * nw) {  // four independent sector reads in flight per thread
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = i < n ? ld_row_elem<LV>(A + cols[j + u * nw] + i * lda) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) tile[(j + u * nw) * 33 + lane] = v[u];
    }
    for (; j < k; j += nw) tile[j * 33 + lane] = i < n ? ld_row_elem<LV>(A + cols[j] + i * lda) : 0.0;
    __syncthreads();
    for (int j = wid; j < k; j += nw)
        if (i < n) __stcs(C + static_cast<int64_t>(j) * n + i, tile[j * 33 + lane]);
}
// Sharded C: this rank holds columns [c_begin, c_end) of M (A_local, or the
// row block of the stored tall A for the dual).  Column j of C is written here
// only when its pivot is local; the owners' broadcasts fill the rest.
__global__ void gather_owned_kernel(const double* __restrict__ A, int64_t lda, int64_t rows,
                                    const long long* __restrict__ cols, int64_t c_begin, int64_t c_end, bool rows_of_a,
                                    double* __restrict__ C) {
    const int j = blockIdx.y;
    const long long g = cols[j];
    if (g < c_begin || g >= c_end) return;
    const int64_t loc = g - c_begin;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        C[static_cast<int64_t>(j) * rows + i] = rows_of_a ? A[loc + i * lda] : A[loc * lda + i];
}
__global__ void copy_pivots_kernel(const long long* __restrict__ src, int k, long long* __restrict__ dst) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) dst[i] = src[i];
}

}  // namespace

// R11 buffer of id_solve_z: k x k, then the inverse diagonal blocks (k > 128).
size_t id_solve_z_scratch(int k) {
    return sizeof(double) * (static_cast<size_t>(k) * k + 1024 * static_cast<size_t>((k + 31) / 32));
}

// Right-hand sides per CTA: 32 while the k x 32 tile fits in ~160 KB.
int id_trsm_nb(int k) {
    const int cap = static_cast<int>((160 * 1024 / sizeof(double)) / (k | 1));
    return cap >= kTrsmNB ? kTrsmNB : (cap < 1 ? 1 : cap);
}

size_t id_trsm_smem_bytes(int k) { return sizeof(double) * static_cast<size_t>(id_trsm_nb(k)) * (k | 1); }

// Z[:, j] for the columns j in [c_begin, c_begin + n) of W (Z has ld k and
// starts at column c_begin); R11 is gathered from the pivot columns of W.
cudaError_t id_solve_z(const double* W, int64_t ldw, int k, int64_t c_begin, int64_t n, const long long* pivots,
                       const long long* pos, double* R11, int* status, double* Z, cudaStream_t stream) {
    const int64_t kk = static_cast<int64_t>(k) * k;
    gather_r11_kernel<<<static_cast<int>(std::min<int64_t>((kk + 255) / 256, 1024)), 256, 0, stream>>>(
        W, ldw, pivots, k, R11, status);
    W += c_begin * ldw;
    pos += c_begin;
    if (n <= 0) return cudaGetLastError();
    const char* te = getenv("IDK_TRSM_DMMA");
    if (k <= 128 && !(te && atoi(te) == 0)) {
        switch ((k + 31) / 32) {
            case 1: return launch_trsm_dmma<1>(W, ldw, R11, k, n, pos, Z, stream);
            case 2: return launch_trsm_dmma<2>(W, ldw, R11, k, n, pos, Z, stream);
            case 3: return launch_trsm_dmma<3>(W, ldw, R11, k, n, pos, Z, stream);
            default: return launch_trsm_dmma<4>(W, ldw, R11, k, n, pos, Z, stream);
        }
    }
    const char* tv = getenv("IDK_TRSM_DINV");
    if (k > 128 && k <= 256 && !(te && atoi(te) == 0) && !(tv && atoi(tv) == 0)) {
        double* Dinv = R11 + static_cast<int64_t>(k) * k;  // carved after R11 (id_solve_z_scratch)
        const char* nbv = getenv("IDK_TRSM_NB");
        const int nbsel = nbv ? atoi(nbv) : 64;  // profiles/trsm_r02.txt
        switch ((k + 31) / 32) {
#define IDK_DINV(NBLK)                                                                                           \
    case NBLK:                                                                                                   \
        if (nbsel == 64) return launch_trsm_dinv<NBLK, 64, 256>(W, ldw, R11, Dinv, k, n, pos, Z, stream);         \
        if (nbsel == 16) return launch_trsm_dinv<NBLK, 16, 128>(W, ldw, R11, Dinv, k, n, pos, Z, stream);         \
        return launch_trsm_dinv<NBLK, 32, 128>(W, ldw, R11, Dinv, k, n, pos, Z, stream);
            IDK_DINV(5) IDK_DINV(6) IDK_DINV(7) IDK_DINV(8)
#undef IDK_DINV
            default: break;
        }
    }
    if (k <= 256 && !(te && atoi(te) == 0)) {
        switch ((k + 31) / 32) {
            case 5: return launch_trsm_dmma_big<5>(W, ldw, R11, k, n, pos, Z, stream);
            case 6: return launch_trsm_dmma_big<6>(W, ldw, R11, k, n, pos, Z, stream);
            case 7: return launch_trsm_dmma_big<7>(W, ldw, R11, k, n, pos, Z, stream);
            default: return launch_trsm_dmma_big<8>(W, ldw, R11, k, n, pos, Z, stream);
        }
    }
    switch ((k + 31) / 32) {
        case 1: return launch_trsm_warp<1>(W, ldw, R11, k, n, pos, Z, stream);
        case 2: return launch_trsm_warp<2>(W, ldw, R11, k, n, pos, Z, stream);
        case 3: return launch_trsm_warp<3>(W, ldw, R11, k, n, pos, Z, stream);
        case 4: return launch_trsm_warp<4>(W, ldw, R11, k, n, pos, Z, stream);
        case 5: return launch_trsm_warp<5>(W, ldw, R11, k, n, pos, Z, stream);
        case 6: return launch_trsm_warp<6>(W, ldw, R11, k, n, pos, Z, stream);
        case 7: return launch_trsm_warp<7>(W, ldw, R11, k, n, pos, Z, stream);
        case 8: return launch_trsm_warp<8>(W, ldw, R11, k, n, pos, Z, stream);
        default: break;  // k > 256: shared-memory kernels below
    }
    // Right-hand sides per CTA: enough CTAs to cover the SMs twice, at most 64,
    // and the k x NB tile within ~150 KB of shared memory.
    int nb = static_cast<int>(std::min<int64_t>(64, std::max<int64_t>(8, n / 296)));
    nb = (nb + 7) & ~7;
    while (nb > 1 && sizeof(double) * (static_cast<size_t>(nb) * (k | 1) + 3 * static_cast<size_t>(k)) > 150 * 1024)
        nb = nb > 8 ? nb - 8 : nb - 1;
    if (sizeof(double) * (static_cast<size_t>(nb) * (k | 1) + 3 * static_cast<size_t>(k)) <= 200 * 1024) {
        const size_t smem = sizeof(double) * (static_cast<size_t>(nb) * (k | 1) + 3 * static_cast<size_t>(k));
        cudaError_t e = cudaFuncSetAttribute(id_trsm_rl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        const int64_t blocks = (n + nb - 1) / nb;
        id_trsm_rl_kernel<<<static_cast<unsigned>(blocks), 256, smem, stream>>>(W, ldw, R11, k, n, pos, Z, nb);
        return cudaGetLastError();
    }
    // very large k: blocked kernel with global R11 reads
    const size_t smem = id_trsm_smem_bytes(k);
    cudaError_t e = cudaFuncSetAttribute(id_trsm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int nb2 = id_trsm_nb(k);
    const int64_t blocks = (n + nb2 - 1) / nb2;
    id_trsm_kernel<<<static_cast<unsigned>(blocks), kTrsmThreads, smem, stream>>>(W, ldw, R11, k, n, pos, Z, nb2);
    return cudaGetLastError();
}

cudaError_t gather_r11(const double* W, int64_t ldw, const long long* pivots, int k, double* R11,
                       cudaStream_t stream) {
    const int64_t kk = static_cast<int64_t>(k) * k;
    gather_r11_kernel<<<static_cast<int>(std::min<int64_t>((kk + 255) / 256, 1024)), 256, 0, stream>>>(
        W, ldw, pivots, k, R11, nullptr);
    return cudaGetLastError();
}

cudaError_t gather_columns(const double* A, int64_t lda, int64_t rows, const long long* cols, int k,
                           bool rows_of_a, double* C, cudaStream_t stream) {
    const int64_t total = rows * k;
    if (total <= 0) return cudaSuccess;
    if (!rows_of_a && rows % 2 == 0 && lda % 2 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
        (reinterpret_cast<uintptr_t>(C) & 15) == 0 && k <= 65535) {
        const int64_t per = 256LL * kGatherVec;  // pairs per CTA
        const dim3 grid(static_cast<unsigned>((rows / 2 + per - 1) / per), static_cast<unsigned>(k));
        gather_columns_vec_kernel<<<grid, 256, 0, stream>>>(A, lda, rows, cols, C);
        return cudaGetLastError();
    }
    if (rows_of_a && sizeof(double) * static_cast<size_t>(k) * 33 <= 200 * 1024) {
        const size_t smem = sizeof(double) * static_cast<size_t>(k) * 33;
        // loads with the .L2::64B prefetch size: each scattered 8-byte element
        // costs a 64-byte L2 fill instead of 128 (cfg5: 33.6 -> 16.8 MB of DRAM reads
        // for 2.1 MB of C; profiles/gather_rows_r02.txt).  IDK_GATHER_ROWS_LD selects
        // the other load forms for A/B.
        const char* lv = getenv("IDK_GATHER_ROWS_LD");
        const int sel = lv ? atoi(lv) : 2;
        auto kern = sel == 1 ? gather_rows_kernel<1> : sel == 2 ? gather_rows_kernel<2>
                  : sel == 3 ? gather_rows_kernel<3> : gather_rows_kernel<0>;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        kern<<<static_cast<unsigned>((rows + 31) / 32), k >= 256 ? 256 : 128, smem, stream>>>(A, lda, rows, cols, k, C);
        return cudaGetLastError();
    }
    gather_columns_kernel<<<static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8)), 256, 0, stream>>>(
        A, lda, rows, cols, k, rows_of_a, C);
    return cudaGetLastError();
}

cudaError_t gather_owned(const double* A, int64_t lda, int64_t rows, const long long* cols, int k, int64_t c_begin,
                         int64_t c_end, bool rows_of_a, double* C, cudaStream_t stream) {
    if (rows <= 0 || k <= 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((rows + 255) / 256, 64)), static_cast<unsigned>(k));
    gather_owned_kernel<<<grid, 256, 0, stream>>>(A, lda, rows, cols, c_begin, c_end, rows_of_a, C);
    return cudaGetLastError();
}

cudaError_t copy_pivots(const long long* src, int k, long long* dst, cudaStream_t stream) {
    copy_pivots_kernel<<<1, 256, 0, stream>>>(src, k, dst);
    return cudaGetLastError();
}

}  // namespace idk
