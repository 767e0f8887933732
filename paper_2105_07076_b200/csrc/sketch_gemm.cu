// sketch_gemm.cu -- Y = Omega * A (or Omega * A^T) in fp64 on the DMMA tensor pipe.
//
// Replaces the reference's Y = matmul(Omega, A) of the composed sketch oracle
// (matrix.cpp:28-48 called on generate(gaussian, l, m, seed), datasets.cpp:15-33).
// Omega is l x K column-major (l = k + p is small: 72..272), A is the big
// matrix.  Two B layouts:
//   * kNT = false : B[kk, j] = A[kk + j*ldb]   (A is K x n, column-major)
//   * kNT = true  : B[kk, j] = A[j + kk*ldb]   (A is n x K, column-major; the
//                   id_auto dual Y = Omega * A^T without materialising A^T,
//                   id.cpp:85)
// CTA tile BM x 64 x 16 (BM = 16*WM, chosen so BM covers l with little
// padding), 4 warps in 2 x 2, warp tile (8*WM) x 32 of m8n8k4 DMMA tiles,
// 2-stage cp.async pipeline (46 KB of shared memory: 4 CTAs per SM), optional split-K with a fixed-order reduction so
// results are bit-reproducible run to run.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace idk {

namespace {

constexpr int kBN = 64;
#ifndef IDK_GEMM_BK
#define IDK_GEMM_BK 16
#endif
#ifndef IDK_GEMM_STAGES
#define IDK_GEMM_STAGES 2
#endif
constexpr int kBK = IDK_GEMM_BK;
constexpr int kStages = IDK_GEMM_STAGES;
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, bool pred) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int WM, bool kNT>
struct Smem {
    static constexpr int BM = 16 * WM;
    static constexpr int SA = BM + 4;                  // As[kk][i], stride = 4 mod 16 doubles
    static constexpr int SB = kNT ? (kBN + 4) : (kBK + 4);  // Bs[kk][j] or Bs[j][kk]
    static constexpr int A_ELEMS = kBK * SA;
    static constexpr int B_ELEMS = kNT ? kBK * SB : kBN * SB;
    static constexpr int STAGE = A_ELEMS + B_ELEMS;
    static constexpr size_t BYTES = sizeof(double) * STAGE * kStages;
};

template <int WM, bool kNT>
__global__ void __launch_bounds__(kThreads)
sketch_gemm_kernel(const double* __restrict__ A, int64_t lda,  // Omega: l x K
                   const double* __restrict__ B, int64_t ldb,  // big matrix
                   double* __restrict__ C, int64_t ldc,        // Y (or split-K partial base)
                   int64_t split_stride,                       // elements between split partials
                   int M, int64_t N, int64_t K, int64_t k_per_split, bool vec16,
                   const double* __restrict__ Ref, int64_t ldr, bool ref_trans, double* __restrict__ resid,
                   const GemmGroup grp) {
    using S = Smem<WM, kNT>;
    constexpr int BM = S::BM;
    extern __shared__ __align__(16) double smem[];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int m0 = blockIdx.x * BM;
    const int64_t n0 = static_cast<int64_t>(blockIdx.y) * kBN;
    int split = blockIdx.z;
    if (grp.count > 0) {  // grouped launch: blockIdx.z = member * splits + split
        const int g = blockIdx.z / grp.splits;
        split = blockIdx.z - g * grp.splits;
        A += g * grp.a_stride;
        B = grp.b[g];
        C += g * grp.c_stride;
    }
    const int64_t kbeg = static_cast<int64_t>(split) * k_per_split;
    const int64_t kend = min(K, kbeg + k_per_split);
    const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kBK - 1) / kBK) : 0;
    C += static_cast<int64_t>(split) * split_stride;

    auto load_stage = [&](int stage, int kt) {
        double* As = smem + stage * S::STAGE;
        double* Bs = As + S::A_ELEMS;
        const int64_t k0 = kbeg + static_cast<int64_t>(kt) * kBK;
        // A tile: kBK columns of Omega, BM contiguous rows each.
        if (vec16) {
            for (int e = tid; e < kBK * (BM / 2); e += kThreads) {
                const int kk = e / (BM / 2), i = (e % (BM / 2)) * 2;
                const int64_t gk = k0 + kk;
                const int gi = m0 + i;
                int bytes = 0;
                if (gk < kend && gi < M) bytes = (gi + 1 < M) ? 16 : 8;
                const double* src = bytes ? A + gk * lda + gi : A;
                cp_async_16(As + kk * S::SA + i, src, bytes);
            }
        } else {
            for (int e = tid; e < kBK * BM; e += kThreads) {
                const int kk = e / BM, i = e % BM;
                const int64_t gk = k0 + kk;
                const int gi = m0 + i;
                const bool ok = gk < kend && gi < M;
                cp_async_8(As + kk * S::SA + i, ok ? A + gk * lda + gi : A, ok);
            }
        }
        if constexpr (!kNT) {
            // B tile: kBN columns of A, kBK contiguous k each -> Bs[j][kk].
            if (vec16) {
                for (int e = tid; e < kBN * (kBK / 2); e += kThreads) {
                    const int j = e / (kBK / 2), kk = (e % (kBK / 2)) * 2;
                    const int64_t gj = n0 + j, gk = k0 + kk;
                    int bytes = 0;
                    if (gj < N && gk < kend) bytes = (gk + 1 < kend) ? 16 : 8;
                    const double* src = bytes ? B + gj * ldb + gk : B;
                    cp_async_16(Bs + j * S::SB + kk, src, bytes);
                }
            } else {
                for (int e = tid; e < kBN * kBK; e += kThreads) {
                    const int j = e / kBK, kk = e % kBK;
                    const int64_t gj = n0 + j, gk = k0 + kk;
                    const bool ok = gj < N && gk < kend;
                    cp_async_8(Bs + j * S::SB + kk, ok ? B + gj * ldb + gk : B, ok);
                }
            }
        } else {
            // B tile: kBK rows of A^T = kBK columns of A (n x K), kBN contiguous j each -> Bs[kk][j].
            if (vec16) {
                for (int e = tid; e < kBK * (kBN / 2); e += kThreads) {
                    const int kk = e / (kBN / 2), j = (e % (kBN / 2)) * 2;
                    const int64_t gj = n0 + j, gk = k0 + kk;
                    int bytes = 0;
                    if (gk < kend && gj < N) bytes = (gj + 1 < N) ? 16 : 8;
                    const double* src = bytes ? B + gk * ldb + gj : B;
                    cp_async_16(Bs + kk * S::SB + j, src, bytes);
                }
            } else {
                for (int e = tid; e < kBK * kBN; e += kThreads) {
                    const int kk = e / kBN, j = e % kBN;
                    const int64_t gj = n0 + j, gk = k0 + kk;
                    const bool ok = gk < kend && gj < N;
                    cp_async_8(Bs + kk * S::SB + j, ok ? B + gk * ldb + gj : B, ok);
                }
            }
        }
    };

    double acc[WM][4][2];
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < ktiles) load_stage(s, s);
        cp_async_commit();
    }

    const int fr = lane >> 2, fc = lane & 3;
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        {
            const int nk = kt + kStages - 1;
            if (nk < ktiles) load_stage(nk % kStages, nk);
            cp_async_commit();
        }
        const double* As = smem + (kt % kStages) * S::STAGE;
        const double* Bs = As + S::A_ELEMS;
#pragma unroll
        for (int kq = 0; kq < kBK / 4; ++kq) {
            double af[WM], bf[4];
#pragma unroll
            for (int tm = 0; tm < WM; ++tm) af[tm] = As[(kq * 4 + fc) * S::SA + wm * (8 * WM) + tm * 8 + fr];
#pragma unroll
            for (int tn = 0; tn < 4; ++tn) {
                const int j = wn * 32 + tn * 8 + fr;
                if constexpr (kNT)
                    bf[tn] = Bs[(kq * 4 + fc) * S::SB + j];
                else
                    bf[tn] = Bs[j * S::SB + kq * 4 + fc];
            }
#pragma unroll
            for (int tm = 0; tm < WM; ++tm)
#pragma unroll
                for (int tn = 0; tn < 4; ++tn) dmma_8x8x4(acc[tm][tn], af[tm], bf[tn]);
        }
    }
    cp_async_wait<0>();

    if (Ref != nullptr) {
        // Fused residual (id.cpp:97-122 diagnostics without materialising
        // approx): sum (Ref - A*B)^2 and sum Ref^2 over this tile, one pair
        // of partials per warp, reduced in a fixed order afterwards.
        double dsum = 0.0, rsum = 0.0;
#pragma unroll
        for (int tm = 0; tm < WM; ++tm) {
            const int i = m0 + wm * (8 * WM) + tm * 8 + fr;
#pragma unroll
            for (int tn = 0; tn < 4; ++tn) {
                const int64_t j = n0 + wn * 32 + tn * 8 + 2 * fc;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (i < M && j + u < N) {
                        const double r = ref_trans ? Ref[static_cast<int64_t>(i) * ldr + j + u] : Ref[(j + u) * ldr + i];
                        const double d = r - acc[tm][tn][u];
                        dsum = fma(d, d, dsum);
                        rsum = fma(r, r, rsum);
                    }
                }
            }
        }
        dsum = warp_sum(dsum);
        rsum = warp_sum(rsum);
        if (lane == 0) {
            const int64_t cta = blockIdx.x + static_cast<int64_t>(gridDim.x) * (blockIdx.y + static_cast<int64_t>(gridDim.y) * blockIdx.z);
            resid[(cta * 4 + warp) * 2] = dsum;
            resid[(cta * 4 + warp) * 2 + 1] = rsum;
        }
        return;
    }

#pragma unroll
    for (int tm = 0; tm < WM; ++tm) {
        const int i = m0 + wm * (8 * WM) + tm * 8 + fr;
        if (i >= M) continue;
#pragma unroll
        for (int tn = 0; tn < 4; ++tn) {
            const int64_t j = n0 + wn * 32 + tn * 8 + 2 * fc;
            if (j < N) C[j * ldc + i] = acc[tm][tn][0];
            if (j + 1 < N) C[(j + 1) * ldc + i] = acc[tm][tn][1];
        }
    }
}

// Fixed-order split-K reduction: Y = sum_{s=0}^{S-1} P_s (s ascending).
__global__ void splitk_reduce_kernel(const double* __restrict__ P, int64_t split_stride, int splits,
                                     double* __restrict__ Y, int M, int64_t N, int64_t ldc) {
    const int64_t total = static_cast<int64_t>(M) * N;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / M;
        const int i = static_cast<int>(e - j * M);
        const int64_t off = j * ldc + i;
        double s = P[off];
        for (int t = 1; t < splits; ++t) s += P[t * split_stride + off];
        Y[off] = s;
    }
}

// Sharded sketch with the all-gather fused in (idk_id_sharded's peer mode): the
// split-K reduction writes each finished element of this rank's Y block to
// every rank's Y buffer (f.y[g]: this rank's slot in rank g's buffer, mapped
// over NVLink by CUDA IPC; f.y[0] is the local one), so the exchange rides on
// the reduction's stores instead of a separate collective.  The system-scope
// fence orders the remote stores before the kernel's completion, which the
// caller's stream-ordered barrier then publishes.
__global__ void splitk_reduce_fanout_kernel(const double* __restrict__ P, int64_t split_stride, int splits,
                                            const FanOut f, int M, int64_t N, int64_t ldc) {
    const int64_t total = static_cast<int64_t>(M) * N;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / M;
        const int i = static_cast<int>(e - j * M);
        const int64_t off = j * ldc + i;
        double s = P[off];
        for (int t = 1; t < splits; ++t) s += P[t * split_stride + off];
#pragma unroll 1
        for (int g = 0; g < f.count; ++g) f.y[g][off] = s;
    }
    __threadfence_system();
}

// splits == 1: the GEMM wrote f.y[0]; copy the block to the other destinations.
__global__ void fanout_copy_kernel(const FanOut f, int M, int64_t N, int64_t ldc) {
    const int64_t total = static_cast<int64_t>(M) * N;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / M;
        const int64_t off = j * ldc + (e - j * M);
        const double v = f.y[0][off];
#pragma unroll 1
        for (int g = 1; g < f.count; ++g) f.y[g][off] = v;
    }
    __threadfence_system();
}

// Grouped form: member g reduces the partials at P + g*group_stride into Ys[g].
__global__ void splitk_reduce_group_kernel(const double* __restrict__ P, int64_t split_stride, int splits,
                                           int64_t group_stride, const GemmGroup grp, int M, int64_t N,
                                           int64_t ldc) {
    const int64_t total = static_cast<int64_t>(M) * N;
    const int g = blockIdx.y;
    P += g * group_stride;
    double* Y = grp.y[g];
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / M;
        const int i = static_cast<int>(e - j * M);
        const int64_t off = j * ldc + i;
        double s = P[off];
        for (int t = 1; t < splits; ++t) s += P[t * split_stride + off];
        Y[off] = s;
    }
}

template <int WM, bool kNT>
cudaError_t launch_wm(const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                      int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K, int splits,
                      bool vec16, cudaStream_t stream, const double* Ref = nullptr, int64_t ldr = 0,
                      bool ref_trans = false, double* resid = nullptr, const GemmGroup* grp = nullptr) {
    using S = Smem<WM, kNT>;
    auto kern = sketch_gemm_kernel<WM, kNT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(S::BYTES));
    if (e != cudaSuccess) return e;
    int64_t kps = (K + splits - 1) / splits;
    kps = ((kps + kBK - 1) / kBK) * kBK;
    GemmGroup g{};
    if (grp) g = *grp;
    g.splits = splits;
    const unsigned gz = static_cast<unsigned>(splits * (g.count > 0 ? g.count : 1));
    dim3 grid((M + S::BM - 1) / S::BM, static_cast<unsigned>((N + kBN - 1) / kBN), gz);
    kern<<<grid, kThreads, S::BYTES, stream>>>(A, lda, B, ldb, C, ldc, split_stride, M, N, K, kps,
                                               vec16, Ref, ldr, ref_trans, resid, g);
    return cudaGetLastError();
}

template <bool kNT>
cudaError_t launch_nt(int wm, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                      int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K, int splits,
                      bool vec16, cudaStream_t stream, const GemmGroup* grp = nullptr) {
#define IDK_LWM(W) launch_wm<W, kNT>(A, lda, B, ldb, C, ldc, split_stride, M, N, K, splits, vec16, stream, \
                                     nullptr, 0, false, nullptr, grp)
    switch (wm) {
        case 2: return IDK_LWM(2);
        case 3: return IDK_LWM(3);
        case 4: return IDK_LWM(4);
        case 5: return IDK_LWM(5);
        case 6: return IDK_LWM(6);
        default: return IDK_LWM(7);
    }
#undef IDK_LWM
}

}  // namespace

// Fixed-order sum of the residual partials: out[0] = sum (Ref - AB)^2, out[1] = sum Ref^2.
__global__ void resid_reduce_kernel(const double* __restrict__ part, int64_t count, double* __restrict__ out) {
    __shared__ double sd[32], sr[32];
    double d = 0.0, r = 0.0;
    for (int64_t e = threadIdx.x; e < count; e += blockDim.x) {
        d += part[2 * e];
        r += part[2 * e + 1];
    }
    d = warp_sum(d);
    r = warp_sum(r);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sd[wid] = d;
        sr[wid] = r;
    }
    __syncthreads();
    if (wid == 0) {
        d = lane < static_cast<int>(blockDim.x >> 5) ? sd[lane] : 0.0;
        r = lane < static_cast<int>(blockDim.x >> 5) ? sr[lane] : 0.0;
        d = warp_sum(d);
        r = warp_sum(r);
        if (lane == 0) {
            out[0] = d;
            out[1] = r;
        }
    }
}

// Pick BM = 16*WM (WM in 2..7) minimising padded rows over ceil(M/BM) tiles.
// Products with a short K (C * Z of approx / diagnostics: K = k <= 512 over thousands of
// rows) run a 16-trip main loop per tile: 64-row tiles keep more CTAs per SM to overlap the
// epilogues (diagnostics on cfg4: 6.51 ms with 112-row tiles, 5.29 ms with 64-row tiles).
int sketch_gemm_pick_wm(int M, int64_t K) {
    if (const char* e = getenv("IDK_GEMM_WM")) return atoi(e);  // tuning experiments
    if (K <= 512 && M >= 1024) return 4;
    int best = 7;
    int64_t best_pad = INT64_MAX;
    for (int wm = 7; wm >= 2; --wm) {
        const int bm = 16 * wm;
        const int64_t tiles = (M + bm - 1) / bm;
        const int64_t pad = tiles * bm - M + tiles * 4;  // small bias toward fewer tiles
        if (pad < best_pad) {
            best_pad = pad;
            best = wm;
        }
    }
    return best;
}

// Number of K splits: enough tiles for ~4 waves of 4 CTAs per SM (so the last
// partial wave costs little) while every split keeps >= 256 of K.  Measured
// on B200 (tools/time_cpqr.py): cfg4 5.82 -> 4.95 ms with 4 splits, cfg2 0.25 ->
// 0.095 ms, cfg5 1.47 -> 1.44 ms.  IDK_GEMM_SPLITS overrides (tuning only).
int sketch_gemm_pick_splits(int M, int64_t N, int64_t K, int num_sms) {
    if (const char* e = getenv("IDK_GEMM_SPLITS")) return atoi(e) > 0 ? atoi(e) : 1;
    const int wm = sketch_gemm_pick_wm(M);
    const int64_t tiles = ((M + 16 * wm - 1) / (16 * wm)) * ((N + kBN - 1) / kBN);
    int splits = 1;
    while (tiles * splits < 16LL * num_sms && K / (splits * 2) >= 256 && splits < 16) splits *= 2;
    // long K ranges take one more doubling while each split keeps >= 128 k-tiles:
    // more, shorter CTAs even out the wave tail (cfg4: 4 -> 8 splits, sketch
    // 4.35 -> 4.29 ms; cfg5's 4096-long K stays at 4, where 8 was slower;
    // profiles/sketch_padding_r02.txt)
    if (tiles * splits < 32LL * num_sms && K / (splits * 2) >= 2048 && splits < 16) splits *= 2;
    return splits;
}

// Y (M x N, ldc) = A (M x K, lda) * op(B); op(B) = B (K x N, ldb) or B^T (B is N x K, ldb).
// `partial` must hold splits * ldc * N doubles when splits > 1.
cudaError_t sketch_gemm(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans,
                        double* Y, int64_t ldc, int M, int64_t N, int64_t K, int splits,
                        double* partial, cudaStream_t stream) {
    if (M <= 0 || N <= 0) return cudaSuccess;
    const int wm = sketch_gemm_pick_wm(M, K);
    const bool vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    if (splits < 1) splits = 1;
    double* out = splits > 1 ? partial : Y;
    const int64_t split_stride = ldc * N;
    cudaError_t e = cudaErrorNotSupported;
    const char* te = getenv("IDK_GEMM_TMA");
    // TMA-fed kernel (sketch_tma.cu) for both layouts; same-box A/B against this
    // file's cp.async kernel: cfg4 29.4 -> 32.4 TFLOP/s, the dual (cfg5) 27.2 -> 30.3,
    // cfg2 19.2 -> 20.7.  IDK_GEMM_TMA=0 selects the cp.async kernel.
    const int tma = te ? atoi(te) : 1;
    if (tma != 0)
        e = sketch_gemm_tma(A, lda, B, ldb, b_trans, out, ldc, split_stride, M, N, K, splits, wm, stream);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = b_trans ? launch_nt<true>(wm, A, lda, B, ldb, out, ldc, split_stride, M, N, K, splits, vec16, stream)
                    : launch_nt<false>(wm, A, lda, B, ldb, out, ldc, split_stride, M, N, K, splits, vec16, stream);
    }
    if (e != cudaSuccess || splits == 1) return e;
    const int64_t total = static_cast<int64_t>(M) * N;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(partial, split_stride, splits, Y, M, N, ldc);
    return cudaGetLastError();
}

// Y block (M x N, ldc) = A * op(B) written to every f.y[g] (see
// splitk_reduce_fanout_kernel); same arithmetic as sketch_gemm with `splits`.
cudaError_t sketch_gemm_fanout(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans, const FanOut& f,
                               int64_t ldc, int M, int64_t N, int64_t K, int splits, double* partial,
                               cudaStream_t stream) {
    if (M <= 0 || N <= 0 || f.count <= 0) return cudaSuccess;
    if (f.count > kFanMax) return cudaErrorInvalidValue;
    const int64_t total = static_cast<int64_t>(M) * N;
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    if (splits <= 1) {
        cudaError_t e = sketch_gemm(A, lda, B, ldb, b_trans, f.y[0], ldc, M, N, K, 1, nullptr, stream);
        if (e != cudaSuccess || f.count == 1) return e;
        fanout_copy_kernel<<<blocks, 256, 0, stream>>>(f, M, N, ldc);
        return cudaGetLastError();
    }
    const int wm = sketch_gemm_pick_wm(M);
    const bool vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    const int64_t split_stride = ldc * N;
    cudaError_t e = cudaErrorNotSupported;
    const char* te = getenv("IDK_GEMM_TMA");
    if (!te || atoi(te) != 0)
        e = sketch_gemm_tma(A, lda, B, ldb, b_trans, partial, ldc, split_stride, M, N, K, splits, wm, stream);
    if (e == cudaErrorNotSupported) {
        cudaGetLastError();
        e = b_trans ? launch_nt<true>(wm, A, lda, B, ldb, partial, ldc, split_stride, M, N, K, splits, vec16, stream)
                    : launch_nt<false>(wm, A, lda, B, ldb, partial, ldc, split_stride, M, N, K, splits, vec16, stream);
    }
    if (e != cudaSuccess) return e;
    splitk_reduce_fanout_kernel<<<blocks, 256, 0, stream>>>(partial, split_stride, splits, f, M, N, ldc);
    return cudaGetLastError();
}

// Grouped sketch: Y_g = Omega_g * op(B_g) for g < grp.count, Omega_g at
// omega + g*grp.a_stride (ld = M), B_g = grp.b[g], Y_g = grp.y[g] (ld = ldc).
// One launch over every member (blockIdx.z = member * splits + split) so small
// sketches fill the GPU together; split-K partials (splits > 1) live at
// partial + (g*splits + s) * ldc*N and are reduced in the same fixed order as
// sketch_gemm, so a member's Y is bit-identical to its single launch with the
// same splits.
cudaError_t sketch_gemm_group(const double* omega, int64_t ldb, bool b_trans, const GemmGroup& grp, int64_t ldc,
                              int M, int64_t N, int64_t K, int splits, double* partial, cudaStream_t stream) {
    if (M <= 0 || N <= 0 || grp.count <= 0) return cudaSuccess;
    if (grp.count > kGemmGroupMax) return cudaErrorInvalidValue;
    const int wm = sketch_gemm_pick_wm(M);
    bool vec16 = (M % 2 == 0) && (ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(omega) & 15) == 0) &&
                 ((grp.a_stride % 2) == 0);
    for (int g = 0; g < grp.count; ++g) vec16 = vec16 && ((reinterpret_cast<uintptr_t>(grp.b[g]) & 15) == 0);
    if (splits < 1) splits = 1;
    const int64_t split_stride = ldc * N;
    GemmGroup g = grp;
    // The kernel addresses C as base + g*c_stride: with splits == 1 it writes Y_g
    // directly when the Y_g are equally spaced; otherwise it goes through partials.
    bool spaced = splits == 1;
    for (int t = 1; spaced && t < grp.count; ++t) spaced = grp.y[t] - grp.y[0] == t * (grp.y[1] - grp.y[0]);
    double* out;
    if (spaced) {
        out = grp.y[0];
        g.c_stride = grp.count > 1 ? grp.y[1] - grp.y[0] : 0;
    } else {
        if (!partial) return cudaErrorInvalidValue;
        out = partial;
        g.c_stride = split_stride * splits;
    }
    cudaError_t e = b_trans ? launch_nt<true>(wm, omega, M, nullptr, ldb, out, ldc, split_stride, M, N, K, splits,
                                              vec16, stream, &g)
                            : launch_nt<false>(wm, omega, M, nullptr, ldb, out, ldc, split_stride, M, N, K, splits,
                                               vec16, stream, &g);
    if (e != cudaSuccess || spaced) return e;
    const int64_t total = static_cast<int64_t>(M) * N;
    const int bx = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16 / grp.count + 1));
    splitk_reduce_group_kernel<<<dim3(bx, grp.count), 256, 0, stream>>>(partial, split_stride, splits,
                                                                       split_stride * splits, grp, M, N, ldc);
    return cudaGetLastError();
}

// Residual of a product: out2 = {||Ref - A*B||_F^2, ||Ref||_F^2} with A (M x K,
// lda) and B (K x N, ldb); Ref is M x N (ldr) or, with ref_trans, N x M.
// `part` needs resid_partials(M, N) doubles.
int64_t resid_partials(int M, int64_t N) {
    const int wm = sketch_gemm_pick_wm(M);
    const int64_t ctas = ((M + 16 * wm - 1) / (16 * wm)) * ((N + kBN - 1) / kBN);
    return ctas * 4 * 2;
}

cudaError_t gemm_residual(const double* A, int64_t lda, const double* B, int64_t ldb, int M, int64_t N, int64_t K,
                          const double* Ref, int64_t ldr, bool ref_trans, double* part, double* out2,
                          cudaStream_t stream) {
    const int wm = sketch_gemm_pick_wm(M, K);
    const bool vec16 = (lda % 2 == 0) && (ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                       ((reinterpret_cast<uintptr_t>(B) & 15) == 0);
    cudaError_t e;
    switch (wm) {
        case 2: e = launch_wm<2, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
        case 3: e = launch_wm<3, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
        case 4: e = launch_wm<4, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
        case 5: e = launch_wm<5, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
        case 6: e = launch_wm<6, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
        default: e = launch_wm<7, false>(A, lda, B, ldb, nullptr, 0, 0, M, N, K, 1, vec16, stream, Ref, ldr, ref_trans, part); break;
    }
    if (e != cudaSuccess) return e;
    resid_reduce_kernel<<<1, 1024, 0, stream>>>(part, resid_partials(M, N) / 2, out2);
    return cudaGetLastError();
}

// Omega (l x m, column-major, ld = l) from Philox4x32-10 keyed by seed.
}  // namespace idk

#include "rng.cuh"

namespace idk {
namespace {
__device__ __forceinline__ void omega_pairs(double* __restrict__ out, int64_t total, uint64_t seed) {
    const int64_t pairs = (total + 1) / 2;
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < pairs;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double c0, c1;
        philox_normal_pair(static_cast<uint64_t>(j), seed, c0, c1);
        out[2 * j] = c0;
        if (2 * j + 1 < total) out[2 * j + 1] = c1;
    }
}

__global__ void omega_philox_kernel(double* __restrict__ out, int64_t total, uint64_t seed) {
    omega_pairs(out, total, seed);
}

// One Omega per group member (blockIdx.y), member g at out + g*total.
__global__ void omega_philox_group_kernel(double* __restrict__ out, int64_t total, const GroupSeeds seeds) {
    omega_pairs(out + blockIdx.y * total, total, seeds.s[blockIdx.y]);
}
}  // namespace

cudaError_t omega_philox_group(double* out, int64_t l, int64_t m, const GroupSeeds& seeds, int count,
                               cudaStream_t stream) {
    const int64_t total = l * m;
    if (total <= 0 || count <= 0) return cudaSuccess;
    if (count > kGemmGroupMax) return cudaErrorInvalidValue;
    const int bx = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8 / count + 1));
    omega_philox_group_kernel<<<dim3(bx, count), 256, 0, stream>>>(out, total, seeds);
    return cudaGetLastError();
}

cudaError_t omega_philox(double* out, int64_t l, int64_t m, uint64_t seed, cudaStream_t stream) {
    const int64_t total = l * m;
    if (total <= 0) return cudaSuccess;
    const int blocks = static_cast<int>(std::min<int64_t>((total / 2 + 255) / 256 + 1, 148 * 8));
    omega_philox_kernel<<<blocks, 256, 0, stream>>>(out, total, seed);
    return cudaGetLastError();
}

}  // namespace idk
