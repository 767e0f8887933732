// sketch_tma.cu -- Y = Omega * A on the DMMA pipe with TMA-fed operands.
//
// Same product and the same fixed-order split-K as sketch_gemm.cu (the
// reference's matmul(Omega, A), matrix.cpp:28-48), but the operand tiles are
// brought in by the Tensor Memory Accelerator: one thread issues
// cp.async.bulk.tensor loads of 16 x 16 (Omega) and 16 x 64 (A) boxes into a
// kStagesT-deep ring (2: measured equal to 3 and 4 CTAs fit per SM) with an mbarrier per stage, so the compute warps do no
// address arithmetic for the loads at all.  Boxes are 128-byte rows with the
// hardware 128B swizzle (16-byte chunk c of row r stored at c ^ (r mod 8)),
// which keeps the DMMA fragment loads free of bank conflicts without padding.
// Out-of-range rows/columns/k are zero-filled by the TMA.  kNT reads A
// transposed (the id_auto dual, id.cpp:85): its 64-column tile is four
// 16 x 16 boxes laid out like Omega's.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace idk {

namespace {

constexpr int kBNT = 64;
constexpr int kBKT = 16;
constexpr int kThreadsT = 128;
#ifndef IDK_TMA_STAGES
#define IDK_TMA_STAGES 2
#endif
constexpr int kStagesT = IDK_TMA_STAGES;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            su32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(su32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_init_t(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_t(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TMA_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TMA_WAIT_%=;\n}" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}

template <int WM>
struct SmemT {
    static constexpr int BM = 16 * WM;
    static constexpr int A_ELEMS = BM * kBKT;    // WM boxes of 16 k-rows x 16 m
    static constexpr int B_ELEMS = kBNT * kBKT;  // 64 n-rows x 16 k
    static constexpr int STAGE = A_ELEMS + B_ELEMS;
    static constexpr size_t BYTES = sizeof(double) * STAGE * kStagesT + 1024;  // + alignment slack
};

// One CTA tile with WMA <= WM live 16-row boxes (the shared-memory layout is
// WM's): the last M tile of cfg4 (l = 272 in 3 x 96 rows) has a box of pure
// padding, which is neither loaded nor multiplied.
template <int WMA, int WM, bool kNT>
__device__ __forceinline__ void sketch_tile(const CUtensorMap& tmA, const CUtensorMap& tmB, double* __restrict__ C,
                                            int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K,
                                            int64_t k_per_split, double* smem, uint64_t* full) {
    using S = SmemT<WM>;
    constexpr int BM = S::BM;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int m0 = blockIdx.x * BM;
    const int n0 = static_cast<int>(blockIdx.y) * kBNT;
    const int64_t kbeg = static_cast<int64_t>(blockIdx.z) * k_per_split;
    const int64_t kend = min(K, kbeg + k_per_split);
    const int ktiles = kend > kbeg ? static_cast<int>((kend - kbeg + kBKT - 1) / kBKT) : 0;
    C += static_cast<int64_t>(blockIdx.z) * split_stride;

    constexpr unsigned kStageBytes = static_cast<unsigned>(sizeof(double) * (WMA * 256 + S::B_ELEMS));
    auto issue = [&](int kt) {  // thread 0 only
        const int st = kt % kStagesT;
        double* As = smem + st * S::STAGE;
        double* Bs = As + S::A_ELEMS;
        const int k0 = static_cast<int>(kbeg) + kt * kBKT;
        mbar_expect_tx_t(&full[st], kStageBytes);
#pragma unroll
        for (int g = 0; g < WMA; ++g) tma_load_2d(As + g * 256, &tmA, m0 + 16 * g, k0, &full[st]);
        if constexpr (kNT) {
#pragma unroll
            for (int b = 0; b < kBNT / 16; ++b) tma_load_2d(Bs + b * 256, &tmB, n0 + 16 * b, k0, &full[st]);
        } else {
            tma_load_2d(Bs, &tmB, k0, n0, &full[st]);
        }
    };

    double acc[WMA][4][2];
#pragma unroll
    for (int a = 0; a < WMA; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    if (tid == 0)
        for (int s = 0; s < kStagesT - 1 && s < ktiles; ++s) issue(s);

    // Warp rows are interleaved by 16-row box: warp wm owns rows 16*tm + 8*wm + fr
    // (tm < WM), so every fragment address is a compile-time offset plus one of
    // two per-lane swizzle values.  In a 128B-swizzled box, element (row r, k)
    // sits at k*16 + (((r>>1) ^ (k&7)) << 1 | (r&1)); with r = 8*wm + fr and
    // k = 4*kq + fc the swizzle term is ((fr>>1) ^ fc) ^ 4*(wm ^ kq), i.e. a
    // lane constant X0 or X1 = X0 ^ 8 (in doubles) picked by the parity of kq.
    const int fr = lane >> 2, fc = lane & 3;
    const int x0 = (((fr >> 1) ^ fc) << 1) + (fr & 1) + fc * 16;
    const int ya = wm ? (x0 ^ 8) : x0, yb = wm ? x0 : (x0 ^ 8);  // kq even / odd
    // B (non-transposed): row j = n index (j & 7 == fr), k index = 4*kq + fc:
    // chunk ((2*kq + (fc>>1)) ^ fr), element fc & 1
    const int bz = ((fc >> 1) ^ (fr & 1)), bf6 = fr & 6;
    const int brow = (wn * 32 + fr) * 16 + (fc & 1);
    // B (transposed, four 16x16 boxes): like A with row = n index within the box
    const int xb0 = (((fr >> 1) ^ fc) << 1) + (fr & 1) + fc * 16;
    for (int kt = 0; kt < ktiles; ++kt) {
        const int st = kt % kStagesT;
        mbar_wait_t(&full[st], static_cast<unsigned>((kt / kStagesT) & 1));
        __syncthreads();  // every warp is done with stage (kt - 1) % kStagesT: refill it
        if (tid == 0 && kt + kStagesT - 1 < ktiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(kt + kStagesT - 1);
        }
        const double* As = smem + st * S::STAGE;
        const double* Bs = As + S::A_ELEMS;
#pragma unroll
        for (int kq = 0; kq < kBKT / 4; ++kq) {
            double af[WMA], bf[4];
            const int ay = (kq & 1) ? yb : ya;
#pragma unroll
            for (int tm = 0; tm < WMA; ++tm) af[tm] = As[tm * 256 + kq * 64 + ay];
#pragma unroll
            for (int tn = 0; tn < 4; ++tn) {
                if constexpr (kNT) {
                    // n index j = wn*32 + tn*8 + fr: box (j >> 4) = 2*wn + (tn >> 1), row within box 8*(tn&1) + fr
                    const int xr = (tn & 1) ? (xb0 ^ 8) : xb0;
                    const int xk = (kq & 1) ? (xr ^ 8) : xr;
                    bf[tn] = Bs[(2 * wn + (tn >> 1)) * 256 + kq * 64 + xk];
                } else {
                    bf[tn] = Bs[brow + tn * 128 + ((((2 * kq) ^ bf6) | bz) << 1)];
                }
            }
#pragma unroll
            for (int tm = 0; tm < WMA; ++tm)
#pragma unroll
                for (int tn = 0; tn < 4; ++tn) dmma(acc[tm][tn], af[tm], bf[tn]);
        }
    }

#pragma unroll
    for (int tm = 0; tm < WMA; ++tm) {
        const int i = m0 + 16 * tm + 8 * wm + fr;
        if (i >= M) continue;
#pragma unroll
        for (int tn = 0; tn < 4; ++tn) {
            const int64_t j = n0 + wn * 32 + tn * 8 + 2 * fc;
            if (j < N) C[j * ldc + i] = acc[tm][tn][0];
            if (j + 1 < N) C[(j + 1) * ldc + i] = acc[tm][tn][1];
        }
    }
}

template <int WM, bool kNT>
__global__ void __launch_bounds__(kThreadsT)
sketch_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  double* __restrict__ C, int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K,
                  int64_t k_per_split) {
    extern __shared__ __align__(1024) double smem_raw[];
    double* smem = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStagesT];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesT; ++s) mbar_init_t(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    __syncthreads();
    if constexpr (WM > 2) {
        if (static_cast<int>(blockIdx.x) * 16 * WM + 16 * (WM - 1) >= M) {  // last tile, last box all padding
            sketch_tile<WM - 1, WM, kNT>(tmA, tmB, C, ldc, split_stride, M, N, K, k_per_split, smem, full);
            return;
        }
    }
    sketch_tile<WM, WM, kNT>(tmA, tmB, C, ldc, split_stride, M, N, K, k_per_split, smem, full);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
    }
    return fn;
}

bool make_map(CUtensorMap* tm, const double* base, uint64_t inner, uint64_t outer, int64_t ld, unsigned box_outer) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
    const cuuint32_t box[2] = {16, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int WM, bool kNT>
cudaError_t launch_t(const CUtensorMap& ta, const CUtensorMap& tb, double* C, int64_t ldc, int64_t split_stride,
                     int M, int64_t N, int64_t K, int splits, cudaStream_t stream) {
    using S = SmemT<WM>;
    auto kern = sketch_tma_kernel<WM, kNT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::BYTES));
    if (e != cudaSuccess) return e;
    int64_t kps = (K + splits - 1) / splits;
    kps = ((kps + kBKT - 1) / kBKT) * kBKT;  // split ranges on box boundaries: no box straddles two splits
    dim3 grid((M + S::BM - 1) / S::BM, static_cast<unsigned>((N + kBNT - 1) / kBNT), splits);
    kern<<<grid, kThreadsT, S::BYTES, stream>>>(ta, tb, C, ldc, split_stride, M, N, K, kps);
    return cudaGetLastError();
}

}  // namespace

// Y (or the split partials) = Omega * A through TMA; cudaErrorNotSupported when
// the operands do not meet TMA's rules (16-byte aligned bases and leading
// dimensions, K < 2^31) or the driver entry point is missing.
cudaError_t sketch_gemm_tma(const double* A, int64_t lda, const double* B, int64_t ldb, bool b_trans, double* out,
                            int64_t ldc, int64_t split_stride, int M, int64_t N, int64_t K, int splits, int wm,
                            cudaStream_t stream) {
    if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) || (lda & 1) || (ldb & 1) ||
        K >= (1LL << 31) - 64 || N >= (1LL << 31) || wm < 2 || wm > 7)
        return cudaErrorNotSupported;
    CUtensorMap ta, tb;
    if (!make_map(&ta, A, static_cast<uint64_t>(M), static_cast<uint64_t>(K), lda, 16) ||
        !(b_trans ? make_map(&tb, B, static_cast<uint64_t>(N), static_cast<uint64_t>(K), ldb, 16)
                  : make_map(&tb, B, static_cast<uint64_t>(K), static_cast<uint64_t>(N), ldb, kBNT)))
        return cudaErrorNotSupported;
#define IDK_TMA_CASE(W)                                                                          \
    case W:                                                                                      \
        return b_trans ? launch_t<W, true>(ta, tb, out, ldc, split_stride, M, N, K, splits, stream) \
                       : launch_t<W, false>(ta, tb, out, ldc, split_stride, M, N, K, splits, stream);
    switch (wm) {
        IDK_TMA_CASE(2)
        IDK_TMA_CASE(3)
        IDK_TMA_CASE(4)
        IDK_TMA_CASE(5)
        IDK_TMA_CASE(6)
        default: return b_trans ? launch_t<7, true>(ta, tb, out, ldc, split_stride, M, N, K, splits, stream)
                                : launch_t<7, false>(ta, tb, out, ldc, split_stride, M, N, K, splits, stream);
    }
#undef IDK_TMA_CASE
}

}  // namespace idk
