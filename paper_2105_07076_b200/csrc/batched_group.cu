// batched_group.cu -- many small IDs (BASELINE cfg3): a group of S threads per column.
//
// Same algorithm as batched_fast.cu (the reference's CPQR qr.cpp:42-126, the
// triangular solve solve.cpp:23-53 and the gather matrix.cpp:121-130 per
// matrix).  batched_fast.cu gives a column to one thread (64 rows in 128
// registers, 8 warps per SM): every phase of a pivot step is a chain of ~60
// dependent FP64 instructions with two warps per scheduler to hide it, and ncu
// shows the step bound by those chains and the three CTA barriers
// (profiles/batched_tuning_r01.txt: issue active 22 %, FP64 pipe 18 %).
//
// Here S threads share a column (row pairs {2p, 2p+1}, p = q + S r', in registers):
//   * S x the warps per SM (16 or 32) and chains S x shorter: dot, axpy and the
//     column's sum of squares are M/S FMAs each plus log2 S shuffles; the pivot
//     column moves through shared memory in 16-byte pieces;
//   * retired rows are zero: when step s finishes, R(s, j) = y_s - w goes to a
//     k x n shared-memory table and the column's row s becomes 0.  So the pivot
//     publishes its registers as they are, every loop runs over all M/S rows
//     without predicates or step specialisation, and sum_i y_i^2 is the
//     column's alpha^2 + tail (the reflector needs only that sum);
//   * only the elected pivot forms its reflector (sqrt, and the two divisions
//     side by side in two lanes), while the other columns already run their dot
//     against the raw pivot column: the column and the reflector scalars are
//     released through two mbarriers (the pivot's lanes arrive; nobody waits
//     for the whole CTA), so a step has the election's two CTA barriers only;
//   * the next matrix streams into shared memory by TMA bulk copies while the
//     current one is factored, as in batched_fast.cu;
//   * Z: R11 is gathered from the table, then a column-oriented back
//     substitution inside the group (the solved entry is broadcast by a
//     shuffle, each lane updates its own rows).
// The pivot rule is exact (lowest position among sqrt(live) >= (1-1e-14)
// sqrt(max)); positions replay the reference's swaps.  Results match the
// reference within rounding (identical columns, ||dZ||/||Z|| <= 1e-10);
// batched.cu remains the bit-identical kernel.
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace idk {

namespace {

constexpr int kGroupCols = 256;  // columns per matrix (one group each)

__device__ __forceinline__ unsigned s32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void g_mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void g_mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void g_mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void g_mbar_wait(uint64_t* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "GWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra GDONE_%=;\n"
        "bra GWAIT_%=;\n"
        "GDONE_%=:\n"
        "}\n" ::"r"(s32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void g_bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(smem)),
                 "l"(gmem), "r"(bytes), "r"(s32(bar))
                 : "memory");
}

// Warp max of non-negative doubles (-1 = none) via two 32-bit redux.sync.
__device__ __forceinline__ double g_wmax_nonneg(double v) {
    const bool has = v >= 0.0;
    const unsigned long long b = has ? static_cast<unsigned long long>(__double_as_longlong(v)) + 1ull : 0ull;
    const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0u);
    const unsigned long long r = (static_cast<unsigned long long>(hi) << 32) | lo;
    return r == 0ull ? -1.0 : __longlong_as_double(static_cast<long long>(r - 1ull));
}

__device__ __noinline__ bool g_tie_band(double v, double vmax) { return sqrt(v) >= (1.0 - 1e-14) * sqrt(vmax); }

__device__ __forceinline__ bool g_tie_ok(double v, double vmax) {  // qr.cpp:71-73, exact
    if (v == vmax) return true;
    if (!(v >= vmax * (1.0 - 4e-14))) return false;
    return g_tie_band(v, vmax);
}

// Sum over the S lanes of a group; every lane gets the same bits (the xor
// butterfly adds the same pairs in every lane).  All 32 lanes take part.
template <int S>
__device__ __forceinline__ double g_sum(double v) {
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// 16-byte shared-memory load the compiler may not hoist or merge
__device__ __forceinline__ double2 g_lds2(const double* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(s32(p)));
    return v;
}

// Column-oriented back substitution T = R11^-1 R12 (solve.cpp:43-51) on the
// group's registers (lane q holds entries q + S r), entry L down to 0: the
// owner lane forms x_L, a shuffle hands it to the group, every lane updates
// its own entries above L.
template <int S, int KZ, int KM, int L>
__device__ __forceinline__ void solve_col(double (&z)[KZ], const double* r11, const double* rinv, int k, int q, int gb) {
    if constexpr (L >= 0) {
        if (L < k) {
            constexpr int rl = L / S, ql = L % S;
            double xl = z[rl] * rinv[L];
            xl = __shfl_sync(0xffffffffu, xl, gb + ql);
            if (q == ql) z[rl] = xl;
#pragma unroll
            for (int r = 0; r * S < L; ++r) {
                const int i = q + S * r;
                if (i < L) z[r] = fma(-r11[L * KM + i], xl, z[r]);
            }
        }
        solve_col<S, KZ, KM, L - 1>(z, r11, rinv, k, q, gb);
    }
}

}  // namespace

#define IDK_REP32(M) \
    M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) \
    M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)

// The reflector a column would produce as the next pivot (qr.cpp:16-28) from
// alpha and sumsq = alpha^2 + tail: rsqrt and one reciprocal instead of a square
// root and two divisions (tau = (beta - alpha) / beta = 1 + |alpha| / sqrt(sumsq),
// scale = 1 / (alpha - beta) = sign(alpha) / (|alpha| + sqrt(sumsq))); within a few
// ulps of the reference's values.
__device__ __forceinline__ void reflector_fast(double pa, double sumsq, int len, double& tau, double& beta,
                                               double& scale) {
    tau = 0.0;
    beta = pa;
    scale = 1.0;
    if (len > 1 && sumsq != mul_rn(pa, pa)) {
        const double rs = rsqrt(sumsq);
        double sq = mul_rn(sumsq, rs);
        sq = fma(fma(-sq, sq, sumsq), 0.5 * rs, sq);  // one Newton step: sqrt(sumsq) to within an ulp
        const double ap = fabs(pa);
        beta = -copysign(sq, pa);
        tau = fma(ap, rs, 1.0);
        scale = copysign(__drcp_rn(ap + sq), pa);
    }
}

template <int M, int S, int KM>
__global__ void __launch_bounds__(kGroupCols * S, 1)
batched_group_kernel(const double* __restrict__ A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                     long long* __restrict__ cols_out, double* __restrict__ Z, double* __restrict__ C,
                     int* __restrict__ status) {
    constexpr int R = M / S;              // rows per thread: pairs {2p, 2p+1}, p = q + S r'
    constexpr int P = R / 2;              // row pairs per thread
    constexpr int T = kGroupCols * S;     // threads
    constexpr int NW = T / 32;            // warps (16 or 32)
    constexpr int NC = kGroupCols;
    constexpr int LDS = M + 2;            // 16-byte aligned column stride of the TMA stage
    constexpr int KZ = KM / S;            // Z entries per thread
    static_assert(M % (2 * S) == 0 && KM % S == 0 && NW <= 32, "layout");
    extern __shared__ __align__(128) double sm[];
    double* stage = sm;                                      // n * LDS (TMA target)
    double* colbuf = stage + static_cast<size_t>(n) * LDS;   // 2 x M: the pivot column as its registers stand
    double* r11 = colbuf + 2 * M;                            // KM x KM, column-major
    double* r12 = r11 + KM * KM;                             // KM x NC: R(s, j) of every column, by step
    __shared__ uint64_t bar_in, bar_col, bar_sc;
    __shared__ double red_d[NW];
    __shared__ unsigned red_u[NW];
    __shared__ double s_sc[2][2];  // tau, scale of the step's reflector (by step parity)
    __shared__ int s_piv[KM];
    __shared__ int s_ppos[2];
    __shared__ double s_rinv[KM];  // 1 / R11(i,i) for the Z solve

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c = tid / S, q = tid % S;
    const bool mine = c < n;
    if (tid == 0) {
        g_mbar_init(&bar_in, 1);
        g_mbar_init(&bar_col, S);
        g_mbar_init(&bar_sc, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto prefetch = [&](int64_t b) {
        if (wid == 0 && b < batch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of stage
            if (lane == 0) g_mbar_expect_tx(&bar_in, static_cast<unsigned>(n) * m * 8u);
            __syncwarp();
            const double* src = A + b * stride;
            for (int j = lane; j < n; j += 32)
                g_bulk_g2s(stage + static_cast<size_t>(j) * LDS, src + j * lda, m * 8u, &bar_in);
        }
    };

    unsigned in_phase = 0, st_phase = 0;
    prefetch(blockIdx.x);
    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        g_mbar_wait(&bar_in, in_phase);
        in_phase ^= 1u;
        double y[R];
#pragma unroll
        for (int rp = 0; rp < P; ++rp) {
            const int i = 2 * (q + S * rp);  // m is even: a pair is inside or outside the matrix
            double2 v = make_double2(0.0, 0.0);
            if (mine && i < m) v = *reinterpret_cast<const double2*>(stage + c * LDS + i);
            y[2 * rp] = v.x;
            y[2 * rp + 1] = v.y;
        }
        __syncthreads();
        prefetch(b + gridDim.x);  // next matrix streams in while this one is factored

        // norms (qr.cpp:56-62): live = sum of squares; pa = row 0 (the first alpha)
        double live, anchor, pa, pt;
        {
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
            for (int r = 0; r < R; r += 4) {
                t0 = fma(y[r], y[r], t0);
                t1 = fma(y[r + 1], y[r + 1], t1);
                t2 = fma(y[r + 2], y[r + 2], t2);
                t3 = fma(y[r + 3], y[r + 3], t3);
            }
            pt = g_sum<S>((t0 + t1) + (t2 + t3));
            pa = g_sum<S>(q == 0 ? y[0] : 0.0);
            live = anchor = pt;
        }
        int pos = c;

        for (int s = 0; s < k; ++s) {
            // ---- pivot: max live, then the lowest qualifying position (qr.cpp:66-78) ----
            const bool cand = mine && pos >= s;
            double mx = g_wmax_nonneg(cand ? live : -1.0);
            if (lane == 0) red_d[wid] = mx;
            __syncthreads();
            mx = g_wmax_nonneg(lane < NW ? red_d[lane] : -1.0);
            const unsigned key = (cand && g_tie_ok(live, mx)) ? static_cast<unsigned>(pos) : 0xffffffffu;
            const unsigned wmin = __reduce_min_sync(0xffffffffu, key);
            if (lane == 0) red_u[wid] = wmin;
            __syncthreads();
            const unsigned best = __reduce_min_sync(0xffffffffu, lane < NW ? red_u[lane] : 0xffffffffu);
            // no candidate (NaN norms): the column at position s pivots, so the step's barriers complete
            const unsigned bsel = best == 0xffffffffu ? static_cast<unsigned>(s) : best;
            const bool piv = mine && static_cast<unsigned>(pos) == bsel;
            const int par = s & 1;
            double* buf = colbuf + par * M;
            const int qs = (s >> 1) % S;  // lane of row s
            if (piv) {
                // Row s (alpha = pa) leaves the registers, so they hold exactly the column
                // below the diagonal and zeros elsewhere: publish them as they stand.
                switch (s) {
#define IDK_ZERO_CASE(sv)                                                        \
    case sv:                                                                     \
        if constexpr (sv < KM) {                                                 \
            if (q == (sv / 2) % S) y[(2 * ((sv / 2) / S) + (sv & 1)) % R] = 0.0; \
        }                                                                        \
        break;
                    IDK_REP32(IDK_ZERO_CASE)
#undef IDK_ZERO_CASE
                    default:
                        break;
                }
#pragma unroll
                for (int rp = 0; rp < P; ++rp)
                    *reinterpret_cast<double2*>(buf + 2 * (q + S * rp)) = make_double2(y[2 * rp], y[2 * rp + 1]);
                if (q == 0) {
                    s_piv[s] = c;
                    s_ppos[par] = pos;
                }
                g_mbar_arrive(&bar_col);
                // reflector (qr.cpp:16-28) from alpha and alpha^2 + tail = pt
                double tau, beta, scale;
                reflector_fast(pa, pt, m - s, tau, beta, scale);
                if (q == 0) {
                    s_sc[par][0] = tau;
                    s_sc[par][1] = scale;
                    r11[s * KM + s] = beta;  // tau == 0: beta = alpha
                    g_mbar_arrive(&bar_sc);
                }
            }
            g_mbar_wait(&bar_col, st_phase);
            if (mine && !piv && pos == s) pos = s_ppos[par];  // the column at position s takes the pivot's place
            if (piv) pos = s;
            const bool upd = mine && !piv && pos > s;

            // ---- dot with the raw pivot column (zeros on rows <= s: no predicates) ----
            double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
            for (int rp = 0; rp < P; rp += 2) {
                const double2 va = g_lds2(buf + 2 * (q + S * rp));
                const double2 vb = g_lds2(buf + 2 * (q + S * (rp + 1)));
                d0 = fma(va.x, y[2 * rp], d0);
                d1 = fma(va.y, y[2 * rp + 1], d1);
                d2 = fma(vb.x, y[2 * rp + 2], d2);
                d3 = fma(vb.y, y[2 * rp + 3], d3);
            }
            const double d = g_sum<S>((d0 + d1) + (d2 + d3));
            g_mbar_wait(&bar_sc, st_phase);
            st_phase ^= 1u;
            const double tau = s_sc[par][0], scale = s_sc[par][1];
            // row s of a live column is the alpha it kept from the last step: w = tau (y_s + scale p^T y);
            // columns that do not take part keep w = 0
            const double ys = pa;
            const double w = (upd && tau != 0.0) ? mul_rn(fma(scale, d, ys), tau) : 0.0;
            const double ws = mul_rn(w, scale);
            // ---- axpy (qr.cpp:93-95) over every row: v = 0 on the retired ones ----
#pragma unroll
            for (int rp = 0; rp < P; rp += 2) {
                const double2 va = g_lds2(buf + 2 * (q + S * rp));
                const double2 vb = g_lds2(buf + 2 * (q + S * (rp + 1)));
                y[2 * rp] = fma(-ws, va.x, y[2 * rp]);
                y[2 * rp + 1] = fma(-ws, va.y, y[2 * rp + 1]);
                y[2 * rp + 2] = fma(-ws, vb.x, y[2 * rp + 2]);
                y[2 * rp + 3] = fma(-ws, vb.y, y[2 * rp + 3]);
            }
            // R(s, j) = y_s - w goes to the table, row s becomes 0; yb = the register that holds row s + 1
            const double head = ys - w;
            if (upd && q == qs) r12[s * NC + c] = head;
            double yb = 0.0;
            switch (s) {
#define IDK_ROW_CASE(sv)                                                                  \
    case sv:                                                                              \
        if constexpr (sv < KM) {                                                          \
            if (upd && q == (sv / 2) % S) y[(2 * ((sv / 2) / S) + (sv & 1)) % R] = 0.0;   \
            yb = y[(2 * (((sv + 1) / 2) / S) + ((sv + 1) & 1)) % R];                      \
        }                                                                                 \
        break;
                IDK_REP32(IDK_ROW_CASE)
#undef IDK_ROW_CASE
                default:
                    break;
            }
            // ---- the next step's alpha (row s + 1) and alpha^2 + tail (every row: retired ones are 0) ----
            double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
#pragma unroll
            for (int r = 0; r < R; r += 4) {
                t0 = fma(y[r], y[r], t0);
                t1 = fma(y[r + 1], y[r + 1], t1);
                t2 = fma(y[r + 2], y[r + 2], t2);
                t3 = fma(y[r + 3], y[r + 3], t3);
            }
            const double na = g_sum<S>(q == ((s + 1) >> 1) % S ? yb : 0.0);
            const double nt = g_sum<S>((t0 + t1) + (t2 + t3));
            if (upd) {
                double lv = sub_rn(live, mul_rn(head, head));
                if (lv < 0.0) lv = 0.0;
                if (lv <= mul_rn(1e-6, anchor)) {  // qr.cpp:100-104
                    lv = nt;
                    anchor = lv;
                }
                live = lv;
                pa = na;
                pt = nt;
            }
        }
        __syncthreads();
        // R11(i, s) = R(i, pivot column of step s), i < s; the diagonal is already in place
        for (int e = tid; e < k * k; e += T) {
            const int sc = e / k, i = e - sc * k;
            if (i < sc) r11[sc * KM + i] = r12[i * NC + s_piv[sc]];
        }
        if (tid < k) s_rinv[tid] = 1.0 / r11[tid * KM + tid];
        __syncthreads();

        // ---- T = R11^-1 R12 per column (solve.cpp:43-51): column-oriented back
        // substitution inside the group, Z written from registers ----
        {
            double z[KZ];
#pragma unroll
            for (int r = 0; r < KZ; ++r) {
                const int i = q + S * r;
                z[r] = (i < k) ? r12[i * NC + c] : 0.0;
            }
            solve_col<S, KZ, KM, KM - 1>(z, r11, s_rinv, k, q, lane & ~(S - 1));
            if (mine) {
                double* zc = Z + b * static_cast<int64_t>(k) * n + static_cast<int64_t>(c) * k;
#pragma unroll
                for (int r = 0; r < KZ; ++r) {
                    const int i = q + S * r;
                    if (i < k) zc[i] = pos < k ? (i == pos ? 1.0 : 0.0) : z[r];
                }
            }
        }
        if (tid == 0) {
            int bad = -1;
            for (int i = 0; i < k; ++i)
                if (fabs(r11[i * KM + i]) <= 1e-300) {
                    bad = i;
                    break;
                }
            status[b] = bad;
        }
        long long* cb = cols_out + b * k;
        for (int j = tid; j < k; j += T) cb[j] = s_piv[j];
        if (C) {
            const double* Ab = A + b * stride;
            double* Cb = C + b * static_cast<int64_t>(m) * k;
            for (int e = tid; e < m * k; e += T) {
                const int j = e / m, i = e - j * m;
                Cb[e] = Ab[static_cast<int64_t>(s_piv[j]) * lda + i];
            }
        }
        __syncthreads();
    }
}

size_t batched_group_smem_bytes(int n, int k) {
    const int M = 64, KM = k <= 16 ? 16 : 32;
    return sizeof(double) * (static_cast<size_t>(n) * (M + 2) + 2 * M + KM * KM + KM * kGroupCols);
}

bool batched_group_ok(const double* A, int64_t lda, int64_t stride, int m, int n, int k, size_t smem_optin) {
    return m <= 64 && m % 2 == 0 && n <= kGroupCols && k <= 32 && lda % 2 == 0 && stride % 2 == 0 &&
           (reinterpret_cast<uintptr_t>(A) & 15) == 0 && batched_group_smem_bytes(n, k) <= smem_optin;
}

template <int S, int KM>
static cudaError_t launch_group(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                                long long* cols, double* Z, double* C, int* status, unsigned grid, size_t smem,
                                cudaStream_t stream) {
    auto kern = batched_group_kernel<64, S, KM>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, kGroupCols * S, smem, stream>>>(A, lda, stride, batch, m, n, k, cols, Z, C, status);
    return cudaGetLastError();
}

cudaError_t batched_id_group(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                             long long* cols, double* Z, double* C, int* status, int num_sms, int group,
                             cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    const size_t smem = batched_group_smem_bytes(n, k);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(batch, num_sms));
    (void)group;  // two threads per column
    if (k <= 16) return launch_group<2, 16>(A, lda, stride, batch, m, n, k, cols, Z, C, status, grid, smem, stream);
    return launch_group<2, 32>(A, lda, stride, batch, m, n, k, cols, Z, C, status, grid, smem, stream);
}

}  // namespace idk
