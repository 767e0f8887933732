// batched_duo.cu -- many small IDs (BASELINE cfg3) with two matrices in flight per SM.
//
// Same algorithm and arithmetic as batched_fast.cu (the reference's CPQR
// qr.cpp:42-126, the triangular solve solve.cpp:23-53 and the gather
// matrix.cpp:121-130 per matrix; FMA, exact pivot rule, reference swaps on
// positions), re-laid out so that two CTAs share an SM:
//   * batched_fast keeps a column's 64 rows in registers (255 registers, one
//     256-thread CTA per SM) and spends most of a pivot step waiting at its
//     three barriers -- 8 warps cannot hide the serial pivot phase;
//   * here a thread keeps rows 32..63 of its column in registers and rows
//     0..31 in shared memory (odd stride: conflict-free), 128 registers, so
//     two 256-thread CTAs are resident per SM and one's pivot phase overlaps
//     the other's column updates.  The top rows are the shared-memory ones:
//     they retire first (rows < s are R), so the shared-memory traffic of a
//     step shrinks as the factorisation advances;
//   * no TMA staging: a CTA loads its next matrix directly (the other CTA
//     computes meanwhile), which frees the 132 KB staging buffer.
#include <climits>

#include "common.cuh"

namespace idk {

namespace {

constexpr int kDuoThreads = 256;  // one thread per column, n <= 256
constexpr int kM = 64;            // rows (padded with zeros)
constexpr int kMS = 32;           // rows 0..31 in shared memory
constexpr int kMR = 32;           // rows 32..63 in registers
constexpr int kLD = kMS + 1;      // shared-memory column stride (odd: conflict-free per lane)

__device__ __forceinline__ double wmax_nn(double v) {  // warp max of non-negative doubles (-1 = none)
    const bool has = v >= 0.0;
    const unsigned long long b = has ? static_cast<unsigned long long>(__double_as_longlong(v)) + 1ull : 0ull;
    const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0u);
    const unsigned long long r = (static_cast<unsigned long long>(hi) << 32) | lo;
    return r == 0ull ? -1.0 : __longlong_as_double(static_cast<long long>(r - 1ull));
}

__device__ __noinline__ bool duo_tie_band(double v, double vmax) { return sqrt(v) >= (1.0 - 1e-14) * sqrt(vmax); }

__device__ __forceinline__ bool duo_tie_ok(double v, double vmax) {  // qr.cpp:71-73, exact
    if (v == vmax) return true;
    if (!(v >= vmax * (1.0 - 4e-14))) return false;
    return duo_tie_band(v, vmax);
}

__device__ __forceinline__ void duo_reflector(double pa, double pt, int len, double& tau, double& beta, double& scale) {
    tau = 0.0;
    beta = pa;
    scale = 1.0;
    if (len > 1 && pt != 0.0) {  // qr.cpp:16-28
        beta = -copysign(sqrt(add_rn(mul_rn(pa, pa), pt)), pa);
        tau = (beta - pa) / beta;
        scale = 1.0 / (pa - beta);
    }
}

__device__ __forceinline__ double lds(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
    return v;
}

// Trailing update of one non-pivot column at compile-time step S (< 32):
// v = [1; scale * p] with p the pivot column below row S (colbuf), rows S+1..31
// of this column in shared memory (my), rows 32..63 in registers (y).
__device__ __forceinline__ void sts(double* p, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(p))), "d"(v));
}

// Trailing update of one non-pivot column at compile-time step S (< 32):
// v = [1; scale * p] with p the pivot column below row S (colbuf), rows S+1..31
// of this column in shared memory (my), rows 32..63 in registers (y).  Shared
// rows are read 4 at a time through volatile loads so the compiler cannot
// hoist a whole column into registers (128 registers per thread: two CTAs per SM).
template <int S>
__device__ __forceinline__ void duo_step(double* __restrict__ my, double (&y)[kMR], const double* __restrict__ pcol,
                                         double tau, double scale, double& live, double& anchor, double& pa,
                                         double& pt, int m, double& rt, double& rb, double& rs) {
    const double ys = lds(my + S);
    double head = ys;
    if (tau != 0.0) {
        double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
        for (int i0 = S + 1; i0 < kMS; i0 += 4) {
            double p[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < kMS) {
                    p[u] = lds(pcol + i0 + u);
                    x[u] = lds(my + i0 + u);
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < kMS) {
                    if (u & 1) d1 = fma(p[u], x[u], d1);
                    else d0 = fma(p[u], x[u], d0);
                }
        }
#pragma unroll
        for (int r0 = 0; r0 < kMR; r0 += 4) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = lds(pcol + kMS + r0 + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (u & 1) d3 = fma(v[u], y[r0 + u], d3);
                else d2 = fma(v[u], y[r0 + u], d2);
            }
        }
        const double w = mul_rn(fma(scale, (d0 + d1) + (d2 + d3), ys), tau);
        const double ws = mul_rn(w, scale);
        head = ys - w;
        sts(my + S, head);
#pragma unroll
        for (int i0 = S + 1; i0 < kMS; i0 += 4) {
            double p[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < kMS) {
                    p[u] = lds(pcol + i0 + u);
                    x[u] = lds(my + i0 + u);
                }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u < kMS) sts(my + i0 + u, fma(-ws, p[u], x[u]));
        }
#pragma unroll
        for (int r0 = 0; r0 < kMR; r0 += 4) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = lds(pcol + kMS + r0 + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) y[r0 + u] = fma(-ws, v[u], y[r0 + u]);
        }
    }
    // next-step reflector inputs: alpha = row S+1, tail = rows S+2..63
    double t0 = 0.0, t1 = 0.0;
#pragma unroll
    for (int i0 = S + 2; i0 < kMS; i0 += 4) {
        double x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < kMS) x[u] = lds(my + i0 + u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u < kMS) {
                if (u & 1) t1 = fma(x[u], x[u], t1);
                else t0 = fma(x[u], x[u], t0);
            }
    }
    constexpr int r_first = S + 2 - kMS > 0 ? S + 2 - kMS : 0;
#pragma unroll
    for (int r = r_first; r < kMR; ++r) {
        if (r & 1) t1 = fma(y[r], y[r], t1);
        else t0 = fma(y[r], y[r], t0);
    }
    if constexpr (S + 1 < kMS) pa = lds(my + S + 1);
    else pa = y[S + 1 - kMS];
    pt = t0 + t1;
    double lv = sub_rn(live, mul_rn(head, head));
    if (lv < 0.0) lv = 0.0;
    if (lv <= mul_rn(1e-6, anchor)) {  // qr.cpp:100-104
        lv = fma(pa, pa, pt);
        anchor = lv;
    }
    live = lv;
    duo_reflector(pa, pt, m - (S + 1), rt, rb, rs);
}

#define IDK_DUO_REP32(M) \
    M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) \
    M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)

}  // namespace

template <int KM>
__global__ void __launch_bounds__(kDuoThreads, 2)
batched_duo_kernel(const double* __restrict__ A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                   long long* __restrict__ cols_out, double* __restrict__ Z, double* __restrict__ C,
                   int* __restrict__ status) {
    extern __shared__ __align__(16) double sm[];
    double* rows = sm;                                                    // n * kLD: rows 0..31 of every column
    double* colbuf = rows + ((static_cast<size_t>(n) * kLD + 1) & ~size_t(1));  // kM: the pivot column
    double* r11 = colbuf + kM;                                            // KM x KM, column-major
    __shared__ double red_d[8];
    __shared__ unsigned red_u[8];
    __shared__ double s_sc[3];
    __shared__ int s_piv[KM];
    __shared__ int s_ppos;
    __shared__ double s_rinv[KM];

    const int c = threadIdx.x, lane = c & 31, wid = c >> 5;
    const bool mine = c < n;
    double* my = rows + static_cast<size_t>(mine ? c : 0) * kLD;

    for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
        // ---- load: rows 0..31 -> shared memory, rows 32..63 -> registers ----
        const double* src = A + b * stride + static_cast<int64_t>(c) * lda;
        double y[kMR];
#pragma unroll
        for (int r = 0; r < kMR; ++r) y[r] = (mine && kMS + r < m) ? __ldg(src + kMS + r) : 0.0;
        double live, anchor, pa, pt;
        {  // rows 0..31 straight into shared memory; norms (qr.cpp:56-62) and the first reflector's inputs
            double s0 = 0.0, s1 = 0.0;
            pa = 0.0;
#pragma unroll
            for (int i = 0; i < kMS; ++i) {
                const double v = (mine && i < m) ? __ldg(src + i) : 0.0;
                if (mine) my[i] = v;
                if (i == 0) pa = v;
                else if (i & 1) s1 = fma(v, v, s1);
                else s0 = fma(v, v, s0);
            }
#pragma unroll
            for (int r = 0; r < kMR; ++r) {
                if (r & 1) s1 = fma(y[r], y[r], s1);
                else s0 = fma(y[r], y[r], s0);
            }
            pt = s0 + s1;
            live = anchor = fma(pa, pa, pt);
        }
        double rt, rb, rs;
        duo_reflector(pa, pt, m, rt, rb, rs);
        int pos = c;

        for (int s = 0; s < k; ++s) {
            // ---- pivot: max live, then the lowest qualifying position (qr.cpp:66-78) ----
            const bool cand = mine && pos >= s;
            double mx = wmax_nn(cand ? live : -1.0);
            if (lane == 0) red_d[wid] = mx;
            __syncthreads();
            mx = wmax_nn(lane < kDuoThreads / 32 ? red_d[lane] : -1.0);
            const unsigned key = (cand && duo_tie_ok(live, mx)) ? static_cast<unsigned>(pos) : 0xffffffffu;
            const unsigned wmin = __reduce_min_sync(0xffffffffu, key);
            if (lane == 0) red_u[wid] = wmin;
            __syncthreads();
            const unsigned best = __reduce_min_sync(0xffffffffu, lane < kDuoThreads / 32 ? red_u[lane] : 0xffffffffu);
            const bool piv = mine && static_cast<unsigned>(pos) == best;
            if (piv) {  // publish the pivot column and its reflector (qr.cpp:16-28)
#pragma unroll
                for (int i = 0; i < kMS; ++i) colbuf[i] = my[i];
                double2* cb2 = reinterpret_cast<double2*>(colbuf + kMS);
#pragma unroll
                for (int r = 0; r < kMR; r += 2) cb2[r >> 1] = make_double2(y[r], y[r + 1]);
                s_sc[0] = rt;
                s_sc[1] = rb;
                s_sc[2] = rs;
                s_piv[s] = c;
                s_ppos = pos;
                r11[s * KM + s] = rt != 0.0 ? rb : pa;
            }
            __syncthreads();
            const double tau = s_sc[0], scale = s_sc[2];
            if (mine && !piv && pos == s) pos = s_ppos;  // the column at position s takes the pivot's place
            if (piv) pos = s;
            if (c < s) r11[s * KM + c] = colbuf[c];  // R(0..s-1, s)
            if (mine && !piv && pos > s) {
                switch (s) {
#define IDK_DUO_CASE(r) \
    case r:             \
        if constexpr (r < KM) duo_step<(r < KM ? r : 0)>(my, y, colbuf, tau, scale, live, anchor, pa, pt, m, rt, rb, rs); \
        break;
                    IDK_DUO_REP32(IDK_DUO_CASE)
#undef IDK_DUO_CASE
                    default:
                        break;
                }
            }
        }
        if (c < k) s_rinv[c] = 1.0 / r11[c * KM + c];
        __syncthreads();

        // ---- T = R11^-1 R12 per column (solve.cpp:43-51), rows 0..k-1 from shared memory ----
        if (mine) {
            double x[KM];
#pragma unroll
            for (int i = 0; i < KM; ++i) x[i] = i < k ? my[i] : 0.0;
            if (pos >= k) {
#pragma unroll
                for (int i = KM - 1; i >= 0; --i) {
                    if (i < k) {
                        double acc = x[i];
#pragma unroll
                        for (int l = i + 1; l < KM; ++l)
                            if (l < k) acc = fma(-r11[l * KM + i], x[l], acc);
                        x[i] = acc * s_rinv[i];
                    }
                }
            }
            double* zc = Z + b * static_cast<int64_t>(k) * n + static_cast<int64_t>(c) * k;
#pragma unroll
            for (int i = 0; i < KM; ++i)
                if (i < k) zc[i] = pos < k ? (i == pos ? 1.0 : 0.0) : x[i];
        }
        if (c == 0) {
            int bad = -1;
            for (int i = 0; i < k; ++i)
                if (fabs(r11[i * KM + i]) <= 1e-300) {
                    bad = i;
                    break;
                }
            status[b] = bad;
        }
        __syncthreads();
        long long* cb = cols_out + b * k;
        for (int j = c; j < k; j += kDuoThreads) cb[j] = s_piv[j];
        if (C) {
            const double* Ab = A + b * stride;
            double* Cb = C + b * static_cast<int64_t>(m) * k;
            for (int e = c; e < m * k; e += kDuoThreads) {
                const int j = e / m, i = e - j * m;
                Cb[e] = Ab[static_cast<int64_t>(s_piv[j]) * lda + i];
            }
        }
        __syncthreads();
    }
}

size_t batched_duo_smem_bytes(int n, int k) {
    const int KM = k <= 16 ? 16 : 32;
    return sizeof(double) * (((static_cast<size_t>(n) * kLD + 1) & ~size_t(1)) + kM + static_cast<size_t>(KM) * KM);
}

bool batched_duo_ok(const double* A, int64_t lda, int64_t stride, int m, int n, int k) {
    (void)A;
    (void)lda;
    (void)stride;
    return m <= kM && n <= kDuoThreads && k <= 32 && k <= m && 2 * batched_duo_smem_bytes(n, k) <= 220 * 1024;
}

cudaError_t batched_id_duo(const double* A, int64_t lda, int64_t stride, int64_t batch, int m, int n, int k,
                           long long* cols, double* Z, double* C, int* status, int num_sms, cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    const size_t smem = batched_duo_smem_bytes(n, k);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(batch, 2LL * num_sms));
    if (k <= 16) {
        auto kern = batched_duo_kernel<16>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<grid, kDuoThreads, smem, stream>>>(A, lda, stride, batch, m, n, k, cols, Z, C, status);
    } else {
        auto kern = batched_duo_kernel<32>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        kern<<<grid, kDuoThreads, smem, stream>>>(A, lda, stride, batch, m, n, k, cols, Z, C, status);
    }
    return cudaGetLastError();
}

}  // namespace idk
