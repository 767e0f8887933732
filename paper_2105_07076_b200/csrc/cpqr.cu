// cpqr.cu -- column-pivoted Householder QR (k steps) as one persistent,
// cooperatively launched kernel.
//
// Reference: qr_column_pivoted, /root/reference/proj/src/qr.cpp:42-126.
//
// Layout.  The pivoted matrix W (m x n, column-major, HBM/L2 resident; the
// sketch Y for RID, a copy of A for deterministic ID) is split into G
// contiguous column blocks, one per CTA.  Each CTA owns the live/anchor
// squared norms and the *position* of its columns in shared memory.
//
// Pivoting.  The reference physically swaps column `step` with the pivot
// (qr.cpp:79-86), so the tie rule "lowest current position with
// sqrt(live) >= (1-1e-14) sqrt(vmax)" (qr.cpp:66-78) is about positions, not
// column ids.  We never move data: every CTA replays the same transposition on
// its position table (the column at position `step` takes the pivot's old
// position), which reproduces the reference's order exactly.
//
// Per step, one grid barrier: every CTA
//   1. reads the pivot column (written by its owner in earlier steps),
//      builds the Householder reflector redundantly in shared memory
//      (qr.cpp:16-28; beta/tau/scale with unfused IEEE ops),
//   2. applies it to its own trailing columns (qr.cpp:31-38, 93-94),
//      downdates live norms and recomputes on cancellation exactly where the
//      reference does (live <= 1e-6 * anchor, qr.cpp:96-106),
//   3. publishes (local max, lowest qualifying position, column id); after
//      the barrier all CTAs reduce the G records identically.  When two CTAs'
//      maxima differ by < 1e-14 relative, a second exact pass decides the tie.
// Trailing update, organised for HBM bandwidth (the matrix does not fit on chip here):
//   * long columns (>= kCoopRows active rows): half a block (16 warps) streams one column
//     at a time -- the dot pass reads it from HBM with kUnroll independent loads per thread,
//     the axpy pass re-reads it from L2 (148 x 2 columns in flight fit) and writes it back,
//     so a step costs two HBM accesses per element instead of three; the two halves of a
//     block work on different columns, so one half's reduction barrier overlaps the other's
//     streaming;
//   * short columns: a warp per column, loads unrolled the same way.
// The owner of pivot s writes beta and the scaled reflector tail back into
// the pivot column at the start of step s+1, so W ends up holding exactly the
// reference's `work` matrix (R above the diagonal, reflectors below).
#include <climits>

#include "common.cuh"

namespace idk {

struct CpqrPub {
    double vmax;      // largest live norm among this CTA's candidates (-1: none)
    long long pos;    // lowest qualifying position (LLONG_MAX: none)
    long long col;    // column id at that position
    long long pad;
};

struct CpqrArgs {
    double* W;
    int64_t ldw;
    int m;
    int64_t n;
    int k;
    int cols_per_cta;
    long long* pos_out;   // n: final position of every column (inverse of perm)
    long long* pivots;    // k: pivot column id per step (== perm[0..k))
    double* taus;         // k
    CpqrPub* pub;         // 2 * G (double-buffered by step parity)
    CpqrPub* pub2;        // G (exact tie pass)
    unsigned* barrier;    // zeroed before launch
    double* xglobal;      // shared reflector (2 x ldx, by step parity) when m doubles do not fit in shared memory
    int64_t ldx;
    const double* Win;    // the matrix as the caller holds it (read once: norms + working copy into W), or W
    int64_t ldin;
};

constexpr int kCpqrThreads = 1024;  // 32 warps per SM: enough loads in flight to stream HBM
constexpr int kUnroll = 8;           // independent 8-byte loads per thread and loop trip
constexpr int kCoopRows = 2048;      // columns at least this long are streamed by half a block each
constexpr double kTieFactor = 1.0 - 1e-14;  // qr.cpp:71
constexpr double kRecompute = 1e-6;          // qr.cpp:100

namespace {

__device__ __forceinline__ double block_max(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    double t = lane < nw ? scratch[lane] : -1.0;
    return warp_max(t);
}

__device__ __forceinline__ long long block_min_ll(long long v, long long* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_min_ll(v);
    __syncthreads();
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    long long t = lane < nw ? scratch[lane] : LLONG_MAX;
    return warp_min_ll(t);
}

}  // namespace

__global__ void __launch_bounds__(kCpqrThreads) cpqr_persistent_kernel(CpqrArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int m = a.m;
    const int nc = a.cols_per_cta;
    // m doubles: pivot column -> reflector; in shared memory, or for tall
    // matrices (m > ~24k rows) this CTA's own L2-resident buffer
    // The reflector: in shared memory, or -- when m doubles do not fit -- ONE L2-resident copy
    // shared by all CTAs, double-buffered by step parity.  Every CTA builds the same values
    // and writes them (identical bits), and reads them only after its own writes, so the
    // copy needs no extra grid barrier; 148 private copies would take 148 x 8m bytes of the
    // L2 that the columns in flight need.
    double* xv = a.xglobal ? a.xglobal : sm;
    double* s_live = a.xglobal ? sm : xv + ((m + 1) & ~1);  // nc
    double* s_anchor = s_live + nc;        // nc
    long long* s_pos = reinterpret_cast<long long*>(s_anchor + nc);  // nc

    __shared__ double red_d[32];
    __shared__ double red_h[64];    // the two half-block reductions of the trailing update
    __shared__ long long red_l[32];
    __shared__ double s_scalar[3];  // tau, beta, scale
    __shared__ long long s_sel[2];  // pivot column, its position before the swap
    __shared__ long long s_col_at;  // scratch for the local arg-min

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int G = gridDim.x;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * nc;
    const int myn = static_cast<int>(max(static_cast<int64_t>(0), min(a.n - c0, static_cast<int64_t>(nc))));
    double* const W = a.W;
    const int64_t ldw = a.ldw;
    unsigned epoch = 0;

    // Few columns per CTA (tall matrices): every warp of the CTA works on one
    // column at a time (rows split over the whole block) instead of a warp per column.
    const bool coop = myn < nwarps;
    // ---- initial squared norms (qr.cpp:56-62); the same pass writes the working copy when the
    // caller's matrix is read in place (no separate copy of A before the factorisation) ----
    const bool copy_in = a.Win != W;
    if (coop) {
        for (int lc = 0; lc < myn; ++lc) {
            const double* src = a.Win + (c0 + lc) * a.ldin;
            double* dst = W + (c0 + lc) * ldw;
            double s = 0.0;
#pragma unroll 4
            for (int i = tid; i < m; i += blockDim.x) {
                const double v = ld_cg(src + i);
                if (copy_in) st_cg(dst + i, v);
                s += v * v;
            }
            s = block_sum(s, red_d);
            if (tid == 0) {
                s_live[lc] = s;
                s_anchor[lc] = s;
                s_pos[lc] = c0 + lc;
            }
        }
    }
    for (int lc = coop ? myn : warp; lc < myn; lc += nwarps) {
        const double* src = a.Win + (c0 + lc) * a.ldin;
        double* dst = W + (c0 + lc) * ldw;
        double ss[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i0 = lane; i0 < m; i0 += 128) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = i0 + 32 * u < m ? ld_cg(src + i0 + 32 * u) : 0.0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (copy_in && i0 + 32 * u < m) st_cg(dst + i0 + 32 * u, v[u]);
                ss[u] += v[u] * v[u];
            }
        }
        const double s = warp_sum((ss[0] + ss[1]) + (ss[2] + ss[3]));
        if (lane == 0) {
            s_live[lc] = s;
            s_anchor[lc] = s;
            s_pos[lc] = c0 + lc;
        }
    }
    __syncthreads();

    // Local candidate summary over columns at positions > after (qr.cpp:66-78).
    auto publish_local = [&](long long after, CpqrPub* slot) {
        double mx = -1.0;
        for (int lc = tid; lc < myn; lc += blockDim.x)
            if (s_pos[lc] > after) mx = fmax(mx, s_live[lc]);
        mx = block_max(mx, red_d);
        long long best = LLONG_MAX;
        if (mx >= 0.0) {
            const double thr = kTieFactor * sqrt(mx);
            for (int lc = tid; lc < myn; lc += blockDim.x)
                if (s_pos[lc] > after && sqrt(s_live[lc]) >= thr) best = min(best, s_pos[lc]);
        }
        best = block_min_ll(best, red_l);
        for (int lc = tid; lc < myn; lc += blockDim.x)
            if (s_pos[lc] == best) s_col_at = c0 + lc;
        __syncthreads();
        if (tid == 0) {
            CpqrPub p;
            p.vmax = mx;
            p.pos = best;
            p.col = best == LLONG_MAX ? -1 : s_col_at;
            p.pad = 0;
            __stcg(reinterpret_cast<double2*>(slot), make_double2(p.vmax, __longlong_as_double(p.pos)));
            __stcg(reinterpret_cast<double2*>(slot) + 1, make_double2(__longlong_as_double(p.col), 0.0));
        }
    };

    // Global selection from the G published records; identical in every CTA.
    auto select_global = [&](long long after, const CpqrPub* slots) {
        if (warp == 0) {
            double vmax = -1.0;
            for (int g = lane; g < G; g += 32) vmax = fmax(vmax, __ldcg(&slots[g].vmax));
            vmax = warp_max(vmax);
            const double thr = kTieFactor * sqrt(vmax);
            long long best = LLONG_MAX, best_col = -1;
            int ambiguous = 0;
            for (int g = lane; g < G; g += 32) {
                const double v = __ldcg(&slots[g].vmax);
                if (v >= 0.0 && sqrt(v) >= thr) {
                    if (v != vmax) ambiguous = 1;
                    const long long p = __ldcg(&slots[g].pos);
                    if (p < best) {
                        best = p;
                        best_col = __ldcg(&slots[g].col);
                    }
                }
            }
            ambiguous = __any_sync(0xffffffffu, ambiguous);
            const long long wbest = warp_min_ll(best);
            const unsigned who = __ballot_sync(0xffffffffu, best == wbest && best != LLONG_MAX);
            const long long wcol = __shfl_sync(0xffffffffu, best_col, who ? __ffs(who) - 1 : 0);
            if (lane == 0) {
                s_sel[0] = ambiguous ? -2 : wcol;
                s_sel[1] = wbest;
                red_d[0] = thr;
            }
        }
        __syncthreads();
        if (s_sel[0] == -2) {
            // Exact pass: lowest position with sqrt(live) >= the global threshold.
            const double thr = red_d[0];
            __syncthreads();
            long long best = LLONG_MAX;
            for (int lc = tid; lc < myn; lc += blockDim.x)
                if (s_pos[lc] > after && sqrt(s_live[lc]) >= thr) best = min(best, s_pos[lc]);
            best = block_min_ll(best, red_l);
            for (int lc = tid; lc < myn; lc += blockDim.x)
                if (s_pos[lc] == best) s_col_at = c0 + lc;
            __syncthreads();
            if (tid == 0) {
                __stcg(&a.pub2[blockIdx.x].pos, best);
                __stcg(&a.pub2[blockIdx.x].col, best == LLONG_MAX ? -1 : s_col_at);
            }
            grid_barrier(a.barrier, epoch);
            if (warp == 0) {
                long long b2 = LLONG_MAX, c2 = -1;
                for (int g = lane; g < G; g += 32) {
                    const long long p = __ldcg(&a.pub2[g].pos);
                    if (p < b2) {
                        b2 = p;
                        c2 = __ldcg(&a.pub2[g].col);
                    }
                }
                const long long wb = warp_min_ll(b2);
                const unsigned who = __ballot_sync(0xffffffffu, b2 == wb);
                const long long wc = __shfl_sync(0xffffffffu, c2, __ffs(who) - 1);
                if (lane == 0) {
                    s_sel[0] = wc;
                    s_sel[1] = wb;
                }
            }
            __syncthreads();
        }
    };

    publish_local(-1, a.pub + blockIdx.x);
    grid_barrier(a.barrier, epoch);
    select_global(-1, a.pub);

    long long prev_piv = -1;
    for (int s = 0; s < a.k; ++s) {
        const long long piv = s_sel[0], ppos = s_sel[1];
        const int len = m - s;
        const double* xvp = xv;  // the previous step's reflector
        if (a.xglobal) xv = a.xglobal + (s & 1) * a.ldx;

        // (0) write back the previous reflector into its column (owner only).
        if (prev_piv >= 0 && prev_piv >= c0 && prev_piv < c0 + myn) {
            double* col = W + prev_piv * ldw + (s - 1);
            for (int i = tid; i < len + 1; i += blockDim.x) __stcg(col + i, i == 0 ? s_scalar[1] : xvp[i]);
        }
        __syncthreads();

        // (1) pivot column -> reflector (qr.cpp:16-28).  The buffer is written once, with the
        // final values (a shared L2 copy is written by every CTA: no read-modify-write).
        const double* pcol = W + piv * ldw + s;
        double t = 0.0;
        for (int i = 1 + tid; i < len; i += blockDim.x) {
            const double v = ld_cg(pcol + i);
            t += v * v;
        }
        const double tail = block_sum(t, red_d);
        if (tid == 0) {
            const double alpha = ld_cg(pcol);
            double tau = 0.0, beta = alpha, scale = 1.0;
            if (len > 1 && tail != 0.0) {
                beta = -copysign(sqrt(add_rn(mul_rn(alpha, alpha), tail)), alpha);
                tau = (beta - alpha) / beta;
                scale = 1.0 / (alpha - beta);
            }
            s_scalar[0] = tau;
            s_scalar[1] = beta;
            s_scalar[2] = scale;
            if (blockIdx.x == 0) {
                a.taus[s] = tau;
                a.pivots[s] = piv;
            }
        }
        __syncthreads();
        const double tau = s_scalar[0];
        {
            const double scale = s_scalar[2];
            for (int i = tid; i < len; i += blockDim.x) {
                const double v = ld_cg(pcol + i);
                xv[i] = (tau != 0.0 && i > 0) ? mul_rn(v, scale) : v;
            }
        }
        // Replay the swap on positions (qr.cpp:79-86).
        for (int lc = tid; lc < myn; lc += blockDim.x) {
            if (c0 + lc == piv) s_pos[lc] = s;
            else if (s_pos[lc] == s) s_pos[lc] = ppos;
        }
        __syncthreads();

        // (2) trailing update + norm downdate (qr.cpp:93-106).
        if (coop || len >= kCoopRows) {
            // half a block per column, rows split over the half's 16 warps; the whole block per
            // column once two columns per SM no longer stay in L2 between their two passes
            // (2 x G columns x len x 8 bytes against ~48 MB of the 126 MB L2)
            const int P = (static_cast<double>(len) * 16.0 * G > 48e6) ? 1 : 2;
            const int H = blockDim.x / P, half = tid / H, ht = tid - half * H;
            const int hw = ht >> 5, hnw = H >> 5;
            double* hred = red_h + half * 32;
            auto half_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "r"(H) : "memory"); };
            auto half_sum = [&](double v) -> double {
                v = warp_sum(v);
                half_sync();  // the scratch of the previous reduction has been read
                if (lane == 0) hred[hw] = v;
                half_sync();
                double t = lane < hnw ? hred[lane] : 0.0;
                return warp_sum(t);
            };
            for (int lc = half; lc < myn; lc += P) {
                if (s_pos[lc] <= s) continue;  // uniform across the half
                double* col = W + (c0 + lc) * ldw + s;
                double head;
                if (tau != 0.0) {
                    double dd[kUnroll];
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) dd[u] = 0.0;
                    for (int i0 = 1 + ht; i0 < len; i0 += H * kUnroll) {
                        double yv[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int i = i0 + u * H;
                            yv[u] = i < len ? ld_cg(col + i) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int i = i0 + u * H;
                            if (i < len) dd[u] += xv[i] * yv[u];
                        }
                    }
                    double d = 0.0;
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) d += dd[u];
                    d = half_sum(d);
                    const double y0 = ld_cg(col);
                    const double w = mul_rn(add_rn(y0, d), tau);
                    head = sub_rn(y0, w);
                    half_sync();  // every thread of the half read y0 before it is overwritten
                    if (ht == 0) st_cg(col, head);
                    for (int i0 = 1 + ht; i0 < len; i0 += H * kUnroll) {  // second pass: L2 hits
                        double yv[kUnroll];
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int i = i0 + u * H;
                            yv[u] = i < len ? ld_cg(col + i) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < kUnroll; ++u) {
                            const int i = i0 + u * H;
                            if (i < len) st_cg(col + i, sub_rn(yv[u], mul_rn(w, xv[i])));
                        }
                    }
                } else {
                    head = ld_cg(col);
                }
                double lv = sub_rn(s_live[lc], mul_rn(head, head));
                if (lv < 0.0) lv = 0.0;
                if (lv <= mul_rn(kRecompute, s_anchor[lc])) {
                    half_sync();  // the updated rows are visible to the whole half
                    double f = 0.0;
                    for (int i = 1 + ht; i < len; i += H) {
                        const double v = ld_cg(col + i);
                        f += v * v;
                    }
                    f = half_sum(f);
                    lv = f;
                    if (ht == 0) s_anchor[lc] = f;
                }
                half_sync();  // s_live / s_anchor of this column have been read by every thread
                if (ht == 0) s_live[lc] = lv;
            }
        } else {
            for (int lc = warp; lc < myn; lc += nwarps) {
                if (s_pos[lc] <= s) continue;
                double* col = W + (c0 + lc) * ldw + s;
                double head;
                if (tau != 0.0) {
                    double dd[4] = {0.0, 0.0, 0.0, 0.0};
                    for (int i0 = 1 + lane; i0 < len; i0 += 128) {
                        double yv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) yv[u] = i0 + 32 * u < len ? ld_cg(col + i0 + 32 * u) : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i0 + 32 * u < len) dd[u] += xv[i0 + 32 * u] * yv[u];
                    }
                    const double d = warp_sum((dd[0] + dd[1]) + (dd[2] + dd[3]));
                    const double y0 = ld_cg(col);
                    const double w = mul_rn(add_rn(y0, d), tau);
                    head = sub_rn(y0, w);
                    __syncwarp();  // every lane read y0 before it is overwritten
                    if (lane == 0) st_cg(col, head);
                    for (int i0 = 1 + lane; i0 < len; i0 += 128) {
                        double yv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) yv[u] = i0 + 32 * u < len ? ld_cg(col + i0 + 32 * u) : 0.0;
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            if (i0 + 32 * u < len) st_cg(col + i0 + 32 * u, sub_rn(yv[u], mul_rn(w, xv[i0 + 32 * u])));
                    }
                } else {
                    head = ld_cg(col);
                }
                double lv = sub_rn(s_live[lc], mul_rn(head, head));
                if (lv < 0.0) lv = 0.0;
                if (lv <= mul_rn(kRecompute, s_anchor[lc])) {
                    __syncwarp();
                    double f = 0.0;
                    for (int i = 1 + lane; i < len; i += 32) {
                        const double v = ld_cg(col + i);
                        f += v * v;
                    }
                    f = warp_sum(f);
                    lv = f;
                    if (lane == 0) s_anchor[lc] = f;
                }
                if (lane == 0) s_live[lc] = lv;
            }
        }
        __syncthreads();
        prev_piv = piv;
        if (s + 1 == a.k) break;

        // (3) next pivot.
        CpqrPub* slots = a.pub + ((s + 1) & 1) * G;
        publish_local(s, slots + blockIdx.x);
        grid_barrier(a.barrier, epoch);
        select_global(s, slots);
    }

    // Final reflector write-back and positions.
    if (prev_piv >= c0 && prev_piv < c0 + myn) {
        const int s = a.k;
        double* col = W + prev_piv * ldw + (s - 1);
        const int len = m - (s - 1);
        for (int i = tid; i < len; i += blockDim.x) __stcg(col + i, i == 0 ? s_scalar[1] : xv[i]);
    }
    for (int lc = tid; lc < myn; lc += blockDim.x) a.pos_out[c0 + lc] = s_pos[lc];
}

// perm[pos[c]] = c
__global__ void invert_positions_kernel(const long long* __restrict__ pos, long long* __restrict__ perm,
                                        int64_t n) {
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < n;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
        perm[pos[c]] = c;
}

// R (k x n, position order; qr.cpp:119-123): R(i, j) = W(i, perm[j]) for i < min(j+1, k).
__global__ void extract_r_kernel(const double* __restrict__ W, int64_t ldw, const long long* __restrict__ perm,
                                 int k, int64_t n, double* __restrict__ R) {
    const int64_t total = static_cast<int64_t>(k) * n;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = e / k;
        const int i = static_cast<int>(e - j * k);
        R[e] = (i <= j) ? W[perm[j] * ldw + i] : 0.0;
    }
}

// Explicit Q (qr.cpp:109-117): column j of Q = H_0 ... H_{k-1} e_j, one CTA per column.
// 1024 threads and four independent loads per thread: a column of a tall matrix is
// streamed (from L2) once per reflector (100000 x 50, 50 steps: 10.5 -> see profiles).
__global__ void __launch_bounds__(1024) form_q_kernel(const double* __restrict__ W, int64_t ldw,
                                                      const long long* __restrict__ pivots,
                                                      const double* __restrict__ taus, int m, int k,
                                                      double* __restrict__ Q) {
    __shared__ double red[32];
    const int j = blockIdx.x;
    const int tid = threadIdx.x, T = blockDim.x;
    double* q = Q + static_cast<int64_t>(j) * m;
    for (int i = tid; i < m; i += T) q[i] = (i == j) ? 1.0 : 0.0;
    __syncthreads();
    for (int step = k - 1; step >= 0; --step) {
        if (step > j) continue;  // H_step leaves e_j (j < step) untouched
        const double tau = taus[step];
        if (tau == 0.0) continue;
        const double* v = W + pivots[step] * ldw + step;
        double* y = q + step;
        const int len = m - step;
        double dd[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i0 = 1 + tid; i0 < len; i0 += 4 * T) {
            double vv[4], yy[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * T;
                vv[u] = i < len ? v[i] : 0.0;
                yy[u] = i < len ? y[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) dd[u] += vv[u] * yy[u];
        }
        const double d = block_sum((dd[0] + dd[1]) + (dd[2] + dd[3]), red);
        const double w = mul_rn(add_rn(y[0], d), tau);
        __syncthreads();
        for (int i0 = tid; i0 < len; i0 += 4 * T) {
            double vv[4], yy[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * T;
                vv[u] = (i < len && i > 0) ? v[i] : 0.0;
                yy[u] = i < len ? y[i] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * T;
                if (i < len) y[i] = (i == 0) ? sub_rn(yy[u], w) : sub_rn(yy[u], mul_rn(w, vv[u]));
            }
        }
        __syncthreads();
    }
}

size_t cpqr_smem_bytes(int m, int cols_per_cta) {
    return sizeof(double) * static_cast<size_t>(((m + 1) & ~1) + 3 * cols_per_cta);
}

// The reflector buffer moves to global memory (L2) when m doubles plus the
// per-column state exceed the shared-memory budget; `xglobal` then needs
// 2 * cpqr_xglobal_ld(m) doubles (one copy shared by all CTAs, double-buffered).
int64_t cpqr_xglobal_ld(int m) { return (static_cast<int64_t>(m) + 31) & ~31LL; }

// Host launcher.  `ws_pub` must hold 3*G CpqrPub, `barrier` one unsigned.
cudaError_t cpqr_launch(double* W, int64_t ldw, int m, int64_t n, int k, long long* pos_out,
                        long long* pivots, double* taus, void* ws_pub, unsigned* barrier, int num_sms,
                        int max_ctas, cudaStream_t stream, double* xglobal, const double* Win, int64_t ldin) {
    // Block-distribute columns: G CTAs, each at most one per SM (co-residency).
    int64_t G = std::min<int64_t>(n, static_cast<int64_t>(max_ctas > 0 ? max_ctas : num_sms));
    int cols = static_cast<int>((n + G - 1) / G);
    G = (n + cols - 1) / cols;
    const bool xg = xglobal && cpqr_smem_bytes(m, cols) > 200 * 1024;
    const size_t smem = xg ? cpqr_smem_bytes(0, cols) : cpqr_smem_bytes(m, cols);
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(cpqr_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(barrier, 0, sizeof(unsigned), stream);
    if (e != cudaSuccess) return e;
    CpqrArgs args;
    args.W = W;
    args.ldw = ldw;
    args.m = m;
    args.n = n;
    args.k = k;
    args.cols_per_cta = cols;
    args.pos_out = pos_out;
    args.pivots = pivots;
    args.taus = taus;
    args.pub = static_cast<CpqrPub*>(ws_pub);
    args.pub2 = static_cast<CpqrPub*>(ws_pub) + 2 * G;
    args.barrier = barrier;
    args.xglobal = xg ? xglobal : nullptr;
    args.ldx = cpqr_xglobal_ld(m);
    args.Win = Win ? Win : W;
    args.ldin = Win ? ldin : ldw;
    void* params[] = {&args};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cpqr_persistent_kernel), dim3(static_cast<unsigned>(G)),
                                       dim3(kCpqrThreads), params, smem, stream);
}

cudaError_t cpqr_finish(const double* W, int64_t ldw, int m, int64_t n, int k, const long long* pos,
                        const long long* pivots, const double* taus, long long* perm, double* R, double* Q,
                        cudaStream_t stream) {
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 4));
    if (perm) {
        invert_positions_kernel<<<blocks, 256, 0, stream>>>(pos, perm, n);
        if (R) {
            const int64_t total = static_cast<int64_t>(k) * n;
            extract_r_kernel<<<static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 8)), 256, 0, stream>>>(
                W, ldw, perm, k, n, R);
        }
    }
    if (Q) form_q_kernel<<<k, 1024, 0, stream>>>(W, ldw, pivots, taus, m, k, Q);
    return cudaGetLastError();
}

}  // namespace idk
