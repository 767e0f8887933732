// cpqr_resident.cu -- column-pivoted Householder QR with the matrix resident on chip.
//
// Reference: qr_column_pivoted, /root/reference/proj/src/qr.cpp:42-126 (same
// reflector convention, norm downdate and recompute rule, and tie rule as
// cpqr.cu, which remains the fallback for shapes that do not fit on chip).
//
// Why.  Each pivot step needs a global argmax before the next reflector
// exists, so CPQR is a chain of k dependent steps.  Streaming the trailing
// matrix through L2 every step (cpqr.cu) costs one L2 round trip per column
// per step; here the matrix is loaded once, kept in registers (the rows that
// stay active longest) and shared memory (the rows retired first), and written
// back once at the end.
//
// Layout.  CTA g owns columns [g*nc, (g+1)*nc).  Each column is handled by a
// group of S consecutive threads; thread (column lc, segment q) owns rows
//   registers : i = l0 + q + S*r,  r < R        (rows l0 .. m-1)
//   shared    : i = q + S*r',      i < l0       (rows 0 .. l0-1, stride lds)
// so rows retire evenly across the group as the step advances.
//
// Exchange.  After its trailing update every CTA publishes one record (local
// max live norm, lowest qualifying position, column id) *and that candidate
// column's active rows*.  After one barrier every CTA reduces the G records
// identically and copies the winner's published column into shared memory:
// the next reflector is then built redundantly in every CTA with no second
// round trip.  Two exchange policies share the code:
//   kCluster = true : one thread-block cluster (<= 16 CTAs), records in shared
//                     memory read through DSMEM, barrier.cluster per step;
//   kCluster = false: one CTA per SM, records in global memory (L2), a
//                     monotonic-counter grid barrier per step.
#include <climits>
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace idk {

struct CpqrRec {
    double vmax;    // largest live norm among this CTA's candidates (-1: none)
    long long pos;  // lowest qualifying position (LLONG_MAX: none)
    long long col;  // its column id
    double tau;     // the candidate's reflector, built before the exchange
    double beta;    //   (qr.cpp:16-28 on its active rows)
    double scale;
};

struct ResidentArgs {
    double* W;
    int64_t ldw;
    int m;
    int64_t n;
    int k;
    int nc;   // columns per CTA
    int l0;   // rows [0, l0) in shared memory, [l0, m) in registers
    int lds;  // shared-memory stride of the l0 rows
    long long* pos_out;
    long long* pivots;
    double* taus;
    // grid-exchange buffers (global); unused in cluster mode
    CpqrRec* rec;     // [2][G]
    double* colbuf;   // [2][G][m]
    CpqrRec* rec2;    // [G]
    double* colbuf2;  // [G][m]
    unsigned* barrier;
    long long* trace;  // optional: %globaltimer at 8 phase marks per step, every CTA
};

namespace {

constexpr double kRecomp = 1e-6;      // qr.cpp:100

template <int S>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (S == 32) {
        return 0xffffffffu;
    } else {
        const unsigned lane = threadIdx.x & 31u;
        return ((1u << S) - 1u) << (lane & ~static_cast<unsigned>(S - 1));
    }
}

template <int S>
__device__ __forceinline__ double group_sum(double v) {
    const unsigned mask = group_mask<S>();
#pragma unroll
    for (int o = S / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
}

template <int R>
constexpr int max_threads_for() {
    return R >= 32 ? 512 : (R >= 16 ? 640 : 768);
}

__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_rec_cg(CpqrRec* p, const CpqrRec& r) {
    double2* d = reinterpret_cast<double2*>(p);
    __stcg(d, make_double2(r.vmax, __longlong_as_double(r.pos)));
    __stcg(d + 1, make_double2(__longlong_as_double(r.col), r.tau));
    __stcg(d + 2, make_double2(r.beta, r.scale));
}

__device__ __forceinline__ CpqrRec ld_rec_cg(const CpqrRec* p) {
    const double2* d = reinterpret_cast<const double2*>(p);
    const double2 a = __ldcg(d), b = __ldcg(d + 1), c = __ldcg(d + 2);
    CpqrRec r;
    r.vmax = a.x;
    r.pos = __double_as_longlong(a.y);
    r.col = __double_as_longlong(b.x);
    r.tau = b.y;
    r.beta = c.x;
    r.scale = c.y;
    return r;
}

// sqrt(v) >= (1 - 1e-14) * sqrt(vmax) (qr.cpp:71-73) evaluated exactly, with
// the sqrt only inside the 4e-14 band where the answer is not obvious.
__device__ __forceinline__ bool qualifies(double v, double vmax) {
    if (v == vmax) return true;
    if (!(v >= vmax * (1.0 - 4e-14))) return false;
    return sqrt(v) >= (1.0 - 1e-14) * sqrt(vmax);
}

// Warp max of non-negative doubles (or -1 = none) via two 32-bit redux.sync.
__device__ __forceinline__ double warp_max_nonneg(double v) {
    const bool has = v >= 0.0;
    const unsigned long long b = has ? static_cast<unsigned long long>(__double_as_longlong(v)) + 1ull : 0ull;
    const unsigned hi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(b >> 32) == hi ? static_cast<unsigned>(b) : 0u);
    const unsigned long long r = (static_cast<unsigned long long>(hi) << 32) | lo;
    return r == 0ull ? -1.0 : __longlong_as_double(static_cast<long long>(r - 1ull));
}

// Reflector scalars from alpha = x[0] and tail = sum x[1..]^2 (qr.cpp:16-28).
__device__ __forceinline__ void reflector(double alpha, double tail, int len, double& tau, double& beta,
                                          double& scale) {
    tau = 0.0;
    beta = alpha;
    scale = 1.0;
    if (len > 1 && tail != 0.0) {
        beta = -copysign(sqrt(add_rn(mul_rn(alpha, alpha), tail)), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
    }
}

}  // namespace

#define IDK_REP32(M) \
    M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) \
    M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)

// xv holds the reflector at offset kGuard, with kGuard zeros in front and
// zeros after the active length: a retired row (i < s) or a padding row
// (i >= m) then reads v = 0, so the row loops need no predicates and every
// lane of a warp takes the same path (the start row depends only on s).
constexpr int kGuard = 32;

template <int S, int R, bool kCluster>
__global__ void __launch_bounds__(max_threads_for<R>())
cpqr_resident_kernel(ResidentArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int m = a.m, nc = a.nc, l0 = a.l0, lds = a.lds;
    const int span = max(m, l0 + R * S);
    const int xlen = ((kGuard + span + S + 1) + 1) & ~1;
    double* xbuf = sm;
    double* xv = xbuf + kGuard;
    double* rows = xbuf + xlen;                               // nc * lds
    double* s_live = rows + static_cast<size_t>(nc) * lds;    // nc
    double* s_anchor = s_live + nc;                           // nc
    long long* s_pos = reinterpret_cast<long long*>(s_anchor + nc);  // nc (positions < 2^31)
    const int mpad = (m + 1) & ~1;
    double* ccol = reinterpret_cast<double*>(s_pos + nc);     // cluster: [2][mpad] + [mpad]

    __shared__ double red_d[32];
    __shared__ long long red_l[32];
    __shared__ double s_sc[3];      // tau, beta, scale of the current pivot
    __shared__ long long s_sel[3];  // pivot column, its position before the swap, winning CTA
    __shared__ double s_cand[3];    // candidate reflector: tau, beta, scale
    __shared__ CpqrRec s_rec[3];    // cluster: own records [2] + tie pass

    const int tid = threadIdx.x, T = blockDim.x;
    const int lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    const int lc = tid / S, q = tid % S;
    const int G = gridDim.x;
    const int me = kCluster ? static_cast<int>(cg::this_cluster().block_rank()) : blockIdx.x;
    const int64_t c0 = static_cast<int64_t>(me) * nc;
    const int myn = static_cast<int>(max(0LL, min(static_cast<long long>(a.n - c0), static_cast<long long>(nc))));
    const bool active = lc < myn;
    const int64_t col = c0 + lc;
    double* const W = a.W;
    const int nsr = l0 / S;  // l0 is a multiple of S
    double* myrows = rows + static_cast<size_t>(lc < nc ? lc : 0) * lds;
    const int gbase = lane & ~(S - 1);
    unsigned epoch = 0;
    // This thread's share of its column's next-reflector inputs: alpha = the
    // entry at the next step's row, tail = sum of squares below it.
    double p_alpha = 0.0, p_tail = 0.0;

    auto trace = [&](int s, int ph) {
        if (a.trace != nullptr && tid == 0) a.trace[(static_cast<size_t>(me) * (a.k + 1) + s) * 8 + ph] = globaltimer();
    };

    auto barrier_all = [&]() {
        if constexpr (kCluster) {
            cg::this_cluster().sync();
        } else {
            grid_barrier(a.barrier, epoch);
        }
    };

    for (int i = tid; i < xlen; i += T) xbuf[i] = 0.0;

    // ---- load (the only read of W) and initial norms (qr.cpp:56-62) ----
    double yr[R];
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = l0 + q + S * r;
        yr[r] = (active && i < m) ? W[col * a.ldw + i] : 0.0;
        part = fma(yr[r], yr[r], part);
        if (i == 0) p_alpha = yr[r];
        else p_tail = fma(yr[r], yr[r], p_tail);
    }
    for (int r = 0; r < nsr; ++r) {
        const int i = q + S * r;
        const double v = active ? W[col * a.ldw + i] : 0.0;
        if (lc < nc) myrows[i] = v;
        part = fma(v, v, part);
        if (i == 0) p_alpha = v;
        else p_tail = fma(v, v, p_tail);
    }
    part = group_sum<S>(part);
    if (active && q == 0) {
        s_live[lc] = part;
        s_anchor[lc] = part;
        s_pos[lc] = col;
    }

    // CTA argmax (qr.cpp:66-78 over this CTA's columns): the max live norm,
    // then the lowest position that qualifies against it; 32-bit redux.sync
    // per warp and one __syncthreads per pass.  Returns the position
    // (INT_MAX: none); the group whose position matches is the candidate.
    auto local_max = [&](bool cand, double lv) -> double {
        const double mx = warp_max_nonneg(cand ? lv : -1.0);
        if (lane == 0) red_d[wid] = mx;
        __syncthreads();
        return warp_max_nonneg(lane < nw ? red_d[lane] : -1.0);
    };
    auto local_pick = [&](bool cand, double lv, long long pos, double vmax, int& winlc) -> int {
        const unsigned key = (cand && qualifies(lv, vmax)) ? static_cast<unsigned>(pos) : 0xffffffffu;
        const unsigned wm = __reduce_min_sync(0xffffffffu, key);
        const unsigned wl = __reduce_min_sync(0xffffffffu, (key == wm) ? static_cast<unsigned>(lc) : 0xffffffffu);
        if (lane == 0) red_l[wid] = static_cast<long long>((static_cast<unsigned long long>(wm) << 32) | wl);
        __syncthreads();
        const unsigned long long mine = lane < nw ? static_cast<unsigned long long>(red_l[lane]) : ~0ull;
        const unsigned best = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(mine >> 32));
        winlc = static_cast<int>(__reduce_min_sync(
            0xffffffffu, static_cast<unsigned>(mine >> 32) == best ? static_cast<unsigned>(mine) : 0xffffffffu));
        return best == 0xffffffffu ? INT_MAX : static_cast<int>(best);
    };

    // Candidate column (local index winlc) -> exchange slot rows first..m-1:
    // its group stores the register rows and turns its (alpha, tail) partials
    // into the next reflector (qr.cpp:16-28); every thread copies a share of
    // its shared-memory rows.
    auto push_candidate = [&](int winlc, int first, double* dst, double pa, double pt) {
        if (winlc >= nc) return;
        if (lc == winlc) {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = l0 + q + S * r;
                if (i >= first && i < m) dst[i - first] = yr[r];
            }
            const double al = group_sum<S>(pa);
            const double tl = group_sum<S>(pt);
            if (q == 0) {
                double tau, beta, scale;
                reflector(al, tl, m - first, tau, beta, scale);
                s_cand[0] = tau;
                s_cand[1] = beta;
                s_cand[2] = scale;
                red_l[31] = c0 + winlc;
            }
        }
        const double* cr = rows + static_cast<size_t>(winlc) * lds;
        for (int i = first + tid; i < l0; i += T) dst[i - first] = cr[i];
    };

    auto write_record = [&](int slot, double mx, int winpos) {
        const bool have = winpos != INT_MAX;
        CpqrRec rc;
        rc.vmax = mx;
        rc.pos = have ? winpos : LLONG_MAX;
        rc.col = have ? red_l[31] : -1;
        rc.tau = have ? s_cand[0] : 0.0;
        rc.beta = have ? s_cand[1] : 0.0;
        rc.scale = have ? s_cand[2] : 1.0;
        if constexpr (kCluster) {
            s_rec[slot] = rc;
        } else {
            st_rec_cg(slot == 2 ? a.rec2 + me : a.rec + static_cast<size_t>(slot) * G + me, rc);
        }
    };

    auto rec_of = [&](int slot, int g) -> CpqrRec {
        if constexpr (kCluster) {
            return *cg::this_cluster().map_shared_rank(&s_rec[slot], g);
        } else {
            return ld_rec_cg(slot == 2 ? a.rec2 + g : a.rec + static_cast<size_t>(slot) * G + g);
        }
    };

    auto col_of = [&](int slot, int g) -> const double* {
        if constexpr (kCluster) {
            return cg::this_cluster().map_shared_rank(ccol + slot * mpad, g);
        } else {
            return slot == 2 ? a.colbuf2 + static_cast<size_t>(g) * m : a.colbuf + (static_cast<size_t>(slot) * G + g) * m;
        }
    };

    auto cand_slot = [&](int slot) -> double* {
        return kCluster ? (ccol + slot * mpad) : (slot == 2 ? a.colbuf2 + static_cast<size_t>(me) * m
                                                            : a.colbuf + (static_cast<size_t>(slot) * G + me) * m);
    };

    // After the barrier warp 0 alone reduces the G records (identical in
    // every CTA) and posts the winner; then all threads copy its column into
    // xv, already scaled by the winner's reflector.
    constexpr int kRecPerLane = kCluster ? 1 : 5;  // G <= 32 (cluster) or <= 160 (grid)
    auto post_winner = [&](const CpqrRec& w, long long wpos, int wg, bool amb) {
        s_sel[0] = amb ? -2 : w.col;
        s_sel[1] = wpos;
        s_sel[2] = wg;
        s_sc[0] = w.tau;
        s_sc[1] = w.beta;
        s_sc[2] = w.scale;
    };
    auto select = [&](int first, int parity) {
        int slot = parity;
        if (wid == 0) {
            CpqrRec r[kRecPerLane];
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) {
                const int g = lane + 32 * t;
                if (g < G) {
                    r[t] = rec_of(parity, g);
                } else {
                    r[t].vmax = -1.0;
                    r[t].pos = LLONG_MAX;
                }
            }
            double vmax = -1.0;
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) vmax = fmax(vmax, r[t].vmax);
            if (first > 0) trace(first - 1, 4);
            vmax = warp_max_nonneg(vmax);
            unsigned best = 0xffffffffu;
            int bt = 0, amb = 0;
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) {
                if (r[t].vmax >= 0.0 && qualifies(r[t].vmax, vmax)) {
                    amb |= r[t].vmax != vmax;
                    if (static_cast<unsigned>(r[t].pos) < best) {
                        best = static_cast<unsigned>(r[t].pos);
                        bt = t;
                    }
                }
            }
            amb = __any_sync(0xffffffffu, amb);
            const unsigned wb = __reduce_min_sync(0xffffffffu, best);
            if (best == wb && best != 0xffffffffu) {  // unique lane: positions are distinct
                CpqrRec w = r[0];
#pragma unroll
                for (int t = 1; t < kRecPerLane; ++t)
                    if (bt == t) w = r[t];
                post_winner(w, wb, lane + 32 * bt, amb != 0);
            }
            if (lane == 0) red_d[0] = vmax;
        }
        __syncthreads();
        if (first > 0) trace(first - 1, 7);
        if (s_sel[0] == -2) {
            // Exact tie pass: lowest position with sqrt(live) >= the global threshold.
            const double vmax = red_d[0];
            const bool cand = active && q == 0 && s_pos[lc] >= first;
            int winlc;
            const int winpos = local_pick(cand, cand ? s_live[lc] : -1.0, cand ? s_pos[lc] : 0, vmax, winlc);
            push_candidate(winpos == INT_MAX ? nc : winlc, first, cand_slot(2), p_alpha, p_tail);
            __syncthreads();
            if (tid == 0) write_record(2, 0.0, winpos);
            barrier_all();
            slot = 2;
            if (wid == 0) {
                unsigned b2 = 0xffffffffu;
                CpqrRec r2;
                int g2 = -1;
                for (int g = lane; g < G; g += 32) {
                    const CpqrRec rr = rec_of(2, g);
                    if (static_cast<unsigned>(rr.pos) < b2) {
                        b2 = static_cast<unsigned>(rr.pos);
                        r2 = rr;
                        g2 = g;
                    }
                }
                const unsigned wb = __reduce_min_sync(0xffffffffu, b2);
                if (b2 == wb && b2 != 0xffffffffu) post_winner(r2, wb, g2, false);
            }
            __syncthreads();
        }
        {
            const int len = m - first;
            const double tau = s_sc[0], scale = s_sc[2];
            const double* src = col_of(slot, static_cast<int>(s_sel[2]));
            for (int i = tid; i < len; i += T) {
                const double x = kCluster ? src[i] : __ldcg(src + i);
                xv[i] = tau != 0.0 ? (i == 0 ? 1.0 : mul_rn(x, scale)) : x;
            }
            for (int i = len + tid; i < span + S; i += T) xv[i] = 0.0;  // stale tail of the previous pivot
        }
        __syncthreads();
    };

    // ---- pivot 0 ----
    {
        const bool cand = active && q == 0;
        const double lv = cand ? s_live[lc] : -1.0;
        const double mx = local_max(cand, lv);
        int winlc;
        const int winpos = local_pick(cand, lv, cand ? s_pos[lc] : 0, mx, winlc);
        push_candidate(winpos == INT_MAX ? nc : winlc, 0, cand_slot(0), p_alpha, p_tail);
        __syncthreads();
        if (tid == 0) write_record(0, mx, winpos);
        barrier_all();
        select(0, 0);
    }

    for (int s = 0; s < a.k; ++s) {
        const long long piv = s_sel[0], ppos = s_sel[1];
        const double tau = s_sc[0];
        trace(s, 0);
        if (me == 0 && tid == 0) {
            a.taus[s] = tau;
            a.pivots[s] = piv;
        }
        // Replay the swap on positions (qr.cpp:79-86); the group leader owns
        // its column's position, every member keeps a copy.
        long long mypos = -1;
        if (active) {
            mypos = s_pos[lc];
            if (col == piv) mypos = s;
            else if (mypos == s) mypos = ppos;
            if (q == 0) s_pos[lc] = mypos;
        }

        // ---- trailing update + downdate (qr.cpp:93-106) ----
        const int dreg = s - l0;
        const int rr0 = dreg <= 0 ? 0 : dreg / S;
        const int sr0 = s / S;
        const double* xr = xv + (l0 + q - s);  // xr[S*r] = v for register row r
        p_alpha = 0.0;
        p_tail = 0.0;
        auto tpart = [&](int i, double v) {
            if (i == s + 1) p_alpha = v;
            else if (i > s + 1) p_tail = fma(v, v, p_tail);
        };
        bool cand = false;
        double lv = -1.0;
        if (active && col == piv) {
            if (tau != 0.0) {  // the pivot column becomes [R; beta; v] like the reference's work
                const double beta = s_sc[1];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = l0 + q + S * r;
                    if (i >= s && i < m) yr[r] = (i == s) ? beta : xv[i - s];
                }
                for (int r = sr0; r < nsr; ++r) {
                    const int i = q + S * r;
                    if (i >= s) myrows[i] = (i == s) ? beta : xv[i - s];
                }
            }
        } else if (mypos > s) {
            double h = 0.0;
            int owner;
            if (s < l0) {
                owner = s % S;
                if (q == owner) h = myrows[s];
            } else {
                owner = dreg % S;
                switch (rr0) {
#define IDK_HEAD_CASE(r) \
    case r:              \
        if constexpr (r < R) h = yr[r]; \
        break;
                    IDK_REP32(IDK_HEAD_CASE)
#undef IDK_HEAD_CASE
                    default:
                        break;
                }
            }
            const double ys = __shfl_sync(group_mask<S>(), h, gbase + owner);
            double head = ys;
            if (tau != 0.0) {
                double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
                int r = sr0;
                for (; r + 4 <= nsr; r += 4) {
                    const int i = q + S * r;
                    const double y0 = myrows[i], y1 = myrows[i + S], y2 = myrows[i + 2 * S], y3 = myrows[i + 3 * S];
                    const double v0 = xv[i - s], v1 = xv[i - s + S], v2 = xv[i - s + 2 * S], v3 = xv[i - s + 3 * S];
                    d0 = fma(v0, y0, d0);
                    d1 = fma(v1, y1, d1);
                    d2 = fma(v2, y2, d2);
                    d3 = fma(v3, y3, d3);
                }
                for (; r < nsr; ++r) {
                    const int i = q + S * r;
                    d0 = fma(xv[i - s], myrows[i], d0);
                }
                switch (rr0) {
#define IDK_DOT_CASE(r)                                                     \
    case r:                                                                 \
        if constexpr (r < R) {                                              \
            if ((r & 3) == 0) d0 = fma(xr[S * r], yr[r], d0);               \
            else if ((r & 3) == 1) d1 = fma(xr[S * r], yr[r], d1);          \
            else if ((r & 3) == 2) d2 = fma(xr[S * r], yr[r], d2);          \
            else d3 = fma(xr[S * r], yr[r], d3);                            \
        }                                                                   \
        [[fallthrough]];
                    IDK_REP32(IDK_DOT_CASE)
#undef IDK_DOT_CASE
                    default:
                        break;
                }
                const double w = mul_rn(group_sum<S>((d0 + d1) + (d2 + d3)), tau);
                r = sr0;
                for (; r + 4 <= nsr; r += 4) {
                    const int i = q + S * r;
                    const double y0 = myrows[i], y1 = myrows[i + S], y2 = myrows[i + 2 * S], y3 = myrows[i + 3 * S];
                    const double v0 = xv[i - s], v1 = xv[i - s + S], v2 = xv[i - s + 2 * S], v3 = xv[i - s + 3 * S];
                    const double n0 = fma(-w, v0, y0), n1 = fma(-w, v1, y1), n2 = fma(-w, v2, y2), n3 = fma(-w, v3, y3);
                    myrows[i] = n0;
                    myrows[i + S] = n1;
                    myrows[i + 2 * S] = n2;
                    myrows[i + 3 * S] = n3;
                    tpart(i, n0);
                    tpart(i + S, n1);
                    tpart(i + 2 * S, n2);
                    tpart(i + 3 * S, n3);
                }
                for (; r < nsr; ++r) {
                    const int i = q + S * r;
                    const double nv = fma(-w, xv[i - s], myrows[i]);
                    myrows[i] = nv;
                    tpart(i, nv);
                }
                switch (rr0) {
#define IDK_AXPY_CASE(r)                                         \
    case r:                                                      \
        if constexpr (r < R) yr[r] = fma(-w, xr[S * r], yr[r]);  \
        [[fallthrough]];
                    IDK_REP32(IDK_AXPY_CASE)
#undef IDK_AXPY_CASE
                    default:
                        break;
                }
                head = ys - w;  // row s has v_0 = 1
            } else {
                for (int r = sr0; r < nsr; ++r) tpart(q + S * r, myrows[q + S * r]);
            }
#pragma unroll
            for (int r = 0; r < R; ++r) tpart(l0 + q + S * r, yr[r]);  // rows >= m hold zeros
            lv = sub_rn(s_live[lc], mul_rn(head, head));
            if (lv < 0.0) lv = 0.0;
            if (lv <= mul_rn(kRecomp, s_anchor[lc])) {
                // fresh = sum_{i > s} y_i^2 (qr.cpp:101-104) = alpha^2 + tail of the next step
                lv = group_sum<S>(fma(p_alpha, p_alpha, p_tail));
                if (q == 0) s_anchor[lc] = lv;
            }
            if (q == 0) s_live[lc] = lv;
            cand = q == 0;
        }
        trace(s, 1);
        if (s + 1 == a.k) break;

        // ---- next pivot: CTA candidate, exchange ----
        const int parity = (s + 1) & 1;
        const double mx = local_max(cand, lv);
        int winlc;
        const int winpos = local_pick(cand, lv, mypos, mx, winlc);
        trace(s, 2);
        push_candidate(winpos == INT_MAX ? nc : winlc, s + 1, cand_slot(parity), p_alpha, p_tail);
        __syncthreads();
        if (tid == 0) write_record(parity, mx, winpos);
        trace(s, 3);
        barrier_all();
        trace(s, 5);
        select(s + 1, parity);
        trace(s, 6);
    }

    // ---- write back (the only write of W) ----
    __syncthreads();
    if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = l0 + q + S * r;
            if (i < m) W[col * a.ldw + i] = yr[r];
        }
        for (int r = 0; r < nsr; ++r) {
            const int i = q + S * r;
            W[col * a.ldw + i] = myrows[i];
        }
        if (q == 0) a.pos_out[col] = s_pos[lc];
    }
    if constexpr (kCluster) cg::this_cluster().sync();  // keep shared memory alive for DSMEM readers
}

// ------------------------------------------------------------------------------------
// host side: plan + dispatch
// ------------------------------------------------------------------------------------

namespace {

int pad_lds(int l0, int S) {
    if (l0 <= 0) return 0;
    if (S >= 16) return l0 | 1;
    int lds = l0;
    while ((lds & 15) != (S & 15)) ++lds;
    return lds;
}

size_t resident_smem(int m, int nc, int l0, int lds, int S, int R, bool cluster) {
    const size_t mpad = static_cast<size_t>((m + 1) & ~1);
    const int span = std::max(m, l0 + R * S);
    const size_t xlen = static_cast<size_t>(((kGuard + span + S + 1) + 1) & ~1);
    size_t d = xlen + static_cast<size_t>(nc) * lds + 2 * static_cast<size_t>(nc) + static_cast<size_t>(nc);
    if (cluster) d += 3 * mpad;
    return d * sizeof(double);
}

ResidentPlan plan_for(int m, int64_t n, int k, int G_target, bool cluster, size_t smem_cap) {
    ResidentPlan best;
    int64_t G = std::min<int64_t>(n, G_target);
    const int nc = static_cast<int>((n + G - 1) / G);
    G = (n + nc - 1) / nc;
    static const int Rs[2] = {32, 16};
    static const int Ss[6] = {32, 16, 8, 4, 2, 1};
    for (int R : Rs) {
        const int maxT = R >= 32 ? 512 : (R >= 16 ? 640 : 768);
        for (int S : Ss) {
            const int threads = ((S * nc + 31) / 32) * 32;
            if (threads > maxT || threads < 32) continue;
            const int reg_rows = R * S;
            // skip plans whose register rows are mostly padding (a smaller R covers m)
            if (R > 16 && (R / 2) * S >= m) continue;
            int l0 = std::max(0, m - reg_rows);
            l0 = ((l0 + S - 1) / S) * S;  // uniform loop bounds need S | l0
            const int lds = pad_lds(l0, S);
            const size_t smem = resident_smem(m, nc, l0, lds, S, R, cluster);
            if (smem > smem_cap) continue;
            // cost model: per-step serial work of one thread (register rows are
            // cheap, shared rows cost ~3 LDS/STS each) -- the step latency --
            // plus a small throughput term for the threads it takes.
            const double cost = (R + 3.0 * (l0 / S)) + threads / 256.0;
            if (!best.ok || cost < best.cost) {
                best.ok = true;
                best.cluster = cluster;
                best.G = static_cast<int>(G);
                best.nc = nc;
                best.S = S;
                best.R = R;
                best.l0 = l0;
                best.lds = lds;
                best.threads = threads;
                best.smem = smem;
                best.cost = cost;
            }
        }
    }
    return best;
}

template <int S, int R, bool C>
void* kernel_ptr() {
    return reinterpret_cast<void*>(cpqr_resident_kernel<S, R, C>);
}

template <bool C>
void* pick_kernel(int S, int R) {
#define IDK_CASE(SS, RR) \
    if (S == SS && R == RR) return kernel_ptr<SS, RR, C>();
    IDK_CASE(32, 32) IDK_CASE(16, 32) IDK_CASE(8, 32) IDK_CASE(4, 32) IDK_CASE(2, 32) IDK_CASE(1, 32)
    IDK_CASE(32, 16) IDK_CASE(16, 16) IDK_CASE(8, 16) IDK_CASE(4, 16) IDK_CASE(2, 16) IDK_CASE(1, 16)
#undef IDK_CASE
    return nullptr;
}

}  // namespace

// Plan the on-chip CPQR of an m x n matrix: a single cluster (<= 16 CTAs,
// DSMEM exchange) when it fits, else one CTA per SM with the grid exchange.
ResidentPlan cpqr_resident_plan(int m, int64_t n, int k, int num_sms, bool allow_cluster) {
    const size_t cap = 200 * 1024;
    if (allow_cluster && n >= 32) {
        ResidentPlan p = plan_for(m, n, k, 16, true, cap);
        if (p.ok) {
            void* fn = pick_kernel<true>(p.S, p.R);
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(p.G);
            cfg.blockDim = dim3(p.threads);
            cfg.dynamicSmemBytes = p.smem;
            cudaLaunchAttribute attr;
            attr.id = cudaLaunchAttributeClusterDimension;
            attr.val.clusterDim.x = p.G;
            attr.val.clusterDim.y = 1;
            attr.val.clusterDim.z = 1;
            cfg.attrs = &attr;
            cfg.numAttrs = 1;
            int clusters = 0;
            if (cudaOccupancyMaxActiveClusters(&clusters, fn, &cfg) == cudaSuccess && clusters >= 1) return p;
            cudaGetLastError();
        }
    }
    return plan_for(m, n, k, num_sms, false, cap);
}

long long* g_trace = nullptr;  // debug: set by idk_debug_cpqr_trace

void cpqr_resident_set_trace(long long* p) { g_trace = p; }

size_t cpqr_resident_exchange_bytes(const ResidentPlan& p, int m) {
    if (!p.ok || p.cluster) return 0;
    const size_t G = static_cast<size_t>(p.G);
    return sizeof(CpqrRec) * 3 * G + sizeof(double) * 3 * G * static_cast<size_t>(m) + 256;
}

cudaError_t cpqr_resident_launch(const ResidentPlan& p, double* W, int64_t ldw, int m, int64_t n, int k,
                                 long long* pos_out, long long* pivots, double* taus, void* exch, unsigned* barrier,
                                 cudaStream_t stream) {
    ResidentArgs a;
    a.W = W;
    a.ldw = ldw;
    a.m = m;
    a.n = n;
    a.k = k;
    a.nc = p.nc;
    a.l0 = p.l0;
    a.lds = p.lds;
    a.pos_out = pos_out;
    a.pivots = pivots;
    a.taus = taus;
    const size_t G = static_cast<size_t>(p.G);
    char* e = static_cast<char*>(exch);
    a.rec = reinterpret_cast<CpqrRec*>(e);
    a.rec2 = a.rec + 2 * G;
    a.colbuf = reinterpret_cast<double*>(e + sizeof(CpqrRec) * 3 * G);
    a.colbuf2 = a.colbuf + 2 * G * static_cast<size_t>(m);
    a.barrier = barrier;
    a.trace = g_trace;
    void* args[] = {&a};
    if (p.cluster) {
        void* fn = pick_kernel<true>(p.S, p.R);
        if (!fn) return cudaErrorInvalidValue;
        cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
        if (err != cudaSuccess) return err;
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(p.G);
        cfg.blockDim = dim3(p.threads);
        cfg.dynamicSmemBytes = p.smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = p.G;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelExC(&cfg, fn, args);
    }
    void* fn = pick_kernel<false>(p.S, p.R);
    if (!fn) return cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(p.smem));
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(barrier, 0, sizeof(unsigned), stream);
    if (err != cudaSuccess) return err;
    return cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(p.threads), args, p.smem, stream);
}

}  // namespace idk
