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
#include <cstdlib>
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace idk {

// Exchange slot of one CTA for one exchange: a 4-double header (candidate
// column id, its next reflector tau/beta/scale) followed by the candidate's
// active rows.  Records: grid mode uses LL-style tagged 64-bit words
// (payload32 << 32 | tag32; aligned 64-bit stores are single-copy atomic), so
// polling the G records is the barrier; cluster mode keeps records in shared
// memory behind barrier.cluster.
constexpr int kHdr = 4;
constexpr int kRecWords = 4;  // vmax hi | vmax lo | pos | pad

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
    // grid-exchange buffers (global, zeroed before launch); unused in cluster mode
    unsigned long long* rec;  // [3][G][kRecWords]
    double* slots;            // [3][G][kHdr + m]
    unsigned* barrier;        // debug: optional grid barrier before each exchange
    long long* trace;         // optional: %globaltimer at 8 phase marks per step, every CTA
};

namespace {

constexpr double kRecomp = 1e-6;  // qr.cpp:100

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

__device__ __forceinline__ unsigned long long tagged(unsigned payload, unsigned tag) {
    return (static_cast<unsigned long long>(payload) << 32) | tag;
}

// Strong (relaxed, gpu scope) 16-byte accesses for the tagged records: each
// 64-bit element is single-copy atomic and takes part in the memory model.
__device__ __forceinline__ void st_relaxed_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long* p, unsigned long long& a,
                                              unsigned long long& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
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
    const int slot_len = kHdr + ((m + 1) & ~1);
    double* xbuf = sm;
    double* xv = xbuf + kGuard;
    double* rows = xbuf + xlen;                                      // nc * lds
    double* s_live = rows + static_cast<size_t>(nc) * lds;           // nc
    double* s_anchor = s_live + nc;                                  // nc
    long long* s_pos = reinterpret_cast<long long*>(s_anchor + nc);  // nc (positions < 2^31)
    double* cslots = reinterpret_cast<double*>(s_pos + nc);          // cluster: [3][slot_len]

    __shared__ double red_d[32];
    __shared__ long long red_l[32];
    __shared__ double s_sc[3];      // tau, beta, scale of the current pivot
    __shared__ long long s_sel[3];  // pivot column, its position before the swap, winning CTA (-2: tie pass)
    __shared__ double s_rec[3][2];  // cluster: own records {vmax, pos}

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

    auto trace = [&](int s, int ph) {
        if (a.trace != nullptr && tid == 0) a.trace[(static_cast<size_t>(me) * (a.k + 1) + s) * 8 + ph] = globaltimer();
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
    }
    for (int r = 0; r < nsr; ++r) {
        const int i = q + S * r;
        const double v = active ? W[col * a.ldw + i] : 0.0;
        if (lc < nc) myrows[i] = v;
        part = fma(v, v, part);
    }
    part = group_sum<S>(part);
    if (active && q == 0) {
        s_live[lc] = part;
        s_anchor[lc] = part;
        s_pos[lc] = col;
    }

    // This group's column: alpha = row `first`, tail = sum of squares below it.
    auto partials = [&](int first, double& al, double& tl) {
        double a0 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = l0 + q + S * r;
            if (i == first) a0 = yr[r];
            else if (i > first) {
                if (r & 1) t1 = fma(yr[r], yr[r], t1);
                else t0 = fma(yr[r], yr[r], t0);
            }
        }
        for (int r = first / S; r < nsr; ++r) {
            const int i = q + S * r;
            const double v = myrows[i];
            if (i == first) a0 = v;
            else if (i > first) t0 = fma(v, v, t0);
        }
        al = group_sum<S>(a0);
        tl = group_sum<S>(t0 + t1);
    };

    // CTA argmax (qr.cpp:66-78 over this CTA's columns): the max live norm,
    // then the lowest position that qualifies against it; 32-bit redux.sync
    // per warp and one __syncthreads per pass.
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

    auto slot_ptr = [&](int slot, int g) -> double* {
        if constexpr (kCluster) {
            double* mineptr = cslots + slot * slot_len;
            return g == me ? mineptr : cg::this_cluster().map_shared_rank(mineptr, g);
        } else {
            return a.slots + (static_cast<size_t>(slot) * G + g) * slot_len;
        }
    };

    // Publish this CTA's candidate (local index winlc, position winpos) for the
    // exchange `tag` in `slot`: header + rows first..m-1, then the record.
    auto publish = [&](int slot, unsigned tag, double mx, int winpos, int winlc, int first) {
        const bool have = winpos != INT_MAX;
        double* dst = slot_ptr(slot, me);
        if (have && lc == winlc) {
            double al, tl;
            partials(first, al, tl);
            double tau, beta, scale;
            reflector(al, tl, m - first, tau, beta, scale);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = l0 + q + S * r;
                if (i >= first && i < m) dst[kHdr + i - first] = yr[r];
            }
            if (q == 0) {
                dst[0] = __longlong_as_double(c0 + winlc);
                dst[1] = tau;
                dst[2] = beta;
                dst[3] = scale;
            }
        }
        if (have) {  // shared-memory rows of the candidate, copied by everyone
            const double* cr = rows + static_cast<size_t>(winlc) * lds;
            for (int i = first + tid; i < l0; i += T) dst[kHdr + i - first] = cr[i];
        }
        __syncthreads();
        if (tid == 0) {
            const unsigned pos32 = have ? static_cast<unsigned>(winpos) : 0xffffffffu;
            if constexpr (kCluster) {
                s_rec[slot][0] = mx;
                s_rec[slot][1] = __longlong_as_double(static_cast<long long>(pos32));
            } else {
                __threadfence();  // slot data before the tagged record (release)
                const unsigned long long vb = static_cast<unsigned long long>(__double_as_longlong(mx));
                unsigned long long* rp = a.rec + (static_cast<size_t>(slot) * G + me) * kRecWords;
                st_relaxed_v2(rp, tagged(static_cast<unsigned>(vb >> 32), tag), tagged(static_cast<unsigned>(vb), tag));
                st_relaxed_v2(rp + 2, tagged(pos32, tag), 0ull);
            }
        }
    };

    // Record of CTA g for exchange `tag`: {vmax, pos}; grid mode spins until
    // all three words carry the tag.
    auto read_rec = [&](int slot, int g, unsigned tag, double& vmax, unsigned& pos) {
        if constexpr (kCluster) {
            const double* rp = cg::this_cluster().map_shared_rank(&s_rec[slot][0], g);
            vmax = rp[0];
            pos = static_cast<unsigned>(__double_as_longlong(rp[1]));
        } else {
            const unsigned long long* rp = a.rec + (static_cast<size_t>(slot) * G + g) * kRecWords;
            unsigned long long x0, x1, x2, x3;
            for (;;) {
                ld_relaxed_v2(rp, x0, x1);
                ld_relaxed_v2(rp + 2, x2, x3);
                if (static_cast<unsigned>(x0) == tag && static_cast<unsigned>(x1) == tag &&
                    static_cast<unsigned>(x2) == tag)
                    break;
            }
            vmax = __longlong_as_double(static_cast<long long>(((x0 >> 32) << 32) | (x1 >> 32)));
            pos = static_cast<unsigned>(x2 >> 32);
        }
    };

    constexpr int kRecPerLane = kCluster ? 1 : 5;  // G <= 32 (cluster) or <= 160 (grid)

    // Wait for every CTA's record of exchange `tag`, reduce them (identical in
    // every CTA), then copy the winner's column -- scaled by its reflector --
    // into xv.  `first` = the step the new pivot is for.
    unsigned epoch = 0;
    auto exchange = [&](int parity, unsigned tag, int first) {
        if constexpr (kCluster) cg::this_cluster().sync();
        if constexpr (!kCluster) {
            if (a.barrier != nullptr) grid_barrier(a.barrier, epoch);
        }
        int slot = parity;
        if (wid == 0) {
            double v[kRecPerLane];
            unsigned p[kRecPerLane];
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) {
                const int g = lane + 32 * t;
                v[t] = -1.0;
                p[t] = 0xffffffffu;
                if (g < G) read_rec(parity, g, tag, v[t], p[t]);
            }
            if constexpr (!kCluster) __threadfence();  // acquire: slot data after the records
            double vmax = -1.0;
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) vmax = fmax(vmax, v[t]);
            vmax = warp_max_nonneg(vmax);
            unsigned best = 0xffffffffu;
            int bt = 0, amb = 0;
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) {
                if (v[t] >= 0.0 && qualifies(v[t], vmax)) {
                    amb |= v[t] != vmax;
                    if (p[t] < best) {
                        best = p[t];
                        bt = t;
                    }
                }
            }
            amb = __any_sync(0xffffffffu, amb);
            const unsigned wb = __reduce_min_sync(0xffffffffu, best);
            if (best == wb && best != 0xffffffffu) {  // unique lane: positions are distinct
                s_sel[0] = amb ? -2 : 0;
                s_sel[1] = wb;
                s_sel[2] = lane + 32 * bt;
            }
            if (lane == 0) red_d[0] = vmax;
        }
        __syncthreads();
        if (s_sel[0] == -2) {
            // Exact tie pass: lowest position with sqrt(live) >= the global threshold.
            const double vmax = red_d[0];
            const bool cand = active && q == 0 && s_pos[lc] >= first;
            int winlc;
            const int winpos = local_pick(cand, cand ? s_live[lc] : -1.0, cand ? s_pos[lc] : 0, vmax, winlc);
            publish(2, tag, 0.0, winpos, winlc, first);
            if constexpr (kCluster) cg::this_cluster().sync();
            slot = 2;
            if (wid == 0) {
                unsigned b2 = 0xffffffffu;
                int g2 = -1;
                for (int g = lane; g < G; g += 32) {
                    double vv;
                    unsigned pp;
                    read_rec(2, g, tag, vv, pp);
                    if (pp < b2) {
                        b2 = pp;
                        g2 = g;
                    }
                }
                if constexpr (!kCluster) __threadfence();
                const unsigned wb = __reduce_min_sync(0xffffffffu, b2);
                if (b2 == wb && b2 != 0xffffffffu) {
                    s_sel[0] = 0;
                    s_sel[1] = wb;
                    s_sel[2] = g2;
                }
            }
            __syncthreads();
        }
        // All threads: header + winner's column (one round trip), scaled into xv.
        const double* src = slot_ptr(slot, static_cast<int>(s_sel[2]));
        const int len = m - first;
        const double h0 = kCluster ? src[0] : __ldcg(src);
        const double tau = kCluster ? src[1] : __ldcg(src + 1);
        const double beta = kCluster ? src[2] : __ldcg(src + 2);
        const double scale = kCluster ? src[3] : __ldcg(src + 3);
        for (int i = tid; i < len; i += T) {
            const double x = kCluster ? src[kHdr + i] : __ldcg(src + kHdr + i);
            xv[i] = tau != 0.0 ? (i == 0 ? 1.0 : mul_rn(x, scale)) : x;
        }
        for (int i = len + tid; i < span + S; i += T) xv[i] = 0.0;  // stale tail of the previous pivot
        if (tid == 0) {
            s_sel[0] = __double_as_longlong(h0);
            s_sc[0] = tau;
            s_sc[1] = beta;
            s_sc[2] = scale;
        }
        __syncthreads();
    };

    // ---- pivot 0 ----
    {
        __syncthreads();
        const bool cand = active && q == 0;
        const double lv = cand ? s_live[lc] : -1.0;
        const double mx = local_max(cand, lv);
        int winlc;
        const int winpos = local_pick(cand, lv, cand ? s_pos[lc] : 0, mx, winlc);
        publish(0, 1u, mx, winpos, winlc, 0);
        exchange(0, 1u, 0);
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
                    myrows[i] = fma(-w, v0, y0);
                    myrows[i + S] = fma(-w, v1, y1);
                    myrows[i + 2 * S] = fma(-w, v2, y2);
                    myrows[i + 3 * S] = fma(-w, v3, y3);
                }
                for (; r < nsr; ++r) {
                    const int i = q + S * r;
                    myrows[i] = fma(-w, xv[i - s], myrows[i]);
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
            }
            lv = sub_rn(s_live[lc], mul_rn(head, head));
            if (lv < 0.0) lv = 0.0;
            if (lv <= mul_rn(kRecomp, s_anchor[lc])) {
                // fresh = sum_{i > s} y_i^2 (qr.cpp:101-104)
                double al, tl;
                partials(s + 1, al, tl);
                lv = fma(al, al, tl);
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
        publish(parity, static_cast<unsigned>(s + 2), mx, winpos, winlc, s + 1);
        trace(s, 3);
        exchange(parity, static_cast<unsigned>(s + 2), s + 1);
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
    const size_t slot_len = kHdr + static_cast<size_t>((m + 1) & ~1);
    const int span = std::max(m, l0 + R * S);
    const size_t xlen = static_cast<size_t>(((kGuard + span + S + 1) + 1) & ~1);
    size_t d = xlen + static_cast<size_t>(nc) * lds + 2 * static_cast<size_t>(nc) + static_cast<size_t>(nc);
    if (cluster) d += 3 * slot_len;
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
    const size_t slot_len = kHdr + static_cast<size_t>((m + 1) & ~1);
    return sizeof(unsigned long long) * kRecWords * 3 * G + sizeof(double) * 3 * G * slot_len + 256;
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
    a.rec = reinterpret_cast<unsigned long long*>(e);
    a.slots = reinterpret_cast<double*>(e + sizeof(unsigned long long) * kRecWords * 3 * G);
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
    // records start untagged (tags are 1..k, so stale records never match)
    err = cudaMemsetAsync(exch, 0, sizeof(unsigned long long) * kRecWords * 3 * G, stream);
    if (err != cudaSuccess) return err;
    a.barrier = nullptr;
    if (getenv("IDK_DEBUG_GRID_BARRIER")) {
        a.barrier = barrier;
        err = cudaMemsetAsync(barrier, 0, sizeof(unsigned), stream);
        if (err != cudaSuccess) return err;
    }
    return cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(p.threads), args, p.smem, stream);
}

}  // namespace idk
