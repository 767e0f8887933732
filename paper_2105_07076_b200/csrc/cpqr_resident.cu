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
// Step structure.  The norm downdate needs only the dot w = tau v^T y of each
// column, so a step is: dot + downdate for every column -> CTA argmax (one
// __syncthreads) -> exchange of the CTA candidates -> select.  Two exchange
// policies share the code:
//   kCluster = true : one thread-block cluster (<= 16 CTAs).  The warp holding
//     the CTA's winner applies that column's pending update to a raw copy with
//     all 32 lanes, builds the next reflector, stages [v | header] in its own
//     slot and bulk-copies it (cp.async.bulk shared::cta -> shared::cluster) to
//     every peer, completing a transaction count on the peer's mbarrier; the
//     other warps apply their deferred trailing axpy while the copies fly.
//     After the mbarrier wait every warp selects the winner from local shared
//     memory and the update reads v straight from the winner's slot copy
//     (push mode).  When G slots of m rows do not fit, only the 48-byte
//     headers are pushed and the winner's rows are pulled over DSMEM (pull).
//   kCluster = false: one CTA per SM (cooperative launch).  Each CTA publishes
//     its candidate column to a global slot and an LL-style tagged record;
//     every thread polls at most a few records (all in flight at once), then
//     the winner's column is copied from L2.
// Reflectors are addressed by absolute row (v_i = 0 for retired and padding
// rows) so the row loops carry no predicates.
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
constexpr int kHdr = 6;  // grid slot header: col, tau, beta, scale, ready flag (epoch | tag), pad
constexpr int kCHdr = 6;  // cluster slot header: col, tau, beta, scale, vmax, pos
constexpr int kRecWords = 4;  // vmax hi | vmax lo | pos | pad
// Copies of each published grid-mode column: after the records every CTA reads
// the winner's column at the same moment, and with one copy all G readers hit
// the same ~17 L2 lines; reader g reads copy g % kColCopies
// (profiles/grid_exchange_r02.txt: cfg4 8.39 -> 7.53 us per step).
constexpr int kColCopies = 4;
constexpr int kPollWarps = 8;  // grid records reduced by their polling warps first (G <= 256)

struct ResidentArgs {
    double* W;
    int64_t ldw;
    const double* Win;  // the matrix read once at the start (W itself, or the caller's A: no working copy)
    int64_t ldin;
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
    int push;                 // cluster: 1 = every CTA holds every candidate (push), 0 = headers only (pull)
    unsigned long long epoch; // grid slot ready flags: per-launch epoch << 32 | exchange tag
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

#ifdef IDK_CPQR_TRACE
__device__ __forceinline__ long long globaltimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// sqrt(v) >= (1 - 1e-14) * sqrt(vmax) (qr.cpp:71-73) evaluated exactly, with
// the sqrt only inside the 4e-14 band where the answer is not obvious.
// The sqrt pair is out of line: the band test almost never reaches it, and
// inlined at every reduction site it was ~750 SASS instructions of cold code
// inside the step loop (instruction-fetch stalls on the serial phases).
__device__ __noinline__ bool qualifies_band(double v, double vmax) {
    return sqrt(v) >= (1.0 - 1e-14) * sqrt(vmax);
}
__device__ __forceinline__ bool qualifies(double v, double vmax) {
    if (v == vmax) return true;
    if (!(v >= vmax * (1.0 - 4e-14))) return false;
    return qualifies_band(v, vmax);
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

// reflector() evaluated by a whole warp: the two divisions run side by side
// in lanes 0 and 1 (one SIMT division instead of two dependent ones); every
// lane returns the same, exactly rounded tau, beta, scale.
__device__ __forceinline__ void reflector_warp(double alpha, double tail, int len, double& tau, double& beta,
                                               double& scale) {
    tau = 0.0;
    beta = alpha;
    scale = 1.0;
    if (len > 1 && tail != 0.0) {
        beta = -copysign(sqrt(add_rn(mul_rn(alpha, alpha), tail)), alpha);
        const unsigned lane = threadIdx.x & 31u;
        const double num = lane == 0 ? beta - alpha : 1.0;
        const double den = lane == 0 ? beta : alpha - beta;
        const double qd = num / den;
        tau = __shfl_sync(0xffffffffu, qd, 0);
        scale = __shfl_sync(0xffffffffu, qd, 1);
    }
}

constexpr int kPubRegs = 4;  // candidate rows per lane kept in registers (m - first <= 128)
constexpr int kHelpWarps = 4;  // warps building a tall (m - first > 128) candidate

__device__ __forceinline__ unsigned long long tagged(unsigned payload, unsigned tag) {
    return (static_cast<unsigned long long>(payload) << 32) | tag;
}

// Strong (relaxed, gpu scope) 16-byte accesses for the tagged records: each
// 64-bit element is single-copy atomic and takes part in the memory model.
__device__ __forceinline__ void st_relaxed_v2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long a) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(a) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void ld_relaxed_v2(const unsigned long long* p, unsigned long long& a,
                                              unsigned long long& b) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// ---- DSMEM bulk push: cp.async.bulk shared::cta -> shared::cluster with an
// mbarrier transaction count on the receiving CTA ----
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ unsigned mapa_u32(unsigned addr, int rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void bulk_push(unsigned dst_cluster, unsigned src_cta, unsigned bytes, unsigned mbar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst_cluster), "r"(src_cta), "r"(bytes), "r"(mbar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned a, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned a, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned a) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned a, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "IDK_MBAR_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra IDK_MBAR_WAIT_%=;\n}"
        ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

}  // namespace

#define IDK_REP32(M) \
    M(0) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) \
    M(16) M(17) M(18) M(19) M(20) M(21) M(22) M(23) M(24) M(25) M(26) M(27) M(28) M(29) M(30) M(31)

// The current reflector is addressed by absolute row: xa[i] = v_i, and
// xa[i] = 0 for every retired row (i < s) and padding row (i >= m), so the row
// loops need no predicates and every lane of a warp takes the same path (the
// start row depends only on s).
//   grid mode   : xa = xbuf, refilled from the winner's global slot each step;
//   cluster mode: xa = the winner's slot in this CTA's own shared memory (every
//                 CTA pushed its candidate to every other CTA before the barrier).

template <int S, int R, bool kCluster>
__global__ void __launch_bounds__(max_threads_for<R>())
cpqr_resident_kernel(ResidentArgs a) {
    extern __shared__ __align__(16) double sm[];
    const int m = a.m, nc = a.nc, l0 = a.l0, lds = a.lds;
    const int G = gridDim.x;
    const int span = max(m, l0 + R * S);
    const int xlen = (span + S + 1) & ~1;       // absolute reflector rows 0 .. span+S-1
    const int gslot = kHdr + ((m + 1) & ~1);    // grid slot: header + rows first .. m-1
    const int cslot = xlen + kCHdr;             // cluster slot: absolute rows, then the header
    double* xbuf = sm;               // grid: the current reflector; cluster: staging scratch
    double* xpull = xbuf + xlen;     // cluster pull mode: reflector double buffer (2 x xlen)
    double* rows = xpull + 2 * xlen;                                 // nc * lds
    double* s_live = rows + static_cast<size_t>(nc) * lds;           // nc
    double* s_anchor = s_live + nc;                                  // nc
    long long* s_pos = reinterpret_cast<long long*>(s_anchor + nc);  // nc (positions < 2^31)
    // cluster slots, 16-B aligned: push mode [3][G][cslot]; pull mode [3][cslot]
    // (own) followed by the header copies [3][G][kCHdr]
    double* cslots = reinterpret_cast<double*>(s_pos + nc);
    cslots += (static_cast<unsigned>(__cvta_generic_to_shared(cslots)) >> 3) & 1u;  // 16-B align (stays a shared-window pointer)
    const bool push = a.push != 0;
    double* chdr = cslots + 3 * cslot;

    __shared__ long long red_l[32];
    __shared__ double s_wv[32];     // per-warp argmax records
    __shared__ unsigned s_wp[32];
    __shared__ unsigned s_wl[32];
    __shared__ long long s_sel[3];  // grid tie pass: -, winning position, winning CTA
    __shared__ double s_help[kHelpWarps + 2];  // tall candidate build: partial norms, pending w, alpha
    __shared__ unsigned long long s_mbar[2];      // cluster: bulk-push barriers, one per slot parity;
                                                  // grid: candidate handed to the publisher / consumed by it
    __shared__ double s_pubw;                     // grid: the candidate's pending axpy weight
    __shared__ int s_publc;                       // grid: the candidate's local column (-1: none)
    __shared__ double s_rv[kCluster ? 1 : 160];  // grid: the G records of this exchange
    __shared__ unsigned s_rp[kCluster ? 1 : 160];
    __shared__ double s_gv[kPollWarps];  // grid: per polling warp (max, lowest qualifying position, its CTA)
    __shared__ unsigned s_gp[kPollWarps];
    __shared__ unsigned s_gg[kPollWarps];

    // grid mode: the last warp only publishes the CTA's candidate (no columns); T counts the workers
    const int tid = threadIdx.x, T = kCluster ? blockDim.x : blockDim.x - 32;
    const bool publisher = !kCluster && tid >= T;
    const int lane = tid & 31, wid = tid >> 5, nw = T >> 5;
    const int lc = tid / S, q = tid % S;
    const int me = kCluster ? static_cast<int>(cg::this_cluster().block_rank()) : blockIdx.x;
    const int64_t c0 = static_cast<int64_t>(me) * nc;
    const int myn = static_cast<int>(max(0LL, min(static_cast<long long>(a.n - c0), static_cast<long long>(nc))));
    const bool active = lc < myn;
    const int64_t col = c0 + lc;
    double* const W = a.W;
    const int nsr = l0 / S;  // l0 is a multiple of S
    double* myrows = rows + static_cast<size_t>(lc < nc ? lc : 0) * lds;
    const int gbase = lane & ~(S - 1);
    constexpr unsigned kFull = 0xffffffffu;

    // barrier over the threads that own columns (grid mode: without the publisher warp)
    auto cta_sync = [&]() {
        if constexpr (kCluster) __syncthreads();
        else asm volatile("bar.sync 3, %0;" ::"r"(T) : "memory");
    };

    // phase marks (tools/trace_cpqr.py) exist only in builds with -DIDK_CPQR_TRACE:
    // the checks cost code size in the step loop, which the serial phases feel
    auto trace_by = [&](bool who, int s, int ph) {
#ifdef IDK_CPQR_TRACE
        if (a.trace != nullptr && who && s >= 0)
            a.trace[(static_cast<size_t>(me) * (a.k + 1) + s) * 16 + ph] = globaltimer();
#else
        (void)who;
        (void)s;
        (void)ph;
#endif
    };
    auto trace = [&](int s, int ph) { trace_by(tid == 0, s, ph); };

#ifdef IDK_CPQR_TRACE
    if (a.trace != nullptr && tid == 0) {  // debug: which SM this CTA runs on (slot 15 of row k)
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[(static_cast<size_t>(me) * (a.k + 1) + a.k) * 16 + 15] = smid;
    }
#endif
    for (int i = tid; i < 3 * xlen; i += T) xbuf[i] = 0.0;
    if constexpr (kCluster) {
        const int zn = push ? 3 * G * cslot : 3 * cslot + 3 * G * kCHdr;
        for (int i = tid; i < zn; i += T) cslots[i] = 0.0;
        if (tid == 0) {
            mbar_init(smem_u32(&s_mbar[0]), 1);
            mbar_init(smem_u32(&s_mbar[1]), 1);
            fence_mbar_init();
        }
    } else {
        if (tid == 0) {
            mbar_init(smem_u32(&s_mbar[0]), 1);  // candidate staged (owner warp -> publisher)
            mbar_init(smem_u32(&s_mbar[1]), 1);  // candidate consumed (publisher -> owner warp)
            fence_mbar_init();
        }
    }
    unsigned mbar_phase = 0;  // bit p = phase parity of s_mbar[p]

    // ---- load (the only read of W) and initial norms (qr.cpp:56-62) ----
    double yr[R];
    double part = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = l0 + q + S * r;
        yr[r] = (active && i < m) ? a.Win[col * a.ldin + i] : 0.0;
        part = fma(yr[r], yr[r], part);
    }
    for (int r = 0; r < nsr; ++r) {
        const int i = q + S * r;
        const double v = active ? a.Win[col * a.ldin + i] : 0.0;
        if (lc < nc) myrows[i] = v;
        part = fma(v, v, part);
    }
    part = group_sum<S>(part);
    if (active && q == 0) {
        s_live[lc] = part;
        s_anchor[lc] = part;
        s_pos[lc] = col;
    }
    if constexpr (kCluster) cg::this_cluster().sync();  // slots zeroed before any CTA pushes
    else __syncthreads();

    // the current pivot (identical in every thread after an exchange)
    long long piv = 0, ppos = 0;
    double tau = 0.0, beta = 0.0;
    const double* xa = xbuf;

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

    // Exact CTA pick against a given threshold vmax (qr.cpp:66-78 over this
    // CTA's columns): the lowest position that qualifies; two 32-bit redux.sync
    // per warp and one __syncthreads.
    auto local_pick = [&](bool cand, double lv, long long pos, double vmax, int& winlc) -> int {
        const unsigned key = (cand && qualifies(lv, vmax)) ? static_cast<unsigned>(pos) : 0xffffffffu;
        const unsigned wm = __reduce_min_sync(kFull, key);
        const unsigned wl = __reduce_min_sync(kFull, (key == wm) ? static_cast<unsigned>(lc) : 0xffffffffu);
        if (lane == 0) red_l[wid] = static_cast<long long>((static_cast<unsigned long long>(wm) << 32) | wl);
        cta_sync();
        const unsigned long long mine = lane < nw ? static_cast<unsigned long long>(red_l[lane]) : ~0ull;
        const unsigned best = __reduce_min_sync(kFull, static_cast<unsigned>(mine >> 32));
        winlc = static_cast<int>(__reduce_min_sync(
            kFull, static_cast<unsigned>(mine >> 32) == best ? static_cast<unsigned>(mine) : 0xffffffffu));
        return best == 0xffffffffu ? INT_MAX : static_cast<int>(best);
    };

    // CTA argmax in one __syncthreads: each warp reduces (max live, lowest
    // position qualifying against it, its column), then every warp combines
    // the warp records identically.  A warp whose max qualifies against the CTA
    // max without equalling it picked against a lower threshold -- ambiguous,
    // resolved exactly by local_pick (rare: needs norms within 4e-14).
    auto cta_argmax = [&](bool cand, double lv, long long pos, int& winpos, int& winlc) -> double {
        const double wm = warp_max_nonneg(cand ? lv : -1.0);
        const unsigned key = (cand && qualifies(lv, wm)) ? static_cast<unsigned>(pos) : 0xffffffffu;
        const unsigned wp = __reduce_min_sync(kFull, key);
        const unsigned wl = __reduce_min_sync(kFull, key == wp ? static_cast<unsigned>(lc) : 0xffffffffu);
        if (lane == 0) {
            s_wv[wid] = wm;
            s_wp[wid] = wp;
            s_wl[wid] = wl;
        }
        cta_sync();
        const double v = lane < nw ? s_wv[lane] : -1.0;
        const unsigned p = lane < nw ? s_wp[lane] : 0xffffffffu;
        const unsigned l = lane < nw ? s_wl[lane] : 0xffffffffu;
        const double cmax = warp_max_nonneg(v);
        const bool qu = v >= 0.0 && qualifies(v, cmax);
        if (__any_sync(kFull, qu && v != cmax)) {
            winpos = local_pick(cand, lv, pos, cmax, winlc);
            return cmax;
        }
        const unsigned bp = __reduce_min_sync(kFull, qu ? p : 0xffffffffu);
        winlc = static_cast<int>(__reduce_min_sync(kFull, (qu && p == bp) ? l : 0xffffffffu));
        winpos = bp == 0xffffffffu ? INT_MAX : static_cast<int>(bp);
        return cmax;
    };

    // Trailing axpy y -= w v of this thread's rows for the current step.  The
    // norm downdate needs only w, so in cluster mode the axpy is deferred and
    // runs while the exchange for the next pivot is in flight.
    bool todo = false;
    double wpend = 0.0;
    int psr0 = 0;
    const double* pxa = xbuf;
    auto do_axpy = [&]() {
        if (!todo) return;
        todo = false;
        const double w = wpend;
        const double* xr = pxa + (l0 + q);
        int r = psr0;
        for (; r + 4 <= nsr; r += 4) {
            const int i = q + S * r;
            const double y0 = myrows[i], y1 = myrows[i + S], y2 = myrows[i + 2 * S], y3 = myrows[i + 3 * S];
            const double v0 = pxa[i], v1 = pxa[i + S], v2 = pxa[i + 2 * S], v3 = pxa[i + 3 * S];
            myrows[i] = fma(-w, v0, y0);
            myrows[i + S] = fma(-w, v1, y1);
            myrows[i + 2 * S] = fma(-w, v2, y2);
            myrows[i + 3 * S] = fma(-w, v3, y3);
        }
        for (; r < nsr; ++r) {
            const int i = q + S * r;
            myrows[i] = fma(-w, pxa[i], myrows[i]);
        }
        // straight-line over every register row (all reflector loads in flight
        // at once); v is zero on retired rows, so they keep their value without a
        // select (ncu: the select was 11 % of the kernel's instructions)
#pragma unroll
        for (int r = 0; r < R; ++r) yr[r] = fma(-w, xr[S * r], yr[r]);
    };

    // ---------------- cluster exchange (push, then all-local select) ----------------
    auto cl_slot = [&](int sl, int g) { return cslots + static_cast<size_t>(sl * G + g) * cslot; };  // push mode
    auto own_slot = [&](int sl) { return cslots + static_cast<size_t>(push ? sl * G + me : sl) * cslot; };
    auto hdr_of = [&](int sl, int g) -> double* {
        return push ? cl_slot(sl, g) + xlen : chdr + static_cast<size_t>(sl * G + g) * kCHdr;
    };

    // Stage this CTA's candidate in its own slot `sl`: header {col, tau, beta,
    // scale, vmax, pos} and v by absolute row, zeros on rows [lo, first).
    auto cl_stage = [&](int sl, double mx, int winpos, int winlc, int first, int lo) {
        const bool have = winpos != INT_MAX;
        double* own = own_slot(sl);
        double* hd = own + xlen;
        if (have && lc == winlc) {
            double al, tl;
            partials(first, al, tl);
            double tu, be, sc;
            reflector(al, tl, m - first, tu, be, sc);
            double* x = own;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int i = l0 + q + S * r;
                if (i >= first && i < m) x[i] = tu != 0.0 ? (i == first ? 1.0 : mul_rn(yr[r], sc)) : yr[r];
            }
            for (int r = first / S; r < nsr; ++r) {
                const int i = q + S * r;
                if (i >= first) x[i] = tu != 0.0 ? (i == first ? 1.0 : mul_rn(myrows[i], sc)) : myrows[i];
            }
            if (q == 0) {
                hd[0] = __longlong_as_double(c0 + winlc);
                hd[1] = tu;
                hd[2] = be;
                hd[3] = sc;
            }
        }
        for (int i = lo + tid; i < first; i += T) own[i] = 0.0;  // retired rows read v = 0
        if (tid == 0) {
            hd[4] = have ? mx : -1.0;
            hd[5] = __longlong_as_double(have ? static_cast<long long>(winpos) : 0xffffffffLL);
        }
    };

    // Tie slot (rare): plain DSMEM stores of the slot (push mode) or of the
    // header (pull mode) to every peer, then barrier.cluster.
    auto cl_push_slow = [&](int sl) {
        __syncthreads();
        cg::cluster_group cluster = cg::this_cluster();
        double* own = own_slot(sl);
        double* src = push ? own : own + xlen;
        double* dst = push ? own : hdr_of(sl, me);
        const int len = push ? cslot : kCHdr;
        if (!push && tid < kCHdr) dst[tid] = src[tid];
        const int tot = (G - 1) * len;
        for (int e = tid; e < tot; e += T) {
            const int gi = e / len, j = e - gi * len;
            const int g = gi < me ? gi : gi + 1;
            cluster.map_shared_rank(dst, g)[j] = src[j];
        }
        cluster.sync();
    };

    // Every warp reduces the G slot headers of `sl` from local shared memory
    // (identical result everywhere, no CTA barrier): winning CTA, its position.
    auto cl_select = [&](int sl, bool& amb, double& gmax, unsigned& bp) -> int {
        const double* h = hdr_of(sl, lane < G ? lane : 0);
        const double v = lane < G ? h[4] : -1.0;
        const unsigned p = lane < G ? static_cast<unsigned>(__double_as_longlong(h[5])) : 0xffffffffu;
        gmax = warp_max_nonneg(v);
        const bool qu = v >= 0.0 && qualifies(v, gmax);
        amb = __any_sync(kFull, qu && v != gmax);
        bp = __reduce_min_sync(kFull, qu ? p : 0xffffffffu);
        return static_cast<int>(__reduce_min_sync(kFull, (qu && p == bp) ? static_cast<unsigned>(lane) : 0xffffffffu));
    };

    // One cluster exchange, for the pivot of step `first`.  The winner group
    // of each CTA finishes its own column's update, stages it and pushes it
    // (warp-level ordering only); every other thread finishes its deferred
    // trailing update meanwhile, so that work overlaps the exchange.
    auto cluster_round = [&](int first, bool cand, double lv, long long pos, int step) {
        int winpos, winlc;
        const double mx = cta_argmax(cand, lv, pos, winpos, winlc);
        trace(step, 2);
        int sl = first & 1;
        const bool have = winpos != INT_MAX;
        const unsigned mb = smem_u32(&s_mbar[sl]);
        // The warp holding the winner column builds the next reflector with all
        // 32 lanes (its deferred update applied on the fly to a raw copy), so
        // the serial path is a few rows per lane, not the group's whole column.
        const int pw = have ? (winlc * S) >> 5 : 0;
        const bool pubwarp = wid == pw;
        // Tall candidates (pull mode, m - first > 32 * kPubRegs) are built by
        // kHelpWarps warps (the publishing warp and the ones after it): each
        // takes every kHelpWarps-th 32-row slice, the partial norms meet in
        // shared memory (named barrier 2), every helper evaluates the same
        // reflector and scales its own rows.
        // (compiled for S >= 4 only: the S = 1, 2 kernels serve m <= 128 in practice and
        // keep their register budget for the resident rows)
        const bool tall = S >= 4 && have && (m - first > 32 * kPubRegs);
        const int nh = tall ? min(kHelpWarps, nw) : 1;
        const int hi = (wid - pw + nw) % nw;
        bool built = false;
        if constexpr (S >= 4) {
        if (tall && hi < nh) {
            built = true;
            double* own = own_slot(sl);
            double* hd = own + xlen;
            const int lo = max(0, first - 2) & ~1;
            const unsigned bytes = push ? static_cast<unsigned>(xlen + kCHdr - lo) * sizeof(double)
                                        : static_cast<unsigned>(kCHdr * sizeof(double));
            const unsigned nthr = static_cast<unsigned>(nh * 32);
            if (pubwarp) {
                const int wl0 = (winlc * S) & 31;
                const double w0 = __shfl_sync(kFull, todo ? wpend : 0.0, wl0);  // 0: already current
                if (lc == winlc) {
#pragma unroll
                    for (int r = 0; r < R; ++r) xbuf[l0 + q + S * r] = yr[r];  // retired / padding rows too
                }
                if (lane == 0) s_help[kHelpWarps] = w0;
            }
            asm volatile("bar.sync 2, %0;" ::"r"(nthr) : "memory");
            trace_by(pubwarp && lane == 0, step, 8);
            const double ww = s_help[kHelpWarps];
            const double* wrow = rows + static_cast<size_t>(winlc) * lds;
            const int stride = 32 * nh;
            double tl = 0.0;
            for (int i0 = first + 32 * hi + lane; i0 < m; i0 += stride * kPubRegs) {
                double yv[kPubRegs];
#pragma unroll
                for (int t = 0; t < kPubRegs; ++t) {
                    const int i = i0 + stride * t;
                    yv[t] = i < m ? fma(-ww, xa[i], i < l0 ? wrow[i] : xbuf[i]) : 0.0;  // the group's axpy
                }
#pragma unroll
                for (int t = 0; t < kPubRegs; ++t) {
                    const int i = i0 + stride * t;
                    if (i < m) {
                        xbuf[i] = yv[t];
                        if (i == first) s_help[kHelpWarps + 1] = yv[t];
                        else tl = fma(yv[t], yv[t], tl);
                    }
                }
            }
            tl = warp_sum(tl);
            if (lane == 0) s_help[hi] = tl;
            asm volatile("bar.sync 2, %0;" ::"r"(nthr) : "memory");
            double tt = 0.0;
            for (int h = 0; h < nh; ++h) tt += s_help[h];  // fixed order: every helper gets the same sum
            const double al = s_help[kHelpWarps + 1];
            trace_by(pubwarp && lane == 0, step, 9);
            // the other warps may start their axpy now: the shared-memory-heavy part of the
            // publish (raw copy, pending update, norm) is done (named barrier 1)
            if (pubwarp) asm volatile("bar.arrive 1, %0;" ::"r"(T) : "memory");
            double tu, be, sc;
            reflector_warp(al, tt, m - first, tu, be, sc);
            trace_by(pubwarp && lane == 0, step, 10);
            for (int i0 = first + 32 * hi + lane; i0 < m; i0 += stride * kPubRegs) {
                double yv[kPubRegs];
#pragma unroll
                for (int t = 0; t < kPubRegs; ++t) yv[t] = i0 + stride * t < m ? xbuf[i0 + stride * t] : 0.0;
#pragma unroll
                for (int t = 0; t < kPubRegs; ++t) {
                    const int i = i0 + stride * t;
                    if (i < m) own[i] = tu != 0.0 ? (i == first ? 1.0 : mul_rn(yv[t], sc)) : yv[t];
                }
            }
            asm volatile("bar.sync 2, %0;" ::"r"(nthr) : "memory");  // every row of v is in the slot
            if (pubwarp) {
                if (lane == 0) {
                    hd[0] = __longlong_as_double(c0 + winlc);
                    hd[1] = tu;
                    hd[2] = be;
                    hd[3] = sc;
                }
                if (lane < first - lo) own[lo + lane] = 0.0;  // retired rows read v = 0
                if (lane == 0) {
                    hd[4] = have ? mx : -1.0;
                    hd[5] = __longlong_as_double(have ? static_cast<long long>(winpos) : 0xffffffffLL);
                    if (!push) {
                        double* mine = hdr_of(sl, me);
                        for (int j = 0; j < kCHdr; ++j) mine[j] = hd[j];
                    }
                }
                trace_by(lane == 0, step, 11);
                fence_proxy_async_smem();  // staging writes (generic proxy) -> bulk-copy reads (async proxy)
                __syncwarp();
                trace_by(lane == 0, step, 12);
                // the arrive releases the local staging to this CTA's waiters; the
                // peers' copies complete the transaction count
                if (lane == 0) mbar_expect_tx(mb, static_cast<unsigned>(G - 1) * bytes);
                if (lane < G - 1) {
                    const int g = lane < me ? lane : lane + 1;
                    const unsigned sa = smem_u32(push ? own + lo : hd);
                    const unsigned da = push ? sa : smem_u32(hdr_of(sl, me));
                    bulk_push(mapa_u32(da, g), sa, bytes, mapa_u32(mb, g));
                }
                trace_by(lane == 0, step, 3);
            } else {
                asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
            }
        }
        }
        if (built) {
        } else if (pubwarp) {
            double* own = own_slot(sl);
            double* hd = own + xlen;
            const int lo = max(0, first - 2) & ~1;
            const unsigned bytes = push ? static_cast<unsigned>(xlen + kCHdr - lo) * sizeof(double)
                                        : static_cast<unsigned>(kCHdr * sizeof(double));
            if (have) {
                const int wl0 = (winlc * S) & 31;
                const double ww = __shfl_sync(kFull, todo ? wpend : 0.0, wl0);  // 0: already current
                if (lc == winlc) {
#pragma unroll
                    for (int r = 0; r < R; ++r) xbuf[l0 + q + S * r] = yr[r];  // retired / padding rows too
                }
                __syncwarp();
                trace_by(lane == 0, step, 8);
                const double* wrow = rows + static_cast<size_t>(winlc) * lds;
                double al = 0.0, tl = 0.0;
                double tu, be, sc;
                if (m - first <= 32 * kPubRegs) {
                    // the updated rows stay in registers (kPubRegs per lane) between
                    // the norm and the scaled write
                    double yv[kPubRegs];
#pragma unroll
                    for (int t = 0; t < kPubRegs; ++t) {
                        const int i = first + lane + 32 * t;
                        yv[t] = 0.0;
                        if (i < m) {
                            const double y = fma(-ww, xa[i], i < l0 ? wrow[i] : xbuf[i]);  // == the group's own axpy
                            yv[t] = y;
                            if (i == first) al = y;
                            else tl = fma(y, y, tl);
                        }
                    }
                    al = __shfl_sync(kFull, al, 0);  // row `first` is lane 0's first row
                    tl = warp_sum(tl);
                    trace_by(lane == 0, step, 9);
                    asm volatile("bar.arrive 1, %0;" ::"r"(T) : "memory");  // see below
                    reflector_warp(al, tl, m - first, tu, be, sc);
                    trace_by(lane == 0, step, 10);
#pragma unroll
                    for (int t = 0; t < kPubRegs; ++t) {
                        const int i = first + lane + 32 * t;
                        if (i < m) own[i] = tu != 0.0 ? (i == first ? 1.0 : mul_rn(yv[t], sc)) : yv[t];
                    }
                } else {
                    // tall candidates (pull mode): kPubRegs rows per lane per batch,
                    // all loads of a batch issued before its stores
                    for (int i0 = first + lane; i0 < m; i0 += 32 * kPubRegs) {
                        double yv[kPubRegs];
#pragma unroll
                        for (int t = 0; t < kPubRegs; ++t) {
                            const int i = i0 + 32 * t;
                            yv[t] = i < m ? fma(-ww, xa[i], i < l0 ? wrow[i] : xbuf[i]) : 0.0;  // the group's axpy
                        }
#pragma unroll
                        for (int t = 0; t < kPubRegs; ++t) {
                            const int i = i0 + 32 * t;
                            if (i < m) {
                                xbuf[i] = yv[t];
                                if (i == first) al = yv[t];
                                else tl = fma(yv[t], yv[t], tl);
                            }
                        }
                    }
                    al = __shfl_sync(kFull, al, 0);
                    tl = warp_sum(tl);
                    trace_by(lane == 0, step, 9);
                    asm volatile("bar.arrive 1, %0;" ::"r"(T) : "memory");
                    reflector_warp(al, tl, m - first, tu, be, sc);
                    trace_by(lane == 0, step, 10);
                    for (int i0 = first + lane; i0 < m; i0 += 32 * kPubRegs) {
                        double yv[kPubRegs];
#pragma unroll
                        for (int t = 0; t < kPubRegs; ++t) yv[t] = i0 + 32 * t < m ? xbuf[i0 + 32 * t] : 0.0;
#pragma unroll
                        for (int t = 0; t < kPubRegs; ++t) {
                            const int i = i0 + 32 * t;
                            if (i < m) own[i] = tu != 0.0 ? (i == first ? 1.0 : mul_rn(yv[t], sc)) : yv[t];
                        }
                    }
                }
                if (lane == 0) {
                    hd[0] = __longlong_as_double(c0 + winlc);
                    hd[1] = tu;
                    hd[2] = be;
                    hd[3] = sc;
                }
            }
            if (lane < first - lo) own[lo + lane] = 0.0;  // retired rows read v = 0
            if (lane == 0) {
                hd[4] = have ? mx : -1.0;
                hd[5] = __longlong_as_double(have ? static_cast<long long>(winpos) : 0xffffffffLL);
                if (!push) {
                    double* mine = hdr_of(sl, me);
                    for (int j = 0; j < kCHdr; ++j) mine[j] = hd[j];
                }
            }
            trace_by(lane == 0, step, 11);
            fence_proxy_async_smem();  // staging writes (generic proxy) -> bulk-copy reads (async proxy)
            __syncwarp();
            trace_by(lane == 0, step, 12);
            // the arrive releases the local staging to this CTA's waiters; the
            // peers' copies complete the transaction count
            if (lane == 0) mbar_expect_tx(mb, static_cast<unsigned>(G - 1) * bytes);
            if (lane < G - 1) {
                const int g = lane < me ? lane : lane + 1;
                const unsigned sa = smem_u32(push ? own + lo : hd);
                const unsigned da = push ? sa : smem_u32(hdr_of(sl, me));
                bulk_push(mapa_u32(da, g), sa, bytes, mapa_u32(mb, g));
            }
            trace_by(lane == 0, step, 3);
            // The other warps' axpys contend for shared memory, so they wait on named barrier 1
            // -- but only until the shared-memory-heavy part of the publish (raw copy, pending
            // update, norm) is done: the arrive sits right after the norm above, and here for a
            // CTA without a candidate.
            if (!have) asm volatile("bar.arrive 1, %0;" ::"r"(T) : "memory");
        } else {
            asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
        }
        do_axpy();
        trace(step, 7);
        mbar_wait(mb, (mbar_phase >> sl) & 1u);
        mbar_phase ^= 1u << sl;
        trace(step, 4);
        bool amb;
        double gmax;
        unsigned bp;
        int gw = cl_select(sl, amb, gmax, bp);
        if (amb) {
            // exact tie pass: lowest position with sqrt(live) >= the global threshold
            const int wp2 = local_pick(cand, lv, pos, gmax, winlc);
            sl = 2;
            cl_stage(2, 0.0, wp2, winlc, first, 0);
            cl_push_slow(2);
            gw = cl_select(2, amb, gmax, bp);
        }
        const double* h = hdr_of(sl, gw);
        piv = __double_as_longlong(h[0]);
        tau = h[1];
        beta = h[2];
        ppos = bp;
        if (push) {
            xa = cl_slot(sl, gw);
        } else {  // pull the winner's rows over DSMEM into the reflector buffer of this parity
            const double* src = cg::this_cluster().map_shared_rank(own_slot(sl), gw);
            double* xb = xpull + (first & 1) * xlen;
            for (int i = tid; i < xlen; i += T) xb[i] = (i >= first && i < m) ? src[i] : 0.0;
            __syncthreads();
            xa = xb;
        }
        trace(step, 5);
    };

    // ---------------- grid exchange (tagged records in L2) ----------------
    auto slot_ptr = [&](int slot, int g) -> double* { return a.slots + (static_cast<size_t>(slot) * G + g) * gslot; };
    // copy c of a slot (c = 0 is slot_ptr itself)
    auto slot_copy = [&](double* base, int c) -> double* { return base + static_cast<size_t>(c) * 3 * G * gslot; };

    // Publish this CTA's candidate (local index winlc, position winpos) for the
    // exchange `tag` in `slot`: header + rows first..m-1, then the record.
    auto publish = [&](int slot, unsigned tag, double mx, int winpos, int winlc, int first) {
        const bool have = winpos != INT_MAX;
        double* dst = slot_ptr(slot, me);
        if (have && lc == winlc) {
            double al, tl;
            partials(first, al, tl);
            double tu, be, sc;
            reflector(al, tl, m - first, tu, be, sc);
#pragma unroll
            for (int cp = 0; cp < kColCopies; ++cp) {
                double* dc = slot_copy(dst, cp);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = l0 + q + S * r;
                    if (i >= first && i < m) dc[kHdr + i - first] = yr[r];
                }
                if (q == 0) {
                    dc[0] = __longlong_as_double(c0 + winlc);
                    dc[1] = tu;
                    dc[2] = be;
                    dc[3] = sc;
                }
            }
        }
        if (have) {  // shared-memory rows of the candidate, copied by everyone
            const double* cr = rows + static_cast<size_t>(winlc) * lds;
            for (int cp = 0; cp < kColCopies; ++cp)
                for (int i = first + tid; i < l0; i += T) slot_copy(dst, cp)[kHdr + i - first] = cr[i];
        }
        cta_sync();
        if (tid < kColCopies) {
            __threadfence();  // slot data before its ready flag (release)
            if (have) st_relaxed_u64(reinterpret_cast<unsigned long long*>(slot_copy(dst, tid) + 4), a.epoch | tag);
        }
        if (tid == 0) {
            const unsigned pos32 = have ? static_cast<unsigned>(winpos) : 0xffffffffu;
            const unsigned long long vb = static_cast<unsigned long long>(__double_as_longlong(mx));
            unsigned long long* rp = a.rec + (static_cast<size_t>(slot) * G + me) * kRecWords;
            st_relaxed_v2(rp, tagged(static_cast<unsigned>(vb >> 32), tag), tagged(static_cast<unsigned>(vb), tag));
            st_relaxed_v2(rp + 2, tagged(pos32, tag), 0ull);
        }
    };

    // Record of CTA g for exchange `tag`: {vmax, pos}; spins until all three
    // words carry the tag.
    auto read_rec = [&](int slot, int g, unsigned tag, double& vmax, unsigned& pos) {
        const unsigned long long* rp = a.rec + (static_cast<size_t>(slot) * G + g) * kRecWords;
        unsigned long long x0, x1, x2, x3;
        for (;;) {
            ld_relaxed_v2(rp, x0, x1);
            ld_relaxed_v2(rp + 2, x2, x3);
            if (static_cast<unsigned>(x0) == tag && static_cast<unsigned>(x1) == tag && static_cast<unsigned>(x2) == tag)
                break;
        }
        vmax = __longlong_as_double(static_cast<long long>(((x0 >> 32) << 32) | (x1 >> 32)));
        pos = static_cast<unsigned>(x2 >> 32);
    };

    constexpr int kRecPerLane = 5;  // G <= 160

    // Wait for every CTA's record of exchange `tag`, reduce them (identical in
    // every CTA), then copy the winner's column -- scaled by its reflector --
    // into xbuf.  `first` = the step the new pivot is for.
#ifdef IDK_CPQR_TRACE
    unsigned epoch = 0;
#endif
    auto grid_exchange = [&](int parity, unsigned tag, int first, bool cand, double lv, long long pos, int step) {
#ifdef IDK_CPQR_TRACE
        if (a.barrier != nullptr) grid_barrier(a.barrier, epoch);  // debug builds: IDK_DEBUG_GRID_BARRIER
#endif
        int slot = parity;
        // every thread polls at most a few records, all in flight at once:
        // one L2 round trip after the last arrival instead of one per record.
        // When every record has its own thread (T >= G), each polling warp also
        // reduces its 32 records before the barrier, so afterwards a warp combines
        // <= 8 warp records instead of all G (ncu: the G-record reduction in every
        // warp was 16 % of the kernel's instructions); a near tie at either level
        // falls back to the exact reduction over all records below.
        const bool two_level = T >= G && G <= 32 * kPollWarps;
        for (int g = tid; g < G; g += T) {
            double vv;
            unsigned pp;
            read_rec(parity, g, tag, vv, pp);
            s_rv[g] = vv;
            s_rp[g] = pp;
        }
        if (two_level && wid < (G + 31) / 32) {
            const double vv = tid < G ? s_rv[tid] : -1.0;  // this thread's own record
            const unsigned pp = tid < G ? s_rp[tid] : 0xffffffffu;
            const double wm = warp_max_nonneg(vv);
            const bool qu = vv >= 0.0 && qualifies(vv, wm);
            const bool wamb = __any_sync(kFull, qu && vv != wm);
            const unsigned wp = __reduce_min_sync(kFull, qu ? pp : 0xffffffffu);
            const unsigned wg = __reduce_min_sync(kFull, (qu && pp == wp) ? static_cast<unsigned>(tid) : 0xffffffffu);
            if (lane == 0) {
                s_gv[wid] = wm;
                s_gp[wid] = wp;
                s_gg[wid] = wamb ? 0xfffffffeu : wg;
            }
        }
        cta_sync();  // records are self-contained; the slot is acquired through its ready flag
        trace(step, 4);
        int gsel = -1;
        unsigned wsel = 0xffffffffu;
        bool done = false;
        if (two_level) {
            const int npw = (G + 31) / 32;
            const double v = lane < npw ? s_gv[lane] : -1.0;
            const unsigned p = lane < npw ? s_gp[lane] : 0xffffffffu;
            const unsigned gg = lane < npw ? s_gg[lane] : 0xffffffffu;
            const double cmax = warp_max_nonneg(v);
            const bool qu = v >= 0.0 && qualifies(v, cmax);
            if (!__any_sync(kFull, (qu && v != cmax) || gg == 0xfffffffeu)) {
                wsel = __reduce_min_sync(kFull, qu ? p : 0xffffffffu);
                gsel = static_cast<int>(__reduce_min_sync(kFull, (qu && p == wsel) ? gg : 0xffffffffu));
                done = wsel != 0xffffffffu;
            }
        }
        if (!done)
        // every warp reduces the G records from shared memory (identical
        // result everywhere): no second CTA barrier before the column copy
        {
            double v[kRecPerLane];
            unsigned p[kRecPerLane];
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) {
                const int g = lane + 32 * t;
                v[t] = g < G ? s_rv[g] : -1.0;
                p[t] = g < G ? s_rp[g] : 0xffffffffu;
            }
            double vmax = -1.0;
#pragma unroll
            for (int t = 0; t < kRecPerLane; ++t) vmax = fmax(vmax, v[t]);
            vmax = warp_max_nonneg(vmax);
            trace(step, 13);
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
            amb = __any_sync(kFull, amb);
            wsel = __reduce_min_sync(kFull, best);
            // positions are distinct, so exactly one lane holds the minimum
            gsel = static_cast<int>(__reduce_min_sync(
                kFull, (best == wsel && best != 0xffffffffu) ? static_cast<unsigned>(lane + 32 * bt) : 0xffffffffu));
            trace(step, 14);
            if (amb) {
                // Exact tie pass: lowest position with sqrt(live) >= the global threshold.
                int winlc;
                const int winpos = local_pick(cand, lv, pos, vmax, winlc);
                publish(2, tag, 0.0, winpos, winlc, first);
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
                    __threadfence();
                    const unsigned wb = __reduce_min_sync(kFull, b2);
                    if (b2 == wb && b2 != 0xffffffffu) {
                        s_sel[1] = wb;
                        s_sel[2] = g2;
                    }
                }
                cta_sync();
                wsel = static_cast<unsigned>(s_sel[1]);
                gsel = static_cast<int>(s_sel[2]);
            }
        }
        trace(step, 5);
        // All threads: header + winner's column (one round trip), scaled into xbuf by absolute row.
        const double* src = slot_copy(slot_ptr(slot, gsel), me % kColCopies);
        {  // the winner published its record before its column: wait for the column's ready flag
            const unsigned long long want = a.epoch | tag;
            const unsigned long long* fp = reinterpret_cast<const unsigned long long*>(src + 4);
            while (ld_acquire_u64(fp) != want) {
            }
        }
        const double h0 = __ldcg(src);
        const double tu = __ldcg(src + 1);
        const double be = __ldcg(src + 2);
        const double sc = __ldcg(src + 3);
        for (int i = tid; i < xlen; i += T) {
            double x = 0.0;
            if (i >= first && i < m) {
                x = __ldcg(src + kHdr + i - first);
                if (tu != 0.0) x = i == first ? 1.0 : mul_rn(x, sc);
            }
            xbuf[i] = x;
        }
        cta_sync();
        piv = __double_as_longlong(h0);
        ppos = wsel;
        tau = tu;
        beta = be;
        xa = xbuf;
    };

    // Grid round.  The warp holding the CTA's winner releases the tagged record, stages the
    // winner's register rows and hands the candidate to the publisher warp, which builds the
    // updated column with all 32 lanes (the winner's deferred update applied to the raw copy),
    // writes it to the L2 slot and sets its ready flags.  The publisher owns no columns and
    // takes no part in the workers' barriers, so no worker waits for the publish of its own
    // CTA (trace before: the publishing warp reached the exchange barrier 3.3 us after the
    // CTA argmax -- 2.4 us of publish plus its own axpy -- and every other warp waited there);
    // only the owner warp waits until the publisher has read the candidate's shared rows
    // before its axpy overwrites them.
    auto grid_round = [&](int first, bool cand, double lv, long long pos, int step) {
        int winpos, winlc;
        const double mx = cta_argmax(cand, lv, pos, winpos, winlc);
        trace(step, 2);
        const int parity = first & 1;
        const unsigned tag = static_cast<unsigned>(first + 1);
        const bool have = winpos != INT_MAX;
        const bool ownwarp = wid == (have ? (winlc * S) >> 5 : 0);
        if (ownwarp) {
            double* xscr = xpull;  // scratch (grid mode keeps the current reflector in xbuf)
            // the record first: the global reduction needs only (norm, position), so it
            // runs while the candidate column is built; readers wait for the column's
            // ready flag (written after a release fence) only for the winner
            if (lane == 0) {
                const unsigned pos32 = have ? static_cast<unsigned>(winpos) : 0xffffffffu;
                const unsigned long long vb = static_cast<unsigned long long>(__double_as_longlong(mx));
                unsigned long long* rp = a.rec + (static_cast<size_t>(parity) * G + me) * kRecWords;
                st_relaxed_v2(rp, tagged(static_cast<unsigned>(vb >> 32), tag), tagged(static_cast<unsigned>(vb), tag));
                st_relaxed_v2(rp + 2, tagged(pos32, tag), 0ull);
            }
            if (have) {
                const int wl0 = (winlc * S) & 31;
                const double ww = __shfl_sync(kFull, todo ? wpend : 0.0, wl0);  // 0: already current
                if (lc == winlc) {
#pragma unroll
                    for (int r = 0; r < R; ++r) xscr[l0 + q + S * r] = yr[r];  // retired / padding rows too: the scratch covers them
                }
                if (lane == 0) {
                    s_pubw = ww;
                    s_publc = winlc;
                }
            } else if (lane == 0) {
                s_publc = -1;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_mbar[0]));
            trace_by(lane == 0, step, 8);
            // With one or two threads per column the staging above is a long serial run of one
            // or two lanes on the winner's critical path: the other warps hold their axpy until
            // the hand-off (named barrier 1; cfg5 CPQR 0.4185 -> 0.4121 ms).  With wider groups
            // the staging is short and the barrier costs more than it gives (cfg4 +0.4 %).
            if constexpr (S <= 2) asm volatile("bar.arrive 1, %0;" ::"r"(T) : "memory");
            mbar_wait(smem_u32(&s_mbar[1]), static_cast<unsigned>(parity));  // candidate rows consumed
        } else {
            if constexpr (S <= 2) asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
        }
        do_axpy();
        trace(step, 7);
        grid_exchange(parity, tag, first, cand, lv, pos, step);
    };

    // The publisher warp's side of exchange `first`.
    auto grid_publish = [&](int first) {
        const int parity = first & 1;
        const unsigned tag = static_cast<unsigned>(first + 1);
        mbar_wait(smem_u32(&s_mbar[0]), static_cast<unsigned>(parity));
        const int winlc = s_publc;
        if (winlc >= 0) {
            const double ww = s_pubw;
            double* dst = slot_ptr(parity, me);
            const double* xscr = xpull;
            const double* wrow = rows + static_cast<size_t>(winlc) * lds;
            double al = 0.0, tl = 0.0;
            for (int i = first + lane; i < m; i += 32) {
                const double y = fma(-ww, xbuf[i], i < l0 ? wrow[i] : xscr[i]);  // == the group's own axpy
#pragma unroll
                for (int cp = 0; cp < kColCopies; ++cp) slot_copy(dst, cp)[kHdr + i - first] = y;
                if (i == first) al = y;
                else tl = fma(y, y, tl);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_mbar[1]));  // shared rows, scratch and reflector read
            al = __shfl_sync(kFull, al, 0);
            tl = warp_sum(tl);
            trace_by(lane == 0, first - 1, 9);
            if (lane < kColCopies) {
                double tu, be, sc;
                reflector(al, tl, m - first, tu, be, sc);
                double* dc = slot_copy(dst, lane);
                dc[0] = __longlong_as_double(c0 + winlc);
                dc[1] = tu;
                dc[2] = be;
                dc[3] = sc;
            }
            trace_by(lane == 0, first - 1, 10);
            __threadfence();  // the column before its ready flag (release)
            __syncwarp();
            trace_by(lane == 0, first - 1, 11);
            if (lane < kColCopies)
                st_relaxed_u64(reinterpret_cast<unsigned long long*>(slot_copy(dst, lane) + 4), a.epoch | tag);
        } else if (lane == 0) {
            mbar_arrive(smem_u32(&s_mbar[1]));
        }
        trace_by(lane == 0, first - 1, 3);
    };

    if (publisher) {
        if constexpr (!kCluster)
            for (int first = 0; first < a.k; ++first) grid_publish(first);
    } else {
    // ---- pivot 0 ----
    {
        const bool cand = active && q == 0;
        const double lv = cand ? s_live[lc] : -1.0;
        if constexpr (kCluster) cluster_round(0, cand, lv, cand ? s_pos[lc] : 0, -1);
        else grid_round(0, cand, lv, cand ? s_pos[lc] : 0, -1);
    }

    for (int s = 0; s < a.k; ++s) {
        trace(s, 0);
        if (me == 0 && tid == 0) {
            a.taus[s] = tau;
            a.pivots[s] = piv;
        }
        // Replay the swap on positions (qr.cpp:79-86); the group leader owns
        // its column's position, every member keeps a copy.
        long long mypos = -1;
        double live0 = 0.0, anchor0 = 0.0;
        if (active) {
            mypos = s_pos[lc];
            live0 = s_live[lc];
            anchor0 = s_anchor[lc];
            if (col == piv) mypos = s;
            else if (mypos == s) mypos = ppos;
        }
        __syncwarp();
        if (active && q == 0) s_pos[lc] = mypos;

        // ---- trailing update + downdate (qr.cpp:93-106) ----
        const int dreg = s - l0;
        const int rr0 = dreg <= 0 ? 0 : dreg / S;
        const int sr0 = s / S;
        const double* xr = xa + (l0 + q);  // xr[S*r] = v for register row r
        bool cand = false;
        double lv = -1.0;
        if (active && col == piv) {
            if (tau != 0.0) {  // the pivot column becomes [R; beta; v] like the reference's work
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = l0 + q + S * r;
                    if (i >= s && i < m) yr[r] = (i == s) ? beta : xa[i];
                }
                for (int r = sr0; r < nsr; ++r) {
                    const int i = q + S * r;
                    if (i >= s) myrows[i] = (i == s) ? beta : xa[i];
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
#pragma unroll 2
                for (; r + 4 <= nsr; r += 4) {
                    const int i = q + S * r;
                    const double y0 = myrows[i], y1 = myrows[i + S], y2 = myrows[i + 2 * S], y3 = myrows[i + 3 * S];
                    const double v0 = xa[i], v1 = xa[i + S], v2 = xa[i + 2 * S], v3 = xa[i + 3 * S];
                    d0 = fma(v0, y0, d0);
                    d1 = fma(v1, y1, d1);
                    d2 = fma(v2, y2, d2);
                    d3 = fma(v3, y3, d3);
                }
                for (; r < nsr; ++r) {
                    const int i = q + S * r;
                    d0 = fma(xa[i], myrows[i], d0);
                }
                // Every register row, retired ones included: v is zero above row s
                // (absolute-row addressing), so the extra terms add exact zeros, and
                // one straight-line block lets all R reflector loads issue back to
                // back instead of one load-use round trip per row.
#pragma unroll
                for (int r = 0; r < R; r += 4) {
                    const double v0 = xr[S * r], v1 = xr[S * (r + 1)], v2 = xr[S * (r + 2)], v3 = xr[S * (r + 3)];
                    d0 = fma(v0, yr[r], d0);
                    d1 = fma(v1, yr[r + 1], d1);
                    d2 = fma(v2, yr[r + 2], d2);
                    d3 = fma(v3, yr[r + 3], d3);
                }
                const double w = mul_rn(group_sum<S>((d0 + d1) + (d2 + d3)), tau);
                wpend = w;
                psr0 = sr0;
                pxa = xa;
                todo = true;
                head = ys - w;  // row s has v_0 = 1
            }
            lv = sub_rn(live0, mul_rn(head, head));
            if (lv < 0.0) lv = 0.0;
            if (lv <= mul_rn(kRecomp, anchor0)) {
                // fresh = sum_{i > s} y_i^2 (qr.cpp:101-104) of the updated column,
                // its rows formed on the fly exactly as the deferred axpy will
                // (same fma, same summation order as partials()); the axpy stays
                // pending, so no second inlined copy of it sits in the step loop
                const double ww = todo ? wpend : 0.0;
                const int first = s + 1;
                double a0 = 0.0, t0 = 0.0, t1 = 0.0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int i = l0 + q + S * r;
                    const double u = fma(-ww, xr[S * r], yr[r]);
                    if (i == first) a0 = u;
                    else if (i > first) {
                        if (r & 1) t1 = fma(u, u, t1);
                        else t0 = fma(u, u, t0);
                    }
                }
                for (int r = first / S; r < nsr; ++r) {
                    const int i = q + S * r;
                    const double u = fma(-ww, xa[i], myrows[i]);
                    if (i == first) a0 = u;
                    else if (i > first) t0 = fma(u, u, t0);
                }
                const double al = group_sum<S>(a0), tl = group_sum<S>(t0 + t1);
                lv = fma(al, al, tl);
                if (q == 0) s_anchor[lc] = lv;
            }
            if (q == 0) s_live[lc] = lv;
            cand = q == 0;
        }
        trace(s, 1);
        if (s + 1 == a.k) break;  // the last step's axpy runs after the loop

        // ---- next pivot: CTA candidate, exchange ----
        if constexpr (kCluster) cluster_round(s + 1, cand, lv, mypos, s);
        else grid_round(s + 1, cand, lv, mypos, s);
        trace(s, 6);
    }
    }  // workers

    do_axpy();
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
    if constexpr (kCluster) cg::this_cluster().sync();  // keep shared memory alive for DSMEM pushes
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

size_t resident_smem(int m, int nc, int l0, int lds, int S, int R, bool cluster, int G, bool push) {
    const int span = std::max(m, l0 + R * S);
    const size_t xlen = static_cast<size_t>((span + S + 1) & ~1);
    size_t d = 3 * xlen + static_cast<size_t>(nc) * lds + 2 * static_cast<size_t>(nc) + static_cast<size_t>(nc);
    if (cluster)  // + alignment pad
        d += (push ? 3 * static_cast<size_t>(G) * (kCHdr + xlen) : 3 * (kCHdr + xlen) + 3 * static_cast<size_t>(G) * kCHdr) + 2;
    return d * sizeof(double);
}

ResidentPlan plan_for(int m, int64_t n, int k, int G_target, bool cluster, size_t smem_cap, bool push) {
    ResidentPlan best;
    int64_t G = std::min<int64_t>(n, G_target);
    const int nc = static_cast<int>((n + G - 1) / G);
    G = (n + nc - 1) / nc;
    static const int Rs[2] = {32, 16};
    static const int Ss[6] = {32, 16, 8, 4, 2, 1};
    for (int R : Rs) {
        // grid mode adds the publisher warp to the launch (the launch bound counts it)
        const int maxT = (R >= 32 ? 512 : (R >= 16 ? 640 : 768)) - (cluster ? 0 : 32);
        for (int S : Ss) {
            const int threads = ((S * nc + 31) / 32) * 32;
            if (threads > maxT || threads < 32) continue;
            const int reg_rows = R * S;
            // skip plans whose register rows are mostly padding (a smaller R covers m)
            if (R > 16 && (R / 2) * S >= m) continue;
            int l0 = std::max(0, m - reg_rows);
            l0 = ((l0 + S - 1) / S) * S;  // uniform loop bounds need S | l0
            const int lds = pad_lds(l0, S);
            const size_t smem = resident_smem(m, nc, l0, lds, S, R, cluster, static_cast<int>(G), push);
            if (smem > smem_cap) continue;
            // cost model: per-step serial work of one thread (register rows are
            // cheap, shared rows cost ~3 LDS/STS each) -- the step latency --
            // plus a small throughput term for the threads it takes.
            const double cost = (R + 3.0 * (l0 / S)) + threads / 256.0;
            if (!best.ok || cost < best.cost) {
                best.ok = true;
                best.cluster = cluster;
                best.push = cluster && push;
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
ResidentPlan cpqr_resident_plan(int m, int64_t n, int k, int num_sms, int cluster_pref) {
    const size_t cap = 200 * 1024;
    if (cluster_pref != 1 && n >= 32) {
        ResidentPlan p;
        if (cluster_pref == 0) p = plan_for(m, n, k, 16, true, cap, true);
        if (!p.ok) p = plan_for(m, n, k, 16, true, cap, false);
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
        if (cluster_pref == 2) return ResidentPlan();
    }
    return plan_for(m, n, k, num_sms, false, cap, false);
}

long long* g_trace = nullptr;  // debug: set by idk_debug_cpqr_trace

void cpqr_resident_set_trace(long long* p) { g_trace = p; }

size_t cpqr_resident_exchange_bytes(const ResidentPlan& p, int m) {
    if (!p.ok || p.cluster) return 0;
    const size_t G = static_cast<size_t>(p.G);
    const size_t slot_len = kHdr + static_cast<size_t>((m + 1) & ~1);
    return sizeof(unsigned long long) * kRecWords * 3 * G + sizeof(double) * kColCopies * 3 * G * slot_len + 256;
}

cudaError_t cpqr_resident_launch(const ResidentPlan& p, double* W, int64_t ldw, int m, int64_t n, int k,
                                 long long* pos_out, long long* pivots, double* taus, void* exch, unsigned* barrier,
                                 cudaStream_t stream, const double* Win, int64_t ldin) {
    ResidentArgs a;
    a.W = W;
    a.ldw = ldw;
    a.Win = Win ? Win : W;
    a.ldin = Win ? ldin : ldw;
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
    a.push = p.push ? 1 : 0;
    static unsigned long long launch_epoch = 0;  // grid slot flags of an earlier launch never match
    a.epoch = (++launch_epoch) << 32;
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
    return cudaLaunchCooperativeKernel(fn, dim3(p.G), dim3(p.threads + 32), args, p.smem, stream);  // + the publisher warp
}

}  // namespace idk
