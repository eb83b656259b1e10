// Thread tiers: one unit per thread, the restricted band of K folded
// diagonals held in registers (K = 16, 24, 32, 48, 64).  Exact reference
// semantics (proj/src/align.cpp:37-155); see xb_kernels.cuh for the
// coordinate system, the drift-space values and the exact running-best chain.
//
// Per slot and antidiagonal the DNA kernel issues 7 instructions over the
// two integer pipes (B200 ALU pipe and FMA pipe, 16 lanes/clk per SMSP each):
//   ALU: VIMNMX3 (recurrence), VIADDMNMX (running best), ISETP (drop test)
//   FMA: IDP.4A (diagonal + score), IMAD (slot key), @p IMAD (kill),
//        @p IMAD (dead-mask bit)
// plus ~10 per 16 slots building the match words, and ~70 per antidiagonal
// of bookkeeping.  Table modes (other schemes) replace the IDP by a PRMT +
// shared-table load.
#include <climits>
#include <cstdint>
#include <utility>

#include "xb_kernels.cuh"

#ifndef XB_COUNTERS
#define XB_COUNTERS 0
#endif
#if XB_COUNTERS
#define XB_COUNT(i) (++xb_dbg[i])
__device__ unsigned long long xb_dbg_unused;
#else
#define XB_COUNT(i) ((void)0)
#endif

namespace xb {

__device__ __forceinline__ uint32_t range_bits(int lo, int hi) {
    if (lo > hi) return 0u;
    return (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo);
}

template <int K>
__device__ __forceinline__ void shift_slots(int32_t (&R)[K], int s) {
    // new slot k <- old slot k + s, vacated slots dead
    for (; s > 0; --s) {
#pragma unroll
        for (int k = 0; k < K - 1; ++k) R[k] = R[k + 1];
        R[K - 1] = kDeadS;
    }
    for (; s < 0; ++s) {
#pragma unroll
        for (int k = K - 1; k > 0; --k) R[k] = R[k - 1];
        R[0] = kDeadS;
    }
}

// rv_r / rh_r: symbols each reader consumes before the next refill point
template <int K, int MODE>
__device__ __forceinline__ void init_windows(TState<K, MODE>& S, const uint32_t* __restrict__ pool,
                                             int rv_r, int rh_r) {
    using St = TState<K, MODE>;
    const int fd = S.d >> 1, cd = S.d - fd;
    const int64_t a = int64_t(fd) - S.ubase - 1;  // v index of slot 0
    const int64_t b = int64_t(cd) + S.ubase - 1;  // h index of slot 0
    if constexpr (MODE == 0) {
#pragma unroll
        for (int w = 0; w < St::NW; ++w) {
            S.HW[w] = chunk_bf(pool, S.h_pos, S.hdir, b + 16 * w);
            S.VW[w] = chunk_tf(pool, S.v_pos, S.vdir, a - 16 * w - 15);
        }
        S.rv.init(pool, S.v_pos, S.vdir, a + 1, rv_r);
        S.rh.init(pool, S.h_pos, S.hdir, b + St::WK, rh_r);
    } else {
        constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
#pragma unroll
        for (int r = 0; r < St::NB; ++r) {
            uint32_t vw = 0, hw = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = 4 * r + q;
                vw |= code_at<ENC>(pool, S.v_pos, S.vdir, S.n, a - k) << (8 * q);
                hw |= code_at<ENC>(pool, S.h_pos, S.hdir, S.m, b + k) << (8 * q);
            }
            S.VW[r] = vw;
            S.HW[r] = hw;
        }
        S.rv.init(pool, S.v_pos, S.vdir, a + 1, rv_r);
        S.rh.init(pool, S.h_pos, S.hdir, b + St::WK, rh_r);
    }
}

// Table modes stream symbols without bounds checks, so once the band reaches
// past the matrix (d >= d_vm) the window bytes of slots whose v or h symbol
// lies past the view's end are overwritten with the sentinel code on every
// such step (its table row and column score -128: those cells never win).
template <int K, int MODE>
__device__ __forceinline__ void sentinel_windows(TState<K, MODE>& S, int d) {
    using St = TState<K, MODE>;
    const int fd = d >> 1, cd = d - fd;
    const int a = fd - S.ubase - 1;  // v index of slot 0
    const int b = cd + S.ubase - 1;  // h index of slot 0
    const int vhi = a - S.n;         // slots 0..vhi: v index >= n
    const int hlo = S.m - b;         // slots hlo..: h index >= m
#pragma unroll
    for (int r = 0; r < St::NB; ++r) {
        const int v1 = min(vhi - 4 * r, 3), h0 = max(hlo - 4 * r, 0);
        const uint32_t mv = v1 < 0 ? 0u : range_bits(0, 8 * v1 + 7);
        const uint32_t mh = h0 > 3 ? 0u : range_bits(8 * h0, 31);
        S.VW[r] = (S.VW[r] & ~mv) | (0x1F1F1F1Fu & mv);
        S.HW[r] = (S.HW[r] & ~mh) | (0x1F1F1F1Fu & mh);
    }
}

// First antidiagonal at which the band's slot range reaches past the matrix
// (i > n for slot 0, j > m for slot K-1) and the step must mask slots, and the
// first at which anything else forces the rare path (end of the matrix,
// pilot cap).
template <int K, int MODE>
__device__ __forceinline__ void set_limits(TState<K, MODE>& S) {
    S.d_vm = min(2 * (S.ubase + S.n + 1), 2 * (S.m - S.ubase - K + 2) - 1);
    S.d_lim = min(S.d_vm, min(S.n + S.m + 2, S.dcap + 1));
}

template <int K, int MODE>
__device__ __forceinline__ void start_unit(TState<K, MODE>& S, int32_t (&E)[K], int32_t (&O)[K],
                                           const TierParams& P, uint32_t unit, int32_t X, unsigned it) {
    const DevUnit u = P.units[unit];
    S.unit = int32_t(unit);
    S.h_pos = u.h_pos;
    S.v_pos = u.v_pos;
    S.m = u.h_len;
    S.n = u.v_len;
    S.hdir = u.dir & 1;
    S.vdir = (u.dir >> 1) & 1;
    S.d = 1;
    S.dcap = P.pilot ? P.pilot_cap : (INT_MAX >> 1);
    S.ubase = -(K / 2);
    S.hs1 = K / 2;  // antidiagonal 0: the origin, u = 0
    S.lr1 = 32 * TState<K, MODE>::NM - 1 - K / 2;
    S.hs2 = S.lr2 = -1;  // antidiagonal -1: empty
    S.stop = 0;
    set_limits(S);
    S.Tc = 64;  // 64 (T + beta d + 1) at d = 0, T = 0
    S.best_d = 0;
    S.best_u = 0;
    S.delta_w = 1;
    S.cells = 1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        O[k] = kDeadS;
        E[k] = (k == K / 2) ? X + 1 : kDeadS;  // s(0,0) = 0 + 0 + off
    }
    // started at the end of iteration it: consumption begins next iteration
    constexpr int PER = TState<K, MODE>::RPER;
    const int r = (PER - 1) - int(it & (PER - 1));
    init_windows(S, P.pool, r, r);
}

// Continues a unit from a resume record written by a narrower tier: the
// saved band is centred in this one, and the windows are rebuilt at d (at
// d-1 when d is even: that iteration only feeds the v symbol, see the loop).
template <int K, int MODE>
__device__ __forceinline__ void resume_unit(TState<K, MODE>& S, int32_t (&E)[K], int32_t (&O)[K],
                                            const TierParams& P, const int32_t* __restrict__ rec,
                                            unsigned it) {
    constexpr int KB = 32 * TState<K, MODE>::NM - 1;
    const int ko = rec[kRecK];
    const int off = (K - ko) >> 1;
    const int d = rec[kRecD];
    S.d = d;
    S.ubase = rec[kRecUbase] - off;
    S.Tc = rec[kRecTc];
    S.best_d = rec[kRecBestD];
    S.best_u = rec[kRecBestU];
    S.cells = rec[kRecCells];
    S.delta_w = rec[kRecDeltaW];
    const int h1 = rec[kRecHs1], l1 = rec[kRecLs1], h2 = rec[kRecHs2], l2 = rec[kRecLs2];
    S.hs1 = h1 < 0 ? -1 : h1 + off;
    S.lr1 = h1 < 0 ? -1 : KB - (l1 + off);
    S.hs2 = h2 < 0 ? -1 : h2 + off;
    S.lr2 = h2 < 0 ? -1 : KB - (l2 + off);
    set_limits(S);
    const bool odd = d & 1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int src = k - off;
        const bool in = src >= 0 && src < ko;
        const int32_t vc = in ? rec[kRecRows + src] : kDeadS;       // row d-2
        const int32_t vp = in ? rec[kRecRows + ko + src] : kDeadS;  // row d-1
        O[k] = odd ? vc : vp;
        E[k] = odd ? vp : vc;
    }
    constexpr int PER = TState<K, MODE>::RPER;
    const int r = (PER - 1) - int(it & (PER - 1));
    S.d = odd ? d : d - 1;
    init_windows(S, P.pool, r, r);
    S.d = d;
}

// ---- one slot -------------------------------------------------------------

struct SlotCtx {
    int32_t c;        // running chain value
    int32_t negC;     // -(64X + 63)
    int32_t r64, one, zero;
};

__device__ __forceinline__ int32_t imad_hi(uint32_t a, uint32_t b, int32_t c) {
    int32_t r;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
__device__ __forceinline__ int32_t imad(int32_t a, int32_t b, int32_t c) {
    int32_t r;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}

// single LOP3s (ptxas otherwise splits a two-constant AND/OR into two)
template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}
template <int LUT, uint32_t B>
__device__ __forceinline__ uint32_t lop3i(uint32_t a, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "n"(B), "r"(c), "n"(LUT));
    return d;
}

// Finishes a slot given its diagonal candidate db and gap sources ln/un:
// recurrence, key, running best, drop test, dead mask.
template <int k>
__device__ __forceinline__ int32_t slot_tail(int32_t db, int32_t ln, int32_t un, SlotCtx& X,
                                             uint32_t& dm) {
    int32_t cand = __vimax3_s32(db, ln, un);
    int32_t key;
    asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(key) : "r"(cand), "r"(X.r64), "n"(k));
    X.c = __viaddmax_s32(key, X.negC, X.c);
    asm("{\n\t.reg .pred p;\n\t"
        "setp.lt.s32 p, %2, %3;\n\t"
        "@p mad.lo.s32 %0, %0, %4, %6;\n\t"
        "@p mad.lo.u32 %1, %5, %7, %1;\n\t}"
        : "+r"(cand), "+r"(dm)
        : "r"(key), "r"(X.c), "r"(X.zero), "r"(X.one), "n"(kDeadS), "n"(1u << (k & 31)));
    return cand;
}

template <int K, int MODE, bool ODD, int k>
__device__ __forceinline__ void slot(int32_t (&cur)[K], const int32_t (&prv)[K],
                                     const uint32_t (&Z)[(K + 15) / 16][4],
                                     const TState<K, MODE>& S, const TierParams& P,
                                     const tab_t* __restrict__ tab, SlotCtx& X,
                                     uint32_t (&dm)[(K + 31) / 32]) {
    const int32_t dg = cur[k];
    int32_t db;
    if constexpr (MODE == 0) {
        // slot f = 4j + q of word w: byte j of Z[w][q] is 1 + 2*match = sim - 2*gap,
        // picked out by a one-hot byte weight (IDP.4A, FMA pipe)
        constexpr int w = k >> 4, f = k & 15, q = f & 3, j = f >> 2;
        db = __dp4a(int(Z[w][q]), 1 << (8 * j), dg);
    } else {
        constexpr int r = k >> 2, q = k & 3;
        // bytes: v code, h code, 0, 0 (sign-replicate of a code byte < 128)
        uint32_t idx;
        asm("prmt.b32 %0, %1, %2, %3;"
            : "=r"(idx) : "r"(S.VW[r]), "r"(S.HW[r]), "n"(q | ((q + 4) << 4) | ((8 | q) << 8) | ((8 | q) << 12)));
        db = imad(tab_lookup(tab, idx), X.one, dg);
    }
    int32_t ln, un;
    if constexpr (ODD) {  // gap sources at u and u+1
        ln = prv[k];
        un = (k < K - 1) ? prv[k < K - 1 ? k + 1 : k] : kDeadS;
    } else {              // gap sources at u-1 and u
        ln = (k > 0) ? prv[k > 0 ? k - 1 : k] : kDeadS;
        un = prv[k];
    }
    cur[k] = slot_tail<k>(db, ln, un, X, dm[k >> 5]);
}

template <int K, int MODE, bool ODD, int... ks>
__device__ __forceinline__ void all_slots(std::integer_sequence<int, ks...>, int32_t (&cur)[K],
                                          const int32_t (&prv)[K], const uint32_t (&Z)[(K + 15) / 16][4],
                                          const TState<K, MODE>& S, const TierParams& P,
                                          const tab_t* __restrict__ tab, SlotCtx& X,
                                          uint32_t (&dm)[(K + 31) / 32]) {
    // descending slot = ascending i: the order of the reference's running best
    (slot<K, MODE, ODD, K - 1 - ks>(cur, prv, Z, S, P, tab, X, dm), ...);
}

// Shifts the symbol windows for antidiagonal d+1 (the symbol entering the
// band after step d: v on odd d, h on even d).
template <int K, int MODE, bool ODD>
__device__ __forceinline__ void feed(TState<K, MODE>& S, const TierParams& P, int d) {
    using St = TState<K, MODE>;
    if constexpr (ODD) {  // floor((d+1)/2) grows: v[a+1] enters at slot 0
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = St::NW - 1; w > 0; --w) S.VW[w] = __funnelshift_l(S.VW[w - 1], S.VW[w], 2);
            S.VW[0] = __funnelshift_l(S.rv.cur, S.VW[0], 2);
            S.rv.cur <<= 2;
        } else {
            const uint32_t code = S.rv.take();
#pragma unroll
            for (int r = St::NB - 1; r > 0; --r) S.VW[r] = __funnelshift_l(S.VW[r - 1], S.VW[r], 8);
            S.VW[0] = (S.VW[0] << 8) | code;
        }
    } else {  // ceil((d+1)/2) grows: h[b+WK] enters at slot WK-1
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = 0; w < St::NW - 1; ++w) S.HW[w] = __funnelshift_r(S.HW[w], S.HW[w + 1], 2);
            S.HW[St::NW - 1] = __funnelshift_r(S.HW[St::NW - 1], S.rh.cur, 2);
            S.rh.cur >>= 2;
        } else {
            const uint32_t code = S.rh.take();
#pragma unroll
            for (int r = 0; r < St::NB - 1; ++r) S.HW[r] = __funnelshift_r(S.HW[r], S.HW[r + 1], 8);
            S.HW[St::NB - 1] = __funnelshift_r(S.HW[St::NB - 1], code, 8);
        }
    }
}

// Where a finished unit's outcome goes: its result row, the next tier's
// escalation list, or (pilot) the widest window seen.
struct Sink {
    uint32_t* esc_list;
    unsigned long long* esc_len;
    long long qidx;
    unsigned long long units, cells, esc;
    bool resumable;  // the next tier takes resume records (a thread or lane-group tier)
};

// Saves the band state of a unit that does not fit at antidiagonal d (the
// step has changed nothing yet: cur = row d-2, prv = row d-1) and returns
// the escalation-list entry: a record index, or the bare unit when the
// records are used up.
template <int K, int MODE>
__device__ __forceinline__ uint32_t save_resume(const TState<K, MODE>& S, const int32_t (&cur)[K],
                                                const int32_t (&prv)[K], const TierParams& P,
                                                int32_t beta) {
    constexpr int KB = 32 * TState<K, MODE>::NM - 1;
    int32_t* rec = nullptr;
    const uint32_t entry = alloc_record<K>(P, rec);
    if (!entry) return uint32_t(S.unit);
    rec[kRecUnit] = S.unit;
    rec[kRecD] = S.d;
    rec[kRecUbase] = S.ubase;
    rec[kRecTc] = S.Tc - (beta << 6);  // as before step d
    rec[kRecBestD] = S.best_d;
    rec[kRecBestU] = S.best_u;
    rec[kRecCells] = S.cells;
    rec[kRecDeltaW] = S.delta_w;
    rec[kRecHs1] = S.hs1;
    rec[kRecLs1] = S.hs1 < 0 ? -1 : KB - S.lr1;
    rec[kRecHs2] = S.hs2;
    rec[kRecLs2] = S.hs2 < 0 ? -1 : KB - S.lr2;
    rec[kRecK] = K;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        rec[kRecRows + k] = cur[k];
        rec[kRecRows + K + k] = prv[k];
    }
    return entry;
}

// Records the outcome of the current unit at the step that decides it (the
// rest of that loop iteration is dead work nobody reads) and sets S.stop.
template <int K, int MODE>
__device__ __forceinline__ void finish_unit(TState<K, MODE>& S, const TierParams& P, int code, int spread,
                                            Sink& sk, int32_t beta, const int32_t (&cur)[K],
                                            const int32_t (&prv)[K]) {
    S.stop = code;
    if (P.pilot) {
        P.pilot_w[sk.qidx] = code == kEscalate ? -1 : S.delta_w;
        return;
    }
    if (code == kEscalate) {
        const uint32_t entry = sk.resumable ? save_resume(S, cur, prv, P, beta) : uint32_t(S.unit);
        // a concurrent consumer may take the entry as soon as it is written:
        // the record first, then the slot, then the entry (volatile)
        __threadfence();
        const unsigned long long slot = atomicAdd(sk.esc_len, 1ull);
        XB_ASSERT(slot < P.ck_units, kChkList);
        *(volatile uint32_t*)&sk.esc_list[slot] = entry;
        ++sk.esc;
        return;
    }
    DevResult res;
    res.cells = S.cells;
    res.delta_w = S.delta_w;
    if (code == kBand) {
        res.score = res.h_ext = res.v_ext = 0;
        res.status = kStatusBand;
        res.spread = spread;
    } else {
        // Tc = 64 (T + beta d + 1) at the current d; the best cell sits on
        // antidiagonal best_d, folded diagonal best_u: i = floor(best_d/2) - best_u
        const int best_i = (S.best_d >> 1) - S.best_u;
        res.score = (S.Tc >> 6) - beta * S.d - 1;
        res.h_ext = S.best_d - best_i;
        res.v_ext = best_i;
        res.status = kStatusOk;
        res.spread = 0;
    }
    XB_ASSERT((unsigned long long)S.unit < P.ck_units, kChkResult);
    P.results[S.unit] = res;
    ++sk.units;
    sk.cells += (unsigned long long)S.cells;
}

__device__ __forceinline__ int bfind32(uint32_t x) {  // highest set bit, -1 for 0
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ int bfind64(uint64_t x) {
    int r;
    asm("bfind.u64 %0, %1;" : "=r"(r) : "l"(x));
    return r;
}

// One antidiagonal d.  cur holds d-2 on entry and d on exit, prv holds d-1.
// A step that decides the unit (finished, failing, outgrowing K) records the
// outcome and sets S.stop; the rest of the loop iteration is harmless dead
// work, which keeps a single exit test per iteration.
//
// Live ranges are kept as hs (highest live slot) and lr = KB - ls (KB =
// 32*NM - 1, ls = lowest live slot), both -1 for an empty row: exactly what
// bfind returns on the live mask and its bit reversal.  With that encoding
// the window of row d is one max per side, an empty row is neutral as long
// as the other row is not, and two empty rows give w <= 0 -- a rare-path
// trigger like every other exception.
template <int K, int MODE, bool ODD>
__device__ __forceinline__ void xstep(TState<K, MODE>& S, int32_t (&cur)[K], int32_t (&prv)[K],
                                      const TierParams& P, const tab_t* __restrict__ tab,
                                      int32_t gap, int32_t X, unsigned it, Sink& sk
#if XB_COUNTERS
                                      , unsigned long long (&xb_dbg)[8]
#endif
                                      ) {
    using St = TState<K, MODE>;
    constexpr int KB = 32 * St::NM - 1;
    XB_COUNT(0);
    const int d = S.d;
    const int32_t beta = -gap;
    S.Tc += beta << 6;  // the running best's drift: c_init of row d
    // Reachable window (align.cpp:68-81) in slot space: a gap step from row
    // d-1 reaches slots [ls1-1, hs1] (d odd) or [ls1, hs1+1] (d even), a
    // diagonal step from d-2 the same slots.  Below d_vm the band lies inside
    // the matrix, so the clamps of align.cpp:80-81 cannot bind.
    const int M = ODD ? max(S.lr1 + 1, S.lr2) : max(S.lr1, S.lr2);  // KB - s_lo
    const int s_hi = ODD ? max(S.hs1, S.hs2) : max(S.hs1 + 1, S.hs2);
    int wm1 = s_hi + M - KB;  // w - 1
    uint32_t vm[St::NM];
#pragma unroll
    for (int q = 0; q < St::NM; ++q) vm[q] = range_bits(0, min(K - 1 - 32 * q, 31));
    [[maybe_unused]] uint32_t inv[St::NW];  // both bits of slots outside the matrix
#pragma unroll
    for (int ww = 0; ww < St::NW; ++ww) inv[ww] = P.zero;
    // one rarely-taken branch for every way a step can stop, reshape or mask
    if ((M > KB || unsigned(s_hi) > unsigned(K - 1) || unsigned(wm1) >= unsigned(P.band) ||
         d >= S.d_lim) && !S.stop) {
        XB_COUNT(1);
        const bool e1 = S.hs1 < 0, e2 = S.hs2 < 0;
        if ((e1 && e2) || d > S.n + S.m + 1 || d > S.dcap) {
            finish_unit(S, P, kDone, 0, sk, beta, cur, prv);  // align.cpp:61-66
        } else {
            int lo = kBig, hi = -kBig;
            if (!e1) {
                lo = KB - S.lr1 - (ODD ? 1 : 0);
                hi = S.hs1 + (ODD ? 0 : 1);
            }
            if (!e2) {
                lo = min(lo, KB - S.lr2);
                hi = max(hi, S.hs2);
            }
            const int fd = d >> 1;
            int A = fd - S.ubase;  // slot k holds i = A - k
            // clamp to the matrix: i <= min(d, n)  and  i >= max(d - m, 0)
            const int w = min(hi, A - max(d - S.m, 0)) - max(lo, A - min(d, S.n)) + 1;
            if (w > P.band) {  // align.cpp:93-94: first overflow, cells so far
                finish_unit(S, P, kBand, w, sk, beta, cur, prv);
            } else {
                if (lo < 0 || hi > K - 1) {
                    // every live source lies inside the unclamped window, so it must fit
                    const int wu = hi - lo + 1;
                    if (wu > K) {
                        finish_unit(S, P, kEscalate, 0, sk, beta, cur, prv);
                    } else {
                        XB_COUNT(3);
                        const int sh = lo - ((K - wu) >> 1);  // new slot 0 = old slot sh
                        shift_slots<K>(cur, sh);
                        shift_slots<K>(prv, sh);
                        S.ubase += sh;
                        if (!e1) {
                            S.hs1 -= sh;
                            S.lr1 += sh;
                        }
                        if (!e2) {
                            S.hs2 -= sh;
                            S.lr2 += sh;
                        }
                        A -= sh;
                        set_limits(S);
                        // symbols left to consume before the next refill (iteration multiple
                        // of 16): this iteration's own consumption counts unless it happened
                        constexpr int PER = St::RPER;
                        const int to_refill = PER - int(it & (PER - 1));
                        init_windows(S, P.pool, ODD ? to_refill : to_refill - 1, to_refill);
                    }
                }
                if (!S.stop && d >= S.d_vm) {
                    XB_COUNT(2);
                    // slots inside the matrix: i <= n  <=>  k >= klo ;  j <= m  <=>  k <= khi
                    const int klo = A - S.n;
                    const int khi = S.m - (d - fd) - S.ubase;
                    const int khk = min(khi, K - 1);
#pragma unroll
                    for (int q = 0; q < St::NM; ++q)
                        vm[q] = range_bits(max(klo - 32 * q, 0), min(khk - 32 * q, 31));
                    if constexpr (MODE == 0) {
#pragma unroll
                        for (int ww = 0; ww < St::NW; ++ww) {
                            const int l = max(klo - 16 * ww, 0), h = min(khi - 16 * ww, 15);
                            inv[ww] = ~range_bits(2 * l, 2 * h + 1);
                        }
                    } else {
                        sentinel_windows(S, d);
                    }
                }
                wm1 = max(w, 0) - 1;  // a clamped-empty row counts no cells (align.cpp:84-90)
            }
        }
    }
    S.cells += wm1 + 1;
    S.delta_w = max(S.delta_w, wm1 + 1);

    // DNA +1/-1/-1: bit 2f+1 of z = ~(x | x << 1), x = (VW ^ HW) | inv, says
    // slot 16w+f is a match inside the matrix; Z[w][q] moves the bits of slots
    // f = 4j + q to bit 1 of byte j and sets bit 0: byte j = 1 + 2*match.
    // 6 ALU (LOP3) + 4 FMA (IMAD) per 16 slots.
    uint32_t Z[St::NW][4];
    if constexpr (MODE == 0) {
#pragma unroll
        for (int ww = 0; ww < St::NW; ++ww) {
            const uint32_t x = lop3<0xBE>(S.VW[ww], S.HW[ww], inv[ww]);  // (a ^ b) | c
            const uint32_t z = lop3<0x03>(x, uint32_t(imad(int32_t(x), P.two, P.zero)), P.zero);  // ~(a | b)
            Z[ww][0] = lop3i<0xEA, 0x02020202u>(z, P.ones);  // (a & b) | c
#pragma unroll
            for (int q = 1; q < 4; ++q)  // z >> 2q on the FMA pipe
                Z[ww][q] = lop3i<0xEA, 0x02020202u>(__umulhi(z, P.mulc[q]), P.ones);
        }
    }

    // exact running best + drop test: chain over k = K-1..0 (ascending i)
    SlotCtx C;
    C.c = S.Tc;  // (T + beta d + off - X) * 64
    C.negC = -((X << 6) + 63);
    C.r64 = P.r64;
    C.one = P.one;
    C.zero = P.zero;
    uint32_t dm[St::NM];
#pragma unroll
    for (int q = 0; q < St::NM; ++q) dm[q] = 0u;
    all_slots<K, MODE, ODD>(std::make_integer_sequence<int, K>{}, cur, prv, Z, S, P, tab, C, dm);

    // running best (align.cpp:123-127): strict improvement, first slot wins.
    // The chain ends above its start exactly when some cell beat T; then
    // (c + 63) rounds up to the new 64 (T' + beta d + 1) and its low bits are
    // the first attaining slot.
    if (C.c != S.Tc) {
        const int32_t c63 = C.c + 63;
        S.Tc = c63 & ~63;
        S.best_d = d;
        S.best_u = S.ubase + (c63 & 63);
    }
    // live slots of row d (align.cpp:138-145); out-of-matrix slots masked
    S.hs2 = S.hs1;
    S.lr2 = S.lr1;
    if constexpr (St::NM == 1) {
        const uint32_t lv = ~dm[0] & vm[0];
        S.hs1 = bfind32(lv);
        S.lr1 = bfind32(__brev(lv));
    } else {
        const uint64_t lv = (uint64_t(~dm[1] & vm[1]) << 32) | (~dm[0] & vm[0]);
        S.hs1 = bfind64(lv);
        S.lr1 = bfind64(__brevll(lv));
    }

    feed<K, MODE, ODD>(S, P, d);
    S.d = d + 1;
}

// resident blocks per SM the register budget is sized for
// (table modes hold two more readers' worth of state: one block fewer from K24)
template <int K, int MODE>
constexpr int tier_min_blocks() {
    return MODE == 0 ? (K <= 24 ? 4 : K <= 32 ? 3 : 2) : (K <= 16 ? 4 : K <= 24 ? 3 : 2);
}

template <int K, int MODE>
__global__ void __launch_bounds__(kTB, tier_min_blocks<K, MODE>()) thread_tier_kernel(TierParams P) {
    __shared__ tab_t tab[MODE == 0 ? 1 : kTabWords];
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    Queue Q;
    if (!make_queue(P, Q)) return;
    if constexpr (MODE != 0) {
        tab_fill(tab, P.scheme, gap);
        __syncthreads();
    }
    const int next_tier = P.esc_to_warp ? kWarpTier : P.tier + 1;
    Sink sk;
    sk.esc_list = P.lists + (long long)next_tier * P.n_units;
    sk.esc_len = &P.ctr->list_len[next_tier];
    sk.qidx = 0;
    sk.units = sk.cells = sk.esc = 0;
    sk.resumable = next_tier != kWarpTier && !P.pilot;
#if XB_COUNTERS
    unsigned long long xb_dbg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

    TState<K, MODE> S;
    int32_t E[K], O[K];
    bool active = false;
    // warp-uniform iteration counter (2 antidiagonals each); the first units
    // start "at the end of iteration -1"
    unsigned it = 0xFFFFFFFFu;
    auto fetch = [&]() {
        active = false;
        uint32_t e;
        while (Q.next(e, sk.qidx)) {
            uint32_t unit = e;
            const int32_t* rec = nullptr;
            if (e & kResumeFlag) {
                rec = record_ptr(P.resume, e);
                unit = uint32_t(rec[kRecUnit]);
            }
            XB_ASSERT(unit < P.ck_units, kChkUnit);
            // units whose values could leave the drift-space range go to the warp tier
            if (P.units[unit].route != 0) {
                if (P.pilot) P.pilot_w[sk.qidx] = -2;  // not a thread-tier unit
                continue;
            }
            start_unit<K, MODE>(S, E, O, P, unit, X, it);
            if (rec) resume_unit<K, MODE>(S, E, O, P, rec, it);
            active = true;
            return;
        }
    };
    fetch();
    it = 0;

    while (__any_sync(0xFFFFFFFFu, active)) {
        if (active) {
            if ((it & (TState<K, MODE>::RPER - 1)) == 0) {  // the same iteration for every thread
                S.rv.refill(P.pool);
                S.rh.refill(P.pool);
            }
            // iterations start on odd d, except right after a resume at an even
            // d, where the odd half only feeds its v symbol
#if XB_COUNTERS
            if (S.d & 1)
                xstep<K, MODE, true>(S, O, E, P, tab, gap, X, it, sk, xb_dbg);
            else
                feed<K, MODE, true>(S, P, S.d - 1);
            xstep<K, MODE, false>(S, E, O, P, tab, gap, X, it, sk, xb_dbg);
#else
            if (S.d & 1)
                xstep<K, MODE, true>(S, O, E, P, tab, gap, X, it, sk);
            else
                feed<K, MODE, true>(S, P, S.d - 1);
            xstep<K, MODE, false>(S, E, O, P, tab, gap, X, it, sk);
#endif
            if (S.stop) {  // outcome already recorded by the deciding step
                XB_COUNT(4);
                fetch();
            }
        }
        ++it;
    }
    if (P.pilot) return;
#if XB_COUNTERS
    for (int q = 0; q < 5; ++q) atomicAdd(&P.ctr->dbg[q], xb_dbg[q]);
#endif
    if (sk.units) atomicAdd(&P.ctr->units[P.tier], sk.units);
    if (sk.cells) atomicAdd(&P.ctr->cells[P.tier], sk.cells);
    if (sk.esc) atomicAdd(&P.ctr->escalated[P.tier], sk.esc);
    if (P.role == kRoleStart) {  // tell a concurrent escalation consumer when the last block is done
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&P.ctr->prod_done, 1u) == gridDim.x - 1) atomicExch(&P.ctr->prod_finished, 1);
        }
    }
}

#define XB_INST(K)                                                   \
    template __global__ void thread_tier_kernel<K, 0>(TierParams);   \
    template __global__ void thread_tier_kernel<K, 1>(TierParams);   \
    template __global__ void thread_tier_kernel<K, 2>(TierParams);
XB_INST(16)
XB_INST(24)
XB_INST(32)
XB_INST(48)
XB_INST(64)
#undef XB_INST

// Picks the start tier from the pilot sample: the width that minimises
// K_t + sum over wider tiers of (share escalating into them) * 1.5 * K.
// One block: the sample is counted by all threads, thread 0 decides.  The
// choice also goes straight to pinned host memory (host_out), so the host's
// read-back does not queue behind other batches' copies on a copy engine.
__global__ void select_tier_kernel(TierParams P, int forced, int32_t* host_out) {
    __shared__ unsigned long long need[kNarrowTiers];  // sample units needing more than tier t
    __shared__ unsigned long long nn;
    if (blockIdx.x != 0) return;
    if (forced >= 0) {
        if (threadIdx.x == 0) {
            P.ctr->start_tier = forced;
            *(volatile int32_t*)host_out = forced;
        }
        return;
    }
    if (threadIdx.x < kNarrowTiers) need[threadIdx.x] = 0;
    if (threadIdx.x == 0) nn = 0;
    __syncthreads();
    unsigned long long my_need[kNarrowTiers] = {0, 0, 0, 0, 0}, my_n = 0;
    for (long long q = threadIdx.x; q < P.pilot_n; q += blockDim.x) {
        const int pw = P.pilot_w[q];
        if (pw == -2) continue;
        const int w = pw < 0 ? (1 << 30) : pw + 2;  // +2: unclamped-window slack
        ++my_n;
        for (int t = 0; t < kNarrowTiers; ++t) my_need[t] += w > tier_width(t) && P.band > tier_width(t);
    }
    for (int t = 0; t < kNarrowTiers; ++t)
        if (my_need[t]) atomicAdd(&need[t], my_need[t]);
    if (my_n) atomicAdd(&nn, my_n);
    __syncthreads();
    if (threadIdx.x != 0) return;
    const double n = double(nn);
    int best = 4;
    double best_cost = 1e30;
    for (int t = 0; t < kNarrowTiers; ++t) {
        double cost = tier_width(t);
        for (int u = t + 1; u < kNarrowTiers; ++u)
            cost += 1.5 * tier_width(u) * (n > 0 ? double(need[u - 1]) / n : 0.0);
        if (cost < best_cost) {
            best_cost = cost;
            best = t;
        }
    }
    // Most of the sample outgrows K64: the whole batch starts on the wide
    // tiers, at K128.  (A K96 start measured slower on config 4 with X = 100:
    // 167 ms plus a 24 ms tail of the 2% of units that outgrow it, against
    // 179 ms at K128 with no tail; K96 stays as the tier K64 escalates into.)
    if (n > 0 && double(need[kNarrowTiers - 1]) > 0.5 * n) best = kWideFirst + 1;
    P.ctr->start_tier = best;
    *(volatile int32_t*)host_out = best;
}

}  // namespace xb
