// Wide tiers: G lanes per unit, K = 96 / 128 / 256 / 512 / 1024 slots of
// the restricted band in registers (S = K/G consecutive slots per lane;
// G = 8, 8, 16, 32, 32: four, four, two, one, one unit per warp).  They take the units whose
// live window outgrows the K64 tier -- large X, low identity, the
// reference's default band of 1024 (pipeline.hpp:28) -- which round 1 left
// to the generic warp tier's global-memory rows.
//
// Exact reference semantics (proj/src/align.cpp:37-155), same coordinates,
// drift-space values and window bookkeeping as the thread tier (see
// xb_kernels.cuh and xb_thread.cu).  What differs from the narrow tiers:
//   * the running best is carried in plain drift-space values, not 64x keys
//     (a slot index no longer fits 6 bits): the drop test of slot k is
//     s_k < max(Tv, max over earlier cells of s_j - X), a lane-local chain
//     seeded by a warp suffix-max over the higher lanes (5 shuffle rounds);
//   * the first cell attaining a new best (the reference's strict '>' in
//     ascending i) is the highest lane holding the antidiagonal maximum, and
//     within it the highest slot: one ballot, taken only on antidiagonals
//     that raise T (warp-uniform: the warp holds one unit);
//   * the live range is two warp reductions (max of the highest live slot,
//     min of the lowest) instead of a gathered bit mask;
//   * a recentre shifts the rows through shared memory (rare).
// The groups of a warp step in lockstep (as the lane-group tiers do): the
// main path uses full-warp shuffles segmented by G; a group whose step
// decides its unit records the outcome and finishes the iteration as dead
// work; the rare path and the fetch of the next unit are group-divergent and
// use the group's mask.  (One warp per unit at K128 cost 4x the instructions
// per cell of the K64 thread tier, measured on config 4 with X = 100:
// per-unit bookkeeping repeated on 32 lanes.)
#include <climits>
#include <cstdint>

#include "xb_kernels.cuh"

namespace xb {

namespace {

__device__ __forceinline__ uint32_t wbits(int lo, int hi) {
    if (lo > hi) return 0u;
    return (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo);
}

__device__ __forceinline__ int wbfind(uint32_t x) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}

template <int LUT>
__device__ __forceinline__ uint32_t wlop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

constexpr int kWideWarps = 4;  // warps per block
constexpr unsigned kFull = 0xFFFFFFFFu;

// Maximum / minimum over the G lanes of a group.  One warp per unit: REDUX.
// Smaller groups: butterfly shuffles on the segment (a REDUX on a partial
// mask compiles to a collective loop with divergent branches).
template <int G>
__device__ __forceinline__ int group_max(int v, unsigned m) {
    if constexpr (G == 32) return __reduce_max_sync(m, v);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(m, v, o, G));
    return v;
}
template <int G>
__device__ __forceinline__ int group_min(int v, unsigned m) {
    if constexpr (G == 32) return __reduce_min_sync(m, v);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(m, v, o, G));
    return v;
}

}  // namespace

template <int K, int G, int MODE>
struct WState {
    static constexpr int S = K / G;            // slots per lane
    static constexpr int NW = (S + 15) / 16;   // 2-bit window words per lane (MODE 0)
    static constexpr int NB = (S + 3) / 4;     // byte window words per lane (table modes)
    static constexpr int KB = K - 1;
    int64_t h_pos, v_pos;
    int32_t m, n, hdir, vdir, unit;
    int32_t d, ubase;
    int32_t lr1, hs1, lr2, hs2;  // hs / KB - ls of rows d-1, d-2; -1 for an empty row
    int32_t d_vm, d_lim, stop;
    int32_t Tv;                  // T + beta d + 1: the chain's start (= Tc / 64 of the narrow tiers)
    int32_t best_d, best_u, cells, delta_w;
    uint32_t VW[NW], HW[NW];     // 2-bit windows of this lane's S slots (MODE 0)
    uint32_t VWb[NB], HWb[NB];   // byte windows (table modes)
    static constexpr int RENC = MODE == 2 ? ENC_5BIT : ENC_2BIT;
    static constexpr int RPER = EncFields<RENC>::PER;
    Reader<true, RENC> rv;       // lane 0 of the group: v symbols entering slot 0
    Reader<false, RENC> rh;      // lane G-1: h symbols entering slot K-1
};

template <int K, int G, int MODE>
__device__ __forceinline__ void w_limits(WState<K, G, MODE>& S) {
    S.d_vm = min(2 * (S.ubase + S.n + 1), 2 * (S.m - S.ubase - K + 2) - 1);
    S.d_lim = min(S.d_vm, S.n + S.m + 2);
}

// symbol windows of this lane's slots at antidiagonal S.d, readers set up for
// rv_r / rh_r symbols before their next refill point (lanes 0 / G-1)
template <int K, int G, int MODE>
__device__ __forceinline__ void w_windows(WState<K, G, MODE>& S, const uint32_t* __restrict__ pool, int lane,
                                          int rv_r, int rh_r) {
    using St = WState<K, G, MODE>;
    constexpr int SS = St::S;
    const int fd = S.d >> 1, cd = S.d - fd;
    const int64_t a = int64_t(fd) - S.ubase - 1;  // v index of group slot 0
    const int64_t b = int64_t(cd) + S.ubase - 1;  // h index of group slot 0
    const int k0 = lane * SS;
    if constexpr (MODE == 0) {
#pragma unroll
        for (int w = 0; w < St::NW; ++w) {
            const int n_in = min(16, SS - 16 * w);
            const uint32_t keep = n_in >= 16 ? 0xFFFFFFFFu : ((1u << (2 * n_in)) - 1u);
            // slot s of word w <- v[a - k0 - 16w - s] at bits 2s; h[b + k0 + 16w + s]
            S.VW[w] = chunk_tf(pool, S.v_pos, S.vdir, a - k0 - 16 * w - 15);  // slots >= n_in: unused
            S.HW[w] = chunk_bf(pool, S.h_pos, S.hdir, b + k0 + 16 * w) & keep;
        }
    } else {
        constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
#pragma unroll
        for (int r = 0; r < St::NB; ++r) {
            uint32_t vw = 0, hw = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int s = 4 * r + q;
                if (s < SS) {
                    vw |= code_at<ENC>(pool, S.v_pos, S.vdir, S.n, a - k0 - s) << (8 * q);
                    hw |= code_at<ENC>(pool, S.h_pos, S.hdir, S.m, b + k0 + s) << (8 * q);
                }
            }
            S.VWb[r] = vw;
            S.HWb[r] = hw;
        }
    }
    // every lane of the group keeps both readers (same words, one transaction):
    // refills and feeds are then straight-line selects, not lane-0 branches
    S.rv.init(pool, S.v_pos, S.vdir, a + 1, rv_r);
    S.rh.init(pool, S.h_pos, S.hdir, b + K, rh_r);
}

// Table modes: sentinel bytes over slots whose v or h symbol lies past the
// view's end (see the thread tier's sentinel_windows).
template <int K, int G, int MODE>
__device__ __forceinline__ void w_sentinels(WState<K, G, MODE>& S, int d, int k0) {
    using St = WState<K, G, MODE>;
    const int fd = d >> 1, cd = d - fd;
    const int vhi = fd - S.ubase - 1 - S.n - k0;
    const int hlo = S.m - (cd + S.ubase - 1) - k0;
#pragma unroll
    for (int r = 0; r < St::NB; ++r) {
        const int v1 = min(vhi - 4 * r, 3), h0 = max(hlo - 4 * r, 0);
        const uint32_t mv = v1 < 0 ? 0u : wbits(0, 8 * v1 + 7);
        const uint32_t mh = h0 > 3 ? 0u : wbits(8 * h0, 31);
        S.VWb[r] = (S.VWb[r] & ~mv) | (0x1F1F1F1Fu & mv);
        S.HWb[r] = (S.HWb[r] & ~mh) | (0x1F1F1F1Fu & mh);
    }
}

// rows shifted by sh slots across the group (new slot k = old slot k + sh,
// vacated slots dead) through the group's shared-memory row
template <int SS, int G>
__device__ __forceinline__ void w_shift(int32_t (&R)[SS], int sh, int lane, int32_t* row, unsigned gmask) {
    constexpr int KK = G * SS;
    __syncwarp(gmask);
#pragma unroll
    for (int s = 0; s < SS; ++s) row[lane * SS + s] = R[s];
    __syncwarp(gmask);
#pragma unroll
    for (int s = 0; s < SS; ++s) {
        const int src = lane * SS + s + sh;
        R[s] = (src >= 0 && src < KK) ? row[src] : kDeadS;
    }
    XB_ASSERT(sh > -KK && sh < KK, kChkSmemRow);
    __syncwarp(gmask);
}

// Symbols entering on d+1 (v after an odd step, h after an even one).  FM:
// the whole warp executes the call (full-mask shuffles); else only the group.
template <int K, int G, int MODE, bool ODD, bool FM>
__device__ __forceinline__ void wfeed(WState<K, G, MODE>& S, int lane, unsigned gmask) {
    using St = WState<K, G, MODE>;
    constexpr int SS = St::S;
    const unsigned m = FM ? kFull : gmask;
    if constexpr (MODE == 0) {
        constexpr int NW = St::NW;
        constexpr int top = 2 * ((SS - 1) & 15);  // bit offset of slot SS-1 in the last word
        if constexpr (ODD) {  // v: slot k <- k-1, new symbol at slot 0 (lane 0's reader)
            const uint32_t out = (S.VW[NW - 1] >> top) & 3u;
            uint32_t in = __shfl_up_sync(m, out, 1, G);
            in = lane == 0 ? S.rv.cur >> 30 : in;
            S.rv.cur <<= 2;
#pragma unroll
            for (int w = NW - 1; w > 0; --w) S.VW[w] = __funnelshift_l(S.VW[w - 1], S.VW[w], 2);
            S.VW[0] = (S.VW[0] << 2) | in;
        } else {  // h: slot k <- k+1, new symbol at slot K-1 (lane G-1's reader)
            const uint32_t out = S.HW[0] & 3u;
            uint32_t in = __shfl_down_sync(m, out, 1, G);
            in = lane == G - 1 ? S.rh.cur & 3u : in;
            S.rh.cur >>= 2;
#pragma unroll
            for (int w = 0; w < NW - 1; ++w) S.HW[w] = __funnelshift_r(S.HW[w], S.HW[w + 1], 2);
            const uint32_t keep = top == 30 ? 0xFFFFFFFFu : ((1u << (top + 2)) - 1u);
            S.HW[NW - 1] = ((S.HW[NW - 1] >> 2) & (keep >> 2)) | (in << top);
        }
    } else {
        constexpr int NB = St::NB;
        constexpr int top = 8 * ((SS - 1) & 3);
        if constexpr (ODD) {
            const uint32_t out = (S.VWb[NB - 1] >> top) & 0xFFu;
            uint32_t in = __shfl_up_sync(m, out, 1, G);
            const uint32_t own = S.rv.take();
            in = lane == 0 ? own : in;
#pragma unroll
            for (int r = NB - 1; r > 0; --r) S.VWb[r] = __funnelshift_l(S.VWb[r - 1], S.VWb[r], 8);
            S.VWb[0] = (S.VWb[0] << 8) | in;
        } else {
            const uint32_t out = S.HWb[0] & 0xFFu;
            uint32_t in = __shfl_down_sync(m, out, 1, G);
            const uint32_t own = S.rh.take();
            in = lane == G - 1 ? own : in;
#pragma unroll
            for (int r = 0; r < NB - 1; ++r) S.HWb[r] = __funnelshift_r(S.HWb[r], S.HWb[r + 1], 8);
            const uint32_t keep = top == 24 ? 0xFFFFFFFFu : ((1u << (top + 8)) - 1u);
            S.HWb[NB - 1] = ((S.HWb[NB - 1] >> 8) & (keep >> 8)) | (in << top);
        }
    }
}

struct WSink {
    uint32_t* esc_list;
    unsigned long long* esc_len;
    unsigned long long units, cells, esc;
    bool resumable;
};

// Records the outcome of the group's unit at the deciding step (see the
// thread tier's finish_unit); the rest of that iteration is dead work.
template <int K, int G, int MODE>
__device__ __forceinline__ void wfinish(WState<K, G, MODE>& S, const TierParams& P, int code, int spread,
                                        WSink& sk, int32_t beta, const int32_t (&cur)[K / G],
                                        const int32_t (&prv)[K / G], int lane, unsigned gmask) {
    constexpr int SS = K / G;
    constexpr int KB = WState<K, G, MODE>::KB;
    S.stop = code;
    if (code == kEscalate) {
        uint32_t entry = uint32_t(S.unit);
        if constexpr (K < tier_width(kWarpTier - 1))  // the widest tier hands bare units to the warp tier
        if (sk.resumable) {
            int32_t* rec = nullptr;
            uint32_t got = 0u;
            if (lane == 0) got = alloc_record<K>(P, rec);
            got = __shfl_sync(gmask, got, 0, G);
            if (got) {
                rec = record_ptr(P.resume, got);
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    rec[kRecRows + lane * SS + s] = cur[s];
                    rec[kRecRows + K + lane * SS + s] = prv[s];
                }
                if (lane == 0) {
                    rec[kRecUnit] = S.unit;
                    rec[kRecD] = S.d;
                    rec[kRecUbase] = S.ubase;
                    rec[kRecTc] = (S.Tv - beta) << 6;  // as before step d, in 64x chain units
                    rec[kRecBestD] = S.best_d;
                    rec[kRecBestU] = S.best_u;
                    rec[kRecCells] = S.cells;
                    rec[kRecDeltaW] = S.delta_w;
                    rec[kRecHs1] = S.hs1;
                    rec[kRecLs1] = S.hs1 < 0 ? -1 : KB - S.lr1;
                    rec[kRecHs2] = S.hs2;
                    rec[kRecLs2] = S.hs2 < 0 ? -1 : KB - S.lr2;
                    rec[kRecK] = K;
                }
                entry = got;
            }
        }
        __syncwarp(gmask);
        if (lane == 0) {
            __threadfence();
            const unsigned long long slot = atomicAdd(sk.esc_len, 1ull);
            XB_ASSERT(slot < P.ck_units, kChkList);
            *(volatile uint32_t*)&sk.esc_list[slot] = entry;
            ++sk.esc;
        }
        return;
    }
    if (lane != 0) return;
    DevResult res;
    res.cells = S.cells;
    res.delta_w = S.delta_w;
    if (code == kBand) {
        res.score = res.h_ext = res.v_ext = 0;
        res.status = kStatusBand;
        res.spread = spread;
    } else {
        const int best_i = (S.best_d >> 1) - S.best_u;
        res.score = S.Tv - beta * S.d - 1;
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

// One antidiagonal d.  cur holds d-2 on entry and d on exit, prv holds d-1.
// FM: every group of the warp executes the step (main loop); else only this
// group (the even step of a unit resumed at an even d, inside fetch).
template <int K, int G, int MODE, bool ODD, bool FM>
__device__ __forceinline__ void wstep(WState<K, G, MODE>& S, int32_t (&cur)[K / G], int32_t (&prv)[K / G],
                                      const TierParams& P, const tab_t* __restrict__ tab, int32_t gap,
                                      int32_t X, unsigned it, int lane, unsigned gmask, WSink& sk,
                                      int32_t* srow) {
    using St = WState<K, G, MODE>;
    constexpr int SS = St::S;
    constexpr int KB = St::KB;
    const unsigned fm = FM ? kFull : gmask;
    const int d = S.d;
    const int k0 = lane * SS;
    const int32_t beta = -gap;
    S.Tv += beta;
    // window of row d, unclamped below d_vm (see the thread tier's xstep)
    const int M = ODD ? max(S.lr1 + 1, S.lr2) : max(S.lr1, S.lr2);  // KB - s_lo
    const int s_hi = ODD ? max(S.hs1, S.hs2) : max(S.hs1 + 1, S.hs2);
    int wm1 = s_hi + M - KB;
    uint32_t vml = wbits(0, SS - 1);  // this lane's in-matrix slots
    [[maybe_unused]] uint32_t inv[St::NW];
#pragma unroll
    for (int w = 0; w < St::NW; ++w) inv[w] = 0u;
    // group-uniform rare path (a decided unit's dead work skips it)
    if ((M > KB || unsigned(s_hi) > unsigned(K - 1) || unsigned(wm1) >= unsigned(P.band) || d >= S.d_lim) &&
        !S.stop) {
        const bool e1 = S.hs1 < 0, e2 = S.hs2 < 0;
        if ((e1 && e2) || d > S.n + S.m + 1) {
            wfinish<K, G, MODE>(S, P, kDone, 0, sk, beta, cur, prv, lane, gmask);  // align.cpp:61-66
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
            int A = fd - S.ubase;
            const int w = min(hi, A - max(d - S.m, 0)) - max(lo, A - min(d, S.n)) + 1;
            if (w > P.band) {  // align.cpp:93-94
                wfinish<K, G, MODE>(S, P, kBand, w, sk, beta, cur, prv, lane, gmask);
            } else {
                if (lo < 0 || hi > K - 1) {
                    const int wu = hi - lo + 1;
                    if (wu > K) {
                        wfinish<K, G, MODE>(S, P, kEscalate, 0, sk, beta, cur, prv, lane, gmask);
                    } else {
                        const int sh = lo - ((K - wu) >> 1);  // new slot 0 = old slot sh
                        w_shift<SS, G>(cur, sh, lane, srow, gmask);
                        w_shift<SS, G>(prv, sh, lane, srow, gmask);
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
                        w_limits(S);
                        constexpr int PER = St::RPER;
                        const int to_refill = PER - int(it & (PER - 1));
                        w_windows(S, P.pool, lane, ODD ? to_refill : to_refill - 1, to_refill);
                    }
                }
                if (!S.stop && d >= S.d_vm) {
                    // slots inside the matrix: i <= n  <=>  k >= klo ;  j <= m  <=>  k <= khi
                    const int klo = A - S.n;
                    const int khi = S.m - (d - fd) - S.ubase;
                    const int l = max(klo - k0, 0), h = min(min(khi, K - 1) - k0, SS - 1);
                    vml = wbits(l, h);
                    if constexpr (MODE == 0) {
#pragma unroll
                        for (int ww = 0; ww < St::NW; ++ww) {
                            const int lw = max(l - 16 * ww, 0), hw = min(h - 16 * ww, 15);
                            inv[ww] = ~((lw > hw) ? 0u : wbits(2 * lw, 2 * hw + 1));
                        }
                    } else {
                        w_sentinels(S, d, k0);
                    }
                }
                wm1 = max(w, 0) - 1;  // a clamped-empty row counts no cells (align.cpp:84-90)
            }
        }
    }
    S.cells += wm1 + 1;
    S.delta_w = max(S.delta_w, wm1 + 1);

    // gap source across the lane edge
    int32_t edge;
    if constexpr (ODD) {
        edge = __shfl_down_sync(fm, prv[0], 1, G);
        if (lane == G - 1) edge = kDeadS;
    } else {
        edge = __shfl_up_sync(fm, prv[SS - 1], 1, G);
        if (lane == 0) edge = kDeadS;
    }
    // match bytes (see the thread tier): byte j of Z[w][q] = 1 + 2*match of slot 16w + 4j + q
    [[maybe_unused]] uint32_t Z[St::NW][4];
    if constexpr (MODE == 0) {
#pragma unroll
        for (int ww = 0; ww < St::NW; ++ww) {
            const uint32_t x = wlop3<0xBE>(S.VW[ww], S.HW[ww], inv[ww]);  // (a ^ b) | c
            const uint32_t z = ~(x | (x << 1));
#pragma unroll
            for (int q = 0; q < 4; ++q) Z[ww][q] = ((z >> (2 * q)) & 0x02020202u) | 0x01010101u;
        }
    }
    // pass 1: candidates and the lane maximum
    int32_t cand[SS];
#pragma unroll
    for (int s = SS - 1; s >= 0; --s) {
        const int32_t dg = cur[s];
        int32_t db;
        if constexpr (MODE == 0) {
            db = __dp4a(int(Z[s >> 4][s & 3]), 1 << (8 * ((s >> 2) & 3)), dg);
        } else {
            const int r = s >> 2, q = s & 3;
            uint32_t idx = 0;
            switch (q) {  // bytes: v code, h code, 0, 0
                case 0: asm("prmt.b32 %0, %1, %2, 0x8840;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                case 1: asm("prmt.b32 %0, %1, %2, 0x9951;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                case 2: asm("prmt.b32 %0, %1, %2, 0xAA62;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                default: asm("prmt.b32 %0, %1, %2, 0xBB73;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
            }
            db = dg + tab_lookup(tab, idx);
        }
        int32_t ln, un;
        if constexpr (ODD) {  // gap sources at u and u+1
            ln = prv[s];
            un = s < SS - 1 ? prv[s < SS - 1 ? s + 1 : s] : edge;
        } else {              // gap sources at u-1 and u
            ln = s > 0 ? prv[s > 0 ? s - 1 : s] : edge;
            un = prv[s];
        }
        cand[s] = __vimax3_s32(db, ln, un);
    }
    // lane maximum with its highest slot: keys 64 cand + s (IMAD on the FMA
    // pipe; the ALU pipe carries the recurrence, chain and compares)
    int32_t mk = -(1 << 30);
#pragma unroll
    for (int s = SS - 1; s >= 0; s -= 2) {
        int32_t k1, k2;
        asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(k1) : "r"(cand[s]), "r"(P.r64), "r"(s));
        if (s >= 1) {
            asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(k2) : "r"(cand[s >= 1 ? s - 1 : 0]), "r"(P.r64), "r"(s - 1));
            mk = __vimax3_s32(mk, k1, k2);
        } else {
            mk = max(mk, k1);
        }
    }
    const int32_t mv = mk >> 6;
    // suffix maximum over the group's lanes (ascending i = descending lane)
    int32_t incl = mv;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const int32_t y = __shfl_down_sync(fm, incl, o, G);
        if (lane + o < G) incl = max(incl, y);
    }
    int32_t above = __shfl_down_sync(fm, incl, 1, G);
    if (lane == G - 1) above = -(1 << 30);
    const int32_t gmax = __shfl_sync(fm, incl, 0, G);
    // pass 2: the lane's chain (align.cpp:122-129: prune against the running
    // best, which includes the cell itself), drop test, live bits
    int32_t c = max(S.Tv, above - X);
    uint32_t dm = 0u;
    int32_t kept[SS];  // the row after the drop test
#pragma unroll
    for (int s = SS - 1; s >= 0; --s) {
        c = __viaddmax_s32(cand[s], -X, c);
        // kill and dead bit as predicated IMADs with opaque constants (FMA
        // pipe; the ALU pipe carries the max / compare chain), as in the
        // thread tier's slot_tail
        kept[s] = cand[s];
        asm("{\n\t.reg .pred p;\n\t"
            "setp.lt.s32 p, %2, %3;\n\t"
            "@p mad.lo.s32 %0, %0, %4, %6;\n\t"
            "@p mad.lo.u32 %1, %5, %7, %1;\n\t}"
            : "+r"(kept[s]), "+r"(dm)
            : "r"(cand[s]), "r"(c), "r"(P.zero), "r"(P.one), "n"(kDeadS), "r"(1u << (s & 31)));
    }
    // running best (align.cpp:123-127): strict improvement, first cell wins:
    // the highest lane holding the maximum, its highest slot holding it.
    // Branch-free (a group-divergent branch here stalled the lockstep warp
    // on branch resolution at most steps): the ballot and the shuffle run
    // every step and the update is a select.
    {
        const bool improve = gmax - X > S.Tv;
        const unsigned bal = __ballot_sync(fm, mv == gmax);
        const unsigned gb = G == 32 ? bal : (bal >> (threadIdx.x & 31 & ~(G - 1))) & ((1u << (G & 31)) - 1u);
        const int bl = 31 - __clz(gb);
        const int bs = __shfl_sync(fm, mk & 63, bl, G);
        S.best_u = improve ? S.ubase + bl * SS + bs : S.best_u;
        S.best_d = improve ? d : S.best_d;
        S.Tv = improve ? gmax - X : S.Tv;
    }
#pragma unroll
    for (int s = 0; s < SS; ++s) cur[s] = kept[s];
    // live slots of row d (align.cpp:138-145): two group reductions
    S.hs2 = S.hs1;
    S.lr2 = S.lr1;
    {
        const uint32_t lv = ~dm & vml;
        const int hs_l = lv ? k0 + wbfind(lv) : -1;
        const int ls_l = lv ? k0 + __ffs(lv) - 1 : kBig;
        const int hs = group_max<G>(hs_l, fm);
        const int ls = group_min<G>(ls_l, fm);
        S.hs1 = hs;
        S.lr1 = hs < 0 ? -1 : KB - ls;
    }
    wfeed<K, G, MODE, ODD, FM>(S, lane, gmask);
    S.d = d + 1;
}

// Resident blocks per SM the register budget is sized for: 128 registers
// at 4 blocks while S <= 16 (the 2-bit table mode needs ~160: 3 blocks).
template <int K, int G, int MODE>
constexpr int wide_min_blocks() {
    return K / G > 16 ? 1 : MODE == 1 ? 3 : 4;
}

// G lanes per unit.  G = 8 (four units per warp) is the throughput form,
// for a wide start tier over a whole batch; G = 32 (one unit per warp, the
// shortest step) serves escalations, which are few and latency-bound.
// kRoleConsumer (G = 32): takes the escalations of a wide start tier while
// it runs, with the lane-group consumer's protocol (xb_group.cu): claim a
// published slot, wait for its entry, leave once the start tier has
// finished and the list is drained; the tail dispatch takes what is left.
template <int K, int G, int MODE>
__global__ void __launch_bounds__(32 * kWideWarps, wide_min_blocks<K, G, MODE>()) wide_tier_kernel(TierParams P) {
    using St = WState<K, G, MODE>;
    constexpr int SS = St::S;
    constexpr int KB = St::KB;
    constexpr int PER = St::RPER;
    __shared__ tab_t tab[MODE == 0 ? 1 : kTabWords];
    __shared__ int32_t rows[kWideWarps * 32 / G][K];  // recentring scratch, one row per group
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    const int wl = threadIdx.x & 31;
    const int lane = wl % G;
    const int gbase = wl - lane;
    const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << gbase;
    int32_t* srow = rows[threadIdx.x / G];
    const int k0 = lane * SS;
    Queue Q;
    const bool consumer = P.role == kRoleConsumer;
    if (P.pilot || !make_queue(P, Q) || (!consumer && Q.len == 0)) return;
    if constexpr (MODE != 0) {
        tab_fill(tab, P.scheme, gap);
        __syncthreads();
    }
    const int next_tier = (P.esc_to_warp || P.tier + 1 >= kWarpTier) ? kWarpTier : P.tier + 1;
    WSink sk;
    sk.esc_list = P.lists + (long long)next_tier * P.n_units;
    sk.esc_len = &P.ctr->list_len[next_tier];
    sk.units = sk.cells = sk.esc = 0;
    sk.resumable = next_tier != kWarpTier;

    // Every group of the warp executes every step; a group without a unit
    // steps on harmless state with stop set (no rare path, no output, no
    // loads: its reader refills are skipped, its windows hold valid codes).
    St S;
    S.m = S.n = 0;
    S.stop = kDone;
    S.rv.cur = S.rh.cur = 0u;
    S.rv.w0 = S.rv.w1 = S.rh.w0 = S.rh.w1 = 0u;
    S.rv.sh = S.rh.sh = 0u;
#pragma unroll
    for (int w = 0; w < St::NW; ++w) S.VW[w] = S.HW[w] = 0u;
#pragma unroll
    for (int r = 0; r < St::NB; ++r) S.VWb[r] = S.HWb[r] = 0u;
    S.hs1 = S.hs2 = S.lr1 = S.lr2 = -1;
    S.Tv = 0;
    S.d = 1;
    S.ubase = 0;
    S.d_vm = S.d_lim = 1 << 30;
    int32_t E[SS], O[SS];
#pragma unroll
    for (int s = 0; s < SS; ++s) E[s] = O[s] = kDeadS;
    bool active = false;
    bool waiting = consumer;  // a consumer group with no unit, still looking for one
    unsigned it = 0xFFFFFFFFu;  // warp-uniform iteration counter (two antidiagonals each)
    // the group's next unit; runs at the end of iteration `it` (group-divergent)
    auto fetch = [&]() __attribute__((always_inline)) {
        active = false;
        for (;;) {
            unsigned long long i = Q.len;
            uint32_t e = 0;
            if (consumer) {
                int st = 0;  // 0 nothing queued yet, 1 claimed slot i (entry e), 2 done
                if (lane == 0) {
                    volatile unsigned long long* lenp = &P.ctr->list_len[P.tier];
                    volatile unsigned long long* curp = Q.cursor;
                    for (;;) {
                        // once the start tier has finished, the tail dispatch (a full
                        // grid) takes what is still queued: stop claiming
                        if (*(volatile int32_t*)&P.ctr->prod_finished) {
                            st = 2;
                            break;
                        }
                        const unsigned long long c = *curp;
                        if (c >= *lenp) break;  // nothing queued yet
                        if (atomicCAS(Q.cursor, c, c + 1) == c) {
                            i = c;
                            const volatile uint32_t* ep = Q.q + (long long)i;
                            while ((e = *ep) == kEmptyEntry) __nanosleep(64);
                            __threadfence();  // the entry's resume record is visible past this point
                            st = 1;
                            break;
                        }
                    }
                }
                st = __shfl_sync(gmask, st, 0, G);
                if (st != 1) {
                    waiting = st == 0;
                    S.stop = kDone;
                    S.m = S.n = 0;
                    return;
                }
                i = __shfl_sync(gmask, i, 0, G);
                e = __shfl_sync(gmask, e, 0, G);
            } else {
                // a plain read first: groups arriving after the queue ran dry leave
                // without queueing on the cursor's atomic
                if (lane == 0 && *(volatile unsigned long long*)Q.cursor < Q.len) i = atomicAdd(Q.cursor, 1ull);
                i = __shfl_sync(gmask, i, 0, G);
                if (i >= Q.len) {
                    S.stop = kDone;
                    S.m = S.n = 0;
                    return;
                }
                XB_ASSERT(i * Q.stride < P.ck_units, kChkList);
                e = Q.q[(long long)i * Q.stride];
            }
            uint32_t unit = e;
            const int32_t* rec = nullptr;
            if (e & kResumeFlag) {
                rec = record_ptr(P.resume, e);
                unit = uint32_t(__ldcg(rec + kRecUnit));
            }
            XB_ASSERT(unit < P.ck_units, kChkUnit);
            const DevUnit u = P.units[unit];
            if (u.route != 0) continue;  // guard failed: the warp tier's (prep listed it there)
            S.unit = int32_t(unit);
            S.h_pos = u.h_pos;
            S.v_pos = u.v_pos;
            S.m = u.h_len;
            S.n = u.v_len;
            S.hdir = u.dir & 1;
            S.vdir = (u.dir >> 1) & 1;
            S.stop = 0;
            const int r = (PER - 1) - int(it & (PER - 1));  // symbols before the next refill point
            if (!rec) {
                S.d = 1;
                S.ubase = -(K / 2);
                S.hs1 = K / 2;
                S.lr1 = KB - K / 2;
                S.hs2 = S.lr2 = -1;
                S.Tv = 1;  // T + beta d + 1 at d = 0, T = 0
                S.best_d = S.best_u = 0;
                S.delta_w = 1;
                S.cells = 1;
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    O[s] = kDeadS;
                    E[s] = (k0 + s == K / 2) ? X + 1 : kDeadS;  // s(0,0) = 0 + 0 + off
                }
                w_limits(S);
                w_windows(S, P.pool, lane, r, r);
            } else {
                // continue from a narrower tier's record, centred (see resume_unit)
                const int ko = __ldcg(rec + kRecK);
                const int off = (K - ko) >> 1;
                const int d = __ldcg(rec + kRecD);
                S.ubase = __ldcg(rec + kRecUbase) - off;
                S.Tv = __ldcg(rec + kRecTc) >> 6;
                S.best_d = __ldcg(rec + kRecBestD);
                S.best_u = __ldcg(rec + kRecBestU);
                S.cells = __ldcg(rec + kRecCells);
                S.delta_w = __ldcg(rec + kRecDeltaW);
                const int h1 = __ldcg(rec + kRecHs1), l1 = __ldcg(rec + kRecLs1);
                const int h2 = __ldcg(rec + kRecHs2), l2 = __ldcg(rec + kRecLs2);
                S.hs1 = h1 < 0 ? -1 : h1 + off;
                S.lr1 = h1 < 0 ? -1 : KB - (l1 + off);
                S.hs2 = h2 < 0 ? -1 : h2 + off;
                S.lr2 = h2 < 0 ? -1 : KB - (l2 + off);
                const bool odd = d & 1;
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    const int src = k0 + s - off;
                    const bool in = src >= 0 && src < ko;
                    const int32_t vc = in ? __ldcg(rec + kRecRows + src) : kDeadS;       // row d-2
                    const int32_t vp = in ? __ldcg(rec + kRecRows + ko + src) : kDeadS;  // row d-1
                    O[s] = odd ? vc : vp;
                    E[s] = odd ? vp : vc;
                }
                // the loop steps odd then even antidiagonals; a record at an even d
                // runs its even step here (readers set up with a full refill period:
                // this happens before the next refill point), and the group joins
                // the loop at an odd d
                S.d = odd ? d : d - 1;
                w_windows(S, P.pool, lane, odd ? r : PER - 1, odd ? r : PER - 1);
                S.d = d;
                w_limits(S);
                if (!odd) {
                    wfeed<K, G, MODE, true, false>(S, lane, gmask);
                    wstep<K, G, MODE, false, false>(S, E, O, P, tab, gap, X, it, lane, gmask, sk, srow);
                    if (!S.stop) w_windows(S, P.pool, lane, r, r);  // the loop's refill schedule
                }
            }
            active = true;
            return;
        }
    };
    fetch();
    it = 0;
    while (__any_sync(kFull, active || waiting)) {
        if (consumer && !__any_sync(kFull, active)) {  // nothing queued for this warp yet
            __nanosleep(2000);
            if (waiting) fetch();
            ++it;
            continue;
        }
        if (active && (it & (PER - 1)) == 0) {  // the same iteration for every group
            S.rv.refill(P.pool);
            S.rh.refill(P.pool);
        }
        wstep<K, G, MODE, true, true>(S, O, E, P, tab, gap, X, it, lane, gmask, sk, srow);
        wstep<K, G, MODE, false, true>(S, E, O, P, tab, gap, X, it, lane, gmask, sk, srow);
        // outcome recorded by the deciding step; idle consumer groups poll every 8th iteration
        if ((active && S.stop) || (consumer && !active && waiting && (it & 7) == 0)) fetch();
        ++it;
    }
    if (lane == 0) {
        if (sk.units) atomicAdd(&P.ctr->units[P.tier], sk.units);
        if (sk.cells) atomicAdd(&P.ctr->cells[P.tier], sk.cells);
        if (sk.esc) atomicAdd(&P.ctr->escalated[P.tier], sk.esc);
    }
    if (P.role == kRoleStart) {  // tell a concurrent escalation consumer when the last block is done
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&P.ctr->prod_done, 1u) == gridDim.x - 1) atomicExch(&P.ctr->prod_finished, 1);
        }
    }
}

#define XB_WINST(K, G)                                                 \
    template __global__ void wide_tier_kernel<K, G, 0>(TierParams);    \
    template __global__ void wide_tier_kernel<K, G, 1>(TierParams);    \
    template __global__ void wide_tier_kernel<K, G, 2>(TierParams);
XB_WINST(96, 8)
XB_WINST(128, 8)
XB_WINST(96, 32)
XB_WINST(128, 32)
XB_WINST(256, 32)
XB_WINST(512, 32)
XB_WINST(1024, 32)
#undef XB_WINST

}  // namespace xb
