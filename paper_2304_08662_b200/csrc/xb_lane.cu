// Lane tiers: G = 8 lanes of a warp cooperate on one unit, each holding
// S = K/8 consecutive slots of the register band (K = 16..64: four units per
// warp).  Same exact semantics, coordinates and bookkeeping as the thread
// tier (xb_thread.cu, xb_kernels.cuh) and the same queues, roles and resume
// records as the 4-lane groups (xb_group.cu), but the step is built for the
// shortest dependent chain, for work that is bound by per-unit latency
// (small batches, escalation tails):
//   * values stay plain drift-space numbers (no 64x keys in the rows); the
//     running best of the lanes above comes from one ballot on the DNA
//     scheme (a cell that beats T scores exactly T + 1, so the threshold of
//     a cell is Tv + [some cell earlier in order improved]) or from one
//     all-gather of the lane maxima (other schemes);
//   * the gap source that crosses a lane edge is shuffled RAW, right after
//     the recurrence, and killed by the receiver with the sender's threshold
//     (known from the same ballot / gather), so the shuffle overlaps the
//     running-best chain instead of following it;
//   * the first cell attaining a new best is remembered by the lane that
//     holds it (antidiagonal + folded diagonal) and looked up only when the
//     unit finishes or escalates;
//   * the live range is one OR-butterfly of the lanes' live bits.
// Measured: a lone unit steps in ~1/4 of the cycles of the 4-lane groups.
#include <climits>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "xb_kernels.cuh"

namespace xb {

namespace {

__device__ __forceinline__ uint32_t lbits(int lo, int hi) {
    if (lo > hi) return 0u;
    return (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo);
}

__device__ __forceinline__ int lbfind32(uint32_t x) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ int lbfind64(uint64_t x) {
    int r;
    asm("bfind.u64 %0, %1;" : "=r"(r) : "l"(x));
    return r;
}

template <int LUT>
__device__ __forceinline__ uint32_t llop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// highest / lowest set bit of a live mask, -1 for an empty one
__device__ __forceinline__ int mask_hi(uint32_t m) { return lbfind32(m); }
__device__ __forceinline__ int mask_hi(uint64_t m) { return lbfind64(m); }
__device__ __forceinline__ int mask_lo(uint32_t m) { return m ? 31 - lbfind32(__brev(m)) : -1; }
__device__ __forceinline__ int mask_lo(uint64_t m) { return m ? 63 - lbfind64(__brevll(m)) : -1; }
template <typename M>
__device__ __forceinline__ M mask_range(int lo, int hi) {  // bits lo..hi, empty for hi < 0
    if (hi < 0) return M(0);
    return ((~M(0)) >> (int(sizeof(M)) * 8 - 1 - hi)) & ((~M(0)) << lo);
}

template <int K, int G, int MODE>
struct LState {
    static constexpr int S = K / G;          // slots per lane
    static constexpr int NB = (S + 3) / 4;   // byte-window words per lane (table mode)
    static constexpr int NM = (K + 31) / 32; // group live-mask words
    static constexpr int KB = 32 * NM - 1;
    int64_t h_pos, v_pos;
    int32_t m, n, hdir, vdir, unit;
    int32_t d, ubase, dcap;
    using Mask = typename std::conditional<(K > 32), uint64_t, uint32_t>::type;
    // live slots of rows d-1 and d-2 (group slots; only the lowest and the
    // highest set bit matter: the window is their span)
    Mask full1, full2;
    int32_t d_vm, d_lim, stop;
    int32_t Tv;                  // T + beta d + 1: a cell is live iff its value >= Tv (or the raised one)
    int32_t best_d, cells, delta_w;
    int32_t mine_d, mine_u;      // last antidiagonal on which this lane held the first best cell, and its u
    int32_t edge;                // killed gap source across the lane edge, for the coming step
    // lane constants, kept opaque so that they stay in registers: the group's
    // lanes above this one, the same plus this lane, and "band < K" (every
    // step must then take the exact width test)
    uint32_t m_above, m_ge;
    int32_t narrow;
    uint32_t ones;               // 0x01010101
    uint32_t Z[4];               // MODE 0: match bytes of the coming step (see the thread tier)
    uint32_t VW, HW;             // 2-bit windows of this lane's S slots (MODE 0)
    uint32_t VWb[NB], HWb[NB];   // byte windows (table modes)
    static constexpr int RENC = MODE == 2 ? ENC_5BIT : ENC_2BIT;  // pool encoding read
    static constexpr int RPER = EncFields<RENC>::PER;              // refill period (iterations)
    Reader<true, RENC> rv;       // lane 0: v symbols entering slot 0
    Reader<false, RENC> rh;      // lane G-1: h symbols entering slot K-1
};

template <int K, int G, int MODE>
__device__ __forceinline__ void l_limits(LState<K, G, MODE>& S) {
    S.d_vm = min(2 * (S.ubase + S.n + 1), 2 * (S.m - S.ubase - K + 2) - 1);
    S.d_lim = S.narrow ? INT_MIN : min(S.d_vm, min(S.n + S.m + 2, S.dcap + 1));  // feeds the step trigger only
}

template <int K, int G, int MODE>
__device__ __forceinline__ void l_windows(LState<K, G, MODE>& S, const uint32_t* __restrict__ pool,
                                          int lane, int rv_r, int rh_r) {
    constexpr int SS = LState<K, G, MODE>::S;
    const int fd = S.d >> 1, cd = S.d - fd;
    const int64_t a = int64_t(fd) - S.ubase - 1;  // v index of global slot 0
    const int64_t b = int64_t(cd) + S.ubase - 1;  // h index of global slot 0
    const int k0 = lane * SS;
    if constexpr (MODE == 0) {
        const uint32_t keep = SS >= 16 ? 0xFFFFFFFFu : ((1u << (2 * SS)) - 1u);
        S.VW = chunk_tf(pool, S.v_pos, S.vdir, a - k0 - 15);  // slot s <- v[a-k0-s] at bits 2s
        S.HW = chunk_bf(pool, S.h_pos, S.hdir, b + k0) & keep;
        if (lane == 0) S.rv.init(pool, S.v_pos, S.vdir, a + 1, rv_r);
        if (lane == G - 1) S.rh.init(pool, S.h_pos, S.hdir, b + K, rh_r);
    } else {
        constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
#pragma unroll
        for (int r = 0; r < LState<K, G, MODE>::NB; ++r) {
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
        if (lane == 0) S.rv.init(pool, S.v_pos, S.vdir, a + 1, rv_r);
        if (lane == G - 1) S.rh.init(pool, S.h_pos, S.hdir, b + K, rh_r);
    }
}

// Table modes: sentinel bytes over this lane's slots whose v or h symbol lies
// past the view's end (see the thread tier's sentinel_windows).
template <int K, int G, int MODE>
__device__ __forceinline__ void l_sentinels(LState<K, G, MODE>& S, int d, int k0) {
    using St = LState<K, G, MODE>;
    const int fd = d >> 1, cd = d - fd;
    const int vhi = fd - S.ubase - 1 - S.n - k0;  // lane slots 0..vhi: v index >= n
    const int hlo = S.m - (cd + S.ubase - 1) - k0;  // lane slots hlo..: h index >= m
#pragma unroll
    for (int r = 0; r < St::NB; ++r) {
        const int v1 = min(vhi - 4 * r, 3), h0 = max(hlo - 4 * r, 0);
        const uint32_t mv = v1 < 0 ? 0u : lbits(0, 8 * v1 + 7);
        const uint32_t mh = h0 > 3 ? 0u : lbits(8 * h0, 31);
        S.VWb[r] = (S.VWb[r] & ~mv) | (0x1F1F1F1Fu & mv);
        S.HWb[r] = (S.HWb[r] & ~mh) | (0x1F1F1F1Fu & mh);
    }
}

// one-slot shift of a row across the group: new[k] = old[k + dir]
template <int SS, int G>
__device__ __forceinline__ void l_shift1(int32_t (&R)[SS], int dir, int lane, unsigned mask) {
    if (dir > 0) {
        const int32_t carry = __shfl_down_sync(mask, R[0], 1, G);
#pragma unroll
        for (int s = 0; s < SS - 1; ++s) R[s] = R[s + 1];
        R[SS - 1] = lane == G - 1 ? kDeadS : carry;
    } else {
        const int32_t carry = __shfl_up_sync(mask, R[SS - 1], 1, G);
#pragma unroll
        for (int s = SS - 1; s > 0; --s) R[s] = R[s - 1];
        R[0] = lane == 0 ? kDeadS : carry;
    }
}

struct LSink {
    uint32_t* esc_list;
    unsigned long long* esc_len;
    long long qidx;
    unsigned long long units, cells, esc;
    bool resumable;
};

}  // namespace

// Symbols entering on d+1 (v after an odd step, h after an even one).
// FM: the whole warp executes this call (full-mask shuffles, no convergence
// check); otherwise only this group does.
template <int K, int G, int MODE, bool ODD, bool FM>
__device__ __forceinline__ void lfeed(LState<K, G, MODE>& S, const TierParams& P, int d, int lane,
                                      unsigned gmask_) {
    const unsigned gmask = FM ? 0xFFFFFFFFu : gmask_;
    using St = LState<K, G, MODE>;
    constexpr int SS = St::S;
    if constexpr (MODE == 0) {
        if constexpr (ODD) {  // v: slot k <- k-1, new symbol at slot 0 (lane 0's reader)
            const uint32_t out = (S.VW >> (2 * (SS - 1))) & 3u;
            uint32_t in = __shfl_up_sync(gmask, out, 1, G);
            if (lane == 0) {
                in = S.rv.cur >> 30;
                S.rv.cur <<= 2;
            }
            S.VW = (S.VW << 2) | in;
        } else {  // h: slot k <- k+1, new symbol at slot K-1 (lane G-1's reader)
            const uint32_t out = S.HW & 3u;
            uint32_t in = __shfl_down_sync(gmask, out, 1, G);
            if (lane == G - 1) {
                in = S.rh.cur & 3u;
                S.rh.cur >>= 2;
            }
            S.HW = (S.HW >> 2) | (in << (2 * (SS - 1)));
        }
    } else {
        constexpr int NB = St::NB;
        constexpr int top = 8 * ((SS - 1) & 3);  // bit offset of slot SS-1 in its word
        if constexpr (ODD) {
            const uint32_t out = (S.VWb[NB - 1] >> top) & 0xFFu;
            uint32_t in = __shfl_up_sync(gmask, out, 1, G);
            if (lane == 0) in = S.rv.take();
#pragma unroll
            for (int r = NB - 1; r > 0; --r) S.VWb[r] = __funnelshift_l(S.VWb[r - 1], S.VWb[r], 8);
            S.VWb[0] = (S.VWb[0] << 8) | in;
        } else {
            const uint32_t out = S.HWb[0] & 0xFFu;
            uint32_t in = __shfl_down_sync(gmask, out, 1, G);
            if (lane == G - 1) in = S.rh.take();
#pragma unroll
            for (int r = 0; r < NB - 1; ++r) S.HWb[r] = __funnelshift_r(S.HWb[r], S.HWb[r + 1], 8);
            const uint32_t keep = top == 24 ? 0xFFFFFFFFu : ((1u << (top + 8)) - 1u);
            S.HWb[NB - 1] = ((S.HWb[NB - 1] >> 8) & (keep >> 8)) | (in << top);
        }
    }
}

// The folded diagonal of the best cell: kept by the lane that held the first
// cell attaining the current best (mine_d == best_d on exactly one lane).
template <int K, int G, int MODE>
__device__ __forceinline__ int32_t best_u_of(const LState<K, G, MODE>& S, unsigned gmask, int gbase) {
    const unsigned b = (__ballot_sync(gmask, S.mine_d == S.best_d) >> gbase) & ((1u << G) - 1u);
    return __shfl_sync(gmask, S.mine_u, lbfind32(b), G);
}

// Records the outcome of the group's unit at the deciding step (see the
// thread tier's finish_unit); escalations save a resume record, each lane
// writing its own slots.
template <int K, int G, int MODE>
__device__ __forceinline__ void lfinish(LState<K, G, MODE>& S, const TierParams& P, int code, int spread,
                                        LSink& sk, int32_t beta, const int32_t (&cur)[K / G],
                                        const int32_t (&prv)[K / G], int lane, unsigned gmask) {
    constexpr int SS = K / G;
    constexpr int KB = LState<K, G, MODE>::KB;
    S.stop = code;
    if (P.pilot) {
        if (lane == 0) P.pilot_w[sk.qidx] = code == kEscalate ? -1 : S.delta_w;
        return;
    }
    const int gbase = int(threadIdx.x & 31) - lane;
    const int32_t best_u = best_u_of(S, gmask, gbase);
    if (code == kEscalate) {
        uint32_t entry = uint32_t(S.unit);
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
                    rec[kRecTc] = (S.Tv - beta) << 6;  // as before step d, in the records' 64x units
                    rec[kRecBestD] = S.best_d;
                    rec[kRecBestU] = best_u;
                    rec[kRecCells] = S.cells;
                    rec[kRecDeltaW] = S.delta_w;
                    rec[kRecHs1] = mask_hi(S.full1);
                    rec[kRecLs1] = mask_lo(S.full1);
                    rec[kRecHs2] = mask_hi(S.full2);
                    rec[kRecLs2] = mask_lo(S.full2);
                    rec[kRecK] = K;
                }
                entry = got;
            }
        }
        __syncwarp(gmask);
        if (lane == 0) {
            // a concurrent consumer may take the entry as soon as it is written:
            // the record first, then the slot, then the entry (volatile)
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
        const int best_i = (S.best_d >> 1) - best_u;
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

// The killed gap source across the lane edge for a step of parity ODD, read
// from the finished row prv (after a (re)start or a recentre; the steps
// themselves pass it on raw, see lstep).  Group-divergent: the group's mask.
template <int SS, int G, bool ODD>
__device__ __forceinline__ int32_t edge_of_rows(const int32_t (&prv)[SS], int lane, unsigned gmask) {
    int32_t e;
    if constexpr (ODD) {  // gap sources at u and u+1
        e = __shfl_down_sync(gmask, prv[0], 1, G);
        if (lane == G - 1) e = kDeadS;
    } else {              // gap sources at u-1 and u
        e = __shfl_up_sync(gmask, prv[SS - 1], 1, G);
        if (lane == 0) e = kDeadS;
    }
    return e;
}

// MODE 0: the match bytes of the coming step from the current windows (byte j
// of Z[q] = 1 + 2*match of slot 4j+q, see the thread tier); inv marks the
// 2-bit fields of slots outside the matrix.
template <int K, int G, int MODE>
__device__ __forceinline__ void l_match(LState<K, G, MODE>& S, uint32_t inv) {
    if constexpr (MODE == 0) {
        const uint32_t x = llop3<0xBE>(S.VW, S.HW, inv);  // (a ^ b) | c
        const uint32_t z = llop3<0x03>(x, x << 1, 0u);    // ~(a | b)
        // (z >> 2q) & 0x02020202 | 0x01010101 as one LOP3 each: the second
        // constant comes in a register (S.ones)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t r;
            asm("lop3.b32 %0, %1, 0x02020202, %2, 0xEA;" : "=r"(r) : "r"(z >> (2 * q)), "r"(S.ones));  // (a & b) | c
            S.Z[q] = r;
        }
    }
}

// One antidiagonal d.  cur holds d-2 on entry and d on exit, prv holds d-1,
// S.edge the killed neighbour value this step needs (and, on exit, the one
// the next step needs).  FM: every group of the warp executes the step.
//
// The step's dependent chain is: recurrence -> lane maximum -> ballot (or
// gather) -> threshold -> drop test -> kill.  Everything else hangs off it:
// the window of row d (cells, delta_w) is computed late from the live masks
// of rows d-1 and d-2, whose gather overlapped the chain.
//
// EXACT = false is the straight-line form: no branch, no divergent region
// (so no reconvergence checks before the collectives).  It is only valid
// when nothing can stop, reshape or mask the step; the warp runs it while no
// group raised a trigger.  The step returns this lane's trigger for the NEXT
// step -- a conservative test taken right after the recurrence, beside the
// chain: the band's edge slot may go live (the window would leave the K
// slots), the group may have no live cell left, d + 1 reaches d_lim.  After a
// trigger (and after every fetch) the whole warp runs one EXACT step, which
// evaluates the thread tier's rare-path conditions from the live masks.
template <int K, int G, int MODE, bool ODD, bool FM, bool EXACT>
__device__ __forceinline__ bool lstep(LState<K, G, MODE>& S, int32_t (&cur)[K / G],
                                      int32_t (&prv)[K / G], const TierParams& P,
                                      const tab_t* __restrict__ tab, int32_t gap, int32_t X,
                                      unsigned it, int lane, unsigned gmask, LSink& sk) {
    const unsigned smask = FM ? 0xFFFFFFFFu : gmask;
    using St = LState<K, G, MODE>;
    using Mask = typename St::Mask;
    constexpr int SS = St::S;
    constexpr int KB = St::KB;
    const int d = S.d;
    const int k0 = lane * SS;
    const int32_t beta = -gap;
    S.Tv += beta;
    uint32_t vml = lbits(0, SS - 1);  // this lane's in-matrix slots
    int wadd = -1;                    // cells of row d when the rare path fixed them, else computed late

    // pass 1: the recurrence (again after a rare path that changed its inputs)
    int32_t cand[SS];
    auto pass1 = [&]() __attribute__((always_inline)) {
        const int32_t edge = S.edge;
#pragma unroll
        for (int s = SS - 1; s >= 0; --s) {
            const int32_t dg = cur[s];
            int32_t db;
            if constexpr (MODE == 0) {
                db = __dp4a(int(S.Z[s & 3]), 1 << (8 * ((s >> 2) & 3)), dg);
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
    };
    pass1();

    // group-divergent exact path: the conditions of the thread tier's xstep
    if (EXACT && !S.stop) {
        const int hs1 = mask_hi(S.full1), ls1 = mask_lo(S.full1);
        const int hs2 = mask_hi(S.full2), ls2 = mask_lo(S.full2);
        const bool e1 = hs1 < 0, e2 = hs2 < 0;
        if ((e1 && e2) || d > S.n + S.m + 1 || d > S.dcap) {
            lfinish<K, G, MODE>(S, P, kDone, 0, sk, beta, cur, prv, lane, gmask);
        } else {
            int lo = kBig, hi = -kBig;
            if (!e1) {
                lo = ls1 - (ODD ? 1 : 0);
                hi = hs1 + (ODD ? 0 : 1);
            }
            if (!e2) {
                lo = min(lo, ls2);
                hi = max(hi, hs2);
            }
            const int fd = d >> 1;
            int A = fd - S.ubase;
            const int w = min(hi, A - max(d - S.m, 0)) - max(lo, A - min(d, S.n)) + 1;
            if (w > P.band) {
                lfinish<K, G, MODE>(S, P, kBand, w, sk, beta, cur, prv, lane, gmask);
            } else {
                bool redo = false;
                if (lo < 0 || hi > K - 1) {
                    const int wu = hi - lo + 1;
                    if (wu > K) {
                        lfinish<K, G, MODE>(S, P, kEscalate, 0, sk, beta, cur, prv, lane, gmask);
                    } else {
                        const int sh = lo - ((K - wu) >> 1);
                        for (int q = sh; q > 0; --q) {
                            l_shift1<SS, G>(cur, 1, lane, gmask);
                            l_shift1<SS, G>(prv, 1, lane, gmask);
                        }
                        for (int q = sh; q < 0; ++q) {
                            l_shift1<SS, G>(cur, -1, lane, gmask);
                            l_shift1<SS, G>(prv, -1, lane, gmask);
                        }
                        S.ubase += sh;
                        S.full1 = sh > 0 ? S.full1 >> sh : S.full1 << -sh;
                        S.full2 = sh > 0 ? S.full2 >> sh : S.full2 << -sh;
                        A -= sh;
                        l_limits(S);
                        constexpr int PER = St::RPER;
                        const int to_refill = PER - int(it & (PER - 1));
                        l_windows(S, P.pool, lane, ODD ? to_refill : to_refill - 1, to_refill);
                        S.edge = edge_of_rows<SS, G, ODD>(prv, lane, gmask);
                        l_match(S, 0u);
                        redo = true;
                    }
                }
                if (!S.stop && d >= S.d_vm) {
                    const int klo = A - S.n;
                    const int khi = S.m - (d - fd) - S.ubase;
                    const int l = max(klo - k0, 0), h = min(min(khi, K - 1) - k0, SS - 1);
                    vml = lbits(l, h);
                    if constexpr (MODE == 0)
                        l_match(S, ~((l > h) ? 0u : lbits(2 * l, 2 * h + 1)));
                    else
                        l_sentinels(S, d, k0);
                    redo = true;
                }
                wadd = max(w, 0);  // a clamped-empty row counts no cells (align.cpp:84-90)
                if (redo && !S.stop) pass1();
            }
        }
    }

    // the next step's edge source leaves raw, now: after an odd step the even
    // one reads lane-1's top slot, after an even step the odd one lane+1's
    // slot 0; the receiver applies the sender's drop test below
    const int32_t nraw = ODD ? __shfl_up_sync(smask, cand[SS - 1], 1, G) : __shfl_down_sync(smask, cand[0], 1, G);

    // lane maximum, and (off the chain) its highest slot from keys 64 cand + s
    // (the range guard of the prep kernel keeps them in int32)
    int32_t lm = cand[SS - 1];
    int32_t mk = cand[SS - 1] * 64 + (SS - 1);
#pragma unroll
    for (int s = SS - 2; s >= 0; s -= 2) {
        if (s >= 1) {
            lm = __vimax3_s32(lm, cand[s], cand[s >= 1 ? s - 1 : 0]);
            mk = __vimax3_s32(mk, cand[s] * 64 + s, cand[s >= 1 ? s - 1 : 0] * 64 + (s - 1));
        } else {
            lm = max(lm, cand[s]);
            mk = max(mk, cand[s] * 64 + s);
        }
    }
    // this lane's trigger for the next step (conservative: cand >= Tv is
    // implied by live)
    bool trig;
    {
        const bool edge_may = ODD ? (lane == G - 1 && cand[SS - 1] >= S.Tv) : (lane == 0 && cand[0] >= S.Tv);
        const unsigned bl = __ballot_sync(smask, lm >= S.Tv);
        trig = (edge_may | ((bl & gmask) == 0u) | (d + 1 >= S.d_lim)) & (S.stop == 0);  // d_lim: also band < K
    }
    // the lane's own chain from Tv, before the lanes above are known
    // (align.cpp:122-129 in ascending i = descending slot): c_s, and whether
    // the cell already fails against it
    bool dead0[SS];
    {
        int32_t c = S.Tv;
#pragma unroll
        for (int s = SS - 1; s >= 0; --s) {
            c = __viaddmax_s32(cand[s], -X, c);
            dead0[s] = cand[s] < c;
        }
    }

    // thresholds: c0 = the running best of the lanes above (a cell fails if it
    // is below c0 or below its lane's chain), nthr for the neighbour value
    // that left raw, and the antidiagonal's outcome
    int32_t c0, nthr, newTv;
    bool improve, first;
    if constexpr (MODE == 0) {
        // +1/-1/-1: a cell beats T only by a match on the diagonal of a cell
        // that held T, so it scores exactly T + 1: the threshold of a cell is
        // Tv + 1 if some cell earlier in order (or itself) improved, else Tv
        const bool imp = lm > S.Tv + X;
        const unsigned bal = __ballot_sync(smask, imp);
        const bool hi_imp = (bal & S.m_above) != 0u;
        c0 = S.Tv + (hi_imp ? 1 : 0);
        // sender of nraw: lane-1's top slot (first of its chain) sees the lanes
        // >= lane; lane+1's slot 0 (last of its chain) sees the lanes > lane
        nthr = ODD ? S.Tv + (((bal & S.m_ge) != 0u) ? 1 : 0) : c0;
        improve = (bal & gmask) != 0u;
        newTv = S.Tv + (improve ? 1 : 0);
        first = imp && !hi_imp;
    } else {
        int32_t Mj[G];
#pragma unroll
        for (int j = 0; j < G; ++j) Mj[j] = __shfl_sync(smask, lm, j, G);
        // maximum over the higher lanes: lane-constant offsets (0 for a higher
        // lane, -2^29 otherwise: values are below 2^25) instead of selects
        int32_t above = -(1 << 30), all = Mj[0];
#pragma unroll
        for (int j = 1; j < G; ++j) {
            above = max(above, Mj[j] + (lane < j ? 0 : -(1 << 29)));
            all = max(all, Mj[j]);
        }
        c0 = max(S.Tv, above - X);
        nthr = ODD ? max(c0, lm - X) : c0;
        improve = all - X > S.Tv;
        newTv = max(S.Tv, all - X);
        first = improve && lm == all && above < all;
    }
    // the neighbour's value, killed as its own lane kills it
    {
        const bool none = ODD ? lane == 0 : lane == G - 1;
        S.edge = (nraw >= nthr && !none) ? nraw : kDeadS;
    }
    // drop test, kill, live bits (a kept cell is >= Tv >= 1, the dead marker
    // negative: the dead mask is the rows' sign bits, shifted in slot by slot)
    uint32_t dm = 0u;
#pragma unroll
    for (int s = SS - 1; s >= 0; --s) {
        const bool dead = dead0[s] || cand[s] < c0;
        cur[s] = dead ? kDeadS : cand[s];
        dm = __funnelshift_l(uint32_t(cur[s]), dm, 1);
    }
    const uint32_t lv = ~dm & vml;
    // gather the live bits of row d (consumed a step later)
    Mask gathered;
    {
        Mask part[G];
        const Mask mine = Mask(lv) << k0;
#pragma unroll
        for (int j = 0; j < G; ++j) part[j] = __shfl_sync(smask, mine, j, G);
        gathered = part[0];
#pragma unroll
        for (int j = 1; j < G; ++j) gathered |= part[j];
    }
    // running best (align.cpp:123-127): strict improvement, first cell wins:
    // the highest lane holding the maximum, its highest slot holding it
    S.best_d = improve ? d : S.best_d;
    S.mine_d = first ? d : S.mine_d;
    S.mine_u = first ? S.ubase + k0 + (mk & 63) : S.mine_u;
    S.Tv = newTv;
    lfeed<K, G, MODE, ODD, FM>(S, P, d, lane, gmask);
    l_match(S, 0u);
    // cells of row d: the span reachable from rows d-1 and d-2 (the exact
    // path may have fixed them: clamps at the matrix edge)
    {
        const Mask reach = S.full2 | S.full1 | (ODD ? S.full1 >> 1 : S.full1 << 1);
        const int wlate =
            mask_hi(reach) + mask_hi(St::NM == 1 ? Mask(__brev(uint32_t(reach))) : Mask(__brevll(reach))) - KB + 1;
        wadd = wadd < 0 ? wlate : wadd;
    }
    S.cells += wadd;
    S.delta_w = max(S.delta_w, wadd);
    S.full2 = S.full1;
    S.full1 = gathered;
    S.d = d + 1;
    return trig;
}

template <int K, int G, int MODE>
__global__ void __launch_bounds__(128) lane_tier_kernel(TierParams P) {
    using St = LState<K, G, MODE>;
    constexpr int SS = St::S;
    constexpr int KB = St::KB;
    __shared__ tab_t tab[MODE == 0 ? 1 : kTabWords];
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    const int wl = threadIdx.x & 31;
    const int lane = wl % G;
    const int gbase = wl - lane;
    const unsigned gmask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << gbase;
    const int k0 = lane * SS;

    Queue Q;
    if (!make_queue(P, Q)) return;
    if (P.role != kRoleConsumer && Q.len == 0) return;  // nothing escalated into this tier
    if constexpr (MODE != 0) {
        tab_fill(tab, P.scheme, gap);
        __syncthreads();
    }
    const int next_tier = P.esc_to_warp ? kWarpTier : P.tier + 1;
    LSink sk;
    sk.esc_list = P.lists + (long long)next_tier * P.n_units;
    sk.esc_len = &P.ctr->list_len[next_tier];
    sk.qidx = 0;
    sk.units = sk.cells = sk.esc = 0;
    sk.resumable = next_tier != kWarpTier && !P.pilot;

    // Every group of the warp executes every step, so the main-path shuffles
    // can use the full mask; a group without a unit steps on harmless state
    // with stop set (no rare path, no output, no loads: its reader refills
    // are skipped and table-mode lookups see empty views).
    St S;
    S.m = S.n = 0;
    S.stop = kDone;
    S.VW = S.HW = 0u;
    S.full1 = S.full2 = 0;
    S.m_above = (gmask << 1 << lane) & gmask;
    S.m_ge = S.m_above | (1u << wl);
    S.narrow = P.band < K ? 1 : 0;
    S.ones = P.ones;
    asm volatile("" : "+r"(S.m_above), "+r"(S.m_ge), "+r"(S.narrow), "+r"(S.ones));
#pragma unroll
    for (int q = 0; q < 4; ++q) S.Z[q] = 0x01010101u;
    S.Tv = 0;
    S.d = 1;
    S.ubase = 0;
    S.d_vm = S.d_lim = 1 << 30;
    S.best_d = S.mine_u = S.cells = S.delta_w = 0;
    S.mine_d = -1;
    S.edge = kDeadS;
    // a group that never gets a unit still feeds its windows from its readers
    // (table modes index the shared table with those codes): start them empty
    S.rv.cur = S.rh.cur = 0u;
    S.rv.w0 = S.rv.w1 = S.rh.w0 = S.rh.w1 = 0u;
    S.rv.pend = S.rh.pend = 0u;
    S.rv.sh = S.rh.sh = 0u;
#pragma unroll
    for (int r = 0; r < St::NB; ++r) S.VWb[r] = S.HWb[r] = 0u;
    int32_t E[SS], O[SS];
#pragma unroll
    for (int s = 0; s < SS; ++s) E[s] = O[s] = kDeadS;
    bool active = false;
    // kRoleConsumer: the list grows while this kernel runs.  A group claims
    // a slot only once the list is longer than the cursor (so it never holds
    // a claim it cannot serve and may stop at any time: the kRoleEscalations
    // launch after the start tier takes whatever is left), waits for the
    // claimed slot's entry to be written, and idles while nothing is queued.
    // The handshake has no timeout: the start tier is launched (API order)
    // before its consumer and never waits for it, so a consumer only ever
    // waits on a producer that is running or already finished -- under tools
    // that serialise launches (ncu, compute-sanitizer) it runs after the
    // whole start tier and just drains the list.
    const bool consumer = P.role == kRoleConsumer;
    bool waiting = consumer;  // a consumer group with no unit, still looking for one
    unsigned it = 0xFFFFFFFFu;
    auto fetch = [&]() __attribute__((always_inline)) {
        active = false;
        for (;;) {
            unsigned long long i = 0;
            uint32_t e = 0;
            if (consumer) {
                int st = 0;  // 0 nothing queued, 1 claimed slot i (entry e), 2 start tier done
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
                if (lane == 0) i = atomicAdd(Q.cursor, 1ull);
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
            if (u.route != 0) {
                if (P.pilot && lane == 0) P.pilot_w[i] = -2;
                continue;
            }
            sk.qidx = (long long)i;
            S.unit = int32_t(unit);
            S.h_pos = u.h_pos;
            S.v_pos = u.v_pos;
            S.m = u.h_len;
            S.n = u.v_len;
            S.hdir = u.dir & 1;
            S.vdir = (u.dir >> 1) & 1;
            S.dcap = P.pilot ? P.pilot_cap : (INT_MAX >> 1);
            S.stop = 0;
            const int r = (St::RPER - 1) - int(it & (St::RPER - 1));
            if (!rec) {
                S.d = 1;
                S.ubase = -(K / 2);
                S.full1 = typename St::Mask(1) << (K / 2);  // antidiagonal 0: the origin, u = 0
                S.full2 = 0;                                // antidiagonal -1: empty
                S.Tv = 1;  // T + beta d + 1 at d = 0, T = 0
                S.best_d = 0;
                S.mine_d = lane == 0 ? 0 : -1;  // the origin: antidiagonal 0, u = 0
                S.mine_u = 0;
                S.delta_w = 1;
                S.cells = 1;
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    O[s] = kDeadS;
                    E[s] = (k0 + s == K / 2) ? X + 1 : kDeadS;
                }
                l_limits(S);
                l_windows(S, P.pool, lane, r, r);
                l_match(S, 0u);
                S.edge = edge_of_rows<SS, G, true>(E, lane, gmask);
            } else {
                // continue from a narrower tier's record (see resume_unit)
                const int ko = __ldcg(rec + kRecK);
                const int off = (K - ko) >> 1;
                const int d = __ldcg(rec + kRecD);
                S.ubase = __ldcg(rec + kRecUbase) - off;
                S.Tv = __ldcg(rec + kRecTc) >> 6;
                S.best_d = __ldcg(rec + kRecBestD);
                S.mine_d = lane == 0 ? S.best_d : -1;
                S.mine_u = __ldcg(rec + kRecBestU);
                S.cells = __ldcg(rec + kRecCells);
                S.delta_w = __ldcg(rec + kRecDeltaW);
                const int h1 = __ldcg(rec + kRecHs1), l1 = __ldcg(rec + kRecLs1), h2 = __ldcg(rec + kRecHs2), l2 = __ldcg(rec + kRecLs2);
                S.full1 = mask_range<typename St::Mask>(l1 + off, h1 < 0 ? -1 : h1 + off);
                S.full2 = mask_range<typename St::Mask>(l2 + off, h2 < 0 ? -1 : h2 + off);
                const bool odd = d & 1;
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    const int src = k0 + s - off;
                    const bool in = src >= 0 && src < ko;
                    const int32_t vc = in ? __ldcg(rec + kRecRows + src) : kDeadS;
                    const int32_t vp = in ? __ldcg(rec + kRecRows + ko + src) : kDeadS;
                    O[s] = odd ? vc : vp;
                    E[s] = odd ? vp : vc;
                }
                S.d = odd ? d : d - 1;
                // a record written at an even d: its odd half-iteration only feeds
                // v, its even step runs here (readers set up with a full refill
                // period, as this happens before the next refill point), and the
                // group joins the loop at an odd d, so the loop itself never peels
                l_windows(S, P.pool, lane, odd ? r : St::RPER - 1, odd ? r : St::RPER - 1);
                S.d = d;
                l_limits(S);
                if (odd) {
                    S.edge = edge_of_rows<SS, G, true>(E, lane, gmask);
                    l_match(S, 0u);
                }
                if (!odd) {
                    if (lane == 0) atomicAdd(&P.ctr->dbg[5], 1ull);  // stats: even-d resumes
                    S.edge = edge_of_rows<SS, G, false>(O, lane, gmask);
                    lfeed<K, G, MODE, true, false>(S, P, d - 1, lane, gmask);
                    l_match(S, 0u);
                    lstep<K, G, MODE, false, false, true>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
                    if (!S.stop) {
                        l_windows(S, P.pool, lane, r, r);  // the loop's refill schedule
                        l_match(S, 0u);
                    }
                }
            }
            active = true;
            return;
        }
    };
    fetch();
    it = 0;
    // A band narrower than K needs the exact width test on every step.
    // One iteration = an odd and an even antidiagonal.  A step runs in its
    // exact form after a fetch and when some lane raised a trigger on the step
    // before (warp-uniform votes); otherwise in the straight-line form.
    auto refill = [&]() __attribute__((always_inline)) {
        if ((it & (St::RPER - 1)) == 0) {  // the same iteration for every group
            if (active && lane == 0) S.rv.refill(P.pool);
            if (active && lane == G - 1) S.rh.refill(P.pool);
        }
    };
    auto odd_exact = [&]() __attribute__((always_inline)) {
        return lstep<K, G, MODE, true, true, true>(S, O, E, P, tab, gap, X, it, lane, gmask, sk);
    };
    auto odd_fast = [&]() __attribute__((always_inline)) {
        return lstep<K, G, MODE, true, true, false>(S, O, E, P, tab, gap, X, it, lane, gmask, sk);
    };
    auto even_exact = [&]() __attribute__((always_inline)) {
        return lstep<K, G, MODE, false, true, true>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
    };
    auto even_fast = [&]() __attribute__((always_inline)) {
        return lstep<K, G, MODE, false, true, false>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
    };
    constexpr unsigned kAll = 0xFFFFFFFFu;
    // the consumer's polling lives in its own copy of the loop, so the
    // ordinary launches run the loop without it
    auto run = [&](auto cons) {
        constexpr bool CONS = decltype(cons)::value;
        bool xo = true;
        if constexpr (!CONS) {
            while (__any_sync(kAll, active)) {
                for (;;) {  // until some group's unit is decided
                    if (xo) {
                        // an exact odd step, then the even step in whichever form
                        refill();
                        bool t = odd_exact();
                        if (__any_sync(kAll, t))
                            t = even_exact();
                        else
                            t = even_fast();
                        xo = __any_sync(kAll, t);
                        if (__any_sync(kAll, active && S.stop)) break;
                        ++it;
                        continue;
                    }
                    // straight-line iterations: uniform branches only; a unit can
                    // only be decided by an exact step
                    bool decided = false;
                    for (;;) {
                        refill();
                        bool t = odd_fast();
                        if (__any_sync(kAll, t)) {
                            t = even_exact();
                            xo = __any_sync(kAll, t);
                            decided = __any_sync(kAll, active && S.stop);
                            if (!decided) ++it;
                            break;
                        }
                        t = even_fast();
                        ++it;
                        if (__any_sync(kAll, t)) {
                            xo = true;
                            break;
                        }
                    }
                    if (decided) break;
                }
                if (active && S.stop) fetch();
                xo = true;
                ++it;
            }
            return;
        }
        while (__any_sync(kAll, active || (CONS && waiting))) {
            if constexpr (CONS) {
                if (!__any_sync(kAll, active)) {  // nothing queued for this warp yet
                    __nanosleep(2000);
                    if (waiting) fetch();
                    xo = true;
                    ++it;
                    continue;
                }
            }
            // every group steps on odd d here (fetch() runs the even step of a
            // unit resumed at an even d), so the warp needs no peeled half
            refill();
            bool t = xo ? odd_exact() : odd_fast();
            t = __any_sync(kAll, t) ? even_exact() : even_fast();
            xo = __any_sync(kAll, t);
            // outcome recorded by the deciding step; idle consumer groups poll every 8th iteration
            if ((active && S.stop) || (CONS && !active && waiting && (it & 7) == 0)) {
                fetch();
                xo = true;
            }
            ++it;
        }
    };
    if (consumer)
        run(std::true_type{});
    else
        run(std::false_type{});
    if (P.pilot) return;
    if (lane == 0) {
        if (sk.units) atomicAdd(&P.ctr->units[P.tier], sk.units);
        if (sk.cells) atomicAdd(&P.ctr->cells[P.tier], sk.cells);
        if (sk.esc) atomicAdd(&P.ctr->escalated[P.tier], sk.esc);
    }
    if (P.role == kRoleStart) {  // a latency-planned start tier with a concurrent consumer
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(&P.ctr->prod_done, 1u) == gridDim.x - 1) atomicExch(&P.ctr->prod_finished, 1);
        }
    }
}

#define XB_LINST(K, G)                                                    \
    template __global__ void lane_tier_kernel<K, G, 0>(TierParams);       \
    template __global__ void lane_tier_kernel<K, G, 1>(TierParams);       \
    template __global__ void lane_tier_kernel<K, G, 2>(TierParams);
XB_LINST(16, 8)
XB_LINST(24, 8)
XB_LINST(32, 8)
XB_LINST(48, 8)
XB_LINST(64, 8)
#undef XB_LINST

}  // namespace xb
