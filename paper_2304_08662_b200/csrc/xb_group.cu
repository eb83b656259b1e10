// Lane-group tiers: G lanes of a warp cooperate on one unit, each holding
// S = K/G consecutive slots of the register band.  Same exact semantics and
// bookkeeping as the thread tier (xb_thread.cu; coordinates and proofs in
// xb_kernels.cuh); what changes is the plumbing between slots that live in
// different lanes:
//   * the one gap source that crosses a lane edge comes by SHFL (up on even
//     antidiagonals, down on odd ones), and so do the symbols entering a
//     lane's window;
//   * the running-best chain, which runs over slots in descending order,
//     becomes: lane-local key maximum -> one all-gather round (G independent
//     shuffles) giving each lane the maximum of the higher lanes and the
//     group maximum -> lane-local chain seeded with it;
//   * the live range is a second all-gather round of the lanes' live bits.
// A step then costs ~S slots of dependent work plus two shuffle rounds on
// its critical path instead of K slots: this tier serves work that is
// latency- rather than throughput-bound (escalation tails, the pilot, and
// batches too small to fill the machine).
#include <climits>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "xb_kernels.cuh"

namespace xb {

namespace {

__device__ __forceinline__ uint32_t gbits(int lo, int hi) {
    if (lo > hi) return 0u;
    return (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo);
}

__device__ __forceinline__ int gbfind32(uint32_t x) {
    int r;
    asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
    return r;
}
__device__ __forceinline__ int gbfind64(uint64_t x) {
    int r;
    asm("bfind.u64 %0, %1;" : "=r"(r) : "l"(x));
    return r;
}

template <int LUT>
__device__ __forceinline__ uint32_t glop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

template <int K, int G, int MODE>
struct GState {
    static constexpr int S = K / G;          // slots per lane
    static constexpr int NB = (S + 3) / 4;   // byte-window words per lane (table mode)
    static constexpr int NM = (K + 31) / 32; // group live-mask words
    static constexpr int KB = 32 * NM - 1;
    int64_t h_pos, v_pos;
    int32_t m, n, hdir, vdir, unit;
    int32_t d, ubase, dcap;
    int32_t lr1, hs1, lr2, hs2;  // group slots; hs / KB - ls, -1 for an empty row
    int32_t d_vm, d_lim, stop;
    int32_t Tc, best_d, best_u, cells, delta_w;
    uint32_t VW, HW;             // 2-bit windows of this lane's S slots (MODE 0)
    uint32_t VWb[NB], HWb[NB];   // byte windows (table modes)
    static constexpr int RENC = MODE == 2 ? ENC_5BIT : ENC_2BIT;  // pool encoding read
    static constexpr int RPER = EncFields<RENC>::PER;              // refill period (iterations)
    Reader<true, RENC> rv;       // lane 0: v symbols entering slot 0
    Reader<false, RENC> rh;      // lane G-1: h symbols entering slot K-1
};

template <int K, int G, int MODE>
__device__ __forceinline__ void g_limits(GState<K, G, MODE>& S) {
    S.d_vm = min(2 * (S.ubase + S.n + 1), 2 * (S.m - S.ubase - K + 2) - 1);
    S.d_lim = min(S.d_vm, min(S.n + S.m + 2, S.dcap + 1));
}

template <int K, int G, int MODE>
__device__ __forceinline__ void g_windows(GState<K, G, MODE>& S, const uint32_t* __restrict__ pool,
                                          int lane, int rv_r, int rh_r) {
    constexpr int SS = GState<K, G, MODE>::S;
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
        for (int r = 0; r < GState<K, G, MODE>::NB; ++r) {
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
__device__ __forceinline__ void g_sentinels(GState<K, G, MODE>& S, int d, int k0) {
    using St = GState<K, G, MODE>;
    const int fd = d >> 1, cd = d - fd;
    const int vhi = fd - S.ubase - 1 - S.n - k0;  // lane slots 0..vhi: v index >= n
    const int hlo = S.m - (cd + S.ubase - 1) - k0;  // lane slots hlo..: h index >= m
#pragma unroll
    for (int r = 0; r < St::NB; ++r) {
        const int v1 = min(vhi - 4 * r, 3), h0 = max(hlo - 4 * r, 0);
        const uint32_t mv = v1 < 0 ? 0u : gbits(0, 8 * v1 + 7);
        const uint32_t mh = h0 > 3 ? 0u : gbits(8 * h0, 31);
        S.VWb[r] = (S.VWb[r] & ~mv) | (0x1F1F1F1Fu & mv);
        S.HWb[r] = (S.HWb[r] & ~mh) | (0x1F1F1F1Fu & mh);
    }
}

// one-slot shift of a row across the group: new[k] = old[k + dir]
template <int SS, int G>
__device__ __forceinline__ void g_shift1(int32_t (&R)[SS], int dir, int lane, unsigned mask) {
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

struct GSink {
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
__device__ __forceinline__ void gfeed(GState<K, G, MODE>& S, const TierParams& P, int d, int lane,
                                      unsigned gmask_) {
    const unsigned gmask = FM ? 0xFFFFFFFFu : gmask_;
    using St = GState<K, G, MODE>;
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

// Records the outcome of the group's unit at the deciding step (see the
// thread tier's finish_unit); escalations save a resume record, each lane
// writing its own slots.
template <int K, int G, int MODE>
__device__ __forceinline__ void gfinish(GState<K, G, MODE>& S, const TierParams& P, int code, int spread,
                                        GSink& sk, int32_t beta, const int32_t (&cur)[K / G],
                                        const int32_t (&prv)[K / G], int lane, unsigned gmask) {
    constexpr int SS = K / G;
    constexpr int KB = GState<K, G, MODE>::KB;
    S.stop = code;
    if (P.pilot) {
        if (lane == 0) P.pilot_w[sk.qidx] = code == kEscalate ? -1 : S.delta_w;
        return;
    }
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

template <int K, int G, int MODE, bool ODD, bool FM>
__device__ __forceinline__ void gstep(GState<K, G, MODE>& S, int32_t (&cur)[K / G],
                                      int32_t (&prv)[K / G], const TierParams& P,
                                      const tab_t* __restrict__ tab, int32_t gap, int32_t X,
                                      unsigned it, int lane, unsigned gmask, GSink& sk) {
    // the main-path shuffles use the full mask when the whole warp steps
    // together; the rare path (group-divergent) always uses the group's mask
    const unsigned smask = FM ? 0xFFFFFFFFu : gmask;
    using St = GState<K, G, MODE>;
    constexpr int SS = St::S;
    constexpr int KB = St::KB;
    const int d = S.d;
    const int k0 = lane * SS;
    const int32_t beta = -gap;
    S.Tc += beta << 6;
    // window of row d, unclamped below d_vm (see the thread tier's xstep)
    const int M = ODD ? max(S.lr1 + 1, S.lr2) : max(S.lr1, S.lr2);  // KB - s_lo
    const int s_hi = ODD ? max(S.hs1, S.hs2) : max(S.hs1 + 1, S.hs2);
    int wm1 = s_hi + M - KB;
    uint32_t vml = gbits(0, SS - 1);  // this lane's in-matrix slots
    [[maybe_unused]] uint32_t inv = 0u;
    const int32_t negC = -((X << 6) + 63);
    int32_t cand[SS], key[SS];
    // Table modes: pass 1 runs speculatively on the current state, beside the
    // rare-path test that the previous step's live-range gather feeds; a
    // group that takes the rare path (which may shift the band or mark the
    // matrix edge) redoes it after.  (Measured: C3 3.61 -> 3.40 ms.  The same
    // reordering made the 2-bit DNA step slower under load, C2 6.63 -> 6.77
    // ms, so that mode keeps pass 1 after the rare path.)
    [[maybe_unused]] auto tpass1 = [&](unsigned msk) __attribute__((always_inline)) {
        // gap source across the lane edge
        int32_t edge;
        if constexpr (ODD) {
            edge = __shfl_down_sync(msk, prv[0], 1, G);
            if (lane == G - 1) edge = kDeadS;
        } else {
            edge = __shfl_up_sync(msk, prv[SS - 1], 1, G);
            if (lane == 0) edge = kDeadS;
        }
        // match bytes (see the thread tier): byte j of Z[q] = 1 + 2*match of slot 4j+q
        [[maybe_unused]] uint32_t Z[4];
        if constexpr (MODE == 0) {
            const uint32_t x = glop3<0xBE>(S.VW, S.HW, inv);  // (a ^ b) | c
            const uint32_t z = ~(x | (x << 1));
    #pragma unroll
            for (int q = 0; q < 4; ++q) Z[q] = ((z >> (2 * q)) & 0x02020202u) | 0x01010101u;
        }

        // pass 1: candidates and keys (key' = 64 cand + s, lane-relative)
    #pragma unroll
        for (int s = SS - 1; s >= 0; --s) {
            const int32_t dg = cur[s];
            int32_t db;
            if constexpr (MODE == 0) {
                db = __dp4a(int(Z[s & 3]), 1 << (8 * ((s >> 2) & 3)), dg);
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
            key[s] = cand[s] * 64 + s;
        }
    };
    if constexpr (MODE != 0) tpass1(smask);
    // group-uniform rare path
    if ((M > KB || unsigned(s_hi) > unsigned(K - 1) || unsigned(wm1) >= unsigned(P.band) ||
         d >= S.d_lim) && !S.stop) {
        const bool e1 = S.hs1 < 0, e2 = S.hs2 < 0;
        if ((e1 && e2) || d > S.n + S.m + 1 || d > S.dcap) {
            gfinish<K, G, MODE>(S, P, kDone, 0, sk, beta, cur, prv, lane, gmask);
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
            if (w > P.band) {
                gfinish<K, G, MODE>(S, P, kBand, w, sk, beta, cur, prv, lane, gmask);
            } else {
                if (lo < 0 || hi > K - 1) {
                    const int wu = hi - lo + 1;
                    if (wu > K) {
                        gfinish<K, G, MODE>(S, P, kEscalate, 0, sk, beta, cur, prv, lane, gmask);
                    } else {
                        const int sh = lo - ((K - wu) >> 1);
                        for (int q = sh; q > 0; --q) {
                            g_shift1<SS, G>(cur, 1, lane, gmask);
                            g_shift1<SS, G>(prv, 1, lane, gmask);
                        }
                        for (int q = sh; q < 0; ++q) {
                            g_shift1<SS, G>(cur, -1, lane, gmask);
                            g_shift1<SS, G>(prv, -1, lane, gmask);
                        }
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
                        g_limits(S);
                        constexpr int PER = St::RPER;
                        const int to_refill = PER - int(it & (PER - 1));
                        g_windows(S, P.pool, lane, ODD ? to_refill : to_refill - 1, to_refill);
                    }
                }
                if (!S.stop && d >= S.d_vm) {
                    const int klo = A - S.n;
                    const int khi = S.m - (d - fd) - S.ubase;
                    const int l = max(klo - k0, 0), h = min(min(khi, K - 1) - k0, SS - 1);
                    vml = gbits(l, h);
                    if constexpr (MODE == 0)
                        inv = ~((l > h) ? 0u : gbits(2 * l, 2 * h + 1));
                    else
                        g_sentinels(S, d, k0);
                }
                wm1 = max(w, 0) - 1;
            }
        }
        if constexpr (MODE != 0) tpass1(gmask);
    }
    S.cells += wm1 + 1;
    S.delta_w = max(S.delta_w, wm1 + 1);

    if constexpr (MODE == 0) {
        // gap source across the lane edge
        int32_t edge;
        if constexpr (ODD) {
            edge = __shfl_down_sync(smask, prv[0], 1, G);
            if (lane == G - 1) edge = kDeadS;
        } else {
            edge = __shfl_up_sync(smask, prv[SS - 1], 1, G);
            if (lane == 0) edge = kDeadS;
        }
        // match bytes (see the thread tier): byte j of Z[q] = 1 + 2*match of slot 4j+q
        [[maybe_unused]] uint32_t Z[4];
        if constexpr (MODE == 0) {
            const uint32_t x = glop3<0xBE>(S.VW, S.HW, inv);  // (a ^ b) | c
            const uint32_t z = ~(x | (x << 1));
    #pragma unroll
            for (int q = 0; q < 4; ++q) Z[q] = ((z >> (2 * q)) & 0x02020202u) | 0x01010101u;
        }

        // pass 1: candidates and keys (key' = 64 cand + s, lane-relative)
    #pragma unroll
        for (int s = SS - 1; s >= 0; --s) {
            const int32_t dg = cur[s];
            int32_t db;
            if constexpr (MODE == 0) {
                db = __dp4a(int(Z[s & 3]), 1 << (8 * ((s >> 2) & 3)), dg);
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
            key[s] = cand[s] * 64 + s;
        }
    }
    // pass 2: one all-gather round of the lane maxima gives every lane the
    // maximum over the higher lanes (its chain input) and the group maximum
    // (the chain's end, i.e. the antidiagonal's running best)
    int32_t Mk = key[0];
#pragma unroll
    for (int s = 1; s < SS; ++s) Mk = max(Mk, key[s]);
    Mk += k0;  // true keys carry the group slot index
    int32_t above = -(1 << 30), all = -(1 << 30);  // below every key, and -C cannot wrap
    {
        int32_t Mj[G];
#pragma unroll
        for (int j = 0; j < G; ++j) Mj[j] = __shfl_sync(smask, Mk, j, G);
        // lane-constant offsets (0 for higher lanes, -2^29 otherwise: keys are
        // below 2^29 by the drift-range guard, so a masked key minus C stays
        // below Tc > 0) instead of a select chain
        static_assert(G == 4, "written for G = 4");
        above = __vimax3_s32(Mj[1] + (lane < 1 ? 0 : -(1 << 29)), Mj[2] + (lane < 2 ? 0 : -(1 << 29)),
                             Mj[3] + (lane < 3 ? 0 : -(1 << 29)));
        all = __vimax3_s32(Mj[0], Mj[1], max(Mj[2], Mj[3]));
    }
    int32_t c = __viaddmax_s32(above, negC, S.Tc);
    // pass 3: lane-local chain, drop test, dead mask (lane-relative keys)
    c -= k0;
    uint32_t dm = 0u;
#pragma unroll
    for (int s = SS - 1; s >= 0; --s) {
        c = __viaddmax_s32(key[s], negC, c);
        if (key[s] < c) {
            cand[s] = kDeadS;
            dm |= 1u << s;
        }
        cur[s] = cand[s];
    }
    // the chain's end: max(Tc, group max key - C)
    const int32_t cf = __viaddmax_s32(all, negC, S.Tc);
    if (cf != S.Tc) {
        const int32_t c63 = cf + 63;
        S.Tc = c63 & ~63;
        S.best_d = d;
        S.best_u = S.ubase + (c63 & 63);
    }
    // live slots of the group: one all-gather round of the lane masks
    S.hs2 = S.hs1;
    S.lr2 = S.lr1;
    {
        const uint32_t lv = ~dm & vml;
        if constexpr (St::NM == 1) {
            const uint32_t mine = lv << k0;
            uint32_t full = 0u;
#pragma unroll
            for (int j = 0; j < G; ++j) full |= __shfl_sync(smask, mine, j, G);
            S.hs1 = gbfind32(full);
            S.lr1 = gbfind32(__brev(full));
        } else {
            const uint64_t mine = uint64_t(lv) << k0;
            uint64_t full = 0ull;
#pragma unroll
            for (int j = 0; j < G; ++j) full |= __shfl_sync(smask, mine, j, G);
            S.hs1 = gbfind64(full);
            S.lr1 = gbfind64(__brevll(full));
        }
    }
    gfeed<K, G, MODE, ODD, FM>(S, P, d, lane, gmask);
    S.d = d + 1;
}

template <int K, int G, int MODE>
__global__ void __launch_bounds__(128) group_tier_kernel(TierParams P) {
    using St = GState<K, G, MODE>;
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
    GSink sk;
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
                S.hs1 = K / 2;
                S.lr1 = KB - K / 2;
                S.hs2 = S.lr2 = -1;
                S.Tc = 64;
                S.best_d = S.best_u = 0;
                S.delta_w = 1;
                S.cells = 1;
#pragma unroll
                for (int s = 0; s < SS; ++s) {
                    O[s] = kDeadS;
                    E[s] = (k0 + s == K / 2) ? X + 1 : kDeadS;
                }
                g_limits(S);
                g_windows(S, P.pool, lane, r, r);
            } else {
                // continue from a narrower tier's record (see resume_unit)
                const int ko = __ldcg(rec + kRecK);
                const int off = (K - ko) >> 1;
                const int d = __ldcg(rec + kRecD);
                S.ubase = __ldcg(rec + kRecUbase) - off;
                S.Tc = __ldcg(rec + kRecTc);
                S.best_d = __ldcg(rec + kRecBestD);
                S.best_u = __ldcg(rec + kRecBestU);
                S.cells = __ldcg(rec + kRecCells);
                S.delta_w = __ldcg(rec + kRecDeltaW);
                const int h1 = __ldcg(rec + kRecHs1), l1 = __ldcg(rec + kRecLs1), h2 = __ldcg(rec + kRecHs2), l2 = __ldcg(rec + kRecLs2);
                S.hs1 = h1 < 0 ? -1 : h1 + off;
                S.lr1 = h1 < 0 ? -1 : KB - (l1 + off);
                S.hs2 = h2 < 0 ? -1 : h2 + off;
                S.lr2 = h2 < 0 ? -1 : KB - (l2 + off);
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
                g_windows(S, P.pool, lane, odd ? r : St::RPER - 1, odd ? r : St::RPER - 1);
                S.d = d;
                g_limits(S);
                if (!odd) {
                    if (lane == 0) atomicAdd(&P.ctr->dbg[5], 1ull);  // stats: even-d resumes
                    gfeed<K, G, MODE, true, false>(S, P, d - 1, lane, gmask);
                    gstep<K, G, MODE, false, false>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
                    if (!S.stop) g_windows(S, P.pool, lane, r, r);  // the loop's refill schedule
                }
            }
            active = true;
            return;
        }
    };
    fetch();
    it = 0;
    // the consumer's polling lives in its own copy of the loop, so the
    // ordinary launches run the loop without it
    auto run = [&](auto cons) {
        constexpr bool CONS = decltype(cons)::value;
        if constexpr (!CONS) {
            // the steps run in an inner loop that fetch() is not part of: it
            // exits (one vote per iteration, as the loop test was) when some
            // group's unit is decided, so the back edge carries no merge with
            // fetch()'s writes
            while (__any_sync(0xFFFFFFFFu, active)) {
                for (;;) {
                    if (active && (it & (St::RPER - 1)) == 0) {
                        if (lane == 0) S.rv.refill(P.pool);
                        if (lane == G - 1) S.rh.refill(P.pool);
                    }
                    gstep<K, G, MODE, true, true>(S, O, E, P, tab, gap, X, it, lane, gmask, sk);
                    gstep<K, G, MODE, false, true>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
                    if (__any_sync(0xFFFFFFFFu, active && S.stop)) break;
                    ++it;
                }
                if (active && S.stop) fetch();
                ++it;
            }
            return;
        }
        while (__any_sync(0xFFFFFFFFu, active || (CONS && waiting))) {
            if constexpr (CONS) {
                if (!__any_sync(0xFFFFFFFFu, active)) {  // nothing queued for this warp yet
                    __nanosleep(2000);
                    if (waiting) fetch();
                    ++it;
                    continue;
                }
            }
            if (active && (it & (St::RPER - 1)) == 0) {
                if (lane == 0) S.rv.refill(P.pool);
                if (lane == G - 1) S.rh.refill(P.pool);
            }
            // every group steps on odd d here (fetch() runs the even step of a
            // unit resumed at an even d), so the warp needs no peeled half
            gstep<K, G, MODE, true, true>(S, O, E, P, tab, gap, X, it, lane, gmask, sk);
            gstep<K, G, MODE, false, true>(S, E, O, P, tab, gap, X, it, lane, gmask, sk);
            // outcome recorded by the deciding step; idle consumer groups poll every 8th iteration
            if ((active && S.stop) || (CONS && !active && waiting && (it & 7) == 0)) fetch();
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

#define XB_GINST(K, G)                                                     \
    template __global__ void group_tier_kernel<K, G, 0>(TierParams);       \
    template __global__ void group_tier_kernel<K, G, 1>(TierParams);       \
    template __global__ void group_tier_kernel<K, G, 2>(TierParams);
XB_GINST(16, 4)
XB_GINST(24, 4)
XB_GINST(32, 4)
XB_GINST(48, 4)
XB_GINST(64, 4)
#undef XB_GINST

}  // namespace xb
