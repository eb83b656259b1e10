// Lane-group tiers: G lanes of a warp cooperate on one unit, each holding
// S = K/G consecutive slots of the register band.  Same exact semantics as
// the thread tier (xb_thread.cu, proofs in xb_kernels.cuh); what changes is
// the plumbing between slots that live in different lanes:
//   * the one gap source that crosses a lane edge comes by SHFL (up on even
//     antidiagonals, down on odd ones), and so do the symbols entering a
//     lane's window;
//   * the running-best chain, which runs over slots in descending order,
//     becomes: lane-local key maximum -> exclusive suffix-max across the
//     group (log2 G shuffles) -> lane-local chain seeded with it;
//   * the live range is an OR-butterfly of the lanes' live bits.
// A step then costs ~S slots of dependent work plus a few shuffle rounds
// instead of K slots, so a unit advances several times faster: this tier
// serves work that is latency- rather than throughput-bound (escalation
// tails, the pilot, and batches too small to fill the machine).
#include <climits>
#include <cstdint>
#include <utility>

#include "xb_kernels.cuh"

namespace xb {

namespace {

__device__ __forceinline__ uint32_t gbits(int lo, int hi) {
    if (lo > hi) return 0u;
    return (0xFFFFFFFFu >> (31 - hi)) & (0xFFFFFFFFu << lo);
}

template <int K, int G, int MODE>
struct GState {
    static constexpr int S = K / G;          // slots per lane
    static constexpr int NB = (S + 3) / 4;   // byte-window words per lane (table mode)
    static constexpr int NM = (K + 31) / 32; // group live-mask words
    int64_t h_pos, v_pos;
    int32_t m, n, hdir, vdir, unit;
    int32_t d, ubase, dcap;
    int32_t ls1, hs1, ls2, hs2;  // global slots, empty = (kBig, -kBig)
    int32_t d_vm, d_lim, stop, spread;
    int32_t T, best_d, best_i, delta_w, cells;
    uint32_t VW, HW;             // 2-bit windows of this lane's S slots (MODE 0)
    uint32_t VWb[NB], HWb[NB];   // byte windows (table modes)
    Reader<true> rv;             // lane 0: v symbols entering slot 0
    Reader<false> rh;            // lane G-1: h symbols entering slot K-1
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

}  // namespace

template <int K, int G, int MODE, bool ODD>
__device__ __forceinline__ void gstep(GState<K, G, MODE>& S, int32_t (&cur)[K / G],
                                      int32_t (&prv)[K / G], const TierParams& P,
                                      const int8_t* __restrict__ tab, int32_t gap, int32_t X,
                                      unsigned it, int lane, unsigned gmask) {
    using St = GState<K, G, MODE>;
    constexpr int SS = St::S;
    const int d = S.d;
    const int k0 = lane * SS;
    int s_lo = ODD ? min(S.ls1 - 1, S.ls2) : min(S.ls1, S.ls2);
    int s_hi = ODD ? max(S.hs1, S.hs2) : max(S.hs1 + 1, S.hs2);
    const int fd = d >> 1;
    int A = fd - S.ubase;
    const int w = min(s_hi, A - max(d - S.m, 0)) - max(s_lo, A - min(d, S.n)) + 1;
    uint32_t vml = gbits(0, SS - 1);                // this lane's in-matrix slots
    uint32_t vmsl = gbits(0, 2 * SS - 1) & 0xAAAAAAAAu;
    // group-uniform rare path
    if ((s_lo < 0 || unsigned(s_hi) > unsigned(K - 1) || w > P.band || d >= S.d_lim) && !S.stop) {
        if (s_hi < 0 || d > S.n + S.m + 1 || d > S.dcap) {
            S.stop = kDone;
        } else if (w > P.band) {
            S.stop = kBand;
            S.spread = w;
        } else {
            if (s_lo < 0 || s_hi > K - 1) {
                const int wu = s_hi - s_lo + 1;
                if (wu > K) {
                    S.stop = kEscalate;
                } else {
                    const int sh = s_lo - ((K - wu) >> 1);
                    for (int q = sh; q > 0; --q) {
                        g_shift1<SS, G>(cur, 1, lane, gmask);
                        g_shift1<SS, G>(prv, 1, lane, gmask);
                    }
                    for (int q = sh; q < 0; ++q) {
                        g_shift1<SS, G>(cur, -1, lane, gmask);
                        g_shift1<SS, G>(prv, -1, lane, gmask);
                    }
                    S.ubase += sh;
                    S.ls1 -= sh;
                    S.hs1 -= sh;
                    S.ls2 -= sh;
                    S.hs2 -= sh;
                    A -= sh;
                    g_limits(S);
                    const int to_refill = 16 - int(it & 15);
                    g_windows(S, P.pool, lane, ODD ? to_refill : to_refill - 1, to_refill);
                }
            }
            if (d >= S.d_vm) {
                const int klo = A - S.n;
                const int khi = S.m - (d - fd) - S.ubase;
                const int l = max(klo - k0, 0), h = min(min(khi, K - 1) - k0, SS - 1);
                vml = gbits(l, h);
                vmsl = (l > h) ? 0u : (gbits(2 * l, 2 * h + 1) & 0xAAAAAAAAu);
            }
        }
    }
    if (!S.stop) {
        S.cells += max(w, 0);
        S.delta_w = max(S.delta_w, w);
    }

    // gap source across the lane edge
    int32_t edge;
    if constexpr (ODD) {
        edge = __shfl_down_sync(gmask, prv[0], 1, G);
        if (lane == G - 1) edge = kDeadS;
    } else {
        edge = __shfl_up_sync(gmask, prv[SS - 1], 1, G);
        if (lane == 0) edge = kDeadS;
    }
    [[maybe_unused]] uint32_t Z = 0;
    if constexpr (MODE == 0) {
        const uint32_t x = S.VW ^ S.HW;
        Z = ~(x | (x << 1)) & vmsl;
    }

    const int32_t beta = -gap;
    const int32_t negC = -((X << 6) + 63);
    const int32_t c_init = (S.T + beta * d + 1) << 6;
    // pass 1: candidates and keys (key' = 64 cand + s, lane-relative)
    int32_t cand[SS], key[SS];
#pragma unroll
    for (int s = SS - 1; s >= 0; --s) {
        const int32_t dg = cur[s];
        int32_t db;
        if constexpr (MODE == 0) {
            const uint32_t t = (3u << (2 * s)) & (Z | P.pat);
            db = s == 0 ? dg + int32_t(t) : dg + int32_t(__umulhi(t, 1u << (32 - 2 * s)));
        } else {
            const int r = s >> 2, q = s & 3;
            uint32_t idx = 0;
            switch (q) {  // bytes: v code, h code, 0, 0
                case 0: asm("prmt.b32 %0, %1, %2, 0x8840;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                case 1: asm("prmt.b32 %0, %1, %2, 0x9951;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                case 2: asm("prmt.b32 %0, %1, %2, 0xAA62;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
                default: asm("prmt.b32 %0, %1, %2, 0xBB73;" : "=r"(idx) : "r"(S.VWb[r]), "r"(S.HWb[r])); break;
            }
            db = dg + int32_t(tab[idx]);
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
    // pass 2: exclusive suffix maximum of (key - C) over the higher lanes
    int32_t M = key[0];
#pragma unroll
    for (int s = 1; s < SS; ++s) M = max(M, key[s]);
    M += k0;  // true keys carry the global slot index
#pragma unroll
    for (int o = 1; o < G; o <<= 1) {
        const int32_t y = __shfl_down_sync(gmask, M, o, G);
        if (lane + o < G) M = max(M, y);
    }
    int32_t above = __shfl_down_sync(gmask, M, 1, G);
    int32_t c = lane == G - 1 ? c_init : __viaddmax_s32(above, negC, c_init);
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
    c += k0;
    // lane 0 ends the chain: the antidiagonal's best
    const int32_t cf = __shfl_sync(gmask, c, 0, G) + ((X << 6) + 63);
    {
        const int32_t qnew = cf >> 6;
        const int32_t qold = S.T + beta * d + X + 1;
        if (qnew > qold && !S.stop) {
            S.T = qnew - beta * d - X - 1;
            S.best_d = d;
            S.best_i = A - (cf & 63);
        }
    }
    // live slots of the group: OR-butterfly of lane masks
    {
        const uint32_t lv = ~dm & vml;
        int hs, ls;
        bool any;
        if constexpr (St::NM == 1) {
            uint32_t full = lv << k0;
#pragma unroll
            for (int o = 1; o < G; o <<= 1) full |= __shfl_xor_sync(gmask, full, o, G);
            any = full != 0u;
            hs = 31 - __clz(full);
            ls = __ffs(full) - 1;
        } else {
            uint64_t full = uint64_t(lv) << k0;
#pragma unroll
            for (int o = 1; o < G; o <<= 1) full |= __shfl_xor_sync(gmask, full, o, G);
            any = full != 0ull;
            hs = 63 - __clzll((long long)full);
            ls = __ffsll((long long)full) - 1;
        }
        S.ls2 = S.ls1;
        S.hs2 = S.hs1;
        S.ls1 = any ? ls : kBig;
        S.hs1 = any ? hs : -kBig;
    }
    // symbols entering on d+1
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
        constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
        constexpr int NB = St::NB;
        constexpr int top = 8 * ((SS - 1) & 3);  // bit offset of slot SS-1 in its word
        if constexpr (ODD) {
            const uint32_t out = (S.VWb[NB - 1] >> top) & 0xFFu;
            uint32_t in = __shfl_up_sync(gmask, out, 1, G);
            if (lane == 0) in = code_at<ENC>(P.pool, S.v_pos, S.vdir, S.n, int64_t(fd) - S.ubase);
#pragma unroll
            for (int r = NB - 1; r > 0; --r) S.VWb[r] = __funnelshift_l(S.VWb[r - 1], S.VWb[r], 8);
            S.VWb[0] = (S.VWb[0] << 8) | in;
        } else {
            const uint32_t out = S.HWb[0] & 0xFFu;
            uint32_t in = __shfl_down_sync(gmask, out, 1, G);
            if (lane == G - 1)
                in = code_at<ENC>(P.pool, S.h_pos, S.hdir, S.m, int64_t(d - fd) + S.ubase - 1 + K);
#pragma unroll
            for (int r = 0; r < NB - 1; ++r) S.HWb[r] = __funnelshift_r(S.HWb[r], S.HWb[r + 1], 8);
            const uint32_t keep = top == 24 ? 0xFFFFFFFFu : ((1u << (top + 8)) - 1u);
            S.HWb[NB - 1] = ((S.HWb[NB - 1] >> 8) & (keep >> 8)) | (in << top);
        }
    }
    S.d = d + 1;
}

template <int K, int G, int MODE>
__global__ void __launch_bounds__(128) group_tier_kernel(TierParams P) {
    using St = GState<K, G, MODE>;
    constexpr int SS = St::S;
    __shared__ int8_t tab[MODE == 0 ? 4 : 32 * 256];
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    const int wl = threadIdx.x & 31;
    const int lane = wl % G;
    const int gbase = wl - lane;
    const unsigned gmask = (G == 32 ? 0xFFFFFFFFu : ((1u << G) - 1u)) << gbase;

    Queue Q;
    if (!make_queue(P, Q)) return;
    if constexpr (MODE != 0) {
        for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) {
            const int h = i >> 8, v = i & 255;
            int val = -128;
            if (v < 32 && h != kSentinel && v != kSentinel) {
                val = P.scheme->sim[v * 32 + h] - 2 * gap;
                val = max(-127, min(127, val));
            }
            tab[i] = int8_t(val);
        }
        __syncthreads();
    }
    const int next_tier = P.esc_to_warp ? kWarpTier : P.tier + 1;
    uint32_t* esc_list = P.lists + (long long)next_tier * P.n_units;
    unsigned long long* esc_len = &P.ctr->list_len[next_tier];
    unsigned long long my_units = 0, my_cells = 0, my_esc = 0;

    St S;
    int32_t E[SS], O[SS];
    bool active = false;
    long long qidx = 0;
    unsigned it = 0xFFFFFFFFu;
    auto fetch = [&]() {
        active = false;
        for (;;) {
            unsigned long long i = 0;
            if (lane == 0) i = atomicAdd(Q.cursor, 1ull);
            i = __shfl_sync(gmask, i, 0, G);
            if (i >= Q.len) return;
            const uint32_t unit = Q.q[(long long)i * Q.stride];
            const DevUnit u = P.units[unit];
            if (u.route != 0) {
                if (P.pilot && lane == 0) P.pilot_w[i] = -2;
                continue;
            }
            qidx = (long long)i;
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
            S.ls1 = S.hs1 = K / 2;
            S.ls2 = kBig;
            S.hs2 = -kBig;
            S.stop = 0;
            S.spread = 0;
            S.T = S.best_d = S.best_i = 0;
            S.delta_w = 1;
            S.cells = 1;
            g_limits(S);
#pragma unroll
            for (int s = 0; s < SS; ++s) {
                O[s] = kDeadS;
                E[s] = (lane * SS + s == K / 2) ? X + 1 : kDeadS;
            }
            const int r = 15 - int(it & 15);
            g_windows(S, P.pool, lane, r, r);
            active = true;
            return;
        }
    };
    fetch();
    it = 0;
    while (__any_sync(0xFFFFFFFFu, active)) {
        if (active) {
            if constexpr (MODE == 0) {
                if ((it & 15) == 0) {
                    if (lane == 0) S.rv.refill(P.pool);
                    if (lane == G - 1) S.rh.refill(P.pool);
                }
            }
            gstep<K, G, MODE, true>(S, O, E, P, tab, gap, X, it, lane, gmask);
            gstep<K, G, MODE, false>(S, E, O, P, tab, gap, X, it, lane, gmask);
            if (S.stop) {
                const int r = S.stop;
                if (lane == 0) {
                    if (P.pilot) {
                        P.pilot_w[qidx] = r == kEscalate ? -1 : S.delta_w;
                    } else if (r == kEscalate) {
                        const unsigned long long slot = atomicAdd(esc_len, 1ull);
                        esc_list[slot] = uint32_t(S.unit);
                        ++my_esc;
                    } else {
                        DevResult res;
                        res.cells = S.cells;
                        res.delta_w = S.delta_w;
                        if (r == kBand) {
                            res.score = res.h_ext = res.v_ext = 0;
                            res.status = kStatusBand;
                            res.spread = S.spread;
                        } else {
                            res.score = S.T;
                            res.h_ext = S.best_d - S.best_i;
                            res.v_ext = S.best_i;
                            res.status = kStatusOk;
                            res.spread = 0;
                        }
                        P.results[S.unit] = res;
                        ++my_units;
                        my_cells += (unsigned long long)S.cells;
                    }
                }
                fetch();
            }
        }
        ++it;
    }
    if (P.pilot || lane != 0) return;
    if (my_units) atomicAdd(&P.ctr->units[P.tier], my_units);
    if (my_cells) atomicAdd(&P.ctr->cells[P.tier], my_cells);
    if (my_esc) atomicAdd(&P.ctr->escalated[P.tier], my_esc);
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
