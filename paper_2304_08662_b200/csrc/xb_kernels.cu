// sm_100a device code: LR split/prep, thread tiers (register band), warp
// tier (exact generic path), and the INT32 issue-rate microbenchmark.
// See xb_kernels.cuh for the coordinate system and DESIGN.md for the proofs.
#include <climits>
#include <cstdint>

#include "xb_kernels.cuh"

namespace xb {

// ------------------------------------------------------------- helpers ----

// contiguous bit range [lo, hi] of a 32-bit word, lo/hi already clamped to
// [0, 31]; empty when lo > hi
__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {
    if (lo > hi) return 0u;
    const uint32_t up = 0xFFFFFFFFu >> (31 - hi);
    return up & (0xFFFFFFFFu << lo);
}

template <int K>
__device__ __forceinline__ void shift_slots(int32_t (&R)[K], int s) {
    // new slot k <- old slot k + s  (s != 0), vacated slots dead
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

// ------------------------------------------------------ thread tier ----

template <int K, int MODE>
__device__ __forceinline__ void init_windows(TState<K, MODE>& S, const uint32_t* __restrict__ pool) {
    const int fd = S.d >> 1, cd = S.d - fd;
    const int64_t a = int64_t(fd) - S.ubase - 1;  // v index of slot 0
    const int64_t b = int64_t(cd) + S.ubase - 1;  // h index of slot 0
    if constexpr (MODE == 0) {
#pragma unroll
        for (int w = 0; w < TState<K, MODE>::NW; ++w) {
            S.HW[w] = chunk_bf(pool, S.h_pos, S.hdir, b + 16 * w);
            S.VW[w] = chunk_tf(pool, S.v_pos, S.vdir, a - 16 * w - 15);
        }
        S.rv.init(pool, S.v_pos, S.vdir, a + 1);
        S.rh.init(pool, S.h_pos, S.hdir, b + K);
    } else {
        constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
#pragma unroll
        for (int r = 0; r < TState<K, MODE>::NB; ++r) {
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
    }
}

template <int K, int MODE>
__device__ __forceinline__ void start_unit(TState<K, MODE>& S, int32_t (&E)[K], int32_t (&O)[K],
                                           const TierParams& P, uint32_t unit, int32_t X) {
    const DevUnit u = P.units[unit];
    S.unit = int32_t(unit);
    S.h_pos = u.h_pos;
    S.v_pos = u.v_pos;
    S.m = u.h_len;
    S.n = u.v_len;
    S.hdir = u.dir & 1;
    S.vdir = (u.dir >> 1) & 1;
    S.d = 1;
    S.ubase = -(K / 2);
    S.fl1 = 0;  // antidiagonal 0: the origin
    S.ll1 = 0;
    S.fl2 = 0;  // antidiagonal -1: empty
    S.ll2 = -1;
    S.T = 0;
    S.best_d = 0;
    S.best_i = 0;
    S.delta_w = 1;
    S.cells = 1;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        O[k] = kDeadS;
        E[k] = (k == K / 2) ? X + 1 : kDeadS;  // s(0,0) = 0 + 0 + off
    }
    init_windows(S, P.pool);
}

// One antidiagonal d.  cur holds d-2 on entry and d on exit, prv holds d-1.
template <int K, int MODE, bool ODD>
__device__ __forceinline__ int xstep(TState<K, MODE>& S, int32_t (&cur)[K], int32_t (&prv)[K],
                                     const TierParams& P, const int8_t* __restrict__ tab,
                                     int32_t gap, int32_t X, int32_t& spread) {
    using St = TState<K, MODE>;
    const int d = S.d;
    if (d > S.n + S.m + 1) return kDone;
    const bool have1 = S.fl1 <= S.ll1, have2 = S.fl2 <= S.ll2;
    if (!have1 && !have2) return kDone;  // align.cpp:64-66

    // reachable window (align.cpp:68-81)
    int lo_u = have1 ? S.fl1 : INT_MAX;
    int hi_u = have1 ? S.ll1 + 1 : INT_MIN;
    if (have2) {
        lo_u = min(lo_u, S.fl2 + 1);
        hi_u = max(hi_u, S.ll2 + 1);
    }
    const int lo = max(lo_u, max(d - S.m, 0));
    const int hi = min(hi_u, min(d, S.n));
    if (lo <= hi) {  // an empty window counts nothing (align.cpp:84-91)
        const int w = hi - lo + 1;
        if (w > P.band) {  // align.cpp:93-94: first overflow, cells so far
            spread = w;
            return kBand;
        }
        S.cells += w;
        S.delta_w = max(S.delta_w, w);
    }

    const int fd = d >> 1, cd = d - fd;
    // every live source lies inside the unclamped window, so it must fit
    {
        const int s_lo = fd - hi_u - S.ubase, s_hi = fd - lo_u - S.ubase;
        if (s_lo < 0 || s_hi > K - 1) {
            const int wu = hi_u - lo_u + 1;
            if (wu > K) return kEscalate;
            const int nb = fd - hi_u - ((K - wu) >> 1);
            shift_slots<K>(cur, nb - S.ubase);
            shift_slots<K>(prv, nb - S.ubase);
            S.ubase = nb;
            init_windows(S, P.pool);
        }
    }

    // slots inside the matrix: i <= n  <=>  k >= klo ;  j <= m  <=>  k <= khi
    const int klo = fd - S.ubase - S.n;
    const int khi = S.m - cd - S.ubase;
    uint32_t vm[St::NM];
    [[maybe_unused]] uint32_t vms[St::NW];
    if (klo <= 0 && khi >= K - 1) {
#pragma unroll
        for (int q = 0; q < St::NM; ++q) vm[q] = 0xFFFFFFFFu;
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = 0; w < St::NW; ++w) vms[w] = 0xAAAAAAAAu;
        }
    } else {
#pragma unroll
        for (int q = 0; q < St::NM; ++q)
            vm[q] = bit_range(max(klo - 32 * q, 0), min(khi - 32 * q, 31));
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = 0; w < St::NW; ++w) {
                const int l = max(klo - 16 * w, 0), h = min(khi - 16 * w, 15);
                vms[w] = bit_range(2 * l, 2 * h + 1) & 0xAAAAAAAAu;
            }
        }
    }

    // DNA +1/-1/-1: bit 2f+1 of Z[w] = slot (16w+f) is a match inside the matrix
    [[maybe_unused]] uint32_t Z[St::NW];
    if constexpr (MODE == 0) {
#pragma unroll
        for (int w = 0; w < St::NW; ++w) {
            const uint32_t x = S.VW[w] ^ S.HW[w];
            Z[w] = ~(x | (x << 1)) & vms[w];
        }
    }

    // exact running best + drop test (see header): chain over k = K-1..0
    const int32_t beta = -gap;
    const int32_t C = (X << 6) + 63;
    int32_t c = (S.T + beta * d + 1) << 6;
    uint32_t dm[St::NM];
#pragma unroll
    for (int q = 0; q < St::NM; ++q) dm[q] = 0u;
    const uint32_t PAT = P.pat;

#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
        const int32_t dg = cur[k];
        int32_t db;
        if constexpr (MODE == 0) {
            const int w = k >> 4, f = k & 15;
            // t = [match bit at 2f+1][1 at 2f]:  (t >> 2f) = 1 + 2*match = sim - 2gap
            const uint32_t t = (3u << (2 * f)) & (Z[w] | PAT);
            db = (f == 0) ? dg + int32_t(t) : dg + int32_t(__umulhi(t, 1u << (32 - 2 * f)));
        } else {
            const int r = k >> 2, q = k & 3;
            const uint32_t idx =
                __byte_perm(S.VW[r], S.HW[r], uint32_t(q | ((q + 4) << 4))) & 0x1F1Fu;
            db = dg + int32_t(tab[idx]);
        }
        int32_t ln, un;
        if constexpr (ODD) {  // gap sources at u and u+1
            ln = prv[k];
            un = (k < K - 1) ? prv[k + 1] : kDeadS;
        } else {              // gap sources at u-1 and u
            ln = (k > 0) ? prv[k - 1] : kDeadS;
            un = prv[k];
        }
        const int32_t cand = __vimax3_s32(db, ln, un);
        const int32_t key = cand * 64 + k;
        c = __viaddmax_s32(key, -C, c);
        const int32_t sn = (key >= c) ? cand : kDeadS;
        dm[k >> 5] = __funnelshift_l(uint32_t(sn), dm[k >> 5], 1);
        cur[k] = sn;
    }

    // running best (align.cpp:123-127)
    {
        const int32_t cf = c + C;
        const int32_t qnew = cf >> 6;
        const int32_t qold = S.T + beta * d + X + 1;
        if (qnew > qold) {
            S.T = qnew - beta * d - X - 1;
            S.best_d = d;
            S.best_i = fd - S.ubase - (cf & 63);
        }
    }
    // live range of row d (align.cpp:138-145); out-of-matrix slots masked
    {
        uint32_t lv[St::NM];
        bool any = false;
#pragma unroll
        for (int q = 0; q < St::NM; ++q) {
            lv[q] = ~dm[q] & vm[q];
            any |= lv[q] != 0u;
        }
        S.fl2 = S.fl1;
        S.ll2 = S.ll1;
        if (!any) {
            S.fl1 = 0;
            S.ll1 = -1;
        } else {
            int hs, ls;
            if constexpr (St::NM == 1) {
                hs = 31 - __clz(lv[0]);
                ls = __ffs(lv[0]) - 1;
            } else {
                hs = lv[1] ? 63 - __clz(lv[1]) : 31 - __clz(lv[0]);
                ls = lv[0] ? __ffs(lv[0]) - 1 : 31 + __ffs(lv[1]);
            }
            S.fl1 = fd - S.ubase - hs;
            S.ll1 = fd - S.ubase - ls;
        }
    }

    // feed the symbol that enters the band on d+1
    if constexpr (ODD) {  // floor((d+1)/2) grows: v[a+1] enters at slot 0
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = St::NW - 1; w > 0; --w) S.VW[w] = __funnelshift_l(S.VW[w - 1], S.VW[w], 2);
            S.VW[0] = __funnelshift_l(S.rv.cur, S.VW[0], 2);
            S.rv.cur <<= 2;
            if (--S.rv.cnt == 0) S.rv.refill(P.pool);
        } else {
            constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
            const uint32_t code =
                code_at<ENC>(P.pool, S.v_pos, S.vdir, S.n, int64_t(fd) - S.ubase);  // a + 1
#pragma unroll
            for (int r = St::NB - 1; r > 0; --r) S.VW[r] = __funnelshift_l(S.VW[r - 1], S.VW[r], 8);
            S.VW[0] = (S.VW[0] << 8) | code;
        }
    } else {  // ceil((d+1)/2) grows: h[b+K] enters at slot K-1
        if constexpr (MODE == 0) {
#pragma unroll
            for (int w = 0; w < St::NW - 1; ++w) S.HW[w] = __funnelshift_r(S.HW[w], S.HW[w + 1], 2);
            S.HW[St::NW - 1] = __funnelshift_r(S.HW[St::NW - 1], S.rh.cur, 2);
            S.rh.cur >>= 2;
            if (--S.rh.cnt == 0) S.rh.refill(P.pool);
        } else {
            constexpr int ENC = MODE == 1 ? ENC_2BIT : ENC_5BIT;
            const uint32_t code =
                code_at<ENC>(P.pool, S.h_pos, S.hdir, S.m, int64_t(cd) + S.ubase - 1 + K);
#pragma unroll
            for (int r = 0; r < St::NB - 1; ++r) S.HW[r] = __funnelshift_r(S.HW[r], S.HW[r + 1], 8);
            S.HW[St::NB - 1] = __funnelshift_r(S.HW[St::NB - 1], code, 8);
        }
    }
    S.d = d + 1;
    return kGo;
}

template <int K, int MODE>
__global__ void __launch_bounds__(kTB) thread_tier_kernel(TierParams P) {
    __shared__ int8_t tab[MODE == 0 ? 4 : 32 * 256];
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    if constexpr (MODE != 0) {
        // tab[h*256 + v] = sim(v, h) - 2*gap; sentinel rows/cols lose
        for (int q = threadIdx.x; q < 32 * 256; q += blockDim.x) {
            const int h = q >> 8, v = q & 255;
            int val = -128;
            if (v < 32 && h != kSentinel && v != kSentinel) {
                val = P.scheme->sim[v * 32 + h] - 2 * gap;
                val = max(-127, min(127, val));
            }
            tab[q] = int8_t(val);
        }
        __syncthreads();
    }
    const unsigned long long qlen = P.queue_len_ptr ? *P.queue_len_ptr : P.queue_len;
    unsigned long long my_units = 0, my_cells = 0, my_esc = 0;

    TState<K, MODE> S;
    int32_t E[K], O[K];
    bool active = false;

    auto fetch = [&]() {
        active = false;
        for (;;) {
            const unsigned long long q = atomicAdd(&P.ctr->cursor[P.tier], 1ull);
            if (q >= qlen) return;
            const uint32_t unit = P.queue[q];
            if (P.tier == 0 && P.units[unit].route != 0) continue;  // sent to the warp tier by prep
            start_unit<K, MODE>(S, E, O, P, unit, X);
            active = true;
            return;
        }
    };
    fetch();

    while (__any_sync(0xFFFFFFFFu, active)) {
        if (active) {
            int32_t spread = 0;
            int r = xstep<K, MODE, true>(S, O, E, P, tab, gap, X, spread);
            if (r == kGo) r = xstep<K, MODE, false>(S, E, O, P, tab, gap, X, spread);
            if (r != kGo) {
                if (r == kEscalate) {
                    const unsigned long long slot = atomicAdd(P.esc_len, 1ull);
                    P.esc_list[slot] = uint32_t(S.unit);
                    ++my_esc;
                } else {
                    DevResult res;
                    if (r == kBand) {
                        res.score = res.h_ext = res.v_ext = 0;
                        res.delta_w = S.delta_w;
                        res.status = kStatusBand;
                        res.spread = spread;
                    } else {
                        res.score = S.T;
                        res.h_ext = S.best_d - S.best_i;
                        res.v_ext = S.best_i;
                        res.delta_w = S.delta_w;
                        res.status = kStatusOk;
                        res.spread = 0;
                    }
                    res.cells = S.cells;
                    P.results[S.unit] = res;
                    ++my_units;
                    my_cells += (unsigned long long)S.cells;
                }
                fetch();
            }
        }
    }
    if (my_units) atomicAdd(&P.ctr->units[P.tier], my_units);
    if (my_cells) atomicAdd(&P.ctr->cells[P.tier], my_cells);
    if (my_esc) atomicAdd(&P.ctr->escalated[P.tier], my_esc);
}

// explicit instantiations used by the engine
template __global__ void thread_tier_kernel<32, 0>(TierParams);
template __global__ void thread_tier_kernel<64, 0>(TierParams);
template __global__ void thread_tier_kernel<32, 1>(TierParams);
template __global__ void thread_tier_kernel<64, 1>(TierParams);
template __global__ void thread_tier_kernel<32, 2>(TierParams);
template __global__ void thread_tier_kernel<64, 2>(TierParams);

// -------------------------------------------------------- warp tier ----
// One warp per unit, int32 values with the reference's explicit dead marker
// (no range assumptions), rows of `band` cells in the reference's folded
// layout (slot = (k - i) mod band, align.cpp:20-35), lanes striding over the
// window 32 cells at a time with an inclusive max-scan for the running best.

constexpr int32_t kDeadW = INT_MIN;

template <int ENC>
__device__ __forceinline__ int slot_of(int k, int i, int band) {
    int u = (k - i) % band;
    return u < 0 ? u + band : u;
}

template <int ENC>
__global__ void __launch_bounds__(128) warp_tier_kernel(TierParams P) {
    __shared__ int32_t simt[32 * 32];
    for (int q = threadIdx.x; q < 32 * 32; q += blockDim.x) simt[q] = P.scheme->sim[q];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int band = P.band;
    int32_t* rows0 = P.warp_scratch + int64_t(gw) * 2 * band;
    int32_t* rows1 = rows0 + band;
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    const unsigned long long qlen = P.queue_len_ptr ? *P.queue_len_ptr : P.queue_len;
    unsigned long long my_units = 0, my_cells = 0;

    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(&P.ctr->cursor[2], 1ull);
        q = __shfl_sync(0xFFFFFFFFu, q, 0);
        if (q >= qlen) break;
        const uint32_t unit = P.queue[q];
        const DevUnit U = P.units[unit];
        const int m = U.h_len, n = U.v_len;

        int32_t* R[2] = {rows0, rows1};
        int rk[2] = {0, 0}, rfl[2] = {0, 0}, rll[2] = {0, -1};
        if (lane == 0) rows0[0] = 0;  // slot_of(0, 0) = 0
        __syncwarp();
        int32_t T = 0;
        int best_d = 0, best_i = 0, delta_w = 1, status = kStatusOk, spread = 0;
        long long cells = 1;

        for (int d = 1; d <= n + m + 1; ++d) {
            const int ci = d & 1, pi = ci ^ 1;
            int32_t* cur = R[ci];
            const int32_t* prev = R[pi];
            const bool have_prev = rfl[pi] <= rll[pi];
            const bool have_pp = rfl[ci] <= rll[ci];
            if (!have_prev && !have_pp) break;
            long long lo = LLONG_MAX, hi = LLONG_MIN;
            if (have_prev) {
                lo = rfl[pi];
                hi = rll[pi] + 1;
            }
            if (have_pp) {
                lo = min(lo, (long long)rfl[ci] + 1);
                hi = max(hi, (long long)rll[ci] + 1);
            }
            lo = max(lo, (long long)(d > m ? d - m : 0));
            hi = min(hi, (long long)min(d, n));
            const int kn = d / 2;
            if (lo > hi) {
                rk[ci] = kn;
                rfl[ci] = 0;
                rll[ci] = -1;
                continue;
            }
            const long long w = hi - lo + 1;
            if (w > band) {
                status = kStatusBand;
                spread = int(w);
                break;
            }
            if (int(w) > delta_w) delta_w = int(w);
            cells += w;
            const int pp_fl = rfl[ci], pp_ll = rll[ci];
            const int pfl = rfl[pi], pll = rll[pi], pk = rk[pi];
            int first = -1, last = -1;
            for (long long base = lo; base <= hi; base += 32) {
                const int i = int(base) + lane;
                const bool act = i <= hi;
                int32_t val = kDeadW;
                int sg = 0;
                if (act) {
                    const int j = d - i;
                    sg = slot_of<ENC>(kn, i, band);
                    if (i - 1 >= pp_fl && i - 1 <= pp_ll) {
                        const int32_t dg = cur[sg];
                        if (dg != kDeadW) {
                            const uint32_t vc = code_at<ENC>(P.pool, U.v_pos, (U.dir >> 1) & 1, n, i - 1);
                            const uint32_t hc = code_at<ENC>(P.pool, U.h_pos, U.dir & 1, m, j - 1);
                            val = dg + simt[vc * 32 + hc];
                        }
                    }
                    if (j >= 1 && i >= pfl && i <= pll) {
                        const int32_t l = prev[slot_of<ENC>(pk, i, band)];
                        if (l != kDeadW) val = max(val, l + gap);
                    }
                    if (i >= 1 && i - 1 >= pfl && i - 1 <= pll) {
                        const int32_t u = prev[slot_of<ENC>(pk, i - 1, band)];
                        if (u != kDeadW) val = max(val, u + gap);
                    }
                }
                // running best in ascending i: inclusive scan over lanes
                int32_t run = val;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int32_t y = __shfl_up_sync(0xFFFFFFFFu, run, o);
                    if (lane >= o) run = max(run, y);
                }
                const int32_t tb = T;
                run = max(run, tb);
                const int32_t M = __shfl_sync(0xFFFFFFFFu, run, 31);
                if (M > tb) {
                    const unsigned bal = __ballot_sync(0xFFFFFFFFu, act && val == M);
                    best_d = d;
                    best_i = int(base) + __ffs(bal) - 1;
                    T = M;
                }
                if (act) {
                    if (val != kDeadW && val < run - X) val = kDeadW;
                    cur[sg] = val;
                }
                const unsigned lb = __ballot_sync(0xFFFFFFFFu, act && val != kDeadW);
                if (lb) {
                    if (first < 0) first = int(base) + __ffs(lb) - 1;
                    last = int(base) + 31 - __clz(lb);
                }
            }
            __syncwarp();
            rk[ci] = kn;
            if (first < 0) {
                rfl[ci] = 0;
                rll[ci] = -1;
            } else {
                rfl[ci] = first;
                rll[ci] = last;
            }
        }
        if (lane == 0) {
            DevResult res;
            if (status == kStatusBand) {
                res.score = res.h_ext = res.v_ext = 0;
            } else {
                res.score = T;
                res.h_ext = best_d - best_i;
                res.v_ext = best_i;
            }
            res.delta_w = delta_w;
            res.cells = cells;
            res.status = status;
            res.spread = spread;
            P.results[unit] = res;
            ++my_units;
            my_cells += (unsigned long long)cells;
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (my_units) atomicAdd(&P.ctr->units[2], my_units);
        if (my_cells) atomicAdd(&P.ctr->cells[2], my_cells);
    }
}

template __global__ void warp_tier_kernel<ENC_2BIT>(TierParams);
template __global__ void warp_tier_kernel<ENC_5BIT>(TierParams);

// ----------------------------------------------------------------- prep ----
// LR split (partition.cpp:45-81) + checked seed score (align.cpp:283-285)
// + cost key + routing, one thread per task.



__device__ __forceinline__ void emit_unit(const PrepParams& P, int64_t idx, int64_t hp, int64_t vp,
                                          int64_t hl, int64_t vl, int dir) {
    DevUnit u;
    u.h_pos = hp;
    u.v_pos = vp;
    u.h_len = int32_t(hl);
    u.v_len = int32_t(vl);
    u.dir = dir;
    // value range guard for the drift-space thread tiers
    const long long mn = hl < vl ? hl : vl;
    const long long bound = (long long)P.max_pos_score * mn + (long long)P.beta * (hl + vl + 2) +
                            P.x + 2;
    const bool ok = P.thread_ok && bound < (1ll << 23) && hl < (1ll << 30) && vl < (1ll << 30);
    u.route = ok ? 0 : 2;
    P.units[idx] = u;
    // longest first: antidiagonals a unit can run before one view is used up
    const long long gapd = hl > vl ? hl - vl : vl - hl;
    const long long est = 2 * mn + (gapd < 64 ? gapd : 64);
    P.keys[idx] = uint32_t(min(est, (long long)0xFFFFFFF0));
    P.vals[idx] = uint32_t(idx);
    if (!ok) {
        const unsigned long long s = atomicAdd(P.warp_len, 1ull);
        P.warp_list[s] = uint32_t(idx);
    }
}

__global__ void prep_kernel(PrepParams P) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= P.n) return;
    const int64_t* q = P.tasks + 4 * t;
    const int64_t hid = q[0], vid = q[1], hs = q[2], vs = q[3];
    const int64_t hb = P.seq_pos[hid], vb = P.seq_pos[vid];
    const int64_t hn = P.seq_len[hid], vn = P.seq_len[vid];
    int32_t ss = 0;
    for (int i = 0; i < P.k; ++i) {
        uint32_t hc, vc;
        if (P.enc == ENC_2BIT) {
            hc = code_at<ENC_2BIT>(P.pool, hb + hs, 1, 1ll << 40, i);
            vc = code_at<ENC_2BIT>(P.pool, vb + vs, 1, 1ll << 40, i);
        } else {
            hc = code_at<ENC_5BIT>(P.pool, hb + hs, 1, 1ll << 40, i);
            vc = code_at<ENC_5BIT>(P.pool, vb + vs, 1, 1ll << 40, i);
        }
        ss += P.scheme->sim[hc * 32 + vc];  // sim(h symbol, v symbol)
    }
    P.seed_score[t] = ss;
    // left: views end at the seed start, walking backwards (origin = seed)
    emit_unit(P, 2 * t, hb + hs - 1, vb + vs - 1, hs, vs, 0);
    // right: views start right after the seed
    emit_unit(P, 2 * t + 1, hb + hs + P.k, vb + vs + P.k, hn - hs - P.k, vn - vs - P.k, 3);
}

// ------------------------------------------------ INT32 microbenchmark ----
// Independent dependency chains, 8 per thread, unrolled; each iteration of
// the alu variant is 8 x (VIADDMNMX, IMNMX, IADD3) = 24 ALU lane-ops.

__global__ void int_peak_alu(int32_t* out, int iters, int32_t seed, long long* clk) {
    int32_t a[8], b = seed ^ threadIdx.x, c = seed + 7;
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * (q + 3);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            a[q] = __viaddmax_s32(a[q], b, c);
            a[q] = max(a[q], b - q);
            asm volatile("add.s32 %0, %0, %1;" : "+r"(a[q]) : "r"(c));
        }
    }
    long long t1 = clock64();
    int32_t s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s ^= a[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

// the thread tier's own mix: per slot 6 ALU (LOP3, VIMNMX3, VIADDMNMX, ISETP,
// SEL, SHF) + LEA/LEA.HI, measured as achieved lane-ops/clk
__global__ void int_peak_mixed(int32_t* out, int iters, int32_t seed, long long* clk) {
    int32_t a[8], b = seed ^ threadIdx.x, c = seed + 7;
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * (q + 3);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            a[q] = __viaddmax_s32(a[q], b, c);
            asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
            a[q] = max(a[q], b - q);
            asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(c), "r"(b));
        }
    }
    long long t1 = clock64();
    int32_t s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s ^= a[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

}  // namespace xb
