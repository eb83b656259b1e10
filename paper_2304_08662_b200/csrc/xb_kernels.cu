// sm_100a device code: LR split/prep, thread tiers (register band), warp
// tier (exact generic path), and the INT32 issue-rate microbenchmark.
// See xb_kernels.cuh for the coordinate system and DESIGN.md for the proofs.
#include <climits>
#include <cstdint>

#include "xb_kernels.cuh"

namespace xb {

#if XB_CHECKS
__device__ PoolRange xb_pool_ranges[kCheckPools];
__device__ unsigned int xb_check_fail;
// a pool-word load must fall inside the registered image its base points into
__device__ __noinline__ bool pool_load_ok(const uint32_t* pool, int64_t wi) {
    const uint32_t* a = pool + wi;
    for (int r = 0; r < kCheckPools; ++r) {
        const PoolRange e = xb_pool_ranges[r];
        if (e.base && pool >= e.base && pool < e.base + e.words) return a >= e.base && a < e.base + e.words;
    }
    return false;
}
#endif

// ------------------------------------------------------------- helpers ----

// contiguous bit range [lo, hi] of a 32-bit word, lo/hi already clamped to
// [0, 31]; empty when lo > hi
__device__ __forceinline__ uint32_t bit_range(int lo, int hi) {
    if (lo > hi) return 0u;
    const uint32_t up = 0xFFFFFFFFu >> (31 - hi);
    return up & (0xFFFFFFFFu << lo);
}

// -------------------------------------------------------- warp tier ----
// One warp per unit, int32 values with the reference's explicit dead marker
// (no range assumptions), rows of `band` cells in the reference's folded
// layout (slot = (k - i) mod band, align.cpp:20-35), lanes striding over the
// window 32 cells at a time with an inclusive max-scan for the running best.

constexpr int32_t kDeadW = INT_MIN;

template <int ENC>
__device__ __forceinline__ int slot_of(long long k, int i, int band) {
    int u = int((k - i) % band);
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
    XB_ASSERT((unsigned long long)gw < P.ck_warp_slots, kChkScratch);
    int32_t* rows0 = P.warp_scratch + int64_t(gw) * 2 * band;
    int32_t* rows1 = rows0 + band;
    const int32_t gap = P.scheme->gap, X = P.scheme->x;
    const unsigned long long qlen = P.ctr->list_len[kWarpTier];
    const uint32_t* queue = P.lists + (long long)kWarpTier * P.n_units;
    unsigned long long my_units = 0, my_cells = 0;

    for (;;) {
        unsigned long long q = 0;
        if (lane == 0) q = atomicAdd(&P.ctr->cursor[kWarpTier], 1ull);
        q = __shfl_sync(0xFFFFFFFFu, q, 0);
        if (q >= qlen) break;
        XB_ASSERT(q < P.ck_units, kChkList);
        const uint32_t unit = queue[q];
        XB_ASSERT(unit < P.ck_units, kChkUnit);
        const DevUnit U = P.units[unit];
        const int m = U.h_len, n = U.v_len;

        int32_t* R[2] = {rows0, rows1};
        long long rk[2] = {0, 0};
        int rfl[2] = {0, 0}, rll[2] = {0, -1};
        if (lane == 0) rows0[0] = 0;  // slot_of(0, 0) = 0
        __syncwarp();
        int32_t T = 0;
        long long best_d = 0;
        int best_i = 0, delta_w = 1, status = kStatusOk, spread = 0;
        long long cells = 1;

        // 64-bit antidiagonals: views up to kMaxViewLen each
        for (long long d = 1; d <= (long long)n + m + 1; ++d) {
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
            hi = min(hi, min(d, (long long)n));
            const long long kn = d / 2;
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
                    const int j = int(d - i);
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
                res.h_ext = int(best_d - best_i);
                res.v_ext = best_i;
            }
            res.delta_w = delta_w;
            res.cells = cells;
            res.status = status;
            res.spread = spread;
            XB_ASSERT(unit < P.ck_units, kChkResult);
            P.results[unit] = res;
            ++my_units;
            my_cells += (unsigned long long)cells;
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (my_units) atomicAdd(&P.ctr->units[kWarpTier], my_units);
        if (my_cells) atomicAdd(&P.ctr->cells[kWarpTier], my_cells);
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
// Independent dependency chains, 8 per thread, each step one SASS instruction
// that ptxas cannot fuse or move to another pipe:
//   alu:   VIADDMNMX (the integer ALU pipe: IADD3/IMNMX/VIADDMNMX class)
//   mixed: VIADDMNMX + IMAD (ALU pipe + FMA pipe: the SM's INT32 issue ceiling)
// Verified in SASS (build/xb_kernels.o): the loop bodies hold exactly these.

__global__ void int_peak_alu(int32_t* out, int iters, int32_t seed, long long* clk) {
    int32_t a[8];
    const int32_t b = seed ^ int32_t(threadIdx.x), c = seed + 7;
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = int32_t(threadIdx.x) * (q + 3);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = __viaddmax_s32(a[q], b, c);
    }
    long long t1 = clock64();
    int32_t s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s ^= a[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void int_peak_mixed(int32_t* out, int iters, int32_t seed, long long* clk) {
    int32_t a[8];
    const int32_t b = seed ^ int32_t(threadIdx.x), c = seed + 7;
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = int32_t(threadIdx.x) * (q + 3);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 2; ++r)
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                a[q] = __viaddmax_s32(a[q], b, c);
                asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[q]) : "r"(b), "r"(c));
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
