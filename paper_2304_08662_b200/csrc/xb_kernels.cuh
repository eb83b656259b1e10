// sm_100a kernels for memory-restricted X-drop seed extension.
//
// Semantics follow the reference kernel proj/src/align.cpp:37-155 exactly
// (window rules 64-98, cell rules 102-136, result 148-154); every result
// field, including cells and delta_w, is bit-identical.  See DESIGN.md for
// the derivation of the tricks used here.
//
// Coordinates.  Antidiagonal d holds cells (i, j), i + j = d, i = offset
// into the vertical view v (length n), j = offset into h (length m).  The
// band is addressed by the folded diagonal u = floor(d/2) - i (the same
// invariant the reference uses, align.cpp:12-19): a cell and its diagonal
// predecessor share u; the gap predecessors sit at u and u-1 (d even) or
// u and u+1 (d odd).  A thread-tier unit keeps K consecutive u values
// (slot k <-> u = ubase + k) of the two live antidiagonals in REGISTERS.
//
// Drift space.  A cell value val is stored as  s = val + beta*d + off  with
// beta = -gap and off = X + 1.  Then the recurrence becomes
//     s_d = max(s_{d-2} + (sim - 2 gap),  s_left,  s_up)
// (one VIMNMX3), every live cell has s >= 1 and the dead sentinel is
// negative, so the liveness bit of a slot is its sign bit.
//
// Exact running best.  The reference updates T cell by cell in ascending i
// and prunes each cell against that running T (align.cpp:122-129).  In slot
// order, ascending i is descending k, so one max chain over k = K-1..0 on
// keys (s*64 + k) gives, per slot, the inclusive prefix maximum AND its
// first-attaining slot; "s_k >= Q_k - X" is then the single compare
// key_k >= c_k with c = running max of (key - 64X - 63).
#pragma once

#include <cstddef>
#include <cstdint>

#include "xb_internal.h"

// Checked builds (make checked, -DXB_CHECKS=1: the bounds-asserting
// library the GPU test-suite also runs against, in place of compute-
// sanitizer, which this pool does not offer): every pool-word load, result
// row, escalation-list slot, resume record and table lookup is checked
// against its buffer; the first failed check's id is kept for the host
// (xb_debug_checks).  Product builds compile the checks away.
#ifndef XB_CHECKS
#define XB_CHECKS 0
#endif

namespace xb {

#if XB_CHECKS
// pool images resident on this device (registered by the host when it
// allocates them): a pool-word load must fall inside the image it reads
struct PoolRange {
    const uint32_t* base;
    unsigned long long words;
};
constexpr int kCheckPools = 32;
extern __device__ PoolRange xb_pool_ranges[kCheckPools];
extern __device__ unsigned int xb_check_fail;  // first failed check id (0: none)
__device__ __noinline__ bool pool_load_ok(const uint32_t* pool, int64_t wi);  // xb_kernels.cu
#define XB_ASSERT(cond, id)                                          \
    do {                                                             \
        if (!(cond)) atomicCAS(&xb::xb_check_fail, 0u, (unsigned)(id)); \
    } while (0)
#else
#define XB_ASSERT(cond, id) ((void)0)
#endif
enum : unsigned {  // check ids
    kChkPool = 1, kChkResult, kChkList, kChkRecord, kChkTable, kChkUnit, kChkScratch, kChkSmemRow
};

constexpr int32_t kDeadS = -(1 << 24);  // dead sentinel in drift space

// Shared score table of the table modes: entry (h, v) = sim(v, h) - 2*gap,
// one 32-bit word at word index 33*h + v (codes < 32; column 32 is padding).
// The pitch of 33 words puts entry (h, v) in bank (h + v) mod 32.  Byte
// entries at h*256 + v had put every row in the same 8 of the 32 banks, and
// protein batches ran at 7.8 shared wavefronts per lookup (ncu, C3 x10).
// The byte offset 4v + 132h comes from the [v, h, 0, 0] index bytes with one
// IDP.4A (tab_offset).
using tab_t = int32_t;
constexpr int kTabPitch = 33;
constexpr int kTabWords = 32 * kTabPitch;
__device__ __forceinline__ int32_t tab_lookup(const tab_t* __restrict__ tab, uint32_t vh_bytes) {
    const uint32_t off = __dp4a(vh_bytes, 4u | (4u * kTabPitch) << 8, 0u);
    XB_ASSERT(off < 4u * kTabWords, kChkTable);
    return *reinterpret_cast<const tab_t*>(reinterpret_cast<const char*>(tab) + off);
}
// fills the table (all threads of the block, then the caller syncs)
__device__ __forceinline__ void tab_fill(tab_t* tab, const DevScheme* scheme, int32_t gap) {
    for (int q = threadIdx.x; q < kTabWords; q += blockDim.x) {
        const int h = q / kTabPitch, v = q % kTabPitch;
        int val = -128;  // sentinel rows/columns and the padding column lose
        if (v < 32 && h != kSentinel && v != kSentinel) {
            val = scheme->sim[v * 32 + h] - 2 * gap;
            val = max(-127, min(127, val));
        }
        tab[q] = val;
    }
}
constexpr int kTB = 128;                // threads per block, thread tiers
constexpr int32_t kBig = 1 << 29;       // empty live range = [kBig, -kBig]

// Tiers: band widths K (slots per unit).  0-4: thread / lane-group tiers
// (K16..K64, register bands); 5-9: wide tiers (G lanes per unit, K96..
// K1024, xb_wide.cu); 10: the generic warp tier (any band).
constexpr int kNumTiers = 11;
constexpr int kNarrowTiers = 5;   // tiers 0..4
constexpr int kWideFirst = 5;
constexpr int kWarpTier = 10;
__host__ __device__ constexpr int tier_width(int t) {
    return t == 0 ? 16 : t == 1 ? 24 : t == 2 ? 32 : t == 3 ? 48 : t == 4 ? 64
         : t == 5 ? 96 : t == 6 ? 128 : t == 7 ? 256 : t == 8 ? 512 : t == 9 ? 1024 : 1 << 30;
}
constexpr int kPilotCursor = 15;  // DevCounters::cursor slot of the pilot sample

struct TierParams {
    const uint32_t* __restrict__ pool;
    const DevUnit* __restrict__ units;
    DevResult* __restrict__ results;
    const uint32_t* __restrict__ order;  // cost-sorted unit indices (main queue)
    uint32_t* __restrict__ lists;        // kNumTiers segments of n_units: escalation inputs
    DevCounters* __restrict__ ctr;
    const DevScheme* __restrict__ scheme;
    long long n_units;
    int32_t* __restrict__ pilot_w;       // pilot: widest window seen per sample (-1: > 64)
    long long pilot_n, pilot_stride;     // pilot sample = order[q * stride], q < pilot_n
    int32_t pilot_cap;                   // pilot: antidiagonals run per sample unit
    int32_t band;
    int32_t tier;                        // this launch's tier index
    int32_t pilot;                       // 1: run the pilot sample, 0: cascade
    int32_t esc_to_warp;                 // escalations skip the wider thread tiers
    int32_t role;                        // kRole*: which of the tier's queues this launch serves
    int32_t* __restrict__ warp_scratch;  // warp tier: 2*band ints per warp slot
    int32_t* __restrict__ resume;        // narrow then wide resume records (xb_internal.h)
    // opaque constants: kept in c[]/uniform registers so ptxas cannot fold
    // them into ALU-pipe forms (LEA, LOP3 immediates, SEL)
    uint32_t pad0;                       // see the static_assert below
    int32_t r64;                         // 64
    int32_t one;                         // 1
    int32_t zero;                        // 0
    int32_t two;                         // 2
    uint32_t ones;                       // 0x01010101
    uint32_t mulc[16];                   // 2^(32-2f), f = 1..15
#if XB_CHECKS
    unsigned long long ck_units;         // result rows = list slots per tier
    unsigned long long ck_warp_slots;    // warp-tier scratch slots
#endif
};
// The K24 loop re-reads these constants from the parameter bank; with r64 at
// an offset = 4 (mod 8) ptxas pairs them so that the loop runs 165 ms on full
// config 5, at 0 (mod 8) 176 ms (A/B over five layouts).
static_assert(offsetof(TierParams, r64) % 8 == 4, "keep the opaque constants' pairing");

// ---------------------------------------------------------------- pool ----

__device__ __forceinline__ uint32_t ldw(const uint32_t* __restrict__ pool, int64_t wi) {
    XB_ASSERT(pool_load_ok(pool, wi), kChkPool);
    return __ldg(pool + wi);
}

// exact reversal of sixteen 2-bit fields
__device__ __forceinline__ uint32_t rev16(uint32_t x) {
    x = __brev(x);
    return ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
}

// 16 symbols starting at pool symbol position q, lowest address in bits 0-1
__device__ __forceinline__ uint32_t chunk_mem(const uint32_t* __restrict__ pool, int64_t q) {
    const int64_t wi = q >> 4;
    const uint32_t sh = uint32_t(q & 15) * 2u;
    return __funnelshift_r(ldw(pool, wi), ldw(pool, wi + 1), sh);
}

// view element t at bits 0-1 ("bottom first")
__device__ __forceinline__ uint32_t chunk_bf(const uint32_t* pool, int64_t pos, int dir, int64_t t) {
    return dir ? chunk_mem(pool, pos + t) : rev16(chunk_mem(pool, pos - t - 15));
}
// view element t at bits 30-31 ("top first")
__device__ __forceinline__ uint32_t chunk_tf(const uint32_t* pool, int64_t pos, int dir, int64_t t) {
    return dir ? rev16(chunk_mem(pool, pos + t)) : chunk_mem(pool, pos - t - 15);
}

// one symbol code (any encoding) of a view, sentinel outside [0, len)
template <int ENC>
__device__ __forceinline__ uint32_t code_at(const uint32_t* __restrict__ pool, int64_t pos, int dir,
                                            int64_t len, int64_t t) {
    if (t < 0 || t >= len) return kSentinel;
    const int64_t p = dir ? pos + t : pos - t;
    if (ENC == ENC_2BIT) return (ldw(pool, p >> 4) >> (uint32_t(p & 15) * 2u)) & 3u;
    const int64_t b = 5 * p;  // 5-bit stream
    return __funnelshift_r(ldw(pool, b >> 5), ldw(pool, (b >> 5) + 1), uint32_t(b & 31)) & 31u;
}

// Field geometry of a reader's chunk: PER symbols of BITS bits per 32-bit
// word.  5-bit pools are read as byte codes: a chunk is 4 symbols unpacked
// from 20 stream bits into 4 bytes (the table modes' window layout).
template <int ENC>
struct EncFields {
    static constexpr int BITS = ENC == ENC_2BIT ? 2 : 8;  // bits per symbol in a chunk word
    static constexpr int PER = 32 / BITS;
    static constexpr int LOG = ENC == ENC_2BIT ? 4 : 2;
};

// exact reversal of the fields of a chunk word
template <int ENC>
__device__ __forceinline__ uint32_t rev_fields(uint32_t x) {
    if constexpr (ENC == ENC_2BIT)
        return rev16(x);
    else
        return __byte_perm(x, 0u, 0x0123);
}

// four 5-bit fields (bits 0-19) -> four bytes
__device__ __forceinline__ uint32_t unpack5(uint32_t x) {
    return (x & 0x1Fu) | ((x << 3) & 0x1F00u) | ((x << 6) & 0x1F0000u) | ((x << 9) & 0x1F000000u);
}

// PER symbols starting at pool symbol position q, lowest address in field 0
template <int ENC>
__device__ __forceinline__ uint32_t chunk_mem_e(const uint32_t* __restrict__ pool, int64_t q) {
    if constexpr (ENC == ENC_5BIT) {
        const int64_t b = 5 * q;
        return unpack5(__funnelshift_r(ldw(pool, b >> 5), ldw(pool, (b >> 5) + 1), uint32_t(b & 31)));
    } else {
        using F = EncFields<ENC>;
        const int64_t wi = q >> F::LOG;
        const uint32_t sh = uint32_t(q & (F::PER - 1)) * uint32_t(F::BITS);
        return __funnelshift_r(ldw(pool, wi), ldw(pool, wi + 1), sh);
    }
}

// Streams consecutive PER-symbol chunks of a view.  Refills happen at
// warp-uniform loop iterations (every PER: 16 for 2-bit, 4 for 5-bit pools),
// so no thread diverges for them: `cur` is filled at (re)initialisation with
// the symbols needed up to the next refill point, and each refill assembles
// the chunk whose words were loaded one refill earlier.  TOP = chunks
// top-first (v side: consume from the top field), else bottom-first (h side).
// A 5-bit pool's chunk is 20 stream bits at a bit offset `sh` into (w0, w1);
// each refill moves 20 bits on, and loads the next word (needed one refill
// later) only when the chunk crosses a word boundary.
// PF: hold one more word (`pend`), loaded a whole refill period before it is
// first read, so no refill waits on a load; without it, the word loaded at a
// refill is consumed right there (one register fewer, for the K <= 24 thread
// tiers whose register budget is exhausted).
template <bool TOP, int ENC = ENC_2BIT, bool PF = true>
struct Reader {
    using F = EncFields<ENC>;
    uint32_t cur;   // remaining symbols until the next refill point
    uint32_t w0, w1;
    uint32_t pend;  // PF: the word after them
    int64_t wnext;  // word index of the next load
    uint32_t sh;
    int32_t dir;

    // t0: view index of the next symbol to consume; r: symbols consumed
    // before the next refill point
    __device__ __forceinline__ void init(const uint32_t* pool, int64_t pos, int d, int64_t t0, int r) {
        dir = d;
        if constexpr (ENC == ENC_2BIT) {
            cur = TOP ? chunk_tf(pool, pos, d, t0) : chunk_bf(pool, pos, d, t0);
        } else {
            const uint32_t c = chunk_mem_e<ENC>(pool, d ? pos + t0 : pos - t0 - (F::PER - 1));
            cur = (TOP ? (d != 0) : (d == 0)) ? rev_fields<ENC>(c) : c;
        }
        const int64_t q = d ? pos + t0 + r : pos - (t0 + r) - (F::PER - 1);
        if constexpr (ENC == ENC_5BIT) {
            const int64_t b = 5 * q, wi = b >> 5;
            sh = uint32_t(b & 31);
            w0 = ldw(pool, wi);
            w1 = ldw(pool, wi + 1);
            wnext = d ? wi + 2 : wi - 1;
            return;
        }
        const int64_t wi = q >> F::LOG;
        sh = uint32_t(q & (F::PER - 1)) * uint32_t(F::BITS);
        w0 = ldw(pool, wi);
        w1 = ldw(pool, wi + 1);
        if constexpr (PF) {
            pend = ldw(pool, d ? wi + 2 : wi - 1);
            wnext = d ? wi + 3 : wi - 2;
        } else {
            wnext = d ? wi + 2 : wi - 1;
        }
    }
    __device__ __forceinline__ void refill(const uint32_t* pool) {
        if constexpr (ENC == ENC_5BIT) {
            const uint32_t c = unpack5(__funnelshift_r(w0, w1, sh));
            cur = (TOP ? (dir != 0) : (dir == 0)) ? rev_fields<ENC>(c) : c;
            if (dir != 0) {  // forward: 20 bits on
                sh += 20u;
                if (sh >= 32u) {
                    sh -= 32u;
                    w0 = w1;
                    w1 = ldw(pool, wnext++);
                }
            } else {         // backward: 20 bits back
                if (sh >= 20u) {
                    sh -= 20u;
                } else {
                    sh += 12u;
                    w1 = w0;
                    w0 = ldw(pool, wnext--);
                }
            }
            return;
        }
        const uint32_t c = __funnelshift_r(w0, w1, sh);
        const bool rev = TOP ? (dir != 0) : (dir == 0);
        cur = rev ? rev_fields<ENC>(c) : c;
        const bool fwd = dir != 0;
        const uint32_t o0 = w0, o1 = w1;
        if constexpr (PF) {
            // the word loaded at the previous refill slides in; the load issued
            // now is first read a whole refill period later (no scoreboard wait)
            w0 = fwd ? o1 : pend;
            w1 = fwd ? pend : o0;
            pend = ldw(pool, wnext);
        } else {
            const uint32_t nw = ldw(pool, wnext);
            w0 = fwd ? o1 : nw;
            w1 = fwd ? nw : o0;
        }
        wnext += fwd ? 1 : -1;
    }
    // the next symbol's code (v side: TOP, h side: !TOP)
    __device__ __forceinline__ uint32_t take() {
        uint32_t c;
        if constexpr (TOP) {
            c = cur >> (32 - F::BITS);
            cur <<= F::BITS;
        } else {
            c = cur & ((1u << F::BITS) - 1u);
            cur >>= F::BITS;
        }
        return c;
    }
};

// ------------------------------------------------------ thread tier ----

template <int K, int MODE>
struct TState {
    static constexpr int WK = (K + 15) / 16 * 16;  // symbol-window slots (multiple of 16)
    static constexpr int NW = WK / 16;             // 2-bit window words
    static constexpr int NB = WK / 4;              // byte window words (table mode)
    static constexpr int NM = (K + 31) / 32;       // liveness mask words
    // unit
    int64_t h_pos, v_pos;
    int32_t m, n, hdir, vdir, unit;
    // progress
    int32_t d, ubase, dcap;
    // rows d-1 (1) and d-2 (2): highest live slot hs and lr = 32*NM-1 - lowest
    // live slot; both -1 for an empty row (xb_thread.cu, xstep)
    int32_t lr1, hs1, lr2, hs2;
    int32_t d_vm, d_lim;         // first d needing matrix masks / any rare-path work
    int32_t stop;                // 0 running, else kDone / kBand / kEscalate
    int32_t Tc;                  // 64 (T + beta d + 1): the running best in chain units
    int32_t best_d, best_u, delta_w;  // best cell: antidiagonal, folded diagonal
    int32_t cells;               // <= 64 (n + m + 1): int32 under the prep guard
    // windows
    uint32_t VW[MODE == 0 ? NW : NB];
    uint32_t HW[MODE == 0 ? NW : NB];
    static constexpr int RENC = MODE == 2 ? ENC_5BIT : ENC_2BIT;  // pool encoding read
    static constexpr int RPER = EncFields<RENC>::PER;              // refill period (iterations)
    static constexpr bool RPF = K >= 32 && MODE == 0;  // register headroom for the prefetched word
    Reader<true, RENC, RPF> rv;
    Reader<false, RENC, RPF> rh;
};

// LR split + seed score + cost keys, one thread per task
struct PrepParams {
    const uint32_t* __restrict__ pool;
    const int64_t* __restrict__ tasks;    // n x {h_id, v_id, h_seed, v_seed} (validated)
    const int64_t* __restrict__ seq_pos;  // pool position of each sequence's symbol 0
    const int64_t* __restrict__ seq_len;
    int64_t n;
    int32_t k;
    int32_t enc;
    int32_t thread_ok;                     // scheme admits the thread tiers at all
    int32_t x, beta, max_pos_score;
    const DevScheme* __restrict__ scheme;
    DevUnit* __restrict__ units;
    uint32_t* __restrict__ keys;
    uint32_t* __restrict__ vals;
    int32_t* __restrict__ seed_score;
    uint32_t* __restrict__ warp_list;
    unsigned long long* __restrict__ warp_len;
};

// Queue roles of a tier launch: a tier can be served by the thread kernel
// for its main queue and by the lane-group kernel for its escalations.
// kRoleConsumer: a few lane-group blocks that take the next tier's
// escalations WHILE the start tier still runs (the start tier publishes them
// with kEmptyEntry-initialised slots), leaving kRoleEscalations a short tail.
enum : int { kRoleAll = 0, kRoleStart = 1, kRoleEscalations = 2, kRoleConsumer = 3 };
constexpr uint32_t kEmptyEntry = 0xFFFFFFFFu;  // escalation-list slot not yet written

// Work source of a launch.  Pilot: a strided sample of the order.  Cascade:
// the start tier takes the whole main queue, each wider tier the units
// escalated into it.
struct Queue {
    const uint32_t* q = nullptr;
    unsigned long long len = 0;
    unsigned long long* cursor = nullptr;
    long long stride = 1;
    __device__ __forceinline__ bool next(uint32_t& unit, long long& idx) {
        const unsigned long long i = atomicAdd(cursor, 1ull);
        if (i >= len) return false;
        idx = (long long)i;
        unit = q[(long long)i * stride];
        return true;
    }
};

__device__ __forceinline__ bool make_queue(const TierParams& P, Queue& Q) {
    if (P.pilot) {
        Q.q = P.order;
        Q.len = (unsigned long long)P.pilot_n;
        Q.stride = P.pilot_stride;
        Q.cursor = &P.ctr->cursor[kPilotCursor];
        return true;
    }
    const int t0 = P.ctr->start_tier;
    if (P.tier < t0) return false;
    if (P.role == kRoleStart && P.tier != t0) return false;
    if ((P.role == kRoleEscalations || P.role == kRoleConsumer) && P.tier == t0) return false;
    Q.cursor = &P.ctr->cursor[P.tier];
    if (P.role == kRoleConsumer) {  // length read as it grows (consumer_claim)
        Q.q = P.lists + (long long)P.tier * P.n_units;
        Q.len = 0;
    } else if (P.tier == t0) {
        Q.q = P.order;
        Q.len = (unsigned long long)P.n_units;
    } else {
        Q.q = P.lists + (long long)P.tier * P.n_units;
        Q.len = P.ctr->list_len[P.tier];
    }
    return true;
}

// Hands out a resume record for a K-slot writer: the escalation-list entry
// (kResumeFlag, + kResumeWideFlag for the wide pool, | index) and the record,
// or 0 when that pool is used up (the unit then restarts from scratch).
template <int K>
__device__ __forceinline__ uint32_t alloc_record(const TierParams& P, int32_t*& rec) {
    static_assert(16 + 2 * K <= kResumeWideStride, "record too small for this writer");
    if constexpr (16 + 2 * K <= kResumeStride) {
        const unsigned long long r = atomicAdd(&P.ctr->resume_next, 1ull);
        if (r >= (unsigned long long)kResumeCap) return 0u;
        rec = P.resume + (long long)r * kResumeStride;
        return kResumeFlag | uint32_t(r);
    } else {
        const unsigned long long r = atomicAdd(&P.ctr->resume_wide_next, 1ull);
        if (r >= (unsigned long long)kResumeWideCap) return 0u;
        rec = P.resume + (long long)kResumeCap * kResumeStride + (long long)r * kResumeWideStride;
        return kResumeFlag | kResumeWideFlag | uint32_t(r);
    }
}

// outcome of one antidiagonal step
enum : int { kGo = 0, kDone = 1, kBand = 2, kEscalate = 3 };

}  // namespace xb
