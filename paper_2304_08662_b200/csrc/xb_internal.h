// Internal device/host shared definitions for the xdrop_b200 engine.
#pragma once

#include <cstdint>

namespace xb {

// Pool encodings. ENC_2BIT: pure ACGT, codes A0 C1 G2 T3, 16 symbols per
// 32-bit word. ENC_5BIT: alphabet index (< 32, 31 = the sentinel) in 5 bits,
// symbol p at bits [5p, 5p+5) of the word stream (protein, DNA with N): 5/8
// of a byte pool.  The kernels' readers unpack 4 symbols at a time into byte
// codes, so the table modes see the same byte windows either way.
enum : int { ENC_2BIT = 2, ENC_5BIT = 5 };

// symbols of zero padding in front of / behind every device pool, so window
// fetches that run past a sequence (masked out later) never leave the buffer
constexpr int64_t kPoolPad = 4096;

// Longest view (extension length) a batch accepts: the result fields are int
// (ExtensionResult, align.hpp:37-45) and the kernels keep lengths in int32.
// Longer views are rejected with XB_E_OUT_OF_RANGE.
constexpr int64_t kMaxViewLen = 0x7FFFFFFF;

// Code reserved for "outside the view": scores -128 (+2gap drift) in the
// thread tier's table, so out-of-matrix diagonals always lose.
constexpr int kSentinel = 31;

// One work unit on the device (a WorkUnit, partition.hpp:54-62, already
// resolved to pool positions). View element t lives at pool symbol
// position  pos + t  (dir Right) or  pos - t  (dir Left).
struct DevUnit {
    int64_t h_pos;
    int64_t v_pos;
    int32_t h_len;
    int32_t v_len;
    int32_t dir;     // bit 0: h view Right, bit 1: v view Right (0 = Left)
    int32_t route;   // 0 thread tier, 2 warp tier directly (guard failed)
};

// Same layout as xb_side_result.
struct DevResult {
    int32_t score, h_ext, v_ext, delta_w;
    int64_t cells;
    int32_t status, spread;
};

// Scheme as the kernels see it.
struct DevScheme {
    int32_t gap;
    int32_t x;
    int32_t fast_dna;     // +1/-1/-1 over a 2-bit pool: bit-parallel sim
    int32_t enc;          // pool encoding
    int32_t max_score;    // max table entry (for overflow guards)
    int32_t min_score;
    int32_t sim[32 * 32]; // code-pair scores [h][v] (sentinel row/col = very negative)
};

// Per-tier counters, device side (tiers: K16 K24 K32 K48 K64 | wide K128
// K256 K512 K1024 | warp; cursor slot 15: the pilot).
struct DevCounters {
    unsigned long long cursor[16];     // work-queue cursors per tier (slot 15: pilot)
    unsigned long long list_len[16];   // escalation-input list lengths per tier
    unsigned long long units[16];
    unsigned long long cells[16];
    unsigned long long escalated[16];
    unsigned long long dbg[8];         // XB_COUNTERS builds: steps, rare, masked, recenters, stops;
                                       // [5] always: lane-group resumes at an even d
    int32_t start_tier;                // chosen by the pilot
    int32_t pad;
    unsigned long long resume_next;    // narrow resume records handed out
    unsigned long long resume_wide_next;  // wide resume records handed out
    unsigned long long patch_n;        // result rows finalised after the start tier
    unsigned int prod_done;            // start-tier blocks finished (concurrent escalation tail)
    int32_t prod_finished;             // 1 once every start-tier block has finished
};

// Resume records: a unit that outgrows its tier saves its band state at the
// antidiagonal that did not fit, and the wider tier continues from there
// instead of re-running it.  An escalation-list entry with kResumeFlag set
// indexes a record; a plain entry is a unit to start from scratch (records
// exhausted, or the next tier is the warp tier).  Writers with K <= 48 use
// the narrow pool; K >= 64 writers (into the wide tiers) use the wide pool,
// which follows the narrow one in the same buffer (kResumeWideFlag set).
constexpr int kResumeCap = 32768;
constexpr int kResumeStride = 128;  // int32 per record: 16 header + 2 * K_old row values
constexpr int kResumeWideCap = 4096;
constexpr int kResumeWideStride = 16 + 2 * 512;
constexpr int64_t kResumeInts = int64_t(kResumeCap) * kResumeStride + int64_t(kResumeWideCap) * kResumeWideStride;
constexpr uint32_t kResumeFlag = 0x80000000u;
constexpr uint32_t kResumeWideFlag = 0x40000000u;
constexpr uint32_t kResumeIndex = 0x3FFFFFFFu;
enum : int {
    kRecUnit = 0, kRecD, kRecUbase, kRecTc, kRecBestD, kRecBestU, kRecCells, kRecDeltaW,
    kRecHs1, kRecLs1, kRecHs2, kRecLs2, kRecK, kRecRows = 16
};

#ifdef __CUDACC__
#define XB_HD __host__ __device__
#else
#define XB_HD
#endif
// the record an escalation-list entry with kResumeFlag points at
XB_HD inline int32_t* record_ptr(int32_t* resume, uint32_t e) {
    const int64_t i = int64_t(e & kResumeIndex);
#if defined(XB_CHECKS) && XB_CHECKS && defined(__CUDA_ARCH__)
    if (i >= ((e & kResumeWideFlag) ? kResumeWideCap : kResumeCap)) return nullptr;  // faults loudly
#endif
    return (e & kResumeWideFlag) ? resume + int64_t(kResumeCap) * kResumeStride + i * kResumeWideStride
                                 : resume + i * kResumeStride;
}

constexpr int kStatusOk = 0;
constexpr int kStatusBand = 1;
constexpr int kStatusEscalated = 2;  // transient: re-run by a wider tier

}  // namespace xb
