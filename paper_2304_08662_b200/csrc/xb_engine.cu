// Host side of the xdrop_b200 C-ABI: scoring schemes, the detached sequence
// pool (2-bit / byte packing, one upload per device), LR split + cost sort
// on the device, the tier cascade, and LPT sharding across devices.
// Reference interfaces replaced are cited per entry point in
// include/xdrop_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <queue>
#include <string>
#include <thread>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/xdrop_b200.h"
#include "xb_internal.h"
#include "xb_kernels.cuh"

namespace xb {
template <int K, int MODE>
__global__ void thread_tier_kernel(TierParams P);
template <int K, int G, int MODE>
__global__ void group_tier_kernel(TierParams P);
template <int K, int G, int MODE>
__global__ void wide_tier_kernel(TierParams P);
template <int K, int G, int MODE>
__global__ void lane_tier_kernel(TierParams P);
template <int ENC>
__global__ void warp_tier_kernel(TierParams P);
__global__ void select_tier_kernel(TierParams P, int forced, int32_t* host_out);
__global__ void prep_kernel(PrepParams P);
__global__ void int_peak_alu(int32_t* out, int iters, int32_t seed, long long* clk);
__global__ void int_peak_mixed(int32_t* out, int iters, int32_t seed, long long* clk);


}  // namespace xb

using namespace xb;

namespace {

thread_local xb_stats g_last_stats{};

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess) {                                                      \
            std::fprintf(stderr, "xdrop_b200: %s failed: %s (%s:%d)\n", #call,        \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                 \
            return XB_E_CUDA;                                                         \
        }                                                                             \
    } while (0)

int n_host_threads() {
    unsigned h = std::thread::hardware_concurrency();
    return int(std::max(1u, std::min(h, 64u)));
}

template <class F>
void parallel_for(int64_t n, F&& f) {
    const int T = n > (1 << 16) ? n_host_threads() : 1;
    if (T <= 1) {
        f(int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + T - 1) / T;
    for (int t = 0; t < T; ++t) {
        const int64_t a = t * chunk, b = std::min(n, a + chunk);
        if (a < b) th.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

// ----------------------------------------------------------------- scheme ----

struct xb_scheme {
    int kind = 0;  // 0 match/mismatch, 1 matrix
    int match = 0, mismatch = 0, gap = -1, x = 0;
    std::string alphabet;
    std::vector<int> cells;  // n*n
    int16_t table[256 * 256];
    bool valid[256];
    int8_t code_of[256];
};

extern "C" {

const char* xb_version(void) { return "xdrop_b200 0.1 (sm_100a)"; }

const char* xb_strerror(int code) {
    switch (code) {
        case XB_OK: return "ok";
        case XB_E_BAD_PARAM: return "invalid parameter";
        case XB_E_DANGLING: return "task references an unknown sequence";
        case XB_E_SEED_OOB: return "seed does not fit inside its sequences";
        case XB_E_UNKNOWN_SYMBOL: return "symbol not in scoring alphabet";
        case XB_E_OUT_OF_RANGE: return "view out of range";
        case XB_E_CUDA: return "CUDA error";
        case XB_E_NO_DEVICE: return "no CUDA device";
        case XB_E_PARSE: return "malformed substitution matrix";
        default: return "unknown error";
    }
}

int xb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

static void scheme_finish(xb_scheme* s) {
    std::memset(s->table, 0, sizeof s->table);
    std::memset(s->valid, 0, sizeof s->valid);
    std::memset(s->code_of, -1, sizeof s->code_of);
    const int n = int(s->alphabet.size());
    for (int i = 0; i < n; ++i) {
        const unsigned char a = (unsigned char)s->alphabet[size_t(i)];
        s->valid[a] = true;
        s->code_of[a] = int8_t(i);  // last occurrence wins, like the table
        for (int j = 0; j < n; ++j) {
            const unsigned char b = (unsigned char)s->alphabet[size_t(j)];
            s->table[a * 256 + b] = int16_t(s->cells[size_t(i * n + j)]);
        }
    }
}

xb_scheme* xb_scheme_match_mismatch(int match, int mismatch, int gap, int x, int* err) {
    if (match <= 0 || mismatch >= 0 || gap >= 0 || x < 0) {
        if (err) *err = XB_E_BAD_PARAM;
        return nullptr;
    }
    auto* s = new xb_scheme();
    s->kind = 0;
    s->match = match;
    s->mismatch = mismatch;
    s->gap = gap;
    s->x = x;
    s->alphabet = "ACGTN";
    s->cells.assign(25, mismatch);
    for (int i = 0; i < 4; ++i) s->cells[size_t(i * 5 + i)] = match;  // N never matches
    scheme_finish(s);
    if (err) *err = XB_OK;
    return s;
}

xb_scheme* xb_scheme_from_matrix(const char* alphabet, int n, const int* cells, int gap, int x,
                                 int* err) {
    if (gap >= 0 || x < 0 || n <= 0 || n > 31 || !alphabet || !cells) {
        if (err) *err = XB_E_BAD_PARAM;
        return nullptr;
    }
    auto* s = new xb_scheme();
    s->kind = 1;
    s->gap = gap;
    s->x = x;
    s->alphabet.assign(alphabet, size_t(n));
    s->cells.assign(cells, cells + size_t(n) * size_t(n));
    scheme_finish(s);
    if (err) *err = XB_OK;
    return s;
}

int xb_parse_submatrix(const char* text, char* alphabet_out, int alphabet_cap, int* cells_out,
                       int cells_cap) {
    if (!text) return -XB_E_BAD_PARAM;
    std::string alpha, labels;
    std::vector<std::vector<int>> rows;
    const char* p = text;
    while (*p) {
        const char* e = std::strchr(p, '\n');
        std::string line = e ? std::string(p, size_t(e - p)) : std::string(p);
        p = e ? e + 1 : p + line.size();
        if (!line.empty() && line.back() == '\r') line.pop_back();
        const size_t pos = line.find_first_not_of(" \t");
        if (pos == std::string::npos || line[pos] == '#') continue;
        // whitespace tokens
        std::vector<std::string> tok;
        size_t q = 0;
        while (q < line.size()) {
            while (q < line.size() && (line[q] == ' ' || line[q] == '\t')) ++q;
            size_t r = q;
            while (r < line.size() && line[r] != ' ' && line[r] != '\t') ++r;
            if (r > q) tok.push_back(line.substr(q, r - q));
            q = r;
        }
        if (alpha.empty()) {
            for (auto& t : tok) {
                if (t.size() != 1) return -XB_E_PARSE;
                alpha += t;
            }
            continue;
        }
        if (tok.empty() || tok[0].size() != 1) return -XB_E_PARSE;
        std::vector<int> row;
        for (size_t i = 1; i < tok.size(); ++i) {
            char* end = nullptr;
            const long v = std::strtol(tok[i].c_str(), &end, 10);
            if (end == tok[i].c_str() || *end) break;  // istream >> int stops here
            row.push_back(int(v));
        }
        if (row.size() != alpha.size()) return -XB_E_PARSE;
        labels += tok[0];
        rows.push_back(std::move(row));
    }
    if (alpha.empty() || rows.size() != alpha.size() || labels != alpha) return -XB_E_PARSE;
    const int n = int(alpha.size());
    if (n + 1 > alphabet_cap || n * n > cells_cap) return -XB_E_BAD_PARAM;
    std::memcpy(alphabet_out, alpha.data(), size_t(n));
    alphabet_out[n] = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) cells_out[i * n + j] = rows[size_t(i)][size_t(j)];
    return n;
}

int xb_scheme_sim(const xb_scheme* s, char a, char b, int* out) {
    if (!s->valid[(unsigned char)a] || !s->valid[(unsigned char)b]) return XB_E_UNKNOWN_SYMBOL;
    *out = s->table[(unsigned char)a * 256 + (unsigned char)b];
    return XB_OK;
}

void xb_scheme_free(xb_scheme* s) { delete s; }

}  // extern "C"

// ------------------------------------------------------------------- pool ----

// One device's copy of the pool.  Sequences become resident on first use:
// a batch uploads the words of the sequences it references that this device
// does not hold yet (or the whole image when that is most of it), so every
// sequence crosses PCIe once per device however many seeds share it, and a
// device serving one shard of the tasks holds only that shard's part.
struct DevPool {
    uint32_t* words = nullptr;
    int64_t* seq_pos = nullptr;
    int64_t* seq_len = nullptr;
    DevScheme* scheme = nullptr;
    int64_t cap_words = 0, cap_seqs = 0;  // allocated sizes (the pool may grow after an upload)
    bool ready = false;                   // the whole image is resident
    bool meta_ready = false;              // seq_pos / seq_len / scheme are current
    std::vector<uint8_t> resident;        // per sequence (when !ready)
    uint32_t* d_stage = nullptr;          // gathered words of a partial upload
    int64_t* d_ranges = nullptr;          // (dst word, src word, words) triples
    int64_t cap_stage = 0, cap_ranges = 0;
};

struct Workspace;

// The detached pool (SequenceStore, sequence.hpp:13-19) keeps no byte copy of
// its sequences: xb_pool_add* validates the symbols and packs them straight
// into one pinned host image of 32-bit words (2-bit DNA, or one byte code per
// symbol), which is what crosses PCIe once per device.  The image grows in
// place; a DNA pool that receives its first 'N' is widened from 2-bit to byte
// codes once (ACGTN codes are 0-4 in both, so the widening is a re-layout).
struct xb_pool {
    xb_scheme scheme;
    std::vector<int64_t> offsets{0};  // symbol offsets of the sequences (no padding)
    int enc = ENC_2BIT;
    uint32_t* host_words = nullptr;   // pinned when host_pinned
    bool host_pinned = false;
    int64_t cap_words = 0;            // allocated words of host_words
    int64_t n_words = 0;              // words covering pad + symbols + pad (+2)
    std::vector<int64_t> seq_pos, seq_len;
    DevScheme dev_scheme{};
    std::map<int, DevPool> dev;
    std::mutex mu;
};

static bool fast_dna(const xb_pool* p) {
    return p->enc == ENC_2BIT && p->scheme.kind == 0 && p->scheme.match == 1 &&
           p->scheme.mismatch == -1 && p->scheme.gap == -1;
}

// Admits the drift-space thread tiers for this scheme (DESIGN.md guards).
static bool thread_tiers_ok(const xb_pool* p) {
    const xb_scheme& s = p->scheme;
    if (s.gap <= -(1 << 10) || s.x >= (1 << 22)) return false;
    if (fast_dna(p)) return true;
    for (int v : s.cells) {
        const long t = long(v) - 2L * s.gap;
        if (t < -127 || t > 127) return false;
    }
    return true;
}

static int enc_bits(int enc) { return enc == ENC_2BIT ? 2 : 5; }
// first / one-past-last word holding image symbol positions [s0, s1)
static int64_t word_lo(int enc, int64_t s0) { return (s0 * enc_bits(enc)) >> 5; }
static int64_t word_hi(int enc, int64_t s1) { return ((s1 * enc_bits(enc)) + 31) >> 5; }
static int64_t words_for(int enc, int64_t total) {
    return word_hi(enc, kPoolPad + total + kPoolPad) + 2;
}

static void host_free(uint32_t* w, bool pinned) {
    if (!w) return;
    if (pinned)
        cudaFreeHost(w);
    else
        std::free(w);
}

// A zeroed image of at least `need` words (pinned when the runtime allows),
// holding the first `keep` words of the old one.
static bool host_reserve(xb_pool* p, int64_t need, int64_t keep) {
    if (need <= p->cap_words) return true;
    const int64_t cap = std::max<int64_t>(need, p->cap_words + p->cap_words / 2);
    uint32_t* w = nullptr;
    bool pinned = cudaMallocHost(&w, size_t(cap) * 4) == cudaSuccess;
    if (!pinned) {
        cudaGetLastError();
        w = static_cast<uint32_t*>(std::malloc(size_t(cap) * 4));
        if (!w) return false;
    }
    parallel_for(cap, [&](int64_t a, int64_t b) {
        const int64_t c = std::min(b, keep);
        if (a < c) std::memcpy(w + a, p->host_words + a, size_t(c - a) * 4);
        if (std::max(a, c) < b) std::memset(w + std::max(a, c), 0, size_t(b - std::max(a, c)) * 4);
    });
    host_free(p->host_words, p->host_pinned);
    p->host_words = w;
    p->host_pinned = pinned;
    p->cap_words = cap;
    return true;
}

// Kernel-side scheme: code-pair table, encoding, guards.
static void pool_scheme(xb_pool* p) {
    const xb_scheme& s = p->scheme;
    DevScheme& d = p->dev_scheme;
    std::memset(&d, 0, sizeof d);
    d.gap = s.gap;
    d.x = s.x;
    d.enc = p->enc;
    d.fast_dna = fast_dna(p) ? 1 : 0;
    d.max_score = INT32_MIN;
    d.min_score = INT32_MAX;
    const int na = int(s.alphabet.size());
    for (int i = 0; i < 32 * 32; ++i) d.sim[i] = -(1 << 20);
    if (p->enc == ENC_2BIT) {
        const char* acgt = "ACGT";
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b)
                d.sim[a * 32 + b] = s.table[(unsigned char)acgt[a] * 256 + (unsigned char)acgt[b]];
    } else {
        for (int a = 0; a < na; ++a)
            for (int b = 0; b < na; ++b)
                d.sim[a * 32 + b] = s.table[(unsigned char)s.alphabet[size_t(a)] * 256 +
                                            (unsigned char)s.alphabet[size_t(b)]];
    }
    for (int v : s.cells) {
        d.max_score = std::max(d.max_score, v);
        d.min_score = std::min(d.min_score, v);
    }
}

// 2-bit image -> byte codes (A0 C1 G2 T3 are the ACGTN scheme's codes too).
static bool widen_to_bytes(xb_pool* p) {
    const int64_t total = p->offsets.back();
    const int64_t nw = words_for(ENC_5BIT, total);
    uint32_t* w = nullptr;
    bool pinned = cudaMallocHost(&w, size_t(nw) * 4) == cudaSuccess;
    if (!pinned) {
        cudaGetLastError();
        w = static_cast<uint32_t*>(std::malloc(size_t(nw) * 4));
        if (!w) return false;
    }
    const uint32_t* old = p->host_words;
    const int64_t nsym = kPoolPad + total + kPoolPad;
    parallel_for(nw, [&](int64_t a, int64_t b) {
        for (int64_t q = a; q < b; ++q) {  // word q holds stream bits [32q, 32q + 32)
            uint64_t acc = 0;
            for (int64_t s = (32 * q) / 5; s <= (32 * q + 31) / 5 && s < nsym; ++s) {
                const uint64_t c = (old[s >> 4] >> (2 * (s & 15))) & 3u;
                const int64_t sh = 5 * s - 32 * q;  // -4 .. 31
                acc |= sh >= 0 ? c << sh : c >> (-sh);
            }
            w[q] = uint32_t(acc);
        }
    });
    host_free(p->host_words, p->host_pinned);
    p->host_words = w;
    p->host_pinned = pinned;
    p->cap_words = nw;
    p->n_words = nw;
    p->enc = ENC_5BIT;
    return true;
}

// Checked builds: the device pool images a pool-word load may read.
#if XB_CHECKS
static std::mutex g_check_mu;
static std::map<int, std::vector<std::pair<const uint32_t*, unsigned long long>>> g_check_pools;
static void check_pools_publish(int dev) {
    PoolRange r[kCheckPools] = {};
    int q = 0;
    for (auto& e : g_check_pools[dev])
        if (q < kCheckPools) r[q++] = PoolRange{e.first, e.second};
    cudaMemcpyToSymbol(xb_pool_ranges, r, sizeof r);
}
static void check_pool_register(int dev, const uint32_t* base, int64_t words) {
    std::lock_guard<std::mutex> g(g_check_mu);
    g_check_pools[dev].push_back({base, (unsigned long long)words});
    check_pools_publish(dev);
}
static void check_pool_unregister(int dev, const uint32_t* base) {
    std::lock_guard<std::mutex> g(g_check_mu);
    auto& v = g_check_pools[dev];
    for (size_t i = 0; i < v.size(); ++i)
        if (v[i].first == base) {
            v.erase(v.begin() + long(i));
            break;
        }
    check_pools_publish(dev);
}
#else
static void check_pool_register(int, const uint32_t*, int64_t) {}
static void check_pool_unregister(int, const uint32_t*) {}
#endif

__global__ void scatter_words_kernel(const uint32_t* __restrict__ src, const int64_t* __restrict__ ranges,
                                     int64_t n_ranges, uint32_t* __restrict__ dst) {
    for (int64_t r = blockIdx.x; r < n_ranges; r += gridDim.x) {
        const int64_t d0 = ranges[3 * r], s0 = ranges[3 * r + 1], len = ranges[3 * r + 2];
        for (int64_t q = threadIdx.x; q < len; q += blockDim.x) dst[d0 + q] = src[s0 + q];
    }
}

// Makes the pool resident on `dev` for a batch referencing the sequences in
// `need` (nullptr: all of them).  The caller's stream orders the copies.
static int pool_device(xb_pool* p, int dev, cudaStream_t st, int64_t* h2d, DevPool** out,
                       const std::vector<uint8_t>* need = nullptr) {
    std::lock_guard<std::mutex> g(p->mu);
    DevPool& D = p->dev[dev];
    CK(cudaSetDevice(dev));
    const int64_t n = int64_t(p->seq_pos.size());
    if (!D.ready) {
        // A pool that grew after an upload (more sequences, or an 'N' that
        // switched it from 2-bit to byte codes) outgrows its device buffers:
        // reallocate.  cudaFree waits for the device to go idle, so no batch
        // still reading the old buffers is cut short.
        if (D.words && (p->n_words > D.cap_words || n > D.cap_seqs)) {
            check_pool_unregister(dev, D.words);
            CK(cudaFree(D.words));
            CK(cudaFree(D.seq_pos));
            CK(cudaFree(D.seq_len));
            D.words = nullptr;
            D.seq_pos = D.seq_len = nullptr;
            D.resident.clear();
        }
        if (!D.words) {
            CK(cudaMalloc(&D.words, size_t(p->n_words) * 4));
            CK(cudaMalloc(&D.seq_pos, size_t(std::max<int64_t>(n, 1)) * 8));
            CK(cudaMalloc(&D.seq_len, size_t(std::max<int64_t>(n, 1)) * 8));
            check_pool_register(dev, D.words, p->n_words);
            D.cap_words = p->n_words;
            D.cap_seqs = std::max<int64_t>(n, 1);
        }
        if (!D.scheme) CK(cudaMalloc(&D.scheme, sizeof(DevScheme)));
        if (!D.meta_ready) {
            if (n) {
                CK(cudaMemcpyAsync(D.seq_pos, p->seq_pos.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(D.seq_len, p->seq_len.data(), size_t(n) * 8, cudaMemcpyHostToDevice, st));
            }
            CK(cudaMemcpyAsync(D.scheme, &p->dev_scheme, sizeof(DevScheme), cudaMemcpyHostToDevice, st));
            if (h2d) *h2d += n * 16 + int64_t(sizeof(DevScheme));
            D.meta_ready = true;
        }
        D.resident.resize(size_t(n), 0);
        // words still missing: one range per run of consecutive missing,
        // needed sequences (merged across shared boundary words)
        std::vector<int64_t> ranges;  // (first word, words)
        int64_t missing = 0;
        if (need) {
            for (int64_t i = 0; i < n; ++i) {
                if (!(*need)[size_t(i)] || D.resident[size_t(i)]) continue;
                const int64_t w0 = word_lo(p->enc, p->seq_pos[size_t(i)]);
                const int64_t w1 = word_hi(p->enc, p->seq_pos[size_t(i)] + std::max<int64_t>(p->seq_len[size_t(i)], 1));
                if (!ranges.empty() && w0 <= ranges[ranges.size() - 2] + ranges.back()) {
                    ranges.back() = std::max(ranges.back(), w1 - ranges[ranges.size() - 2]);
                } else {
                    ranges.push_back(w0);
                    ranges.push_back(w1 - w0);
                }
            }
            for (size_t r = 1; r < ranges.size(); r += 2) missing += ranges[r];
        }
        if (!need || 2 * missing > p->n_words) {
            // the whole image (most of it is needed anyway: one contiguous copy)
            CK(cudaMemcpyAsync(D.words, p->host_words, size_t(p->n_words) * 4, cudaMemcpyHostToDevice, st));
            if (h2d) *h2d += p->n_words * 4;
            D.ready = true;
            D.resident.assign(size_t(n), 1);
        } else if (missing) {
            const int64_t nr = int64_t(ranges.size()) / 2;
            if (nr <= 64) {  // few runs (a locality shard of a pool in genome order): copy them directly
                for (int64_t r = 0; r < nr; ++r)
                    CK(cudaMemcpyAsync(D.words + ranges[size_t(2 * r)], p->host_words + ranges[size_t(2 * r)],
                                       size_t(ranges[size_t(2 * r + 1)]) * 4, cudaMemcpyHostToDevice, st));
            } else {  // many runs: gather into one staged copy, scatter on the device
                if (missing > D.cap_stage) {
                    cudaFree(D.d_stage);
                    CK(cudaMalloc(&D.d_stage, size_t(missing) * 4));
                    D.cap_stage = missing;
                }
                if (nr > D.cap_ranges) {
                    cudaFree(D.d_ranges);
                    CK(cudaMalloc(&D.d_ranges, size_t(nr) * 24));
                    D.cap_ranges = nr;
                }
                uint32_t* hs = nullptr;
                int64_t* hr = nullptr;
                CK(cudaMallocHost(&hs, size_t(missing) * 4));
                CK(cudaMallocHost(&hr, size_t(nr) * 24));
                int64_t at = 0;
                for (int64_t r = 0; r < nr; ++r) {
                    const int64_t w0 = ranges[size_t(2 * r)], len = ranges[size_t(2 * r + 1)];
                    std::memcpy(hs + at, p->host_words + w0, size_t(len) * 4);
                    hr[3 * r] = w0;
                    hr[3 * r + 1] = at;
                    hr[3 * r + 2] = len;
                    at += len;
                }
                CK(cudaMemcpyAsync(D.d_stage, hs, size_t(missing) * 4, cudaMemcpyHostToDevice, st));
                CK(cudaMemcpyAsync(D.d_ranges, hr, size_t(nr) * 24, cudaMemcpyHostToDevice, st));
                scatter_words_kernel<<<unsigned(std::min<int64_t>(nr, 4096)), 256, 0, st>>>(D.d_stage, D.d_ranges,
                                                                                        nr, D.words);
                CK(cudaGetLastError());
                CK(cudaStreamSynchronize(st));  // the staging buffers are released here
                cudaFreeHost(hs);
                cudaFreeHost(hr);
            }
            if (h2d) *h2d += missing * 4;
            for (int64_t i = 0; i < n; ++i)
                if ((*need)[size_t(i)]) D.resident[size_t(i)] = 1;
        }
    }
    *out = &D;
    return XB_OK;
}

static void pool_drop_devices(xb_pool* p) {
    for (auto& kv : p->dev) {
        cudaSetDevice(kv.first);
        if (kv.second.words) check_pool_unregister(kv.first, kv.second.words);
        cudaFree(kv.second.words);
        cudaFree(kv.second.seq_pos);
        cudaFree(kv.second.seq_len);
        cudaFree(kv.second.scheme);
        cudaFree(kv.second.d_stage);
        cudaFree(kv.second.d_ranges);
    }
    p->dev.clear();
}


extern "C" {

xb_pool* xb_pool_create(const xb_scheme* s, int* err) {
    if (!s) {
        if (err) *err = XB_E_BAD_PARAM;
        return nullptr;
    }
    auto* p = new xb_pool();
    p->scheme = *s;
    p->enc = s->kind == 0 ? ENC_2BIT : ENC_5BIT;
    if (!host_reserve(p, words_for(p->enc, 0), 0)) {
        delete p;
        if (err) *err = XB_E_BAD_PARAM;
        return nullptr;
    }
    p->n_words = words_for(p->enc, 0);
    pool_scheme(p);
    if (err) *err = XB_OK;
    return p;
}

int64_t xb_pool_add_bulk(xb_pool* p, const char* concat, const int64_t* offsets, int64_t n) {
    if (!p || n < 0 || (n && (!concat || !offsets))) return -XB_E_BAD_PARAM;
    const int64_t total = n ? offsets[n] - offsets[0] : 0;
    // validate (io.cpp:82-89 ingestion rule) before touching the pool
    std::atomic<int> bad{0};
    std::atomic<bool> non_acgt{false};
    const char* base = concat + (n ? offsets[0] : 0);
    parallel_for(total, [&](int64_t a, int64_t b) {
        bool na = false;
        for (int64_t i = a; i < b; ++i) {
            const unsigned char c = (unsigned char)base[i];
            if (!p->scheme.valid[c]) {
                bad = 1;
                return;
            }
            na |= (c != 'A' && c != 'C' && c != 'G' && c != 'T');
        }
        if (na) non_acgt = true;
    });
    if (bad) return -XB_E_UNKNOWN_SYMBOL;
    std::lock_guard<std::mutex> g(p->mu);
    const bool widened = non_acgt && p->enc == ENC_2BIT;
    if (widened && !widen_to_bytes(p)) return -XB_E_BAD_PARAM;
    const int64_t first = int64_t(p->offsets.size()) - 1;
    const int64_t at = p->offsets.back();
    const int64_t nw = words_for(p->enc, at + total);
    if (!host_reserve(p, nw, p->n_words)) return -XB_E_BAD_PARAM;
    // pack the new symbols into the words they fall in; the image past the
    // old symbols is zero, so a word shared with them is OR-ed into
    uint8_t code[256];
    for (int c = 0; c < 256; ++c) code[c] = p->scheme.code_of[c] < 0 ? 0 : uint8_t(p->scheme.code_of[c]);
    const int bits = enc_bits(p->enc);
    const int64_t s0 = kPoolPad + at, s1 = s0 + total;  // image symbol positions of the new run
    const int64_t q0 = word_lo(p->enc, s0), q1 = word_hi(p->enc, s1);
    uint32_t* W = p->host_words;
    parallel_for(q1 - q0, [&](int64_t a, int64_t b) {
        for (int64_t q = q0 + a; q < q0 + b; ++q) {  // word q: stream bits [32q, 32q + 32)
            const int64_t lo = std::max((32 * q) / bits, s0), hi = std::min((32 * q + 31) / bits + 1, s1);
            uint64_t acc = 0;
            for (int64_t s = lo; s < hi; ++s) {
                const uint64_t c = code[(unsigned char)base[s - s0]];
                const int64_t sh = bits * s - 32 * q;  // > -bits: a field may start in the previous word
                acc |= sh >= 0 ? c << sh : c >> (-sh);
            }
            W[q] |= uint32_t(acc);
        }
    });
    p->n_words = nw;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t o0 = at + offsets[i] - offsets[0], o1 = at + offsets[i + 1] - offsets[0];
        p->offsets.push_back(o1);
        p->seq_pos.push_back(kPoolPad + o0);
        p->seq_len.push_back(o1 - o0);
    }
    pool_scheme(p);
    for (auto& kv : p->dev) {  // new sequences are not resident; a widened image none at all
        kv.second.ready = false;
        kv.second.meta_ready = false;
        if (widened) kv.second.resident.clear();
    }
    return first;
}

int64_t xb_pool_add(xb_pool* p, const char* symbols, int64_t len) {
    const int64_t off[2] = {0, len};
    return xb_pool_add_bulk(p, symbols, off, 1);
}

int64_t xb_pool_size(const xb_pool* p) { return int64_t(p->offsets.size()) - 1; }

int64_t xb_pool_seq_len(const xb_pool* p, int64_t id) {
    if (id < 0 || id >= xb_pool_size(p)) return -XB_E_DANGLING;
    return p->offsets[size_t(id) + 1] - p->offsets[size_t(id)];
}

int xb_pool_bits_per_symbol(const xb_pool* p) { return enc_bits(p->enc); }

void xb_pool_evict(xb_pool* p) {
    std::lock_guard<std::mutex> g(p->mu);
    for (auto& kv : p->dev) {
        kv.second.ready = false;
        kv.second.meta_ready = false;
        kv.second.resident.clear();
    }
}

void xb_pool_free(xb_pool* p) {
    if (!p) return;
    pool_drop_devices(p);
    host_free(p->host_words, p->host_pinned);
    delete p;
}

}  // extern "C"

// ------------------------------------------------------------------ batch ----

// Device buffers + pinned staging of one batch on one device.  Cached per
// (pool, device) and reused by later batches, so repeated calls do not pay
// cudaMalloc / page-locking on every step.
// Throughput-planned batches fill every SM with persistent start-tier blocks,
// so on one device their cascades run one after another: a batch's start
// tier waits for the previous such batch's last kernel (its escalation tail
// would otherwise starve behind the newer batch's resident blocks until that
// whole start tier ends).  Their uploads and planning (prep, sort, pilot)
// still overlap the previous batch.  Latency-planned batches are not ordered.
struct CascadeOrder {
    std::mutex mu;
    std::map<int, cudaEvent_t> last;  // device -> event after the last ordered cascade
};
static CascadeOrder& cascade_order() {
    static CascadeOrder* o = new CascadeOrder();
    return *o;
}

// h_misc (pinned, 4 KiB per workspace): the counters are
// copied to its start; the pilot's start tier is written by the kernel here.
constexpr int kMiscStartTier = 1000;

// Events of a run on its stream: start, after prep + sort, after the pilot,
// after tier t (kEvTier + t), after the warp tier, after the result copy
// (fetch), the cascade-order marker, and the early result copy.
enum : int { kEvStart = 0, kEvPrep = 1, kEvPilot = 2, kEvTier = 3, kEvWarp = kEvTier + kWarpTier,
             kEvFetch, kEvOrder, kEvCopy, kNumEv };
static_assert(kNumEv <= 20, "Workspace::ev");

struct Workspace {
    int dev = 0;
    bool in_use = false;
    int64_t capU = 0, capI = 0;
    size_t scratch_bytes = 0, cub_bytes = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[20] = {};  // kEv* below
    int64_t* d_tasks = nullptr;
    DevUnit* d_units = nullptr;
    uint32_t *d_keys = nullptr, *d_vals = nullptr, *d_keys2 = nullptr, *d_order = nullptr;
    DevResult* d_res = nullptr;
    int32_t* d_seed = nullptr;
    uint32_t* d_lists = nullptr;
    DevCounters* d_ctr = nullptr;
    int32_t* d_scratch = nullptr;
    int32_t* d_resume = nullptr;  // narrow + wide escalation records (kResumeInts)
    int32_t* d_pilot = nullptr;
    void* d_cub = nullptr;
    DevResult* h_res = nullptr;
    int32_t* h_seed = nullptr;
    int64_t* h_tasks = nullptr;
    // rows finished after the start tier (escalations, warp tier), gathered
    // so that the bulk of the results can cross PCIe during the cascade tail
    cudaStream_t copy_stream = nullptr;
    cudaStream_t aux_stream = nullptr;  // high priority: the concurrent escalation consumer
    cudaEvent_t aux_ev[2] = {};
    int32_t* h_misc = nullptr;  // pinned (4 KiB): start tier after the pilot, counters

    void release_units() {
        cudaFree(d_units);
        cudaFree(d_keys);
        cudaFree(d_vals);
        cudaFree(d_keys2);
        cudaFree(d_order);
        cudaFree(d_res);
        cudaFree(d_lists);
        cudaFree(d_pilot);
        cudaFree(d_cub);
        if (h_res) cudaFreeHost(h_res);
        d_units = nullptr;
        d_keys = d_vals = d_keys2 = d_order = d_lists = nullptr;
        d_res = nullptr;
        d_pilot = nullptr;
        d_cub = nullptr;
        h_res = nullptr;
        capU = 0;
        cub_bytes = 0;
    }
    void release_items() {
        cudaFree(d_tasks);
        cudaFree(d_seed);
        if (h_seed) cudaFreeHost(h_seed);
        if (h_tasks) cudaFreeHost(h_tasks);
        d_tasks = nullptr;
        d_seed = nullptr;
        h_seed = nullptr;
        h_tasks = nullptr;
        capI = 0;
    }
    void destroy() {
        {
            CascadeOrder& o = cascade_order();
            std::lock_guard<std::mutex> g(o.mu);
            auto it = o.last.find(dev);
            if (it != o.last.end() && it->second == ev[kEvOrder]) o.last.erase(it);
        }
        cudaSetDevice(dev);
        release_units();
        release_items();
        cudaFree(d_ctr);
        cudaFree(d_scratch);
        cudaFree(d_resume);
        if (h_misc) cudaFreeHost(h_misc);
        for (auto& e : ev)
            if (e) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (aux_stream) cudaStreamDestroy(aux_stream);
        for (auto& e : aux_ev)
            if (e) cudaEventDestroy(e);
    }
};


struct DevBatch {
    int dev = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaStream_t aux_stream = nullptr;
    cudaEvent_t* aux_ev = nullptr;
    int t0 = -1;               // start tier, when known on the host
    bool early_copy = false;   // results copied by run_cascade on the copy stream
    int32_t* h_misc = nullptr;
    TierParams tp{};           // planned launch parameters (run_plan -> run_cascade)
    bool all_group = false, no_group = false;
    int group_fam = 1;  // several-lanes-per-unit launches of the narrow tiers: 1 = 4-lane groups, 2 = lane tiers
    // small batches only (at most kPlanUnits units): the longest unit's and the
    // whole batch's estimated antidiagonals (unit_est), for the family choice
    double est_max = 0, est_sum = 0;
    Workspace* ws = nullptr;
    DevPool* pool = nullptr;
    std::vector<int64_t> tasks;  // global task (or unit) indices of this shard
    int64_t n_items = 0;         // tasks (or units) on this device
    int64_t n_units = 0;
    int64_t* d_tasks = nullptr;
    DevUnit* d_units = nullptr;
    uint32_t *d_keys = nullptr, *d_vals = nullptr, *d_keys2 = nullptr, *d_order = nullptr;
    DevResult* d_res = nullptr;
    int32_t* d_seed = nullptr;
    uint32_t* d_lists = nullptr;  // kNumTiers x n_units escalation inputs
    DevCounters* d_ctr = nullptr;
    int32_t* d_scratch = nullptr;
    int32_t* d_resume = nullptr;
    int32_t* d_pilot = nullptr;
    int scratch_warps = 0;
    void* d_cub = nullptr;
    size_t cub_bytes = 0;
    cudaEvent_t* ev = nullptr;
    int sm_count = 0;
    int occ[kWarpTier] = {};   // resident blocks per SM: thread kernels (0-4), wide kernels (5-8)
    int gocc[kWarpTier] = {};  // lane-group kernels (0-4), one-warp-per-unit wide kernels (5-9)
    int locc[kWarpTier] = {};  // lane-tier kernels (0-4)
    int mode = 0;
    int launches = 0;
    // host staging (pinned)
    DevResult* h_res = nullptr;
    int32_t* h_seed = nullptr;
    int64_t* h_tasks = nullptr;
    // host-built units (units mode)
    std::vector<DevUnit> h_units;
};

struct xb_batch {
    xb_pool* pool = nullptr;
    int k = 0, band = 0, flags = 0;
    bool units_mode = false;
    int64_t n = 0;
    std::vector<DevBatch> devs;
    int64_t h2d = 0, d2h = 0;
    bool ran = false;
};

// Batch workspaces hold no pool data, so they are reused across calls and
// pools: a process-wide idle list per device, bounded in count and bytes.
// (Never destroyed at exit: the CUDA runtime may already be gone then.)
struct WorkspaceCache {
    std::mutex mu;
    std::map<int, std::vector<Workspace*>> idle;
};
static WorkspaceCache& ws_cache() {
    static WorkspaceCache* c = new WorkspaceCache();
    return *c;
}
constexpr size_t kIdleWorkspaces = 16;
constexpr int64_t kIdleBytes = 8LL << 30;

static int64_t ws_bytes(const Workspace* w) {
    return w->capU * 160 + w->capI * 40 + int64_t(w->scratch_bytes) + kResumeInts * 4;
}

static void free_dev(xb_pool*, DevBatch& D) {
    if (!D.ws) return;
    Workspace* w = D.ws;
    D.ws = nullptr;
    WorkspaceCache& c = ws_cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto& v = c.idle[w->dev];
        int64_t held = 0;
        for (Workspace* x : v) held += ws_bytes(x);
        if (v.size() < kIdleWorkspaces && held + ws_bytes(w) <= kIdleBytes) {
            w->in_use = false;
            v.push_back(w);
            return;
        }
    }
    w->destroy();
    delete w;
}

// longest-first estimate for a unit, shared with the prep kernel
static inline long long unit_est(long long hl, long long vl) {
    const long long mn = std::min(hl, vl);
    const long long gd = hl > vl ? hl - vl : vl - hl;
    return 2 * mn + std::min(gd, 64LL);
}

static Workspace* acquire_workspace(int dev) {
    WorkspaceCache& c = ws_cache();
    std::lock_guard<std::mutex> g(c.mu);
    auto& v = c.idle[dev];
    if (!v.empty()) {
        Workspace* w = v.back();  // most recently used: its buffers are likely big enough
        v.pop_back();
        w->in_use = true;
        return w;
    }
    auto* w = new Workspace();
    w->dev = dev;
    w->in_use = true;
    return w;
}

// The sequences a device's batch references (tasks: this device's shard;
// units mode: its units), or an empty vector when the device already holds
// the whole pool.  The scan is a relaxed byte store per reference on all
// host threads (~0.5 ms for config 5's 4M references); a dense batch is no
// sign of a full one (a rank's locality shard references every sequence of
// its part of the pool many times, and only that part).
static void referenced_sequences(const xb_batch* B, const DevBatch& D, const void* items,
                                 std::vector<uint8_t>& need) {
    need.clear();
    int64_t ns = 0;
    {
        std::lock_guard<std::mutex> g(B->pool->mu);
        ns = int64_t(B->pool->seq_pos.size());
        auto it = B->pool->dev.find(D.dev);
        if (ns == 0 || (it != B->pool->dev.end() && it->second.ready)) return;
    }
    need.assign(size_t(ns), 0);
    uint8_t* m = need.data();
    const bool sh = !D.tasks.empty();
    if (B->units_mode) {
        const xb_unit* U = static_cast<const xb_unit*>(items);
        parallel_for(D.n_items, [&](int64_t a, int64_t b) {
            for (int64_t q = a; q < b; ++q) {
                const xb_unit& u = U[sh ? D.tasks[size_t(q)] : q];
                __atomic_store_n(&m[u.h_id], uint8_t(1), __ATOMIC_RELAXED);
                __atomic_store_n(&m[u.v_id], uint8_t(1), __ATOMIC_RELAXED);
            }
        });
    } else {
        const xb_task* T = static_cast<const xb_task*>(items);
        parallel_for(D.n_items, [&](int64_t a, int64_t b) {
            for (int64_t q = a; q < b; ++q) {
                const xb_task& t = T[sh ? D.tasks[size_t(q)] : q];
                __atomic_store_n(&m[t.h_id], uint8_t(1), __ATOMIC_RELAXED);
                __atomic_store_n(&m[t.v_id], uint8_t(1), __ATOMIC_RELAXED);
            }
        });
    }
}

static int setup_device(xb_batch* B, DevBatch& D, const xb_exec* ex, const void* items) {
    CK(cudaSetDevice(D.dev));
    D.ws = acquire_workspace(D.dev);
    Workspace& W = *D.ws;
    if (!W.stream) {
        CK(cudaStreamCreateWithFlags(&W.stream, cudaStreamNonBlocking));
        for (auto& e : W.ev) CK(cudaEventCreate(&e));
        CK(cudaMalloc(&W.d_ctr, sizeof(DevCounters)));
        CK(cudaMalloc(&W.d_resume, size_t(kResumeInts) * 4));
        CK(cudaStreamCreateWithFlags(&W.copy_stream, cudaStreamNonBlocking));
        int lo_pri = 0, hi_pri = 0;
        CK(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
        CK(cudaStreamCreateWithPriority(&W.aux_stream, cudaStreamNonBlocking, hi_pri));
        for (auto& e : W.aux_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaMallocHost(&W.h_misc, 4096));
        static_assert(sizeof(DevCounters) <= 4096, "h_misc holds the counters");
    }
    D.stream = (ex && ex->stream && B->devs.size() == 1) ? (cudaStream_t)ex->stream : W.stream;
    D.ev = W.ev;
    CK(cudaDeviceGetAttribute(&D.sm_count, cudaDevAttrMultiProcessorCount, D.dev));
    std::vector<uint8_t> need;
    referenced_sequences(B, D, items, need);
    const int rc = pool_device(B->pool, D.dev, D.stream, &B->h2d, &D.pool, need.empty() ? nullptr : &need);
    if (rc) return rc;
    const int64_t U = std::max<int64_t>(D.n_units, 1);
    if (U > W.capU) {
        W.release_units();
        CK(cudaMalloc(&W.d_units, size_t(U) * sizeof(DevUnit)));
        CK(cudaMalloc(&W.d_keys, size_t(U) * 4));
        CK(cudaMalloc(&W.d_vals, size_t(U) * 4));
        CK(cudaMalloc(&W.d_keys2, size_t(U) * 4));
        CK(cudaMalloc(&W.d_order, size_t(U) * 4));
        CK(cudaMalloc(&W.d_res, size_t(U) * sizeof(DevResult)));
        CK(cudaMalloc(&W.d_lists, size_t(U) * 4 * kNumTiers));
        CK(cudaMalloc(&W.d_pilot, size_t(U / 512 + 128) * 4));
        CK(cudaMallocHost(&W.h_res, size_t(U) * sizeof(DevResult)));
        CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, W.cub_bytes, W.d_keys, W.d_keys2,
                                                     W.d_vals, W.d_order, int(U), 0, 32, D.stream));
        CK(cudaMalloc(&W.d_cub, std::max<size_t>(W.cub_bytes, 16)));
        W.capU = U;
    }
    const int64_t I = std::max<int64_t>(D.n_items, 1);
    if (!B->units_mode && I > W.capI) {
        W.release_items();
        CK(cudaMalloc(&W.d_tasks, size_t(I) * 32));
        CK(cudaMalloc(&W.d_seed, size_t(I) * 4));
        CK(cudaMallocHost(&W.h_seed, size_t(I) * 4));
        CK(cudaMallocHost(&W.h_tasks, size_t(I) * 32));
        W.capI = I;
    }
    // warp-tier scratch: 2*band ints per warp slot, capped at 1 GiB (down to
    // a single warp when one warp's rows alone are that large)
    {
        const int64_t per_warp = 2LL * B->band * 4;
        // one warp slot per unit at most: a small batch with a huge band (the
        // band survey: band = L + 1) needs kilobytes, not the full 16 per SM
        int64_t warps = std::min<int64_t>(int64_t(D.sm_count) * 16, std::max<int64_t>(D.n_units, 1));
        warps = std::min<int64_t>(warps, std::max<int64_t>(1, (1LL << 30) / per_warp));
        if (warps > 4) warps = (warps + 3) / 4 * 4;
        D.scratch_warps = int(warps);
        const size_t need = size_t(warps * per_warp);
        if (need > W.scratch_bytes) {
            cudaFree(W.d_scratch);
            CK(cudaMalloc(&W.d_scratch, need));
            W.scratch_bytes = need;
        }
    }
    D.d_units = W.d_units;
    D.d_keys = W.d_keys;
    D.d_vals = W.d_vals;
    D.d_keys2 = W.d_keys2;
    D.d_order = W.d_order;
    D.d_res = W.d_res;
    D.d_lists = W.d_lists;
    D.d_ctr = W.d_ctr;
    D.d_pilot = W.d_pilot;
    D.d_cub = W.d_cub;
    D.cub_bytes = W.cub_bytes;
    D.d_scratch = W.d_scratch;
    D.d_resume = W.d_resume;
    D.copy_stream = W.copy_stream;
    D.aux_stream = W.aux_stream;
    D.aux_ev = W.aux_ev;
    D.h_misc = W.h_misc;
    D.h_res = W.h_res;
    D.d_tasks = W.d_tasks;
    D.d_seed = W.d_seed;
    D.h_seed = W.h_seed;
    D.h_tasks = W.h_tasks;
    return XB_OK;
}

static int upload_inputs(xb_batch* B, DevBatch& D, const void* items) {
    CK(cudaSetDevice(D.dev));
    if (B->units_mode) {
        const size_t U = size_t(D.n_units);
        if (U) {
            CK(cudaMemcpyAsync(D.d_units, D.h_units.data(), U * sizeof(DevUnit),
                               cudaMemcpyHostToDevice, D.stream));
            CK(cudaStreamSynchronize(D.stream));  // h_units is pageable
            B->h2d += int64_t(U * sizeof(DevUnit));
        }
    } else if (D.n_items) {
        const xb_task* T = static_cast<const xb_task*>(items);
        int64_t* h = D.h_tasks;
        const bool sh = !D.tasks.empty();
        const int64_t* map = sh ? D.tasks.data() : nullptr;
        parallel_for(D.n_items, [&](int64_t a, int64_t b) {
            for (int64_t q = a; q < b; ++q) {
                const xb_task& t = T[sh ? map[q] : q];
                h[4 * q + 0] = t.h_id;
                h[4 * q + 1] = t.v_id;
                h[4 * q + 2] = int64_t(t.h_seed);
                h[4 * q + 3] = int64_t(t.v_seed);
            }
        });
        CK(cudaMemcpyAsync(D.d_tasks, h, size_t(D.n_items) * 32, cudaMemcpyHostToDevice, D.stream));
        B->h2d += D.n_items * 32;
    }
    return XB_OK;
}

constexpr int kGroupLanes = 4;  // lanes per unit in the lane-group tiers (xb_group.cu)
constexpr int kLaneLanes = 8;   // lanes per unit in the lane tiers (xb_lane.cu)
// Batches of at most this many units are planned with host-side estimates of
// their work (est_sum / est_max); every latency-planned batch is smaller.
constexpr int64_t kPlanUnits = 1 << 16;

// 4-lane groups (1) or lane tiers (2) for a latency-planned batch of nu
// units.  Both families finish when the longest unit does or when the
// machine is through the work, whichever is later; in cycles of SMSP time,
// measured on configs 1-3 at several scales:
//   groups: a step every 490 cycles with one warp per SMSP, 620 with two;
//           33 cycles of issue per unit and antidiagonal
//   lanes:  300 / 450 cycles per step; 55 (DNA) or 62 (table modes) of issue
template <typename DB>
static int pick_group_family(const DB& D, bool table_mode, int64_t nu) {
    const double sm = double(D.sm_count), smsp = 4.0 * sm;
    if (D.est_max <= 0) return nu <= int64_t(D.sm_count) * 16 ? 2 : 1;
    const double over = std::min(1.0, std::max(0.0, (double(nu) - 32.0 * sm) / (32.0 * sm)));
    const double groups = std::max((490.0 + 130.0 * over) * D.est_max, 33.0 * D.est_sum / smsp);
    const double lanes = std::max((double(nu) <= 16.0 * sm ? 300.0 : 450.0) * D.est_max,
                                  (table_mode ? 62.0 : 55.0) * D.est_sum / smsp);
    return lanes < 0.95 * groups ? 2 : 1;
}
static int family_lanes(int fam) { return fam == 2 ? kLaneLanes : fam == 1 ? kGroupLanes : 1; }

// Kernel families of the narrow tiers (K16..K64): 0 = one thread per unit,
// 1 = 4-lane groups (xb_group.cu), 2 = lane tiers (8 lanes per unit,
// xb_lane.cu).  The lane tiers step a lone unit ~1.6x sooner at ~2.5x the
// instructions per unit and antidiagonal, so they take the batches that are
// pure latency: few enough units that every SMSP holds at most one warp.
// XB_GROUP_FAMILY=4|8 overrides the choice (A/B runs).
static int forced_group_family() {
    static const int v = [] {
        const char* e = std::getenv("XB_GROUP_FAMILY");
        return e ? (std::atoi(e) == 8 ? 2 : 1) : 0;
    }();
    return v;
}

template <int FAM, int K, int MODE>
static void* tier_fn() {
    if constexpr (FAM == 2)
        return reinterpret_cast<void*>(lane_tier_kernel<K, kLaneLanes, MODE>);
    else if constexpr (FAM == 1)
        return reinterpret_cast<void*>(group_tier_kernel<K, kGroupLanes, MODE>);
    else
        return reinterpret_cast<void*>(thread_tier_kernel<K, MODE>);
}

template <int FAM, int MODE>
static void* tier_fn_t(int t) {
    switch (t) {
        case 0: return tier_fn<FAM, 16, MODE>();
        case 1: return tier_fn<FAM, 24, MODE>();
        case 2: return tier_fn<FAM, 32, MODE>();
        case 3: return tier_fn<FAM, 48, MODE>();
        default: return tier_fn<FAM, 64, MODE>();
    }
}

// wide tiers: G = 8 lanes per unit for a throughput start tier (K96,
// K128), else one warp per unit (escalations, consumers, latency mode)
template <int MODE>
static void* wide_fn_t(int t, bool latency) {
    switch (t) {
        case 5: return latency ? reinterpret_cast<void*>(wide_tier_kernel<96, 32, MODE>)
                               : reinterpret_cast<void*>(wide_tier_kernel<96, 8, MODE>);
        case 6: return latency ? reinterpret_cast<void*>(wide_tier_kernel<128, 32, MODE>)
                               : reinterpret_cast<void*>(wide_tier_kernel<128, 8, MODE>);
        case 7: return reinterpret_cast<void*>(wide_tier_kernel<256, 32, MODE>);
        case 8: return reinterpret_cast<void*>(wide_tier_kernel<512, 32, MODE>);
        default: return reinterpret_cast<void*>(wide_tier_kernel<1024, 32, MODE>);
    }
}

// tiers 0-4: the kernel of family `fam`; 5-9: the wide kernels, where any
// fam != 0 selects the latency form (one warp per unit)
static void* tier_kernel(int fam, int mode, int t) {
    if (t >= kWideFirst)
        return mode == 0 ? wide_fn_t<0>(t, fam != 0) : mode == 1 ? wide_fn_t<1>(t, fam != 0) : wide_fn_t<2>(t, fam != 0);
    if (fam == 2) return mode == 0 ? tier_fn_t<2, 0>(t) : mode == 1 ? tier_fn_t<2, 1>(t) : tier_fn_t<2, 2>(t);
    if (fam == 1) return mode == 0 ? tier_fn_t<1, 0>(t) : mode == 1 ? tier_fn_t<1, 1>(t) : tier_fn_t<1, 2>(t);
    return mode == 0 ? tier_fn_t<0, 0>(t) : mode == 1 ? tier_fn_t<0, 1>(t) : tier_fn_t<0, 2>(t);
}

static cudaError_t launch_tier(int fam, int mode, int t, const TierParams& P, int blocks,
                               cudaStream_t st) {
    TierParams q = P;
    void* args[] = {&q};
    return cudaLaunchKernel(tier_kernel(fam, mode, t), dim3(unsigned(blocks)), dim3(kTB), args, 0, st);
}

static int occupancy_blocks(int fam, int t, int mode, int* out) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tier_kernel(fam, mode, t), kTB, 0) != cudaSuccess)
        return XB_E_CUDA;
    *out = std::max(1, b);
    return XB_OK;
}

static int run_plan(xb_batch* B, DevBatch& D) {
    CK(cudaSetDevice(D.dev));
    xb_pool* p = B->pool;
    const int mode = p->dev_scheme.fast_dna ? 0 : (p->enc == ENC_2BIT ? 1 : 2);
    const bool tok = thread_tiers_ok(p);
    D.launches = 0;
    CK(cudaEventRecord(D.ev[kEvStart], D.stream));
    CK(cudaMemsetAsync(D.d_ctr, 0, sizeof(DevCounters), D.stream));
    const int64_t nu = D.n_units;
    D.early_copy = false;
    D.t0 = -1;
    if (nu == 0) {
        for (int q = kEvPrep; q <= kEvWarp; ++q) CK(cudaEventRecord(D.ev[q], D.stream));
        return XB_OK;
    }
    // ---- LR split + seed score + cost keys (or host-built units) ----
    if (!B->units_mode) {
        PrepParams pp{};
        pp.pool = D.pool->words;
        pp.tasks = D.d_tasks;
        pp.seq_pos = D.pool->seq_pos;
        pp.seq_len = D.pool->seq_len;
        pp.n = D.n_items;
        pp.k = B->k;
        pp.enc = p->enc;
        pp.thread_ok = (tok && !(B->flags & XB_FLAG_GENERIC_ONLY)) ? 1 : 0;
        pp.x = p->scheme.x;
        pp.beta = -p->scheme.gap;
        pp.max_pos_score = std::max(0, p->dev_scheme.max_score);
        pp.scheme = D.pool->scheme;
        pp.units = D.d_units;
        pp.keys = D.d_keys;
        pp.vals = D.d_vals;
        pp.seed_score = D.d_seed;
        pp.warp_list = D.d_lists + int64_t(kWarpTier) * nu;
        pp.warp_len = &D.d_ctr->list_len[kWarpTier];
        const int tb = 256;
        prep_kernel<<<unsigned((D.n_items + tb - 1) / tb), tb, 0, D.stream>>>(pp);
        CK(cudaGetLastError());
        ++D.launches;
    } else {
        // keys/vals/warp list for host-built units
        std::vector<uint32_t> keys(static_cast<size_t>(nu)), vals(static_cast<size_t>(nu)), wl;
        for (int64_t u = 0; u < nu; ++u) {
            DevUnit& x = D.h_units[size_t(u)];
            if (!tok || (B->flags & XB_FLAG_GENERIC_ONLY)) x.route = 2;
            keys[size_t(u)] = uint32_t(std::min<long long>(unit_est(x.h_len, x.v_len), 0xFFFFFFF0LL));
            vals[size_t(u)] = uint32_t(u);
            if (x.route) wl.push_back(uint32_t(u));
        }
        CK(cudaMemcpyAsync(D.d_units, D.h_units.data(), size_t(nu) * sizeof(DevUnit),
                           cudaMemcpyHostToDevice, D.stream));
        CK(cudaMemcpyAsync(D.d_keys, keys.data(), size_t(nu) * 4, cudaMemcpyHostToDevice, D.stream));
        CK(cudaMemcpyAsync(D.d_vals, vals.data(), size_t(nu) * 4, cudaMemcpyHostToDevice, D.stream));
        unsigned long long wlen = wl.size();
        if (!wl.empty())
            CK(cudaMemcpyAsync(D.d_lists + int64_t(kWarpTier) * nu, wl.data(), wl.size() * 4,
                               cudaMemcpyHostToDevice, D.stream));
        CK(cudaMemcpyAsync(&D.d_ctr->list_len[kWarpTier], &wlen, 8, cudaMemcpyHostToDevice, D.stream));
        CK(cudaStreamSynchronize(D.stream));  // host vectors die at scope end
    }
    // units are ready: the pilot (below) may start on the aux stream while
    // the main stream sorts them
    CK(cudaEventRecord(D.aux_ev[0], D.stream));
    // ---- longest first ----
    const uint32_t* order = D.d_vals;
    if (!(B->flags & XB_FLAG_NO_SORT)) {
        size_t tmp = D.cub_bytes;
        CK(cub::DeviceRadixSort::SortPairsDescending(D.d_cub, tmp, D.d_keys, D.d_keys2, D.d_vals,
                                                     D.d_order, int(nu), 0, 32, D.stream));
        order = D.d_order;
    }
    CK(cudaEventRecord(D.ev[kEvPrep], D.stream));

    TierParams tp{};
    tp.pool = D.pool->words;
    tp.units = D.d_units;
    tp.results = D.d_res;
    tp.order = order;
    tp.lists = D.d_lists;
    tp.ctr = D.d_ctr;
    tp.scheme = D.pool->scheme;
    tp.n_units = nu;
    tp.band = B->band;
    tp.warp_scratch = D.d_scratch;
    tp.resume = D.d_resume;
#if XB_CHECKS
    tp.ck_units = (unsigned long long)nu;
    tp.ck_warp_slots = (unsigned long long)D.scratch_warps;
#endif
    tp.r64 = 64;
    tp.one = 1;
    tp.zero = 0;
    tp.two = 2;
    tp.ones = 0x01010101u;
    for (int f = 0; f < 16; ++f) tp.mulc[f] = f ? (1u << (32 - 2 * f)) : 0u;
    const int forced = (B->flags & XB_FLAG_FORCE_TIER) ? ((B->flags >> 8) & 15) : -1;
    D.mode = mode;
    // Lane groups (several lanes per unit) finish a unit several times
    // sooner at ~1.8x the instructions per cell: they take the work whose
    // wall time is set by per-unit latency, not by throughput -- the pilot,
    // escalations, and batches too small to fill the SMs with thread units.
    const bool latency_mode = nu <= int64_t(D.sm_count) * 256 && !(B->flags & XB_FLAG_THROUGHPUT);
    const bool all_group = (B->flags & XB_FLAG_GROUP) || (!(B->flags & XB_FLAG_NO_GROUP) && latency_mode);
    const bool no_group = (B->flags & XB_FLAG_NO_GROUP) && !(B->flags & XB_FLAG_GROUP);
    // pilot: a strided sample of the order, each unit run for at most
    // pilot_cap antidiagonals on the widest thread tier, to measure widths.
    // A latency-bound batch skips it: the pilot would cost about as much as
    // the batch, and there a start a little too wide (K32) costs far less
    // than an escalation, which re-runs the unit after the whole start tier.
    const long long pn = (forced >= 0 || (B->flags & XB_FLAG_GENERIC_ONLY) || latency_mode)
                             ? 0 : std::min<long long>(nu, 64 + nu / 512);
    // Latency-planned batches have no pilot (it would cost as much as the
    // batch) and start at K32 lane groups, or at K16 for DNA with X <= 10.
    // Measured: config 1 (X = 10) K16 0.223 ms, K24 0.239, K32 0.263, no
    // escalations; configs 2 and 3 (X = 15, 20) are fastest at K32: at K24
    // their few escalating units (38, 209) finish in the tail, 7.4 ms / 3.6 ms
    // even with a concurrent consumer (whose polling slowed the start tier),
    // against 6.4 / 3.4 ms.
    int latency_start = (p->scheme.kind == 0 && p->scheme.x <= 10) ? 0 : 2;
    if (const char* e = std::getenv("XB_LATENCY_START")) latency_start = std::atoi(e);
    const int default_start = latency_mode ? latency_start : 4;
    tp.pilot_n = pn;
    tp.pilot_stride = pn ? std::max<long long>(1, nu / pn) : 1;
    // 512 antidiagonals: config 5 and 4 keep their start tiers (K24, K64; 256 sent config 4
    // to K48 at a third of the rate), the pilot on a config-5 shard of 8 takes 0.08 ms, not 0.29
    tp.pilot_cap = std::getenv("XB_PILOT_CAP") ? std::atoi(std::getenv("XB_PILOT_CAP")) : 512;
    tp.pilot_w = D.d_pilot;
    tp.esc_to_warp = (B->flags & XB_FLAG_ESC_TO_WARP) ? 1 : 0;
    for (int t = 0; t < kWarpTier; ++t) {
        if (!D.occ[t]) CK(occupancy_blocks(0, t, mode, &D.occ[t]) ? cudaErrorUnknown : cudaSuccess);
        if (!D.gocc[t]) CK(occupancy_blocks(1, t, mode, &D.gocc[t]) ? cudaErrorUnknown : cudaSuccess);
        if (!D.locc[t]) CK(occupancy_blocks(2, t, mode, &D.locc[t]) ? cudaErrorUnknown : cudaSuccess);
    }
    if (pn > 0) {
        // The pilot samples a stride of the units in input order (d_vals is
        // the identity), so it needs only the prep kernel's units: it runs on
        // the aux stream concurrently with the cost sort on the main stream.
        TierParams pp = tp;
        pp.order = D.d_vals;
        pp.tier = 4;
        pp.pilot = 1;
        pp.role = kRoleAll;
        const bool g = !no_group;
        const long long lanes = pn * (g ? kGroupLanes : 1);
        const int blocks = int(std::min<long long>(D.sm_count * (g ? D.gocc[4] : D.occ[4]), (lanes + kTB - 1) / kTB));
        CK(cudaStreamWaitEvent(D.aux_stream, D.aux_ev[0], 0));
        CK(launch_tier(g ? 1 : 0, mode, 4, pp, blocks, D.aux_stream));
        CK(cudaEventRecord(D.aux_ev[1], D.aux_stream));
        CK(cudaStreamWaitEvent(D.stream, D.aux_ev[1], 0));
        ++D.launches;
    }
    tp.pilot = 0;
    select_tier_kernel<<<1, 256, 0, D.stream>>>(tp, forced >= 0 ? forced : (pn > 0 ? -1 : default_start),
                                                D.h_misc + kMiscStartTier);
    CK(cudaGetLastError());
    ++D.launches;
    CK(cudaEventRecord(D.ev[kEvPilot], D.stream));
    D.tp = tp;
    D.all_group = all_group;
    D.no_group = no_group;
    // a latency-planned batch that puts at most one lane-tier warp on every
    // SMSP runs on the lane tiers (config 1: 0.217 -> 0.139 ms); larger ones
    // are bound by instruction issue, where the 4-lane groups cost less
    // (config 3: 3.4 ms against 3.8 ms, config 2: 6.4 against 11 ms)
    D.group_fam = (B->flags & XB_FLAG_LANES) ? 2 : (B->flags & XB_FLAG_NO_LANES) ? 1
                  : forced_group_family() ? forced_group_family()
                  : latency_mode ? pick_group_family(D, mode != 0, nu) : 1;
    D.t0 = forced >= 0 ? forced : (pn > 0 ? -1 : default_start);  // -1: read back after the pilot
    return XB_OK;  // a pilot-chosen start tier arrives in h_misc[kMiscStartTier] (written by the kernel)
}

// ---- the cascade tail, dispatched on the device --------------------------
// After the start tier, the wider tiers take only the units escalated into
// them -- usually none or a few.  Launching every wider tier from the host
// cost ~6 us per empty launch, and ~40 us while the early result copy held
// PCIe (measured on config 5 shards).  Instead one single-thread kernel
// looks at each tier's escalation list on the device and tail-launches
// (CUDA dynamic parallelism, cudaStreamTailLaunch) only the tiers with work,
// re-launching itself behind each so that it sees the list after that tier
// has finished, then the warp tier.
struct TailPlan {
    TierParams tp;                 // tier / role set per launch
    int32_t grid[kNumTiers];       // blocks for each tier's launch
    int32_t group[kNumTiers];      // narrow tiers: 0 one thread per unit, 1 4-lane groups, 2 lane tiers
    int32_t mode;
    int32_t t0;
    int32_t warp_blocks, warp_threads, warp_enc;
};

template <int MODE>
__device__ void tail_launch_tier(int t, int group, const TierParams& P, int grid) {
    const dim3 g = dim3(unsigned(grid)), b = dim3(kTB);
    switch (t) {
#define XB_TAIL_NARROW(T, K)                                                                        \
    case T:                                                                                         \
        if (group == 2)                                                                             \
            lane_tier_kernel<K, kLaneLanes, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P);            \
        else if (group)                                                                             \
            group_tier_kernel<K, kGroupLanes, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P);          \
        else                                                                                        \
            thread_tier_kernel<K, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P);                      \
        break;
        XB_TAIL_NARROW(0, 16)
        XB_TAIL_NARROW(1, 24)
        XB_TAIL_NARROW(2, 32)
        XB_TAIL_NARROW(3, 48)
        XB_TAIL_NARROW(4, 64)
#undef XB_TAIL_NARROW
        // escalations on the wide tiers: one warp per unit (latency-bound)
        case 5: wide_tier_kernel<96, 32, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P); break;
        case 6: wide_tier_kernel<128, 32, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P); break;
        case 7: wide_tier_kernel<256, 32, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P); break;
        case 8: wide_tier_kernel<512, 32, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P); break;
        default: wide_tier_kernel<1024, 32, MODE><<<g, b, 0, cudaStreamTailLaunch>>>(P); break;
    }
}

__global__ void tail_dispatch_kernel(TailPlan plan, int t) {
    DevCounters* ctr = plan.tp.ctr;
    for (; t < kWarpTier; ++t) {
        // work left in tier t's list (a concurrent consumer may have taken all of it)
        if (ctr->cursor[t] < ctr->list_len[t] && plan.grid[t] > 0) {
            TierParams P = plan.tp;
            P.tier = t;
            P.role = kRoleEscalations;
            if (plan.mode == 0)
                tail_launch_tier<0>(t, plan.group[t], P, plan.grid[t]);
            else if (plan.mode == 1)
                tail_launch_tier<1>(t, plan.group[t], P, plan.grid[t]);
            else
                tail_launch_tier<2>(t, plan.group[t], P, plan.grid[t]);
            tail_dispatch_kernel<<<1, 1, 0, cudaStreamTailLaunch>>>(plan, t + 1);
            ctr->dbg[6] += 2;  // device-side launches (xb_stats.launches)
            return;
        }
    }
    if (t == kWarpTier) {
        TierParams P = plan.tp;
        P.tier = kWarpTier;
        if (ctr->list_len[kWarpTier] > 0) {
            if (plan.warp_enc == ENC_2BIT)
                warp_tier_kernel<ENC_2BIT><<<plan.warp_blocks, plan.warp_threads, 0, cudaStreamTailLaunch>>>(P);
            else
                warp_tier_kernel<ENC_5BIT><<<plan.warp_blocks, plan.warp_threads, 0, cudaStreamTailLaunch>>>(P);
            ctr->dbg[6] += 1;
        }
    }
}

// Resident lane-group blocks per SM for a latency-bound start tier.  A block
// puts one warp (8 groups) on each SMSP.  A lone warp advances one step per
// ~490 cycles of latency while issuing ~160 instructions, so a second warp per
// SMSP fits in the latency shadow and a third only slows every step down --
// including the longest unit's, which sets the batch's wall time.  Batches
// that fit one block per SM keep one warp per SMSP: spreading the units over
// more SMSPs shortens every step.  Measured on 1 B200 (scripts/lat_sweep.sh,
// tier ms at 4/3/2/1 blocks, first version): C1 0.57/0.45/0.35/0.31,
// C2 10.6/8.8/7.4/12.6, C3 4.97/4.98/4.98/5.52; after the step-loop changes
// (batch ms at 3/2/1 blocks): C1 0.50/0.40/0.36, C2 8.13/6.49/11.7,
// C3 3.18/3.17/4.46 (2 for C2 and C3, 1 for C1: the engine's choice).
// Lane-group blocks that consume the next tier's escalations while a
// throughput start tier runs.  Each one displaces about one start-tier block
// (1/592 of the machine); 4 blocks serve 128 escalated units at a time, which
// keeps up with config 5's ~3,000 escalations over the 165 ms start tier.
constexpr int kConsumerBlocks = 4;

// XB_LATENCY_BLOCKS overrides the choice (the sweep).
static int latency_blocks_per_sm(const DevBatch& D) {
    if (const char* e = std::getenv("XB_LATENCY_BLOCKS")) return std::max(1, std::atoi(e));
    const int64_t groups_per_block = kTB / family_lanes(D.group_fam);
    return D.n_units <= int64_t(D.sm_count) * groups_per_block ? 1 : 2;
}

// The cascade: the start tier takes the queue (with a concurrent consumer of
// its escalations), a device-side dispatch runs the wider tiers that have
// escalations and the warp tier, then the results cross PCIe on the copy
// stream (overlapping the next batch's kernels in a stream of batches).
static int run_cascade(xb_batch* B, DevBatch& D) {
    if (D.n_units == 0) return XB_OK;
    CK(cudaSetDevice(D.dev));
    xb_pool* p = B->pool;
    const int mode = D.mode;
    if (D.t0 < 0) D.t0 = D.h_misc[kMiscStartTier];  // the stream was synchronised by xb_batch_run
    TierParams tp = D.tp;
    // the next tier's escalations are consumed concurrently with the start
    // tier (lane groups, when there is a wider lane-group tier); the tail
    // dispatch after the start tier finishes what is left
    const bool concurrent = !D.all_group && !D.no_group && D.t0 + 1 < kWarpTier &&
                            !(B->flags & (XB_FLAG_ESC_TO_WARP | XB_FLAG_SERIAL_TAIL));
    std::unique_lock<std::mutex> order;
    if (!D.all_group) {  // throughput-planned: after the previous such cascade
        CascadeOrder& o = cascade_order();
        order = std::unique_lock<std::mutex>(o.mu);
        auto it = o.last.find(D.dev);
        if (it != o.last.end()) CK(cudaStreamWaitEvent(D.stream, it->second, 0));
    }
    for (int t = 0; t < D.t0 && t < kWarpTier; ++t) CK(cudaEventRecord(D.ev[kEvTier + t], D.stream));
    const int t0 = D.t0;
    if (t0 < kWarpTier) {
        // ---- the start tier ----
        tp.tier = t0;
        if (D.no_group || D.all_group) {
            tp.role = kRoleAll;
            const int* gocc = D.group_fam == 2 && t0 < kNarrowTiers ? D.locc : D.gocc;
            int per_sm = D.all_group ? gocc[t0] : D.occ[t0];
            if (D.all_group && t0 < kNarrowTiers) per_sm = std::min(per_sm, latency_blocks_per_sm(D));
            const int blocks = D.sm_count * per_sm;
            CK(launch_tier(D.all_group ? D.group_fam : 0, mode, t0, tp, blocks, D.stream));
        } else {  // throughput: one thread per unit (or 8 lanes, wide), the concurrent consumer beside it
            if (concurrent) {
                // the next tier's list starts empty-marked
                CK(cudaMemsetAsync(D.d_lists + int64_t(t0 + 1) * D.n_units, 0xFF, size_t(D.n_units) * 4,
                                   D.stream));
                CK(cudaEventRecord(D.aux_ev[0], D.stream));
            }
            tp.role = kRoleStart;
            // leave the consumer's blocks room to be resident whichever kernel
            // the hardware dispatches first (start-tier blocks are persistent)
            CK(launch_tier(0, mode, t0, tp,
                           std::max(1, D.sm_count * D.occ[t0] - (concurrent ? kConsumerBlocks : 0)), D.stream));
            if (concurrent) {
                // a few high-priority blocks take the start tier's escalations while
                // it runs (lane groups, or one warp per unit on the wide tiers).
                // Launched after it (API order), so tools that serialise launches
                // run the consumer after the whole start tier: the consumer never
                // waits on a producer that cannot run (no timeout)
                CK(cudaStreamWaitEvent(D.aux_stream, D.aux_ev[0], 0));
                TierParams cp = tp;
                cp.tier = t0 + 1;
                cp.role = kRoleConsumer;
                CK(launch_tier(1, mode, t0 + 1, cp, kConsumerBlocks, D.aux_stream));
                CK(cudaEventRecord(D.aux_ev[1], D.aux_stream));
                ++D.launches;
            }
        }
        ++D.launches;
        CK(cudaEventRecord(D.ev[kEvTier + t0], D.stream));
        if (concurrent) CK(cudaStreamWaitEvent(D.stream, D.aux_ev[1], 0));
    }
    // ---- the tail: wider tiers and the warp tier (device-dispatched) ----
    {
        TailPlan plan{};
        plan.tp = tp;
        plan.mode = mode;
        plan.t0 = t0;
        for (int t = t0 + 1; t < kWarpTier; ++t) {
            if (t >= kWideFirst) {  // escalations: one warp per unit, at full occupancy
                plan.grid[t] = D.sm_count * D.gocc[t];
                plan.group[t] = 1;
            } else if (D.no_group) {
                plan.grid[t] = D.sm_count * D.occ[t];
                plan.group[t] = 0;
            } else {
                // lane groups; in latency mode no more resident blocks than the start
                // tier (their work is its long units)
                const int fam = D.all_group ? D.group_fam : 1;
                const int occ = fam == 2 ? D.locc[t] : D.gocc[t];
                plan.grid[t] = D.sm_count * (D.all_group ? std::min(occ, latency_blocks_per_sm(D)) : occ);
                plan.group[t] = fam;
            }
        }
        // one warp per scratch slot: blocks of 4 warps, or one smaller block
        const int wpb = std::min(4, D.scratch_warps);
        plan.warp_blocks = D.scratch_warps / wpb;
        plan.warp_threads = 32 * wpb;
        plan.warp_enc = p->enc;
        tail_dispatch_kernel<<<1, 1, 0, D.stream>>>(plan, std::max(t0 + 1, 0));
        CK(cudaGetLastError());
        ++D.launches;
    }
    // The tail's kernels are children of the dispatch grid, so an event
    // recorded now completes after all of them: the tail's time is reported
    // as the warp tier's (xb_stats.ms_tier[9]).  No event per tail tier: the
    // front end handles every stream command slowly while a large D2H copy
    // runs (~30-40 us each, measured), so the cascade issues as few as it can.
    CK(cudaEventRecord(D.ev[kEvWarp], D.stream));
    // results (and seed scores) cross PCIe on the copy stream after the
    // cascade; with a stream of batches they overlap the next batch's kernels
    {
        CK(cudaStreamWaitEvent(D.copy_stream, D.ev[kEvWarp], 0));
        CK(cudaMemcpyAsync(D.h_res, D.d_res, size_t(D.n_units) * sizeof(DevResult), cudaMemcpyDeviceToHost,
                           D.copy_stream));
        if (!B->units_mode && D.n_items)
            CK(cudaMemcpyAsync(D.h_seed, D.d_seed, size_t(D.n_items) * 4, cudaMemcpyDeviceToHost, D.copy_stream));
        CK(cudaEventRecord(D.ev[kEvCopy], D.copy_stream));
        D.early_copy = true;
        B->d2h += D.n_units * int64_t(sizeof(DevResult)) + (B->units_mode ? 0 : D.n_items * 4);
    }
    if (order.owns_lock()) {
        CK(cudaEventRecord(D.ev[kEvOrder], D.stream));
        cascade_order().last[D.dev] = D.ev[kEvOrder];
    }
    return XB_OK;
}

static int fetch_device(xb_batch* B, DevBatch& D) {
    CK(cudaSetDevice(D.dev));
    if (D.early_copy) return XB_OK;  // bulk copy already issued by run_cascade
    if (D.n_units)
        CK(cudaMemcpyAsync(D.h_res, D.d_res, size_t(D.n_units) * sizeof(DevResult),
                           cudaMemcpyDeviceToHost, D.stream));
    if (!B->units_mode && D.n_items)
        CK(cudaMemcpyAsync(D.h_seed, D.d_seed, size_t(D.n_items) * 4, cudaMemcpyDeviceToHost,
                           D.stream));
    CK(cudaEventRecord(D.ev[kEvFetch], D.stream));
    B->d2h += D.n_units * int64_t(sizeof(DevResult)) + (B->units_mode ? 0 : D.n_items * 4);
    return XB_OK;
}

// LPT over estimated task cost (partition.cpp:231-305 without the tile
// memory test): heaviest first onto the least loaded device.
static void shard_lpt(const std::vector<long long>& cost, int G, std::vector<std::vector<int64_t>>& out) {
    out.assign(size_t(G), {});
    std::vector<int64_t> idx(cost.size());
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return cost[size_t(a)] > cost[size_t(b)]; });
    using E = std::pair<long long, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> pq;
    for (int g = 0; g < G; ++g) pq.push({0, g});
    for (int64_t t : idx) {
        E e = pq.top();
        pq.pop();
        out[size_t(e.second)].push_back(t);
        e.first += cost[size_t(t)];
        pq.push(e);
    }
    for (auto& v : out) std::sort(v.begin(), v.end());
}

// Estimated cost of each task: its two units' longest-first estimates (the
// prep kernel's key), the linear proxy of SURVEY §8(e) for h_len * v_len
// (partition.cpp:79-81).  The caller holds p->mu.
static void task_costs(const xb_pool* p, const xb_task* tasks, int64_t n, int k, std::vector<long long>& cost) {
    cost.resize(size_t(n));
    parallel_for(n, [&](int64_t a, int64_t b) {
        for (int64_t t = a; t < b; ++t) {
            const xb_task& q = tasks[t];
            const long long hl = p->offsets[q.h_id + 1] - p->offsets[q.h_id];
            const long long vl = p->offsets[q.v_id + 1] - p->offsets[q.v_id];
            cost[size_t(t)] = unit_est((long long)q.h_seed, (long long)q.v_seed) +
                              unit_est(hl - (long long)q.h_seed - k, vl - (long long)q.v_seed - k) + 1;
        }
    });
}

// Locality-aware shards (the reference packs
// sequences into IPU tiles with a greedy graph partition, partition.cpp:
// 110-184).  Sequences are nodes, tasks edges.  Each
// connected component is ordered by a breadth-first sweep started from a
// peripheral node (the last node of a first BFS), so that neighbouring
// sequences get nearby ranks -- on a read-overlap graph the sweep runs along
// the genome.  Tasks are ordered by the lower rank of their two sequences
// and cut into n_shards contiguous runs of equal estimated cost: each shard
// references a compact neighbourhood of the pool, which is all a device
// then uploads (pool_device's per-sequence residency).
static void shard_locality(const xb_pool* p, const xb_task* tasks, int64_t n, const std::vector<long long>& cost,
                           int G, std::vector<std::vector<int64_t>>& out) {
    const int64_t ns = int64_t(p->offsets.size()) - 1;
    std::vector<int64_t> deg(size_t(ns) + 1, 0);
    for (int64_t t = 0; t < n; ++t) {
        ++deg[tasks[t].h_id];
        if (tasks[t].v_id != tasks[t].h_id) ++deg[tasks[t].v_id];
    }
    std::vector<int64_t> start(size_t(ns) + 1, 0);
    for (int64_t i = 0; i < ns; ++i) start[size_t(i) + 1] = start[size_t(i)] + deg[size_t(i)];
    std::vector<int64_t> adj(static_cast<size_t>(start[size_t(ns)]));
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t t = 0; t < n; ++t) {
        const int64_t h = tasks[t].h_id, v = tasks[t].v_id;
        adj[size_t(fill[size_t(h)]++)] = v;
        if (v != h) adj[size_t(fill[size_t(v)]++)] = h;
    }
    std::vector<int64_t> rank(size_t(ns), -1), mark(size_t(ns), -1), queue;
    queue.reserve(size_t(ns));
    int64_t next_rank = 0;
    auto bfs = [&](int64_t s, int64_t stamp, bool assign) {  // returns the last node reached
        queue.clear();
        queue.push_back(s);
        mark[size_t(s)] = stamp;
        for (size_t h = 0; h < queue.size(); ++h) {
            const int64_t u = queue[h];
            if (assign) rank[size_t(u)] = next_rank++;
            for (int64_t e = start[size_t(u)]; e < start[size_t(u) + 1]; ++e) {
                const int64_t w = adj[size_t(e)];
                if (mark[size_t(w)] != stamp) {
                    mark[size_t(w)] = stamp;
                    queue.push_back(w);
                }
            }
        }
        return queue.back();
    };
    for (int64_t s = 0; s < ns; ++s) {
        if (rank[size_t(s)] >= 0 || deg[size_t(s)] == 0) continue;
        const int64_t far = bfs(s, 2 * s, false);
        bfs(far, 2 * s + 1, true);
    }
    std::vector<int64_t> idx(static_cast<size_t>(n));
    std::iota(idx.begin(), idx.end(), 0);
    auto key = [&](int64_t t) { return std::min(rank[tasks[t].h_id], rank[tasks[t].v_id]); };
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
    long double total = 0;
    for (long long c : cost) total += c;
    out.assign(size_t(G), {});
    long double acc = 0;
    int g = 0;
    for (int64_t t : idx) {
        // cut where the running cost passes the next equal share
        while (g < G - 1 && acc >= total * (g + 1) / G) ++g;
        out[size_t(g)].push_back(t);
        acc += cost[size_t(t)];
    }
    for (auto& v : out) std::sort(v.begin(), v.end());
}

static int exec_devices(const xb_exec* ex, std::vector<int>& ids) {
    const int avail = xb_device_count();
    if (avail <= 0) return XB_E_NO_DEVICE;
    const int n = (ex && ex->n_devices > 1) ? ex->n_devices : 1;
    for (int g = 0; g < n; ++g) {
        int id = (ex && ex->device_ids) ? ex->device_ids[g] : (n == 1 ? -1 : g);
        if (id < 0) {
            if (cudaGetDevice(&id) != cudaSuccess) id = 0;
        }
        if (id >= avail) return XB_E_BAD_PARAM;
        ids.push_back(id);
    }
    return XB_OK;
}

// align.cpp:271-279 order: any dangling id (first such task) before any seed
// out of bounds (first such task); the scan runs on all host threads.
static int validate_tasks(const xb_pool* p, const xb_task* tasks, int64_t n, int k, int64_t* bad) {
    const int64_t ns = xb_pool_size(p);
    const int T = n > (1 << 16) ? n_host_threads() : 1;
    const int64_t chunk = (n + T - 1) / std::max(T, 1);
    std::vector<int64_t> first_dangling(size_t(std::max(T, 1)), INT64_MAX);
    std::vector<int64_t> first_oob(size_t(std::max(T, 1)), INT64_MAX);
    std::vector<int64_t> first_long(size_t(std::max(T, 1)), INT64_MAX);  // a view of 2^31+ symbols
    auto scan = [&](int c) {
        const int64_t a = c * chunk, b = std::min(n, a + chunk);
        for (int64_t t = a; t < b; ++t) {
            const xb_task& q = tasks[t];
            if (int64_t(q.h_id) >= ns || int64_t(q.v_id) >= ns) {
                first_dangling[size_t(c)] = t;
                return;  // nothing later in this chunk can matter
            }
            if (first_oob[size_t(c)] != INT64_MAX) continue;
            const int64_t hl = p->offsets[q.h_id + 1] - p->offsets[q.h_id];
            const int64_t vl = p->offsets[q.v_id + 1] - p->offsets[q.v_id];
            if (int64_t(q.h_seed) + k > hl || int64_t(q.v_seed) + k > vl ||
                q.h_seed > uint64_t(hl) || q.v_seed > uint64_t(vl))
                first_oob[size_t(c)] = t;
            else if (first_long[size_t(c)] == INT64_MAX &&
                     (int64_t(q.h_seed) > kMaxViewLen || int64_t(q.v_seed) > kMaxViewLen ||
                      hl - int64_t(q.h_seed) - k > kMaxViewLen || vl - int64_t(q.v_seed) - k > kMaxViewLen))
                first_long[size_t(c)] = t;
        }
    };
    if (T <= 1) {
        scan(0);
    } else {
        std::vector<std::thread> th;
        for (int c = 0; c < T; ++c) th.emplace_back(scan, c);
        for (auto& x : th) x.join();
    }
    const int64_t dg = *std::min_element(first_dangling.begin(), first_dangling.end());
    if (dg != INT64_MAX) {
        if (bad) *bad = dg;
        return XB_E_DANGLING;
    }
    const int64_t ob = *std::min_element(first_oob.begin(), first_oob.end());
    if (ob != INT64_MAX) {
        if (bad) *bad = ob;
        return XB_E_SEED_OOB;
    }
    const int64_t lg = *std::min_element(first_long.begin(), first_long.end());
    if (lg != INT64_MAX) {
        if (bad) *bad = lg;
        return XB_E_OUT_OF_RANGE;
    }
    return XB_OK;
}

extern "C" {

xb_batch* xb_batch_create(xb_pool* p, const xb_task* tasks, int64_t n, int k, int band,
                          const xb_exec* exec, int64_t* bad_task, int* err) {
    auto fail = [&](int code, xb_batch* b) -> xb_batch* {
        if (err) *err = code;
        if (b) xb_batch_free(b);
        return nullptr;
    };
    if (!p || n < 0 || k < 0 || band < 1 || (n && !tasks)) return fail(XB_E_BAD_PARAM, nullptr);
    std::unique_lock<std::mutex> lk(p->mu);  // the pool must not grow under the scans
    int rc = validate_tasks(p, tasks, n, k, bad_task);
    if (rc) return fail(rc, nullptr);
    std::vector<int> ids;
    rc = exec_devices(exec, ids);
    if (rc) return fail(rc, nullptr);
    auto* B = new xb_batch();
    B->pool = p;
    B->k = k;
    B->band = band;
    B->flags = exec ? exec->flags : 0;
    B->n = n;
    B->devs.resize(ids.size());
    if (ids.size() > 1) {
        std::vector<long long> cost;
        task_costs(p, tasks, n, k, cost);
        std::vector<std::vector<int64_t>> sh;
        if (B->flags & XB_FLAG_LOCALITY)
            shard_locality(p, tasks, n, cost, int(ids.size()), sh);
        else
            shard_lpt(cost, int(ids.size()), sh);
        for (size_t g = 0; g < ids.size(); ++g) B->devs[g].tasks = std::move(sh[g]);
    }
    for (size_t g = 0; g < ids.size(); ++g) {  // planning estimates of small batches
        DevBatch& D = B->devs[g];
        const int64_t ni = ids.size() > 1 ? int64_t(D.tasks.size()) : n;
        if (2 * ni > kPlanUnits) continue;
        for (int64_t q = 0; q < ni; ++q) {
            const xb_task& t = tasks[ids.size() > 1 ? D.tasks[size_t(q)] : q];
            const long long hl = p->offsets[t.h_id + 1] - p->offsets[t.h_id];
            const long long vl = p->offsets[t.v_id + 1] - p->offsets[t.v_id];
            const long long l = unit_est((long long)t.h_seed, (long long)t.v_seed);
            const long long r = unit_est(hl - (long long)t.h_seed - k, vl - (long long)t.v_seed - k);
            D.est_sum += double(l + r);
            D.est_max = std::max(D.est_max, double(std::max(l, r)));
        }
    }
    lk.unlock();
    for (size_t g = 0; g < ids.size(); ++g) {
        DevBatch& D = B->devs[g];
        D.dev = ids[g];
        D.n_items = ids.size() > 1 ? int64_t(D.tasks.size()) : n;
        D.n_units = 2 * D.n_items;
        rc = setup_device(B, D, exec, tasks);
        if (rc) return fail(rc, B);
        rc = upload_inputs(B, D, tasks);
        if (rc) return fail(rc, B);
    }
    for (auto& D : B->devs) {  // pool + task uploads done (see pool_device)
        if (cudaSetDevice(D.dev) != cudaSuccess || cudaStreamSynchronize(D.stream) != cudaSuccess)
            return fail(XB_E_CUDA, B);
    }
    if (err) *err = XB_OK;
    return B;
}

int xb_batch_run(xb_batch* B) {
    if (!B) return XB_E_BAD_PARAM;
    for (auto& D : B->devs) {  // prep, sort, pilot, start-tier choice on every device
        const int rc = run_plan(B, D);
        if (rc) return rc;
    }
    for (auto& D : B->devs) {  // a pilot-chosen start tier is read back (after ~1 ms)
        if (D.n_units && D.t0 < 0) {
            CK(cudaSetDevice(D.dev));
            CK(cudaStreamSynchronize(D.stream));
        }
    }
    for (auto& D : B->devs) {
        const int rc = run_cascade(B, D);
        if (rc) return rc;
    }
    B->ran = true;
    return XB_OK;
}

int xb_batch_sync(xb_batch* B) {
    for (auto& D : B->devs) {
        CK(cudaSetDevice(D.dev));
        CK(cudaStreamSynchronize(D.stream));
    }
    return XB_OK;
}

int xb_batch_fetch(xb_batch* B, xb_side_result* out, int32_t* seed_score) {
    if (!B || !B->ran) return XB_E_BAD_PARAM;
    for (auto& D : B->devs) {
        const int rc = fetch_device(B, D);
        if (rc) return rc;
    }
    for (auto& D : B->devs) {
        CK(cudaSetDevice(D.dev));
        const bool sharded = B->devs.size() > 1;
        // local unit q -> caller's row
        auto row = [&](int64_t q) -> int64_t {
            if (B->units_mode) return sharded ? D.tasks[size_t(q)] : q;
            return sharded ? 2 * D.tasks[size_t(q >> 1)] + (q & 1) : q;
        };
        auto copy_rows = [&](const DevResult* src) {
            if (!sharded) {
                parallel_for(D.n_units, [&](int64_t a, int64_t b) {
                    std::memcpy(out + a, src + a, size_t(b - a) * sizeof(xb_side_result));
                });
            } else {
                parallel_for(D.n_units, [&](int64_t a, int64_t b) {
                    for (int64_t q = a; q < b; ++q) std::memcpy(&out[row(q)], &src[q], sizeof(xb_side_result));
                });
            }
        };
        // every row: copied once the whole cascade had finished (run_cascade)
        CK(cudaEventSynchronize(D.early_copy ? D.ev[kEvCopy] : D.ev[kEvFetch]));
        copy_rows(D.h_res);
        if (seed_score && !B->units_mode) {
            if (!sharded)
                std::memcpy(seed_score, D.h_seed, size_t(D.n_items) * 4);
            else
                for (int64_t q = 0; q < D.n_items; ++q) seed_score[D.tasks[size_t(q)]] = D.h_seed[q];
        }
    }
    return XB_OK;
}

int xb_batch_stats(xb_batch* B, xb_stats* st) {
    if (!B || !st) return XB_E_BAD_PARAM;
    std::memset(st, 0, sizeof *st);
    st->n_devices = int(B->devs.size());
    st->start_tier = -1;
    for (auto& D : B->devs) {
        CK(cudaSetDevice(D.dev));
        CK(cudaStreamSynchronize(D.stream));
        DevCounters c{};
        CK(cudaMemcpyAsync(D.h_misc, D.d_ctr, sizeof c, cudaMemcpyDeviceToHost, D.stream));
        CK(cudaStreamSynchronize(D.stream));
        std::memcpy(&c, D.h_misc, sizeof c);
        float ms[3 + kNumTiers] = {0};
        if (D.n_units && B->ran) {  // before the first run no event has been recorded
            CK(cudaEventElapsedTime(&ms[0], D.ev[kEvStart], D.ev[kEvWarp]));  // whole run
            CK(cudaEventElapsedTime(&ms[1], D.ev[kEvStart], D.ev[kEvPrep]));  // prep + sort
            CK(cudaEventElapsedTime(&ms[2], D.ev[kEvPrep], D.ev[kEvPilot]));  // pilot + select
            // tiers up to the start tier: from the previous tier's end (the pilot's
            // for t = 0); the device-dispatched tail is reported as the warp tier
            const int t0 = std::min(std::max(D.t0, -1), kWarpTier - 1);
            for (int t = 0; t <= t0; ++t)
                CK(cudaEventElapsedTime(&ms[3 + t], D.ev[kEvTier + t - 1], D.ev[kEvTier + t]));
            CK(cudaEventElapsedTime(&ms[3 + kWarpTier], D.ev[kEvTier + t0], D.ev[kEvWarp]));
        }
        st->ms_total = std::max(st->ms_total, double(ms[0]));
        st->ms_prep = std::max(st->ms_prep, double(ms[1]));
        st->ms_pilot = std::max(st->ms_pilot, double(ms[2]));
        for (int t = 0; t < kNumTiers; ++t) {
            st->ms_tier[t] = std::max(st->ms_tier[t], double(ms[3 + t]));
            st->units_tier[t] += int64_t(c.units[t]);
            st->cells_tier[t] += int64_t(c.cells[t]);
            st->escalated[t] += int64_t(c.escalated[t]);
        }
        st->start_tier = c.start_tier;
        st->start_lane_groups = (D.n_units && D.all_group) ? D.group_fam : 0;
        for (int q = 0; q < 6; ++q) st->dbg[q] += int64_t(c.dbg[q]);
        st->launches += D.launches + int(c.dbg[6]);  // host launches + the tail's device launches
        st->sm_count = D.sm_count;
    }
    st->h2d_bytes = B->h2d;
    st->d2h_bytes = B->d2h;
    return XB_OK;
}

void xb_batch_free(xb_batch* B) {
    if (!B) return;
    for (auto& D : B->devs) {  // nothing may still write into a workspace handed back
        if (D.ws && cudaSetDevice(D.dev) == cudaSuccess) {
            if (D.stream) cudaStreamSynchronize(D.stream);
            if (D.copy_stream) cudaStreamSynchronize(D.copy_stream);
        }
        free_dev(B->pool, D);
    }
    delete B;
}

int xb_extend_batch(xb_pool* p, const xb_task* tasks, int64_t n, int k, int band,
                    xb_side_result* out, int32_t* seed_score, int64_t* bad_task,
                    const xb_exec* exec) {
    int err = 0;
    xb_batch* B = xb_batch_create(p, tasks, n, k, band, exec, bad_task, &err);
    if (!B) return err;
    int rc = xb_batch_run(B);
    if (!rc) rc = xb_batch_fetch(B, out, seed_score);
    if (!rc) rc = xb_batch_stats(B, &g_last_stats);
    xb_batch_free(B);
    return rc;
}

int xb_extend_units(xb_pool* p, const xb_unit* units, int64_t n, int band, xb_side_result* out,
                    int64_t* bad_unit, const xb_exec* exec) {
    if (!p || n < 0 || band < 1 || (n && !units)) return XB_E_BAD_PARAM;
    std::unique_lock<std::mutex> lk(p->mu);  // the pool must not grow under the scan
    const int64_t ns = xb_pool_size(p);
    std::vector<DevUnit> all(static_cast<size_t>(n));
    for (int64_t q = 0; q < n; ++q) {
        const xb_unit& u = units[q];
        if (int64_t(u.h_id) >= ns || int64_t(u.v_id) >= ns) {
            if (bad_unit) *bad_unit = q;
            return XB_E_DANGLING;
        }
        const int64_t hn = p->seq_len[u.h_id], vn = p->seq_len[u.v_id];
        // make_view range checks (sequence.cpp:5-15)
        auto bad_view = [&](int64_t len, uint64_t origin, int dir, uint64_t length) {
            if (origin > uint64_t(len)) return true;
            const uint64_t room = dir ? uint64_t(len) - origin : origin;
            return length > room;
        };
        // views of 2^31 symbols or more: the result fields (int h_ext/v_ext,
        // align.hpp:37-45) and the kernels' int32 lengths cannot hold them
        if (bad_view(hn, u.h_origin, u.h_dir, u.h_len) || bad_view(vn, u.v_origin, u.v_dir, u.v_len) ||
            u.h_len > uint64_t(kMaxViewLen) || u.v_len > uint64_t(kMaxViewLen)) {
            if (bad_unit) *bad_unit = q;
            return XB_E_OUT_OF_RANGE;
        }
        DevUnit& d = all[size_t(q)];
        d.h_pos = p->seq_pos[u.h_id] + int64_t(u.h_origin) - (u.h_dir ? 0 : 1);
        d.v_pos = p->seq_pos[u.v_id] + int64_t(u.v_origin) - (u.v_dir ? 0 : 1);
        d.h_len = int32_t(u.h_len);
        d.v_len = int32_t(u.v_len);
        d.dir = (u.h_dir ? 1 : 0) | (u.v_dir ? 2 : 0);
        const long long mn = std::min<long long>(u.h_len, u.v_len);
        const long long bound = (long long)std::max(0, p->dev_scheme.max_score) * mn +
                                (long long)(-p->scheme.gap) * (long long)(u.h_len + u.v_len + 2) +
                                p->scheme.x + 2;
        d.route = (bound < (1LL << 23) && u.h_len < (1ull << 30) && u.v_len < (1ull << 30)) ? 0 : 2;
    }
    lk.unlock();
    std::vector<int> ids;
    int rc = exec_devices(exec, ids);
    if (rc) return rc;
    auto* B = new xb_batch();
    B->pool = p;
    B->band = band;
    B->flags = exec ? exec->flags : 0;
    B->units_mode = true;
    B->n = n;
    B->devs.resize(ids.size());
    std::vector<std::vector<int64_t>> sh;
    if (ids.size() > 1) {
        std::vector<long long> cost(static_cast<size_t>(n));
        for (int64_t q = 0; q < n; ++q) cost[size_t(q)] = unit_est(all[size_t(q)].h_len, all[size_t(q)].v_len) + 1;
        shard_lpt(cost, int(ids.size()), sh);
    }
    for (size_t g = 0; g < ids.size(); ++g) {
        DevBatch& D = B->devs[g];
        D.dev = ids[g];
        if (ids.size() > 1) {
            D.tasks = sh[g];
            for (int64_t q : D.tasks) D.h_units.push_back(all[size_t(q)]);
        } else {
            D.h_units = all;
        }
        D.n_items = int64_t(D.h_units.size());
        D.n_units = D.n_items;
        if (D.n_units <= kPlanUnits)
            for (const DevUnit& x : D.h_units) {
                const long long e = unit_est(x.h_len, x.v_len);
                D.est_sum += double(e);
                D.est_max = std::max(D.est_max, double(e));
            }
        rc = setup_device(B, D, exec, units);
        if (!rc) rc = upload_inputs(B, D, nullptr);
        if (rc) {
            xb_batch_free(B);
            return rc;
        }
    }
    rc = xb_batch_run(B);
    if (!rc) rc = xb_batch_fetch(B, out, nullptr);
    if (!rc) rc = xb_batch_stats(B, &g_last_stats);
    xb_batch_free(B);
    return rc;
}

int xb_sweep_band(uint64_t length, const int32_t* xs, int32_t nx, const double* ps, int32_t np,
                  uint64_t rng_seed, int32_t* delta_w, const xb_exec* exec) {
    if (nx < 0 || np < 0 || (nx && !xs) || (np && !ps) || (nx && np && !delta_w)) return XB_E_BAD_PARAM;
    if (length + 1 > uint64_t(INT32_MAX)) return XB_E_BAD_PARAM;
    for (int32_t a = 0; a < nx; ++a)
        if (xs[a] < 0) return XB_E_BAD_PARAM;  // scoring.cpp:17-20
    if (!nx || !np) return XB_OK;
    // the np pairs (pipeline.cpp:188-195), shared by every X
    std::vector<char> sym;
    std::vector<int64_t> off{0};
    for (int32_t b = 0; b < np; ++b) {
        int err = 0;
        xb_synth* S = xb_synth_pairs(1, length, ps[b], 17, 0, rng_seed, &err);
        if (!S) return err;
        int64_t z[6];
        xb_synth_sizes(S, z);
        const size_t base = sym.size();
        sym.resize(base + size_t(z[1]));
        std::vector<int64_t> o(size_t(z[0]) + 1);
        xb_synth_copy(S, sym.data() + base, o.data(), nullptr);
        xb_synth_free(S);
        for (size_t q = 1; q < o.size(); ++q) off.push_back(int64_t(base) + o[q]);
    }
    // full views, both Right (pipeline.cpp:196-199); band = length + 1
    std::vector<xb_unit> units(static_cast<size_t>(np));
    for (int32_t b = 0; b < np; ++b)
        units[size_t(b)] = xb_unit{uint32_t(2 * b), uint32_t(2 * b + 1), 1, 1, 0, 0, length, length};
    std::vector<int> rcs(static_cast<size_t>(nx), XB_OK);
    auto one_x = [&](int32_t a) {
        int err = 0;
        xb_scheme* sc = xb_scheme_match_mismatch(1, -1, -1, xs[a], &err);
        if (!sc) {
            rcs[size_t(a)] = err;
            return;
        }
        xb_pool* pool = xb_pool_create(sc, &err);
        xb_scheme_free(sc);
        if (!pool) {
            rcs[size_t(a)] = err;
            return;
        }
        const int64_t id = xb_pool_add_bulk(pool, sym.data(), off.data(), int64_t(off.size()) - 1);
        std::vector<xb_side_result> out(static_cast<size_t>(np));
        int64_t bad = -1;
        int rc = id < 0 ? int(-id) : xb_extend_units(pool, units.data(), np, int(length + 1), out.data(), &bad, exec);
        for (int32_t b = 0; b < np && !rc; ++b) delta_w[size_t(a) * size_t(np) + size_t(b)] = out[size_t(b)].delta_w;
        xb_pool_free(pool);
        rcs[size_t(a)] = rc;
    };
    // the X values are independent batches: run them concurrently
    std::vector<std::thread> th;
    for (int32_t a = 0; a < nx; ++a) th.emplace_back(one_x, a);
    for (auto& t : th) t.join();
    for (int rc : rcs)
        if (rc) return rc;
    return XB_OK;
}

int xb_shard_tasks(xb_pool* p, const xb_task* tasks, int64_t n, int k, int n_shards, int mode,
                   int32_t* shard_of, int64_t* bad_task) {
    if (!p || n < 0 || k < 0 || n_shards < 1 || (n && (!tasks || !shard_of)) ||
        (mode != XB_SHARD_LPT && mode != XB_SHARD_LOCALITY))
        return XB_E_BAD_PARAM;
    std::lock_guard<std::mutex> g(p->mu);
    const int rc = validate_tasks(p, tasks, n, k, bad_task);
    if (rc) return rc;
    std::vector<long long> cost;
    task_costs(p, tasks, n, k, cost);
    std::vector<std::vector<int64_t>> sh;
    if (mode == XB_SHARD_LOCALITY)
        shard_locality(p, tasks, n, cost, n_shards, sh);
    else
        shard_lpt(cost, n_shards, sh);
    for (int s = 0; s < n_shards; ++s)
        for (int64_t t : sh[size_t(s)]) shard_of[t] = s;
    return XB_OK;
}

int xb_plan_group_family(int sm_count, int table_mode, int64_t n_units, double est_max, double est_sum) {
    struct { int sm_count; double est_max, est_sum; } d{sm_count, est_max, est_sum};
    return pick_group_family(d, table_mode != 0, n_units);
}

int xb_debug_checks(int device, uint32_t* failed) {
    if (failed) *failed = 0;
#if XB_CHECKS
    if (cudaSetDevice(device) != cudaSuccess) return XB_E_CUDA;
    unsigned int v = 0, zero = 0;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpyFromSymbol(&v, xb_check_fail, sizeof v));
    CK(cudaMemcpyToSymbol(xb_check_fail, &zero, sizeof zero));
    if (failed) *failed = v;
    return XB_OK;
#else
    (void)device;
    return -1;  // a product build: the checks are compiled out
#endif
}

int xb_last_stats(xb_stats* st) {
    if (!st) return XB_E_BAD_PARAM;
    *st = g_last_stats;
    return XB_OK;
}

int xb_measure_int32_peak(int device, double* alu, double* mixed, double* clk_mhz, int* sm_count) {
    if (xb_device_count() <= device) return XB_E_NO_DEVICE;
    CK(cudaSetDevice(device));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int tb = 256, bps = 8, blocks = sms * bps, iters = 1 << 14;
    int32_t* out = nullptr;
    long long* clk = nullptr;
    CK(cudaMalloc(&out, size_t(blocks) * tb * 4));
    CK(cudaMalloc(&clk, size_t(blocks) * 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double res[2] = {0, 0};
    double mhz = 0;
    for (int v = 0; v < 2; ++v) {
        for (int rep = 0; rep < 3; ++rep) {  // warm, then keep the best
            CK(cudaEventRecord(e0));
            if (v == 0) int_peak_alu<<<blocks, tb>>>(out, iters, 7, clk);
            else int_peak_mixed<<<blocks, tb>>>(out, iters, 7, clk);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::vector<long long> c(static_cast<size_t>(blocks));
            CK(cudaMemcpy(c.data(), clk, size_t(blocks) * 8, cudaMemcpyDeviceToHost));
            const long long cmax = *std::max_element(c.begin(), c.end());
            const double ops = double(blocks) * tb * iters * 32.0;  // 32 SASS instructions per iteration
            // per-SM clock cycles: blocks run concurrently (bps resident per SM)
            const double per_clk_sm = ops / (double(cmax) * sms);
            res[v] = std::max(res[v], per_clk_sm);
            mhz = std::max(mhz, double(cmax) / (ms * 1e3));
        }
    }
    cudaFree(out);
    cudaFree(clk);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (alu) *alu = res[0];
    if (mixed) *mixed = res[1];
    if (clk_mhz) *clk_mhz = mhz;
    if (sm_count) *sm_count = sms;
    return XB_OK;
}

}  // extern "C"
