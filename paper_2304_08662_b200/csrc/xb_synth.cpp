// Deterministic synthetic inputs for the five BASELINE.json configs
// (SURVEY.md §8d).  The paper's ELBA/PASTIS datasets are not available, so
// these seeded generators stand in for them with the configs' shapes, sizes,
// mutation models and seed placement.  Raw std::mt19937_64 draws only, as
// the reference generator does (proj/src/io.cpp:205-212); one engine per
// pair / read, seeded from splitmix64(config seed, index), so the output is
// identical for any thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xdrop_b200.h"

namespace {

constexpr char kBases[4] = {'A', 'C', 'G', 'T'};
constexpr char kAmino[21] = "ARNDCQEGHILKMFPSTWYV";

uint64_t splitmix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct Rng {
    std::mt19937_64 e;
    explicit Rng(uint64_t s) : e(s) {}
    uint64_t operator()() { return e(); }
    double unit() { return double(e() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) { return n ? e() % n : 0; }
};

struct Interval {
    int64_t a, b;  // [a, b) in source coordinates, copied verbatim
};

// Copies src with per-position events at `rate`: substitution / insertion /
// deletion chosen with weights ws:wi:wd.  Protected intervals (seeds) are
// copied exactly.  map[p] = output position of source position p (-1 if
// deleted).  `sub` draws a substituted symbol for a source symbol.
template <class Sub, class Ins>
void mutate(Rng& r, const char* src, int64_t n, double rate, int ws, int wi, int wd,
            const std::vector<Interval>& prot, std::string& out, std::vector<int64_t>* map, Sub sub,
            Ins ins) {
    out.clear();
    out.reserve(size_t(n + n / 8 + 16));
    if (map) map->assign(size_t(n), -1);
    size_t pi = 0;
    const int wt = ws + wi + wd;
    for (int64_t p = 0; p < n; ++p) {
        while (pi < prot.size() && prot[pi].b <= p) ++pi;
        const bool guarded = pi < prot.size() && prot[pi].a <= p;
        if (!guarded && r.unit() < rate) {
            const int ev = int(r.below(uint64_t(wt)));
            if (ev < ws) {
                if (map) (*map)[size_t(p)] = int64_t(out.size());
                out.push_back(sub(r, src[p]));
                continue;
            } else if (ev < ws + wi) {
                out.push_back(ins(r));
            } else {
                continue;  // deletion
            }
        }
        if (map) (*map)[size_t(p)] = int64_t(out.size());
        out.push_back(src[p]);
    }
}

char dna_sub(Rng& r, char c) {
    int cur = 0;
    while (kBases[cur] != c) ++cur;
    return kBases[(cur + 1 + int(r.below(3))) % 4];
}
char dna_ins(Rng& r) { return kBases[r.below(4)]; }

void random_dna(Rng& r, char* out, int64_t n) {
    int64_t i = 0;
    while (i < n) {
        uint64_t w = r();
        for (int q = 0; q < 32 && i < n; ++q, ++i, w >>= 2) out[i] = kBases[w & 3];
    }
}

template <class F>
void par(int64_t n, int T, F&& f) {
    if (T <= 1 || n < 64) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int64_t> next{0};
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&] {
            for (;;) {
                const int64_t i0 = next.fetch_add(16);
                if (i0 >= n) return;
                for (int64_t i = i0; i < std::min(n, i0 + 16); ++i) f(i);
            }
        });
    for (auto& x : th) x.join();
}

}  // namespace

struct xb_synth {
    std::vector<char> symbols;
    std::vector<int64_t> offsets{0};
    std::vector<int64_t> tasks;  // 4 per task
    int k = 17, x = 15, band = 1024;
};

namespace {

struct PairOut {
    std::string h, v;
    std::vector<int64_t> seeds;  // h_seed, v_seed pairs
};

void assemble(xb_synth* S, std::vector<PairOut>& pairs, bool shared_pool) {
    int64_t total = 0;
    for (auto& p : pairs) total += int64_t(p.h.size() + p.v.size());
    S->symbols.reserve(size_t(total));
    for (size_t i = 0; i < pairs.size(); ++i) {
        const int64_t hid = int64_t(S->offsets.size()) - 1;
        S->symbols.insert(S->symbols.end(), pairs[i].h.begin(), pairs[i].h.end());
        S->offsets.push_back(int64_t(S->symbols.size()));
        S->symbols.insert(S->symbols.end(), pairs[i].v.begin(), pairs[i].v.end());
        S->offsets.push_back(int64_t(S->symbols.size()));
        for (size_t q = 0; q + 1 < pairs[i].seeds.size(); q += 2) {
            S->tasks.push_back(hid);
            S->tasks.push_back(hid + 1);
            S->tasks.push_back(pairs[i].seeds[q]);
            S->tasks.push_back(pairs[i].seeds[q + 1]);
        }
        std::string().swap(pairs[i].h);
        std::string().swap(pairs[i].v);
    }
    (void)shared_pool;
}

// cfg 1, 2, 4: DNA pairs, v = mutate(h) at 15% / 5% (1:1:1), seeds protected
void make_dna_pairs(xb_synth* S, int cfg, double scale, uint64_t seed, int T) {
    int64_t n_pairs;
    if (cfg == 1) n_pairs = std::max<int64_t>(1, llround(1000 * scale));
    else if (cfg == 2) n_pairs = std::max<int64_t>(1, llround(10000 * scale));
    else n_pairs = std::max<int64_t>(1, llround(40000 * scale));
    const double rate = cfg == 1 ? 0.05 : 0.15;
    const int k = 17;
    std::vector<PairOut> pairs(static_cast<size_t>(n_pairs));
    par(n_pairs, T, [&](int64_t pi) {
        Rng r(splitmix(seed * 1000003ull + uint64_t(pi)));
        int64_t L;
        if (cfg == 1) L = 1000;
        else if (cfg == 2) L = 10000;
        else L = int64_t(std::floor(1000.0 * std::exp(r.unit() * std::log(25.0))));  // log-uniform
        PairOut& P = pairs[size_t(pi)];
        P.h.resize(size_t(L));
        random_dna(r, &P.h[0], L);
        std::vector<int64_t> hs;
        if (cfg == 1) {
            hs.push_back((L - k) / 2);  // the aligned midpoint
        } else if (cfg == 2) {
            hs.push_back(int64_t(r.below(uint64_t(L - k + 1))));
        } else {
            const int ns = 1 + int(r.below(4));
            for (int tries = 0; int(hs.size()) < ns && tries < 64; ++tries) {
                const int64_t s = int64_t(r.below(uint64_t(L - k + 1)));
                bool clash = false;
                for (int64_t o : hs) clash |= (s < o + k && o < s + k);
                if (!clash) hs.push_back(s);
            }
            std::sort(hs.begin(), hs.end());
        }
        std::vector<Interval> prot;
        for (int64_t s : hs) prot.push_back({s, s + k});
        std::vector<int64_t> map;
        mutate(r, P.h.data(), L, rate, 1, 1, 1, prot, P.v, &map, dna_sub, dna_ins);
        for (int64_t s : hs) {
            P.seeds.push_back(s);
            P.seeds.push_back(map[size_t(s)]);
        }
    });
    if (cfg == 4) {
        // exactly the configured number of extensions
        const int64_t want = std::max<int64_t>(1, llround(100000 * scale));
        int64_t have = 0;
        for (auto& p : pairs) have += int64_t(p.seeds.size() / 2);
        for (int64_t pi = n_pairs - 1; pi >= 0 && have > want; --pi) {
            auto& sd = pairs[size_t(pi)].seeds;
            while (have > want && sd.size() > 2) {
                sd.resize(sd.size() - 2);
                --have;
            }
        }
    }
    S->k = k;
    S->x = cfg == 1 ? 10 : cfg == 2 ? 15 : 50;
    S->band = cfg == 2 ? 256 : 1024;
    assemble(S, pairs, cfg == 4);
}

// cfg 3: protein pairs, BLOSUM62 conditional substitutions + 5% indels
int make_protein(xb_synth* S, double scale, uint64_t seed, const char* matrix_text, int T) {
    char alpha[64];
    int cells[64 * 64];
    const int n = xb_parse_submatrix(matrix_text, alpha, 64, cells, 64 * 64);
    if (n <= 0) return XB_E_PARSE;
    // conditional substitution table over the 20 standard residues:
    // P(b | a) proportional to 2^(S(a,b)/2), b != a (1/2-bit units)
    int idx[20];
    for (int a = 0; a < 20; ++a) {
        const char* p = std::strchr(alpha, kAmino[a]);
        if (!p) return XB_E_PARSE;
        idx[a] = int(p - alpha);
    }
    double cum[20][20];
    for (int a = 0; a < 20; ++a) {
        double acc = 0;
        for (int b = 0; b < 20; ++b) {
            if (b != a) acc += std::pow(2.0, cells[idx[a] * n + idx[b]] / 2.0);
            cum[a][b] = acc;
        }
        for (int b = 0; b < 20; ++b) cum[a][b] /= acc;
    }
    int code[256];
    for (int a = 0; a < 20; ++a) code[(unsigned char)kAmino[a]] = a;
    const int64_t n_pairs = std::max<int64_t>(1, llround(10000 * scale));
    const int k = 6;
    std::vector<PairOut> pairs(static_cast<size_t>(n_pairs));
    par(n_pairs, T, [&](int64_t pi) {
        Rng r(splitmix(seed * 1000003ull + uint64_t(pi)));
        const int64_t L = 1000 + int64_t(r.below(4001));
        PairOut& P = pairs[size_t(pi)];
        P.h.resize(size_t(L));
        for (int64_t i = 0; i < L; ++i) P.h[size_t(i)] = kAmino[r.below(20)];  // uniform stand-in
        const int64_t s = int64_t(r.below(uint64_t(L - k + 1)));
        std::vector<Interval> prot{{s, s + k}};
        // 30% substitutions then 5% indels (half insertions, half deletions)
        std::string mid;
        mutate(
            r, P.h.data(), L, 0.30, 1, 0, 0, prot, mid, nullptr,
            [&](Rng& rr, char c) {
                const int a = code[(unsigned char)c];
                const double u = rr.unit();
                int b = 0;
                while (b < 19 && cum[a][b] < u) ++b;
                if (b == a) b = (b + 1) % 20;
                return kAmino[b];
            },
            [](Rng& rr) { return kAmino[rr.below(20)]; });
        std::vector<int64_t> map;
        mutate(
            r, mid.data(), int64_t(mid.size()), 0.05, 0, 1, 1, prot, P.v, &map,
            [](Rng&, char c) { return c; }, [](Rng& rr) { return kAmino[rr.below(20)]; });
        P.seeds.push_back(s);
        P.seeds.push_back(map[size_t(s)]);
    });
    S->k = k;
    S->x = 20;
    S->band = 1024;
    assemble(S, pairs, false);
    return XB_OK;
}

// cfg 5: genome-based overlap workload.  Reads are sampled from a random
// genome (log-normal lengths, median 10 kb, sigma 0.5, clipped to 1-25 kb),
// each with 7.5% errors (1:1:1) so pairs differ by ~15%.  Pairs are read
// pairs with a true dovetail overlap of 2-8 kb; each carries 1-3 exact 17-mer
// seeds planted on the true overlap diagonal (copied error-free into both
// reads).
void make_overlap(xb_synth* S, double scale, uint64_t seed, int T) {
    const int64_t n_reads = std::max<int64_t>(4, llround(200000 * scale));
    const int64_t want = std::max<int64_t>(1, llround(2000000 * scale));
    const int64_t G = n_reads * 900;
    const int k = 17;
    Rng master(splitmix(seed));
    std::vector<int64_t> len(static_cast<size_t>(n_reads)), start(static_cast<size_t>(n_reads));
    for (int64_t i = 0; i < n_reads; ++i) {
        // Box-Muller from raw draws
        const double u1 = std::max(master.unit(), 1e-300), u2 = master.unit();
        const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
        int64_t L = int64_t(std::llround(10000.0 * std::exp(0.5 * z)));
        L = std::min<int64_t>(25000, std::max<int64_t>(1000, L));
        len[size_t(i)] = L;
    }
    for (int64_t i = 0; i < n_reads; ++i)
        start[size_t(i)] = int64_t(master.below(uint64_t(G - len[size_t(i)])));
    // ids in genome order
    std::vector<int64_t> ord(static_cast<size_t>(n_reads));
    for (int64_t i = 0; i < n_reads; ++i) ord[size_t(i)] = i;
    std::sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return start[size_t(a)] < start[size_t(b)] || (start[size_t(a)] == start[size_t(b)] && a < b);
    });
    std::vector<int64_t> st(static_cast<size_t>(n_reads)), ln(static_cast<size_t>(n_reads));
    for (int64_t i = 0; i < n_reads; ++i) {
        st[size_t(i)] = start[size_t(ord[size_t(i)])];
        ln[size_t(i)] = len[size_t(ord[size_t(i)])];
    }
    // dovetail pairs (A before B): overlap = end(A) - start(B) in [2000, 8000], B ends after A
    struct Pr {
        int64_t a, b;
    };
    std::vector<Pr> prs;
    for (int64_t a = 0; a < n_reads; ++a) {
        const int64_t ea = st[size_t(a)] + ln[size_t(a)];
        for (int64_t b = a + 1; b < n_reads && st[size_t(b)] <= ea - 2000; ++b) {
            const int64_t ov = ea - st[size_t(b)];
            if (ov >= 2000 && ov <= 8000 && st[size_t(b)] + ln[size_t(b)] > ea) prs.push_back({a, b});
        }
    }
    for (int64_t i = int64_t(prs.size()) - 1; i > 0; --i)
        std::swap(prs[size_t(i)], prs[master.below(uint64_t(i + 1))]);
    // planted seeds: genome positions g, per pair, until `want` extensions
    struct Sd {
        int64_t a, b, g;
    };
    std::vector<Sd> seeds;
    std::vector<std::vector<int64_t>> per_read(static_cast<size_t>(n_reads));
    for (const Pr& p : prs) {
        if (int64_t(seeds.size()) >= want) break;
        const int64_t lo = st[size_t(p.b)], hi = st[size_t(p.a)] + ln[size_t(p.a)] - k;  // [lo, hi]
        const int ns = 1 + int(master.below(3));
        std::vector<int64_t> gs;
        for (int tries = 0; int(gs.size()) < ns && tries < 32; ++tries) {
            const int64_t g = lo + int64_t(master.below(uint64_t(hi - lo + 1)));
            bool clash = false;
            for (int64_t o : gs) clash |= (g < o + k && o < g + k);
            if (!clash) gs.push_back(g);
        }
        for (int64_t g : gs) {
            if (int64_t(seeds.size()) >= want) break;
            seeds.push_back({p.a, p.b, g});
            per_read[size_t(p.a)].push_back(g);
            per_read[size_t(p.b)].push_back(g);
        }
    }
    // genome, chunked engines
    std::vector<char> genome(static_cast<size_t>(G));
    const int64_t CH = 1 << 20;
    par((G + CH - 1) / CH, T, [&](int64_t c) {
        Rng r(splitmix(seed ^ 0xABCDEF12345ull) + uint64_t(c));
        random_dna(r, genome.data() + c * CH, std::min(CH, G - c * CH));
    });
    // reads
    std::vector<std::string> reads(static_cast<size_t>(n_reads));
    std::vector<std::vector<int64_t>> seed_pos(static_cast<size_t>(n_reads));  // read pos per per_read[] entry
    par(n_reads, T, [&](int64_t i) {
        Rng r(splitmix(seed * 7919ull + uint64_t(i)));
        auto& g = per_read[size_t(i)];
        std::vector<int64_t> sorted = g;
        std::sort(sorted.begin(), sorted.end());
        std::vector<Interval> prot;
        for (int64_t x : sorted) {
            const int64_t a = x - st[size_t(i)];
            if (!prot.empty() && prot.back().b >= a) prot.back().b = std::max(prot.back().b, a + k);
            else prot.push_back({a, a + k});
        }
        std::vector<int64_t> map;
        mutate(r, genome.data() + st[size_t(i)], ln[size_t(i)], 0.075, 1, 1, 1, prot,
               reads[size_t(i)], &map, dna_sub, dna_ins);
        seed_pos[size_t(i)].resize(g.size());
        for (size_t q = 0; q < g.size(); ++q) seed_pos[size_t(i)][q] = map[size_t(g[q] - st[size_t(i)])];
    });
    // pool = reads in genome order; tasks = (A, B, posA(g), posB(g))
    int64_t total = 0;
    for (auto& rd : reads) total += int64_t(rd.size());
    S->symbols.reserve(size_t(total));
    for (int64_t i = 0; i < n_reads; ++i) {
        S->symbols.insert(S->symbols.end(), reads[size_t(i)].begin(), reads[size_t(i)].end());
        S->offsets.push_back(int64_t(S->symbols.size()));
        std::string().swap(reads[size_t(i)]);
    }
    std::vector<size_t> cursor(static_cast<size_t>(n_reads), 0);
    S->tasks.reserve(seeds.size() * 4);
    for (const Sd& s : seeds) {
        const int64_t pa = seed_pos[size_t(s.a)][cursor[size_t(s.a)]++];
        const int64_t pb = seed_pos[size_t(s.b)][cursor[size_t(s.b)]++];
        S->tasks.push_back(s.a);
        S->tasks.push_back(s.b);
        S->tasks.push_back(pa);
        S->tasks.push_back(pb);
    }
    S->k = k;
    S->x = 15;
    S->band = 256;
}

}  // namespace

namespace {

// The reference's own pair generator (proj/src/io.cpp:198-255), restated:
// H uniform over ACGT from raw mt19937_64 draws, V a copy whose non-seed
// positions change to a strictly different base with probability 1 - p,
// the seed at the centre (or uniform), h_seed = v_seed.  Raw engine draws
// only, so every standard library gives the same bytes.
int make_reference_pairs(xb_synth* S, uint64_t pairs, uint64_t length, double p_match, int k,
                         int uniform, uint64_t seed) {
    if (k < 1 || uint64_t(k) > length) return XB_E_BAD_PARAM;  // io.cpp:199-202 InputError
    static const char kBases[4] = {'A', 'C', 'G', 'T'};
    std::mt19937_64 rng(seed);
    auto draw = [&]() -> uint64_t { return rng(); };
    auto unit_interval = [&]() -> double { return double(draw() >> 11) * 0x1.0p-53; };
    const bool never = p_match >= 1.0, always = p_match <= 0.0;
    S->k = k;
    S->symbols.reserve(size_t(2 * pairs * length));
    for (uint64_t q = 0; q < pairs; ++q) {
        std::string h(size_t(length), 'A');
        for (uint64_t i = 0; i < length; ++i) h[size_t(i)] = kBases[draw() % 4];
        uint64_t pos = (length - uint64_t(k)) / 2;
        if (uniform) pos = draw() % (length - uint64_t(k) + 1);
        std::string v = h;
        for (uint64_t i = 0; i < length; ++i) {
            if (i >= pos && i < pos + uint64_t(k)) continue;
            if (never) continue;
            if (!always && unit_interval() < p_match) continue;
            int cur = 0;
            while (kBases[cur] != v[size_t(i)]) ++cur;
            v[size_t(i)] = kBases[(cur + 1 + int(draw() % 3)) % 4];
        }
        for (const std::string* x : {&h, &v}) {
            S->symbols.insert(S->symbols.end(), x->begin(), x->end());
            S->offsets.push_back(int64_t(S->symbols.size()));
        }
        S->tasks.insert(S->tasks.end(), {int64_t(2 * q), int64_t(2 * q + 1), int64_t(pos), int64_t(pos)});
    }
    return XB_OK;
}

}  // namespace

extern "C" {

xb_synth* xb_synth_make(int cfg, double scale, uint64_t seed, const char* matrix_text, int n_threads,
                        int* err) {
    if (cfg < 1 || cfg > 5 || !(scale > 0)) {
        if (err) *err = XB_E_BAD_PARAM;
        return nullptr;
    }
    const int T = n_threads > 0 ? n_threads : int(std::max(1u, std::thread::hardware_concurrency()));
    if (seed == 0) seed = 20230417ull + uint64_t(cfg);  // SURVEY §8d seeding
    auto* S = new xb_synth();
    int rc = XB_OK;
    if (cfg == 3) {
        if (!matrix_text) rc = XB_E_BAD_PARAM;
        else rc = make_protein(S, scale, seed, matrix_text, T);
    } else if (cfg == 5) {
        make_overlap(S, scale, seed, T);
    } else {
        make_dna_pairs(S, cfg, scale, seed, T);
    }
    if (rc) {
        delete S;
        if (err) *err = rc;
        return nullptr;
    }
    if (err) *err = XB_OK;
    return S;
}

void xb_synth_sizes(const xb_synth* s, int64_t* z) {
    z[0] = int64_t(s->offsets.size()) - 1;
    z[1] = int64_t(s->symbols.size());
    z[2] = int64_t(s->tasks.size() / 4);
    z[3] = s->k;
    z[4] = s->x;
    z[5] = s->band;
}

void xb_synth_copy(const xb_synth* s, char* symbols, int64_t* offsets, int64_t* tasks) {
    if (symbols) std::memcpy(symbols, s->symbols.data(), s->symbols.size());
    if (offsets) std::memcpy(offsets, s->offsets.data(), s->offsets.size() * 8);
    if (tasks) std::memcpy(tasks, s->tasks.data(), s->tasks.size() * 8);
}

xb_synth* xb_synth_pairs(uint64_t pairs, uint64_t length, double p_match, int k, int uniform_seed,
                         uint64_t rng_seed, int* err) {
    auto* S = new xb_synth();
    const int rc = make_reference_pairs(S, pairs, length, p_match, k, uniform_seed, rng_seed);
    if (rc) {
        delete S;
        if (err) *err = rc;
        return nullptr;
    }
    if (err) *err = XB_OK;
    return S;
}

void xb_synth_free(xb_synth* s) { delete s; }

}  // extern "C"
