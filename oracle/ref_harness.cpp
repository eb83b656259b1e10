/*
 * TEST INFRASTRUCTURE ONLY -- a C shim over the UNMODIFIED reference library.
 *
 * oracle/Makefile compiles the reference sources where they lie
 * (/root/reference/proj/src/*.cpp, nothing copied) together with this file
 * into oracle/_ref/libxband_ref.so.  It exists to
 *   (1) pin the C oracle (oracle/xdrop_oracle.c) against the real thing,
 *   (2) generate tests/golden/ fixtures, and
 *   (3) time the reference CPU path on the GPU box's host cores (bench.py
 *       cpu_baseline leg and `bench.py --impl reference`).
 * The batch entry point follows the reference batch loop
 * (proj/src/pipeline.cpp:103-136): split_lr, checked seed score, then both
 * sides through xdrop_extend with one BandBuffers scratch per thread, which
 * the reference declares re-entrant (proj/include/xband/align.hpp:53-56).
 */
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "xband/align.hpp"
#include "xband/errors.hpp"
#include "xband/io.hpp"
#include "xband/partition.hpp"
#include "xband/pipeline.hpp"
#include "xband/scoring.hpp"

using namespace xband;

namespace {
struct RefResult {  // same layout as xo_result / xb_side_result
    int32_t score, h_ext, v_ext, delta_w;
    int64_t cells;
    int32_t status, spread;
};
void fill(RefResult* o, const ExtensionResult& r) {
    o->score = r.score;
    o->h_ext = r.h_ext;
    o->v_ext = r.v_ext;
    o->delta_w = r.delta_w;
    o->cells = r.cells;
    o->status = 0;
    o->spread = 0;
}
void fill_fail(RefResult* o, const BandExceededError& e) {
    std::memset(o, 0, sizeof *o);
    o->cells = e.cells;
    o->status = 1;
    o->spread = e.observed_spread;
}
}  // namespace

extern "C" {

void* ref_scheme_mm(int match, int mismatch, int gap, int x) {
    try {
        return new ScoringScheme(ScoringScheme::match_mismatch(match, mismatch, gap, x));
    } catch (...) {
        return nullptr;
    }
}

void* ref_scheme_matrix(const char* text, int gap, int x) {
    try {
        return new ScoringScheme(ScoringScheme::from_matrix(parse_submatrix(text), gap, x));
    } catch (...) {
        return nullptr;
    }
}

void ref_scheme_free(void* s) { delete static_cast<ScoringScheme*>(s); }

/* matrix as parsed by the reference: alphabet into `alpha` (n+1 bytes),
 * n*n cells row-major into `cells`; returns n or -1 */
int ref_parse_matrix(const char* text, char* alpha, int cap, int* cells) {
    try {
        SubMatrix m = parse_submatrix(text);
        int n = (int)m.alphabet.size();
        if (n * n > cap) return -1;
        std::memcpy(alpha, m.alphabet.data(), size_t(n));
        alpha[n] = 0;
        for (int i = 0; i < n * n; ++i) cells[i] = m.cells[size_t(i)];
        return n;
    } catch (...) {
        return -1;
    }
}

int ref_sim(const void* s, char a, char b, int* out) {
    try {
        *out = sim(*static_cast<const ScoringScheme*>(s), a, b);
        return 0;
    } catch (...) {
        return -1;
    }
}

/* One kernel call on views into two standalone sequences. dir: 1 Right, 0 Left.
 * Returns 0 ok, 1 band exceeded (payload in out), 2 input error. */
int ref_xdrop_extend(const char* hs, int64_t hn, int64_t h_origin, int h_dir, int64_t h_len,
                     const char* vs, int64_t vn, int64_t v_origin, int v_dir, int64_t v_len,
                     const void* scheme, int band, RefResult* out) {
    Sequence H{0, "h", std::string(hs, size_t(hn))};
    Sequence V{1, "v", std::string(vs, size_t(vn))};
    try {
        SeqView hv = make_view(H, size_t(h_origin), h_dir ? Dir::Right : Dir::Left, size_t(h_len));
        SeqView vv = make_view(V, size_t(v_origin), v_dir ? Dir::Right : Dir::Left, size_t(v_len));
        fill(out, xdrop_extend(hv, vv, *static_cast<const ScoringScheme*>(scheme), band));
        return 0;
    } catch (const BandExceededError& e) {
        fill_fail(out, e);
        return 1;
    } catch (...) {
        return 2;
    }
}

int ref_full_oracle(const char* hs, int64_t hn, const char* vs, int64_t vn, const void* scheme,
                    RefResult* out) {
    Sequence H{0, "h", std::string(hs, size_t(hn))};
    Sequence V{1, "v", std::string(vs, size_t(vn))};
    SeqView hv = make_view(H, 0, Dir::Right, size_t(hn));
    SeqView vv = make_view(V, 0, Dir::Right, size_t(vn));
    fill(out, xdrop_full_oracle(hv, vv, *static_cast<const ScoringScheme*>(scheme)));
    return 0;
}

/* extend_seed on a two-sequence store; returns 0 ok, 1 band exceeded
 * (side in *side), 2 dangling, 3 seed out of bounds, 4 other input error */
int ref_extend_seed(const char* hs, int64_t hn, const char* vs, int64_t vn, int64_t h_seed,
                    int64_t v_seed, int h_id, int v_id, int k, const void* scheme, int band,
                    RefResult* left, RefResult* right, int32_t* seed_score, int32_t* total,
                    char* side, int32_t* spread) {
    SequenceStore store;
    store.push_back(Sequence{0, "h", std::string(hs, size_t(hn))});
    store.push_back(Sequence{1, "v", std::string(vs, size_t(vn))});
    ExtensionTask t{0, uint32_t(h_id), uint32_t(v_id), size_t(h_seed), size_t(v_seed)};
    try {
        SeedAlignment a =
            extend_seed(t, store, k, *static_cast<const ScoringScheme*>(scheme), band);
        fill(left, a.left);
        fill(right, a.right);
        *seed_score = a.seed_score;
        *total = a.total;
        return 0;
    } catch (const BandExceededError& e) {
        *side = e.side;
        *spread = e.observed_spread;
        return 1;
    } catch (const DanglingReference&) {
        return 2;
    } catch (const SeedOutOfBounds&) {
        return 3;
    } catch (...) {
        return 4;
    }
}

/* ---- pool + multi-threaded batch (the CPU baseline) ---- */

void* ref_pool_create(const char* concat, const int64_t* off, int64_t n) {
    auto* st = new SequenceStore();
    st->reserve(size_t(n));
    for (int64_t i = 0; i < n; ++i)
        st->push_back(Sequence{uint32_t(i), "s", std::string(concat + off[i], size_t(off[i + 1] - off[i]))});
    return st;
}

void ref_pool_free(void* p) { delete static_cast<SequenceStore*>(p); }

/* tasks: n x {h_id, v_id, h_seed, v_seed}; out: 2n (L, R); order: optional
 * processing order (e.g. cost-sorted), results still land at task index.
 * Returns 0, or 2/3/4 on the first input error (task index in *bad). */
int ref_extend_batch(const void* pool, const void* scheme, const int64_t* tasks, int64_t n,
                     const int64_t* order, int k, int band, int n_threads, RefResult* out,
                     int32_t* seed_score, int64_t* bad) {
    const SequenceStore& store = *static_cast<const SequenceStore*>(pool);
    const ScoringScheme& sc = *static_cast<const ScoringScheme*>(scheme);
    std::atomic<int64_t> next{0};
    std::atomic<int> err{0};
    std::atomic<int64_t> err_task{-1};
    auto worker = [&]() {
        BandBuffers scratch(band);
        for (;;) {
            int64_t q0 = next.fetch_add(16);
            if (q0 >= n || err.load()) return;
            int64_t q1 = std::min<int64_t>(n, q0 + 16);
            for (int64_t q = q0; q < q1; ++q) {
                int64_t ti = order ? order[q] : q;
                const int64_t* tq = tasks + 4 * ti;
                ExtensionTask t{int(ti), uint32_t(tq[0]), uint32_t(tq[1]), size_t(tq[2]),
                                size_t(tq[3])};
                try {
                    auto [l, r] = split_lr(t, store, k);
                    const Sequence& hs = store[t.h_id];
                    const Sequence& vs = store[t.v_id];
                    int32_t ss = 0;
                    for (int i = 0; i < k; ++i)
                        ss += sim(sc, hs.symbols[t.h_seed + size_t(i)],
                                  vs.symbols[t.v_seed + size_t(i)]);
                    seed_score[ti] = ss;
                    for (const WorkUnit* u : {&l, &r}) {
                        const Dir dir = (u->side == Side::L) ? Dir::Left : Dir::Right;
                        SeqView hv = make_view(hs, u->h_origin, dir, u->h_len);
                        SeqView vv = make_view(vs, u->v_origin, dir, u->v_len);
                        RefResult* o = &out[2 * ti + (u->side == Side::L ? 0 : 1)];
                        try {
                            fill(o, xdrop_extend(hv, vv, sc, band, &scratch));
                        } catch (const BandExceededError& e) {
                            fill_fail(o, e);
                        }
                    }
                } catch (const DanglingReference&) {
                    err = 2;
                    err_task = ti;
                } catch (const SeedOutOfBounds&) {
                    err = 3;
                    err_task = ti;
                } catch (...) {
                    err = 4;
                    err_task = ti;
                }
            }
        }
    };
    if (n_threads <= 1) {
        worker();
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < n_threads; ++i) th.emplace_back(worker);
        for (auto& t : th) t.join();
    }
    if (bad) *bad = err_task.load();
    return err.load();
}

/* run_pipeline on the reference's own synthetic generator; writes the
 * results text (truncated to cap) and returns its length, or -1. */
int64_t ref_pipeline_synth(int64_t pairs, int64_t length, double p_match, int x, int band,
                           int k, uint64_t seed, int uniform_seed, char* buf, int64_t cap,
                           int* exit_code) {
    RunConfig cfg;
    cfg.use_synth = true;
    cfg.synth.pairs = size_t(pairs);
    cfg.synth.length = size_t(length);
    cfg.synth.p_match = p_match;
    cfg.synth.k = k;
    cfg.synth.rng_seed = seed;
    cfg.synth.placement = uniform_seed ? SeedPlacement::UniformRandom : SeedPlacement::Center;
    cfg.k = k;
    cfg.x = x;
    cfg.band = band;
    std::ostringstream log;
    PipelineResult r = run_pipeline(cfg, log);
    *exit_code = r.exit_code;
    int64_t len = int64_t(r.results_text.size());
    std::memcpy(buf, r.results_text.data(), size_t(std::min(len, cap)));
    return len;
}

/* the reference's own synthetic dataset, for the pipeline drop-in check */
int64_t ref_generate_synthetic(int64_t pairs, int64_t length, double p_match, int k,
                               uint64_t seed, int uniform_seed, char* symbols, int64_t* off,
                               int64_t* tasks) {
    SynthParams sp;
    sp.pairs = size_t(pairs);
    sp.length = size_t(length);
    sp.p_match = p_match;
    sp.k = k;
    sp.rng_seed = seed;
    sp.placement = uniform_seed ? SeedPlacement::UniformRandom : SeedPlacement::Center;
    Dataset ds = generate_synthetic(sp);
    int64_t pos = 0;
    for (size_t i = 0; i < ds.store.size(); ++i) {
        off[i] = pos;
        std::memcpy(symbols + pos, ds.store[i].symbols.data(), ds.store[i].symbols.size());
        pos += int64_t(ds.store[i].symbols.size());
    }
    off[ds.store.size()] = pos;
    for (size_t t = 0; t < ds.tasks.size(); ++t) {
        tasks[4 * t + 0] = ds.tasks[t].h_id;
        tasks[4 * t + 1] = ds.tasks[t].v_id;
        tasks[4 * t + 2] = int64_t(ds.tasks[t].h_seed);
        tasks[4 * t + 3] = int64_t(ds.tasks[t].v_seed);
    }
    return int64_t(ds.tasks.size());
}

/* the reference's band survey (pipeline.cpp:181-208): TSV x / error_rate / delta_w */
int64_t ref_sweep_band(int64_t length, const int* xs, int nx, const double* ps, int np,
                       uint64_t seed, char* buf, int64_t cap) {
    std::vector<int> xv(xs, xs + nx);
    std::vector<double> pv(ps, ps + np);
    const std::string t = sweep_band(size_t(length), xv, pv, seed);
    const int64_t len = int64_t(t.size());
    if (buf) std::memcpy(buf, t.data(), size_t(std::min(len, cap)));
    return len;
}

/* the reference's parsers (io.cpp:58-196), for the ingest parity tests:
 * kind codes as XB_PARSE_* in include/xdrop_b200.h */
static int parse_kind(const std::exception& e, int64_t* line) {
    *line = 0;
    if (auto* x = dynamic_cast<const InvalidSymbol*>(&e)) { *line = int64_t(x->line); return 3; }
    if (auto* x = dynamic_cast<const MalformedLine*>(&e)) { *line = int64_t(x->line); return 4; }
    if (dynamic_cast<const MissingHeader*>(&e)) return 1;
    if (dynamic_cast<const EmptyRecord*>(&e)) return 2;
    if (dynamic_cast<const NegativeIndex*>(&e)) return 5;
    if (dynamic_cast<const BadHeader*>(&e)) return 6;
    if (dynamic_cast<const IndexOutOfDeclaredShape*>(&e)) return 7;
    return 99;
}

static void put_msg(const std::exception& e, char* msg, int64_t cap) {
    const std::string m = e.what();
    const size_t n = std::min<size_t>(m.size(), size_t(cap) - 1);
    std::memcpy(msg, m.data(), n);
    msg[n] = 0;
}

/* returns records (sym/off/names/name_off filled; buffers sized by the
 * caller from len) or -1 with kind/line/msg */
int64_t ref_parse_fasta(const char* text, int64_t len, const char* allowed, char* sym, int64_t* off,
                        char* names, int64_t* name_off, int* kind, int64_t* line, char* msg) {
    try {
        SequenceStore st = parse_fasta(std::string(text, size_t(len)), std::string(allowed));
        int64_t a = 0, b = 0;
        off[0] = 0;
        name_off[0] = 0;
        for (size_t i = 0; i < st.size(); ++i) {
            std::memcpy(sym + a, st[i].symbols.data(), st[i].symbols.size());
            a += int64_t(st[i].symbols.size());
            off[i + 1] = a;
            std::memcpy(names + b, st[i].name.data(), st[i].name.size());
            b += int64_t(st[i].name.size());
            name_off[i + 1] = b;
        }
        *kind = 0;
        return int64_t(st.size());
    } catch (const std::exception& e) {
        *kind = parse_kind(e, line);
        put_msg(e, msg, 256);
        return -1;
    }
}

/* which = 0 seeds, 1 overlaps; tasks: 5 int64 per task (task_id, h, v, hs, vs) */
int64_t ref_parse_tasks(int which, const char* text, int64_t len, int64_t* tasks, int64_t cap,
                        int* kind, int64_t* line, char* msg) {
    try {
        const std::string t(text, size_t(len));
        std::vector<ExtensionTask> v = which ? parse_overlaps(t) : parse_seeds(t);
        for (size_t i = 0; i < v.size() && int64_t(i) < cap; ++i) {
            tasks[5 * i + 0] = v[i].task_id;
            tasks[5 * i + 1] = v[i].h_id;
            tasks[5 * i + 2] = v[i].v_id;
            tasks[5 * i + 3] = int64_t(v[i].h_seed);
            tasks[5 * i + 4] = int64_t(v[i].v_seed);
        }
        *kind = 0;
        return int64_t(v.size());
    } catch (const std::exception& e) {
        *kind = parse_kind(e, line);
        put_msg(e, msg, 256);
        return -1;
    }
}

}  // extern "C"
