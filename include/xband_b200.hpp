// Header-only C++ shim: the reference's xband types and calls on top of the
// xdrop_b200 C-ABI, so existing xband callers (proj/src/pipeline.cpp:99-137,
// proj/tests/test_align.cpp) swap only the loop body.  Semantics preserved:
//   * ExtensionTask / ExtensionResult / SeedAlignment field meanings
//     (proj/include/xband/align.hpp:16-51);
//   * extend_seed: the left side's BandExceededError is thrown before the
//     right side's (align.cpp:289-305), with side 'L' / 'R';
//   * batch: both sides always computed, FailedUnit per failing side
//     (pipeline.cpp:115-131), results in task order.
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "xdrop_b200.h"

namespace xband_b200 {

struct InputError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DanglingReference : InputError {
    using InputError::InputError;
};
struct SeedOutOfBounds : InputError {
    using InputError::InputError;
};
struct UnknownSymbol : InputError {
    using InputError::InputError;
};
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct BandExceededError : std::runtime_error {
    BandExceededError(int spread, long long done, char s)
        : std::runtime_error("antidiagonal spread " + std::to_string(spread) +
                             " exceeds allocated band"),
          observed_spread(spread), cells(done), side(s) {}
    int observed_spread;
    long long cells;
    char side;
};

inline void check(int rc, const std::string& what) {
    switch (rc) {
        case XB_OK: return;
        case XB_E_DANGLING: throw DanglingReference(what + ": " + xb_strerror(rc));
        case XB_E_SEED_OOB: throw SeedOutOfBounds(what + ": " + xb_strerror(rc));
        case XB_E_UNKNOWN_SYMBOL: throw UnknownSymbol(what + ": " + xb_strerror(rc));
        case XB_E_BAD_PARAM:
        case XB_E_PARSE:
        case XB_E_OUT_OF_RANGE: throw InputError(what + ": " + xb_strerror(rc));
        default: throw DeviceError(what + ": " + xb_strerror(rc));
    }
}

struct ExtensionTask {
    int task_id = 0;
    uint32_t h_id = 0, v_id = 0;
    size_t h_seed = 0, v_seed = 0;
};

struct ExtensionResult {
    int score = 0;
    int h_ext = 0;
    int v_ext = 0;
    long long cells = 0;
    int delta_w = 0;
    bool operator==(const ExtensionResult&) const = default;
};

struct SeedAlignment {
    int task_id = 0;
    ExtensionResult left, right;
    int seed_score = 0;
    int total = 0;
};

struct FailedUnit {
    int task_id = 0;
    char side = '?';
    int observed_spread = 0;
};

// ScoringScheme (scoring.hpp:28-54)
class ScoringScheme {
public:
    static ScoringScheme match_mismatch(int match, int mismatch, int gap, int x) {
        int err = 0;
        xb_scheme* s = xb_scheme_match_mismatch(match, mismatch, gap, x, &err);
        check(err, "match_mismatch");
        return ScoringScheme(s);
    }
    static ScoringScheme from_matrix(const std::string& alphabet, const std::vector<int>& cells,
                                     int gap, int x) {
        int err = 0;
        xb_scheme* s = xb_scheme_from_matrix(alphabet.data(), int(alphabet.size()), cells.data(),
                                             gap, x, &err);
        check(err, "from_matrix");
        return ScoringScheme(s);
    }
    ScoringScheme(ScoringScheme&& o) noexcept : s_(o.s_) { o.s_ = nullptr; }
    ScoringScheme(const ScoringScheme&) = delete;
    ~ScoringScheme() { xb_scheme_free(s_); }
    int sim(char a, char b) const {
        int v = 0;
        check(xb_scheme_sim(s_, a, b, &v), "sim");
        return v;
    }
    const xb_scheme* get() const { return s_; }

private:
    explicit ScoringScheme(xb_scheme* s) : s_(s) {}
    xb_scheme* s_;
};

// The detached pool (SequenceStore, sequence.hpp:13-19), packed and
// uploaded once per device on first use.
class SequencePool {
public:
    explicit SequencePool(const ScoringScheme& s) {
        int err = 0;
        p_ = xb_pool_create(s.get(), &err);
        check(err, "pool");
    }
    SequencePool(const SequencePool&) = delete;
    ~SequencePool() { xb_pool_free(p_); }
    uint32_t add(const std::string& symbols) {
        const int64_t id = xb_pool_add(p_, symbols.data(), int64_t(symbols.size()));
        if (id < 0) check(int(-id), "pool add");
        return uint32_t(id);
    }
    size_t size() const { return size_t(xb_pool_size(p_)); }
    xb_pool* get() const { return p_; }

private:
    xb_pool* p_;
};

inline ExtensionResult to_result(const xb_side_result& r) {
    return ExtensionResult{r.score, r.h_ext, r.v_ext, r.cells, r.delta_w};
}

// The batch loop of pipeline.cpp:103-136 in one call.
inline void extend_batch(SequencePool& pool, const std::vector<ExtensionTask>& tasks, int k,
                         int band, std::vector<SeedAlignment>& done,
                         std::vector<FailedUnit>& failed, std::vector<long long>* unit_cells = nullptr,
                         const xb_exec* exec = nullptr) {
    std::vector<xb_task> t(tasks.size());
    for (size_t q = 0; q < tasks.size(); ++q)
        t[q] = xb_task{tasks[q].task_id, tasks[q].h_id, tasks[q].v_id, tasks[q].h_seed, tasks[q].v_seed};
    std::vector<xb_side_result> out(2 * tasks.size());
    std::vector<int32_t> ss(tasks.size());
    int64_t bad = -1;
    check(xb_extend_batch(pool.get(), t.data(), int64_t(t.size()), k, band, out.data(), ss.data(),
                          &bad, exec),
          "extend_batch");
    if (unit_cells) unit_cells->assign(2 * tasks.size(), 0);
    for (size_t q = 0; q < tasks.size(); ++q) {
        bool ok = true;
        for (int s = 0; s < 2; ++s) {
            const xb_side_result& r = out[2 * q + size_t(s)];
            if (unit_cells) (*unit_cells)[2 * q + size_t(s)] = r.cells;
            if (r.status == XB_SIDE_BAND_EXCEEDED) {
                failed.push_back({tasks[q].task_id, s ? 'R' : 'L', r.spread});
                ok = false;
            }
        }
        if (ok) {
            SeedAlignment a;
            a.task_id = tasks[q].task_id;
            a.left = to_result(out[2 * q]);
            a.right = to_result(out[2 * q + 1]);
            a.seed_score = ss[q];
            a.total = a.left.score + a.seed_score + a.right.score;
            done.push_back(a);
        }
    }
}

// extend_seed (align.cpp:268-309) for one task.
inline SeedAlignment extend_seed(SequencePool& pool, const ExtensionTask& task, int k, int band) {
    xb_task t{task.task_id, task.h_id, task.v_id, task.h_seed, task.v_seed};
    xb_side_result out[2];
    int32_t ss = 0;
    check(xb_extend_batch(pool.get(), &t, 1, k, band, out, &ss, nullptr, nullptr), "extend_seed");
    for (int s = 0; s < 2; ++s)
        if (out[s].status == XB_SIDE_BAND_EXCEEDED)
            throw BandExceededError(out[s].spread, out[s].cells, s ? 'R' : 'L');
    SeedAlignment a;
    a.task_id = task.task_id;
    a.left = to_result(out[0]);
    a.right = to_result(out[1]);
    a.seed_score = ss;
    a.total = a.left.score + ss + a.right.score;
    return a;
}

// sweep_band (pipeline.hpp:58, pipeline.cpp:181-208): the band survey TSV.
inline std::string sweep_band(size_t length, const std::vector<int>& xs,
                              const std::vector<double>& p_grid, uint64_t rng_seed,
                              const xb_exec* exec = nullptr) {
    std::vector<int32_t> dw(xs.size() * p_grid.size());
    std::vector<int32_t> x32(xs.begin(), xs.end());
    check(xb_sweep_band(length, x32.data(), int32_t(xs.size()), p_grid.data(), int32_t(p_grid.size()),
                        rng_seed, dw.data(), exec),
          "sweep_band");
    std::string out = "x\terror_rate\tdelta_w\n";
    char buf[64];
    for (size_t a = 0; a < xs.size(); ++a)
        for (size_t b = 0; b < p_grid.size(); ++b) {
            std::snprintf(buf, sizeof buf, "%d\t%.2f\t%d\n", xs[a], 1.0 - p_grid[b],
                          dw[a * p_grid.size() + b]);
            out += buf;
        }
    return out;
}

}  // namespace xband_b200
