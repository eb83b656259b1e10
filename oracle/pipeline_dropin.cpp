// TEST INFRASTRUCTURE ONLY -- the drop-in check of SURVEY §8(f) item 1.
//
// The reference's end-to-end run (run_pipeline, proj/src/pipeline.cpp:56-179)
// with its kernel loop (pipeline.cpp:99-137: split_lr, checked seed score,
// xdrop_extend per side, unit_cells, FailedUnit) replaced by ONE batch call
// of the product (xband_b200::extend_batch over the xdrop_b200 C-ABI, i.e.
// the sm_100a kernels).  Everything around the loop is the reference's own
// code, compiled from /root/reference/proj/src by oracle/Makefile:
// generate_synthetic (io.cpp:198-256), the partitions and batches
// (partition.cpp), the measured-cost replay on the IPU simulator
// (run_devices, bsp.cpp:142-171, fed the product's per-unit cells) and
// write_results (io.cpp:258-298).  The results text -- rows, '# total', and
// the summary block built from the replay -- must be byte-identical to the
// reference's own run_pipeline (tests/test_pipeline_dropin.py: SHA-256 of
// Appendix B and acceptance criterion 9).
//
// Built into oracle/_ref/libxband_dropin.so (it needs the reference sources,
// so it is built in the dev container and travels prebuilt).
#include <cstdint>
#include <cstring>
#include <sstream>
#include <unordered_map>
#include <vector>

#include "../include/xband_b200.hpp"
#include "xband/align.hpp"
#include "xband/bsp.hpp"
#include "xband/io.hpp"
#include "xband/partition.hpp"
#include "xband/pipeline.hpp"
#include "xband/scoring.hpp"

namespace {

struct DropinConfig {
    int64_t pairs, length;
    double p_match;
    int32_t k, uniform_seed;
    uint64_t seed;
    int32_t x, band, tiles, devices, multicomparison, work_steal;
};

xband::RunConfig to_run_config(const DropinConfig& c) {
    xband::RunConfig cfg;
    cfg.use_synth = true;
    cfg.synth.pairs = size_t(c.pairs);
    cfg.synth.length = size_t(c.length);
    cfg.synth.p_match = c.p_match;
    cfg.synth.k = c.k;
    cfg.synth.rng_seed = c.seed;
    cfg.synth.placement = c.uniform_seed ? xband::SeedPlacement::UniformRandom : xband::SeedPlacement::Center;
    cfg.k = c.k;
    cfg.x = c.x;
    cfg.band = c.band;
    cfg.tiles = c.tiles;
    cfg.devices = c.devices;
    cfg.multicomparison = c.multicomparison != 0;
    cfg.policy = c.work_steal ? xband::Policy::WorkSteal : xband::Policy::StaticRoundRobin;
    return cfg;
}

int64_t emit(const std::string& text, char* buf, int64_t cap) {
    const int64_t len = int64_t(text.size());
    if (buf && cap > 0) std::memcpy(buf, text.data(), size_t(std::min(len, cap)));
    return len;
}

}  // namespace

extern "C" {

// The reference pipeline itself, unmodified (the expected bytes).
int64_t dropin_reference(const DropinConfig* c, char* buf, int64_t cap, int* exit_code) {
    std::ostringstream log;
    xband::PipelineResult r = xband::run_pipeline(to_run_config(*c), log);
    *exit_code = r.exit_code;
    return emit(r.results_text, buf, cap);
}

// The same run with the kernel loop swapped for the product's batch call.
int64_t dropin_product(const DropinConfig* c, char* buf, int64_t cap, int* exit_code) {
    const xband::RunConfig cfg = to_run_config(*c);
    // the pieces of run_pipeline ahead of the loop (pipeline.cpp:59-72)
    const xband::ScoringScheme scheme =
        xband::ScoringScheme::match_mismatch(cfg.match, cfg.mismatch, cfg.gap, cfg.x);
    const xband::Dataset ds = xband::generate_synthetic(cfg.synth);
    const xband::TileBudget budget = xband::TileBudget::make(cfg.band, cfg.workers, cfg.tile_memory);
    std::vector<xband::Partition> parts =
        cfg.multicomparison ? xband::greedy_partition(xband::build_graph(ds.tasks, ds.store), budget)
                            : xband::singleton_partitions(ds.tasks, ds.store, budget);
    xband::attach_units(parts, ds.tasks, ds.store, ds.k);
    std::vector<xband::Batch> batches = xband::schedule_batches(parts, cfg.tiles, budget);

    // ---- the replaced loop: one batch through the C-ABI ----
    xband_b200::ScoringScheme ours =
        xband_b200::ScoringScheme::match_mismatch(cfg.match, cfg.mismatch, cfg.gap, cfg.x);
    xband_b200::SequencePool pool(ours);
    for (const xband::Sequence& s : ds.store) pool.add(s.symbols);
    std::vector<xband_b200::ExtensionTask> tasks;
    tasks.reserve(ds.tasks.size());
    for (const xband::ExtensionTask& t : ds.tasks)
        tasks.push_back({t.task_id, t.h_id, t.v_id, t.h_seed, t.v_seed});
    std::vector<xband_b200::SeedAlignment> done;
    std::vector<xband_b200::FailedUnit> failed;
    std::vector<long long> cells;  // [2q + side]
    xband_b200::extend_batch(pool, tasks, ds.k, cfg.band, done, failed, &cells);

    xband::PipelineResult res;
    std::unordered_map<int, long long> unit_cells;  // unit_id = 2 task_id + side (split_lr)
    for (size_t q = 0; q < tasks.size(); ++q)
        for (int s = 0; s < 2; ++s) unit_cells[2 * tasks[q].task_id + s] = cells[2 * q + size_t(s)];
    for (const auto& a : done) {
        xband::SeedAlignment b;
        b.task_id = a.task_id;
        b.left = {a.left.score, a.left.h_ext, a.left.v_ext, a.left.cells, a.left.delta_w};
        b.right = {a.right.score, a.right.h_ext, a.right.v_ext, a.right.cells, a.right.delta_w};
        b.seed_score = a.seed_score;
        b.total = a.total;
        res.alignments.push_back(b);
    }
    for (const auto& f : failed) res.failed.push_back({f.task_id, f.side, f.observed_spread});

    // ---- after the loop: the reference's replay and results text ----
    xband::CostModel model;
    model.mode = xband::CostModel::Mode::Measured;
    model.frequency = cfg.frequency;
    model.unit_cells = &unit_cells;
    model.store = &ds.store;
    model.scheme = &scheme;
    model.band = cfg.band;
    res.sim = xband::run_devices(batches, parts, cfg.devices, cfg.policy, model, cfg.workers);
    res.summary.wall_cost = res.sim.wall_cost;
    res.summary.wall_seconds = xband::time_from_cost(res.sim.wall_cost, cfg.frequency);
    res.summary.batch_count = batches.size();
    res.summary.transmitted_bytes = res.sim.transmitted_bytes;
    res.summary.transmitted_seqs = res.sim.transmitted_seqs;
    res.summary.failed_units = res.failed.size();
    for (const auto& kv : unit_cells) res.summary.total_cells += kv.second;
    if (res.summary.wall_seconds > 0.0) {
        double products = 0.0;
        for (const xband::ExtensionTask& t : ds.tasks)
            products += double(ds.store[t.h_id].symbols.size()) * double(ds.store[t.v_id].symbols.size());
        res.summary.gcups = xband::gcups(products, 1.0, res.summary.wall_seconds);
    }
    res.results_text = xband::write_results(res.alignments, res.failed, res.summary);
    *exit_code = res.failed.empty() ? 0 : 3;
    return emit(res.results_text, buf, cap);
}

}  // extern "C"
