/*
 * xdrop_b200 -- C-ABI for the B200-native X-drop seed-extension batch.
 *
 * This is the drop-in boundary for the reference's batch path (xband,
 * /root/reference/proj).  The reference is a C++ library with no FFI; its
 * callers run the loop at proj/src/pipeline.cpp:103-136 over
 * xband::extend_seed-style calls.  Each entry point below names the
 * reference interface it replaces.  Plain pointers and sizes only -- no
 * torch or CUDA types cross this boundary (a cudaStream_t may be passed as
 * an opaque void* in xb_exec).
 *
 * Error model (mirrors proj/include/xband/errors.hpp): calls return XB_OK or
 * an XB_E_* code; BandExceededError becomes a per-side status
 * (XB_SIDE_BAND_EXCEEDED) carrying observed_spread and cells, exactly as the
 * pipeline records FailedUnit (pipeline.cpp:124-130).
 */
#ifndef XDROP_B200_H
#define XDROP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes (errors.hpp:14-93) ---- */
#define XB_OK 0
#define XB_E_BAD_PARAM 1       /* InputError: band < 1, k < 0, bad scheme (scoring.cpp:17-20,37-40) */
#define XB_E_DANGLING 2        /* DanglingReference (align.cpp:271-273) */
#define XB_E_SEED_OOB 3        /* SeedOutOfBounds (align.cpp:276-279) */
#define XB_E_UNKNOWN_SYMBOL 4  /* UnknownSymbol (scoring.cpp:55-59, io.cpp ingestion) */
#define XB_E_OUT_OF_RANGE 5    /* OutOfRange from make_view (sequence.cpp:5-15) */
#define XB_E_CUDA 6            /* device failure (no reference analogue) */
#define XB_E_NO_DEVICE 7       /* no CUDA device visible: the product never falls back to CPU */
#define XB_E_PARSE 8           /* NonSquare / MissingEntry / header errors of parse_submatrix */

/* ---- per-side status ---- */
#define XB_SIDE_OK 0
#define XB_SIDE_BAND_EXCEEDED 1 /* BandExceededError: spread + cells set, score fields 0 */

/* ExtensionTask (align.hpp:16-20): same field order and widths. */
typedef struct {
    int32_t task_id;
    uint32_t h_id, v_id;
    uint64_t h_seed, v_seed;
} xb_task;

/* ExtensionResult (align.hpp:37-45) + BandExceededError payload
 * (errors.hpp:85-93).  32 bytes. */
typedef struct {
    int32_t score;
    int32_t h_ext;
    int32_t v_ext;
    int32_t delta_w;
    int64_t cells;
    int32_t status; /* XB_SIDE_* */
    int32_t spread; /* observed_spread when status == XB_SIDE_BAND_EXCEEDED */
} xb_side_result;

/* One explicit extension (a WorkUnit, partition.hpp:54-62, or the two
 * SeqViews handed to xdrop_extend, align.hpp:57-59).  dir: 0 Left (element
 * i = symbols[origin-1-i]), 1 Right (element i = symbols[origin+i]),
 * sequence.hpp:35-38. */
typedef struct {
    uint32_t h_id, v_id;
    int32_t h_dir, v_dir;
    uint64_t h_origin, v_origin;
    uint64_t h_len, v_len;
} xb_unit;

/* Execution options.  NULL means: device 0, internal stream. */
typedef struct {
    int32_t n_devices;         /* 0 or 1 = single device */
    const int32_t* device_ids; /* n_devices ids; NULL = 0..n_devices-1 */
    void* stream;              /* cudaStream_t for single-device calls, or NULL */
    int32_t flags;             /* XB_FLAG_* */
} xb_exec;

#define XB_FLAG_NO_SORT 1       /* skip the longest-first cost sort (ablation) */
#define XB_FLAG_GENERIC_ONLY 2  /* route every unit to the warp tier (testing) */
#define XB_FLAG_FORCE_TIER 8    /* start at tier (flags >> 8) & 15, no pilot (testing) */
#define XB_FLAG_ESC_TO_WARP 16  /* units outgrowing the start tier go straight to the warp tier */
#define XB_FLAG_GROUP 32        /* every thread-tier launch runs as lane groups (testing) */
#define XB_FLAG_NO_GROUP 64     /* never use lane groups: one thread per unit throughout (ablation) */
#define XB_FLAG_THROUGHPUT 128  /* plan a small batch like a large one: pilot + cost model (testing) */
#define XB_FLAG_SERIAL_TAIL 4096 /* wider tiers only after the start tier (no concurrent escalation consumer; ablation) */
#define XB_FLAG_LOCALITY 8192   /* multi-device batches: locality-aware shards (xb_shard_tasks XB_SHARD_LOCALITY) */
#define XB_FLAG_LANES 16384     /* several-lanes-per-unit launches of the narrow tiers use the lane tiers (8 lanes per unit; testing) */
#define XB_FLAG_NO_LANES 32768  /* ... never the lane tiers: the 4-lane groups (testing) */

/* Per-call device statistics (summed over devices; times are the max).
 * Tiers: 0..4 = one unit per thread (or per 4-lane group) with a
 * K = 16/24/32/48/64 slot register band; 5..9 = 8-32 lanes per unit with a
 * K = 96/128/256/512/1024 slot register band; 10 = one warp per unit, rows
 * in global memory (exact generic path, any band).  Tiers after the start
 * tier are dispatched on the device; their time is reported as tier 10's. */
#define XB_NUM_TIERS 11
typedef struct {
    int32_t n_devices;
    int32_t launches;            /* kernels launched by the last run */
    double ms_total;             /* device time of the whole run */
    double ms_prep;              /* LR split + seed scores + cost sort */
    double ms_pilot;             /* pilot sample + start-tier choice */
    double ms_tier[XB_NUM_TIERS];
    int64_t units_tier[XB_NUM_TIERS];  /* units finished per tier */
    int64_t cells_tier[XB_NUM_TIERS];  /* sum of ExtensionResult.cells finished per tier */
    int64_t escalated[XB_NUM_TIERS];   /* units handed from tier t to tier t+1 */
    int64_t h2d_bytes, d2h_bytes;
    int32_t sm_count;
    int32_t start_tier;          /* tier the pilot chose */
    int64_t dbg[6];              /* [0..4] instrumented builds only (-DXB_COUNTERS=1), else 0;
                                    [5] units a lane-group tier resumed at an even antidiagonal */
    int32_t start_lane_groups;   /* latency-bound batch: the start tier ran as 4-lane groups (1) or on the lane tiers (2) */
    int32_t reserved;
} xb_stats;

typedef struct xb_scheme xb_scheme;
typedef struct xb_pool xb_pool;
typedef struct xb_batch xb_batch;

const char* xb_version(void);
const char* xb_strerror(int code);
/* number of visible CUDA devices (0 on a CPU-only host) */
int xb_device_count(void);

/* ---- scoring (scoring.hpp:30-56) ---- */
/* ScoringScheme::match_mismatch (scoring.cpp:16-34): alphabet ACGTN, N never matches. */
xb_scheme* xb_scheme_match_mismatch(int match, int mismatch, int gap, int x, int* err);
/* ScoringScheme::from_matrix (scoring.cpp:36-53): n <= 31 symbols. */
xb_scheme* xb_scheme_from_matrix(const char* alphabet, int n, const int* cells, int gap, int x,
                                 int* err);
/* parse_submatrix (scoring.cpp:61-105): NCBI text -> alphabet + n*n cells; returns n or -XB_E_*. */
int xb_parse_submatrix(const char* text, char* alphabet_out, int alphabet_cap, int* cells_out,
                       int cells_cap);
/* checked sim (scoring.cpp:55-59) */
int xb_scheme_sim(const xb_scheme* s, char a, char b, int* out);
void xb_scheme_free(xb_scheme* s);

/* ---- detached sequence pool (SequenceStore, sequence.hpp:13-19) ---- */
/* Symbols are validated against the scheme alphabet and packed: 2 bits per
 * base when every sequence is pure ACGT, else one byte (alphabet code) per symbol. */
xb_pool* xb_pool_create(const xb_scheme* s, int* err);
/* returns the new dense id (>= 0) or -XB_E_* */
int64_t xb_pool_add(xb_pool* p, const char* symbols, int64_t len);
/* bulk add: concat holds n sequences, offsets has n+1 entries; returns first id or -XB_E_* */
int64_t xb_pool_add_bulk(xb_pool* p, const char* concat, const int64_t* offsets, int64_t n);
int64_t xb_pool_size(const xb_pool* p);
int64_t xb_pool_seq_len(const xb_pool* p, int64_t id);
int xb_pool_bits_per_symbol(const xb_pool* p);
/* drop device copies (the next call re-uploads; used to time end-to-end runs) */
void xb_pool_evict(xb_pool* p);
void xb_pool_free(xb_pool* p);

/* ---- the batch entry points ---- */
/* Replaces the loop at pipeline.cpp:103-136 (extend_seed per task,
 * align.cpp:268-309): out[2t] = left, out[2t+1] = right, seed_score[t];
 * the task's total is left.score + seed_score + right.score when both sides
 * are XB_SIDE_OK.  On XB_E_DANGLING / XB_E_SEED_OOB / XB_E_UNKNOWN_SYMBOL,
 * *bad_task (if non-NULL) is the first offending task index. */
int xb_extend_batch(xb_pool* p, const xb_task* tasks, int64_t n, int k, int band,
                    xb_side_result* out, int32_t* seed_score, int64_t* bad_task,
                    const xb_exec* exec);

/* Explicit units: each entry is one xdrop_extend call (align.cpp:165-177). */
int xb_extend_units(xb_pool* p, const xb_unit* units, int64_t n, int band, xb_side_result* out,
                    int64_t* bad_unit, const xb_exec* exec);

/* Device-resident form used to time the kernels alone: create uploads the
 * pool and the tasks, run enqueues LR split + sort + the kernel tiers on the
 * stream (no host sync), fetch downloads the results. */
xb_batch* xb_batch_create(xb_pool* p, const xb_task* tasks, int64_t n, int k, int band,
                          const xb_exec* exec, int64_t* bad_task, int* err);
int xb_batch_run(xb_batch* b);
int xb_batch_sync(xb_batch* b);
int xb_batch_fetch(xb_batch* b, xb_side_result* out, int32_t* seed_score);
int xb_batch_stats(xb_batch* b, xb_stats* st);
void xb_batch_free(xb_batch* b);

/* ---- sharding across processes / devices (partition.cpp:110-305) ---- */
/* Splits a task list into n_shards (one per GPU: torchrun ranks, or the
 * devices of one xb_exec): shard_of[t] in [0, n_shards), deterministic.
 * XB_SHARD_LPT: longest-processing-time on the estimated task cost (the
 *   assignment xb_extend_batch uses across devices; schedule_batches,
 *   partition.cpp:231-305, without the tile-memory test).
 * XB_SHARD_LOCALITY: tasks ordered along a breadth-first sweep of the
 *   sequence graph and cut into contiguous runs of equal cost, so each shard
 *   references a compact part of the pool (the reference's graph partition,
 *   partition.cpp:110-184, re-targeted from IPU tiles to GPUs); a device then
 *   uploads only the sequences its shard references.
 * Validation and error codes as xb_extend_batch. */
#define XB_SHARD_LPT 0
#define XB_SHARD_LOCALITY 1
int xb_shard_tasks(xb_pool* p, const xb_task* tasks, int64_t n, int k, int n_shards, int mode,
                   int32_t* shard_of, int64_t* bad_task);

/* stats of the last xb_extend_batch / xb_extend_units call on this thread */
int xb_last_stats(xb_stats* st);

/* ---- measurement helpers (not part of the reference surface) ---- */
/* INT32 issue-rate microbenchmark on `device`: lane-ops/clk/SM for chains of
 * IADD3/IMNMX/VIADDMNMX (alu) and for the kernel's own ALU+FMA mix; also the
 * SM clock seen (MHz) and SM count. */
int xb_measure_int32_peak(int device, double* alu_ops_per_clk_sm, double* mixed_ops_per_clk_sm,
                          double* clk_mhz, int* sm_count);

/* Checked builds only (make checked: -DXB_CHECKS=1, libxdrop_b200_checked.so):
 * waits for `device`, returns in *failed the id of the first bounds check
 * that failed since the last call (0: none) and clears it.  Product builds
 * return -1 (checks compiled out). */
int xb_debug_checks(int device, uint32_t* failed);

/* The planner's choice for a latency-planned batch (no reference analogue; the
 * reference schedules IPU tiles, partition.cpp:231-305): which kernels run
 * several lanes per unit -- 1 = 4-lane groups, 2 = lane tiers (8 lanes) --
 * given the SM count, the scoring mode (0 = +1/-1/-1 DNA, else table), the
 * number of units and the estimated antidiagonals of the longest unit and of
 * the whole batch.  Pure host arithmetic: no device needed. */
int xb_plan_group_family(int sm_count, int table_mode, int64_t n_units, double est_max, double est_sum);

/* ---- deterministic synthetic configs (BASELINE.json configs[0..4]) ---- */
/* Builds config `cfg` (1..5) at `scale` (1.0 = the BASELINE size).  Returns
 * a handle; query sizes then copy out.  Matrix configs (cfg 3) take the
 * NCBI matrix text for the BLOSUM62 conditional substitutions. */
typedef struct xb_synth xb_synth;
xb_synth* xb_synth_make(int cfg, double scale, uint64_t seed, const char* matrix_text,
                        int n_threads, int* err);
/* sizes: [0] n_seqs, [1] total symbols, [2] n_tasks, [3] k, [4] x, [5] band */
void xb_synth_sizes(const xb_synth* s, int64_t* sizes6);
/* symbols: total bytes; offsets: n_seqs+1; tasks: 4*n_tasks int64 (h_id, v_id, h_seed, v_seed) */
void xb_synth_copy(const xb_synth* s, char* symbols, int64_t* offsets, int64_t* tasks);
void xb_synth_free(xb_synth* s);
/* The reference's pair generator (generate_synthetic, proj/src/io.cpp:198-255,
 * SynthParams io.hpp:35-42): `pairs` pairs of length `length`, V mutated at
 * rate 1 - p_match outside a k-mer seed at the centre (uniform_seed = 0) or a
 * uniform position; byte-identical to the reference for the same parameters.
 * k < 1 or k > length: XB_E_BAD_PARAM (the reference's InputError). */
xb_synth* xb_synth_pairs(uint64_t pairs, uint64_t length, double p_match, int k, int uniform_seed,
                         uint64_t rng_seed, int* err);

/* ---- ingest of the reference's input formats (proj/src/io.cpp:58-196) ---- */
/* Parse errors carry the reference's exception kind (errors.hpp:54-82), the
 * 1-based line where the exception has one (InvalidSymbol, MalformedLine;
 * else 0, the line is then in the text) and its what() text. */
#define XB_PARSE_OK 0
#define XB_PARSE_MISSING_HEADER 1   /* MissingHeader */
#define XB_PARSE_EMPTY_RECORD 2     /* EmptyRecord */
#define XB_PARSE_INVALID_SYMBOL 3   /* InvalidSymbol (line) */
#define XB_PARSE_MALFORMED_LINE 4   /* MalformedLine (line) */
#define XB_PARSE_NEGATIVE_INDEX 5   /* NegativeIndex */
#define XB_PARSE_BAD_HEADER 6       /* BadHeader */
#define XB_PARSE_OUT_OF_SHAPE 7     /* IndexOutOfDeclaredShape */
#define XB_PARSE_BAD_ARGUMENT 8     /* null text / negative length (no reference analogue) */
typedef struct {
    int32_t kind;
    int32_t reserved;
    int64_t line;
    char message[256];
} xb_parse_error;

/* parse_fasta (io.cpp:58-96): records of `text` (LF or CRLF), symbols
 * upper-cased and checked against `allowed`, into one contiguous buffer on
 * all host threads (n_threads <= 0: all).  NULL on a parse error (*err). */
typedef struct xb_fasta xb_fasta;
xb_fasta* xb_fasta_parse(const char* text, int64_t len, const char* allowed, int n_threads,
                         xb_parse_error* err);
/* sizes: [0] records, [1] symbol bytes, [2] name bytes */
void xb_fasta_sizes(const xb_fasta* f, int64_t* sizes3);
/* symbols; offsets (records+1); names concatenated; name_offsets (records+1) */
void xb_fasta_copy(const xb_fasta* f, char* symbols, int64_t* offsets, char* names,
                   int64_t* name_offsets);
/* appends every record to the pool (ids in file order, as xb_pool_add_bulk) */
int64_t xb_pool_add_fasta(xb_pool* p, const xb_fasta* f);
void xb_fasta_free(xb_fasta* f);
/* parse_seeds (io.cpp:98-127) / parse_overlaps (io.cpp:129-196, Matrix
 * Market coordinate pattern|integer general, 1-based ids): tasks in input
 * order, task_id = ordinal.  Returns the task count (at most `cap` written;
 * call with cap 0 to size), or -XB_E_PARSE with *err filled. */
int64_t xb_parse_seeds(const char* text, int64_t len, xb_task* out, int64_t cap, xb_parse_error* err);
int64_t xb_parse_overlaps(const char* text, int64_t len, xb_task* out, int64_t cap,
                          xb_parse_error* err);

/* ---- band survey (sweep_band, proj/src/pipeline.cpp:181-208) ---- */
/* For every X in xs and every p in ps: one synthetic pair (xb_synth_pairs
 * with pairs = 1, k = 17, centred seed, rng_seed), extended over the full
 * views with +1/-1/-1 scoring and band = length + 1; delta_w[ix*np + ip]
 * receives its delta_w.  The X values run as concurrent batches.  The
 * reference prints "x\terror_rate\tdelta_w" rows with error_rate = 1 - p
 * as %.2f (xband_b200::sweep_band and xband.sweep_band reproduce the text). */
int xb_sweep_band(uint64_t length, const int32_t* xs, int32_t nx, const double* ps, int32_t np,
                  uint64_t rng_seed, int32_t* delta_w, const xb_exec* exec);

#ifdef __cplusplus
}
#endif

#endif
