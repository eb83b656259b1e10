/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the X-drop hot path.
 *
 * This is a from-scratch C restatement of the reference xband kernel
 * (/root/reference/proj/src/align.cpp) used as the parity checker for the
 * sm_100a engine.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_2304_08662_b200) never links or calls anything in this directory.
 *
 * Parity is pinned: tests/test_oracle.py checks it against the reference's
 * own compiled library (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and against the golden vectors in tests/golden/.
 */
#ifndef XDROP_ORACLE_H
#define XDROP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes carried in xo_result.status */
#define XO_OK 0
#define XO_BAND_EXCEEDED 1

/* ScoringScheme (scoring.hpp:28-54): flat 256x256 byte-pair table. */
typedef struct {
    int16_t table[256 * 256];
    unsigned char valid[256];
    int gap;
    int x;
} xo_scheme;

/* ExtensionResult (align.hpp:37-45) plus the BandExceededError payload
 * (errors.hpp:85-93): on status XO_BAND_EXCEEDED, `spread` is the observed
 * spread and `cells` the work done before the abort. */
typedef struct {
    int32_t score;
    int32_t h_ext;
    int32_t v_ext;
    int32_t delta_w;
    int64_t cells;
    int32_t status;
    int32_t spread;
} xo_result;

/* A SeqView (sequence.hpp:27-39): `origin` points at symbols[origin] of the
 * backing sequence; dir 1 = Right (element i = origin[i]), dir 0 = Left
 * (element i = origin[-1-i]). */
typedef struct {
    const unsigned char* origin;
    int64_t length;
    int32_t dir;
} xo_view;

/* returns 0, or -1 on invalid parameters (scoring.cpp:17-20,37-40) */
int xo_scheme_match_mismatch(xo_scheme* s, int match, int mismatch, int gap, int x);
int xo_scheme_from_matrix(xo_scheme* s, const char* alphabet, int n, const int* cells,
                          int gap, int x);

/* xdrop_extend (align.cpp:37-177): banded kernel.  Returns -1 if band < 1. */
int xo_xdrop_extend(xo_view h, xo_view v, const xo_scheme* s, int band, xo_result* out);

/* xdrop_full_oracle (align.cpp:179-266): dense matrix restatement. */
int xo_full_oracle(xo_view h, xo_view v, const xo_scheme* s, xo_result* out);

/* Batch of seed tasks over a pool (pipeline.cpp:103-136 loop body):
 * pool = concatenated symbols, seq_off[i]..seq_off[i+1] = sequence i.
 * tasks = n x {h_id, v_id, h_seed, v_seed}.  out = 2n results (L then R per
 * task), seed_score = n.  Returns 0, 2 dangling id, 3 seed out of bounds
 * (first offending task index in *bad_task). */
int xo_extend_batch(const unsigned char* pool, const int64_t* seq_off, int64_t n_seqs,
                    const int64_t* tasks, int64_t n, int k, const xo_scheme* s, int band,
                    xo_result* out, int32_t* seed_score, int64_t* bad_task, int n_threads);

#ifdef __cplusplus
}
#endif

#endif
