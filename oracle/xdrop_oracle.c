/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the X-drop seed-extension path.
 * See xdrop_oracle.h for the rules on who may call this.
 *
 * A plain-C restatement of the reference algorithm, written from its
 * semantics rather than its code:
 *   - scoring tables ............ proj/src/scoring.cpp:16-53 (N never matches)
 *   - the reversing view op ..... proj/include/xband/sequence.hpp:35-38
 *   - banded X-drop kernel ...... proj/src/align.cpp:37-155 (window rules
 *                                 70-98, cell rules 102-136, result 148-154)
 *   - dense reference ........... proj/src/align.cpp:179-266
 *   - seed stitching ............ proj/src/align.cpp:268-309
 *   - batch loop ................ proj/src/pipeline.cpp:103-136
 *
 * Storage differs from the reference on purpose (three rows addressed by
 * i - row_lo instead of two folded rows); only the observable results must
 * agree, and tests/test_oracle.py checks that against oracle/_ref.
 */
#include "xdrop_oracle.h"

#include <limits.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define DEAD INT32_MIN

static const char kDna[] = "ACGTN";

int xo_scheme_match_mismatch(xo_scheme* s, int match, int mismatch, int gap, int x) {
    if (match <= 0 || mismatch >= 0 || gap >= 0 || x < 0) return -1;
    memset(s, 0, sizeof *s);
    s->gap = gap;
    s->x = x;
    for (int a = 0; a < 5; ++a) {
        s->valid[(unsigned char)kDna[a]] = 1;
        for (int b = 0; b < 5; ++b) {
            /* 'N' is an unknown base: it scores as a mismatch even against N */
            int same = (a == b) && kDna[a] != 'N';
            s->table[(unsigned char)kDna[a] * 256 + (unsigned char)kDna[b]] =
                (int16_t)(same ? match : mismatch);
        }
    }
    return 0;
}

int xo_scheme_from_matrix(xo_scheme* s, const char* alphabet, int n, const int* cells,
                          int gap, int x) {
    if (gap >= 0 || x < 0 || n <= 0) return -1;
    memset(s, 0, sizeof *s);
    s->gap = gap;
    s->x = x;
    for (int a = 0; a < n; ++a) {
        s->valid[(unsigned char)alphabet[a]] = 1;
        for (int b = 0; b < n; ++b)
            s->table[(unsigned char)alphabet[a] * 256 + (unsigned char)alphabet[b]] =
                (int16_t)cells[a * n + b];
    }
    return 0;
}

static inline unsigned char elem(const xo_view* w, int64_t i) {
    return w->dir ? w->origin[i] : w->origin[-1 - i];
}

static inline int32_t score_of(const xo_scheme* s, unsigned char a, unsigned char b) {
    return s->table[(size_t)a * 256 + b];
}

/* One antidiagonal's worth of cells: values for i in [lo, lo + cap), live
 * (unpruned) cells confined to [fl, ll]; fl > ll means nothing survived. */
typedef struct {
    int32_t* val;
    int64_t lo;
    int64_t fl, ll;
} diag_row;

static inline int32_t peek(const diag_row* r, int64_t i) {
    if (i < r->fl || i > r->ll) return DEAD;
    return r->val[i - r->lo];
}

static inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
static inline int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

int xo_xdrop_extend(xo_view h, xo_view v, const xo_scheme* s, int band, xo_result* out) {
    if (band < 1) return -1;
    const int64_t m = h.length, n = v.length;
    const int32_t gap = s->gap, x = s->x;

    int32_t* store = (int32_t*)malloc(sizeof(int32_t) * 3 * ((size_t)band + 1));
    diag_row rows[3];
    for (int r = 0; r < 3; ++r) {
        rows[r].val = store + (size_t)r * ((size_t)band + 1);
        rows[r].lo = 0;
        rows[r].fl = 0;
        rows[r].ll = -1;
    }
    /* antidiagonal 0 is the origin cell, antidiagonal -1 is empty */
    rows[0].val[0] = 0;
    rows[0].fl = rows[0].ll = 0;

    int32_t best = 0;
    int64_t best_d = 0, best_i = 0, cells = 1;
    int32_t widest = 1;
    out->status = XO_OK;
    out->spread = 0;

    for (int64_t d = 1; d <= n + m + 1; ++d) {
        diag_row* prev = &rows[(d - 1) % 3];
        diag_row* prev2 = &rows[(d + 1) % 3]; /* (d - 2) mod 3 */
        diag_row* cur = &rows[d % 3];
        const int prev_live = prev->fl <= prev->ll;
        const int prev2_live = prev2->fl <= prev2->ll;
        if (!prev_live && !prev2_live) break;

        /* reachable span: a gap step from d-1 or a diagonal step from d-2 */
        int64_t lo = INT64_MAX, hi = INT64_MIN;
        if (prev_live) {
            lo = prev->fl;
            hi = prev->ll + 1;
        }
        if (prev2_live) {
            lo = min64(lo, prev2->fl + 1);
            hi = max64(hi, prev2->ll + 1);
        }
        lo = max64(lo, d > m ? d - m : 0);
        hi = min64(hi, min64(d, n));
        if (lo > hi) {
            cur->fl = 0;
            cur->ll = -1;
            continue;
        }
        const int64_t w = hi - lo + 1;
        if (w > band) {
            out->status = XO_BAND_EXCEEDED;
            out->spread = (int32_t)w;
            out->cells = cells;
            out->score = 0;
            out->h_ext = out->v_ext = 0;
            out->delta_w = widest;
            free(store);
            return 0;
        }
        if (w > widest) widest = (int32_t)w;
        cells += w;

        cur->lo = lo;
        int64_t first = -1, last = -1;
        for (int64_t i = lo; i <= hi; ++i) {
            const int64_t j = d - i;
            int32_t val = DEAD;
            const int32_t dg = peek(prev2, i - 1); /* live only when i,j >= 1 */
            if (dg != DEAD) val = dg + score_of(s, elem(&v, i - 1), elem(&h, j - 1));
            if (j >= 1) {
                const int32_t left = peek(prev, i);
                if (left != DEAD && left + gap > val) val = left + gap;
            }
            if (i >= 1) {
                const int32_t up = peek(prev, i - 1);
                if (up != DEAD && up + gap > val) val = up + gap;
            }
            if (val != DEAD) {
                /* running best first (strict: earliest cell wins), then the
                 * drop test against that running best */
                if (val > best) {
                    best = val;
                    best_d = d;
                    best_i = i;
                }
                if (val < best - x) val = DEAD;
            }
            cur->val[i - lo] = val;
            if (val != DEAD) {
                if (first < 0) first = i;
                last = i;
            }
        }
        if (first < 0) {
            cur->fl = 0;
            cur->ll = -1;
        } else {
            cur->fl = first;
            cur->ll = last;
        }
    }

    out->score = best;
    out->h_ext = (int32_t)(best_d - best_i);
    out->v_ext = (int32_t)best_i;
    out->cells = cells;
    out->delta_w = widest;
    free(store);
    return 0;
}

int xo_full_oracle(xo_view h, xo_view v, const xo_scheme* s, xo_result* out) {
    const int64_t m = h.length, n = v.length;
    const int64_t cols = m + 1;
    int32_t* M = (int32_t*)malloc(sizeof(int32_t) * (size_t)((n + 1) * cols));
    for (int64_t q = 0; q < (n + 1) * cols; ++q) M[q] = DEAD;
#define AT(i, j) M[(i) * cols + (j)]
    int32_t best = 0;
    int64_t best_d = 0, best_i = 0;
    AT(0, 0) = 0;
    int64_t fl1 = 0, ll1 = 0;  /* live range of d-1 */
    int64_t fl2 = 0, ll2 = -1; /* live range of d-2 */
    int32_t widest = 1;
    for (int64_t d = 1; d <= n + m; ++d) {
        const int64_t ilo = max64(0, d - m), ihi = min64(d, n);
        int64_t first = -1, last = -1;
        for (int64_t i = ilo; i <= ihi; ++i) {
            const int64_t j = d - i;
            int32_t val = DEAD;
            if (i >= 1 && j >= 1 && AT(i - 1, j - 1) != DEAD)
                val = AT(i - 1, j - 1) + score_of(s, elem(&v, i - 1), elem(&h, j - 1));
            if (j >= 1 && AT(i, j - 1) != DEAD && AT(i, j - 1) + s->gap > val)
                val = AT(i, j - 1) + s->gap;
            if (i >= 1 && AT(i - 1, j) != DEAD && AT(i - 1, j) + s->gap > val)
                val = AT(i - 1, j) + s->gap;
            if (val != DEAD) {
                if (val > best) {
                    best = val;
                    best_d = d;
                    best_i = i;
                }
                if (val < best - s->x) val = DEAD;
                if (val != DEAD) {
                    if (first < 0) first = i;
                    last = i;
                }
            }
            AT(i, j) = val;
        }
        /* the window the banded kernel would have opened on this d */
        if (fl1 <= ll1 || fl2 <= ll2) {
            int64_t lo = INT64_MAX, hi = INT64_MIN;
            if (fl1 <= ll1) {
                lo = fl1;
                hi = ll1 + 1;
            }
            if (fl2 <= ll2) {
                lo = min64(lo, fl2 + 1);
                hi = max64(hi, ll2 + 1);
            }
            lo = max64(lo, ilo);
            hi = min64(hi, ihi);
            if (lo <= hi && hi - lo + 1 > widest) widest = (int32_t)(hi - lo + 1);
        }
        fl2 = fl1;
        ll2 = ll1;
        if (first < 0) {
            fl1 = 0;
            ll1 = -1;
        } else {
            fl1 = first;
            ll1 = last;
        }
    }
#undef AT
    out->score = best;
    out->h_ext = (int32_t)(best_d - best_i);
    out->v_ext = (int32_t)best_i;
    out->cells = (n + 1) * (m + 1);
    out->delta_w = widest;
    out->status = XO_OK;
    out->spread = 0;
    free(M);
    return 0;
}

/* ---- batch of seed tasks (pipeline.cpp:103-136 semantics) ---- */

typedef struct {
    const unsigned char* pool;
    const int64_t* seq_off;
    const int64_t* tasks;
    int64_t n;
    int k;
    const xo_scheme* s;
    int band;
    xo_result* out;
    int32_t* seed_score;
    int64_t next; /* shared cursor, guarded by mu */
    pthread_mutex_t mu;
} batch_ctx;

static void run_task(batch_ctx* c, int64_t t) {
    const int64_t* q = c->tasks + 4 * t;
    const int64_t hid = q[0], vid = q[1], hs = q[2], vs = q[3];
    const unsigned char* H = c->pool + c->seq_off[hid];
    const unsigned char* V = c->pool + c->seq_off[vid];
    const int64_t hl = c->seq_off[hid + 1] - c->seq_off[hid];
    const int64_t vl = c->seq_off[vid + 1] - c->seq_off[vid];
    int32_t ss = 0;
    for (int i = 0; i < c->k; ++i) ss += score_of(c->s, H[hs + i], V[vs + i]);
    c->seed_score[t] = ss;
    xo_view hlv = {H + hs, hs, 0}, vlv = {V + vs, vs, 0};
    xo_xdrop_extend(hlv, vlv, c->s, c->band, &c->out[2 * t]);
    xo_view hrv = {H + hs + c->k, hl - hs - c->k, 1}, vrv = {V + vs + c->k, vl - vs - c->k, 1};
    xo_xdrop_extend(hrv, vrv, c->s, c->band, &c->out[2 * t + 1]);
}

static void* batch_worker(void* arg) {
    batch_ctx* c = (batch_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        int64_t t0 = c->next;
        c->next += 64;
        pthread_mutex_unlock(&c->mu);
        if (t0 >= c->n) break;
        int64_t t1 = t0 + 64 < c->n ? t0 + 64 : c->n;
        for (int64_t t = t0; t < t1; ++t) run_task(c, t);
    }
    return NULL;
}

int xo_extend_batch(const unsigned char* pool, const int64_t* seq_off, int64_t n_seqs,
                    const int64_t* tasks, int64_t n, int k, const xo_scheme* s, int band,
                    xo_result* out, int32_t* seed_score, int64_t* bad_task, int n_threads) {
    if (band < 1 || k < 0) return 1;
    /* validation first, as extend_seed does (align.cpp:271-279) */
    for (int64_t t = 0; t < n; ++t) {
        const int64_t* q = tasks + 4 * t;
        if (q[0] < 0 || q[1] < 0 || q[0] >= n_seqs || q[1] >= n_seqs) {
            if (bad_task) *bad_task = t;
            return 2;
        }
        const int64_t hl = seq_off[q[0] + 1] - seq_off[q[0]];
        const int64_t vl = seq_off[q[1] + 1] - seq_off[q[1]];
        if (q[2] < 0 || q[3] < 0 || q[2] + k > hl || q[3] + k > vl) {
            if (bad_task) *bad_task = t;
            return 3;
        }
        for (int i = 0; i < k; ++i)
            if (!s->valid[pool[seq_off[q[0]] + q[2] + i]] ||
                !s->valid[pool[seq_off[q[1]] + q[3] + i]]) {
                if (bad_task) *bad_task = t;
                return 4;
            }
    }
    batch_ctx c;
    memset(&c, 0, sizeof c);
    c.pool = pool;
    c.seq_off = seq_off;
    c.tasks = tasks;
    c.n = n;
    c.k = k;
    c.s = s;
    c.band = band;
    c.out = out;
    c.seed_score = seed_score;
    pthread_mutex_init(&c.mu, NULL);
    if (n_threads <= 1) {
        batch_worker(&c);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
        for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, batch_worker, &c);
        for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&c.mu);
    return 0;
}
