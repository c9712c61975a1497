/*
 * oracle.h -- the CPU oracle for the flip-graph random walk of arXiv 2511.20317.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load liboracle.so.  The product path
 * (paper_2511_20317_b200/, libfg.so) never links, imports or calls anything here,
 * and this code shares nothing with it (no headers, no helpers, no tables).
 *
 * What it is: a plain, slow, obviously-correct C99 implementation of what the
 * walk computes, written from PAPER.md (/root/reference/PAPER.md, cited as
 * PAPER:<line>) and the readings fixed in DESIGN.md ("Readings", R1-R23, which
 * follow SURVEY.md section 8(c)).  Coefficients are stored as plain int8 values
 * in {-1,0,1}; ternary arithmetic is integer arithmetic with a range check (the
 * definition), NOT the paper's bit-plane encoding.  The paper's bit formulas
 * are implemented separately in or_bits_* so the tests can pin
 * them against integer arithmetic; the walk does not use them.
 *
 * Every step rebuilds its flip-candidate list from scratch (O(r^2)).  Nothing is
 * blocked, fused or reordered.
 *
 * Pins (tests/test_oracle_*.py): T1 PAPER:132-182 (2,2,3:11) verifies only in the
 * C^T layout; T2 PAPER:433-497 normalisation example; T3 PAPER:403-422 bit
 * formulas vs integers (exhaustive); T4 PAPER:656 additions; T5 PAPER:515-524
 * invariants; T6 Random123 Philox known-answer vectors; tensor invariance of every
 * move; brute-force neighbour counts; Strassen rediscovery from naive (2,2,2)
 * (PAPER:11).  The exact walk TRAJECTORY (which move is taken at each step) is
 * "parity unpinned" by the paper: it follows the readings R8-R17, and the GPU
 * path must reproduce it bit-exactly.
 */
#ifndef FG_ORACLE_H
#define FG_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OR_MAXLEN 64          /* <= 64 elements per factor */
#define OR_RING_ZT 0          /* Z_T = {-1,0,1} */
#define OR_RING_Z2 1          /* Z_2 = {0,1} */
#define OR_NCNT 12

/* per-walker counters (same meaning as the GPU path's) */
enum { OR_C_STEPS = 0, OR_C_DRAWS, OR_C_FLIPS, OR_C_FLIP_FAIL, OR_C_EXPAND_OK,
       OR_C_EXPAND_REJECT, OR_C_MERGES, OR_C_ZERO_REMOVED, OR_C_BEST_COPIES,
       OR_C_IMPROVEMENTS, OR_C_REDUCE_CALLS, OR_C_VERIFY_FAIL };

typedef struct {
    uint32_t k_flip;        /* max flip draws per step (R11) */
    uint32_t thr_accept_eq; /* Bernoulli(0.01) as u32 threshold (R9) */
    uint32_t thr_reduce;    /* p_reduce threshold */
    uint32_t thr_expand;    /* p_expand threshold */
    int32_t  expand_slack;  /* "best_rank + 2" */
    uint32_t mode;          /* 0 = Alg. 1 walk, 1 = naive-complexity minimisation (R24) */
} or_params;

typedef struct {
    int m, n, p, ring, R;   /* format, ring, row capacity */
    int len[3];             /* m*n, n*p, p*m */
    int r;                  /* current rank */
    int best_r;
    int best_adds;          /* naive additions of the best scheme */
    uint64_t walker_id;     /* global id, Philox counter word 2 (R8) */
    uint64_t step;          /* Alg.1 iteration index since seeding (R8) */
    uint64_t digest;        /* running event digest */
    uint64_t cnt[OR_NCNT];
    int8_t *rows;           /* R*3*OR_MAXLEN: rows[(l*3+X)*OR_MAXLEN + e] */
    int8_t *best;           /* same layout */
} or_walker;

/* --- Philox4x32-10 (Random123), R8 --- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t or_word(uint64_t seed, uint64_t step, uint64_t walker_id, int slot);

/* --- the paper's bit formulas, PAPER:403-422 (pinned by T3; unused by the walk) --- */
void or_bits_add(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb,
                 uint64_t *d, uint64_t *s, int *valid);
void or_bits_sub(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb,
                 uint64_t *d, uint64_t *s, int *valid);
int or_bits_eq(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb);
int or_bits_negeq(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb);
/* batch form for the exhaustive test: n pairs, outputs d,s,valid,eq,negeq */
void or_bits_batch(int64_t n, const uint64_t *da, const uint64_t *sa, const uint64_t *db,
                   const uint64_t *sb, int op /*0 add,1 sub*/, uint64_t *d, uint64_t *s,
                   int32_t *valid, int32_t *eq, int32_t *negeq);

/* --- schemes as int8 rows [u(mn) | v(np) | w(pm)] --- */
int  or_verify(int m, int n, int p, int ring, const int8_t *coeffs, int rank,
               int32_t first_fail[3]);                    /* 0 = pass, 1 = fail, <0 arg */
int  or_additions(int m, int n, int p, const int8_t *coeffs, int rank);
void or_normalize_rows(int m, int n, int p, int8_t *coeffs, int rank);
int  or_naive(int m, int n, int p, int8_t *coeffs_out);   /* returns rank m*n*p */
/* type invariant PAPER:516: out[(ru*65+rv)*65+rw] += 1 for each row; out has 65^3 ints */
int  or_type_invariant(int m, int n, int p, const int8_t *coeffs, int rank, int32_t *out);
int  or_sym_invariant(int m, int n, int p, const int8_t *coeffs, int rank, int32_t *out);
int  or_matrix_rank(const int8_t *a, int rows, int cols);

/* --- walker --- */
int  or_walker_init(or_walker *w, int m, int n, int p, int ring, int R, uint64_t walker_id);
void or_walker_free(or_walker *w);
int  or_seed_rows(or_walker *w, const int8_t *coeffs, int rank);  /* normalises (ZT) */
int  or_seed_naive(or_walker *w);
void or_walk(or_walker *w, uint64_t steps, uint64_t seed, const or_params *prm);
int  or_get_rows(const or_walker *w, int which /*0 cur,1 best*/, int8_t *coeffs_out);
void or_restart(or_walker *w, const int8_t *coeffs, int rank);     /* R23 */

/* single moves, for property tests */
int  or_count_candidates(or_walker *w);                        /* |C|, R10 */
int  or_get_candidate(or_walker *w, int idx, int32_t out[4]);   /* (X,i,j,sigma) */
int  or_apply_flip(or_walker *w, int cand, int d, int e);       /* 1 = committed */
int  or_apply_expand(or_walker *w, int plus, int i, int j, int perm); /* 1 = applied */
void or_reduce_all_public(or_walker *w);
void or_local_reduce_public(or_walker *w, int a, int b);

/* --- meta operators, meta.c: int8 rows in and out, not normalised --- */
int or_meta_transpose(int m, int n, int p, const int8_t *in, int rank, int8_t *out);   /* -> (p,n,m) */
int or_meta_rotate(int m, int n, int p, const int8_t *in, int rank, int8_t *out);      /* -> (n,p,m) */
int or_meta_swap_sizes(int m, int n, int p, const int8_t *in, int rank, int8_t *out);  /* -> (m,p,n) */
int or_meta_project(int m, int n, int p, const int8_t *in, int rank, int8_t *out, int *rank_out);
int or_meta_extend(int m, int n, int p, const int8_t *in, int rank, int8_t *out, int *rank_out);
int or_meta_merge(int m, int n, int p1, int p2, const int8_t *a, int ra, const int8_t *b, int rb, int8_t *out);
int or_meta_product(int m1, int n1, int p1, const int8_t *a, int ra, int m2, int n2, int p2, const int8_t *b,
                    int rb, int8_t *out);

int or_resize(int *m, int *n, int *p, int8_t *coeffs, int *rank, int r_cap, int nbest, const int32_t *bfmt,
              const int32_t *brank, const int8_t *const *bcoeffs, uint32_t thr_resize, uint64_t seed,
              uint64_t round, uint64_t walker_id, int *op_out);                 /* Alg. 2, R31 */

int or_lift_exhaustive(int m, int n, int p, const int8_t *z2, int rank, int8_t *out);  /* lift.c */

/* many walkers in one flat call (bench cpu baseline / tests): walker k has global
   id id_base+k, all seeded naive (or from coeffs if rank>0).  Output per walker:
   r, best_r, digest, cnt[OR_NCNT], and optionally rows/best (R*(mn+np+pm) int8). */
/* ids (may be NULL): explicit global ids; else id_base + k */
int  or_run_walkers(int m, int n, int p, int ring, int R, int64_t count, uint64_t id_base,
                    const uint64_t *ids,
                    const int8_t *seed_coeffs, int seed_rank, uint64_t steps, uint64_t seed,
                    const or_params *prm, int threads,
                    int32_t *r_out, int32_t *best_r_out, uint64_t *digest_out,
                    uint64_t *cnt_out, int8_t *rows_out, int8_t *best_out);

#ifdef __cplusplus
}
#endif
#endif
