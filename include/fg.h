/*
 * fg.h -- C ABI of libfg.so, the B200 (sm_100a) flip-graph walker of
 * arXiv 2511.20317 ("FlipGraphGPU"; PAPER.md lines cited as PAPER:<line>).
 *
 * What the library computes (the hot path):
 *   thousands of independent walkers, each holding one (m,n,p:r) matrix-
 *   multiplication scheme with coefficients in
 *   Z_T = {-1,0,1} or Z_2, run the RandomWalk
 *   of Algorithm 1: flips, reductions
 *   (PAPER:233-238), expand = plus/split, sign-symmetry
 *   normalisation, best tracking with 1% plateau acceptance
 *   (PAPER:310-313).  Every strict rank improvement is checked against
 *   the Brent equations by a batched device verifier.  Readings of
 *   points the paper leaves open are R1-R23 in DESIGN.md.
 *
 * Conventions for every function:
 *   - returns FG_OK (0) or a negative fg_status; nothing throws across the ABI;
 *     on error no output buffer is partially written;
 *   - every pointer argument is a HOST pointer owned by the caller, except where
 *     stated; the ctx owns all device memory it allocates;
 *   - one ctx per host thread; no callbacks; work is enqueued on the CUDA stream
 *     given to fg_create and the call synchronises that stream before returning
 *     unless stated otherwise;
 *   - determinism: (seed, global walker id, step index) fully determine every
 *     trajectory (reading R8), independent of launch geometry, GPU count or how
 *     the steps are split over fg_walk calls.
 *
 * Scheme interchange layout ("coeffs", SPEC:637-642 / PAPER:177-182): int8 rows,
 * one row per rank-one term, row = [u (m*n) | v (n*p) | w (p*m)], with
 *   u[i*n + j] = coefficient of a_ij, v[j*p + k] = coefficient of b_jk,
 *   w[k*m + i] = coefficient of the term in c_ik (C^T order).
 * Values in {-1,0,1} (Z_T) or {0,1} (Z_2).
 */
#ifndef FG_H
#define FG_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FG_MAX_LEN  64    /* a factor has <= 64 elements (one u64 word) */
#define FG_MAX_RCAP 512   /* rows reserved per walker (R1) */
#define FG_MAX_KFLIP 64   /* flip draws per step (R11: draw a uses Philox slot 7 + a, a >= 1) */
#define FG_NCNT     12    /* per-walker counters, see fg_get_walkers */

enum fg_ring { FG_ZT = 0, FG_Z2 = 1 };

enum fg_status {
    FG_OK = 0,
    FG_E_ARG = -1,            /* bad argument (null pointer, range, format < 1) */
    FG_E_CAPACITY = -2,       /* mn, np or pm > 64; rank > r_cap; r_cap > 512 */
    FG_E_DOMAIN = -3,         /* coefficient not in {-1,0,1} (Z_T) or {0,1} (Z_2); zero factor in a seed */
    FG_E_INVALID_SCHEME = -4, /* a seed fails the Brent equations */
    FG_E_CUDA = -5,           /* a CUDA call failed (no device, launch failure, OOM) */
    FG_E_STATE = -6,          /* call out of order (e.g. walk before seed) */
    FG_E_UNSUPPORTED = -7     /* format / r_cap combination without a kernel in this build */
};

/* Walk parameters (Alg. 1 inputs).  Probabilities are u32 thresholds:
   an event with probability q fires when a Philox word x satisfies x < q*2^32
   (reading R9).  fg_params_default() fills the defaults of DESIGN.md. */
typedef struct fg_params {
    uint32_t k_flip;        /* max flip draws per step, 1..FG_MAX_KFLIP (R11); default 16 */
    uint32_t thr_accept_eq; /* equal-rank acceptance, "random() < 0.01": 42949672 */
    uint32_t thr_reduce;    /* p_reduce: default 0.5 -> 2147483648 */
    uint32_t thr_expand;    /* p_expand: default 0.01 -> 42949672 */
    int32_t  expand_slack;  /* Alg. 1 "best_rank + 2": default 2 */
    uint32_t phase_steps;   /* steps per kernel launch inside fg_walk (0 = all in one) */
    uint32_t flags;         /* 0, or FG_FLAG_COMPLEXITY */
} fg_params;

/* fg_params.flags: naive-additive-complexity minimisation ("random flips
   without reduction edges", Table 4; reading R24 in DESIGN.md): each
   step is try_flip only -- a draw producing a zero factor is rejected, no local or
   global reduction, no expand, so the rank never changes -- and the best scheme is
   the minimum of (rank, naive additions PAPER:656), ties replaced with the 1%
   plateau acceptance.  Every strict improvement is verified. */
#define FG_FLAG_COMPLEXITY 1u

typedef struct fg_ctx fg_ctx;   /* opaque: owns the device pool and its host mirror */

void fg_params_default(fg_params *out);
const char *fg_strerror(int status);

/* Create a pool of num_walkers walkers for format (m,n,p) over `ring`, each with
   room for r_cap rows, on CUDA device `device`; work goes to `cuda_stream`
   (a cudaStream_t; NULL = the legacy default stream).  walker_id_base is the
   global id of local walker 0 (multi-GPU sharding); global
   ids must stay below 2^32 (Philox counter word 2, R8).  Errors: FG_E_ARG,
   FG_E_CAPACITY (R1), FG_E_UNSUPPORTED (no kernel variant), FG_E_CUDA. */
int fg_create(int m, int n, int p, int ring, int r_cap, int64_t num_walkers,
              int64_t walker_id_base, int device, void *cuda_stream, fg_ctx **out);
void fg_destroy(fg_ctx *ctx);

/* seed every walker with the naive (m,n,p : m*n*p) scheme, rows
   ordered l = (i*n + j)*p + k; this is also each walker's initial best
   (rank assessment).  Resets step counters, digests and counters.
   Errors: FG_E_CAPACITY if m*n*p > r_cap. */
int fg_seed_naive(fg_ctx *ctx);

/* seed walkers [w_begin, w_end) (local indices) with one scheme of
   `rank` rows in the interchange layout; it is verified and
   sign-normalised on entry and duplicated over the range.  Walkers
   outside the range are untouched.  Errors: FG_E_DOMAIN, FG_E_CAPACITY,
   FG_E_INVALID_SCHEME, FG_E_ARG. */
int fg_seed_pool(fg_ctx *ctx, const int8_t *coeffs, int rank, int64_t w_begin, int64_t w_end);

/* Load walkers [w_begin, w_begin+count) with one scheme EACH: coeffs is count * r_cap
   rows (row-padded), ranks[k] rows used by walker w_begin+k.  Every scheme is
   verified and sign-normalised; each walker's best is its scheme, its step index,
   digest and counters restart.  Used by exploratory search after a
   Resize round.  Errors as fg_seed_pool. */
int fg_load_walkers(fg_ctx *ctx, const int8_t *coeffs, const int32_t *ranks, int64_t w_begin, int64_t count);

/* Run `steps` iterations of Algorithm 1 (reading R17) on every
   walker, Philox key = seed (R8).  Split into launches of params->phase_steps
   steps.  After the walk: the batched verifier checks every strict improvement
   queued by the walk (R19), and the local best (rank, naive additions, walker id)
   is recomputed (R20, R21).  params may be NULL (defaults).  Synchronous.
   Errors: FG_E_STATE (not seeded), FG_E_ARG, FG_E_CUDA. */
int fg_walk(fg_ctx *ctx, uint64_t steps, uint64_t seed, const fg_params *params);

/* Pure host, exact Brent check (reading R7) of one scheme in the
   interchange layout.  Returns FG_OK if it verifies; FG_E_INVALID_SCHEME if not,
   with the lexicographically first failing (a,b,c) in first_fail (else -1s);
   FG_E_DOMAIN / FG_E_CAPACITY / FG_E_ARG on bad input.  Needs no GPU. */
int fg_verify(int m, int n, int p, int ring, const int8_t *coeffs, int rank,
              int32_t first_fail[3]);

/* Batched device Brent check of `count` schemes (the walk's verifier kernel,
   exposed): coeffs is count * r_cap rows (row-padded), ranks[k] rows used.
   ok_out[k] = 1 if scheme k verifies, first_fail_out[3k..3k+2] as fg_verify. */
int fg_verify_batch(fg_ctx *ctx, const int8_t *coeffs, const int32_t *ranks, int64_t count,
                    int32_t *ok_out, int32_t *first_fail_out);

/* Best scheme known to this ctx: the lexicographic minimum of (rank, naive
   additions PAPER:656, global walker id) over the local walkers' bests and every
   record imported with fg_import_best (R20).  coeffs_out (may be NULL) receives
   rank rows; it must hold r_cap rows. */
int fg_best(const fg_ctx *ctx, int *rank, int *naive_additions, int64_t *walker_id,
            int8_t *coeffs_out);

/* Bulk read of local walkers [w_begin, w_end) for parity and debugging.  Any
   output may be NULL.  Per walker: r, best_r, naive additions of the best scheme,
   digest,
   step index, FG_NCNT counters (steps, draws, flips, flip_fail, expand_ok,
   expand_reject, merges, zero_removed, best_copies, improvements, reduce_calls,
   verify_fail), and r_cap rows (zero-padded) of the current and best schemes. */
int fg_get_walkers(const fg_ctx *ctx, int64_t w_begin, int64_t w_end, int32_t *r,
                   int32_t *best_r, int32_t *best_adds, uint64_t *digest, uint64_t *step,
                   uint64_t *cnt, int8_t *rows, int8_t *best);

/* Single-walker convenience form of fg_get_walkers. */
int fg_get_walker(const fg_ctx *ctx, int64_t w, int *rank, int *best_rank, uint64_t *digest,
                  int8_t *coeffs_out, int8_t *best_out);

/* Fixed-size best records for the multi-GPU pool sync (DESIGN.md
   section 6): header (format, ring, r_cap, rank, additions, walker id) + the best
   scheme as 6*r_cap u64 bit planes.  All records of one job have the same size. */
size_t fg_record_bytes(int r_cap);
int fg_export_best(const fg_ctx *ctx, void *record);
/* Merge `count` records (e.g. the all-gathered records of every rank) into the
   ctx's pool best; invalid or other-format records are rejected with FG_E_ARG. */
int fg_import_best(fg_ctx *ctx, const void *records, int count);
/* Host-only deterministic merge (R20) of `count` records into *out. */
int fg_record_merge(const void *records, int count, void *out);
/* Host-only: build a record from a scheme (interchange layout). */
int fg_record_pack(int m, int n, int p, int ring, int r_cap, const int8_t *coeffs, int rank,
                   int64_t walker_id, void *record);
/* Host-only: read a record back (rank, additions, walker id, coeffs r_cap rows). */
int fg_record_unpack(const void *record, int *m, int *n, int *p, int *ring, int *rank,
                     int *additions, int64_t *walker_id, int8_t *coeffs_out);

/* Reading R23 (plateau restart, off unless called): every local walker whose
   best rank exceeds the pool best rank + slack is re-seeded with the pool best
   scheme (current and best); its step counter, counters continue and its digest
   records the restart.  *restarted receives the number re-seeded. */
int fg_restart(fg_ctx *ctx, int slack, int64_t *restarted);

/* Checkpoint / resume and host-buffer I/O: the complete walker state (planes of
   current and best schemes, ranks, step indices, digests, counters) as an opaque
   byte image of fg_state_bytes(ctx) bytes (64-byte header whose word 10 is the bytes
   per plane word, walker headers, current and best planes packed to 2 / 4 / 8 bytes
   per plane word for factors of <= 16 / 32 / 64 elements, and for the linked-class
   kernel walk_wl its per-walker class image).  Packing and unpacking run on the device
   around one copy each way.  Resuming from it continues every trajectory bit-exactly
   (R8).  fg_load_state rejects an image of another format, ring, capacity, walker
   count or plane width (FG_E_ARG). */
size_t fg_state_bytes(const fg_ctx *ctx);
int fg_save_state(const fg_ctx *ctx, void *host_buf);
int fg_load_state(fg_ctx *ctx, const void *host_buf);

/* Totals since create: out[0] steps, [1] draws, [2] flips, [3] expands,
   [4] merges + zero removals, [5] verified candidates, [6] verify failures,
   [7] verify-queue overflows, [8] kernel launches, [9] walk kernel ms (x1000),
   [10] verify kernel ms (x1000), [11] walk launches.  out must hold 12. */
int fg_stats(const fg_ctx *ctx, uint64_t out[12]);

/* ---- Meta operators (section 3.3.2; readings R25-R30 in DESIGN.md) ----
   Host only (no GPU), the orchestration between walks: schemes in the interchange
   layout in and out, output rows NOT sign-normalised (fg_seed_pool normalises).
   The caller sizes `out` for the result rank stated per function; the result
   format must satisfy R1 (else FG_E_CAPACITY).  Errors as fg_verify.             */
/* C = AB <=> C^T = B^T A^T: (m,n,p:r) -> (p,n,m:r) */
int fg_meta_transpose(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out);
/* cyclic symmetry of the matmul tensor: (u,v,w) -> (v,w,u), (m,n,p:r) -> (n,p,m:r) */
int fg_meta_rotate(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out);
/* swap sizes: (m,n,p:r) -> (m,p,n:r) = rotate(rotate(transpose)) */
int fg_meta_swap_sizes(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out);
/* project: (m,n,p) -> (m,n,p-1), drop the last column of B and C and the
   terms left with a zero factor; *rank_out <= rank rows written */
int fg_meta_project(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out, int *rank_out);
/* extend: (m,n,p:r) -> (m,n,p+1 : r+mn), a naive (m,n,1) block appended */
int fg_meta_extend(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out, int *rank_out);
/* merge: (m,n,p1:ra) + (m,n,p2:rb) -> (m,n,p1+p2 : ra+rb), B = [B1 | B2] */
int fg_meta_merge(int m, int n, int p1, int p2, int ring, const int8_t *a, int ra, const int8_t *b, int rb,
                  int8_t *out);
/* double: merge with itself, (m,n,p:r) -> (m,n,2p:2r) */
int fg_meta_double(int m, int n, int p, int ring, const int8_t *in, int rank, int8_t *out);
/* product: Kronecker, (m1,n1,p1:ra) x (m2,n2,p2:rb) -> (m1m2,n1n2,p1p2 : ra*rb),
   block index i = i1*m2 + i2 (same for j, k), row l = l1*rb + l2.  Block matrix
   multiplication with Strassen is the product with a (2,2,2:7) scheme. */
int fg_meta_product(int m1, int n1, int p1, const int8_t *a, int ra, int m2, int n2, int p2, const int8_t *b,
                    int rb, int ring, int8_t *out);

/* Alg. 2 Resize of one scheme, reading R31 in DESIGN.md; host only.
   Decisions come from Philox blocks 0x100 / 0x101 of counter (round lo, round hi,
   walker id, block) under key `seed`: swap sizes with probability 1/2; try to merge
   with a best scheme picked uniformly (same m and n); if not merged, with
   probability thr_resize/2^32: project 5% / product with a best scheme 50% / double
   30% / extend 15%.  A result outside R1, max(m,n,p) <= 16
   or rank <= r_cap is not applied.  (m,n,p), rank and coeffs are updated in place;
   coeffs must hold r_cap rows of the widest format (3*64 int8).  bests: nbest
   schemes, formats bfmt[3k..3k+2], ranks brank[k], rows bcoeffs[k].  op_out (may
   be NULL): bit 0 = swapped; bits 1..3 = 1 merge, 2 project, 3 product, 4 double,
   5 extend, 0 none.  Outputs are not sign-normalised. */
int fg_resize(int *m, int *n, int *p, int ring, int8_t *coeffs, int *rank, int r_cap, int nbest,
              const int32_t *bfmt, const int32_t *brank, const int8_t *const *bcoeffs, uint32_t thr_resize,
              uint64_t seed, uint64_t round, uint64_t walker_id, int *op_out);

/* Z_2 -> Z_T lifting (reading R32): find signs for the nonzero
   coefficients of a Z_2 scheme (rank rows of {0,1}) so that the Brent equations
   hold over the integers.  Depth-first search with the first nonzero of every row's
   u and v pinned to +1 and per-equation reachability pruning, at most
   node_budget nodes.  FG_OK: `out` holds the lifted scheme (rank rows in {-1,0,1},
   same support); FG_E_INVALID_SCHEME: no lift exists (search exhausted, or the
   input is not a Z_2 scheme); FG_E_STATE: budget exhausted (no conclusion).
   *nodes_used (may be NULL) reports the search size.  Host only. */
int fg_lift(int m, int n, int p, const int8_t *z2, int rank, int64_t node_budget, int8_t *out,
            int64_t *nodes_used);

/* Type invariant: counts[(ru*65 + rv)*65 + rw] = number of terms whose
   U, V, W factor matrices (m x n, n x p, p x m) have ranks (ru, rv, rw) over Q;
   rank_sums = the exponents of the rank-sum polynomial.  The
   symmetrised polynomial is the S_3 orbit sum of the type counts.
   counts must hold 65^3 ints.  Host only. */
int fg_type_invariant(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int32_t *counts,
                      int32_t rank_sums[3]);
/* Symmetrised polynomial invariant: sym[(a*65 + b)*65 + c] = the
   coefficient of x^a y^b z^c in sum_{pi in S_3} pi(sum_i x^{rank U_i} y^{rank V_i}
   z^{rank W_i}), ranks as in fg_type_invariant.  Invariant under the cyclic symmetry and
   transposition (meta operators), unlike the type polynomial.  sym must hold 65^3
   ints (caller-owned, overwritten).  FG_E_ARG on a NULL buffer, the fg_type_invariant
   errors otherwise.  Host only. */
int fg_sym_invariant(int m, int n, int p, int ring, const int8_t *coeffs, int rank, int32_t *sym);
/* Canonical 64-bit key of a scheme up to row order and per-row sign normalisation
   (PAPER:429): for pool de-duplication.  Host only. */
int fg_scheme_key(int m, int n, int p, int ring, const int8_t *coeffs, int rank, uint64_t *key);

/* Exact time-to-rank: out[k] (k = 0..max_rank) = the smallest
   walker step index (0-based Alg. 1 iteration since seeding, R8) in which some walker
   of this ctx made a VERIFIED strict improvement to rank k (R19), 0 for the seeded
   rank, UINT64_MAX if rank k was never reached that way.  A strict improvement whose
   verify-queue entry overflowed is not recorded (fg_stats [7] counts overflows).
   The box time to rank <= t is then min over k <= t.  FG_E_STATE before seeding. */
int fg_rank_first_steps(const fg_ctx *ctx, int max_rank, uint64_t *out);

/* Which kernel variant fg_walk uses for this ctx ("warp32_zt_u32k", ...). */
const char *fg_kernel_name(const fg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
