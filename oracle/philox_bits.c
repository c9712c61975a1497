/*
 * oracle/philox_bits.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * (1) Philox4x32-10, the counter-based generator of reading R8 (the paper only
 *     says each scheme has "its own random number generator for consistent
 *     results").  Constants and round function are Random123's
 *     published Philox4x32 (Salmon et al., SC'11); pinned by the three Random123
 *     known-answer vectors in tests/golden/philox_kat.txt (T6).
 * (2) The paper's bit-level ternary arithmetic, PAPER:403-422 (section 3.5.2),
 *     transcribed formula by formula.  Pinned exhaustively against integer
 *     arithmetic (T3).  The oracle's walk does NOT use these: it uses integer
 *     arithmetic on int8 coefficients (walk.c), the plain definition.
 */
#include "oracle.h"

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint64_t p0 = (uint64_t)PHILOX_M0 * c[0];
    uint64_t p1 = (uint64_t)PHILOX_M1 * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    int round;
    for (round = 0; round < 10; round++) {
        if (round > 0) { k[0] += PHILOX_W0; k[1] += PHILOX_W1; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* R8: word t of step s of walker w:
   key = (seed lo, seed hi); counter = (s lo, s hi, w, t >> 2); word = out[t & 3]. */
uint32_t or_word(uint64_t seed, uint64_t step, uint64_t walker_id, int slot)
{
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t ctr[4] = {(uint32_t)step, (uint32_t)(step >> 32), (uint32_t)walker_id,
                       (uint32_t)(slot >> 2)};
    uint32_t out[4];
    or_philox4x32_10(ctr, key, out);
    return out[slot & 3];
}

/* PAPER:403-408 (Addition), transcribed:
   digits_{a+b} = digits_a XOR digits_b
   signs_{a+b}  = (signs_a AND digits_a OR signs_b AND digits_b) AND digits_{a+b}
   valid_{a+b}  = (digits_a AND digits_b AND NOT(signs_a XOR signs_b)) == 0       */
void or_bits_add(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb,
                 uint64_t *d, uint64_t *s, int *valid)
{
    uint64_t digits = da ^ db;
    uint64_t signs = ((sa & da) | (sb & db)) & digits;
    *d = digits;
    *s = signs;
    *valid = ((da & db & ~(sa ^ sb)) == 0);
}

/* PAPER:410-415 (Subtraction), transcribed:
   digits_{a-b} = digits_a XOR digits_b
   signs_{a-b}  = (signs_a AND digits_a OR NOT(signs_b) AND digits_b) AND digits_{a-b}
   valid_{a-b}  = (digits_a AND digits_b AND (signs_a XOR signs_b)) == 0          */
void or_bits_sub(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb,
                 uint64_t *d, uint64_t *s, int *valid)
{
    uint64_t digits = da ^ db;
    uint64_t signs = ((sa & da) | (~sb & db)) & digits;
    *d = digits;
    *s = signs;
    *valid = ((da & db & (sa ^ sb)) == 0);
}

/* a = b  <=>  (digits_a = digits_b) AND (signs_a = signs_b) */
int or_bits_eq(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb)
{
    return (da == db) && (sa == sb);
}

/* a = -b <=> (digits_a = digits_b) AND (signs_a = NOT(signs_b) AND digits_b).
   The zero vector satisfies this formula; reading R4 makes zero
   "equal", never "negated", so the zero case is excluded here. */
int or_bits_negeq(uint64_t da, uint64_t sa, uint64_t db, uint64_t sb)
{
    return (da == db) && (sa == (~sb & db)) && (da != 0);
}

void or_bits_batch(int64_t n, const uint64_t *da, const uint64_t *sa, const uint64_t *db,
                   const uint64_t *sb, int op, uint64_t *d, uint64_t *s,
                   int32_t *valid, int32_t *eq, int32_t *negeq)
{
    int64_t i;
    for (i = 0; i < n; i++) {
        int v;
        if (op == 0) or_bits_add(da[i], sa[i], db[i], sb[i], &d[i], &s[i], &v);
        else         or_bits_sub(da[i], sa[i], db[i], sb[i], &d[i], &s[i], &v);
        valid[i] = v;
        eq[i] = or_bits_eq(da[i], sa[i], db[i], sb[i]);
        negeq[i] = or_bits_negeq(da[i], sa[i], db[i], sb[i]);
    }
}
