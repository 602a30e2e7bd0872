/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked or loaded by the product
 * library (paper_2002_01119_b200/lib/libringmix_b200.so).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker.
 *
 * Plain-C restatement of the integer chain behind the reference's
 * permutation_for_step (reference: pkg/src/ringmix/mixing.py:79-86) and
 * sample_permutation (mixing.py:72-76), whose randomness comes from
 * seeding.stream (pkg/src/ringmix/seeding.py:27-37):
 *
 *     np.random.default_rng(np.random.SeedSequence((seed, TAG, idx...)))
 *         .permutation(n)
 *
 * The algorithm lives in a third-party dependency absent from
 * /root/reference: numpy (pinned here to 2.3.5, the version the golden
 * fixtures in tests/golden/ were frozen under).  Restated from numpy's
 * published algorithm:
 *   - bit_generator.pyx  _coerce_to_uint32_array / SeedSequence.mix_entropy /
 *     SeedSequence.generate_state  (hashmix/mix constants below),
 *   - pcg64.h  pcg_setseq_128_srandom_r, pcg_setseq_128_xsl_rr_64_random_r,
 *     pcg64_next32 (buffered upper half),
 *   - distributions.c  random_interval (masked rejection),
 *   - _generator.pyx  Generator.shuffle (Fisher-Yates, i = n-1 .. 1).
 *
 * Parity is pinned against tests/golden/perms.npz, produced by running the
 * reference itself (tests/golden/make_golden.py).
 */
#include <stdint.h>
#include <stddef.h>

typedef unsigned __int128 u128;

#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_POOL 4

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

/* _int_to_uint32_array: 0 -> [0]; otherwise little-endian 32-bit limbs. */
int or_limbs(uint64_t v, uint32_t *out) {
    int n = 0;
    if (v == 0) {
        out[0] = 0;
        return 1;
    }
    while (v) {
        out[n++] = (uint32_t)v;
        v >>= 32;
    }
    return n;
}

/* SeedSequence(entropy words).generate_state(4, uint64). */
void or_seedseq_state(const uint32_t *ent, int n, uint64_t out[4]) {
    uint32_t pool[SS_POOL];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < SS_POOL; i++) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, &hc);
    for (int s = 0; s < SS_POOL; s++)
        for (int d = 0; d < SS_POOL; d++)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = SS_POOL; s < n; s++)
        for (int d = 0; d < SS_POOL; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
    uint32_t hb = SS_INIT_B;
    uint32_t w[8];
    for (int i = 0; i < 8; i++) {
        uint32_t v = pool[i % SS_POOL];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        w[i] = v;
    }
    for (int i = 0; i < 4; i++) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

typedef struct {
    u128 state, inc;
    int has32;
    uint32_t buf32;
} or_pcg64;

static const u128 PCG_MULT =
    (((u128)2549297995355413924ULL) << 64) | (u128)4865540595714422341ULL;

static void pcg_step(or_pcg64 *g) { g->state = g->state * PCG_MULT + g->inc; }

static void pcg_seed(or_pcg64 *g, const uint64_t v[4]) {
    u128 initstate = ((u128)v[0] << 64) | v[1];
    u128 initseq = ((u128)v[2] << 64) | v[3];
    g->state = 0;
    g->inc = (initseq << 1) | 1u;
    pcg_step(g);
    g->state += initstate;
    pcg_step(g);
    g->has32 = 0;
    g->buf32 = 0;
}

static uint64_t pcg_next64(or_pcg64 *g) {
    pcg_step(g);
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(g->state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static uint32_t pcg_next32(or_pcg64 *g) {
    if (g->has32) {
        g->has32 = 0;
        return g->buf32;
    }
    uint64_t n = pcg_next64(g);
    g->has32 = 1;
    g->buf32 = (uint32_t)(n >> 32);
    return (uint32_t)n;
}

static uint64_t random_interval(or_pcg64 *g, uint64_t max) {
    if (max == 0) return 0;
    uint64_t mask = max, v;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    if (max <= 0xffffffffULL) {
        while ((v = (pcg_next32(g) & mask)) > max) {}
    } else {
        while ((v = (pcg_next64(g) & mask)) > max) {}
    }
    return v;
}

static void shuffle_arange(or_pcg64 *g, int64_t n, int64_t *a) {
    for (int64_t i = 0; i < n; i++) a[i] = i;
    for (int64_t i = n - 1; i >= 1; i--) {
        int64_t j = (int64_t)random_interval(g, (uint64_t)i);
        int64_t t = a[i];
        a[i] = a[j];
        a[j] = t;
    }
}

/* permutation_for_step for an arbitrary entropy prefix (limbs of seed and
 * tag, computed by the caller for any Python int) followed by limbs(step). */
int or_permutation(const uint32_t *prefix, int nprefix, uint64_t step, int64_t n, int64_t *out) {
    uint32_t ent[64];
    if (nprefix < 0 || nprefix > 60) return -1;
    for (int i = 0; i < nprefix; i++) ent[i] = prefix[i];
    int ne = nprefix + or_limbs(step, ent + nprefix);
    uint64_t st[4];
    or_seedseq_state(ent, ne, st);
    or_pcg64 g;
    pcg_seed(&g, st);
    shuffle_arange(&g, n, out);
    return 0;
}

/* monte_carlo_consensus draw pattern (reference spectral.py:273-277): one
 * stream per index, `count` permutations drawn back to back from it (the
 * PCG state and the buffered 32-bit half carry across draws). */
int or_permutation_sequential(const uint32_t *prefix, int nprefix, uint64_t idx, int64_t n,
                              int count, int64_t *out) {
    uint32_t ent[64];
    if (nprefix < 0 || nprefix > 60) return -1;
    for (int i = 0; i < nprefix; i++) ent[i] = prefix[i];
    int ne = nprefix + or_limbs(idx, ent + nprefix);
    uint64_t st[4];
    or_seedseq_state(ent, ne, st);
    or_pcg64 g;
    pcg_seed(&g, st);
    for (int c = 0; c < count; c++) shuffle_arange(&g, n, out + (int64_t)c * n);
    return 0;
}

/* Raw generator outputs (used by tests to pin next64 against numpy). */
int or_raw64(const uint32_t *ent, int nent, int count, uint64_t *out) {
    uint64_t st[4];
    or_seedseq_state(ent, nent, st);
    or_pcg64 g;
    pcg_seed(&g, st);
    for (int c = 0; c < count; c++) out[c] = pcg_next64(&g);
    return 0;
}
