/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see perm_oracle.c header).
 *
 * Scalar C restatement of numpy 2.3.5's Generator.standard_normal for a
 * SeedSequence-seeded PCG64 stream, the noise source of the reference's
 * quadratic oracle (reference objectives.py:84-90 `batch.rng().standard_normal(d)`
 * with batch.rng() = seeding.stream(seed, TAG_GRADIENT, k, l), simulation.py:235).
 * numpy's published algorithm (distributions.c random_standard_normal): a
 * 256-layer ziggurat on 64-bit draws — idx = r & 0xff, sign = bit 8,
 * rabs = next 52 bits; fast accept rabs < ki[idx]; base-strip tail by
 * Marsaglia's exponential method with log1p; wedge test against exp(-x^2/2).
 * The ki/wi/fi tables are numpy's own doubles (read from the installed
 * libnpyrandom.a by tools/gen_ziggurat_tables.py) and passed in by the caller.
 */
#include <math.h>
#include <stdint.h>

typedef unsigned __int128 u128;

/* from perm_oracle.c */
void or_seedseq_state(const uint32_t *ent, int n, uint64_t out[4]);

static const u128 NRM_MULT =
    (((u128)2549297995355413924ULL) << 64) | (u128)4865540595714422341ULL;

typedef struct {
    u128 state, inc;
    int64_t draws;
} nrm_pcg;

static void nrm_step(nrm_pcg *g) { g->state = g->state * NRM_MULT + g->inc; }

static uint64_t nrm_next64(nrm_pcg *g) {
    nrm_step(g);
    g->draws++;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(g->state >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static double nrm_next_double(nrm_pcg *g) {
    return (double)(nrm_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

static const double ZIG_R = 3.6541528853610087963519472518;
static const double ZIG_INV_R = 0.27366123732975827203338247596;

static double nrm_one(nrm_pcg *g, const uint64_t *ki, const double *wi, const double *fi) {
    for (;;) {
        uint64_t r = nrm_next64(g);
        int idx = (int)(r & 0xff);
        r >>= 8;
        int sign = (int)(r & 0x1);
        uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * wi[idx];
        if (sign & 0x1) x = -x;
        if (rabs < ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                volatile double xx = -ZIG_INV_R * log1p(-nrm_next_double(g));
                volatile double yy = -log1p(-nrm_next_double(g));
                if (yy + yy > xx * xx)
                    return ((rabs >> 8) & 0x1) ? -(ZIG_R + xx) : ZIG_R + xx;
            }
        } else {
            volatile double lhs = (fi[idx - 1] - fi[idx]) * nrm_next_double(g);
            lhs = lhs + fi[idx];
            if (lhs < exp(-0.5 * x * x)) return x;
        }
    }
}

/* stream(entropy words).standard_normal(n); returns raw 64-bit draws consumed. */
int64_t or_standard_normal(const uint32_t *words, int nwords, int64_t n, const uint64_t *ki,
                           const double *wi, const double *fi, double *out) {
    uint64_t v[4];
    or_seedseq_state(words, nwords, v);
    nrm_pcg g;
    u128 initstate = ((u128)v[0] << 64) | v[1];
    u128 initseq = ((u128)v[2] << 64) | v[3];
    g.state = 0;
    g.inc = (initseq << 1) | 1u;
    g.draws = 0;
    nrm_step(&g);
    g.state += initstate;
    nrm_step(&g);
    for (int64_t i = 0; i < n; i++) out[i] = nrm_one(&g, ki, wi, fi);
    return g.draws;
}
