/*
 * oracle/countsketch.c -- TEST INFRASTRUCTURE ONLY (CPU checker, never shipped,
 * never on the product path).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's build.
 *
 * Plain-C restatement of the CountSketch construction the reference performs in
 *   /root/reference/pkg/src/skpower/sketching.py:114-124  (SketchOperator.__init__)
 *   /root/reference/pkg/src/skpower/sketching.py:141-150  (_draw_countsketch)
 * The arithmetic lives in numpy 2.3.5 (third-party, not vendored in the
 * reference).  Restated here from numpy's published algorithms:
 *   - PCG64 = PCG "XSL-RR 128/64": state' = state * M + inc (mod 2^128),
 *     output = rotr64(hi(state') ^ lo(state'), hi(state') >> 58)  [O'Neill 2014]
 *   - Generator.random(): (u64 >> 11) * 2^-53
 *   - np.argpartition(keys, s-1)[:, :s]: the s smallest keys; the order of the
 *     first s entries is ascending-key on numpy 2.3.5 (SURVEY.md §7 hard part 2;
 *     pinned by tests/golden against the live reference).
 *   - Generator.integers(0, R): Lemire's nearly-divisionless bounded draw on
 *     32-bit values; PCG64's next_uint32 returns the low half of a 64-bit draw
 *     and keeps the high half in the BIT GENERATOR (has_uint32 / uinteger),
 *     so the buffer persists across integers() calls: after an odd number of
 *     32-bit column draws (s == 1) the first sign is that buffered half.
 *     64-bit draws (random()) neither use nor clear it.
 * Ties between equal 53-bit keys are broken by the lower column index.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static const u128 PCG_MULT =
    (((u128)2549297995355413924ULL) << 64) | (u128)4865540595714422341ULL;

typedef struct {
    u128 state;
    u128 inc;
    /* PCG64's 32-bit buffer (numpy pcg64_state.has_uint32 / uinteger):
     * part of the bit generator, persists across integers() calls */
    uint64_t buf;
    int bcnt;
} pcg64_t;

static inline uint64_t pcg64_next(pcg64_t* g) {
    g->state = g->state * PCG_MULT + g->inc;
    uint64_t hi = (uint64_t)(g->state >> 64), lo = (uint64_t)g->state;
    unsigned rot = (unsigned)(hi >> 58);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
}

static inline uint32_t buffered_u32(pcg64_t* g) {
    if (!g->bcnt) {
        g->buf = pcg64_next(g);
        g->bcnt = 1;
    } else {
        g->buf >>= 32;
        g->bcnt = 0;
    }
    return (uint32_t)g->buf;
}

/* Lemire bounded draw in [0, rng] with rng < 2^32-1 (numpy's
 * buffered_bounded_lemire_uint32). */
static inline uint32_t lemire_u32(pcg64_t* g, uint32_t rng) {
    uint32_t excl = rng + 1u;
    uint64_t m = (uint64_t)buffered_u32(g) * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
        uint32_t thr = (uint32_t)(0u - excl) % excl;
        while (left < thr) {
            m = (uint64_t)buffered_u32(g) * excl;
            left = (uint32_t)m;
        }
    }
    return (uint32_t)(m >> 32);
}

/* Generator.integers(0, hi, size=cnt) into out[] (int64 path, use_masked=False). */
static void integers_fill(pcg64_t* g, uint64_t hi, int64_t cnt, int64_t* out) {
    uint64_t rng = hi - 1;
    if (rng == 0) {
        for (int64_t i = 0; i < cnt; ++i) out[i] = 0;
        return;
    }
    for (int64_t i = 0; i < cnt; ++i) out[i] = (int64_t)lemire_u32(g, (uint32_t)rng);
}

/* Advance a PCG64 state by delta steps (numpy BitGenerator.advance). */
void skpo_pcg64_advance(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                        uint64_t delta, uint64_t* out_hi, uint64_t* out_lo) {
    u128 acc_m = 1, acc_p = 0, cur_m = PCG_MULT;
    u128 cur_p = ((u128)inc_hi << 64) | inc_lo;
    u128 st = ((u128)st_hi << 64) | st_lo;
    while (delta) {
        if (delta & 1u) {
            acc_m *= cur_m;
            acc_p = acc_p * cur_m + cur_p;
        }
        cur_p = (cur_m + 1) * cur_p;
        cur_m *= cur_m;
        delta >>= 1;
    }
    st = acc_m * st + acc_p;
    *out_hi = (uint64_t)(st >> 64);
    *out_lo = (uint64_t)st;
}

/* First `cnt` raw 64-bit outputs (for known-answer tests of the generator). */
void skpo_pcg64_raw(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                    int64_t cnt, uint64_t* out) {
    pcg64_t g = {((u128)st_hi << 64) | st_lo, ((u128)inc_hi << 64) | inc_lo, 0, 0};
    for (int64_t i = 0; i < cnt; ++i) out[i] = pcg64_next(&g);
}

/* _draw_countsketch(rng, n, r, s): cols (n*s, int64) and signs (n*s, int8 +-1).
 * Returns 0 on success, 1 on bad arguments. */
int skpo_countsketch(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                     int64_t n, int64_t r, int32_t s, int64_t* cols, int8_t* signs) {
    if (n < 1 || r < 1 || s < 1 || s > r || r > 0xFFFFFFFFLL) return 1;
    pcg64_t g = {((u128)st_hi << 64) | st_lo, ((u128)inc_hi << 64) | inc_lo, 0, 0};
    if (s == 1) {
        /* rng.integers(0, r, size=(n, 1)) -- sketching.py:144 */
        integers_fill(&g, (uint64_t)r, n, cols);
    } else {
        /* rng.random((n, r)) then argpartition(keys, s-1)[:, :s] -- sketching.py:147-148 */
        uint64_t* best = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)s);
        int64_t* bidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)s);
        if (!best || !bidx) { free(best); free(bidx); return 1; }
        for (int64_t j = 0; j < n; ++j) {
            int cnt = 0;
            for (int64_t c = 0; c < r; ++c) {
                uint64_t key = pcg64_next(&g) >> 11;
                if (cnt == s && key >= best[s - 1]) continue;
                int p = cnt < s ? cnt++ : s - 1;
                while (p > 0 && best[p - 1] > key) {
                    best[p] = best[p - 1];
                    bidx[p] = bidx[p - 1];
                    --p;
                }
                best[p] = key;
                bidx[p] = c;
            }
            memcpy(cols + j * s, bidx, sizeof(int64_t) * (size_t)s);
        }
        free(best);
        free(bidx);
    }
    /* rng.integers(0, 2, size=(n, s)) * 2 - 1 -- sketching.py:149 */
    int64_t tot = n * (int64_t)s;
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)tot);
    if (!tmp) return 1;
    integers_fill(&g, 2, tot, tmp);
    for (int64_t e = 0; e < tot; ++e) signs[e] = (int8_t)(tmp[e] * 2 - 1);
    free(tmp);
    return 0;
}
