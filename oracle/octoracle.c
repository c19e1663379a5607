/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the octsca GPU path. See
 * octoracle.h for the contract and how it is pinned. Each function cites the
 * reference lines (/root/reference/proj/...) whose behaviour it restates.
 * Deliberately simple, scalar and unoptimised: it is the checker.
 */
#include "octoracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

static inline uint64_t wmask(uint32_t w) { return w >= 64 ? ~(uint64_t)0 : (((uint64_t)1 << w) - 1); }
static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

/* ---- rng.hpp:25-32, 65-70 (splitmix64 seeding) ---- */
static uint64_t splitmix64(uint64_t* x) {
    uint64_t z = (*x += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void oo_rng_from_seed(uint64_t seed, uint64_t st[4]) {
    for (int i = 0; i < 4; ++i) st[i] = splitmix64(&seed);
    if ((st[0] | st[1] | st[2] | st[3]) == 0) st[0] = 1;
}

/* ---- rng.hpp:34-44 (xoshiro256++ next) ---- */
uint64_t oo_rng_next(uint64_t s[4]) {
    uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

/* ---- rng.hpp:47-60 (jump = 2^128 draws) ---- */
void oo_rng_jump(uint64_t s[4]) {
    static const uint64_t J[4] = {0x180ec6d33cfd0abaULL, 0xd5a61266f0c9392cULL, 0xa9582618e03fc9aaULL,
                                  0x39abdc4529b1661cULL};
    uint64_t acc[4] = {0, 0, 0, 0};
    for (int i = 0; i < 4; ++i)
        for (int b = 0; b < 64; ++b) {
            if (J[i] & ((uint64_t)1 << b))
                for (int j = 0; j < 4; ++j) acc[j] ^= s[j];
            oo_rng_next(s);
        }
    memcpy(s, acc, sizeof acc);
}

/* ---- rng.hpp:84-94 (stream i = i jumps from from_seed) ---- */
void oo_stream_set(uint64_t seed, uint32_t n, uint64_t* states) {
    uint64_t s[4];
    oo_rng_from_seed(seed, s);
    for (uint32_t i = 0; i < n; ++i) {
        memcpy(states + 4 * (size_t)i, s, sizeof s);
        if (i + 1 < n) oo_rng_jump(s);
    }
}

/* ---- rng.cpp:7-30 (dyadic plan) ---- */
int oo_dyadic_plan(double r, uint32_t max_words, uint32_t* k_out, uint64_t* m_out) {
    if (!(r > 0.0 && r < 1.0)) return 0;
    double scaled = ldexp(r, (int)max_words);
    if (scaled != floor(scaled)) return 0;
    uint64_t m = (uint64_t)scaled;
    uint32_t k = max_words;
    while (k > 0 && (m & 1) == 0) {
        m >>= 1;
        --k;
    }
    *k_out = k;
    *m_out = m;
    return 1;
}

/* ---- params.hpp:34-69 (ProbSpec::resolve, auto and forced) ---- */
static void resolve_auto(double r, oo_prob* o) {
    o->r = r;
    o->k = 0;
    o->m = 0;
    if (r == 0.0)
        o->mode = OO_ZERO;
    else if (r == 0.5)
        o->mode = OO_HALF;
    else if (oo_dyadic_plan(r, 16, &o->k, &o->m))
        o->mode = OO_DYADIC;
    else
        o->mode = OO_ARBITRARY;
}

int oo_resolve(double r, int forced, oo_prob* o) {
    if (r < 0.0 || r > 1.0) return 1;
    resolve_auto(r, o);
    if (forced < 0 || forced == o->mode) return 0;
    switch (forced) {
    case OO_ZERO:
        if (r != 0.0) return 1;
        break;
    case OO_HALF:
        if (r != 0.5) return 1;
        break;
    case OO_DYADIC:
        if (oo_dyadic_plan(r, 16, &o->k, &o->m)) {
            o->mode = OO_DYADIC;
            return 0;
        }
        return 1;
    case OO_ARBITRARY:
        if (r == 0.0) return 1;
        o->mode = OO_ARBITRARY;
        o->k = 0;
        o->m = 0;
        return 0;
    default:
        return 1;
    }
    return 0;
}

/* ---- params.hpp:72-80 ---- */
uint32_t oo_draws_per_word(const oo_prob* p, uint32_t w) {
    switch (p->mode) {
    case OO_ZERO: return 0;
    case OO_HALF: return 1;
    case OO_DYADIC: return p->k;
    default: return w;
    }
}

/* ---- opt-in counter-based streams (NOT in the reference; include/octgpu.h octgpu_set_rng):
 * SplitMix64's finaliser (the reference's seeding mixer, rng.hpp splitmix64) over a Weyl
 * sequence whose origin hashes (seed, global sweep sigma, row y). st[0] holds the Weyl value. */
#define OO_GAMMA 0x9E3779B97F4A7C15ull
static uint64_t oo_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t ctr_sweep_key(uint64_t seed, uint64_t sigma) { return oo_mix64(seed + (sigma + 1) * OO_GAMMA); }
static uint64_t ctr_row_origin(uint64_t key, uint32_t y) { return oo_mix64(key + ((uint64_t)y + 1) * OO_GAMMA); }
uint64_t oo_ctr_draw(uint64_t seed, uint64_t sigma, uint32_t y, uint64_t i) {
    return oo_mix64(ctr_row_origin(ctr_sweep_key(seed, sigma), y) + (i + 1) * OO_GAMMA);
}

/* one draw from a row's source: xoshiro state (ctr = 0) or Weyl counter in st[0] (ctr = 1) */
static uint64_t src_next(uint64_t st[4], int ctr) {
    if (!ctr) return oo_rng_next(st);
    st[0] += OO_GAMMA;
    return oo_mix64(st[0]);
}

/* ---- rng.hpp:135-179, params.hpp:84-92 (xi words) ---- */
static uint64_t xi_word_src(uint64_t st[4], const oo_prob* p, uint32_t w, int ctr) {
    switch (p->mode) {
    case OO_ZERO: return 0;
    case OO_HALF: return src_next(st, ctr) & wmask(w);
    case OO_DYADIC: {
        uint64_t acc = src_next(st, ctr) & wmask(w);
        for (uint32_t i = 1; i < p->k; ++i) {
            uint64_t xi = src_next(st, ctr) & wmask(w);
            acc = ((p->m >> i) & 1) ? (acc | xi) : (acc & xi);
        }
        return acc;
    }
    default: {
        uint64_t word = 0;
        for (uint32_t i = 0; i < w; ++i) {
            double u = (double)(src_next(st, ctr) >> 11) * 0x1.0p-53;
            word |= (uint64_t)(u < p->r) << i;
        }
        return word;
    }
    }
}

uint64_t oo_xi_word(uint64_t st[4], const oo_prob* p, uint32_t w) { return xi_word_src(st, p, w, 0); }

/* ---- slope_field.hpp:110-118 (flat start) ---- */
void oo_new_flat(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes) {
    size_t pw = (size_t)Y * (X / (2 * w));
    for (int p = 0; p < 4; ++p) {
        uint64_t v = (p & 1) ? wmask(w) : 0;
        for (size_t i = 0; i < pw; ++i) planes[p * pw + i] = v;
    }
}

/* ---- engine_vec.hpp:25-30 ---- */
static inline uint64_t update_mask(uint64_t sxm, uint64_t sym, uint64_t sxp, uint64_t syp, uint64_t xp,
                                   uint64_t xq) {
    uint64_t mp = xp & ~(sxm | sym) & sxp & syp;
    uint64_t mq = xq & ~(sxp | syp) & sxm & sym;
    return mp ^ mq;
}

/* Row accessor for a (possibly striped) lattice. */
typedef struct {
    uint32_t X, Y, w, n, y0, y1;
    uint64_t* planes; /* 4 planes x (y1-y0) rows */
    uint64_t* ghost;  /* row y1 mod Y of the y-plane of the other parity, or NULL if full lattice */
    uint32_t yoff;    /* global row of buffer row y is y + yoff (site parity uses the global row) */
} lat_t;

static uint64_t* row_of(const lat_t* L, int plane, uint32_t y) {
    size_t rows = L->y1 - L->y0;
    uint32_t ly = y - L->y0;
    if (ly == rows) {
        if (L->ghost) return L->ghost;
        ly = 0; /* full lattice: periodic wrap to row 0 */
    }
    return L->planes + (size_t)plane * rows * L->n + (size_t)ly * L->n;
}

/* ---- engine_vec.hpp:98-137 (detail::sweep_rows) ---- */
/* ctr = 0: row y draws from states[y - y0] (xoshiro); ctr = 1: from the counter stream of
 * sweep key `key` (states unused) */
static void sweep_range_src(const lat_t* L, int parity, const oo_prob* p, const oo_prob* q, uint64_t* states,
                            uint32_t ya, uint32_t yb, uint64_t* mask_log, int ctr, uint64_t key) {
    const uint32_t n = L->n, w = L->w;
    const uint64_t M = wmask(w);
    const int with_q = q->mode != OO_ZERO;
    uint64_t* xbuf = malloc(n * sizeof(uint64_t));
    uint64_t* mbuf = malloc(n * sizeof(uint64_t));
    for (uint32_t y = ya; y < yb; ++y) {
        uint64_t cst[4] = {0, 0, 0, 0};
        if (ctr) cst[0] = ctr_row_origin(key, y + L->yoff);
        uint64_t* st = ctr ? cst : states + 4 * (size_t)(y - L->y0);
        uint64_t* px = row_of(L, 0 * 2 + parity, y);
        uint64_t* py = row_of(L, 1 * 2 + parity, y);
        uint64_t* qy1 = row_of(L, 1 * 2 + (parity ^ 1), y + 1);
        uint64_t* raw = row_of(L, 0 * 2 + (parity ^ 1), y);
        const int shifted = ((uint32_t)parity ^ (y + L->yoff)) & 1u; /* engine_vec.hpp:59-61 */
        if (shifted) /* rotate_row_down, engine_vec.hpp:34-41 */
            for (uint32_t k = 0; k < n; ++k) {
                uint64_t nx = raw[k + 1 == n ? 0 : k + 1];
                xbuf[k] = ((raw[k] >> 1) | (nx << (w - 1))) & M;
            }
        else
            memcpy(xbuf, raw, n * sizeof(uint64_t));
        for (uint32_t k = 0; k < n; ++k) {
            uint64_t xp = xi_word_src(st, p, w, ctr);
            uint64_t xq = with_q ? xi_word_src(st, q, w, ctr) : 0;
            uint64_t m = update_mask(px[k], py[k], xbuf[k], qy1[k], xp, xq) & M;
            mbuf[k] = m;
            px[k] ^= m;
            py[k] ^= m;
            qy1[k] ^= m;
        }
        if (shifted) { /* scatter_rotated_xor, engine_vec.hpp:45-54 */
            uint64_t prev_top = mbuf[n - 1] >> (w - 1);
            for (uint32_t k = 0; k < n; ++k) {
                uint64_t cur = mbuf[k];
                raw[k] ^= ((cur << 1) | prev_top) & M;
                prev_top = cur >> (w - 1);
            }
        } else {
            for (uint32_t k = 0; k < n; ++k) raw[k] ^= mbuf[k];
        }
        if (mask_log) memcpy(mask_log + (size_t)y * n, mbuf, n * sizeof(uint64_t));
    }
    free(xbuf);
    free(mbuf);
}

static void sweep_range(const lat_t* L, int parity, const oo_prob* p, const oo_prob* q, uint64_t* states,
                        uint32_t ya, uint32_t yb, uint64_t* mask_log) {
    sweep_range_src(L, parity, p, q, states, ya, yb, mask_log, 0, 0);
}

static void sweep_rows(const lat_t* L, int parity, const oo_prob* p, const oo_prob* q, uint64_t* states,
                       uint64_t* mask_log) {
    sweep_range(L, parity, p, q, states, L->y0, L->y1, mask_log);
}

/* ---- engine_vec.hpp:145-168 (sublattice_sweep) ---- */
int oo_sweep(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, uint64_t* states, int* phase, int parity,
             const oo_prob* p, const oo_prob* q, uint64_t* mask_log) {
    if (*phase != parity) return 2;
    lat_t L = {X, Y, w, X / (2 * w), 0, Y, planes, NULL, 0};
    sweep_rows(&L, parity, p, q, states, mask_log);
    *phase ^= 1;
    return 0;
}

/* ---- engine_vec.hpp:171-177 (mcs_step) ---- */
int oo_step(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, uint64_t* states, int* phase, uint64_t* t,
            const oo_prob* p, const oo_prob* q, uint64_t n_mcs) {
    for (uint64_t i = 0; i < n_mcs; ++i) {
        oo_sweep(X, Y, w, planes, states, phase, *phase, p, q, NULL);
        oo_sweep(X, Y, w, planes, states, phase, *phase, p, q, NULL);
        ++*t;
    }
    return 0;
}

/* n MCS with the counter-based streams: sweeps phase then !phase, sigma = 2 t + 0 / 1 */
int oo_step_ctr(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, int* phase, uint64_t* t, const oo_prob* p,
                const oo_prob* q, uint64_t seed, uint64_t n_mcs) {
    lat_t L = {X, Y, w, X / (2 * w), 0, Y, planes, NULL, 0};
    for (uint64_t i = 0; i < n_mcs; ++i) {
        for (int h = 0; h < 2; ++h) {
            sweep_range_src(&L, *phase, p, q, NULL, 0, Y, NULL, 1, ctr_sweep_key(seed, 2 * *t + (uint64_t)h));
            *phase ^= 1;
        }
        ++*t;
    }
    return 0;
}

void oo_sweep_stripe(uint32_t X, uint32_t Y, uint32_t w, uint32_t y0, uint32_t y1, uint64_t* stripe_planes,
                     uint64_t* ghost, uint64_t* states, int parity, const oo_prob* p, const oo_prob* q) {
    lat_t L = {X, Y, w, X / (2 * w), y0, y1, stripe_planes, (y1 - y0 == Y) ? NULL : ghost, 0};
    sweep_rows(&L, parity, p, q, states, NULL);
}

/* ---- slope_field.hpp:232-246 (FNV-1a over planes then t_mcs) ---- */
static void fnv_mix(uint64_t* h, uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) {
        *h ^= (v >> (8 * i)) & 0xff;
        *h *= 0x100000001b3ULL;
    }
}

uint64_t oo_field_checksum(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint64_t t_mcs) {
    uint64_t h = 0xcbf29ce484222325ULL;
    size_t total = 4 * (size_t)Y * (X / (2 * w));
    /* mix(uint64_t(w)) widens each word to 8 bytes for both word sizes */
    for (size_t i = 0; i < total; ++i) fnv_mix(&h, planes[i], 8);
    fnv_mix(&h, t_mcs, 8);
    return h;
}

uint64_t oo_states_digest(const uint64_t* states, uint32_t n) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (size_t i = 0; i < 4 * (size_t)n; ++i) fnv_mix(&h, states[i], 8);
    return h;
}

/* ---- slope_field.hpp:59-64 (minus_bit) ---- */
static int minus_bit(const uint64_t* planes, uint32_t X, uint32_t Y, uint32_t w, int axis, uint32_t x,
                     uint32_t y) {
    uint32_t n = X / (2 * w);
    int par = (int)((x ^ y) & 1);
    uint32_t j = x >> 1;
    const uint64_t* r = planes + (size_t)(axis * 2 + par) * Y * n + (size_t)y * n;
    return (int)((r[j / w] >> (j % w)) & 1);
}

static inline int pm(int b) { return b ? 1 : -1; }

/* ---- slope_field.hpp:159-174 (curl_check) ---- */
uint64_t oo_curl_check(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint32_t* fx, uint32_t* fy) {
    uint64_t bad = 0;
    for (uint32_t y = 0; y < Y; ++y) {
        uint32_t ym = y == 0 ? Y - 1 : y - 1;
        for (uint32_t x = 0; x < X; ++x) {
            uint32_t xm = x == 0 ? X - 1 : x - 1;
            int lhs = pm(minus_bit(planes, X, Y, w, 0, x, y)) - pm(minus_bit(planes, X, Y, w, 0, x, ym));
            int rhs = pm(minus_bit(planes, X, Y, w, 1, x, y)) - pm(minus_bit(planes, X, Y, w, 1, xm, y));
            if (lhs != rhs) {
                if (bad == 0) {
                    *fx = x;
                    *fy = y;
                }
                ++bad;
            }
        }
    }
    return bad;
}

/* ---- slope_field.hpp:206-229 (reconstruct_heights) ---- */
int oo_reconstruct(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, int32_t* h, int* kind,
                   uint32_t* where) {
    uint32_t fx = 0, fy = 0;
    if (oo_curl_check(X, Y, w, planes, &fx, &fy)) {
        *kind = 1;
        *where = fy * X + fx;
        return 2;
    }
    memset(h, 0, (size_t)X * Y * sizeof(int32_t));
    for (uint32_t x = 1; x < X; ++x) h[x] = h[x - 1] + pm(minus_bit(planes, X, Y, w, 0, x, 0));
    if (h[X - 1] + pm(minus_bit(planes, X, Y, w, 0, 0, 0)) != h[0]) {
        *kind = 2;
        *where = 0;
        return 2;
    }
    for (uint32_t x = 0; x < X; ++x) {
        for (uint32_t y = 1; y < Y; ++y)
            h[(size_t)y * X + x] = h[(size_t)(y - 1) * X + x] + pm(minus_bit(planes, X, Y, w, 1, x, y));
        if (h[(size_t)(Y - 1) * X + x] + pm(minus_bit(planes, X, Y, w, 1, x, 0)) != h[x]) {
            *kind = 3;
            *where = x;
            return 2;
        }
    }
    *kind = 0;
    return 0;
}

void oo_power_sums(uint32_t X, uint32_t Y, const int32_t* h, uint64_t* out8) {
    i128 s[4] = {0, 0, 0, 0};
    size_t N = (size_t)X * Y;
    for (size_t i = 0; i < N; ++i) {
        i128 v = h[i];
        i128 v2 = v * v;
        s[0] += v;
        s[1] += v2;
        s[2] += v2 * v;
        s[3] += v2 * v2;
    }
    for (int k = 0; k < 4; ++k) {
        out8[2 * k] = (uint64_t)s[k];
        out8[2 * k + 1] = (uint64_t)((unsigned __int128)s[k] >> 64);
    }
}

/* ---- slope_field.hpp:159-229 + measure.cpp:24-51 at scale: the same reconstruction (curl_check, row 0
 * by its sigma_x- prefix and closure, every column by its sigma_y- walk from row 0 and closure), reduced
 * to the exact power sums without materialising the HeightMap; OpenMP over rows (curl) and over column
 * blocks (the column walks keep the reference's y order). For the at-scale parity tests (2^32+ sites),
 * where the scalar oo_reconstruct + oo_power_sums would need 16+ GiB and minutes. Returns 0, or 2 with
 * *kind = 1 curl (*where = y * X + x of the first bad plaquette, *count), 2 row 0, 3 column (*where). */
int oo_measure_planes_mt(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint64_t* out8, int* kind,
                         uint64_t* where, uint64_t* count) {
    uint64_t bad = 0, first = ~(uint64_t)0;
#pragma omp parallel for schedule(static) reduction(+ : bad) reduction(min : first)
    for (uint32_t y = 0; y < Y; ++y) {
        uint32_t ym = y == 0 ? Y - 1 : y - 1;
        for (uint32_t x = 0; x < X; ++x) {
            uint32_t xm = x == 0 ? X - 1 : x - 1;
            int lhs = pm(minus_bit(planes, X, Y, w, 0, x, y)) - pm(minus_bit(planes, X, Y, w, 0, x, ym));
            int rhs = pm(minus_bit(planes, X, Y, w, 1, x, y)) - pm(minus_bit(planes, X, Y, w, 1, xm, y));
            if (lhs != rhs) {
                uint64_t idx = (uint64_t)y * X + x;
                if (idx < first) first = idx;
                ++bad;
            }
        }
    }
    *count = bad;
    if (bad) {
        *kind = 1;
        *where = first;
        return 2;
    }
    int64_t* row0 = (int64_t*)malloc((size_t)X * sizeof(int64_t));
    row0[0] = 0;
    for (uint32_t x = 1; x < X; ++x) row0[x] = row0[x - 1] + pm(minus_bit(planes, X, Y, w, 0, x, 0));
    if (row0[X - 1] + pm(minus_bit(planes, X, Y, w, 0, 0, 0)) != row0[0]) {
        free(row0);
        *kind = 2;
        *where = 0;
        return 2;
    }
    const uint32_t CB = 256;  /* columns per task */
    const uint32_t nblk = (X + CB - 1) / CB;
    i128 S[4] = {0, 0, 0, 0};
    uint64_t col_bad = ~(uint64_t)0;
#pragma omp parallel
    {
        i128 s[4] = {0, 0, 0, 0};
        int64_t h[256];
        uint64_t cb = ~(uint64_t)0;
#pragma omp for schedule(dynamic, 1)
        for (uint32_t b = 0; b < nblk; ++b) {
            uint32_t xa = b * CB, xb = xa + CB < X ? xa + CB : X;
            for (uint32_t x = xa; x < xb; ++x) h[x - xa] = row0[x];
            for (uint32_t y = 0; y < Y; ++y) {
                int64_t s1 = 0;
                i128 s2 = 0, s3 = 0, s4 = 0;
                for (uint32_t x = xa; x < xb; ++x) {
                    if (y) h[x - xa] += pm(minus_bit(planes, X, Y, w, 1, x, y));
                    i128 v = h[x - xa], v2 = v * v;
                    s1 += h[x - xa];
                    s2 += v2;
                    s3 += v2 * v;
                    s4 += v2 * v2;
                }
                s[0] += s1;
                s[1] += s2;
                s[2] += s3;
                s[3] += s4;
            }
            for (uint32_t x = xa; x < xb; ++x)
                if (h[x - xa] + pm(minus_bit(planes, X, Y, w, 1, x, 0)) != row0[x] && x < cb) cb = x;
        }
#pragma omp critical
        {
            for (int k = 0; k < 4; ++k) S[k] += s[k];
            if (cb < col_bad) col_bad = cb;
        }
    }
    free(row0);
    if (col_bad != ~(uint64_t)0) {
        *kind = 3;
        *where = col_bad;
        return 2;
    }
    for (int k = 0; k < 4; ++k) {
        out8[2 * k] = (uint64_t)S[k];
        out8[2 * k + 1] = (uint64_t)((unsigned __int128)S[k] >> 64);
    }
    *kind = 0;
    return 0;
}

/* ---- measure.cpp:24-51 (height_moments, sequential double) ---- */
void oo_height_moments(uint32_t X, uint32_t Y, const int32_t* h, double* out6) {
    size_t N = (size_t)X * Y;
    double n = (double)N, mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0, skew, kurt;
    for (size_t i = 0; i < N; ++i) mean += h[i];
    mean /= n;
    for (size_t i = 0; i < N; ++i) {
        double d = h[i] - mean;
        double d2 = d * d;
        m2 += d2;
        m3 += d2 * d;
        m4 += d2 * d2;
    }
    m2 /= n;
    m3 /= n;
    m4 /= n;
    if (m2 > 0.0) {
        skew = m3 / pow(m2, 1.5);
        kurt = m4 / (m2 * m2) - 3.0;
    } else {
        skew = NAN;
        kurt = NAN;
    }
    out6[0] = mean; out6[1] = m2; out6[2] = m3; out6[3] = m4; out6[4] = skew; out6[5] = kurt;
}

/* ---- measure.cpp:143-165 (log_schedule) ---- */
uint32_t oo_log_schedule(uint64_t t_max, uint32_t ppd, uint64_t* out, uint32_t cap) {
    if (t_max < 1 || ppd < 1) return 0;
    uint32_t cnt = 0;
    uint64_t prev = 0;
    for (uint32_t k = 0;; ++k) {
        double exact = pow(10.0, (double)k / (double)ppd);
        if (exact > (double)t_max * (1.0 + 1e-12)) break;
        uint64_t t = (uint64_t)llround(exact);
        if (t <= prev) t = prev + 1;
        if (t > t_max) break;
        if (cnt < cap) out[cnt] = t;
        ++cnt;
        prev = t;
    }
    if (cnt == 0 || (cnt <= cap && out[cnt - 1] != t_max) || (cnt > cap && prev != t_max)) {
        if (cnt < cap) out[cnt] = t_max;
        ++cnt;
    }
    return cnt;
}

/* k MCS (2k sweeps f, f^1, ...) of a row stripe held with halos, as the GPU
 * multi-stripe path organises it (not a reference function; built from
 * sweep_range, so it is exactly the reference's sweeps restricted to the rows
 * the stripe can complete): R = L + HA + HB buffer rows (HA = 5, HB = 6 on the
 * GPU path), 0..HA-1 halo above, HA..HA+L-1 own, then the halo below. Sweep i
 * (1-based) runs on rows [i-1, R-i): each sweep needs the previous one on rows
 * y-1..y+1, so the valid band shrinks by one row per side; sweep 2k <= HA + 1
 * still covers the own rows. Afterwards the own rows are final except y-plane f
 * of row HA (completed by the previous stripe's boundary row), and y-plane f of
 * row HA+L is the boundary row for the next stripe. yoff = global row of buffer
 * row 0 (= y0 - HA mod Y). */
void oo_mcs_stripe(uint32_t X, uint32_t w, uint32_t R, uint32_t nsweeps, uint32_t yoff, uint64_t* planes,
                   uint64_t* states, int f, const oo_prob* p, const oo_prob* q) {
    lat_t Lt = {X, R, w, X / (2 * w), 0, R, planes, NULL, yoff};
    for (uint32_t i = 1; i <= nsweeps; ++i) sweep_range(&Lt, f ^ (int)((i - 1) & 1), p, q, states, i - 1, R - i, NULL);
}
