/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle (checker) for the octsca GPU path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj,
 * "octsca" 0.1.0). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, and only as the checker. The product library
 * (paper_1606_00310_b200/csrc/liboctgpu.so) never links or calls it.
 *
 * Pinning: tests/test_oracle.py checks every function here against
 *   (a) the golden vectors in tests/golden/ (generated from the unmodified
 *       reference by tests/golden/make_goldens.py, plus SURVEY.md Appendix A), and
 *   (b) the reference itself (oracle/_ref/libocref.so) when it is built.
 *
 * Storage convention = the reference's SlopeField (slope_field.hpp:15-53):
 * 4 planes in order x/even, x/odd, y/even, y/odd; each Y rows x n words,
 * row-major; n = X / (2w). Words are held in uint64_t; for w = 32 only the
 * low 32 bits are used (exactly the values of SlopeField<uint32_t>).
 */
#ifndef OCTORACLE_H
#define OCTORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OO_ZERO = 0, OO_HALF = 1, OO_DYADIC = 2, OO_ARBITRARY = 3 };

typedef struct {
    double r;
    int mode;
    uint32_t k;  /* dyadic: r = m / 2^k */
    uint64_t m;  /* dyadic: odd numerator */
} oo_prob;

/* rng.hpp:17-120 */
void oo_rng_from_seed(uint64_t seed, uint64_t st[4]);
uint64_t oo_rng_next(uint64_t st[4]);
void oo_rng_jump(uint64_t st[4]);
void oo_stream_set(uint64_t seed, uint32_t n, uint64_t* states);

/* rng.cpp:7-30, params.hpp:34-92 */
int oo_dyadic_plan(double r, uint32_t max_words, uint32_t* k, uint64_t* m);
int oo_resolve(double r, int forced, oo_prob* out); /* 0 ok, 1 ConfigError */
uint32_t oo_draws_per_word(const oo_prob* p, uint32_t w);
uint64_t oo_xi_word(uint64_t st[4], const oo_prob* p, uint32_t w);

/* slope_field.hpp:110-118 */
void oo_new_flat(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes);

/* engine_vec.hpp:98-177. Returns 0, or 2 on phase mismatch. */
int oo_sweep(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, uint64_t* states, int* phase, int parity,
             const oo_prob* p, const oo_prob* q, uint64_t* mask_log);
/* opt-in counter-based streams (include/octgpu.h octgpu_set_rng; no reference equivalent) */
uint64_t oo_ctr_draw(uint64_t seed, uint64_t sigma, uint32_t y, uint64_t i);
int oo_step_ctr(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, int* phase, uint64_t* t, const oo_prob* p,
                const oo_prob* q, uint64_t seed, uint64_t n_mcs);
int oo_step(uint32_t X, uint32_t Y, uint32_t w, uint64_t* planes, uint64_t* states, int* phase, uint64_t* t,
            const oo_prob* p, const oo_prob* q, uint64_t n_mcs);

/* Row-stripe form of detail::sweep_rows (engine_vec.hpp:98-137): the stripe
 * owns rows [y0, y1) (stripe_planes: 4 planes x (y1-y0) rows x n words,
 * states: (y1-y0) x 4) and borrows one ghost plane-row, y-plane of parity
 * !parity at row y1 mod Y, owned by the next stripe. Used by the multi-rank
 * CPU tests of the stripe protocol. */
void oo_sweep_stripe(uint32_t X, uint32_t Y, uint32_t w, uint32_t y0, uint32_t y1, uint64_t* stripe_planes,
                     uint64_t* ghost, uint64_t* states, int parity, const oo_prob* p, const oo_prob* q);

/* Fused MCS of a row stripe with 1 halo row above and 2 below (see .c) */
void oo_mcs_stripe(uint32_t X, uint32_t w, uint32_t R, uint32_t nsweeps, uint32_t yoff, uint64_t* planes,
                   uint64_t* states, int f, const oo_prob* p, const oo_prob* q);

/* slope_field.hpp:232-246 */
uint64_t oo_field_checksum(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint64_t t_mcs);
/* FNV-1a over per-row RNG states (SURVEY Appendix A digest) */
uint64_t oo_states_digest(const uint64_t* states, uint32_t n);

/* slope_field.hpp:159-174: number of violating plaquettes, first in scan order */
uint64_t oo_curl_check(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint32_t* fx, uint32_t* fy);
/* slope_field.hpp:206-229: 0 ok, 2 InvariantError (kind: 1 curl, 2 row0, 3 column; *where = column) */
int oo_reconstruct(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, int32_t* h, int* kind,
                   uint32_t* where);

/* Exact integer power sums S_k = sum h^k, k = 1..4, as (lo, hi) int128 halves */
void oo_power_sums(uint32_t X, uint32_t Y, const int32_t* h, uint64_t* out8);
/* reconstruct_heights + the exact power sums at scale (OpenMP; no HeightMap): see .c */
int oo_measure_planes_mt(uint32_t X, uint32_t Y, uint32_t w, const uint64_t* planes, uint64_t* out8, int* kind,
                         uint64_t* where, uint64_t* count);
/* measure.cpp:24-51 restated: {mean, m2, m3, m4, skew, kurt} in sequential double */
void oo_height_moments(uint32_t X, uint32_t Y, const int32_t* h, double* out6);
/* measure.cpp:143-165 */
uint32_t oo_log_schedule(uint64_t t_max, uint32_t ppd, uint64_t* out, uint32_t cap);

#ifdef __cplusplus
}
#endif
#endif
