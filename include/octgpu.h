/*
 * octgpu — C-ABI of the B200-native bit-vectorized octahedron-model SCA.
 *
 * This is the drop-in boundary for the reference engine
 * `octsca::VecEngine<Word>` (/root/reference/proj/include/octsca/engine_vec.hpp:184-213)
 * as consumed by `octsca::run` (run.hpp:18-38) and `run_session`'s `drive`
 * (session.cpp:37-85). Plain pointers and sizes only; no C++ or torch types.
 * Every entry point names the reference interface it replaces.
 *
 * Conventions
 *  - Plane buffers on the host side use the reference SlopeField layout
 *    (slope_field.hpp:15-53, 207-210): 4 planes in order x/even, x/odd,
 *    y/even, y/odd; each Y rows x n words, row-major; n = X / (2w); words
 *    are uint64_t for w = 64 and uint32_t for w = 32, LSB-first, bit 1 =
 *    slope +1.
 *  - RNG states: one xoshiro256++ state (4 x uint64_t) per lattice row, in
 *    row order (RngStreamSet::states(), rng.hpp:102-108).
 *  - Errors: every function returning int returns an octgpu_status; the
 *    message of the last failure on the calling thread is available from
 *    octgpu_last_error(). The codes map 1:1 to the reference exceptions
 *    (errors.hpp:8-25; CLI exit codes SPEC.md:475). There is NO CPU
 *    fallback: if CUDA is unavailable the call fails with OCTGPU_ERR_CUDA.
 *  - Engines are not thread-safe (same as VecEngine). All work is enqueued
 *    on the engine's CUDA stream; calls that return data synchronise.
 */
#ifndef OCTGPU_H
#define OCTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    OCTGPU_OK = 0,
    OCTGPU_ERR_CONFIG = 1,    /* octsca::ConfigError    (errors.hpp:8-12)  */
    OCTGPU_ERR_INVARIANT = 2, /* octsca::InvariantError (errors.hpp:14-19) */
    OCTGPU_ERR_IO = 3,        /* octsca::IoError        (errors.hpp:21-25) */
    OCTGPU_ERR_CUDA = 4       /* device/runtime failure (no reference analogue) */
} octgpu_status;

/* octsca::ProbMode (params.hpp:13) */
typedef enum { OCTGPU_ZERO = 0, OCTGPU_HALF = 1, OCTGPU_DYADIC = 2, OCTGPU_ARBITRARY = 3 } octgpu_mode;

/* octsca::ProbSpec (params.hpp:28-44): value + generation mode (+ DyadicPlan
 * rng.hpp:142-151 as r = m / 2^k with m odd; ops follow the bits of m). */
typedef struct {
    double value;
    int32_t mode;
    uint32_t k;
    uint64_t m;
} octgpu_prob;

/* octsca::UpdateParams (params.hpp:95-102) */
typedef struct {
    octgpu_prob p;
    octgpu_prob q;
} octgpu_params;

/* MeasurementRecord (measure.hpp:11-17) plus the exact integer sufficient
 * statistics it is derived from: S_k = sum_{x,y} h(x,y)^k with the
 * reference's gauge h(0,0) = 0 (slope_field.hpp:214), as two's-complement
 * int128 split into (lo, hi). */
typedef struct {
    uint64_t t;
    uint64_t n_sites;
    uint64_t s_lo[4];
    int64_t s_hi[4];
    double W2;
    double mean_h;
    double skew;
    double kurt;
} octgpu_moments;

typedef struct octgpu_engine octgpu_engine;

/* ---- host-side parameter plumbing (no GPU needed) ---- */

/* ProbSpec::resolve(r) when forced_mode < 0, else ProbSpec::resolve(r, forced)
 * (params.hpp:34-69, dyadic_plan rng.cpp:7-30). */
int octgpu_resolve(double r, int forced_mode, octgpu_prob* out);
/* ProbSpec::draws_per_word (params.hpp:72-80) */
uint32_t octgpu_draws_per_word(const octgpu_prob* p, uint32_t w);
/* LatticeConfig::validate (lattice.hpp:31-39) */
int octgpu_validate_lattice(uint32_t X, uint32_t Y, uint32_t w);
/* RngStreamSet(master_seed, n).states() (rng.hpp:84-94, 102-108) into out[n*4] */
int octgpu_stream_states(uint64_t master_seed, uint32_t n, uint64_t* out);
/* log_schedule (measure.cpp:143-165); returns the number of points, writes up to cap */
uint32_t octgpu_log_schedule(uint64_t t_max, uint32_t points_per_decade, uint64_t* out, uint32_t cap);

/* height_moments (measure.cpp:24-51) over a host HeightMap (row-major int32),
 * restated with the reference's sequential double accumulation so results are
 * bit-identical: out = {mean, m2, m3, m4, skew, kurt}. */
void octgpu_height_moments(uint32_t X, uint32_t Y, const int32_t* h, double* out6);

/* ---- engine lifecycle ---- */

/* VecEngine(LatticeConfig{X,Y,w}, seed, workers) (engine_vec.hpp:187-189):
 * new_flat field (slope_field.hpp:110-118), RngStreamSet(seed, Y). */
int octgpu_create(uint32_t X, uint32_t Y, uint32_t w, uint64_t seed, int device, octgpu_engine** out);
/* VecEngine(SlopeField, RngStreamSet, workers) (engine_vec.hpp:191-193) —
 * resume from any state, including phase = 1 (mid-MCS). planes: host,
 * reference layout; states: host, n_states >= Y rows of 4 words. */
int octgpu_create_from(uint32_t X, uint32_t Y, uint32_t w, uint64_t t_mcs, int phase, const void* planes,
                       const uint64_t* states, uint32_t n_states, uint64_t master_seed, int device,
                       octgpu_engine** out);
void octgpu_destroy(octgpu_engine* e);
/* Replace the whole state of an existing engine (same geometry): the write-back
 * half of VecEngine's mutable field()/streams() accessors (engine_vec.hpp:200-214). */
int octgpu_set_state(octgpu_engine* e, uint64_t t_mcs, int phase, const void* planes, const uint64_t* states,
                     uint32_t n_states);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream); NULL restores the engine's own. */
int octgpu_set_stream(octgpu_engine* e, void* cuda_stream);
/* Block until all enqueued work finished; surfaces asynchronous CUDA errors. */
int octgpu_sync(octgpu_engine* e);
/* Periodic engines take their two plane sets from a library-private stream-ordered pool
 * (cudaMemPoolCreate) that keeps freed memory for the next engine of the process (no
 * re-mapping on resume / re-creation). This returns the pool's unused memory on `device`
 * to the driver (for cudaMalloc, PyTorch, NCCL). No reference counterpart. */
int octgpu_release_pool(int device);

/* ---- the hot path ---- */

/* n_mcs x VecEngine::step(prm) = mcs_step (engine_vec.hpp:171-177, 197). */
int octgpu_step(octgpu_engine* e, const octgpu_params* prm, uint64_t n_mcs);
/* sublattice_sweep(field, parity, prm, plan, streams, mask_log)
 * (engine_vec.hpp:145-168). mask_log: NULL or host buffer of Y*n words
 * (reference row-major), receives the applied mask of every (row, word). */
int octgpu_sweep(octgpu_engine* e, int parity, const octgpu_params* prm, void* mask_log);
/* Random tile-origin shifts (DTr-style, BASELINE.json north_star): seed != 0 moves the row origin of the
 * kernels' block tiling by a pseudo-random offset every pass (periodic lattices, TMA kernels); 0 = off.
 * Result-neutral: sites of one sublattice share no slopes (engine_vec.hpp:95-97). */
int octgpu_set_tile_shift(octgpu_engine* e, uint64_t seed);

/* xi source of octgpu_step. OCTGPU_RNG_XOSHIRO (default): the reference's per-row
 * xoshiro256++ streams (rng.hpp:17-124), bit-exact with VecEngine. OCTGPU_RNG_COUNTER:
 * opt-in counter-based streams with NO reference equivalent (BASELINE north_star,
 * SURVEY.md 8f row 4): draw i of row y in global sweep sigma = 2 t + (0 | 1) is
 * mix64(o + (i+1) g), o = mix64(mix64(seed + (sigma+1) g) + (y+1) g), g = 0x9E3779B97F4A7C15,
 * mix64 = the SplitMix64 finaliser; seed = octgpu_master_seed. The xi words are built from
 * these draws exactly as from xoshiro draws (half / dyadic / arbitrary); y is the GLOBAL row,
 * so row stripes (w = 64, >= 8 words per row; set the same kind on every stripe) reproduce the
 * periodic engine. Counter steps leave the xoshiro states untouched; single sweeps
 * (octgpu_sweep) are xoshiro-only (OCTGPU_ERR_CONFIG). Results are pinned by
 * oracle/octoracle.c oo_step_ctr. */
#define OCTGPU_RNG_XOSHIRO 0
#define OCTGPU_RNG_COUNTER 1
int octgpu_set_rng(octgpu_engine* e, int kind);
int octgpu_get_rng(const octgpu_engine* e);

/* The fused pass octgpu_step (or, on a row stripe, octgpu_stripe_max_mcs) launches for prm on this engine:
 * *kernel = OCTGPU_KERNEL_* and *sweeps_per_launch = sublattice sweeps one full-length launch covers (2 per
 * MCS: 6 for a 3-MCS k_mcs_deep pass, 2 for the one-MCS kernels, 1 for in-place sweeps). No reference
 * counterpart (the reference's sweeps are OpenMP loops); used by benchmarks to attribute kernel time. */
#define OCTGPU_KERNEL_MCS 0   /* k_mcs: register-prefetch one-MCS pass */
#define OCTGPU_KERNEL_BULK 1  /* k_mcs_bulk: TMA one-MCS pass */
#define OCTGPU_KERNEL_DEEP 2  /* k_mcs_deep: TMA, temporally blocked (2 or 3 MCS per pass) */
#define OCTGPU_KERNEL_SWEEP 3 /* k_sweep_ctr: one in-place sweep */
int octgpu_pass_plan(octgpu_engine* e, const octgpu_params* prm, int* kernel, int* sweeps_per_launch);

/* ---- state access ---- */

uint64_t octgpu_t(const octgpu_engine* e);         /* VecEngine::t (engine_vec.hpp:199) */
int octgpu_phase(const octgpu_engine* e);          /* SlopeField::phase (slope_field.hpp:44) */
uint64_t octgpu_master_seed(const octgpu_engine* e); /* RngStreamSet::master_seed (rng.hpp:97) */
/* VecEngine::field() planes (engine_vec.hpp:200-201), reference layout, 4*Y*n words */
int octgpu_get_planes(octgpu_engine* e, void* out);
/* VecEngine::streams().states() (rng.hpp:102-108), Y*4 words */
int octgpu_get_states(octgpu_engine* e, uint64_t* out);
/* field_checksum(field()) (slope_field.hpp:232-246). On a row stripe: the same FNV-1a over the
 * stripe's own rows (4 planes x L rows, reference layout) then t, i.e. the checksum of the stripe as an
 * L-row field (a per-stripe correctness digest; sync the whole group first). */
int octgpu_field_checksum(octgpu_engine* e, uint64_t* out);

/* ---- measurement ---- */

/* measure_heights(t(), heights()) (run.hpp:28, measure.cpp:53-56) computed on
 * the device without materialising the HeightMap: curl_check + closure checks
 * as reconstruct_heights (slope_field.hpp:206-229, same InvariantError
 * messages), exact int128 power sums, doubles derived from them. */
int octgpu_measure(octgpu_engine* e, octgpu_moments* out);
/* VecEngine::heights() = reconstruct_heights(field) (engine_vec.hpp:207):
 * out[y*X + x] int32, h(0,0) = 0. */
int octgpu_heights(octgpu_engine* e, int32_t* out);
/* row_balances(field) / col_balances(field) (slope_field.hpp:177-202): rows_out[y] =
 * sum_x sigma_x-(x,y) (Y entries), cols_out[x] = sum_y sigma_y-(x,y) (X entries); either
 * pointer may be NULL. On a row stripe: its own rows (rows_out: L entries, global rows
 * y0..y0+L-1) and column sums over them (the lattice's col_balances = the sum over stripes). */
int octgpu_balances(octgpu_engine* e, int64_t* rows_out, int64_t* cols_out);

/* ---- row stripes (multi-GPU) ----
 * A stripe engine owns global rows [y0, y1) (at least 4) of an X x Y periodic
 * lattice (sublattice partition as the reference's SweepPlan row blocks,
 * params.hpp:107-127; results do not depend on the partition). One pass of
 * k = 1 MCS (or k = octgpu_stripe_max_mcs(), 3 for constant xi: the
 * temporally blocked kernel):
 *   octgpu_halo_pack -> exchange (to_prev -> rank-1, to_next -> rank+1) ->
 *   octgpu_halo_unpack -> octgpu_stripe_mcs_n(k) -> exchange boundary (-> rank+1) ->
 *   octgpu_stripe_finish.
 * to_prev carries the stripe's first 4 rows, to_next its last 3 (4 plane-rows
 * + the row's xoshiro state each); boundary is one plane-row.
 * All buffers are DEVICE memory (e.g. NCCL send/recv buffers); all work is on
 * the engine's stream. octgpu_get_planes / octgpu_get_states return the
 * stripe's own rows. planes/states NULL = flat start, RngStreamSet(seed, Y)
 * rows y0..y1-1. */
typedef struct {
    uint64_t t;
    uint64_t n_sites;
    uint64_t s_lo[4]; /* power sums in the stripe-local gauge (h = 0 at column 0 above row y0) */
    int64_t s_hi[4];
    int64_t col_sum;       /* sum of sigma_y-(0, y) over the stripe's rows */
    int64_t sy_first;      /* sigma_y-(0, y0) */
    int64_t row_first_sum; /* sum_x sigma_x-(x, y0) */
    uint64_t curl_count;
    uint64_t curl_first;   /* global y * X + x of the first violation, ~0 if none */
} octgpu_stripe_moments;

int octgpu_create_stripe(uint32_t X, uint32_t Y, uint32_t w, uint32_t y0, uint32_t y1, uint64_t t_mcs, int phase,
                         const void* planes, const uint64_t* states, uint64_t master_seed, int device,
                         octgpu_engine** out);
int octgpu_stripe_sizes(const octgpu_engine* e, uint64_t* to_prev_bytes, uint64_t* to_next_bytes,
                        uint64_t* boundary_bytes);
int octgpu_halo_pack(octgpu_engine* e, void* to_prev, void* to_next);
int octgpu_halo_unpack(octgpu_engine* e, const void* from_prev, const void* from_next);
int octgpu_stripe_mcs(octgpu_engine* e, const octgpu_params* prm, void* boundary_out); /* k = 1 */
int octgpu_stripe_mcs_n(octgpu_engine* e, const octgpu_params* prm, uint32_t n_mcs, void* boundary_out);
/* largest n_mcs one pass may take for these parameters (1 or 2); 0 on error */
int octgpu_stripe_max_mcs(octgpu_engine* e, const octgpu_params* prm);
int octgpu_stripe_finish(octgpu_engine* e, const void* boundary_in);
/* local moments; needs fresh halos (pack/exchange/unpack) for the curl check of row y0 */
int octgpu_measure_stripe(octgpu_engine* e, octgpu_stripe_moments* out);
/* Global measure_heights from the stripes' local moments, in row order (parts[0] holds row 0):
 * reconstruct_heights' checks (curl, row 0, column 0; InvariantError messages as the periodic
 * engine) and the exact int128 sums shifted binomially by the column-0 prefix of the stripes
 * above. Host-only (no GPU). */
int octgpu_stripes_combine(const octgpu_stripe_moments* parts, uint32_t n_parts, uint32_t X, uint32_t Y,
                           octgpu_moments* out);
uint32_t octgpu_stripe_y0(const octgpu_engine* e);
uint32_t octgpu_stripe_rows(const octgpu_engine* e);

/* ---- device-side halo exchange over peer memory (NVLink P2P / same GPU) ----
 * Replaces pack -> NCCL -> unpack -> boundary -> finish with kernels that read
 * the neighbours' rows and write the boundary plane-row directly in their
 * memory, synchronised by per-stripe "passes done" counters in device memory
 * (no host round trip, no NCCL). Stripes must step in lockstep (same number of
 * passes with the same k). Needs w = 64 and X >= 1024 (the TMA kernels).
 *   octgpu_stripe_peer        this stripe's device memory, as seen by this process
 *   octgpu_stripe_ipc_export  the same as a CUDA IPC blob (OCTGPU_IPC_BYTES) for another process
 *   octgpu_stripe_ipc_open    map a neighbour's blob into this process
 *   octgpu_stripe_connect     set the ring neighbours (the same peer twice for 2 stripes) and pull the
 *                             initial halo rows with their xoshiro states
 *   octgpu_stripe_pass        one pass of n_mcs (1, or 2 with constant xi): pull -> MCS -> push + signal
 *   octgpu_stripe_pull        refresh the halo rows (before octgpu_measure_stripe)
 *   octgpu_stripe_disconnect  unmap the neighbours (every rank, then a barrier, before any rank frees its stripe)
 * A neighbour that stops stepping makes the waits time out (~10 s): the next
 * octgpu_measure_stripe / octgpu_sync reports OCTGPU_ERR_CUDA. */
#define OCTGPU_IPC_BYTES 512
typedef struct {
    uint64_t planes[2]; /* device addresses of the two plane sets */
    uint64_t rng[2];    /* device addresses of the two rng-state sets */
    uint64_t done;      /* device address of the passes-done counter */
    uint32_t alloc_rows;
    uint32_t rows;
    uint32_t n;
    uint32_t w;
    int32_t device;
    int32_t pad;
} octgpu_peer;
int octgpu_stripe_peer(const octgpu_engine* e, octgpu_peer* out);
int octgpu_stripe_ipc_export(const octgpu_engine* e, void* out);
int octgpu_stripe_ipc_open(octgpu_engine* e, const void* blob, octgpu_peer* out);
int octgpu_stripe_connect(octgpu_engine* e, const octgpu_peer* prev, const octgpu_peer* next);
int octgpu_stripe_pass(octgpu_engine* e, const octgpu_params* prm, uint32_t n_mcs);
int octgpu_stripe_pull(octgpu_engine* e);
int octgpu_stripe_disconnect(octgpu_engine* e);

/* ---- diagnostics ---- */
const char* octgpu_last_error(void);
const char* octgpu_version(void);
/* Number of kernel launches this engine has issued (for launch accounting). */
uint64_t octgpu_launch_count(const octgpu_engine* e);

#ifdef __cplusplus
}
#endif
#endif /* OCTGPU_H */
