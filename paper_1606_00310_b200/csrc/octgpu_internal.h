// Internal declarations shared by the host engine (engine.cu) and the device
// kernels (kernels.cu). Not part of the C-ABI; see include/octgpu.h for that.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace octgpu {

// Per-probability generation mode as the device sees it. ZERO/HALF/DYADIC/ARB
// mirror octsca::ProbMode (params.hpp:13); ONE is ARB with r == 1, whose xi is
// the all-ones word (to_unit(x) < 1.0 always holds, rng.hpp:167-177) while the
// stream still advances w draws per word.
enum Mode : int { M_ZERO = 0, M_HALF = 1, M_DYADIC = 2, M_ARB = 3, M_ONE = 4 };

struct ProbDev {
    int mode;
    uint32_t k;   // dyadic: r = m / 2^k, ops from bit 1 of m upward (rng.cpp:24-28)
    uint64_t m;
    uint64_t T;   // ARB: xi bit = (draw < T), T = ceil(r * 2^53) << 11
};

// Device layout ("word-major"): plane p, row y, word k lives at
//   base + p * plane_stride + k * Y + y
// so a warp whose lanes own 32 consecutive rows touches one contiguous 256-B
// (w=64) segment per plane per word: every access is coalesced and any
// contiguous window of rows is contiguous in memory.
//
// Rows are addressed through a "virtual" row index v: the kernels compute the
// rows v in [c0, c1) ("core" rows) and may read the rows just outside that
// range; physical row = wrap ? v % wrap : v. A full periodic lattice is
// {Y = lattice rows, c0 = 1, c1 = Y + 1, wrap = Y}; a row stripe of L rows
// held with one halo row above and two below (plus padding) is
// {Y = allocated rows, c0 = 1, c1 = L + 1, wrap = 0}.
struct Geom {
    uint32_t Y;            // rows stored per plane (row stride in words)
    uint32_t n;            // words per plane-row = X / (2w)
    size_t plane_stride;   // n * Y words
    uint32_t c0, c1;       // core rows (virtual)
    uint32_t wrap;         // periodic modulus in y, or 0
    uint32_t ypar;         // parity of the global row of physical row 0 (site parity uses global rows)
    uint32_t ghost;        // periodic: rows wrap..wrap+ghost-1 mirror rows (i mod wrap), so block windows never wrap
    uint32_t pf = 0;       // TMA kernels: L2 prefetch distance in ring stages (0 = off)
    // counter-based rng: global row of physical row r = (r + gy0) mod gytot (gytot = 0: r itself)
    uint32_t gy0 = 0, gytot = 0;
};

// cache operator of the fused kernels' plane stores ("" = default write-back, ".cs" = streaming / evict-first)
#ifndef OCTGPU_ST_HINT
#define OCTGPU_ST_HINT ""
#endif

#ifndef OCTGPU_BULK_WARPS
#define OCTGPU_BULK_WARPS 4
#endif
constexpr uint32_t kMcsConsumerWarps = OCTGPU_BULK_WARPS;  // k_mcs_bulk: compute warps per block (+1 producer)
constexpr uint32_t kTmaBoxRows = 30 * kMcsConsumerWarps + 4;  // k_mcs_bulk window rows (124)

// k_mcs_deep block shape (mcs_deep.cu): kDeepWarps compute warps whose 32 * kDeepWarps lanes own that many
// consecutive rows (the block's TMA window) + 1 producer warp. Warp-edge rows are exchanged through shared
// memory every word, so only the block's own edges are halo rows: 256 - 2 L core rows for an L-sweep pass.
#ifndef OCTGPU_DEEP_WARPS
#define OCTGPU_DEEP_WARPS 8
#endif
// k_mcs_deep words per ring stage: the two words of a stage are unrolled, so the sweeps' carried state
// ping-pongs between two register sets instead of being copied every word. Block-wide kernel, ms/MCS at
// KS = 1 / 2 / 4: c2 0.165 / 0.150 / 0.171, c2' 0.318 / 0.249 / 0.242 (tools/r2_deep_var2.sh; S = 2..5 within
// 1%)
#ifndef OCTGPU_DEEP_KS
#define OCTGPU_DEEP_KS 2
#endif
constexpr int kDeepKS = OCTGPU_DEEP_KS;          // k_mcs_deep words per ring stage
constexpr int kDeepWarps = OCTGPU_DEEP_WARPS;
constexpr int kDeepLanes = 32 * kDeepWarps;      // rows per block window (TMA box rows, <= 256)
static_assert(kDeepLanes <= 256, "a TMA box dimension holds at most 256 rows");
#ifndef OCTGPU_DEEP_MINB
#define OCTGPU_DEEP_MINB 2
#endif
constexpr int kDeepMinBlocks = OCTGPU_DEEP_MINB;  // resident blocks per SM the register budget targets
// sweeps per k_mcs_deep pass (even): 6 (3 MCS) for constant xi, 4 (2 MCS) for live streams
constexpr int kDeepSweepsConst = 6;
constexpr int kDeepSweepsLive = 4;
constexpr int kDeepSweepsLong = 8;  // 4-MCS constant-xi passes on periodic lattices: absorb remainders of 3-MCS schedules
constexpr int kStripeSweeps = kDeepSweepsConst;  // the longest stripe pass (its halo rows are sized for it)
constexpr int deep_box_rows() { return kDeepLanes; }
constexpr int deep_core_rows(int L) { return kDeepLanes - 2 * L; }  // even: block windows start 16-B aligned

constexpr int kGraphPasses = 16;  // passes per CUDA graph replayed by octgpu_step (even)

// Row stripes: halo rows above / below the core rows (local rows 0..HA-1 and
// HA+L..HA+L+HB-1): enough for k_mcs_deep's 3-MCS pass (5 rows of shrinking
// lanes each side + stage 1's Y(s)[y+1]); shorter passes use fewer of them.
constexpr uint32_t kStripeHA = uint32_t(kStripeSweeps) - 1;
constexpr uint32_t kStripeHB = uint32_t(kStripeSweeps);

// periodic lattices keep this many ghost rows (>= every TMA window + the random tile-origin shift) so windows
// never wrap
constexpr uint32_t kGhostRows = 320;
static_assert(kTmaBoxRows <= kGhostRows && uint32_t(deep_box_rows()) + 64 <= kGhostRows, "ghost rows");

// Per-row RNG states are stored SoA: s[j * Y + y], j = 0..3.

struct StripeLink;  // below

// ---- launchers (return the launch error, never synchronise) ----
// host layout [4][rows][n] (compact) <-> device rows 0..rows-1 of each plane
cudaError_t launch_import(int w, const void* host_layout_dev, void* planes, Geom g, uint32_t rows, cudaStream_t st);
cudaError_t launch_export(int w, const void* planes, void* host_layout_dev, Geom g, uint32_t rows, cudaStream_t st);
// w = 64 planes: rows 0..ghost-1 -> wrap..wrap+ghost-1 of each of the `cols` (plane, word) columns of Y rows
cudaError_t launch_ghost_copy(void* planes, uint32_t Y, uint32_t wrap, uint32_t ghost, uint32_t cols,
                              cudaStream_t st);
// periodic lattices: rewrite the ghost rows (planes, and rng when non-null) from rows 0..ghost-1
cudaError_t launch_refresh_ghosts(int w, void* planes, uint64_t* rng, Geom g, cudaStream_t st);

// One sublattice sweep in place (engine_vec.hpp:145-168), optional mask log in
// reference row-major layout.
// one in-place sweep with counter-based xi (sweep sigma of the run keyed by seed; octgpu_set_rng)
cudaError_t launch_sweep_ctr(int w, void* planes, int parity, Geom g, const ProbDev& p, const ProbDev& q,
                             uint64_t seed, uint64_t sigma, cudaStream_t st);
cudaError_t launch_sweep(int w, void* planes, uint64_t* rng, int parity, Geom g, const ProbDev& p,
                         const ProbDev& q, bool rng_live, void* mask_log, cudaStream_t st);

// One full MCS (sweep f then sweep f^1, engine_vec.hpp:171-177) fused into a
// single pass, src -> dst (ping-pong). jtab: 4-bit table of T^(n*D) (the
// second sweep's stream offset); unused when !rng_live.
cudaError_t launch_mcs(int w, const void* src, void* dst, const uint64_t* rng_src, uint64_t* rng_dst, int f,
                       Geom g, const ProbDev& p, const ProbDev& q, bool rng_live, const uint64_t* jtab,
                       cudaStream_t st);

// Same as launch_mcs with shared-memory staging by cp.async.bulk (mcs_bulk.cu):
// w = 64, n >= 8, periodic Y >= kGhostRows only. ks = words per stage (1, 2 or 4), S = stages.
// tmK / tmK1: 3-D tensor maps (rows x words x planes) of the src plane set with
// boxes of kTmaBoxRows rows x ks and x ks+1 words (see engine.cu ensure_tmaps).
cudaError_t launch_mcs_bulk(const void* src, void* dst, const uint64_t* rng_src, uint64_t* rng_dst, int f, Geom g,
                            const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int ks, int S,
                            const CUtensorMap* tmK, const CUtensorMap* tmK1, cudaStream_t st,
                            const StripeLink* link = nullptr);
size_t mcs_bulk_stage_bytes(int ks);
// k_mcs_bulk with counter-based xi (KS = 2 tensor maps): sweeps sigma (phase f) and sigma + 1 of seed's streams
cudaError_t launch_mcs_bulk_ctr(const void* src, void* dst, int f, Geom g, const ProbDev& p, const ProbDev& q,
                                uint64_t seed, uint64_t sigma, int S, const CUtensorMap* tmK, const CUtensorMap* tmK1,
                                cudaStream_t st, const StripeLink* link = nullptr);
size_t mcs_bulk_smem(int ks, int S);  // dynamic smem of a block (kMcsConsumerWarps + 1 warps)

// Temporally blocked variant (mcs_deep.cu): L sweeps (L/2 MCS, starting with
// parity f) in one pass, L in {4, 6} (6: constant xi only). The geometry's core
// rows must start at virtual row L - 1 (see engine.cu deep_geom). tmK / tmK1:
// tensor maps with boxes of deep_box_rows() rows x kDeepKS and x kDeepKS + 1 words.
bool mcs_deep_supported(int p_mode, int q_mode);
bool mcs_deep_supported_l(int p_mode, int q_mode, int L, bool ctr);
size_t mcs_deep_smem(int p_mode, int q_mode, int L, int S, bool ctr = false);  // S ring stages
// k_mcs_deep with counter-based xi: sweeps sigma .. sigma + L - 1 of seed's streams (octgpu_set_rng)
// link: a row stripe's halo exchange fused into the pass (nullptr: none)
cudaError_t launch_mcs_deep_ctr(const void* src, void* dst, int f, Geom g, const ProbDev& p, const ProbDev& q,
                                uint64_t seed, uint64_t sigma, int L, int S, const CUtensorMap* tmK,
                                const CUtensorMap* tmK1, cudaStream_t st, const StripeLink* link = nullptr);
cudaError_t launch_mcs_deep(const void* src, void* dst, const uint64_t* rng_src, uint64_t* rng_dst, int f, Geom g,
                            const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int L, int S,
                            const CUtensorMap* tmK, const CUtensorMap* tmK1, cudaStream_t st,
                            const StripeLink* link = nullptr);

// s <- M s for every row state, M given as a 4-bit table (64 x 16 x 4 u64).
cudaError_t launch_apply_jump(uint64_t* rng, uint32_t Y, const uint64_t* tab, cudaStream_t st);

// Measurement: column scan + per-row pass + final reduction. For a periodic
// lattice the gauge is the reference's h(0,0) = 0; for a stripe it is local
// (h = 0 at the virtual row c0 - 1, column 0) and the host shifts the power
// sums binomially when combining stripes.
size_t measure_scratch_bytes(uint32_t Y);
cudaError_t launch_measure(int w, const void* planes, Geom g, uint32_t X, void* scratch, void* result_dev,
                           cudaStream_t st);

// Row-stripe halo exchange: gather rows [r0, r0+nrows) of all 4 planes (and
// their rng states when rng != null) into a contiguous buffer laid out
// [plane][row][word] + [row][4] state words, or scatter such a buffer back.
cudaError_t launch_rows_gather(int w, const void* planes, const uint64_t* rng, Geom g, uint32_t r0, uint32_t nrows,
                               void* buf, cudaStream_t st);
cudaError_t launch_rows_scatter(int w, void* planes, uint64_t* rng, Geom g, uint32_t r0, uint32_t nrows,
                                const void* buf, cudaStream_t st);
// one plane-row (word k = 0..n-1 of row r) <-> contiguous n words
cudaError_t launch_planerow_copy(int w, void* planes, int plane, Geom g, uint32_t r, void* buf, bool to_buf,
                                 cudaStream_t st);
// Device-side halo exchange over peer memory (p2p.cu). A neighbour stripe as
// this device sees it: its current plane / rng set (pass parity), allocated
// rows, core rows and its "passes done" counter.
struct PeerView {
    const void* planes;
    const uint64_t* rng;
    const uint64_t* done;
    uint32_t Y;  // allocated rows (row stride)
    uint32_t L;  // core rows
    long long timeout;  // wait limit in SM clock cycles (the prev view's value is used)
};
// A stripe pass fused with its halo exchange (one launch; csrc/stripe_link.cuh): the blocks whose TMA window
// covers halo rows wait for the neighbour(s) to report done >= need and copy their boundary core rows into the
// local halo rows of the source set before their first TMA load; the blocks that write the boundary core rows
// (and the one that completes Y(f) of the first halo row below, which it also pushes into the next stripe's new
// set) publish done = value through a ticket once all of them are finished. active = 0: a periodic lattice.
struct StripeLink {
    PeerView prev, next;
    uint64_t need;          // neighbours' passes done before ours may read their rows
    uint32_t* err;          // wait timeout flag
    uint64_t* done;         // ours: passes completed (read by the neighbours)
    uint32_t* ticket;       // ours: signalling blocks finished in this pass
    uint64_t value;         // done after this pass
    void* next_planes;      // the next stripe's NEW plane set (the push target)
    uint32_t next_Y;        // its allocated rows
    int push_plane;         // Y(f) = 2 + f
    int active;
};
constexpr long long kP2PTimeoutCycles = 20'000'000'000ll;  // default ~10 s at 2 GHz: a dead neighbour is an error, not a hang
// wait for prev.done >= need && next.done >= need, then copy the neighbours' boundary core rows (+ states)
// into the local halo rows (kStripeHA above, kStripeHB below)
cudaError_t launch_halo_pull(int w, void* planes, uint64_t* rng, Geom g, const PeerView& prev, const PeerView& next,
                             uint64_t need, uint32_t* err, bool with_rng, cudaStream_t st);
// copy plane-row (plane, local row kStripeHA + L) into the next stripe's row kStripeHA, then publish *done = value
cudaError_t launch_push_signal(int w, const void* planes, int plane, Geom g, void* next_planes, uint32_t next_Y,
                               uint64_t* done, uint64_t value, cudaStream_t st);

// row_balances / col_balances (slope_field.hpp:177-202) over physical rows r0 .. r0+R-1: rows_out[R] and
// cols_out[X] (either may be null); tmp: X u64 of device scratch for the column counts.
cudaError_t launch_balances(int w, const void* planes, Geom g, uint32_t r0, uint32_t R, uint32_t X,
                            long long* rows_out, long long* cols_out, void* tmp, cudaStream_t st);

// Heights (reference HeightMap layout, row-major int32), after launch_measure.
cudaError_t launch_heights(int w, const void* planes, Geom g, uint32_t X, const void* scratch, int32_t* out,
                           cudaStream_t st);

// Result of launch_measure (device struct, copied back by the host).
struct MeasureResult {
    uint64_t s_lo[4];       // S_k = sum h^k, k=1..4, int128 as (lo, hi)
    int64_t s_hi[4];
    unsigned long long curl_count;
    unsigned long long curl_first;  // y * X + x of the first violating plaquette, ~0 if none
    long long row0_sum;             // sum_x sigma_x-(x, y) of the first core row (global row 0 if periodic)
    long long col0_sum;             // sum_y sigma_y-(0, y) over the core rows
    long long sy_first;             // sigma_y-(0, first core row)
    long long pad;
};

}  // namespace octgpu
