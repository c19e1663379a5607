// sm_100a device code for the bit-vectorized octahedron SCA.
//
// Hot path: the reference's
//   VecEngine::step -> mcs_step -> sublattice_sweep -> detail::sweep_rows
// (engine_vec.hpp:98-177) with per-row xoshiro256++ xi words
// (rng.hpp:17-179, params.hpp:84-92), and the measurement
//   reconstruct_heights -> height_moments (slope_field.hpp:206-229, measure.cpp:24-56).
//
// Mapping (B200-first, not the paper's thread-per-word CTA-per-row kernel):
//  * one LANE owns one lattice ROW and walks its words k = 0..n-1 in order,
//    so each row's xoshiro stream is consumed exactly in the reference order
//    (ξp then ξq per word, engine_vec.hpp:123-125) without any jump;
//  * planes are stored word-major (see Geom), so the 32 lanes of a warp read
//    and write one contiguous 256-B segment per plane per word (coalesced);
//  * loads are software-pipelined PF words ahead in registers;
//  * k_mcs fuses both sublattice sweeps of one MCS into one pass (0.5 B of
//    HBM traffic per site update instead of the reference's 1 B), using
//    warp shuffles for the y-neighbour exchange and a GF(2) jump table for
//    the second sweep's stream position.
#include <algorithm>
#include <cstdint>

#include "device_common.cuh"
#include "octgpu_internal.h"

namespace octgpu {

// -------------------------------------------------------------------------
// Single sublattice sweep, in place (sublattice_sweep, engine_vec.hpp:145-168)

// One row y of the sweep; R is the row's xi source (Xo: the reference's
// xoshiro stream; Ctr: the opt-in counter-based stream).
template <typename Word, int PM, int QM, int PF, typename R>
__device__ __forceinline__ void sweep_row(Word* __restrict__ planes, int parity, const Geom& g, const ProbDev& p,
                                          const ProbDev& q, Word* __restrict__ mask_log, uint32_t y, R& s) {
    constexpr int W = int(sizeof(Word) * 8);
    const uint32_t Y = g.wrap, LD = g.Y, n = g.n;  // periodic lattice: Y rows, row stride LD
    const size_t PS = g.plane_stride;
    Word* px = planes + size_t(0 + parity) * PS + y;                         // X(pi)[y]
    Word* py = planes + size_t(2 + parity) * PS + y;                         // Y(pi)[y]
    Word* qy = planes + size_t(2 + (parity ^ 1)) * PS + (y + 1 == Y ? 0 : y + 1);  // Y(!pi)[y+1]
    Word* xr = planes + size_t(0 + (parity ^ 1)) * PS + y;                   // X(!pi)[y]
    const bool shifted = ((uint32_t(parity) ^ y) & 1u) != 0;                  // engine_vec.hpp:59-61

    const Word raw0 = xr[0];
    Word bA[PF], bB[PF], bC[PF], bR[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        if (uint32_t(j) < n) {
            const size_t o = size_t(j) * LD;
            bA[j] = px[o];
            bB[j] = py[o];
            bC[j] = qy[o];
            bR[j] = (uint32_t(j) + 1 < n) ? xr[o + LD] : raw0;
        }
    }
    Word cur = raw0, carry = 0, new0 = 0;
    for (uint32_t kb = 0; kb < n; kb += PF) {
#pragma unroll
        for (int j = 0; j < PF; ++j) {
            const uint32_t k = kb + j;
            if (k < n) {
                const size_t o = size_t(k) * LD;
                const Word A = bA[j], B = bB[j], Cn = bC[j], nxt = bR[j];
                const uint32_t kk = k + PF;
                if (kk < n) {  // refill this slot PF words ahead
                    const size_t oo = size_t(kk) * LD;
                    bA[j] = px[oo];
                    bB[j] = py[oo];
                    bC[j] = qy[oo];
                    bR[j] = (kk + 1 < n) ? xr[oo + LD] : raw0;
                }
                const Word sxp = shifted ? Word((cur >> 1) | (nxt << (W - 1))) : cur;  // rotate_row_down
                Word xp, xq;
                gen_xi<PM, QM, Word>(s, p, q, xp, xq);
                const Word m = update_mask<Word>(A, B, sxp, Cn, xp, xq);
                px[o] = A ^ m;
                py[o] = B ^ m;
                qy[o] = Cn ^ m;
                const Word sc = shifted ? Word((m << 1) | carry) : m;  // scatter_rotated_xor
                carry = Word(m >> (W - 1));
                if (k == 0)
                    new0 = cur ^ sc;  // word 0 waits for the PBC carry of word n-1
                else
                    xr[o] = cur ^ sc;
                if (mask_log) mask_log[size_t(y) * n + k] = m;
                cur = nxt;
            }
        }
    }
    if (shifted) new0 ^= carry;
    xr[0] = new0;
}

template <typename Word, int PM, int QM, int PF>
__global__ void __launch_bounds__(128) k_sweep(Word* __restrict__ planes, uint64_t* __restrict__ rng, int parity,
                                               Geom g, ProbDev p, ProbDev q, Word* __restrict__ mask_log) {
    const uint32_t y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= g.wrap) return;
    Xo s{0, 0, 0, 0};
    if constexpr (Plan<PM, QM>::live) s = load_state(rng, g.Y, y);
    sweep_row<Word, PM, QM, PF>(planes, parity, g, p, q, mask_log, y, s);
    if constexpr (Plan<PM, QM>::live) store_state(rng, g.Y, y, s);
}

// The same sweep with counter-based xi (octgpu_set_rng; device_common.cuh Ctr):
// row y's draws start from ctr_row(key, y), key = ctr_sweep_key(seed, sigma).
template <typename Word, int PM, int QM, int PF>
__global__ void __launch_bounds__(128) k_sweep_ctr(Word* __restrict__ planes, int parity, Geom g, ProbDev p,
                                                   ProbDev q, uint64_t key) {
    const uint32_t y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= g.wrap) return;
    Ctr s = ctr_row(key, y);
    sweep_row<Word, PM, QM, PF>(planes, parity, g, p, q, static_cast<Word*>(nullptr), y, s);
}

// -------------------------------------------------------------------------
// Fused MCS: sweep f then sweep s = f^1 in one pass, src -> dst.
//
// Warp w owns "core" rows [30w, 30w+30) ∩ [0, Y). Lane L holds row
// y_L = (30w - 1 + L) mod Y; lanes 0 and 31 are halo rows whose FIRST sweep
// is recomputed redundantly (from src, so duplicates are bit-identical).
// Per word k every lane loads X(f)[y], Y(f)[y], X(s)[y] and Y(s)[y+1] - four
// contiguous windows. The second sweep of row y needs only first-sweep
// results of rows y-1, y, y+1 (same word and its right neighbour), obtained
// through shuffles, so the second sweep trails the first by one word.
// The periodic x seam (word n-1 -> word 0) is handled by drawing the second
// sweep's word-0 xi first (stream order) but applying it last.

template <typename Word, int PM, int QM, int PF>
__global__ void __launch_bounds__(128) k_mcs(const Word* __restrict__ src, Word* __restrict__ dst,
                                             const uint64_t* __restrict__ rs, uint64_t* __restrict__ rd, int f,
                                             Geom g, ProbDev p, ProbDev q, const uint64_t* __restrict__ jtab) {
    constexpr int W = int(sizeof(Word) * 8);
    constexpr bool LIVE = Plan<PM, QM>::live;
    const uint32_t Y = g.Y, n = g.n;
    const int lane = threadIdx.x & 31;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid * 30u >= g.c1 - g.c0) return;  // warp-uniform
    const uint32_t v = g.c0 - 1 + wid * 30u + lane;  // virtual row
    const uint32_t y = g.wrap ? v % g.wrap : v;
    const uint32_t y1 = g.wrap ? (v + 1) % g.wrap : v + 1;
    const bool core = lane >= 1 && lane <= 30 && v < g.c1;
    const bool wyf = lane >= 2 && v - 1 < g.c1;  // lane-1 is core
    const int s = f ^ 1;
    const size_t PS = g.plane_stride;
    const Word* sXf = src + size_t(0 + f) * PS + y;
    const Word* sYf = src + size_t(2 + f) * PS + y;
    const Word* sXs = src + size_t(0 + s) * PS + y;
    const Word* sYs1 = src + size_t(2 + s) * PS + y1;
    Word* dXf = dst + size_t(0 + f) * PS + y;
    Word* dYf = dst + size_t(2 + f) * PS + y;
    Word* dXs = dst + size_t(0 + s) * PS + y;
    Word* dYs = dst + size_t(2 + s) * PS + y;
    const bool sh1 = ((uint32_t(f) ^ y ^ g.ypar) & 1u) != 0;  // first sweep shifts x+ of this row
    const bool sh2 = !sh1;                           // second sweep does

    Xo s1{0, 0, 0, 0}, s2{0, 0, 0, 0};
    if constexpr (LIVE) {
        s1 = load_state(rs, Y, y);
        s2 = apply_table(jtab, s1);  // stream position n*D draws ahead
    }
    Word xi2p0, xi2q0;  // second sweep, word 0: drawn first, applied last
    gen_xi<PM, QM, Word>(s2, p, q, xi2p0, xi2q0);

    const Word raw0 = sXs[0];
    Word bA[PF], bB[PF], bC[PF], bR[PF];
#pragma unroll
    for (int j = 0; j < PF; ++j) {
        if (uint32_t(j) < n) {
            const size_t o = size_t(j) * Y;
            bA[j] = sXf[o];
            bB[j] = sYf[o];
            bC[j] = sYs1[o];
            bR[j] = (uint32_t(j) + 1 < n) ? sXs[o + Y] : raw0;
        }
    }

    // post-first-sweep values of word 0 and 1 kept for the seam
    Word A0 = 0, B0 = 0, C0 = 0, R0 = 0, A1 = 0;
    // previous word (k-1), post-first
    Word pA = 0, pB = 0, pC = 0, pR = 0;
    Word cur = raw0, carry1 = 0;
    Word m2last = 0;     // m2 of the most recent second-sweep word (j-1)
    Word xf1 = 0;        // X(f)[y][1] pending the carry of m2[0]

    // second sweep of word j >= 1 (needs post-first words j and j+1)
    auto second = [&](uint32_t j, Word Aj, Word Ajn, Word Bj, Word Cj, Word Rj, Word x2p, Word x2q) {
        const Word Cup = __shfl_up_sync(0xffffffffu, Cj, 1);    // Y(s)[y] post-first (row y-1 wrote it)
        const Word Bdn = __shfl_down_sync(0xffffffffu, Bj, 1);  // Y(f)[y+1] post-first
        const Word sxp2 = sh2 ? Word((Aj >> 1) | (Ajn << (W - 1))) : Aj;
        const Word m2 = update_mask<Word>(Rj, Cup, sxp2, Bdn, x2p, x2q);
        const Word mup = __shfl_up_sync(0xffffffffu, m2, 1);
        const size_t o = size_t(j) * Y;
        if (core) {
            dXs[o] = Rj ^ m2;
            dYs[o] = Cup ^ m2;
        }
        if (wyf) dYf[o] = Bj ^ mup;
        return m2;
    };

    for (uint32_t kb = 0; kb < n; kb += PF) {
#pragma unroll
        for (int jj = 0; jj < PF; ++jj) {
            const uint32_t k = kb + jj;
            if (k < n) {
                const Word A = bA[jj], B = bB[jj], Cn = bC[jj], nxt = bR[jj];
                const uint32_t kk = k + PF;
                if (kk < n) {
                    const size_t oo = size_t(kk) * Y;
                    bA[jj] = sXf[oo];
                    bB[jj] = sYf[oo];
                    bC[jj] = sYs1[oo];
                    bR[jj] = (kk + 1 < n) ? sXs[oo + Y] : raw0;
                }
                // ---- first sweep, word k ----
                const Word sxp = sh1 ? Word((cur >> 1) | (nxt << (W - 1))) : cur;
                Word x1p, x1q;
                gen_xi<PM, QM, Word>(s1, p, q, x1p, x1q);
                const Word m1 = update_mask<Word>(A, B, sxp, Cn, x1p, x1q);
                const Word Ap = A ^ m1, Bp = B ^ m1, Cp = Cn ^ m1;
                const Word sc1 = sh1 ? Word((m1 << 1) | carry1) : m1;
                carry1 = Word(m1 >> (W - 1));
                const Word Rp = cur ^ sc1;  // word 0 still lacks the seam carry
                cur = nxt;
                if (k == 0) {
                    A0 = Ap; B0 = Bp; C0 = Cp; R0 = Rp;
                } else {
                    if (k == 1) A1 = Ap;
                    // ---- second sweep, word j = k-1 (j >= 1) ----
                    if (k >= 2) {
                        const uint32_t j = k - 1;
                        Word x2p, x2q;
                        gen_xi<PM, QM, Word>(s2, p, q, x2p, x2q);
                        const Word m2 = second(j, pA, Ap, pB, pC, pR, x2p, x2q);
                        const Word xfj = pA ^ (sh2 ? Word(m2 << 1) : m2);
                        if (j == 1) {
                            xf1 = xfj;  // needs m2[0] >> (W-1)
                        } else {
                            if (core) dXf[size_t(j) * Y] = xfj ^ (sh2 ? Word(m2last >> (W - 1)) : Word(0));
                        }
                        m2last = m2;
                    }
                }
                pA = Ap; pB = Bp; pC = Cp; pR = Rp;
            }
        }
    }
    // seam of the first sweep: carry of m1[n-1] into word 0
    if (sh1) R0 ^= carry1;
    if (n >= 2) {
        // second sweep, word n-1 (right neighbour wraps to word 0)
        const uint32_t j = n - 1;
        Word x2p, x2q;
        gen_xi<PM, QM, Word>(s2, p, q, x2p, x2q);
        const Word Rj = (j == 0) ? R0 : pR;
        const Word m2 = second(j, pA, A0, pB, pC, Rj, x2p, x2q);
        const Word xfj = pA ^ (sh2 ? Word(m2 << 1) : m2);
        if (j == 1) {
            xf1 = xfj;
        } else {
            if (core) dXf[size_t(j) * Y] = xfj ^ (sh2 ? Word(m2last >> (W - 1)) : Word(0));
        }
        m2last = m2;
    }
    {
        // second sweep, word 0 (xi drawn first, applied last)
        const Word Anext = (n >= 2) ? A1 : A0;
        const Word m2 = second(0, A0, Anext, B0, C0, R0, xi2p0, xi2q0);
        const Word top_prev = (n >= 2) ? Word(m2last >> (W - 1)) : Word(m2 >> (W - 1));
        const Word xf0 = A0 ^ (sh2 ? Word((m2 << 1) | top_prev) : m2);
        if (core) {
            dXf[0] = xf0;
            if (n >= 2) dXf[Y] = xf1 ^ (sh2 ? Word(m2 >> (W - 1)) : Word(0));
        }
    }
    if constexpr (LIVE) {
        if (core) store_state(rd, Y, y, s2);
    }
}

// -------------------------------------------------------------------------
// Jump application (GF(2) matrix on every row state)

__global__ void k_apply_jump(uint64_t* __restrict__ rng, uint32_t Y, const uint64_t* __restrict__ tab) {
    const uint32_t y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= Y) return;
    Xo s = load_state(rng, Y, y);
    s = apply_table(tab, s);
    store_state(rng, Y, y, s);
}

// -------------------------------------------------------------------------
// Layout transposes: reference SlopeField rows (row-major [Y][n] per plane)
// <-> device word-major ([n][Y] per plane).

template <typename Word, bool TO_DEVICE>
__global__ void k_transpose(const Word* __restrict__ in, Word* __restrict__ out, Geom g, uint32_t rows) {
    __shared__ Word tile[32][33];
    const uint32_t n = g.n;
    const size_t hoff = size_t(blockIdx.z) * rows * n;      // host plane
    const size_t doff = size_t(blockIdx.z) * g.plane_stride;  // device plane
    // host: [rows][n] (row-major); device: word k of row r at k * g.Y + r
    const uint32_t R = TO_DEVICE ? rows : n, Cc = TO_DEVICE ? n : rows;  // dims of `in`
    const uint32_t c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint32_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < Cc)
            tile[i][threadIdx.x] = TO_DEVICE ? in[hoff + size_t(r) * n + c] : in[doff + size_t(r) * g.Y + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const uint32_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < Cc) {
            if (TO_DEVICE)
                out[doff + size_t(c) * g.Y + r] = tile[threadIdx.x][i];
            else
                out[hoff + size_t(c) * n + r] = tile[threadIdx.x][i];
        }
    }
}

// Ghost rows of a periodic lattice: row wrap + i = row (i mod wrap).
template <typename Word>
__global__ void k_refresh_ghosts(Word* __restrict__ planes, uint64_t* __restrict__ rng, Geom g) {
    const uint32_t per = g.ghost * g.n, total = 4 * per;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        const uint32_t p = t / per, rem = t % per, k = rem / g.ghost, i = rem % g.ghost;
        Word* base = planes + size_t(p) * g.plane_stride + size_t(k) * g.Y;
        base[g.wrap + i] = base[i % g.wrap];
    }
    if (rng)
        for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < 4 * g.ghost; t += gridDim.x * blockDim.x) {
            const uint32_t j = t / g.ghost, i = t % g.ghost;
            rng[size_t(j) * g.Y + g.wrap + i] = rng[size_t(j) * g.Y + i % g.wrap];
        }
}

// -------------------------------------------------------------------------
// Launchers

namespace {

constexpr int kPF = 4;

template <template <typename, int, int, int> class K, typename Word>
struct Dispatch;

template <typename Word, int PM, int QM>
cudaError_t sweep_pq(void* planes, uint64_t* rng, int parity, Geom g, const ProbDev& p, const ProbDev& q,
                     void* mask_log, cudaStream_t st) {
    const uint32_t threads = 128, blocks = (g.wrap + threads - 1) / threads;
    k_sweep<Word, PM, QM, kPF><<<blocks, threads, 0, st>>>(static_cast<Word*>(planes), rng, parity, g, p, q,
                                                          static_cast<Word*>(mask_log));
    return cudaGetLastError();
}

template <typename Word, int PM, int QM>
cudaError_t sweep_ctr_pq(void* planes, int parity, Geom g, const ProbDev& p, const ProbDev& q, uint64_t key,
                         cudaStream_t st) {
    const uint32_t threads = 128, blocks = (g.wrap + threads - 1) / threads;
    k_sweep_ctr<Word, PM, QM, kPF><<<blocks, threads, 0, st>>>(static_cast<Word*>(planes), parity, g, p, q, key);
    return cudaGetLastError();
}

template <typename Word, int PM, int QM>
cudaError_t mcs_pq(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g, const ProbDev& p,
                   const ProbDev& q, const uint64_t* jtab, cudaStream_t st) {
    const uint32_t warps = (g.c1 - g.c0 + 29) / 30;
    const uint32_t threads = 128, blocks = (warps * 32 + threads - 1) / threads;
    k_mcs<Word, PM, QM, kPF><<<blocks, threads, 0, st>>>(static_cast<const Word*>(src), static_cast<Word*>(dst),
                                                        rs, rd, f, g, p, q, jtab);
    return cudaGetLastError();
}

#define OCT_Q_CASES(FN, WORD, PM, ...)                        \
    switch (q.mode) {                                         \
    case M_ZERO: return FN<WORD, PM, M_ZERO>(__VA_ARGS__);     \
    case M_HALF: return FN<WORD, PM, M_HALF>(__VA_ARGS__);     \
    case M_DYADIC: return FN<WORD, PM, M_DYADIC>(__VA_ARGS__); \
    case M_ARB: return FN<WORD, PM, M_ARB>(__VA_ARGS__);       \
    case M_ONE: return FN<WORD, PM, M_ONE>(__VA_ARGS__);       \
    default: return cudaErrorInvalidValue;                    \
    }

#define OCT_PQ_CASES(FN, WORD, ...)                                      \
    switch (p.mode) {                                                    \
    case M_ZERO: OCT_Q_CASES(FN, WORD, M_ZERO, __VA_ARGS__)               \
    case M_HALF: OCT_Q_CASES(FN, WORD, M_HALF, __VA_ARGS__)               \
    case M_DYADIC: OCT_Q_CASES(FN, WORD, M_DYADIC, __VA_ARGS__)           \
    case M_ARB: OCT_Q_CASES(FN, WORD, M_ARB, __VA_ARGS__)                 \
    case M_ONE: OCT_Q_CASES(FN, WORD, M_ONE, __VA_ARGS__)                 \
    default: return cudaErrorInvalidValue;                               \
    }

}  // namespace

cudaError_t launch_sweep(int w, void* planes, uint64_t* rng, int parity, Geom g, const ProbDev& p,
                         const ProbDev& q, bool, void* mask_log, cudaStream_t st) {
    if (w == 64) {
        OCT_PQ_CASES(sweep_pq, uint64_t, planes, rng, parity, g, p, q, mask_log, st)
    } else {
        OCT_PQ_CASES(sweep_pq, uint32_t, planes, rng, parity, g, p, q, mask_log, st)
    }
}

cudaError_t launch_sweep_ctr(int w, void* planes, int parity, Geom g, const ProbDev& p, const ProbDev& q,
                             uint64_t seed, uint64_t sigma, cudaStream_t st) {
    const uint64_t key = ctr_sweep_key(seed, sigma);
    if (w == 64) {
        OCT_PQ_CASES(sweep_ctr_pq, uint64_t, planes, parity, g, p, q, key, st)
    } else {
        OCT_PQ_CASES(sweep_ctr_pq, uint32_t, planes, parity, g, p, q, key, st)
    }
}

cudaError_t launch_mcs(int w, const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                       const ProbDev& p, const ProbDev& q, bool, const uint64_t* jtab, cudaStream_t st) {
    if (w == 64) {
        OCT_PQ_CASES(mcs_pq, uint64_t, src, dst, rs, rd, f, g, p, q, jtab, st)
    } else {
        OCT_PQ_CASES(mcs_pq, uint32_t, src, dst, rs, rd, f, g, p, q, jtab, st)
    }
}

cudaError_t launch_apply_jump(uint64_t* rng, uint32_t Y, const uint64_t* tab, cudaStream_t st) {
    const uint32_t threads = 128, blocks = (Y + threads - 1) / threads;
    k_apply_jump<<<blocks, threads, 0, st>>>(rng, Y, tab);
    return cudaGetLastError();
}

template <typename Word, bool TO>
static cudaError_t transpose_w(const void* in, void* out, Geom g, uint32_t rows, cudaStream_t st) {
    const uint32_t R = TO ? rows : g.n, Cc = TO ? g.n : rows;
    dim3 grid((Cc + 31) / 32, (R + 31) / 32, 4), block(32, 8);
    k_transpose<Word, TO><<<grid, block, 0, st>>>(static_cast<const Word*>(in), static_cast<Word*>(out), g, rows);
    return cudaGetLastError();
}

cudaError_t launch_import(int w, const void* in, void* planes, Geom g, uint32_t rows, cudaStream_t st) {
    return w == 64 ? transpose_w<uint64_t, true>(in, planes, g, rows, st)
                   : transpose_w<uint32_t, true>(in, planes, g, rows, st);
}

cudaError_t launch_export(int w, const void* planes, void* out, Geom g, uint32_t rows, cudaStream_t st) {
    return w == 64 ? transpose_w<uint64_t, false>(planes, out, g, rows, st)
                   : transpose_w<uint32_t, false>(planes, out, g, rows, st);
}

// rows 0..ghost-1 -> rows wrap..wrap+ghost-1 of every (plane, word) column (word-major: a column's rows are
// contiguous), 16 B per thread; requires ghost <= wrap and 16-B aligned columns (Y even, ghost even)
__global__ void k_ghost_copy(uint64_t* __restrict__ planes, uint32_t Y, uint32_t wrap, uint32_t ghost, uint32_t cols) {
    const uint32_t per = ghost / 2, total = per * cols;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t c = i / per, r = (i - c * per) * 2;
        uint64_t* col = planes + size_t(c) * Y;
        *reinterpret_cast<ulonglong2*>(col + wrap + r) = *reinterpret_cast<const ulonglong2*>(col + r);
    }
}

cudaError_t launch_ghost_copy(void* planes, uint32_t Y, uint32_t wrap, uint32_t ghost, uint32_t cols,
                              cudaStream_t st) {
    const uint32_t total = ghost / 2 * cols;
    const uint32_t blocks = std::min<uint32_t>(1184, (total + 255) / 256);
    k_ghost_copy<<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(planes), Y, wrap, ghost, cols);
    return cudaGetLastError();
}

cudaError_t launch_refresh_ghosts(int w, void* planes, uint64_t* rng, Geom g, cudaStream_t st) {
    if (!g.ghost) return cudaSuccess;
    const uint32_t blocks = std::min<uint32_t>(256, (4 * g.ghost * g.n + 255) / 256);
    if (w == 64)
        k_refresh_ghosts<uint64_t><<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(planes), rng, g);
    else
        k_refresh_ghosts<uint32_t><<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(planes), rng, g);
    return cudaGetLastError();
}

}  // namespace octgpu

// -------------------------------------------------------------------------
// Row-stripe halo exchange helpers (multi-GPU path). Tiny and strided: a few
// plane-rows per MCS, so plain grid-stride loops.
namespace octgpu {

template <typename Word>
__global__ void k_rows_gather(const Word* __restrict__ planes, const uint64_t* __restrict__ rng, Geom g, uint32_t r0,
                              uint32_t nrows, Word* __restrict__ buf) {
    const uint32_t n = g.n, per = nrows * n, total = 4 * per;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t p = i / per, rem = i % per, r = rem / n, k = rem % n;
        buf[i] = planes[size_t(p) * g.plane_stride + size_t(k) * g.Y + r0 + r];
    }
    if (rng && blockIdx.x == 0)
        for (uint32_t t = threadIdx.x; t < 4 * nrows; t += blockDim.x)  // [row][j]
            reinterpret_cast<uint64_t*>(buf + total)[t] = rng[size_t(t & 3) * g.Y + r0 + (t >> 2)];
}

template <typename Word>
__global__ void k_rows_scatter(Word* __restrict__ planes, uint64_t* __restrict__ rng, Geom g, uint32_t r0,
                               uint32_t nrows, const Word* __restrict__ buf) {
    const uint32_t n = g.n, per = nrows * n, total = 4 * per;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t p = i / per, rem = i % per, r = rem / n, k = rem % n;
        planes[size_t(p) * g.plane_stride + size_t(k) * g.Y + r0 + r] = buf[i];
    }
    if (rng && blockIdx.x == 0)
        for (uint32_t t = threadIdx.x; t < 4 * nrows; t += blockDim.x)
            rng[size_t(t & 3) * g.Y + r0 + (t >> 2)] = reinterpret_cast<const uint64_t*>(buf + total)[t];
}

template <typename Word>
__global__ void k_planerow_copy(Word* __restrict__ planes, int plane, Geom g, uint32_t r, Word* __restrict__ buf,
                                int to_buf) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < g.n; k += gridDim.x * blockDim.x) {
        Word* p = planes + size_t(plane) * g.plane_stride + size_t(k) * g.Y + r;
        if (to_buf)
            buf[k] = *p;
        else
            *p = buf[k];
    }
}

namespace {
inline uint32_t small_grid(uint32_t work) { return std::min<uint32_t>(1024, (work + 255) / 256 + 1); }
}  // namespace

cudaError_t launch_rows_gather(int w, const void* planes, const uint64_t* rng, Geom g, uint32_t r0, uint32_t nrows,
                               void* buf, cudaStream_t st) {
    const uint32_t blocks = small_grid(4 * nrows * g.n);
    if (w == 64)
        k_rows_gather<uint64_t><<<blocks, 256, 0, st>>>(static_cast<const uint64_t*>(planes), rng, g, r0, nrows,
                                                        static_cast<uint64_t*>(buf));
    else
        k_rows_gather<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t*>(planes), rng, g, r0, nrows,
                                                        static_cast<uint32_t*>(buf));
    return cudaGetLastError();
}

cudaError_t launch_rows_scatter(int w, void* planes, uint64_t* rng, Geom g, uint32_t r0, uint32_t nrows,
                                const void* buf, cudaStream_t st) {
    const uint32_t blocks = small_grid(4 * nrows * g.n);
    if (w == 64)
        k_rows_scatter<uint64_t><<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(planes), rng, g, r0, nrows,
                                                         static_cast<const uint64_t*>(buf));
    else
        k_rows_scatter<uint32_t><<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(planes), rng, g, r0, nrows,
                                                         static_cast<const uint32_t*>(buf));
    return cudaGetLastError();
}

cudaError_t launch_planerow_copy(int w, void* planes, int plane, Geom g, uint32_t r, void* buf, bool to_buf,
                                 cudaStream_t st) {
    const uint32_t blocks = small_grid(g.n);
    if (w == 64)
        k_planerow_copy<uint64_t><<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(planes), plane, g, r,
                                                          static_cast<uint64_t*>(buf), to_buf);
    else
        k_planerow_copy<uint32_t><<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(planes), plane, g, r,
                                                          static_cast<uint32_t*>(buf), to_buf);
    return cudaGetLastError();
}

}  // namespace octgpu
