// Temporally blocked MCS kernel: L sweeps (L/2 MCS) of a periodic lattice in
// ONE pass over the planes (Appendix B.5 extended).
//
// Same warp-specialised TMA pipeline as k_mcs_bulk (mcs_bulk.cu), but every
// lane carries its row through L sublattice sweeps f, s, f, s, ... before the
// planes go back to HBM, so DRAM traffic per MCS drops from ~0.5 B to
// ~0.5·2/L B per site update. Results are bit-identical to L/2 launches of the
// one-MCS kernel (and to the reference's mcs_step, engine_vec.hpp:171-177).
//
// Dependencies that make this possible (engine_vec.hpp:95-137):
//  * sweep ℓ of row y, word j, reads only sweep-(ℓ-1) values of rows y-1..y+1
//    and words j..j+1, plus the x-carry of sweep ℓ's own word j-1;
//  * so sweep ℓ runs one word behind sweep ℓ-1 (software pipeline over the
//    word index) and one lane narrower on each side (halo rows recomputed by
//    the neighbouring warp): a warp keeps lanes L-1 .. 32-L as core rows
//    (26 of 32 for L = 4);
//  * the periodic x seam: sweep ℓ processes words ℓ-1, ..., n-1, 0, ..., ℓ-2
//    (its wrapped words need sweep ℓ-1's word 0 carry, available only after
//    sweep ℓ-1 wrapped). The reference draws the xi of words 0..ℓ-2 of stream
//    ℓ first: they are drawn at the start (stream order kept) and parked in
//    shared memory with the first/second-word outputs each sweep leaves for
//    the next one's wrap.
//  * stream ℓ starts (ℓ-1)·n·D draws after stream 1: one GF(2) table jump per
//    sweep per row (the same T^(nD) table as k_mcs_bulk).
//
// Iteration i of a row runs sweep ℓ on word (i-(ℓ-1)) mod n when
// 2(ℓ-1) <= i < n + 2(ℓ-1); iterations 2L..n-1 are the branch-free steady
// state. Used for periodic w = 64 lattices with n >= 8, Y >= kGhostRows and
// probabilities whose xi is cheap (zero / half / dyadic / one): arbitrary
// probabilities are issue-bound and keep the one-MCS kernel (30 of 32 rows).
#include <cuda.h>

#include <cstdint>

#include "device_common.cuh"
#include "octgpu_internal.h"
#include "stripe_link.cuh"

namespace octgpu {

namespace {

constexpr int kDP = kDeepWarps;   // compute warps per block (+1 producer)
constexpr int kKS = kDeepKS;      // words per ring stage
constexpr int kSMax = 8;          // ring stages: runtime S <= kSMax (barrier slots)
constexpr int kLanes = kDeepLanes;  // rows per block = compute lanes = parking-slot stride
// xoshiro streams kept in registers in a live pass; the others live in parking slots (loaded / stored
// around each use). With the block-wide lane layout a 4-sweep pass keeps all four in registers.
#ifndef OCTGPU_DEEP_REG_STREAMS
#define OCTGPU_DEEP_REG_STREAMS 4
#endif
constexpr int kRegStreams = OCTGPU_DEEP_REG_STREAMS;

constexpr int kXchBar = 1;  // named barrier of the compute warps' edge exchange (0 = __syncthreads)

template <int L>
struct DeepGeo {
    // core lanes L-1 .. kLanes-2-L: lane kLanes-1-L would still be exact, but an even core-row count keeps
    // every block's window start even (a TMA box must start 16-B aligned in its innermost, row dimension)
    static constexpr int kFirst = L - 1;           // first core lane
    static constexpr int kLast = kLanes - 2 - L;   // last core lane
    static constexpr int kRows = kLast - kFirst + 1;  // core rows per block
    static constexpr int kWin = kLanes;            // window rows (TMA box)
    static_assert(kRows == deep_core_rows(L), "host core-row count must match");
    static_assert(kWin == deep_box_rows(), "host tensor-map box must match");
    static_assert(kWin + 64 <= int(kGhostRows), "ghost rows must cover the window overhang and tile shifts");
};

constexpr int align16w(int words) { return (words + 15) / 16 * 16; }

template <int L>
struct DeepStage {  // ring stage: Xf[KS][W] | Yf[KS][W] | Ys[KS][W] | Xs[KS+1][W], 128-B aligned segments
    static constexpr int W = DeepGeo<L>::kWin;
    static constexpr int kSeg = align16w(kKS * W);
    static constexpr int kXf = 0, kYf = kSeg, kYs = 2 * kSeg, kXs = 3 * kSeg;
    static constexpr int kWords = 3 * kSeg + align16w((kKS + 1) * W);
    static constexpr uint32_t kTx = (4 * kKS + 1) * W * 8;
};

// Per-lane parking slots in shared memory ([slot][kLanes] u64), then the edge exchange buffers.
template <int L, int PM, int QM, bool CTR = false>
struct DeepSlots {
    static constexpr bool kPreP = !(PM == M_ZERO || PM == M_ONE);
    static constexpr bool kPreQ = !(QM == M_ZERO || QM == M_ONE);
    // stages 1..L-1: A,B,C,R,A1 of their first two words; stage L: R
    __host__ __device__ static constexpr int save() { return 5 * (L - 1) + 1; }
    // xi words 0..l-2 of streams l = 2..L
    __host__ __device__ static constexpr int npre() { return L * (L - 1) / 2; }
    __host__ __device__ static constexpr int preP0() { return save(); }
    __host__ __device__ static constexpr int preQ0() { return save() + (kPreP ? npre() : 0); }
    // streams kRegStreams..L-1 (0-based) of a live pass are parked in shared memory (4 slots each)
    static constexpr bool kLive = kPreP || kPreQ || !(PM == M_ZERO || PM == M_ONE) || !(QM == M_ZERO || QM == M_ONE);
    // (counter-based streams are one word each: all of them stay in registers)
    __host__ __device__ static constexpr int parked() { return !CTR && kLive && L > kRegStreams ? L - kRegStreams : 0; }
    __host__ __device__ static constexpr int st0() { return preQ0() + (kPreQ ? npre() : 0); }
    __host__ __device__ static constexpr int count() { return st0() + 4 * parked(); }
    __host__ __device__ static constexpr int pre(int l, int j) { return (l - 1) * (l - 2) / 2 + j; }
    // edge exchange: [2 buffers][kDP warps][C of lane 31 | B of lane 0][L words, L-1 used] u64
    __host__ __device__ static constexpr int xch_words() { return 2 * kDP * 2 * L; }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* tm, uint32_t row, uint32_t word, uint32_t plane,
                                      uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(row), "r"(word), "r"(plane), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of a TMA box (no shared memory, no barrier): SASS UTMAPF
__device__ __forceinline__ void tma3d_prefetch(const CUtensorMap* tm, uint32_t row, uint32_t word, uint32_t plane) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(row), "r"(word), "r"(plane)
                 : "memory");
}
// named barrier of the compute lanes; the non-.aligned form: the lanes reach it from lane-divergent code
__device__ __forceinline__ void xch_barrier() {
    __syncwarp();
    asm volatile("barrier.sync %0, %1;" ::"n"(kXchBar), "n"(kLanes) : "memory");
}

__device__ __forceinline__ void st_pred(uint64_t* p, uint64_t v, bool pred) {
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.b32 q, %2, 0;\n"
        "@q st.global" OCTGPU_ST_HINT ".b64 [%0], %1;\n"
        "}\n" ::"l"(p),
        "l"(v), "r"(int(pred)));
}

__device__ __forceinline__ Xo slot_state(const uint64_t* save, int slot) {
    return Xo{save[(slot + 0) * kLanes], save[(slot + 1) * kLanes], save[(slot + 2) * kLanes], save[(slot + 3) * kLanes]};
}
__device__ __forceinline__ void slot_store(uint64_t* save, int slot, const Xo& s) {
    save[(slot + 0) * kLanes] = s.a;
    save[(slot + 1) * kLanes] = s.b;
    save[(slot + 2) * kLanes] = s.c;
    save[(slot + 3) * kLanes] = s.d;
}

// Lane context shared by every iteration.
struct DeepCtx {
    uint32_t n, Y;
    uint64_t* d0;   // dst at this lane's physical row y
    uint64_t* d1;   // dst at physical row y + 1 (Y(f) of the row below)
    uint32_t wrap;
    uint32_t sf1, sf2;   // x+ neighbour shifted by one packed bit in sweeps of parity f / s
    int up, dn;          // shuffle source lanes of rows y - 1 / y + 1 (rotating: see edge exchange)
    bool core, ghost_row;  // ghost_row: the row's stream state is mirrored into the ghost rows
    uint64_t* save;  // this lane's parking slots: save[slot * kLanes]
};

template <int L, typename Src = Xo>
struct DeepState {
    uint64_t pA[L], pB[L], pC[L], pR[L];  // each sweep's outputs at its previous word
    uint32_t ml[L];                       // high word of each sweep's mask at its previous word (x carry)
    Src rs[L];                            // stream of each sweep (xoshiro, or the opt-in counter stream)
    uint64_t cur, raw0;                   // sweep 1: original X(s)[y][j], X(s)[y][0]
};

// plane stores of the last sweep (the host mirrors rows 0..ghost-1 into a periodic lattice's ghost rows after
// the pass: one strided device copy instead of a branch per store here)
__device__ __forceinline__ void put(uint64_t* ptr, uint64_t val, bool pred) { st_pred(ptr, val, pred); }

// Edge exchange after every word: lane 31 of warp w publishes its rows' C outputs (row y+1's Y input of the
// next sweep) and lane 0 its B outputs (row y-1's Y(s)[y+1] input); after the barrier lane 31 of warp w+1
// takes warp w's C and lane 0 of warp w-1 takes warp w's B. Lane 31's own C and lane 0's own B are consumed
// only by the neighbouring warp, so they are overwritten in place and the rotating shuffles of the next word
// (lane 0 <- lane 31, lane 31 <- lane 0) deliver the other warp's row.
// predicated shared-memory accesses (no branch around the edge lanes' exchange)
__device__ __forceinline__ void sts2_pred(uint64_t* p, uint64_t a, uint64_t b, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q st.shared.v2.u64 [%0], {%1, %2};\n}\n" ::"r"(smem_u32(p)),
                 "l"(a), "l"(b), "r"(int(pred))
                 : "memory");
}
__device__ __forceinline__ void sts1_pred(uint64_t* p, uint64_t a, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q st.shared.u64 [%0], %1;\n}\n" ::"r"(smem_u32(p)), "l"(a),
                 "r"(int(pred))
                 : "memory");
}
__device__ __forceinline__ void lds2_pred(const uint64_t* p, uint64_t& a, uint64_t& b, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %3, 0;\n@q ld.shared.v2.u64 {%0, %1}, [%2];\n}\n"
                 : "+l"(a), "+l"(b)
                 : "r"(smem_u32(p)), "r"(int(pred))
                 : "memory");
}
__device__ __forceinline__ void lds1_pred(const uint64_t* p, uint64_t& a, bool pred) {
    asm volatile("{\n.reg .pred q;\nsetp.ne.b32 q, %2, 0;\n@q ld.shared.u64 %0, [%1];\n}\n"
                 : "+l"(a)
                 : "r"(smem_u32(p)), "r"(int(pred))
                 : "memory");
}
// v[0..L-2] <-> a 16-B aligned row of L words
template <int L>
__device__ __forceinline__ void xrow_store(uint64_t* row, const uint64_t* v, bool pred) {
#pragma unroll
    for (int l = 0; l + 1 < L - 1; l += 2) sts2_pred(row + l, v[l], v[l + 1], pred);
    if constexpr ((L - 1) % 2) sts1_pred(row + L - 2, v[L - 2], pred);
}
template <int L>
__device__ __forceinline__ void xrow_load(const uint64_t* row, uint64_t* v, bool pred) {
#pragma unroll
    for (int l = 0; l + 1 < L - 1; l += 2) lds2_pred(row + l, v[l], v[l + 1], pred);
    if constexpr ((L - 1) % 2) lds1_pred(row + L - 2, v[L - 2], pred);
}

template <int L, typename StateT>
__device__ __forceinline__ void edge_exchange(StateT& S, uint64_t* xch, uint32_t i, int wib, int lane) {
    // buffer i&1: [kDP warps][C of lane 31 | B of lane 0][L words (L-1 used)]
    uint64_t* buf = xch + size_t(i & 1u) * (kDP * 2 * L);
    xrow_store<L>(buf + (wib * 2 + 0) * L, S.pC, lane == 31);
    xrow_store<L>(buf + (wib * 2 + 1) * L, S.pB, lane == 0);
    xch_barrier();
    xrow_load<L>(buf + ((wib - 1) * 2 + 0) * L, S.pC, lane == 31 && wib > 0);
    xrow_load<L>(buf + ((wib + 1) * 2 + 1) * L, S.pB, lane == 0 && wib < kDP - 1);
}

// Split-phase edge exchange (the one-draw live passes): publish (store the edge rows of iteration i, then one
// arrive per warp on the iteration's mbarrier) and collect (wait for every warp's publish of iteration i, then
// load the neighbours' rows). Between them a warp runs the next word's first sweep, which needs no neighbour
// values, instead of idling at the block barrier. Iteration i uses buffer / mbarrier i & 1, phase (i >> 1) & 1;
// a warp can publish iteration i + 2 into the same buffer only after collecting i + 1, i.e. after every warp has
// collected i. Measured: c2' 0.249 -> 0.243 ms/MCS; the constant-xi and two-draw passes are faster with the
// barrier (the release-arrive also orders the sweep's global stores), so they keep it.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int L, typename StateT>
__device__ __forceinline__ void xch_publish(StateT& S, uint64_t* xch, uint64_t* xbar, uint32_t i, int wib, int lane) {
    uint64_t* buf = xch + size_t(i & 1u) * (kDP * 2 * L);
    xrow_store<L>(buf + (wib * 2 + 0) * L, S.pC, lane == 31);
    xrow_store<L>(buf + (wib * 2 + 1) * L, S.pB, lane == 0);
    __syncwarp();
    if (lane == 0) mbar_arrive(&xbar[i & 1u]);
}
template <int L, typename StateT>
__device__ __forceinline__ void xch_collect(StateT& S, const uint64_t* xch, uint64_t* xbar, uint32_t i, int wib,
                                            int lane) {
    mbar_wait(&xbar[i & 1u], (i >> 1) & 1u);
    const uint64_t* buf = xch + size_t(i & 1u) * (kDP * 2 * L);
    xrow_load<L>(buf + ((wib - 1) * 2 + 0) * L, S.pC, lane == 31 && wib > 0);
    xrow_load<L>(buf + ((wib + 1) * 2 + 1) * L, S.pB, lane == 0 && wib < kDP - 1);
}

// One iteration i: sweep l on word (i-(l-1)) mod n for every active l.
// STEADY: all sweeps active, no first/second/last words, no wrap (i in [2L, n-1]).
// (sweeps LO..HI into nA..nR; every sweep reads the state of iteration i - 1: deep_commit after the last range)
template <int PM, int QM, int L, bool STEADY, bool CTR, int LO, int HI>
__device__ __forceinline__ void deep_sweeps(DeepState<L, typename std::conditional<CTR, Ctr, Xo>::type>& S,
                                            const DeepCtx& c, uint32_t i, const uint64_t* sb, int jj,
                                            const ProbDev& p, const ProbDev& q, const Geom& g, int f,
                                            uint64_t (&nA)[L], uint64_t (&nB)[L], uint64_t (&nC)[L],
                                            uint64_t (&nR)[L], bool (&act)[L]) {
    // plane offsets of the last sweep's stores, formed from the kernel parameters (uniform, no registers)
    const size_t oXf = size_t(f) * g.plane_stride, oXs = size_t(f ^ 1) * g.plane_stride;
    const size_t oYf = size_t(2 + f) * g.plane_stride, oYs = size_t(3 - f) * g.plane_stride;
    using ST = DeepStage<L>;
    using SL = DeepSlots<L, PM, QM, CTR>;
    const uint32_t n = c.n;
#pragma unroll
    for (int l = LO; l <= HI; ++l) {
        const int li = l - 1;
        uint32_t j = i - uint32_t(l - 1);
        bool active = true;
        if constexpr (!STEADY) {
            active = i >= uint32_t(2 * (l - 1)) && i < n + uint32_t(2 * (l - 1));
            if (j >= n) j -= n;
        }
        act[li] = active;
        if (!active) continue;  // block-uniform
        const bool first = !STEADY && j == uint32_t(l - 1);
        const bool second = !STEADY && j == uint32_t(l);
        const bool last = !STEADY && j == (l == 1 ? n - 1 : uint32_t(l - 2));

        // ---- xi of word j of stream l (stream order: pre-drawn words 0..l-2 come first) ----
        uint64_t xp, xq;
        if (STEADY || l == 1 || j >= uint32_t(l - 1)) {
            if constexpr (SL::parked() > 0) {
                if (li >= kRegStreams) {  // li is a constant after unrolling
                    const int sl = SL::st0() + 4 * (li - kRegStreams);
                    Xo st = slot_state(c.save, sl);
                    gen_xi<PM, QM, uint64_t>(st, p, q, xp, xq);
                    slot_store(c.save, sl, st);
                } else {
                    gen_xi<PM, QM, uint64_t>(S.rs[li], p, q, xp, xq);
                }
            } else {
                gen_xi<PM, QM, uint64_t>(S.rs[li], p, q, xp, xq);
            }
        } else {
            const int k = SL::pre(l, int(j));
            if constexpr (SL::kPreP) xp = c.save[(SL::preP0() + k) * kLanes];
            else xp = (PM == M_ONE) ? ~uint64_t(0) : 0;
            if constexpr (SL::kPreQ) xq = c.save[(SL::preQ0() + k) * kLanes];
            else xq = (QM == M_ONE) ? ~uint64_t(0) : 0;
        }

        // ---- inputs: own X, own Y, Y[y+1] of the other parity, x+ neighbour words j, j+1 ----
        uint64_t xo, yo, yn, x0, x1;
        if (l == 1) {
            xo = sb[ST::kXf + jj * ST::W];
            yo = sb[ST::kYf + jj * ST::W];
            yn = sb[ST::kYs + jj * ST::W + 1];
            const uint64_t nxt = (j + 1 == n) ? S.raw0 : sb[ST::kXs + (jj + 1) * ST::W];
            x0 = S.cur;
            x1 = nxt;
            S.cur = nxt;
        } else {
            const int sv = 5 * (l - 2);  // slots of sweep l-1
            if (!STEADY && j == uint32_t(l - 2)) {  // sweep l-1's first word (parked; rows y±1 = lanes t±1)
                x0 = c.save[(sv + 0) * kLanes];
                yn = c.save[(sv + 1) * kLanes + 1];
                yo = c.save[(sv + 2) * kLanes - 1];
                xo = c.save[(sv + 3) * kLanes];
            } else {
                x0 = S.pA[li - 1];
                yn = __shfl_sync(0xffffffffu, S.pB[li - 1], c.dn);
                yo = __shfl_sync(0xffffffffu, S.pC[li - 1], c.up);
                xo = S.pR[li - 1];
            }
            uint64_t nxa = nA[li - 1];
            if constexpr (!STEADY) {
                const uint32_t jn = (j + 1 == n) ? 0u : j + 1;
                if (jn == uint32_t(l - 2)) nxa = c.save[(sv + 0) * kLanes];
                else if (j == uint32_t(l - 2)) nxa = c.save[(sv + 4) * kLanes];
            }
            x1 = nxa;
        }
        const uint32_t sh = (l & 1) ? c.sf1 : c.sf2;
        const uint64_t rot = rot_sel(x0, x1, sh);
        const uint64_t m = update_mask<uint64_t>(xo, yo, rot, yn, xp, xq);
        const uint64_t mprev = first ? uint64_t(0) : (uint64_t(S.ml[li]) << 32);  // carry_sel reads its high word
        nA[li] = xo ^ m;
        nB[li] = yo ^ m;
        nC[li] = yn ^ m;
        nR[li] = x0 ^ carry_sel(m, mprev, sh);
        S.ml[li] = uint32_t(m >> 32);

        if constexpr (!STEADY) {
            const int sv = 5 * (l - 1);
            if (first) {
                if (l < L) {
                    c.save[(sv + 0) * kLanes] = nA[li];
                    c.save[(sv + 1) * kLanes] = nB[li];
                    c.save[(sv + 2) * kLanes] = nC[li];
                    c.save[(sv + 3) * kLanes] = nR[li];
                } else {
                    c.save[sv * kLanes] = nR[li];
                }
            }
            if (second && l < L) c.save[(sv + 4) * kLanes] = nA[li];
            if (last) {  // the x carry of the last word completes X(other) of the first word
                const uint64_t carry = carry_sel(0, m, sh);
                if (l < L) {
                    c.save[(sv + 3) * kLanes] ^= carry;
                } else {
                    const uint64_t xf = c.save[sv * kLanes] ^ carry;
                    put(c.d0 + (((L & 1) ? oXs : oXf) + size_t(l - 1) * c.Y), xf, c.core);
                }
            }
        }
        if (l == L) {
            // sweep L has parity s (L even): X(s), Y(s) own; Y(f)[y+1] = C^L[y]; X(f) via the carry
            const size_t o = size_t(j) * c.Y;
            put(c.d0 + (oXs + o), nA[li], c.core);
            put(c.d0 + (oYs + o), nB[li], c.core);
            put(c.d1 + (oYf + o), nC[li], c.core);
            if (!first) put(c.d0 + (oXf + o), nR[li], c.core);
        }
    }
}

template <int L, typename StateT>
__device__ __forceinline__ void deep_commit(StateT& S, const uint64_t (&nA)[L], const uint64_t (&nB)[L],
                                            const uint64_t (&nC)[L], const uint64_t (&nR)[L], const bool (&act)[L]) {
#pragma unroll
    for (int l = 0; l < L; ++l) {
        if (act[l]) {
            S.pA[l] = nA[l];
            S.pB[l] = nB[l];
            S.pC[l] = nC[l];
            S.pR[l] = nR[l];
        }
    }
}

// One iteration: every sweep, then commit (the block-barrier exchange follows in the caller)
template <int PM, int QM, int L, bool STEADY, bool CTR = false>
__device__ __forceinline__ void deep_iter(DeepState<L, typename std::conditional<CTR, Ctr, Xo>::type>& S,
                                          const DeepCtx& c, uint32_t i, const uint64_t* sb, int jj,
                                          const ProbDev& p, const ProbDev& q, const Geom& g, int f) {
    uint64_t nA[L] = {}, nB[L] = {}, nC[L] = {}, nR[L] = {};
    bool act[L];
    deep_sweeps<PM, QM, L, STEADY, CTR, 1, L>(S, c, i, sb, jj, p, q, g, f, nA, nB, nC, nR, act);
    deep_commit<L>(S, nA, nB, nC, nR, act);
}

// One iteration with the split-phase exchange: sweep 1 of word i, collect iteration i - 1, `refill` (thread 0's
// ring refill), sweeps 2..L, commit, publish iteration i.
template <int PM, int QM, int L, bool STEADY, bool CTR, typename Refill>
__device__ __forceinline__ void deep_iter_split(DeepState<L, typename std::conditional<CTR, Ctr, Xo>::type>& S,
                                                const DeepCtx& c, uint32_t i, const uint64_t* sb, int jj,
                                                const ProbDev& p, const ProbDev& q, const Geom& g, int f,
                                                uint64_t* xch, uint64_t* xbar, int wib, int lane, Refill&& refill) {
    uint64_t nA[L] = {}, nB[L] = {}, nC[L] = {}, nR[L] = {};
    bool act[L];
    deep_sweeps<PM, QM, L, STEADY, CTR, 1, 1>(S, c, i, sb, jj, p, q, g, f, nA, nB, nC, nR, act);
    if (STEADY || i > 0) xch_collect<L>(S, xch, xbar, i - 1, wib, lane);
    refill();
    deep_sweeps<PM, QM, L, STEADY, CTR, 2, L>(S, c, i, sb, jj, p, q, g, f, nA, nB, nC, nR, act);
    deep_commit<L>(S, nA, nB, nC, nR, act);
    xch_publish<L>(S, xch, xbar, i, wib, lane);
}

// Ring stage `slot` <- word block b of the four source planes (one 3-D TMA box each), completing on full[slot].
template <int L>
__device__ __forceinline__ void deep_issue(uint64_t* ring, uint64_t* full, const CUtensorMap* tmK,
                                           const CUtensorMap* tmK1, uint32_t blk_r0, int f, uint32_t pf,
                                           uint32_t nblocks, uint32_t b, uint32_t slot) {
    using ST = DeepStage<L>;
    uint64_t* base = ring + size_t(slot) * ST::kWords;
    const uint32_t kb = b * kKS, s_ = uint32_t(f ^ 1);
    mbar_expect_tx(&full[slot], ST::kTx);
    tma3d(base + ST::kXf, tmK, blk_r0, kb, uint32_t(f), &full[slot]);
    tma3d(base + ST::kYf, tmK, blk_r0, kb, uint32_t(2 + f), &full[slot]);
    tma3d(base + ST::kYs, tmK, blk_r0, kb, 2 + s_, &full[slot]);
    tma3d(base + ST::kXs, tmK1, blk_r0, kb, s_, &full[slot]);
    if (pf > 0 && b + pf < nblocks) {  // warm L2 pf stages ahead of the ring
        const uint32_t kp = (b + pf) * kKS;
        tma3d_prefetch(tmK, blk_r0, kp, uint32_t(f));
        tma3d_prefetch(tmK, blk_r0, kp, uint32_t(2 + f));
        tma3d_prefetch(tmK, blk_r0, kp, 2 + s_);
        tma3d_prefetch(tmK1, blk_r0, kp, s_);
    }
}

}  // namespace

// CTR: xi from the opt-in counter-based streams (octgpu_set_rng): sweep l of the pass is global sweep
// sigma0 + l - 1 of seed's streams; no stream state is loaded, parked or stored.
template <int PM, int QM, int L, bool CTR>
__global__ void __launch_bounds__(32 * kDP, kDeepMinBlocks)
    k_mcs_deep(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst, const uint64_t* __restrict__ rs,
               uint64_t* __restrict__ rd, int f, Geom g, ProbDev p, ProbDev q, const uint64_t* __restrict__ jtab, int S,
               const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmK1, uint64_t ctr_seed,
               uint64_t sigma0, const __grid_constant__ StripeLink lk) {
    static_assert(L % 2 == 0 && L >= 2, "whole MCS only");
    using GEO = DeepGeo<L>;
    using ST = DeepStage<L>;
    using SL = DeepSlots<L, PM, QM, CTR>;
    using Src = typename std::conditional<CTR, Ctr, Xo>::type;
    constexpr bool LIVE = Plan<PM, QM>::live;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t n = g.n;
    const int lane = threadIdx.x & 31;
    const int wib = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
    const uint32_t blk_r0 = g.c0 - uint32_t(L - 1) + blockIdx.x * uint32_t(GEO::kRows);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* ring = reinterpret_cast<uint64_t*>(smem_raw + 128);
    uint64_t* slots = ring + S * ST::kWords;
    uint64_t* xch = slots + SL::count() * kLanes;
    const uint32_t nblocks = (n + kKS - 1) / kKS;

    // No producer warp: thread 0 refills a ring stage right after the exchange barrier that follows the
    // word which consumed it (every warp has read the stage by then), so the ring needs only "full" barriers
    // and the block is 8 warps: two blocks per SM leave 128 registers per thread. (The tensor maps are
    // passed by address straight from the __grid_constant__ parameters: a copy in local memory is not a
    // valid TMA descriptor.)
    // a row stripe's fused halo exchange: this block's roles (block-uniform)
    bool sig = false, push = false;
    uint32_t nsig = 0;
    if (lk.active) {
        const uint32_t c0 = g.c0, c1 = g.c1, nb = gridDim.x;
        auto core_lo = [&](uint32_t b) { return max(c0, c0 + b * uint32_t(GEO::kRows)); };
        auto core_hi = [&](uint32_t b) { return min(c1, c0 + (b + 1) * uint32_t(GEO::kRows)); };  // exclusive
        auto signals = [&](uint32_t b) {  // writes what the neighbours pull: the first HB / last HA core rows
            return core_lo(b) < c0 + kStripeHB || core_hi(b) > c1 - kStripeHA;
        };
        for (uint32_t b = 0; b < nb; ++b) nsig += signals(b) ? 1u : 0u;
        sig = signals(blockIdx.x);
        push = core_hi(blockIdx.x) == c1;
        const bool above = blk_r0 < kStripeHA, below = blk_r0 + uint32_t(kLanes) > c1;
        if ((above || below) && !link_pull(lk, const_cast<uint64_t*>(src), g, above, below)) return;
    }
    // one-draw live passes: the split-phase exchange (xch_publish / xch_collect)
    constexpr bool kSplit = !CTR && ((PM == M_HALF && QM == M_ZERO) || (PM == M_ZERO && QM == M_HALF));
    uint64_t* xbar = full + kSMax;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
        if constexpr (kSplit) {
            mbar_init(&xbar[0], kDP);
            mbar_init(&xbar[1], kDP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t b = 0; b < uint32_t(S) && b < nblocks; ++b)
            deep_issue<L>(ring, full, &tmK, &tmK1, blk_r0, f, g.pf, nblocks, b, b);
    }
    __syncthreads();

    const int t = int(threadIdx.x);  // block lane = row blk_r0 + t
    const uint32_t v = blk_r0 + uint32_t(t);
    const uint32_t y = g.wrap ? v % g.wrap : v;
    const uint32_t y1 = g.wrap ? (v + 1) % g.wrap : v + 1;
    const size_t PS = g.plane_stride;
    const int s = f ^ 1;

    DeepCtx c;
    c.n = n;
    c.Y = g.Y;
    c.wrap = g.wrap;
    c.d0 = dst + y;
    c.d1 = dst + y1;
    c.sf1 = (uint32_t(f) ^ y ^ g.ypar) & 1u;
    c.sf2 = c.sf1 ^ 1u;
    c.up = (lane + 31) & 31;
    c.dn = (lane + 1) & 31;
    c.core = t >= GEO::kFirst && t <= GEO::kLast && v < g.c1;
    c.ghost_row = g.ghost && y < g.ghost;
    c.save = slots + t;

    DeepState<L, Src> R;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        R.pA[l] = R.pB[l] = R.pC[l] = R.pR[l] = 0;
        R.ml[l] = 0;
        R.rs[l] = Src{};
    }
    if constexpr (CTR && LIVE) {
#pragma unroll
        for (int l = 1; l <= L; ++l) {
            Ctr cur = ctr_row(ctr_sweep_key(ctr_seed, sigma0 + uint64_t(l - 1)), ctr_global_row(g, y));
            // words 0..l-2 of streams l >= 2 are processed last: drawn first into their slots, as for xoshiro
#pragma unroll
            for (int jw = 0; jw <= l - 2; ++jw) {
                uint64_t xp, xq;
                gen_xi<PM, QM, uint64_t>(cur, p, q, xp, xq);
                if constexpr (SL::kPreP) c.save[(SL::preP0() + SL::pre(l, jw)) * kLanes] = xp;
                if constexpr (SL::kPreQ) c.save[(SL::preQ0() + SL::pre(l, jw)) * kLanes] = xq;
            }
            R.rs[l - 1] = cur;
        }
    } else if constexpr (LIVE) {
        Xo base = load_state(rs, g.Y, y);
#pragma unroll
        for (int l = 1; l <= L; ++l) {
            if (l > 1) base = apply_table(jtab, base);  // stream l starts (l-1) n D draws after stream 1
            Xo cur = base;
            // words 0..l-2 of streams l >= 2 are processed last but drawn first
#pragma unroll
            for (int jw = 0; jw <= l - 2; ++jw) {
                uint64_t xp, xq;
                gen_xi<PM, QM, uint64_t>(cur, p, q, xp, xq);
                if constexpr (SL::kPreP) c.save[(SL::preP0() + SL::pre(l, jw)) * kLanes] = xp;
                if constexpr (SL::kPreQ) c.save[(SL::preQ0() + SL::pre(l, jw)) * kLanes] = xq;
            }
            if constexpr (SL::parked() > 0) {
                if (l - 1 >= kRegStreams)
                    slot_store(c.save, SL::st0() + 4 * (l - 1 - kRegStreams), cur);
                else
                    R.rs[l - 1] = cur;
            } else {
                R.rs[l - 1] = cur;
            }
        }
    }

    uint32_t st = 0, ph = 0;
    for (uint32_t b = 0; b < nblocks; ++b) {
        mbar_wait(&full[st], ph);
        const uint64_t* sb = ring + size_t(st) * ST::kWords + t;
        const uint32_t kb = b * kKS;
        if (b == 0) {
            R.cur = sb[ST::kXs];
            R.raw0 = R.cur;
        }
        if constexpr (kSplit) {
            // the previous stage is refilled once every warp has published its last word (the collect of this
            // block's first word): by then every warp has read it
            const uint32_t pst = st == 0 ? uint32_t(S) - 1 : st - 1;
            auto refill = [&](int jj) {
                if (jj == 0 && threadIdx.x == 0 && b > 0 && b - 1 + uint32_t(S) < nblocks)
                    deep_issue<L>(ring, full, &tmK, &tmK1, blk_r0, f, g.pf, nblocks, b - 1 + uint32_t(S), pst);
            };
            if (kb >= uint32_t(2 * L) && kb + kKS < n) {
#pragma unroll
                for (int jj = 0; jj < kKS; ++jj)
                    deep_iter_split<PM, QM, L, true, CTR>(R, c, kb + jj, sb, jj, p, q, g, f, xch, xbar, wib, lane,
                                                          [&] { refill(jj); });
            } else {
#pragma unroll 1
                for (int jj = 0; jj < kKS; ++jj)
                    if (kb + jj < n)
                        deep_iter_split<PM, QM, L, false, CTR>(R, c, kb + jj, sb, jj, p, q, g, f, xch, xbar, wib,
                                                               lane, [&] { refill(jj); });
            }
            if (++st == uint32_t(S)) {
                st = 0;
                ph ^= 1u;
            }
            continue;
        }
        if (kb >= uint32_t(2 * L) && kb + kKS < n) {  // i = n-1 is sweep 1's last word: generic
#pragma unroll
            for (int jj = 0; jj < kKS; ++jj) {
                deep_iter<PM, QM, L, true, CTR>(R, c, kb + jj, sb, jj, p, q, g, f);
                edge_exchange<L>(R, xch, kb + jj, wib, lane);
            }
        } else {
#pragma unroll 1
            for (int jj = 0; jj < kKS; ++jj) {
                if (kb + jj < n) {
                    deep_iter<PM, QM, L, false, CTR>(R, c, kb + jj, sb, jj, p, q, g, f);
                    edge_exchange<L>(R, xch, kb + jj, wib, lane);
                }
            }
        }
        // every warp is past this stage's last word (the exchange barrier): refill it
        if (threadIdx.x == 0 && b + uint32_t(S) < nblocks)
            deep_issue<L>(ring, full, &tmK, &tmK1, blk_r0, f, g.pf, nblocks, b + uint32_t(S), st);
        if (++st == uint32_t(S)) {
            st = 0;
            ph ^= 1u;
        }
    }
    // drain: sweeps 2..L finish their wrapped words
#pragma unroll 1
    for (uint32_t i = n; i < n + uint32_t(2 * L - 2); ++i) {
        if constexpr (kSplit) {
            deep_iter_split<PM, QM, L, false, CTR>(R, c, i, nullptr, 0, p, q, g, f, xch, xbar, wib, lane, [] {});
        } else {
            deep_iter<PM, QM, L, false, CTR>(R, c, i, nullptr, 0, p, q, g, f);
            edge_exchange<L>(R, xch, i, wib, lane);
        }
    }

    if constexpr (LIVE && !CTR) {
        Xo fin = R.rs[L - 1];
        if constexpr (SL::parked() > 0) fin = slot_state(c.save, SL::st0() + 4 * (L - 1 - kRegStreams));
        if (c.core) {
            store_state(rd, g.Y, y, fin);
            if (c.ghost_row) store_state(rd, g.Y, y + g.wrap, fin);
        }
    }
    if (sig) link_signal<true>(lk, dst, g, push, nsig, kLanes);
}

namespace {

template <int PM, int QM, int L, bool CTR = false>
cudaError_t deep_go(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g, const ProbDev& p,
                    const ProbDev& q, const uint64_t* jtab, int S, const CUtensorMap* tmK, const CUtensorMap* tmK1,
                    cudaStream_t st, uint64_t ctr_seed, uint64_t sigma0, const StripeLink* link) {
    using GEO = DeepGeo<L>;
    const uint32_t blocks = (g.c1 - g.c0 + GEO::kRows - 1) / GEO::kRows;
    const size_t smem = mcs_deep_smem(p.mode, q.mode, L, S, CTR);
    auto kern = k_mcs_deep<PM, QM, L, CTR>;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    StripeLink lk{};
    if (link) lk = *link;
    kern<<<blocks, 32 * kDP, smem, st>>>(static_cast<const uint64_t*>(src), static_cast<uint64_t*>(dst), rs,
                                               rd, f, g, p, q, jtab, S, *tmK, *tmK1, ctr_seed, sigma0, lk);
    return cudaGetLastError();
}

template <int L>
size_t deep_smem_l(int pm, int qm, int S, bool ctr) {
    const bool pp = !(pm == M_ZERO || pm == M_ONE), pq = !(qm == M_ZERO || qm == M_ONE);
    const int parked = !ctr && (pp || pq) && L > kRegStreams ? L - kRegStreams : 0;
    const int slots = 5 * (L - 1) + 1 + (pp ? L * (L - 1) / 2 : 0) + (pq ? L * (L - 1) / 2 : 0) + 4 * parked;
    const int xch = 2 * kDP * 2 * L;
    return 128 + size_t(S) * DeepStage<L>::kWords * 8 + size_t(slots) * kLanes * 8 + size_t(xch) * 8;
}

constexpr bool cheap_mode(int m) { return m == M_ZERO || m == M_HALF || m == M_DYADIC || m == M_ONE; }
constexpr bool const_mode(int m) { return m == M_ZERO || m == M_ONE; }

}  // namespace

bool mcs_deep_supported(int pm, int qm) {
    const bool live = !(const_mode(pm) && const_mode(qm));
    // M_ONE next to a live stream still steps w draws per word: issue-bound, keep one MCS per pass
    return cheap_mode(pm) && cheap_mode(qm) && !(live && (pm == M_ONE || qm == M_ONE));
}

// L = 6 / 8 (3 / 4 MCS per pass) only with constant xi (xoshiro streams advance lazily); a live pass keeps
// four 256-bit states per lane in registers at L = 4 (8 with counter streams would spill).
bool mcs_deep_supported_l(int pm, int qm, int L, bool ctr) {
    if (!mcs_deep_supported(pm, qm)) return false;
    if (L == kDeepSweepsLive) return true;
    if (L == kDeepSweepsConst || L == kDeepSweepsLong) return const_mode(pm) && const_mode(qm);
    return false;
}

size_t mcs_deep_smem(int pm, int qm, int L, int S, bool ctr) {
    if (L == 4) return deep_smem_l<4>(pm, qm, S, ctr);
    if (L == 6) return deep_smem_l<6>(pm, qm, S, ctr);
    if (L == 8) return deep_smem_l<8>(pm, qm, S, ctr);
    return 0;
}

namespace {

template <int PM, int QM, bool CTR>
cudaError_t deep_l(int L, const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                   const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int S, const CUtensorMap* tmK,
                   const CUtensorMap* tmK1, cudaStream_t st, uint64_t seed, uint64_t sigma,
                   const StripeLink* link) {
    if (L == 4)
        return deep_go<PM, QM, 4, CTR>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    if constexpr (const_mode(PM) && const_mode(QM)) {
        if (L == 6)
            return deep_go<PM, QM, 6, CTR>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
        if (L == 8)
            return deep_go<PM, QM, 8, CTR>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    }
    return cudaErrorInvalidValue;
}

template <int PM, bool CTR>
cudaError_t deep_q(int L, const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                   const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int S, const CUtensorMap* tmK,
                   const CUtensorMap* tmK1, cudaStream_t st, uint64_t seed, uint64_t sigma,
                   const StripeLink* link) {
    switch (q.mode) {
    case M_ZERO: return deep_l<PM, M_ZERO, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_HALF: return deep_l<PM, M_HALF, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_DYADIC:
        return deep_l<PM, M_DYADIC, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_ONE: return deep_l<PM, M_ONE, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    default: return cudaErrorInvalidValue;
    }
}

template <bool CTR>
cudaError_t deep_p(int L, const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                   const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int S, const CUtensorMap* tmK,
                   const CUtensorMap* tmK1, cudaStream_t st, uint64_t seed, uint64_t sigma,
                   const StripeLink* link) {
    if (S < 2 || S > kSMax || !mcs_deep_supported_l(p.mode, q.mode, L, CTR)) return cudaErrorInvalidValue;
    switch (p.mode) {
    case M_ZERO: return deep_q<M_ZERO, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_HALF: return deep_q<M_HALF, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_DYADIC: return deep_q<M_DYADIC, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    case M_ONE: return deep_q<M_ONE, CTR>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, seed, sigma, link);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_mcs_deep(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                            const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int L, int S,
                            const CUtensorMap* tmK, const CUtensorMap* tmK1, cudaStream_t st, const StripeLink* link) {
    return deep_p<false>(L, src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, 0, 0, link);
}

// counter-based streams (octgpu_set_rng): sweeps sigma .. sigma + L - 1 of seed's streams
cudaError_t launch_mcs_deep_ctr(const void* src, void* dst, int f, Geom g, const ProbDev& p, const ProbDev& q,
                                uint64_t seed, uint64_t sigma, int L, int S, const CUtensorMap* tmK,
                                const CUtensorMap* tmK1, cudaStream_t st, const StripeLink* link) {
    return deep_p<true>(L, src, dst, nullptr, nullptr, f, g, p, q, nullptr, S, tmK, tmK1, st, seed, sigma, link);
}

}  // namespace octgpu
