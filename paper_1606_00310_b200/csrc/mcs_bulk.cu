// Fused MCS kernel, v3: warp-specialised TMA pipeline.
// Each block = kP consumer warps (30 core rows each, one halo row on each side
// recomputed redundantly) + 1 producer warp. The producer streams the block's
// (30*kP + 4)-row window of the four src planes, KS words per stage, into an
// S-stage shared-memory ring with 3-D TMA tile copies (SASS UTMALDG) that
// complete on per-stage "full" mbarriers; the consumers release a stage by
// arriving on its "empty" mbarrier.
// Measured predecessors (profiles/): v2 issued the copies from lane 0 of every
// compute warp, 34-row boxes per warp: the issuing warp stalled on the TMA
// issue (36% of stall samples on the UTMALDG loop) and the 34/30 row overlap
// re-read 9% of the planes from DRAM. One block box of 124 rows per plane cuts
// the copy count 4x and the overlap to 124/120.
//
// Same algorithm and bit-exact results as k_mcs in kernels.cu (sweep f, then
// sweep f^1, src -> dst). Lane -> row mapping: consumer warp c of block b owns
// the virtual rows r0 = c0 - 1 + 30*(kP*b + c) + lane, core lanes 1..30.
// Stores are predicated in PTX (no divergent branches).
// Used for w = 64, n >= 8 and (periodic) Y >= kGhostRows; smaller lattices take k_mcs.
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "device_common.cuh"
#include "octgpu_internal.h"
#include "stripe_link.cuh"

namespace octgpu {

namespace {

constexpr int kP = kMcsConsumerWarps;  // consumer warps per block
constexpr int kWin = kTmaBoxRows;      // window rows: 30*kP core rows + halos, lane 31's Y(s)[y+1], even
static_assert(kWin == 30 * kP + 4, "TMA box rows must cover the block window");

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
    // relaxed: the producer has no generic-proxy writes to publish
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Consumer release of a stage. relaxed: the default .release would fence
// (MEMBAR.ALL.CTA) every outstanding global store; the stage's shared-memory
// reads have completed anyway, since the stores issued before this arrive
// consume their values (in-order issue).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// One 3-D TMA tile copy (SASS UTMALDG): box at (row, word, plane) of the
// tensor map lands in shared memory as [words][rows]. Operands are uniform.
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

__device__ __forceinline__ void st_pred(uint64_t* p, uint64_t v, bool pred) {
    asm volatile(
        "{\n"
        ".reg .pred q;\n"
        "setp.ne.b32 q, %2, 0;\n"
        "@q st.global" OCTGPU_ST_HINT ".b64 [%0], %1;\n"
        "}\n" ::"l"(p),
        "l"(v), "r"(int(pred)));
}

// Stage layout (uint64 words), every segment 128-B aligned for the TMA:
// Xf[KS][kWin] | Yf[KS][kWin] | Ys[KS][kWin] | Xs[KS+1][kWin]
constexpr int align16w(int words) { return (words + 15) / 16 * 16; }
template <int KS>
struct StageLayout {
    static constexpr int kSeg = align16w(KS * kWin);
    static constexpr int kXf = 0;
    static constexpr int kYf = kSeg;
    static constexpr int kYs = 2 * kSeg;
    static constexpr int kXs = 3 * kSeg;
    static constexpr int kWords = 3 * kSeg + align16w((KS + 1) * kWin);
    static constexpr int kBytes = kWords * 8;
    static constexpr uint32_t kTx = (4 * KS + 1) * kWin * 8;  // bytes landed per stage (full boxes)
};

constexpr int kBarBytes = 2 * 8 * 8;  // full[8] | empty[8]

}  // namespace

size_t mcs_bulk_stage_bytes(int ks) {
    return ks == 4 ? StageLayout<4>::kBytes : ks == 2 ? StageLayout<2>::kBytes : StageLayout<1>::kBytes;
}

// CTR: xi from the opt-in counter-based streams (octgpu_set_rng): sweep keys ck1 / ck2, no stream state
// loaded or stored.
template <int PM, int QM, int KS, bool CTR>
__global__ void __launch_bounds__(32 * (kP + 1), kP >= 8 ? 2 : 4) k_mcs_bulk(const uint64_t* __restrict__ src,
                                                            uint64_t* __restrict__ dst,
                                                            const uint64_t* __restrict__ rs,
                                                            uint64_t* __restrict__ rd, int f, Geom g, ProbDev p,
                                                            ProbDev q, const uint64_t* __restrict__ jtab, int S,
                                                            const __grid_constant__ CUtensorMap tmK,
                                                            const __grid_constant__ CUtensorMap tmK1,
                                                            uint64_t ck1, uint64_t ck2,
                                                            const __grid_constant__ StripeLink lk) {
    using Word = uint64_t;
    using LY = StageLayout<KS>;
    constexpr bool LIVE = Plan<PM, QM>::live;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t Y = g.Y, n = g.n;
    const int lane = threadIdx.x & 31;
    // warp in block, through a shuffle so the compiler sees it as warp-uniform
    const int wib = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0);
    const uint32_t rows = g.c1 - g.c0;
    const uint32_t blk_r0 = g.c0 - 1 + blockIdx.x * (30u * kP);  // virtual row of the window's first row
    // consumer warps of this block that own core rows (the last block may have fewer)
    const uint32_t left = rows - blockIdx.x * (30u * kP);
    const uint32_t nact = min(uint32_t(kP), (left + 29) / 30);
    const uint32_t s_ = uint32_t(f ^ 1);

    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + 8;
    Word* ring = reinterpret_cast<Word*>(smem_raw + kBarBytes);
    const uint32_t nblocks = (n + KS - 1) / KS;

    // a row stripe's fused halo exchange (stripe_link.cuh): this block's roles (block-uniform)
    bool sig = false, push = false;
    uint32_t nsig = 0;
    if (lk.active) {
        const uint32_t c0 = g.c0, c1 = g.c1, nb = gridDim.x, K = 30u * kP;
        auto core_lo = [&](uint32_t b) { return c0 + b * K; };
        auto core_hi = [&](uint32_t b) { return min(c1, c0 + (b + 1) * K); };  // exclusive
        auto signals = [&](uint32_t b) { return core_lo(b) < c0 + kStripeHB || core_hi(b) > c1 - kStripeHA; };
        for (uint32_t b = 0; b < nb; ++b) nsig += signals(b) ? 1u : 0u;
        sig = signals(blockIdx.x);
        push = core_hi(blockIdx.x) == c1;
        const bool above = blk_r0 < kStripeHA, below = blk_r0 + uint32_t(kWin) > c1;
        if ((above || below) && !link_pull(lk, const_cast<uint64_t*>(src), g, above, below)) return;
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], nact);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (wib == kP) {
        // ---- producer warp: one lane streams the window, KS words per stage ----
        if (lane == 0) {
            if (lk.active) asm volatile("fence.proxy.async.global;" ::: "memory");  // after a halo pull
            uint32_t st = 0, ph = 0;  // stage, and the parity of its fill round
            for (uint32_t b = 0; b < nblocks; ++b) {
                if (b >= uint32_t(S)) mbar_wait(&empty[st], ph ^ 1u);
                Word* base = ring + size_t(st) * LY::kWords;
                const uint32_t kb = b * KS;
                mbar_expect_tx(&full[st], LY::kTx);
                tma3d(base + LY::kXf, &tmK, blk_r0, kb, uint32_t(f), &full[st]);
                tma3d(base + LY::kYf, &tmK, blk_r0, kb, uint32_t(2 + f), &full[st]);
                tma3d(base + LY::kYs, &tmK, blk_r0, kb, 2 + s_, &full[st]);
                tma3d(base + LY::kXs, &tmK1, blk_r0, kb, s_, &full[st]);
                if (g.pf > 0 && b + g.pf < nblocks) {  // warm L2 pf stages ahead of the ring
                    const uint32_t kp = (b + g.pf) * KS;
                    tma3d_prefetch(&tmK, blk_r0, kp, uint32_t(f));
                    tma3d_prefetch(&tmK, blk_r0, kp, uint32_t(2 + f));
                    tma3d_prefetch(&tmK, blk_r0, kp, 2 + s_);
                    tma3d_prefetch(&tmK1, blk_r0, kp, s_);
                }
                if (++st == uint32_t(S)) {
                    st = 0;
                    ph ^= 1u;
                }
            }
        }
        return;
    }
    if (uint32_t(wib) >= nact) return;  // warp-uniform
    const uint32_t r0 = blk_r0 + 30u * wib;  // virtual row of lane 0
    const int wrow = 30 * wib + lane;        // this lane's row in the window
    const uint32_t v = r0 + lane;  // virtual row
    const uint32_t y = g.wrap ? v % g.wrap : v;
    const bool core = lane >= 1 && lane <= 30 && v < g.c1;
    const bool wyf = lane >= 2 && v - 1 < g.c1;  // row v-1 is core: this lane writes Y(f)[v]
    const int s = f ^ 1;
    const size_t PS = g.plane_stride;
    Word* dXf = dst + size_t(0 + f) * PS + y;
    Word* dYf = dst + size_t(2 + f) * PS + y;
    Word* dXs = dst + size_t(0 + s) * PS + y;
    Word* dYs = dst + size_t(2 + s) * PS + y;
    const uint32_t sf1 = (uint32_t(f) ^ y ^ g.ypar) & 1u;  // first sweep: x+ neighbour shifted by one bit
    const uint32_t sf2 = sf1 ^ 1u;

    // Periodic lattices keep ghost rows wrap..wrap+ghost-1 equal to rows
    // 0..ghost-1, so a block window never wraps; warps that store rows
    // 0..ghost-1 (the first few and the last) also refresh those ghosts.
    const bool ghostw = g.ghost && (r0 + 1 < g.ghost || r0 + 31 >= g.wrap);  // warp-uniform
    const bool ghost_row = ghostw && y < g.ghost;

    using Src = typename std::conditional<CTR, Ctr, Xo>::type;
    Src st1{}, st2{};  // first / second sweep streams
    if constexpr (CTR) {
        const uint32_t gy = ctr_global_row(g, y);
        st1 = ctr_row(ck1, gy);
        st2 = ctr_row(ck2, gy);
    } else if constexpr (LIVE) {
        st1 = load_state(rs, Y, y);
        st2 = apply_table(jtab, st1);
    }
    Word xi2p0, xi2q0;
    gen_xi<PM, QM, Word>(st2, p, q, xi2p0, xi2q0);

    Word A0 = 0, B0 = 0, C0 = 0, R0 = 0, A1 = 0;
    Word pA = 0, pB = 0, pC = 0, pR = 0;
    Word m1last = 0, m2last = 0, xf1 = 0;
    Word cur = 0, raw0 = 0;

    // predicated store, mirrored into the ghost row when this is one of rows 0..ghost-1;
    // gh = integral_constant: 0 / 1 = warp-uniform ghostw hoisted out of the loop, 2 = checked here
    auto putg = [&](auto gh, Word* ptr, Word val, bool pred) {
        st_pred(ptr, val, pred);
        if constexpr (decltype(gh)::value == 1) st_pred(ptr + g.wrap, val, pred && ghost_row);
        if constexpr (decltype(gh)::value == 2)
            if (ghostw) st_pred(ptr + g.wrap, val, pred && ghost_row);
    };
    auto put = [&](Word* ptr, Word val, bool pred) {
        st_pred(ptr, val, pred);
        if (ghostw) st_pred(ptr + g.wrap, val, pred && ghost_row);
    };

    auto second = [&](auto gh, uint32_t j, Word Aj, Word Ajn, Word Bj, Word Cj, Word Rj, Word x2p, Word x2q) {
        const Word Cup = __shfl_up_sync(0xffffffffu, Cj, 1);
        const Word Bdn = __shfl_down_sync(0xffffffffu, Bj, 1);
        const Word sxp2 = rot_sel(Aj, Ajn, sf2);
        const Word m2 = update_mask<Word>(Rj, Cup, sxp2, Bdn, x2p, x2q);
        const Word mup = __shfl_up_sync(0xffffffffu, m2, 1);
        const uint32_t o = j * Y;  // < 2^32: n * Y words per plane
        putg(gh, dXs + o, Rj ^ m2, core);
        putg(gh, dYs + o, Cup ^ m2, core);
        putg(gh, dYf + o, Bj ^ mup, wyf);
        return m2;
    };
    const std::integral_constant<int, 2> GHOST{};

    uint32_t st = 0, ph = 0;  // ring stage and the parity of its current fill
    for (uint32_t b = 0; b < nblocks; ++b) {
        mbar_wait(&full[st], ph);
        const Word* sb = ring + size_t(st) * LY::kWords;
        const uint32_t kb = b * KS;
        if (b == 0) {
            cur = sb[LY::kXs + wrow];  // X(s)[y][0], original
            raw0 = cur;
        }
        // arbitrary-probability bodies are ~10^4 instructions per word: keep them rolled (I-cache)
        constexpr int kUnroll = (PM == M_ARB || QM == M_ARB) ? 1 : KS;
        if (kb >= 3 && kb + KS <= n) {
            // steady state: words k >= 3, second sweep of word k-1 >= 2, no special cases
            auto steady = [&](auto gh) {
#pragma unroll kUnroll
                for (int jj = 0; jj < KS; ++jj) {
                    const uint32_t k = kb + jj;
                    const Word A = sb[LY::kXf + jj * kWin + wrow];
                    const Word B = sb[LY::kYf + jj * kWin + wrow];
                    const Word Cn = sb[LY::kYs + jj * kWin + wrow + 1];
                    const Word nxt = (k + 1 == n) ? raw0 : sb[LY::kXs + (jj + 1) * kWin + wrow];
                    Word x1p, x1q, x2p, x2q;
                    gen_xi_pair<PM, QM, Word>(st1, st2, p, q, x1p, x1q, x2p, x2q);
                    const Word sxp = rot_sel(cur, nxt, sf1);
                    const Word m1 = update_mask<Word>(A, B, sxp, Cn, x1p, x1q);
                    const Word Ap = A ^ m1, Bp = B ^ m1, Cp = Cn ^ m1;
                    const Word Rp = cur ^ carry_sel(m1, m1last, sf1);
                    m1last = m1;
                    cur = nxt;
                    const Word m2 = second(gh, k - 1, pA, Ap, pB, pC, pR, x2p, x2q);
                    putg(gh, dXf + (k - 1) * Y, pA ^ carry_sel(m2, m2last, sf2), core);
                    m2last = m2;
                    pA = Ap; pB = Bp; pC = Cp; pR = Rp;
                }
            };
            if constexpr (kUnroll == 1) {  // arbitrary-p bodies: one copy (instruction cache)
                steady(std::integral_constant<int, 2>{});
            } else if (ghostw) {
                steady(std::integral_constant<int, 1>{});
            } else {
                steady(std::integral_constant<int, 0>{});
            }
        } else {
#pragma unroll kUnroll
            for (int jj = 0; jj < KS; ++jj) {
                const uint32_t k = kb + jj;
                if (k >= n) break;
                const Word A = sb[LY::kXf + jj * kWin + wrow];
                const Word B = sb[LY::kYf + jj * kWin + wrow];
                const Word Cn = sb[LY::kYs + jj * kWin + wrow + 1];
                const Word nxt = (k + 1 == n) ? raw0 : sb[LY::kXs + (jj + 1) * kWin + wrow];
                // ---- xi for first sweep word k and (k >= 2) second sweep word k-1, interleaved ----
                Word x1p, x1q, x2p = 0, x2q = 0;
                if (k >= 2)
                    gen_xi_pair<PM, QM, Word>(st1, st2, p, q, x1p, x1q, x2p, x2q);
                else
                    gen_xi<PM, QM, Word>(st1, p, q, x1p, x1q);
                // ---- first sweep, word k ----
                const Word sxp = rot_sel(cur, nxt, sf1);
                const Word m1 = update_mask<Word>(A, B, sxp, Cn, x1p, x1q);
                const Word Ap = A ^ m1, Bp = B ^ m1, Cp = Cn ^ m1;
                const Word Rp = cur ^ carry_sel(m1, m1last, sf1);  // word 0: m1last = 0, carry of word n-1 added last
                m1last = m1;
                cur = nxt;
                if (k == 0) {
                    A0 = Ap; B0 = Bp; C0 = Cp; R0 = Rp;
                } else {
                    if (k == 1) A1 = Ap;
                    if (k >= 2) {
                        const uint32_t j = k - 1;
                        const Word m2 = second(GHOST, j, pA, Ap, pB, pC, pR, x2p, x2q);
                        if (j == 1)
                            xf1 = pA ^ carry_sel(m2, 0, sf2);  // word 0's carry comes last
                        else
                            put(dXf + j * Y, pA ^ carry_sel(m2, m2last, sf2), core);
                        m2last = m2;
                    }
                }
                pA = Ap; pB = Bp; pC = Cp; pR = Rp;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (++st == uint32_t(S)) {
            st = 0;
            ph ^= 1u;
        }
    }
    R0 ^= carry_sel(0, m1last, sf1);  // periodic seam: carry of word n-1 into word 0
    {
        const uint32_t j = n - 1;  // n >= 8 here
        Word x2p, x2q;
        gen_xi<PM, QM, Word>(st2, p, q, x2p, x2q);
        const Word m2 = second(GHOST, j, pA, A0, pB, pC, pR, x2p, x2q);
        put(dXf + j * Y, pA ^ carry_sel(m2, m2last, sf2), core);
        m2last = m2;
    }
    {
        const Word m2 = second(GHOST, 0, A0, A1, B0, C0, R0, xi2p0, xi2q0);
        put(dXf, A0 ^ carry_sel(m2, m2last, sf2), core);
        put(dXf + Y, xf1 ^ carry_sel(0, m2, sf2), core);
    }
    if constexpr (LIVE && !CTR) {
        // a row stripe also advances the streams of the halo rows next to its core rows
        // (the peer-memory halo exchange pulls neighbour states only once, p2p.cu)
        const bool halo_state = g.wrap == 0 && (v + 1 == g.c0 || v == g.c1);
        if (core || halo_state) store_state(rd, Y, y, st2);
        if (core && ghost_row) store_state(rd, Y, y + g.wrap, st2);
    }
    if (sig) link_signal<false>(lk, dst, g, push, nsig, 32u * nact);  // the compute warps (producer / idle ones exited)
}

namespace {

template <int PM, int QM, int KS, bool CTR = false>
cudaError_t bulk_go(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g, const ProbDev& p,
                    const ProbDev& q, const uint64_t* jtab, int S, const CUtensorMap* tmK, const CUtensorMap* tmK1,
                    cudaStream_t st, uint64_t ck1, uint64_t ck2, const StripeLink* link) {
    const uint32_t warps = (g.c1 - g.c0 + 29) / 30;
    const uint32_t threads = 32 * (kP + 1), blocks = (warps + kP - 1) / kP;
    const size_t smem = mcs_bulk_smem(KS, S);
    auto kern = k_mcs_bulk<PM, QM, KS, CTR>;
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    StripeLink lk{};
    if (link) lk = *link;
    kern<<<blocks, threads, smem, st>>>(static_cast<const uint64_t*>(src), static_cast<uint64_t*>(dst), rs, rd, f, g,
                                        p, q, jtab, S, *tmK, *tmK1, ck1, ck2, lk);
    return cudaGetLastError();
}

template <int PM, int QM>
cudaError_t bulk_pq(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g, const ProbDev& p,
                    const ProbDev& q, const uint64_t* jtab, int ks, int S, const CUtensorMap* tmK,
                    const CUtensorMap* tmK1, cudaStream_t st, const StripeLink* link) {
    switch (ks) {
    case 1: return bulk_go<PM, QM, 1>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, 0, 0, link);
    case 2: return bulk_go<PM, QM, 2>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, 0, 0, link);
    case 4: return bulk_go<PM, QM, 4>(src, dst, rs, rd, f, g, p, q, jtab, S, tmK, tmK1, st, 0, 0, link);
    default: return cudaErrorInvalidValue;
    }
}

#define OCT_BQ(PM)                                                                              \
    switch (q.mode) {                                                                           \
    case M_ZERO: return bulk_pq<PM, M_ZERO>(src, dst, rs, rd, f, g, p, q, jtab, ks, S, tmK, tmK1, st, link);     \
    case M_HALF: return bulk_pq<PM, M_HALF>(src, dst, rs, rd, f, g, p, q, jtab, ks, S, tmK, tmK1, st, link);     \
    case M_DYADIC: return bulk_pq<PM, M_DYADIC>(src, dst, rs, rd, f, g, p, q, jtab, ks, S, tmK, tmK1, st, link); \
    case M_ARB: return bulk_pq<PM, M_ARB>(src, dst, rs, rd, f, g, p, q, jtab, ks, S, tmK, tmK1, st, link);       \
    case M_ONE: return bulk_pq<PM, M_ONE>(src, dst, rs, rd, f, g, p, q, jtab, ks, S, tmK, tmK1, st, link);       \
    default: return cudaErrorInvalidValue;                                                      \
    }

}  // namespace

size_t mcs_bulk_smem(int ks, int S) { return kBarBytes + size_t(S) * mcs_bulk_stage_bytes(ks); }

cudaError_t launch_mcs_bulk(const void* src, void* dst, const uint64_t* rs, uint64_t* rd, int f, Geom g,
                            const ProbDev& p, const ProbDev& q, const uint64_t* jtab, int ks, int S,
                            const CUtensorMap* tmK, const CUtensorMap* tmK1, cudaStream_t st, const StripeLink* link) {
    switch (p.mode) {
    case M_ZERO: OCT_BQ(M_ZERO)
    case M_HALF: OCT_BQ(M_HALF)
    case M_DYADIC: OCT_BQ(M_DYADIC)
    case M_ARB: OCT_BQ(M_ARB)
    case M_ONE: OCT_BQ(M_ONE)
    default: return cudaErrorInvalidValue;
    }
}

// counter-based streams: KS = 2 only (the engine's plan)
#define OCT_CTR_ARGS src, dst, nullptr, nullptr, f, g, p, q, nullptr, S, tmK, tmK1, st, k1, k2, link
#define OCT_BQC(PM)                                                           \
    switch (q.mode) {                                                         \
    case M_ZERO: return bulk_go<PM, M_ZERO, 2, true>(OCT_CTR_ARGS);         \
    case M_HALF: return bulk_go<PM, M_HALF, 2, true>(OCT_CTR_ARGS);         \
    case M_DYADIC: return bulk_go<PM, M_DYADIC, 2, true>(OCT_CTR_ARGS);     \
    case M_ARB: return bulk_go<PM, M_ARB, 2, true>(OCT_CTR_ARGS);           \
    case M_ONE: return bulk_go<PM, M_ONE, 2, true>(OCT_CTR_ARGS);           \
    default: return cudaErrorInvalidValue;                                    \
    }

cudaError_t launch_mcs_bulk_ctr(const void* src, void* dst, int f, Geom g, const ProbDev& p, const ProbDev& q,
                                uint64_t seed, uint64_t sigma, int S, const CUtensorMap* tmK, const CUtensorMap* tmK1,
                                cudaStream_t st, const StripeLink* link) {
    const uint64_t k1 = ctr_sweep_key(seed, sigma), k2 = ctr_sweep_key(seed, sigma + 1);
    switch (p.mode) {
    case M_ZERO: OCT_BQC(M_ZERO)
    case M_HALF: OCT_BQC(M_HALF)
    case M_DYADIC: OCT_BQC(M_DYADIC)
    case M_ARB: OCT_BQC(M_ARB)
    case M_ONE: OCT_BQC(M_ONE)
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace octgpu
