// Device helpers shared by the sm_100a kernels: xoshiro256++ and the opt-in
// counter-based streams, xi words, the Kawasaki mask. Included by kernels.cu,
// mcs_bulk.cu and mcs_deep.cu.
#pragma once
#include <cstdint>
#include <type_traits>

#include "octgpu_internal.h"

namespace octgpu {

// -------------------------------------------------------------------------
// xoshiro256++ (rng.hpp:34-44) on the device

struct Xo {
    uint64_t a, b, c, d;
};

// 64-bit shifts and rotations of the xoshiro step, spelled out on 32-bit
// halves. The arbitrary-probability path (64 draws per word) is bound by the
// ALU pipe (ncu pipe_alu 95%) while the FMA pipe idles, and the generic
// lowering of (x << k) | (x >> (64 - k)) costs 4-6 ALU instructions per
// rotation. Each half of a rotation is either one funnel shift (SHF.L.W, ALU
// pipe) or an IMAD.HI (x >> (32-k) as the high word of x * 2^k) plus an IMAD
// (x * 2^k + that) on the FMA pipe; which rotation goes to which pipe is a
// compile-time choice (OCTGPU_ROT23_FMA / OCTGPU_ROT45_FMA / OCTGPU_SHL17_FMA).
// Measured at c4 (profiles/r1_xoshiro_variants.json): all funnel shifts
// 10.39 ms/MCS; rot23 on IMAD 10.86; rot23+rot45 11.21; all IMAD 11.80 (the
// IMAD.HI issue cost outweighs the ALU relief) -> funnel shifts everywhere.
#ifndef OCTGPU_ROT23_FMA
#define OCTGPU_ROT23_FMA 0
#endif
#ifndef OCTGPU_ROT45_FMA
#define OCTGPU_ROT45_FMA 0
#endif
#ifndef OCTGPU_SHL17_FMA
#define OCTGPU_SHL17_FMA 0
#endif
__device__ __forceinline__ uint64_t pack64(uint32_t lo, uint32_t hi) { return (uint64_t(hi) << 32) | lo; }

template <int K, bool FMA>  // high 32 bits of (hi:lo) << K, 0 < K < 32
__device__ __forceinline__ uint32_t fsl(uint32_t lo, uint32_t hi) {
    if constexpr (!FMA) {
        return __funnelshift_l(lo, hi, K);
    } else {
        uint32_t r;
        asm("{\n\t.reg .u32 t;\n\tmul.hi.u32 t, %1, %3;\n\tmad.lo.u32 %0, %2, %3, t;\n\t}"
            : "=r"(r)
            : "r"(lo), "r"(hi), "n"(1u << K));
        return r;
    }
}

template <int K, bool FMA>  // 0 < K < 32
__device__ __forceinline__ uint64_t rotl64_lo(uint64_t x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    return pack64(fsl<K, FMA>(hi, lo), fsl<K, FMA>(lo, hi));
}

template <int K, bool FMA>  // 32 < K < 64: swap halves, then rotate by K - 32
__device__ __forceinline__ uint64_t rotl64_hi(uint64_t x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    return pack64(fsl<K - 32, FMA>(lo, hi), fsl<K - 32, FMA>(hi, lo));
}

template <int K, bool FMA>  // 0 < K < 32
__device__ __forceinline__ uint64_t shl64(uint64_t x) {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    return pack64(lo << K, fsl<K, FMA>(lo, hi));
}

// The xoshiro xor network as four three-input LOP3 per 32-bit half: b' = b ^ c ^ a, c' = c ^ a ^ t,
// d' = d ^ b, a' = a ^ d' (the sequential statement order of rng.hpp:34-44 compiles to 9.5 LOP3 per step:
// c ^ a is materialised and reused). OCTGPU_XO_ASM=0 restores the plain C++ statements.
#ifndef OCTGPU_XO_ASM
#define OCTGPU_XO_ASM 1
#endif
#if OCTGPU_XO_ASM
#define OCTGPU_XO_STEP_PTX                               \
    "shl.b32 t0, b0, 17;\n\t" /* t = b << 17 */         \
    "shf.l.wrap.b32 t1, b0, b1, 17;\n\t"                 \
    "xor.b32 e0, d0, b0;\n\t" /* d' = d ^ b */          \
    "xor.b32 e1, d1, b1;\n\t"                           \
    "lop3.b32 b0, b0, c0, a0, 0x96;\n\t" /* b ^ c ^ a */ \
    "lop3.b32 b1, b1, c1, a1, 0x96;\n\t"                \
    "lop3.b32 c0, c0, a0, t0, 0x96;\n\t" /* c ^ a ^ t */ \
    "lop3.b32 c1, c1, a1, t1, 0x96;\n\t"                \
    "xor.b32 a0, a0, e0;\n\t" /* a ^ d' */              \
    "xor.b32 a1, a1, e1;\n\t"                           \
    "shf.l.wrap.b32 d0, e0, e1, 13;\n\t" /* rotl 45 */   \
    "shf.l.wrap.b32 d1, e1, e0, 13;\n\t"
#define OCTGPU_XO_IN                                          \
    ".reg .u32 a0, a1, b0, b1, c0, c1, d0, d1, t0, t1, e0, e1;\n\t" \
    "mov.b64 {a0, a1}, %1;\n\t"                            \
    "mov.b64 {b0, b1}, %2;\n\t"                            \
    "mov.b64 {c0, c1}, %3;\n\t"                            \
    "mov.b64 {d0, d1}, %4;\n\t"
#define OCTGPU_XO_OUT                \
    "mov.b64 %1, {a0, a1};\n\t"     \
    "mov.b64 %2, {b0, b1};\n\t"     \
    "mov.b64 %3, {c0, c1};\n\t"     \
    "mov.b64 %4, {d0, d1};\n\t"
#endif

__device__ __forceinline__ void xo_step(Xo& s) {
#if OCTGPU_XO_ASM
    uint32_t dummy = 0;
    asm("{\n\t" OCTGPU_XO_IN OCTGPU_XO_STEP_PTX OCTGPU_XO_OUT "}"
        : "+r"(dummy), "+l"(s.a), "+l"(s.b), "+l"(s.c), "+l"(s.d));
#else
    const uint64_t t = shl64<17, OCTGPU_SHL17_FMA>(s.b);
    s.c ^= s.a;
    s.d ^= s.b;
    s.b ^= s.c;
    s.a ^= s.d;
    s.c ^= t;
    s.d = rotl64_hi<45, OCTGPU_ROT45_FMA>(s.d);
#endif
}

__device__ __forceinline__ uint64_t xo_next(Xo& s) {
    const uint64_t r = rotl64_lo<23, OCTGPU_ROT23_FMA>(s.a + s.d) + s.a;
    xo_step(s);
    return r;
}

// -------------------------------------------------------------------------
// Counter-based streams (opt-in rng mode, NOT the reference's generator; see
// octgpu_set_rng): draw i of row y in global sweep sigma is
//   mix64(origin(seed, sigma, y) + (i + 1) * gamma),
//   origin = mix64(mix64(seed + (sigma + 1) * gamma) + (y + 1) * gamma),
// i.e. SplitMix64 (the reference's seeding mixer, rng.hpp splitmix64) run as a
// Weyl sequence from a hashed per-(sweep, row) origin. No state is stored: a
// row's draws are a pure function of (seed, sigma, y, i).
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Ctr {
    uint64_t x;
};

__host__ __device__ __forceinline__ uint64_t ctr_sweep_key(uint64_t seed, uint64_t sigma) {
    return mix64(seed + (sigma + 1) * kGamma);
}

__device__ __forceinline__ Ctr ctr_row(uint64_t sweep_key, uint32_t y) {
    return Ctr{mix64(sweep_key + (uint64_t(y) + 1) * kGamma)};
}

// the lattice row whose counter stream physical row y uses (row stripes: local rows -> global rows)
__device__ __forceinline__ uint32_t ctr_global_row(const Geom& g, uint32_t y) {
    return g.gytot ? (y + g.gy0) % g.gytot : y;
}

__device__ __forceinline__ uint64_t rng_next(Ctr& s) {
    s.x += kGamma;
    return mix64(s.x);
}
__device__ __forceinline__ uint64_t rng_next(Xo& s) { return xo_next(s); }

__device__ __forceinline__ Xo load_state(const uint64_t* __restrict__ r, uint32_t Y, uint32_t y) {
    return Xo{r[y], r[size_t(Y) + y], r[2 * size_t(Y) + y], r[3 * size_t(Y) + y]};
}

__device__ __forceinline__ void store_state(uint64_t* __restrict__ r, uint32_t Y, uint32_t y, const Xo& s) {
    r[y] = s.a;
    r[size_t(Y) + y] = s.b;
    r[2 * size_t(Y) + y] = s.c;
    r[3 * size_t(Y) + y] = s.d;
}

// s <- M s with M given as a 4-bit ("four Russians") table: 64 nibble
// positions x 16 values x 4 u64 (32 KB, L1-resident after first touch).
__device__ __forceinline__ Xo apply_table(const uint64_t* __restrict__ tab, const Xo& s) {
    const uint64_t v[4] = {s.a, s.b, s.c, s.d};
    Xo r{0, 0, 0, 0};
#pragma unroll 16
    for (int i = 0; i < 64; ++i) {
        const uint32_t nib = uint32_t(v[i >> 4] >> (4 * (i & 15))) & 15u;
        const ulonglong2* e = reinterpret_cast<const ulonglong2*>(tab + (size_t(i) * 16 + nib) * 4);
        const ulonglong2 lo = __ldg(e), hi = __ldg(e + 1);
        r.a ^= lo.x;
        r.b ^= lo.y;
        r.c ^= hi.x;
        r.d ^= hi.y;
    }
    return r;
}

// -------------------------------------------------------------------------
// Arbitrary-probability xi bits, 32 draws at a time (rng.hpp:174-179).
// acc = 2*acc + (r >= T): the 64-bit compare is a subtract whose carry-out
// (= no borrow; PTX sub.cc/subc.cc, SASS IADD3 + IADD3.X) feeds an
// add-with-carry, 3 instructions per draw instead of 2 compares + select +
// or. Draw j lands at bit 31-j; one bit reverse puts it at bit j and one NOT
// turns (r >= T) into the xi bit (r < T). Rolled by bytes: fully unrolled copies of the 64-draw word at
// every call site overflow the instruction cache.
__device__ __forceinline__ uint32_t acc_ge(uint32_t acc, uint64_t r, uint64_t T) {
    uint32_t out;
    asm("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %3;\n\tsubc.cc.u32 d, %2, %4;\n\taddc.u32 %0, %5, %5;\n\t}"
        : "=r"(out)
        : "r"(uint32_t(r)), "r"(uint32_t(r >> 32)), "r"(uint32_t(T)), "r"(uint32_t(T >> 32)), "r"(acc));
    return out;
}

// One draw + compare + xoshiro step, spelled out so that the xor network is four three-input LOP3 per half
// (b ^ c ^ a, c ^ a ^ t, d ^ b, a ^ d') instead of the 9.5 LOP3 per draw the compiler derives from the
// sequential xoshiro statement order: the arbitrary-p path is bound by the ALU pipe, which LOP3, SHF and IADD3
// share. (64-bit adds as mad.wide by a runtime 1, to move them to the FMA pipe, do not survive ptxas: it splits
// them back into IMAD.WIDE + IADD3 + IMAD.X.) Same values as acc_ge(acc, xo_next(s), T).
__device__ __forceinline__ uint32_t arb_draw(Xo& s, uint32_t T0, uint32_t T1, uint32_t acc) {
#if OCTGPU_XO_ASM
    asm("{\n\t" OCTGPU_XO_IN
        ".reg .u32 u0, u1, r0, r1, x0, x1, z;\n\t"
        "add.cc.u32 u0, a0, d0;\n\t"  // u = a + d
        "addc.u32 u1, a1, d1;\n\t"
        "shf.l.wrap.b32 r1, u0, u1, 23;\n\t"  // rotl(u, 23)
        "shf.l.wrap.b32 r0, u1, u0, 23;\n\t"
        "add.cc.u32 x0, r0, a0;\n\t"  // x = rotl(u, 23) + a
        "addc.u32 x1, r1, a1;\n\t"
        "sub.cc.u32 z, x0, %5;\n\t"  // acc = 2 acc + (x >= T)
        "subc.cc.u32 z, x1, %6;\n\t"
        "addc.u32 %0, %0, %0;\n\t" OCTGPU_XO_STEP_PTX OCTGPU_XO_OUT "}"
        : "+r"(acc), "+l"(s.a), "+l"(s.b), "+l"(s.c), "+l"(s.d)
        : "r"(T0), "r"(T1));
    return acc;
#else
    return acc_ge(acc, xo_next(s), (uint64_t(T1) << 32) | T0);
#endif
}

template <typename Word>
__device__ __forceinline__ uint32_t arb_half(Xo& s, const ProbDev& pd) {
    const uint32_t T0 = uint32_t(pd.T), T1 = uint32_t(pd.T >> 32);
    uint32_t acc = 0;
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) acc = arb_draw(s, T0, T1, acc);
    }
    return ~__brev(acc);
}

// two independent streams interleaved draw by draw (instruction-level parallelism)
__device__ __forceinline__ void arb_half_pair(Xo& a, Xo& b, const ProbDev& pd, uint32_t& ra, uint32_t& rb) {
    const uint32_t T0 = uint32_t(pd.T), T1 = uint32_t(pd.T >> 32);
    uint32_t acca = 0, accb = 0;
#pragma unroll 1
    for (int it = 0; it < 4; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acca = arb_draw(a, T0, T1, acca);
            accb = arb_draw(b, T0, T1, accb);
        }
    }
    ra = ~__brev(acca);
    rb = ~__brev(accb);
}

// -------------------------------------------------------------------------
// xi words (rng.hpp:129-179, params.hpp:84-92)

template <int MODE, typename Word, typename R>
__device__ __forceinline__ Word xi_word(R& s, const ProbDev& pd) {
    constexpr int W = int(sizeof(Word) * 8);
    constexpr bool XO = std::is_same<R, Xo>::value;
    if constexpr (MODE == M_ZERO) {
        return Word(0);
    } else if constexpr (MODE == M_HALF) {
        return Word(rng_next(s));  // xi_half: low w bits of one draw
    } else if constexpr (MODE == M_DYADIC) {
        Word acc = Word(rng_next(s));  // Horner over the digits of m, LSB first
        for (uint32_t i = 1; i < pd.k; ++i) {
            const Word x = Word(rng_next(s));
            acc = ((pd.m >> i) & 1) ? Word(acc | x) : Word(acc & x);
        }
        return acc;
    } else if constexpr (MODE == M_ARB) {
        // xi_arbitrary: bit i = to_unit(draw_i) < r  <=>  draw_i < T (integer threshold)
        if constexpr (XO) {
            const uint32_t lo = arb_half<Word>(s, pd);
            if constexpr (W == 32) {
                return Word(lo);
            } else {
                return Word(pack64(lo, arb_half<Word>(s, pd)));
            }
        } else {
            Word acc = 0;
#pragma unroll 4
            for (int i = 0; i < W; ++i) acc |= Word(rng_next(s) < pd.T ? 1 : 0) << i;
            return acc;
        }
    } else {  // M_ONE: every bit accepted, stream still advances w draws
        if constexpr (XO) {
#pragma unroll 8
            for (int i = 0; i < W; ++i) xo_step(s);
        } else {
            s.x += uint64_t(W) * kGamma;
        }
        return Word(~Word(0));
    }
}

template <int PM, int QM>
struct Plan {
    static constexpr bool p_const = (PM == M_ZERO || PM == M_ONE);
    static constexpr bool q_const = (QM == M_ZERO || QM == M_ONE);
    static constexpr bool live = !(p_const && q_const);  // any draw needs a live stream
};

template <int PM, int QM, typename Word, typename R>
__device__ __forceinline__ void gen_xi(R& s, const ProbDev& p, const ProbDev& q, Word& xp, Word& xq) {
    if constexpr (Plan<PM, QM>::live) {
        xp = xi_word<PM, Word>(s, p);
        xq = (QM == M_ZERO) ? Word(0) : xi_word<QM, Word>(s, q);  // engine_vec.hpp:105,125
    } else {
        xp = (PM == M_ONE) ? Word(~Word(0)) : Word(0);
        xq = (QM == M_ONE) ? Word(~Word(0)) : Word(0);
    }
}

// Two independent streams at once (the fused MCS kernel's first-sweep stream
// for word k and second-sweep stream for word k-1): the same draws in the
// same per-stream order, interleaved draw by draw for instruction-level
// parallelism (each xoshiro step is a serial dependency chain).
template <int MODE, typename Word>
__device__ __forceinline__ void xi_word_pair(Xo& a, Xo& b, const ProbDev& pd, Word& wa, Word& wb) {
    constexpr int W = int(sizeof(Word) * 8);
    if constexpr (MODE == M_ZERO) {
        wa = wb = Word(0);
    } else if constexpr (MODE == M_HALF) {
        wa = Word(xo_next(a));
        wb = Word(xo_next(b));
    } else if constexpr (MODE == M_DYADIC) {
        Word ra = Word(xo_next(a)), rb = Word(xo_next(b));
        for (uint32_t i = 1; i < pd.k; ++i) {
            const Word xa = Word(xo_next(a)), xb = Word(xo_next(b));
            const bool orop = (pd.m >> i) & 1;
            ra = orop ? Word(ra | xa) : Word(ra & xa);
            rb = orop ? Word(rb | xb) : Word(rb & xb);
        }
        wa = ra;
        wb = rb;
    } else if constexpr (MODE == M_ARB) {
        uint32_t la, lb;
        arb_half_pair(a, b, pd, la, lb);
        if constexpr (W == 32) {
            wa = Word(la);
            wb = Word(lb);
        } else {
            uint32_t ha, hb;
            arb_half_pair(a, b, pd, ha, hb);
            wa = Word(pack64(la, ha));
            wb = Word(pack64(lb, hb));
        }
    } else {  // M_ONE
#pragma unroll 8
        for (int i = 0; i < W; ++i) {
            xo_step(a);
            xo_step(b);
        }
        wa = wb = Word(~Word(0));
    }
}

// counter-based streams: two independent draw chains as they are (no state to interleave)
template <int PM, int QM, typename Word>
__device__ __forceinline__ void gen_xi_pair(Ctr& a, Ctr& b, const ProbDev& p, const ProbDev& q, Word& ap, Word& aq,
                                            Word& bp, Word& bq) {
    gen_xi<PM, QM, Word>(a, p, q, ap, aq);
    gen_xi<PM, QM, Word>(b, p, q, bp, bq);
}

template <int PM, int QM, typename Word>
__device__ __forceinline__ void gen_xi_pair(Xo& a, Xo& b, const ProbDev& p, const ProbDev& q, Word& ap, Word& aq,
                                            Word& bp, Word& bq) {
    if constexpr (Plan<PM, QM>::live) {
        xi_word_pair<PM, Word>(a, b, p, ap, bp);
        if constexpr (QM == M_ZERO) {
            aq = bq = Word(0);
        } else {
            xi_word_pair<QM, Word>(a, b, q, aq, bq);
        }
    } else {
        ap = bp = (PM == M_ONE) ? Word(~Word(0)) : Word(0);
        aq = bq = (QM == M_ONE) ? Word(~Word(0)) : Word(0);
    }
}

// x+ neighbour alignment and its inverse as branch-free funnel shifts, with
// s = 1 on rows whose sites sit at odd packed positions (engine_vec.hpp:34-88):
//   rot_sel(x0, x1, s)     = s ? (x0 >> 1) | (x1 << 63) : x0     (gather_xplus, word k and k+1)
//   carry_sel(m, mp, s)    = s ? (m << 1) | (mp >> 63) : m       (scatter_xplus, word k and k-1)
// Two SHF.R.W / SHF.L.W per 64-bit result instead of shift + shift + or + 2 selects.
__device__ __forceinline__ uint64_t rot_sel(uint64_t x0, uint64_t x1, uint32_t s) {
    const uint32_t l0 = uint32_t(x0), h0 = uint32_t(x0 >> 32), l1 = uint32_t(x1);
    return (uint64_t(__funnelshift_r(h0, l1, s)) << 32) | __funnelshift_r(l0, h0, s);
}
__device__ __forceinline__ uint64_t carry_sel(uint64_t m, uint64_t mp, uint32_t s) {
    const uint32_t l = uint32_t(m), h = uint32_t(m >> 32), hp = uint32_t(mp >> 32);
    return (uint64_t(__funnelshift_l(l, h, s)) << 32) | __funnelshift_l(hp, l, s);
}

// engine_vec.hpp:25-30
template <typename Word>
__device__ __forceinline__ Word update_mask(Word sxm, Word sym, Word sxp, Word syp, Word xp, Word xq) {
    const Word mp = xp & ~(sxm | sym) & sxp & syp;
    const Word mq = xq & ~(sxp | syp) & sxm & sym;
    return Word(mp ^ mq);
}

}  // namespace octgpu
