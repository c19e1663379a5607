// Device helpers shared by the sm_100a kernels: xoshiro256++, xi words,
// the Kawasaki mask. Included by kernels.cu and mcs_bulk.cu only.
#pragma once
#include <cstdint>

#include "octgpu_internal.h"

namespace octgpu {

// -------------------------------------------------------------------------
// xoshiro256++ (rng.hpp:34-44) on the device

struct Xo {
    uint64_t a, b, c, d;
};

__device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

__device__ __forceinline__ void xo_step(Xo& s) {
    const uint64_t t = s.b << 17;
    s.c ^= s.a;
    s.d ^= s.b;
    s.b ^= s.c;
    s.a ^= s.d;
    s.c ^= t;
    s.d = rotl64(s.d, 45);
}

__device__ __forceinline__ uint64_t xo_next(Xo& s) {
    const uint64_t r = rotl64(s.a + s.d, 23) + s.a;
    xo_step(s);
    return r;
}

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
// xi words (rng.hpp:129-179, params.hpp:84-92)

template <int MODE, typename Word>
__device__ __forceinline__ Word xi_word(Xo& s, const ProbDev& pd) {
    constexpr int W = int(sizeof(Word) * 8);
    if constexpr (MODE == M_ZERO) {
        return Word(0);
    } else if constexpr (MODE == M_HALF) {
        return Word(xo_next(s));  // xi_half: low w bits of one draw
    } else if constexpr (MODE == M_DYADIC) {
        Word acc = Word(xo_next(s));  // Horner over the digits of m, LSB first
        for (uint32_t i = 1; i < pd.k; ++i) {
            const Word x = Word(xo_next(s));
            acc = ((pd.m >> i) & 1) ? Word(acc | x) : Word(acc & x);
        }
        return acc;
    } else if constexpr (MODE == M_ARB) {
        // xi_arbitrary: bit i = to_unit(draw_i) < r  <=>  draw_i < T (integer threshold).
        // Rolled by bytes: the word is ~W x 22 instructions, and fully unrolled
        // copies at every call site overflow the instruction cache.
        Word word = 0;
#pragma unroll 1
        for (int i0 = 0; i0 < W; i0 += 8) {
            uint32_t byte = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) byte |= uint32_t(xo_next(s) < pd.T) << j;
            word |= Word(byte) << i0;
        }
        return word;
    } else {  // M_ONE: every bit accepted, stream still advances w draws
#pragma unroll 8
        for (int i = 0; i < W; ++i) xo_step(s);
        return Word(~Word(0));
    }
}

template <int PM, int QM>
struct Plan {
    static constexpr bool p_const = (PM == M_ZERO || PM == M_ONE);
    static constexpr bool q_const = (QM == M_ZERO || QM == M_ONE);
    static constexpr bool live = !(p_const && q_const);  // any draw needs a live stream
};

template <int PM, int QM, typename Word>
__device__ __forceinline__ void gen_xi(Xo& s, const ProbDev& p, const ProbDev& q, Word& xp, Word& xq) {
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
        Word ra = 0, rb = 0;
#pragma unroll 1
        for (int i0 = 0; i0 < W; i0 += 8) {
            uint32_t ba = 0, bb = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ba |= uint32_t(xo_next(a) < pd.T) << j;
                bb |= uint32_t(xo_next(b) < pd.T) << j;
            }
            ra |= Word(ba) << i0;
            rb |= Word(bb) << i0;
        }
        wa = ra;
        wb = rb;
    } else {  // M_ONE
#pragma unroll 8
        for (int i = 0; i < W; ++i) {
            xo_step(a);
            xo_step(b);
        }
        wa = wb = Word(~Word(0));
    }
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

// engine_vec.hpp:25-30
template <typename Word>
__device__ __forceinline__ Word update_mask(Word sxm, Word sym, Word sxp, Word syp, Word xp, Word xq) {
    const Word mp = xp & ~(sxm | sym) & sxp & syp;
    const Word mq = xq & ~(sxp | syp) & sxm & sym;
    return Word(mp ^ mq);
}

}  // namespace octgpu
