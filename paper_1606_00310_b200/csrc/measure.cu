// Device-side measurement: reconstruct_heights + height_moments
// (slope_field.hpp:159-229, measure.cpp:24-56) without materialising the
// HeightMap, in exact integer arithmetic.
//
// Heights: h(x,y) = H_y + r(x,y), H_y = sum sigma_y-(0,y') over the rows from the first
// scanned row to y (column 0) and r(x,y) = sum_{x'=1..x} sigma_x-(x',y) (row prefix). This
// equals the reference's row-0-then-columns integration whenever curl_check passes, which is
// checked in the same pass. With u(x) = sum_{x'<=x} sigma_x-(x',y) (inclusive from x = 0),
// h = G_y + u(x), G_y = H_y - sigma_x-(0,y), so S_k = sum_y sum_j C(k,j) G_y^(k-j) U_j(y)
// with U_j(y) = sum_x u(x)^j.
//
// Kernels (one measurement = 3 launches):
//   k_col_scan      one block: the column-0 prefix G_y = H_y - sigma_x-(0, y) of every core row (global
//                   gauge), the column closure sum and sigma_y-(0, c0).
//   k_measure_rows  persistent blocks of kSeg warps; a block takes a row group of 32 rows (lane per row)
//                   and warp s the group's x-segment s (plane-major coalesced loads). Word-parallel curl
//                   check; U_j per segment from 32-site units read through four chained 8-site tables (each
//                   indexed by the partial net step of the ones before, entries summed as packed 64-bit
//                   words), unit sums accumulated in 32-bit registers relative to a 4-word chunk and folded
//                   into the segment's sums once per chunk (16-site units: OCTGPU_MEAS_UNIT=16). Each thread then
//                   shifts its own segment's sums by the segment's global start height (G_y plus the net
//                   steps of the segments before it, exchanged through shared memory: one block barrier per
//                   group) and keeps the block's sums in registers; one block reduction at the end.
//   k_measure_final one block: sum of the blocks' partial sums, closure data.
// Scan order = virtual rows c0 .. c1-1 (periodic: physical rows 1 .. Y-1, 0; a stripe: its core
// rows); the gauge H is 0 at virtual row c0 - 1. For a periodic lattice that is the reference's
// h(0,0) = 0 whenever the column closes (otherwise the measurement fails with the reference's
// column error before the sums are used).
#include <algorithm>
#include <cstdint>
#include <type_traits>

#include "octgpu_internal.h"

namespace octgpu {

struct Partial {  // one row-pass block's sums
    __int128 S[4];                   // sum h^k over the block's sites (global gauge)
    unsigned long long curl_count;
    unsigned long long curl_first;   // row_id * X + x, ~0 if none
    long long row0;                  // sum_x sigma_x- of row_id 0 (its share of the row's segments)
    unsigned long long n_sites;
};

namespace {

constexpr int kRowsPerGroup = 32;  // lane per row; lane 0 reads the row above for the curl check
#ifndef OCTGPU_MEAS_SEG
#define OCTGPU_MEAS_SEG 16  // x-segments per row group: one warp each
#endif
constexpr int kSeg = OCTGPU_MEAS_SEG;
#ifndef OCTGPU_MEAS_MINB
#define OCTGPU_MEAS_MINB 1  // resident blocks per SM the register budget targets: 1 x 16 warps, 128 registers
#endif
constexpr int kMThreads = 32 * kSeg;

__host__ __device__ inline uint32_t measure_groups(uint32_t rows) { return (rows + kRowsPerGroup - 1) / kRowsPerGroup; }

__device__ __forceinline__ __int128 shfl_down_i128(__int128 v, int off) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)((unsigned __int128)v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, off);
    hi = __shfl_down_sync(0xffffffffu, hi, off);
    return (__int128)(((unsigned __int128)hi << 64) | lo);
}

// ---- 8-site tables ---------------------------------------------------------------
// A byte = 8 consecutive sites of a row: bits 0..3 the 4 even-x sites (one packed plane's nibble),
// bits 4..7 the 4 odd-x sites; sites interleave e0 o0 e1 o1 ... (slope_field.hpp:15-53). For an
// offset o (the height just before the byte, relative to the 16-site unit start; o is even) the entry
// holds q_k = sum_i (o + p_i)^k over the byte's inclusive prefix values p_i, k = 1..4, and d = p_8.
// T0 = offset 0 (first byte of a unit), T1[(o + 8) * 256 + b] = offsets -8..8 (second byte, indexed by
// the first byte's d + 8; odd rows unused). Since p_i = i (mod 2) and o is even, q1 is even, q2 = 0
// (mod 4) and q4 = 4 (mod 16), so an entry packs into 64 bits with room for the sum of two:
//   lo = q3 + B3 (16 bits) | q1 / 2 + B1 (8 bits) | d + 8 (8 bits)
//   hi = q2 / 4 (9 bits) | (q4 - 4) / 16 (23 bits)
// B3 = 1296 (T0) / 17200 (T1), B1 = 18 / 50. A unit (T0 + T1 entry) decodes as
//   q3 = Q3 - 18496, q1 = 2 (Q1 - 68), d = D - 16, q2 = 4 Q2, q4 = 16 Q4 + 8.
constexpr int kUnitB1 = 68, kUnitB3 = 18496;

struct MeasTab {
    uint2 t0[256];
    uint2 t1[17 * 256];
};

__host__ __device__ constexpr uint2 tab_entry(int b, int o, bool second) {
    int p = 0, q1 = 0, q2 = 0, q3 = 0, q4 = 0;
    for (int i = 0; i < 8; ++i) {
        const int bit = (i & 1) ? (b >> (4 + (i >> 1))) & 1 : (b >> (i >> 1)) & 1;
        p += bit ? 1 : -1;
        const int v = o + p;
        q1 += v;
        q2 += v * v;
        q3 += v * v * v;
        q4 += v * v * v * v;
    }
    const int b1 = second ? 50 : 18, b3 = second ? 17200 : 1296;
    const uint32_t lo = uint32_t(q3 + b3) | (uint32_t(q1 / 2 + b1) << 16) | (uint32_t(p + 8) << 24);
    const uint32_t hi = uint32_t(q2 / 4) | (uint32_t((q4 - 4) / 16) << 9);
    return uint2{lo, hi};
}

struct MeasTabInit : MeasTab {
    constexpr MeasTabInit() : MeasTab{} {
        for (int b = 0; b < 256; ++b) t0[b] = tab_entry(b, 0, false);
        for (int o = -8; o <= 8; o += 2)
            for (int b = 0; b < 256; ++b) t1[(o + 8) * 256 + b] = tab_entry(b, o, true);
    }
};

__device__ const MeasTab g_tab = MeasTabInit();

#ifndef OCTGPU_MEAS_UNIT
#define OCTGPU_MEAS_UNIT 32  // sites per unit: 32 (four chained 8-site tables) or 16 (two)
#endif
constexpr int kUnit = OCTGPU_MEAS_UNIT;
static_assert(kUnit == 16 || kUnit == 32, "OCTGPU_MEAS_UNIT must be 16 or 32");

// ---- 32-site units: four chained 8-site tables -----------------------------------------
// Byte j of a unit (j = 0..3) is read at offset o in -8j..8j (even): T0 (o = 0) and Tj (o = 2 (f - 4j),
// f = 0..8j the partial step field of the entries so far). An entry is one 64-bit word of five fields,
// each sized for the SUM of a unit's four entries (no carries between fields):
//   bits  0..16  F3 = (q3 - q1) / 6 + B3_j   (v^3 - v is divisible by 6)
//   bits 17..28  F2 = q2 / 4
//   bits 29..38  F1 = q1 / 2 + B1_j
//   bits 39..57  F4 = (q4 - 4) / 16
//   bits 58..63  FD = d / 2 + 4 = popcount(byte)   (the unit's partial sum indexes the next table)
// B1_j, B3_j = minus the field's minimum over Tj (the all-down byte at o = -8j), so a unit decodes as
//   q1 = 2 (F1 - B1), q2 = 4 F2, q3 = 6 (F3 - B3) + q1, q4 = 16 F4 + 16, d = 2 (FD - 16).
// Unit ranges: |q1| <= 528, q2 <= 11440, |q3 - q1| / 6 <= 46376, q4 <= 7246096, |d| <= 32.
constexpr int kTRows = 9 + 17 + 25;           // T1, T2, T3 (even offsets only)
__host__ __device__ constexpr int tab_base(int j) { return j <= 1 ? 0 : j == 2 ? 9 : 26; }  // Tj's first row
struct TabQ {
    long long q1, q2, q3, q4;
    int pc;
};
__host__ __device__ constexpr TabQ tab_q(int b, int o) {
    TabQ t{0, 0, 0, 0, 0};
    int p = 0;
    for (int i = 0; i < 8; ++i) {
        const int bit = (i & 1) ? (b >> (4 + (i >> 1))) & 1 : (b >> (i >> 1)) & 1;
        p += bit ? 1 : -1;
        t.pc += bit;
        const long long v = o + p, v2 = v * v;
        t.q1 += v;
        t.q2 += v2;
        t.q3 += v2 * v;
        t.q4 += v2 * v2;
    }
    return t;
}
__host__ __device__ constexpr long long tab_b1(int j) { return -tab_q(0, -8 * j).q1 / 2; }
__host__ __device__ constexpr long long tab_b3(int j) { return -(tab_q(0, -8 * j).q3 - tab_q(0, -8 * j).q1) / 6; }
constexpr long long kU32B1 = tab_b1(0) + tab_b1(1) + tab_b1(2) + tab_b1(3);
constexpr long long kU32B3 = tab_b3(0) + tab_b3(1) + tab_b3(2) + tab_b3(3);
static_assert(kU32B1 == 264 && kU32B3 == 46376, "unit biases");

__host__ __device__ constexpr unsigned long long tab32_entry(int b, int o, long long b1, long long b3) {
    const TabQ t = tab_q(b, o);
    return (unsigned long long)((t.q3 - t.q1) / 6 + b3) | ((unsigned long long)(t.q2 / 4) << 17) |
           ((unsigned long long)(t.q1 / 2 + b1) << 29) | ((unsigned long long)((t.q4 - 4) / 16) << 39) |
           ((unsigned long long)t.pc << 58);
}

struct MeasTab32 {
    unsigned long long t0[256];
    unsigned long long tj[kTRows * 256];
};
struct MeasTab32Init : MeasTab32 {
    constexpr MeasTab32Init() : MeasTab32{} {
        for (int b = 0; b < 256; ++b) t0[b] = tab32_entry(b, 0, tab_b1(0), tab_b3(0));
        for (int j = 1; j < 4; ++j) {
            const long long b1 = tab_b1(j), b3 = tab_b3(j);
            for (int f = 0; f <= 8 * j; ++f)
                for (int b = 0; b < 256; ++b) tj[(tab_base(j) + f) * 256 + b] = tab32_entry(b, 2 * (f - 4 * j), b1, b3);
        }
    }
};
__device__ const MeasTab32 g_tab32 = MeasTab32Init();

// shared memory: T0 replicated x16 (entry b at [b][lane & 15]: every warp lookup conflict-free), the
// chained tables once, then two buffers of the threads' segment net steps (groups alternate)
constexpr int kRep = 16;
// 32-site units: table j is replicated R_j times, entry b of copy c at [b][c] and lane l reads copy l % R_j.
// A 64-bit entry spans a bank pair and a warp's LDS.64 is served per half-warp: the wavefronts of one lookup
// are the sum over the two half-warps of the fullest pair. Entry b of copy c sits in pair (R_j b + c) mod 16,
// so a half-warp splits into R_j lane groups with disjoint pairs. Measured wavefronts per lookup (random
// bytes, ncu source page): R = 1: 6.9, 2: 6.4, 4: 5.5, 8: 4.0, 16: 2.0 (conflict-free). Default T0 x 16
// (32 KB), T1 x 4 (72 KB), T2, T3 once (34 + 50 KB): larger copies shrink the L1 the plane loads stream
// through and measured slower (tools/r2_u32rep.sh, tools/r2_u32load.sh).
#ifndef OCTGPU_MEAS_R0
#define OCTGPU_MEAS_R0 16
#endif
#ifndef OCTGPU_MEAS_R1
#define OCTGPU_MEAS_R1 4
#endif
#ifndef OCTGPU_MEAS_R2
#define OCTGPU_MEAS_R2 1
#endif
#ifndef OCTGPU_MEAS_R3
#define OCTGPU_MEAS_R3 1
#endif
__host__ __device__ constexpr int tab_rep(int j) {
    return j == 0 ? OCTGPU_MEAS_R0 : j == 1 ? OCTGPU_MEAS_R1 : j == 2 ? OCTGPU_MEAS_R2 : OCTGPU_MEAS_R3;
}
__host__ __device__ constexpr int tab_rows(int j) { return j == 0 ? 1 : 8 * j + 1; }
// first entry of table j's copies in shared memory
__host__ __device__ constexpr int tab_off(int j) {
    return j == 0 ? 0 : tab_off(j - 1) + 256 * tab_rows(j - 1) * tab_rep(j - 1);
}
constexpr int kT0Words = kUnit == 32 ? 0 : 256 * kRep;  // 8-byte entries
constexpr int kT1Words = kUnit == 32 ? tab_off(4) : 17 * 256;
// Up to this many sites per segment (R <= 2^13) the segment sums T1..T3 and the per-chunk increment of T4
// fit 64 bits (T3 <= 2^13 2^39; 4 R^3 C1 <= 2^59, R^4 ns <= 2^61 with C1 <= 2^18, ns = 512); T4 itself is
// summed in 128. Wider segments (X > 2^17) form everything in 128 bits.
constexpr uint32_t kNarrowSegSites = 8192;
constexpr size_t kMeasSmem = sizeof(uint2) * (kT0Words + kT1Words) + 2 * sizeof(long long) * kMThreads +
                             kSeg * sizeof(Partial);

}  // namespace

// device scratch of a measurement (engine.cu allocates measure_scratch_bytes and zeroes it once)
struct MeasScratch {
    long long* G;           // [Y] column-0 gauge G_y, relative to the row's 1024-row scan chunk
    long long* col;         // [2] the column's total (closure), sigma_y-(0, c0)
    unsigned int* ticket;   // k_col_scan: blocks done (the last one scans the chunk totals, resets it)
    long long* tot;         // [chunks] chunk totals, then (in place) their exclusive prefix
    Partial* part;          // [row-pass blocks]
};
constexpr uint32_t kColChunk = 1024;  // rows per k_col_scan block

__host__ __device__ inline MeasScratch scratch_layout(void* base, uint32_t Y) {
    MeasScratch m;
    m.G = static_cast<long long*>(base);
    m.col = m.G + Y;
    m.ticket = reinterpret_cast<unsigned int*>(m.col + 2);
    m.tot = m.col + 3;
    const size_t chunks = Y / kColChunk + 2;
    m.part = reinterpret_cast<Partial*>(m.tot + ((chunks + 1) & ~size_t(1)) + ((Y + 3) & 1));  // 16-B aligned
    return m;
}

size_t measure_scratch_bytes(uint32_t Y) {
    const MeasScratch m = scratch_layout(nullptr, Y);
    return size_t(reinterpret_cast<char*>(m.part) - static_cast<char*>(nullptr)) +
           size_t(measure_groups(Y + 1) + 1) * sizeof(Partial) + 64;
}

namespace {

// signed 32 x 32 -> 64-bit multiply-add in one IMAD.WIDE
__device__ __forceinline__ long long madw(int a, int b, long long c) {
    long long d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

// Unit accumulators of a chunk: r = height at the unit start relative to the chunk start (|r| <= 512),
// Q* the biased unit fields (tab_entry); every sum stays in 32 bits over a 32-unit chunk except the three
// held in 64 (sum r^3, sum r^4, sum r^3 Q1).
struct UnitAcc {
    int ar, ar2, aq1, aq2, aq3, aq4, x11, x12, x13, x21;
    unsigned int x22;
    long long ar3, ar4, x31;
    __device__ __forceinline__ void clear() {
        ar = ar2 = aq1 = aq2 = aq3 = aq4 = x11 = x12 = x13 = x21 = 0;
        x22 = 0;
        ar3 = ar4 = x31 = 0;
    }
};

// one 16-site unit: byte un of evn (first 8 sites), byte un of odd (next 8)
__device__ __forceinline__ void unit(UnitAcc& A, int& r, uint32_t evn, uint32_t odd, uint32_t un, const uint2* t0l,
                                     const uint2* t1) {
    const uint2 e0 = t0l[__byte_perm(evn, 0, 0x4440 + un) * kRep];
    const uint2 e1 = t1[__byte_perm(odd, e0.x >> 24, 0x5540 + un)];  // (d0 + 8) * 256 + byte
    const uint32_t lo = e0.x + e1.x, hi = e0.y + e1.y;
    const int q3 = int(lo & 0xffffu), q1 = int(__byte_perm(lo, 0, 0x4442)), q2 = int(hi & 0x1ffu), q4 = int(hi >> 9);
    const int r2 = r * r, r3 = r2 * r;
    A.ar += r;
    A.ar2 += r2;
    A.ar3 = madw(r2, r, A.ar3);
    A.ar4 = madw(r2, r2, A.ar4);
    A.aq1 += q1;
    A.aq2 += q2;
    A.aq3 += q3;
    A.aq4 += q4;
    A.x11 += r * q1;
    A.x12 += r * q2;
    A.x13 += r * q3;
    A.x21 += r2 * q1;
    A.x22 += uint32_t(r2) * uint32_t(q2);
    A.x31 = madw(r3, q1, A.x31);
    r += int(lo >> 24) - 16;
}

// Fold a chunk of K units (net step r, ns sites) into the segment sums T (relative to the segment start;
// R = the chunk's start height there). The chunk's own sums C_k = sum (16 r^k + ... ) decode the biased
// unit fields; then T_k += sum_j C(k, j) R^(k-j) C_j (C_0 = ns).
template <typename TT>
__device__ __forceinline__ void flush_chunk(UnitAcc& A, int K, int ns, long long R, TT& T1, TT& T2, TT& T3,
                                            __int128& T4) {
    const long long k = K;
    const long long C1 = 16ll * A.ar + 2ll * A.aq1 - 2ll * kUnitB1 * k;
    const long long C2 = 16ll * A.ar2 + 4ll * A.x11 - 4ll * kUnitB1 * A.ar + 4ll * A.aq2;
    const long long C3 = 16ll * A.ar3 + 6ll * A.x21 - 6ll * kUnitB1 * A.ar2 + 12ll * A.x12 + A.aq3 - kUnitB3 * k;
    const long long C4 = 16ll * A.ar4 + 8ll * A.x31 - 8ll * kUnitB1 * A.ar3 + 24ll * (long long)A.x22 +
                         4ll * A.x13 - 4ll * kUnitB3 * A.ar + 16ll * A.aq4 + 8ll * k;
    const TT r1 = R, r2 = r1 * r1, r3 = r2 * r1;
    T1 += C1 + r1 * ns;
    T2 += C2 + 2 * r1 * C1 + r2 * ns;
    T3 += C3 + 3 * r1 * C2 + 3 * r2 * C1 + r3 * ns;
    T4 += C4 + 4 * r1 * C3 + 6 * r2 * C2 + 4 * r3 * C1 + r2 * r2 * ns;  // 64-bit increment when narrow
    A.clear();
}

// Unit accumulators of a chunk of 32-site units: s = r / 2, r = the height at the unit start relative to
// the chunk start (|s| <= 240 over 16 units); F* the biased unit fields. 32-bit sums except s^4 and s^3 F1.
struct UnitAcc32 {
    int as, as2, as3, f1, f2, f3, f4, sf1, sf2, sf3, s2f1, s2f2;
    long long as4, s3f1;
    __device__ __forceinline__ void clear() {
        as = as2 = as3 = f1 = f2 = f3 = f4 = sf1 = sf2 = sf3 = s2f1 = s2f2 = 0;
        as4 = s3f1 = 0;
    }
};

// a lane's copies of the four tables (tab_off / tab_rep)
struct TabLanes {
    const unsigned long long *t0, *t1, *t2, *t3;
};

// one 32-site unit v of a 64-site half: bytes 2v (evn), 2v (odd), 2v + 1 (evn), 2v + 1 (odd)
__device__ __forceinline__ void unit32(UnitAcc32& A, int& s, uint32_t evn, uint32_t odd, uint32_t v,
                                       const TabLanes& T) {
    const uint32_t k0 = 2 * v, k1 = 2 * v + 1;
    unsigned long long e = T.t0[__byte_perm(evn, 0, 0x4440 + k0) * tab_rep(0)];
    e += T.t1[__byte_perm(odd, uint32_t(e >> 58), 0x5540 + k0) * tab_rep(1)];
    e += T.t2[__byte_perm(evn, uint32_t(e >> 58), 0x5540 + k1) * tab_rep(2)];
    e += T.t3[__byte_perm(odd, uint32_t(e >> 58), 0x5540 + k1) * tab_rep(3)];
    const uint32_t lo = uint32_t(e), hi = uint32_t(e >> 32);
    const int F3 = int(lo & 0x1ffffu), F2 = int((lo >> 17) & 0xfffu), F1 = int(__funnelshift_r(lo, hi, 29) & 0x3ffu),
              F4 = int((hi >> 7) & 0x7ffffu), FD = int(hi >> 26);
    const int s2 = s * s, s3 = s2 * s;
    A.as += s;
    A.as2 += s2;
    A.as3 += s3;
    A.as4 = madw(s2, s2, A.as4);
    A.f1 += F1;
    A.f2 += F2;
    A.f3 += F3;
    A.f4 += F4;
    A.sf1 += s * F1;
    A.sf2 += s * F2;
    A.sf3 += s * F3;
    A.s2f1 += s2 * F1;
    A.s2f2 += s2 * F2;
    A.s3f1 = madw(s3, F1, A.s3f1);
    s += FD - 16;
}

// Fold a chunk of K 32-site units (ns sites) into the segment sums; with r = 2 s and the unit decode above,
// C_k = sum over units of sum_j C(k, j) r^(k-j) q_j (q_0 = 32), then T_k += sum_j C(k, j) R^(k-j) C_j.
template <typename TT>
__device__ __forceinline__ void flush_chunk32(UnitAcc32& A, int K, int ns, long long R, TT& T1, TT& T2, TT& T3,
                                              __int128& T4) {
    const long long k = K, B1 = kU32B1, B3 = kU32B3;
    const long long as = A.as, as2 = A.as2, as3 = A.as3, f1 = A.f1;
    const long long C1 = 64 * as + 2 * f1 - 2 * B1 * k;
    const long long C2 = 128 * as2 + 8ll * A.sf1 - 8 * B1 * as + 4ll * A.f2;
    const long long C3 = 256 * as3 + 24ll * A.s2f1 - 24 * B1 * as2 + 24ll * A.sf2 + 6ll * A.f3 - 6 * B3 * k + 2 * f1 -
                         2 * B1 * k;
    const long long C4 = 512 * A.as4 + 64 * A.s3f1 - 64 * B1 * as3 + 96ll * A.s2f2 + 48ll * A.sf3 - 48 * B3 * as +
                         16ll * A.sf1 - 16 * B1 * as + 16ll * A.f4 + 16 * k;
    const TT r1 = R, r2 = r1 * r1, r3 = r2 * r1;
    T1 += C1 + r1 * ns;
    T2 += C2 + 2 * r1 * C1 + r2 * ns;
    T3 += C3 + 3 * r1 * C2 + 3 * r2 * C1 + r3 * ns;
    T4 += C4 + 4 * r1 * C3 + 6 * r2 * C2 + 4 * r3 * C1 + r2 * r2 * ns;
    A.clear();
}

// base[o] through one 32 x 32 -> 64-bit address multiply-add (keeps the per-word address arithmetic at one
// instruction per plane)
template <typename Word>
__device__ __forceinline__ Word ldg_word(const Word* base, uint32_t o) {
    if constexpr (sizeof(Word) == 8) {
        unsigned long long v;
        asm("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %2, 8, %1;\n\tld.global.nc.u64 %0, [a];\n\t}"
            : "=l"(v) : "l"(base), "r"(o));
        return Word(v);
    } else {
        unsigned int v;
        asm("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %2, 4, %1;\n\tld.global.nc.u32 %0, [a];\n\t}"
            : "=r"(v) : "l"(base), "r"(o));
        return Word(v);
    }
}

template <typename Word>
struct Curl {  // word-parallel curl check of one word
    static constexpr int W = int(sizeof(Word) * 8);
    // parity ya (even-x sites, D rotated up one packed bit with the previous word's top bit) and parity !ya
    // (odd-x sites, D aligned); bxa / bxb: the row above's X words
    __device__ __forceinline__ static void eval(Word xa, Word xb, Word ca, Word cb, Word bxa, Word bxb, Word pcb,
                                                Word& V1, Word& V2) {
        const Word D1 = Word((cb << 1) | (pcb >> (W - 1)));
        V1 = (xa ^ bxa ^ ca ^ D1) | ((xa ^ bxa) & (xa ^ ca));
        V2 = (xb ^ bxb ^ cb ^ ca) | ((xb ^ bxb) & (xb ^ cb));
    }
};

}  // namespace

// ---- row pass -------------------------------------------------------------------------
// Persistent blocks of kSeg warps walk the row groups (32 rows each, lane per row): warp s handles
// x-segment s (words [s n / kSeg, (s+1) n / kSeg)) of the group's rows and shifts its sums to the global
// gauge (Gg: k_col_scan); part[blockIdx.x] = the block's sums.
template <typename Word, bool WIDE>
__global__ void __launch_bounds__(kMThreads, OCTGPU_MEAS_MINB) k_measure_rows(const Word* __restrict__ planes, Geom g, uint32_t X,
                                                               const long long* __restrict__ Gg,
                                                               const long long* __restrict__ pre,
                                                               Partial* __restrict__ part) {
    constexpr int W = int(sizeof(Word) * 8);
    constexpr int kChunkWords = 256 / W;  // 512 sites per chunk
    constexpr bool kU32 = kUnit == 32 && W > 0;  // (dependent: the other unit's branch is discarded)
    extern __shared__ __align__(16) unsigned char msm[];
    uint2* t0rep = reinterpret_cast<uint2*>(msm);
    uint2* t1 = t0rep + kT0Words;
    long long* Dbuf = reinterpret_cast<long long*>(t1 + kT1Words);
    if constexpr (kU32) {  // the replicated copies of T0..T3
        unsigned long long* tq = reinterpret_cast<unsigned long long*>(msm);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const unsigned long long* src = j == 0 ? g_tab32.t0 : g_tab32.tj + tab_base(j) * 256;
            const int n = 256 * tab_rows(j) * tab_rep(j);
            for (int i = threadIdx.x; i < n; i += kMThreads) tq[tab_off(j) + i] = src[i / tab_rep(j)];
        }
    } else {
        for (int i = threadIdx.x; i < kT0Words; i += kMThreads) t0rep[i] = g_tab.t0[i / kRep];
        const uint4* src1 = reinterpret_cast<const uint4*>(g_tab.t1);
        uint4* dst1 = reinterpret_cast<uint4*>(t1);
        for (int i = threadIdx.x; i < kT1Words / 2; i += kMThreads) dst1[i] = src1[i];
    }
    __syncthreads();

    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const uint32_t n = g.n, Y = g.Y;
    const size_t PS = g.plane_stride;
    const uint32_t kbeg = uint32_t(seg) * n / kSeg, kend = uint32_t(seg + 1) * n / kSeg;
    const uint32_t ngroups = measure_groups(g.c1 - g.c0);
    const uint2* t0l = t0rep + (lane % kRep);
    TabLanes TL{};
    if constexpr (kU32) {
        const unsigned long long* tq = reinterpret_cast<const unsigned long long*>(msm);
        TL = TabLanes{tq + tab_off(0) + lane % tab_rep(0), tq + tab_off(1) + lane % tab_rep(1),
                      tq + tab_off(2) + lane % tab_rep(2), tq + tab_off(3) + lane % tab_rep(3)};
    }

    // the block's sums, one slot per warp (each warp adds its group shares; no contention)
    Partial* wsum = reinterpret_cast<Partial*>(Dbuf + 2 * kMThreads);
    if (lane == 0) {
        Partial z{};
        z.curl_first = ~0ull;
        wsum[seg] = z;
    }
    uint32_t gen = 0;
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t first = g.c0 + grp * uint32_t(kRowsPerGroup);  // the group's first row
        const uint32_t v = first + uint32_t(lane);
        const uint32_t y = g.wrap ? v % g.wrap : v;
        const bool core = v < g.c1;
        const uint32_t row_id = g.wrap ? y : v - g.c0;
        const int ya = int((y ^ g.ypar) & 1u);
        // even-x sites of row y are in X(ya), odd-x in X(!ya); C = Y(ya), its partner Y(!ya)
        const Word* pXa = planes + size_t(ya) * PS + y;
        const Word* pXb = planes + size_t(ya ^ 1) * PS + y;
        const Word* pCa = planes + size_t(2 + ya) * PS + y;
        const Word* pCb = planes + size_t(3 - ya) * PS + y;
        // lane 0: the row above (its X words, which the other lanes take from lane - 1); parity !ya
        const uint32_t yu = g.wrap ? (v - 1) % g.wrap : v - 1;
        const Word* pUa = planes + size_t(ya ^ 1) * PS + yu;
        const Word* pUb = planes + size_t(ya) * PS + yu;

        using TT = typename std::conditional<WIDE, __int128, long long>::type;
        TT T1 = 0, T2 = 0, T3 = 0;
        __int128 T4 = 0;
        long long R = 0;
        Word bad = 0;
        if (kend > kbeg) {
            typename std::conditional<kU32, UnitAcc32, UnitAcc>::type A;
            A.clear();
            int r = 0;
            Word pcb = pCb[size_t(kbeg == 0 ? n - 1 : kbeg - 1) * Y];
            uint32_t o = kbeg * Y;  // word offset within a plane (n Y < 2^32: launch_measure)
            // plane-major loads (a warp's 32 rows of one plane: one contiguous 256-B segment), the parity
            // selects at use: lane l reads X(ya) / X(!ya) / Y(ya) / Y(!ya) of its row from planes 0..3
            const Word* P0 = planes + y;
            const Word* P1 = planes + PS + y;
            const Word* P2 = planes + 2 * PS + y;
            const Word* P3 = planes + 3 * PS + y;
            const Word* U0 = planes + yu;
            const Word* U1 = planes + PS + yu;
            Word nw0 = ldg_word(P0, o), nw1 = ldg_word(P1, o), nw2 = ldg_word(P2, o), nw3 = ldg_word(P3, o), nu0 = 0,
                 nu1 = 0;
            if (lane == 0) {
                nu0 = ldg_word(U0, o);
                nu1 = ldg_word(U1, o);
            }
            for (uint32_t kc = kbeg; kc < kend; kc += kChunkWords) {
                const uint32_t kce = min(kend, kc + kChunkWords);
#pragma unroll
                for (uint32_t i = 0; i < uint32_t(kChunkWords); ++i) {  // unrolled: the prefetch rotates by renaming
                    const uint32_t k = kc + i;
                    if (k >= kce) break;
                    const Word xa = ya ? nw1 : nw0, xb = ya ? nw0 : nw1, ca = ya ? nw3 : nw2, cb = ya ? nw2 : nw3;
                    const Word ua = ya ? nu0 : nu1, ub = ya ? nu1 : nu0;
                    // prefetch the next word (the segment's last word re-reads itself: no branch, no copies)
                    o += k + 1 < kend ? Y : 0u;
                    nw0 = ldg_word(P0, o);
                    nw1 = ldg_word(P1, o);
                    nw2 = ldg_word(P2, o);
                    nw3 = ldg_word(P3, o);
                    if (lane == 0) {
                        nu0 = ldg_word(U0, o);
                        nu1 = ldg_word(U1, o);
                    }
                    Word bxa = __shfl_up_sync(0xffffffffu, xa, 1);
                    Word bxb = __shfl_up_sync(0xffffffffu, xb, 1);
                    if (lane == 0) {
                        bxa = ua;
                        bxb = ub;
                    }
                    Word V1, V2;
                    Curl<Word>::eval(xa, xb, ca, cb, bxa, bxb, pcb, V1, V2);
                    bad |= V1 | V2;
                    pcb = cb;
#pragma unroll
                    for (int half = 0; half < W / 32; ++half) {
                        const uint32_t a32 = uint32_t(uint64_t(xa) >> (32 * half));
                        const uint32_t b32 = uint32_t(uint64_t(xb) >> (32 * half));
                        const uint32_t evn = (a32 & 0x0F0F0F0Fu) | ((b32 & 0x0F0F0F0Fu) << 4);  // chunks 0,2,4,6
                        const uint32_t odd = ((a32 >> 4) & 0x0F0F0F0Fu) | (b32 & 0xF0F0F0F0u);  // chunks 1,3,5,7
                        if constexpr (kU32) {
                            unit32(A, r, evn, odd, 0, TL);
                            unit32(A, r, evn, odd, 1, TL);
                        } else {
#pragma unroll
                            for (uint32_t un = 0; un < 4; ++un) unit(A, r, evn, odd, un, t0l, t1);
                        }
                    }
                }
                const int words = int(kce - kc);
                if constexpr (kU32) {
                    flush_chunk32(A, words * (W / 16), words * 2 * W, R, T1, T2, T3, T4);
                    R += 2 * r;  // r holds s = (height step) / 2
                } else {
                    flush_chunk(A, words * (W / 8), words * 2 * W, R, T1, T2, T3, T4);
                    R += r;
                }
                r = 0;
            }
        }
        unsigned int rc = 0, rfirst = 0xffffffffu;
        if (!core) bad = 0;
        if (__any_sync(0xffffffffu, bad != 0)) {
            // rare: exact curl count and first plaquette of the segment (the reference's error message)
            Word pcb = kend > kbeg ? pCb[size_t(kbeg == 0 ? n - 1 : kbeg - 1) * Y] : 0;
            for (uint32_t k = kbeg; k < kend; ++k) {
                const size_t o = size_t(k) * Y;
                const Word xa = pXa[o], xb = pXb[o], ca = pCa[o], cb = pCb[o];
                Word bxa = __shfl_up_sync(0xffffffffu, xa, 1);
                Word bxb = __shfl_up_sync(0xffffffffu, xb, 1);
                if (lane == 0) {
                    bxa = pUa[o];
                    bxb = pUb[o];
                }
                Word V1, V2;
                Curl<Word>::eval(xa, xb, ca, cb, bxa, bxb, pcb, V1, V2);
                pcb = cb;
                if (core && (V1 | V2)) {
                    rc += __popcll((unsigned long long)V1) + __popcll((unsigned long long)V2);
                    if (V1)
                        rfirst = min(rfirst, 2u * (k * W + uint32_t(__ffsll((long long)(unsigned long long)V1) - 1)));
                    if (V2)
                        rfirst = min(rfirst,
                                     2u * (k * W + uint32_t(__ffsll((long long)(unsigned long long)V2) - 1)) + 1u);
                }
            }
        }
        // this segment's start height: G_y + the net steps of the row's segments before it
        long long* Dg = Dbuf + size_t(gen & 1u) * kMThreads;
        Dg[threadIdx.x] = R;
        __syncthreads();  // (the double-buffered D slots need no second barrier per group)
        {
            __int128 S[4] = {0, 0, 0, 0};
            unsigned long long ccount = 0, cfirst = ~0ull;
            long long row0 = 0;
            if (core) {
                long long off = Gg[y] + pre[(v - g.c0) / kColChunk];  // global gauge
                for (int s2 = 0; s2 < seg; ++s2) off += Dg[s2 * 32 + lane];
                // S_k = sum_j C(k, j) off^(k-j) T_j, T_0 = the segment's sites
                const __int128 c = off, c2 = c * c, c3 = c2 * c, c4 = c2 * c2;
                const __int128 ns = (__int128)(kend - kbeg) * 2 * W, t1 = T1, t2 = T2, t3 = T3;
                S[0] = c * ns + t1;
                S[1] = c2 * ns + 2 * c * t1 + t2;
                S[2] = c3 * ns + 3 * c2 * t1 + 3 * c * t2 + t3;
                S[3] = c4 * ns + 4 * c3 * t1 + 6 * c2 * t2 + 4 * c * t3 + T4;
                ccount = rc;
                if (rfirst != 0xffffffffu) cfirst = (unsigned long long)row_id * X + rfirst;
                if (row_id == 0) row0 = R;  // sum_x sigma_x- of row 0 (over its segments)
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                for (int o = 16; o > 0; o >>= 1) S[k] += shfl_down_i128(S[k], o);
            const bool any_curl = __any_sync(0xffffffffu, ccount != 0), any_r0 = __any_sync(0xffffffffu, row0 != 0);
            if (any_curl || any_r0)
                for (int o = 16; o > 0; o >>= 1) {
                    ccount += __shfl_down_sync(0xffffffffu, ccount, o);
                    const unsigned long long f = __shfl_down_sync(0xffffffffu, cfirst, o);
                    cfirst = f < cfirst ? f : cfirst;
                    row0 += __shfl_down_sync(0xffffffffu, row0, o);
                }
            if (lane == 0) {
                Partial& pw = wsum[seg];
                for (int k = 0; k < 4; ++k) pw.S[k] += S[k];
                pw.curl_count += ccount;
                pw.curl_first = cfirst < pw.curl_first ? cfirst : pw.curl_first;
                pw.row0 += row0;
                pw.n_sites += (unsigned long long)min(uint32_t(kRowsPerGroup), g.c1 - first) * (kend - kbeg) * 2 * W;
            }
        }
        ++gen;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial pr{};
        pr.curl_first = ~0ull;
        for (int w2 = 0; w2 < kSeg; ++w2) {
            const Partial& pw = wsum[w2];
            for (int k = 0; k < 4; ++k) pr.S[k] += pw.S[k];
            pr.curl_count += pw.curl_count;
            pr.curl_first = pw.curl_first < pr.curl_first ? pw.curl_first : pr.curl_first;
            pr.row0 += pw.row0;
            pr.n_sites += pw.n_sites;
        }
        part[blockIdx.x] = pr;
    }
}

// Column 0: G_y = H_y - sigma_x-(0, y) for the virtual rows c0 .. c1-1, H_y the inclusive prefix of
// sigma_y-(0, y') from c0. Block b scans rows [1024 b, 1024 b + 1024) (coalesced: one row per thread) and
// stores G relative to its chunk; the last block to finish turns the chunk totals into their exclusive
// prefix (the global gauge is G_y + tot[i / 1024]) and writes the column's total and sigma_y-(0, c0).
template <typename Word>
__global__ void __launch_bounds__(1024) k_col_scan(const Word* __restrict__ planes, Geom g, MeasScratch m) {
    __shared__ long long wt[32];
    __shared__ bool last;
    const uint32_t R = g.c1 - g.c0, t = threadIdx.x, lane = t & 31, wp = t >> 5;
    const uint32_t i = blockIdx.x * kColChunk + t;
    const size_t PS = g.plane_stride;
    int sy = 0, sx = 0;
    uint32_t y = 0;
    if (i < R) {
        const uint32_t v = g.c0 + i;
        y = g.wrap ? v % g.wrap : v;
        const int ya = int((y ^ g.ypar) & 1u);
        sy = (planes[size_t(2 + ya) * PS + y] & 1) ? 1 : -1;
        sx = (planes[size_t(ya) * PS + y] & 1) ? 1 : -1;
    }
    long long incl = sy;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= uint32_t(o)) incl += u;
    }
    if (lane == 31) wt[wp] = incl;
    __syncthreads();
    if (wp == 0) {
        long long u = wt[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long z = __shfl_up_sync(0xffffffffu, u, o);
            if (lane >= uint32_t(o)) u += z;
        }
        wt[lane] = u;
    }
    __syncthreads();
    incl += wp > 0 ? wt[wp - 1] : 0;
    if (i < R) m.G[y] = incl - sx;
    if (i == 0) m.col[1] = sy;
    if (t == 0) {
        m.tot[blockIdx.x] = wt[31];
        __threadfence();
        last = atomicAdd(m.ticket, 1u) + 1u == gridDim.x;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // exclusive prefix of the chunk totals (gridDim.x <= 2^16 / ... chunks; a sequential pass per 1024)
    long long carry = 0;
    for (uint32_t b0 = 0; b0 < gridDim.x; b0 += 1024) {
        const uint32_t b = b0 + t;
        const long long v = b < gridDim.x ? ((volatile long long*)m.tot)[b] : 0;
        long long c = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long z = __shfl_up_sync(0xffffffffu, c, o);
            if (lane >= uint32_t(o)) c += z;
        }
        if (lane == 31) wt[wp] = c;
        __syncthreads();
        if (wp == 0) {
            long long u = wt[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long z = __shfl_up_sync(0xffffffffu, u, o);
                if (lane >= uint32_t(o)) u += z;
            }
            wt[lane] = u;
        }
        __syncthreads();
        c += (wp > 0 ? wt[wp - 1] : 0) + carry;
        if (b < gridDim.x) m.tot[b] = c - v;
        carry += wt[31];
        __syncthreads();
    }
    if (t == 0) {
        m.col[0] = carry;
        *m.ticket = 0;
    }
}

__global__ void __launch_bounds__(1024) k_measure_final(const Partial* __restrict__ part, uint32_t nb,
                                                        const long long* __restrict__ col,
                                                        MeasureResult* __restrict__ res) {
    __shared__ __int128 sh_s[4][32];
    __shared__ unsigned long long sh_cc[32], sh_cf[32];
    __shared__ long long sh_r0[32];
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    __int128 S[4] = {0, 0, 0, 0};
    unsigned long long cc = 0, cf = ~0ull;
    long long r0 = 0;
    for (uint32_t i = t; i < nb; i += 1024) {
        const Partial& p = part[i];
        for (int k = 0; k < 4; ++k) S[k] += p.S[k];
        cc += p.curl_count;
        cf = p.curl_first < cf ? p.curl_first : cf;
        r0 += p.row0;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        __int128 vs = S[k];
        for (int off = 16; off > 0; off >>= 1) vs += shfl_down_i128(vs, off);
        if (lane == 0) sh_s[k][wp] = vs;
    }
    for (int off = 16; off > 0; off >>= 1) {
        cc += __shfl_down_sync(0xffffffffu, cc, off);
        const unsigned long long o = __shfl_down_sync(0xffffffffu, cf, off);
        cf = o < cf ? o : cf;
        r0 += __shfl_down_sync(0xffffffffu, r0, off);
    }
    if (lane == 0) {
        sh_cc[wp] = cc;
        sh_cf[wp] = cf;
        sh_r0[wp] = r0;
    }
    __syncthreads();
    if (t == 0) {
        __int128 tot[4] = {0, 0, 0, 0};
        unsigned long long tc = 0, tf = ~0ull;
        long long tr = 0;
        for (int i = 0; i < 32; ++i) {
            for (int k = 0; k < 4; ++k) tot[k] += sh_s[k][i];
            tc += sh_cc[i];
            tf = sh_cf[i] < tf ? sh_cf[i] : tf;
            tr += sh_r0[i];
        }
        for (int k = 0; k < 4; ++k) {
            res->s_lo[k] = (uint64_t)tot[k];
            res->s_hi[k] = (int64_t)(tot[k] >> 64);
        }
        res->curl_count = tc;
        res->curl_first = tf;
        res->row0_sum = tr;
        res->col0_sum = col[0];
        res->sy_first = col[1];
        res->pad = 0;
    }
}

// Heights (reference HeightMap layout): one warp per row, lane l owns words
// l, l+32, ...; h(x,y) = G_y + u(x) (G_y: k_col_scan of the last measurement).
template <typename Word>
__global__ void k_heights(const Word* __restrict__ planes, Geom g, uint32_t X, const long long* __restrict__ G,
                          const long long* __restrict__ pre, int32_t* __restrict__ out) {
    constexpr int W = int(sizeof(Word) * 8);
    const uint32_t Y = g.wrap, LD = g.Y, n = g.n;  // periodic only
    const uint32_t y = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (y >= Y) return;
    const size_t PS = g.plane_stride;
    const int ya = int(y & 1u);
    const Word* Xa = planes + size_t(ya) * PS + y;
    const Word* Xb = planes + size_t(ya ^ 1) * PS + y;
    const uint32_t vrow = y < g.c0 ? y + g.wrap : y;  // scan position of physical row y
    long long carry = G[y] + pre[(vrow - g.c0) / kColChunk];  // global gauge (k_col_scan)
    int32_t* row = out + size_t(y) * X;
    for (uint32_t kb = 0; kb < n; kb += 32) {
        const uint32_t k = kb + lane;
        Word a = 0, b = 0;
        int delta = 0;
        if (k < n) {
            a = Xa[size_t(k) * LD];
            b = Xb[size_t(k) * LD];
            delta = 2 * (__popcll((unsigned long long)a) + __popcll((unsigned long long)b)) - 2 * W;
        }
        int incl = delta;
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        long long h = carry + (incl - delta);
        if (k < n) {
            int32_t* dst = row + size_t(k) * 2 * W;
            for (int bb = 0; bb < W; ++bb) {
                h += ((a >> bb) & 1) ? 1 : -1;
                dst[2 * bb] = int32_t(h);
                h += ((b >> bb) & 1) ? 1 : -1;
                dst[2 * bb + 1] = int32_t(h);
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

// ---- row / column balances (slope_field.hpp:177-202) ----------------------------
// Rows r0 .. r0+R-1 (physical); the site parity of physical row r is (r ^ ypar) & 1.
// row_balances: out[y] = 2 * popcount(sigma_x- bits of row r0+y) - X, lane per row.
template <typename Word>
__global__ void k_row_balances(const Word* __restrict__ planes, Geom g, uint32_t r0, uint32_t R, uint32_t X,
                               long long* __restrict__ out) {
    const uint32_t y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= R) return;
    const size_t PS = g.plane_stride;
    const Word* a = planes + r0 + y;
    const Word* b = planes + PS + r0 + y;
    long long pop = 0;
    for (uint32_t k = 0; k < g.n; ++k)
        pop += __popcll((unsigned long long)a[size_t(k) * g.Y]) + __popcll((unsigned long long)b[size_t(k) * g.Y]);
    out[y] = 2 * pop - (long long)X;
}

// col_balances: out[x] += sum over rows of sigma_y-(x, y) (out zeroed by the caller). Warp per (word k,
// chunk of rows); lane = row. Column x = 2 (W k + b) + e takes its bit from plane Y((e ^ parity(row)) & 1),
// so each lane's two y-plane words are the even-x (wa) and odd-x (wb) columns of its row; the per-bit
// counts over the warp's rows come from ballots.
template <typename Word>
__global__ void k_col_balances(const Word* __restrict__ planes, Geom g, uint32_t r0, uint32_t R, uint32_t chunk,
                               unsigned long long* __restrict__ cnt) {
    constexpr int W = int(sizeof(Word) * 8);
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t chunks = (R + chunk - 1) / chunk;
    const uint32_t k = warp / chunks, c = warp % chunks;
    if (k >= g.n) return;
    const size_t PS = g.plane_stride;
    const uint32_t ya = c * chunk, yb = min(R, ya + chunk);
    unsigned int ce[W / 32] = {}, co[W / 32] = {};  // lane holds bits lane, lane + 32 (w = 64)
    for (uint32_t y0 = ya; y0 < yb; y0 += 32) {
        const uint32_t y = y0 + lane;
        Word wa = 0, wb = 0;
        if (y < yb) {
            const uint32_t r = r0 + y;
            const int par = int((r ^ g.ypar) & 1u);
            const Word v0 = planes[2 * PS + size_t(k) * g.Y + r], v1 = planes[3 * PS + size_t(k) * g.Y + r];
            wa = par ? v1 : v0;  // even x: plane parity = row parity
            wb = par ? v0 : v1;
        }
#pragma unroll
        for (int b = 0; b < W; ++b) {
            const unsigned int ma = __ballot_sync(0xffffffffu, (wa >> b) & 1);
            const unsigned int mb = __ballot_sync(0xffffffffu, (wb >> b) & 1);
            if (lane == (b & 31)) {
                ce[b >> 5] += __popc(ma);
                co[b >> 5] += __popc(mb);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < W / 32; ++h) {
        const uint32_t j = uint32_t(W) * k + 32u * h + lane;  // packed index: columns 2j, 2j + 1
        atomicAdd(cnt + 2 * size_t(j), (unsigned long long)ce[h]);
        atomicAdd(cnt + 2 * size_t(j) + 1, (unsigned long long)co[h]);
    }
}

__global__ void k_counts_to_balance(const unsigned long long* __restrict__ cnt, uint32_t X, uint32_t R,
                                    long long* __restrict__ out) {
    const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x < X) out[x] = 2 * (long long)cnt[x] - (long long)R;
}

cudaError_t launch_balances(int w, const void* planes, Geom g, uint32_t r0, uint32_t R, uint32_t X,
                            long long* rows_out, long long* cols_out, void* tmp, cudaStream_t st) {
    if (rows_out) {
        const uint32_t nb = (R + 255) / 256;
        if (w == 64)
            k_row_balances<uint64_t><<<nb, 256, 0, st>>>(static_cast<const uint64_t*>(planes), g, r0, R, X, rows_out);
        else
            k_row_balances<uint32_t><<<nb, 256, 0, st>>>(static_cast<const uint32_t*>(planes), g, r0, R, X, rows_out);
    }
    if (cols_out) {
        unsigned long long* cnt = static_cast<unsigned long long*>(tmp);
        cudaError_t e = cudaMemsetAsync(cnt, 0, size_t(X) * sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        const uint32_t chunk = 1024, chunks = (R + chunk - 1) / chunk;
        const uint32_t warps = g.n * chunks, nb = (warps * 32 + 255) / 256;
        if (w == 64)
            k_col_balances<uint64_t><<<nb, 256, 0, st>>>(static_cast<const uint64_t*>(planes), g, r0, R, chunk, cnt);
        else
            k_col_balances<uint32_t><<<nb, 256, 0, st>>>(static_cast<const uint32_t*>(planes), g, r0, R, chunk, cnt);
        k_counts_to_balance<<<(X + 255) / 256, 256, 0, st>>>(cnt, X, R, cols_out);
    }
    return cudaGetLastError();
}

// ---- launchers -----------------------------------------------------------------

cudaError_t launch_measure(int w, const void* planes, Geom g, uint32_t X, void* scratch, void* result_dev,
                           cudaStream_t st) {
    const MeasScratch m = scratch_layout(scratch, g.Y);
    Partial* part = m.part;
    const uint32_t ngroups = measure_groups(g.c1 - g.c0);
    const uint32_t cblocks = (g.c1 - g.c0 + kColChunk - 1) / kColChunk;
    if (w == 64)
        k_col_scan<uint64_t><<<cblocks, kColChunk, 0, st>>>(static_cast<const uint64_t*>(planes), g, m);
    else
        k_col_scan<uint32_t><<<cblocks, kColChunk, 0, st>>>(static_cast<const uint32_t*>(planes), g, m);
    // persistent grid: exactly the blocks that are resident at once (registers / shared memory)
    auto persistent = [&](auto kern, uint32_t& grid) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMeasSmem));
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 0, per_sm = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMThreads, kMeasSmem)) != cudaSuccess)
            return e;
        grid = std::max<uint32_t>(1, std::min<uint32_t>(ngroups, uint32_t(std::max(per_sm, 1) * sms)));
        return cudaSuccess;
    };
    // segments of more than kNarrowSegSites sites (X > 2^17) keep all four segment sums in 128 bits
    const bool wide = (X + kSeg - 1) / kSeg > kNarrowSegSites;
    if (uint64_t(g.n) * g.Y >= (uint64_t(1) << 32)) return cudaErrorInvalidValue;  // 32-bit word offsets
    uint32_t grid = 1;
    auto go = [&](auto kern, const auto* pl) -> cudaError_t {
        const cudaError_t e = persistent(kern, grid);
        if (e != cudaSuccess) return e;
        kern<<<grid, kMThreads, kMeasSmem, st>>>(pl, g, X, m.G, m.tot, part);
        return cudaSuccess;
    };
    cudaError_t e;
    if (w == 64) {
        const uint64_t* pl = static_cast<const uint64_t*>(planes);
        e = wide ? go(k_measure_rows<uint64_t, true>, pl) : go(k_measure_rows<uint64_t, false>, pl);
    } else {
        const uint32_t* pl = static_cast<const uint32_t*>(planes);
        e = wide ? go(k_measure_rows<uint32_t, true>, pl) : go(k_measure_rows<uint32_t, false>, pl);
    }
    if (e != cudaSuccess) return e;
    k_measure_final<<<1, 1024, 0, st>>>(part, grid, m.col, static_cast<MeasureResult*>(result_dev));
    return cudaGetLastError();
}

cudaError_t launch_heights(int w, const void* planes, Geom g, uint32_t X, const void* scratch, int32_t* out,
                           cudaStream_t st) {
    const MeasScratch m = scratch_layout(const_cast<void*>(scratch), g.Y);
    const uint32_t threads = 128, blocks = (g.wrap * 32 + threads - 1) / threads;
    if (w == 64)
        k_heights<uint64_t><<<blocks, threads, 0, st>>>(static_cast<const uint64_t*>(planes), g, X, m.G, m.tot, out);
    else
        k_heights<uint32_t><<<blocks, threads, 0, st>>>(static_cast<const uint32_t*>(planes), g, X, m.G, m.tot, out);
    return cudaGetLastError();
}

}  // namespace octgpu
