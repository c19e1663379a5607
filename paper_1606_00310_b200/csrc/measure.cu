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
// Kernels (one measurement = 2 launches):
//   k_measure_rows  per block: 4 row groups of 31 rows (lane per row; lane 0 is the row above,
//                   for the curl check) x 4 x-segments (one warp each). Word-parallel curl
//                   check; U_j per segment from 16-site units read through two 8-site tables
//                   (the second indexed by the first's net step, so a unit costs one combine);
//                   segments and rows combined in int128 in a block-local column-0 gauge.
//   k_measure_final one block: exclusive prefix of the blocks' column-0 increments, binomial
//                   shift of each block's sums to the global gauge, reduction, closure data.
// Scan order = virtual rows c0 .. c1-1 (periodic: physical rows 1 .. Y-1, 0; a stripe: its core
// rows); the gauge H is 0 at virtual row c0 - 1. For a periodic lattice that is the reference's
// h(0,0) = 0 whenever the column closes (otherwise the measurement fails with the reference's
// column error before the sums are used).
#include <algorithm>
#include <cstdint>

#include "octgpu_internal.h"

namespace octgpu {

struct Partial {
    __int128 S[4];                   // block sums in the block-local gauge (H = 0 before its first row)
    unsigned long long curl_count;
    unsigned long long curl_first;   // row_id * X + x, ~0 if none
    long long row0;                  // sum_x sigma_x- of row_id 0 (the block holding it)
    long long delta;                 // sum of sigma_y-(0, y) over the block's rows
    long long sy_first;              // sigma_y-(0, c0) (block 0)
    long long prefix;                // written by k_measure_final: H offset of the block
    unsigned long long n_sites;
    long long pad;
};

namespace {

constexpr int kRowsPerGroup = 31;  // lane 0 is the y-1 halo for the curl check
constexpr int kSeg = 8;            // x-segments per row: one warp each; a block = one row group at a time
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
// offset o (the height just before the byte, relative to the unit start) the entry holds
// q_k = sum_i (o + p_i)^k over the byte's inclusive prefix values p_i, k = 1..4, and d = p_7.
// T0 = offset 0 (first byte of a 16-site unit), T1[o + 8] = offsets -8..8 (second byte, indexed
// by the first byte's d). Biased fields; the sum of a T0 and a T1 entry is the unit's, without
// carries between fields:  lo = q3 + B3 (16 bits) | q1 + B1 << 16 (9 bits) | d + 8 << 25,
// hi = q2 (11 bits) | q4 << 11 (18 bits); unit biases B1 = 136 (36 + 100), B3 = 18496 (1296 + 17200),
// d: 16.
constexpr int kUnitB1 = 136, kUnitB3 = 18496, kUnitD = 16;

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
    const int b1 = second ? 100 : 36, b3 = second ? 17200 : 1296;
    const uint32_t lo = uint32_t(q3 + b3) | (uint32_t(q1 + b1) << 16) | (uint32_t(p + 8) << 25);
    const uint32_t hi = uint32_t(q2) | (uint32_t(q4) << 11);
    return uint2{lo, hi};
}

struct MeasTabInit : MeasTab {
    constexpr MeasTabInit() : MeasTab{} {
        for (int b = 0; b < 256; ++b) t0[b] = tab_entry(b, 0, false);
        for (int o = -8; o <= 8; ++o)
            for (int b = 0; b < 256; ++b) t1[(o + 8) * 256 + b] = tab_entry(b, o, true);
    }
};

__device__ const MeasTab g_tab = MeasTabInit();

// shared memory: T0 replicated x16 (entry b at [b][lane & 15]: every warp lookup conflict-free),
// T1 once; reused for the cross-warp combine after the row pass
#ifndef OCTGPU_MEAS_REP
#define OCTGPU_MEAS_REP 16  // T0 replicas: 16 = every lookup conflict-free
#endif
#ifndef OCTGPU_MEAS_MINB
#define OCTGPU_MEAS_MINB 2  // resident blocks per SM the register budget targets
#endif
constexpr int kRep = OCTGPU_MEAS_REP;
constexpr int kT0Words = 256 * kRep;  // uint2
constexpr int kT1Words = 17 * 256;
struct SegOut {                      // one lane's segment result (int128 sums, delta, curl)
    __int128 T[4];
    long long D;
    unsigned int rc, rfirst;
};
constexpr size_t kMeasSmem = sizeof(uint2) * (kT0Words + kT1Words) + sizeof(SegOut) * kMThreads;

}  // namespace

size_t measure_scratch_bytes(uint32_t Y) {
    return size_t(Y + 2) * sizeof(long long) + size_t(measure_groups(Y + 1) + 1) * sizeof(Partial) + 64;
}

namespace {

// signed 32 x 32 -> 64-bit multiply-add in one IMAD.WIDE (the compiler otherwise emits the unsigned form
// plus a sign correction when it can prove one factor non-negative)
__device__ __forceinline__ long long madw(int a, int b, long long c) {
    long long d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}

// Unit accumulators since the last flush; heights relative to the segment base + u.
struct UnitAcc {
    int Au1, Au2, Aq1, Aq2, Aq3, X11, X12, units;
    unsigned int Aq4;
    long long Au3, Au4, X13, X21, X22, X31;
    __device__ __forceinline__ void clear() {
        Au1 = Au2 = Aq1 = Aq2 = Aq3 = X11 = X12 = units = 0;
        Aq4 = 0;
        Au3 = Au4 = X13 = X21 = X22 = X31 = 0;
    }
};

// T_k += sum_j C(k,j) B^(k-j) t_j for the unit sums t_j of heights B + u (u = offset within the flush)
__device__ __noinline__ void flush_units(UnitAcc& A, long long B, __int128* T) {
    const long long K = A.units;
    const long long t1 = 16ll * A.Au1 + A.Aq1 - kUnitB1 * K;
    const long long t2 = 16ll * A.Au2 + 2ll * (A.X11 - (long long)kUnitB1 * A.Au1) + A.Aq2;
    const long long t3 = 16ll * A.Au3 + 3ll * (A.X21 - (long long)kUnitB1 * A.Au2) + 3ll * A.X12 + A.Aq3 -
                         (long long)kUnitB3 * K;
    const long long t4 = 16ll * A.Au4 + 4ll * (A.X31 - (long long)kUnitB1 * A.Au3) + 6ll * A.X22 +
                         4ll * (A.X13 - (long long)kUnitB3 * A.Au1) + (long long)A.Aq4;
    const __int128 b = B, b2 = b * b, b3 = b2 * b, b4 = b2 * b2, t0 = 16 * K;
    T[0] += b * t0 + t1;
    T[1] += b2 * t0 + 2 * b * t1 + t2;
    T[2] += b3 * t0 + 3 * b2 * t1 + 3 * b * t2 + t3;
    T[3] += b4 * t0 + 4 * b3 * t1 + 6 * b2 * t2 + 4 * b * t3 + t4;
    A.clear();
}

// one 16-site unit: byte b0 (first 8 sites) then b1 (next 8) of the row. t0b = this lane's replica of
// T0 (entry b at t0b + 16 b), t1b = T1.
__device__ __forceinline__ void unit(UnitAcc& A, int& u, uint32_t b0, uint32_t b1, const uint2* t0b,
                                     const uint2* t1b) {
    const uint2 e0 = t0b[b0 * kRep];
    const uint2 e1 = t1b[(e0.x >> 25) * 256 + b1];
    const uint32_t lo = e0.x + e1.x, hi = e0.y + e1.y;
    const int q3b = int(lo & 0xffffu), q1b = int((lo >> 16) & 0x1ffu), Db = int(lo >> 25);
    const int q2 = int(hi & 0x7ffu);
    const unsigned int q4 = hi >> 11;
    const int u2 = u * u, u3 = u2 * u;
    A.Au1 += u;
    A.Au2 += u2;
    A.Au3 += (long long)u3;
    A.Au4 = madw(u2, u2, A.Au4);
    A.Aq1 += q1b;
    A.Aq2 += q2;
    A.Aq3 += q3b;
    A.Aq4 += q4;
    A.X11 += u * q1b;
    A.X12 += u * q2;
    A.X13 = madw(u, q3b, A.X13);
    A.X21 = madw(u2, q1b, A.X21);
    A.X22 = madw(u2, q2, A.X22);
    A.X31 = madw(u3, q1b, A.X31);
    u += Db - kUnitD;
    ++A.units;
}

}  // namespace

// ---- row pass -------------------------------------------------------------------------
// Persistent blocks of kSeg warps walk the row groups (31 core rows each, lane 0 = the row above):
// warp s handles x-segment s (words [s n / kSeg, (s+1) n / kSeg)) of the group's 32 rows, then warp 0
// combines the segments of each row and the group's rows into one Partial (group-local gauge).
template <typename Word>
__global__ void __launch_bounds__(kMThreads, OCTGPU_MEAS_MINB) k_measure_rows(const Word* __restrict__ planes, Geom g, uint32_t X,
                                                               long long* __restrict__ Gout, Partial* __restrict__ part) {
    constexpr int W = int(sizeof(Word) * 8);
    extern __shared__ __align__(16) unsigned char msm[];
    uint2* t0rep = reinterpret_cast<uint2*>(msm);
    uint2* t1 = t0rep + kT0Words;
    SegOut* so = reinterpret_cast<SegOut*>(t1 + kT1Words);
    for (int i = threadIdx.x; i < kT0Words; i += kMThreads) t0rep[i] = g_tab.t0[i / kRep];
    {
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
    const uint2* t0b = t0rep + (lane % kRep);

    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t first = g.c0 + grp * uint32_t(kRowsPerGroup);  // the group's first core row
        const uint32_t v = first - 1 + uint32_t(lane);                // lane 0: the row above
        const uint32_t y = g.wrap ? v % g.wrap : v;
        const bool core = lane >= 1 && v < g.c1;
        const uint32_t row_id = g.wrap ? y : v - g.c0;
        const int ya = int((y ^ g.ypar) & 1u);
        // even-x sites of row y are in X(ya), odd-x in X(!ya); C = Y(ya), its partner Y(!ya)
        const Word* pXa = planes + size_t(ya) * PS + y;
        const Word* pXb = planes + size_t(ya ^ 1) * PS + y;
        const Word* pCa = planes + size_t(2 + ya) * PS + y;
        const Word* pCb = planes + size_t(3 - ya) * PS + y;

        __int128 T[4] = {0, 0, 0, 0};
        long long B = 0;
        unsigned int rc = 0, rfirst = 0xffffffffu;
        {
            UnitAcc A;
            A.clear();
            int u = 0;
            Word pcb = 0, nxa = 0, nxb = 0, nca = 0, ncb = 0;
            if (kend > kbeg) {
                pcb = pCb[size_t(kbeg == 0 ? n - 1 : kbeg - 1) * Y];
                const size_t o = size_t(kbeg) * Y;
                nxa = pXa[o];
                nxb = pXb[o];
                nca = pCa[o];
                ncb = pCb[o];
            }
            for (uint32_t k = kbeg; k < kend; ++k) {
                const Word xa = nxa, xb = nxb, ca = nca, cb = ncb;
                if (k + 1 < kend) {  // prefetch the next word (the loads were the top stall)
                    const size_t o = size_t(k + 1) * Y;
                    nxa = pXa[o];
                    nxb = pXb[o];
                    nca = pCa[o];
                    ncb = pCb[o];
                }
                const Word bxa = __shfl_up_sync(0xffffffffu, xa, 1);
                const Word bxb = __shfl_up_sync(0xffffffffu, xb, 1);
                // curl check, word-parallel: parity ya (even-x sites, D rotated up one packed
                // bit with the previous word's top bit) and parity !ya (odd-x sites, D aligned)
                const Word D1 = Word((cb << 1) | (pcb >> (W - 1)));
                const Word V1 = (xa ^ bxa ^ ca ^ D1) | ((xa ^ bxa) & (xa ^ ca));
                const Word V2 = (xb ^ bxb ^ cb ^ ca) | ((xb ^ bxb) & (xb ^ cb));
                pcb = cb;
                if (V1 | V2) {
                    rc += __popcll((unsigned long long)V1) + __popcll((unsigned long long)V2);
                    if (V1)
                        rfirst = min(rfirst, 2u * (k * W + uint32_t(__ffsll((long long)(unsigned long long)V1) - 1)));
                    if (V2)
                        rfirst = min(rfirst,
                                     2u * (k * W + uint32_t(__ffsll((long long)(unsigned long long)V2) - 1)) + 1u);
                }
                // rebase before the 32-bit unit accumulators could overflow: |u| <= 1024, <= 1024 units
                if (u > 1024 - 2 * W || u < -(1024 - 2 * W) || A.units > 1024 - W / 4) {
                    flush_units(A, B, T);
                    B += u;
                    u = 0;
                }
#pragma unroll
                for (int half = 0; half < W / 32; ++half) {
                    const uint32_t a32 = uint32_t(uint64_t(xa) >> (32 * half));
                    const uint32_t b32 = uint32_t(uint64_t(xb) >> (32 * half));
                    const uint32_t evn = (a32 & 0x0F0F0F0Fu) | ((b32 & 0x0F0F0F0Fu) << 4);  // chunks 0,2,4,6
                    const uint32_t odd = ((a32 >> 4) & 0x0F0F0F0Fu) | (b32 & 0xF0F0F0F0u);  // chunks 1,3,5,7
#pragma unroll
                    for (int un = 0; un < 4; ++un)
                        unit(A, u, __byte_perm(evn, 0, 0x4440 + un), __byte_perm(odd, 0, 0x4440 + un), t0b, t1);
                }
            }
            flush_units(A, B, T);
            B += u;
        }
        {
            SegOut& m = so[threadIdx.x];
            for (int k = 0; k < 4; ++k) m.T[k] = T[k];
            m.D = B;
            m.rc = rc;
            m.rfirst = rfirst;
        }
        __syncthreads();
        if (seg == 0) {
            // column 0 in the group gauge: inclusive prefix of sigma_y-(0, y) over the core rows
            // sigma_y-(0, y) and sigma_x-(0, y): bit 0 of word 0 of Y(ya) and X(ya)
            const int sy0 = (pCa[0] & 1) ? 1 : -1, sx0 = (pXa[0] & 1) ? 1 : -1;
            long long incl = core ? sy0 : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const long long t = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= off) incl += t;
            }
            __int128 S[4] = {0, 0, 0, 0};
            unsigned long long ccount = 0, cfirst = ~0ull;
            long long row0 = 0;
            if (core) {
                const long long G = incl - sx0;  // group-local G_y = H'_y - sigma_x-(0, y)
                Gout[y] = G;
                // the row's U_j: segments in order, each shifted by the net step of the segments before it
                __int128 U[4] = {0, 0, 0, 0};
                long long off = 0;
                unsigned int crc = 0, cfst = 0xffffffffu;
                for (int s2 = 0; s2 < kSeg; ++s2) {
                    const SegOut& m = so[s2 * 32 + lane];
                    const __int128 c = off, c2 = c * c, c3 = c2 * c, c4 = c2 * c2;
                    const __int128 ns = (__int128)(uint32_t(s2 + 1) * n / kSeg - uint32_t(s2) * n / kSeg) * 2 * W;
                    U[0] += c * ns + m.T[0];
                    U[1] += c2 * ns + 2 * c * m.T[0] + m.T[1];
                    U[2] += c3 * ns + 3 * c2 * m.T[0] + 3 * c * m.T[1] + m.T[2];
                    U[3] += c4 * ns + 4 * c3 * m.T[0] + 6 * c2 * m.T[1] + 4 * c * m.T[2] + m.T[3];
                    off += m.D;
                    crc += m.rc;
                    cfst = min(cfst, m.rfirst);
                }
                const __int128 Gq = G, g2 = Gq * Gq, g3 = g2 * Gq, g4 = g2 * g2, U0 = X;
                S[0] = Gq * U0 + U[0];
                S[1] = g2 * U0 + 2 * Gq * U[0] + U[1];
                S[2] = g3 * U0 + 3 * g2 * U[0] + 3 * Gq * U[1] + U[2];
                S[3] = g4 * U0 + 4 * g3 * U[0] + 6 * g2 * U[1] + 4 * Gq * U[2] + U[3];
                ccount = crc;
                if (cfst != 0xffffffffu) cfirst = (unsigned long long)row_id * X + cfst;
                if (row_id == 0) row0 = off;  // sum_x sigma_x- of the row
            }
            const long long delta = __shfl_sync(0xffffffffu, incl, 31);
            const long long syf = __shfl_sync(0xffffffffu, (long long)sy0, 1);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                for (int off = 16; off > 0; off >>= 1) S[k] += shfl_down_i128(S[k], off);
            for (int off = 16; off > 0; off >>= 1) {
                ccount += __shfl_down_sync(0xffffffffu, ccount, off);
                const unsigned long long o = __shfl_down_sync(0xffffffffu, cfirst, off);
                cfirst = o < cfirst ? o : cfirst;
                row0 += __shfl_down_sync(0xffffffffu, row0, off);
            }
            if (lane == 0) {
                Partial pr;
                for (int k = 0; k < 4; ++k) pr.S[k] = S[k];
                pr.curl_count = ccount;
                pr.curl_first = cfirst;
                pr.row0 = row0;
                pr.delta = delta;
                pr.sy_first = syf;
                pr.prefix = 0;
                pr.n_sites = (unsigned long long)min(uint32_t(kRowsPerGroup), g.c1 - first) * X;
                pr.pad = 0;
                part[grp] = pr;
            }
        }
        __syncthreads();  // the segment buffer is rewritten by the next group
    }
}

__global__ void __launch_bounds__(1024) k_measure_final(Partial* __restrict__ part, uint32_t nb,
                                                        MeasureResult* __restrict__ res) {
    __shared__ __int128 sh_s[4][32];
    __shared__ unsigned long long sh_cc[32], sh_cf[32];
    __shared__ long long sh_r0[32], sh_tot[32];
    __shared__ long long carry_sh;
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    if (t == 0) carry_sh = 0;
    __syncthreads();
    __int128 S[4] = {0, 0, 0, 0};
    unsigned long long cc = 0, cf = ~0ull;
    long long r0 = 0;
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t i = base + t;
        Partial p{};
        if (i < nb) p = part[i];
        // exclusive prefix of the blocks' column-0 increments (block order = scan order)
        long long incl = i < nb ? p.delta : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) sh_tot[wp] = incl;
        __syncthreads();
        if (wp == 0) {
            long long v = sh_tot[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const long long o = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += o;
            }
            sh_tot[lane] = v;
        }
        __syncthreads();
        const long long carry = carry_sh;
        const long long pre = carry + incl - (i < nb ? p.delta : 0) + (wp > 0 ? sh_tot[wp - 1] : 0);
        if (i < nb) {
            part[i].prefix = pre;
            const __int128 c = pre, c2 = c * c, c3 = c2 * c, c4 = c2 * c2, ns = (__int128)p.n_sites;
            S[0] += c * ns + p.S[0];
            S[1] += c2 * ns + 2 * c * p.S[0] + p.S[1];
            S[2] += c3 * ns + 3 * c2 * p.S[0] + 3 * c * p.S[1] + p.S[2];
            S[3] += c4 * ns + 4 * c3 * p.S[0] + 6 * c2 * p.S[1] + 4 * c * p.S[2] + p.S[3];
            cc += p.curl_count;
            cf = p.curl_first < cf ? p.curl_first : cf;
            r0 += p.row0;
        }
        __syncthreads();
        if (t == 1023) carry_sh = pre + (i < nb ? p.delta : 0);
        __syncthreads();
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
        res->col0_sum = carry_sh;
        res->sy_first = part[0].sy_first;
        res->pad = 0;
    }
}

// Heights (reference HeightMap layout): one warp per row, lane l owns words
// l, l+32, ...; h(x,y) = G_y + u(x) with G_y = block-local G + the block's prefix.
template <typename Word>
__global__ void k_heights(const Word* __restrict__ planes, Geom g, uint32_t X, const long long* __restrict__ G,
                          const Partial* __restrict__ part, int32_t* __restrict__ out) {
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
    long long carry = G[y] + part[(vrow - g.c0) / kRowsPerGroup].prefix;
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
    long long* G = static_cast<long long*>(scratch);
    Partial* part = reinterpret_cast<Partial*>(G + ((g.Y + 2) & ~1u));  // 16-B aligned (int128)
    const uint32_t ngroups = measure_groups(g.c1 - g.c0);
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
    uint32_t grid = 1;
    if (w == 64) {
        cudaError_t e = persistent(k_measure_rows<uint64_t>, grid);
        if (e != cudaSuccess) return e;
        k_measure_rows<uint64_t><<<grid, kMThreads, kMeasSmem, st>>>(static_cast<const uint64_t*>(planes), g, X, G,
                                                                      part);
    } else {
        cudaError_t e = persistent(k_measure_rows<uint32_t>, grid);
        if (e != cudaSuccess) return e;
        k_measure_rows<uint32_t><<<grid, kMThreads, kMeasSmem, st>>>(static_cast<const uint32_t*>(planes), g, X, G,
                                                                      part);
    }
    k_measure_final<<<1, 1024, 0, st>>>(part, ngroups, static_cast<MeasureResult*>(result_dev));
    return cudaGetLastError();
}

cudaError_t launch_heights(int w, const void* planes, Geom g, uint32_t X, const void* scratch, int32_t* out,
                           cudaStream_t st) {
    const long long* G = static_cast<const long long*>(scratch);
    const Partial* part = reinterpret_cast<const Partial*>(G + ((g.Y + 2) & ~1u));
    const uint32_t threads = 128, blocks = (g.wrap * 32 + threads - 1) / threads;
    if (w == 64)
        k_heights<uint64_t><<<blocks, threads, 0, st>>>(static_cast<const uint64_t*>(planes), g, X, G, part, out);
    else
        k_heights<uint32_t><<<blocks, threads, 0, st>>>(static_cast<const uint32_t*>(planes), g, X, G, part, out);
    return cudaGetLastError();
}

}  // namespace octgpu
