// Device-side measurement: reconstruct_heights + height_moments
// (slope_field.hpp:159-229, measure.cpp:24-56) without materialising the
// HeightMap, in exact integer arithmetic.
//
// Heights: h(x,y) = H_y + r(x,y), H_y = sum_{y'=1..y} sigma_y-(0,y') (column
// 0) and r(x,y) = sum_{x'=1..x} sigma_x-(x',y) (row prefix). This equals the
// reference's row-0-then-columns integration whenever curl_check passes,
// which is checked in the same pass. With u(x) = sum_{x'<=x} sigma_x-(x',y)
// (inclusive from x = 0) we have h = G_y + u(x), G_y = H_y - sigma_x-(0,y),
// so S_k = sum_y sum_j C(k,j) G_y^(k-j) U_j(y) with U_j(y) = sum_x u(x)^j.
//
// Kernels (one measurement = 3 launches):
//   k_col_scan     single block: G_y for all rows (column-0 prefix) + column closure
//   k_measure_rows per row: word-parallel curl check, U_j via an 8-site lookup
//                  table, binomial shift by G_y, int128 block reduction
//   k_measure_final single block: sums the per-block partials
#include <cstdint>

#include "octgpu_internal.h"

namespace octgpu {

struct Partial {
    __int128 S[4];
    unsigned long long curl_count;
    unsigned long long curl_first;
    long long row0;
    long long pad;
};

namespace {

constexpr int kRowsPerWarp = 31;  // lane 0 is the y-1 halo for the curl check
constexpr int kThreads = 128;

uint32_t measure_blocks(uint32_t rows) {
    const uint32_t warps = (rows + kRowsPerWarp - 1) / kRowsPerWarp;
    return (warps * 32 + kThreads - 1) / kThreads;
}

__device__ __forceinline__ __int128 shfl_down_i128(__int128 v, int off) {
    unsigned long long lo = (unsigned long long)v, hi = (unsigned long long)((unsigned __int128)v >> 64);
    lo = __shfl_down_sync(0xffffffffu, lo, off);
    hi = __shfl_down_sync(0xffffffffu, hi, off);
    return (__int128)(((unsigned __int128)hi << 64) | lo);
}

}  // namespace

size_t measure_scratch_bytes(uint32_t Y) {
    return size_t(Y) * sizeof(long long) + size_t(measure_blocks(Y + 1)) * sizeof(Partial) + 64;
}

// ---- column 0: G_y and the column-0 closure ------------------------------
// Rows [start, start + count) in order; G[row] = sum_{rows <= row} sigma_y-(0,.) - sigma_x-(0,row)
// (- sigma_y-(0,start) when exclude_first: the periodic gauge h(0,0) = 0).
template <typename Word>
__global__ void __launch_bounds__(1024) k_col_scan(const Word* __restrict__ planes, Geom g, uint32_t start,
                                                   uint32_t count, int exclude_first, long long* __restrict__ G,
                                                   long long* __restrict__ col_sum, long long* __restrict__ sy_first) {
    __shared__ int warp_tot[32];
    __shared__ long long carry_sh;
    const size_t PS = g.plane_stride;
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    if (t == 0) carry_sh = 0;
    __syncthreads();
    const int par0 = int((start ^ g.ypar) & 1u);
    const int sy00 = (planes[(2 + par0) * PS + start] & 1) ? 1 : -1;
    const int excl = exclude_first ? sy00 : 0;
    for (uint32_t base = 0; base < count; base += 1024) {
        const uint32_t i = base + t;
        const uint32_t y = start + i;
        int sy = 0, s0 = 0;
        if (i < count) {
            const int par = int((y ^ g.ypar) & 1u);  // site (0,y) has parity (global y)&1
            sy = (planes[(2 + par) * PS + y] & 1) ? 1 : -1;
            s0 = (planes[par * PS + y] & 1) ? 1 : -1;
        }
        int incl = sy;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int o = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += o;
        }
        if (lane == 31) warp_tot[wp] = incl;
        __syncthreads();
        if (wp == 0) {
            int v = warp_tot[lane];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, v, off);
                if (lane >= off) v += o;
            }
            warp_tot[lane] = v;  // inclusive over warps
        }
        __syncthreads();
        const long long carry = carry_sh;
        const long long run = carry + incl + (wp > 0 ? warp_tot[wp - 1] : 0);  // sum_{y'<=y} sy
        if (i < count) G[y] = (run - excl) - s0;
        __syncthreads();
        if (t == 1023) carry_sh = run;
        __syncthreads();
    }
    if (t == 0) {
        *col_sum = carry_sh;
        *sy_first = sy00;
    }
}

// ---- per-row pass ------------------------------------------------------------
// 8-site table: index = nibble of the even-x plane | nibble of the odd-x plane << 4
// (sites interleave a0 b0 a1 b1 ...). Entry = d (net step), q_j = sum_i p_i^j
// over the chunk's 8 prefix values, packed: lo = q3:12 | q1:7 | d:5 | q2:8, hi = q4.
// 16 replicas (one per lane mod 16) make every warp lookup conflict-free.
__device__ __forceinline__ uint64_t lut_entry(uint32_t idx) {
    int p = 0, q1 = 0, q2 = 0, q3 = 0, q4 = 0;
    for (int i = 0; i < 8; ++i) {
        const uint32_t bit = (i & 1) ? (idx >> (4 + (i >> 1))) & 1 : (idx >> (i >> 1)) & 1;
        p += bit ? 1 : -1;
        q1 += p;
        q2 += p * p;
        q3 += p * p * p;
        q4 += p * p * p * p;
    }
    const uint32_t lo = (uint32_t(q3) & 0xfffu) | ((uint32_t(q1) & 0x7fu) << 12) | ((uint32_t(p) & 0x1fu) << 19) |
                        (uint32_t(q2) << 24);
    return (uint64_t(uint32_t(q4)) << 32) | lo;
}

template <typename Word>
__global__ void __launch_bounds__(kThreads, 4) k_measure_rows(const Word* __restrict__ planes, Geom g, uint32_t X,
                                                           const long long* __restrict__ Gv,
                                                           Partial* __restrict__ part) {
    constexpr int W = int(sizeof(Word) * 8);
    __shared__ uint64_t lut[256 * 16];
    __shared__ __int128 sh_s[4][kThreads / 32];
    __shared__ unsigned long long sh_cc[kThreads / 32], sh_cf[kThreads / 32];
    __shared__ long long sh_r0[kThreads / 32];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        const uint64_t e = lut_entry(i);
#pragma unroll
        for (int r = 0; r < 16; ++r) lut[i * 16 + r] = e;
    }
    __syncthreads();

    const uint32_t Y = g.Y, n = g.n;
    const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
    const uint32_t wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    __int128 S[4] = {0, 0, 0, 0};
    unsigned long long ccount = 0, cfirst = ~0ull;
    long long row0 = 0;
    if (wid * kRowsPerWarp < g.c1 - g.c0) {  // warp-uniform
        const uint32_t v = g.c0 - 1 + wid * kRowsPerWarp + lane;  // lane 0: the y-1 halo row
        const uint32_t y = g.wrap ? v % g.wrap : v;
        const bool core = lane >= 1 && v < g.c1;
        const uint32_t row_id = g.wrap ? y : v - g.c0;  // position of this row in the result's scan order
        const size_t PS = g.plane_stride;
        const Word* X0 = planes + y;
        const Word* X1 = planes + PS + y;
        const Word* Y0 = planes + 2 * PS + y;
        const Word* Y1 = planes + 3 * PS + y;
        const int ya = int((y ^ g.ypar) & 1u);
        const uint64_t* lrep = lut + (lane & 15);
        const size_t last = size_t(n - 1) * Y;
        Word pD0 = Y0[last], pD1 = Y1[last];
        long long U1 = 0, U2 = 0, rowsum = 0;
        __int128 U3 = 0, U4 = 0;
        int u0 = 0;
        unsigned int rc = 0, rfirst = 0xffffffffu;
        for (uint32_t k = 0; k < n; ++k) {
            const size_t o = size_t(k) * Y;
            const Word x0 = X0[o], x1 = X1[o], yy0 = Y0[o], yy1 = Y1[o];
            const Word bx0 = __shfl_up_sync(0xffffffffu, x0, 1);
            const Word bx1 = __shfl_up_sync(0xffffffffu, x1, 1);
#pragma unroll
            for (int pi = 0; pi < 2; ++pi) {  // curl check, word-parallel
                const Word A = pi ? x1 : x0;
                const Word B = pi ? bx0 : bx1;
                const Word C = pi ? yy1 : yy0;
                const Word Dr = pi ? yy0 : yy1;
                const Word Dp = pi ? pD0 : pD1;
                const bool even_x = ((uint32_t(pi) ^ y ^ g.ypar) & 1u) == 0;
                const Word D = even_x ? Word((Dr << 1) | (Dp >> (W - 1))) : Dr;
                const Word Vv = (A ^ B ^ C ^ D) | ((A ^ B) & (A ^ C));
                if (Vv) {
                    rc += __popcll((unsigned long long)Vv);
                    const uint32_t b = __ffsll((long long)(unsigned long long)Vv) - 1;
                    rfirst = min(rfirst, 2u * (k * W + b) + (even_x ? 0u : 1u));
                }
            }
            pD0 = yy0;
            pD1 = yy1;
            const Word xa = ya ? x1 : x0;  // even-x sites of row y
            const Word xb = ya ? x0 : x1;  // odd-x sites
            rowsum += 2 * (__popcll((unsigned long long)xa) + __popcll((unsigned long long)xb)) - 2 * W;
            // 8-site chunk indices, nibble of xa | nibble of xb << 4, gathered per 32-bit half
            int u = 0, c1 = 0, c2 = 0, c3 = 0;
            unsigned long long c4 = 0;
#pragma unroll
            for (int half = 0; half < W / 32; ++half) {
                const uint32_t a32 = uint32_t(uint64_t(xa) >> (32 * half));
                const uint32_t b32 = uint32_t(uint64_t(xb) >> (32 * half));
                const uint32_t evn = (a32 & 0x0F0F0F0Fu) | ((b32 & 0x0F0F0F0Fu) << 4);  // chunks 0,2,4,6
                const uint32_t odd = ((a32 >> 4) & 0x0F0F0F0Fu) | (b32 & 0xF0F0F0F0u);  // chunks 1,3,5,7
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    const uint32_t idx = (((ch & 1) ? odd : evn) >> (8 * (ch >> 1))) & 0xffu;
                    const uint64_t e = lrep[idx * 16];
                    const uint32_t lo = uint32_t(e);
                    const int q3 = int(lo << 20) >> 20;
                    const int q1 = int(lo << 13) >> 25;
                    const int d = int(lo << 8) >> 27;
                    const int q2 = int(lo >> 24);
                    const int q4 = int(e >> 32);
                    const int u2 = u * u, u3 = u2 * u, u4 = u2 * u2;  // |u| <= 120: u4 < 2^28
                    c1 += 8 * u + q1;
                    c2 += 8 * u2 + 2 * u * q1 + q2;
                    c3 += 8 * u3 + 3 * u2 * q1 + 3 * u * q2 + q3;
                    // sum_i (u + p_i)^4 over the chunk: >= 0 and < 2^31 for |u| <= 120
                    const int t4 = 8 * u4 + 4 * u3 * q1 + 6 * u2 * q2 + 4 * u * q3 + q4;
                    c4 += (unsigned long long)(unsigned)t4;
                    u += d;
                }
            }
            constexpr long long NS = 2 * W;
            if (u0 >= -4096 && u0 <= 4096) {  // 32x32->64 products only, then one int128 add each
                const int a = u0, aa = a * a;                     // aa <= 2^24
                const long long aaa = (long long)aa * a;          // <= 2^36
                const long long a4 = (long long)aa * aa;          // <= 2^48
                U1 += (long long)(NS * a) + c1;
                U2 += (long long)aa * NS + (long long)(2 * a) * c1 + c2;
                U3 += (__int128)(aaa * NS + (long long)(3 * aa) * c1 + (long long)(3 * a) * c2 + c3);
                U4 += (__int128)(a4 * NS + 4 * aaa * c1 + (long long)(6 * aa) * c2 + (long long)(4 * a) * c3 +
                                 (long long)c4);
            } else {
                const long long uu = (long long)u0 * u0;
                const __int128 uuu = (__int128)uu * u0;
                U1 += NS * u0 + c1;
                U2 += NS * uu + 2ll * u0 * c1 + c2;
                U3 += (__int128)NS * uuu + (__int128)(3 * uu) * c1 + (__int128)(3ll * u0) * c2 + c3;
                U4 += (__int128)NS * uuu * u0 + (__int128)4 * uuu * c1 + (__int128)(6 * uu) * c2 +
                      (__int128)(4ll * u0) * c3 + (__int128)c4;
            }
            u0 += u;
        }
        if (core) {
            const __int128 G = Gv[y];
            const __int128 g2 = G * G, g3 = g2 * G, g4 = g3 * G;
            const __int128 U0 = X;
            S[0] = G * U0 + U1;
            S[1] = g2 * U0 + 2 * G * U1 + U2;
            S[2] = g3 * U0 + 3 * g2 * U1 + 3 * G * U2 + U3;
            S[3] = g4 * U0 + 4 * g3 * U1 + 6 * g2 * U2 + 4 * G * U3 + U4;
            ccount = rc;
            if (rfirst != 0xffffffffu) cfirst = (unsigned long long)row_id * X + rfirst;
            if (row_id == 0) row0 = rowsum;
        }
    }
    // block reduction
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        __int128 vs = S[k];
        for (int off = 16; off > 0; off >>= 1) vs += shfl_down_i128(vs, off);
        if (lane == 0) sh_s[k][wp] = vs;
    }
    for (int off = 16; off > 0; off >>= 1) {
        ccount += __shfl_down_sync(0xffffffffu, ccount, off);
        const unsigned long long o = __shfl_down_sync(0xffffffffu, cfirst, off);
        cfirst = o < cfirst ? o : cfirst;
        row0 += __shfl_down_sync(0xffffffffu, row0, off);
    }
    if (lane == 0) {
        sh_cc[wp] = ccount;
        sh_cf[wp] = cfirst;
        sh_r0[wp] = row0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial pr;
        for (int k = 0; k < 4; ++k) pr.S[k] = 0;
        pr.curl_count = 0;
        pr.curl_first = ~0ull;
        pr.row0 = 0;
        pr.pad = 0;
        for (int i = 0; i < kThreads / 32; ++i) {
            for (int k = 0; k < 4; ++k) pr.S[k] += sh_s[k][i];
            pr.curl_count += sh_cc[i];
            pr.curl_first = sh_cf[i] < pr.curl_first ? sh_cf[i] : pr.curl_first;
            pr.row0 += sh_r0[i];
        }
        part[blockIdx.x] = pr;
    }
}

__global__ void __launch_bounds__(256) k_measure_final(const Partial* __restrict__ part, uint32_t nb,
                                                       const long long* __restrict__ col_sum,
                                                       const long long* __restrict__ sy_first,
                                                       MeasureResult* __restrict__ res) {
    __shared__ __int128 sh_s[4][8];
    __shared__ unsigned long long sh_cc[8], sh_cf[8];
    __shared__ long long sh_r0[8];
    const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
    __int128 S[4] = {0, 0, 0, 0};
    unsigned long long cc = 0, cf = ~0ull;
    long long r0 = 0;
    for (uint32_t i = t; i < nb; i += blockDim.x) {
        const Partial p = part[i];
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
        for (int i = 0; i < 8; ++i) {
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
        res->col0_sum = *col_sum;
        res->sy_first = *sy_first;
        res->pad = 0;
    }
}

// Heights (reference HeightMap layout): one warp per row, lane l owns words
// l, l+32, ...; h(x,y) = G_y + u(x).
template <typename Word>
__global__ void k_heights(const Word* __restrict__ planes, Geom g, uint32_t X, const long long* __restrict__ G,
                          int32_t* __restrict__ out) {
    constexpr int W = int(sizeof(Word) * 8);
    const uint32_t Y = g.wrap, LD = g.Y, n = g.n;  // periodic only
    const uint32_t y = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (y >= Y) return;
    const size_t PS = g.plane_stride;
    const int ya = int(y & 1u);
    const Word* Xa = planes + size_t(ya) * PS + y;
    const Word* Xb = planes + size_t(ya ^ 1) * PS + y;
    long long carry = G[y];
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
    Partial* part = reinterpret_cast<Partial*>(G + g.Y);
    const uint32_t rows = g.c1 - g.c0;
    const uint32_t nb = measure_blocks(rows);
    long long* col = reinterpret_cast<long long*>(part + measure_blocks(g.Y + 1));
    long long* syf = col + 1;
    // periodic: rows 0..Y-1 in the reference's gauge; stripe: its core rows, local gauge
    const uint32_t start = g.wrap ? 0 : g.c0;
    const int excl = g.wrap ? 1 : 0;
    if (w == 64) {
        k_col_scan<uint64_t><<<1, 1024, 0, st>>>(static_cast<const uint64_t*>(planes), g, start, rows, excl, G, col,
                                                  syf);
        k_measure_rows<uint64_t><<<nb, kThreads, 0, st>>>(static_cast<const uint64_t*>(planes), g, X, G, part);
    } else {
        k_col_scan<uint32_t><<<1, 1024, 0, st>>>(static_cast<const uint32_t*>(planes), g, start, rows, excl, G, col,
                                                  syf);
        k_measure_rows<uint32_t><<<nb, kThreads, 0, st>>>(static_cast<const uint32_t*>(planes), g, X, G, part);
    }
    k_measure_final<<<1, 256, 0, st>>>(part, nb, col, syf, static_cast<MeasureResult*>(result_dev));
    return cudaGetLastError();
}

cudaError_t launch_heights(int w, const void* planes, Geom g, uint32_t X, const void* scratch, int32_t* out,
                           cudaStream_t st) {
    const long long* G = static_cast<const long long*>(scratch);
    const uint32_t threads = 128, blocks = (g.wrap * 32 + threads - 1) / threads;
    if (w == 64)
        k_heights<uint64_t><<<blocks, threads, 0, st>>>(static_cast<const uint64_t*>(planes), g, X, G, out);
    else
        k_heights<uint32_t><<<blocks, threads, 0, st>>>(static_cast<const uint32_t*>(planes), g, X, G, out);
    return cudaGetLastError();
}

}  // namespace octgpu
