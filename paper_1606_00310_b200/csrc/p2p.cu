// Device-side halo exchange between row stripes over peer memory (NVLink /
// NVSwitch P2P, or the same device): no NCCL, no host round trip per pass.
//
// Each stripe engine exposes its two plane sets, two rng-state sets and a
// "done" counter (passes completed) to its ring neighbours. One pass P of a
// stripe is, on its own stream:
//   k_halo_pull      wait until both neighbours report done >= P-1, then read
//                    their boundary core rows straight from their memory into
//                    the local halo rows (xoshiro states only once, at connect:
//                    afterwards every pass advances the streams of its halo
//                    rows itself, so no stripe reads a neighbour's states
//                    while that neighbour applies a lazy jump in place)
//   MCS kernel       k_mcs_deep (2 MCS) or k_mcs_bulk (1 MCS), unchanged
//   k_push_signal    write the finished y-plane f of the first halo row below
//                    into the next stripe's first core row (its own pass never
//                    writes that plane-row), then publish done = P
//                    (threadfence.sys + st.release.sys)
// Why this is race-free with ping-pong plane sets (set index = pass parity,
// identical on every stripe):
//  * pass P reads the neighbours' set P%2 (their pass P-1 output, complete
//    when done >= P-1) and writes the local set (P+1)%2;
//  * the push writes the next stripe's set (P+1)%2, which that stripe last
//    READ in its pass P-1 (done >= P-1 was awaited) and whose plane-row it
//    never writes itself;
//  * a neighbour cannot start pass P+1 (overwriting its set P%2 that we read)
//    before we publish done = P, after our pull.
// Waits are bounded (clock64): on timeout the kernel raises an error flag the
// host reports as OCTGPU_ERR_CUDA instead of hanging the GPU.
#include <algorithm>
#include <cstdint>

#include "octgpu_internal.h"

namespace octgpu {

namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// thread 0 of the block waits for both counters; the block then proceeds
__device__ __forceinline__ bool block_wait(const uint64_t* a, const uint64_t* b, uint64_t need, uint32_t* err,
                                           long long limit) {
    __shared__ int ok;
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        ok = 1;
        while (ld_acquire_sys(a) < need || ld_acquire_sys(b) < need) {
            if (clock64() - t0 > limit) {
                atomicExch(err, 1u);
                ok = 0;
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    return ok != 0;
}

template <typename Word>
__global__ void k_halo_pull(Word* __restrict__ planes, uint64_t* __restrict__ rng, Geom g, PeerView prev,
                            PeerView next, uint64_t need, uint32_t* err, int with_rng) {
    if (!block_wait(prev.done, next.done, need, err, prev.timeout)) return;
    const uint32_t n = g.n;
    const uint32_t rows = kStripeHA + kStripeHB;
    const uint32_t per = rows * n, total = 4 * per;
    const uint32_t L = g.c1 - g.c0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t p = i / per, rem = i % per, r = rem / n, k = rem % n;
        const bool above = r < kStripeHA;
        const PeerView& pv = above ? prev : next;
        // above: the previous stripe's last HA core rows; below: the next stripe's first HB core rows
        const uint32_t src_row = above ? pv.L + r : kStripeHA + (r - kStripeHA);
        const uint32_t dst_row = above ? r : kStripeHA + L + (r - kStripeHA);
        const Word* sp = static_cast<const Word*>(pv.planes);
        planes[size_t(p) * g.plane_stride + size_t(k) * g.Y + dst_row] =
            sp[size_t(p) * size_t(n) * pv.Y + size_t(k) * pv.Y + src_row];
    }
    if (with_rng && blockIdx.x == 0)
        for (uint32_t t = threadIdx.x; t < 4 * rows; t += blockDim.x) {
            const uint32_t j = t & 3, r = t >> 2;
            const bool above = r < kStripeHA;
            const PeerView& pv = above ? prev : next;
            const uint32_t src_row = above ? pv.L + r : kStripeHA + (r - kStripeHA);
            const uint32_t dst_row = above ? r : kStripeHA + L + (r - kStripeHA);
            rng[size_t(j) * g.Y + dst_row] = pv.rng[size_t(j) * pv.Y + src_row];
        }
}

template <typename Word>
__global__ void k_push_signal(const Word* __restrict__ planes, int plane, Geom g, Word* __restrict__ next_planes,
                              uint32_t next_Y, uint64_t* done, uint64_t value) {
    const uint32_t L = g.c1 - g.c0;
    for (uint32_t k = threadIdx.x; k < g.n; k += blockDim.x)
        next_planes[size_t(plane) * size_t(g.n) * next_Y + size_t(k) * next_Y + kStripeHA] =
            planes[size_t(plane) * g.plane_stride + size_t(k) * g.Y + kStripeHA + L];
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(done, value);
    }
}

}  // namespace

cudaError_t launch_halo_pull(int w, void* planes, uint64_t* rng, Geom g, const PeerView& prev, const PeerView& next,
                             uint64_t need, uint32_t* err, bool with_rng, cudaStream_t st) {
    const uint32_t work = 4 * (kStripeHA + kStripeHB) * g.n;
    const uint32_t blocks = std::min<uint32_t>(32, (work + 255) / 256);
    if (w == 64)
        k_halo_pull<uint64_t><<<blocks, 256, 0, st>>>(static_cast<uint64_t*>(planes), rng, g, prev, next, need, err,
                                                       int(with_rng));
    else
        k_halo_pull<uint32_t><<<blocks, 256, 0, st>>>(static_cast<uint32_t*>(planes), rng, g, prev, next, need, err,
                                                       int(with_rng));
    return cudaGetLastError();
}

cudaError_t launch_push_signal(int w, const void* planes, int plane, Geom g, void* next_planes, uint32_t next_Y,
                               uint64_t* done, uint64_t value, cudaStream_t st) {
    if (w == 64)
        k_push_signal<uint64_t><<<1, 256, 0, st>>>(static_cast<const uint64_t*>(planes), plane, g,
                                                   static_cast<uint64_t*>(next_planes), next_Y, done, value);
    else
        k_push_signal<uint32_t><<<1, 256, 0, st>>>(static_cast<const uint32_t*>(planes), plane, g,
                                                   static_cast<uint32_t*>(next_planes), next_Y, done, value);
    return cudaGetLastError();
}

}  // namespace octgpu
