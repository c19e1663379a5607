// A row stripe's pass fused with its device-side halo exchange (the three launches of p2p.cu -- pull, MCS
// kernel, push + signal -- as one): included by the TMA MCS kernels. Same protocol and race argument as
// p2p.cu, refined per block:
//  * a block whose TMA window covers halo rows waits (thread 0, ld.acquire.sys, bounded) for the neighbour on
//    that side to report done >= need, copies the neighbour's boundary core rows of its set P%2 into the local
//    halo rows of the source set, and only then issues its first TMA load (fence.proxy.async: the generic
//    stores must be visible to the async proxy). Interior blocks start at once: their rows overlap the wait.
//  * the blocks that write the first 4 / last 3 core rows (what the neighbours pull next pass) and the block
//    that completes Y(f) of the first halo row below (pushed into the next stripe's new set, whose pass never
//    writes that plane-row) take a ticket when done; the last of them publishes done = value
//    (threadfence.sys + st.release.sys) and resets the ticket.
//  * a neighbour rewrites the set we pulled from only in its next pass, whose boundary blocks first wait for our
//    done >= P; the rows we push are read by the next stripe's block 0 after it waited for the same.
#pragma once
#include <cstdint>

#include "octgpu_internal.h"

namespace octgpu {

__device__ __forceinline__ uint64_t link_ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void link_st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide: wait for the neighbours on the requested sides, then copy their boundary core rows into this
// stripe's halo rows (rows 0..HA-1 from the previous stripe's last HA core rows, rows HA+L.. from the next
// stripe's first HB core rows) of `planes` (the pass's source set). Returns false on a timeout (err set).
template <typename Word>
__device__ bool link_pull(const StripeLink& lk, Word* __restrict__ planes, const Geom& g, bool above, bool below) {
    __shared__ int ok;
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        ok = 1;
        while ((above && link_ld_acquire_sys(lk.prev.done) < lk.need) ||
               (below && link_ld_acquire_sys(lk.next.done) < lk.need)) {
            if (clock64() - t0 > lk.prev.timeout) {
                atomicExch(lk.err, 1u);
                ok = 0;
                break;
            }
            __nanosleep(256);
        }
    }
    __syncthreads();
    if (!ok) return false;
    const uint32_t n = g.n, L = g.c1 - g.c0;
    const uint32_t rows = (above ? kStripeHA : 0u) + (below ? kStripeHB : 0u);
    const uint32_t total = 4 * rows * n;
    for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) {
        const uint32_t p = i / (rows * n), rem = i % (rows * n), r = rem / n, k = rem % n;
        const bool up = above && r < kStripeHA;
        const uint32_t rb = up ? r : r - (above ? kStripeHA : 0u);  // row within its side
        const PeerView& pv = up ? lk.prev : lk.next;
        const uint32_t src_row = up ? pv.L + rb : kStripeHA + rb;
        const uint32_t dst_row = up ? rb : kStripeHA + L + rb;
        const Word* sp = static_cast<const Word*>(pv.planes);
        planes[size_t(p) * g.plane_stride + size_t(k) * g.Y + dst_row] =
            sp[size_t(p) * size_t(n) * pv.Y + size_t(k) * pv.Y + src_row];
    }
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // before this block's TMA
    return true;
}

__device__ __forceinline__ void link_bar(uint32_t nthreads) {
    asm volatile("barrier.sync 2, %0;" ::"r"(nthreads) : "memory");
}

// At the end of a signalling block, by its threads 0..nthreads-1 (the compute warps; a multiple of 32): push (if
// this block completed it) the Y(f) plane-row of the first halo row below into the next stripe's new set, then
// take a ticket; the last of `nsig` blocks publishes done. WHOLE: every thread of the block takes part
// (k_mcs_deep: __syncthreads; a named barrier with a runtime count there cost the live 2-MCS pass a register
// spill in its main loop, 0.249 -> 0.291 ms/MCS)
template <bool WHOLE, typename Word>
__device__ void link_signal(const StripeLink& lk, const Word* __restrict__ dst, const Geom& g, bool push,
                            uint32_t nsig, uint32_t nthreads) {
    if constexpr (WHOLE) {
        nthreads = blockDim.x;
        __syncthreads();
    } else {
        link_bar(nthreads);  // every store of these threads issued (named barrier 2: producers may have exited)
    }
    if (push) {
        const uint32_t L = g.c1 - g.c0;
        Word* np = static_cast<Word*>(lk.next_planes);
        for (uint32_t k = threadIdx.x; k < g.n; k += nthreads)
            np[size_t(lk.push_plane) * size_t(g.n) * lk.next_Y + size_t(k) * lk.next_Y + kStripeHA] =
                dst[size_t(lk.push_plane) * g.plane_stride + size_t(k) * g.Y + kStripeHA + L];
        if constexpr (WHOLE)
            __syncthreads();
        else
            link_bar(nthreads);
    }
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (atomicAdd(lk.ticket, 1u) + 1u == nsig) {
            *lk.ticket = 0;
            __threadfence_system();
            link_st_release_sys(lk.done, lk.value);
        }
    }
}

}  // namespace octgpu
