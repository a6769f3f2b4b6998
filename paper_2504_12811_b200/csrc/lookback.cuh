// lookback.cuh — decoupled look-back (single-pass prefix over CTAs taken in ticket order),
// used by the candidate scan (K2), the ordered pair emission (K3) and the onesweep sort (K4).
// A state word packs a 2-bit flag (0 = not ready, 1 = aggregate, 2 = inclusive prefix) over a
// 30-bit value, so one 32-bit store publishes both atomically.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace aaa {

constexpr uint32_t LB_AGG = 1u << 30, LB_PRE = 2u << 30, LB_VAL = (1u << 30) - 1u;

__device__ __forceinline__ void lb_store(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lb_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Called by one full warp. Publishes `local` for CTA `ticket` and returns the exclusive prefix
// of all earlier tickets (to every lane). Warp-parallel window of 32 predecessors.
__device__ __forceinline__ uint32_t lookback_warp(uint32_t* state, uint32_t ticket, uint32_t local) {
    int lane = threadIdx.x & 31;
    if (ticket == 0) {
        if (lane == 0) lb_store(&state[0], LB_PRE | local);
        return 0;
    }
    if (lane == 0) lb_store(&state[ticket], LB_AGG | local);
    uint32_t excl = 0;
    int64_t base = (int64_t)ticket - 1;
    while (true) {
        int64_t idx = base - lane;
        uint32_t v = LB_PRE;
        if (idx >= 0) {
            do {
                v = lb_load(&state[idx]);
            } while ((v & ~LB_VAL) == 0);
        }
        uint32_t pmask = __ballot_sync(0xffffffffu, (v & ~LB_VAL) == LB_PRE);
        if (pmask) {
            int first = __ffs(pmask) - 1;
            excl += warp_sum(lane <= first ? (v & LB_VAL) : 0u);
            break;
        }
        excl += warp_sum(v & LB_VAL);
        base -= 32;
    }
    if (lane == 0) lb_store(&state[ticket], LB_PRE | (excl + local));
    return excl;
}

// Block-wide exclusive scan of one value per thread (blockDim.x <= 1024, multiple of 32).
// Returns the exclusive prefix; *total receives the block sum. `sh` needs 32 words.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* sh, uint32_t* total) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < nw ? sh[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < nw) sh[lane] = s;
    }
    __syncthreads();
    uint32_t warp_excl = w > 0 ? sh[w - 1] : 0u;
    *total = sh[nw - 1];
    __syncthreads();
    return warp_excl + x - v;
}

}  // namespace aaa
