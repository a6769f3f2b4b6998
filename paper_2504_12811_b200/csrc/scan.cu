// scan.cu — K2: exclusive prefix sum of the per-Gaussian candidate-tile counts (the flattened
// (Gaussian, tile) index space of K3; tile duplication). Single pass, decoupled
// look-back; HBM-bound (8 B per Gaussian).
#include "aaa_internal.cuh"
#include "lookback.cuh"

namespace aaa {

constexpr int SCAN_THREADS = 256, SCAN_ITEMS = 16, SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__global__ void __launch_bounds__(SCAN_THREADS) k_scan(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                       int64_t n, uint32_t* total, uint32_t* state,
                                                       uint32_t* ticket_ctr) {
    __shared__ uint32_t s_items[SCAN_TILE + SCAN_TILE / 32];
    __shared__ uint32_t s_scan[32];
    __shared__ uint32_t s_ticket, s_excl;
    if (threadIdx.x == 0) s_ticket = atomicAdd(ticket_ctr, 1u);
    __syncthreads();
    uint32_t b = s_ticket;
    int64_t start = (int64_t)b * SCAN_TILE;
    // striped coalesced load -> padded smem -> blocked per-thread items
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int i = k * SCAN_THREADS + threadIdx.x;
        int64_t gi = start + i;
        s_items[i + (i >> 5)] = gi < n ? in[gi] : 0u;
    }
    __syncthreads();
    uint32_t v[SCAN_ITEMS], sum = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int i = threadIdx.x * SCAN_ITEMS + k;
        v[k] = s_items[i + (i >> 5)];
        sum += v[k];
    }
    uint32_t btot;
    uint32_t texcl = block_exclusive_scan(sum, s_scan, &btot);
    if (threadIdx.x < 32) {
        uint32_t e = lookback_warp(state, b, btot);
        if (threadIdx.x == 0) s_excl = e;
    }
    __syncthreads();
    uint32_t run = s_excl + texcl;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int i = threadIdx.x * SCAN_ITEMS + k;
        s_items[i + (i >> 5)] = run;
        run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        int i = k * SCAN_THREADS + threadIdx.x;
        int64_t gi = start + i;
        if (gi < n) out[gi] = s_items[i + (i >> 5)];
    }
    if (threadIdx.x == 0 && start + SCAN_TILE >= n) *total = s_excl + btot;
}

size_t scan_state_words(int64_t n) { return (size_t)((n + SCAN_TILE - 1) / SCAN_TILE) + 1; }

void launch_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, uint32_t* state, uint32_t* ticket,
                 cudaStream_t st) {
    if (n == 0) {
        cudaMemsetAsync(total, 0, sizeof(uint32_t), st);
        return;
    }
    unsigned blocks = (unsigned)((n + SCAN_TILE - 1) / SCAN_TILE);
    k_scan<<<blocks, SCAN_THREADS, 0, st>>>(in, out, n, total, state, ticket);
}

}  // namespace aaa
