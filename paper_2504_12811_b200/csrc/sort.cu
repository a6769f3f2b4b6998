// sort.cu — K4: stable LSD onesweep radix sort of the (tile, depth) keys with their Gaussian
// indices, and K5: per-tile [start, end) ranges of the sorted list.
//
// The paper does not name its sort; the global (tile, depth) order is the
// first level of the hierarchical re-sort. Design (B200, HBM-bound):
//  * one upfront histogram pass computes the 256-bin digit histograms of every pass at once
//    (reads 8 B per key once);
//  * each digit pass is one kernel: a CTA ranks 4096 keys with warp-level multisplit
//    (match.any + popc, stable within the warp), publishes its per-digit counts with a
//    decoupled look-back over CTAs taken in ticket order, reorders the keys in shared memory
//    and writes digit runs (reads 12 B, writes 12 B per key per pass).
// Keys are 32-bit (tile << key_db | log-depth code, see aaa_internal.cuh): 4 passes of 8-bit digits.
#include "aaa_internal.cuh"
#include "lookback.cuh"

namespace aaa {

#ifndef AAA_SORT_ITEMS
#define AAA_SORT_ITEMS 20  // A/B on c3: 12 -> 0.252, 16 -> 0.242, 20 -> 0.232 ms
#endif
#ifndef AAA_SORT_MINB
#define AAA_SORT_MINB 3  // 80 registers, 3 CTAs per SM (A/B on c3: 1 -> 0.25-0.35 ms, 3 -> 0.215 ms)
#endif
constexpr int SORT_THREADS = 256, SORT_ITEMS = AAA_SORT_ITEMS, SORT_TILE = SORT_THREADS * SORT_ITEMS, SORT_WARPS = 8;
constexpr int MAX_PASSES = 8;

int sort_passes(int key_bits) { return (key_bits + 7) / 8; }

size_t sort_state_words(uint32_t cap, int passes) {
    size_t blocks = (cap + SORT_TILE - 1) / SORT_TILE + 1;
    return (size_t)passes * blocks * 256;
}

__global__ void __launch_bounds__(256) k_sort_hist(const skey_t* __restrict__ keys, const uint32_t* d_count,
                                                    int passes, uint32_t* hist, bool drop) {
    __shared__ uint32_t sh[MAX_PASSES * 256];
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t P = *d_count;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        skey_t k = keys[i];
        if (drop && k == SKEY_NONE) continue;
        for (int p = 0; p < passes; p++) atomicAdd(&sh[p * 256 + ((k >> (8 * p)) & 0xFF)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// exclusive scan of each pass's 256-bin histogram, in place (one CTA of 256 threads per pass)
__global__ void k_sort_hist_scan(uint32_t* hist) {
    __shared__ uint32_t s_scan[32];
    uint32_t* h = hist + blockIdx.x * 256;
    uint32_t v = h[threadIdx.x], tot;
    uint32_t e = block_exclusive_scan(v, s_scan, &tot);
    h[threadIdx.x] = e;
}

__global__ void __launch_bounds__(SORT_THREADS, AAA_SORT_MINB) k_onesweep(const skey_t* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           skey_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           const uint32_t* d_count, int shift,
                                                           const uint32_t* __restrict__ digit_base,
                                                           uint32_t* state, uint32_t* ticket_ctr, bool drop) {
    extern __shared__ __align__(16) unsigned char smem[];
    skey_t* s_keys = reinterpret_cast<skey_t*>(smem);                             // SORT_TILE
    uint32_t* s_vals = reinterpret_cast<uint32_t*>(s_keys + SORT_TILE);          // SORT_TILE
    uint32_t* s_whist = s_vals + SORT_TILE;                                      // SORT_WARPS * 256
    uint32_t* s_base = s_whist + SORT_WARPS * 256;                               // 256 (global base per digit)
    uint32_t* s_bin = s_base + 256;                                              // 256 (block-local start)
    uint32_t* s_scan = s_bin + 256;                                              // 32
    uint32_t* s_ticket = s_scan + 32;
    uint32_t* s_nvalid = s_ticket + 1;

    const uint32_t P = *d_count;
    if (threadIdx.x == 0) *s_ticket = atomicAdd(ticket_ctr, 1u);
    for (int i = threadIdx.x; i < SORT_WARPS * 256; i += SORT_THREADS) s_whist[i] = 0;
    __syncthreads();
    const uint32_t b = *s_ticket;
    const uint64_t start = (uint64_t)b * SORT_TILE;
    if (start >= P) return;  // no later ticket looks back past the last real block
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;

    skey_t k[SORT_ITEMS];
    uint32_t v[SORT_ITEMS];
    uint32_t rank[SORT_ITEMS];
    // warp w owns the contiguous segment [w*512, w*512+512) of the tile, round r covers 32 keys
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; r++) {
        uint64_t idx = start + w * (SORT_ITEMS * 32) + r * 32 + lane;
        bool valid = idx < P;
        k[r] = valid ? kin[idx] : ~0u;
        v[r] = valid ? vin[idx] : 0u;
    }
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; r++) {
        uint64_t idx = start + w * (SORT_ITEMS * 32) + r * 32 + lane;
        bool valid = idx < P && !(drop && k[r] == SKEY_NONE);  // drop: culled candidates leave here
        uint32_t d = valid ? (uint32_t)((k[r] >> shift) & 0xFF) : (0x100u | lane);
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t prev = valid ? s_whist[w * 256 + d] : 0u;
        __syncwarp();
        if (valid && (peers & lt_mask) == 0) s_whist[w * 256 + d] = prev + __popc(peers);
        __syncwarp();
        rank[r] = prev + __popc(peers & lt_mask);
    }
    __syncthreads();
    // per digit (thread = digit): across-warp exclusive prefix, block total, look-back
    {
        const int d = threadIdx.x;
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < SORT_WARPS; ww++) {
            uint32_t c = s_whist[ww * 256 + d];
            s_whist[ww * 256 + d] = run;
            run += c;
        }
        uint32_t tot;
        uint32_t bin = block_exclusive_scan(run, s_scan, &tot);
        s_bin[d] = bin;
        if (d == 0) *s_nvalid = tot;
        // decoupled look-back for digit d over earlier tickets
        uint32_t* st = state + (size_t)b * 256 + d;
        uint32_t excl = 0;
        if (b == 0) {
            lb_store(st, LB_PRE | run);
        } else {
            lb_store(st, LB_AGG | run);
            int64_t j = (int64_t)b - 1;
            while (j >= 0) {
                uint32_t sv;
                do {
                    sv = lb_load(state + (size_t)j * 256 + d);
                } while ((sv & ~LB_VAL) == 0);
                excl += sv & LB_VAL;
                if ((sv & ~LB_VAL) == LB_PRE) break;
                j--;
            }
            lb_store(st, LB_PRE | (excl + run));
        }
        s_base[d] = digit_base[d] + excl - bin;
    }
    __syncthreads();
    // reorder in shared memory (block-stable order), then write digit runs
#pragma unroll
    for (int r = 0; r < SORT_ITEMS; r++) {
        uint64_t idx = start + w * (SORT_ITEMS * 32) + r * 32 + lane;
        if (idx < P && !(drop && k[r] == SKEY_NONE)) {
            uint32_t d = (uint32_t)((k[r] >> shift) & 0xFF);
            uint32_t pos = s_bin[d] + s_whist[w * 256 + d] + rank[r];
            s_keys[pos] = k[r];
            s_vals[pos] = v[r];
        }
    }
    __syncthreads();
    const uint32_t nvalid = *s_nvalid;
    for (uint32_t i = threadIdx.x; i < nvalid; i += SORT_THREADS) {
        skey_t key = s_keys[i];
        uint32_t d = (uint32_t)((key >> shift) & 0xFF);
        uint32_t o = s_base[d] + i;
        kout[o] = key;
        vout[o] = s_vals[i];
    }
}

static size_t onesweep_smem() {
    return (size_t)SORT_TILE * (sizeof(skey_t) + 4) + (SORT_WARPS * 256 + 256 + 256 + 32 + 4 + 4) * 4;
}

// d_kept != nullptr: the input holds culled candidates (key SKEY_NONE, K3's dense emission), d_kept
// of the d_count keys are real; the first pass drops the culled ones (they would sort last) and
// the later passes sort only the d_kept real keys.
// hist_ready: the digit histograms were accumulated by K3 (AAA_K3_HIST; hist zeroed before it)
int launch_sort(SortBufs& sb, const uint32_t* d_count, uint32_t cap, int key_bits, cudaStream_t st,
                const uint32_t* d_kept, bool hist_ready) {
    int passes = sort_passes(key_bits);
    if (cap == 0) return 0;
    unsigned blocks = (cap + SORT_TILE - 1) / SORT_TILE;
    size_t per_pass = (size_t)(blocks + 1) * 256;
    if (!hist_ready) cudaMemsetAsync(sb.hist, 0, sizeof(uint32_t) * 256 * passes, st);
    cudaMemsetAsync(sb.state, 0, sizeof(uint32_t) * per_pass * passes, st);
    cudaMemsetAsync(sb.tickets, 0, sizeof(uint32_t) * passes, st);
    unsigned hblocks = min(blocks, 148u * 4u);
    const bool drop = d_kept != nullptr;
    if (!hist_ready) k_sort_hist<<<hblocks, 256, 0, st>>>(sb.keys[0], d_count, passes, sb.hist, drop);
    k_sort_hist_scan<<<passes, 256, 0, st>>>(sb.hist);
    if (ensure_smem_attr((const void*)k_onesweep, onesweep_smem()) != cudaSuccess) return 0;
    int cur = 0;
    for (int p = 0; p < passes; p++) {
        k_onesweep<<<blocks, SORT_THREADS, onesweep_smem(), st>>>(sb.keys[cur], sb.vals[cur], sb.keys[cur ^ 1],
                                                                   sb.vals[cur ^ 1], (drop && p > 0) ? d_kept : d_count,
                                                                   8 * p, sb.hist + 256 * p, sb.state + per_pass * p,
                                                                   sb.tickets + p, drop && p == 0);
        cur ^= 1;
    }
    return cur;
}

// Global-order ablations (AAA_FLAG_NO_HIER_SORT / NO_3D): the list order among equal keys is the
// blend order, and its tie rule is the caller's Gaussian index (DESIGN readings). The scene is
// stored in Morton order, so each run of equal keys (short: equal tile and mean-depth code) is
// re-sorted by the caller's index perm[g]; the exact mode needs no fix (its per-pixel order is by
// z*; exact float ties are order-ambiguous by definition, reading 4).
__global__ void k_tie_fix(const skey_t* __restrict__ keys, uint32_t* vals, const uint32_t* d_count,
                          const uint32_t* __restrict__ perm) {
    const uint32_t P = *d_count;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        const skey_t k = keys[i];
        if (i > 0 && keys[i - 1] == k) continue;           // not the start of a run
        if (i + 1 >= P || keys[i + 1] != k) continue;        // run of one
        uint32_t j = i + 1;
        while (j < P && keys[j] == k) j++;
        for (uint32_t a = i + 1; a < j; a++) {                // insertion sort by the caller's index
            const uint32_t v = vals[a], pv = perm[v & VAL_INDEX_MASK];
            uint32_t b = a;
            while (b > i && perm[vals[b - 1] & VAL_INDEX_MASK] > pv) {
                vals[b] = vals[b - 1];
                b--;
            }
            vals[b] = v;
        }
    }
}

void launch_tie_fix(const skey_t* keys, uint32_t* vals, const uint32_t* d_count, uint32_t cap, const uint32_t* perm,
                    cudaStream_t st) {
    if (cap == 0 || !perm) return;
    k_tie_fix<<<min((cap + 255) / 256, 148u * 8u), 256, 0, st>>>(keys, vals, d_count, perm);
}

// ------------------------------------------------------------------ K5: tile ranges
__global__ void k_ranges(const skey_t* __restrict__ keys, const uint32_t* d_count, uint2* ranges, int key_db) {
    uint32_t P = *d_count;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
        uint32_t t = keys[i] >> key_db;
        if (i == 0 || (keys[i - 1] >> key_db) != t) ranges[t].x = i;
        if (i + 1 == P || (keys[i + 1] >> key_db) != t) ranges[t].y = i + 1;
    }
}

void launch_ranges(const skey_t* keys, const uint32_t* d_count, uint32_t cap, uint2* ranges, int n_tiles, int key_db,
                   cudaStream_t st) {
    cudaMemsetAsync(ranges, 0, sizeof(uint2) * n_tiles, st);
    if (cap == 0) return;
    unsigned blocks = min((cap + 255) / 256, 148u * 8u);
    k_ranges<<<blocks, 256, 0, st>>>(keys, d_count, ranges, key_db);
}

}  // namespace aaa
