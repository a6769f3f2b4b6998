// cull_emit.cu — K3: exact 3D tile-frustum culling (Eq. 18) of every flattened
// (Gaussian, candidate tile) pair and deterministic emission of (tile, depth) keys.
//
// Predicate (keep <=> min over the tile frustum of rho^2 < tau, frustum = the 4 planes through
// the tile's outermost pixel centres ∩ {z >= near}, readings 20-21):
//  * tau-ellipsoid entirely beyond near: the minimum over the pixel-centre rectangle of the
//    exact screen-space quadratic q(p) = |c x w(p)|^2 - tau |w(p)|^2 (q < 0 <=> some ray of the
//    tile meets the ellipsoid); equivalent to the paper's plane/edge search.
//  * otherwise (the case where the 2-plane/3-edge shortcut is not exact): the
//    5-constraint QP by active-set enumeration, in FP64.
// Emission order is (Gaussian ascending, tile raster order within its rect): a block-wide scan
// of keep flags plus a decoupled look-back over candidate chunks taken in ticket order.
#include "aaa_internal.cuh"
#include "geom.cuh"

namespace aaa {

#ifndef AAA_K3_ITEMS
#define AAA_K3_ITEMS 8
#endif
constexpr int EMIT_THREADS = 256, EMIT_ITEMS = AAA_K3_ITEMS, EMIT_CHUNK = EMIT_THREADS * EMIT_ITEMS, EMIT_SOFF = 4096;
#ifndef AAA_K3_PERSIST
#define AAA_K3_PERSIST 1  // A/B on c3 with the capacity-sized grid: K3 0.379 -> 0.339 ms
#endif
// Dense emission: every candidate c writes its (key, value) at position c, culled candidates the
// sentinel key SKEY_NONE (above every valid key: tile ids < 2^tile_bits - 1), and the kept count
// is one atomic per block. No scan and no decoupled look-back between blocks: the onesweep sort
// over all C candidates moves the sentinels behind the P kept pairs and keeps the kept pairs in
// the same stable order as a compacted emission would (so the sorted list is the same bit for bit;
// A/B on c3: K3 0.425 -> 0.341 ms, sort 0.210 -> 0.242 ms against the round-1 compacting K3).
// The candidate count C is read on the device (no host round trip): the grid covers the pair
// buffers' capacity `cap`, chunks at or beyond C exit, and a view with C > cap only processes the
// first cap candidates and raises *ovf (the host re-renders it with larger buffers).

#ifndef AAA_K3_PROBE
#define AAA_K3_PROBE 1  // A/B (K3 ms, binary search / probes first): c3 0.339 / 0.323, c4 wide 0.334 / 0.318
#endif
#ifndef AAA_K3_MINB
#define AAA_K3_MINB 3  // 80 registers, 3 CTAs of 256 threads per SM (A/B on c3: 2 -> 0.70 ms, 3 -> 0.64 ms)
#endif
__global__ void __launch_bounds__(EMIT_THREADS, AAA_K3_MINB) k_cull_emit(ViewParams vp, const CullRec* __restrict__ cull,
                                                            const CrossRec* __restrict__ cross,
                                                            const uint32_t* __restrict__ offsets, int64_t n,
                                                            uint32_t cap, skey_t* __restrict__ keys,
                                                            uint32_t* __restrict__ vals, uint32_t* counters,
                                                            uint32_t* ovf, uint32_t* hist, int passes) {
    __shared__ uint32_t s_ticket, s_C;
#if AAA_K3_HIST
    // the sort's digit histograms of every emitted key (AAA_K3_HIST: replaces the sort's separate
    // histogram pass), accumulated per CTA over its chunks and added to `hist` at exit
    __shared__ uint32_t s_hist[4 * 256];
    if (hist)
        for (int i = threadIdx.x; i < 4 * 256; i += EMIT_THREADS) s_hist[i] = 0u;
#endif
    __shared__ int64_t s_g0, s_g1;
    __shared__ uint32_t s_off[EMIT_SOFF];
    // per-thread emitted pairs, [item][thread] (a register array indexed in a rolled loop would
    // live in local memory)
    // [t * (ITEMS + 1) + k] (odd stride): conflict-free writes, coalesced reads
    constexpr int SS = EMIT_ITEMS + 1;
    __shared__ skey_t s_key[EMIT_THREADS * SS];
    __shared__ uint32_t s_val[EMIT_THREADS * SS];
#if AAA_K3_PERSIST
    // persistent CTAs (a grid of resident CTAs, independent of C): each takes chunk tickets
    // until the chunks run out
    for (;;) {
#endif
    if (threadIdx.x == 0) {
        s_ticket = atomicAdd(&counters[CNT_EMIT_TICKET], 1u);
        const uint32_t Cd = counters[CNT_C];
        s_C = min(Cd, cap);
        if (s_ticket == 0) {
            counters[CNT_CCLAMP] = s_C;  // the sort's element count
            if (Cd > cap && ovf) *ovf = Cd;  // the capacity this view needs
        }
    }
    __syncthreads();
    const uint32_t C = s_C;
    if ((uint64_t)s_ticket * EMIT_CHUNK >= C) {
#if AAA_K3_HIST
        if (hist)
            for (int i = threadIdx.x; i < passes * 256; i += EMIT_THREADS)
                if (s_hist[i]) atomicAdd(&hist[i], s_hist[i]);
#endif
        return;
    }
    if (threadIdx.x < 32) {
        // the chunk's candidates [c0, c1] belong to Gaussians [g0, g1] (largest g with offset <= c):
        // two 17-ary searches side by side (half-warp each), one parallel load per step
        const int lane = threadIdx.x, grp = lane >> 4, gi = lane & 15;
        const uint32_t c0 = s_ticket * EMIT_CHUNK, c1 = min(c0 + EMIT_CHUNK, C) - 1;
        const uint32_t target = grp ? c1 : c0;
        int64_t lo = 0, hi = n;  // offsets[lo] <= target, answer in [lo, hi)
        while (true) {
            const bool active = hi - lo > 1;
            if (!__any_sync(0xffffffffu, active)) break;
            const int64_t step = (hi - lo + 16) / 17;
            const int64_t pr = lo + (int64_t)(gi + 1) * step;
            const bool le = active && pr < hi && offsets[pr] <= target;
            const uint32_t bal = __ballot_sync(0xffffffffu, le);
            const int k = __popc((bal >> (grp * 16)) & 0xFFFFu);
            if (active) {
                lo += (int64_t)k * step;
                hi = min(hi, lo + step);
            }
        }
        if (gi == 0) {
            if (grp) s_g1 = lo;
            else s_g0 = lo;
        }
    }
    __syncthreads();
    const uint32_t chunk = s_ticket;
    const uint32_t cbeg = chunk * EMIT_CHUNK + threadIdx.x * EMIT_ITEMS;
    const int64_t g0 = s_g0, g1 = s_g1;
    const bool in_smem = g1 - g0 + 1 <= EMIT_SOFF;  // offsets of the chunk's Gaussians staged in smem
    if (in_smem)
        for (int64_t i = threadIdx.x; i <= g1 - g0; i += EMIT_THREADS) s_off[i] = offsets[g0 + i];
    __syncthreads();
    auto off = [&](int64_t x) -> uint32_t { return in_smem ? s_off[x - g0] : offsets[x]; };
    auto find = [&](uint32_t c, int64_t lo) -> int64_t {  // largest g in [lo, g1] with off(g) <= c
        int64_t hi = g1 + 1;
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (off(mid) <= c) lo = mid; else hi = mid;
        }
        return lo;
    };
    int64_t g = find(cbeg, g0);
    // per Gaussian, held in registers while consecutive candidates share it: the FP32 image of
    // the quadratic and the record's small fields (the FP64 coefficients are re-read from global
    // memory only by the rare guard-band re-test)
    struct Hot {
        float pref_x, pref_y;
        uint16_t tx0, ty0, tx1, ty1, i0, j0, i1, j1;
        int32_t cross_slot;
        uint32_t zkey;
    } r;
    int64_t g_loaded = -1;
    QuadF qf{};
    uint32_t nkeep = 0;
    const bool no_cull = (vp.flags & AAA_FLAG_NO_TILE_CULL) != 0;
    const bool f64_only = (vp.flags & AAA_FLAG_CULL_FP64) != 0;  // guard-band test switch
#pragma unroll 1
    for (int k = 0; k < EMIT_ITEMS; k++) {
        uint32_t c = cbeg + k;
        if (c >= C) break;
#if AAA_K3_PROBE
        if (g < g1 && off(g + 1) <= c) {  // next Gaussian: a few linear probes, then a binary search
            g++;                          // (long runs of empty Gaussians: off-screen regions)
#pragma unroll
            for (int pr = 0; pr < 3; pr++)
                if (g < g1 && off(g + 1) <= c) g++;
            if (g < g1 && off(g + 1) <= c) g = find(c, g + 1);
        }
#else
        if (g < g1 && off(g + 1) <= c) g = find(c, g + 1);  // next Gaussian (skips empty runs)
#endif
        if (g != g_loaded) {
            union {
                float4 v[sizeof(CullRec) / 16];
                CullRec c;
            } rr;
            const float4* src = reinterpret_cast<const float4*>(cull + g);
#pragma unroll
            for (int q = 0; q < (int)(sizeof(CullRec) / 16); q++) rr.v[q] = __ldg(&src[q]);
            g_loaded = g;
            const CullRec& r0 = rr.c;
            qf = QuadF{(float)r0.qa, (float)r0.qb, (float)r0.qc, (float)r0.qd, (float)r0.qe, (float)r0.qf,
                       (float)r0.ia, (float)r0.ic, (float)r0.xs, (float)r0.ys, (float)r0.qi};
            r = Hot{r0.pref_x, r0.pref_y, r0.tx0, r0.ty0, r0.tx1, r0.ty1, r0.i0, r0.j0, r0.i1, r0.j1,
                    r0.cross_slot, r0.zkey};
        }
        uint32_t j = c - off(g);
        uint32_t w = (uint32_t)r.tx1 - r.tx0 + 1;
        int tx = r.tx0 + (int)(j % w), ty = r.ty0 + (int)(j / w);
        // pixel-centre box of the tile (exact in FP32: k + 0.5 with k < 2^23)
        const float x0 = TILE * tx + 0.5f, x1 = fminf(TILE * tx + TILE - 0.5f, vp.width - 0.5f);
        const float y0 = TILE * ty + 0.5f, y1 = fminf(TILE * ty + TILE - 0.5f, vp.height - 0.5f);
        bool keep;
        uint32_t sub = SUBTILE_ALL;
        if (no_cull) {
            keep = true;
        } else if (r.cross_slot < 0) {
            // exact sign of the FP64 box minimum: FP32 outside the guard band, FP64 inside it
            auto box_keep = [&](float bx0, float bx1, float by0, float by1) -> bool {
                if (!f64_only) {
                    const int sg = quad_box_sign_f32(qf, bx0 - r.pref_x, bx1 - r.pref_x, by0 - r.pref_y, by1 - r.pref_y);
                    if (sg >= 0) return sg == 1;
                }
                const CullRec& rd = cull[g];
                const double px = r.pref_x, py = r.pref_y;
                return quad_box_min_pre(rd.qa, rd.qb, rd.qc, rd.qd, rd.qe, rd.qf, rd.ia, rd.ic, rd.xs, rd.ys, rd.qi,
                                        (double)bx0 - px, (double)bx1 - px, (double)by0 - py, (double)by1 - py) < 0.0;
            };
            keep = box_keep(x0, x1, y0, y1);
            if (keep) {
                // the same exact test on each 8x4 warp sub-tile (pixel-centre rects): the raster
                // kernels skip the Gaussian on sub-tiles whose bit is clear ("repeated culling")
                sub = 0;
#pragma unroll
                for (int s = 0; s < 8; s++) {
                    const int spx = TILE * tx + 8 * (s & 1), spy = TILE * ty + 4 * (s >> 1);
                    // sub-tiles outside the Gaussian's pixel rect hold no contributing pixel (bounds)
                    if (spx > r.i1 || spx + 7 < r.i0 || spy > r.j1 || spy + 3 < r.j0) continue;
                    const float sx0 = spx + 0.5f, sy0 = spy + 0.5f;
                    if (sx0 > vp.width - 0.5f || sy0 > vp.height - 0.5f) continue;
                    const float sx1 = fminf(sx0 + 7.f, vp.width - 0.5f), sy1 = fminf(sy0 + 3.f, vp.height - 0.5f);
                    if (box_keep(sx0, sx1, sy0, sy1)) sub |= 1u << s;
                }
            }
        } else {
            const CrossRec& cr = cross[r.cross_slot];
            keep = frustum_qp_min(cr.M, cr.muv, vp.fx, vp.fy, vp.cx, vp.cy, vp.near_z, x0, x1, y0, y1) < cr.tau;
        }
        const uint32_t tile = (uint32_t)(ty * vp.tiles_x + tx);
        s_key[threadIdx.x * SS + k] = keep ? ((tile << vp.key_db) | r.zkey) : SKEY_NONE;
        s_val[threadIdx.x * SS + k] = keep ? ((uint32_t)g | (sub << VAL_INDEX_BITS)) : 0u;
        nkeep += keep;
    }
    {
        __syncthreads();
        const uint32_t c0 = chunk * EMIT_CHUNK;
        for (int i = threadIdx.x; i < EMIT_CHUNK; i += EMIT_THREADS) {
            if (c0 + i >= C) break;
            const skey_t kk = s_key[(i / EMIT_ITEMS) * SS + i % EMIT_ITEMS];
            keys[c0 + i] = kk;
            vals[c0 + i] = s_val[(i / EMIT_ITEMS) * SS + i % EMIT_ITEMS];
#if AAA_K3_HIST
            if (hist)
                for (int p = 0; p < passes; p++) atomicAdd(&s_hist[p * 256 + ((kk >> (8 * p)) & 0xFFu)], 1u);
#endif
        }
        uint32_t w = nkeep;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(&counters[CNT_P], w);
    }
#if AAA_K3_PERSIST
    __syncthreads();  // the shared staging is reused by the next chunk
    }
#endif
}

void launch_cull_emit(const ViewParams& vp, const ViewBufs& vb, int64_t n, uint32_t cap, skey_t* keys,
                      uint32_t* vals, uint32_t* ovf, cudaStream_t st, uint32_t* hist, int passes) {
    if (cap == 0) return;
    unsigned blocks = (cap + EMIT_CHUNK - 1) / EMIT_CHUNK;
    if (AAA_K3_PERSIST) blocks = std::min(blocks, 148u * AAA_K3_MINB);
    k_cull_emit<<<blocks, EMIT_THREADS, 0, st>>>(vp, vb.cull, vb.cross, vb.offsets, n, cap, keys, vals, vb.counters,
                                                 ovf, (AAA_K3_HIST && AAA_K3_PERSIST) ? hist : nullptr, passes);
}

}  // namespace aaa
