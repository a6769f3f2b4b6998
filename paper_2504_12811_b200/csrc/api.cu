// api.cu — the C ABI (include/aaa.h): context, scene residency, per-view pipeline driver.
//
// Pipeline per view:
//   compute stream: K1 preprocess -> K2 scan -> K3 cull+emit (candidate count read on the device,
//                   grid over the pair capacity) -> K4 onesweep sort -> K5 ranges -> K6 raster -> K6s
//   (one host synchronisation per call, at its end: views whose candidates outgrew the pair
//   buffers are rendered again with larger ones)
//   copy stream:    (host outputs) D2H of the image, overlapping the next view's kernels
// Every per-view buffer lives in one of two slots used alternately; the events prep_done /
// raster_done of a slot order the two streams. (Running view v+1's K1-K5 concurrently with view
// v's K6 on a second compute stream was measured 1% slower on c3: every stage is latency-bound
// and they only contend.) Both streams are library-owned and non-blocking; the caller's stream is
// joined at entry and exit of each call.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <vector>

#include "aaa_internal.cuh"

#ifndef AAA_SORT_DROP
#define AAA_SORT_DROP 0  // 1: the sort's first pass drops K3's culled candidates (A/B c3: sort 0.216 either way; latency-bound passes)
#endif

using namespace aaa;

cudaError_t aaa::ensure_smem_attr(const void* func, size_t bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, size_t>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(func, dev, bytes);
    if (done.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

namespace {

// all buffers one view in flight needs (the scene is shared by both slots)
struct Slot {
    ViewBufs vb{};
    int64_t vb_n = -1;
    size_t scan_state_cap = 0;
    SortBufs sb{};
    uint32_t pair_cap = 0;
    size_t sort_state_cap = 0;
    uint2* ranges = nullptr;
    uint32_t* tile_order = nullptr;  // K6 tile launch order (longest list first)
    uint4* gdesc = nullptr;          // giant sub-tile descriptors (tiles x 8)
    uint2* gtab = nullptr;           // sub-tile list of every long tile (tiles x 8)
    int ranges_cap = 0;
    SpillHdr* spill_hdr = nullptr;
    float4* spill_e = nullptr;
    size_t spill_cap = 0;
    int spill_k = 0;
    SpillHdr* deep_hdr = nullptr;  // K6s -> K6d queue
    float4* deep_e = nullptr;
    size_t deep_slots = 0;
    int deep_k = 0;
    float* d_out = nullptr;  // staging image for host outputs
    size_t d_out_cap = 0;
    cudaEvent_t prep_done = nullptr, raster_done = nullptr, k6_done = nullptr;
    bool k6_pending = false;  // k6_done has been recorded for this slot's last view
    ViewParams vp{};
    uint32_t C = 0;
    int sorted = 0;
};

}  // namespace

struct aaa_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;             // caller's stream
    cudaStream_t pstream = nullptr, rstream = nullptr;  // compute / image-copy streams
    cudaStream_t kstream = nullptr;  // K6 stream when K1/K2 of the next view overlap K6 (overlap_k1)
    bool overlap_k1 = false;
    cudaEvent_t ev_entry = nullptr, ev_exit = nullptr;
    aaa_config cfg{};
    aaa_camera cam{};
    bool have_cam = false, loaded = false;
    SceneDev scene{};
    Slot slot[2];
    int cur = 0;  // slot of the last view
    uint32_t* h_counters = nullptr;  // pinned
    std::string err;
    // per-view stage events (AAA_FLAG_TIMING): a pool reused across views, read at get_stats
    std::vector<std::vector<cudaEvent_t>> ev_pool;
    size_t ev_used = 0;
    int64_t launches = 0;
    std::vector<uint32_t> h_perm;  // internal -> caller Gaussian index (host copy of scene.perm)
    // backward support (AAA_FLAG_SAVE_CONTRIBS): the last single-view render's blend records
    float2* rec = nullptr;
    size_t rec_cap_px = 0;  // pixels x entries the record buffer holds
    uint32_t rec_cap = 256; // recorded blends per pixel (grown when a render needs more)
    uint32_t* rec_n = nullptr;
    bool saved = false;     // rec holds the render of slot `cur`
    float* bwd_acc = nullptr;
    size_t bwd_acc_cap = 0;
    // tile-band cost model (aaa_render_band / aaa_tile_row_costs): device row difference array
    // per-call overflow words of the views (K3: candidate count above the pair capacity), host copy
    uint32_t* d_ovf = nullptr;
    size_t ovf_cap = 0;
    std::vector<uint32_t> h_ovf;
    uint32_t c_hint = 0;  // pair capacity the last overflow asked for
    unsigned long long* d_rowdiff = nullptr;
    unsigned long long* h_rowdiff = nullptr;  // pinned
    int rowdiff_cap = 0;
    uint32_t* bwd_overflow = nullptr;
};



// compute stream: e0 K1 e1 K2 e2 [sync] e3 K3 e4 sort e5 ranges e6 | e10 K6 e7 K6s e8 | [copy] e9
constexpr int N_EV = 11;

namespace {

aaa_status fail(aaa_ctx* c, aaa_status s, const std::string& m) {
    if (c) c->err = m;
    return s;
}

#define CU(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? AAA_ERR_OOM : AAA_ERR_CUDA,        \
                        std::string(#expr) + ": " + cudaGetErrorString(e_));                      \
    } while (0)

// every entry point that allocates, launches or synchronises first selects the context's device
#define SETDEV(ctx) CU(cudaSetDevice((ctx)->device))

template <typename T>
cudaError_t grow(T*& p, size_t& cap, size_t need) {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    size_t n = need + need / 4 + 256;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    cap = e == cudaSuccess ? n : 0;
    return e;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

aaa_status check_camera(aaa_ctx* ctx, const aaa_camera* c) {
    if (!c) return fail(ctx, AAA_ERR_INVALID_ARG, "camera is null");
    if (c->width < 1 || c->height < 1 || c->width > 65535 || c->height > 65535)
        return fail(ctx, AAA_ERR_INVALID_ARG, "camera width/height out of range");
    if (!(c->fx > 0) || !(c->fy > 0) || !(c->near_z > 0) || !std::isfinite(c->cx) || !std::isfinite(c->cy))
        return fail(ctx, AAA_ERR_INVALID_ARG, "camera fx, fy, near must be > 0 and cx, cy finite");
    const float* M = c->world_to_view;
    for (int i = 0; i < 16; i++)
        if (!std::isfinite(M[i])) return fail(ctx, AAA_ERR_INVALID_ARG, "world_to_view not finite");
    double R[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) R[i][j] = M[4 * i + j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double d = R[i][0] * R[j][0] + R[i][1] * R[j][1] + R[i][2] * R[j][2];
            if (std::fabs(d - (i == j ? 1.0 : 0.0)) > 1e-4)
                return fail(ctx, AAA_ERR_INVALID_ARG, "world_to_view rotation not orthonormal");
        }
    double det = R[0][0] * (R[1][1] * R[2][2] - R[1][2] * R[2][1]) - R[0][1] * (R[1][0] * R[2][2] - R[1][2] * R[2][0]) +
                 R[0][2] * (R[1][0] * R[2][1] - R[1][1] * R[2][0]);
    if (det < 0) return fail(ctx, AAA_ERR_INVALID_ARG, "world_to_view rotation has det -1");
    if (M[12] != 0.f || M[13] != 0.f || M[14] != 0.f || M[15] != 1.f)
        return fail(ctx, AAA_ERR_INVALID_ARG, "world_to_view last row must be (0,0,0,1)");
    return AAA_OK;
}

// Tiles with a list longer than a threshold are rendered pixel by pixel (one warp per pixel, K6s)
// instead of by 8x4 sub-tile warps (K6): on giant lists (c4 zoom-out) a sub-tile warp's serial walk
// is the kernel's critical path. 0 = the automatic threshold (k_tile_order); AAA_GIANT_LIST=N fixes
// it for A/B runs (N = 0: never).
uint32_t giant_list_threshold() {
    static const uint32_t v = [] {
        const char* e = getenv("AAA_GIANT_LIST");
        if (!e) return 0u;
        const uint32_t n = (uint32_t)strtoul(e, nullptr, 10);
        return n ? n : UINT32_MAX;
    }();
    return v;
}

ViewParams make_view(const aaa_ctx* ctx, const aaa_camera& c, int row_begin, int row_end) {
    ViewParams vp{};
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) vp.Rv[3 * i + j] = c.world_to_view[4 * i + j];
        vp.tv[i] = c.world_to_view[4 * i + 3];
    }
    // The camera is the given affine map x_v = Rv x + t (reading 37). Its float32 rotation block is
    // orthonormal only to ~1e-7, so the inverse (camera centre, world -> Gaussian-space ray
    // directions) is the exact 3x3 inverse in FP64, not Rv^T: with |t| ~ 2 and near = 0.01 the
    // transpose shortcut would move z* near the near plane by ~1e-5 relative.
    {
        const double* a = vp.Rv;
        const double c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
        const double det = a[0] * c00 + a[1] * c01 + a[2] * c02, id = 1.0 / det;
        vp.Rvi[0] = c00 * id; vp.Rvi[1] = (a[2] * a[7] - a[1] * a[8]) * id; vp.Rvi[2] = (a[1] * a[5] - a[2] * a[4]) * id;
        vp.Rvi[3] = c01 * id; vp.Rvi[4] = (a[0] * a[8] - a[2] * a[6]) * id; vp.Rvi[5] = (a[2] * a[3] - a[0] * a[5]) * id;
        vp.Rvi[6] = c02 * id; vp.Rvi[7] = (a[1] * a[6] - a[0] * a[7]) * id; vp.Rvi[8] = (a[0] * a[4] - a[1] * a[3]) * id;
    }
    for (int i = 0; i < 3; i++) vp.o[i] = -(vp.Rvi[3 * i] * vp.tv[0] + vp.Rvi[3 * i + 1] * vp.tv[1] + vp.Rvi[3 * i + 2] * vp.tv[2]);
    vp.fx = c.fx; vp.fy = c.fy; vp.cx = c.cx; vp.cy = c.cy; vp.near_z = c.near_z;
    vp.width = c.width; vp.height = c.height;
    vp.tiles_x = (c.width + TILE - 1) / TILE;
    vp.tiles_y = (c.height + TILE - 1) / TILE;
    vp.k = ctx->cfg.k;
    vp.tau_fixed = ctx->cfg.tau_fixed;
    vp.alpha_max = ctx->cfg.alpha_max;
    vp.T_eps = ctx->cfg.T_eps;
    vp.tau_mode = ctx->cfg.tau_mode;
    for (int i = 0; i < 3; i++) vp.bg[i] = ctx->cfg.background[i];
    vp.flags = ctx->cfg.flags;
    vp.sh_degree = ctx->scene.sh_degree;
    // 32-bit sort key: tile bits + log-depth code bits (see aaa_internal.cuh)
    int tb = 0;
    while ((1u << tb) <= (uint32_t)(vp.tiles_x * vp.tiles_y)) tb++;  // tile ids < 2^tb - 1: SKEY_NONE is never a key
    vp.key_db = std::min(KEY_BITS - tb, 28);
    vp.key_scale = std::ldexp(1.0, vp.key_db) / KEY_LOG_RANGE;
    float nl = (float)(c.near_z * (1.0 - 1e-5));
    if ((double)nl > c.near_z * (1.0 - 1e-5)) nl = std::nextafter(nl, 0.f);
    vp.key_near_f = nl;
    vp.key_near = (double)nl;
    float is = (float)(1.0 / vp.key_scale);
    if ((double)is > 1.0 / vp.key_scale) is = std::nextafter(is, 0.f);
    vp.key_inv_scale_f = is;
    vp.inv_fx = 1.0 / vp.fx;
    vp.inv_fy = 1.0 / vp.fy;
    vp.key_zmul = (1.0 - ZKEY_PAD) / vp.key_near;
    vp.giant_list = (ctx->cfg.flags & AAA_FLAG_FORCE_GIANT) ? 1u : giant_list_threshold();
    set_rows(vp, row_begin, row_end);
    return vp;
}

void free_slot(Slot& s) {
    ViewBufs& vb = s.vb;
    cudaFree(vb.cull); cudaFree(vb.raster); cudaFree(vb.color); cudaFree(vb.counts); cudaFree(vb.offsets);
    cudaFree(vb.cross); cudaFree(vb.dbg); cudaFree(vb.counters); cudaFree(vb.scan_state);
    for (int i = 0; i < 2; i++) cudaFree(s.sb.keys[i]);  // keys and vals share one allocation
    cudaFree(s.sb.hist); cudaFree(s.sb.state); cudaFree(s.sb.tickets);
    cudaFree(s.ranges); cudaFree(s.tile_order); cudaFree(s.gdesc); cudaFree(s.gtab); cudaFree(s.spill_hdr); cudaFree(s.spill_e); cudaFree(s.deep_hdr); cudaFree(s.deep_e);
    cudaFree(s.d_out);
    if (s.prep_done) cudaEventDestroy(s.prep_done);
    if (s.raster_done) cudaEventDestroy(s.raster_done);
    if (s.k6_done) cudaEventDestroy(s.k6_done);
    s = Slot{};
}

aaa_status ensure_view_bufs(aaa_ctx* ctx, Slot& sl, int64_t n) {
    if (sl.vb_n >= n && sl.vb.counters) return AAA_OK;
    ViewBufs& vb = sl.vb;
    cudaFree(vb.cull); cudaFree(vb.raster); cudaFree(vb.color); cudaFree(vb.counts); cudaFree(vb.offsets);
    cudaFree(vb.cross); cudaFree(vb.dbg); cudaFree(vb.counters);
    uint32_t* keep_state = vb.scan_state;
    vb = ViewBufs{};
    vb.scan_state = keep_state;
    size_t m = (size_t)(n > 0 ? n : 1);
    CU(cudaMalloc(&vb.cull, m * sizeof(CullRec)));
    CU(cudaMalloc(&vb.raster, m * RASTER_REC_F4 * sizeof(float4)));
    CU(cudaMalloc(&vb.color, m * sizeof(float4)));
    CU(cudaMalloc(&vb.counts, m * sizeof(uint32_t)));
    CU(cudaMalloc(&vb.offsets, m * sizeof(uint32_t)));
    CU(cudaMalloc(&vb.cross, m * sizeof(CrossRec)));
    CU(cudaMalloc(&vb.counters, CNT_TOTAL * sizeof(uint32_t)));
    CU(cudaMemset(vb.counters, 0, CNT_TOTAL * sizeof(uint32_t)));
    sl.vb_n = n;
    return AAA_OK;
}

aaa_status ensure_tiles(aaa_ctx* ctx, Slot& sl, int n_tiles) {
    if (n_tiles <= sl.ranges_cap) return AAA_OK;
    cudaFree(sl.ranges);
    cudaFree(sl.tile_order);
    cudaFree(sl.gdesc);
    cudaFree(sl.gtab);
    sl.ranges = nullptr;
    sl.tile_order = nullptr;
    sl.gdesc = nullptr;
    sl.gtab = nullptr;
    CU(cudaMalloc(&sl.ranges, (size_t)n_tiles * sizeof(uint2)));
    CU(cudaMalloc(&sl.tile_order, (size_t)n_tiles * sizeof(uint32_t)));
    CU(cudaMalloc(&sl.gdesc, (size_t)n_tiles * 8 * sizeof(uint4)));  // giant sub-tile descriptors
    CU(cudaMalloc(&sl.gtab, (size_t)n_tiles * 8 * sizeof(uint2)));   // long tiles' sub-tile lists
    sl.ranges_cap = n_tiles;
    return AAA_OK;
}

// Spill slots for pixels whose K6 window fills: one per pixel up to 4M per view (beyond that a
// pixel is counted as unresolved by aaa_get_stats), each holding the window's K entries.
constexpr size_t MAX_SPILL = (size_t)1 << 22;
// Deep queue: pixels whose K6s pending set outgrows its AAA_SP_CAP_LVL1 entries (none on c1-c5 so
// far; beyond the queue's slots a pixel is counted as unresolved). AAA_FLAG_FORCE_DEEP (K6s limit
// 32) uses a wider, shallower queue.
constexpr size_t DEEP_SLOTS = 4096, DEEP_SLOTS_FORCED = (size_t)1 << 18;

aaa_status ensure_deep(aaa_ctx* ctx, Slot& sl, bool forced) {
    const size_t slots = forced ? DEEP_SLOTS_FORCED : DEEP_SLOTS;
    const int k = forced ? 32 : AAA_SP_CAP_LVL1;
    if (sl.deep_hdr && sl.deep_slots == slots && sl.deep_k == k) return AAA_OK;
    cudaFree(sl.deep_hdr);
    cudaFree(sl.deep_e);
    sl.deep_hdr = nullptr;
    sl.deep_e = nullptr;
    sl.deep_slots = 0;
    CU(cudaMalloc(&sl.deep_hdr, slots * sizeof(SpillHdr)));
    CU(cudaMalloc(&sl.deep_e, slots * (size_t)k * sizeof(float4)));
    sl.deep_slots = slots;
    sl.deep_k = k;
    return AAA_OK;
}

aaa_status ensure_spill(aaa_ctx* ctx, Slot& sl, size_t pixels, int k) {
    size_t cap = std::min(pixels, MAX_SPILL);
    if (cap <= sl.spill_cap && k <= sl.spill_k) return AAA_OK;
    cudaFree(sl.spill_hdr);
    cudaFree(sl.spill_e);
    sl.spill_hdr = nullptr;
    sl.spill_e = nullptr;
    sl.spill_cap = 0;
    CU(cudaMalloc(&sl.spill_hdr, cap * sizeof(SpillHdr)));
    CU(cudaMalloc(&sl.spill_e, cap * (size_t)k * sizeof(float4)));
    sl.spill_cap = cap;
    sl.spill_k = k;
    return AAA_OK;
}

aaa_status ensure_pairs(aaa_ctx* ctx, Slot& sl, uint32_t C) {
    if (C > sl.pair_cap || !sl.sb.keys[0]) {
        for (int i = 0; i < 2; i++) {
            cudaFree(sl.sb.keys[i]);  // keys and vals of a ping-pong side share one allocation
            sl.sb.keys[i] = nullptr;
            sl.sb.vals[i] = nullptr;
        }
        uint32_t cap = C + C / 4 + 4096;
        for (int i = 0; i < 2; i++) {
            // one contiguous 2 x cap words per side: after the sort the free side is K6's giant
            // sub-tile list buffer (RasterArgs::gsub)
            CU(cudaMalloc(&sl.sb.keys[i], (size_t)cap * (sizeof(skey_t) + sizeof(uint32_t))));
            sl.sb.vals[i] = reinterpret_cast<uint32_t*>(sl.sb.keys[i] + cap);
        }
        sl.pair_cap = cap;
        if (!sl.sb.hist) CU(cudaMalloc(&sl.sb.hist, 256 * 8 * sizeof(uint32_t)));
        if (!sl.sb.tickets) CU(cudaMalloc(&sl.sb.tickets, 8 * sizeof(uint32_t)));
    }
    size_t need = sort_state_words(sl.pair_cap, 8);
    CU(grow(sl.sb.state, sl.sort_state_cap, need));
    // K2/K3 look-back state shares one buffer (K2 has finished when this grows)
    size_t sneed = scan_state_words(sl.vb_n) + (size_t)sl.pair_cap / 2048 + 8;
    CU(grow(sl.vb.scan_state, sl.scan_state_cap, sneed));
    return AAA_OK;
}

aaa_status ensure_out(aaa_ctx* ctx, Slot& sl, size_t floats) {
    CU(grow(sl.d_out, sl.d_out_cap, floats));
    return AAA_OK;
}

aaa_status ensure_rowdiff(aaa_ctx* ctx, int rows) {
    if (rows + 1 <= ctx->rowdiff_cap) return AAA_OK;
    cudaFree(ctx->d_rowdiff);
    cudaFreeHost(ctx->h_rowdiff);
    ctx->d_rowdiff = nullptr;
    ctx->h_rowdiff = nullptr;
    ctx->rowdiff_cap = 0;
    CU(cudaMalloc(&ctx->d_rowdiff, (size_t)(rows + 1) * sizeof(unsigned long long)));
    CU(cudaMallocHost(&ctx->h_rowdiff, (size_t)(rows + 1) * sizeof(unsigned long long)));
    ctx->rowdiff_cap = rows + 1;
    return AAA_OK;
}

// per-row band costs (device histogram, one small D2H; syncs ps): the candidate pairs of the slot's
// full-frame K1, or with AAA_BAND_APPROX the projected-disc model of the means and scales (no K1)
aaa_status row_costs(aaa_ctx* ctx, const Slot& sl, const ViewParams& vp, int rows, cudaStream_t ps,
                     std::vector<int64_t>& out) {
    aaa_status s = ensure_rowdiff(ctx, rows);
    if (s) return s;
    if (AAA_BAND_APPROX) launch_row_costs_approx(ctx->scene, vp, rows, ctx->d_rowdiff, ps);
    else launch_row_costs(sl.vb, ctx->scene.n, rows, ctx->d_rowdiff, ps);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(ctx->h_rowdiff, ctx->d_rowdiff, (size_t)(rows + 1) * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, ps));
    CU(cudaStreamSynchronize(ps));
    out.assign(rows, 0);
    int64_t acc = 0;
    for (int r = 0; r < rows; r++) {
        acc += (int64_t)ctx->h_rowdiff[r];
        out[r] = acc;
    }
    return AAA_OK;
}

// contiguous bands of near-equal cost: cut k is the first row whose cost prefix reaches k/world of
// the total (every row also counts 1e-9, so empty rows still split), each band >= 1 row
void split_bands(const std::vector<int64_t>& cost, int world, int32_t* cuts) {
    const int R = (int)cost.size();
    std::vector<double> pref(R + 1, 0.0);
    for (int r = 0; r < R; r++) pref[r + 1] = pref[r] + (double)cost[r] + 1e-9;
    cuts[0] = 0;
    for (int k = 1; k < world; k++) {
        const double target = pref[R] * k / world;
        const int r = (int)(std::lower_bound(pref.begin(), pref.end(), target) - pref.begin());
        cuts[k] = std::min(std::max(r, cuts[k - 1] + 1), R - (world - k));
    }
    cuts[world] = R;
}

// Run the pipeline for one view in slot ctx->cur into device buffers rgb (3 x out_h x W) / T
// (nullptr = the slot's staging image, copied to host_rgb / host_T on the raster stream).
// stop_after: 1 = after K3 (unsorted pairs kept, nothing on the raster stream), 0 = full render.
// band_world > 0: tile-band mode (aaa_render_band): K1 for the whole frame, then this rank's band
// of the cost-balanced split (cuts written to band_cuts).
aaa_status run_view(aaa_ctx* ctx, const aaa_camera& cam, int row_begin, int row_end, float* rgb, float* T,
                    float* host_rgb, float* host_T, bool debug_k1, int stop_after, int band_rank = -1,
                    int band_world = 0, int32_t* band_cuts = nullptr, uint32_t* ovf = nullptr,
                    bool sync_size = false) {
    Slot& sl = ctx->slot[ctx->cur];
    cudaStream_t ps = ctx->pstream, rs = ctx->rstream;
    const int64_t n = ctx->scene.n;
    ViewParams vp = make_view(ctx, cam, row_begin, row_end);
    // the slot's previous view must have left the raster stream before its buffers are reused
    CU(cudaStreamWaitEvent(ps, sl.raster_done, 0));
    aaa_status s = ensure_view_bufs(ctx, sl, n);
    if (s) return s;
    s = ensure_tiles(ctx, sl, vp.tiles_x * vp.tiles_y);
    if (s) return s;
    if (debug_k1 && !sl.vb.dbg)
        CU(cudaMalloc(&sl.vb.dbg, (size_t)(sl.vb_n > 0 ? sl.vb_n : 1) * AAA_DBG_GAUSS_FIELDS * sizeof(double)));  // slot capacity (>= n)
    CU(grow(sl.vb.scan_state, sl.scan_state_cap, scan_state_words(n) + 8));
    const bool timing = (ctx->cfg.flags & AAA_FLAG_TIMING) != 0 && stop_after == 0;
    cudaEvent_t* ev = nullptr;
    if (timing) {
        if (ctx->ev_used == ctx->ev_pool.size()) {
            std::vector<cudaEvent_t> e(N_EV);
            for (int i = 0; i < N_EV; i++) CU(cudaEventCreate(&e[i]));
            ctx->ev_pool.push_back(e);
        }
        ev = ctx->ev_pool[ctx->ev_used++].data();
    }
    auto mark = [&](int i, cudaStream_t st) {
        if (ev) cudaEventRecord(ev[i], st);
    };
    CU(cudaMemsetAsync(sl.vb.counters, 0, CNT_TOTAL * sizeof(uint32_t), ps));
    size_t s2 = scan_state_words(n);
    CU(cudaMemsetAsync(sl.vb.scan_state, 0, s2 * sizeof(uint32_t), ps));
    mark(0, ps);
    if (AAA_BAND_APPROX && band_world > 0) {
        // cut first (model of the means and scales), then K1 for this band only
        std::vector<int64_t> cost;
        s = row_costs(ctx, sl, vp, vp.tiles_y, ps, cost);
        if (s) return s;
        split_bands(cost, band_world, band_cuts);
        row_begin = band_cuts[band_rank];
        row_end = band_cuts[band_rank + 1];
        set_rows(vp, row_begin, row_end);
        if (n > 0) ctx->launches += 1;
    }
    const int k1_launches = launch_preprocess(ctx->scene, vp, sl.vb, debug_k1, ps);
    if (!AAA_BAND_APPROX && band_world > 0) {
        std::vector<int64_t> cost;
        s = row_costs(ctx, sl, vp, vp.tiles_y, ps, cost);
        if (s) return s;
        split_bands(cost, band_world, band_cuts);
        row_begin = band_cuts[band_rank];
        row_end = band_cuts[band_rank + 1];
        set_rows(vp, row_begin, row_end);
        launch_band_clip(sl.vb, n, row_begin, row_end, ps);
        if (n > 0) ctx->launches += 2;
    }
    mark(1, ps);
    if (n > 0) ctx->launches += k1_launches + 1;  // K1 (+ K1c), K2
    launch_scan(sl.vb.counts, sl.vb.offsets, n, &sl.vb.counters[CNT_C], sl.vb.scan_state,
                &sl.vb.counters[CNT_SCAN_TICKET], ps);
    CU(cudaGetLastError());
    mark(2, ps);
    // The pair buffers keep the capacity earlier views needed: K3 and the sort read the candidate
    // count C on the device and size nothing from it on the host, so a view costs no host round
    // trip. The first view of a slot, debug views and re-renders (sync_size) read C back once to
    // size the buffers; a view whose C exceeds the capacity raises *ovf and the call re-renders it
    // after growing them (render_common).
    if (sync_size || sl.pair_cap == 0 || stop_after == 1 || ctx->c_hint > sl.pair_cap) {
        CU(cudaMemcpyAsync(ctx->h_counters, sl.vb.counters, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, ps));
        CU(cudaStreamSynchronize(ps));
        s = ensure_pairs(ctx, sl, std::max(ctx->h_counters[CNT_C], ctx->c_hint));
        if (s) return s;
    }
    const uint32_t cap = sl.pair_cap;
    const int key_bits = KEY_BITS;
    // overlap_k1: K1/K2 of this view ran beside the previous view's K6 (K1 needs registers, K6
    // shared memory, so they share SMs); K3 onwards need the whole GPU and wait for that K6
    Slot& prev = ctx->slot[ctx->cur ^ 1];
    if (ctx->overlap_k1 && prev.k6_pending) CU(cudaStreamWaitEvent(ps, prev.k6_done, 0));
    mark(3, ps);
    // AAA_K3_HIST: K3 accumulates the sort's digit histograms (zeroed here), no histogram pass
    const bool k3_hist = AAA_K3_HIST && !AAA_SORT_DROP && stop_after == 0;
    if (k3_hist) CU(cudaMemsetAsync(sl.sb.hist, 0, sizeof(uint32_t) * 256 * sort_passes(key_bits), ps));
    launch_cull_emit(vp, sl.vb, n, cap, sl.sb.keys[0], sl.sb.vals[0], ovf, ps, k3_hist ? sl.sb.hist : nullptr,
                     sort_passes(key_bits));
    mark(4, ps);
    ctx->launches += 1;
    sl.vp = vp;
    if (stop_after == 1) {
        sl.sorted = 0;
        CU(cudaGetLastError());
        return AAA_OK;
    }
    // sort all min(C, cap) candidates (dense K3 emission: sentinels last, the first P are kept pairs)
    int sorted = launch_sort(sl.sb, &sl.vb.counters[CNT_CCLAMP], cap, key_bits, ps,
                             AAA_SORT_DROP ? &sl.vb.counters[CNT_P] : nullptr, k3_hist);
    sl.sorted = sorted;
    if (ctx->scene.perm && (ctx->cfg.flags & (AAA_FLAG_NO_HIER_SORT | AAA_FLAG_NO_3D))) {
        launch_tie_fix(sl.sb.keys[sorted], sl.sb.vals[sorted], &sl.vb.counters[CNT_P], cap, ctx->scene.perm, ps);
        ctx->launches += 1;
    }
    mark(5, ps);
    launch_ranges(sl.sb.keys[sorted], &sl.vb.counters[CNT_P], cap, sl.ranges, vp.tiles_x * vp.tiles_y, vp.key_db, ps);
    mark(6, ps);
    ctx->launches += (k3_hist ? 2 : 3) + sort_passes(key_bits);  // [histogram,] scan, passes, ranges
    const int out_h = std::min(row_end * TILE, cam.height) - row_begin * TILE;
    const size_t plane = (size_t)out_h * cam.width;
    RasterArgs ra{};
    ra.keys = sl.sb.keys[sorted];
    ra.vals = sl.sb.vals[sorted];
    ra.ranges = sl.ranges;
    ra.tile_order = sl.tile_order;
    ra.raster = sl.vb.raster;
    ra.color = sl.vb.color;
    if (!rgb || (!T && host_T)) {
        s = ensure_out(ctx, sl, 4 * plane);
        if (s) return s;
    }
    ra.out_rgb = rgb ? rgb : sl.d_out;
    ra.out_T = T ? T : (host_T ? sl.d_out + 3 * plane : nullptr);
    ra.out_row0 = row_begin * TILE;
    ra.out_h = out_h;
    const int win_k = (ctx->cfg.flags & AAA_FLAG_FORCE_FALLBACK) ? 1 : ctx->cfg.window_k;
    s = ensure_spill(ctx, sl, (size_t)cam.width * cam.height, std::max(win_k, sl.spill_k));
    if (s) return s;
    ra.spill_hdr = sl.spill_hdr;
    ra.spill_e = sl.spill_e;
    ra.spill_cap = (uint32_t)sl.spill_cap;
    ra.spill_k = (uint32_t)sl.spill_k;
    s = ensure_deep(ctx, sl, (ctx->cfg.flags & AAA_FLAG_FORCE_DEEP) != 0);
    if (s) return s;
    ra.deep_hdr = sl.deep_hdr;
    ra.deep_e = sl.deep_e;
    ra.deep_cap = (uint32_t)sl.deep_slots;
    ra.deep_k = (uint32_t)sl.deep_k;
    ra.counters = sl.vb.counters;
    ra.gdesc = AAA_K6_GSUB ? sl.gdesc : nullptr;
    ra.gtab = (AAA_K6_GSUB && AAA_K6S_SUBL) ? sl.gtab : nullptr;
    ra.gsub = sl.sb.keys[sorted ^ 1];
    ra.gsub_cap = (ctx->cfg.flags & AAA_FLAG_NO_GSUB) ? 0u : 2 * cap;  // 0: every giant pixel walks the full list
    if (ctx->cfg.flags & AAA_FLAG_SAVE_CONTRIBS) {
        const size_t npx = (size_t)cam.width * cam.height;
        if (npx * ctx->rec_cap > ctx->rec_cap_px) {
            cudaFree(ctx->rec);
            cudaFree(ctx->rec_n);
            ctx->rec = nullptr;
            ctx->rec_n = nullptr;
            ctx->rec_cap_px = 0;
            CU(cudaMalloc(&ctx->rec, npx * ctx->rec_cap * sizeof(float2)));
            CU(cudaMalloc(&ctx->rec_n, npx * sizeof(uint32_t) + 16));
            ctx->rec_cap_px = npx * ctx->rec_cap;
        }
        CU(cudaMemsetAsync(ctx->rec_n, 0, npx * sizeof(uint32_t), ps));
        ra.rec = ctx->rec;
        ra.rec_n = ctx->rec_n;
        ra.rec_cap = ctx->rec_cap;
    }
    cudaStream_t ks = ps;
    if (ctx->overlap_k1) {
        ks = ctx->kstream;
        CU(cudaEventRecord(sl.prep_done, ps));
        CU(cudaStreamWaitEvent(ks, sl.prep_done, 0));
    }
    mark(10, ks);
    launch_raster(vp, ra, ctx->cfg.window_k, ks);
    mark(7, ks);
    launch_raster_fallback(vp, ra, ks);
    mark(8, ks);
    if (ctx->overlap_k1) {
        CU(cudaEventRecord(sl.k6_done, ks));
        sl.k6_pending = true;
    }
    if (vp.tile_row_end > vp.tile_row_begin)  // [tile order,] K6, K6s, K6d
        ctx->launches += (ctx->cfg.flags & (AAA_FLAG_NO_3D | AAA_FLAG_NO_HIER_SORT)) ? 3 : 4;
    if (host_rgb || host_T) {
        // image D2H on the copy stream, overlapping the next view's kernels
        CU(cudaEventRecord(sl.prep_done, ks));
        CU(cudaStreamWaitEvent(rs, sl.prep_done, 0));
        if (host_rgb) CU(cudaMemcpyAsync(host_rgb, ra.out_rgb, 3 * plane * sizeof(float), cudaMemcpyDeviceToHost, rs));
        if (host_T) CU(cudaMemcpyAsync(host_T, ra.out_T, plane * sizeof(float), cudaMemcpyDeviceToHost, rs));
        mark(9, rs);
        CU(cudaEventRecord(sl.raster_done, rs));
    } else {
        mark(9, ks);
        CU(cudaEventRecord(sl.raster_done, ks));
    }
    CU(cudaGetLastError());
    return AAA_OK;
}

// join the caller's stream: library streams start after the caller's prior work ...
aaa_status enter(aaa_ctx* ctx) {
    CU(cudaSetDevice(ctx->device));
    CU(cudaEventRecord(ctx->ev_entry, ctx->stream));
    CU(cudaStreamWaitEvent(ctx->pstream, ctx->ev_entry, 0));
    CU(cudaStreamWaitEvent(ctx->rstream, ctx->ev_entry, 0));
    CU(cudaStreamWaitEvent(ctx->kstream, ctx->ev_entry, 0));
    return AAA_OK;
}

// ... and the caller's later work starts after everything the call enqueued
aaa_status leave(aaa_ctx* ctx) {
    CU(cudaEventRecord(ctx->ev_exit, ctx->rstream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_exit, 0));
    CU(cudaEventRecord(ctx->ev_exit, ctx->pstream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_exit, 0));
    CU(cudaEventRecord(ctx->ev_exit, ctx->kstream));
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_exit, 0));
    return AAA_OK;
}

// AAA_WARN_UNRESOLVED when a pixel of the last view could not be finished exactly (spill queue
// full: the pixel holds its partial state); needs the streams synchronised
aaa_status unresolved_status(aaa_ctx* ctx) {
    const Slot& sl = ctx->slot[ctx->cur];
    if (!sl.vb.counters) return AAA_OK;
    uint32_t u = 0;
    CU(cudaMemcpy(&u, &sl.vb.counters[CNT_UNRESOLVED], sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (u) return fail(ctx, AAA_WARN_UNRESOLVED, std::to_string(u) + " pixels unresolved (spill queue full); they hold a partial blend");
    return AAA_OK;
}

aaa_status sync_all(aaa_ctx* ctx) {
    CU(cudaStreamSynchronize(ctx->pstream));
    CU(cudaStreamSynchronize(ctx->rstream));
    CU(cudaStreamSynchronize(ctx->kstream));
    CU(cudaStreamSynchronize(ctx->stream));
    return AAA_OK;
}

aaa_status render_common(aaa_ctx* ctx, const aaa_camera* cams, int n_views, int row_begin, int row_end, float* rgb,
                         float* T, int band_rank = -1, int band_world = 0, int32_t* band_cuts = nullptr) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->loaded) return fail(ctx, AAA_ERR_STATE, "render before aaa_load_gaussians");
    if (!rgb) return fail(ctx, AAA_ERR_INVALID_ARG, "rgb output is null");
    const int W = cams[0].width, H = cams[0].height;
    for (int v = 0; v < n_views; v++) {
        aaa_status s = check_camera(ctx, &cams[v]);
        if (s) return s;
        if (cams[v].width != W || cams[v].height != H)
            return fail(ctx, AAA_ERR_INVALID_ARG, "all views of a batch need the same width/height");
    }
    const int ty = (H + TILE - 1) / TILE;
    if (row_begin < 0 || row_end > ty || row_begin >= row_end)
        return fail(ctx, AAA_ERR_INVALID_ARG, "tile row band out of range");
    const int out_h = std::min(row_end * TILE, H) - row_begin * TILE;
    size_t plane = (size_t)out_h * W;
    const bool dev_rgb = is_device_ptr(rgb);
    const bool dev_T = T ? is_device_ptr(T) : true;
    const bool save = (ctx->cfg.flags & AAA_FLAG_SAVE_CONTRIBS) != 0;
    if (save && (n_views != 1 || row_begin != 0 || row_end != ty || band_world > 0 ||
                 (ctx->cfg.flags & (AAA_FLAG_NO_HIER_SORT | AAA_FLAG_NO_3D))))
        return fail(ctx, AAA_ERR_INVALID_ARG, "AAA_FLAG_SAVE_CONTRIBS needs a single full-image default render");
    ctx->saved = false;
    aaa_status s = enter(ctx);
    if (s) return s;
    if ((size_t)n_views > ctx->ovf_cap) {
        cudaFree(ctx->d_ovf);
        ctx->d_ovf = nullptr;
        ctx->ovf_cap = 0;
        CU(cudaMalloc(&ctx->d_ovf, (size_t)n_views * sizeof(uint32_t)));
        ctx->ovf_cap = (size_t)n_views;
    }
    CU(cudaMemsetAsync(ctx->d_ovf, 0, (size_t)n_views * sizeof(uint32_t), ctx->pstream));
    auto view_ptrs = [&](int v, float*& r, float*& t, float*& hr, float*& ht) {
        r = dev_rgb ? rgb + 3 * plane * v : nullptr;
        t = T && dev_T ? T + plane * v : nullptr;
        hr = dev_rgb ? nullptr : rgb + 3 * plane * v;
        ht = T && !dev_T ? T + plane * v : nullptr;
    };
    for (int v = 0; v < n_views && !s; v++) {
        ctx->cur ^= 1;
        float *r, *t, *hr, *ht;
        view_ptrs(v, r, t, hr, ht);
        s = run_view(ctx, cams[v], row_begin, row_end, r, t, hr, ht, false, 0, band_rank, band_world, band_cuts,
                     ctx->d_ovf + v);
    }
    if (!s) {
        // the call's one host synchronisation: did any view need more pair capacity than its slot
        // had (K3 then covered only part of its candidates)? Those views are rendered again with
        // buffers sized from their own count.
        ctx->h_ovf.resize((size_t)n_views);
        CU(cudaMemcpyAsync(ctx->h_ovf.data(), ctx->d_ovf, (size_t)n_views * sizeof(uint32_t), cudaMemcpyDeviceToHost,
                           ctx->pstream));
        CU(cudaStreamSynchronize(ctx->pstream));
        for (int v = 0; v < n_views && !s; v++) {
            if (!ctx->h_ovf[v]) continue;
            ctx->c_hint = std::max(ctx->c_hint, ctx->h_ovf[v]);
            ctx->cur ^= 1;
            float *r, *t, *hr, *ht;
            view_ptrs(v, r, t, hr, ht);
            s = run_view(ctx, cams[v], row_begin, row_end, r, t, hr, ht, false, 0, band_rank, band_world, band_cuts,
                         nullptr, true);
        }
    }
    if (save && !s) {
        // a pixel that blended more than rec_cap contributions: grow the record and render again
        const size_t npx = (size_t)W * H;
        uint32_t* d_max = ctx->rec_n + npx;  // spare word after the counts
        CU(cudaEventRecord(ctx->ev_exit, ctx->kstream));  // the records come from K6 (kstream)
        CU(cudaStreamWaitEvent(ctx->pstream, ctx->ev_exit, 0));
        CU(cudaMemsetAsync(d_max, 0, sizeof(uint32_t), ctx->pstream));
        launch_max_u32(ctx->rec_n, npx, d_max, ctx->pstream);
        uint32_t mx = 0;
        CU(cudaMemcpyAsync(&mx, d_max, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->pstream));
        CU(cudaStreamSynchronize(ctx->pstream));
        if (mx > ctx->rec_cap) {
            while (ctx->rec_cap < mx) ctx->rec_cap *= 2;
            s = run_view(ctx, cams[0], row_begin, row_end, dev_rgb ? rgb : nullptr, T && dev_T ? T : nullptr,
                         dev_rgb ? nullptr : rgb, T && !dev_T ? T : nullptr, false, 0, -1, 0, nullptr, nullptr, true);
        }
    }
    aaa_status s2 = leave(ctx);
    if (s) return s;
    if (s2) return s2;
    ctx->saved = save;
    if (!dev_rgb || !dev_T) return sync_all(ctx);
    return AAA_OK;
}

// run a view up to K3 (or K1 with the debug record) and wait for it
aaa_status run_debug_view(aaa_ctx* ctx, bool debug_k1) {
    const int ty = (ctx->cam.height + TILE - 1) / TILE;
    aaa_status s = enter(ctx);
    if (s) return s;
    ctx->cur ^= 1;
    ctx->saved = false;
    s = run_view(ctx, ctx->cam, 0, ty, nullptr, nullptr, nullptr, nullptr, debug_k1, 1);
    aaa_status s2 = leave(ctx);
    if (s) return s;
    if (s2) return s2;
    return sync_all(ctx);
}

}  // namespace

extern "C" {

int32_t aaa_version(void) { return 1; }

aaa_status aaa_create(int32_t device, void* stream, aaa_ctx** out) {
    if (!out) return AAA_ERR_INVALID_ARG;
    *out = nullptr;
    aaa_ctx* ctx = new aaa_ctx();
    ctx->device = device;
    ctx->stream = (cudaStream_t)stream;
    aaa_default_config(&ctx->cfg);
    auto bail = [&](cudaError_t e) {
        cudaGetLastError();
        aaa_destroy(ctx);
        return e == cudaErrorMemoryAllocation ? AAA_ERR_OOM : AAA_ERR_CUDA;
    };
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return bail(e);
    if ((e = cudaMallocHost(&ctx->h_counters, CNT_TOTAL * sizeof(uint32_t))) != cudaSuccess) return bail(e);
    int lo = 0, hi = 0;
    if ((e = cudaDeviceGetStreamPriorityRange(&lo, &hi)) != cudaSuccess) return bail(e);
    if ((e = cudaStreamCreateWithPriority(&ctx->pstream, cudaStreamNonBlocking, hi)) != cudaSuccess) return bail(e);
    if ((e = cudaStreamCreateWithPriority(&ctx->rstream, cudaStreamNonBlocking, lo)) != cudaSuccess) return bail(e);
    if ((e = cudaStreamCreateWithPriority(&ctx->kstream, cudaStreamNonBlocking, lo)) != cudaSuccess) return bail(e);
    {
        // off by default: A/B on c3 258.2 -> 258.9 FPS, c2 1581 -> 1623 FPS, but K1 beside K6 slows K6
        // by about what it hides (c3: K6 2.66 -> 3.07 ms measured with K1 inside it), which blurs
        // the per-kernel timings the roofline figures are computed from
        const char* ov = getenv("AAA_OVERLAP_K1");
        ctx->overlap_k1 = ov && ov[0] == '1';
    }
    if ((e = cudaEventCreateWithFlags(&ctx->ev_entry, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    if ((e = cudaEventCreateWithFlags(&ctx->ev_exit, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    for (auto& sl : ctx->slot) {
        if ((e = cudaEventCreateWithFlags(&sl.prep_done, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
        if ((e = cudaEventCreateWithFlags(&sl.raster_done, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
        if ((e = cudaEventCreateWithFlags(&sl.k6_done, cudaEventDisableTiming)) != cudaSuccess) return bail(e);
    }
    *out = ctx;
    return AAA_OK;
}

void aaa_destroy(aaa_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->pstream) cudaStreamSynchronize(ctx->pstream);
    if (ctx->rstream) cudaStreamSynchronize(ctx->rstream);
    if (ctx->kstream) cudaStreamSynchronize(ctx->kstream);
    SceneDev& s = ctx->scene;
    cudaFree(s.geomA); cudaFree(s.geomB); cudaFree(s.geomC); cudaFree(s.sh); cudaFree(s.perm);
    for (auto& sl : ctx->slot) free_slot(sl);
    cudaFree(ctx->rec); cudaFree(ctx->rec_n); cudaFree(ctx->bwd_acc); cudaFree(ctx->bwd_overflow);
    cudaFree(ctx->d_rowdiff);
    if (ctx->h_rowdiff) cudaFreeHost(ctx->h_rowdiff);
    cudaFree(ctx->d_ovf);
    if (ctx->h_counters) cudaFreeHost(ctx->h_counters);
    for (auto& e : ctx->ev_pool)
        for (auto x : e) cudaEventDestroy(x);
    if (ctx->ev_entry) cudaEventDestroy(ctx->ev_entry);
    if (ctx->ev_exit) cudaEventDestroy(ctx->ev_exit);
    if (ctx->pstream) cudaStreamDestroy(ctx->pstream);
    if (ctx->rstream) cudaStreamDestroy(ctx->rstream);
    if (ctx->kstream) cudaStreamDestroy(ctx->kstream);
    delete ctx;
}

aaa_status aaa_set_stream(aaa_ctx* ctx, void* stream) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    ctx->stream = (cudaStream_t)stream;
    return AAA_OK;
}

aaa_status aaa_default_config(aaa_config* c) {
    if (!c) return AAA_ERR_INVALID_ARG;
    c->k = 0.3f;
    c->tau_mode = 0;
    c->tau_fixed = 9.0f;
    c->alpha_max = 0.99f;
    c->T_eps = 1e-4f;
    c->background[0] = c->background[1] = c->background[2] = 0.f;
    c->window_k = 32;
    c->flags = 0;
    return AAA_OK;
}

aaa_status aaa_set_config(aaa_ctx* ctx, const aaa_config* c) {
    if (!ctx || !c) return AAA_ERR_INVALID_ARG;
    if (!(c->k >= 0) || !(c->alpha_max > 0 && c->alpha_max <= 1) || !(c->T_eps >= 0 && c->T_eps < 1) ||
        (c->tau_mode != 0 && c->tau_mode != 1) || (c->tau_mode == 1 && !(c->tau_fixed > 0)) ||
        (c->window_k != 16 && c->window_k != 32))
        return fail(ctx, AAA_ERR_INVALID_ARG, "invalid config (k>=0, 0<alpha_max<=1, 0<=T_eps<1, tau_mode 0/1, window_k 16/32)");
    ctx->cfg = *c;
    return AAA_OK;
}

// Store the validated scene in Morton order of its means (SceneDev::perm): AABB (per-block partial
// min/max, reduced on the host), 30-bit codes, the onesweep sort, one gather per array. The
// caller's index of internal Gaussian i is perm[i]; ctx->h_perm keeps a host copy for the debug
// records.
aaa_status reorder_scene(aaa_ctx* ctx, cudaStream_t st) {
    SceneDev& s = ctx->scene;
    const int64_t n = s.n;
    const int blk = aabb_blocks(n);
    float* d_blk = nullptr;
    CU(cudaMalloc(&d_blk, (size_t)blk * 6 * sizeof(float)));
    launch_aabb(s, d_blk, st);
    std::vector<float> hb((size_t)blk * 6);
    CU(cudaMemcpyAsync(hb.data(), d_blk, hb.size() * sizeof(float), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    cudaFree(d_blk);
    float lh[6] = {hb[0], hb[1], hb[2], hb[3], hb[4], hb[5]};
    for (int b = 1; b < blk; b++)
        for (int k = 0; k < 3; k++) {
            lh[k] = std::min(lh[k], hb[6 * b + k]);
            lh[3 + k] = std::max(lh[3 + k], hb[6 * b + 3 + k]);
        }
    SortBufs sb{};
    uint32_t* d_count = nullptr;
    const uint32_t cap = (uint32_t)n;
    for (int i = 0; i < 2; i++) {
        CU(cudaMalloc(&sb.keys[i], (size_t)cap * sizeof(skey_t)));
        CU(cudaMalloc(&sb.vals[i], (size_t)cap * sizeof(uint32_t)));
    }
    CU(cudaMalloc(&sb.hist, 256 * 8 * sizeof(uint32_t)));
    CU(cudaMalloc(&sb.tickets, 8 * sizeof(uint32_t)));
    CU(cudaMalloc(&sb.state, sort_state_words(cap, 4) * sizeof(uint32_t)));
    CU(cudaMalloc(&d_count, sizeof(uint32_t)));
    CU(cudaMemcpyAsync(d_count, &cap, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    launch_morton_order(s, sb.keys[0], sb.vals[0], lh, st);
    const int cur = launch_sort(sb, d_count, cap, 32, st);
    uint32_t* perm = sb.vals[cur];
    float4 *a2 = nullptr, *b2 = nullptr, *c2 = nullptr, *sh2 = nullptr;
    CU(cudaMalloc(&a2, (size_t)n * sizeof(float4)));
    CU(cudaMalloc(&b2, (size_t)n * sizeof(float4)));
    CU(cudaMalloc(&c2, (size_t)n * sizeof(float4)));
    CU(cudaMalloc(&sh2, (size_t)n * s.sh_chunks * sizeof(float4)));
    launch_permute(s.geomA, a2, perm, n, 1, st);
    launch_permute(s.geomB, b2, perm, n, 1, st);
    launch_permute(s.geomC, c2, perm, n, 1, st);
    launch_permute(s.sh, sh2, perm, n, s.sh_chunks, st);
    CU(cudaGetLastError());
    ctx->h_perm.resize((size_t)n);
    CU(cudaMemcpyAsync(ctx->h_perm.data(), perm, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    cudaFree(s.geomA); cudaFree(s.geomB); cudaFree(s.geomC); cudaFree(s.sh);
    s.geomA = a2; s.geomB = b2; s.geomC = c2; s.sh = sh2;
    s.perm = perm;
    cudaFree(sb.vals[cur ^ 1]);
    for (int i = 0; i < 2; i++) cudaFree(sb.keys[i]);
    cudaFree(sb.hist); cudaFree(sb.tickets); cudaFree(sb.state); cudaFree(d_count);
    return AAA_OK;
}

aaa_status aaa_load_gaussians(aaa_ctx* ctx, const aaa_gaussians* g, int64_t* first_bad) {
    if (!ctx || !g) return AAA_ERR_INVALID_ARG;
    if (first_bad) *first_bad = -1;
    if (g->n < 0 || g->sh_degree < 0 || g->sh_degree > 3)
        return fail(ctx, AAA_ERR_INVALID_ARG, "n must be >= 0 and sh_degree in 0..3");
    if (g->n > 0 && (!g->means || !g->scales || !g->quats || !g->opacities || !g->sh || !g->v_train))
        return fail(ctx, AAA_ERR_INVALID_ARG, "null scene array");
    if (g->n > MAX_GAUSSIANS) return fail(ctx, AAA_ERR_INVALID_ARG, "n too large (<= 2^24 Gaussians per context)");
    CU(cudaSetDevice(ctx->device));
    {
        aaa_status s = sync_all(ctx);  // views in flight still read the old scene
        if (s) return s;
    }
    cudaStream_t st = ctx->stream;
    SceneDev& s = ctx->scene;
    cudaFree(s.geomA); cudaFree(s.geomB); cudaFree(s.geomC); cudaFree(s.sh); cudaFree(s.perm);
    s = SceneDev{};
    ctx->loaded = false;
    ctx->saved = false;
    const int64_t n = g->n;
    const int nf = 3 * (g->sh_degree + 1) * (g->sh_degree + 1);
    s.n = n;
    s.sh_degree = g->sh_degree;
    s.sh_chunks = (nf + 3) / 4;
    size_t m = (size_t)(n > 0 ? n : 1);
    CU(cudaMalloc(&s.geomA, m * sizeof(float4)));
    CU(cudaMalloc(&s.geomB, m * sizeof(float4)));
    CU(cudaMalloc(&s.geomC, m * sizeof(float4)));
    CU(cudaMalloc(&s.sh, m * s.sh_chunks * sizeof(float4)));
    int64_t* d_bad = nullptr;
    CU(cudaMalloc(&d_bad, sizeof(int64_t)));
    int64_t init = INT64_MAX;
    CU(cudaMemcpyAsync(d_bad, &init, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    if (n > 0) {
        const float *dm = g->means, *ds = g->scales, *dq = g->quats, *dop = g->opacities, *dsh = g->sh, *dv = g->v_train;
        float* tmp = nullptr;
        if (!g->device_ptrs) {
            size_t tot = (size_t)n * (3 + 3 + 4 + 1 + nf + 1);
            CU(cudaMalloc(&tmp, tot * sizeof(float)));
            float* p = tmp;
            auto up = [&](const float* src, size_t cnt, const float*& dst) -> cudaError_t {
                cudaError_t e = cudaMemcpyAsync(p, src, cnt * sizeof(float), cudaMemcpyHostToDevice, st);
                dst = p;
                p += cnt;
                return e;
            };
            CU(up(g->means, (size_t)n * 3, dm));
            CU(up(g->scales, (size_t)n * 3, ds));
            CU(up(g->quats, (size_t)n * 4, dq));
            CU(up(g->opacities, (size_t)n, dop));
            CU(up(g->sh, (size_t)n * nf, dsh));
            CU(up(g->v_train, (size_t)n, dv));
        }
        launch_load_pack(*g, dm, ds, dq, dop, dsh, dv, s, d_bad, st);
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(st));
        if (tmp) cudaFree(tmp);
    }
    int64_t bad = INT64_MAX;
    CU(cudaMemcpyAsync(&bad, d_bad, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    cudaFree(d_bad);
    if (bad != INT64_MAX) {
        if (first_bad) *first_bad = bad;
        char msg[160];
        snprintf(msg, sizeof msg,
                 "Gaussian %lld invalid: need finite values, q != 0, s > 0, 0 < o < 1, v_train > 0 (S:113)",
                 (long long)bad);
        return fail(ctx, AAA_ERR_INVALID_GAUSSIAN, msg);
    }
    ctx->h_perm.clear();
#ifndef AAA_NO_REORDER
    if (n > 1) {
        aaa_status rs = reorder_scene(ctx, st);
        if (rs) return rs;
    }
#endif
    ctx->loaded = true;
    return AAA_OK;
}

aaa_status aaa_set_camera(aaa_ctx* ctx, const aaa_camera* cam) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    aaa_status s = check_camera(ctx, cam);
    if (s) return s;
    ctx->cam = *cam;
    ctx->have_cam = true;
    return AAA_OK;
}

aaa_status aaa_render(aaa_ctx* ctx, float* rgb, float* T) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->have_cam) return fail(ctx, AAA_ERR_STATE, "render before aaa_set_camera");
    const int ty = (ctx->cam.height + TILE - 1) / TILE;
    return render_common(ctx, &ctx->cam, 1, 0, ty, rgb, T);
}

aaa_status aaa_render_batch(aaa_ctx* ctx, const aaa_camera* cams, int32_t n_views, float* rgb, float* T) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!cams || n_views < 1) return fail(ctx, AAA_ERR_INVALID_ARG, "need >= 1 camera");
    const int ty = (cams[0].height + TILE - 1) / TILE;
    return render_common(ctx, cams, n_views, 0, ty, rgb, T);
}

aaa_status aaa_render_tiles(aaa_ctx* ctx, int32_t row_begin, int32_t row_end, float* rgb, float* T) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->have_cam) return fail(ctx, AAA_ERR_STATE, "render before aaa_set_camera");
    return render_common(ctx, &ctx->cam, 1, row_begin, row_end, rgb, T);
}

aaa_status aaa_tile_row_costs(aaa_ctx* ctx, int64_t* out, int32_t n_rows) {
    if (!ctx || !out) return AAA_ERR_INVALID_ARG;
    if (!ctx->loaded || !ctx->have_cam) return fail(ctx, AAA_ERR_STATE, "need scene and camera");
    const int ty = (ctx->cam.height + TILE - 1) / TILE;
    if (n_rows < ty) return fail(ctx, AAA_ERR_INVALID_ARG, "n_rows < tile rows");
    aaa_status s = enter(ctx);
    if (s) return s;
    ctx->cur ^= 1;
    ctx->saved = false;
    Slot& sl = ctx->slot[ctx->cur];
    cudaStream_t ps = ctx->pstream;
    CU(cudaStreamWaitEvent(ps, sl.raster_done, 0));
    s = ensure_view_bufs(ctx, sl, ctx->scene.n);
    if (s) return s;
    ViewParams vp = make_view(ctx, ctx->cam, 0, ty);
    CU(cudaMemsetAsync(sl.vb.counters, 0, CNT_TOTAL * sizeof(uint32_t), ps));
    if (!AAA_BAND_APPROX) launch_preprocess(ctx->scene, vp, sl.vb, false, ps);
    sl.vp = vp;
    std::vector<int64_t> cost;
    s = row_costs(ctx, sl, vp, ty, ps, cost);
    if (s) return s;
    CU(cudaEventRecord(sl.raster_done, ps));
    for (int r = 0; r < n_rows; r++) out[r] = r < ty ? cost[r] : 0;
    s = leave(ctx);
    if (s) return s;
    return sync_all(ctx);
}

aaa_status aaa_render_band(aaa_ctx* ctx, int32_t rank, int32_t world, float* rgb, float* T, int32_t* cuts) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->have_cam) return fail(ctx, AAA_ERR_STATE, "render before aaa_set_camera");
    if (!cuts) return fail(ctx, AAA_ERR_INVALID_ARG, "cuts is null");
    const int ty = (ctx->cam.height + TILE - 1) / TILE;
    if (world < 1 || rank < 0 || rank >= world || world > ty)
        return fail(ctx, AAA_ERR_INVALID_ARG, "need 1 <= world <= tile rows and 0 <= rank < world");
    return render_common(ctx, &ctx->cam, 1, 0, ty, rgb, T, rank, world, cuts);
}

aaa_status aaa_compute_vtrain(aaa_ctx* ctx, const aaa_camera* cams, int32_t n_cams, float* out, int32_t store) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->loaded) return fail(ctx, AAA_ERR_STATE, "aaa_compute_vtrain before aaa_load_gaussians");
    if (n_cams < 0 || (n_cams > 0 && !cams)) return fail(ctx, AAA_ERR_INVALID_ARG, "need n_cams >= 0 cameras");
    if (!out && !store) return fail(ctx, AAA_ERR_INVALID_ARG, "out is null and store == 0");
    SETDEV(ctx);
    std::vector<VtCam> h(n_cams > 0 ? n_cams : 1);
    for (int i = 0; i < n_cams; i++) {
        aaa_status s = check_camera(ctx, &cams[i]);
        if (s) return s;
        const aaa_camera& c = cams[i];
        VtCam& v = h[i];
        for (int r = 0; r < 3; r++) {
            for (int k = 0; k < 3; k++) v.R[3 * r + k] = c.world_to_view[4 * r + k];
            v.t[r] = c.world_to_view[4 * r + 3];
        }
        v.fx = c.fx; v.fy = c.fy; v.cx = c.cx; v.cy = c.cy; v.near_z = c.near_z;
        v.f = std::max((double)c.fx, (double)c.fy);
        v.w = c.width; v.h = c.height;
    }
    {
        aaa_status s = sync_all(ctx);  // renders in flight still read v_train
        if (s) return s;
    }
    cudaStream_t st = ctx->stream;
    VtCam* d_cams = nullptr;
    CU(cudaMalloc(&d_cams, h.size() * sizeof(VtCam)));
    CU(cudaMemcpyAsync(d_cams, h.data(), h.size() * sizeof(VtCam), cudaMemcpyHostToDevice, st));
    const size_t bytes = (size_t)ctx->scene.n * sizeof(float);
    const bool dev_out = out && is_device_ptr(out);
    float* d_out = dev_out ? out : nullptr;
    if (out && !dev_out && bytes) CU(cudaMalloc(&d_out, bytes));
    launch_vtrain(ctx->scene, d_cams, n_cams, d_out, store != 0, st);
    if (store) ctx->saved = false;  // a saved render's K1 state no longer matches v_train
    CU(cudaGetLastError());
    if (out && !dev_out && bytes) CU(cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (out && !dev_out) cudaFree(d_out);
    cudaFree(d_cams);
    return AAA_OK;
}

aaa_status aaa_render_backward(aaa_ctx* ctx, const float* dL_drgb, const float* dL_dT, float* d_means,
                               float* d_scales, float* d_quats, float* d_opac, float* d_sh) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    if (!ctx->saved) return fail(ctx, AAA_ERR_STATE, "no render saved with AAA_FLAG_SAVE_CONTRIBS");
    if (!dL_drgb || !d_means || !d_scales || !d_quats || !d_opac || !d_sh)
        return fail(ctx, AAA_ERR_INVALID_ARG, "null pointer");
    SETDEV(ctx);
    const Slot& sl = ctx->slot[ctx->cur];
    const int64_t n = ctx->scene.n;
    CU(grow(ctx->bwd_acc, ctx->bwd_acc_cap, (size_t)(n > 0 ? n : 1) * BWD_ACC));
    if (!ctx->bwd_overflow) CU(cudaMalloc(&ctx->bwd_overflow, sizeof(uint32_t)));
    aaa_status s = enter(ctx);
    if (s) return s;
    cudaStream_t ps = ctx->pstream;
    CU(cudaMemsetAsync(ctx->bwd_overflow, 0, sizeof(uint32_t), ps));
    BwdArgs ba{};
    ba.rec = ctx->rec;
    ba.rec_n = ctx->rec_n;
    ba.rec_cap = ctx->rec_cap;
    ba.dL_drgb = dL_drgb;
    ba.dL_dT = dL_dT;
    ba.raster = sl.vb.raster;
    ba.color = sl.vb.color;
    ba.acc = ctx->bwd_acc;
    ba.overflow = ctx->bwd_overflow;
    ba.d_means = d_means; ba.d_scales = d_scales; ba.d_quats = d_quats; ba.d_opac = d_opac; ba.d_sh = d_sh;
    launch_backward(ctx->scene, sl.vp, ba, ps);
    CU(cudaGetLastError());
    s = leave(ctx);
    if (s) return s;
    s = sync_all(ctx);
    if (s) return s;
    uint32_t ov = 0;
    CU(cudaMemcpy(&ov, ctx->bwd_overflow, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    if (ov) return fail(ctx, AAA_ERR_STATE, std::to_string(ov) + " pixels blended more than 256 contributions");
    return AAA_OK;
}

aaa_status aaa_get_stats(aaa_ctx* ctx, aaa_stats* out) {
    if (!ctx || !out) return AAA_ERR_INVALID_ARG;
    SETDEV(ctx);
    {
        aaa_status s = sync_all(ctx);
        if (s) return s;
    }
    memset(out, 0, sizeof(*out));
    out->n = ctx->scene.n;
    const Slot& sl = ctx->slot[ctx->cur];
    if (!sl.vb.counters) return AAA_OK;
    uint32_t h[CNT_TOTAL];
    CU(cudaMemcpy(h, sl.vb.counters, sizeof(h), cudaMemcpyDeviceToHost));
    out->visible = h[CNT_VISIBLE];
    out->candidates = h[CNT_C];
    out->pairs = h[CNT_P];
    out->spilled_pixels = h[CNT_SPILL];
    out->unresolved_pixels = h[CNT_UNRESOLVED];
    out->crossing = h[CNT_CROSS];
    out->deep_pixels = h[CNT_DEEP];
    out->giant_pixels = h[CNT_GIANT];
    out->evaluations = h[CNT_EVAL];
#ifdef AAA_DEBUG_STATS
    {
        const unsigned long long* u = reinterpret_cast<const unsigned long long*>(&h[20]);
        fprintf(stderr, "[aaa debug] inserts=%llu shifts=%llu far_shifts=%llu sum_cnt=%llu ins_cnt16=%llu k6s_max_pending=%u"
                " k6s_rounds=%u k6s_matched=%u k6s_max_rounds=%u\n",
                u[0], u[1], u[2], u[3], u[4], h[30], h[18], h[19], h[31]);
    }
#endif
    out->launches = ctx->launches;
    // per-stage means over the timed views since the previous call
    // stages: K1, K2, K3, sort, ranges, K6, K6s, host-sync gap, output copy, total
    const int a[10] = {0, 1, 3, 4, 5, 10, 7, 2, 8, 0}, b[10] = {1, 2, 4, 5, 6, 7, 8, 3, 9, 9};
    double acc[10] = {0};
    int64_t nv = 0;
    for (size_t v = 0; v < ctx->ev_used; v++) {
        cudaEvent_t* e = ctx->ev_pool[v].data();
        float t[10];
        bool ok = true;
        for (int i = 0; i < 10; i++) ok = ok && cudaEventElapsedTime(&t[i], e[a[i]], e[b[i]]) == cudaSuccess;
        if (!ok) { cudaGetLastError(); continue; }
        for (int i = 0; i < 10; i++) acc[i] += t[i];
        nv++;
    }
    ctx->ev_used = 0;
    out->timed_views = nv;
    for (int i = 0; i < 10; i++) out->ms[i] = nv ? (float)(acc[i] / nv) : 0.f;
    return out->unresolved_pixels ? fail(ctx, AAA_WARN_UNRESOLVED, std::to_string(out->unresolved_pixels) +
                                                                       " pixels unresolved (spill queue full)")
                                  : AAA_OK;
}

aaa_status aaa_synchronize(aaa_ctx* ctx) {
    if (!ctx) return AAA_ERR_INVALID_ARG;
    SETDEV(ctx);
    aaa_status s = sync_all(ctx);
    if (s) return s;
    return unresolved_status(ctx);
}

aaa_status aaa_debug_copy(aaa_ctx* ctx, int32_t what, void* dst, size_t cap, size_t* len) {
    if (!ctx || !dst || !len) return AAA_ERR_INVALID_ARG;
    if (!ctx->loaded || !ctx->have_cam) return fail(ctx, AAA_ERR_STATE, "need scene and camera");
    SETDEV(ctx);
    aaa_status s = AAA_OK;
    if (what == AAA_DBG_GAUSS || what == AAA_DBG_KEYS_UNSORTED || what == AAA_DBG_VALS_UNSORTED)
        s = run_debug_view(ctx, what == AAA_DBG_GAUSS);
    else if (what >= AAA_DBG_GAUSS && what <= AAA_DBG_COLOR)
        s = sync_all(ctx);
    else
        return fail(ctx, AAA_ERR_INVALID_ARG, "unknown debug buffer");
    if (s) return s;
    const Slot& sl = ctx->slot[ctx->cur];
    if (!sl.vb.counters) return fail(ctx, AAA_ERR_STATE, "no view rendered yet");
    const void* src = nullptr;
    size_t bytes = 0;
    std::vector<unsigned char> dense_tmp;
    uint32_t h[CNT_TOTAL];
    CU(cudaMemcpy(h, sl.vb.counters, sizeof(h), cudaMemcpyDeviceToHost));
    switch (what) {
        case AAA_DBG_GAUSS:
            src = sl.vb.dbg;
            bytes = (size_t)ctx->scene.n * AAA_DBG_GAUSS_FIELDS * sizeof(double);
            break;
        case AAA_DBG_KEYS_UNSORTED:
        case AAA_DBG_VALS_UNSORTED:
            {  // the kept pairs in emission order: compact the candidate array (dense K3 emission)
                const size_t cn = std::min<size_t>(h[CNT_C], sl.pair_cap);
                std::vector<skey_t> k(cn);
                std::vector<uint32_t> v(cn);
                if (cn) {
                    CU(cudaMemcpy(k.data(), sl.sb.keys[0], cn * sizeof(skey_t), cudaMemcpyDeviceToHost));
                    CU(cudaMemcpy(v.data(), sl.sb.vals[0], cn * 4, cudaMemcpyDeviceToHost));
                }
                size_t m = 0;
                for (size_t i = 0; i < cn; i++)
                    if (k[i] != SKEY_NONE) { k[m] = k[i]; v[m] = v[i]; m++; }
                dense_tmp.resize(m * 4);
                if (what == AAA_DBG_KEYS_UNSORTED) memcpy(dense_tmp.data(), k.data(), m * 4);
                else memcpy(dense_tmp.data(), v.data(), m * 4);
                src = nullptr;
                bytes = m * 4;
            }
            break;
        case AAA_DBG_KEYS: src = sl.sb.keys[sl.sorted]; bytes = (size_t)h[CNT_P] * sizeof(skey_t); break;
        case AAA_DBG_VALS: src = sl.sb.vals[sl.sorted]; bytes = (size_t)h[CNT_P] * 4; break;
        case AAA_DBG_RANGES: src = sl.ranges; bytes = (size_t)sl.vp.tiles_x * sl.vp.tiles_y * sizeof(uint2); break;
        case AAA_DBG_SPILL:
            src = sl.spill_hdr;
            bytes = (size_t)std::min((size_t)h[CNT_SPILL], sl.spill_cap) * sizeof(SpillHdr);
            break;
        case AAA_DBG_RASTER: src = sl.vb.raster; bytes = (size_t)ctx->scene.n * RASTER_REC_F4 * sizeof(float4); break;
        case AAA_DBG_COLOR: src = sl.vb.color; bytes = (size_t)ctx->scene.n * sizeof(float4); break;
    }
    *len = bytes;
    if (bytes > cap) return fail(ctx, AAA_ERR_INVALID_ARG, "debug buffer too small");
    if (bytes && src) CU(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    if (bytes && !src) memcpy(dst, dense_tmp.data(), bytes);
    // records and indices in the caller's Gaussian order (the scene is stored in Morton order)
    const std::vector<uint32_t>& pm = ctx->h_perm;
    if (bytes && !pm.empty()) {
        if (what == AAA_DBG_GAUSS || what == AAA_DBG_RASTER || what == AAA_DBG_COLOR) {
            const size_t row = bytes / (size_t)ctx->scene.n;
            std::vector<unsigned char> tmp(bytes);
            const unsigned char* in = static_cast<const unsigned char*>(dst);
            for (size_t i = 0; i < (size_t)ctx->scene.n; i++) memcpy(&tmp[(size_t)pm[i] * row], in + i * row, row);
            memcpy(dst, tmp.data(), bytes);
        } else if (what == AAA_DBG_VALS || what == AAA_DBG_VALS_UNSORTED) {
            uint32_t* v = static_cast<uint32_t*>(dst);
            for (size_t i = 0; i < bytes / 4; i++) v[i] = (v[i] & ~VAL_INDEX_MASK) | pm[v[i] & VAL_INDEX_MASK];
        }
    }
    return AAA_OK;
}

const char* aaa_last_error(const aaa_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

}  // extern "C"
