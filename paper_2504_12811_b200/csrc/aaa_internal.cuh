// aaa_internal.cuh — device-side layouts and launch entry points shared by the kernels of the
// B200 forward renderer. See DESIGN.md "Data layout in HBM" for sizes.
#pragma once
#include <cmath>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/aaa.h"

namespace aaa {

constexpr int TILE = 16;                // 16x16 pixel tiles (reading 24)
// Sort key (32 bits): tile << key_db | dcode. dcode = floor(S log2(z_lb / near_lo)), a log-depth code
// over KEY_LOG_RANGE octaves above near (S = 2^key_db / KEY_LOG_RANGE codes per octave); its decode
// near_lo 2^(dcode / S) is a lower bound of z_lb, so the key stays a valid depth lower bound.
using skey_t = uint32_t;
constexpr skey_t SKEY_NONE = 0xFFFFFFFFu;  // K3 dense emission: culled candidate (sorts last)
#ifndef AAA_KEY_BITS
#define AAA_KEY_BITS 32  // sort key width: 8-bit radix passes = AAA_KEY_BITS / 8
#endif
#ifndef AAA_KEY_LOG_RANGE
#define AAA_KEY_LOG_RANGE 24.0
#endif
constexpr int KEY_BITS = AAA_KEY_BITS;
constexpr double KEY_LOG_RANGE = AAA_KEY_LOG_RANGE;
constexpr int RASTER_REC_F4 = 7;        // raster record: 7 float4 = 112 B
constexpr float ANGLE_EPS = 1e-4f;      // Eq. 17 epsilon (reading 17)
constexpr double ZKEY_PAD = 1e-5;       // relative downward pad of the depth key (reading 23)
// pair value: Gaussian index (low 24 bits) | 8-bit mask of the 8x4 warp sub-tiles it may touch
constexpr int VAL_INDEX_BITS = 24;
constexpr uint32_t VAL_INDEX_MASK = (1u << VAL_INDEX_BITS) - 1u;
constexpr uint32_t SUBTILE_ALL = 0xFFu;
constexpr int64_t MAX_GAUSSIANS = 1ll << VAL_INDEX_BITS;

// Per-view constants passed by value to every kernel (camera in double for the FP64 geometry).
struct ViewParams {
    double Rv[9];       // world->view rotation (row-major)
    double tv[3];       // world->view translation
    double Rvi[9];      // Rv^-1 (row-major; the exact inverse of the given float32 matrix, reading 37)
    double o[3];        // camera centre in world space, -Rv^-1 tv
    double fx, fy, cx, cy, near_z;
    int width, height;
    int tiles_x, tiles_y;
    int tile_row_begin, tile_row_end;   // band [begin, end) of tile rows to emit
    double fr_norm[4];  // K1 sphere exit: |normal| of the 4 pixel-centre frustum planes (set_rows)
    float k, tau_fixed, alpha_max, T_eps;
    int tau_mode;
    float bg[3];
    uint32_t flags;
    int sh_degree;
    int key_db;            // depth-code bits of the 32-bit key (32 - tile bits)
    double key_scale;      // S: codes per octave
    double key_near;       // near_lo (encode base, = key_near_f promoted)
    float key_inv_scale_f; // 1/S rounded down (decode)
    float key_near_f;      // near_lo rounded down (decode)
    double inv_fx, inv_fy; // 1/fx, 1/fy
    double key_zmul;       // (1 - ZKEY_PAD) / key_near (encode)
    uint32_t giant_list;   // K6: tiles whose list is longer go pixel by pixel to K6s (0 = the automatic
                           // threshold k_tile_order computes; UINT32_MAX = never)
};

// Scene residency (L0): structure of float4 arrays, 16-byte aligned.
// the rendered tile rows of a view and the frustum-plane norms that depend on them (K1's sphere
// exit: sqrt(fx^2 + x0^2) etc., the same expressions K1 used to evaluate per Gaussian)
inline void set_rows(ViewParams& vp, int row_begin, int row_end) {
    vp.tile_row_begin = row_begin;
    vp.tile_row_end = row_end;
    const double x0 = 0.5 - vp.cx, x1 = vp.width - 0.5 - vp.cx;
    const double y0 = TILE * row_begin + 0.5 - vp.cy;
    const double y1 = std::fmin((double)(TILE * row_end), (double)vp.height) - 0.5 - vp.cy;
    vp.fr_norm[0] = std::sqrt(vp.fx * vp.fx + x0 * x0);
    vp.fr_norm[1] = std::sqrt(vp.fx * vp.fx + x1 * x1);
    vp.fr_norm[2] = std::sqrt(vp.fy * vp.fy + y0 * y0);
    vp.fr_norm[3] = std::sqrt(vp.fy * vp.fy + y1 * y1);
}

struct SceneDev {
    int64_t n;
    int sh_degree;
    float4* geomA;   // mu.x, mu.y, mu.z, opacity
    float4* geomB;   // s.x, s.y, s.z, v_train
    float4* geomC;   // q.w, q.x, q.y, q.z (normalised at load)
    float4* sh;      // SoA chunks: sh[c * n + g], c < 3*(deg+1)^2/4 (rounded up); floats in
                     // coefficient-major, channel-minor order
    int sh_chunks;
    // internal -> caller index: the scene is stored in Morton order of the means (aaa_load_gaussians)
    // so that warps and tile lists touch spatially coherent Gaussians; per-Gaussian outputs
    // (gradients, v_train, debug records) are written back in the caller's order through it
    uint32_t* perm;
};

// K3 input per visible Gaussian (128 B): screen-space quadratic q(p) = N(p) - tau Q(p) relative
// to p_ref (exact tile predicate for non-crossing Gaussians, K3) with its per-Gaussian
// box-minimum helpers precomputed (no FP64 division per tile), tile rect, key.
struct __align__(16) CullRec {
    double qa, qb, qc, qd, qe, qf;  // q = qa dx^2 + 2 qb dx dy + qc dy^2 + 2 qd dx + 2 qe dy + qf
    double ia, ic;                  // 1/qa, 1/qc when positive (edge critical points), else 0
    double xs, ys, qi;              // interior critical point and its value (qi = +inf unless PD)
    float pref_x, pref_y;
    uint16_t tx0, ty0, tx1, ty1;    // inclusive tile rect (band-clipped)
    uint16_t i0, j0, i1, j1;        // inclusive pixel rect of the bounds (sub-tile pre-reject)
    int32_t cross_slot;             // >= 0: index into CrossRec (exact QP path); -1 otherwise
    uint32_t zkey;                  // log-depth code of the depth lower bound (reading 23)
};
// the tile rect read as one 16-byte word (x = tx0 | ty0 << 16, y = tx1 | ty1 << 16)
constexpr int CULLREC_RECT_U4 = 6;
static_assert(offsetof(CullRec, tx0) == 16 * CULLREC_RECT_U4 && offsetof(CullRec, tx1) == 16 * CULLREC_RECT_U4 + 4,
              "CullRec rect layout");
static_assert(sizeof(CullRec) == 128, "CullRec is 128 B");

// Gaussians whose tau-ellipsoid reaches z <= near: the exact QP culling path needs T_view.
struct CrossRec {
    double M[9];    // view <- Gaussian-space linear map (row-major), filtered scales
    double muv[3];
    double tau;
    double pad;
};

// Per-view scratch owned by the context.
struct ViewBufs {
    CullRec* cull;        // n
    float4* raster;       // n * RASTER_REC_F4
    float4* color;        // n (rgb, unused)
    uint32_t* counts;     // n candidate tiles per Gaussian
    uint32_t* offsets;    // n exclusive scan
    CrossRec* cross;      // n (worst case)
    double* dbg;          // n * AAA_DBG_GAUSS_FIELDS (only when debugging)
    // device counters: [0] visible, [1] crossing slots, [2] C total, [3] P pairs,
    // [4] spilled pixels (K6 windows that filled), [5] K6s ticket, [6] unresolved pixels,
    // [7] tickets (scratch), [8..15] sort tickets, [16] K3 ticket
    uint32_t* counters;
    uint32_t* scan_state; // decoupled look-back state for the scan / emit / sort
};

// K6s pending-set capacity per pixel (first spill level; the deep level K6d holds 2048)
#ifndef AAA_SP_CAP
#define AAA_SP_CAP 256
#endif
constexpr int AAA_SP_CAP_LVL1 = AAA_SP_CAP;
constexpr int CNT_VISIBLE = 0, CNT_CROSS = 1, CNT_C = 2, CNT_P = 3, CNT_SPILL = 4, CNT_SPILL_TICKET = 5,
              CNT_UNRESOLVED = 6, CNT_SCAN_TICKET = 7, CNT_SORT_TICKET = 8, CNT_EMIT_TICKET = 16, CNT_EVAL = 17,
              CNT_DEEP = 32, CNT_DEEP_TICKET = 33, CNT_GIANT = 34, CNT_GIANT_THR = 35, CNT_CCLAMP = 36, CNT_GDESC = 37,
              CNT_GSUB = 38, CNT_GTICKET = 39, CNT_TOTAL = 40;

// ---- launchers (each file implements its own) ----
void launch_load_pack(const aaa_gaussians& in, const float* dmeans, const float* dscales, const float* dquats,
                      const float* dopac, const float* dsh, const float* dvt, SceneDev& sc, int64_t* d_bad,
                      cudaStream_t st);
int launch_preprocess(const SceneDev& sc, const ViewParams& vp, ViewBufs& vb, bool debug, cudaStream_t st);  // launches
size_t scan_state_words(int64_t n);
void launch_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* total, uint32_t* state, uint32_t* ticket,
                 cudaStream_t st);
// K3 over the first min(C, cap) candidates (C read on the device); raises *ovf when C > cap
void launch_cull_emit(const ViewParams& vp, const ViewBufs& vb, int64_t n, uint32_t cap, skey_t* keys,
                      uint32_t* vals, uint32_t* ovf, cudaStream_t st,
                      uint32_t* hist = nullptr, int passes = 0);
struct SortBufs {
    skey_t* keys[2];
    uint32_t* vals[2];
    uint32_t* hist;        // passes * 256
    uint32_t* state;       // passes * blocks * 256
    uint32_t* tickets;     // passes
    int cap_blocks;
};
int sort_passes(int key_bits);
size_t sort_state_words(uint32_t cap, int passes);
// returns the index (0/1) of the buffer holding the sorted output
int launch_sort(SortBufs& sb, const uint32_t* d_count, uint32_t cap, int key_bits, cudaStream_t st,
                const uint32_t* d_kept = nullptr, bool hist_ready = false);
int sort_passes(int key_bits);
void launch_tie_fix(const skey_t* keys, uint32_t* vals, const uint32_t* d_count, uint32_t cap, const uint32_t* perm,
                    cudaStream_t st);
void launch_ranges(const skey_t* keys, const uint32_t* d_count, uint32_t cap, uint2* ranges, int n_tiles, int key_db,
                   cudaStream_t st);
// exact state of a pixel whose K6 window filled: K6s resumes it at list position `pos`
struct SpillHdr {
    uint32_t pixel, pos, cnt;
    float T, Cr, Cg, Cb;
    uint32_t pad;
};
struct RasterArgs {
    const skey_t* keys;
    const uint32_t* vals;
    const uint2* ranges;
    uint32_t* tile_order;  // K6 launch order of the tiles (written by k_tile_order)
    const float4* raster;
    const float4* color;
    float* out_rgb;       // 3 x out_h x W
    float* out_T;         // out_h x W (nullable)
    int out_row0;         // first image row stored in out (band renders)
    int out_h;
    SpillHdr* spill_hdr;  // spilled pixel states (K6 -> K6s)
    float4* spill_e;      // spill_k window entries per spilled pixel: (z, alpha, g bits, 0)
    uint32_t spill_cap;
    uint32_t spill_k;
    SpillHdr* deep_hdr;   // pixels whose K6s pending set overflowed (K6s -> K6d)
    float4* deep_e;       // deep_k entries per deep pixel: (z, alpha, g bits, order bits)
    uint32_t deep_cap;    // slots
    uint32_t deep_k;      // >= the K6s pending limit
    uint32_t* counters;
    // backward support (AAA_FLAG_SAVE_CONTRIBS): every blended contribution of pixel p, in blend
    // order, as (g bits, alpha) at rec[p * rec_cap + i]; rec_n[p] = count (may exceed rec_cap:
    // overflow, reported by the backward pass). Null when not saving.
    float2* rec;
    uint32_t* rec_n;
    uint32_t rec_cap;
    // giant tiles (AAA_K6_GSUB): each giant sub-tile's K6 warp writes the sub-tile's list — the
    // list positions carrying its bit — into the sort's free ping-pong buffer (gsub, gsub_cap words)
    // and one descriptor (tile, sub, list start, length; gdesc, tiles x 8 capacity); K6s walks the
    // list for the sub-tile's pixels. Null gdesc: giant pixels go through the spill queue.
    uint4* gdesc;
    uint32_t* gsub;
    uint32_t gsub_cap;
    // AAA_K6S_SUBL: every tile list longer than GIANT_MIN gets sub-tile lists too; gtab[tile * 8 +
    // sub] = (start in gsub, length or GSUB_FULL), read by K6s for the spilled pixels of those tiles
    uint2* gtab;
};
#ifndef AAA_K6S_SUBL
#define AAA_K6S_SUBL 0  // A/B (FPS, off / on): c3 306.3 / 299.7, c4 wide 264.9 / 268.5 (K6s 0.41 -> 0.32 ms), c4 inside 324.2 / 320.8
#endif
#ifndef AAA_K6_GSUB
#define AAA_K6_GSUB 1  // A/B (FPS, off / on): c4 zoom-out 231.5 / 269.7, c3 301.6 / 300.1, c4 wide 256.4 / 255.6; images bit-identical
#endif
// gdesc[].w of a sub-tile whose list did not fit: its pixels walk the full tile list
constexpr uint32_t GSUB_FULL = 0xFFFFFFFFu;
void launch_raster(const ViewParams& vp, const RasterArgs& ra, int window_k, cudaStream_t st);

// backward pass (backward.cu): per-Gaussian accumulators of dL/dc (3), dL/dW (9, row-major
// W[j][i]), dL/doA (1), dL/drgb (3)
constexpr int BWD_ACC = 16;
struct BwdArgs {
    const float2* rec;      // recorded blends (RasterArgs::rec)
    const uint32_t* rec_n;
    uint32_t rec_cap;
    const float* dL_drgb;   // 3 x H x W
    const float* dL_dT;     // H x W (nullable)
    const float4* raster;   // the view's raster records
    const float4* color;
    float* acc;             // N x BWD_ACC
    uint32_t* overflow;     // pixels whose record overflowed
    float *d_means, *d_scales, *d_quats, *d_opac, *d_sh;
};
void launch_backward(const SceneDev& sc, const ViewParams& vp, const BwdArgs& ba, cudaStream_t st);
void launch_max_u32(const uint32_t* a, size_t n, uint32_t* out, cudaStream_t st);

// v_hat_train cameras (Eq. 6): world->view rotation/translation, intrinsics, f = max(fx, fy)
struct VtCam {
    double R[9], t[3];
    double fx, fy, cx, cy, near_z, f, w, h;
};
void launch_morton_order(const SceneDev& sc, uint32_t* keys, uint32_t* vals, const float* lo_hi, cudaStream_t st);
int aabb_blocks(int64_t n);
void launch_aabb(const SceneDev& sc, float* d_blk, cudaStream_t st);
void launch_permute(const float4* in, float4* out, const uint32_t* perm, int64_t n, int chunks, cudaStream_t st);
void launch_vtrain(const SceneDev& sc, const VtCam* cams, int n_cams, float* out, bool store, cudaStream_t st);
void launch_raster_fallback(const ViewParams& vp, const RasterArgs& ra, cudaStream_t st);
void launch_row_costs(const ViewBufs& vb, int64_t n, int rows, unsigned long long* diff, cudaStream_t st);
void launch_row_costs_approx(const SceneDev& sc, const ViewParams& vp, int rows, unsigned long long* diff,
                             cudaStream_t st);
#ifndef AAA_K3_HIST
#define AAA_K3_HIST 1  // K3 accumulates the sort's digit histograms, no separate pass (A/B: c3 305.8 -> 307.1 FPS, c2 1801 -> 1829)
#endif
#ifndef AAA_BAND_APPROX
#define AAA_BAND_APPROX 1  // tile bands: cost model from the means and scales, K1 on the band only (c5, 8 bands: slowest 2.64 -> 1.90 ms)
#endif
void launch_band_clip(const ViewBufs& vb, int64_t n, int row_begin, int row_end, cudaStream_t st);
// cudaFuncAttributeMaxDynamicSharedMemorySize is per device: set it once per (kernel, device, size)
// for the current device (thread-safe); a failure is returned and also left in cudaGetLastError()
// for the launching entry point to report.
cudaError_t ensure_smem_attr(const void* func, size_t bytes);

}  // namespace aaa
