/* aaa.h — C ABI of the B200-native AAA-Gaussians forward renderer (arxiv 2504.12811).
 *
 * The library renders a set of 3D Gaussians (mean mu, scale s, rotation q, opacity o,
 * SH colour, stored training frequency v_train) from a pinhole
 * camera (V, P, M_vp, f) with the paper's four stages:
 *   1. per-Gaussian preprocess: adaptive 3D smoothing filter and perpendicular amplitude
 *      (Eq. 6-13), SH colour, view-space bounding (Eq. 14-17),
 *      camera-inside discard, whole-view-frustum cull;
 *   2. 3D tile-frustum culling (Eq. 18) and (tile, depth) key emission;
 *   3. a global onesweep radix sort of the keys and per-tile ranges;
 *   4. per-tile hierarchical re-sort with per-pixel 3D evaluation at the maximum-response
 *      point (Eq. 4-5), front-to-back blending with early termination.
 * All of it runs in hand-written sm_100a CUDA kernels; nothing here falls back to the CPU.
 *
 * Conventions: view space +z forward, y down; pixel (i, j) has its
 * centre at (i + 0.5, j + 0.5); x_pix = fx X/Z + cx. Quaternions are (w, x, y, z).
 * Inputs are post-activation (scales > 0, opacity in (0,1)).
 *
 * Threading: one context per host thread; calls on one context are not thread-safe.
 * Errors: every call returns aaa_status; aaa_last_error() gives a per-context message that
 * stays valid until the next call on that context. Asynchronous CUDA errors surface at the
 * next synchronising call as AAA_ERR_CUDA.
 * Determinism: identical inputs give bit-identical images, keys and values.
 */
#ifndef AAA_H_
#define AAA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    AAA_WARN_UNRESOLVED = 1,       /* results written, but some pixels of the last view hit a
                                      full spill queue and hold a partial (inexact) blend; only
                                      aaa_get_stats / aaa_synchronize return it (stats filled) */
    AAA_OK = 0,
    AAA_ERR_INVALID_ARG = -1,      /* null pointer, bad camera/config value, bad sizes      */
    AAA_ERR_INVALID_GAUSSIAN = -2, /* load-time validation failed; see first_bad   */
    AAA_ERR_CUDA = -3,             /* CUDA runtime error (message from cudaGetErrorString) */
    AAA_ERR_OOM = -4,              /* device allocation failed                              */
    AAA_ERR_STATE = -5             /* call out of order (e.g. render before load/camera)    */
} aaa_status;

typedef struct aaa_ctx aaa_ctx; /* opaque; owns all device state of one renderer */

/* Pinhole camera. world_to_view: row-major 4x4 rigid transform whose upper
 * 3x3 is a rotation (det +1) and whose last row is (0,0,0,1). Requirements: width, height
 * in [1, 65535]; fx, fy > 0; near_z > 0 (default 0.01, reading 7). */
typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
    float world_to_view[16];
    float near_z;
} aaa_camera;

/* Render configuration. Defaults from aaa_default_config():
 *   k = 0.3; tau_mode 0: tau = 2 ln(255 o A) per Gaussian (reading 1), tau_mode 1:
 *   tau = min(tau_fixed, 2 ln(255 o A)) with tau_fixed = 9; alpha_max = 0.99 (reading 2);
 *   T_eps = 1e-4 (reading 3); background black; window_k = 32 (per-pixel re-sort window,
 *   16 or 32); flags = 0. */
typedef struct {
    float k;
    int32_t tau_mode;
    float tau_fixed;
    float alpha_max;
    float T_eps;
    float background[3];
    int32_t window_k;
    uint32_t flags;
} aaa_config;

/* Scene arrays, structure-of-arrays, float32:
 *   means N x 3, scales N x 3 (standard deviations, > 0), quats N x 4 (w,x,y,z, nonzero),
 *   opacities N (in (0,1)), sh N x (deg+1)^2 x 3 (coefficient-major, channel-minor),
 *   v_train N (> 0 or +inf).
 * device_ptrs = 1: the pointers are CUDA device memory on the context's device; 0: host. */
typedef struct {
    const float *means, *scales, *quats, *opacities, *sh, *v_train;
    int64_t n;
    int32_t sh_degree; /* 0..3 */
    int32_t device_ptrs;
} aaa_gaussians;

/* Counters of the last rendered view: N loaded, V visible after preprocessing,
 * C candidate (Gaussian, tile) pairs from the bounds, P pairs kept by 3D tile culling,
 * pixels whose K6 per-pixel window filled (their exact state is spilled and finished by the
 * K6s kernel), pixels K6s could not resolve exactly (0 unless the image is wrong),
 * Gaussians taking the near-plane-crossing cull path, pixel-Gaussian evaluations in the
 * raster kernels, and the number of kernels this context has launched since creation.
 * ms[]: mean per-view device time of each stage over the views rendered with AAA_FLAG_TIMING
 * since the previous aaa_get_stats call (timed_views of them; the accumulation is reset by
 * the call): 0 preprocess (K1), 1 scan (K2), 2 cull/emit (K3), 3 sort (K4), 4 ranges (K5),
 * 5 raster (K6), 6 spilled-pixel continuation (K6s), 7 host-sync gap after K2, 8 output copy
 * (host outputs only), 9 total. deep_pixels: spilled pixels whose pending set outgrew K6s's
 * 256 entries (finished by K6d with 2048). giant_pixels: pixels of tiles whose list exceeded the
 * giant-list threshold, rendered one warp per pixel by K6s from the list start (counted in
 * spilled_pixels too). */
typedef struct {
    int64_t n, visible, candidates, pairs, spilled_pixels, unresolved_pixels, crossing;
    int64_t evaluations, launches, timed_views;
    float ms[10];
    int64_t deep_pixels, giant_pixels;
} aaa_stats;

/* aaa_config.flags:
 *   AAA_FLAG_TIMING          per-stage CUDA events (read back by aaa_get_stats)
 *   AAA_FLAG_NO_TILE_CULL    Table 5 "w/o culling": every tile of the bounds rect is kept
 *                            (no 3D tile test, no sub-tile masks); the image is unchanged
 *   AAA_FLAG_FORCE_FALLBACK  window K = 1: every pixel with two pending entries continues in the
 *                            spill kernel (test of the exact continuation; the image is unchanged)
 *   AAA_FLAG_FORCE_DEEP      K6s hands every pixel whose pending set exceeds 32 entries to K6d
 *                            (test of the second spill level; the image is unchanged)
 *   AAA_FLAG_CULL_FP64       K3 decides every tile / sub-tile test in FP64 (no FP32 guard-band
 *                            fast path; test of the guard band: the pairs are unchanged)
 *   AAA_FLAG_FORCE_GIANT     every tile with a list of more than one entry takes the giant-list
 *                            path (one warp per pixel in K6s from the list start; test of that
 *                            path: the image is unchanged)
 *   AAA_FLAG_NO_GSUB         giant-list pixels walk their tile's whole list instead of their
 *                            sub-tile's list (the path taken when the sub-tile lists do not fit in
 *                            the free sort buffer; test of it: the image is unchanged)
 *   AAA_FLAG_NO_HIER_SORT    Table 5 "w/o hier. sort": blend in the global per-Gaussian
 *                            order only — tile lists sorted by the view depth of the mean, no
 *                            per-pixel re-sort (the image changes where that order is not z*)
 *   AAA_FLAG_NO_3D           Table 5 "w/o 3D": affine 2D splat evaluation (EWA projection
 *                            J Sigma_hat_view J^T of the filtered Gaussian, J the perspective
 *                            Jacobian at the mean; rho^2 = d^T Sigma'^-1 d), exact 2D tile culling,
 *                            the global mean-depth order (implies NO_HIER_SORT); Gaussians whose
 *                            mean is closer than near are dropped, no camera-inside test.
 *                            With NO_TILE_CULL and k = 0 this is a 3DGS-style baseline path. */
enum {
    AAA_FLAG_TIMING = 1u,
    AAA_FLAG_NO_TILE_CULL = 2u,
    AAA_FLAG_FORCE_FALLBACK = 4u,
    AAA_FLAG_NO_HIER_SORT = 8u,
    AAA_FLAG_NO_3D = 16u,
    AAA_FLAG_SAVE_CONTRIBS = 32u  /* aaa_render records each pixel's blended contributions (in blend
                                   * order) for aaa_render_backward; single full-image default renders
                                   * only; the call synchronises */
    , AAA_FLAG_FORCE_DEEP = 64u
    , AAA_FLAG_CULL_FP64 = 128u
    , AAA_FLAG_FORCE_GIANT = 256u
    , AAA_FLAG_NO_GSUB = 512u
};

/* what for aaa_debug_copy (parity tests only; synchronises) */
enum {
    AAA_DBG_GAUSS = 0,  /* N x AAA_DBG_GAUSS_FIELDS float64 per-Gaussian preprocess record  */
    AAA_DBG_KEYS = 1,   /* P uint32 keys, sorted (tile << (32 - tile bits) | log-depth code) */
    AAA_DBG_VALS = 2,   /* P uint32 Gaussian indices, sorted                                  */
    AAA_DBG_KEYS_UNSORTED = 3, /* P uint32 keys in emission order                         */
    AAA_DBG_VALS_UNSORTED = 4, /* P uint32 values in emission order                       */
    AAA_DBG_RANGES = 5, /* tiles x 2 uint32 [start, end)                                     */
    AAA_DBG_SPILL = 6,   /* spilled pixels: 8 x 32-bit (pixel, list pos, count, T, r, g, b, 0) */
    AAA_DBG_RASTER = 7,  /* N x 28 float32 raster records of the last view (K6 inputs)         */
    AAA_DBG_COLOR = 8    /* N x 4 float32 colours of the last view                              */
};
/* per-Gaussian debug record: v_hat, v_eff, s_hat[3], A, oA, tau, valid(after inside test),
 * inside, inside_rho2, colour[3], visible (kept by the whole-view cull), crossing,
 * tile rect tx0, ty0, tx1, ty1 (inclusive; empty if tx0 > tx1), z key (float), pixel rect
 * x0, x1, y0, y1 (continuous pixel coordinates of the angular bounds) */
enum { AAA_DBG_GAUSS_FIELDS = 26 };

int32_t aaa_version(void);

/* Create a context on `device`; `cuda_stream` (a cudaStream_t, may be NULL = legacy default
 * stream) is borrowed, not owned: every kernel and copy of the context is enqueued on it. */
aaa_status aaa_create(int32_t device, void* cuda_stream, aaa_ctx** out);
void aaa_destroy(aaa_ctx* ctx);
aaa_status aaa_set_stream(aaa_ctx* ctx, void* cuda_stream);

aaa_status aaa_default_config(aaa_config* cfg);
aaa_status aaa_set_config(aaa_ctx* ctx, const aaa_config* cfg);

/* Copy the Gaussians into the context's packed device buffers (caller may free its arrays
 * when this returns; synchronises). Validates q != 0, s > 0, o in (0,1), finite values,
 * v_train > 0: on failure returns AAA_ERR_INVALID_GAUSSIAN and writes
 * the first bad index to *first_bad (nullable). n = 0 is a valid empty scene. */
aaa_status aaa_load_gaussians(aaa_ctx* ctx, const aaa_gaussians* g, int64_t* first_bad);

/* Validate and store the camera used by aaa_render. */
aaa_status aaa_set_camera(aaa_ctx* ctx, const aaa_camera* cam);

/* Render the current camera. rgb: 3 x H x W float32 (CHW), T: H x W final transmittance
 * (nullable). Pointers may be device memory (rendered in place on the context's stream) or host
 * memory (copied back; the call returns after the copy). The views themselves need no host round
 * trip (K3 and the sort read the candidate count on the device); the call synchronises once at its
 * end to check that no view outgrew the context's pair buffers, and renders any that did again
 * with larger buffers (the first call of a context also reads the count back once per slot). */
aaa_status aaa_render(aaa_ctx* ctx, float* rgb, float* T);

/* Render n_views cameras (all with the same width/height) into rgb n x 3 x H x W and
 * T n x H x W (nullable). Same pointer rules as aaa_render. */
aaa_status aaa_render_batch(aaa_ctx* ctx, const aaa_camera* cams, int32_t n_views, float* rgb, float* T);

/* Render only tile rows [tile_row_begin, tile_row_end) of the current camera (screen-space
 * band partition for multi-GPU single frames). rgb_band: 3 x band_h x W with
 * band_h = min(16*tile_row_end, H) - 16*tile_row_begin; T_band nullable. */
aaa_status aaa_render_tiles(aaa_ctx* ctx, int32_t tile_row_begin, int32_t tile_row_end, float* rgb_band,
                            float* T_band);

/* Per-tile-row candidate cost of the current camera (sum of candidate tiles of every visible
 * Gaussian on each tile row), used to balance tile bands; out: host, ceil(H/16) int64. Runs K1
 * and a device row histogram only. Syncs. */
aaa_status aaa_tile_row_costs(aaa_ctx* ctx, int64_t* out, int32_t n_rows);

/* One frame split across `world` ranks by screen-space tile-row bands (the c5 partition of
 * SURVEY 8(e); the paper itself renders on one GPU): K1 runs on every Gaussian for the whole
 * frame (replicated on every rank), its per-row candidate costs (as aaa_tile_row_costs) cut the R
 * tile rows into `world` contiguous bands of near-equal cost — the same cut on every rank, no
 * communication — and K2-K6 run for this rank's band only. cuts (host, world + 1 int32, out): band
 * r is tile rows [cuts[r], cuts[r+1]). rgb (device or host): capacity 3 x H x W floats; the band is
 * written as 3 planes of band_h x W, band_h = min(16 cuts[rank+1], H) - 16 cuts[rank]; T (nullable):
 * band_h x W. Output is bit-identical to the same rows of aaa_render.
 * Errors: AAA_ERR_INVALID_ARG (world < 1, rank outside [0, world), world > R, null rgb/cuts),
 * AAA_ERR_STATE (no scene or camera). Synchronises twice internally (row costs, pair count). */
aaa_status aaa_render_band(aaa_ctx* ctx, int32_t rank, int32_t world, float* rgb, float* T, int32_t* cuts);

/* Training sampling frequency v_hat_train (Eq. 6): for every loaded
 * Gaussian, the maximum over the cameras whose view frustum contains its mean of f / z, with z
 * the mean's view depth and f = max(fx, fy) (reading 10). "Contains" is the culling frustum of
 * reading 20 applied to the mean point: z >= near_z and the projection inside the pixel-centre
 * rectangle [0.5, W - 0.5] x [0.5, H - 0.5]. +inf when no camera sees the mean or n_cams == 0
 * (S:192). Computed in FP64 from the float32 inputs, rounded to float32.
 * cams: n_cams host cameras (validated like aaa_set_camera). out: N floats, device or host
 * pointer, nullable when store != 0. store != 0 also replaces the context's per-Gaussian
 * v_train, so later renders use it (the next step of the pipeline).
 * Errors: AAA_ERR_INVALID_ARG (n_cams < 0, bad camera, out null with store == 0),
 * AAA_ERR_STATE (no scene loaded). Synchronises. */
aaa_status aaa_compute_vtrain(aaa_ctx* ctx, const aaa_camera* cams, int32_t n_cams, float* out, int32_t store);

/* Backward pass (the paper trains with this rasterizer): gradients of
 * a scalar loss L through the last aaa_render made with AAA_FLAG_SAVE_CONTRIBS (full image, no
 * ablation flags). In (device float32): dL_drgb 3 x H x W, dL_dT H x W (nullable = 0). Out
 * (device float32, overwritten): d_means N x 3, d_scales N x 3, d_quats N x 4 (w.r.t. the raw,
 * unnormalised input quaternion), d_opac N, d_sh N x (deg+1)^2 x 3 (the load layout). The blend
 * order and the contribution set of the forward are held fixed (the tau cutoff, near plane,
 * culling and early termination carry no derivative); v_train is not differentiated.
 * Errors: AAA_ERR_STATE (no saved render, or the scene/camera changed since), AAA_ERR_INVALID_ARG
 * (null pointers), AAA_ERR_CUDA. The saving render sizes its per-pixel record to the largest
 * blend count (re-rendering once when it grows). Synchronises. */
aaa_status aaa_render_backward(aaa_ctx* ctx, const float* dL_drgb, const float* dL_dT, float* d_means,
                               float* d_scales, float* d_quats, float* d_opac, float* d_sh);

/* Both synchronise; both return AAA_WARN_UNRESOLVED (stats still filled) when pixels of the last
 * view were left inexact because a spill queue was full (stats.unresolved_pixels; never seen on
 * c1-c5). */
aaa_status aaa_get_stats(aaa_ctx* ctx, aaa_stats* out);
aaa_status aaa_synchronize(aaa_ctx* ctx);

/* Copy an internal buffer of the last render to host memory (parity tests only). *len
 * receives the byte size; returns AAA_ERR_INVALID_ARG if cap is too small. */
aaa_status aaa_debug_copy(aaa_ctx* ctx, int32_t what, void* host_dst, size_t cap, size_t* len);

const char* aaa_last_error(const aaa_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* AAA_H_ */
