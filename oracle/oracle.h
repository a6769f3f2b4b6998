/* oracle.h — float64 CPU brute-force oracle for the AAA-Gaussians forward renderer.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load or call this library. It shares
 * no code, headers, tables or helpers with the CUDA path under
 * paper_2504_12811_b200/ and include/aaa.h, and uses a different algebra:
 * per-pixel rays are minimised with the explicit inverse covariance
 * (SPEC S:509), the amplitude uses the matrix form Eq. 10, and
 * tile culling is an exact convex QP by active-set enumeration of the paper's
 * frustum planes pulled back to Gaussian space (Eq. 5; Eq. 18).
 *
 * All arithmetic is IEEE double; f32 inputs are promoted exactly.
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_scene orc_scene;

typedef struct {
    int32_t width, height;
    double fx, fy, cx, cy;
    double world_to_view[16]; /* row-major rigid transform */
    double near_z;
} orc_camera;

typedef struct {
    double k;          /* filter kernel size, 0.3 */
    int32_t tau_mode;  /* 0: tau = 2 ln(255 o A); 1: tau = min(tau_fixed, 2 ln(255 o A)) */
    double tau_fixed;
    double alpha_max;  /* 0.99 */
    double T_eps;      /* 1e-4 */
    double bg[3];
    /* ambiguity bands */
    double band_rho;   /* |rho^2 - tau| < band_rho            (4e-3) */
    double band_near;  /* |z* - near| < band_near * max(1,z*)  (1e-5) */
    double band_tie;   /* (z_{k+1}-z_k)/z_k < band_tie          (4e-6) */
    double band_gauss; /* Gaussian-level margins, relative      (1e-5) */
    /* blend order (Table 5 "w/o hier. sort"):
     *   0: exact per-ray order by (z*, g) (reading 4)
     *   1: the global per-Gaussian order only (3DGS-style sort by the view depth of the mean):
     *      by (code, g), code = floor(clamp(order_scale * log2(max(mu_z, order_near) / order_near),
     *      0, order_qmax)) — the depth code of the renderer's sort key */
    int32_t order_mode;
    double order_scale, order_near, order_qmax;
    /* evaluation (Table 5 "w/o 3D"): 0: 3D maximum-response evaluation;
     * 1: affine 2D splat — Sigma' = J Sigma_hat_view J^T with the perspective Jacobian J at the
     *    mean, rho^2 = d^T Sigma'^-1 d, d = pixel centre - projected mean; a Gaussian whose mean
     *    is closer than near is dropped; no camera-inside test (use with order_mode 1) */
    int32_t eval_mode;
} orc_config;

/* per-Gaussian record exported by orc_gaussian (indices into out[]) */
enum {
    ORC_G_VHAT = 0, ORC_G_VEFF, ORC_G_SHAT0, ORC_G_SHAT1, ORC_G_SHAT2, ORC_G_A, ORC_G_OA,
    ORC_G_TAU, ORC_G_VALID, ORC_G_INSIDE, ORC_G_INSIDE_RHO2, ORC_G_R, ORC_G_G, ORC_G_B,
    ORC_G_MUV0, ORC_G_MUV1, ORC_G_MUV2, ORC_G_COUNT
};

/* contribution record exported by orc_pixel_contribs */
enum {
    ORC_C_Z = 0, ORC_C_ALPHA, ORC_C_RHO2, ORC_C_TAU, ORC_C_G, ORC_C_R, ORC_C_GG, ORC_C_B,
    ORC_C_INCLUDED, ORC_C_FLAGS, ORC_C_COUNT
};

/* pixel / contribution ambiguity flags */
enum {
    ORC_F_CUTOFF = 1u, ORC_F_NEAR = 2u, ORC_F_TIE = 4u, ORC_F_GAUSS = 8u, ORC_F_TERMINATED = 16u
};

orc_scene* orc_create(int64_t n, int32_t sh_degree, const float* means, const float* scales,
                      const float* quats, const float* opacities, const float* sh,
                      const float* v_train);
void orc_destroy(orc_scene* s);
int32_t orc_num_threads(void);

/* Per-Gaussian preprocessing for one view (filter, amplitude, tau, colour, inside). */
int32_t orc_set_view(orc_scene* s, const orc_camera* cam, const orc_config* cfg);

/* Copy ORC_G_COUNT doubles describing Gaussian g for the current view. */
int32_t orc_gaussian(const orc_scene* s, int64_t g, double* out);

/* All N records at once: N x ORC_G_COUNT doubles. */
int32_t orc_gaussians(const orc_scene* s, double* out);

/* Render npix pixels (integer pixel indices; centres at +0.5). out_rgbT: 4 doubles
 * per pixel (r,g,b,T). out_flags: OR of ORC_F_* over the pixel's decisions.
 * use_rejects = 0 evaluates every Gaussian on every ray (pure brute force). */
int32_t orc_render_pixels(const orc_scene* s, int64_t npix, const int32_t* px, const int32_t* py,
                          int32_t use_rejects, double* out_rgbT, uint32_t* out_flags,
                          int32_t* out_nblend);

/* All contributions and near-miss candidates of one pixel, sorted by (z*, g):
 * ORC_C_COUNT doubles each. Returns the count (may exceed cap; only cap written). */
int64_t orc_pixel_contribs(const orc_scene* s, int32_t px, int32_t py, double* out, int64_t cap);

/* Exact min over the frustum {pixel-centre rect [x0,x1]x[y0,y1]} ∩ {z >= near} of
 * rho^2 for Gaussian g (convex QP, active-set enumeration). m queries. */
int32_t orc_frustum_min_rho2(const orc_scene* s, int64_t m, const int64_t* g, const double* rects,
                             double* out);

/* test hooks */
void orc_sh_basis(const double* d, double* Y16);
double orc_qp_min_norm(int32_t nc, const double* a, const double* b);

/* v_hat_train (Eq. 6): out[g] = max over the cameras whose frustum
 * contains the mean (view depth z >= near, projection inside the pixel-centre rectangle
 * [0.5, W-0.5] x [0.5, H-0.5], reading 20) of max(fx, fy) / z; +inf if none. amb[g] = 1 when
 * some camera's decision lies within a relative 1e-9 of a frustum boundary (FP rounding may flip
 * it). Independent of the view set by orc_set_view. */
int32_t orc_vtrain(const orc_scene* s, int32_t n_cams, const orc_camera* cams, double* out, int32_t* amb);

#ifdef __cplusplus
}
#endif
