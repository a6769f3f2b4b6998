// oracle.cpp — plain, slow, float64 CPU oracle of the AAA-Gaussians forward render.
//
// TEST INFRASTRUCTURE ONLY (see oracle.h). Every function cites the passage of
// /root/reference/PAPER.md (P:line) or SPEC.md (S:line) it follows, or the
// reading in DESIGN.md "Readings" (= SURVEY.md §8c row N) where the paper is silent.
//
// What it computes, in the paper's order:
//   per Gaussian:  R(q) (Eq. 3), view-space mean, v_hat = f/d (Eq. 6),
//       v' = min(v_train, v_hat) (Eq. 13), Sigma_hat = Sigma + k/v'^2 I,
//       A = sqrt(|Sigma| d^T Sigma^-1 d / (|Sigma_hat| d^T Sigma_hat^-1 d)) (Eq. 10, matrix form),
//       tau = 2 ln(255 o A) (reading 1), colour from SH at d (reading 15),
//       camera-inside discard (reading 8).
//   per pixel: maximum-response point on the pixel ray by explicit minimisation
//       of (x-mu)^T Sigma_hat^-1 (x-mu) along the ray; contributes iff rho^2 < tau and
//       z* >= near (readings 1, 6); alpha = min(0.99, o A exp(-rho^2/2)) (Eq. 9, reading 2);
//       exact sort by (z*, g) (reading 4); front-to-back blend with the 3DGS termination rule
//       (reading 3).
//   culling (Eq. 18): exact min of rho^2 over the tile frustum (4 pixel-centre planes
//       plus z >= near, readings 20-21), planes pulled back to Gaussian space by T_view^T (Eq. 5),
//       QP solved by enumerating every active set of <= 3 constraints.
//
// Exact rejects: a Gaussian whose bounding sphere of radius
// sqrt((tau+band) * lambda_max(Sigma_hat)) misses a tile's cone or a pixel's ray line
// provably has rho^2 >= tau + band on that ray, so skipping it changes nothing; a self-test
// checks use_rejects=1 and use_rejects=0 agree bit for bit.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

typedef double M3[3][3];

struct Prepared {
    bool valid;        // tau > 0 and camera outside the ellipsoid
    bool inside;
    double inside_rho2;
    double vhat, veff, shat[3], A, oA, tau;
    double rgb[3];
    double mu[3];      // world mean
    double muv[3];     // view mean
    double Sinv[3][3]; // Sigma_hat^-1
    double radius;     // sqrt((tau + band_rho) * max shat)
    bool gauss_margin; // inside-test margin within band_gauss
    double order_code; // order_mode 1: depth code of the mean (orc_config)
    double pm[2];      // eval_mode 1: projected mean (pixels)
    double conic[3];   // eval_mode 1: Sigma'^-1 = [[c0, c1], [c1, c2]]
    double radius2d;   // eval_mode 1: sqrt((tau + band) lambda_max(Sigma')) (exact reject radius)
};

}  // namespace

struct orc_scene {
    int64_t n;
    int deg;
    std::vector<double> means, scales, quats, opac, sh, vtrain;
    orc_camera cam;
    orc_config cfg;
    double Rv[3][3], Rvi[3][3], tv[3], o[3];  // world->view rotation (and its inverse), translation, camera centre
    std::vector<Prepared> prep;
    bool have_view = false;
};

namespace {

// ---- tiny linear algebra -------------------------------------------------
inline double dot3(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }

inline double det3(const M3 m) {
    return m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
           m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
           m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]);
}

// inverse by the adjugate (explicit; the oracle deliberately inverts)
inline void inv3(const M3 m, M3 out) {
    double d = det3(m);
    out[0][0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) / d;
    out[0][1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) / d;
    out[0][2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) / d;
    out[1][0] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) / d;
    out[1][1] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) / d;
    out[1][2] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) / d;
    out[2][0] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) / d;
    out[2][1] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) / d;
    out[2][2] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) / d;
}

inline double quad3(const M3 m, const double* v) {  // v^T m v
    double s = 0;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) s += v[i] * m[i][j] * v[j];
    return s;
}

// Rotation from a (w,x,y,z) Hamilton quaternion, normalised.
void quat_rot(const double* q_in, M3 R) {
    double n = std::sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
    double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
    R[0][0] = 1 - 2 * (y * y + z * z); R[0][1] = 2 * (x * y - w * z);     R[0][2] = 2 * (x * z + w * y);
    R[1][0] = 2 * (x * y + w * z);     R[1][1] = 1 - 2 * (x * x + z * z); R[1][2] = 2 * (y * z - w * x);
    R[2][0] = 2 * (x * z - w * y);     R[2][1] = 2 * (y * z + w * x);     R[2][2] = 1 - 2 * (x * x + y * y);
}

// Real spherical-harmonic basis, degree <= 3, in the 3DGS sign convention (reading 15).
// Written from the textbook polynomial forms Y_lm(x,y,z) on the unit sphere.
void sh_basis(const double* d, double* Y) {
    const double PI = 3.14159265358979323846;
    double x = d[0], y = d[1], z = d[2];
    Y[0] = 0.5 * std::sqrt(1.0 / PI);
    double c1 = std::sqrt(3.0 / (4.0 * PI));
    Y[1] = -c1 * y;
    Y[2] = c1 * z;
    Y[3] = -c1 * x;
    double c2a = 0.5 * std::sqrt(15.0 / PI), c2b = 0.25 * std::sqrt(5.0 / PI), c2c = 0.25 * std::sqrt(15.0 / PI);
    Y[4] = c2a * x * y;
    Y[5] = -c2a * y * z;
    Y[6] = c2b * (3.0 * z * z - 1.0);
    Y[7] = -c2a * x * z;
    Y[8] = c2c * (x * x - y * y);
    double c3a = 0.25 * std::sqrt(35.0 / (2.0 * PI)), c3b = 0.5 * std::sqrt(105.0 / PI),
           c3c = 0.25 * std::sqrt(21.0 / (2.0 * PI)), c3d = 0.25 * std::sqrt(7.0 / PI),
           c3e = 0.25 * std::sqrt(105.0 / PI);
    Y[9] = -c3a * y * (3.0 * x * x - y * y);
    Y[10] = c3b * x * y * z;
    Y[11] = -c3c * y * (5.0 * z * z - 1.0);
    Y[12] = c3d * z * (5.0 * z * z - 3.0);
    Y[13] = -c3c * x * (5.0 * z * z - 1.0);
    Y[14] = c3e * z * (x * x - y * y);
    Y[15] = -c3a * x * (x * x - 3.0 * y * y);
}

// Per-Gaussian preprocessing for the current view.
void prepare_one(const orc_scene* s, int64_t g, Prepared& P) {
    const orc_config& cfg = s->cfg;
    const orc_camera& cam = s->cam;
    const double* mu = &s->means[3 * g];
    const double* sc = &s->scales[3 * g];
    M3 R;
    quat_rot(&s->quats[4 * g], R);
    for (int i = 0; i < 3; i++) P.mu[i] = mu[i];
    for (int i = 0; i < 3; i++) P.muv[i] = dot3(s->Rv[i], mu) + s->tv[i];
    // Eq. 6: v_hat = f / d, d = view-space z of the mean; f = max(fx, fy) (reading 10);
    // v_hat = +inf when the mean is not in front (reading 9).
    double f = std::max(cam.fx, cam.fy);
    P.vhat = P.muv[2] > 0 ? f / P.muv[2] : std::numeric_limits<double>::infinity();
    // Eq. 13: v' = min(v_train, v_hat)
    P.veff = std::min(s->vtrain[g], P.vhat);
    double cf = std::isinf(P.veff) ? 0.0 : cfg.k / (P.veff * P.veff);
    // Sigma = R S S^T R^T (Eq. 3) and Sigma_hat = Sigma + k/v'^2 I (with v', reading 12)
    M3 Sig, Shat;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double v = 0;
            for (int m = 0; m < 3; m++) v += R[i][m] * sc[m] * sc[m] * R[j][m];
            Sig[i][j] = v;
            Shat[i][j] = v + (i == j ? cf : 0.0);
        }
    for (int i = 0; i < 3; i++) P.shat[i] = sc[i] * sc[i] + cf;  // eigenvalues of Sigma_hat (Eq. 12 notation)
    // Eq. 10, explicit determinants and inverses; d = (mu - o)/|mu - o|
    double d[3] = {mu[0] - s->o[0], mu[1] - s->o[1], mu[2] - s->o[2]};
    double dn = std::sqrt(dot3(d, d));
    for (int i = 0; i < 3; i++) d[i] /= dn;
    M3 Sinv, Shinv;
    inv3(Sig, Sinv);
    inv3(Shat, Shinv);
    if (cf == 0.0) {
        P.A = 1.0;  // Sigma_hat == Sigma: the ratio is exactly 1
    } else {
        double num = det3(Sig) * quad3(Sinv, d);
        double den = det3(Shat) * quad3(Shinv, d);
        P.A = std::sqrt(num / den);
    }
    // alpha uses o * A (Eq. 9, reading 13); tau: the alpha >= 1/255 level set (reading 1)
    P.oA = s->opac[g] * P.A;
    double tau_op = 2.0 * std::log(255.0 * P.oA);
    P.tau = cfg.tau_mode == 0 ? tau_op : std::min(cfg.tau_fixed, tau_op);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) P.Sinv[i][j] = Shinv[i][j];
    // camera inside the tau-ellipsoid -> discard (reading 8)
    double om[3] = {s->o[0] - mu[0], s->o[1] - mu[1], s->o[2] - mu[2]};
    P.inside_rho2 = quad3(Shinv, om);
    P.inside = P.inside_rho2 < P.tau;
    P.gauss_margin = std::fabs(P.inside_rho2 - P.tau) <= cfg.band_gauss * std::max(1.0, std::fabs(P.tau));
    P.valid = (P.tau > 0) && !P.inside;
    // colour: SH at direction d, + 0.5, clamped below at 0 (reading 15)
    double Y[16];
    sh_basis(d, Y);
    int K = (s->deg + 1) * (s->deg + 1);
    for (int c = 0; c < 3; c++) {
        double v = 0;
        for (int k = 0; k < K; k++) v += Y[k] * s->sh[(g * K + k) * 3 + c];
        P.rgb[c] = std::max(0.0, v + 0.5);
    }
    // eval_mode 1 (Table 5 "w/o 3D"): EWA projection Sigma' = J (Rv Sigma_hat Rv^T) J^T
    if (cfg.eval_mode == 1) {
        M3 Sv;
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                double v = 0;
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++) v += s->Rv[i][a] * Shat[a][b] * s->Rv[j][b];
                Sv[i][j] = v;
            }
        const double x = P.muv[0], y = P.muv[1], z = P.muv[2];
        const double J[2][3] = {{cam.fx / z, 0.0, -cam.fx * x / (z * z)}, {0.0, cam.fy / z, -cam.fy * y / (z * z)}};
        double S2[2][2];
        for (int i = 0; i < 2; i++)
            for (int j = 0; j < 2; j++) {
                double v = 0;
                for (int a = 0; a < 3; a++)
                    for (int b = 0; b < 3; b++) v += J[i][a] * Sv[a][b] * J[j][b];
                S2[i][j] = v;
            }
        const double det = S2[0][0] * S2[1][1] - S2[0][1] * S2[1][0];
        P.conic[0] = S2[1][1] / det;
        P.conic[1] = -S2[0][1] / det;
        P.conic[2] = S2[0][0] / det;
        P.pm[0] = cam.fx * x / z + cam.cx;
        P.pm[1] = cam.fy * y / z + cam.cy;
        const double hm = 0.5 * (S2[0][0] + S2[1][1]), hd = 0.5 * (S2[0][0] - S2[1][1]);
        const double lmax2 = hm + std::sqrt(hd * hd + S2[0][1] * S2[0][1]);
        P.radius2d = std::sqrt(std::max(0.0, P.tau + cfg.band_rho) * lmax2);
        // 3DGS mean-frustum rule (reading 36): projected mean within 1.3x the image about its centre
        const bool in_fr = std::fabs(P.pm[0] - 0.5 * cam.width) <= 0.65 * cam.width &&
                           std::fabs(P.pm[1] - 0.5 * cam.height) <= 0.65 * cam.height;
        P.valid = (P.tau > 0) && (z >= cam.near_z) && det > 0 && in_fr;
        P.inside = false;
        P.gauss_margin = false;
    }
    // order_mode 1 (Table 5 "w/o hier. sort"): global order by the mean's view depth code
    P.order_code = 0.0;
    if (cfg.order_mode == 1) {
        double u = cfg.order_scale * std::log2(std::max(P.muv[2], cfg.order_near) / cfg.order_near);
        P.order_code = std::floor(std::min(std::max(u, 0.0), cfg.order_qmax));
    }
    double lmax = std::max(P.shat[0], std::max(P.shat[1], P.shat[2]));
    P.radius = std::sqrt(std::max(0.0, P.tau + cfg.band_rho) * lmax);
}

struct Contrib {
    double z, alpha, rho2, tau, rgb[3];
    int64_t g;
    bool included;
    uint32_t flags;
};

// World-space direction v of pixel centre p with view-z component 1 (reading 26).
inline void pixel_dir(const orc_scene* s, double px, double py, double* v) {
    double r[3] = {(px - s->cam.cx) / s->cam.fx, (py - s->cam.cy) / s->cam.fy, 1.0};
    for (int i = 0; i < 3; i++) v[i] = s->Rvi[i][0] * r[0] + s->Rvi[i][1] * r[1] + s->Rvi[i][2] * r[2];
}

// Maximum-response point of Gaussian g along the ray o + t v, by explicit
// minimisation with Sigma_hat^-1: t* = v^T S^-1 (mu - o) / v^T S^-1 v.
inline void eval_ray(const orc_scene* s, const Prepared& P, const double* v, double* t_out, double* rho2_out) {
    double mo[3] = {P.mu[0] - s->o[0], P.mu[1] - s->o[1], P.mu[2] - s->o[2]};
    double Sv[3], Smo[3];
    for (int i = 0; i < 3; i++) {
        Sv[i] = dot3(P.Sinv[i], v);
        Smo[i] = dot3(P.Sinv[i], mo);
    }
    double t = dot3(v, Smo) / dot3(v, Sv);
    double e[3] = {s->o[0] + t * v[0] - P.mu[0], s->o[1] + t * v[1] - P.mu[1], s->o[2] + t * v[2] - P.mu[2]};
    *t_out = t;                 // view depth z*, since v has view-z 1 (reading 5)
    *rho2_out = quad3(P.Sinv, e);
}

// Collect the contributions (and near-miss candidates) of one pixel from a candidate list.
void pixel_contribs(const orc_scene* s, const std::vector<int64_t>* cand, int px, int py, bool use_rejects,
                    std::vector<Contrib>& out) {
    const orc_config& cfg = s->cfg;
    double v[3];
    pixel_dir(s, px + 0.5, py + 0.5, v);
    double vn = std::sqrt(dot3(v, v));
    double vh[3] = {v[0] / vn, v[1] / vn, v[2] / vn};
    out.clear();
    int64_t m = cand ? (int64_t)cand->size() : s->n;
    for (int64_t i = 0; i < m; i++) {
        int64_t g = cand ? (*cand)[i] : i;
        const Prepared& P = s->prep[g];
        if (cfg.eval_mode == 1) {  // affine 2D splat (Table 5 "w/o 3D")
            if (!P.valid) continue;
            const double dx = px + 0.5 - P.pm[0], dy = py + 0.5 - P.pm[1];
            const double rho2 = P.conic[0] * dx * dx + 2.0 * P.conic[1] * dx * dy + P.conic[2] * dy * dy;
            const bool in_rho = rho2 < P.tau, near_rho = std::fabs(rho2 - P.tau) < cfg.band_rho;
            if (!in_rho && !near_rho) continue;
            Contrib c;
            c.z = P.muv[2];
            c.rho2 = rho2;
            c.tau = P.tau;
            c.alpha = std::min(cfg.alpha_max, P.oA * std::exp(-0.5 * rho2));
            for (int k = 0; k < 3; k++) c.rgb[k] = P.rgb[k];
            c.g = g;
            c.included = in_rho;
            c.flags = near_rho ? ORC_F_CUTOFF : 0u;
            out.push_back(c);
            continue;
        }
        if (!(P.tau > 0) || (P.inside && !P.gauss_margin)) continue;
        if (use_rejects) {  // exact sphere-vs-line reject (rho^2 >= dist^2 / lambda_max)
            double d[3] = {P.mu[0] - s->o[0], P.mu[1] - s->o[1], P.mu[2] - s->o[2]};
            double a = dot3(d, vh);
            double dist2 = dot3(d, d) - a * a;
            if (dist2 > P.radius * P.radius * (1.0 + 1e-9)) continue;
        }
        double t, rho2;
        eval_ray(s, P, v, &t, &rho2);
        bool in_rho = rho2 < P.tau;
        bool near_rho = std::fabs(rho2 - P.tau) < cfg.band_rho;
        bool in_near = t >= s->cam.near_z;  // reading 6
        bool near_near = std::fabs(t - s->cam.near_z) < cfg.band_near * std::max(1.0, std::fabs(t));
        bool included = in_rho && in_near && !P.inside;
        bool flippable = near_rho || near_near || P.gauss_margin;
        if (!included && !flippable) continue;
        if (!included && !(in_rho || near_rho)) continue;
        if (!in_near && !near_near) continue;  // max-response point behind near: never a contribution
        Contrib c;
        c.z = t;
        c.rho2 = rho2;
        c.tau = P.tau;
        c.alpha = std::min(cfg.alpha_max, P.oA * std::exp(-0.5 * rho2));
        for (int k = 0; k < 3; k++) c.rgb[k] = P.rgb[k];
        c.g = g;
        c.included = included;
        c.flags = (near_rho ? ORC_F_CUTOFF : 0u) | (near_near ? ORC_F_NEAR : 0u) | (P.gauss_margin ? ORC_F_GAUSS : 0u);
        out.push_back(c);
    }
    if (cfg.order_mode == 1) {  // global per-Gaussian order only (orc_config.order_mode)
        std::sort(out.begin(), out.end(), [s](const Contrib& a, const Contrib& b) {
            const double ca = s->prep[a.g].order_code, cb = s->prep[b.g].order_code;
            return ca < cb || (ca == cb && a.g < b.g);
        });
        return;
    }
    // exact per-ray order: ascending z*, ties by index (reading 4)
    std::sort(out.begin(), out.end(), [](const Contrib& a, const Contrib& b) {
        return a.z < b.z || (a.z == b.z && a.g < b.g);
    });
}

// Front-to-back blend (reading 3): stop when T (1 - alpha) < T_eps, else C += alpha c T, T *= 1 - alpha.
void blend(const orc_scene* s, std::vector<Contrib>& cs, double* rgbT, uint32_t* flags, int32_t* nblend) {
    const orc_config& cfg = s->cfg;
    double C[3] = {0, 0, 0}, T = 1.0;
    uint32_t f = 0;
    int nb = 0;
    // tie flags among included neighbours; none in the global-order mode
    int prev = -1;
    for (size_t i = 0; i < cs.size() && cfg.order_mode == 0; i++) {
        if (!cs[i].included && !(cs[i].flags)) continue;
        if (prev >= 0) {
            double gap = (cs[i].z - cs[prev].z) / std::max(std::fabs(cs[prev].z), 1e-300);
            if (gap < cfg.band_tie) {
                cs[i].flags |= ORC_F_TIE;
                cs[prev].flags |= ORC_F_TIE;
            }
        }
        prev = (int)i;
    }
    bool done = false;
    for (size_t i = 0; i < cs.size(); i++) {
        const Contrib& c = cs[i];
        if (!done) f |= c.flags;
        if (!c.included || done) continue;
        double testT = T * (1.0 - c.alpha);
        if (testT < cfg.T_eps) {
            done = true;
            f |= ORC_F_TERMINATED;
            continue;
        }
        for (int k = 0; k < 3; k++) C[k] += c.alpha * c.rgb[k] * T;
        T = testT;
        nb++;
    }
    for (int k = 0; k < 3; k++) rgbT[k] = C[k] + T * cfg.bg[k];
    rgbT[3] = T;
    *flags = f;
    *nblend = nb;
}

// Tile-level exact reject: sphere (mu, radius) vs the cone of the tile's pixel-centre rays.
void tile_candidates(const orc_scene* s, int tx, int ty, std::vector<int64_t>& out) {
    const orc_camera& cam = s->cam;
    double x0 = 16.0 * tx + 0.5, x1 = std::min(16.0 * tx + 15.5, cam.width - 0.5);
    double y0 = 16.0 * ty + 0.5, y1 = std::min(16.0 * ty + 15.5, cam.height - 0.5);
    double axis[3];
    pixel_dir(s, 0.5 * (x0 + x1), 0.5 * (y0 + y1), axis);
    double an = std::sqrt(dot3(axis, axis));
    for (int i = 0; i < 3; i++) axis[i] /= an;
    double beta = 0;
    const double cx[4] = {x0, x1, x0, x1}, cy[4] = {y0, y0, y1, y1};
    for (int k = 0; k < 4; k++) {
        double v[3];
        pixel_dir(s, cx[k], cy[k], v);
        double cr[3] = {axis[1] * v[2] - axis[2] * v[1], axis[2] * v[0] - axis[0] * v[2], axis[0] * v[1] - axis[1] * v[0]};
        beta = std::max(beta, std::atan2(std::sqrt(dot3(cr, cr)), dot3(axis, v)));
    }
    out.clear();
    for (int64_t g = 0; g < s->n; g++) {
        const Prepared& P = s->prep[g];
        if (s->cfg.eval_mode == 1) {  // 2D splat: disc (projected mean, radius) vs the tile rectangle
            if (!P.valid) continue;
            const double qx = std::min(std::max(P.pm[0], x0), x1), qy = std::min(std::max(P.pm[1], y0), y1);
            const double ddx = qx - P.pm[0], ddy = qy - P.pm[1];
            if (ddx * ddx + ddy * ddy <= P.radius2d * P.radius2d * (1.0 + 1e-9)) out.push_back(g);
            continue;
        }
        if (!(P.tau > 0) || (P.inside && !P.gauss_margin)) continue;
        double d[3] = {P.mu[0] - s->o[0], P.mu[1] - s->o[1], P.mu[2] - s->o[2]};
        double dl = std::sqrt(dot3(d, d));
        if (dl <= P.radius * (1.0 + 1e-9)) { out.push_back(g); continue; }
        double cr[3] = {axis[1] * d[2] - axis[2] * d[1], axis[2] * d[0] - axis[0] * d[2], axis[0] * d[1] - axis[1] * d[0]};
        double gamma = std::atan2(std::sqrt(dot3(cr, cr)), dot3(axis, d));
        if (gamma <= beta + std::asin(std::min(1.0, P.radius / dl)) + 1e-9) out.push_back(g);
    }
}

// Exact min of |u|^2 subject to a_k . u + b_k >= 0 (k < nc), by active-set enumeration:
// every subset of <= 3 constraints held with equality, least-norm point, keep if feasible.
double qp_min_norm(int nc, const double a[][3], const double* b) {
    double best = std::numeric_limits<double>::infinity();
    auto feasible = [&](const double* u) {
        for (int k = 0; k < nc; k++) {
            double an = std::sqrt(dot3(a[k], a[k]));
            double un = std::sqrt(dot3(u, u));
            double val = dot3(a[k], u) + b[k];
            if (val < -1e-10 * (an * un + std::fabs(b[k]))) return false;
        }
        return true;
    };
    auto consider = [&](const double* u) {
        if (feasible(u)) best = std::min(best, dot3(u, u));
    };
    double zero[3] = {0, 0, 0};
    consider(zero);
    for (int i = 0; i < nc; i++) {  // one active plane: u = -b a / |a|^2
        double aa = dot3(a[i], a[i]);
        double u[3] = {-b[i] * a[i][0] / aa, -b[i] * a[i][1] / aa, -b[i] * a[i][2] / aa};
        consider(u);
    }
    for (int i = 0; i < nc; i++)
        for (int j = i + 1; j < nc; j++) {  // two active: u = A^T (A A^T)^-1 (-b)
            double g11 = dot3(a[i], a[i]), g12 = dot3(a[i], a[j]), g22 = dot3(a[j], a[j]);
            double det = g11 * g22 - g12 * g12;
            if (det <= 1e-14 * g11 * g22) continue;
            double l1 = (-b[i] * g22 + b[j] * g12) / det;
            double l2 = (-b[j] * g11 + b[i] * g12) / det;
            double u[3];
            for (int m = 0; m < 3; m++) u[m] = l1 * a[i][m] + l2 * a[j][m];
            consider(u);
        }
    for (int i = 0; i < nc; i++)
        for (int j = i + 1; j < nc; j++)
            for (int k = j + 1; k < nc; k++) {  // three active: solve the 3x3 system
                M3 Am = {{a[i][0], a[i][1], a[i][2]}, {a[j][0], a[j][1], a[j][2]}, {a[k][0], a[k][1], a[k][2]}};
                double d = det3(Am);
                double sc = std::sqrt(dot3(a[i], a[i]) * dot3(a[j], a[j]) * dot3(a[k], a[k]));
                if (std::fabs(d) <= 1e-12 * sc) continue;
                M3 Ai;
                inv3(Am, Ai);
                double rhs[3] = {-b[i], -b[j], -b[k]};
                double u[3] = {dot3(Ai[0], rhs), dot3(Ai[1], rhs), dot3(Ai[2], rhs)};
                consider(u);
            }
    return best;
}

// Min rho^2 over the frustum of rect [x0,x1]x[y0,y1] ∩ {z >= near} (readings 20-21).
// The frustum half-spaces are written in view space, then pulled back to Gaussian space
// with T_view^T (Eq. 5; T_view = V T built with the filtered scales).
double frustum_min_rho2(const orc_scene* s, int64_t g, double x0, double x1, double y0, double y1) {
    const orc_camera& cam = s->cam;
    const Prepared& P = s->prep[g];
    M3 R;
    quat_rot(&s->quats[4 * g], R);
    // view-space columns of T_view's linear part: M = Rv R diag(sqrt(shat))
    M3 M;
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double v = 0;
            for (int m = 0; m < 3; m++) v += s->Rv[i][m] * R[m][j];
            M[i][j] = v * std::sqrt(P.shat[j]);
        }
    // view-space half-spaces n . x + d >= 0
    double n[5][3] = {{cam.fx, 0, cam.cx - x0}, {-cam.fx, 0, -(cam.cx - x1)},
                      {0, cam.fy, cam.cy - y0}, {0, -cam.fy, -(cam.cy - y1)}, {0, 0, 1}};
    double dd[5] = {0, 0, 0, 0, -cam.near_z};
    double a[5][3], b[5];
    for (int k = 0; k < 5; k++) {
        for (int j = 0; j < 3; j++) a[k][j] = n[k][0] * M[0][j] + n[k][1] * M[1][j] + n[k][2] * M[2][j];
        b[k] = dot3(n[k], P.muv) + dd[k];
    }
    return qp_min_norm(5, a, b);
}

}  // namespace

extern "C" {

orc_scene* orc_create(int64_t n, int32_t deg, const float* means, const float* scales, const float* quats,
                      const float* opac, const float* sh, const float* vtrain) {
    orc_scene* s = new orc_scene();
    s->n = n;
    s->deg = deg;
    int K = (deg + 1) * (deg + 1);
    s->means.assign(means, means + 3 * n);
    s->scales.assign(scales, scales + 3 * n);
    s->quats.assign(quats, quats + 4 * n);
    s->opac.assign(opac, opac + n);
    s->sh.assign(sh, sh + 3 * K * n);
    s->vtrain.assign(vtrain, vtrain + n);
    return s;
}

void orc_destroy(orc_scene* s) { delete s; }

int32_t orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int32_t orc_set_view(orc_scene* s, const orc_camera* cam, const orc_config* cfg) {
    s->cam = *cam;
    s->cfg = *cfg;
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++) s->Rv[i][j] = cam->world_to_view[4 * i + j];
        s->tv[i] = cam->world_to_view[4 * i + 3];
    }
    // The camera is the affine map x_v = Rv x + t as given (reading 37): the camera centre
    // and the world-space pixel rays use the exact inverse Rv^-1 (the float32 matrix is
    // orthonormal only to ~1e-7; Rv^T in its place moves z* by ~1e-5 relative near the near plane)
    inv3(s->Rv, s->Rvi);
    for (int i = 0; i < 3; i++)  // o = -Rv^-1 t
        s->o[i] = -(s->Rvi[i][0] * s->tv[0] + s->Rvi[i][1] * s->tv[1] + s->Rvi[i][2] * s->tv[2]);
    s->prep.assign(s->n, Prepared());
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < s->n; g++) prepare_one(s, g, s->prep[g]);
    s->have_view = true;
    return 0;
}

int32_t orc_gaussian(const orc_scene* s, int64_t g, double* out) {
    if (!s->have_view || g < 0 || g >= s->n) return -1;
    const Prepared& P = s->prep[g];
    out[ORC_G_VHAT] = P.vhat;
    out[ORC_G_VEFF] = P.veff;
    for (int i = 0; i < 3; i++) out[ORC_G_SHAT0 + i] = P.shat[i];
    out[ORC_G_A] = P.A;
    out[ORC_G_OA] = P.oA;
    out[ORC_G_TAU] = P.tau;
    out[ORC_G_VALID] = P.valid ? 1.0 : 0.0;
    out[ORC_G_INSIDE] = P.inside ? 1.0 : 0.0;
    out[ORC_G_INSIDE_RHO2] = P.inside_rho2;
    for (int i = 0; i < 3; i++) out[ORC_G_R + i] = P.rgb[i];
    for (int i = 0; i < 3; i++) out[ORC_G_MUV0 + i] = P.muv[i];
    return 0;
}

int32_t orc_render_pixels(const orc_scene* s, int64_t npix, const int32_t* px, const int32_t* py,
                          int32_t use_rejects, double* out_rgbT, uint32_t* out_flags, int32_t* out_nblend) {
    if (!s->have_view) return -1;
    // group pixels by 16x16 tile (for the tile-level reject only; results do not depend on it)
    int tw = (s->cam.width + 15) / 16;
    std::vector<int64_t> order(npix);
    for (int64_t i = 0; i < npix; i++) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
        int64_t ta = (int64_t)(py[a] / 16) * tw + px[a] / 16, tb = (int64_t)(py[b] / 16) * tw + px[b] / 16;
        return ta < tb || (ta == tb && a < b);
    });
    std::vector<std::pair<int64_t, int64_t>> groups;  // [begin, end) in order
    for (int64_t i = 0; i < npix;) {
        int64_t t = (int64_t)(py[order[i]] / 16) * tw + px[order[i]] / 16;
        int64_t j = i;
        while (j < npix && (int64_t)(py[order[j]] / 16) * tw + px[order[j]] / 16 == t) j++;
        groups.push_back({i, j});
        i = j;
    }
#pragma omp parallel
    {
        std::vector<int64_t> cand;
        std::vector<Contrib> cs;
#pragma omp for schedule(dynamic, 1)
        for (int64_t gi = 0; gi < (int64_t)groups.size(); gi++) {
            int64_t b = groups[gi].first, e = groups[gi].second;
            int64_t p0 = order[b];
            if (use_rejects) tile_candidates(s, px[p0] / 16, py[p0] / 16, cand);
            for (int64_t k = b; k < e; k++) {
                int64_t p = order[k];
                pixel_contribs(s, use_rejects ? &cand : nullptr, px[p], py[p], use_rejects != 0, cs);
                blend(s, cs, &out_rgbT[4 * p], &out_flags[p], &out_nblend[p]);
            }
        }
    }
    return 0;
}

int32_t orc_gaussians(const orc_scene* s, double* out) {
    if (!s->have_view) return -1;
    for (int64_t g = 0; g < s->n; g++) orc_gaussian(s, g, out + g * ORC_G_COUNT);
    return 0;
}

int64_t orc_pixel_contribs(const orc_scene* s, int32_t px, int32_t py, double* out, int64_t cap) {
    if (!s->have_view) return -1;
    std::vector<Contrib> cs;
    pixel_contribs(s, nullptr, px, py, false, cs);
    double rgbT[4];
    uint32_t f;
    int32_t nb;
    blend(s, cs, rgbT, &f, &nb);  // sets tie flags
    for (int64_t i = 0; i < (int64_t)cs.size() && i < cap; i++) {
        double* o = out + i * ORC_C_COUNT;
        o[ORC_C_Z] = cs[i].z;
        o[ORC_C_ALPHA] = cs[i].alpha;
        o[ORC_C_RHO2] = cs[i].rho2;
        o[ORC_C_TAU] = cs[i].tau;
        o[ORC_C_G] = (double)cs[i].g;
        o[ORC_C_R] = cs[i].rgb[0];
        o[ORC_C_GG] = cs[i].rgb[1];
        o[ORC_C_B] = cs[i].rgb[2];
        o[ORC_C_INCLUDED] = cs[i].included ? 1.0 : 0.0;
        o[ORC_C_FLAGS] = (double)cs[i].flags;
    }
    return (int64_t)cs.size();
}

int32_t orc_frustum_min_rho2(const orc_scene* s, int64_t m, const int64_t* g, const double* rects, double* out) {
    if (!s->have_view) return -1;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < m; i++)
        out[i] = frustum_min_rho2(s, g[i], rects[4 * i], rects[4 * i + 1], rects[4 * i + 2], rects[4 * i + 3]);
    return 0;
}

// test hook: SH basis values (pinned against scipy's spherical harmonics)
void orc_sh_basis(const double* d, double* Y16) { sh_basis(d, Y16); }

// test hook: the raw QP, so tests can pin it against brute force on arbitrary constraints
double orc_qp_min_norm(int32_t nc, const double* a, const double* b) {
    return qp_min_norm(nc, reinterpret_cast<const double(*)[3]>(a), b);
}

}  // extern "C"

// Eq. 6, frustum membership of the mean point as in S:154 with the culling frustum
// of reading 20: near plane and the pixel-centre planes; f = max(fx, fy) (reading 10).
int32_t orc_vtrain(const orc_scene* s, int32_t n_cams, const orc_camera* cams, double* out, int32_t* amb) {
    const double INF = std::numeric_limits<double>::infinity();
#pragma omp parallel for schedule(static)
    for (int64_t g = 0; g < s->n; g++) {
        const double* mu = &s->means[3 * g];
        double best = -INF;
        int32_t a = 0;
        for (int32_t c = 0; c < n_cams; c++) {
            const orc_camera& cam = cams[c];
            const double* M = cam.world_to_view;
            double v[3];
            for (int i = 0; i < 3; i++) v[i] = M[4 * i] * mu[0] + M[4 * i + 1] * mu[1] + M[4 * i + 2] * mu[2] + M[4 * i + 3];
            const double z = v[2];
            const double eps = 1e-9;
            if (std::fabs(z - cam.near_z) <= eps * std::max(1.0, std::fabs(z))) a = 1;
            if (!(z >= cam.near_z)) continue;
            const double px = cam.fx * v[0] / z + cam.cx, py = cam.fy * v[1] / z + cam.cy;
            const double bx[2] = {0.5, cam.width - 0.5}, by[2] = {0.5, cam.height - 0.5};
            for (int k = 0; k < 2; k++) {
                if (std::fabs(px - bx[k]) <= eps * std::max(1.0, std::fabs(px))) a = 1;
                if (std::fabs(py - by[k]) <= eps * std::max(1.0, std::fabs(py))) a = 1;
            }
            if (px < bx[0] || px > bx[1] || py < by[0] || py > by[1]) continue;
            best = std::max(best, std::max(cam.fx, cam.fy) / z);
        }
        out[g] = best > 0 ? best : INF;
        if (amb) amb[g] = a;
    }
    return 0;
}
