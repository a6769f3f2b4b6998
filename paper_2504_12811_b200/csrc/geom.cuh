// geom.cuh — FP64 device geometry shared by K1 (preprocess) and K3 (tile cull).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

namespace aaa {

__device__ __forceinline__ double dot3(const double* a, const double* b) {
    return fma(a[0], b[0], fma(a[1], b[1], a[2] * b[2]));
}
__device__ __forceinline__ void cross3(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}
__device__ __forceinline__ void mat3_vec(const double* M, const double* v, double* o) {
    for (int i = 0; i < 3; i++) o[i] = M[3 * i] * v[0] + M[3 * i + 1] * v[1] + M[3 * i + 2] * v[2];
}
__device__ __forceinline__ void mat3_mul(const double* A, const double* B, double* C) {
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) C[3 * i + j] = A[3 * i] * B[j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}
// rotation matrix (row-major) of a normalised (w,x,y,z) quaternion (Eq. 3 R)
__device__ __forceinline__ void quat_to_rot(float4 q, double* R) {
    double w = q.x, x = q.y, y = q.z, z = q.w;
    double inv = 1.0 / sqrt(w * w + x * x + y * y + z * z);  // normalise in FP64
    w *= inv; x *= inv; y *= inv; z *= inv;
    R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z);       R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);       R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);       R[7] = 2.0 * (y * z + w * x);       R[8] = 1.0 - 2.0 * (x * x + y * y);
}

// Minimum over the box [x0,x1]x[y0,y1] of q = a x^2 + 2b xy + c y^2 + 2d x + 2e y + f:
// the 4 corners, the 4 edge critical points, and the interior critical point when q is
// positive definite. Exact for any quadratic (the minimum of a quadratic over a box lies at
// one of these candidates).
__device__ __forceinline__ double quad_box_min(double a, double b, double c, double d, double e, double f,
                                               double x0, double x1, double y0, double y1) {
    auto q = [&](double x, double y) { return (a * x + 2.0 * b * y + 2.0 * d) * x + (c * y + 2.0 * e) * y + f; };
    double m = fmin(fmin(q(x0, y0), q(x1, y0)), fmin(q(x0, y1), q(x1, y1)));
    if (c > 0.0) {
        double ya = -(b * x0 + e) / c, yb = -(b * x1 + e) / c;
        if (ya > y0 && ya < y1) m = fmin(m, q(x0, ya));
        if (yb > y0 && yb < y1) m = fmin(m, q(x1, yb));
    }
    if (a > 0.0) {
        double xa = -(b * y0 + d) / a, xb = -(b * y1 + d) / a;
        if (xa > x0 && xa < x1) m = fmin(m, q(xa, y0));
        if (xb > x0 && xb < x1) m = fmin(m, q(xb, y1));
    }
    double det = a * c - b * b;
    if (a > 0.0 && det > 0.0) {
        double xs = (b * e - c * d) / det, ys = (b * d - a * e) / det;
        if (xs >= x0 && xs <= x1 && ys >= y0 && ys <= y1) m = fmin(m, q(xs, ys));
    }
    return m;
}

// quad_box_min with the per-Gaussian parts precomputed: ia = 1/a (a > 0) else 0, ic likewise,
// (xs, ys, qi) the interior critical point and value (qi = +inf unless q is positive definite).
__device__ __forceinline__ double quad_box_min_pre(double a, double b, double c, double d, double e, double f,
                                                   double ia, double ic, double xs, double ys, double qi,
                                                   double x0, double x1, double y0, double y1) {
    auto q = [&](double x, double y) { return (a * x + 2.0 * b * y + 2.0 * d) * x + (c * y + 2.0 * e) * y + f; };
    double m = fmin(fmin(q(x0, y0), q(x1, y0)), fmin(q(x0, y1), q(x1, y1)));
    if (ic > 0.0) {
        double ya = -(b * x0 + e) * ic, yb = -(b * x1 + e) * ic;
        if (ya > y0 && ya < y1) m = fmin(m, q(x0, ya));
        if (yb > y0 && yb < y1) m = fmin(m, q(x1, yb));
    }
    if (ia > 0.0) {
        double xa = -(b * y0 + d) * ia, xb = -(b * y1 + d) * ia;
        if (xa > x0 && xa < x1) m = fmin(m, q(xa, y0));
        if (xb > x0 && xb < x1) m = fmin(m, q(xb, y1));
    }
    if (xs >= x0 && xs <= x1 && ys >= y0 && ys <= y1) m = fmin(m, qi);
    return m;
}

// FP32 image of quad_box_min_pre's coefficients (K3's fast path).
struct QuadF {
    float a, b, c, d, e, f, ia, ic, xs, ys, qi;
};

// Sign of quad_box_min_pre decided in FP32 with a guard band, FP64 only inside the band.
// Every FP32 candidate value differs from its FP64 counterpart by at most ~8 * 2^-24 * S, where
// S = |a|X^2 + 2|b|XY + 2|d|X + |c|Y^2 + 2|e|Y + |f| (X, Y the box's largest |x|, |y|): one
// rounding per coefficient, per coordinate and per FMA of the Horner form, each bounded by the
// magnitude of the terms; an edge critical point computed in FP32 moves q by O(c dy^2), second
// order. With the band at 2^-17 S (16x that bound) a decision outside the band is the FP64
// decision, so the kept set is bit-identical to the all-FP64 test.
// Returns 1 (q < 0 somewhere: keep), 0 (reject), -1 (inside the band: re-test in FP64).
__device__ __forceinline__ int quad_box_sign_f32(const QuadF& Q, float x0, float x1, float y0, float y1) {
    auto q = [&](float x, float y) {
        return fmaf(fmaf(Q.a, x, fmaf(2.f * Q.b, y, 2.f * Q.d)), x, fmaf(fmaf(Q.c, y, 2.f * Q.e), y, Q.f));
    };
    float m = fminf(fminf(q(x0, y0), q(x1, y0)), fminf(q(x0, y1), q(x1, y1)));
    if (Q.ic > 0.f) {
        const float ya = -fmaf(Q.b, x0, Q.e) * Q.ic, yb = -fmaf(Q.b, x1, Q.e) * Q.ic;
        if (ya > y0 && ya < y1) m = fminf(m, q(x0, ya));
        if (yb > y0 && yb < y1) m = fminf(m, q(x1, yb));
    }
    if (Q.ia > 0.f) {
        const float xa = -fmaf(Q.b, y0, Q.d) * Q.ia, xb = -fmaf(Q.b, y1, Q.d) * Q.ia;
        if (xa > x0 && xa < x1) m = fminf(m, q(xa, y0));
        if (xb > x0 && xb < x1) m = fminf(m, q(xb, y1));
    }
    if (Q.xs >= x0 && Q.xs <= x1 && Q.ys >= y0 && Q.ys <= y1) m = fminf(m, Q.qi);
    const float X = fmaxf(fabsf(x0), fabsf(x1)), Y = fmaxf(fabsf(y0), fabsf(y1));
    const float S = fmaf(fmaf(fabsf(Q.a), X, 2.f * fmaf(fabsf(Q.b), Y, fabsf(Q.d))), X,
                         fmaf(fmaf(fabsf(Q.c), Y, 2.f * fabsf(Q.e)), Y, fabsf(Q.f)));
    // a non-finite or tiny scale (FP32 underflow of the coefficients) always takes the FP64 test
    if (!(S > 1e-30f && S < 1e30f)) return -1;
    const float band = S * 0x1p-17f;
    if (m < -band) return 1;
    if (m > band) return 0;
    return -1;
}

// Exact minimum of rho^2 = |u|^2 over the frustum {pixel-centre rect [x0,x1]x[y0,y1]} ∩
// {z >= near} (readings 20-21). The five view-space half-spaces n.x + d >= 0 are
// pulled back to Gaussian space through x = M u + mu_v (Eq. 5); the convex QP is solved by
// trying every set of <= 3 active constraints (least-norm point on their intersection) and
// keeping feasible candidates. Used for Gaussians whose tau-ellipsoid reaches z <= near, where
// the paper's 2-plane/3-edge shortcut is not exact.
static __device__ __noinline__ double frustum_qp_min(const double* M, const double* muv, double fx, double fy, double cx,
                                              double cy, double near_z, double x0, double x1, double y0,
                                              double y1) {
    double n[5][3] = {{fx, 0.0, cx - x0}, {-fx, 0.0, x1 - cx}, {0.0, fy, cy - y0}, {0.0, -fy, y1 - cy},
                      {0.0, 0.0, 1.0}};
    double a[5][3], b[5], an[5];
    for (int k = 0; k < 5; k++) {
        for (int j = 0; j < 3; j++) a[k][j] = n[k][0] * M[j] + n[k][1] * M[3 + j] + n[k][2] * M[6 + j];
        b[k] = n[k][0] * muv[0] + n[k][1] * muv[1] + n[k][2] * muv[2] - (k == 4 ? near_z : 0.0);
        an[k] = sqrt(dot3(a[k], a[k]));
    }
    double best = CUDART_INF;
    for (int mask = 0; mask < 32; mask++) {
        int cnt = __popc(mask);
        if (cnt > 3) continue;
        int id[3];
        int m = 0;
        for (int k = 0; k < 5; k++)
            if (mask & (1 << k)) id[m++] = k;
        double u[3] = {0.0, 0.0, 0.0};
        if (cnt == 1) {
            double s = -b[id[0]] / dot3(a[id[0]], a[id[0]]);
            for (int j = 0; j < 3; j++) u[j] = s * a[id[0]][j];
        } else if (cnt == 2) {
            const double *p = a[id[0]], *q = a[id[1]];
            double g11 = dot3(p, p), g12 = dot3(p, q), g22 = dot3(q, q);
            double det = g11 * g22 - g12 * g12;
            if (!(det > 1e-14 * g11 * g22)) continue;
            double l1 = (-b[id[0]] * g22 + b[id[1]] * g12) / det;
            double l2 = (-b[id[1]] * g11 + b[id[0]] * g12) / det;
            for (int j = 0; j < 3; j++) u[j] = l1 * p[j] + l2 * q[j];
        } else if (cnt == 3) {
            const double *p = a[id[0]], *q = a[id[1]], *r = a[id[2]];
            double qr[3], rp[3], pq[3];
            cross3(q, r, qr);
            cross3(r, p, rp);
            cross3(p, q, pq);
            double det = dot3(p, qr);
            if (!(fabs(det) > 1e-12 * an[id[0]] * an[id[1]] * an[id[2]])) continue;
            // solve [p;q;r] u = -b via the adjugate (Cramer)
            for (int j = 0; j < 3; j++) u[j] = -(b[id[0]] * qr[j] + b[id[1]] * rp[j] + b[id[2]] * pq[j]) / det;
        }
        double un = sqrt(dot3(u, u));
        bool ok = true;
        for (int k = 0; k < 5 && ok; k++)
            ok = dot3(a[k], u) + b[k] >= -1e-10 * (an[k] * un + fabs(b[k]));
        if (ok) best = fmin(best, dot3(u, u));
    }
    return best;
}

}  // namespace aaa
