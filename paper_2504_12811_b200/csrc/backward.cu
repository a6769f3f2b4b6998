// backward.cu — gradients of a scalar loss through the forward render (the paper
// trains with this rasterizer). Two kernels:
//
//  KB6 (per pixel): replays the pixel's blended contributions recorded by K6/K6s in their exact
//      blend order and back-propagates the front-to-back compositing (reading 3)
//          C = sum_i alpha_i c_i T_i + T_n bg,  T_{i+1} = T_i (1 - alpha_i)
//      in reverse (T_i = T_{i+1} / (1 - alpha_i), the colour behind i accumulated), then
//      alpha = oA exp(-rho^2 / 2) (unless clamped at alpha_max) and the 3D evaluation
//      rho^2(p) = |c x w(p)|^2 / |w(p)|^2, w(p) = W r(p) (DESIGN K6):
//          d rho^2 / d c = 2 (w x u) / Q,   d rho^2 / d w = 2 (u x c) / Q - 2 rho^2 w / Q,
//      u = c x w, Q = |w|^2; accumulated per Gaussian into (dL/dc, dL/dW, dL/doA, dL/drgb).
//  KB1 (per Gaussian): chains those through K1's per-Gaussian map theta = (mu, s, q, o) ->
//      (c, W, oA, rgb) — quaternion normalisation, the adaptive filter (Eq. 6, 12, 13), the
//      amplitude A (Eq. 12), W = diag(1/sigma_hat) (R_v R)^T, c = -W mu_v, SH colour — by forward-
//      mode dual numbers over the 11 inputs (the same FP64 formulas as K1); SH gradients are
//      dL/drgb x basis.
// The contribution set (tau cutoff, near plane, culling, early termination) is held fixed: its
// boundaries carry no derivative (as in 3DGS). v_train is an input and is not differentiated.
#include <math_constants.h>

#include "aaa_internal.cuh"
#include "geom.cuh"

namespace aaa {

// ------------------------------------------------------------------ KB6
__global__ void __launch_bounds__(128) k_bwd_pixels(ViewParams vp, BwdArgs ba) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t npx = (int64_t)vp.width * vp.height;
    if (p >= npx) return;
    const int px = (int)(p % vp.width), py = (int)(p / vp.width);
    uint32_t n = ba.rec_n[p];
    if (n > ba.rec_cap) {
        atomicAdd(ba.overflow, 1u);
        return;
    }
    const float2* rec = ba.rec + p * ba.rec_cap;
    const size_t plane = (size_t)npx;
    const float dC[3] = {ba.dL_drgb[p], ba.dL_drgb[plane + p], ba.dL_drgb[2 * plane + p]};
    const float dT = ba.dL_dT ? ba.dL_dT[p] : 0.f;
    // final transmittance, exactly as the forward blend computed it
    float Tn = 1.f;
    for (uint32_t i = 0; i < n; i++) Tn = Tn * (1.f - rec[i].y);
    const float pxf = px + 0.5f, pyf = py + 0.5f;
    const float rx = (pxf - (float)vp.cx) * (float)vp.inv_fx, ry = (pyf - (float)vp.cy) * (float)vp.inv_fy;
    float B[3] = {vp.bg[0], vp.bg[1], vp.bg[2]};  // colour behind entry i, in units of T_{i+1}
    float T = Tn;
    for (int i = (int)n - 1; i >= 0; i--) {
        const uint32_t g = __float_as_uint(rec[i].x);
        const float a = rec[i].y;
        const float Ti = T / (1.f - a);
        const float4 col = __ldg(&ba.color[g]);
        const float c3[3] = {col.x, col.y, col.z};
        float dA = -dT * Tn / (1.f - a);
        float* acc = ba.acc + (size_t)g * BWD_ACC;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            dA += dC[k] * Ti * (c3[k] - B[k]);
            atomicAdd(&acc[13 + k], dC[k] * a * Ti);  // dL/drgb
            B[k] = a * c3[k] + (1.f - a) * B[k];
        }
        T = Ti;
        // alpha = min(alpha_max, oA exp(-rho^2/2)): no gradient through the clamp
        if (a >= vp.alpha_max) continue;
        const float4* r = ba.raster + (size_t)g * RASTER_REC_F4;
        const float4 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3], r4 = r[4], r5 = r[5], r6 = r[6];
        const float dx = pxf - r0.x, dy = pyf - r0.y;
        const float u0 = fmaf(dy, r2.z, fmaf(dx, r1.w, r1.x));
        const float u1 = fmaf(dy, r2.w, fmaf(dx, r2.x, r1.y));
        const float u2 = fmaf(dy, r3.x, fmaf(dx, r2.y, r1.z));
        const float w0 = fmaf(dy, r4.w, fmaf(dx, r4.x, r3.y));
        const float w1 = fmaf(dy, r5.x, fmaf(dx, r4.y, r3.z));
        const float w2 = fmaf(dy, r5.y, fmaf(dx, r4.z, r3.w));
        const float c0 = r6.y, c1 = r6.z, c2 = r6.w;
        const float N = u0 * u0 + u1 * u1 + u2 * u2, Q = w0 * w0 + w1 * w1 + w2 * w2;
        const float iQ = 1.f / Q, rho2 = N * iQ;
        const float oA = r0.z;
        atomicAdd(&acc[12], dA * __expf(-0.5f * rho2));  // dL/doA
        const float dR = -0.5f * a * dA;                   // dL/drho^2
        // d rho^2 / d c = 2 (w x u) / Q
        const float s = 2.f * dR * iQ;
        atomicAdd(&acc[0], s * (w1 * u2 - w2 * u1));
        atomicAdd(&acc[1], s * (w2 * u0 - w0 * u2));
        atomicAdd(&acc[2], s * (w0 * u1 - w1 * u0));
        // d rho^2 / d w = 2 (u x c) / Q - 2 rho^2 w / Q; dL/dW = (dL/dw) r^T
        const float gw0 = s * ((u1 * c2 - u2 * c1) - rho2 * w0);
        const float gw1 = s * ((u2 * c0 - u0 * c2) - rho2 * w1);
        const float gw2 = s * ((u0 * c1 - u1 * c0) - rho2 * w2);
        const float gw[3] = {gw0, gw1, gw2}, rr[3] = {rx, ry, 1.f};
#pragma unroll
        for (int j = 0; j < 3; j++)
#pragma unroll
            for (int k = 0; k < 3; k++) atomicAdd(&acc[3 + 3 * j + k], gw[j] * rr[k]);
        (void)oA;
    }
}

// ------------------------------------------------------------------ dual numbers for KB1
constexpr int ND = 11;  // d/d(mu 3, s 3, q 4, o 1)
struct Dn {
    double v, d[ND];
};
__device__ __forceinline__ Dn dconst(double v) {
    Dn r;
    r.v = v;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = 0.0;
    return r;
}
__device__ __forceinline__ Dn dvar(double v, int k) {
    Dn r = dconst(v);
    r.d[k] = 1.0;
    return r;
}
__device__ __forceinline__ Dn operator+(const Dn& a, const Dn& b) {
    Dn r;
    r.v = a.v + b.v;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = a.d[i] + b.d[i];
    return r;
}
__device__ __forceinline__ Dn operator-(const Dn& a, const Dn& b) {
    Dn r;
    r.v = a.v - b.v;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = a.d[i] - b.d[i];
    return r;
}
__device__ __forceinline__ Dn operator-(const Dn& a) {
    Dn r;
    r.v = -a.v;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = -a.d[i];
    return r;
}
__device__ __forceinline__ Dn operator*(const Dn& a, const Dn& b) {
    Dn r;
    r.v = a.v * b.v;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
    return r;
}
__device__ __forceinline__ Dn operator*(const Dn& a, double b) {
    Dn r;
    r.v = a.v * b;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = a.d[i] * b;
    return r;
}
__device__ __forceinline__ Dn operator*(double b, const Dn& a) { return a * b; }
__device__ __forceinline__ Dn operator+(const Dn& a, double b) {
    Dn r = a;
    r.v += b;
    return r;
}
__device__ __forceinline__ Dn operator/(const Dn& a, const Dn& b) {
    Dn r;
    const double ib = 1.0 / b.v;
    r.v = a.v * ib;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = (a.d[i] - r.v * b.d[i]) * ib;
    return r;
}
__device__ __forceinline__ Dn operator/(double a, const Dn& b) { return dconst(a) / b; }
__device__ __forceinline__ Dn dsqrt(const Dn& a) {
    Dn r;
    r.v = sqrt(a.v);
    const double h = r.v > 0.0 ? 0.5 / r.v : 0.0;
#pragma unroll
    for (int i = 0; i < ND; i++) r.d[i] = a.d[i] * h;
    return r;
}
__device__ __forceinline__ double dot_up(const Dn& x, int k) { return x.d[k]; }

// ------------------------------------------------------------------ KB1
__global__ void __launch_bounds__(64) k_bwd_gaussians(SceneDev sc, ViewParams vp, BwdArgs ba) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= sc.n) return;
    const float* acc = ba.acc + (size_t)g * BWD_ACC;
    const int K = (sc.sh_degree + 1) * (sc.sh_degree + 1);
    float up[BWD_ACC];
    bool any = false;
#pragma unroll
    for (int i = 0; i < BWD_ACC; i++) {
        up[i] = acc[i];
        any |= up[i] != 0.f;
    }
    double grad[ND];
#pragma unroll
    for (int i = 0; i < ND; i++) grad[i] = 0.0;
    const int64_t go = sc.perm ? (int64_t)sc.perm[g] : g;  // the caller's index of Gaussian g
    float* dsh = ba.d_sh + (size_t)go * K * 3;
    if (!any) {
        for (int i = 0; i < 3; i++) ba.d_means[3 * go + i] = 0.f, ba.d_scales[3 * go + i] = 0.f;
        for (int i = 0; i < 4; i++) ba.d_quats[4 * go + i] = 0.f;
        ba.d_opac[go] = 0.f;
        for (int i = 0; i < 3 * K; i++) dsh[i] = 0.f;
        return;
    }
    const float4 A4 = sc.geomA[g], B4 = sc.geomB[g], C4 = sc.geomC[g];
    const Dn mu[3] = {dvar(A4.x, 0), dvar(A4.y, 1), dvar(A4.z, 2)};
    const Dn s[3] = {dvar(B4.x, 3), dvar(B4.y, 4), dvar(B4.z, 5)};
    Dn qw = dvar(C4.x, 6), qx = dvar(C4.y, 7), qy = dvar(C4.z, 8), qz = dvar(C4.w, 9);
    const Dn op = dvar(A4.w, 10);
    // R(q), q normalised, as quat_to_rot
    {
        const Dn inv = 1.0 / dsqrt(qw * qw + qx * qx + qy * qy + qz * qz);
        qw = qw * inv; qx = qx * inv; qy = qy * inv; qz = qz * inv;
    }
    Dn R[9];
    R[0] = dconst(1.0) - 2.0 * (qy * qy + qz * qz); R[1] = 2.0 * (qx * qy - qw * qz); R[2] = 2.0 * (qx * qz + qw * qy);
    R[3] = 2.0 * (qx * qy + qw * qz); R[4] = dconst(1.0) - 2.0 * (qx * qx + qz * qz); R[5] = 2.0 * (qy * qz - qw * qx);
    R[6] = 2.0 * (qx * qz - qw * qy); R[7] = 2.0 * (qy * qz + qw * qx); R[8] = dconst(1.0) - 2.0 * (qx * qx + qy * qy);
    Dn muv[3];
    for (int i = 0; i < 3; i++) muv[i] = mu[0] * vp.Rv[3 * i] + mu[1] * vp.Rv[3 * i + 1] + mu[2] * vp.Rv[3 * i + 2] + vp.tv[i];
    // adaptive filter (Eq. 6, 13, 12): v_hat = f / mu_z, v' = min(v_train, v_hat), c_f = k / v'^2
    const double f = fmax(vp.fx, vp.fy);
    Dn cf = dconst(0.0);
    {
        const double vhat = muv[2].v > 0.0 ? f / muv[2].v : CUDART_INF;
        const double vt = (double)B4.w;
        if (vhat < vt) {
            const Dn vh = f / muv[2];
            cf = (double)vp.k / (vh * vh);
        } else if (!isinf(vt)) {
            cf = dconst((double)vp.k / (vt * vt));
        }
    }
    Dn shat[3], sig[3];
    for (int i = 0; i < 3; i++) {
        shat[i] = s[i] * s[i] + cf;
        sig[i] = dsqrt(shat[i]);
    }
    Dn dv[3];
    {
        Dn d0 = mu[0] + (-vp.o[0]), d1 = mu[1] + (-vp.o[1]), d2 = mu[2] + (-vp.o[2]);
        const Dn idn = 1.0 / dsqrt(d0 * d0 + d1 * d1 + d2 * d2);
        dv[0] = d0 * idn; dv[1] = d1 * idn; dv[2] = d2 * idn;
    }
    Dn Amp = dconst(1.0);
    if (cf.v > 0.0) {  // Eq. 12 with d' = R^T d
        const Dn dp0 = R[0] * dv[0] + R[3] * dv[1] + R[6] * dv[2];
        const Dn dp1 = R[1] * dv[0] + R[4] * dv[1] + R[7] * dv[2];
        const Dn dp2 = R[2] * dv[0] + R[5] * dv[1] + R[8] * dv[2];
        const Dn s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
        const Dn num = dp0 * dp0 * s2[1] * s2[2] + dp1 * dp1 * s2[0] * s2[2] + dp2 * dp2 * s2[0] * s2[1];
        const Dn den = dp0 * dp0 * shat[1] * shat[2] + dp1 * dp1 * shat[0] * shat[2] + dp2 * dp2 * shat[0] * shat[1];
        Amp = dsqrt(num / den);
    }
    const Dn oA = op * Amp;
    // W = diag(1/sig) R^T R_v^-1 (reading 37); c = -W mu_v
    auto addg = [&](const Dn& x, float u) {
        if (u != 0.f)
            for (int k = 0; k < ND; k++) grad[k] += (double)u * x.d[k];
    };
    Dn W[9];
    for (int j = 0; j < 3; j++) {
        const Dn isg = 1.0 / sig[j];
        for (int i = 0; i < 3; i++) {
            const Dn Qij = R[j] * vp.Rvi[i] + R[3 + j] * vp.Rvi[3 + i] + R[6 + j] * vp.Rvi[6 + i];
            W[3 * j + i] = Qij * isg;
        }
    }
    for (int j = 0; j < 3; j++) {
        const Dn cj = -(W[3 * j] * muv[0] + W[3 * j + 1] * muv[1] + W[3 * j + 2] * muv[2]);
        addg(cj, up[j]);
    }
    for (int k = 0; k < 9; k++) addg(W[k], up[3 + k]);
    addg(oA, up[12]);
    // SH colour (reading 15) at d: value and direction derivative
    const Dn x = dv[0], y = dv[1], z = dv[2];
    const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                          0.5462742152960396};
    const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                          -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    Dn b[16];
    b[0] = dconst(C0);
    b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    const Dn xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = C2[0] * xy; b[5] = C2[1] * yz; b[6] = C2[2] * (2.0 * zz - xx - yy); b[7] = C2[3] * xz;
    b[8] = C2[4] * (xx - yy);
    b[9] = C3[0] * y * (3.0 * xx - yy); b[10] = C3[1] * xy * z; b[11] = C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy); b[13] = C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = C3[5] * z * (xx - yy); b[15] = C3[6] * x * (xx - 3.0 * yy);
    for (int ch = 0; ch < 3; ch++) {
        Dn v = dconst(0.5);
        for (int k = 0; k < K; k++) {
            const int e = 3 * k + ch;
            const float4 chunk = sc.sh[(int64_t)(e >> 2) * sc.n + g];
            const float coef = (e & 3) == 0 ? chunk.x : (e & 3) == 1 ? chunk.y : (e & 3) == 2 ? chunk.z : chunk.w;
            v = v + b[k] * (double)coef;
        }
        const bool live = v.v > 0.0;  // colour = max(0, SH + 0.5)
        const float u = live ? up[13 + ch] : 0.f;
        addg(v, u);
        for (int k = 0; k < K; k++) dsh[3 * k + ch] = (float)((double)u * b[k].v);
    }
    for (int i = 0; i < 3; i++) ba.d_means[3 * go + i] = (float)grad[i];
    for (int i = 0; i < 3; i++) ba.d_scales[3 * go + i] = (float)grad[3 + i];
    for (int i = 0; i < 4; i++) ba.d_quats[4 * go + i] = (float)grad[6 + i];
    ba.d_opac[go] = (float)grad[10];
}

__global__ void k_max_u32(const uint32_t* __restrict__ a, size_t n, uint32_t* out) {
    uint32_t m = 0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        m = max(m, a[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

void launch_max_u32(const uint32_t* a, size_t n, uint32_t* out, cudaStream_t st) {
    if (n) k_max_u32<<<148 * 4, 256, 0, st>>>(a, n, out);
}

void launch_backward(const SceneDev& sc, const ViewParams& vp, const BwdArgs& ba, cudaStream_t st) {
    const int64_t npx = (int64_t)vp.width * vp.height;
    cudaMemsetAsync(ba.acc, 0, (size_t)(sc.n > 0 ? sc.n : 1) * BWD_ACC * sizeof(float), st);
    if (npx > 0) k_bwd_pixels<<<(unsigned)((npx + 127) / 128), 128, 0, st>>>(vp, ba);
    if (sc.n > 0) k_bwd_gaussians<<<(unsigned)((sc.n + 63) / 64), 64, 0, st>>>(sc, vp, ba);
}

}  // namespace aaa
