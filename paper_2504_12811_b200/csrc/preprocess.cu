// preprocess.cu — L0 scene packing and K1, the per-Gaussian preprocess kernel.
//
// K1 (one thread per Gaussian; HBM-bound: 48 B geometry + SH of survivors in, ~200 B out):
//   filter      v_hat = f/z (Eq. 6), v' = min(v_train, v_hat) (Eq. 13),
//               s_hat_i = s_i^2 + k/v'^2 and the perpendicular amplitude A (Eq. 12);
//   tau         2 ln(255 o A) (DESIGN reading 1); camera-inside discard;
//   bounds      view-space tangent-plane angles (Eq. 14-15) with the rotation step
//               (Eq. 16) and clamp (Eq. 17), full axis on a negative
//               discriminant; readings 16-19;
//   view cull   exact min of rho^2 over the view frustum — screen-space quadratic box
//               minimum when the ellipsoid lies beyond near, 5-plane QP otherwise;
//   key         tight lower bound of the per-ray max-response depth (reading 23);
//   records     K3 cull record (FP64 quadratic), K6 raster record (FP32, re-centred at p_ref).
// Geometry runs in FP64 (B200 has full-rate-class FP64 for this per-Gaussian work).
#include <math_constants.h>

#include <algorithm>

#include "aaa_internal.cuh"
#include "geom.cuh"

namespace aaa {

// ------------------------------------------------------------------ L0: validate + pack
__global__ void k_load_pack(int64_t n, int deg, const float* __restrict__ means, const float* __restrict__ scales,
                            const float* __restrict__ quats, const float* __restrict__ opac,
                            const float* __restrict__ sh, const float* __restrict__ vt, float4* geomA,
                            float4* geomB, float4* geomC, float4* shp, int chunks,
                            unsigned long long* first_bad) {
    int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    float mx = means[3 * g], my = means[3 * g + 1], mz = means[3 * g + 2];
    float sx = scales[3 * g], sy = scales[3 * g + 1], sz = scales[3 * g + 2];
    float qw = quats[4 * g], qx = quats[4 * g + 1], qy = quats[4 * g + 2], qz = quats[4 * g + 3];
    float o = opac[g], v = vt[g];
    bool ok = isfinite(mx) && isfinite(my) && isfinite(mz) && isfinite(sx) && isfinite(sy) && isfinite(sz) &&
              sx > 0.f && sy > 0.f && sz > 0.f && isfinite(qw) && isfinite(qx) && isfinite(qy) && isfinite(qz) &&
              o > 0.f && o < 1.f && v > 0.f && !isnan(v);
    double qn = sqrt((double)qw * qw + (double)qx * qx + (double)qy * qy + (double)qz * qz);
    ok = ok && qn > 0.0;
    int nf = 3 * (deg + 1) * (deg + 1);
    const float* s = sh + g * nf;
    for (int i = 0; i < nf; i++) ok = ok && isfinite(s[i]);
    if (!ok) atomicMin(first_bad, (unsigned long long)g);
    geomA[g] = make_float4(mx, my, mz, o);
    geomB[g] = make_float4(sx, sy, sz, v);
    // raw quaternion: K1 normalises it in FP64 (a f32-rounded unit quaternion would perturb R by ~1e-7)
    geomC[g] = ok ? make_float4(qw, qx, qy, qz) : make_float4(1.f, 0.f, 0.f, 0.f);
    for (int c = 0; c < chunks; c++) {
        float e[4];
        for (int j = 0; j < 4; j++) e[j] = (4 * c + j < nf) ? s[4 * c + j] : 0.f;
        shp[(int64_t)c * n + g] = make_float4(e[0], e[1], e[2], e[3]);
    }
}

void launch_load_pack(const aaa_gaussians& in, const float* dm, const float* ds, const float* dq, const float* dop,
                      const float* dsh, const float* dvt, SceneDev& sc, int64_t* d_bad, cudaStream_t st) {
    if (sc.n == 0) return;
    int threads = 256;
    unsigned blocks = (unsigned)((sc.n + threads - 1) / threads);
    k_load_pack<<<blocks, threads, 0, st>>>(sc.n, sc.sh_degree, dm, ds, dq, dop, dsh, dvt, sc.geomA, sc.geomB,
                                            sc.geomC, sc.sh, sc.sh_chunks, (unsigned long long*)d_bad);
}

// ------------------------------------------------------------------ L0: spatial order
// Morton (Z-order) codes of the means over the scene's bounding box, 10 bits per axis: sorting
// the scene by them at load puts spatially close Gaussians in the same warps of K1 (coherent
// culling and bounds branches) and next to each other in memory (K6 gathers their records).
__global__ void __launch_bounds__(256) k_aabb(const float4* __restrict__ A, int64_t n, float* __restrict__ out) {
    float lo[3] = {CUDART_INF_F, CUDART_INF_F, CUDART_INF_F}, hi[3] = {-CUDART_INF_F, -CUDART_INF_F, -CUDART_INF_F};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 a = __ldg(&A[i]);
        lo[0] = fminf(lo[0], a.x); lo[1] = fminf(lo[1], a.y); lo[2] = fminf(lo[2], a.z);
        hi[0] = fmaxf(hi[0], a.x); hi[1] = fmaxf(hi[1], a.y); hi[2] = fmaxf(hi[2], a.z);
    }
    __shared__ float s[6][8];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; k++) s[k][w] = lo[k], s[3 + k][w] = hi[k];
    __syncthreads();
    if (threadIdx.x < 6) {
        float v = s[threadIdx.x][0];
        for (int i = 1; i < (int)(blockDim.x >> 5); i++)
            v = threadIdx.x < 3 ? fminf(v, s[threadIdx.x][i]) : fmaxf(v, s[threadIdx.x][i]);
        out[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

int aabb_blocks(int64_t n) { return (int)std::min<int64_t>(1024, (n + 255) / 256); }

void launch_aabb(const SceneDev& sc, float* d_blk, cudaStream_t st) {
    k_aabb<<<aabb_blocks(sc.n), 256, 0, st>>>(sc.geomA, sc.n, d_blk);
}

__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void k_morton(const float4* __restrict__ A, int64_t n, float lx, float ly, float lz, float sx, float sy,
                         float sz, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float4 a = __ldg(&A[i]);
    auto q = [](float v) { return (uint32_t)fminf(fmaxf(v, 0.f), 1023.f); };
    keys[i] = spread10(q((a.x - lx) * sx)) | (spread10(q((a.y - ly) * sy)) << 1) | (spread10(q((a.z - lz) * sz)) << 2);
    vals[i] = (uint32_t)i;
}

void launch_morton_order(const SceneDev& sc, uint32_t* keys, uint32_t* vals, const float* lh, cudaStream_t st) {
    auto sc_of = [](float lo, float hi) { return hi > lo ? 1023.f / (hi - lo) : 0.f; };
    k_morton<<<(unsigned)((sc.n + 255) / 256), 256, 0, st>>>(sc.geomA, sc.n, lh[0], lh[1], lh[2], sc_of(lh[0], lh[3]),
                                                             sc_of(lh[1], lh[4]), sc_of(lh[2], lh[5]), keys, vals);
}

// out[c * n + i] = in[c * n + perm[i]] for each of `chunks` SoA chunks
__global__ void k_permute(const float4* __restrict__ in, float4* __restrict__ out, const uint32_t* __restrict__ perm,
                          int64_t n, int chunks) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = perm[i];
    for (int c = 0; c < chunks; c++) out[(int64_t)c * n + i] = __ldg(&in[(int64_t)c * n + p]);
}

void launch_permute(const float4* in, float4* out, const uint32_t* perm, int64_t n, int chunks, cudaStream_t st) {
    if (n > 0) k_permute<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, out, perm, n, chunks);
}

// ------------------------------------------------------------------ K1 helpers
// Spherical-harmonic colour, degree <= 3, 3DGS real basis (reading 15), direction d (unit).
__device__ __forceinline__ void sh_color(const float4* __restrict__ sh, int64_t n, int64_t g, int deg, float3 d,
                                         float out[3]) {
    float f[48];
    int chunks = (3 * (deg + 1) * (deg + 1) + 3) / 4;
#pragma unroll
    for (int c = 0; c < 12; c++) {
        if (c < chunks) {
            float4 v = __ldg(&sh[(int64_t)c * n + g]);
            f[4 * c] = v.x; f[4 * c + 1] = v.y; f[4 * c + 2] = v.z; f[4 * c + 3] = v.w;
        } else {
            f[4 * c] = f[4 * c + 1] = f[4 * c + 2] = f[4 * c + 3] = 0.f;
        }
    }
    const float C0 = 0.28209479177387814f, C1 = 0.4886025119029199f;
    const float C2[5] = {1.0925484305920792f, -1.0925484305920792f, 0.31539156525252005f, -1.0925484305920792f,
                         0.5462742152960396f};
    const float C3[7] = {-0.5900435899266435f, 2.890611442640554f, -0.4570457994644658f, 0.3731763325901154f,
                         -0.4570457994644658f, 1.445305721320277f, -0.5900435899266435f};
    float x = d.x, y = d.y, z = d.z;
    float b[16];
    b[0] = C0;
    b[1] = -C1 * y; b[2] = C1 * z; b[3] = -C1 * x;
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[4] = C2[0] * xy; b[5] = C2[1] * yz; b[6] = C2[2] * (2.f * zz - xx - yy); b[7] = C2[3] * xz;
    b[8] = C2[4] * (xx - yy);
    b[9] = C3[0] * y * (3.f * xx - yy); b[10] = C3[1] * xy * z; b[11] = C3[2] * y * (4.f * zz - xx - yy);
    b[12] = C3[3] * z * (2.f * zz - 3.f * xx - 3.f * yy); b[13] = C3[4] * x * (4.f * zz - xx - yy);
    b[14] = C3[5] * z * (xx - yy); b[15] = C3[6] * x * (xx - 3.f * yy);
    int K = (deg + 1) * (deg + 1);
#pragma unroll
    for (int ch = 0; ch < 3; ch++) {
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < 16; k++)
            if (k < K) acc = fmaf(b[k], f[3 * k + ch], acc);
        out[ch] = fmaxf(acc + 0.5f, 0.f);
    }
}

// One screen axis of the view-space bounds (Eq. 14-17). s_ii, s_i3, s33: the quadric
// coefficients of Appendix B; disc: cancellation-free discriminant s_i3^2 - s_ii s33.
// Returns false when no front-facing ray of this plane family meets the ellipsoid.
__device__ bool axis_bounds(double s_ii, double s_i3, double s33, double disc, double mu_i, double mu_z, double f,
                            double c, double& lo, double& hi) {
    if (!(disc >= 0.0)) {  // the ellipsoid meets the plane family's axis: full axis
        lo = -CUDART_INF;
        hi = CUDART_INF;
        return true;
    }
    double sq = sqrt(disc);
    double num = s_i3 + copysign(sq, s_i3);
    double mn = sqrt(mu_i * mu_i + mu_z * mu_z);
    if (num == 0.0 || mn == 0.0) {
        lo = -CUDART_INF;
        hi = CUDART_INF;
        return true;
    }
    // Angles are handled as unit vectors v(theta) = (sin theta, cos theta) in the (x|y, z) view
    // plane, so no trigonometry is needed: tan theta = v.x / v.y.
    // The two tangent-plane roots (Eq. 14-15): tan r1 = (s_i3 +- sqrt(D)) / s33 and, in the
    // cancellation-free form, tan r2 = s_ii / (s_i3 +- sqrt(D)).
    double n1 = rhypot(num, s33), n2 = rhypot(s_ii, num);
    double d1x = num * n1, d1y = s33 * n1, d2x = s_ii * n2, d2y = num * n2;
    const double imn = 1.0 / mn;
    double mx = mu_i * imn, my = mu_z * imn;  // v(theta_mu)
    // rotation step (Eq. 16, reading 16): representative of each root in (theta_mu - pi, theta_mu]
    // <=> sin(theta_mu - r) >= 0 <=> cross(v(theta_mu), v(r)) >= 0
    if (mx * d1y - my * d1x < 0.0) { d1x = -d1x; d1y = -d1y; }
    if (mx * d2y - my * d2x < 0.0) { d2x = -d2x; d2y = -d2y; }
    // theta1 = the larger representative (closer to theta_mu: larger cos), theta2 = smaller + pi
    double lx, ly, ux, uy;
    if (mx * d1x + my * d1y >= mx * d2x + my * d2y) {
        lx = d1x; ly = d1y; ux = -d2x; uy = -d2y;
    } else {
        lx = d2x; ly = d2y; ux = -d1x; uy = -d1y;
    }
    // The ray-angle interval [theta1, theta2] (< pi long, through theta_mu) meets the front half
    // (cos > 0) in one arc; an end behind the camera leaves that side unbounded (the clamp of
    // Eq. 17 at +-(pi/2 - eps) maps to |x| ~ 1e4 f, beyond any viewport).
    const bool lf = ly > 0.0, uf = uy > 0.0;
    if (!lf && !uf) return false;  // no front-facing ray of this plane family meets the ellipsoid
    lo = lf ? f * (lx / ly) + c : -CUDART_INF;
    hi = uf ? f * (ux / uy) + c : CUDART_INF;
    return true;
}

// ------------------------------------------------------------------ K1
// Table 5 "w/o 3D" (AAA_FLAG_NO_3D): the affine 2D splat of the filtered Gaussian.
// Sigma' = J (M M^T) J^T, J the perspective Jacobian at the mean (EWA); the cull record carries
// the exact 2D quadratic q(d) = d^T Sigma'^-1 d - tau around the projected mean, so K3's box
// minimum performs exact 2D tile / sub-tile culling; the key is the mean-depth code.
// (A separate kernel, so the 3D K1's register allocation is untouched; its prelude — filter,
// amplitude, tau — is the same arithmetic as K1's.)
__global__ void __launch_bounds__(128) k_preprocess_2d(SceneDev sc, ViewParams vp, ViewBufs vb) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= sc.n) return;
    const float4 A4 = __ldg(&sc.geomA[g]), B4 = __ldg(&sc.geomB[g]), C4 = __ldg(&sc.geomC[g]);
    vb.counts[g] = 0;
    const double mu[3] = {A4.x, A4.y, A4.z};
    const double s[3] = {B4.x, B4.y, B4.z};
    double R[9];
    quat_to_rot(C4, R);
    double muv[3];
    mat3_vec(vp.Rv, mu, muv);
    for (int i = 0; i < 3; i++) muv[i] += vp.tv[i];
    const double f = fmax(vp.fx, vp.fy);
    const double vhat = muv[2] > 0.0 ? f / muv[2] : CUDART_INF;
    const double veff = fmin((double)B4.w, vhat);
    const double cf = isinf(veff) ? 0.0 : (double)vp.k / (veff * veff);
    double shat[3], sig[3];
    for (int i = 0; i < 3; i++) {
        shat[i] = s[i] * s[i] + cf;
        sig[i] = sqrt(shat[i]);
    }
    double d[3] = {mu[0] - vp.o[0], mu[1] - vp.o[1], mu[2] - vp.o[2]};
    const double idn = 1.0 / sqrt(dot3(d, d));
    for (int i = 0; i < 3; i++) d[i] *= idn;
    double Amp = 1.0;
    if (cf > 0.0) {  // Eq. 12 with d' = R^T d (Eq. 11)
        const double dp0 = R[0] * d[0] + R[3] * d[1] + R[6] * d[2];
        const double dp1 = R[1] * d[0] + R[4] * d[1] + R[7] * d[2];
        const double dp2 = R[2] * d[0] + R[5] * d[1] + R[8] * d[2];
        const double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
        const double num = dp0 * dp0 * s2[1] * s2[2] + dp1 * dp1 * s2[0] * s2[2] + dp2 * dp2 * s2[0] * s2[1];
        const double den = dp0 * dp0 * shat[1] * shat[2] + dp1 * dp1 * shat[0] * shat[2] + dp2 * dp2 * shat[0] * shat[1];
        Amp = sqrt(num / den);
    }
    const double oA = (double)A4.w * Amp;
    double tau = 2.0 * log(255.0 * oA);
    if (vp.tau_mode == 1) tau = fmin((double)vp.tau_fixed, tau);
    if (!(tau > 0.0)) return;
    double Q[9], M[9];
    mat3_mul(vp.Rv, R, Q);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = Q[3 * i + j] * sig[j];

    const double x = muv[0], y = muv[1], z = muv[2];
    if (!(z >= vp.near_z)) return;
    // 3DGS mean-frustum rule: the projected mean within 1.3x the image about its centre
    {
        const double pmx = vp.fx * x / z + vp.cx, pmy = vp.fy * y / z + vp.cy;
        if (fabs(pmx - 0.5 * vp.width) > 0.65 * vp.width || fabs(pmy - 0.5 * vp.height) > 0.65 * vp.height) return;
    }
    double S[9];  // view-space covariance M M^T
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) S[3 * i + j] = dot3(&M[3 * i], &M[3 * j]);
    const double iz = 1.0 / z;
    const double J0[3] = {vp.fx * iz, 0.0, -vp.fx * x * iz * iz}, J1[3] = {0.0, vp.fy * iz, -vp.fy * y * iz * iz};
    double SJ0[3], SJ1[3];
    mat3_vec(S, J0, SJ0);
    mat3_vec(S, J1, SJ1);
    const double a = dot3(J0, SJ0), b = dot3(J0, SJ1), c = dot3(J1, SJ1);
    const double det = a * c - b * b;
    if (!(det > 0.0)) return;
    const double ca = c / det, cb = -b / det, cc = a / det;  // conic Sigma'^-1
    const double hm = 0.5 * (a + c), hd = 0.5 * (a - c);
    const double r = sqrt(tau * (hm + sqrt(hd * hd + b * b)));
    const double pmx = vp.fx * x * iz + vp.cx, pmy = vp.fy * y * iz + vp.cy;
    const double PAD = 1.0;
    const double ixlo = ceil(fmax(pmx - r - PAD - 0.5, -1.0)), ixhi = floor(fmin(pmx + r + PAD - 0.5, (double)vp.width));
    const double iylo = ceil(fmax(pmy - r - PAD - 0.5, -1.0)), iyhi = floor(fmin(pmy + r + PAD - 0.5, (double)vp.height));
    const int i0 = max(0, (int)ixlo), i1 = min(vp.width - 1, (int)ixhi);
    const int j0 = max(0, (int)iylo), j1 = min(vp.height - 1, (int)iyhi);
    if (i0 > i1 || j0 > j1) return;
    const float prx_f = (float)pmx, pry_f = (float)pmy;
    const double prx = prx_f, pry = pry_f;
    // q relative to p_ref = the f32-rounded projected mean: d = p - p_ref + e, e = p_ref - pm
    const double ex = prx - pmx, ey = pry - pmy;
    double qd = ca * ex + cb * ey, qe = cb * ex + cc * ey;
    double qf = ca * ex * ex + 2.0 * cb * ex * ey + cc * ey * ey - tau;
    const double px0 = i0 + 0.5, px1 = i1 + 0.5, py0 = j0 + 0.5, py1 = j1 + 0.5;
    if (!(quad_box_min(ca, cb, cc, qd, qe, qf, px0 - prx, px1 - prx, py0 - pry, py1 - pry) < 0.0)) return;
    int tx0 = i0 / TILE, tx1 = i1 / TILE, ty0 = j0 / TILE, ty1 = j1 / TILE;
    ty0 = max(ty0, vp.tile_row_begin);
    ty1 = min(ty1, vp.tile_row_end - 1);
    const double qmax = (double)((1u << vp.key_db) - 1u);
    const double um = vp.key_scale * log2(fmax(z, vp.key_near) / vp.key_near);
    const uint32_t zkey = (uint32_t)fmin(fmax(floor(um), 0.0), qmax);
    float rgb[3];
    sh_color(sc.sh, sc.n, g, sc.sh_degree, make_float3((float)d[0], (float)d[1], (float)d[2]), rgb);
    CullRec cu;
    cu.qa = ca; cu.qb = cb; cu.qc = cc; cu.qd = qd; cu.qe = qe; cu.qf = qf;
    cu.ia = 1.0 / ca;
    cu.ic = 1.0 / cc;
    const double dq = ca * cc - cb * cb;
    cu.xs = (cb * qe - cc * qd) / dq;
    cu.ys = (cb * qd - ca * qe) / dq;
    cu.qi = (ca * cu.xs + 2.0 * cb * cu.ys + 2.0 * qd) * cu.xs + (cc * cu.ys + 2.0 * qe) * cu.ys + qf;
    cu.pref_x = prx_f;
    cu.pref_y = pry_f;
    cu.tx0 = (uint16_t)tx0; cu.ty0 = (uint16_t)ty0; cu.tx1 = (uint16_t)tx1; cu.ty1 = (uint16_t)ty1;
    cu.i0 = (uint16_t)i0; cu.j0 = (uint16_t)j0; cu.i1 = (uint16_t)i1; cu.j1 = (uint16_t)j1;
    cu.cross_slot = -1;
    cu.zkey = zkey;
    vb.cull[g] = cu;
    // raster record (2D): [p_ref, oA, tau], [conic a, b, c, e.x], [e.y, -, -, -]
    float4* rr = vb.raster + g * RASTER_REC_F4;
    rr[0] = make_float4(prx_f, pry_f, (float)oA, (float)tau);
    rr[1] = make_float4((float)ca, (float)cb, (float)cc, (float)ex);
    rr[2] = make_float4((float)ey, 0.f, 0.f, 0.f);
    vb.color[g] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
    const uint32_t cnt = (ty0 <= ty1) ? (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1) : 0u;
    vb.counts[g] = cnt;
    atomicAdd(&vb.counters[CNT_VISIBLE], 1u);
}

#ifndef AAA_K1_MINB
#define AAA_K1_MINB 3  // 168 registers: 3 CTAs of 128 threads per SM (A/B: 0.78 -> 0.69 ms on c3)
#endif
// DBG: the parity-test instantiation that also writes the per-Gaussian debug fields
#ifndef AAA_K1_SPLIT
#define AAA_K1_SPLIT 0  // A/B on c3: K1 0.410 ms inline vs K1 + K1c 0.455 ms split
#endif
#ifndef AAA_K1_ITEMS
#define AAA_K1_ITEMS 1
#endif
// A/B (round 2, K1 ms without / with the sphere exit): c3 0.410 / 0.408, c4 inside 0.292 / 0.242,
// c4 wide 0.454 / 0.468, c4 zoom-out 0.475 / 0.493 — kept (whole frames: c4 inside +1.2%, others
// within 0.5%)
#ifndef AAA_K1_TMAX32
#define AAA_K1_TMAX32 1  // A/B (K1 ms, FP64 / FP32 log in the sphere exit): c3 0.395 / 0.387, c4 wide 0.459 / 0.449
#endif
#ifndef AAA_K1_SHPF
#define AAA_K1_SHPF 2  // A/B (K1 ms, 0 / 1 L2 / 2 L1): c3 0.404 / 0.394 / 0.394, c4 wide 0.465 / 0.458 / 0.458
#endif
#ifndef AAA_K1_SPHERE
#define AAA_K1_SPHERE 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

template <bool DBG>
__device__ __forceinline__ void k1_one(const SceneDev& sc, const ViewParams& vp, ViewBufs& vb, int64_t g);

// K1 is latency-bound at 12 warps per SM (FP64 registers). AAA_K1_ITEMS > 1: each thread walks
// AAA_K1_ITEMS Gaussians grid-strided and prefetches the next one's geometry (L1) and SH (L2)
// before working on the current one, so its loads are in flight during the FP64 work.
template <bool DBG>
__global__ void __launch_bounds__(128, AAA_K1_MINB) k_preprocess(SceneDev sc, ViewParams vp, ViewBufs vb) {
    if (AAA_K1_ITEMS == 1) {
        const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (g < sc.n) k1_one<DBG>(sc, vp, vb, g);
        return;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < sc.n; g += stride) {
        if (AAA_K1_ITEMS > 1 && g + stride < sc.n) {
            const int64_t gn = g + stride;
            prefetch_l1(&sc.geomA[gn]);
            prefetch_l1(&sc.geomB[gn]);
            prefetch_l1(&sc.geomC[gn]);
            const int chunks = (3 * (sc.sh_degree + 1) * (sc.sh_degree + 1) + 3) / 4;
            for (int c = 0; c < chunks; c++) prefetch_l2(&sc.sh[(int64_t)c * sc.n + gn]);
        }
        k1_one<DBG>(sc, vp, vb, g);
    }
}

template <bool DBG>
__device__ __forceinline__ void k1_one(const SceneDev& sc, const ViewParams& vp, ViewBufs& vb, int64_t g) {
    const double INF = CUDART_INF;
    float4 A4 = __ldg(&sc.geomA[g]), B4 = __ldg(&sc.geomB[g]), C4 = __ldg(&sc.geomC[g]);
    double* dbg = DBG ? vb.dbg + g * AAA_DBG_GAUSS_FIELDS : nullptr;
    if (dbg)
        for (int i = 0; i < AAA_DBG_GAUSS_FIELDS; i++) dbg[i] = 0.0;
    vb.counts[g] = 0;

    double mu[3] = {A4.x, A4.y, A4.z};
    double s[3] = {B4.x, B4.y, B4.z};
    double muv[3];
    mat3_vec(vp.Rv, mu, muv);
    for (int i = 0; i < 3; i++) muv[i] += vp.tv[i];

    // --- adaptive 3D filter (Eq. 6, 12, 13)
    double f = fmax(vp.fx, vp.fy);
    double vhat = muv[2] > 0.0 ? f / muv[2] : INF;
    double veff = fmin((double)B4.w, vhat);
    double cf = isinf(veff) ? 0.0 : (double)vp.k / (veff * veff);
#if AAA_K1_SPHERE
    if (!DBG) {
        // Conservative early exit (the exact whole-view cull below decides every survivor): the
        // tau-ellipsoid lies in the sphere of radius sqrt(tau lambda_max), tau <= 2 ln(255 o) (A <= 1)
        // and lambda_max <= max s_i^2 + k / v'^2; a sphere entirely outside one plane of the
        // pixel-centre frustum (4 planes through the camera + z >= near) holds nothing visible.
        // With the scene in Morton order, whole warps of off-screen Gaussians leave here.
#if AAA_K1_TMAX32
        // an upper bound suffices here: FP32 log (a few ulp) widened by 1e-5 relative + 1e-6
        const double tmax = (double)(2.f * __logf(255.f * A4.w)) * (1.0 + 1e-5) + 1e-6;
#else
        const double tmax = 2.0 * log(255.0 * (double)A4.w);
#endif
        const double lmax = fmax(fmax(s[0] * s[0], s[1] * s[1]), s[2] * s[2]) + cf;
        const double r = sqrt(fmax(tmax, 0.0) * lmax) * (1.0 + 1e-6) + 1e-9 * fabs(muv[2]);
        // pixel-centre frustum of the rendered tile rows (the whole image, or a band / row range);
        // the planes' normal lengths come with the view (set_rows)
        const double x0 = 0.5 - vp.cx, x1 = vp.width - 0.5 - vp.cx;
        const double y0 = TILE * vp.tile_row_begin + 0.5 - vp.cy;
        const double y1 = fmin((double)(TILE * vp.tile_row_end), (double)vp.height) - 0.5 - vp.cy;
        const bool out = !(tmax > 0.0) || muv[2] + r < vp.near_z ||
                         vp.fx * muv[0] - x0 * muv[2] < -r * vp.fr_norm[0] ||
                         -vp.fx * muv[0] + x1 * muv[2] < -r * vp.fr_norm[1] ||
                         vp.fy * muv[1] - y0 * muv[2] < -r * vp.fr_norm[2] ||
                         -vp.fy * muv[1] + y1 * muv[2] < -r * vp.fr_norm[3];
        if (out) return;
    }
#endif
#if AAA_K1_SHPF
    if (!DBG) {
        // the SH coefficients are read last (colour); start their loads now so they arrive in the
        // cache while the FP64 geometry runs (1 = L2, 2 = L1; K1 uses no shared memory)
        const int chunks = (3 * (sc.sh_degree + 1) * (sc.sh_degree + 1) + 3) / 4;
        for (int c = 0; c < chunks; c++) {
            if (AAA_K1_SHPF == 2) prefetch_l1(&sc.sh[(int64_t)c * sc.n + g]);
            else prefetch_l2(&sc.sh[(int64_t)c * sc.n + g]);
        }
    }
#endif
    double R[9];
    quat_to_rot(C4, R);
    double shat[3], sig[3], isig[3];
    for (int i = 0; i < 3; i++) {
        shat[i] = s[i] * s[i] + cf;
        sig[i] = sqrt(shat[i]);
        isig[i] = rsqrt(shat[i]);
    }
    double d[3] = {mu[0] - vp.o[0], mu[1] - vp.o[1], mu[2] - vp.o[2]};
    double dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    const double idn = 1.0 / dn;
    for (int i = 0; i < 3; i++) d[i] *= idn;
    double Amp = 1.0;
    if (cf > 0.0) {  // Eq. 12 with d' = R^T d (Eq. 11)
        double dp0 = R[0] * d[0] + R[3] * d[1] + R[6] * d[2];
        double dp1 = R[1] * d[0] + R[4] * d[1] + R[7] * d[2];
        double dp2 = R[2] * d[0] + R[5] * d[1] + R[8] * d[2];
        double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
        double num = dp0 * dp0 * s2[1] * s2[2] + dp1 * dp1 * s2[0] * s2[2] + dp2 * dp2 * s2[0] * s2[1];
        double den = dp0 * dp0 * shat[1] * shat[2] + dp1 * dp1 * shat[0] * shat[2] + dp2 * dp2 * shat[0] * shat[1];
        Amp = sqrt(num / den);
    }
    double oA = (double)A4.w * Amp;
    double tau = 2.0 * log(255.0 * oA);
    if (vp.tau_mode == 1) tau = fmin((double)vp.tau_fixed, tau);
    if (dbg) {
        dbg[0] = vhat; dbg[1] = veff; dbg[2] = shat[0]; dbg[3] = shat[1]; dbg[4] = shat[2];
        dbg[5] = Amp; dbg[6] = oA; dbg[7] = tau;
    }
    if (!(tau > 0.0)) return;

    // --- T_view linear part M = Rv R diag(sig); W = M^-1 = diag(1/sig) R^T Rv^-1; c = -W mu_v
    double Q[9];
    mat3_mul(vp.Rv, R, Q);
    double M[9];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) M[3 * i + j] = Q[3 * i + j] * sig[j];
    double Wm[9];  // Rv^-1 exactly (reading 37); R is orthonormal to FP64 rounding (normalised q)
    for (int j = 0; j < 3; j++)
        for (int i = 0; i < 3; i++)
            Wm[3 * j + i] = (R[j] * vp.Rvi[i] + R[3 + j] * vp.Rvi[3 + i] + R[6 + j] * vp.Rvi[6 + i]) * isig[j];
    double c[3];
    mat3_vec(Wm, muv, c);
    for (int i = 0; i < 3; i++) c[i] = -c[i];
    double c2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    bool inside = c2 < tau;  // camera inside the tau-ellipsoid
    if (dbg) {
        dbg[8] = inside ? 0.0 : 1.0;
        dbg[9] = inside ? 1.0 : 0.0;
        dbg[10] = c2;
    }
    if (inside) return;

    // --- depth extent; entirely closer than near -> no pixel can take it (reading 6)
    double gz[3] = {M[6], M[7], M[8]};
    double szz = gz[0] * gz[0] + gz[1] * gz[1] + gz[2] * gz[2];
    double zext = sqrt(tau * szz);
    if (muv[2] + zext < vp.near_z) return;
    bool crossing = (muv[2] - zext) <= vp.near_z;

    // --- bounds (Eq. 14-17): s_ij = tau (M M^T)_ij - mu_i mu_j, discriminant cancellation-free
    const double* Mx = &M[0];
    const double* My = &M[3];
    const double* Mz = &M[6];
    double sxx = tau * dot3(Mx, Mx) - muv[0] * muv[0];
    double sxz = tau * dot3(Mx, Mz) - muv[0] * muv[2];
    double syy = tau * dot3(My, My) - muv[1] * muv[1];
    double syz = tau * dot3(My, Mz) - muv[1] * muv[2];
    double szz3 = tau * szz - muv[2] * muv[2];
    double ex[3], ey[3], cxz[3], cyz[3];
    for (int j = 0; j < 3; j++) {
        ex[j] = muv[2] * Mx[j] - muv[0] * Mz[j];
        ey[j] = muv[2] * My[j] - muv[1] * Mz[j];
    }
    cross3(Mx, Mz, cxz);
    cross3(My, Mz, cyz);
    double discx = tau * (dot3(ex, ex) - tau * dot3(cxz, cxz));
    double discy = tau * (dot3(ey, ey) - tau * dot3(cyz, cyz));
    double xlo, xhi, ylo, yhi;
    if (!axis_bounds(sxx, sxz, szz3, discx, muv[0], muv[2], vp.fx, vp.cx, xlo, xhi)) return;
    if (!axis_bounds(syy, syz, szz3, discy, muv[1], muv[2], vp.fy, vp.cy, ylo, yhi)) return;
    if (dbg) {
        dbg[21] = xlo; dbg[22] = xhi; dbg[23] = ylo; dbg[24] = yhi;
    }
    // pixel-centre index range with 1 px padding, clipped to the image
    const double PAD = 1.0;
    double ixlo = ceil(fmax(xlo - PAD - 0.5, -1.0)), ixhi = floor(fmin(xhi + PAD - 0.5, (double)vp.width));
    double iylo = ceil(fmax(ylo - PAD - 0.5, -1.0)), iyhi = floor(fmin(yhi + PAD - 0.5, (double)vp.height));
    int i0 = max(0, (int)ixlo), i1 = min(vp.width - 1, (int)ixhi);
    int j0 = max(0, (int)iylo), j1 = min(vp.height - 1, (int)iyhi);
    if (i0 > i1 || j0 > j1) return;

    // --- p_ref: projected mean clamped into the pixel rect, else the rect centre (rounded to f32)
    double px0 = i0 + 0.5, px1 = i1 + 0.5, py0 = j0 + 0.5, py1 = j1 + 0.5;
    double prx, pry;
    if (muv[2] > 0.0) {
        prx = fmin(fmax(vp.fx * muv[0] / muv[2] + vp.cx, px0), px1);
        pry = fmin(fmax(vp.fy * muv[1] / muv[2] + vp.cy, py0), py1);
    } else {
        prx = 0.5 * (px0 + px1);
        pry = 0.5 * (py0 + py1);
    }
    float prx_f = (float)prx, pry_f = (float)pry;
    prx = prx_f;
    pry = pry_f;
    // pixel ray r(p) = ((px-cx)/fx, (py-cy)/fy, 1); unit-space direction w(p) = W r(p) is affine in p
    double rref[3] = {(prx - vp.cx) * vp.inv_fx, (pry - vp.cy) * vp.inv_fy, 1.0};
    double wref[3], wa[3], wb[3];
    mat3_vec(Wm, rref, wref);
    for (int j = 0; j < 3; j++) {
        wa[j] = Wm[3 * j + 0] * vp.inv_fx;
        wb[j] = Wm[3 * j + 1] * vp.inv_fy;
    }
    // rho^2(p) = |c x w(p)|^2 / |w(p)|^2,  c x w(p) = F0 + dx E1 + dy E2 (re-centred, DESIGN K6)
    double F0[3], E1[3], E2[3];
    cross3(c, wref, F0);
    cross3(c, wa, E1);
    cross3(c, wb, E2);
    // screen-space quadratic q(p) = |c x w|^2 - tau |w|^2 (< 0 <=> rho^2 < tau), relative to p_ref
    double qa = dot3(E1, E1) - tau * dot3(wa, wa);
    double qb = dot3(E1, E2) - tau * dot3(wa, wb);
    double qc = dot3(E2, E2) - tau * dot3(wb, wb);
    double qd = dot3(F0, E1) - tau * dot3(wref, wa);
    double qe = dot3(F0, E2) - tau * dot3(wref, wb);
    double qf = dot3(F0, F0) - tau * dot3(wref, wref);

    // --- whole-view frustum cull, exact: over the bounds rect (which holds every pixel
    // centre of the tau-ellipsoid's projection), quadratic box minimum or the 5-plane QP
    bool visible;
    if (!crossing) {
        visible = quad_box_min(qa, qb, qc, qd, qe, qf, px0 - prx, px1 - prx, py0 - pry, py1 - pry) < 0.0;
    } else {
        visible = frustum_qp_min(M, muv, vp.fx, vp.fy, vp.cx, vp.cy, vp.near_z, px0, px1, py0, py1) < tau;
    }
    if (dbg) dbg[15] = crossing ? 1.0 : 0.0;
    if (!visible) return;

    // --- tile rect, band-clipped
    int tx0 = i0 / TILE, tx1 = i1 / TILE, ty0 = j0 / TILE, ty1 = j1 / TILE;
    ty0 = max(ty0, vp.tile_row_begin);
    ty1 = min(ty1, vp.tile_row_end - 1);

    // --- depth key: tight lower bound of z* over every contributing ray (reading 23)
    double cn = sqrt(c2);
    const double icn = 1.0 / cn;
    double ch[3] = {c[0] * icn, c[1] * icn, c[2] * icn};
    double gc = dot3(gz, ch);
    double gp[3] = {gz[0] - gc * ch[0], gz[1] - gc * ch[1], gz[2] - gc * ch[2]};
    double zlb = muv[2] - sqrt(tau) * sqrt(dot3(gp, gp)) - (tau * icn) * fmax(0.0, -gc);
    zlb = fmax(zlb, vp.near_z);
    // log-depth code, rounded down (decode <= z_lb (1 - pad)); zlb >= near > near_lo keeps u >= 0
    const double u = vp.key_scale * log2(zlb * vp.key_zmul);
    const double qmax = (double)((1u << vp.key_db) - 1u);
    uint32_t zkey = (uint32_t)fmin(fmax(floor(u), 0.0), qmax);
    if (vp.flags & AAA_FLAG_NO_HIER_SORT) {  // Table 5 "w/o hier. sort": depth code of the mean
        const double um = vp.key_scale * log2(fmax(muv[2], vp.key_near) / vp.key_near);
        zkey = (uint32_t)fmin(fmax(floor(um), 0.0), qmax);
    }

    int slot = -1;
    if (crossing) {
        slot = (int)atomicAdd(&vb.counters[CNT_CROSS], 1u);
        CrossRec cr;
        for (int i = 0; i < 9; i++) cr.M[i] = M[i];
        for (int i = 0; i < 3; i++) cr.muv[i] = muv[i];
        cr.tau = tau;
        cr.pad = 0.0;
        vb.cross[slot] = cr;
    }
    CullRec cu;
    cu.qa = qa; cu.qb = qb; cu.qc = qc; cu.qd = qd; cu.qe = qe; cu.qf = qf;
    cu.ia = qa > 0.0 ? 1.0 / qa : 0.0;
    cu.ic = qc > 0.0 ? 1.0 / qc : 0.0;
    {
        double det = qa * qc - qb * qb;
        if (qa > 0.0 && det > 0.0) {
            cu.xs = (qb * qe - qc * qd) / det;
            cu.ys = (qb * qd - qa * qe) / det;
            cu.qi = (qa * cu.xs + 2.0 * qb * cu.ys + 2.0 * qd) * cu.xs + (qc * cu.ys + 2.0 * qe) * cu.ys + qf;
        } else {
            cu.xs = cu.ys = 0.0;
            cu.qi = CUDART_INF;
        }
    }
    cu.pref_x = prx_f;
    cu.pref_y = pry_f;
    cu.tx0 = (uint16_t)tx0; cu.ty0 = (uint16_t)ty0; cu.tx1 = (uint16_t)tx1; cu.ty1 = (uint16_t)ty1;
    cu.i0 = (uint16_t)i0; cu.j0 = (uint16_t)j0; cu.i1 = (uint16_t)i1; cu.j1 = (uint16_t)j1;
    cu.cross_slot = slot;
    cu.zkey = zkey;
    vb.cull[g] = cu;

    float4* rr = vb.raster + g * RASTER_REC_F4;
    rr[0] = make_float4(prx_f, pry_f, (float)oA, (float)tau);
    rr[1] = make_float4((float)F0[0], (float)F0[1], (float)F0[2], (float)E1[0]);
    rr[2] = make_float4((float)E1[1], (float)E1[2], (float)E2[0], (float)E2[1]);
    rr[3] = make_float4((float)E2[2], (float)wref[0], (float)wref[1], (float)wref[2]);
    rr[4] = make_float4((float)wa[0], (float)wa[1], (float)wa[2], (float)wb[0]);
    rr[5] = make_float4((float)wb[1], (float)wb[2], (float)dot3(c, wref), (float)dot3(c, wa));
    rr[6] = make_float4((float)dot3(c, wb), (float)c[0], (float)c[1], (float)c[2]);  // c: backward only

    // --- colour (reading 15): SH at d = (mu - o)/|mu - o|. By default a separate streaming kernel
    // (K1c, k_color) evaluates it for the visible Gaussians: K1 is latency-bound at 12 warps per SM
    // (168 registers of FP64 geometry), and the 192 B of SH per Gaussian were its largest source
    // of memory stalls; K1c runs at full occupancy. Same d, same arithmetic: identical colours.
    float rgb[3] = {0.f, 0.f, 0.f};
    if (DBG || !AAA_K1_SPLIT) {
        sh_color(sc.sh, sc.n, g, sc.sh_degree, make_float3((float)d[0], (float)d[1], (float)d[2]), rgb);
        vb.color[g] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
    }

    uint32_t cnt = (ty0 <= ty1) ? (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1) : 0u;
    vb.counts[g] = cnt;
    {  // one atomic per warp for the visible count (a per-thread atomic serialises on one address)
        const unsigned act = __activemask();
        if ((threadIdx.x & 31) == __ffs(act) - 1) atomicAdd(&vb.counters[CNT_VISIBLE], (unsigned)__popc(act));
    }
    if (dbg) {
        dbg[11] = rgb[0]; dbg[12] = rgb[1]; dbg[13] = rgb[2];
        dbg[14] = 1.0;
        dbg[16] = tx0; dbg[17] = ty0; dbg[18] = tx1; dbg[19] = ty1;
        dbg[20] = vp.key_near * exp2((double)zkey / vp.key_scale);
        dbg[25] = zlb;
    }
}

// K1c: SH colour of every Gaussian K1 kept (count > 0; the debug instantiation of K1 computes it
// inline) — d in FP64 exactly as K1 computes it, then the same FP32 evaluation
__global__ void __launch_bounds__(256) k_color(SceneDev sc, ViewParams vp, ViewBufs vb) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= sc.n || vb.counts[g] == 0) return;
    const float4 A4 = __ldg(&sc.geomA[g]);
    double d[3] = {(double)A4.x - vp.o[0], (double)A4.y - vp.o[1], (double)A4.z - vp.o[2]};
    const double idn = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int i = 0; i < 3; i++) d[i] *= idn;
    float rgb[3];
    sh_color(sc.sh, sc.n, g, sc.sh_degree, make_float3((float)d[0], (float)d[1], (float)d[2]), rgb);
    vb.color[g] = make_float4(rgb[0], rgb[1], rgb[2], 0.f);
}

int launch_preprocess(const SceneDev& sc, const ViewParams& vp, ViewBufs& vb, bool debug, cudaStream_t st) {
    if (sc.n == 0) return 0;
    int threads = 128;
    unsigned blocks = (unsigned)((sc.n + threads - 1) / threads);
    if (vp.flags & AAA_FLAG_NO_3D) {
        k_preprocess_2d<<<blocks, threads, 0, st>>>(sc, vp, vb);
    } else if (debug) {
        k_preprocess<true><<<blocks, threads, 0, st>>>(sc, vp, vb);
    } else {
        const unsigned b1 = (unsigned)((sc.n + threads * AAA_K1_ITEMS - 1) / (threads * AAA_K1_ITEMS));
        k_preprocess<false><<<b1, threads, 0, st>>>(sc, vp, vb);
        if (AAA_K1_SPLIT) {
            k_color<<<(unsigned)((sc.n + 255) / 256), 256, 0, st>>>(sc, vp, vb);
            return 2;
        }
    }
    return 1;
}

// Tile-band cost model: per tile row, the number of candidate (Gaussian, rect
// tile) pairs of a full-frame K1 — identical on every rank, so every rank derives the same bands
// without communication. Difference array over rows (+w at ty0, -w at ty1 + 1, w = rect width),
// accumulated per block in shared memory and flushed with one 64-bit atomic per row per block.
constexpr int ROWCOST_SMEM_ROWS = 2048;
__global__ void __launch_bounds__(256) k_row_costs(const CullRec* __restrict__ cull, const uint32_t* __restrict__ counts,
                                                   int64_t n, int rows, unsigned long long* diff) {
    __shared__ int32_t h[ROWCOST_SMEM_ROWS + 1];
    const bool sm = rows <= ROWCOST_SMEM_ROWS;
    if (sm)
        for (int i = threadIdx.x; i <= rows; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
        if (counts[g] == 0) continue;
        const uint4 rr = reinterpret_cast<const uint4*>(cull + g)[CULLREC_RECT_U4];
        const int tx0 = rr.x & 0xFFFF, ty0 = rr.x >> 16, tx1 = rr.y & 0xFFFF, ty1 = rr.y >> 16;
        const int w = tx1 - tx0 + 1;
        if (sm) {
            atomicAdd(&h[ty0], w);
            atomicAdd(&h[ty1 + 1], -w);
        } else {
            atomicAdd(&diff[ty0], (unsigned long long)(long long)w);
            atomicAdd(&diff[ty1 + 1], (unsigned long long)(long long)(-w));
        }
    }
    __syncthreads();
    if (sm)
        for (int i = threadIdx.x; i <= rows; i += blockDim.x)
            if (h[i]) atomicAdd(&diff[i], (unsigned long long)(long long)h[i]);
}

// Approximate tile-band cost model (AAA_BAND_APPROX): per tile row, the tile-rect width of every
// Gaussian whose projected bounding disc (3 sigma of its largest scale widened by the 3D filter's
// smallest variance, FP32) covers the row — from the means and scales alone, before any K1, so a
// band rank runs K1 only where its band can see (the sphere exit). Only the load balance depends
// on it: any cut renders the same stacked frame. Identical on every rank (same inputs, same
// arithmetic, integer atomics).
__global__ void __launch_bounds__(256) k_row_costs_approx(SceneDev sc, ViewParams vp, int rows,
                                                          unsigned long long* diff) {
    __shared__ int32_t h[ROWCOST_SMEM_ROWS + 1];
    const bool sm = rows <= ROWCOST_SMEM_ROWS;
    if (sm)
        for (int i = threadIdx.x; i <= rows; i += blockDim.x) h[i] = 0;
    __syncthreads();
    float R[9], t[3];
    for (int i = 0; i < 9; i++) R[i] = (float)vp.Rv[i];
    for (int i = 0; i < 3; i++) t[i] = (float)vp.tv[i];
    const float fx = (float)vp.fx, fy = (float)vp.fy, cx = (float)vp.cx, cy = (float)vp.cy, nz = (float)vp.near_z;
    const float fmx = fmaxf(fx, fy), kf = vp.k;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < sc.n; g += (int64_t)gridDim.x * blockDim.x) {
        const float4 A = __ldg(&sc.geomA[g]), B = __ldg(&sc.geomB[g]);
        const float x = fmaf(R[0], A.x, fmaf(R[1], A.y, fmaf(R[2], A.z, t[0])));
        const float y = fmaf(R[3], A.x, fmaf(R[4], A.y, fmaf(R[5], A.z, t[1])));
        const float z = fmaf(R[6], A.x, fmaf(R[7], A.y, fmaf(R[8], A.z, t[2])));
        if (!(z > nz)) continue;
        const float smax = fmaxf(fmaxf(B.x, B.y), B.z), zf = z / fmx;
        const float r = 3.f * sqrtf(fmaf(smax, smax, kf * zf * zf)), iz = 1.f / z;
        const float xc = fmaf(fx * x, iz, cx), yc = fmaf(fy * y, iz, cy), rx = fx * r * iz, ry = fy * r * iz;
        const int tx0 = max(0, (int)floorf((xc - rx) / TILE)), tx1 = min(vp.tiles_x - 1, (int)floorf((xc + rx) / TILE));
        const int ty0 = max(0, (int)floorf((yc - ry) / TILE)), ty1 = min(rows - 1, (int)floorf((yc + ry) / TILE));
        if (tx0 > tx1 || ty0 > ty1) continue;
        const int w = tx1 - tx0 + 1;
        if (sm) {
            atomicAdd(&h[ty0], w);
            atomicAdd(&h[ty1 + 1], -w);
        } else {
            atomicAdd(&diff[ty0], (unsigned long long)(long long)w);
            atomicAdd(&diff[ty1 + 1], (unsigned long long)(long long)(-w));
        }
    }
    __syncthreads();
    if (sm)
        for (int i = threadIdx.x; i <= rows; i += blockDim.x)
            if (h[i]) atomicAdd(&diff[i], (unsigned long long)(long long)h[i]);
}

void launch_row_costs_approx(const SceneDev& sc, const ViewParams& vp, int rows, unsigned long long* diff,
                             cudaStream_t st) {
    cudaMemsetAsync(diff, 0, (size_t)(rows + 1) * sizeof(unsigned long long), st);
    if (sc.n == 0) return;
    const unsigned blocks = (unsigned)std::min<int64_t>((sc.n + 255) / 256, 148 * 8);
    k_row_costs_approx<<<blocks, 256, 0, st>>>(sc, vp, rows, diff);
}

// clip every visible Gaussian's tile rect to the band [row_begin, row_end) and recount its
// candidates (after a full-frame K1): K2/K3 then emit only the band's pairs
__global__ void __launch_bounds__(256) k_band_clip(CullRec* cull, uint32_t* counts, int64_t n, int row_begin,
                                                   int row_end) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || counts[g] == 0) return;
    uint4* p = reinterpret_cast<uint4*>(cull + g) + CULLREC_RECT_U4;
    uint4 rr = *p;
    const int tx0 = rr.x & 0xFFFF, tx1 = rr.y & 0xFFFF;
    const int ty0 = max((int)(rr.x >> 16), row_begin), ty1 = min((int)(rr.y >> 16), row_end - 1);
    counts[g] = ty0 <= ty1 ? (uint32_t)(tx1 - tx0 + 1) * (uint32_t)(ty1 - ty0 + 1) : 0u;
    if (ty0 <= ty1) {
        rr.x = (uint32_t)tx0 | ((uint32_t)ty0 << 16);
        rr.y = (uint32_t)tx1 | ((uint32_t)ty1 << 16);
        *p = rr;
    }
}

void launch_row_costs(const ViewBufs& vb, int64_t n, int rows, unsigned long long* diff, cudaStream_t st) {
    cudaMemsetAsync(diff, 0, (size_t)(rows + 1) * sizeof(unsigned long long), st);
    if (n == 0) return;
    const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
    k_row_costs<<<blocks, 256, 0, st>>>(vb.cull, vb.counts, n, rows, diff);
}

void launch_band_clip(const ViewBufs& vb, int64_t n, int row_begin, int row_end, cudaStream_t st) {
    if (n == 0) return;
    k_band_clip<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vb.cull, vb.counts, n, row_begin, row_end);
}

}  // namespace aaa
