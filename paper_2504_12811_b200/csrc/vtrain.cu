// vtrain.cu — v_hat_train (Eq. 6): per Gaussian, the maximum over the
// training cameras whose frustum contains the mean of f / z (f = max(fx, fy), reading 10).
// The frustum is the culling frustum of reading 20 applied to the mean point. One thread per
// Gaussian, the cameras staged in shared memory in chunks; FP64 arithmetic, f32 result.
#include <math_constants.h>

#include "aaa_internal.cuh"

namespace aaa {

constexpr int VT_THREADS = 256, VT_CAMS = 128;

__global__ void __launch_bounds__(VT_THREADS) k_vtrain(const float4* __restrict__ geomA, int64_t n,
                                                       const VtCam* __restrict__ cams, int n_cams,
                                                       float* __restrict__ out, float4* geomB_store,
                                                       const uint32_t* __restrict__ perm) {
    __shared__ VtCam s_cam[VT_CAMS];
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double mu[3] = {0.0, 0.0, 0.0};
    if (g < n) {
        const float4 a = __ldg(&geomA[g]);
        mu[0] = a.x; mu[1] = a.y; mu[2] = a.z;
    }
    double best = -CUDART_INF;
    for (int c0 = 0; c0 < n_cams; c0 += VT_CAMS) {
        const int nc = min(VT_CAMS, n_cams - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < nc; i += blockDim.x) s_cam[i] = cams[c0 + i];
        __syncthreads();
        for (int i = 0; i < nc; i++) {
            const VtCam& c = s_cam[i];
            const double z = fma(c.R[6], mu[0], fma(c.R[7], mu[1], fma(c.R[8], mu[2], c.t[2])));
            if (!(z >= c.near_z)) continue;
            const double x = fma(c.R[0], mu[0], fma(c.R[1], mu[1], fma(c.R[2], mu[2], c.t[0])));
            const double y = fma(c.R[3], mu[0], fma(c.R[4], mu[1], fma(c.R[5], mu[2], c.t[1])));
            const double px = c.fx * x / z + c.cx, py = c.fy * y / z + c.cy;
            if (px < 0.5 || px > c.w - 0.5 || py < 0.5 || py > c.h - 0.5) continue;
            best = fmax(best, c.f / z);
        }
    }
    if (g >= n) return;
    const float v = best > 0.0 ? (float)best : CUDART_INF_F;
    if (out) out[perm ? (int64_t)perm[g] : g] = v;  // the caller's order
    if (geomB_store) geomB_store[g].w = v;
}

void launch_vtrain(const SceneDev& sc, const VtCam* cams, int n_cams, float* out, bool store, cudaStream_t st) {
    if (sc.n == 0) return;
    const unsigned blocks = (unsigned)((sc.n + VT_THREADS - 1) / VT_THREADS);
    k_vtrain<<<blocks, VT_THREADS, 0, st>>>(sc.geomA, sc.n, cams, n_cams, out, store ? sc.geomB : nullptr, sc.perm);
}

}  // namespace aaa
