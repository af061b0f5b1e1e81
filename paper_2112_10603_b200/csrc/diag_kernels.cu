// diag_kernels.cu -- coarse-scale diagnostics of interpolate(..., diagnostics=True)
// (interp.py:119-127): for levels 0 and 1, ScaleDiagnostics.mask and .blend_luma.
//
// Off the hot path (diagnostics only), so these kernels replay the reference's
// arithmetic literally instead of the exact fixed-point forms of the synthesis
// kernels: warp_flow in f64 (_kernels.py:78-107), np.gradient on f32, and
// scipy's uniform_filter1d(size 3, nearest) as its running sum -- one thread
// per column for axis 0, one per row for axis 1 (at the coarse levels the
// column pass over non-integer warped luma is order dependent as well).
// Inputs are the engine's own level planes: luma s16 / s4 (exact 16x / 4x
// level values) and the level flows in fixed point (exact f32).
#include <cuda_runtime.h>

#include <cstdint>

#include "fvv_device.cuh"

namespace fvv {

struct LDiag {  // scratch planes (n = level pixels)
    double *wl, *wr, *ad, *tad;
    float *ol, *orr, *tol, *tor;
};

__device__ __forceinline__ double level_luma(const Geometry& g, const uint8_t* ws, const Planes& P, int pair,
                                             int level, int side, int i, const LDiagSrc& src) {
    if (src.lum[side]) return (double)src.lum[side][i];
    if (level == 0) return (double)((float)cplane<uint16_t>(ws, P, P.s16[side], pair)[i] * 0.0625f);
    return (double)((float)cplane<uint16_t>(ws, P, P.s4[side], pair)[i] * 0.25f);
}

// the level's flow (f32, exact from the fixed point) times -0.5 (FlowField.scaled, f32)
__device__ __forceinline__ float2 level_mid_flow(const Geometry& g, const uint8_t* ws, const Planes& P, int pair,
                                                 int level, int d, int i, const LDiagSrc& src) {
    if (src.flow[d]) return make_float2(src.flow[d][i].x * -0.5f, src.flow[d][i].y * -0.5f);
    const int2 v = cplane<int2>(ws, P, level == 0 ? P.flow0[d] : P.flow1[d], pair)[i];
    const float sc = 1.0f / (float)(1 << g.fb[level]);
    return make_float2(((float)v.x * sc) * -0.5f, ((float)v.y * sc) * -0.5f);
}

// pass 1 (per pixel): warped levels, |wl - wr|, occlusion cue inputs max(0, -div f_m)
__global__ void k_ldiag_warp(Geometry g, const uint8_t* __restrict__ ws, Planes P, int pair, int level, LDiag s,
                             LDiagSrc src) {
    const Level L = g.lv[level];
    const int h = L.h, w = L.w;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h * w) return;
    const int y = i / w, x = i - (i / w) * w;
    double wv[2];
    for (int d = 0; d < 2; d++) {
        const float2 f = level_mid_flow(g, ws, P, pair, level, d, i, src);
        double sx = (double)x + (double)f.x, sy = (double)y + (double)f.y;
        if (sx < 0.0) sx = 0.0; else if (sx > w - 1) sx = (double)(w - 1);
        if (sy < 0.0) sy = 0.0; else if (sy > h - 1) sy = (double)(h - 1);
        int x0 = (int)sx, y0 = (int)sy;
        if (x0 > w - 2) x0 = w > 1 ? w - 2 : 0;
        if (y0 > h - 2) y0 = h > 1 ? h - 2 : 0;
        const double fx = sx - x0, fy = sy - y0;
        const int x1 = w > 1 ? x0 + 1 : x0, y1 = h > 1 ? y0 + 1 : y0;
        auto sv = [&](int yy, int xx) { return level_luma(g, ws, P, pair, level, d, yy * w + xx, src); };
        const double top = (1.0 - fx) * sv(y0, x0) + fx * sv(y0, x1);
        const double bot = (1.0 - fx) * sv(y1, x0) + fx * sv(y1, x1);
        wv[d] = (1.0 - fy) * top + fy * bot;
        // np.gradient (f32, edge order 1) of f_m.x along x and f_m.y along y
        auto fm = [&](int yy, int xx) { return level_mid_flow(g, ws, P, pair, level, d, yy * w + xx, src); };
        float gx, gy;
        if (w < 2) gx = 0.0f;
        else if (x == 0) gx = (fm(y, 1).x - fm(y, 0).x) / 1.0f;
        else if (x == w - 1) gx = (fm(y, w - 1).x - fm(y, w - 2).x) / 1.0f;
        else gx = (fm(y, x + 1).x - fm(y, x - 1).x) / 2.0f;
        if (h < 2) gy = 0.0f;
        else if (y == 0) gy = (fm(1, x).y - fm(0, x).y) / 1.0f;
        else if (y == h - 1) gy = (fm(h - 1, x).y - fm(h - 2, x).y) / 1.0f;
        else gy = (fm(y + 1, x).y - fm(y - 1, x).y) / 2.0f;
        const float v = -(gx + gy);
        (d ? s.orr : s.ol)[i] = v > 0.0f ? v : 0.0f;
    }
    s.wl[i] = wv[0];
    s.wr[i] = wv[1];
    s.ad[i] = fabs(wv[0] - wv[1]);
}

// scipy uniform_filter1d(size 3, mode nearest) on one line: tmp = (p0 + p1) + p2,
// out = tmp / 3, tmp += p[i+2] - p[i-1] (the padded line p repeats the ends)
template <typename In, typename F>
__device__ __forceinline__ void ufilt3(In at, long n, F put) {
    auto P = [&](long k) { return (double)(k <= 0 ? at(0) : (k >= n + 1 ? at(n - 1) : at(k - 1))); };
    double tmp = (P(0) + P(1)) + P(2);
    put(0, tmp / 3.0);
    for (long i = 1; i < n; i++) {
        tmp = tmp + (P(i + 2) - P(i - 1));
        put(i, tmp / 3.0);
    }
}

// pass 2: axis 0 of smooth3, one thread per column (f64 stays f64, f32 stored as f32)
__global__ void k_ldiag_cols(int h, int w, LDiag s) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= w) return;
    ufilt3([&](long k) { return s.ad[k * w + x]; }, h, [&](long k, double v) { s.tad[k * w + x] = v; });
    ufilt3([&](long k) { return s.ol[k * w + x]; }, h, [&](long k, double v) { s.tol[k * w + x] = (float)v; });
    ufilt3([&](long k) { return s.orr[k * w + x]; }, h, [&](long k, double v) { s.tor[k * w + x] = (float)v; });
}

// pass 3: axis 1, one thread per row, then the level's mask (no clip) and blend
__global__ void k_ldiag_rows(int h, int w, LDiag s, double eps, double eps2, double* __restrict__ mask,
                             double* __restrict__ blend) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= h) return;
    const long r = (long)y * w;
    // the occlusion row passes land in the (now free) pass-1 planes, the diff in ad
    ufilt3([&](long k) { return s.tol[r + k]; }, w, [&](long k, double v) { s.ol[r + k] = (float)v; });
    ufilt3([&](long k) { return s.tor[r + k]; }, w, [&](long k, double v) { s.orr[r + k] = (float)v; });
    ufilt3([&](long k) { return s.tad[r + k]; }, w, [&](long k, double v) { s.ad[r + k] = v; });
    for (long k = 0; k < w; k++) {
        const float ql = 0.5f + 4.0f * s.ol[r + k], qr = 0.5f + 4.0f * s.orr[r + k];
        const double el = s.ad[r + k] * (double)ql, er = s.ad[r + k] * (double)qr;
        const double m = (er + eps) / (el + er + eps2);
        mask[r + k] = m;
        blend[r + k] = m * s.wl[r + k] + (1.0 - m) * s.wr[r + k];
    }
}

size_t level_mask_scratch_bytes(const Geometry& g, int level) {
    const size_t n = (size_t)g.lv[level].w * g.lv[level].h;
    return n * (4 * sizeof(double) + 4 * sizeof(float)) + 256;
}

cudaError_t run_level_mask(const Geometry& g, uint8_t* ws, const Planes& P, int pair, int level, void* scratch,
                           double* mask, double* blend, const LDiagSrc& src, cudaStream_t st) {
    const int h = g.lv[level].h, w = g.lv[level].w;
    const size_t n = (size_t)h * w;
    LDiag s;
    double* dp = static_cast<double*>(scratch);
    s.wl = dp; s.wr = dp + n; s.ad = dp + 2 * n; s.tad = dp + 3 * n;
    float* fp = reinterpret_cast<float*>(dp + 4 * n);
    s.ol = fp; s.orr = fp + n; s.tol = fp + 2 * n; s.tor = fp + 3 * n;
    k_ldiag_warp<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, ws, P, pair, level, s, src);
    k_ldiag_cols<<<(w + 63) / 64, 64, 0, st>>>(h, w, s);
    k_ldiag_rows<<<(h + 63) / 64, 64, 0, st>>>(h, w, s, g.eps, g.eps2, mask, blend);
    return cudaGetLastError();
}

}  // namespace fvv
