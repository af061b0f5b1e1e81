// literal_kernels.cu -- the reference's interpolation replayed literally on the
// device, for configurations outside the fixed-point domain of the fast path
// (block sizes other than 2, 4, 8; max_span > 120): InterpConfig accepts any
// block >= 2 and radius >= 1 (interp.py:32-36), and with a block of e.g. 6 the
// _block_to_pixel weights (i - 2.5) / 6 are not dyadic, so the flows are
// arbitrary f32 values and every downstream f64 expression must be evaluated
// exactly as the reference orders it (no FMA: the library builds --fmad=false).
//
// One pair at a time, simple kernels: thread per pixel (pyramid, warps,
// block_to_pixel, upscale), thread per block (SAD search + tie-rule argmin),
// thread per column / row for scipy's running-sum passes (order dependent in
// both axes on non-dyadic data).  The same arithmetic as the CPU oracle
// (oracle/fvv_oracle.c), which is pinned to the reference's golden vectors.
//   interp.py:67-71 pyramid        flow.py:47-54 upscale_flow     flow.py:69-91 block match
//   flow.py:94-98 block_to_pixel   _kernels.py:78-107 warp_flow   warp.py:27-88 warp/mask/blend
//   interp.py:78-94 _mask_inputs (scipy uniform_filter size 3, nearest)
#include <cuda_runtime.h>

#include <cstdint>

#include "fvv_device.cuh"
#include "literal.h"

namespace fvv {

namespace {

__device__ __forceinline__ uint8_t lit_u8(double v) {  // to_uint8: clip(rint(v), 0, 255)
    double r = rint(v);
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    return (uint8_t)r;
}

// _grid_bilinear_jit (_kernels.py:136-167) at one output (sy, sx), values at v(y, x)
template <typename V>
__device__ __forceinline__ double grid_bl(V v, int h, int w, double sy, double sx) {
    if (sy < 0.0) sy = 0.0; else if (sy > h - 1) sy = (double)(h - 1);
    int y0 = (int)sy;
    if (y0 > h - 2) y0 = h > 1 ? h - 2 : 0;
    const double fy = sy - y0;
    const int y1 = h > 1 ? y0 + 1 : y0;
    if (sx < 0.0) sx = 0.0; else if (sx > w - 1) sx = (double)(w - 1);
    int x0 = (int)sx;
    if (x0 > w - 2) x0 = w > 1 ? w - 2 : 0;
    const double fx = sx - x0;
    const int x1 = w > 1 ? x0 + 1 : x0;
    const double top = (1.0 - fx) * v(y0, x0) + fx * v(y0, x1);
    const double bot = (1.0 - fx) * v(y1, x0) + fx * v(y1, x1);
    return (1.0 - fy) * top + fy * bot;
}

// _warp_flow_jit (_kernels.py:78-107)
template <typename V>
__device__ __forceinline__ double warp_px(V src, int h, int w, int y, int x, float fxv, float fyv) {
    double sx = (double)x + (double)fxv, sy = (double)y + (double)fyv;
    if (sx < 0.0) sx = 0.0; else if (sx > w - 1) sx = (double)(w - 1);
    if (sy < 0.0) sy = 0.0; else if (sy > h - 1) sy = (double)(h - 1);
    int x0 = (int)sx, y0 = (int)sy;
    if (x0 > w - 2) x0 = w > 1 ? w - 2 : 0;
    if (y0 > h - 2) y0 = h > 1 ? h - 2 : 0;
    const double fx = sx - x0, fy = sy - y0;
    const int x1 = w > 1 ? x0 + 1 : x0, y1 = h > 1 ? y0 + 1 : y0;
    const double top = (1.0 - fx) * src(y0, x0) + fx * src(y0, x1);
    const double bot = (1.0 - fx) * src(y1, x0) + fx * src(y1, x1);
    return (1.0 - fy) * top + fy * bot;
}

template <typename In, typename F>
__device__ __forceinline__ void ufilt3(In at, long n, F put) {  // scipy uniform_filter1d(3, nearest)
    auto P = [&](long k) { return (double)(k <= 0 ? at(0) : (k >= n + 1 ? at(n - 1) : at(k - 1))); };
    double tmp = (P(0) + P(1)) + P(2);
    put(0, tmp / 3.0);
    for (long i = 1; i < n; i++) {
        tmp = tmp + (P(i + 2) - P(i - 1));
        put(i, tmp / 3.0);
    }
}

// ---- pyramid (interp.py:67-71, frame.py:68-75) ------------------------------
__global__ void k_lit_luma(const uint8_t* __restrict__ f, int fmt, int n, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (fmt == FVV_RGB8) {
        const double r = f[3 * i], g = f[3 * i + 1], b = f[3 * i + 2];
        double y = 0.299 * r + 0.587 * g;
        y = y + 0.114 * b;
        out[i] = (float)(uint8_t)rint(y);
    } else {
        out[i] = (float)f[i];
    }
}

__global__ void k_lit_box2(const float* __restrict__ a, int h, int w, float* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int oh = h / 2, ow = w / 2;
    if (i >= oh * ow) return;
    const int y = i / ow, x = i - (i / ow) * ow;
    const float s = (a[(2 * y) * w + 2 * x] + a[(2 * y) * w + 2 * x + 1]) +
                    (a[(2 * y + 1) * w + 2 * x] + a[(2 * y + 1) * w + 2 * x + 1]);
    out[i] = s / 4.0f;
}

// ---- one flow level (flow.py:101-131) ----------------------------------------
// base = upscale_flow(prev) or 0; target warped by base; q planes for the search
__global__ void k_lit_base(const float2* __restrict__ prev, int ph, int pw, int h, int w, const float* __restrict__ tgt,
                           float2* __restrict__ base, double* __restrict__ tw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h * w) return;
    const int y = i / w, x = i - (i / w) * w;
    float2 b = make_float2(0.0f, 0.0f);
    if (prev) {
        const double ry = (double)ph / h, rx = (double)pw / w;
        const double sy = ((double)y + 0.5) * ry - 0.5, sx = ((double)x + 0.5) * rx - 0.5;
        const double bx = grid_bl([&](int yy, int xx) { return (double)prev[yy * pw + xx].x; }, ph, pw, sy, sx);
        const double by = grid_bl([&](int yy, int xx) { return (double)prev[yy * pw + xx].y; }, ph, pw, sy, sx);
        b = make_float2((float)(bx * 2.0), (float)(by * 2.0));
    }
    base[i] = b;
    tw[i] = prev ? warp_px([&](int yy, int xx) { return (double)tgt[yy * w + xx]; }, h, w, y, x, b.x, b.y)
                 : (double)tgt[i];
}

// block search: thread per block, candidates in tie-rule rank order, first minimum
// (flow.py:57-91, _kernels.py:28-49); SAD of rint(8 ref) (f32) vs rint(8 target) (f64)
__global__ void k_lit_search(const float* __restrict__ ref, const double* __restrict__ tw, int h, int w, int r,
                             int B, const int16_t* __restrict__ cand_of_rank, float2* __restrict__ off,
                             int* __restrict__ best_sad) {
    const int nbx = (w + B - 1) / B, nby = (h + B - 1) / B;
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nbx * nby) return;
    const int by = b / nbx, bx = b - (b / nbx) * nbx;
    const int ys = by * B, ye = min(ys + B, h), xs = bx * B, xe = min(xs + B, w);
    const int side = 2 * r + 1, n = side * side;
    int best = 0x7fffffff, bk = 0;
    for (int k = 0; k < n; k++) {
        const int c = cand_of_rank[k];
        const int dy = c / side - r, dx = c % side - r;  // stack index (dy + r) * side + (dx + r)
        int acc = 0;
        for (int y = ys; y < ye; y++) {
            const int sy = min(max(y + dy, 0), h - 1);  // np.pad mode="edge"
            for (int x = xs; x < xe; x++) {
                const int sx = min(max(x + dx, 0), w - 1);
                const int q = (int)rint(tw[sy * w + sx] * 8.0);
                const int p = (int)rintf(ref[y * w + x] * 8.0f);
                const int d = q - p;
                acc += d >= 0 ? d : -d;
            }
        }
        if (acc < best) { best = acc; bk = k; }
    }
    const int c = cand_of_rank[bk];
    off[b] = make_float2((float)(c % side - r), (float)(c / side - r));
    best_sad[b] = best;
}

// flow = base + f32(block_to_pixel(offsets))  (flow.py:94-98, 129)
__global__ void k_lit_flow(const float2* __restrict__ base, const float2* __restrict__ off, int h, int w, int B,
                           float2* __restrict__ flow) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h * w) return;
    const int y = i / w, x = i - (i / w) * w;
    const int nbx = (w + B - 1) / B, nby = (h + B - 1) / B;
    const double c = (B - 1) / 2.0;
    const double sy = ((double)y - c) / B, sx = ((double)x - c) / B;
    const double px = grid_bl([&](int yy, int xx) { return (double)off[yy * nbx + xx].x; }, nby, nbx, sy, sx);
    const double py = grid_bl([&](int yy, int xx) { return (double)off[yy * nbx + xx].y; }, nby, nbx, sy, sx);
    flow[i] = make_float2(base[i].x + (float)px, base[i].y + (float)py);
}

// match-error map of a level: block_to_pixel(best / (area * 8)) (flow.py:86-91, 130)
__global__ void k_lit_err(const int* __restrict__ best_sad, int h, int w, int B, double* __restrict__ err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= h * w) return;
    const int y = i / w, x = i - (i / w) * w;
    const int nbx = (w + B - 1) / B, nby = (h + B - 1) / B;
    auto e = [&](int by, int bx) {
        const int rows = min(by * B + B, h) - by * B, cols = min(bx * B + B, w) - bx * B;
        return (double)best_sad[by * nbx + bx] / ((double)((long long)rows * cols) * 8.0);
    };
    const double c = (B - 1) / 2.0;
    err[i] = grid_bl(e, nby, nbx, ((double)y - c) / B, ((double)x - c) / B);
}

// ---- synthesis (interp.py:129-141, warp.py) ------------------------------------
// mid flows f32, backward warps of every plane (to_uint8), warped luma (f64), |wl - wr|,
// occlusion cue inputs
__global__ void k_lit_warp(const uint8_t* __restrict__ fl, const uint8_t* __restrict__ fr, int fmt, int W, int H,
                           const float2* __restrict__ flr, const float2* __restrict__ frl, LitSynth s) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= W * H) return;
    const int y = i / W, x = i - (i / W) * W;
    const uint8_t* fr2[2] = {fl, fr};
    const float2* fw[2] = {flr, frl};
    double lum[2];
    for (int d = 0; d < 2; d++) {
        const float fx = fw[d][i].x * -0.5f, fy = fw[d][i].y * -0.5f;  // FlowField.scaled(-0.5), f32
        const uint8_t* f = fr2[d];
        uint8_t* wd = d ? s.wr : s.wl;
        if (fmt == FVV_RGB8) {
            uint8_t c3[3];
            for (int c = 0; c < 3; c++)
                c3[c] = lit_u8(warp_px([&](int yy, int xx) { return (double)f[(yy * W + xx) * 3 + c]; }, H, W, y, x, fx, fy));
            for (int c = 0; c < 3; c++) wd[i * 3 + c] = c3[c];
            double l = 0.299 * (double)c3[0] + 0.587 * (double)c3[1];
            l = l + 0.114 * (double)c3[2];
            lum[d] = (double)(uint8_t)rint(l);
        } else {
            const uint8_t v = lit_u8(warp_px([&](int yy, int xx) { return (double)f[yy * W + xx]; }, H, W, y, x, fx, fy));
            wd[i] = v;
            lum[d] = (double)v;
        }
        // occlusion cue input: max(0, -(d/dx f_m.x + d/dy f_m.y)), np.gradient on f32
        auto fm = [&](int yy, int xx) { return make_float2(fw[d][yy * W + xx].x * -0.5f, fw[d][yy * W + xx].y * -0.5f); };
        float gx, gy;
        if (W < 2) gx = 0.0f;
        else if (x == 0) gx = (fm(y, 1).x - fm(y, 0).x) / 1.0f;
        else if (x == W - 1) gx = (fm(y, W - 1).x - fm(y, W - 2).x) / 1.0f;
        else gx = (fm(y, x + 1).x - fm(y, x - 1).x) / 2.0f;
        if (H < 2) gy = 0.0f;
        else if (y == 0) gy = (fm(1, x).y - fm(0, x).y) / 1.0f;
        else if (y == H - 1) gy = (fm(H - 1, x).y - fm(H - 2, x).y) / 1.0f;
        else gy = (fm(y + 1, x).y - fm(y - 1, x).y) / 2.0f;
        const float v = -(gx + gy);
        (d ? s.or_ : s.ol)[i] = v > 0.0f ? v : 0.0f;
    }
    s.ad[i] = fabs(lum[0] - lum[1]);
}

// chroma planes of 4:2:0 (imageops.py:40-48 halve_flow: f32 2x2 mean, times 0.5)
__global__ void k_lit_warp_chroma(const uint8_t* __restrict__ fl, const uint8_t* __restrict__ fr, int W, int H,
                                  const float2* __restrict__ flr, const float2* __restrict__ frl, LitSynth s) {
    const int cw = W / 2, ch = H / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cw * ch) return;
    const int y = i / cw, x = i - (i / cw) * cw;
    const uint8_t* fr2[2] = {fl, fr};
    const float2* fw[2] = {flr, frl};
    for (int d = 0; d < 2; d++) {
        auto hv = [&](int yy, int xx) {
            float c[2];
            for (int k = 0; k < 2; k++) {
                auto g = [&](int a, int b) {
                    const float2 v = fw[d][(2 * yy + a) * W + 2 * xx + b];
                    return (k ? v.y : v.x) * -0.5f;
                };
                const float sum = (g(0, 0) + g(0, 1)) + (g(1, 0) + g(1, 1));
                c[k] = (sum / 4.0f) * 0.5f;
            }
            return make_float2(c[0], c[1]);
        };
        const float2 f = hv(y, x);
        uint8_t* wd = d ? s.wr : s.wl;
        for (int p = 0; p < 2; p++) {
            const uint8_t* pl = fr2[d] + (size_t)W * H + (size_t)p * cw * ch;
            wd[(size_t)W * H + (size_t)p * cw * ch + i] =
                lit_u8(warp_px([&](int yy, int xx) { return (double)pl[yy * cw + xx]; }, ch, cw, y, x, f.x, f.y));
        }
    }
}

// axis-0 passes of smooth3 (one thread per column): diff (f64) and both occlusion maps (f32)
__global__ void k_lit_cols(int H, int W, LitSynth s) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= W) return;
    ufilt3([&](long k) { return s.ad[k * W + x]; }, H, [&](long k, double v) { s.tad[k * W + x] = v; });
    ufilt3([&](long k) { return s.ol[k * W + x]; }, H, [&](long k, double v) { s.tol[k * W + x] = (float)v; });
    ufilt3([&](long k) { return s.or_[k * W + x]; }, H, [&](long k, double v) { s.tor[k * W + x] = (float)v; });
}

// axis-1 passes (one thread per row), errors, mask (warp.py:49-63, clipped)
__global__ void k_lit_rows(int H, int W, LitSynth s, double eps, double eps2) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= H) return;
    const long r = (long)y * W;
    ufilt3([&](long k) { return s.tol[r + k]; }, W, [&](long k, double v) { s.ol[r + k] = (float)v; });
    ufilt3([&](long k) { return s.tor[r + k]; }, W, [&](long k, double v) { s.or_[r + k] = (float)v; });
    ufilt3([&](long k) { return s.tad[r + k]; }, W, [&](long k, double v) { s.ad[r + k] = v; });
    for (long k = 0; k < W; k++) {
        const float ql = 0.5f + 4.0f * s.ol[r + k], qr = 0.5f + 4.0f * s.or_[r + k];
        const double el = s.ad[r + k] * (double)ql, er = s.ad[r + k] * (double)qr;
        const double m = (er + eps) / (el + er + eps2);
        s.mask[r + k] = m < 0.0 ? 0.0 : (m > 1.0 ? 1.0 : m);
    }
}

// blend (warp.py:66-88): to_uint8(m a + (1 - m) b); 4:2:0 chroma with the 2x2-mean mask
__global__ void k_lit_blend(int fmt, int W, int H, LitSynth s, uint8_t* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = W * H;
    if (i < n) {
        const double m = s.mask[i];
        const int ch = fmt == FVV_RGB8 ? 3 : 1;
        for (int c = 0; c < ch; c++)
            out[i * ch + c] = lit_u8(m * (double)s.wl[i * ch + c] + (1.0 - m) * (double)s.wr[i * ch + c]);
    }
    if (fmt == FVV_YUV420) {
        const int cw = W / 2, chh = H / 2;
        if (i < cw * chh) {
            const int y = i / cw, x = i - (i / cw) * cw;
            const double* m = s.mask;
            const double sm = (m[(2 * y) * W + 2 * x] + m[(2 * y) * W + 2 * x + 1]) +
                              (m[(2 * y + 1) * W + 2 * x] + m[(2 * y + 1) * W + 2 * x + 1]);
            const double mc = sm / 4.0;
            for (int p = 0; p < 2; p++) {
                const size_t o = (size_t)n + (size_t)p * cw * chh + i;
                out[o] = lit_u8(mc * (double)s.wl[o] + (1.0 - mc) * (double)s.wr[o]);
            }
        }
    }
}

inline unsigned g1(long n, int t = 256) { return (unsigned)((n + t - 1) / t); }

}  // namespace

LitLayout lit_layout(int W, int H, int fmt, const int* block) {
    LitLayout L{};
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o = (o + bytes + 255) / 256 * 256; return r; };
    const size_t n = (size_t)W * H;
    for (int s = 0; s < 3; s++) {
        const int f = s == 0 ? 4 : (s == 1 ? 2 : 1);
        const size_t ns = (size_t)(W / f) * (H / f);
        const size_t nb = (size_t)((W / f + block[s] - 1) / block[s]) * ((H / f + block[s] - 1) / block[s]);
        for (int side = 0; side < 2; side++) L.lum[s][side] = take(ns * 4);
        for (int d = 0; d < 2; d++) {
            L.flow[s][d] = take(ns * 8);
            L.sad[s][d] = take(nb * 4);
        }
        L.off[s] = take(nb * 8);
    }
    L.base = take(n * 8);
    L.tw = take(n * 8);
    size_t fb = fmt == FVV_GRAY8 ? n : (fmt == FVV_RGB8 ? 3 * n : n + 2 * (size_t)(W / 2) * (H / 2));
    L.wl = take(fb);
    L.wr = take(fb);
    L.ad = take(n * 8);
    L.tad = take(n * 8);
    L.mask = take(n * 8);
    L.ol = take(n * 4);
    L.orr = take(n * 4);
    L.tol = take(n * 4);
    L.tor = take(n * 4);
    L.bytes = o;
    return L;
}

cudaError_t lit_interpolate(const LitLayout& L, uint8_t* ws, int W, int H, int fmt, const int* block,
                            const int* radius, const int16_t* const* cand_of_rank, double eps,
                            const uint8_t* left, const uint8_t* right, uint8_t* out, cudaStream_t st) {
    auto F = [&](size_t off) { return reinterpret_cast<float*>(ws + off); };
    auto F2 = [&](size_t off) { return reinterpret_cast<float2*>(ws + off); };
    const int n = W * H;
    // pyramid
    const uint8_t* fr[2] = {left, right};
    for (int side = 0; side < 2; side++) {
        k_lit_luma<<<g1(n), 256, 0, st>>>(fr[side], fmt, n, F(L.lum[2][side]));
        k_lit_box2<<<g1(n / 4), 256, 0, st>>>(F(L.lum[2][side]), H, W, F(L.lum[1][side]));
        k_lit_box2<<<g1(n / 16), 256, 0, st>>>(F(L.lum[1][side]), H / 2, W / 2, F(L.lum[0][side]));
    }
    // flow levels (flow.py:101-131): direction 0 = ref left, target right
    for (int s = 0; s < 3; s++) {
        const int f = s == 0 ? 4 : (s == 1 ? 2 : 1);
        const int w = W / f, h = H / f, B = block[s];
        const int nb = ((w + B - 1) / B) * ((h + B - 1) / B);
        for (int d = 0; d < 2; d++) {
            const float2* prev = s ? F2(L.flow[s - 1][d]) : nullptr;
            k_lit_base<<<g1((long)w * h), 256, 0, st>>>(prev, s ? h / 2 : 0, s ? w / 2 : 0, h, w, F(L.lum[s][1 - d]),
                                                        F2(L.base), reinterpret_cast<double*>(ws + L.tw));
            k_lit_search<<<g1(nb, 64), 64, 0, st>>>(F(L.lum[s][d]), reinterpret_cast<double*>(ws + L.tw), h, w,
                                                    radius[s], B, cand_of_rank[s], F2(L.off[s]),
                                                    reinterpret_cast<int*>(ws + L.sad[s][d]));
            k_lit_flow<<<g1((long)w * h), 256, 0, st>>>(F2(L.base), F2(L.off[s]), h, w, B, F2(L.flow[s][d]));
        }
    }
    // synthesis
    LitSynth sy;
    sy.wl = ws + L.wl; sy.wr = ws + L.wr;
    sy.ad = reinterpret_cast<double*>(ws + L.ad); sy.tad = reinterpret_cast<double*>(ws + L.tad);
    sy.mask = reinterpret_cast<double*>(ws + L.mask);
    sy.ol = F(L.ol); sy.or_ = F(L.orr); sy.tol = F(L.tol); sy.tor = F(L.tor);
    k_lit_warp<<<g1(n), 256, 0, st>>>(left, right, fmt, W, H, F2(L.flow[2][0]), F2(L.flow[2][1]), sy);
    if (fmt == FVV_YUV420)
        k_lit_warp_chroma<<<g1(n / 4), 256, 0, st>>>(left, right, W, H, F2(L.flow[2][0]), F2(L.flow[2][1]), sy);
    k_lit_cols<<<g1(W, 64), 64, 0, st>>>(H, W, sy);
    k_lit_rows<<<g1(H, 64), 64, 0, st>>>(H, W, sy, eps, 2.0 * eps);
    k_lit_blend<<<g1(n), 256, 0, st>>>(fmt, W, H, sy, out);
    return cudaGetLastError();
}

cudaError_t lit_level_err(const LitLayout& L, uint8_t* ws, int W, int H, const int* block, int level, int d,
                          double* err, cudaStream_t st) {
    const int f = level == 0 ? 4 : (level == 1 ? 2 : 1);
    const int w = W / f, h = H / f;
    k_lit_err<<<g1((long)w * h), 256, 0, st>>>(reinterpret_cast<const int*>(ws + L.sad[level][d]), h, w,
                                                block[level], err);
    return cudaGetLastError();
}

}  // namespace fvv
