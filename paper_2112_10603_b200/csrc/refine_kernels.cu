// refine_kernels.cu -- the non-convolution kernels of RefineNet + ContextNet
// (architecture in vinet_params.py, fp32 oracle
// oracle/vinet_ref.py refine_view).  The 21 convolution layers per view run
// on the tcgen05 kernel (conv_tc.cu) through fvv_conv2d_bf16; these kernels
// build the U-Net input, the flow pyramid, the warped context features (written
// straight into the U-Net's concat buffers at a channel offset), the skip
// copies and the residual output.
//
// Layouts: activations NHWC bf16 [n][h][w][cstride]; flows f32 planar.
// The network runs on the 64-aligned canvas (Wp, Hp) of the VINet engine,
// edge-replicated from the frame (W, H).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "fvv_device.cuh"
#include "refine.h"

namespace fvv {

// net_image (vinet_ref.py): (3, H, W) in [0, 1] -- RGB, (Y, U, V) with chroma
// repeated 2x2, or (Y, 0.5, 0.5)
__device__ __forceinline__ float3 net_px(const uint8_t* __restrict__ f, int fmt, int W, int H, int x, int y) {
    const float k = 1.0f / 255.0f;
    if (fmt == FVV_RGB8) {
        const uint8_t* p = f + ((size_t)y * W + x) * 3;
        return make_float3(p[0] * k, p[1] * k, p[2] * k);
    }
    const float Y = f[(size_t)y * W + x] * k;
    if (fmt == FVV_GRAY8) return make_float3(Y, 127.5f * k, 127.5f * k);
    const int cw = (W + 1) / 2, ch = (H + 1) / 2;
    const size_t co = (size_t)(y >> 1) * cw + (x >> 1);
    return make_float3(Y, f[(size_t)W * H + co] * k, f[(size_t)W * H + (size_t)cw * ch + co] * k);
}

// warp (vinet_ref.py): backward bilinear at (x + fx, y + fy), clamped
__device__ __forceinline__ float3 warp_px(const uint8_t* __restrict__ f, int fmt, int W, int H, int x, int y,
                                          float fx, float fy) {
    const float sx = fminf(fmaxf((float)x + fx, 0.0f), (float)(W - 1));
    const float sy = fminf(fmaxf((float)y + fy, 0.0f), (float)(H - 1));
    const int x0 = min((int)floorf(sx), W - 2), y0 = min((int)floorf(sy), H - 2);
    const float ax = sx - (float)x0, ay = sy - (float)y0;
    const float3 a = net_px(f, fmt, W, H, x0, y0), b = net_px(f, fmt, W, H, x0 + 1, y0);
    const float3 c = net_px(f, fmt, W, H, x0, y0 + 1), d = net_px(f, fmt, W, H, x0 + 1, y0 + 1);
    auto bl = [&](float pa, float pb, float pc, float pd) {
        const float top = (1.0f - ax) * pa + ax * pb, bot = (1.0f - ax) * pc + ax * pd;
        return (1.0f - ay) * top + ay * bot;
    };
    return make_float3(bl(a.x, b.x, c.x, d.x), bl(a.y, b.y, c.y, d.y), bl(a.z, b.z, c.z, d.z));
}

// Context-net input: the canvas image of every source frame, NHWC bf16 cstride 16
__global__ void k_ref_img(RefSrc src, int nsrc, int fmt, int W, int H, int Wp, int Hp,
                          __nv_bfloat16* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, s = blockIdx.z;
    if (x >= Wp || s >= nsrc) return;
    const float3 v = net_px(src.frame[s], fmt, W, H, min(x, W - 1), min(y, H - 1));
    __nv_bfloat16* o = out + (((size_t)s * Hp + y) * Wp + x) * 16;
    __align__(16) __nv_bfloat16 buf[16];
#pragma unroll
    for (int i = 0; i < 16; i++) buf[i] = __float2bfloat16_rn(0.0f);
    buf[0] = __float2bfloat16_rn(v.x);
    buf[1] = __float2bfloat16_rn(v.y);
    buf[2] = __float2bfloat16_rn(v.z);
    reinterpret_cast<uint4*>(o)[0] = reinterpret_cast<const uint4*>(buf)[0];
    reinterpret_cast<uint4*>(o)[1] = reinterpret_cast<const uint4*>(buf)[1];
}

// U-Net input of every view (refine_inputs): x0 NHWC bf16 cstride 32 =
// (A, B, warp(A, F_l,t), warp(B, F_r,t), w_t, F_l,t, F_r,t); merged (3, H, W) f32;
// the canvas flows (F_l,t, F_r,t) f32 planar (4, Hp, Wp) for the context pyramid
__global__ void k_ref_in(RefViews rv, int nloop, int fmt, int W, int H, int Wp, int Hp, __nv_bfloat16* __restrict__ x0,
                         float* __restrict__ merged, float* __restrict__ flow0) {
    // nloop > 1: views b0 .. b0 + nloop - 1 share their source pair and state (a
    // refine batch of one camera gap): the state, the mask and the unwarped frames
    // are read once per pixel and only the t-dependent channels are redone
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, b0 = blockIdx.z * nloop;
    if (x >= Wp) return;
    const int xs = min(x, W - 1), ys = min(y, H - 1);
    const uint8_t* L = rv.left[b0];
    const uint8_t* R = rv.right[b0];
    const float* S = rv.state[b0];
    const size_t plane = (size_t)W * H, pix = (size_t)ys * W + xs;
    const float sfx = S[pix], sfy = S[plane + pix], sgx = S[2 * plane + pix], sgy = S[3 * plane + pix];
    const float m = 1.0f / (1.0f + expf(-S[4 * plane + pix]));
    const float3 A = net_px(L, fmt, W, H, xs, ys), B = net_px(R, fmt, W, H, xs, ys);
    const size_t cp = (size_t)Wp * Hp, co = (size_t)y * Wp + x;
    for (int k = 0; k < nloop; k++) {
        const int b = b0 + k;
        const float t = rv.t[b];
        const float tl = 2.0f * t, tr = 2.0f * (1.0f - t);
        const float flx = sfx * tl, fly = sfy * tl;
        const float frx = sgx * tr, fry = sgy * tr;
        const float wt = (1.0f - t) * m / ((1.0f - t) * m + t * (1.0f - m));
        const float3 wl = warp_px(L, fmt, W, H, xs, ys, flx, fly), wr = warp_px(R, fmt, W, H, xs, ys, frx, fry);
        __align__(16) __nv_bfloat16 buf[32];
        const float v[17] = {A.x, A.y, A.z, B.x, B.y, B.z, wl.x, wl.y, wl.z, wr.x, wr.y, wr.z, wt, flx, fly, frx, fry};
#pragma unroll
        for (int i = 0; i < 32; i++) buf[i] = __float2bfloat16_rn(i < 17 ? v[i] : 0.0f);
        uint4* o = reinterpret_cast<uint4*>(x0 + (((size_t)b * Hp + y) * Wp + x) * 32);
#pragma unroll
        for (int i = 0; i < 4; i++) o[i] = reinterpret_cast<const uint4*>(buf)[i];
        float* fo = flow0 + (size_t)b * 4 * cp;
        fo[co] = flx;
        fo[cp + co] = fly;
        fo[2 * cp + co] = frx;
        fo[3 * cp + co] = fry;
        if (x < W && y < H) {
            float* mo = merged + (size_t)b * 3 * plane;
            mo[pix] = wt * wl.x + (1.0f - wt) * wr.x;
            mo[plane + pix] = wt * wl.y + (1.0f - wt) * wr.y;
            mo[2 * plane + pix] = wt * wl.z + (1.0f - wt) * wr.z;
        }
    }
}

// context flow pyramid: pool2(flow) * 0.5, 4 planar channels
__global__ void k_ref_flow_pool(const float* __restrict__ in, float* __restrict__ out, int w, int h, int nb) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, bc = blockIdx.z;
    const int wo = w / 2, ho = h / 2;
    if (x >= wo || bc >= nb * 4) return;
    const float* p = in + (size_t)bc * w * h + (size_t)(2 * y) * w + 2 * x;
    out[(size_t)bc * wo * ho + (size_t)y * wo + x] = (((p[0] + p[1]) + (p[w] + p[w + 1])) * 0.25f) * 0.5f;
}

// warp NHWC bf16 features (channels [0, C) of feat, cstride fs) of source src_of(b)
// with flow channels (2 comp, 2 comp + 1) of the level-k flow -> dst channels
// [coff, coff + C) (cstride ds).  One thread = 8 channels of one pixel.
__global__ void k_ref_warp_feat(const __nv_bfloat16* __restrict__ feat, int fs, int C, int w, int h,
                                const float* __restrict__ flow, int comp, int src_mul, int src_add,
                                __nv_bfloat16* __restrict__ dst, int ds, int coff, int nb) {
    const int cg = C / 8;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long per = (long long)w * h * cg;
    const int b = (int)(i / per);
    if (b >= nb) return;
    const long long r = i - (long long)b * per;
    const int pix = (int)(r / cg), g = (int)(r - (long long)pix * cg);
    const int y = pix / w, x = pix - y * w;
    const size_t cp = (size_t)w * h;
    const float* fb = flow + (size_t)b * 4 * cp;
    const float fx = fb[(size_t)comp * cp + pix], fy = fb[(size_t)(comp + 1) * cp + pix];
    const float sx = fminf(fmaxf((float)x + fx, 0.0f), (float)(w - 1));
    const float sy = fminf(fmaxf((float)y + fy, 0.0f), (float)(h - 1));
    const int x0 = min((int)floorf(sx), w - 2), y0 = min((int)floorf(sy), h - 2);
    const float ax = sx - (float)x0, ay = sy - (float)y0;
    const int s = b * src_mul + src_add;
    const __nv_bfloat16* base = feat + (size_t)s * cp * fs + (size_t)g * 8;
    auto ld = [&](int yy, int xx, float (&v)[8]) {
        const uint4 q = *reinterpret_cast<const uint4*>(base + ((size_t)yy * w + xx) * fs);
        const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const float2 f = __bfloat1622float2(p[k]);
            v[2 * k] = f.x;
            v[2 * k + 1] = f.y;
        }
    };
    float a[8], bb[8], c[8], d[8];
    ld(y0, x0, a);
    ld(y0, x0 + 1, bb);
    ld(y0 + 1, x0, c);
    ld(y0 + 1, x0 + 1, d);
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const float top = (1.0f - ax) * a[k] + ax * bb[k], bot = (1.0f - ax) * c[k] + ax * d[k];
        o[k] = __float2bfloat16_rn((1.0f - ay) * top + ay * bot);
    }
    *reinterpret_cast<uint4*>(dst + ((size_t)b * cp + pix) * ds + coff + (size_t)g * 8) =
        *reinterpret_cast<const uint4*>(o);
}

// skip connection: channels [0, C) of src (cstride ss) -> dst channels [coff, coff + C) (cstride ds)
__global__ void k_nhwc_copy(const __nv_bfloat16* __restrict__ src, int ss, int C, __nv_bfloat16* __restrict__ dst,
                            int ds, int coff, long long npix) {
    const int cg = C / 8;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= npix * cg) return;
    const long long p = i / cg;
    const int g = (int)(i - p * cg);
    *reinterpret_cast<uint4*>(dst + p * ds + coff + g * 8) = *reinterpret_cast<const uint4*>(src + p * ss + g * 8);
}

// output: out = clip(merged + 2 sigmoid(r) - 1, 0, 1) -> packed uint8 view
// (RGB: rint per channel; Y: rint; U, V: rint of the 2x2 mean of 255 * out).
// One thread = one 2x2 pixel block.
__global__ void k_ref_out(RefViews rv, int fmt, int W, int H, int Wp, int Hp, const float* __restrict__ r,
                          int rs, const float* __restrict__ merged) {
    const int bx = blockIdx.x * blockDim.x + threadIdx.x, by = blockIdx.y, b = blockIdx.z;
    if (2 * bx >= W) return;
    const size_t plane = (size_t)W * H;
    const float* mo = merged + (size_t)b * 3 * plane;
    const float* rb = r + (size_t)b * Hp * Wp * rs;
    uint8_t* out = rv.out[b];
    float acc1 = 0.0f, acc2 = 0.0f, c1[4], c2[4];
    int q = 0;
    for (int dy = 0; dy < 2; dy++)
        for (int dx = 0; dx < 2; dx++, q++) {
            const int x = 2 * bx + dx, y = 2 * by + dy;
            const size_t pix = (size_t)y * W + x;
            const float* rp = rb + ((size_t)y * Wp + x) * rs;
            float o[3];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const float s = 1.0f / (1.0f + expf(-rp[c]));
                o[c] = fminf(fmaxf(mo[c * plane + pix] + (s * 2.0f - 1.0f), 0.0f), 1.0f) * 255.0f;
            }
            if (fmt == FVV_RGB8) {
#pragma unroll
                for (int c = 0; c < 3; c++) out[pix * 3 + c] = (uint8_t)fminf(fmaxf(rintf(o[c]), 0.0f), 255.0f);
            } else {
                out[pix] = (uint8_t)fminf(fmaxf(rintf(o[0]), 0.0f), 255.0f);
            }
            c1[q] = o[1];
            c2[q] = o[2];
        }
    if (fmt == FVV_YUV420) {
        acc1 = ((c1[0] + c1[1]) + (c1[2] + c1[3])) * 0.25f;
        acc2 = ((c2[0] + c2[1]) + (c2[2] + c2[3])) * 0.25f;
        const int cw = (W + 1) / 2, ch = (H + 1) / 2;
        const size_t co = (size_t)by * cw + bx;
        out[plane + co] = (uint8_t)fminf(fmaxf(rintf(acc1), 0.0f), 255.0f);
        out[plane + (size_t)cw * ch + co] = (uint8_t)fminf(fmaxf(rintf(acc2), 0.0f), 255.0f);
    }
}

cudaError_t ref_img(const RefSrc& src, int nsrc, int fmt, int W, int H, int Wp, int Hp, void* out, cudaStream_t st) {
    k_ref_img<<<dim3((Wp + 127) / 128, Hp, nsrc), 128, 0, st>>>(src, nsrc, fmt, W, H, Wp, Hp,
                                                               static_cast<__nv_bfloat16*>(out));
    return cudaGetLastError();
}

cudaError_t ref_inputs(const RefViews& rv, int nb, int fmt, int W, int H, int Wp, int Hp, void* x0, float* merged,
                       float* flow0, cudaStream_t st) {
    bool shared = true;
    for (int b = 1; b < nb; b++)
        shared = shared && rv.left[b] == rv.left[0] && rv.right[b] == rv.right[0] && rv.state[b] == rv.state[0];
    const int nloop = shared ? nb : 1;
    k_ref_in<<<dim3((Wp + 127) / 128, Hp, nb / nloop), 128, 0, st>>>(rv, nloop, fmt, W, H, Wp, Hp,
                                                                    static_cast<__nv_bfloat16*>(x0), merged, flow0);
    return cudaGetLastError();
}

cudaError_t ref_flow_pool(const float* in, float* out, int w, int h, int nb, cudaStream_t st) {
    k_ref_flow_pool<<<dim3((w / 2 + 127) / 128, h / 2, nb * 4), 128, 0, st>>>(in, out, w, h, nb);
    return cudaGetLastError();
}

cudaError_t ref_warp_feat(const void* feat, int fs, int C, int w, int h, const float* flow, int comp, int src_mul,
                          int src_add, void* dst, int ds, int coff, int nb, cudaStream_t st) {
    const long long n = (long long)nb * w * h * (C / 8);
    k_ref_warp_feat<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(feat), fs, C, w, h, flow, comp, src_mul, src_add,
        static_cast<__nv_bfloat16*>(dst), ds, coff, nb);
    return cudaGetLastError();
}

cudaError_t nhwc_copy(const void* src, int ss, int C, void* dst, int ds, int coff, long long npix, cudaStream_t st) {
    const long long n = npix * (C / 8);
    k_nhwc_copy<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), ss, C,
                                                             static_cast<__nv_bfloat16*>(dst), ds, coff, npix);
    return cudaGetLastError();
}

cudaError_t ref_out(const RefViews& rv, int nb, int fmt, int W, int H, int Wp, int Hp, const float* r, int rs,
                    const float* merged, cudaStream_t st) {
    k_ref_out<<<dim3((W / 2 + 127) / 128, H / 2, nb), 128, 0, st>>>(rv, fmt, W, H, Wp, Hp, r, rs, merged);
    return cudaGetLastError();
}

}  // namespace fvv
