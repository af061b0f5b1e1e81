// refine.h -- host interface of the RefineNet / ContextNet kernels (refine_kernels.cu)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace fvv {

constexpr int kRefMaxViews = 64;

struct RefSrc {  // source frames of the context net
    const uint8_t* frame[2 * kRefMaxViews];
};
struct RefViews {  // one entry per view of a refine batch
    const uint8_t* left[kRefMaxViews];
    const uint8_t* right[kRefMaxViews];
    const float* state[kRefMaxViews];  // (5, H, W) f32: F_m->l, F_m->r, mask logit
    float t[kRefMaxViews];
    uint8_t* out[kRefMaxViews];
};

cudaError_t ref_img(const RefSrc& src, int nsrc, int fmt, int W, int H, int Wp, int Hp, void* out, cudaStream_t st);
cudaError_t ref_inputs(const RefViews& rv, int nb, int fmt, int W, int H, int Wp, int Hp, void* x0, float* merged,
                       float* flow0, cudaStream_t st);
cudaError_t ref_flow_pool(const float* in, float* out, int w, int h, int nb, cudaStream_t st);
cudaError_t ref_warp_feat(const void* feat, int fs, int C, int w, int h, const float* flow, int comp, int src_mul,
                          int src_add, void* dst, int ds, int coff, int nb, cudaStream_t st);
cudaError_t nhwc_copy(const void* src, int ss, int C, void* dst, int ds, int coff, long long npix, cudaStream_t st);
cudaError_t ref_out(const RefViews& rv, int nb, int fmt, int W, int H, int Wp, int Hp, const float* r, int rs,
                    const float* merged, cudaStream_t st);

}  // namespace fvv
