// conv_tc.h -- host interface of the tcgen05 implicit-GEMM convolution (conv_tc.cu)
#pragma once
#include <cuda_runtime.h>

namespace fvv {

constexpr int kConvMaxTaps = 16;

struct ConvTCParams {
    int B, cpad, wrow0, kc_per_tap;          // filled in by conv_tc()
    int Hg, Wg;                              // output grid (per image / per phase)
    int sy, sx, by0, bx0;                    // input coordinate of tap 0 = g * s + b0
    int ntaps;
    int tdy[kConvMaxTaps], tdx[kConvMaxTaps];  // per-tap input offsets
    int omy, omx, oay, oax;                  // output coordinate = g * om + oa
    int Hout, Wout, ostride, ocoff, N;       // output tensor, channel placement, real channels
    int act, out_f32;                        // 1 = ReLU; 1 = fp32 output (else bf16)
    int shuffle_c;                           // > 0: sub-pixel output (fp32 or bf16): channel n = phase * shuffle_c + c
                                             // lands at (2 gy + phase / 2, 2 gx + phase % 2), channel c
};

cudaError_t conv_tc(const void* x, int B, int Hin, int Win, int cpad, const void* w, int wrows, int wrow0,
                    int ntile, const float* bias, void* out, const ConvTCParams& p, cudaStream_t st);

}  // namespace fvv
