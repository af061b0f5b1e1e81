// literal.h -- host interface of the literal (any InterpConfig) interpolation path
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace fvv {

struct LitLayout {             // byte offsets in the engine's literal workspace (one pair)
    size_t lum[3][2];          // f32 level luma per side
    size_t flow[3][2];         // float2 level flows per direction (kept for diagnostics)
    size_t sad[3][2];          // int best SAD per block
    size_t off[3];             // float2 block offsets (scratch)
    size_t base, tw;           // float2 base flow, f64 warped target (scratch)
    size_t wl, wr;             // u8 warped frames
    size_t ad, tad, mask;      // f64 planes
    size_t ol, orr, tol, tor;  // f32 occlusion planes
    size_t bytes;
};

struct LitSynth {
    uint8_t *wl, *wr;
    double *ad, *tad, *mask;
    float *ol, *or_, *tol, *tor;
};

LitLayout lit_layout(int W, int H, int fmt, const int* block);
cudaError_t lit_interpolate(const LitLayout& L, uint8_t* ws, int W, int H, int fmt, const int* block,
                            const int* radius, const int16_t* const* cand_of_rank, double eps,
                            const uint8_t* left, const uint8_t* right, uint8_t* out, cudaStream_t st);
cudaError_t lit_level_err(const LitLayout& L, uint8_t* ws, int W, int H, const int* block, int level, int d,
                          double* err, cudaStream_t st);

}  // namespace fvv
