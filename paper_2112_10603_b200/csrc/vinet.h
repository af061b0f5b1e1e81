// vinet.h -- host interface of the VINet engine (vinet_kernels.cu)
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "fvv_device.cuh"

namespace fvv {

constexpr int kVinMaxPairs = 64;

struct VinPairs {
    const uint8_t* left[kVinMaxPairs];
    const uint8_t* right[kVinMaxPairs];
};

struct VinWeights {                 // packed layer weights (convtc.py layouts), 3 blocks x 10 layers
    const void* w[3][10];
    const float* b[3][10];
};

struct VinLayout {
    int W, H, Wp, Hp, B;            // frame, 64-aligned canvas, pairs per chunk
    size_t img[3], state[3];        // per level: images (B, 2, 3, h, w) f32, state (B, 5, h, w) f32
    size_t xin, a0, a1, a2, head;   // block input (bf16 NHWC, cpad <= 32), activations, head (f32)
    size_t flows;                   // (B, 5, H, W) f32 scratch for fvv_vinet_rig
    size_t tiles;                   // VinTileDst[2 * kVinMaxViews] (fused tiling)
    size_t bytes;
};

struct VinTileDst {                 // one cluster tile of a synthesized view (fused tiling)
    long long off;                  // cluster frame's byte offset in the clusters buffer
    int sw;                         // its stitched width
    int cell;                       // small-tile index (col * 4 + row), -1 = none
    int pad;
};
constexpr int kVinMaxViews = 8192;
constexpr int kVinViewTab = 64;      // per-view synthesis constants passed as a kernel parameter
struct VinViewK {
    float t[kVinViewTab], kl[kVinViewTab], kr[kVinViewTab];
};  // tile-table capacity (global views per rig frame)

VinLayout vin_layout(int W, int H, int B);
cudaError_t vin_flows(const VinLayout& L, const VinWeights& w, const VinPairs& pp, int fmt, uint8_t* ws, float* out,
                      Prof* prof, cudaStream_t st);
cudaError_t vin_synth(const VinPairs& pp, int npairs, const float* state, int fmt, int W, int H, int nviews,
                      uint8_t* views, size_t frame_bytes, size_t pair_stride, cudaStream_t st);
cudaError_t vin_tile_table(const ClusterJobs& cj, int njobs, int nviews_total, VinTileDst* tab, cudaStream_t st);
cudaError_t vin_synth_tiled(const VinPairs& pp, int npairs, const float* state, int fmt, int W, int H, int nviews,
                            uint8_t* views, size_t frame_bytes, size_t pair_stride, const VinTileDst* tab, int v0,
                            int period, uint8_t* clusters, cudaStream_t st);

}  // namespace fvv
