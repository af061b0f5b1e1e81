// encode.h -- host interface of the tile encoder's device stage (encode_kernels.cu)
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace fvv {

// One (tile, plane) of a frame record: codec.py:174-216 encode_frame's per-plane
// _encode_plane call.  `src` points at the tile's plane inside the stitched
// cluster frame (row pitch `pitch`); prev / recon are compact w x h planes of
// the tile's reconstruction (P reference in, committed reconstruction out).
struct EncJob {
    const uint8_t* src;
    const uint8_t* prev;  // null for I frames
    uint8_t* recon;
    long long block0;     // first 8x8 block of this job in the batch
    int pitch, w, h;
    int nbx, nby;
    int is_p, step, pad;
};

cudaError_t enc_set_constants(const double* dct64, const uint8_t* zz64);
cudaError_t enc_blocks(const EncJob* jobs, int njobs, long long total_blocks, int lossless, int16_t* zz, int* ntok,
                       cudaStream_t st);
cudaError_t enc_tokens(const int16_t* zz, const long long* tok_off, long long nblocks, uint8_t* out,
                       cudaStream_t st);

}  // namespace fvv
