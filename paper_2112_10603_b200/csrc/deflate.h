// deflate.h -- host interface of the device DEFLATE (deflate_kernels.cu):
// zlib.compress(stream, 6)[2:-4] of many independent byte streams at once,
// byte for byte (the raw DEFLATE data codec.py:148 keeps).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace fvv {

// Scratch for a batch of streams with lengths len[0..S) (host).
size_t zd_scratch_bytes(const int64_t* len, int nstreams);

// data: device bytes, stream s = data[in_off[s], in_off[s+1]) (host offsets).
// out: device, capacity >= zd_out_capacity(len, S); zeroed and filled here,
// the streams packed back to back: stream s = out[out_off[s], out_off[s+1])
// (out_off: device, S + 1 entries, written by the call).
size_t zd_out_capacity(const int64_t* len, int nstreams);
cudaError_t zd_deflate(const uint8_t* data, const int64_t* in_off, int nstreams, uint8_t* out, int64_t* out_off,
                       void* scratch, size_t scratch_bytes, cudaStream_t st);

}  // namespace fvv
