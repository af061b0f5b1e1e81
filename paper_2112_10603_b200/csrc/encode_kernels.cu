// encode_kernels.cu -- the FVT1 tile encoder's transform stage on the device
// (the encoder hand-off after the tiling).
//
// Reference: codec.py:138-153 _encode_plane, codec.py:174-216 encode_frame,
// dct.py:9-36 (orthonormal DCT-II by einsum), dct.py:39-81 (lossless lifting),
// dct.py:84-95 (zigzag).  Per 8x8 block of an edge-padded plane (or P-frame
// residual against the previous reconstruction):
//   lossy:    q = rint(DCT(b) / step); recon = rint(IDCT(q * step))
//   lossless: q = lift(b);            recon = b
// then recon is committed clip(ref + recon, 0, 255) (P) or clip(recon) (I),
// and q is written in zigzag order with the (run, level) token count of the
// block.  k_enc_tokens then writes the 3-byte token stream (codec.py:68-98
// _tokens_encode); the host only runs DEFLATE (zlib level 6) and frames the
// record.
//
// Bit-exactness of the DCT: numpy evaluates dct8_blocks' einsum as two BLAS
// dgemm contractions (einsum_path: "njk,ij->ikn" then "ikn,lk->nil"), and the
// OpenBLAS kernel of the reference's host accumulates every output as a
// sequential FMA chain over k = 0..7 from 0.  The same chains here
// (__fma_rn, j ascending) give the same doubles; tests/test_encoder.py pins
// the model against the reference's own dct8_blocks / idct8_blocks, and the
// GPU test compares whole records with reference-generated goldens.
#include <cuda_runtime.h>

#include <cstdint>

#include "encode.h"

namespace fvv {

__constant__ double c_dct[64];  // dct.py:9-17 _C, uploaded from exact host constants
__constant__ uint8_t c_zz[64];  // dct.py:84-91 zigzag order

__device__ __forceinline__ int clamp255(int v) { return v < 0 ? 0 : (v > 255 ? 255 : v); }

// lifting (dct.py:39-56) on 8 values with stride s, in place: [L3, H3, H2 x2, H1 x4]
__device__ __forceinline__ void lift8(int* a, int s) {
    int tmp[8];
    for (int n = 8; n > 1; n >>= 1) {
        for (int i = 0; i < n / 2; i++) {
            const int e = a[(2 * i) * s], o = a[(2 * i + 1) * s];
            tmp[i] = (e + o) >> 1;
            tmp[n / 2 + i] = e - o;
        }
        for (int i = 0; i < n; i++) a[i * s] = tmp[i];
    }
}

// One CTA = 4 blocks x 64 threads; thread (i, k) of a block owns coefficient (i, k).
__global__ void __launch_bounds__(256) k_enc_blocks(const EncJob* __restrict__ jobs, int njobs, long long total,
                                                    int lossless, int16_t* __restrict__ zz, int* __restrict__ ntok) {
    __shared__ double sb[4][64];   // block samples, then stage-1 products
    __shared__ double st[4][64];
    __shared__ int si[4][64];
    const int sub = threadIdx.x >> 6, e = threadIdx.x & 63;
    const int i = e >> 3, k = e & 7;
    const long long gblk = (long long)blockIdx.x * 4 + sub;
    // job lookup: jobs sorted by block0 (binary search, last job with block0 <= gblk)
    int lo = 0, hi = njobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].block0 <= gblk) lo = mid;
        else hi = mid - 1;
    }
    const EncJob J = jobs[lo];
    const long long lb = gblk - J.block0;
    const bool live = gblk < total && lb < (long long)J.nbx * J.nby;
    const int by = live ? (int)(lb / J.nbx) : 0, bx = live ? (int)(lb - (long long)by * J.nbx) : 0;
    // edge-padded sample (codec.py:56-61 np.pad mode="edge"), minus the reference for P
    const int y = min(by * 8 + i, J.h - 1), x = min(bx * 8 + k, J.w - 1);
    int v = 0;
    if (live) {
        v = J.src[(long long)y * J.pitch + x];
        if (J.is_p) v -= J.prev[(long long)y * J.w + x];
    }
    if (lossless) {  // kernel-wide (quality 100): the CTA's barriers stay uniform
        si[sub][e] = v;
        __syncthreads();
        if (live && e < 8) lift8(&si[sub][e * 8], 1);   // rows
        __syncthreads();
        if (live && e < 8) lift8(&si[sub][e], 8);       // columns
        __syncthreads();
        if (live) {
            // recon == the residual / samples exactly (unlift . lift = id)
            if (i + by * 8 < J.h && k + bx * 8 < J.w) {
                const int ry = by * 8 + i, rx = bx * 8 + k;
                const int ref = J.is_p ? J.prev[(long long)ry * J.w + rx] : 0;
                J.recon[(long long)ry * J.w + rx] = (uint8_t)clamp255(ref + v);
            }
        }
    } else {
        sb[sub][e] = (double)v;
        __syncthreads();
        // stage 1 ("njk,ij->ikn"): T[i][k] = sum_j C[i][j] * B[j][k]
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) acc = __fma_rn(c_dct[i * 8 + j], sb[sub][j * 8 + k], acc);
        st[sub][e] = acc;
        __syncthreads();
        // stage 2 ("ikn,lk->nil"): O[i][l] = sum_k T[i][k] * C[l][k]   (thread e = (i, l))
        double o = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk++) o = __fma_rn(st[sub][i * 8 + kk], c_dct[k * 8 + kk], o);
        const int q = __double2int_rn(__ddiv_rn(o, (double)J.step));  // np.rint(coeffs / step)
        si[sub][e] = q;
        __syncthreads();
        // reconstruction: rint(idct(q * step)), idct8_blocks = einsum("ji,njk,kl->nil")
        // path "njk,ji->ikn" then "ikn,kl->nil"
        sb[sub][e] = (double)(q * J.step);
        __syncthreads();
        double a1 = 0.0;
#pragma unroll
        for (int j = 0; j < 8; j++) a1 = __fma_rn(c_dct[j * 8 + i], sb[sub][j * 8 + k], a1);
        st[sub][e] = a1;
        __syncthreads();
        double a2 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; kk++) a2 = __fma_rn(st[sub][i * 8 + kk], c_dct[kk * 8 + k], a2);
        if (live) {
            const int ry = by * 8 + i, rx = bx * 8 + k;
            if (ry < J.h && rx < J.w) {
                const int r = __double2int_rn(a2);
                const int ref = J.is_p ? J.prev[(long long)ry * J.w + rx] : 0;
                J.recon[(long long)ry * J.w + rx] = (uint8_t)clamp255(ref + r);
            }
        }
    }
    __syncthreads();
    // zigzag (codec.py:147 qc.reshape(-1, 64)[:, ZIGZAG]) and the block's token count
    const int zval = si[sub][c_zz[e]];
    if (live) zz[gblk * 64 + e] = (int16_t)zval;
    const unsigned nz = __ballot_sync(0xffffffffu, zval != 0);
    __shared__ int cnt[4][2];
    if ((e & 31) == 0) cnt[sub][e >> 5] = __popc(nz);
    __syncthreads();
    if (live && e == 0) ntok[gblk] = cnt[sub][0] + cnt[sub][1] + 1;  // + EOB
}

// 3-byte tokens of every block (codec.py:68-98): (run, level lo, level hi) per
// nonzero coefficient, (0xFF, 0, 0) at the end of the block.  off = exclusive
// prefix sum of ntok per job's first block (tokens of a job are contiguous).
__global__ void k_enc_tokens(const int16_t* __restrict__ zz, const long long* __restrict__ tok_off,
                             long long nblocks, uint8_t* __restrict__ out) {
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nblocks) return;
    uint8_t* o = out + tok_off[b] * 3;
    const int16_t* z = zz + b * 64;
    int prev = -1;
    for (int p = 0; p < 64; p++) {
        const int v = z[p];
        if (v) {
            o[0] = (uint8_t)(p - prev - 1);
            o[1] = (uint8_t)(v & 0xFF);
            o[2] = (uint8_t)((v >> 8) & 0xFF);
            o += 3;
            prev = p;
        }
    }
    o[0] = 0xFF;
    o[1] = 0;
    o[2] = 0;
}

cudaError_t enc_set_constants(const double* dct64, const uint8_t* zz64) {
    cudaError_t e = cudaMemcpyToSymbol(c_dct, dct64, 64 * sizeof(double));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_zz, zz64, 64);
    return e;
}

cudaError_t enc_blocks(const EncJob* jobs, int njobs, long long total_blocks, int lossless, int16_t* zz, int* ntok,
                       cudaStream_t st) {
    const long long n = total_blocks;
    if (n <= 0) return cudaSuccess;
    k_enc_blocks<<<(unsigned)((n + 3) / 4), 256, 0, st>>>(jobs, njobs, n, lossless, zz, ntok);
    return cudaGetLastError();
}

cudaError_t enc_tokens(const int16_t* zz, const long long* tok_off, long long nblocks, uint8_t* out,
                       cudaStream_t st) {
    if (nblocks <= 0) return cudaSuccess;
    k_enc_tokens<<<(unsigned)((nblocks + 127) / 128), 128, 0, st>>>(zz, tok_off, nblocks, out);
    return cudaGetLastError();
}

}  // namespace fvv
