// tile_kernels.cu -- dense-view tiling (cluster.py:77-191) on the device.
//
//   k_downscale      downscale(frame, f): f x f box mean, rint    cluster.py:77-89
//   k_assemble       assemble_cluster_frame from explicit tiles   cluster.py:143-191
//   k_rig_clusters   every cluster of a rig frame straight from   server/pipeline.py:273-292
//                    the global views buffer, downscale fused
//
// All integer: a box sum of uint8 samples is exact in the reference's f64,
// /f^2 is a power-of-two scaling for f = 2, 4 (exact), rint is half-even.
#include <cstdint>
#include <cuda_runtime.h>

#include "fvv_device.cuh"

namespace fvv {

// rint(s / n) for an exact integer sum s (n = factor^2), half to even.
__device__ __forceinline__ uint8_t box_round(int s, int n) {
    return to_u8(__ddiv_rn((double)s, (double)n));
}

struct FrameDims {
    int W, H, fmt, cw, ch;
    long bytes;
};

__host__ __device__ inline FrameDims dims_of(int W, int H, int fmt) {
    FrameDims d;
    d.W = W; d.H = H; d.fmt = fmt;
    d.cw = (W + 1) / 2; d.ch = (H + 1) / 2;
    d.bytes = fmt == FVV_GRAY8 ? (long)W * H
            : fmt == FVV_RGB8 ? (long)W * H * 3 : (long)W * H + 2L * d.cw * d.ch;
    return d;
}

// value of the downscaled frame `src` (dims s) at output byte offset `o` of
// the factor-f reduced frame (dims q)
__device__ __forceinline__ uint8_t downscaled_byte(const uint8_t* src, const FrameDims& s,
                                                   const FrameDims& q, int f, long o) {
    if (s.fmt == FVV_RGB8) {
        const int c = (int)(o % 3);
        const long p = o / 3;
        const int y = (int)(p / q.W), x = (int)(p % q.W);
        int acc = 0;
        for (int i = 0; i < f; i++)
            for (int j = 0; j < f; j++) acc += src[((long)(y * f + i) * s.W + x * f + j) * 3 + c];
        return box_round(acc, f * f);
    }
    const long ysz = (long)q.W * q.H;
    const uint8_t* pl = src;
    int pw = s.W, ow = q.W;
    long r = o;
    if (o >= ysz) {  // chroma planes (YUV420)
        const long csz = (long)q.cw * q.ch;
        const int p = (int)((o - ysz) / csz);
        r = (o - ysz) - p * csz;
        pl = src + (long)s.W * s.H + p * (long)s.cw * s.ch;
        pw = s.cw;
        ow = q.cw;
    }
    const int y = (int)(r / ow), x = (int)(r % ow);
    int acc = 0;
    for (int i = 0; i < f; i++)
        for (int j = 0; j < f; j++) acc += pl[(long)(y * f + i) * pw + x * f + j];
    return box_round(acc, f * f);
}

__global__ void k_downscale(FrameDims s, FrameDims q, int f, const uint8_t* __restrict__ frames,
                            uint8_t* __restrict__ out) {
    const long o = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const int n = blockIdx.y;
    if (o >= q.bytes) return;
    out[(long)n * q.bytes + o] = downscaled_byte(frames + (long)n * s.bytes, s, q, f, o);
}

// --- cluster geometry (cluster.py:135-140, 143-191) -------------------------


// Scalar form: one thread = one stitched byte (any geometry the reference accepts).
// skip_period > 0: tiles of views whose index is not a multiple of skip_period
// (the synthesized ones) were written by the synthesis kernel (fused tiling).
__global__ void k_rig_clusters_1(FrameDims fd, ClusterJobs jobs, ViewSrc vs,
                                 uint8_t* __restrict__ clusters, int skip_period) {
    pdl_enter();
    const uint8_t* __restrict__ views = vs.views;
    const ClusterJob jb = jobs.job[blockIdx.z];
    const int sw = jb.sw, sh = fd.H;
    const long ysz = (long)sw * sh;
    const long csz = (long)(sw / 2) * (sh / 2);
    const long total = fd.fmt == FVV_YUV420 ? ysz + 2 * csz : ysz;
    const long o = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= total) return;
    int p = 0;
    long r = o;
    if (o >= ysz) { p = 1 + (int)((o - ysz) / csz); r = (o - ysz) - (p - 1) * csz; }
    const int pw = p ? sw / 2 : sw;
    const int y = (int)(r / pw), x = (int)(r % pw);
    const int W = fd.W, H = fd.H;
    const int cellw = W / 4, cellh = H / 4;
    const int bx = p ? 2 * x : x, byy = p ? 2 * y : y;
    uint8_t v;
    if (bx < W) {
        const uint8_t* a = views + (long)(jb.anchor_view - vs.view_base) * fd.bytes;
        v = p ? a[(long)W * H + (p - 1) * (long)fd.cw * fd.ch + (long)y * fd.cw + x] : a[(long)y * W + x];
    } else {
        const int col = (bx - W) / cellw, row = byy / cellh;
        const int i = col * 4 + row;
        if (i >= jb.nsmall) {
            v = p ? 128 : 0;
        } else {
            int vi = jb.first_small + i;
            if (vi >= jb.skip) vi += 1;
            if (skip_period && vi % skip_period) return;
            const int tx = p ? x - (W + col * cellw) / 2 : x - (W + col * cellw);
            const int ty = p ? y - (row * cellh) / 2 : y - row * cellh;
            if (vi - vs.halo_first >= 0 && vi - vs.halo_first < vs.halo_count) {  // pre-downscaled
                const FrameDims qd = dims_of(cellw, cellh, fd.fmt);
                const uint8_t* q = vs.halo + (long)(vi - vs.halo_first) * qd.bytes;
                v = p ? q[(long)cellw * cellh + (p - 1) * (long)qd.cw * qd.ch + (long)ty * qd.cw + tx]
                      : q[(long)ty * cellw + tx];
            } else {
                const uint8_t* src = views + (long)(vi - vs.view_base) * fd.bytes;
                const uint8_t* pl = p ? src + (long)W * H + (p - 1) * (long)fd.cw * fd.ch : src;
                const int spw = p ? fd.cw : W;
                int acc = 0;
                for (int ii = 0; ii < 4; ii++)
                    for (int jj = 0; jj < 4; jj++) acc += pl[(long)(ty * 4 + ii) * spw + tx * 4 + jj];
                v = box_round(acc, 16);
            }
        }
    }
    clusters[jb.out_offset + o] = v;
}

// Vector form (W % 32 == 0): one thread = 4 consecutive bytes of one plane
// row: anchor copy, quarter-tile 4x4 box mean of view `vi` (one 16-byte
// read per source row), or padding (0 luma / 128 chroma).  With W % 32 == 0
// every cell edge and source row is 16-byte aligned, so a group never
// straddles a cell.
__global__ void k_rig_clusters(FrameDims fd, ClusterJobs jobs, ViewSrc vs,
                               uint8_t* __restrict__ clusters, int skip_period) {
    pdl_enter();
    const uint8_t* __restrict__ views = vs.views;
    const ClusterJob jb = jobs.job[blockIdx.z];
    const int sw = jb.sw, sh = fd.H;
    // 32-bit index math (a cluster frame is < 2^31 bytes: checked on the host): the
    // 64-bit divisions this replaces are software sequences of ~70 instructions each
    const unsigned ysz = (unsigned)sw * sh;
    const unsigned csz = (unsigned)(sw / 2) * (sh / 2);
    const unsigned total = fd.fmt == FVV_YUV420 ? ysz + 2 * csz : ysz;
    const unsigned o = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
    if (o >= total) return;
    int p = 0;
    unsigned r = o;
    if (o >= ysz) { p = o - ysz >= csz ? 2 : 1; r = (o - ysz) - (p - 1) * csz; }
    const unsigned pw = p ? sw / 2 : sw;
    const int y = (int)(r / pw), x = (int)(r - (unsigned)y * pw);
    const int W = fd.W, H = fd.H;
    const int cellw = W / 4, cellh = H / 4;
    const int bx = p ? 2 * x : x, byy = p ? 2 * y : y;  // luma-grid position
    uchar4 v;
    if (bx < W) {
        const uint8_t* a = views + (long)(jb.anchor_view - vs.view_base) * fd.bytes;
        const uint8_t* src = p ? a + (long)W * H + (p - 1) * (long)fd.cw * fd.ch + (long)y * fd.cw + x
                               : a + (long)y * W + x;
        v = *reinterpret_cast<const uchar4*>(src);
    } else {
        const int col = (bx - W) / cellw, row = byy / cellh;
        const int i = col * 4 + row;
        if (i >= jb.nsmall) {
            const uint8_t f = p ? 128 : 0;
            v = make_uchar4(f, f, f, f);
        } else {
            int vi = jb.first_small + i;
            if (vi >= jb.skip) vi += 1;
            if (skip_period && vi % skip_period) return;
            const int tx = p ? x - (W + col * cellw) / 2 : x - (W + col * cellw);
            const int ty = p ? y - (row * cellh) / 2 : y - row * cellh;
            if (vi - vs.halo_first >= 0 && vi - vs.halo_first < vs.halo_count) {  // pre-downscaled
                const FrameDims qd = dims_of(cellw, cellh, fd.fmt);
                const uint8_t* q = vs.halo + (long)(vi - vs.halo_first) * qd.bytes;
                const uint8_t* qs = p ? q + (long)cellw * cellh + (p - 1) * (long)qd.cw * qd.ch + (long)ty * qd.cw + tx
                                      : q + (long)ty * cellw + tx;
                *reinterpret_cast<uchar4*>(clusters + jb.out_offset + o) = *reinterpret_cast<const uchar4*>(qs);
                return;
            }
            const uint8_t* src = views + (long)(vi - vs.view_base) * fd.bytes;
            const uint8_t* pl = p ? src + (long)W * H + (p - 1) * (long)fd.cw * fd.ch : src;
            const int spw = p ? fd.cw : W;
            int acc[4] = {0, 0, 0, 0};
#pragma unroll
            for (int ii = 0; ii < 4; ii++) {
                const uint8_t* rowp = pl + (long)(ty * 4 + ii) * spw + tx * 4;
                const uint4 q = *reinterpret_cast<const uint4*>(rowp);  // 16 source bytes
                const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int k = 0; k < 4; k++)
                    acc[k] += (int)(w4[k] & 0xFF) + (int)((w4[k] >> 8) & 0xFF) +
                              (int)((w4[k] >> 16) & 0xFF) + (int)(w4[k] >> 24);
            }
            v = make_uchar4(box_round(acc[0], 16), box_round(acc[1], 16), box_round(acc[2], 16),
                            box_round(acc[3], 16));
        }
    }
    *reinterpret_cast<uchar4*>(clusters + jb.out_offset + o) = v;
}

// assemble_cluster_frame from explicit small tiles (already downscaled)
struct SmallTable {
    const uint8_t* small[256];
};

__global__ void k_assemble(FrameDims fd, int nsmall, int sw, const uint8_t* __restrict__ anchor,
                           SmallTable st, uint8_t* __restrict__ out) {
    const int sh = fd.H;
    const long ysz = (long)sw * sh;
    const long csz = (long)(sw / 2) * (sh / 2);
    const long total = fd.fmt == FVV_YUV420 ? ysz + 2 * csz : ysz;
    const long o = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= total) return;
    int p = 0;
    long r = o;
    if (o >= ysz) { p = 1 + (int)((o - ysz) / csz); r = (o - ysz) - (p - 1) * csz; }
    const int pw = p ? sw / 2 : sw;
    const int y = (int)(r / pw), x = (int)(r % pw);
    const int W = fd.W, H = fd.H;
    const int cellw = W / 4, cellh = H / 4;
    const FrameDims qd = dims_of(cellw, cellh, fd.fmt);
    const int bx = p ? 2 * x : x, byy = p ? 2 * y : y;
    uint8_t v;
    if (bx < W) {
        v = p ? anchor[(long)W * H + (p - 1) * (long)fd.cw * fd.ch + (long)y * fd.cw + x]
              : anchor[(long)y * W + x];
    } else {
        const int col = (bx - W) / cellw, row = byy / cellh;
        const int i = col * 4 + row;
        if (i >= nsmall) {
            v = p ? 128 : 0;
        } else {
            const uint8_t* s = st.small[i];
            const int tx = p ? x - (W + col * cellw) / 2 : x - (W + col * cellw);
            const int ty = p ? y - (row * cellh) / 2 : y - row * cellh;
            v = p ? s[(long)cellw * cellh + (p - 1) * (long)qd.cw * qd.ch + (long)ty * qd.cw + tx]
                  : s[(long)ty * cellw + tx];
        }
    }
    out[o] = v;
}

cudaError_t launch_rig_clusters_src(int W, int H, int fmt, const ClusterJob* jobs, int njobs,
                                    long max_cluster_bytes, const ViewSrc& vs, uint8_t* out,
                                    cudaStream_t st, int skip_period);

cudaError_t launch_downscale(int W, int H, int fmt, const uint8_t* frames, int n, int f,
                             uint8_t* out, cudaStream_t st) {
    FrameDims s = dims_of(W, H, fmt), q = dims_of(W / f, H / f, fmt);
    if (n <= 0) return cudaSuccess;
    dim3 grd((unsigned)((q.bytes + 255) / 256), n);
    k_downscale<<<grd, 256, 0, st>>>(s, q, f, frames, out);
    return cudaGetLastError();
}

cudaError_t launch_assemble(int W, int H, int fmt, const uint8_t* anchor,
                            const uint8_t* const* smalls, int nsmall, int sw, uint8_t* out,
                            cudaStream_t st) {
    FrameDims fd = dims_of(W, H, fmt);
    SmallTable t;
    for (int i = 0; i < nsmall && i < 256; i++) t.small[i] = smalls[i];
    const long total = (long)sw * H + (fmt == FVV_YUV420 ? 2L * (sw / 2) * (H / 2) : 0);
    k_assemble<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(fd, nsmall, sw, anchor, t, out);
    return cudaGetLastError();
}

cudaError_t launch_rig_clusters(int W, int H, int fmt, const ClusterJob* jobs, int njobs,
                                long max_cluster_bytes, const uint8_t* views, uint8_t* out,
                                cudaStream_t st, int skip_period) {
    ViewSrc vs{views, 0, nullptr, 0, 0};
    return launch_rig_clusters_src(W, H, fmt, jobs, njobs, max_cluster_bytes, vs, out, st, skip_period);
}

cudaError_t launch_rig_clusters_src(int W, int H, int fmt, const ClusterJob* jobs, int njobs,
                                    long max_cluster_bytes, const ViewSrc& vs, uint8_t* out,
                                    cudaStream_t st, int skip_period) {
    FrameDims fd = dims_of(W, H, fmt);
    for (int b = 0; b < njobs; b += kMaxClusters) {
        ClusterJobs cj;
        cudaError_t e;
        int n = njobs - b < kMaxClusters ? njobs - b : kMaxClusters;
        for (int i = 0; i < n; i++) cj.job[i] = jobs[b + i];
        if (W % 32 == 0) {
            dim3 grd((unsigned)((max_cluster_bytes / 4 + 255) / 256), 1, n);
            e = launch_k(true, k_rig_clusters, grd, dim3(256), 0, st, fd, cj, vs, out, skip_period);
        } else {
            dim3 grd((unsigned)((max_cluster_bytes + 255) / 256), 1, n);
            e = launch_k(true, k_rig_clusters_1, grd, dim3(256), 0, st, fd, cj, vs, out, skip_period);
        }
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace fvv
