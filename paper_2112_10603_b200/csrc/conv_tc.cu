// conv_tc.cu -- implicit-GEMM convolution on the 5th-generation tensor cores
// (tcgen05 + TMEM + TMA) for the VINet flow/fusion blocks (PAPER.md:320-337,
// SURVEY.md sec. 8(b)/(c)/(d) north-star rows).
//
// GEMM view: D[m][n] = sum_k A[m][k] * B[n][k] with
//   m = an output pixel of one output row (tile: 128 consecutive pixels),
//   n = an output channel (tile: NT <= 256),
//   k = (tap, input channel); one K chunk = one tap x (SW / 2) channels.
// A chunk is an input-row segment of 128 pixels (stride sx) x chunk channels,
// fetched by one 4-D TMA copy from the NHWC bf16 activation tensor; TMA's
// out-of-bounds zero fill is the convolution padding.  B chunks come from the
// K-major bf16 weight matrix by a 2-D TMA copy.  Both land in the canonical
// K-major swizzled layout (SW = 32/64/128 bytes per row) the UMMA descriptors
// describe.  One elected thread issues tcgen05.mma (M=128, N=NT, K=16) into a
// TMEM accumulator; the 4 warps read it back with tcgen05.ld and apply
// bias + activation in the epilogue.
//
// Roles (128 threads): warp 0 / lane 0 = TMA producer, warp 1 / lane 0 = MMA
// issuer, warp 2 = TMEM allocator; all 4 warps = epilogue (warp w owns TMEM
// lanes 32w..32w+31, i.e. output pixels 32w..32w+31 of the tile).
// Pipeline: kStages smem stages, full/empty mbarriers, one accumulator barrier.
//
// Transposed convolutions (k4 s2 p1) run as four 2x2-tap phase convolutions
// on the input grid whose outputs interleave (omy = omx = 2).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>

#include "conv_tc.h"

namespace fvv {


// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}
// K-major, swizzled canonical layout: rows of SW bytes, 8-row groups SBO = 8*SW apart
template <int SW>
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    constexpr uint64_t layout = SW == 128 ? 2 : (SW == 64 ? 4 : 6);
    uint64_t d = (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)1 << 16;                        // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * SW) >> 4) << 32;          // SBO
    d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
    d |= layout << 61;
    return d;
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// ---------------------------------------------------------------------------
// the kernel: persistent, warp-specialised, double-buffered accumulators
// ---------------------------------------------------------------------------
// A CTA loops over output tiles (128 pixels of one output row x NT channels).
// Warp 0 / lane 0 streams K chunks with TMA into kStages smem stages; warp 1 /
// lane 0 issues the MMAs of tile i into TMEM accumulator i % 2; warps 2-5 drain
// accumulator (i - 1) % 2 meanwhile (tcgen05.ld, bias, ReLU, stores) -- the
// epilogue of one tile overlaps the MMAs of the next.
// MT output rows per tile (MT accumulators of 128 x NT per buffer) share each
// weight chunk; MT = 2 whenever two double-buffered sets fit TMEM (NT <= 128).
// RR > 0 (row reuse, 3x3 stride-1 convolutions with a small N): a tile is RR output rows;
// one stage holds the RR + 2 input-row segments of one (dx, channel chunk) and the three
// weight chunks of taps (0..2, dx), and output row r takes rows r + dy with B_dy -- every
// input row segment is fetched once per tile instead of once per (row, dy) tap.
#ifndef FVV_CONV_RR_STAGES
#define FVV_CONV_RR_STAGES 4  // row-reuse stages when they fit (the 108 KB NT32/SW128 stage fits 2)
#endif
#ifndef FVV_CONV_RR_MAXN
#define FVV_CONV_RR_MAXN 64   // row-reuse tiles for 3x3 stride-1 convolutions with ntile <= this
#endif
template <int NT, int SW, int RR = 0>
struct ConvTile {
    static constexpr int MT = RR > 0 ? RR : (NT <= 128 ? 2 : 1);
    static constexpr int kARows = RR > 0 ? RR + 2 : MT;
    static constexpr int kBChunks = RR > 0 ? 3 : 1;
    static constexpr int kABytes = 128 * SW;                 // one 128-pixel row segment
    static constexpr int kBBytes = NT * SW;
    static constexpr int kStageBytes = kARows * kABytes + kBChunks * kBBytes;
    // as many stages as fit the 227 KB opt-in shared memory (1 KB alignment slack + barriers), at most 6
    static constexpr int kFit = (232448 - 1280) / kStageBytes;
    static constexpr int kStages = RR > 0 ? (kFit < FVV_CONV_RR_STAGES ? (kFit >= 1 ? kFit : 1) : FVV_CONV_RR_STAGES)
                                          : (kFit < 6 ? kFit : 6);
    static constexpr int kTmemCols = 2 * MT * NT < 32 ? 32 : 2 * MT * NT;  // two accumulator sets
    static constexpr size_t kSmem = 1024 /* alignment slack */ + (size_t)kStages * kStageBytes + 256;
};
constexpr int kConvThreads = 192;

struct TileCoord {
    int b, gy, gx0, n0;
};
__device__ __forceinline__ TileCoord tile_of(int t, const ConvTCParams& p, int ntx, int nn, int NT, int MT) {
    TileCoord c;
    const int tn = t % nn;
    t /= nn;
    const int tx = t % ntx;
    t /= ntx;
    const int nty = (p.Hg + MT - 1) / MT;
    c.gy = (t % nty) * MT;
    c.b = t / nty;
    c.gx0 = tx * 128;
    c.n0 = tn * NT;
    return c;
}

template <int NT, int SW, int RR = 0>
__global__ void __launch_bounds__(kConvThreads, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const float* __restrict__ bias, void* __restrict__ out, ConvTCParams p) {
    using T = ConvTile<NT, SW, RR>;
    static_assert(NT % 16 == 0 && NT >= 16 && NT <= 256, "UMMA N (M = 128)");
    constexpr int S = T::kStages;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * T::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;    // [2] accumulator ready
    uint64_t* tempty = tfull + 2;   // [2] accumulator drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntx = (p.Wg + 127) / 128, nn = (p.N + NT - 1) / NT;
    constexpr int MT = T::MT;
    const int ntiles = ntx * nn * ((p.Hg + MT - 1) / MT) * p.B;
    const int nk = (RR > 0 ? 3 : p.ntaps) * p.kc_per_tap;  // RR: K chunks = (dx, channel chunk)

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 4);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(T::kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---- TMA producer ----
            int kg = 0;  // global K-chunk counter (stage / phase continue across tiles)
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const TileCoord c = tile_of(t, p, ntx, nn, NT, MT);
                const int ix0 = c.gx0 * p.sx + p.bx0, iy0 = c.gy * p.sy + p.by0;
                for (int kc = 0; kc < nk; kc++, kg++) {
                    const int s = kg % S;
                    if (kg >= S) mbar_wait(&empty[s], ((kg / S) - 1) & 1);
                    const int tap = kc / p.kc_per_tap, c0 = (kc - tap * p.kc_per_tap) * (SW / 2);
                    uint8_t* sa = smem + s * T::kStageBytes;
                    mbar_expect_tx(&full[s], T::kStageBytes);
                    if constexpr (RR > 0) {
                        // tap = dx here: input rows iy0 .. iy0 + RR + 1, weights of taps (dy, dx)
#pragma unroll
                        for (int j = 0; j < T::kARows; j++)
                            tma_load_4d(sa + j * T::kABytes, &tmA, &full[s], c0, ix0 + p.tdx[tap], iy0 + j, c.b);
#pragma unroll
                        for (int dy = 0; dy < 3; dy++)
                            tma_load_2d(sa + T::kARows * T::kABytes + dy * T::kBBytes, &tmB, &full[s],
                                        (dy * 3 + tap) * p.cpad + c0, p.wrow0 + c.n0);
                    } else {
#pragma unroll
                        for (int r = 0; r < MT; r++)  // rows past Hg load real or zero rows; the epilogue skips them
                            tma_load_4d(sa + r * T::kABytes, &tmA, &full[s], c0, ix0 + p.tdx[tap],
                                        iy0 + r * p.sy + p.tdy[tap], c.b);
                        tma_load_2d(sa + MT * T::kABytes, &tmB, &full[s], tap * p.cpad + c0, p.wrow0 + c.n0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---- MMA issuer ----
            constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                                       ((uint32_t)(128 >> 4) << 24);
            int kg = 0, i = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x, i++) {
                const int acc = i & 1;
                if (i >= 2) mbar_wait(&tempty[acc], ((i >> 1) - 1) & 1);  // drained by the epilogue
                asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                const uint32_t td = tmem + acc * MT * NT;
                for (int kc = 0; kc < nk; kc++, kg++) {
                    const int s = kg % S;
                    mbar_wait(&full[s], (kg / S) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
                    const uint32_t sa = smem_u32(smem + s * T::kStageBytes), sb = sa + T::kARows * T::kABytes;
                    // descriptors of the stage's operands: base + (byte offset >> 4) in the start-address
                    // field (smem < 256 KB, so the 14-bit field never carries) -- one add per MMA
                    const uint64_t da0 = umma_desc<SW>(sa), db0 = umma_desc<SW>(sb);
                    if constexpr (RR > 0) {
#pragma unroll
                        for (int k = 0; k < SW / 32; k++)
#pragma unroll
                            for (int dy = 0; dy < 3; dy++) {
                                const uint64_t db = db0 + (uint64_t)((dy * T::kBBytes + 32 * k) >> 4);
#pragma unroll
                                for (int r = 0; r < MT; r++)
                                    umma_bf16(td + r * NT, da0 + (uint64_t)(((r + dy) * T::kABytes + 32 * k) >> 4),
                                              db, idesc, (kc > 0 || k > 0 || dy > 0) ? 1u : 0u);
                            }
                    } else {
#pragma unroll
                        for (int k = 0; k < SW / 32; k++) {
                            const uint64_t db = db0 + (uint64_t)((32 * k) >> 4);
#pragma unroll
                            for (int r = 0; r < MT; r++)
                                umma_bf16(td + r * NT, da0 + (uint64_t)((r * T::kABytes + 32 * k) >> 4), db, idesc,
                                          (kc > 0 || k > 0) ? 1u : 0u);
                        }
                    }
                    umma_commit(&empty[s]);  // frees the stage once these MMAs have read it
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else {
        // ---- epilogue warps 2..5: TMEM lanes 32 * (warp % 4) .. +31 ----
        const int q = warp & 3;
        const int row = q * 32 + lane;
        constexpr int CW = NT < 32 ? NT : 32;  // columns per tcgen05.ld
        int i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, i++) {
            const TileCoord c0t = tile_of(t, p, ntx, nn, NT, MT);
            const int acc = i & 1;
            mbar_wait(&tfull[acc], (i >> 1) & 1);
            __syncwarp();
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const int gx = c0t.gx0 + row;
#pragma unroll 1
            for (int ccm = 0; ccm < MT * NT; ccm += CW) {
                const int sub = ccm / NT, cc = ccm - sub * NT;
                TileCoord c = c0t;
                c.gy += sub;
                const bool valid = gx < p.Wg && c.gy < p.Hg;
                const int oy = c.gy * p.omy + p.oay, ox = gx * p.omx + p.oax;
                const size_t obase = (((size_t)c.b * p.Hout + oy) * p.Wout + ox) * p.ostride + p.ocoff;
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + acc * MT * NT + ccm;
                if (CW == 32) {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
                          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
                          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                        : "r"(taddr));
                } else {
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
                        "%14,%15}, [%16];\n"
                        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                          "=r"(r[14]), "=r"(r[15])
                        : "r"(taddr));
                }
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                if (valid) {
                    const int nb = c.n0 + cc;
                    float v[32];
#pragma unroll
                    for (int j = 0; j < CW; j++) {
                        float x = __uint_as_float(r[j]) + (nb + j < p.N ? bias[nb + j] : 0.0f);
                        if (p.act == 1) x = fmaxf(x, 0.0f);
                        v[j] = x;
                    }
                    if (p.shuffle_c && !p.out_f32 && (p.shuffle_c & 7) == 0 && (p.ostride & 7) == 0 &&
                        (p.ocoff & 7) == 0 && (nb % p.shuffle_c) == 0 && nb + CW <= p.N) {
                        // sub-pixel, bf16: 8 consecutive channels of one phase per 16-byte store
#pragma unroll
                        for (int j = 0; j < CW; j += 8) {
                            const int n = nb + j;
                            const int ph = n / p.shuffle_c, ch = n - ph * p.shuffle_c;
                            const size_t o = (((size_t)c.b * p.Hout + 2 * c.gy + (ph >> 1)) * p.Wout + 2 * gx +
                                              (ph & 1)) * p.ostride + p.ocoff + ch;
                            uint4 u;
                            __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
                            __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
                            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
                            __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
                            memcpy(&u.x, &h0, 4); memcpy(&u.y, &h1, 4); memcpy(&u.z, &h2, 4); memcpy(&u.w, &h3, 4);
                            *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + o) = u;
                        }
                    } else if (p.shuffle_c) {
                        // sub-pixel (transposed-conv) head: one 3x3 GEMM emits all 4 output phases
#pragma unroll
                        for (int j = 0; j < CW; j++) {
                            const int n = nb + j;
                            if (n < p.N) {
                                const int ph = n / p.shuffle_c, ch = n - ph * p.shuffle_c;
                                const size_t o = (((size_t)c.b * p.Hout + 2 * c.gy + (ph >> 1)) * p.Wout + 2 * gx +
                                                  (ph & 1)) * p.ostride + p.ocoff + ch;
                                if (p.out_f32) reinterpret_cast<float*>(out)[o] = v[j];
                                else reinterpret_cast<__nv_bfloat16*>(out)[o] = __float2bfloat16_rn(v[j]);
                            }
                        }
                    } else if (p.out_f32) {
                        float* o = reinterpret_cast<float*>(out) + obase;
#pragma unroll
                        for (int j = 0; j < CW; j++)
                            if (nb + j < p.N) o[nb + j] = v[j];
                    } else {
                        __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(out) + obase + nb;
                        if (nb + CW <= p.N && ((obase + nb) & 7) == 0) {
#pragma unroll
                            for (int j = 0; j < CW; j += 8) {
                                uint4 u;
                                __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
                                __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
                                __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
                                __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
                                memcpy(&u.x, &h0, 4); memcpy(&u.y, &h1, 4); memcpy(&u.z, &h2, 4); memcpy(&u.w, &h3, 4);
                                *reinterpret_cast<uint4*>(o + j) = u;
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < CW; j++)
                                if (nb + j < p.N) o[j] = __float2bfloat16_rn(v[j]);
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&tempty[acc]))
                                        : "memory");
        }
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(T::kTmemCols)
                     : "memory");
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

static int sm_count(int dev) {
    static std::atomic<int> cache[64];
    int n = cache[dev & 63].load(std::memory_order_relaxed);
    if (!n) {
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
        cache[dev & 63].store(n, std::memory_order_relaxed);
    }
    return n;
}

static bool getenv_flag_off(const char* name) {  // NAME=0 disables a fast path (A/B timing only)
    const char* v = getenv(name);
    return v && v[0] == '0';
}

static CUtensorMapSwizzle swz(int sw) {
    return sw == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// activation map: NHWC bf16 [B][H][W][C] as 4-D (C, W, H, B); box = chunk x 128 pixels (stride sx)
static bool make_act_map(CUtensorMap* m, const void* x, int B, int H, int W, int C, int sw, int sx) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    const cuuint32_t box[4] = {(cuuint32_t)(sw / 2), (cuuint32_t)(128 * sx), 1, 1};
    const cuuint32_t estr[4] = {1, (cuuint32_t)sx, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(x), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz(sw), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// weight map: bf16 [rows][K] K-major; box = chunk x NT rows
static bool make_w_map(CUtensorMap* m, const void* w, int rows, int K, int sw, int nt) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {(cuuint32_t)(sw / 2), (cuuint32_t)nt};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(w), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz(sw), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NT, int SW, int RR = 0>
static cudaError_t launch_nt_sw(const CUtensorMap& a, const CUtensorMap& w, const float* bias, void* out,
                                const ConvTCParams& p, int ntiles, cudaStream_t st) {
    using T = ConvTile<NT, SW, RR>;
    auto kern = k_conv_tc<NT, SW, RR>;
    // per-device state: the >48 KB shared-memory attribute is a property of the
    // function on each device, and SM counts may differ between devices
    static std::atomic<unsigned long long> attr_done{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (!(attr_done.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)T::kSmem);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();  // do not leave the error for the next launch check to find
            return e;
        }
        attr_done.fetch_or(bit, std::memory_order_release);
    }
    (void)ntiles;
    const int nsm = sm_count(dev);
    const int tiles = (p.Wg + 127) / 128 * ((p.Hg + T::MT - 1) / T::MT) * p.B * ((p.N + NT - 1) / NT);
    kern<<<tiles < nsm ? tiles : nsm, kConvThreads, T::kSmem, st>>>(a, w, bias, out, p);
    return cudaGetLastError();
}

template <int SW>
static cudaError_t launch_sw(int nt, const CUtensorMap& a, const CUtensorMap& w, const float* bias, void* out,
                             const ConvTCParams& p, int ntiles, cudaStream_t st) {
    switch (nt) {
        case 16: return launch_nt_sw<16, SW>(a, w, bias, out, p, ntiles, st);
        case 32: return launch_nt_sw<32, SW>(a, w, bias, out, p, ntiles, st);
        case 64: return launch_nt_sw<64, SW>(a, w, bias, out, p, ntiles, st);
        case 128: return launch_nt_sw<128, SW>(a, w, bias, out, p, ntiles, st);
        case 256: return launch_nt_sw<256, SW>(a, w, bias, out, p, ntiles, st);
        default: return cudaErrorInvalidValue;
    }
}

// One convolution (or one phase of a transposed convolution).  x: NHWC bf16
// [B][Hin][Win][cpad]; w: bf16 [rows][ntaps*cpad] (this conv's rows start at
// wrow0); out: NHWC (bf16 or f32) [B][Hout][Wout][ostride], channels
// [ocoff, ocoff + N).  ntile = UMMA N tile (16..256).
cudaError_t conv_tc(const void* x, int B, int Hin, int Win, int cpad, const void* w, int wrows, int wrow0,
                    int ntile, const float* bias, void* out, const ConvTCParams& p0, cudaStream_t st) {
    ConvTCParams p = p0;
    p.B = B;
    p.cpad = cpad;
    p.wrow0 = wrow0;
    const int sw = cpad >= 64 ? 128 : (cpad == 32 ? 64 : (cpad == 16 ? 32 : 0));
    if (!sw || (cpad > 64 && cpad % 64) || p.ntaps < 1 || p.ntaps > kConvMaxTaps) return cudaErrorInvalidValue;
    if (p.sx < 1 || p.sx > 2) return cudaErrorInvalidValue;
    p.kc_per_tap = cpad * 2 / sw;
    CUtensorMap ma, mw;
    if (!make_act_map(&ma, x, B, Hin, Win, cpad, sw, p.sx)) return cudaErrorInvalidValue;
    if (!make_w_map(&mw, w, wrows, p.ntaps * cpad, sw, ntile)) return cudaErrorInvalidValue;
    const int npad = ((p.N + ntile - 1) / ntile) * ntile;
    const int ntiles = npad / ntile;
    // small-N 3x3 stride-1 convolutions (the VINet head) are A-load bound: row-reuse tiles
    bool std3x3 = p.ntaps == 9 && p.sy == 1 && p.sx == 1 && p.omy == 1 && p.omx == 1;
    for (int t = 0; t < 9 && std3x3; t++) std3x3 = p.tdy[t] == t / 3 && p.tdx[t] == t % 3;
    if (std3x3 && ntile <= FVV_CONV_RR_MAXN && !getenv_flag_off("FVV_CONV_RR")) {
        // small-N 3x3 stride-1 layers (the VINet head, RefineNet's narrow full / half resolution
        // layers) are A-load bound: row-reuse tiles fetch each input row once per (dx, chunk)
        switch (ntile * 1000 + sw) {
            case 16032: return launch_nt_sw<16, 32, 4>(ma, mw, bias, out, p, ntiles, st);
            case 16064: return launch_nt_sw<16, 64, 4>(ma, mw, bias, out, p, ntiles, st);
            case 16128: return launch_nt_sw<16, 128, 4>(ma, mw, bias, out, p, ntiles, st);
            case 32032: return launch_nt_sw<32, 32, 4>(ma, mw, bias, out, p, ntiles, st);
            case 32064: return launch_nt_sw<32, 64, 4>(ma, mw, bias, out, p, ntiles, st);
            case 32128: return launch_nt_sw<32, 128, 4>(ma, mw, bias, out, p, ntiles, st);
            case 64064: return launch_nt_sw<64, 64, 4>(ma, mw, bias, out, p, ntiles, st);
            case 64128: return launch_nt_sw<64, 128, 4>(ma, mw, bias, out, p, ntiles, st);
            default: break;
        }
    }
    switch (sw) {
        case 128: return launch_sw<128>(ntile, ma, mw, bias, out, p, ntiles, st);
        case 64: return launch_sw<64>(ntile, ma, mw, bias, out, p, ntiles, st);
        default: return launch_sw<32>(ntile, ma, mw, bias, out, p, ntiles, st);
    }
}

}  // namespace fvv
