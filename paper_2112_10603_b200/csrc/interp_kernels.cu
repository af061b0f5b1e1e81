// interp_kernels.cu -- the per-stage kernels of interpolate() (interp.py:97-148)
// for a batch of camera/view pairs.  One launch of each kernel covers every
// pair of a recursion stage and both flow directions.
//
//   k_pyramid    luma + exact 2x2 / 4x4 pyramid sums      interp.py:67-71
//   k_sad<L>     exhaustive SAD block search + tie rule    flow.py:69-91, _kernels.py:28-49
//   k_flow<L>    flow = upscale(prev) + block_to_pixel     flow.py:47-54, 94-98, 129
//   k_warpq<L>   target warped by the base flow, *8, rint  flow.py:123-124, 77-78
//   k_mask_cols  final flows, mid warps, |wl-wr| column    interp.py:131-136, 78-94
//                sums, occlusion cue (exact, order-free)   warp.py:27-46
//   k_scan_carry scipy's running sum along rows (ordered)  imageops.py:51-52
//   k_blend      replay of 8-column chain segments, mask,  warp.py:49-88
//                blend of every plane
//
// Numerics: see DESIGN.md sec. 3 -- integer SAD, literal f64 bilinear
// arithmetic (no FMA), and the row-sequential replay of scipy's running sum
// where the reference's rounding is order dependent.
#include <algorithm>
#include <type_traits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <mutex>

#include "fvv_device.cuh"

// minimum resident CTAs per SM (register budgets), tuned on B200 -- see profiles/
#ifndef FVV_MINB_MASK
#define FVV_MINB_MASK 8
#endif
#ifndef FVV_MINB_SAD8
#define FVV_MINB_SAD8 4
#endif
#ifndef FVV_MINB_SADP
#define FVV_MINB_SADP 6
#endif

namespace fvv {

// ---------------------------------------------------------------------------
// k_pyramid: one thread per level-0 pixel (a 4x4 luma block).
// s4 = 4 x level-1 value, s16 = 16 x level-0 value: box_downsample of the
// integer luma is exact, so the f32 pyramid of interp.py:67-71 equals
// s4/4 and s16/16 exactly.
// ---------------------------------------------------------------------------
__global__ void k_pyramid(Geometry g, PairTable pt, uint8_t* __restrict__ ws, Planes P) {
    pdl_enter();
    const int w0 = g.lv[0].w, h0 = g.lv[0].h;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int pair = blockIdx.z >> 1, side = blockIdx.z & 1;
    if (x >= w0 || y >= h0) return;
    const uint8_t* fr = side ? pt.right[pair] : pt.left[pair];
    const int W = g.W;
    int v[4][4];
    if (g.fmt == FVV_RGB8) {
        uint8_t* luma = plane<uint8_t>(ws, P, P.luma[side], pair);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint8_t* row = fr + ((size_t)(4 * y + i) * W + 4 * x) * 3;
            uchar4 o;
            uint8_t t[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                t[j] = bt601(row[3 * j], row[3 * j + 1], row[3 * j + 2]);
                v[i][j] = t[j];
            }
            o.x = t[0]; o.y = t[1]; o.z = t[2]; o.w = t[3];
            *reinterpret_cast<uchar4*>(luma + (size_t)(4 * y + i) * W + 4 * x) = o;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; i++) {
            uchar4 q = *reinterpret_cast<const uchar4*>(fr + (size_t)(4 * y + i) * W + 4 * x);
            v[i][0] = q.x; v[i][1] = q.y; v[i][2] = q.z; v[i][3] = q.w;
        }
    }
    uint16_t* s4 = plane<uint16_t>(ws, P, P.s4[side], pair);
    const int w1 = g.lv[1].w;
    int s16 = 0;
#pragma unroll
    for (int a = 0; a < 2; a++) {
        int s0 = (v[2 * a][0] + v[2 * a][1]) + (v[2 * a + 1][0] + v[2 * a + 1][1]);
        int s1 = (v[2 * a][2] + v[2 * a][3]) + (v[2 * a + 1][2] + v[2 * a + 1][3]);
        *reinterpret_cast<ushort2*>(s4 + (size_t)(2 * y + a) * w1 + 2 * x) =
            make_ushort2((uint16_t)s0, (uint16_t)s1);
        s16 += s0 + s1;
    }
    plane<uint16_t>(ws, P, P.s16[side], pair)[(size_t)y * w0 + x] = (uint16_t)s16;
    // rint(8 * s16/16) = rint(s16/2), half to even (flow.py:77-78 at level 0)
    plane<uint16_t>(ws, P, P.q0[side], pair)[(size_t)y * w0 + x] =
        (uint16_t)(((uint32_t)s16 + (((uint32_t)s16 >> 1) & 1u)) >> 1);
}

// rint(8 * s16/16) = rint(s16/2), half to even (flow.py:77-78 at level 0)
__device__ __forceinline__ uint32_t q0_of(uint32_t s) { return (s + ((s >> 1) & 1u)) >> 1; }

// ---------------------------------------------------------------------------
// Level-specific sample access for the search.  d = direction: the reference
// block is on side d, the target on side 1-d (flow.py:119).
// ---------------------------------------------------------------------------
template <int LEVEL>
struct SadSrc {
    const uint16_t* q0_ref;   // level 0 (quantized, k_pyramid)
    const uint16_t* s16_ref;  // level 0
    const uint16_t* s16_tgt;
    const uint16_t* s4_ref;   // level 1
    const uint8_t* y_ref;     // level 2
    const uint16_t* tq;       // levels 1, 2: quantized warped target
    __device__ __forceinline__ uint32_t ref(int idx) const {
        if (LEVEL == 0) return q0_of(s16_ref[idx]);
        if (LEVEL == 1) return 2u * s4_ref[idx];
        return 8u * y_ref[idx];
    }
    // reference samples (idx, idx+1) packed as u16 pair (idx even, 4-byte aligned)
    __device__ __forceinline__ uint32_t ref_pair(int idx) const {
        if (LEVEL == 0) return *reinterpret_cast<const uint32_t*>(q0_ref + idx);
        if (LEVEL == 1) return *reinterpret_cast<const uint32_t*>(s4_ref + idx) << 1;  // 2*s <= 2040
        const uint32_t y2 = *reinterpret_cast<const uint16_t*>(y_ref + idx);
        return ((y2 & 0xFFu) | ((y2 & 0xFF00u) << 8)) << 3;                      // 8*Y pair
    }
    __device__ __forceinline__ uint32_t tgt(int idx) const {
        return tq[idx];
    }
};

template <int LEVEL>
__device__ __forceinline__ SadSrc<LEVEL> make_src(const Geometry& g, const PairTable& pt,
                                                  uint8_t* ws, const Planes& P, int pair, int d) {
    SadSrc<LEVEL> s;
    s.q0_ref = cplane<uint16_t>(ws, P, P.q0[d], pair);
    s.s16_ref = cplane<uint16_t>(ws, P, P.s16[d], pair);
    s.s16_tgt = cplane<uint16_t>(ws, P, P.s16[1 - d], pair);
    s.s4_ref = cplane<uint16_t>(ws, P, P.s4[d], pair);
    if (g.fmt == FVV_RGB8) s.y_ref = cplane<uint8_t>(ws, P, P.luma[d], pair);
    else s.y_ref = d ? pt.right[pair] : pt.left[pair];
    s.tq = LEVEL == 0 ? cplane<uint16_t>(ws, P, P.q0[1 - d], pair)
         : LEVEL == 1 ? cplane<uint16_t>(ws, P, P.tq1[d], pair)
                      : cplane<uint16_t>(ws, P, P.tq2[d], pair);
    return s;
}

struct SadLaunch {
    int nbx_cta;      // blocks per CTA (horizontal strip)
    int bx_begin;     // first block column covered by this launch
    int bx_end;       // one past the last block column
    int groups;       // dx groups per dy row (G)
    int pw;           // pair-plane pitch (u32) -- covers every thread's reads
    const int16_t* rank_of;      // stack index -> tie-rule rank  (flow.py:57-66)
    const int16_t* cand_of_rank; // tie-rule rank -> stack index
};

// ---------------------------------------------------------------------------
// k_sad: exhaustive SAD over the (2r+1)^2 candidates of every block of one
// block row strip, fused with the reference's tie rule.
//
// SAD = sum |a - b| = 2 * sum max(a, b) - sum a - sum b.  Samples are
// <= 2040 (8 * 255), so two candidates (dx, dx+1) share one 32-bit register
// as u16 lanes: max via VIMNMX.U16x2, sums accumulated lane-wise in plain
// 32-bit adds (no carry crosses lanes while a lane holds <= 32 samples) and
// flushed to 32-bit totals.  Exact integer arithmetic: order free.
// Winner = min over (sad, tie-rule rank) -> first minimum of
// np.argmin over the lexsorted candidate stack (flow.py:81-82).
// ---------------------------------------------------------------------------
template <int LEVEL, int KP, bool FULL8>
__global__ void __launch_bounds__(256) k_sad(Geometry g, PairTable pt, uint8_t* __restrict__ ws,
                                             Planes P, SadLaunch sl) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    const Level L = g.lv[LEVEL];
    const int B = L.block, r = L.r, side = 2 * r + 1;
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int by = blockIdx.y;
    const int bx0 = sl.bx_begin + blockIdx.x * sl.nbx_cta;
    const int nb = min(sl.nbx_cta, sl.bx_end - bx0);  // blocks in this CTA
    const int stripW = sl.nbx_cta * B;
    const int RW = stripW;                 // ref row pitch (u32)
    const int PW = sl.pw;                  // pair-plane pitch (u32)
    const int PH = B + 2 * r;
    uint32_t* Rs = reinterpret_cast<uint32_t*>(smem);                 // B x RW
    uint32_t* Ps = Rs + B * RW;                                        // PH x PW
    unsigned long long* best = reinterpret_cast<unsigned long long*>(
        smem + (((size_t)(B * RW + PH * PW) * 4 + 7) & ~(size_t)7));
    int* suma = reinterpret_cast<int*>(best + sl.nbx_cta);
    int16_t* rk = reinterpret_cast<int16_t*>(suma + sl.nbx_cta);      // side*side

    const SadSrc<LEVEL> src = make_src<LEVEL>(g, pt, ws, P, pair, d);
    const int w = L.w, h = L.h;
    const int ys = by * B;
    const int rows = min(B, h - ys);
    const int nthreads = blockDim.x;
    const int tid = threadIdx.x;

    // stage the reference strip (duplicated into both u16 lanes) and the
    // edge-padded target window (np.pad mode="edge", flow.py:78) as pairs
    for (int i = tid; i < B * RW; i += nthreads) {
        int yy = i / RW, xx = i % RW;
        int gx = bx0 * B + xx, gy = ys + yy;
        uint32_t q = 0;
        if (gy < h && gx < w && xx < nb * B) q = src.ref(gy * w + gx);
        Rs[i] = q | (q << 16);
    }
    for (int i = tid; i < PH * PW; i += nthreads) {
        int yy = i / PW, xx = i % PW;
        int gy = clampi(ys - r + yy, 0, h - 1);
        int gx0 = clampi(bx0 * B - r + xx, 0, w - 1);
        int gx1 = clampi(bx0 * B - r + xx + 1, 0, w - 1);
        Ps[i] = src.tgt(gy * w + gx0) | (src.tgt(gy * w + gx1) << 16);
    }
    for (int i = tid; i < side * side; i += nthreads) rk[i] = sl.rank_of[i];
    for (int i = tid; i < sl.nbx_cta; i += nthreads) best[i] = ~0ull;
    __syncthreads();
    // sum of reference samples per block (valid region only)
    for (int kb = tid; kb < nb; kb += nthreads) {
        int cols = min(B, w - (bx0 + kb) * B);
        int s = 0;
        for (int yy = 0; yy < rows; yy++)
            for (int xx = 0; xx < cols; xx++) s += (int)(Rs[yy * RW + kb * B + xx] & 0xFFFFu);
        suma[kb] = s;
    }

    const int per_block = side * sl.groups;
    const int kb = tid / per_block;
    const int rem = tid - kb * per_block;
    const int iy = rem / sl.groups;             // dy + r
    const int grp = rem - iy * sl.groups;
    const int dxo = grp * 2 * KP;               // dx + r of this thread's first candidate
    const bool active = kb < nb;

    int tot_lo[KP], tot_hi[KP];  // 2*sum(max) - sum(b), per candidate
#pragma unroll
    for (int k = 0; k < KP; k++) tot_lo[k] = tot_hi[k] = 0;

    if (active) {
        const int cols = min(B, w - (bx0 + kb) * B);
        const uint32_t* Rb = Rs + kb * B;
        const uint32_t* Pb = Ps + iy * PW + kb * B + dxo;
        if (FULL8) {
            // B == 8, full block: 4-row packed accumulation then flush
#pragma unroll 1
            for (int y0 = 0; y0 < 8; y0 += 4) {
                uint32_t am[KP], ab[KP];
#pragma unroll
                for (int k = 0; k < KP; k++) am[k] = ab[k] = 0;
#pragma unroll
                for (int yy = y0; yy < y0 + 4; yy++) {
                    if (yy < rows) {
                        uint32_t pv[2 * KP + 6];
#pragma unroll
                        for (int j = 0; j < 2 * KP + 6; j++) pv[j] = Pb[yy * PW + j];
#pragma unroll
                        for (int xx = 0; xx < 8; xx++) {
                            const uint32_t rv = Rb[yy * RW + xx];
#pragma unroll
                            for (int k = 0; k < KP; k++) {
                                const uint32_t p = pv[xx + 2 * k];
                                am[k] += __vmaxu2(p, rv);
                                ab[k] += p;
                            }
                        }
                    }
                }
#pragma unroll
                for (int k = 0; k < KP; k++) {
                    tot_lo[k] += 2 * (int)(am[k] & 0xFFFFu) - (int)(ab[k] & 0xFFFFu);
                    tot_hi[k] += 2 * (int)(am[k] >> 16) - (int)(ab[k] >> 16);
                }
            }
        } else {
            // general block size / ragged block: guarded, flush every row
            for (int yy = 0; yy < rows; yy++) {
                uint32_t am[KP], ab[KP];
#pragma unroll
                for (int k = 0; k < KP; k++) am[k] = ab[k] = 0;
                for (int xx = 0; xx < cols; xx++) {
                    const uint32_t rv = Rb[yy * RW + xx];
#pragma unroll
                    for (int k = 0; k < KP; k++) {
                        const uint32_t p = Pb[yy * PW + xx + 2 * k];
                        am[k] += __vmaxu2(p, rv);
                        ab[k] += p;
                    }
                }
#pragma unroll
                for (int k = 0; k < KP; k++) {
                    tot_lo[k] += 2 * (int)(am[k] & 0xFFFFu) - (int)(ab[k] & 0xFFFFu);
                    tot_hi[k] += 2 * (int)(am[k] >> 16) - (int)(ab[k] >> 16);
                }
            }
        }
    }
    __syncthreads();  // suma ready
    if (active) {
        const int sa = suma[kb];
        unsigned long long mine = ~0ull;
#pragma unroll
        for (int k = 0; k < KP; k++) {
            const int c0 = dxo + 2 * k;
            if (c0 < side) {
                unsigned long long key = ((unsigned long long)(uint32_t)(tot_lo[k] - sa) << 32) |
                                         (uint32_t)rk[iy * side + c0];
                mine = key < mine ? key : mine;
            }
            if (c0 + 1 < side) {
                unsigned long long key = ((unsigned long long)(uint32_t)(tot_hi[k] - sa) << 32) |
                                         (uint32_t)rk[iy * side + c0 + 1];
                mine = key < mine ? key : mine;
            }
        }
        atomicMin(&best[kb], mine);
    }
    __syncthreads();
    for (int k = tid; k < nb; k += nthreads) {
        const unsigned long long key = best[k];
        const int idx = sl.cand_of_rank[(int)(key & 0xFFFFFFFFu)];
        BlockHit hit;
        hit.dy = (int16_t)(idx / side - r);
        hit.dx = (int16_t)(idx % side - r);
        hit.sad = (int32_t)(key >> 32);
        plane<BlockHit>(ws, P, P.hit[LEVEL][d], pair)[by * L.nbx + bx0 + k] = hit;
    }
}

// warp_fixed with 32-bit coordinates (frames <= 8192 px, validated on the host)
template <typename Src>
__device__ __forceinline__ long long warp_fixed32(const Src& src, int h, int w, int y, int x,
                                                  int fxn, int fyn, int vb) {
    const ITap tx = clamp_itap32((x << vb) + fxn, vb, w);
    const ITap ty = clamp_itap32((y << vb) + fyn, vb, h);
    const int V = 1 << vb;
    (void)V;
    return (long long)bilerp_u(src(ty.i0, tx.i0), src(ty.i0, tx.i1), src(ty.i1, tx.i0), src(ty.i1, tx.i1),
                               tx.f, ty.f, vb);
}

__device__ __forceinline__ int2 lerp_i2(int2 a, int2 b, int den, int f) {
    return make_int2((den - f) * a.x + f * b.x, (den - f) * a.y + f * b.y);
}

// Builds the edge-padded pair plane P[yy][j] = T[y][xs-r+j] | T[y][xs-r+j+1] << 16
// of a search window.  Interior windows (no column clamping, even start)
// read two 32-bit words of the u16 target row per pair of P words and form
// the odd pair with one PRMT -- no u16 staging pass.  Edge windows take the
// clamped path through `Ts`.
template <int LEVEL>
__device__ __forceinline__ void stage_pairs(const SadSrc<LEVEL>& src, int w, int h, int r, int ys, int xs,
                                            int PH, int PW, uint32_t* Ps, uint16_t* Ts, int TW,
                                            int warp, int nwarps, int lane) {
    const int x0 = xs - r;
    const bool interior = x0 >= 0 && ((x0 & 1) == 0) && x0 + PW + 3 <= w;  // reads T[x0 .. x0+PW+2]
    if (interior) {
        for (int yy = warp; yy < PH; yy += nwarps) {
            const int gy = clampi(ys - r + yy, 0, h - 1);
            const uint32_t* row = reinterpret_cast<const uint32_t*>(src.tq + (size_t)gy * w + x0);
            for (int m = lane; 2 * m < PW; m += 32) {
                const uint32_t w0 = row[m], w1 = row[m + 1];
                Ps[yy * PW + 2 * m] = w0;
                if (2 * m + 1 < PW) Ps[yy * PW + 2 * m + 1] = __byte_perm(w0, w1, 0x5432);
            }
        }
        __syncthreads();
        return;
    }
    for (int yy = warp; yy < PH; yy += nwarps) {
        const int gy = clampi(ys - r + yy, 0, h - 1);
        for (int xx = lane; xx < TW; xx += 32)
            Ts[yy * TW + xx] = (uint16_t)src.tgt(gy * w + clampi(x0 + xx, 0, w - 1));
    }
    __syncthreads();
    for (int yy = warp; yy < PH; yy += nwarps)
        for (int j = lane; j < PW; j += 32)
            Ps[yy * PW + j] = j + 1 < TW ? (uint32_t)Ts[yy * TW + j] | ((uint32_t)Ts[yy * TW + j + 1] << 16) : 0u;
}

// ---------------------------------------------------------------------------
// k_sad8: the 8x8-block search (every BASELINE config) -- same arithmetic as
// k_sad, restructured for throughput: a CTA covers NBY x NBX blocks, the
// window is staged with 2-D warp-row loops (no index division), and every
// thread (one block, one dy, all 2r+1 dx) reads its reference row and its
// candidate pairs with 16-byte LDS (pair-plane pitch = 4 mod 8 words: eight
// consecutive dy rows hit eight distinct 16-byte bank groups).
// ---------------------------------------------------------------------------
struct Sad8Launch {
    int nbx, nby;                // blocks per CTA (x, y)
    int bx_begin, bx_end;        // block columns of this launch (full 8-wide columns)
    int pw;                      // pair-plane pitch (u32 words), = 4 mod 8
    int tw;                      // staged target window width (u16 samples)
    const int16_t* rank_of;
    const int16_t* cand_of_rank;
};

template <int LEVEL, int KP>
__global__ void __launch_bounds__(256, FVV_MINB_SAD8) k_sad8(Geometry g, PairTable pt, uint8_t* __restrict__ ws,
                                              Planes P, Sad8Launch sl) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    const Level L = g.lv[LEVEL];
    const int r = L.r, side = 2 * r + 1;
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int bx0 = sl.bx_begin + blockIdx.x * sl.nbx, by0 = blockIdx.y * sl.nby;
    const int nbx = min(sl.nbx, sl.bx_end - bx0), nby = min(sl.nby, L.nby - by0);
    const int RW = sl.nbx * 8, RH = sl.nby * 8;      // reference strip (u32 words, duplicated)
    const int PW = sl.pw, PH = RH + 2 * r;           // pair plane
    const int TW = sl.tw;                            // raw u16 target window width
    uint32_t* Rs = reinterpret_cast<uint32_t*>(smem);            // RH x RW
    uint32_t* Ps = Rs + RH * RW;                                  // PH x PW
    uint16_t* Ts = reinterpret_cast<uint16_t*>(Ps + PH * PW);     // PH x TW (staging)
    size_t off = ((size_t)(RH * RW + PH * PW) * 4 + (size_t)PH * TW * 2 + 15) & ~(size_t)15;
    unsigned long long* best = reinterpret_cast<unsigned long long*>(smem + off);
    int* suma = reinterpret_cast<int*>(best + sl.nbx * sl.nby);
    int16_t* rk = reinterpret_cast<int16_t*>(suma + sl.nbx * sl.nby);

    const SadSrc<LEVEL> src = make_src<LEVEL>(g, pt, ws, P, pair, d);
    const int w = L.w, h = L.h;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int ys = by0 * 8, xs = bx0 * 8;

    // reference strip (duplicated into both u16 lanes)
    for (int yy = warp; yy < RH; yy += nwarps) {
        const int gy = ys + yy;
        for (int xx = lane; xx < RW; xx += 32) {
            uint32_t q = 0;
            if (gy < h && xx < nbx * 8) q = src.ref(gy * w + xs + xx);
            Rs[yy * RW + xx] = q | (q << 16);
        }
    }
    for (int i = tid; i < side * side; i += blockDim.x) rk[i] = sl.rank_of[i];
    for (int i = tid; i < sl.nbx * sl.nby; i += blockDim.x) best[i] = ~0ull;
    // edge-padded target window (np.pad mode="edge", flow.py:78) as candidate pairs
    stage_pairs<LEVEL>(src, w, h, r, ys, xs, PH, PW, Ps, Ts, TW, warp, nwarps, lane);
    // sum of reference samples per block (valid rows only; columns are full here)
    for (int k = tid; k < sl.nbx * sl.nby; k += blockDim.x) {
        const int kbx = k % sl.nbx, kby = k / sl.nbx;
        const int rows = min(8, h - (by0 + kby) * 8);
        int sacc = 0;
        for (int yy = 0; yy < rows; yy++)
            for (int xx = 0; xx < 8; xx++) sacc += (int)(Rs[(kby * 8 + yy) * RW + kbx * 8 + xx] & 0xFFFFu);
        suma[k] = sacc;
    }
    __syncthreads();

    const int kb = tid / side, iy = tid - kb * side;   // block (in CTA), dy + r
    const int kbx = kb % sl.nbx, kby = kb / sl.nbx;
    const bool active = kb < sl.nbx * sl.nby && kbx < nbx && kby < nby;
    if (active) {
        const int rows = min(8, h - (by0 + kby) * 8);
        const uint32_t* Rb = Rs + (kby * 8) * RW + kbx * 8;
        const uint32_t* Pb = Ps + (kby * 8 + iy) * PW + kbx * 8;
        int tot_lo[KP], tot_hi[KP];
#pragma unroll
        for (int k = 0; k < KP; k++) tot_lo[k] = tot_hi[k] = 0;
#pragma unroll 1
        for (int y0 = 0; y0 < 8; y0 += 4) {
            uint32_t am[KP], ab[KP];
#pragma unroll
            for (int k = 0; k < KP; k++) am[k] = ab[k] = 0;
#pragma unroll
            for (int yy = y0; yy < y0 + 4; yy++) {
                if (yy < rows) {
                    constexpr int NP = (2 * KP + 6 + 3) / 4;  // 16-byte groups of candidate pairs
                    uint32_t pv[4 * NP];
#pragma unroll
                    for (int q = 0; q < NP; q++) {
                        const uint4 v = *reinterpret_cast<const uint4*>(Pb + yy * PW + 4 * q);
                        pv[4 * q] = v.x; pv[4 * q + 1] = v.y; pv[4 * q + 2] = v.z; pv[4 * q + 3] = v.w;
                    }
                    const uint4 ra = *reinterpret_cast<const uint4*>(Rb + yy * RW);
                    const uint4 rb = *reinterpret_cast<const uint4*>(Rb + yy * RW + 4);
                    const uint32_t rv[8] = {ra.x, ra.y, ra.z, ra.w, rb.x, rb.y, rb.z, rb.w};
#pragma unroll
                    for (int xx = 0; xx < 8; xx++) {
#pragma unroll
                        for (int k = 0; k < KP; k++) {
                            const uint32_t pp = pv[xx + 2 * k];
                            am[k] += __vmaxu2(pp, rv[xx]);
                            ab[k] += pp;
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < KP; k++) {
                tot_lo[k] += 2 * (int)(am[k] & 0xFFFFu) - (int)(ab[k] & 0xFFFFu);
                tot_hi[k] += 2 * (int)(am[k] >> 16) - (int)(ab[k] >> 16);
            }
        }
        const int sa = suma[kb];
        unsigned long long mine = ~0ull;
#pragma unroll
        for (int k = 0; k < KP; k++) {
            const int c0 = 2 * k;
            if (c0 < side) {
                const unsigned long long key = ((unsigned long long)(uint32_t)(tot_lo[k] - sa) << 32) |
                                               (uint32_t)rk[iy * side + c0];
                mine = key < mine ? key : mine;
            }
            if (c0 + 1 < side) {
                const unsigned long long key = ((unsigned long long)(uint32_t)(tot_hi[k] - sa) << 32) |
                                               (uint32_t)rk[iy * side + c0 + 1];
                mine = key < mine ? key : mine;
            }
        }
        atomicMin(&best[kb], mine);
    }
    __syncthreads();
    for (int k = tid; k < sl.nbx * sl.nby; k += blockDim.x) {
        const int kx = k % sl.nbx, ky = k / sl.nbx;
        if (kx >= nbx || ky >= nby) continue;
        const unsigned long long key = best[k];
        const int idx = sl.cand_of_rank[(int)(key & 0xFFFFFFFFu)];
        BlockHit hit;
        hit.dy = (int16_t)(idx / side - r);
        hit.dx = (int16_t)(idx % side - r);
        hit.sad = (int32_t)(key >> 32);
        plane<BlockHit>(ws, P, P.hit[LEVEL][d], pair)[(by0 + ky) * L.nbx + bx0 + kx] = hit;
    }
}

// ---------------------------------------------------------------------------
// k_sadp: 8x8-block search with PIXEL-pair packing.  One 32-bit register
// holds two horizontally adjacent samples: the reference pair (R[x], R[x+1])
// and, from the pair plane, the target pair (T[x+dx], T[x+dx+1]).  One
// VIMNMX.U16x2 then gives max() of one candidate at two pixels, so a row of
// 8 pixels costs 4 VIMNMX + 4 lane-wise adds per candidate, any (2r+1)
// candidates, no wasted slot.  A lane sums at most 32 samples per block
// (<= 32 * 2040 < 2^16): the accumulators never overflow, no flush needed.
// One thread = one block, one dy, all 2r+1 dx (SIDE = 2r+1, compile time).
// ---------------------------------------------------------------------------
struct SadPLaunch {
    int nbx, nby;         // blocks per CTA
    int bx_begin, bx_end; // full 8-wide block columns of this launch
    int pw;               // pair-plane pitch (words), = 4 mod 8
    int tw;               // raw target window width
    const int16_t* rank_of;
    const int16_t* cand_of_rank;
};

template <int LEVEL, int SIDE>
__global__ void __launch_bounds__(256, FVV_MINB_SADP) k_sadp(Geometry g, PairTable pt, uint8_t* __restrict__ ws,
                                              Planes P, SadPLaunch sl) {
    pdl_enter();
    extern __shared__ __align__(16) uint8_t smem[];
    const Level L = g.lv[LEVEL];
    constexpr int r = SIDE / 2;
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int bx0 = sl.bx_begin + blockIdx.x * sl.nbx, by0 = blockIdx.y * sl.nby;
    const int nbx = min(sl.nbx, sl.bx_end - bx0), nby = min(sl.nby, L.nby - by0);
    const int RW = sl.nbx * 4, RH = sl.nby * 8;      // reference pixel pairs (words)
    const int PW = sl.pw, PH = RH + 2 * r;
    const int TW = sl.tw;
    uint32_t* Rs = reinterpret_cast<uint32_t*>(smem);            // RH x RW
    uint32_t* Ps = Rs + RH * RW;                                  // PH x PW
    uint16_t* Ts = reinterpret_cast<uint16_t*>(Ps + PH * PW);     // PH x TW (staging)
    size_t off = ((size_t)(RH * RW + PH * PW) * 4 + (size_t)PH * TW * 2 + 15) & ~(size_t)15;
    unsigned long long* best = reinterpret_cast<unsigned long long*>(smem + off);
    int* suma = reinterpret_cast<int*>(best + sl.nbx * sl.nby);
    int16_t* rk = reinterpret_cast<int16_t*>(suma + sl.nbx * sl.nby);

    const SadSrc<LEVEL> src = make_src<LEVEL>(g, pt, ws, P, pair, d);
    const int w = L.w, h = L.h;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int ys = by0 * 8, xs = bx0 * 8;

    for (int yy = warp; yy < RH; yy += nwarps) {
        const int gy = ys + yy;
        for (int xx = lane; xx < RW; xx += 32)
            Rs[yy * RW + xx] = (gy < h && 2 * xx < nbx * 8) ? src.ref_pair(gy * w + xs + 2 * xx) : 0u;
    }
    for (int i = tid; i < SIDE * SIDE; i += blockDim.x) rk[i] = sl.rank_of[i];
    for (int i = tid; i < sl.nbx * sl.nby; i += blockDim.x) best[i] = ~0ull;
    stage_pairs<LEVEL>(src, w, h, r, ys, xs, PH, PW, Ps, Ts, TW, warp, nwarps, lane);
    for (int k = tid; k < sl.nbx * sl.nby; k += blockDim.x) {
        const int kbx = k % sl.nbx, kby = k / sl.nbx;
        const int rows = min(8, h - (by0 + kby) * 8);
        int sacc = 0;
        for (int yy = 0; yy < rows; yy++)
            for (int xx = 0; xx < 4; xx++) {
                const uint32_t v = Rs[(kby * 8 + yy) * RW + kbx * 4 + xx];
                sacc += (int)(v & 0xFFFFu) + (int)(v >> 16);
            }
        suma[k] = sacc;
    }
    __syncthreads();

    const int kb = tid / SIDE, iy = tid - kb * SIDE;   // block (in CTA), dy + r
    const int kbx = kb % sl.nbx, kby = kb / sl.nbx;
    const bool active = kb < sl.nbx * sl.nby && kbx < nbx && kby < nby;
    if (active) {
        const int rows = min(8, h - (by0 + kby) * 8);
        const uint32_t* Rb = Rs + (kby * 8) * RW + kbx * 4;
        const uint32_t* Pb = Ps + (kby * 8 + iy) * PW + kbx * 8;
        uint32_t am[SIDE], ab[SIDE];
#pragma unroll
        for (int c = 0; c < SIDE; c++) am[c] = ab[c] = 0;
        constexpr int NP = (SIDE + 6 + 3) / 4;  // 16-byte groups covering words 0..SIDE+5
#pragma unroll 2
        for (int yy = 0; yy < 8; yy++) {
            if (yy < rows) {
                uint32_t pv[4 * NP];
#pragma unroll
                for (int q = 0; q < NP; q++) {
                    const uint4 v = *reinterpret_cast<const uint4*>(Pb + yy * PW + 4 * q);
                    pv[4 * q] = v.x; pv[4 * q + 1] = v.y; pv[4 * q + 2] = v.z; pv[4 * q + 3] = v.w;
                }
                const uint4 rq = *reinterpret_cast<const uint4*>(Rb + yy * RW);
                const uint32_t rv[4] = {rq.x, rq.y, rq.z, rq.w};
#pragma unroll
                for (int k = 0; k < 4; k++)
#pragma unroll
                    for (int c = 0; c < SIDE; c++) {
                        const uint32_t pp = pv[2 * k + c];
                        am[c] += __vmaxu2(pp, rv[k]);
                        ab[c] += pp;
                    }
            }
        }
        const int sa = suma[kb];
        unsigned long long mine = ~0ull;
#pragma unroll
        for (int c = 0; c < SIDE; c++) {
            const int sad = 2 * ((int)(am[c] & 0xFFFFu) + (int)(am[c] >> 16)) -
                            ((int)(ab[c] & 0xFFFFu) + (int)(ab[c] >> 16)) - sa;
            const unsigned long long key = ((unsigned long long)(uint32_t)sad << 32) |
                                           (uint32_t)rk[iy * SIDE + c];
            mine = key < mine ? key : mine;
        }
        atomicMin(&best[kb], mine);
    }
    __syncthreads();
    for (int k = tid; k < sl.nbx * sl.nby; k += blockDim.x) {
        const int kx = k % sl.nbx, ky = k / sl.nbx;
        if (kx >= nbx || ky >= nby) continue;
        const unsigned long long key = best[k];
        const int idx = sl.cand_of_rank[(int)(key & 0xFFFFFFFFu)];
        BlockHit hit;
        hit.dy = (int16_t)(idx / SIDE - r);
        hit.dx = (int16_t)(idx % SIDE - r);
        hit.sad = (int32_t)(key >> 32);
        plane<BlockHit>(ws, P, P.hit[LEVEL][d], pair)[(by0 + ky) * L.nbx + bx0 + kx] = hit;
    }
}

// ---------------------------------------------------------------------------
// k_flow<L>: flow_L = base + f32(block_to_pixel(offsets))  (flow.py:122-129)
// base = 0 at level 0, f32(2 * upscale(flow_{L-1})) otherwise.  Exact fixed
// point (units 2^-fb[L]), equal to the reference's f32 values; both bilinear
// terms are evaluated separably per 16x64 tile (x-lerp rows, then y-lerp).
// ---------------------------------------------------------------------------
constexpr int kFH = 64, kFW = 64;
#ifndef FVV_FLOW_PAIR
#define FVV_FLOW_PAIR 1
#endif
template <int LEVEL>
__global__ void __launch_bounds__(256) k_flow(Geometry g, uint8_t* __restrict__ ws, Planes P) {
    pdl_enter();
    __shared__ __align__(16) int2 hu[kFH / 2 + 3][kFW];   // x-lerped rows of flow_{L-1}
    __shared__ __align__(16) int2 hb[kFH / 2 + 3][kFW];   // x-lerped block rows (B >= 2)
    __shared__ ITap cu[kFW], cb[kFW];
    __shared__ int4 rtab[kFH];  // per tile row: block-grid y tap (i0 - b_lo, i1 - b_lo, f), base-flow y tap (i0 - s_lo, i1 - s_lo) packed
    const Level L = g.lv[LEVEL];
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int x0 = blockIdx.x * kFW, y0 = blockIdx.y * kFH;
    const int tid = threadIdx.x, tx = tid & 63, tg = tid >> 6;
    const int B = L.block, D = 2 * B, lgD = 31 - __clz(D);
    const Level Lp = g.lv[LEVEL > 0 ? LEVEL - 1 : 0];
    const int xc = min(x0 + tx, L.w - 1);
    if (tid < kFW) {
        cb[tid] = clamp_itap32(2 * xc - B + 1, lgD, L.nbx);
        if (LEVEL > 0) cu[tid] = clamp_itap32(2 * xc - 1, 2, Lp.w);
    }
    const int ylast = min(y0 + kFH - 1, L.h - 1);
    const int b_lo = clamp_itap32(2 * y0 - B + 1, lgD, L.nby).i0;
    const int b_n = clamp_itap32(2 * ylast - B + 1, lgD, L.nby).i1 - b_lo + 1;
    const int s_lo = LEVEL > 0 ? clamp_itap32(2 * y0 - 1, 2, Lp.h).i0 : 0;
    const int s_n = LEVEL > 0 ? clamp_itap32(2 * ylast - 1, 2, Lp.h).i1 - s_lo + 1 : 0;
    if (tid < kFH) {  // the row taps, once per tile instead of once per pixel
        const int y = min(y0 + tid, L.h - 1);
        const ITap t = clamp_itap32(2 * y - B + 1, lgD, L.nby);
        int w = 0;
        if (LEVEL > 0) {
            const ITap u = clamp_itap32(2 * y - 1, 2, Lp.h);
            w = (u.i0 - s_lo) | ((u.i1 - s_lo) << 8) | (u.f << 16);  // indices < kFH / 2 + 3, f <= 4
        }
        rtab[tid] = make_int4(t.i0 - b_lo, t.i1 - b_lo, t.f, w);
    }
    __syncthreads();
    const BlockHit* hit = cplane<BlockHit>(ws, P, P.hit[LEVEL][d], pair);
    for (int row = tg; row < b_n; row += 4) {
        const BlockHit* hr = hit + (size_t)(b_lo + row) * L.nbx;
        const ITap t = cb[tx];
        const BlockHit p = hr[t.i0], q = hr[t.i1];
        hb[row][tx] = lerp_i2(make_int2(p.dx, p.dy), make_int2(q.dx, q.dy), D, t.f);
    }
    if (LEVEL > 0) {
        const int2* prev = cplane<int2>(ws, P, P.flow0[d], pair);
        for (int row = tg; row < s_n; row += 4) {
            const int2* pr = prev + (size_t)(s_lo + row) * Lp.w;
            const ITap t = cu[tx];
            hu[row][tx] = lerp_i2(pr[t.i0], pr[t.i1], 4, t.f);
        }
    }
    __syncthreads();
    const int rs = g.fb[LEVEL] - g.rb[LEVEL];
    const int bs = LEVEL > 0 ? g.fb[LEVEL] - (g.fb[LEVEL - 1] + 3) : 0;
    int2* out = plane<int2>(ws, P, LEVEL == 0 ? P.flow0[d] : P.flow1[d], pair);
#if FVV_FLOW_PAIR
    {
        // two adjacent columns per thread (8 rows apart per step): 16-byte reads of the
        // x-lerped rows, one 16-byte store when the row pitch keeps it aligned
        const int px = tid & 31, rg = tid >> 5;
        const int xq = x0 + 2 * px;
        if (xq >= L.w) return;
        const bool two = xq + 1 < L.w, vec = two && (L.w & 1) == 0;
        for (int ty = rg; ty < kFH; ty += 8) {
            const int y = y0 + ty;
            if (y >= L.h) break;
            const int4 rt = rtab[ty];
            const int4 ba = *reinterpret_cast<const int4*>(&hb[rt.x][2 * px]);
            const int4 bb = *reinterpret_cast<const int4*>(&hb[rt.y][2 * px]);
            const int2 r0 = lerp_i2(make_int2(ba.x, ba.y), make_int2(bb.x, bb.y), D, rt.z);
            const int2 r1 = lerp_i2(make_int2(ba.z, ba.w), make_int2(bb.z, bb.w), D, rt.z);
            int4 f = make_int4(r0.x << rs, r0.y << rs, r1.x << rs, r1.y << rs);
            if (LEVEL > 0) {
                const int4 ua = *reinterpret_cast<const int4*>(&hu[rt.w & 0xFF][2 * px]);
                const int4 ub = *reinterpret_cast<const int4*>(&hu[(rt.w >> 8) & 0xFF][2 * px]);
                const int2 u0 = lerp_i2(make_int2(ua.x, ua.y), make_int2(ub.x, ub.y), 4, rt.w >> 16);
                const int2 u1 = lerp_i2(make_int2(ua.z, ua.w), make_int2(ub.z, ub.w), 4, rt.w >> 16);
                f.x += u0.x << bs;
                f.y += u0.y << bs;
                f.z += u1.x << bs;
                f.w += u1.y << bs;
            }
            int2* o = out + (size_t)y * L.w + xq;
            if (vec) {
                *reinterpret_cast<int4*>(o) = f;
            } else {
                o[0] = make_int2(f.x, f.y);
                if (two) o[1] = make_int2(f.z, f.w);
            }
        }
        return;
    }
#endif
    const int x = x0 + tx;
    if (x >= L.w) return;
    for (int ty = tg; ty < kFH; ty += 4) {
        const int y = y0 + ty;
        if (y >= L.h) break;
        const int4 rt = rtab[ty];
        const int2 res = lerp_i2(hb[rt.x][tx], hb[rt.y][tx], D, rt.z);
        int2 f = make_int2(res.x << rs, res.y << rs);
        if (LEVEL > 0) {
            const int2 base = lerp_i2(hu[rt.w & 0xFF][tx], hu[(rt.w >> 8) & 0xFF][tx], 4, rt.w >> 16);
            f.x += base.x << bs;
            f.y += base.y << bs;
        }
        out[(size_t)y * L.w + x] = f;
    }
}

// ---------------------------------------------------------------------------
// k_warpq<L> (L = 1, 2): pad_q source = rint(8 * warp_plane(target, base))
// (flow.py:123-124 then :78); the edge padding is applied by the search.
// Exact integer bilinear: base = 2x upscale of flow_{L-1} (units
// 2^-(fb[L-1]+3)), computed separably per 16x64 tile; level-1 samples in
// units 1/4 (s4), level-2 samples integral (luma).
// ---------------------------------------------------------------------------
constexpr int kQH = 64, kQW = 64;  // 16 pixels per thread amortise the tile setup
#ifndef FVV_WARPQ_UNROLL
#define FVV_WARPQ_UNROLL 4  // interior loop unroll (16 rows per thread)
#endif
constexpr int kWarpqUnroll = FVV_WARPQ_UNROLL;
#ifndef FVV_WARPQ_PAIR
#define FVV_WARPQ_PAIR 1  // interior tiles: two adjacent columns per thread
#endif
#ifndef FVV_WARPQ_L1PF
#define FVV_WARPQ_L1PF 0  // > 0: L1 prefetch of the luma row this many iterations ahead (r2 sweep 1/2/4: no change), off
#endif
template <int LEVEL>
__global__ void __launch_bounds__(256) k_warpq(Geometry g, PairTable pt, uint8_t* __restrict__ ws,
                                               Planes P) {
    pdl_enter();
    __shared__ __align__(16) int2 h[kQH / 2 + 3][kQW];
    __shared__ ITap cxt[kQW];
    __shared__ int4 rt[kQH];  // per tile row: base-flow y tap (i0 - s_lo, i1 - s_lo, f)
    const Level& L = g.lv[LEVEL];
    const Level& Lp = g.lv[LEVEL - 1];
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int x0 = blockIdx.x * kQW, y0 = blockIdx.y * kQH;
    const int tid = threadIdx.x, tx = tid & 63, tg = tid >> 6;
    const int2* prev = cplane<int2>(ws, P, LEVEL == 1 ? P.flow0[d] : P.flow1[d], pair);
    const int ylast = min(y0 + kQH - 1, L.h - 1);
    const int s_lo = clamp_itap32(2 * y0 - 1, 2, Lp.h).i0;
    const int s_n = clamp_itap32(2 * ylast - 1, 2, Lp.h).i1 - s_lo + 1;
    if (tid < kQW) {
        cxt[tid] = clamp_itap32(2 * min(x0 + tid, L.w - 1) - 1, 2, Lp.w);
        const ITap t = clamp_itap32(2 * min(y0 + tid, L.h - 1) - 1, 2, Lp.h);
        rt[tid] = make_int4(t.i0 - s_lo, t.i1 - s_lo, t.f, 0);
    }
    __syncthreads();
    for (int row = tg; row < s_n; row += 4) {
        const int2* pr = prev + (size_t)(s_lo + row) * Lp.w;
        const ITap t = cxt[tx];
        h[row][tx] = lerp_i2(pr[t.i0], pr[t.i1], 4, t.f);
    }
    __syncthreads();
    const int vb = g.fb[LEVEL - 1] + 3;
    const int w = L.w;
    uint16_t* outp = plane<uint16_t>(ws, P, LEVEL == 1 ? P.tq1[d] : P.tq2[d], pair);
    const uint16_t* s4 = cplane<uint16_t>(ws, P, P.s4[1 - d], pair);
    const uint8_t* yp = g.fmt == FVV_RGB8 ? cplane<uint8_t>(ws, P, P.luma[1 - d], pair)
                                          : (d ? pt.left[pair] : pt.right[pair]);
    const int M = g.qmargin[LEVEL];
    const bool interior = x0 >= M && x0 + kQW - 1 + M <= w - 2 && y0 >= M && y0 + kQH - 1 + M <= L.h - 2;
#if FVV_WARPQ_PAIR
    if (interior) {
        // two adjacent columns per thread (x, x + 1; 8 rows apart per step): one 16-byte
        // read of the x-lerped base rows and one 32-bit store serve both pixels
        const int k = LEVEL == 1 ? 2 * vb - 1 : 2 * vb - 3;
        const int fmask = (1 << vb) - 1;
        const int px = tid & 31, rg = tid >> 5;
        const int xp = x0 + 2 * px;
        const int xs0 = xp << vb, xs1 = (xp + 1) << vb;
        uint32_t* op = reinterpret_cast<uint32_t*>(outp + (size_t)(y0 + rg) * w + xp);  // xp, w even
#pragma unroll kWarpqUnroll
        for (int ty = rg; ty < kQH; ty += 8) {
            const int y = y0 + ty;
            const int4 r = rt[ty];
            const int4 ha = *reinterpret_cast<const int4*>(&h[r.x][2 * px]);
            const int4 hb = *reinterpret_cast<const int4*>(&h[r.y][2 * px]);
            const int2 bc[2] = {lerp_i2(make_int2(ha.x, ha.y), make_int2(hb.x, hb.y), 4, r.z),
                                lerp_i2(make_int2(ha.z, ha.w), make_int2(hb.z, hb.w), 4, r.z)};
            uint32_t q[2];
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const int sx = (c ? xs1 : xs0) + bc[c].x, sy = (y << vb) + bc[c].y;
                const int fx = sx & fmask, fy = sy & fmask;
                const int off = (sy >> vb) * w + (sx >> vb);
                int a, b, cc, e;
                if (LEVEL == 1) {
                    const uint16_t* p0 = s4 + (unsigned)off;
                    a = p0[0]; b = p0[1]; cc = p0[w]; e = p0[w + 1];
                } else {
                    const uint8_t* p0 = yp + (unsigned)off;
                    a = p0[0]; b = p0[1]; cc = p0[w]; e = p0[w + 1];
                }
                q[c] = (uint32_t)rne64((long long)bilerp_u(a, b, cc, e, fx, fy, vb), k);
            }
            *op = q[0] | (q[1] << 16);
            op += 4 * (size_t)w;  // 8 rows of u16 pairs
        }
        return;
    }
#endif
    const int x = x0 + tx;
    if (x >= L.w) return;
    if (interior) {
        // every sample position (x, y) + base lies in [0, n-2] + [0, 1): no clamping,
        // taps are a shift and a mask (bit-identical to the clamped form here)
        const int k = LEVEL == 1 ? 2 * vb - 1 : 2 * vb - 3;
        const int fmask = (1 << vb) - 1;
        const int xs = x << vb;
        uint16_t* op = outp + (size_t)(y0 + tg) * w + x;
#pragma unroll kWarpqUnroll
        for (int ty = tg; ty < kQH; ty += 4) {
            const int y = y0 + ty;
            const int4 r = rt[ty];
            const int2 base = lerp_i2(h[r.x][tx], h[r.y][tx], 4, r.z);
            const int sx = xs + base.x, sy = (y << vb) + base.y;
            const int fx = sx & fmask, fy = sy & fmask;
            const int off = (sy >> vb) * w + (sx >> vb);
            int a, b, c, e;
            if (LEVEL == 1) {
                const uint16_t* p0 = s4 + (unsigned)off;
                a = p0[0]; b = p0[1]; c = p0[w]; e = p0[w + 1];
            } else {
                const uint8_t* p0 = yp + (unsigned)off;
#if FVV_WARPQ_L1PF
                // this thread's row FVV_WARPQ_L1PF iterations ahead (4 tile rows per iteration)
                if (ty + 4 * FVV_WARPQ_L1PF < kQH)
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p0 + 4 * FVV_WARPQ_L1PF * (size_t)w));
#endif
                a = p0[0]; b = p0[1]; c = p0[w]; e = p0[w + 1];
            }
            *op = (uint16_t)rne64((long long)bilerp_u(a, b, c, e, fx, fy, vb), k);
            op += 4 * (size_t)w;
        }
        return;
    }
    for (int ty = tg; ty < kQH; ty += 4) {
        const int y = y0 + ty;
        if (y >= L.h) break;
        const int4 r = rt[ty];
        const int2 base = lerp_i2(h[r.x][tx], h[r.y][tx], 4, r.z);
        int q;
        if (LEVEL == 1) {
            // value = v / (4 * 2^(2vb)); rint(8 * value) = rint(v / 2^(2vb - 1))
            q = rne64(bilin_fixed(s4, w, L.h, w, y, x, base.x, base.y, vb), 2 * vb - 1);
        } else {
            q = rne64(bilin_fixed(yp, w, L.h, w, y, x, base.x, base.y, vb), 2 * vb - 3);
        }
        outp[(size_t)y * w + x] = (uint16_t)q;
    }
}

// ---------------------------------------------------------------------------
// k_mask_cols: everything of _mask_inputs (interp.py:78-94) that does not
// depend on scipy's order of summation, plus the mid warps of every plane
// (warp.py:27-46).  Exactness: with power-of-two blocks
// every flow value is a dyadic rational with <= 24 significant bits, so
// np.gradient, the f32 occlusion cue and BOTH smoothing passes over it are
// exact sums -- scipy's running sum equals the plain 3-tap sum bitwise.
// |wl - wr| is integral, so its column pass is exact too; only its row pass
// (k_scan_carry / k_blend) must replay scipy in order.  Structure: a register-streaming
// column walker.  A warp owns kMW output columns (lanes 2..kMW+1; two halo
// lanes per side supply x-neighbours through shuffles) and walks down a
// kMH-row band, carrying lagged sliding windows:
//   F(y)      mid flows of both directions (separable: x-lerped source rows
//             are cached and re-used until the row tap moves)
//   gx(y)     x-gradient of f_m.x (shuffles), occ(y-1) = max(0, -(gx + gy))
//   O0(y-2)   column pass of smooth3 on occ (exact), O(y-2) row pass (shuffles)
//   d(y)      |wl - wr| of the luma warps at y, Sd(y-1) its column sum
//   chroma    at odd rows, from the 2x2 mid flows of the lane pair (x, x+1)
// Edge rows/columns follow the reference: one-sided np.gradient, nearest
// padding for smooth3.  No shared memory, no index division.
// ---------------------------------------------------------------------------
#ifndef FVV_KMH
// walker band height (Geometry::mh, chosen per launch): r2 v10 sweep (cfg4, 6 rig frames in
// flight; views/s and the one-frame k_mask_cols2 ms) 32: 11392 / 3.62, 48: 11592 / 3.50,
// 64: 11697 / 3.49, 96: 11782 / 3.49, 128: 11833 / 3.65.  96-row bands cut the halo rows but
// also the CTAs: small launches (cfg1, cfg2's 1-4 pair stages) lose latency with them
// (cfg1 0.15 -> 0.19 ms, cfg2 0.95 -> 1.08 ms), so launches of fewer than kMaskBigCtas
// 96-row CTAs keep 64-row bands.
#define FVV_KMH 64
#endif
#ifndef FVV_KMH_BIG
#define FVV_KMH_BIG 96
#endif
#ifndef FVV_MASK_BIG_CTAS
#define FVV_MASK_BIG_CTAS 1480  // two waves of 5 CTAs per SM on 148 SMs
#endif
#ifndef FVV_MASK_UNROLL
#define FVV_MASK_UNROLL 1
#endif
#ifndef FVV_MASK_NC
#define FVV_MASK_NC 0  // no-clamp interior rows: r2 sweep 4.02 -> 4.92 ms (register pressure), off
#endif
constexpr int kMW = 28, kMWarps = 4, kMH = FVV_KMH, kMaskUnroll = FVV_MASK_UNROLL;

template <int FMT>
__global__ void __launch_bounds__(kMWarps * 32, FVV_MINB_MASK) k_mask_cols(Geometry g, PairTable pt,
                                                               uint8_t* __restrict__ ws, Planes P) {
    pdl_enter();
    const int W = g.W, H = g.H;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.z;
    const int y0 = blockIdx.y * g.mh;
    const int xw0 = (blockIdx.x * kMWarps + wid) * kMW;
    if (xw0 >= W) return;  // whole warp outside the frame (no block-level sync in this kernel)
    const int x = xw0 - 2 + lane;
    const int xc = clampi(x, 0, W - 1);
    const bool own = lane >= 2 && lane < 2 + kMW && x < W;
    const Level& L1 = g.lv[1];
    const Level& L2 = g.lv[2];
    const int B2 = L2.block, D2 = 2 * B2, lgD2 = 31 - __clz(D2);
    const int mb = g.fb[2] + 1, kY = 2 * mb;
    const int bs = g.fb[2] - (g.fb[1] + 3), rs = g.fb[2] - g.rb[2];
    const ITap tu = clamp_itap32(2 * xc - 1, 2, L1.w);
    const ITap tb = clamp_itap32(2 * xc - B2 + 1, lgD2, L2.nbx);
    // x-neighbour lanes with the reference's edge rules folded in: np.gradient is
    // one-sided at x = 0 / W-1 (neighbour = self, difference doubled in our
    // units), smooth3's nearest padding repeats the edge value (neighbour = self)
    const int srcL = x <= 0 ? lane : lane - 1, srcR = x >= W - 1 ? lane : lane + 1;
    const int gmul = (W >= 2 && (x == 0 || x == W - 1)) ? 2 : (W >= 2 ? 1 : 0);
    const int2* f1[2] = {cplane<int2>(ws, P, P.flow1[0], pair), cplane<int2>(ws, P, P.flow1[1], pair)};
    const BlockHit* hh[2] = {cplane<BlockHit>(ws, P, P.hit[2][0], pair),
                             cplane<BlockHit>(ws, P, P.hit[2][1], pair)};
    const uint8_t* frL = pt.left[pair];
    const uint8_t* frR = pt.right[pair];
    uint8_t* o_wl = plane<uint8_t>(ws, P, P.wl, pair);
    uint8_t* o_wr = plane<uint8_t>(ws, P, P.wr, pair);
    uint16_t* o_sd = plane<uint16_t>(ws, P, P.sd, pair);
    float* o_ol = plane<float>(ws, P, P.occ_l, pair);
    float* o_or = plane<float>(ws, P, P.occ_r, pair);
    const float oscale = 1.0f / (float)(1 << (mb + 1));
    const int ys = max(0, y0 - 2), ye = min(H - 1, y0 + g.mh + 1);
    const int yo1 = min(H, y0 + g.mh);  // output rows [y0, yo1)

    auto xl_u = [&](int d, int row) {
        const int2* r = f1[d] + row * L1.w;
        return lerp_i2(r[tu.i0], r[tu.i1], 4, tu.f);
    };
    auto xl_b = [&](int d, int row) {
        const BlockHit* r = hh[d] + row * L2.nbx;
        const BlockHit p = r[tb.i0], q = r[tb.i1];
        return lerp_i2(make_int2(p.dx, p.dy), make_int2(q.dx, q.dy), D2, tb.f);
    };
    // exact f32(f64(a + b + c) / 3) of three f32 smooth3 column outputs
    auto rowpass = [&](float o0v) {
        const float a = __shfl_sync(0xffffffffu, o0v, srcL), c = __shfl_sync(0xffffffffu, o0v, srcR);
        if (a == 0.0f && o0v == 0.0f && c == 0.0f) return 0.0f;
        return (float)div3(__dadd_rn(__dadd_rn((double)a, (double)o0v), (double)c));
    };
    const double c3k = 0x1.5555555555555p-2 * (double)oscale;  // RN(1/3) * 2^-(mb+1), exact
    auto colpass = [&](int a, int b, int c) {  // f32(f64(sum/3)) of occ in units 2^-(mb+1)
        const int sn = a + b + c;  // >= 0, < 2^31: (double)sn built exactly off the XU pipe
        return sn ? third_scaled_f32((uint32_t)sn, c3k) : 0.0f;
    };

    // source-row caches: x-lerped rows ua, ua+1 of flow1 and ba, ba+1 of the block grid
    int ua = -10, ba = -10;
    int2 hu0[2], hu1[2], hb0[2], hb1[2];
    int2 F0[2], F1[2], F2[2];
    int gx1[2] = {0, 0}, gx2[2] = {0, 0};
    int oc0[2] = {0, 0}, oc1[2] = {0, 0}, oc2[2] = {0, 0};
    int d0 = 0, d1 = 0, d2 = 0;
#pragma unroll
    for (int d = 0; d < 2; d++) F0[d] = F1[d] = F2[d] = make_int2(0, 0);

    auto emit_o = [&](int t, int a0, int a1, int b0, int b1, int c0, int c1) {
        // O0(t) from occ(t-1), occ(t), occ(t+1) per direction, then the row pass.
        // Smooth flow has no convergence: when the occlusion cue of the warp's
        // 3 rows is zero in every lane, both passes are exactly zero (warp-uniform skip)
        float ol = 0.0f, orr = 0.0f;
        if (__any_sync(0xffffffffu, (a0 | a1 | b0 | b1 | c0 | c1) != 0)) {
            ol = rowpass(colpass(a0, b0, c0));
            orr = rowpass(colpass(a1, b1, c1));
        }
        if (own) {
            o_ol[(unsigned)(t * W + x)] = ol;
            o_or[(unsigned)(t * W + x)] = orr;
        }
    };

    // one walker row; GEN = general row (band edges, image top), else every
    // output of the row is in range and no edge rule applies (the band interior)
    auto step = [&](int yy, auto gen, auto nclamp) {
        constexpr bool GEN = decltype(gen)::value;
        // NC: every bilinear tap of this row (luma and chroma, both directions,
        // every lane) provably stays inside its plane (|mid flow| <= max_span / 2,
        // Geometry::mmargin), so the clamps of tap2 are identities and are skipped
        constexpr bool NC = decltype(nclamp)::value;
        // ---- mid flows F(yy) (flow.py:122-129 at level 2, interp.py:131-132) ----
        const Tap2 ty = tap2(2 * yy - 1, 2, L1.h);  // L1.h >= 2
        if (ty.i0 != ua) {
#pragma unroll
            for (int d = 0; d < 2; d++) {
                hu0[d] = ty.i0 == ua + 1 ? hu1[d] : xl_u(d, ty.i0);
                hu1[d] = xl_u(d, ty.i0 + 1);
            }
            ua = ty.i0;
        }
        const ITap tby = clamp_itap32(2 * yy - B2 + 1, lgD2, L2.nby);
        if (tby.i0 != ba) {
#pragma unroll
            for (int d = 0; d < 2; d++) {
                hb0[d] = tby.i0 == ba + 1 ? hb1[d] : xl_b(d, tby.i0);
                hb1[d] = xl_b(d, tby.i1);
            }
            ba = tby.i0;
        }
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const int2 base = lerp_i2(hu0[d], hu1[d], 4, ty.f);
            const int2 res = lerp_i2(hb0[d], hb1[d], D2, tby.f);
            F0[d] = F1[d];
            F1[d] = F2[d];
            F2[d] = make_int2(-((base.x << bs) + (res.x << rs)), -((base.y << bs) + (res.y << rs)));
            // x-gradient at yy (np.gradient edge order 1), units 2^-(mb+1)
            const int xl = __shfl_sync(0xffffffffu, F2[d].x, srcL);
            const int xr = __shfl_sync(0xffffffffu, F2[d].x, srcR);
            gx1[d] = gx2[d];
            gx2[d] = gmul * (xr - xl);
        }
        // ---- luma warps at yy (warp.py:37), d = |wl - wr| ----
        int wl, wr;
        if (FMT == FVV_RGB8) {
            uint8_t cl[3], cr[3];
#pragma unroll
            for (int c = 0; c < 3; c++) {
                auto sl = [&](int a, int b) { return (int)frL[((size_t)a * W + b) * 3 + c]; };
                auto sr = [&](int a, int b) { return (int)frR[((size_t)a * W + b) * 3 + c]; };
                cl[c] = (uint8_t)rne64(warp_fixed32(sl, H, W, yy, xc, F2[0].x, F2[0].y, mb), kY);
                cr[c] = (uint8_t)rne64(warp_fixed32(sr, H, W, yy, xc, F2[1].x, F2[1].y, mb), kY);
            }
            wl = bt601(cl[0], cl[1], cl[2]);
            wr = bt601(cr[0], cr[1], cr[2]);
            if (own && (!GEN || (yy >= y0 && yy < yo1))) {
                uint8_t* o = plane<uint8_t>(ws, P, P.wrgb, pair) + ((size_t)yy * W + x) * 6;
#pragma unroll
                for (int c = 0; c < 3; c++) { o[c] = cl[c]; o[3 + c] = cr[c]; }
            }
        } else if (NC) {
            const int fm = (1 << mb) - 1;
            auto nc = [&](const uint8_t* fr, int2 f) {
                const int sx = (xc << mb) + f.x, sy = (yy << mb) + f.y;
                const uint8_t* r0 = fr + (unsigned)((sy >> mb) * W + (sx >> mb));
                return rne64((long long)bilerp_u(r0[0], r0[1], r0[W], r0[W + 1], sx & fm, sy & fm, mb), kY);
            };
            wl = nc(frL, F2[0]);
            wr = nc(frR, F2[1]);
        } else {
            wl = rne64(bilin_fixed(frL, W, H, W, yy, xc, F2[0].x, F2[0].y, mb), kY);
            wr = rne64(bilin_fixed(frR, W, H, W, yy, xc, F2[1].x, F2[1].y, mb), kY);
        }
        d0 = d1;
        d1 = d2;
        d2 = abs(wl - wr);
        if (own && (!GEN || (yy >= y0 && yy < yo1))) {
            o_wl[(unsigned)(yy * W + x)] = (uint8_t)wl;
            o_wr[(unsigned)(yy * W + x)] = (uint8_t)wr;
        }
        // ---- Sd(yy-1): column sum of d with nearest padding ----
        {
            const int t = yy - 1;
            if (own && (!GEN || (t >= y0 && t < yo1))) o_sd[(unsigned)(t * W + x)] = (uint16_t)(((GEN && t == 0) ? d1 : d0) + d1 + d2);
        }
        // ---- occ(yy-1) then O0/O(yy-2) ----
        {
            const int r = yy - 1;
            if (!GEN || (r >= ys && (r == 0 || r - 1 >= ys))) {
#pragma unroll
                for (int d = 0; d < 2; d++) {
                    const int gy = H < 2 ? 0 : ((GEN && r == 0) ? 2 * (F2[d].y - F1[d].y) : F2[d].y - F0[d].y);
                    const int v = -(gx1[d] + gy);
                    oc0[d] = oc1[d];
                    oc1[d] = oc2[d];
                    oc2[d] = v > 0 ? v : 0;
                }
                const int t2 = yy - 2;  // occ(t2 - 1) = oc0 (or occ(0) at the top), occ(t2) = oc1, occ(t2 + 1) = oc2
                if (!GEN || (t2 >= y0 && t2 < yo1)) {
                    if (GEN && t2 == 0) emit_o(t2, oc1[0], oc1[1], oc1[0], oc1[1], oc2[0], oc2[1]);
                    else emit_o(t2, oc0[0], oc0[1], oc1[0], oc1[1], oc2[0], oc2[1]);
                }
            }
        }
        // ---- chroma warps for chroma row (yy-1)/2 at odd yy (imageops.py:40-48) ----
        if (FMT == FVV_YUV420 && (yy & 1) && (!GEN || (yy - 1 >= y0 && yy - 1 < yo1 && yy - 1 >= ys))) {
            const int cw = g.cw, chh = g.ch, cb = mb + 3, kC = 2 * cb;
            int2 cv[2];
#pragma unroll
            for (int d = 0; d < 2; d++) {
                const int sx = F1[d].x + F2[d].x, sy = F1[d].y + F2[d].y;
                cv[d] = make_int2(sx + __shfl_xor_sync(0xffffffffu, sx, 1),
                                  sy + __shfl_xor_sync(0xffffffffu, sy, 1));
            }
            if (own) {
                const int cy = (yy - 1) >> 1, cx = x >> 1;
                const int p = x & 1;  // even lane: U plane, odd lane: V plane
                const uint8_t* pl = frL + (size_t)W * H + (size_t)p * cw * chh;
                const uint8_t* pr = frR + (size_t)W * H + (size_t)p * cw * chh;
                uint8_t vl, vr;
                if (NC) {
                    const int fm = (1 << cb) - 1;
                    auto nc = [&](const uint8_t* pp, int2 f) {
                        const int sx = (cx << cb) + f.x, sy = (cy << cb) + f.y;
                        const uint8_t* r0 = pp + (unsigned)((sy >> cb) * cw + (sx >> cb));
                        return (uint8_t)rne64((long long)bilerp_u(r0[0], r0[1], r0[cw], r0[cw + 1], sx & fm, sy & fm, cb),
                                              kC);
                    };
                    vl = nc(pl, cv[0]);
                    vr = nc(pr, cv[1]);
                } else {
                    vl = (uint8_t)rne64(bilin_fixed(pl, cw, chh, cw, cy, cx, cv[0].x, cv[0].y, cb), kC);
                    vr = (uint8_t)rne64(bilin_fixed(pr, cw, chh, cw, cy, cx, cv[1].x, cv[1].y, cb), kC);
                }
                uint8_t* wc = reinterpret_cast<uint8_t*>(plane<uchar4>(ws, P, P.wc, pair) + (unsigned)(cy * cw + cx));
                wc[2 * p] = vl;
                wc[2 * p + 1] = vr;
            }
        }
    };
    const int b0 = min(max(y0 + 2, 3), yo1), b1 = max(b0, yo1);  // interior rows [b0, b1)
    // rows whose taps (luma row yy, chroma row (yy-1)/2) stay inside their planes,
    // and whether this warp's columns (all 32 lanes' luma taps, the owned lanes'
    // chroma taps) do: the no-clamp walker runs on their intersection
    const int mm = g.mmargin, cm = g.cmargin;
    const bool cols_in = FMT != FVV_RGB8 && xw0 - 2 >= mm && xw0 + 29 <= W - 2 - mm &&
                         (FMT != FVV_YUV420 || ((xw0 >> 1) >= cm && ((xw0 + kMW - 1) >> 1) <= g.cw - 2 - cm));
    const int r_lo = FMT == FVV_YUV420 ? max(mm, 2 * cm + 1) : mm;
    const int r_hi = FMT == FVV_YUV420 ? min(H - 2 - mm, 2 * (g.ch - 2 - cm) + 1) : H - 2 - mm;  // inclusive
    int yy = ys;
    for (; yy < b0; yy++) step(yy, std::true_type{}, std::false_type{});
    if (FVV_MASK_NC && cols_in && r_lo <= r_hi) {
        const int n0 = min(b1, max(yy, r_lo)), n1 = min(b1, max(n0, r_hi + 1));
        for (; yy < n0; yy++) step(yy, std::false_type{}, std::false_type{});
#pragma unroll kMaskUnroll
        for (; yy < n1; yy++) step(yy, std::false_type{}, std::true_type{});
    }
    for (; yy < b1; yy++) step(yy, std::false_type{}, std::false_type{});
    for (; yy <= ye; yy++) step(yy, std::true_type{}, std::false_type{});
    // ---- bottom edge: occ(H-1) (one-sided gy), O0/O(H-2), O0/O(H-1), Sd(H-1) ----
    if (ye == H - 1) {
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const int gy = H < 2 ? 0 : 2 * (F2[d].y - F1[d].y);
            const int v = -(gx2[d] + gy);
            oc0[d] = oc1[d];
            oc1[d] = oc2[d];
            oc2[d] = v > 0 ? v : 0;
        }
        if (H - 2 >= y0 && H - 2 < yo1) emit_o(H - 2, oc0[0], oc0[1], oc1[0], oc1[1], oc2[0], oc2[1]);
        if (H - 1 >= y0 && H - 1 < yo1) emit_o(H - 1, oc1[0], oc1[1], oc2[0], oc2[1], oc2[0], oc2[1]);
        if (own && H - 1 >= y0 && H - 1 < yo1) o_sd[(size_t)(H - 1) * W + x] = (uint16_t)(d1 + d2 + d2);
    }
}

// ---------------------------------------------------------------------------
// k_mask_cols2: the same computation as k_mask_cols (gray / 4:2:0), with each
// lane walking TWO adjacent columns x = 2m, 2m+1.  A warp covers 64 columns
// and owns 60 (one halo column pair per side instead of two halo lanes: 6 %
// of the lanes' work is halo instead of 12.5 %); per-row uniform work, the
// x-neighbour shuffles (one up + one down per direction serve both columns),
// the stores (u8x2 / u16x2 / f32x2) and the chroma pixel (x/2: the lane's own
// 2x2 block, no pair shuffle) are shared by the two columns.  Both columns'
// windows live in registers (twice the state of k_mask_cols at half the warps).
// Column semantics are identical to k_mask_cols: clamped sample column xc,
// nearest / one-sided neighbours at the frame edges.
// ---------------------------------------------------------------------------
#ifndef FVV_MINB_MASK2
#define FVV_MINB_MASK2 5  // r2 sweep: 4 (128 regs, no spills) 4.03 ms, 5 (96 regs) 3.85 ms per cfg4 step; r2 v10 (6 frames in flight): 4 = +0.9 % views/s but +0.19 ms one-frame latency, 6 = -1.4 %
#endif
#ifndef FVV_MASK2_HB_CACHE
#define FVV_MASK2_HB_CACHE 1
#endif
#ifndef FVV_MASK2_L1PF
#define FVV_MASK2_L1PF 4  // prefetch.global.L1 of the luma rows 4 rows ahead: r2 sweep 3.83 -> 3.70 ms (2: 3.70, 8: 3.71)
#endif
#ifndef FVV_MASK2_L1PF_C
#define FVV_MASK2_L1PF_C 0  // also the chroma rows
#endif
#ifndef FVV_MASK2_L2PF
#define FVV_MASK2_L2PF 0  // > 0: prefetch.global.L2 of the luma rows this many rows ahead
#endif
#ifndef FVV_MASK2_FPF
#define FVV_MASK2_FPF 1  // > 0: L1 prefetch of the level-1 flow row this many rows past the next reload: r2 sweep 0 / 1 / 2 / 3 = 3.58 / 3.49 / 3.50 / 3.50 ms
#endif
#ifndef FVV_MASK2_HPF
#define FVV_MASK2_HPF 0  // L1 prefetch of the next block-hit row: r2 sweep 3.49 -> 3.55 ms, off
#endif
#ifndef FVV_MASK2_UNROLL
#define FVV_MASK2_UNROLL 1  // interior-row loop unroll: r2 sweep 1 / 2 / 3 = 3.59 / 4.00 / 4.55 ms, keep 1
#endif
#ifndef FVV_MASK2_PF
#define FVV_MASK2_PF 0  // luma taps loaded one row ahead: r2 sweep 3.79 -> 3.94 ms (128 regs, spills), off
#endif
#ifndef FVV_MASK2_RTAB
#define FVV_MASK2_RTAB 0  // walker rows' y taps from a per-CTA shared table: r2 sweep 3.49 -> 3.55 ms (more spills), off
#endif
#if FVV_MASK2_RTAB && FVV_MASK2_PF
#error "FVV_MASK2_RTAB is for the default (no tap prefetch) walker"
#endif
#ifndef FVV_MASK2_DLERP
#define FVV_MASK2_DLERP 0  // row lerps from (scaled base, difference) pairs, one IMAD per component: timed-path parity green, but more spills at 96 registers (r2 v8: 3.51 -> 3.66 ms), off
#endif
#if FVV_MASK2_DLERP && (FVV_MASK2_PF || !FVV_MASK2_HB_CACHE)
#error "FVV_MASK2_DLERP needs the block-grid row cache and no tap prefetch"
#endif
#if FVV_MASK2_PF && !FVV_MASK2_HB_CACHE
#error "FVV_MASK2_PF needs the block-grid row cache"
#endif
constexpr int kM2Own = 60, kM2Warps = 4, kMask2Unroll = FVV_MASK2_UNROLL;

template <int FMT>
__global__ void __launch_bounds__(kM2Warps * 32, FVV_MINB_MASK2) k_mask_cols2(Geometry g, PairTable pt,
                                                                  uint8_t* __restrict__ ws, Planes P) {
    pdl_enter();
    static_assert(FMT != FVV_RGB8, "RGB8 runs k_mask_cols");
    const int W = g.W, H = g.H;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int pair = blockIdx.z;
    const int y0 = blockIdx.y * g.mh;
    const int xw0 = (blockIdx.x * kM2Warps + wid) * kM2Own;  // even
#if FVV_MASK2_RTAB
    // the walker rows' y taps (level-1 flow rows, level-2 block rows), once per CTA:
    // rows ys .. ye as (ty.i0, ty.f, tby.i0, tby.i1 | tby.f << 16)
    __shared__ int4 rtab[(kMH > FVV_KMH_BIG ? kMH : FVV_KMH_BIG) + 4];
    {
        const int ys_ = max(0, y0 - 2), ye_ = min(H - 1, y0 + g.mh + 1);
        const int B2_ = g.lv[2].block, lg_ = 31 - __clz(2 * B2_);
        for (int i = threadIdx.x; i <= ye_ - ys_; i += blockDim.x) {
            const int yy = ys_ + i;
            const Tap2 t = tap2(2 * yy - 1, 2, g.lv[1].h);
            const ITap b = clamp_itap32(2 * yy - B2_ + 1, lg_, g.lv[2].nby);
            rtab[i] = make_int4(t.i0, t.f, b.i0, b.i1 | (b.f << 16));
        }
        __syncthreads();  // the only block-level barrier: before any warp leaves
    }
#endif
    if (xw0 >= W) return;
    const int xa = xw0 - 2 + 2 * lane;  // this lane's columns xa, xa + 1 (xa even)
    int xcl[2], gmul[2];
    bool selfL[2], selfR[2];
#pragma unroll
    for (int c = 0; c < 2; c++) {
        const int x = xa + c;
        xcl[c] = clampi(x, 0, W - 1);
        selfL[c] = x <= 0;
        selfR[c] = x >= W - 1;
        gmul[c] = (W >= 2 && (x == 0 || x == W - 1)) ? 2 : (W >= 2 ? 1 : 0);
    }
    const bool own = lane >= 1 && lane <= 30 && xa < W;  // W even: xa + 1 < W as well
    const Level& L1 = g.lv[1];
    const Level& L2 = g.lv[2];
    const int B2 = L2.block, D2 = 2 * B2, lgD2 = 31 - __clz(D2);
    const int mb = g.fb[2] + 1, kY = 2 * mb;
    const int bs = g.fb[2] - (g.fb[1] + 3), rs = g.fb[2] - g.rb[2];
    ITap tu[2], tb[2];
#pragma unroll
    for (int c = 0; c < 2; c++) {
        tu[c] = clamp_itap32(2 * xcl[c] - 1, 2, L1.w);
        tb[c] = clamp_itap32(2 * xcl[c] - B2 + 1, lgD2, L2.nbx);
    }
    const int2* f1[2] = {cplane<int2>(ws, P, P.flow1[0], pair), cplane<int2>(ws, P, P.flow1[1], pair)};
    const BlockHit* hh[2] = {cplane<BlockHit>(ws, P, P.hit[2][0], pair),
                             cplane<BlockHit>(ws, P, P.hit[2][1], pair)};
    const uint8_t* frL = pt.left[pair];
    const uint8_t* frR = pt.right[pair];
    uint8_t* o_wl = plane<uint8_t>(ws, P, P.wl, pair);
    uint8_t* o_wr = plane<uint8_t>(ws, P, P.wr, pair);
    uint16_t* o_sd = plane<uint16_t>(ws, P, P.sd, pair);
    float* o_ol = plane<float>(ws, P, P.occ_l, pair);
    float* o_or = plane<float>(ws, P, P.occ_r, pair);
    uchar4* o_wc = FMT == FVV_YUV420 ? plane<uchar4>(ws, P, P.wc, pair) : nullptr;
    const double c3k = 0x1.5555555555555p-2 * (double)(1.0f / (float)(1 << (mb + 1)));  // exact
    const int ys = max(0, y0 - 2), ye = min(H - 1, y0 + g.mh + 1);
    const int yo1 = min(H, y0 + g.mh);

    // neighbour values of a per-column quantity v[2] with the edge rules folded in
    auto nbrs = [&](const int (&v)[2], int (&l)[2], int (&r)[2]) {
        const int up = __shfl_up_sync(0xffffffffu, v[1], 1);    // column xa - 1
        const int dn = __shfl_down_sync(0xffffffffu, v[0], 1);  // column xa + 2
        l[0] = selfL[0] ? v[0] : up;
        r[0] = selfR[0] ? v[0] : v[1];
        l[1] = selfL[1] ? v[1] : v[0];
        r[1] = selfR[1] ? v[1] : dn;
    };
    auto colpass = [&](int a, int b, int c) {  // f32(f64(sum/3)) of occ in units 2^-(mb+1)
        const int sn = a + b + c;
        return sn ? third_scaled_f32((uint32_t)sn, c3k) : 0.0f;
    };
    auto row3 = [&](float a, float b, float c) {  // f32(f64(a + b + c) / 3)
        if (a == 0.0f && b == 0.0f && c == 0.0f) return 0.0f;
        return (float)div3(__dadd_rn(__dadd_rn((double)a, (double)b), (double)c));
    };

    int ua = -10;
#if FVV_MASK2_HB_CACHE
    int ba = -10;
#endif
    int2 hu0[2][2], hu1[2][2];  // [dir][col]
#if FVV_MASK2_HB_CACHE
    int2 hb0[2][2], hb1[2][2];
#endif
    int2 Fp[2][2], Fc[2][2];                          // F(yy-1), F(yy)
    int Fpp_y[2][2];                                  // F(yy-2).y
    int gxp[2][2], gxc[2][2];                         // gx(yy-1), gx(yy)
    int oc0[2][2], oc1[2][2], oc2[2][2];
    uint32_t dp1 = 0, dp2 = 0;  // |wl - wr| of rows yy-2, yy-1, both columns packed (col 0 | col 1 << 16)
#pragma unroll
    for (int d = 0; d < 2; d++)
#pragma unroll
        for (int c = 0; c < 2; c++) {
            Fp[d][c] = Fc[d][c] = make_int2(0, 0);
            Fpp_y[d][c] = 0;
            gxp[d][c] = gxc[d][c] = 0;
            oc0[d][c] = oc1[d][c] = oc2[d][c] = 0;
        }

    auto xl_u = [&](int d, int row, int c) {
        const int2* r = f1[d] + row * L1.w;
        return lerp_i2(r[tu[c].i0], r[tu[c].i1], 4, tu[c].f);
    };
    auto xl_b = [&](int d, int row, int c) {
        const BlockHit* r = hh[d] + row * L2.nbx;
        const BlockHit p = r[tb[c].i0], q = r[tb[c].i1];
        return lerp_i2(make_int2(p.dx, p.dy), make_int2(q.dx, q.dy), D2, tb[c].f);
    };
    auto emit_o = [&](int t, const int (&a)[2][2], const int (&b)[2][2], const int (&cc)[2][2]) {
        float o[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};
        if (__any_sync(0xffffffffu, (a[0][0] | a[0][1] | a[1][0] | a[1][1] | b[0][0] | b[0][1] | b[1][0] | b[1][1] |
                                     cc[0][0] | cc[0][1] | cc[1][0] | cc[1][1]) != 0)) {
#pragma unroll
            for (int d = 0; d < 2; d++) {
                float v[2];
#pragma unroll
                for (int c = 0; c < 2; c++) v[c] = colpass(a[d][c], b[d][c], cc[d][c]);
                int vi[2] = {__float_as_int(v[0]), __float_as_int(v[1])}, li[2], ri[2];
                nbrs(vi, li, ri);
#pragma unroll
                for (int c = 0; c < 2; c++) o[d][c] = row3(__int_as_float(li[c]), v[c], __int_as_float(ri[c]));
            }
        }
        if (own) {
            *reinterpret_cast<float2*>(o_ol + (unsigned)(t * W + xa)) = make_float2(o[0][0], o[0][1]);
            *reinterpret_cast<float2*>(o_or + (unsigned)(t * W + xa)) = make_float2(o[1][0], o[1][1]);
        }
    };

#if FVV_MASK2_PF
    int2 Fn[2][2];
    int gxn[2][2];
    int T[2][2][4];   // the luma taps of the next row, per (direction, column), loaded one row ahead
    int2 TF[2][2];    // their bilinear weights (fx, fy) in units 2^-mb
    auto flows_of = [&](int yy, int2 (&Fo)[2][2], int (&gxo)[2][2]) {
        const Tap2 ty = tap2(2 * yy - 1, 2, L1.h);
        if (ty.i0 != ua) {
#pragma unroll
            for (int d = 0; d < 2; d++)
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    hu0[d][c] = ty.i0 == ua + 1 ? hu1[d][c] : xl_u(d, ty.i0, c);
                    hu1[d][c] = xl_u(d, ty.i0 + 1, c);
                }
            ua = ty.i0;
        }
        const ITap tby = clamp_itap32(2 * yy - B2 + 1, lgD2, L2.nby);
        if (tby.i0 != ba) {
#pragma unroll
            for (int d = 0; d < 2; d++)
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    hb0[d][c] = tby.i0 == ba + 1 ? hb1[d][c] : xl_b(d, tby.i0, c);
                    hb1[d][c] = xl_b(d, tby.i1, c);
                }
            ba = tby.i0;
        }
#pragma unroll
        for (int d = 0; d < 2; d++) {
            int fx[2];
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const int2 base = lerp_i2(hu0[d][c], hu1[d][c], 4, ty.f);
                const int2 res = lerp_i2(hb0[d][c], hb1[d][c], D2, tby.f);
                Fo[d][c] = make_int2(-((base.x << bs) + (res.x << rs)), -((base.y << bs) + (res.y << rs)));
                fx[c] = Fo[d][c].x;
            }
            int l[2], r[2];
            nbrs(fx, l, r);
#pragma unroll
            for (int c = 0; c < 2; c++) gxo[d][c] = gmul[c] * (r[c] - l[c]);
        }
    };
    auto issue = [&](int yy) {  // bilin_fixed's taps of row yy, loads only
#pragma unroll
        for (int d = 0; d < 2; d++) {
            const uint8_t* fr = d ? frR : frL;
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const Tap2 tx = tap2((xcl[c] << mb) + Fn[d][c].x, mb, W), tyy = tap2((yy << mb) + Fn[d][c].y, mb, H);
                const uint8_t* r0 = fr + (unsigned)(tyy.i0 * W + tx.i0);
                T[d][c][0] = r0[0];
                T[d][c][1] = r0[1];
                T[d][c][2] = r0[W];
                T[d][c][3] = r0[W + 1];
                TF[d][c] = make_int2(tx.f, tyy.f);
            }
        }
    };
#endif
    auto step = [&](int yy, auto gen) {
        constexpr bool GEN = decltype(gen)::value;
#if FVV_MASK2_PF
        // rotate the windows (F(yy) and gx(yy) were computed one row ahead)
#pragma unroll
        for (int d = 0; d < 2; d++)
#pragma unroll
            for (int c = 0; c < 2; c++) {
                Fpp_y[d][c] = Fp[d][c].y;
                Fp[d][c] = Fc[d][c];
                Fc[d][c] = Fn[d][c];
                gxp[d][c] = gxc[d][c];
                gxc[d][c] = gxn[d][c];
            }
        // ---- luma warps at yy from the taps loaded during the previous row ----
        int wl[2], wr[2];
#pragma unroll
        for (int c = 0; c < 2; c++) {
            wl[c] = rne64((long long)bilerp_u(T[0][c][0], T[0][c][1], T[0][c][2], T[0][c][3], TF[0][c].x, TF[0][c].y, mb), kY);
            wr[c] = rne64((long long)bilerp_u(T[1][c][0], T[1][c][1], T[1][c][2], T[1][c][3], TF[1][c].x, TF[1][c].y, mb), kY);
        }
        // ---- next row: its flows, then its tap loads, in flight behind this row's work ----
        if (yy < ye) {
            flows_of(yy + 1, Fn, gxn);
            issue(yy + 1);
        }
#else
#if FVV_MASK2_RTAB
        const int4 rtv = rtab[yy - ys];
        Tap2 ty;
        ty.i0 = rtv.x;
        ty.f = rtv.y;
#else
        const Tap2 ty = tap2(2 * yy - 1, 2, L1.h);
#endif
        if (ty.i0 != ua) {
#pragma unroll
            for (int d = 0; d < 2; d++)
#pragma unroll
                for (int c = 0; c < 2; c++) {
#if FVV_MASK2_DLERP
                    // (hu0, hu1) = (4 u0, u1 - u0): the row lerp is one multiply-add per component
                    const int2 a = ty.i0 == ua + 1 ? make_int2((hu0[d][c].x >> 2) + hu1[d][c].x, (hu0[d][c].y >> 2) + hu1[d][c].y)
                                                   : xl_u(d, ty.i0, c);
                    const int2 b = xl_u(d, ty.i0 + 1, c);
                    hu0[d][c] = make_int2(a.x << 2, a.y << 2);
                    hu1[d][c] = make_int2(b.x - a.x, b.y - a.y);
#else
                    hu0[d][c] = ty.i0 == ua + 1 ? hu1[d][c] : xl_u(d, ty.i0, c);
                    hu1[d][c] = xl_u(d, ty.i0 + 1, c);
#endif
                }
#if FVV_MASK2_FPF
            // the flow row the next reload reads (two walker rows on), into L1 now:
            // F -> luma address -> gather is a dependent chain behind it
            if (ty.i0 + 1 + FVV_MASK2_FPF < L1.h) {
#pragma unroll
                for (int d = 0; d < 2; d++)
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(f1[d] + (ty.i0 + 1 + FVV_MASK2_FPF) * L1.w + tu[0].i0));
            }
#endif
            ua = ty.i0;
        }
#if FVV_MASK2_RTAB
        ITap tby;
        tby.i0 = rtv.z;
        tby.i1 = rtv.w & 0xFFFF;
        tby.f = rtv.w >> 16;
#else
        const ITap tby = clamp_itap32(2 * yy - B2 + 1, lgD2, L2.nby);
#endif
#if FVV_MASK2_HB_CACHE
        if (tby.i0 != ba) {
#pragma unroll
            for (int d = 0; d < 2; d++)
#pragma unroll
                for (int c = 0; c < 2; c++) {
#if FVV_MASK2_DLERP
                    // (hb0, hb1) = (D2 p, q - p)
                    const int2 a = tby.i0 == ba + 1 ? make_int2((hb0[d][c].x >> lgD2) + hb1[d][c].x, (hb0[d][c].y >> lgD2) + hb1[d][c].y)
                                                    : xl_b(d, tby.i0, c);
                    const int2 b = xl_b(d, tby.i1, c);
                    hb0[d][c] = make_int2(a.x << lgD2, a.y << lgD2);
                    hb1[d][c] = make_int2(b.x - a.x, b.y - a.y);
#else
                    hb0[d][c] = tby.i0 == ba + 1 ? hb1[d][c] : xl_b(d, tby.i0, c);
                    hb1[d][c] = xl_b(d, tby.i1, c);
#endif
                }
#if FVV_MASK2_HPF
            if (tby.i1 + 1 < L2.nby) {
#pragma unroll
                for (int d = 0; d < 2; d++)
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(hh[d] + (tby.i1 + 1) * L2.nbx + tb[0].i0));
            }
#endif
            ba = tby.i0;
        }
#else
        // block-grid rows re-lerped every row from L1-resident hits (saves 16 registers)
        int2 hb0[2][2], hb1[2][2];
#pragma unroll
        for (int d = 0; d < 2; d++)
#pragma unroll
            for (int c = 0; c < 2; c++) {
                hb0[d][c] = xl_b(d, tby.i0, c);
                hb1[d][c] = xl_b(d, tby.i1, c);
            }
#endif
        // ---- mid flows F(yy), x-gradients gx(yy) ----
#pragma unroll
        for (int d = 0; d < 2; d++) {
            int fx[2];
#pragma unroll
            for (int c = 0; c < 2; c++) {
#if FVV_MASK2_DLERP
                const int2 base = make_int2(hu0[d][c].x + ty.f * hu1[d][c].x, hu0[d][c].y + ty.f * hu1[d][c].y);
                const int2 res = make_int2(hb0[d][c].x + tby.f * hb1[d][c].x, hb0[d][c].y + tby.f * hb1[d][c].y);
#else
                const int2 base = lerp_i2(hu0[d][c], hu1[d][c], 4, ty.f);
                const int2 res = lerp_i2(hb0[d][c], hb1[d][c], D2, tby.f);
#endif
                Fpp_y[d][c] = Fp[d][c].y;
                Fp[d][c] = Fc[d][c];
                Fc[d][c] = make_int2(-((base.x << bs) + (res.x << rs)), -((base.y << bs) + (res.y << rs)));
                fx[c] = Fc[d][c].x;
            }
            int l[2], r[2];
            nbrs(fx, l, r);
#pragma unroll
            for (int c = 0; c < 2; c++) {
                gxp[d][c] = gxc[d][c];
                gxc[d][c] = gmul[c] * (r[c] - l[c]);
            }
        }
#if FVV_MASK2_L1PF
        // pull the luma rows the walker reaches FVV_MASK2_L1PF rows from now into L1 (the
        // gathers' long-scoreboard stalls are mostly first touches of a row's lines)
        {
            const int yq = yy + FVV_MASK2_L1PF;
#pragma unroll
            for (int d = 0; d < 2; d++) {
                const int sy = min(max(yq + (Fc[d][0].y >> mb), 0), H - 1);
                const int sx = min(max(xcl[0] + (Fc[d][0].x >> mb), 0), W - 1);
                asm volatile("prefetch.global.L1 [%0];\n" ::"l"((d ? frR : frL) + (unsigned)(sy * W + sx)));
#if FVV_MASK2_L2PF
                const int sy2 = min(max(yy + FVV_MASK2_L2PF + (Fc[d][0].y >> mb), 0), H - 1);
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"((d ? frR : frL) + (unsigned)(sy2 * W + sx)));
#endif
#if FVV_MASK2_L1PF_C
                if (FMT == FVV_YUV420 && (yy & 1)) {  // the chroma rows of the same 2x2 blocks
                    const int cw = g.cw, chh = g.ch;
                    const int cy = min(max((yq >> 1) + (Fc[d][0].y >> (mb + 1)), 0), chh - 1);
                    const int cx = min(max((xa >> 1) + (Fc[d][0].x >> (mb + 1)), 0), cw - 1);
                    const uint8_t* cp = (d ? frR : frL) + (size_t)W * H + (unsigned)(cy * cw + cx);
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(cp));
                    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(cp + (size_t)cw * chh));
                }
#endif
            }
        }
#endif
        // ---- luma warps at yy, d = |wl - wr| ----
        int wl[2], wr[2];
#pragma unroll
        for (int c = 0; c < 2; c++) {
            wl[c] = rne64(bilin_fixed(frL, W, H, W, yy, xcl[c], Fc[0][c].x, Fc[0][c].y, mb), kY);
            wr[c] = rne64(bilin_fixed(frR, W, H, W, yy, xcl[c], Fc[1][c].x, Fc[1][c].y, mb), kY);
        }
#endif
        const uint32_t dp0 = dp1;
        dp1 = dp2;
        dp2 = (uint32_t)abs(wl[0] - wr[0]) | ((uint32_t)abs(wl[1] - wr[1]) << 16);
        if (own && (!GEN || (yy >= y0 && yy < yo1))) {
            *reinterpret_cast<uint16_t*>(o_wl + (unsigned)(yy * W + xa)) = (uint16_t)(wl[0] | (wl[1] << 8));
            *reinterpret_cast<uint16_t*>(o_wr + (unsigned)(yy * W + xa)) = (uint16_t)(wr[0] | (wr[1] << 8));
        }
        // ---- Sd(yy-1) ----
        {
            const int t = yy - 1;
            if (own && (!GEN || (t >= y0 && t < yo1))) {  // lane-wise sums < 2^16: packed adds
                const uint32_t sp = ((GEN && t == 0) ? dp1 : dp0) + dp1 + dp2;
                *reinterpret_cast<uint32_t*>(o_sd + (unsigned)(t * W + xa)) = sp;
            }
        }
        // ---- occ(yy-1) then O0/O(yy-2) ----
        {
            const int r = yy - 1;
            if (!GEN || (r >= ys && (r == 0 || r - 1 >= ys))) {
#pragma unroll
                for (int d = 0; d < 2; d++) {
#pragma unroll
                    for (int c = 0; c < 2; c++) {
                        const int gy = H < 2 ? 0 : ((GEN && r == 0) ? 2 * (Fc[d][c].y - Fp[d][c].y)
                                                                    : Fc[d][c].y - Fpp_y[d][c]);
                        const int v = -(gxp[d][c] + gy);
                        oc0[d][c] = oc1[d][c];
                        oc1[d][c] = oc2[d][c];
                        oc2[d][c] = v > 0 ? v : 0;
                    }
                }
                const int t2 = yy - 2;
                if (!GEN || (t2 >= y0 && t2 < yo1)) {
                    if (GEN && t2 == 0) emit_o(t2, oc1, oc1, oc2);
                    else emit_o(t2, oc0, oc1, oc2);
                }
            }
        }
        // ---- chroma pixel (xa/2, (yy-1)/2) at odd yy: the lane's own 2x2 block ----
        if (FMT == FVV_YUV420 && (yy & 1) && (!GEN || (yy - 1 >= y0 && yy - 1 < yo1 && yy - 1 >= ys))) {
            if (own) {
                const int cw = g.cw, chh = g.ch, cb = mb + 3, kC = 2 * cb;
                const int cy = (yy - 1) >> 1, cx = xa >> 1;
                int2 cv[2];
#pragma unroll
                for (int d = 0; d < 2; d++)
                    cv[d] = make_int2((Fp[d][0].x + Fc[d][0].x) + (Fp[d][1].x + Fc[d][1].x),
                                      (Fp[d][0].y + Fc[d][0].y) + (Fp[d][1].y + Fc[d][1].y));
                const uint8_t* ul = frL + (size_t)W * H;
                const uint8_t* ur = frR + (size_t)W * H;
                const size_t cpl = (size_t)cw * chh;
                const uint8_t a0 = (uint8_t)rne64(bilin_fixed(ul, cw, chh, cw, cy, cx, cv[0].x, cv[0].y, cb), kC);
                const uint8_t a1 = (uint8_t)rne64(bilin_fixed(ur, cw, chh, cw, cy, cx, cv[1].x, cv[1].y, cb), kC);
                const uint8_t b0 = (uint8_t)rne64(bilin_fixed(ul + cpl, cw, chh, cw, cy, cx, cv[0].x, cv[0].y, cb), kC);
                const uint8_t b1 = (uint8_t)rne64(bilin_fixed(ur + cpl, cw, chh, cw, cy, cx, cv[1].x, cv[1].y, cb), kC);
                o_wc[(unsigned)(cy * cw + cx)] = make_uchar4(a0, a1, b0, b1);
            }
        }
    };
#if FVV_MASK2_PF
    flows_of(ys, Fn, gxn);
    issue(ys);
#endif
    const int b0 = min(max(y0 + 2, 3), yo1), b1 = max(b0, yo1);
    int yy = ys;
    for (; yy < b0; yy++) step(yy, std::true_type{});
#pragma unroll kMask2Unroll
    for (; yy < b1; yy++) step(yy, std::false_type{});
    for (; yy <= ye; yy++) step(yy, std::true_type{});
    if (ye == H - 1) {
#pragma unroll
        for (int d = 0; d < 2; d++) {
#pragma unroll
            for (int c = 0; c < 2; c++) {
                const int gy = H < 2 ? 0 : 2 * (Fc[d][c].y - Fp[d][c].y);
                const int v = -(gxc[d][c] + gy);
                oc0[d][c] = oc1[d][c];
                oc1[d][c] = oc2[d][c];
                oc2[d][c] = v > 0 ? v : 0;
            }
        }
        if (H - 2 >= y0 && H - 2 < yo1) emit_o(H - 2, oc0, oc1, oc2);
        if (H - 1 >= y0 && H - 1 < yo1) emit_o(H - 1, oc1, oc2, oc2);
        if (own && H - 1 >= y0 && H - 1 < yo1)
            *reinterpret_cast<uint32_t*>(o_sd + (size_t)(H - 1) * W + xa) = dp1 + dp2 + dp2;
    }
}

// ---------------------------------------------------------------------------
// Per-pixel mask and blend (warp.py:49-88), shared by k_blend.
// ---------------------------------------------------------------------------
// mask (warp.py:63) and clip for one pixel from the row-pass running sum
__device__ __forceinline__ double mask_of(double tsum, float occ_l, float occ_r, const Geometry& g) {
    const double D = div3(tsum);
    const float ql = __fadd_rn(0.5f, __fmul_rn(4.0f, occ_l));
    const float qr = __fadd_rn(0.5f, __fmul_rn(4.0f, occ_r));
    const double el = __dmul_rn(D, f2d_posnormal(ql));  // ql, qr >= 0.5
    const double er = __dmul_rn(D, f2d_posnormal(qr));
    const double num = __dadd_rn(er, g.eps), den = __dadd_rn(__dadd_rn(el, er), g.eps2);
    const double m = g.fastdiv ? ddiv_fast(num, den) : __ddiv_rn(num, den);
    return m < 0.0 ? 0.0 : (m > 1.0 ? 1.0 : m);  // np.clip (m is never NaN: den >= 2 eps)
}
// blend (warp.py:66-67): to_uint8(m * a + (1 - m) * b)
__device__ __forceinline__ uint8_t blend_px(double m, int a, int b) {
    return to_u8_small(__dadd_rn(__dmul_rn(m, u2d_exact(a)), __dmul_rn(__dsub_rn(1.0, m), u2d_exact(b))));
}

// ---------------------------------------------------------------------------
// Split row scan.  The only order-dependent part of the mask is scipy's
// running sum along each row of smooth3(|wl - wr|) (tmp(x) = tmp(x-1) +
// (p[x+2] - p[x-1]), f64).  k_scan_carry runs that chain once per row and
// stores tmp at every 8th column; k_blend then replays the <= 7 chain steps
// of its own 8-column group from the stored carry -- the same additions in
// the same order, so the same doubles -- and evaluates mask + blend fully in
// parallel (thread = 2 rows x 8 columns, chroma from the row pair).
// ---------------------------------------------------------------------------
#ifndef FVV_KCC
#define FVV_KCC 96  // r2 v13 sweep (cfg4 scan ms per rig frame): 32 / 64 / 96 / 128 = 0.392 / 0.365 / 0.334 / 0.344
#endif
#ifndef FVV_SCAN_TSTORE
#define FVV_SCAN_TSTORE 1
#endif
constexpr int kCR = 32, kCC = FVV_KCC;  // carry kernel: rows per CTA (one lane each), chunk columns
constexpr int kCT = kCC + 16;       // staged u16 per row and chunk: sd[c0-8 .. c0+72)
constexpr int kCTP = kCT + 4;       // row pitch: 2*kCTP B (168 B = 21 x 8 B at kCC 64, 232 B = 29 x 8 B at 96): odd 8-byte count, 16 lanes hit 16 bank pairs
// the double2 carry stores step by 2 up to kCC/8 and the transpose moves kCC/16 pieces per row
static_assert(kCC % 16 == 0 && kCC >= 16, "FVV_KCC must be a positive multiple of 16");
static_assert(((2 * kCTP) / 8) % 2 == 1 && (2 * kCTP) % 8 == 0, "carry row pitch must be an odd number of 8-byte words");

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ double d0_of(int s) { return div3(u2d_exact(s)); }  // == s / 3.0 (IEEE)

template <bool COOP>
__global__ void __launch_bounds__(kCR) k_scan_carry(Geometry g, const uint8_t* __restrict__ ws,
                                                    Planes P) {
    pdl_enter();
    __shared__ __align__(16) uint16_t tile[2][kCR][kCTP];  // per lane: its own row segment
#if FVV_SCAN_TSTORE
    __shared__ __align__(16) double ctile[kCR][kCC / 8 + 2];  // carry transpose (80 B pitch: no conflicts)
#endif
    const int W = g.W, H = g.H;
    const int pair = blockIdx.y, y0 = blockIdx.x * kCR;
    const int lane = threadIdx.x;
    const uint16_t* sd = cplane<uint16_t>(ws, P, P.sd, pair);
    double* carry = reinterpret_cast<double*>(const_cast<uint8_t*>(ws) + P.stride * (size_t)pair + P.carry);
    const int ng = (W + 7) / 8;
    const int y = min(y0 + lane, H - 1);
    const bool live = y0 + lane < H;
    const uint16_t* row = sd + (size_t)y * W;
    const int nchunks = (W + kCC - 1) / kCC;
    const bool vec = (W % 4) == 0;  // 8-byte aligned row segments (always, frames are W % 4 == 0)
    // stage chunk k into tile[k & 1][r] for the warp's 32 rows r: entry j holds
    // sd[clamp(c0 - 8 + j)].  In-range entries come in 8-byte cp.async pieces
    // (c0 - 8 and W are multiples of 4), issued cooperatively when COOP: consecutive
    // lanes take consecutive pieces of the same row, so one instruction touches
    // ~2 rows' contiguous bytes instead of 32 rows (r1 v21 ncu: the per-lane-row
    // staging was MIO/LSU-throttled).  Only the clamped ends are written with
    // plain stores, each lane into its own row (the only row it reads).
    auto stage = [&](int k) {
        const int c0 = k * kCC;
        uint16_t* t = tile[k & 1][lane];
        if (vec) {
            const int jlo = max(0, 8 - c0);                  // first in-range entry
            const int jhi = min(kCT, W - (c0 - 8));          // one past the last
            if (!COOP) {
                for (int j = jlo; j < jhi; j += 4) cp_async8(t + j, row + c0 - 8 + j);
            } else if (jlo == 0 && jhi == kCT) {
                constexpr int NP = kCT / 4;                   // pieces per row
#pragma unroll 4
                for (int i = lane; i < kCR * NP; i += 32) {
                    const int r = i / NP, j = 4 * (i - r * NP);
                    const uint16_t* rw = sd + (size_t)min(y0 + r, H - 1) * W;
                    cp_async8(&tile[k & 1][r][j], rw + c0 - 8 + j);
                }
            } else {
                const int np = (jhi - jlo) >> 2;
                for (int r = 0; r < kCR; r++) {
                    const uint16_t* rw = sd + (size_t)min(y0 + r, H - 1) * W;
                    for (int q = lane; q < np; q += 32)
                        cp_async8(&tile[k & 1][r][jlo + 4 * q], rw + c0 - 8 + jlo + 4 * q);
                }
            }
            if (jlo > 0) {
                const uint16_t v = row[0];
                for (int j = 0; j < jlo; j++) t[j] = v;
            }
            if (jhi < kCT) {
                const uint16_t v = row[W - 1];
                for (int j = max(jhi, 0); j < kCT; j++) t[j] = v;
            }
        } else {
            for (int j = 0; j < kCT; j++) t[j] = row[clampi(c0 - 8 + j, 0, W - 1)];
        }
        cp_async_commit();
    };
    stage(0);
    double tmp = 0.0;
    double ep[3] = {0.0, 0.0, 0.0};  // D0 of sd[x0-2 .. x0] carried from the previous group
    for (int k = 0; k < nchunks; k++) {
        if (k + 1 < nchunks) {
            stage(k + 1);
            cp_async_wait_1();
        } else {
            cp_async_wait_0();
        }
        __syncwarp();
        const int c0 = k * kCC;
        const int n = min(kCC, W - c0);
        const uint16_t* tl = tile[k & 1][lane];  // tl[j] = sd[clamp(c0 - 8 + j)]
        double* cr = carry + (size_t)y * ng + c0 / 8;
        double cv[kCC / 8];   // this chunk's carries: one 64-byte row segment per lane
#pragma unroll
        for (int i = 0; i < kCC / 8; i++) cv[i] = 0.0;
        if (n == kCC && c0 > 0) {
            // full interior chunk: no data-dependent exits, so the D0 work of every
            // group is free to be scheduled ahead of the ordered DADD chain
#pragma unroll
            for (int c8 = 0; c8 < kCC; c8 += 8) {
                const int x0 = c0 + c8;
                double e[11];                       // e[i] = D0(sd[clamp(x0 - 2 + i)])
                e[0] = ep[0]; e[1] = ep[1]; e[2] = ep[2];
                {
                    const uint2 qa = *reinterpret_cast<const uint2*>(tl + c8 + 8);   // sd[x0 .. x0+3]
                    const uint2 qb = *reinterpret_cast<const uint2*>(tl + c8 + 12);  // sd[x0+4 .. x0+7]
                    const uint2 qc = *reinterpret_cast<const uint2*>(tl + c8 + 16);  // sd[x0+8 .. x0+11]
                    e[3] = d0_of(qa.x >> 16);    e[4] = d0_of(qa.y & 0xFFFF); e[5] = d0_of(qa.y >> 16);
                    e[6] = d0_of(qb.x & 0xFFFF); e[7] = d0_of(qb.x >> 16);    e[8] = d0_of(qb.y & 0xFFFF);
                    e[9] = d0_of(qb.y >> 16);    e[10] = d0_of(qc.x & 0xFFFF);
                }
                ep[0] = e[8]; ep[1] = e[9]; ep[2] = e[10];
                (void)x0;
                tmp = __dadd_rn(tmp, __dsub_rn(e[3], e[0]));
                cv[c8 >> 3] = tmp;
#pragma unroll
                for (int j = 1; j < 8; j++) tmp = __dadd_rn(tmp, __dsub_rn(e[j + 3], e[j]));
            }
        } else {
#pragma unroll
        for (int c8 = 0; c8 < kCC; c8 += 8) {
            if (c8 >= n) break;
            const int x0 = c0 + c8;
            // sd[x0+1 .. x0+8] = tl[c8+9 .. c8+16]: new D0 values of this group
            double e[11];                       // e[i] = D0(sd[clamp(x0 - 2 + i)])
            if (x0 == 0) {
                const uint2 h = *reinterpret_cast<const uint2*>(tl + c8 + 8);  // sd[0..3]
                e[2] = d0_of(h.x & 0xFFFF);
                e[0] = e[1] = e[2];
            } else {
                e[0] = ep[0]; e[1] = ep[1]; e[2] = ep[2];
            }
            {
                const uint2 qa = *reinterpret_cast<const uint2*>(tl + c8 + 8);   // sd[x0 .. x0+3]
                const uint2 qb = *reinterpret_cast<const uint2*>(tl + c8 + 12);  // sd[x0+4 .. x0+7]
                const uint2 qc = *reinterpret_cast<const uint2*>(tl + c8 + 16);  // sd[x0+8 .. x0+11]
                e[3] = d0_of(qa.x >> 16);    e[4] = d0_of(qa.y & 0xFFFF); e[5] = d0_of(qa.y >> 16);
                e[6] = d0_of(qb.x & 0xFFFF); e[7] = d0_of(qb.x >> 16);    e[8] = d0_of(qb.y & 0xFFFF);
                e[9] = d0_of(qb.y >> 16);    e[10] = d0_of(qc.x & 0xFFFF);
            }
            ep[0] = e[8]; ep[1] = e[9]; ep[2] = e[10];
            // delta(x0 + j) = D0(sd[x0+j+1]) - D0(sd[x0+j-2]) = e[j+3] - e[j]
            if (x0 == 0) {
                tmp = __dadd_rn(__dadd_rn(e[2], e[2]), W > 1 ? e[3] : e[2]);
            } else {
                tmp = __dadd_rn(tmp, __dsub_rn(e[3], e[0]));
            }
            cv[c8 >> 3] = tmp;
            if (n - c8 >= 8) {
#pragma unroll
                for (int j = 1; j < 8; j++) tmp = __dadd_rn(tmp, __dsub_rn(e[j + 3], e[j]));
            } else {
                const int m = n - c8;
#pragma unroll
                for (int j = 1; j < 8; j++)
                    if (j < m) tmp = __dadd_rn(tmp, __dsub_rn(e[j + 3], e[j]));
            }
        }
        }
#if FVV_SCAN_TSTORE
        if (COOP && n == kCC && (ng & 1) == 0 && y0 + kCR <= H) {
            // full chunk of 32 live rows: transpose the carries through shared memory so
            // consecutive lanes store consecutive 16-byte pieces of the same row
            double2* cs = reinterpret_cast<double2*>(&ctile[lane][0]);
#pragma unroll
            for (int i = 0; i < kCC / 8; i += 2) cs[i / 2] = make_double2(cv[i], cv[i + 1]);
            __syncwarp();
            constexpr int PR = kCC / 16;  // double2 pieces per row
#pragma unroll
            for (int i = lane; i < kCR * PR; i += 32) {
                const int r = i / PR, q = i - (i / PR) * PR;
                *reinterpret_cast<double2*>(carry + (size_t)(y0 + r) * ng + c0 / 8 + 2 * q) =
                    reinterpret_cast<const double2*>(&ctile[r][0])[q];
            }
        } else
#endif
        if (live) {
            const int ngc = (n + 7) / 8;
            if (ngc == kCC / 8 && (ng & 1) == 0) {   // 16-byte aligned full segment
#pragma unroll
                for (int i = 0; i < kCC / 8; i += 2)
                    *reinterpret_cast<double2*>(cr + i) = make_double2(cv[i], cv[i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < kCC / 8; i++)
                    if (i < ngc) cr[i] = cv[i];
            }
        }
        __syncwarp();
    }
}

#ifndef FVV_MINB_BLEND
#define FVV_MINB_BLEND 10
#endif
#ifndef FVV_BLEND_HALF
#define FVV_BLEND_HALF 0  // m = 1/2 shortcut for groups with equal cues: exact, but rare on the bench rig (1.16 -> 1.18 ms), off
#endif
template <int FMT>
__global__ void __launch_bounds__(128, FVV_MINB_BLEND) k_blend(Geometry g, PairTable pt, const uint8_t* __restrict__ ws,
                                               Planes P, int pair_base, bool write_frame,
                                               double* mask_out /* nullable: (launch pairs, H, W) */) {
    pdl_enter();
    // thread = one 8-column group of ONE row; a warp holds 16 groups x the 2 rows
    // of a row pair (lanes 0-15: upper row, 16-31: lower row), so the chroma
    // 2x2-mean mask comes from a shuffle and each thread keeps one row's state
    const int W = g.W, H = g.H;
    const int pair = blockIdx.z + pair_base;
    const int ng = (W + 7) / 8;
    const int lane = threadIdx.x & 31;
    const int rr = lane >> 4;                                               // row within the pair
    const int gxr = blockIdx.x * (blockDim.x / 2) + (threadIdx.x >> 5) * 16 + (lane & 15);
    const bool active = gxr < ng;
    const int gx = active ? gxr : ng - 1;                                   // 8-column group
    const int yp = blockIdx.y;                                              // row pair
    const int x0 = gx * 8, n = min(8, W - x0);
    const uint16_t* sd = cplane<uint16_t>(ws, P, P.sd, pair);
    const double* carry = cplane<double>(ws, P, P.carry, pair);
    const float* ol = cplane<float>(ws, P, P.occ_l, pair);
    const float* orr = cplane<float>(ws, P, P.occ_r, pair);
    const uint8_t* wl = cplane<uint8_t>(ws, P, P.wl, pair);
    const uint8_t* wr = cplane<uint8_t>(ws, P, P.wr, pair);
    uint8_t* out = pt.out[pair];
    double csum[4];  // chroma: per column pair, m(2j) + m(2j+1) of this thread's row
    {
        const int y = 2 * yp + rr;
        const size_t ro = (size_t)y * W;
        const uint16_t* srow = sd + ro;
        float vl[8], vr[8];
        uint8_t al[8], ar[8];
        if (n == 8) {
            const float4 a = *reinterpret_cast<const float4*>(ol + ro + x0);
            const float4 b = *reinterpret_cast<const float4*>(ol + ro + x0 + 4);
            const float4 c = *reinterpret_cast<const float4*>(orr + ro + x0);
            const float4 d = *reinterpret_cast<const float4*>(orr + ro + x0 + 4);
            vl[0] = a.x; vl[1] = a.y; vl[2] = a.z; vl[3] = a.w; vl[4] = b.x; vl[5] = b.y; vl[6] = b.z; vl[7] = b.w;
            vr[0] = c.x; vr[1] = c.y; vr[2] = c.z; vr[3] = c.w; vr[4] = d.x; vr[5] = d.y; vr[6] = d.z; vr[7] = d.w;
            if (FMT != FVV_RGB8) {
                // u8 rows are only 4-byte aligned (W % 4 == 0)
                const uint2 p = make_uint2(*reinterpret_cast<const uint32_t*>(wl + ro + x0),
                                           *reinterpret_cast<const uint32_t*>(wl + ro + x0 + 4));
                const uint2 q = make_uint2(*reinterpret_cast<const uint32_t*>(wr + ro + x0),
                                           *reinterpret_cast<const uint32_t*>(wr + ro + x0 + 4));
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    al[j] = (p.x >> (8 * j)) & 0xFF; al[4 + j] = (p.y >> (8 * j)) & 0xFF;
                    ar[j] = (q.x >> (8 * j)) & 0xFF; ar[4 + j] = (q.y >> (8 * j)) & 0xFF;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++) {
                const int xx = min(x0 + j, W - 1);
                vl[j] = ol[ro + xx]; vr[j] = orr[ro + xx];
                if (FMT != FVV_RGB8) { al[j] = wl[ro + xx]; ar[j] = wr[ro + xx]; }
            }
        }
        double mrow[8];
        // equal occlusion cues (in smooth flow both are 0): e_l == e_r, so den = (2 e_r) + 2 eps =
        // 2 (e_r + eps) exactly and m = 1/2 whatever the smoothed difference is (warp.py:63) --
        // the running-sum replay, its sd / carry loads and the mask division are skipped
        bool half = FVV_BLEND_HALF != 0;
#pragma unroll
        for (int j = 0; j < 8; j++) half = half && (j >= n || vl[j] == vr[j]);
        if (half) {
#pragma unroll
            for (int j = 0; j < 8; j++) mrow[j] = j < n ? 0.5 : 0.0;
        } else {
            int s[11];  // sd[clamp(x0 - 2 + j)]
            if ((W & 7) == 0 && x0 >= 2 && x0 + 8 < W) {
                // interior: sd[x0-2 .. x0-1] (4-byte aligned), sd[x0 .. x0+7] (16-byte), sd[x0+8]
                const uint32_t a = *reinterpret_cast<const uint32_t*>(srow + x0 - 2);
                const uint4 b = *reinterpret_cast<const uint4*>(srow + x0);
                s[0] = a & 0xFFFF; s[1] = a >> 16;
                s[2] = b.x & 0xFFFF; s[3] = b.x >> 16; s[4] = b.y & 0xFFFF; s[5] = b.y >> 16;
                s[6] = b.z & 0xFFFF; s[7] = b.z >> 16; s[8] = b.w & 0xFFFF; s[9] = b.w >> 16;
                s[10] = srow[x0 + 8];
            } else {
#pragma unroll
                for (int j = 0; j < 11; j++) s[j] = srow[clampi(x0 - 2 + j, 0, W - 1)];
            }
            // replay the running sum inside the group: tmp(x0) from the carry, then x0+1 ..
            double tmp = carry[(size_t)y * ng + gx];
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (j > 0) tmp = __dadd_rn(tmp, __dsub_rn(d0_of(s[j + 3]), d0_of(s[j])));
                mrow[j] = j < n ? mask_of(tmp, vl[j], vr[j], g) : 0.0;
            }
        }
        if (write_frame && active) {
            if (FMT == FVV_RGB8) {
                const uint8_t* px = cplane<uint8_t>(ws, P, P.wrgb, pair) + (ro + x0) * 6;
                uint8_t* o = out + (ro + x0) * 3;
#pragma unroll
                for (int j = 0; j < 8; j++)
                    if (j < n)
#pragma unroll
                        for (int ch = 0; ch < 3; ch++)
                            o[3 * j + ch] = blend_px(mrow[j], px[6 * j + ch], px[6 * j + 3 + ch]);
            } else {
                uint32_t lo = 0, hi = 0;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    lo |= (uint32_t)blend_px(mrow[j], al[j], ar[j]) << (8 * j);
                    hi |= (uint32_t)blend_px(mrow[4 + j], al[4 + j], ar[4 + j]) << (8 * j);
                }
                *reinterpret_cast<uint32_t*>(out + ro + x0) = lo;  // W % 4 == 0: n is 4 or 8
                if (n == 8) *reinterpret_cast<uint32_t*>(out + ro + x0 + 4) = hi;
            }
        }
        if (mask_out && active) {
            double* mo = mask_out + (size_t)blockIdx.z * W * H;  // this launch's pair
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < n) mo[ro + x0 + j] = mrow[j];
        }
        if (FMT == FVV_YUV420) {
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const double p = __dadd_rn(mrow[2 * j], mrow[2 * j + 1]);
                const double up = __shfl_xor_sync(0xffffffffu, p, 16);  // the other row's pair sum
                csum[j] = rr == 0 ? p : __dadd_rn(up, p);                // (a + b) + (c + d)
            }
        }
    }
    // chroma blend with the 2x2-mean mask (warp.py:83-88)
    if (FMT == FVV_YUV420 && write_frame && active && rr == 1) {
        const int cw = g.cw, chh = g.ch;
        const int cx0 = x0 / 2, nc = n / 2;
        const uchar4* wc = cplane<uchar4>(ws, P, P.wc, pair) + (size_t)yp * cw + cx0;
        uint8_t* uo = out + (size_t)W * H + (size_t)yp * cw + cx0;
        uint8_t* vo = uo + (size_t)cw * chh;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            if (j >= nc) break;
            const double mc = __dmul_rn(csum[j], 0.25);  // /4 == *0.25 exactly
            const uchar4 q = wc[j];
            uo[j] = blend_px(mc, q.x, q.y);
            vo[j] = blend_px(mc, q.z, q.w);
        }
    }
}

// k_blend_s: k_blend streamed per pixel -- the same operations in the same
// order (bit-identical), but each pixel's mask is consumed (blend byte, mask
// store, chroma pair sum) as soon as it is formed instead of staging 8 masks,
// the warped luma and the sd window stay packed in their load registers, and
// the chroma row is split across the row pair (upper lanes U, lower lanes V;
// both hold the full 2x2 sum: RN((a+b)+(c+d)) either way round).  Its loads
// (including the chroma sources) are all issued up front.
#ifndef FVV_BLEND_STREAM
#define FVV_BLEND_STREAM 1
#endif
#ifndef FVV_BLEND_WQ_EARLY
#define FVV_BLEND_WQ_EARLY 0  // chroma sources loaded with the luma-row inputs (costs 4 live registers)
#endif
#ifndef FVV_MINB_BLEND_S
#define FVV_MINB_BLEND_S 8  // r2 sweep (cfg4 ms per rig frame): 6 / 7 / 8 / 9 / 10 = 1.091 / 1.031 / 0.992 / 1.032 / 1.069 (k_blend 1.166)
#endif
template <int FMT>
__global__ void __launch_bounds__(128, FVV_MINB_BLEND_S) k_blend_s(Geometry g, PairTable pt, const uint8_t* __restrict__ ws,
                                                   Planes P, int pair_base, bool write_frame,
                                                   double* mask_out /* nullable: (launch pairs, H, W) */) {
    pdl_enter();
    const int W = g.W, H = g.H;
    const int pair = blockIdx.z + pair_base;
    const int ng = (W + 7) / 8;
    const int lane = threadIdx.x & 31;
    const int rr = lane >> 4;                                               // row within the pair
    const int gxr = blockIdx.x * (blockDim.x / 2) + (threadIdx.x >> 5) * 16 + (lane & 15);
    const bool active = gxr < ng;
    const int gx = active ? gxr : ng - 1;                                   // 8-column group
    const int yp = blockIdx.y;                                              // row pair
    const int x0 = gx * 8, n = min(8, W - x0);
    const uint16_t* sd = cplane<uint16_t>(ws, P, P.sd, pair);
    const double* carry = cplane<double>(ws, P, P.carry, pair);
    const float* ol = cplane<float>(ws, P, P.occ_l, pair);
    const float* orr = cplane<float>(ws, P, P.occ_r, pair);
    const uint8_t* wl = cplane<uint8_t>(ws, P, P.wl, pair);
    const uint8_t* wr = cplane<uint8_t>(ws, P, P.wr, pair);
    uint8_t* out = pt.out[pair];
    const int y = 2 * yp + rr;
    const size_t ro = (size_t)y * W;
    const uint16_t* srow = sd + ro;
    // ---- loads ----
    float vl[8], vr[8];
    uint2 pl = make_uint2(0, 0), pr = make_uint2(0, 0);  // warped luma, 8 bytes per side
    if (n == 8) {
        const float4 a = *reinterpret_cast<const float4*>(ol + ro + x0);
        const float4 b = *reinterpret_cast<const float4*>(ol + ro + x0 + 4);
        const float4 c = *reinterpret_cast<const float4*>(orr + ro + x0);
        const float4 d = *reinterpret_cast<const float4*>(orr + ro + x0 + 4);
        vl[0] = a.x; vl[1] = a.y; vl[2] = a.z; vl[3] = a.w; vl[4] = b.x; vl[5] = b.y; vl[6] = b.z; vl[7] = b.w;
        vr[0] = c.x; vr[1] = c.y; vr[2] = c.z; vr[3] = c.w; vr[4] = d.x; vr[5] = d.y; vr[6] = d.z; vr[7] = d.w;
        if (FMT != FVV_RGB8) {  // u8 rows are only 4-byte aligned (W % 4 == 0)
            pl = make_uint2(*reinterpret_cast<const uint32_t*>(wl + ro + x0), *reinterpret_cast<const uint32_t*>(wl + ro + x0 + 4));
            pr = make_uint2(*reinterpret_cast<const uint32_t*>(wr + ro + x0), *reinterpret_cast<const uint32_t*>(wr + ro + x0 + 4));
        }
    } else {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int xx = min(x0 + j, W - 1);
            vl[j] = ol[ro + xx]; vr[j] = orr[ro + xx];
            if (FMT != FVV_RGB8) {
                const int sh = 8 * (j & 3);
                if (j < 4) { pl.x |= (uint32_t)wl[ro + xx] << sh; pr.x |= (uint32_t)wr[ro + xx] << sh; }
                else { pl.y |= (uint32_t)wl[ro + xx] << sh; pr.y |= (uint32_t)wr[ro + xx] << sh; }
            }
        }
    }
    // sd[clamp(x0 - 2 + j)], j = 0..10: sa = (s0, s1), sb = (s2 .. s9), s10
    uint32_t sa;
    uint4 sb;
    int s10;
    if ((W & 7) == 0 && x0 >= 2 && x0 + 8 < W) {
        sa = *reinterpret_cast<const uint32_t*>(srow + x0 - 2);
        sb = *reinterpret_cast<const uint4*>(srow + x0);
        s10 = srow[x0 + 8];
    } else {
        uint32_t t[10];
#pragma unroll
        for (int j = 0; j < 10; j++) t[j] = srow[clampi(x0 - 2 + j, 0, W - 1)];
        sa = t[0] | (t[1] << 16);
        sb = make_uint4(t[2] | (t[3] << 16), t[4] | (t[5] << 16), t[6] | (t[7] << 16), t[8] | (t[9] << 16));
        s10 = srow[clampi(x0 + 8, 0, W - 1)];
    }
    auto sj = [&](int j) -> int {  // j compile time after unrolling
        const uint32_t wv = j < 2 ? sa : (j < 4 ? sb.x : (j < 6 ? sb.y : (j < 8 ? sb.z : sb.w)));
        return j == 10 ? s10 : (int)((j & 1) ? (wv >> 16) : (wv & 0xFFFFu));
    };
    double tmp = carry[(size_t)y * ng + gx];
    // chroma sources of this group's 2x2 blocks (Ul, Ur, Vl, Vr), loaded with the rest
    const int cw = g.cw, chh = g.ch;
    const int cx0 = x0 / 2, nc = n / 2;
    uchar4 wq[4];
    auto load_wq = [&]() {
        if (FMT == FVV_YUV420 && write_frame && active) {
            const uchar4* wc = cplane<uchar4>(ws, P, P.wc, pair) + (size_t)yp * cw + cx0;
            if (nc == 4 && (cw & 3) == 0) {
                const uint4 v = *reinterpret_cast<const uint4*>(wc);
                wq[0] = *reinterpret_cast<const uchar4*>(&v.x); wq[1] = *reinterpret_cast<const uchar4*>(&v.y);
                wq[2] = *reinterpret_cast<const uchar4*>(&v.z); wq[3] = *reinterpret_cast<const uchar4*>(&v.w);
            } else {
#pragma unroll
                for (int j = 0; j < 4; j++) wq[j] = wc[min(j, nc - 1)];
            }
        }
    };
#if FVV_BLEND_WQ_EARLY
    load_wq();
#endif
    // ---- per pixel: replay, mask, blend, stores ----
    uint32_t lo = 0, hi = 0;
    double csum[4];
    double pe = 0.0;
    double* mo = mask_out ? mask_out + (size_t)blockIdx.z * W * H + ro + x0 : nullptr;  // this launch's pair
#pragma unroll
    for (int j = 0; j < 8; j++) {
        if (j > 0) tmp = __dadd_rn(tmp, __dsub_rn(d0_of(sj(j + 3)), d0_of(sj(j))));
        const double m = j < n ? mask_of(tmp, vl[j], vr[j], g) : 0.0;
        if (write_frame && active) {
            if (FMT == FVV_RGB8) {
                if (j < n) {
                    const uint8_t* px = cplane<uint8_t>(ws, P, P.wrgb, pair) + (ro + x0 + j) * 6;
                    uint8_t* o = out + (ro + x0 + j) * 3;
#pragma unroll
                    for (int ch = 0; ch < 3; ch++) o[ch] = blend_px(m, px[ch], px[3 + ch]);
                }
            } else {
                const int sh = 8 * (j & 3);
                const uint32_t a = ((j < 4 ? pl.x : pl.y) >> sh) & 0xFFu, b = ((j < 4 ? pr.x : pr.y) >> sh) & 0xFFu;
                const uint32_t v = (uint32_t)blend_px(m, (int)a, (int)b) << sh;
                if (j < 4) lo |= v; else hi |= v;
            }
        }
        if (mo && active && j < n) mo[j] = m;
        if (FMT == FVV_YUV420) {
            if (j & 1) {
                const double p = __dadd_rn(pe, m);                               // m(2k) + m(2k+1) of this row
                const double o = __shfl_xor_sync(0xffffffffu, p, 16);            // the other row's pair sum
                csum[j >> 1] = rr == 0 ? __dadd_rn(p, o) : __dadd_rn(o, p);      // (a + b) + (c + d)
            } else {
                pe = m;
            }
        }
    }
    if (FMT != FVV_RGB8 && write_frame && active) {
        *reinterpret_cast<uint32_t*>(out + ro + x0) = lo;  // W % 4 == 0: n is 4 or 8
        if (n == 8) *reinterpret_cast<uint32_t*>(out + ro + x0 + 4) = hi;
    }
    // chroma blend with the 2x2-mean mask (warp.py:83-88): upper lanes U, lower lanes V
#if !FVV_BLEND_WQ_EARLY
    load_wq();
#endif
    if (FMT == FVV_YUV420 && write_frame && active) {
        uint8_t* co = out + (size_t)W * H + (size_t)rr * cw * chh + (size_t)yp * cw + cx0;
        uint32_t pk = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const double mc = __dmul_rn(csum[j], 0.25);  // /4 == *0.25 exactly
            const uint8_t v = rr == 0 ? blend_px(mc, wq[j].x, wq[j].y) : blend_px(mc, wq[j].z, wq[j].w);
            pk |= (uint32_t)v << (8 * j);
        }
        if (nc == 4 && (cw & 3) == 0) {
            *reinterpret_cast<uint32_t*>(co) = pk;
        } else {
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (j < nc) co[j] = (uint8_t)(pk >> (8 * j));
        }
    }
}

// ---------------------------------------------------------------------------
// host-side launch helpers (called from api.cu)
// ---------------------------------------------------------------------------
using BlendKernel = void (*)(Geometry, PairTable, const uint8_t*, Planes, int, bool, double*);
static BlendKernel blend_kernel(int fmt) {
#if FVV_BLEND_STREAM
    return fmt == FVV_YUV420 ? k_blend_s<FVV_YUV420> : fmt == FVV_RGB8 ? k_blend_s<FVV_RGB8> : k_blend_s<FVV_GRAY8>;
#else
    return fmt == FVV_YUV420 ? k_blend<FVV_YUV420> : fmt == FVV_RGB8 ? k_blend<FVV_RGB8> : k_blend<FVV_GRAY8>;
#endif
}
// ---------------------------------------------------------------------------
// k_sadw: the 8x8-block search for 8-aligned levels (w % 8 == 0) -- pixel-pair
// packing as k_sadp, restructured so that nearly every issued instruction is
// search arithmetic:
//  * the target window is staged RAW (u16 samples, 16-byte cp.async straight
//    into shared memory, edge replication at chunk granularity); the odd
//    pixel pairs are formed in registers with one PRMT each;
//  * the reference strip is staged once per block as pixel-pair words, with
//    the per-block reference sum accumulated during staging;
//  * sum(max) is accumulated with IDP.2A (lo + hi + acc, fma pipe) so that the
//    alu pipe -- the bound: VIMNMX, PRMT, IADD3 all issue there at half rate --
//    carries only the max and the column sums;
//  * sum(b) per candidate comes from per-thread column sums of the target
//    pair words (SIDE + 6 adds per row instead of 4 * SIDE);
//  * thread = (dy, dx group, block) with the block index fastest: the 8
//    threads of a shared-memory phase read 8 consecutive 16-byte groups of
//    one row (conflict-free by construction), the CTA is 8 x NBY blocks;
//  * winner key = sad << 10 | tie-rule rank (< 2^27), 32-bit smem atomicMin.
// Candidates of one thread: dx + r in [c0, c0 + CG); with more than one group
// CG is even, so every group shares the pair parity of group 0.  Same exact integer SAD as k_sad.
// ---------------------------------------------------------------------------
#ifndef FVV_MINB_SADW
#define FVV_MINB_SADW(side) ((side) > 13 ? FVV_MINB_SADW25 : ((side) > 9 ? 3 : 4))
#endif
#ifndef FVV_MINB_SADW25
#define FVV_MINB_SADW25 2
#endif
#ifdef FVV_DEBUG
#include <cassert>
#define FVV_DBG_ALIGN(p, a) assert((reinterpret_cast<uintptr_t>(p) & ((a) - 1)) == 0)
#else
#define FVV_DBG_ALIGN(p, a) ((void)0)
#endif
template <int SIDE, int CG, int RB_ = 0>
struct SadW {
    static constexpr int R = SIDE / 2;
    static constexpr int NG = (SIDE + CG - 1) / CG;        // dx groups per dy row
#ifndef FVV_SADW_NBY25
#define FVV_SADW_NBY25 0  // > 0: block rows per CTA at 25x25 (default 1: 200 of 224 lanes per dx group busy); r2 sweep NBY 2 (min blocks 1): 1.04 -> 1.12 ms, off
#endif
    static constexpr int NBY = (SIDE == 25 && FVV_SADW_NBY25 > 0) ? FVV_SADW_NBY25
                             : (256 / (8 * SIDE * NG)) > 0 ? 256 / (8 * SIDE * NG) : 1;
    static constexpr int NB = 8 * NBY;                     // blocks per CTA (8 x NBY)
    static constexpr int TPG = ((NB * SIDE + 31) / 32) * 32; // threads per dx group (whole warps)
    static constexpr int THREADS = TPG * NG;
    static constexpr int XPAD = 8 * ((R + 7) / 8);         // left apron, chunk aligned
    static constexpr int NPJ = CG + 6;                     // pair words per row and thread
    static constexpr int LASTW = 4 * 7 + 4 * (((XPAD - R + (NG - 1) * CG + NPJ) / 2) / 4) + 3;  // last word read
    static constexpr int WW = 8 * ((LASTW / 4) + 1) > 64 + 2 * XPAD ? 8 * ((LASTW / 4) + 1)
                                                                    : 64 + 2 * XPAD;  // samples
    static constexpr int TWW = WW / 2;                     // words per window row
    // each thread searches RB blocks stacked vertically (NBY block rows apart):
    // setup, rank table and the window apron are shared by twice the work
#ifndef FVV_SADW_RB5
#define FVV_SADW_RB5 3
#endif
#ifndef FVV_SADW_RB9
#define FVV_SADW_RB9 4
#endif
#ifndef FVV_SADW_RB25
#define FVV_SADW_RB25 4
#endif
    static constexpr int RB = RB_ > 0 ? RB_
                            : (SIDE <= 5 ? FVV_SADW_RB5 : (SIDE <= 9 ? FVV_SADW_RB9 : (SIDE == 25 ? FVV_SADW_RB25 : 1)));
    static constexpr int NBYT = NBY * RB;                  // block rows per CTA
    static constexpr int WH = 8 * NBYT + 2 * R;            // window rows
    // + 8: the window's TMA mbarrier (between the reference sums and the ranks, 8-aligned)
    static constexpr size_t SMEM = (size_t)WH * TWW * 4 + (size_t)8 * NBYT * 32 * 4 +
                                   (size_t)NB * RB * 8 + 8 + (size_t)SIDE * SIDE * 2;
};

// The target window arrives by one TMA tile copy per CTA (FVV_SADW_TMA): box
// WW x WH samples of the level's u16 target plane, viewed as a 3-D tensor
// (x, y, pair slot) whose pair stride is the workspace slot stride, so one map
// per (level, direction) serves every pair of the launch.  TMA zero-fills
// outside the plane; CTAs on the frame edge then overwrite those samples with
// the replicated edge (the window is clamp-indexed, flow.py:57-91 via
// _kernels.py's edge padding).  FVV_SADW_TMA=0 keeps the per-thread cp.async
// staging for A/B timing.
#ifndef FVV_SADW_TMA
#define FVV_SADW_TMA 1
#endif
__device__ __forceinline__ void sadw_mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void sadw_tma_window(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                                int z, uint32_t bytes) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
        "l"(map), "r"(x), "r"(y), "r"(z), "r"(b)
        : "memory");
}
__device__ __forceinline__ void sadw_mbar_wait0(uint64_t* bar) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SADW_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        "@!p bra SADW_WAIT_%=;\n"
        "}\n" ::"r"(a)
        : "memory");
}

struct SadWLaunch {
    int bx_end;                  // full 8-wide block columns (w / 8)
    const int16_t* rank_of;
    const int16_t* cand_of_rank;
};

template <int LEVEL>
__device__ __forceinline__ const uint16_t* sadw_tgt(const Geometry& g, const PairTable& pt, uint8_t* ws,
                                                    const Planes& P, int pair, int d) {
    return LEVEL == 0 ? cplane<uint16_t>(ws, P, P.q0[1 - d], pair)
         : LEVEL == 1 ? cplane<uint16_t>(ws, P, P.tq1[d], pair)
                      : cplane<uint16_t>(ws, P, P.tq2[d], pair);
}

// Full 16-byte shared load, never narrowed: a quarter-warp phase (8 blocks of
// one block row) then reads 8 distinct 16-byte bank groups.  Narrowed 32-bit
// loads would put the 4 block rows of a warp on the same banks.
__device__ __forceinline__ uint4 lds128(const uint32_t* p) {
    uint4 v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// One thread's search: dx + r in [G*CG, G*CG + CG), every row of its block.
// Word offsets are compile time, so the window reads are aligned LDS.128.
template <int SIDE, int CG, int G>
__device__ __forceinline__ uint32_t sadw_group(const uint32_t* Rb, const uint32_t* Tb, int rows, int sa,
                                               const int16_t* rki) {
    using S = SadW<SIDE, CG>;
    constexpr int base = S::XPAD - S::R + G * CG;          // window sample of pair 0
    constexpr int ch0 = (base / 2) / 4, ch1 = ((base + S::NPJ) / 2) / 4;
    constexpr int JF = (2 * S::NPJ) / 3;   // alu : fma balance of the inner loop
    uint32_t am[CG], cs[S::NPJ];
#pragma unroll
    for (int c = 0; c < CG; c++) am[c] = 0;
#pragma unroll
    for (int j = 0; j < S::NPJ; j++) cs[j] = 0;
#pragma unroll 2
    for (int yy = 0; yy < rows; yy++) {
        uint32_t wv[4 * (ch1 - ch0 + 1)];
#pragma unroll
        for (int q = ch0; q <= ch1; q++) {
            FVV_DBG_ALIGN(Tb + yy * S::TWW + 4 * q, 16);
            const uint4 t4 = lds128(Tb + yy * S::TWW + 4 * q);
            wv[4 * (q - ch0)] = t4.x; wv[4 * (q - ch0) + 1] = t4.y;
            wv[4 * (q - ch0) + 2] = t4.z; wv[4 * (q - ch0) + 3] = t4.w;
        }
        FVV_DBG_ALIGN(Rb + yy * 32, 16);
        const uint4 r4 = lds128(Rb + yy * 32);
        const uint32_t rv[4] = {r4.x, r4.y, r4.z, r4.w};
        uint32_t pv[S::NPJ];
#pragma unroll
        for (int j = 0; j < S::NPJ; j++) {
            const int sidx = base + j;                           // compile time
            const int wi = sidx / 2 - 4 * ch0;
            pv[j] = (sidx & 1) ? __byte_perm(wv[wi], wv[wi + 1], 0x5432) : wv[wi];
            // pipe balance: the first JF column sums go to the fma pipe as lo + hi
            // (IDP), the rest stay packed on the alu pipe (one IADD3 per two rows)
            if (j < JF) cs[j] = __dp2a_lo(pv[j], 0x0101u, cs[j]);
            else cs[j] += pv[j];
        }
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int c = 0; c < CG; c++) am[c] = __dp2a_lo(__vmaxu2(pv[2 * k + c], rv[k]), 0x0101u, am[c]);
    }
    uint32_t mine = 0xFFFFFFFFu;
#pragma unroll
    for (int c = 0; c < CG; c++) {
        const int cc = G * CG + c;
        if (cc < SIDE) {
            int ab = 0;  // sum of the target samples of candidate c
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const int j = c + 2 * k;
                ab += j < JF ? (int)cs[j] : (int)((cs[j] & 0xFFFFu) + (cs[j] >> 16));
            }
            const int sad = 2 * (int)am[c] - ab - sa;
            mine = min(mine, ((uint32_t)sad << 10) | (uint32_t)rki[cc]);
        }
    }
    return mine;
}

template <int LEVEL, int SIDE, int CG, int RB_>
__global__ void __launch_bounds__(SadW<SIDE, CG, RB_>::THREADS, FVV_MINB_SADW(SIDE))
k_sadw(Geometry g, PairTable pt, uint8_t* __restrict__ ws, Planes P, SadWLaunch sl,
       const __grid_constant__ CUtensorMap tmw0, const __grid_constant__ CUtensorMap tmw1) {
    pdl_enter();
    using S = SadW<SIDE, CG, RB_>;
    extern __shared__ __align__(128) uint8_t sadw_smem[];          // TMA destination: 128-byte aligned
    uint32_t* Ts = reinterpret_cast<uint32_t*>(sadw_smem);         // WH x TWW raw words
    uint32_t* Rs = Ts + S::WH * S::TWW;                            // 8*NBYT x 32 pair words
    uint32_t* best = Rs + 8 * S::NBYT * 32;                        // NB*RB keys
    int* suma = reinterpret_cast<int*>(best + S::NB * S::RB);      // NB*RB reference sums
    uint64_t* wbar = reinterpret_cast<uint64_t*>(suma + S::NB * S::RB);  // window TMA barrier
    int16_t* rk = reinterpret_cast<int16_t*>(wbar + 1);            // SIDE^2 ranks

    const Level& L = g.lv[LEVEL];
    const int w = L.w, h = L.h;
    const int pair = blockIdx.z >> 1, d = blockIdx.z & 1;
    const int bx0 = blockIdx.x * 8, by0 = blockIdx.y * S::NBYT;
    const int tid = threadIdx.x;

    // ---- stage: target window (raw u16, edge replicated) -------------------
    const uint16_t* tg = sadw_tgt<LEVEL>(g, pt, ws, P, pair, d);
    const int xa = bx0 * 8 - S::XPAD, ya = by0 * 8 - S::R;
    constexpr int NCH = S::WW / 8;                                  // 16-byte chunks per row
    static_assert(NCH <= 16, "two window rows per warp pass");
#if FVV_SADW_TMA
    static_assert(S::WW <= 256 && S::WH <= 256, "TMA box dimensions");
    (void)tg;
    if (tid == 0) {
        sadw_mbar_init(wbar);
        sadw_tma_window(Ts, d ? &tmw1 : &tmw0, wbar, xa, ya, pair, (uint32_t)(S::WH * S::TWW * 4));
    }
#else
    (void)tmw0; (void)tmw1;
    {
        const int lane = tid & 31, q = lane & 15;                   // chunk of this lane
        const int gx = xa + 8 * q;
        const bool inside = gx >= 0 && gx + 8 <= w;
        const int cx = gx < 0 ? 0 : w - 1;                           // replicated edge column
        if (q < NCH) {
            for (int t = 2 * (tid >> 5) + (lane >> 4); t < S::WH; t += 2 * (S::THREADS / 32)) {
                const uint16_t* row = tg + (size_t)clampi(ya + t, 0, h - 1) * w;
                uint32_t* dst = Ts + t * S::TWW + 4 * q;
                if (inside) {
                    FVV_DBG_ALIGN(dst, 16); FVV_DBG_ALIGN(row + gx, 16);
                    cp_async16(dst, row + gx);
                } else {
                    const uint32_t v = row[cx];
                    const uint32_t vv = v | (v << 16);
                    *reinterpret_cast<uint4*>(dst) = make_uint4(vv, vv, vv, vv);
                }
            }
        }
    }
    cp_async_commit();
#endif
    // ---- stage: reference strip as pixel-pair words + per-block sums -------
    for (int i = tid; i < S::NB * S::RB; i += S::THREADS) { best[i] = 0xFFFFFFFFu; suma[i] = 0; }
    for (int i = tid; i < SIDE * SIDE; i += S::THREADS) rk[i] = sl.rank_of[i];
    __syncthreads();
    const uint8_t* yp = LEVEL != 2 ? nullptr
                      : g.fmt == FVV_RGB8 ? cplane<uint8_t>(ws, P, P.luma[d], pair)
                                          : (d ? pt.right[pair] : pt.left[pair]);
    const bool yal = (reinterpret_cast<uintptr_t>(yp) & 7) == 0;  // w % 8 == 0: every row 8-aligned
    for (int i = tid; i < 8 * S::NBYT * 8; i += S::THREADS) {      // (row, block column)
        const int kx = i & 7, yy = i >> 3;
        const int gy = by0 * 8 + yy, gx = (bx0 + kx) * 8;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (gy < h && gx < w) {
            const size_t o = (size_t)gy * w + gx;
            if (LEVEL == 2) {
                uint2 b;
                if (yal) {
                    b = *reinterpret_cast<const uint2*>(yp + o);
                } else {
                    b.x = yp[o] | (yp[o + 1] << 8) | (yp[o + 2] << 16) | ((uint32_t)yp[o + 3] << 24);
                    b.y = yp[o + 4] | (yp[o + 5] << 8) | (yp[o + 6] << 16) | ((uint32_t)yp[o + 7] << 24);
                }
                v.x = __byte_perm(b.x, 0, 0x4140) << 3; v.y = __byte_perm(b.x, 0, 0x4342) << 3;
                v.z = __byte_perm(b.y, 0, 0x4140) << 3; v.w = __byte_perm(b.y, 0, 0x4342) << 3;
            } else {
                const uint16_t* rp = LEVEL == 0 ? cplane<uint16_t>(ws, P, P.q0[d], pair)
                                                : cplane<uint16_t>(ws, P, P.s4[d], pair);
                FVV_DBG_ALIGN(rp + o, 16);
                v = *reinterpret_cast<const uint4*>(rp + o);
                if (LEVEL == 1) { v.x <<= 1; v.y <<= 1; v.z <<= 1; v.w <<= 1; }  // 2 * s4 <= 2040
            }
            const uint32_t ps = v.x + v.y + v.z + v.w;                // lanes <= 4 * 2040
            atomicAdd(&suma[(yy >> 3) * 8 + kx], (int)((ps & 0xFFFFu) + (ps >> 16)));
        }
        FVV_DBG_ALIGN(Rs + yy * 32 + 4 * kx, 16);
        *reinterpret_cast<uint4*>(Rs + yy * 32 + 4 * kx) = v;
    }
#if FVV_SADW_TMA
    sadw_mbar_wait0(wbar);
    if (xa < 0 || xa + S::WW > w || ya < 0 || ya + S::WH > h) {  // CTA-uniform: frame-edge windows
        // columns: whole 16-byte chunks lie outside the plane (xa, w multiples of 8);
        // they take the row's edge sample (row 0 / h-1 rows are fixed up next)
        const uint16_t* Th = reinterpret_cast<const uint16_t*>(Ts);
        for (int i = tid; i < S::WH * NCH; i += S::THREADS) {
            const int t = i / NCH, q = i - t * NCH, gx = xa + 8 * q;
            if (gx < 0 || gx + 8 > w) {
                const uint32_t v = Th[t * S::WW + (gx < 0 ? -xa : w - 1 - xa)];
                const uint32_t vv = v | (v << 16);
                *reinterpret_cast<uint4*>(Ts + t * S::TWW + 4 * q) = make_uint4(vv, vv, vv, vv);
            }
        }
        __syncthreads();
        // rows outside the plane: copies of row 0 / h-1 (both inside the window)
        for (int i = tid; i < S::WH * NCH; i += S::THREADS) {
            const int t = i / NCH, q = i - t * NCH, gy = ya + t;
            if (gy < 0 || gy > h - 1) {
                const int ts = (gy < 0 ? 0 : h - 1) - ya;
                *reinterpret_cast<uint4*>(Ts + t * S::TWW + 4 * q) =
                    *reinterpret_cast<const uint4*>(Ts + ts * S::TWW + 4 * q);
            }
        }
    }
#else
    cp_async_wait_0();
#endif
    __syncthreads();

    // ---- search ---------------------------------------------------------------
    const int gq = tid / S::TPG, rest = tid - gq * S::TPG;      // dx group is warp-uniform
    const int kb = rest % S::NB, iy = rest / S::NB;
    const int kx = kb & 7, ky = kb >> 3;
#pragma unroll 1
    for (int rb = 0; rb < S::RB; rb++) {
        const int kyr = ky + rb * S::NBY, kbr = kb + rb * S::NB;    // block row / slot of this pass
        const bool active = iy < SIDE && bx0 + kx < sl.bx_end && by0 + kyr < L.nby;
        if (active) {
            const int rows = min(8, h - (by0 + kyr) * 8);
            const uint32_t* Rb = Rs + (kyr * 8) * 32 + 4 * kx;
            const uint32_t* Tb = Ts + (kyr * 8 + iy) * S::TWW + 4 * kx;
            const int sa = suma[kbr];
            const int16_t* rki = rk + iy * SIDE;
            uint32_t mine;
            if (S::NG == 1 || gq == 0) mine = sadw_group<SIDE, CG, 0>(Rb, Tb, rows, sa, rki);
            else mine = sadw_group<SIDE, CG, (S::NG > 1 ? 1 : 0)>(Rb, Tb, rows, sa, rki);
            atomicMin(&best[kbr], mine);
        }
    }
    __syncthreads();
    for (int i = tid; i < S::NB * S::RB; i += S::THREADS) {
        const int hx = bx0 + (i & 7), hy = by0 + (i >> 3);
        if (hx < sl.bx_end && hy < L.nby) {
            const uint32_t key = best[i];
            const int idx = sl.cand_of_rank[key & 1023u];
            BlockHit hit;
            hit.dy = (int16_t)(idx / SIDE - S::R);
            hit.dx = (int16_t)(idx % SIDE - S::R);
            hit.sad = (int32_t)(key >> 10);
            plane<BlockHit>(ws, P, P.hit[LEVEL][d], pair)[hy * L.nbx + hx] = hit;
        }
    }
}

// host: the (x, y, pair slot) u16 view of one target plane for the window copies
static PFN_cuTensorMapEncodeTiled_v12000 sadw_encode_fn() {
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
static bool sadw_window_map(CUtensorMap* m, const void* base, int w, int h, int npairs, size_t pair_stride, int bw,
                            int bh) {
    auto fn = sadw_encode_fn();
    if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || (pair_stride & 15) || ((size_t)w * 2) % 16) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)std::max(npairs, 1)};
    const cuuint64_t strides[2] = {(cuuint64_t)w * 2, (cuuint64_t)pair_stride};
    const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int LEVEL, int SIDE, int CG, int RB_>
static cudaError_t launch_sadw_rb(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                                  SadWLaunch sl, int npairs, cudaStream_t st) {
    using S = SadW<SIDE, CG, RB_>;
    const Level& L = g.lv[LEVEL];
    auto kern = k_sadw<LEVEL, SIDE, CG, RB_>;
    if (S::SMEM > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((sl.bx_end + 7) / 8, (L.nby + S::NBYT - 1) / S::NBYT, 2 * npairs);
    CUtensorMap tm[2];
    memset(tm, 0, sizeof(tm));
#if FVV_SADW_TMA
    for (int d = 0; d < 2; d++) {
        const size_t off = LEVEL == 0 ? P.q0[1 - d] : LEVEL == 1 ? P.tq1[d] : P.tq2[d];
        if (!sadw_window_map(&tm[d], ws + off, L.w, L.h, npairs, P.stride, S::WW, S::WH))
            return cudaErrorInvalidValue;
    }
#endif
    cudaError_t le = launch_k(g.pdl, kern, grid, dim3(S::THREADS), S::SMEM, st, g, pt, ws, P, sl, tm[0], tm[1]);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

// Stacked blocks per thread (RB) trade parallelism for amortised setup: small
// launches (fewer than two CTAs per SM with stacking) take RB = 1.
template <int LEVEL, int SIDE, int CG>
static cudaError_t launch_sadw(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                               SadWLaunch sl, int npairs, cudaStream_t st) {
    using S = SadW<SIDE, CG>;
    const Level& L = g.lv[LEVEL];
    const long ctas = (long)((sl.bx_end + 7) / 8) * ((L.nby + S::NBYT - 1) / S::NBYT) * 2 * npairs;
    if (S::RB > 1 && ctas < g.sadw_rb_min_ctas) return launch_sadw_rb<LEVEL, SIDE, CG, 1>(g, pt, ws, P, sl, npairs, st);
    return launch_sadw_rb<LEVEL, SIDE, CG, S::RB>(g, pt, ws, P, sl, npairs, st);
}

template <int LEVEL, int KP, bool FULL8>
static cudaError_t launch_sad_kp(const Geometry& g, const PairTable& pt, uint8_t* ws,
                                 const Planes& P, SadLaunch sl, int npairs, cudaStream_t st) {
    const Level& L = g.lv[LEVEL];
    const int side = 2 * L.r + 1;
    const int nbx = sl.bx_end - sl.bx_begin;
    if (nbx <= 0) return cudaSuccess;
    const int threads_needed = sl.nbx_cta * side * sl.groups;
    const int threads = ((threads_needed + 31) / 32) * 32;
    const int RW = sl.nbx_cta * L.block, PW = sl.pw, PH = L.block + 2 * L.r;
    size_t smem = (size_t)L.block * RW * 4 + (size_t)PH * PW * 4;
    smem = (smem + 7) & ~(size_t)7;
    smem += (size_t)sl.nbx_cta * 8 + (size_t)sl.nbx_cta * 4 + (size_t)side * side * 2 + 16;
    auto kern = k_sad<LEVEL, KP, FULL8>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((nbx + sl.nbx_cta - 1) / sl.nbx_cta, L.nby, 2 * npairs);
    cudaError_t le = launch_k(g.pdl, kern, grid, dim3(threads), smem, st, g, pt, ws, P, sl);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

template <int LEVEL, bool FULL8>
static cudaError_t launch_sad_level(const Geometry& g, const PairTable& pt, uint8_t* ws,
                                    const Planes& P, SadLaunch sl, int kp, int npairs,
                                    cudaStream_t st) {
    switch (kp) {
        case 3: return launch_sad_kp<LEVEL, 3, FULL8>(g, pt, ws, P, sl, npairs, st);
        case 5: return launch_sad_kp<LEVEL, 5, FULL8>(g, pt, ws, P, sl, npairs, st);
        case 7: return launch_sad_kp<LEVEL, 7, FULL8>(g, pt, ws, P, sl, npairs, st);
        case 9: return launch_sad_kp<LEVEL, 9, FULL8>(g, pt, ws, P, sl, npairs, st);
        case 13: return launch_sad_kp<LEVEL, 13, FULL8>(g, pt, ws, P, sl, npairs, st);
        default: return launch_sad_kp<LEVEL, 16, FULL8>(g, pt, ws, P, sl, npairs, st);
    }
}

// Choose KP (candidate pairs per thread) and G (threads per dy row).
static void pick_kp(int side, int* kp, int* groups) {
    static const int opts[] = {3, 5, 7, 9, 13, 16};
    const int need = (side + 1) / 2;  // candidate pairs per dy row
    int best_kp = 16, best_g = (need + 15) / 16, best_waste = 1 << 30;
    for (int o : opts) {
        int gcount = (need + o - 1) / o;
        int waste = gcount * o - need;
        if (waste < best_waste || (waste == best_waste && gcount < best_g)) {
            best_waste = waste; best_kp = o; best_g = gcount;
        }
    }
    *kp = best_kp;
    *groups = best_g;
}

template <int LEVEL, int KP>
static cudaError_t launch_sad8_kp(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                                  Sad8Launch sl, int npairs, cudaStream_t st) {
    const Level& L = g.lv[LEVEL];
    const int side = 2 * L.r + 1;
    const int ncols = sl.bx_end - sl.bx_begin;
    if (ncols <= 0) return cudaSuccess;
    const int threads = ((sl.nbx * sl.nby * side + 31) / 32) * 32;
    const int RW = sl.nbx * 8, RH = sl.nby * 8, PH = RH + 2 * L.r;
    size_t smem = (size_t)(RH * RW + PH * sl.pw) * 4 + (size_t)PH * sl.tw * 2;
    smem = (smem + 15) & ~(size_t)15;
    smem += (size_t)sl.nbx * sl.nby * 12 + (size_t)side * side * 2 + 16;
    auto kern = k_sad8<LEVEL, KP>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    dim3 grid((ncols + sl.nbx - 1) / sl.nbx, (L.nby + sl.nby - 1) / sl.nby, 2 * npairs);
    cudaError_t le = launch_k(g.pdl, kern, grid, dim3(threads), smem, st, g, pt, ws, P, sl);
    if (le != cudaSuccess) return le;
    return cudaGetLastError();
}

template <int LEVEL>
static cudaError_t run_sad(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                           const int16_t* rank_of, const int16_t* cand_of_rank, int npairs,
                           cudaStream_t st) {
    const Level& L = g.lv[LEVEL];
    const int side = 2 * L.r + 1;
    int kp, groups;
    pick_kp(side, &kp, &groups);
    const bool fast = L.block == 8;
    const int full_cols = fast ? L.w / 8 : 0;  // block columns with 8 valid columns
    cudaError_t e;
    // pixel-pair packing wins for small candidate rows; at 2r+1 = 25 its 50
    // accumulators cost occupancy, and the candidate-pair kernel is faster
    const bool pix = full_cols > 0 && (side == 3 || side == 5 || side == 9 || side == 13 ||
                                       side == 17);
    if (fast && (L.w & 7) == 0 && (side == 3 || side == 5 || side == 9 || side == 13 || side == 17 ||
                                   side == 25)) {
        SadWLaunch sw;
        sw.bx_end = full_cols;
        sw.rank_of = rank_of;
        sw.cand_of_rank = cand_of_rank;
        switch (side) {
            case 3: return launch_sadw<LEVEL, 3, 3>(g, pt, ws, P, sw, npairs, st);
            case 5: return launch_sadw<LEVEL, 5, 5>(g, pt, ws, P, sw, npairs, st);
            case 9: return launch_sadw<LEVEL, 9, 9>(g, pt, ws, P, sw, npairs, st);
            case 13: return launch_sadw<LEVEL, 13, 13>(g, pt, ws, P, sw, npairs, st);
            case 17: return launch_sadw<LEVEL, 17, 17>(g, pt, ws, P, sw, npairs, st);
            default: return launch_sadw<LEVEL, 25, 13>(g, pt, ws, P, sw, npairs, st);
        }
    }
    if (pix) {
        SadPLaunch sp;
        sp.rank_of = rank_of;
        sp.cand_of_rank = cand_of_rank;
        sp.bx_begin = 0;
        sp.bx_end = full_cols;
        int nbx = 256 / side;
        if (nbx > 32) nbx = 32;
        int nby = 1;
        if (L.r <= 6) { nby = nbx >= 24 ? 3 : (nbx >= 16 ? 2 : 1); nbx /= nby; }
        sp.nbx = nbx;
        sp.nby = nby;
        const int need = 8 * (nbx - 1) + ((side + 6 + 3) / 4) * 4;
        int pw = std::max(8 * nbx + 2 * L.r, need);
        while (pw % 8 != 4) pw++;
        sp.pw = pw;
        sp.tw = pw + 1;
        const int threads = ((nbx * nby * side + 31) / 32) * 32;
        const int RW = nbx * 4, RH = nby * 8, PH = RH + 2 * L.r;
        size_t smem = (size_t)(RH * RW + PH * pw) * 4 + (size_t)PH * sp.tw * 2;
        smem = (smem + 15) & ~(size_t)15;
        smem += (size_t)nbx * nby * 12 + (size_t)side * side * 2 + 16;
        dim3 grid((full_cols + nbx - 1) / nbx, (L.nby + nby - 1) / nby, 2 * npairs);
        auto go = [&](auto kern) -> cudaError_t {
            if (smem > 48 * 1024) {
                cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e2 != cudaSuccess) return e2;
            }
            cudaError_t le = launch_k(g.pdl, kern, grid, dim3(threads), smem, st, g, pt, ws, P, sp);
            return le != cudaSuccess ? le : cudaGetLastError();
        };
        switch (side) {
            case 3: e = go(k_sadp<LEVEL, 3>); break;
            case 5: e = go(k_sadp<LEVEL, 5>); break;
            case 9: e = go(k_sadp<LEVEL, 9>); break;
            case 13: e = go(k_sadp<LEVEL, 13>); break;
            default: e = go(k_sadp<LEVEL, 17>); break;
        }
        if (e != cudaSuccess) return e;
    } else if (full_cols > 0 && groups == 1) {
        // k_sad8: CTA = nby x nbx blocks, one thread per (block, dy)
        Sad8Launch s8;
        s8.rank_of = rank_of;
        s8.cand_of_rank = cand_of_rank;
        s8.bx_begin = 0;
        s8.bx_end = full_cols;
        const int per_block = side;
        int nbx = 256 / per_block;                        // blocks per CTA
        if (nbx > 32) nbx = 32;
        int nby = 1;
        if (L.r <= 6) { nby = nbx >= 24 ? 3 : (nbx >= 16 ? 2 : 1); nbx /= nby; }
        s8.nbx = nbx;
        s8.nby = nby;
        const int need = 8 * (nbx - 1) + ((2 * kp + 6 + 3) / 4) * 4;  // words read by the last block
        int pw = std::max(8 * nbx + 2 * L.r, need);
        while (pw % 8 != 4) pw++;
        s8.pw = pw;
        s8.tw = pw + 1;
        e = [&]() -> cudaError_t {
            switch (kp) {
                case 3: return launch_sad8_kp<LEVEL, 3>(g, pt, ws, P, s8, npairs, st);
                case 5: return launch_sad8_kp<LEVEL, 5>(g, pt, ws, P, s8, npairs, st);
                case 7: return launch_sad8_kp<LEVEL, 7>(g, pt, ws, P, s8, npairs, st);
                case 9: return launch_sad8_kp<LEVEL, 9>(g, pt, ws, P, s8, npairs, st);
                case 13: return launch_sad8_kp<LEVEL, 13>(g, pt, ws, P, s8, npairs, st);
                default: return launch_sad8_kp<LEVEL, 16>(g, pt, ws, P, s8, npairs, st);
            }
        }();
        if (e != cudaSuccess) return e;
    }
    SadLaunch sl;
    sl.groups = groups;
    sl.rank_of = rank_of;
    sl.cand_of_rank = cand_of_rank;
    int per_block = side * groups;
    sl.nbx_cta = per_block >= 256 ? 1 : (256 / per_block < 32 ? 256 / per_block : 32);
    // every thread reads pair columns [kb*B + dxo, kb*B + dxo + 2*KP + 6)
    sl.pw = sl.nbx_cta * L.block + std::max(2 * L.r + 1, 2 * kp * groups + 6) + 1;
    if ((sl.pw & 1) == 0) sl.pw += 1;  // odd pitch: dy rows fall in distinct banks
    // full block columns take the FULL8 path (it guards ragged rows itself);
    // a ragged last block column or other block sizes take the general path
    if (full_cols > 0 && groups != 1 && !pix) {
        sl.bx_begin = 0;
        sl.bx_end = full_cols;
        e = launch_sad_level<LEVEL, true>(g, pt, ws, P, sl, kp, npairs, st);
        if (e != cudaSuccess) return e;
    }
    if (full_cols < L.nbx) {
        sl.bx_begin = full_cols;
        sl.bx_end = L.nbx;
        e = launch_sad_level<LEVEL, false>(g, pt, ws, P, sl, kp, npairs, st);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

thread_local int g_failed_class = -1;

cudaError_t run_interp_stage(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P,
                             const int16_t* const* rank_of, const int16_t* const* cand_of_rank,
                             int npairs, double* mask_out, Prof* prof, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    // FVV_SYNC_CHECK=1: synchronise after every kernel class and report the
    // class that faulted (debugging aid; off by default, never in a graph)
    static const bool sync_check = getenv("FVV_SYNC_CHECK") && *getenv("FVV_SYNC_CHECK") == '1';
    int cur = -1;
    auto B = [&](int c) { cur = c; if (prof) prof->begin(c, st); };
    auto E = [&]() {
        if (prof) prof->end(st);
        cudaError_t ce = cudaGetLastError();
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (ce == cudaSuccess && sync_check && cudaStreamIsCapturing(st, &cap) == cudaSuccess &&
            cap == cudaStreamCaptureStatusNone)
            ce = cudaStreamSynchronize(st);
        if (ce != cudaSuccess) g_failed_class = cur;
        return ce;
    };

    B(KC_PYRAMID);
    e = launch_k(g.pdl, k_pyramid, dim3((g.lv[0].w + 31) / 32, (g.lv[0].h + 7) / 8, 2 * npairs), dim3(32, 8),
                 0, st, g, pt, ws, P);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_SAD0);
    e = run_sad<0>(g, pt, ws, P, rank_of[0], cand_of_rank[0], npairs, st);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_FLOW0);
    e = launch_k(g.pdl, k_flow<0>, dim3((g.lv[0].w + kFW - 1) / kFW, (g.lv[0].h + kFH - 1) / kFH, 2 * npairs),
                 dim3(256), 0, st, g, ws, P);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_WARPQ1);
    e = launch_k(g.pdl, k_warpq<1>, dim3((g.lv[1].w + kQW - 1) / kQW, (g.lv[1].h + kQH - 1) / kQH, 2 * npairs),
                 dim3(256), 0, st, g, pt, ws, P);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_SAD1);
    e = run_sad<1>(g, pt, ws, P, rank_of[1], cand_of_rank[1], npairs, st);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_FLOW1);
    e = launch_k(g.pdl, k_flow<1>, dim3((g.lv[1].w + kFW - 1) / kFW, (g.lv[1].h + kFH - 1) / kFH, 2 * npairs),
                 dim3(256), 0, st, g, ws, P);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_WARPQ2);
    e = launch_k(g.pdl, k_warpq<2>, dim3((g.lv[2].w + kQW - 1) / kQW, (g.lv[2].h + kQH - 1) / kQH, 2 * npairs),
                 dim3(256), 0, st, g, pt, ws, P);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_SAD2);
    e = run_sad<2>(g, pt, ws, P, rank_of[2], cand_of_rank[2], npairs, st);
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_MASK_PROD);
    {
        const bool two = g.fmt != FVV_RGB8 && g.mask_cols2;
        const int cols = two ? kM2Own * kM2Warps : kMW * kMWarps;
        const long big = (long)((g.W + cols - 1) / cols) * ((g.H + FVV_KMH_BIG - 1) / FVV_KMH_BIG) * npairs;
        Geometry gm = g;
        gm.mh = big >= FVV_MASK_BIG_CTAS ? FVV_KMH_BIG : kMH;
        const dim3 grd((g.W + cols - 1) / cols, (g.H + gm.mh - 1) / gm.mh, npairs);
        if (two)
            e = launch_k(g.pdl, g.fmt == FVV_YUV420 ? k_mask_cols2<FVV_YUV420> : k_mask_cols2<FVV_GRAY8>, grd,
                         dim3(kM2Warps * 32), 0, st, gm, pt, ws, P);
        else
            e = launch_k(g.pdl, g.fmt == FVV_YUV420 ? k_mask_cols<FVV_YUV420>
                                : g.fmt == FVV_RGB8 ? k_mask_cols<FVV_RGB8> : k_mask_cols<FVV_GRAY8>,
                         grd, dim3(kMWarps * 32), 0, st, gm, pt, ws, P);
    }
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;

    B(KC_SCAN);
    {
        // cooperative row staging pays once the launch has several warps per SM;
        // below that the per-warp critical path (its index math) dominates
        const dim3 grid((g.H + kCR - 1) / kCR, npairs);
        e = launch_k(g.pdl, (int)(grid.x * grid.y) >= g.scan_coop_min ? k_scan_carry<true> : k_scan_carry<false>,
                     grid, dim3(kCR), 0, st, g, ws, P);
    }
    if (e != cudaSuccess || (e = E()) != cudaSuccess) return e;
    B(KC_BLEND);
    {
        const dim3 grd(((g.W + 7) / 8 + 63) / 64, g.H / 2, npairs);
        e = launch_k(g.pdl, blend_kernel(g.fmt), grd, dim3(128), 0, st, g, pt, ws, P, 0, true, mask_out);
    }
    if (e != cudaSuccess) return e;
    return E();
}

// diagnostics: final flows (InterpDiagnostics.scales[-1].flow_lr/rl) and mask
__global__ void k_diag_flow(Geometry g, const uint8_t* __restrict__ ws, Planes P, int pair,
                            float2* flow_lr, float2* flow_rl) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.z;
    if (i >= g.W * g.H) return;
    float2* out = d ? flow_rl : flow_lr;
    if (!out) return;
    const int y = i / g.W, x = i - (i / g.W) * g.W;
    const Level L1 = g.lv[1], L2 = g.lv[2];
    const int2 base = up2_fixed(cplane<int2>(ws, P, P.flow1[d], pair), L1.h, L1.w, y, x);
    const int2 res = b2p_fixed(cplane<BlockHit>(ws, P, P.hit[2][d], pair), L2.nby, L2.nbx, L2.block,
                               y, x);
    const int bs = g.fb[2] - (g.fb[1] + 3), rs = g.fb[2] - g.rb[2];
    const float sc = 1.0f / (float)(1 << g.fb[2]);  // exact: values < 2^24 units
    out[i] = make_float2((float)((base.x << bs) + (res.x << rs)) * sc,
                         (float)((base.y << bs) + (res.y << rs)) * sc);
}

// per-level diagnostics (InterpDiagnostics.scales[s], interp.py:49-56, 114-128):
// the level's flows (f32, exact from the fixed point) and the match-error maps
// _block_to_pixel(best_sad / (area * 8)) in the reference's literal f64.
template <int LEVEL>
__global__ void k_diag_level(Geometry g, const uint8_t* __restrict__ ws, Planes P, int pair,
                             float2* flow_lr, float2* flow_rl, double* err_lr, double* err_rl) {
    const Level L = g.lv[LEVEL];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.z;
    if (i >= L.w * L.h) return;
    const int y = i / L.w, x = i - (i / L.w) * L.w;
    const BlockHit* hit = cplane<BlockHit>(ws, P, P.hit[LEVEL][d], pair);
    float2* fo = d ? flow_rl : flow_lr;
    if (fo) {
        int2 f;
        if (LEVEL == 2) {
            const Level L1 = g.lv[1];
            const int2 base = up2_fixed(cplane<int2>(ws, P, P.flow1[d], pair), L1.h, L1.w, y, x);
            const int2 res = b2p_fixed(hit, L.nby, L.nbx, L.block, y, x);
            const int bs = g.fb[2] - (g.fb[1] + 3), rs = g.fb[2] - g.rb[2];
            f = make_int2((base.x << bs) + (res.x << rs), (base.y << bs) + (res.y << rs));
        } else {
            f = cplane<int2>(ws, P, LEVEL == 0 ? P.flow0[d] : P.flow1[d], pair)[i];
        }
        const float sc = 1.0f / (float)(1 << g.fb[LEVEL]);
        fo[i] = make_float2((float)f.x * sc, (float)f.y * sc);
    }
    double* eo = d ? err_rl : err_lr;
    if (eo) {
        auto err_of = [&](int by, int bx) {
            const int rows = min(by * L.block + L.block, L.h) - by * L.block;
            const int cols = min(bx * L.block + L.block, L.w) - bx * L.block;
            const double area8 = __dmul_rn((double)((long long)rows * cols), 8.0);
            return __ddiv_rn((double)hit[by * L.nbx + bx].sad, area8);
        };
        const double c = (double)(L.block - 1) / 2.0;
        const double sy = __ddiv_rn(__dsub_rn((double)y, c), (double)L.block);
        const double sx = __ddiv_rn(__dsub_rn((double)x, c), (double)L.block);
        const Tap ty = clamp_tap(sy, L.nby), tx = clamp_tap(sx, L.nbx);
        eo[i] = bilerp(err_of(ty.i0, tx.i0), err_of(ty.i0, tx.i1), err_of(ty.i1, tx.i0),
                       err_of(ty.i1, tx.i1), tx.f, ty.f);
    }
}

// direct-t state of pair `pair` (fvv_dense_views mode 1): the VINet synthesis
// state (5, H, W) f32 = (F_m->l, F_m->r, logit M) from the engine's final
// flows (exact: FlowField.scaled(-0.5) of the level-2 flow) and the f64 mask
__global__ void k_direct_state(Geometry g, const uint8_t* __restrict__ ws, Planes P, int pair,
                               const double* __restrict__ mask, float* __restrict__ state) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t n = (size_t)g.W * g.H;
    if (i >= (int)n) return;
    const int y = i / g.W, x = i - (i / g.W) * g.W;
    const Level L1 = g.lv[1], L2 = g.lv[2];
    const float sc = 1.0f / (float)(1 << g.fb[2]);
    for (int d = 0; d < 2; d++) {
        const int2 base = up2_fixed(cplane<int2>(ws, P, P.flow1[d], pair), L1.h, L1.w, y, x);
        const int2 res = b2p_fixed(cplane<BlockHit>(ws, P, P.hit[2][d], pair), L2.nby, L2.nbx, L2.block, y, x);
        const int bs = g.fb[2] - (g.fb[1] + 3), rs = g.fb[2] - g.rb[2];
        state[(size_t)(2 * d) * n + i] = ((float)((base.x << bs) + (res.x << rs)) * sc) * -0.5f;
        state[(size_t)(2 * d + 1) * n + i] = ((float)((base.y << bs) + (res.y << rs)) * sc) * -0.5f;
    }
    const double m = fmin(fmax(mask[i], 1e-7), 1.0 - 1e-7);
    state[4 * n + i] = (float)log(m / (1.0 - m));
}

cudaError_t run_direct_state(const Geometry& g, uint8_t* ws, const Planes& P, int pair, const double* mask,
                             float* state, cudaStream_t st) {
    const int n = g.W * g.H;
    k_direct_state<<<(n + 255) / 256, 256, 0, st>>>(g, ws, P, pair, mask, state);
    return cudaGetLastError();
}

cudaError_t run_level_diag(const Geometry& g, uint8_t* ws, const Planes& P, int pair, int level,
                           float* flow_lr, float* flow_rl, double* err_lr, double* err_rl,
                           cudaStream_t st) {
    const Level& L = g.lv[level];
    dim3 grd((L.w * L.h + 255) / 256, 1, 2);
    auto f2 = [](float* p) { return reinterpret_cast<float2*>(p); };
    if (level == 0) k_diag_level<0><<<grd, 256, 0, st>>>(g, ws, P, pair, f2(flow_lr), f2(flow_rl), err_lr, err_rl);
    else if (level == 1) k_diag_level<1><<<grd, 256, 0, st>>>(g, ws, P, pair, f2(flow_lr), f2(flow_rl), err_lr, err_rl);
    else k_diag_level<2><<<grd, 256, 0, st>>>(g, ws, P, pair, f2(flow_lr), f2(flow_rl), err_lr, err_rl);
    return cudaGetLastError();
}

cudaError_t run_diag(const Geometry& g, const PairTable& pt, uint8_t* ws, const Planes& P, int pair,
                     float* flow_lr, float* flow_rl, double* mask, cudaStream_t st) {
    if (flow_lr || flow_rl) {
        dim3 grd((g.W * g.H + 255) / 256, 1, 2);
        k_diag_flow<<<grd, 256, 0, st>>>(g, ws, P, pair, reinterpret_cast<float2*>(flow_lr),
                                         reinterpret_cast<float2*>(flow_rl));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (mask) {
        const dim3 grd(((g.W + 7) / 8 + 63) / 64, g.H / 2, 1);
        const cudaError_t e = launch_k(false, blend_kernel(g.fmt), grd, dim3(128), 0, st, g, pt, ws, P, pair, false, mask);
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    return cudaSuccess;
}

}  // namespace fvv
