// deflate_kernels.cu -- zlib.compress(stream, 6) for many streams at once on
// the device, byte-identical (the FVT1 encoder's per-plane DEFLATE,
// codec.py:148; algorithm and its zlib 1.3 provenance in zdeflate_core.h).
//
// Pipeline (one launch each, all streams of the batch together):
//   k_zd_chain   per 16K-position chunk: hash-chain links (distance to the newest
//                earlier same-hash position), window heads by shared-memory
//                atomicMax, then the chunk in position order by one warp with
//                __match_any_sync resolving same-hash lanes
//   k_zd_match   per 4K-position chunk: longest_match for every position, both
//                chain limits, window bytes and links staged in shared memory
//   k_zd_spec    per 16K-position segment: deflate_slow's lazy parse started
//                from a fresh state at the segment start (speculative), with the
//                sync code of every loop top it visits
//   k_zd_fix     per stream: walk the segments; from each true entry state
//                re-parse until a loop top whose sync code the speculative parse
//                shares (typically a few symbols), then adopt the speculative rest
//   k_zd_compact per segment: the true symbols into the stream's symbol array
//   k_zd_tree    per block (every 16383 symbols): histogram, zlib's Huffman
//                trees, static / dynamic choice, exact sizes
//   k_zd_layout  per stream: block byte ranges, the stored-block decision
//                (needs the block's start and the window position), bit offsets,
//                packed output offsets
//   k_zd_emit    per block: header / tree description, then every symbol's
//                bits at its scanned offset (atomicOr into the zeroed output)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "deflate.h"
#include "zdeflate_core.h"

namespace fvv {
using namespace zd;

namespace {

constexpr int kCH1 = 16384;   // chain chunk (positions)
constexpr int kCH2 = 4096;    // search chunk (positions)
#ifndef FVV_ZD_SEG
#define FVV_ZD_SEG 16384
#endif
constexpr int kSeg = FVV_ZD_SEG;  // speculative parse segment (positions)
constexpr int kSegPad = 260;  // symbols a segment's parse may run past its end
constexpr int kPW = 2048;     // parse window (records staged per refill)
constexpr size_t kChainSmem = 4 * 32768 + 2 * kCH1 + 2 * kCH1 + 64;
constexpr size_t kMatchSmem = 2 * (size_t)(kWSize + kCH2) + (kWSize + kCH2 + kMaxMatch + 8);

struct ZStream {
    int64_t in_off, n, blk_base;
    int32_t blk_cap, seg0, nseg, pad;
};
struct ZChunk {
    int32_t s, pad;
    int64_t c0;
};
struct ZSeg {
    int32_t s, k;
    int64_t g0, g1, sym_base;
};
struct SegExit {  // parse state at the first loop top at or past the segment end
    int64_t s, ms, cnt;
    int32_t ml, avail, final_lit, pad;
};
struct SegFix {
    int64_t fix_cnt, skip, out_base;
};
struct StreamSyms {
    int64_t nsym;
    int32_t final_lit, nblk;
};
struct BlockInfo {
    int64_t byte0, nbytes;
    uint64_t opt_lenb;
    int32_t flush_back;  // loop top of the flushing iteration = block end - flush_back
    int32_t type_ns;     // static or dynamic (stored is decided by the layout)
};

struct Plan {
    int S = 0, C1 = 0, C2 = 0, B = 0, G = 0;
    int64_t N = 0, SY = 0;
    size_t streams, ch1, ch2, segs, blkmap, pdist, rec, canon, spec, fix, syms, sexit, sfix, ssyms, binfo, codes,
        boff, slen, total;
};

size_t up(size_t x) { return (x + 255) & ~(size_t)255; }

Plan make_plan(const int64_t* len, int S) {
    Plan p;
    p.S = S;
    for (int s = 0; s < S; s++) {
        const int64_t n = std::max<int64_t>(0, len[s]);
        p.N += n;
        p.C1 += (int)((std::max<int64_t>(0, n - 2) + kCH1 - 1) / kCH1);
        p.C2 += (int)((n + kCH2 - 1) / kCH2);
        p.B += (int)(n / kBlockSyms + 2);
        const int64_t g = std::max<int64_t>(1, (n + kSeg - 1) / kSeg);
        p.G += (int)g;
        p.SY += n + g * kSegPad;
    }
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o += up(bytes); return at; };
    p.streams = take(sizeof(ZStream) * (size_t)S);
    p.ch1 = take(sizeof(ZChunk) * (size_t)std::max(1, p.C1));
    p.ch2 = take(sizeof(ZChunk) * (size_t)std::max(1, p.C2));
    p.segs = take(sizeof(ZSeg) * (size_t)p.G);
    p.blkmap = take(sizeof(int32_t) * (size_t)p.B);
    p.pdist = take(sizeof(uint16_t) * (size_t)(p.N + 8));
    p.rec = take(sizeof(uint2) * (size_t)(p.N + 8));
    p.canon = take((size_t)p.N + 8);
    p.spec = take(sizeof(uint32_t) * (size_t)p.SY);
    p.fix = take(sizeof(uint32_t) * (size_t)p.SY);
    p.syms = take(sizeof(uint32_t) * (size_t)(p.N + 8));
    p.sexit = take(sizeof(SegExit) * (size_t)p.G);
    p.sfix = take(sizeof(SegFix) * (size_t)p.G);
    p.ssyms = take(sizeof(StreamSyms) * (size_t)S);
    p.binfo = take(sizeof(BlockInfo) * (size_t)p.B);
    p.codes = take(sizeof(BlockCode) * (size_t)p.B);
    p.boff = take(sizeof(uint64_t) * (size_t)p.B);
    p.slen = take(sizeof(int64_t) * (size_t)S);
    p.total = o;
    return p;
}

// Links are only ordered among positions of the same hash, so the chunk is
// split by hash into 8 groups (h & 7), each a position-ordered list walked by
// its own warp: 8 independent serial walks instead of one.
__global__ void __launch_bounds__(256) k_zd_chain(const uint8_t* __restrict__ data, const ZStream* __restrict__ zs,
                                                  const ZChunk* __restrict__ ch, uint16_t* __restrict__ pdist) {
    extern __shared__ __align__(16) uint8_t zsm[];
    uint32_t* head = reinterpret_cast<uint32_t*>(zsm);                    // 32768 hash heads (0: none)
    uint16_t* hs = reinterpret_cast<uint16_t*>(zsm + 4 * 32768);           // hashes of the chunk
    uint16_t* lst = reinterpret_cast<uint16_t*>(zsm + 4 * 32768 + 2 * kCH1);  // chunk offsets grouped by h & 7
    int* gcount = reinterpret_cast<int*>(zsm + 4 * 32768 + 4 * kCH1);        // [8] group sizes, then starts
    const ZChunk ck = ch[blockIdx.x];
    const ZStream sd = zs[ck.s];
    const uint8_t* d = data + sd.in_off;
    const int64_t n = sd.n, c0 = ck.c0;
    const int64_t c1 = min(c0 + (int64_t)kCH1, n - 2);  // positions <= n - 3 carry a hash
    const int cn = (int)(c1 - c0);
    const int64_t base = c0 - kMaxDist - 1;                // head values: position - base (>= 1)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int i = tid; i < 32768; i += blockDim.x) head[i] = 0;
    if (tid < 16) gcount[tid] = 0;
    __syncthreads();
    // newest position of each hash within MAX_DIST before the chunk (position 0 is NIL)
    for (int64_t q = max((int64_t)1, c0 - kMaxDist) + tid; q < c0; q += blockDim.x)
        atomicMax(&head[hash3(d + q)], (uint32_t)(q - base));
    // thread t hashes chunk offsets [32 t, 32 t + 32) and counts them per group
    int cnt[8];
#pragma unroll
    for (int g = 0; g < 8; g++) cnt[g] = 0;
    const int i0 = tid * (kCH1 / 256);
    for (int k = 0; k < kCH1 / 256; k++) {
        const int i = i0 + k;
        if (i < cn) {
            const uint32_t h = hash3(d + c0 + i);
            hs[i] = (uint16_t)h;
#pragma unroll
            for (int g = 0; g < 8; g++) cnt[g] += (int)((h & 7) == (uint32_t)g);
        }
    }
    // exclusive scan of the per-thread counts, per group (thread order = position order)
    int off[8];
#pragma unroll
    for (int g = 0; g < 8; g++) {
        int v = cnt[g];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += u;
        }
        off[g] = v - cnt[g];  // within the warp
    }
    __shared__ int wtot[8][8];  // [warp][group]
#pragma unroll
    for (int g = 0; g < 8; g++)
        if (lane == 31) wtot[wid][g] = off[g] + cnt[g];
    __syncthreads();
    if (tid < 8) {  // group sizes and starts
        int tot = 0;
        for (int w = 0; w < 8; w++) tot += wtot[w][tid];
        gcount[tid] = tot;
    }
    __syncthreads();
    int gstart[8];
    {
        int a = 0;
#pragma unroll
        for (int g = 0; g < 8; g++) {
            gstart[g] = a;
            a += gcount[g];
        }
    }
#pragma unroll
    for (int g = 0; g < 8; g++) {
        int wo = 0;
        for (int w = 0; w < wid; w++) wo += wtot[w][g];
        off[g] += gstart[g] + wo;
    }
    for (int k = 0; k < kCH1 / 256; k++) {
        const int i = i0 + k;
        if (i < cn) {
            const int g = hs[i] & 7;
            int o = 0;
#pragma unroll
            for (int gg = 0; gg < 8; gg++)
                if (gg == g) o = off[gg]++;
            lst[o] = (uint16_t)i;
        }
    }
    __syncthreads();
    // warp w walks group w in position order
    const int gs = gstart[wid], ge = gs + gcount[wid];
    for (int b = gs; b < ge; b += 32) {
        const bool act = b + lane < ge;
        const int i = act ? lst[b + lane] : 0;
        const int64_t p = c0 + i;
        const uint32_t h = act ? hs[i] : (0x8000u | lane);
        const uint32_t m = __match_any_sync(0xffffffffu, h);
        const uint32_t lower = m & ((1u << lane) - 1u);
        const int src = lower ? 31 - __clz(lower) : lane;
        const int iq = __shfl_sync(0xffffffffu, i, src);
        int64_t q;
        if (lower) {
            q = c0 + iq;
        } else {
            const uint32_t r = act ? head[h] : 0u;
            q = r ? base + r : 0;
        }
        const uint16_t pd = (act && q > 0 && p - q <= kMaxDist) ? (uint16_t)(p - q) : (uint16_t)0;
        __syncwarp();
        if (act && (m >> lane) == 1u) head[h] = p == 0 ? 0u : (uint32_t)(p - base);
        __syncwarp();
        if (act) pdist[sd.in_off + p] = pd;
    }
}

__global__ void __launch_bounds__(512) k_zd_match(const uint8_t* __restrict__ data, const ZStream* __restrict__ zs,
                                                  const ZChunk* __restrict__ ch, const uint16_t* __restrict__ pdist,
                                                  uint2* __restrict__ rec) {
    extern __shared__ __align__(16) uint8_t zsm[];
    const ZChunk ck = ch[blockIdx.x];
    const ZStream sd = zs[ck.s];
    const uint8_t* d = data + sd.in_off;
    const uint16_t* pg = pdist + sd.in_off;
    const int64_t n = sd.n, c0 = ck.c0, c1 = min(c0 + (int64_t)kCH2, n);
    const int64_t wb = max((int64_t)0, c0 - kWSize), we = min(n, c1 + kMaxMatch);
    const int64_t pe = min(c1, n - 2);
    uint16_t* sp = reinterpret_cast<uint16_t*>(zsm);
    uint8_t* sb = zsm + 2 * (size_t)(kWSize + kCH2);
    for (int64_t i = threadIdx.x; i < pe - wb; i += blockDim.x) sp[i] = pg[wb + i];
    for (int64_t i = threadIdx.x; i < we - wb; i += blockDim.x) sb[i] = d[wb + i];
    __syncthreads();
    // shared-window addresses for the search's explicit ld.shared: taken through a
    // volatile mov after the barrier, so no load can be scheduled above it
    ShWin win;
    asm volatile("mov.u32 %0, %1;" : "=r"(win.sb) : "r"((uint32_t)__cvta_generic_to_shared(sb)));
    asm volatile("mov.u32 %0, %1;" : "=r"(win.sp) : "r"((uint32_t)__cvta_generic_to_shared(sp)));
    uint2* out = rec + sd.in_off;
    for (int64_t p = c0 + threadIdx.x; p < c1; p += blockDim.x) {
        MatchRec r{0u, 0u};
        const int64_t la = n - p;
        if (la >= kMinMatch) {
            const int P = (int)(p - wb);
            const int pd0 = sp[P];
            if (pd0 && !nil_at_slide(p, n, (uint32_t)pd0))
                r = match_search32w(win, P, (int)min(la, (int64_t)(1 << 20)), pd0);
        }
        out[p] = make_uint2(r.r128, r.r32);
    }
}

// Speculative parse of one segment: one warp stages record / byte windows,
// lane 0 parses.  The last segment of a stream runs to the end of the input.
__global__ void __launch_bounds__(32) k_zd_spec(const uint8_t* __restrict__ data, const ZStream* __restrict__ zs,
                                                const ZSeg* __restrict__ segs, const uint2* __restrict__ rec,
                                                uint8_t* __restrict__ canon, uint32_t* __restrict__ spec,
                                                SegExit* __restrict__ sexit) {
    __shared__ uint2 wr[kPW];
    __shared__ uint8_t wbt[kPW + 1];
    const ZSeg sg = segs[blockIdx.x];
    const ZStream sd = zs[sg.s];
    const uint8_t* d = data + sd.in_off;
    const uint2* rg = rec + sd.in_off;
    uint8_t* cn = canon + sd.in_off;
    uint32_t* sy = spec + sg.sym_base;
    const int64_t n = sd.n, g1 = sg.g1;
    const bool last = sg.k == sd.nseg - 1;
    const int lane = threadIdx.x;
    ParseState st;
    parse_init(st, sg.g0);
    int64_t cnt = 0, wbeg = -1;
    bool more = true;
    if (lane == 0 && sg.g0 < n) cn[sg.g0] = 1;
    while (more) {
        const int64_t s0 = __shfl_sync(0xffffffffu, st.s, 0);
        if (wbeg < 0 || s0 >= wbeg + kPW) {
            wbeg = s0;
            for (int i = lane; i < kPW; i += 32) {
                const int64_t p = wbeg + i;
                wr[i] = p < n ? rg[p] : make_uint2(0u, 0u);
            }
            for (int i = lane; i < kPW + 1; i += 32) {
                const int64_t p = wbeg - 1 + i;
                wbt[i] = (p >= 0 && p < n) ? d[p] : (uint8_t)0;
            }
            __syncwarp();
        }
        if (lane == 0) {
            auto rc = [&](int64_t p) {
                const uint2 v = wr[p - wbeg];
                return MatchRec{v.x, v.y};
            };
            auto by = [&](int64_t p) { return wbt[p - wbeg + 1]; };
            auto em = [&](uint32_t v) { sy[cnt++] = v; };
            for (;;) {
                if (st.s >= g1 && !(last && st.s >= n)) {
                    more = false;  // first loop top past the segment
                    break;
                }
                if (st.s >= wbeg + kPW) break;  // refill
                if (!parse_iter(st, n, rc, by, em)) {
                    more = false;  // the input is done (last segment)
                    break;
                }
                if (st.s < g1) cn[st.s] = (uint8_t)sync_code(st);
            }
        }
        more = __shfl_sync(0xffffffffu, more, 0);
        __syncwarp();
    }
    if (lane == 0) sexit[blockIdx.x] = SegExit{st.s, st.ms, cnt, st.ml, st.avail, st.final_lit, 0};
}

// Per stream: the true parse across its segments.
__global__ void __launch_bounds__(128) k_zd_fix(const uint8_t* __restrict__ data, const ZStream* __restrict__ zs,
                                                int S, const ZSeg* __restrict__ segs,
                                                const uint2* __restrict__ rec, const uint8_t* __restrict__ canon,
                                                const uint32_t* __restrict__ spec, uint32_t* __restrict__ fix,
                                                const SegExit* __restrict__ sexit, SegFix* __restrict__ sfix,
                                                StreamSyms* __restrict__ ssyms) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const ZStream sd = zs[s];
    const uint8_t* d = data + sd.in_off;
    const uint2* rg = rec + sd.in_off;
    const uint8_t* cn = canon + sd.in_off;
    const int64_t n = sd.n;
    auto rc = [&](int64_t p) {
        const uint2 v = rg[p];
        return MatchRec{v.x, v.y};
    };
    auto by = [&](int64_t p) { return d[p]; };
    SegExit e0 = sexit[sd.seg0];
    ParseState cur;
    parse_init(cur, e0.s);
    cur.ms = e0.ms; cur.ml = e0.ml; cur.avail = e0.avail; cur.final_lit = e0.final_lit;
    int64_t total = e0.cnt;
    sfix[sd.seg0] = SegFix{0, 0, 0};
    for (int k = 1; k < sd.nseg; k++) {
        const int gi = sd.seg0 + k;
        const ZSeg sg = segs[gi];
        const bool last = k == sd.nseg - 1;
        const int64_t g1 = sg.g1;
        ParseState st = cur;
        int64_t fc = 0;
        uint32_t* fy = fix + sg.sym_base;
        auto em = [&](uint32_t v) { fy[fc++] = v; };
        auto synced = [&]() {
            const int c = sync_code(st);
            return c != 0 && st.s < g1 && cn[st.s] == c;
        };
        bool sync = synced();
        while (!sync && st.s < g1) {
            if (!parse_iter(st, n, rc, by, em)) break;
            sync = synced();
        }
        const SegExit ex = sexit[gi];
        int64_t skip;
        if (sync) {
            const int64_t target = st.s - st.avail;  // a pending literal is not emitted yet
            const uint32_t* sy = spec + sg.sym_base;
            int64_t cov = sg.g0, i = 0;
            while (cov < target) cov += sym_cover(sy[i++]);
            skip = i;
            parse_init(cur, ex.s);
            cur.ms = ex.ms; cur.ml = ex.ml; cur.avail = ex.avail; cur.final_lit = ex.final_lit;
        } else {
            skip = ex.cnt;
            if (last)
                while (parse_iter(st, n, rc, by, em)) {
                }
            cur = st;
        }
        sfix[gi] = SegFix{fc, skip, total};
        total += fc + ex.cnt - skip;
    }
    ssyms[s] = StreamSyms{total, cur.final_lit, (int32_t)((total - cur.final_lit) / kBlockSyms + 1)};
}

__global__ void __launch_bounds__(256) k_zd_compact(const ZStream* __restrict__ zs, const ZSeg* __restrict__ segs,
                                                    const uint32_t* __restrict__ spec,
                                                    const uint32_t* __restrict__ fix,
                                                    const SegExit* __restrict__ sexit,
                                                    const SegFix* __restrict__ sfix, uint32_t* __restrict__ syms) {
    const ZSeg sg = segs[blockIdx.x];
    const SegFix f = sfix[blockIdx.x];
    const int64_t cnt = sexit[blockIdx.x].cnt;
    uint32_t* out = syms + zs[sg.s].in_off + f.out_base;
    for (int64_t i = threadIdx.x; i < f.fix_cnt; i += blockDim.x) out[i] = fix[sg.sym_base + i];
    out += f.fix_cnt;
    for (int64_t i = f.skip + threadIdx.x; i < cnt; i += blockDim.x) out[i - f.skip] = spec[sg.sym_base + i];
}

__global__ void __launch_bounds__(256) k_zd_tree(const ZStream* __restrict__ zs, const int32_t* __restrict__ blkmap,
                                                 const StreamSyms* __restrict__ ssyms,
                                                 const uint32_t* __restrict__ syms, BlockInfo* __restrict__ binfo,
                                                 BlockCode* __restrict__ codes) {
    __shared__ ZTab t;
    __shared__ TreeWork w;
    __shared__ __align__(16) BlockCode bc;
    __shared__ uint32_t lf[kLCodes], df[kDCodes];
    __shared__ unsigned long long nbytes;
    const int slot = blockIdx.x;
    const int s = blkmap[slot];
    const ZStream sd = zs[s];
    const StreamSyms ss = ssyms[s];
    const int b = slot - (int)sd.blk_base;
    if (b >= ss.nblk) return;
    const int64_t j0 = (int64_t)b * kBlockSyms, j1 = b == ss.nblk - 1 ? ss.nsym : j0 + kBlockSyms;
    for (int i = threadIdx.x; i < kLCodes; i += blockDim.x) lf[i] = 0;
    for (int i = threadIdx.x; i < kDCodes; i += blockDim.x) df[i] = 0;
    if (threadIdx.x == 0) {
        ztab_fill(t);
        nbytes = 0;
    }
    __syncthreads();
    const uint32_t* sy = syms + sd.in_off;
    uint64_t cov = 0;
    for (int64_t i = j0 + threadIdx.x; i < j1; i += blockDim.x) {
        const uint32_t v = sy[i], dist = v >> 8, lc = v & 0xff;
        cov += sym_cover(v);
        if (dist == 0) {
            atomicAdd(&lf[lc], 1u);
        } else {
            atomicAdd(&lf[t.lcode[lc] + 257], 1u);
            atomicAdd(&df[d_code(t, dist - 1)], 1u);
        }
    }
    atomicAdd(&nbytes, (unsigned long long)cov);
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kHeapSize; i++) w.lfc[i] = w.ldl[i] = 0;
        for (int i = 0; i < 2 * kDCodes + 1; i++) w.dfc[i] = w.ddl[i] = 0;
        for (int i = 0; i < 2 * kBLCodes + 1; i++) w.bfc[i] = w.bdl[i] = 0;
        for (int i = 0; i < kLCodes; i++) w.lfc[i] = (uint16_t)lf[i];
        for (int i = 0; i < kDCodes; i++) w.dfc[i] = (uint16_t)df[i];
        w.lfc[kEndBlock] = 1;
        uint64_t opt_lenb;
        const int ty = block_trees_ns(w, t, opt_lenb);
        block_code(bc, w, t, ty, (int64_t)nbytes);
        const uint32_t lastsym = j1 > j0 ? sy[j1 - 1] : 0u;
        binfo[slot] = BlockInfo{0, (int64_t)nbytes, opt_lenb,
                                (lastsym >> 8) ? sym_cover(lastsym) - 1 : 0, ty};
    }
    __syncthreads();
    const uint32_t* src = reinterpret_cast<const uint32_t*>(&bc);
    uint32_t* dst = reinterpret_cast<uint32_t*>(codes + slot);
    for (int i = threadIdx.x; i < (int)(sizeof(BlockCode) / 4); i += blockDim.x) dst[i] = src[i];
}

__global__ void __launch_bounds__(1024) k_zd_layout(const ZStream* __restrict__ zs, int S,
                                                    const StreamSyms* __restrict__ ssyms,
                                                    BlockInfo* __restrict__ binfo, BlockCode* __restrict__ codes,
                                                    uint64_t* __restrict__ boff, int64_t* __restrict__ slen,
                                                    int64_t* __restrict__ out_off) {
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        const ZStream sd = zs[s];
        const int nblk = ssyms[s].nblk;
        uint64_t off = 0;
        int64_t byte0 = 0;
        for (int b = 0; b < nblk; b++) {
            const int64_t slot = sd.blk_base + b;
            BlockInfo bi = binfo[slot];
            const bool last = b == nblk - 1;
            const int64_t end = byte0 + bi.nbytes;
            const int64_t top = last ? sd.n : end - bi.flush_back;
            const bool buf_ok = byte0 >= (int64_t)kWSize * slides_at(top, sd.n);
            const int type = take_stored(bi.nbytes, bi.opt_lenb, buf_ok) ? kStored : bi.type_ns;
            codes[slot].type = type;
            bi.byte0 = byte0;
            binfo[slot] = bi;
            boff[slot] = off;
            if (type == kStored) off = ((off + 3 + 7) & ~(uint64_t)7) + 32 + 8 * (uint64_t)bi.nbytes;
            else off += codes[slot].bits;
            byte0 = end;
        }
        slen[s] = (int64_t)((off + 7) >> 3);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t o = 0;
        out_off[0] = 0;
        for (int s = 0; s < S; s++) out_off[s + 1] = (o += slen[s]);
    }
}

__global__ void __launch_bounds__(256) k_zd_emit(const uint8_t* __restrict__ data, const ZStream* __restrict__ zs,
                                                 const int32_t* __restrict__ blkmap,
                                                 const StreamSyms* __restrict__ ssyms,
                                                 const uint32_t* __restrict__ syms, const BlockInfo* __restrict__ binfo,
                                                 const BlockCode* __restrict__ codes,
                                                 const uint64_t* __restrict__ boff,
                                                 const int64_t* __restrict__ out_off, uint64_t* __restrict__ out) {
    __shared__ ZTab t;
    __shared__ uint32_t lcl[kLCodes], dcl[kDCodes];
    __shared__ uint64_t part[256];
    __shared__ uint64_t sym_base;
    const int slot = blockIdx.x;
    const int s = blkmap[slot];
    const ZStream sd = zs[s];
    const StreamSyms ss = ssyms[s];
    const int b = slot - (int)sd.blk_base;
    if (b >= ss.nblk) return;
    const BlockInfo bi = binfo[slot];
    const BlockCode* bc = codes + slot;
    const int type = bc->type, last = b == ss.nblk - 1;
    const uint64_t base = (uint64_t)out_off[s] * 8 + boff[slot];
    if (type == kStored) {
        if (threadIdx.x == 0) put_bits(out, base, (uint64_t)last, 3);
        const uint64_t P = (base + 3 + 7) >> 3;
        const uint32_t len = (uint32_t)bi.nbytes, nlen = ~len & 0xffffu;
        const uint8_t* src = data + sd.in_off + bi.byte0;
        for (int64_t i = threadIdx.x; i < 4 + bi.nbytes; i += blockDim.x) {
            const uint32_t v = i == 0 ? (len & 0xff) : i == 1 ? (len >> 8) & 0xff : i == 2 ? (nlen & 0xff)
                             : i == 3 ? (nlen >> 8) : src[i - 4];
            put_bits(out, (P + (uint64_t)i) * 8, v, 8);
        }
        return;
    }
    if (threadIdx.x == 0) ztab_fill(t);
    for (int i = threadIdx.x; i < kLCodes; i += blockDim.x) lcl[i] = bc->lcl[i];
    for (int i = threadIdx.x; i < kDCodes; i += blockDim.x) dcl[i] = bc->dcl[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        put_bits(out, base, (uint64_t)((type << 1) + last), 3);
        uint64_t o = base + 3;
        if (type == kDynamic) o = send_trees(out, o, bc->h, t);
        sym_base = o;
    }
    auto lco = [&](int c) { return lcl[c]; };
    auto dco = [&](int c) { return dcl[c]; };
    auto llen = [&](int c) { return (int)(lcl[c] & 0xff); };
    auto dlen = [&](int c) { return (int)(dcl[c] & 0xff); };
    const int64_t j0 = (int64_t)b * kBlockSyms;
    const int nsym = (int)((last ? ss.nsym : j0 + kBlockSyms) - j0);
    const int per = (nsym + blockDim.x - 1) / blockDim.x;
    const int i0 = min(nsym, (int)threadIdx.x * per), i1 = min(nsym, i0 + per);
    const uint32_t* sy = syms + sd.in_off + j0;
    uint64_t bits = 0;
    for (int i = i0; i < i1; i++) bits += (uint64_t)sym_bits(t, sy[i], llen, dlen);
    part[threadIdx.x] = bits;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t acc = 0;
        for (int i = 0; i < (int)blockDim.x; i++) {
            const uint64_t v = part[i];
            part[i] = acc;
            acc += v;
        }
        const uint32_t e = lcl[kEndBlock];
        put_bits(out, sym_base + acc, e >> 8, (int)(e & 0xff));
    }
    __syncthreads();
    uint64_t off = sym_base + part[threadIdx.x];
    for (int i = i0; i < i1; i++) off += (uint64_t)put_sym(out, off, t, sy[i], lco, dco);
}

}  // namespace

size_t zd_scratch_bytes(const int64_t* len, int nstreams) { return make_plan(len, nstreams).total; }

size_t zd_out_capacity(const int64_t* len, int nstreams) {
    uint64_t c = 16;
    for (int s = 0; s < nstreams; s++) c += compress_bound((uint64_t)std::max<int64_t>(0, len[s]));
    return (size_t)((c + 7) & ~(uint64_t)7);
}

cudaError_t zd_deflate(const uint8_t* data, const int64_t* in_off, int S, uint8_t* out, int64_t* out_off,
                       void* scratch, size_t scratch_bytes, cudaStream_t st) {
    if (S <= 0) return cudaSuccess;
    std::vector<int64_t> len(S);
    for (int s = 0; s < S; s++) len[s] = in_off[s + 1] - in_off[s];
    const Plan p = make_plan(len.data(), S);
    if (scratch_bytes < p.total) return cudaErrorInvalidValue;
    uint8_t* sc = static_cast<uint8_t*>(scratch);
    std::vector<ZStream> zs(S);
    std::vector<ZChunk> c1, c2;
    std::vector<ZSeg> sg;
    std::vector<int32_t> bm;
    c1.reserve(p.C1);
    c2.reserve(p.C2);
    sg.reserve(p.G);
    bm.reserve(p.B);
    int64_t bb = 0, sb = 0;
    for (int s = 0; s < S; s++) {
        const int64_t n = len[s];
        const int nseg = (int)std::max<int64_t>(1, (n + kSeg - 1) / kSeg);
        zs[s] = ZStream{in_off[s], n, bb, (int32_t)(n / kBlockSyms + 2), (int32_t)sg.size(), nseg, 0};
        for (int64_t c = 0; c < n - 2; c += kCH1) c1.push_back(ZChunk{s, 0, c});
        for (int64_t c = 0; c < n; c += kCH2) c2.push_back(ZChunk{s, 0, c});
        for (int k = 0; k < nseg; k++) {
            const int64_t g0 = (int64_t)k * kSeg, g1 = std::min(n, g0 + kSeg);
            sg.push_back(ZSeg{s, k, g0, g1, sb});
            sb += (g1 - g0) + kSegPad;
        }
        for (int i = 0; i < zs[s].blk_cap; i++) bm.push_back(s);
        bb += zs[s].blk_cap;
    }
    cudaError_t e;
    auto h2d = [&](size_t off, const void* src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(sc + off, src, bytes, cudaMemcpyHostToDevice, st) : cudaSuccess;
    };
    if ((e = h2d(p.streams, zs.data(), sizeof(ZStream) * zs.size()))) return e;
    if ((e = h2d(p.ch1, c1.data(), sizeof(ZChunk) * c1.size()))) return e;
    if ((e = h2d(p.ch2, c2.data(), sizeof(ZChunk) * c2.size()))) return e;
    if ((e = h2d(p.segs, sg.data(), sizeof(ZSeg) * sg.size()))) return e;
    if ((e = h2d(p.blkmap, bm.data(), sizeof(int32_t) * bm.size()))) return e;
    if ((e = cudaMemsetAsync(out, 0, zd_out_capacity(len.data(), S), st))) return e;
    if ((e = cudaMemsetAsync(sc + p.canon, 0, (size_t)p.N + 8, st))) return e;
    static thread_local int attrs_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attrs_dev != dev) {  // per device: the >48 KB shared memory opt-in
        if ((e = cudaFuncSetAttribute(k_zd_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChainSmem)))
            return e;
        if ((e = cudaFuncSetAttribute(k_zd_match, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMatchSmem)))
            return e;
        attrs_dev = dev;
    }
    const ZStream* dzs = reinterpret_cast<const ZStream*>(sc + p.streams);
    const ZSeg* dsg = reinterpret_cast<const ZSeg*>(sc + p.segs);
    const int32_t* bmap = reinterpret_cast<const int32_t*>(sc + p.blkmap);
    uint16_t* pdist = reinterpret_cast<uint16_t*>(sc + p.pdist);
    uint2* rec = reinterpret_cast<uint2*>(sc + p.rec);
    uint8_t* canon = sc + p.canon;
    uint32_t* spec = reinterpret_cast<uint32_t*>(sc + p.spec);
    uint32_t* fix = reinterpret_cast<uint32_t*>(sc + p.fix);
    uint32_t* syms = reinterpret_cast<uint32_t*>(sc + p.syms);
    SegExit* sexit = reinterpret_cast<SegExit*>(sc + p.sexit);
    SegFix* sfix = reinterpret_cast<SegFix*>(sc + p.sfix);
    StreamSyms* ssyms = reinterpret_cast<StreamSyms*>(sc + p.ssyms);
    BlockInfo* binfo = reinterpret_cast<BlockInfo*>(sc + p.binfo);
    BlockCode* codes = reinterpret_cast<BlockCode*>(sc + p.codes);
    uint64_t* boff = reinterpret_cast<uint64_t*>(sc + p.boff);
    if (p.C1) k_zd_chain<<<p.C1, 256, kChainSmem, st>>>(data, dzs, reinterpret_cast<const ZChunk*>(sc + p.ch1), pdist);
    if (p.C2)
        k_zd_match<<<p.C2, 512, kMatchSmem, st>>>(data, dzs, reinterpret_cast<const ZChunk*>(sc + p.ch2), pdist, rec);
    k_zd_spec<<<p.G, 32, 0, st>>>(data, dzs, dsg, rec, canon, spec, sexit);
    k_zd_fix<<<(S + 127) / 128, 128, 0, st>>>(data, dzs, S, dsg, rec, canon, spec, fix, sexit, sfix, ssyms);
    k_zd_compact<<<p.G, 256, 0, st>>>(dzs, dsg, spec, fix, sexit, sfix, syms);
    k_zd_tree<<<p.B, 256, 0, st>>>(dzs, bmap, ssyms, syms, binfo, codes);
    k_zd_layout<<<1, 1024, 0, st>>>(dzs, S, ssyms, binfo, codes, boff, reinterpret_cast<int64_t*>(sc + p.slen),
                                   out_off);
    k_zd_emit<<<p.B, 256, 0, st>>>(data, dzs, bmap, ssyms, syms, binfo, codes, boff, out_off,
                                   reinterpret_cast<uint64_t*>(out));
    return cudaGetLastError();
}

}  // namespace fvv
