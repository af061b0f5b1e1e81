// zdeflate_core.h -- zlib's DEFLATE at level 6 (windowBits 15, memLevel 8,
// default strategy: what zlib.compress(data, 6) runs, codec.py:148), restated
// as independent steps a GPU can run in parallel.  Shared by the device
// kernels (deflate_kernels.cu) and the host model (tools/zdeflate_model.cpp).
//
// Third-party algorithm: zlib 1.3 (the image's libz.so.1.3 and the zlib
// compiled into the interpreter: zlib.ZLIB_VERSION == "1.3").  The output must
// be byte-identical to zlib's, so every decision below restates zlib's
// published deflate_slow / longest_match / trees.c behaviour:
//
//  * hash chains.  deflate_slow inserts EVERY position p <= n-3 into the hash
//    chains (also inside emitted matches), with the 15-bit hash
//    ((b0 << 10) ^ (b1 << 5) ^ b2) & 0x7fff of the rolling UPDATE_HASH.  So the
//    chain of p is content-determined: all earlier positions with the same
//    hash, newest first.  Position 0 is never a candidate (it equals NIL).
//  * longest_match(p) walks at most max_chain candidates (128; 32 once the
//    previous match is >= good_length 8), the first within MAX_DIST (<=), the
//    others strictly nearer; it returns the longest match and the FIRST
//    (nearest) candidate reaching it, stopping at the first candidate of
//    length >= nice (128, capped by the lookahead).  Its start value
//    best_len = prev_length only thresholds the result, so the search is
//    precomputed once per position for both chain limits (match_search).
//  * the lazy parse (deflate_slow's state machine) consumes those records
//    sequentially (parse_*), emitting zlib's symbols; a block is flushed every
//    lit_bufsize - 1 = 16383 symbols and at the end.
//  * per block: zlib's Huffman construction (build_tree / gen_bitlen /
//    gen_codes / scan_tree / build_bl_tree), the stored / static / dynamic
//    choice of _tr_flush_block, and the exact bit layout.
//  * the sliding window only matters at two places, both handled exactly: a
//    block may be stored only while its start is still inside the window, and
//    the slide at strstart == wsize + MAX_DIST at the very end of the input
//    turns a candidate at exactly MAX_DIST into NIL.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define ZHD __host__ __device__ __forceinline__
#else
#define ZHD inline
#endif

namespace zd {

constexpr int kWSize = 32768;
constexpr int kMinMatch = 3, kMaxMatch = 258;
constexpr int kMinLookahead = kMaxMatch + kMinMatch + 1;  // 262
constexpr int kMaxDist = kWSize - kMinLookahead;          // 32506
constexpr int kTooFar = 4096;
constexpr int kGoodLength = 8, kMaxLazy = 16, kNiceLength = 128, kMaxChain = 128;
constexpr int kBlockSyms = (1 << 14) - 1;  // lit_bufsize - 1 (memLevel 8)
constexpr int kLCodes = 286, kDCodes = 30, kBLCodes = 19;
constexpr int kHeapSize = 2 * kLCodes + 1;
constexpr int kMaxBits = 15, kMaxBLBits = 7;
constexpr int kEndBlock = 256;
constexpr int kStored = 0, kStatic = 1, kDynamic = 2;

ZHD uint32_t hash3(const uint8_t* p) {
    return (((uint32_t)p[0] << 10) ^ ((uint32_t)p[1] << 5) ^ (uint32_t)p[2]) & 0x7fffu;
}

// zlib's compressBound: the output capacity per stream
ZHD uint64_t compress_bound(uint64_t n) { return n + (n >> 12) + (n >> 14) + (n >> 25) + 13; }

// ---------------------------------------------------------------------------
// Static tables (tr_static_init)
// ---------------------------------------------------------------------------
struct ZTab {
    uint8_t lcode[256];   // match length - 3 -> length code 0..28
    uint8_t dcode[512];   // d_code table
    uint16_t base_len[29];
    uint16_t base_dist[30];
    uint8_t xl[29], xd[30], xbl[19], bl_order[19];
    uint16_t s_lcode[288];
    uint8_t s_llen[288];
    uint16_t s_dcode[30];
    uint8_t s_dlen[30];
};

ZHD uint32_t bi_reverse(uint32_t code, int len) {
    uint32_t r = 0;
    do {
        r |= code & 1;
        code >>= 1;
        r <<= 1;
    } while (--len > 0);
    return r >> 1;
}

ZHD void ztab_fill(ZTab& t) {
    const uint8_t xl[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
    const uint8_t xd[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
    const uint8_t blo[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    for (int i = 0; i < 29; i++) t.xl[i] = xl[i];
    for (int i = 0; i < 30; i++) t.xd[i] = xd[i];
    for (int i = 0; i < 19; i++) { t.xbl[i] = i == 16 ? 2 : (i == 17 ? 3 : (i == 18 ? 7 : 0)); t.bl_order[i] = blo[i]; }
    int length = 0, code;
    for (code = 0; code < 28; code++) {
        t.base_len[code] = (uint16_t)length;
        for (int n = 0; n < (1 << xl[code]); n++) t.lcode[length++] = (uint8_t)code;
    }
    t.lcode[255] = 28;  // length 258: code 285 rather than 284 + 5 bits
    t.base_len[28] = 0;
    int dist = 0;
    for (code = 0; code < 16; code++) {
        t.base_dist[code] = (uint16_t)dist;
        for (int n = 0; n < (1 << xd[code]); n++) t.dcode[dist++] = (uint8_t)code;
    }
    dist >>= 7;
    for (; code < 30; code++) {
        t.base_dist[code] = (uint16_t)(dist << 7);
        for (int n = 0; n < (1 << (xd[code] - 7)); n++) t.dcode[256 + dist++] = (uint8_t)code;
    }
    // static literal/length tree: 8/9/7/8-bit canonical codes (gen_codes)
    uint16_t blc[kMaxBits + 1];
    for (int b = 0; b <= kMaxBits; b++) blc[b] = 0;
    for (int n = 0; n < 288; n++) {
        const int l = n <= 143 ? 8 : (n <= 255 ? 9 : (n <= 279 ? 7 : 8));
        t.s_llen[n] = (uint8_t)l;
        blc[l]++;
    }
    uint16_t next[kMaxBits + 1];
    uint32_t c = 0;
    for (int b = 1; b <= kMaxBits; b++) {
        c = (c + blc[b - 1]) << 1;
        next[b] = (uint16_t)c;
    }
    for (int n = 0; n < 288; n++) t.s_lcode[n] = (uint16_t)bi_reverse(next[t.s_llen[n]]++, t.s_llen[n]);
    for (int n = 0; n < 30; n++) {
        t.s_dlen[n] = 5;
        t.s_dcode[n] = (uint16_t)bi_reverse((uint32_t)n, 5);
    }
}

ZHD int d_code(const ZTab& t, uint32_t dist /* distance - 1 */) {
    return dist < 256 ? t.dcode[dist] : t.dcode[256 + (dist >> 7)];
}

// ---------------------------------------------------------------------------
// Per-position match search (longest_match for every position, both chain
// limits).  prevdist[p]: distance to the newest earlier same-hash position
// (0: none, or farther than MAX_DIST, or position 0 = NIL).
// Record: (len << 16) | dist, 0 = no usable match (len <= 2, or a length-3
// match farther than TOO_FAR, which deflate_slow discards when it is the
// result: only possible from prev_length 2).
// ---------------------------------------------------------------------------
struct MatchRec {
    uint32_t r128, r32;
};

// The slide at strstart == wsize + MAX_DIST (only at the end of the input:
// n <= p + 261) maps the candidate at exactly MAX_DIST to window index 0 = NIL.
ZHD bool nil_at_slide(int64_t p, int64_t n, uint32_t pd) {
    return pd == (uint32_t)kMaxDist && p >= kWSize + kMaxDist && (p - (kWSize + kMaxDist)) % kWSize == 0 &&
           n <= p + kMinLookahead - 1;
}

ZHD uint32_t finish_rec(int best, int64_t p, int64_t bc) {
    if (best <= 2) return 0;
    const uint32_t dist = (uint32_t)(p - bc);
    if (best == kMinMatch && dist > (uint32_t)kTooFar) return 0;
    return ((uint32_t)best << 16) | dist;
}

// win(i) returns the byte at stream position i (any i in [p - MAX_DIST, n)),
// pdist(i) the prevdist of position i.
template <typename Win, typename PDist>
ZHD MatchRec match_search(int64_t p, int64_t n, const Win& win, const PDist& pdist) {
    MatchRec r{0, 0};
    const int64_t la = n - p;
    if (la < kMinMatch) return r;
    const uint32_t pd = pdist(p);
    if (pd == 0 || nil_at_slide(p, n, pd)) return r;
    const int nice = la < kNiceLength ? (int)la : kNiceLength;
    const int maxlen = la < kMaxMatch ? (int)la : kMaxMatch;
    int best = 2, cnt = 0;
    int64_t bc = 0, c = p - pd;
    const uint8_t s0 = win(p), s1 = win(p + 1);
    bool have32 = false;
    for (;;) {
        cnt++;
        // zlib's quick rejection (match[best_len], match[best_len-1], bytes 0, 1);
        // byte 2 is equal on a chain (equal hashes and bytes 0, 1)
        if (win(c + best) == win(p + best) && win(c + best - 1) == win(p + best - 1) && win(c) == s0 &&
            win(c + 1) == s1) {
            int len = 3;
            while (len < maxlen && win(c + len) == win(p + len)) len++;
            if (len > best) {
                best = len;
                bc = c;
                if (len >= nice) break;
            }
        }
        if (cnt == kMaxChain >> 2) {
            r.r32 = finish_rec(best, p, bc);
            have32 = true;
        }
        if (cnt == kMaxChain) break;
        const uint32_t d = pdist(c);
        if (d == 0) break;
        c -= d;
        if (p - c >= kMaxDist) break;  // later candidates: strictly within MAX_DIST
    }
    r.r128 = finish_rec(best, p, bc);
    if (!have32) r.r32 = r.r128;
    return r;
}

// match_search with 32-bit window-relative indices over plain arrays (the
// device form): sb / sp hold the bytes and links of positions [wb, ...), P is
// the position relative to wb, la = n - p; the NIL edge is checked by the caller.
ZHD uint32_t finish_rec32(int best, int dist) {
    if (best <= 2 || (best == kMinMatch && dist > kTooFar)) return 0;
    return ((uint32_t)best << 16) | (uint32_t)dist;
}
// 4 bytes at byte offset i (little endian) of a 4-byte aligned buffer with 8
// bytes of readable padding past its end
ZHD uint32_t ld32u(const uint8_t* b, int i) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(b + (i & ~3));
    const int sh = (i & 3) * 8;
#ifdef __CUDA_ARCH__
    return __funnelshift_r(w[0], w[1], sh);
#else
    return (uint32_t)((((uint64_t)w[1] << 32) | w[0]) >> sh);
#endif
}

ZHD int ctz32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __ffs((int)x) - 1;
#else
    return __builtin_ctz(x);
#endif
}

// Every candidate's match length from a branch-free 8-byte compare (scan words
// cached), the continuation loop only for candidates matching 8+ bytes.  zlib's
// quick rejection (bytes best-1, best, 0, 1) only skips candidates that cannot
// beat best, so measuring them changes nothing: the running best, the first
// (nearest) candidate reaching it, the nice cut and the 32 / 128 chain limits
// are longest_match's and the result equals match_search's.  (A filter that
// passes ~7 % of the candidates keeps most of a warp idle while a few lanes
// measure; measuring all keeps the lanes together.)
// Window access for match_search32: the bytes as aligned 32-bit words and the
// links.  Host: plain pointers.  Device (ShWin): 32-bit shared-window addresses
// with explicit ld.shared, so the compiler does not rebuild a generic pointer
// to the dynamic shared array inside the candidate loop.
struct PtrWin {
    const uint8_t* sb;
    const uint16_t* sp;
    ZHD uint32_t word(int wi) const { return reinterpret_cast<const uint32_t*>(sb)[wi]; }
    ZHD int link(int i) const { return sp[i]; }
};
#ifdef __CUDACC__
struct ShWin {
    uint32_t sb, sp;  // shared-window addresses (sb 4-byte aligned)
    __device__ __forceinline__ uint32_t word(int wi) const {
        uint32_t v;
        asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(sb + 4u * (uint32_t)wi));
        return v;
    }
    __device__ __forceinline__ int link(int i) const {
        unsigned short v;
        asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(sp + 2u * (uint32_t)i));
        return (int)v;
    }
};
#endif

template <typename Win>
ZHD uint32_t win32u(const Win& W, int i) {  // 4 bytes at byte offset i
    const int wi = i >> 2, sh = (i & 3) * 8;
    const uint32_t w0 = W.word(wi), w1 = W.word(wi + 1);
#ifdef __CUDA_ARCH__
    return __funnelshift_r(w0, w1, sh);
#else
    return (uint32_t)((((uint64_t)w1 << 32) | w0) >> sh);
#endif
}

template <typename Win>
ZHD MatchRec match_search32w(const Win& W, int P, int la, int pd0) {
    MatchRec r{0, 0};
    const int nice = la < kNiceLength ? la : kNiceLength;
    const int maxlen = la < kMaxMatch ? la : kMaxMatch;
    const int lim = P - kMaxDist;  // later candidates must lie above (distance < MAX_DIST)
    const uint32_t p0 = win32u(W, P), p1 = win32u(W, P + 4);
    int best = 2, bc = P, cnt = 0, c = P - pd0;
    uint32_t pb = 0;  // scan bytes best-3 .. best once best >= 8
    bool done = false;
    for (int phase = 0; phase < 2 && !done; phase++) {
        const int stop = phase ? kMaxChain : (kMaxChain >> 2);
        while (cnt < stop) {
            cnt++;
            const int d = W.link(c);
            uint32_t x0, x1;
            {  // 8 bytes at c from three aligned words
                const int wi = c >> 2, sh = (c & 3) * 8;
                const uint32_t w0 = W.word(wi), w1 = W.word(wi + 1), w2 = W.word(wi + 2);
#ifdef __CUDA_ARCH__
                x0 = __funnelshift_r(w0, w1, sh) ^ p0;
                x1 = __funnelshift_r(w1, w2, sh) ^ p1;
#else
                x0 = (uint32_t)((((uint64_t)w1 << 32) | w0) >> sh) ^ p0;
                x1 = (uint32_t)((((uint64_t)w2 << 32) | w1) >> sh) ^ p1;
#endif
            }
            int len;
            if ((x0 | x1) != 0) {  // the common case: fewer than 8 equal bytes, no branch
                const uint32_t y = x0 ? x0 : x1;
                len = (ctz32(y) >> 3) + (x0 ? 0 : 4);
            } else if (best >= 8 && win32u(W, c + best - 3) != pb) {
                len = 8;  // differs within bytes best-3 .. best: cannot beat best
            } else {
                len = 8;
                uint32_t x = 0;
                while (len < maxlen && (x = win32u(W, c + len) ^ win32u(W, P + len)) == 0) len += 4;
                if (x) len += ctz32(x) >> 3;
            }
            len = len < maxlen ? len : maxlen;
            const bool imp = len > best;
            best = imp ? len : best;
            bc = imp ? c : bc;
            if (imp) {
                if (len >= nice) { done = true; break; }
                if (best >= 8) pb = win32u(W, P + best - 3);
            }
            if (d == 0) { done = true; break; }
            c -= d;
            if (c <= lim) { done = true; break; }
        }
        if (phase == 0) r.r32 = finish_rec32(best, P - bc);
    }
    r.r128 = finish_rec32(best, P - bc);
    return r;
}


ZHD MatchRec match_search32(const uint8_t* sb, const uint16_t* sp, int P, int la, int pd0) {
    return match_search32w(PtrWin{sb, sp}, P, la, pd0);
}

// ---------------------------------------------------------------------------
// Lazy parse (deflate_slow).  Symbols: (dist << 8) | lc as zlib's sym_buf
// (dist 0: literal lc; else lc = match length - 3).
// ---------------------------------------------------------------------------
// the k-th window slide happens at the first loop top s >= slide_at(k)
ZHD int64_t slide_at(int64_t k, int64_t n) {
    const int64_t base = (int64_t)kWSize * k;
    if (n > base + 2 * kWSize) return base + kWSize + kMaxDist + 1;  // input still flowing in
    const int64_t a = base + kWSize + kMaxDist, b = n - (kMinLookahead - 1);
    return a > b ? a : b;
}

struct BlockDesc {
    int64_t sym0;      // first symbol (stream-relative index)
    int32_t nsym;
    int32_t flags;     // bit 0: last block; bit 1: block start still in the window (stored allowed)
    int64_t byte0;     // input range [byte0, byte0 + nbytes)
    int64_t nbytes;
};

struct ParseState {
    int64_t s;          // strstart (loop top)
    int ml;             // match_length
    int64_t ms;         // match_start
    int avail;          // match_available
    int final_lit;      // the input ended with a pending literal (emitted after the loop)
    int64_t slides;     // window slides so far
    int64_t nsym;       // symbols emitted
    int64_t blk_sym0, blk_byte0;
    int32_t nblocks;
};

ZHD void parse_init(ParseState& st, int64_t s0 = 0) {
    st.s = s0; st.ml = kMinMatch - 1; st.ms = 0; st.avail = 0; st.final_lit = 0; st.slides = 0; st.nsym = 0;
    st.blk_sym0 = 0; st.blk_byte0 = 0; st.nblocks = 0;
}

// The parse's decisions depend on (s, match_length, match_start, match_available)
// only, and with match_length 2 (no match pending: right after a match, in a run
// of literals, or at a fresh start) match_start is never read again.  Two parses
// of the same data that meet at a loop top with equal sync codes stay identical.
// 0: not a sync state; 1: match_length 2, nothing pending; 2: match_length 2,
// literal s - 1 pending.
ZHD int sync_code(const ParseState& st) { return st.ml == kMinMatch - 1 ? 1 + st.avail : 0; }
ZHD bool canonical(const ParseState& st) { return st.ml == kMinMatch - 1 && st.avail == 0; }

// input bytes a symbol covers
ZHD int sym_cover(uint32_t sym) { return (sym >> 8) ? (int)(sym & 0xff) + kMinMatch : 1; }

// One deflate_slow iteration without the block bookkeeping (blocks are cut
// from the finished symbol stream: every 16383 symbols).  At s >= n: the
// pending literal, then false.
template <typename Rec, typename Byte, typename Emit>
ZHD bool parse_iter(ParseState& st, int64_t n, const Rec& rec, const Byte& byte, const Emit& emit) {
    if (st.s >= n) {
        if (st.avail) {
            emit((uint32_t)byte(st.s - 1));
            st.avail = 0;
            st.final_lit = 1;
        }
        return false;
    }
    const int64_t la = n - st.s;
    const int pl = st.ml;
    const int64_t pm = st.ms;
    st.ml = kMinMatch - 1;
    if (la >= kMinMatch && pl < kMaxLazy) {
        const MatchRec m = rec(st.s);
        const uint32_t r = pl < kGoodLength ? m.r128 : m.r32;
        const int len = (int)(r >> 16);
        if (len > pl) {
            st.ml = len;
            st.ms = st.s - (int64_t)(r & 0xffffu);
        }
    }
    if (pl >= kMinMatch && st.ml <= pl) {
        emit(((uint32_t)(st.s - 1 - pm) << 8) | (uint32_t)(pl - kMinMatch));
        st.s += pl - 1;
        st.avail = 0;
        st.ml = kMinMatch - 1;
    } else if (st.avail) {
        emit((uint32_t)byte(st.s - 1));
        st.s++;
    } else {
        st.avail = 1;
        st.s++;
    }
    return true;
}

// window slides done by loop top s (deflate_slow / fill_window)
ZHD int64_t slides_at(int64_t s, int64_t n) {
    int64_t k = 0;
    while (slide_at(k, n) <= s) k++;
    return k;
}

// One iteration of deflate_slow's loop at loop top st.s; after the input is
// consumed, the final literal and the last block.  Returns false once done.
template <typename Rec, typename Byte, typename Emit, typename Block>
ZHD bool parse_step(ParseState& st, int64_t n, const Rec& rec, const Byte& byte, const Emit& emit,
                    const Block& block) {
    auto flush = [&](int64_t end, int last) {
        BlockDesc b;
        b.sym0 = st.blk_sym0;
        b.nsym = (int32_t)(st.nsym - st.blk_sym0);
        b.byte0 = st.blk_byte0;
        b.nbytes = end - st.blk_byte0;
        b.flags = (last ? 1 : 0) | (st.blk_byte0 >= (int64_t)kWSize * st.slides ? 2 : 0);
        block(st.nblocks++, b);
        st.blk_sym0 = st.nsym;
        st.blk_byte0 = end;
    };
    while (st.s >= slide_at(st.slides, n)) st.slides++;
    if (st.s >= n) {
        if (st.avail) emit(st.nsym++, (uint32_t)byte(st.s - 1));
        st.avail = 0;
        flush(n, 1);
        return false;
    }
    const int64_t la = n - st.s;
    const int pl = st.ml;
    const int64_t pm = st.ms;
    st.ml = kMinMatch - 1;
    if (la >= kMinMatch && pl < kMaxLazy) {
        const MatchRec m = rec(st.s);
        const uint32_t r = pl < kGoodLength ? m.r128 : m.r32;
        const int len = (int)(r >> 16);
        if (len > pl) {
            st.ml = len;
            st.ms = st.s - (int64_t)(r & 0xffffu);
        }
    }
    if (pl >= kMinMatch && st.ml <= pl) {
        emit(st.nsym++, ((uint32_t)(st.s - 1 - pm) << 8) | (uint32_t)(pl - kMinMatch));
        st.s += pl - 1;
        st.avail = 0;
        st.ml = kMinMatch - 1;
        if (st.nsym - st.blk_sym0 == kBlockSyms) flush(st.s, 0);
    } else if (st.avail) {
        emit(st.nsym++, (uint32_t)byte(st.s - 1));
        if (st.nsym - st.blk_sym0 == kBlockSyms) flush(st.s, 0);
        st.s++;
    } else {
        st.avail = 1;
        st.s++;
    }
    return true;
}

template <typename Rec, typename Byte, typename Emit, typename Block>
ZHD void parse_stream(int64_t n, const Rec& rec, const Byte& byte, const Emit& emit, const Block& block) {
    ParseState st;
    parse_init(st);
    while (parse_step(st, n, rec, byte, emit, block)) {
    }
}

// ---------------------------------------------------------------------------
// Huffman trees of one block (trees.c), Freq/Code and Dad/Len unions kept as
// the same storage so every read sees what zlib's would.
// ---------------------------------------------------------------------------
struct TreeWork {
    uint16_t lfc[kHeapSize], ldl[kHeapSize];
    uint16_t dfc[2 * kDCodes + 1], ddl[2 * kDCodes + 1];
    uint16_t bfc[2 * kBLCodes + 1], bdl[2 * kBLCodes + 1];
    uint16_t lreal[kLCodes], dreal[kDCodes], breal[kBLCodes];  // frequencies before the dummy nodes
    int16_t heap[kHeapSize];
    uint8_t depth[kHeapSize];
    uint16_t bl_count[kMaxBits + 1];
    int heap_len, heap_max;
    uint64_t opt_len, static_len;
    int lmax, dmax, blmax;  // max_code of each tree, max_blindex
};

struct TreeDesc {
    uint16_t* fc;
    uint16_t* dl;
    const uint8_t* slen;   // static tree lengths (null for the bit-length tree)
    const uint8_t* extra;
    int extra_base, elems, max_length;
};

ZHD bool zsmaller(const uint16_t* fc, int n, int m, const uint8_t* depth) {
    return fc[n] < fc[m] || (fc[n] == fc[m] && depth[n] <= depth[m]);
}

ZHD void pqdownheap(TreeWork& w, const uint16_t* fc, int k) {
    const int v = w.heap[k];
    int j = k << 1;
    while (j <= w.heap_len) {
        if (j < w.heap_len && zsmaller(fc, w.heap[j + 1], w.heap[j], w.depth)) j++;
        if (zsmaller(fc, v, w.heap[j], w.depth)) break;
        w.heap[k] = w.heap[j];
        k = j;
        j <<= 1;
    }
    w.heap[k] = (int16_t)v;
}

ZHD void gen_bitlen(TreeWork& w, const TreeDesc& d, int max_code) {
    uint16_t* fc = d.fc;
    uint16_t* dl = d.dl;
    int overflow = 0;
    for (int b = 0; b <= kMaxBits; b++) w.bl_count[b] = 0;
    dl[w.heap[w.heap_max]] = 0;  // root
    int h;
    for (h = w.heap_max + 1; h < kHeapSize; h++) {
        const int n = w.heap[h];
        int bits = dl[dl[n]] + 1;
        if (bits > d.max_length) bits = d.max_length, overflow++;
        dl[n] = (uint16_t)bits;
        if (n > max_code) continue;
        w.bl_count[bits]++;
        int xbits = 0;
        if (n >= d.extra_base) xbits = d.extra[n - d.extra_base];
        const uint64_t f = fc[n];
        w.opt_len += f * (uint64_t)(bits + xbits);
        if (d.slen) w.static_len += f * (uint64_t)(d.slen[n] + xbits);
    }
    if (overflow == 0) return;
    do {
        int bits = d.max_length - 1;
        while (w.bl_count[bits] == 0) bits--;
        w.bl_count[bits]--;
        w.bl_count[bits + 1] += 2;
        w.bl_count[d.max_length]--;
        overflow -= 2;
    } while (overflow > 0);
    for (int bits = d.max_length; bits != 0; bits--) {
        int n = w.bl_count[bits];
        while (n != 0) {
            const int m = w.heap[--h];
            if (m > max_code) continue;
            if (dl[m] != (unsigned)bits) {
                w.opt_len += ((uint64_t)bits - dl[m]) * (uint64_t)fc[m];
                dl[m] = (uint16_t)bits;
            }
            n--;
        }
    }
}

ZHD void gen_codes(uint16_t* fc, const uint16_t* dl, int max_code, const uint16_t* bl_count) {
    uint16_t next[kMaxBits + 1];
    uint32_t code = 0;
    for (int bits = 1; bits <= kMaxBits; bits++) {
        code = (code + bl_count[bits - 1]) << 1;
        next[bits] = (uint16_t)code;
    }
    for (int n = 0; n <= max_code; n++) {
        const int len = dl[n];
        if (len == 0) continue;
        fc[n] = (uint16_t)bi_reverse(next[len]++, len);
    }
}

ZHD int build_tree(TreeWork& w, const TreeDesc& d) {
    uint16_t* fc = d.fc;
    uint16_t* dl = d.dl;
    const int elems = d.elems;
    int max_code = -1;
    w.heap_len = 0;
    w.heap_max = kHeapSize;
    for (int n = 0; n < elems; n++) {
        if (fc[n] != 0) {
            w.heap[++w.heap_len] = (int16_t)(max_code = n);
            w.depth[n] = 0;
        } else {
            dl[n] = 0;
        }
    }
    while (w.heap_len < 2) {
        const int node = w.heap[++w.heap_len] = (int16_t)(max_code < 2 ? ++max_code : 0);
        fc[node] = 1;
        w.depth[node] = 0;
        w.opt_len--;
        if (d.slen) w.static_len -= d.slen[node];
    }
    for (int n = w.heap_len / 2; n >= 1; n--) pqdownheap(w, fc, n);
    int node = elems;
    do {
        const int n = w.heap[1];
        w.heap[1] = w.heap[w.heap_len--];
        pqdownheap(w, fc, 1);
        const int m = w.heap[1];
        w.heap[--w.heap_max] = (int16_t)n;
        w.heap[--w.heap_max] = (int16_t)m;
        fc[node] = (uint16_t)(fc[n] + fc[m]);
        w.depth[node] = (uint8_t)((w.depth[n] >= w.depth[m] ? w.depth[n] : w.depth[m]) + 1);
        dl[n] = dl[m] = (uint16_t)node;
        w.heap[1] = (int16_t)node++;
        pqdownheap(w, fc, 1);
    } while (w.heap_len >= 2);
    w.heap[--w.heap_max] = w.heap[1];
    gen_bitlen(w, d, max_code);
    gen_codes(fc, dl, max_code, w.bl_count);
    return max_code;
}

ZHD void scan_tree(TreeWork& w, uint16_t* dl, int max_code) {
    int prevlen = -1, curlen, nextlen = dl[0], count = 0, max_count = 7, min_count = 4;
    if (nextlen == 0) max_count = 138, min_count = 3;
    dl[max_code + 1] = 0xffff;  // guard
    for (int n = 0; n <= max_code; n++) {
        curlen = nextlen;
        nextlen = dl[n + 1];
        if (++count < max_count && curlen == nextlen) {
            continue;
        } else if (count < min_count) {
            w.bfc[curlen] += (uint16_t)count;
        } else if (curlen != 0) {
            if (curlen != prevlen) w.bfc[curlen]++;
            w.bfc[16]++;
        } else if (count <= 10) {
            w.bfc[17]++;
        } else {
            w.bfc[18]++;
        }
        count = 0;
        prevlen = curlen;
        if (nextlen == 0) max_count = 138, min_count = 3;
        else if (curlen == nextlen) max_count = 6, min_count = 3;
        else max_count = 7, min_count = 4;
    }
}

// Histogram already in w.lfc[0..285] / w.dfc[0..29] (END_BLOCK counted).
// Builds the three trees; returns static or dynamic and (opt_lenb) the byte
// size _tr_flush_block compares a stored block against.
ZHD int block_trees_ns(TreeWork& w, const ZTab& t, uint64_t& opt_lenb_out) {
    w.opt_len = w.static_len = 0;
    for (int n = 0; n < kLCodes; n++) w.lreal[n] = w.lfc[n];
    for (int n = 0; n < kDCodes; n++) w.dreal[n] = w.dfc[n];
    for (int n = 0; n < kBLCodes; n++) w.bfc[n] = 0;
    const TreeDesc ld{w.lfc, w.ldl, t.s_llen, t.xl, 257, kLCodes, kMaxBits};
    const TreeDesc dd{w.dfc, w.ddl, t.s_dlen, t.xd, 0, kDCodes, kMaxBits};
    const TreeDesc bd{w.bfc, w.bdl, nullptr, t.xbl, 0, kBLCodes, kMaxBLBits};
    w.lmax = build_tree(w, ld);
    w.dmax = build_tree(w, dd);
    scan_tree(w, w.ldl, w.lmax);
    scan_tree(w, w.ddl, w.dmax);
    for (int n = 0; n < kBLCodes; n++) w.breal[n] = w.bfc[n];
    build_tree(w, bd);
    int mb;
    for (mb = kBLCodes - 1; mb >= 3; mb--)
        if (w.bdl[t.bl_order[mb]] != 0) break;
    w.blmax = mb;
    w.opt_len += 3 * ((uint64_t)mb + 1) + 5 + 5 + 4;
    uint64_t opt_lenb = (w.opt_len + 3 + 7) >> 3;
    const uint64_t static_lenb = (w.static_len + 3 + 7) >> 3;
    if (static_lenb <= opt_lenb) opt_lenb = static_lenb;
    opt_lenb_out = opt_lenb;
    return static_lenb == opt_lenb ? kStatic : kDynamic;
}

// _tr_flush_block's choice: stored when it is no larger and the block's start
// is still in the window (buf != NULL), else static or dynamic
ZHD bool take_stored(int64_t stored_len, uint64_t opt_lenb, bool buf_ok) {
    return (uint64_t)stored_len + 4 <= opt_lenb && buf_ok;
}

ZHD int block_trees(TreeWork& w, const ZTab& t, int64_t stored_len, bool buf_ok) {
    uint64_t ob;
    const int ty = block_trees_ns(w, t, ob);
    return take_stored(stored_len, ob, buf_ok) ? kStored : ty;
}

// bits of one symbol under code lengths (llen, dlen)
template <typename LLen, typename DLen>
ZHD int sym_bits(const ZTab& t, uint32_t sym, const LLen& llen, const DLen& dlen) {
    const uint32_t dist = sym >> 8, lc = sym & 0xff;
    if (dist == 0) return llen(lc);
    const int code = t.lcode[lc];
    const int dc = d_code(t, dist - 1);
    return llen(code + 257) + t.xl[code] + dlen(dc) + t.xd[dc];
}

// Exact size in bits of the dynamic tree description (what send_all_trees writes)
ZHD uint64_t dyn_header_bits(const TreeWork& w, const ZTab& t) {
    uint64_t b = 5 + 5 + 4 + 3 * (uint64_t)(w.blmax + 1);
    for (int n = 0; n < kBLCodes; n++) b += (uint64_t)w.breal[n] * (w.bdl[n] + t.xbl[n]);
    return b;
}

// ---------------------------------------------------------------------------
// Bit writer: LSB-first into 64-bit little-endian words (OR into a zeroed
// buffer; atomic on the device, where neighbouring blocks share words).
// ---------------------------------------------------------------------------
ZHD void put_bits(uint64_t* words, uint64_t off, uint64_t val, int nbits) {
    if (nbits == 0) return;
    const uint64_t wi = off >> 6;
    const int sh = (int)(off & 63);
#ifdef __CUDA_ARCH__
    atomicOr((unsigned long long*)&words[wi], (unsigned long long)(val << sh));
    if (sh + nbits > 64) atomicOr((unsigned long long*)&words[wi + 1], (unsigned long long)(val >> (64 - sh)));
#else
    words[wi] |= val << sh;
    if (sh + nbits > 64) words[wi + 1] |= val >> (64 - sh);
#endif
}

// What the bit writer needs of a dynamic block's trees.
struct TreeHdr {
    uint16_t ldl[kLCodes + 2];   // literal/length code lengths (0..lmax)
    uint16_t ddl[kDCodes + 2];   // distance code lengths (0..dmax)
    uint16_t bcode[kBLCodes];    // bit-length tree codes (bit-reversed) and lengths
    uint8_t blen[kBLCodes];
    int16_t lmax, dmax, blmax;
};

ZHD void tree_hdr(TreeHdr& h, const TreeWork& w) {
    for (int n = 0; n < kLCodes + 2; n++) h.ldl[n] = n <= w.lmax ? w.ldl[n] : 0;
    for (int n = 0; n < kDCodes + 2; n++) h.ddl[n] = n <= w.dmax ? w.ddl[n] : 0;
    for (int n = 0; n < kBLCodes; n++) {
        h.bcode[n] = w.bfc[n];
        h.blen[n] = (uint8_t)w.bdl[n];
    }
    h.lmax = (int16_t)w.lmax;
    h.dmax = (int16_t)w.dmax;
    h.blmax = (int16_t)w.blmax;
}

// send_all_trees: the dynamic block's tree description, returns the new offset
ZHD uint64_t send_trees(uint64_t* out, uint64_t off, const TreeHdr& h, const ZTab& t) {
    const int lcodes = h.lmax + 1, dcodes = h.dmax + 1, blcodes = h.blmax + 1;
    put_bits(out, off, (uint64_t)(lcodes - 257), 5); off += 5;
    put_bits(out, off, (uint64_t)(dcodes - 1), 5); off += 5;
    put_bits(out, off, (uint64_t)(blcodes - 4), 4); off += 4;
    for (int r = 0; r < blcodes; r++) {
        put_bits(out, off, h.blen[t.bl_order[r]], 3);
        off += 3;
    }
    auto code = [&](int c) {
        put_bits(out, off, h.bcode[c], h.blen[c]);
        off += h.blen[c];
    };
    for (int tree = 0; tree < 2; tree++) {
        const uint16_t* dl = tree ? h.ddl : h.ldl;
        const int max_code = tree ? h.dmax : h.lmax;
        int prevlen = -1, curlen, nextlen = dl[0], count = 0, max_count = 7, min_count = 4;
        if (nextlen == 0) max_count = 138, min_count = 3;
        for (int n = 0; n <= max_code; n++) {
            curlen = nextlen;
            nextlen = n + 1 <= max_code ? dl[n + 1] : 0xffff;  // the guard scan_tree wrote
            if (++count < max_count && curlen == nextlen) {
                continue;
            } else if (count < min_count) {
                do { code(curlen); } while (--count != 0);
            } else if (curlen != 0) {
                if (curlen != prevlen) {
                    code(curlen);
                    count--;
                }
                code(16);
                put_bits(out, off, (uint64_t)(count - 3), 2); off += 2;
            } else if (count <= 10) {
                code(17);
                put_bits(out, off, (uint64_t)(count - 3), 3); off += 3;
            } else {
                code(18);
                put_bits(out, off, (uint64_t)(count - 11), 7); off += 7;
            }
            count = 0;
            prevlen = curlen;
            if (nextlen == 0) max_count = 138, min_count = 3;
            else if (curlen == nextlen) max_count = 6, min_count = 3;
            else max_count = 7, min_count = 4;
        }
    }
    return off;
}

// Everything the emitter needs of one block: type, codes, exact size in bits
// (header included; a stored block's alignment depends on its offset and is
// added by the layout pass).
struct BlockCode {
    TreeHdr h;
    uint32_t lcl[kLCodes];  // (code << 8) | len
    uint32_t dcl[kDCodes];
    uint64_t bits;
    int32_t type, pad;
};

// Finish a block after block_trees: codes and size.
ZHD void block_code(BlockCode& bc, const TreeWork& w, const ZTab& t, int type, int64_t nbytes) {
    bc.type = type;
    if (type == kStored) {
        bc.bits = 3 + 32 + 8 * (uint64_t)nbytes;  // + alignment
        return;
    }
    uint64_t bits = 3;
    if (type == kStatic) {
        for (int n = 0; n < kLCodes; n++) bc.lcl[n] = ((uint32_t)t.s_lcode[n] << 8) | t.s_llen[n];
        for (int n = 0; n < kDCodes; n++) bc.dcl[n] = ((uint32_t)t.s_dcode[n] << 8) | t.s_dlen[n];
    } else {
        tree_hdr(bc.h, w);
        bits += dyn_header_bits(w, t);
        for (int n = 0; n < kLCodes; n++) bc.lcl[n] = n <= w.lmax ? (((uint32_t)w.lfc[n] << 8) | w.ldl[n]) : 0;
        for (int n = 0; n < kDCodes; n++) bc.dcl[n] = n <= w.dmax ? (((uint32_t)w.dfc[n] << 8) | w.ddl[n]) : 0;
    }
    for (int n = 0; n < kLCodes; n++)
        bits += (uint64_t)w.lreal[n] * ((bc.lcl[n] & 0xff) + (n >= 257 ? t.xl[n - 257] : 0));
    for (int n = 0; n < kDCodes; n++) bits += (uint64_t)w.dreal[n] * ((bc.dcl[n] & 0xff) + t.xd[n]);
    bc.bits = bits;
}

// one symbol with codes (lcode/llen, dcode/dlen) at off
template <typename L, typename D>
ZHD int put_sym(uint64_t* out, uint64_t off, const ZTab& t, uint32_t sym, const L& lc_of, const D& dc_of) {
    const uint32_t dist = sym >> 8, lc = sym & 0xff;
    if (dist == 0) {
        const uint32_t cl = lc_of(lc);  // (code << 8) | len
        put_bits(out, off, cl >> 8, (int)(cl & 0xff));
        return (int)(cl & 0xff);
    }
    const int code = t.lcode[lc];
    const uint32_t cl = lc_of(code + 257);
    uint64_t v = cl >> 8;
    int nb = (int)(cl & 0xff);
    const int xl = t.xl[code];
    if (xl) v |= (uint64_t)(lc - t.base_len[code]) << nb;  // code 285 (length 258) has no extra bits
    nb += xl;
    const uint32_t d = dist - 1;
    const int dc = d_code(t, d);
    const uint32_t dcl = dc_of(dc);
    v |= (uint64_t)(dcl >> 8) << nb;
    nb += (int)(dcl & 0xff);
    if (t.xd[dc]) v |= (uint64_t)(d - t.base_dist[dc]) << nb;
    nb += t.xd[dc];
    put_bits(out, off, v, nb);  // <= 15 + 5 + 15 + 13 = 48 bits
    return nb;
}

}  // namespace zd
