// Host model of the device DEFLATE pipeline (csrc/zdeflate_core.h run as plain
// loops) checked byte for byte against the system zlib's compress2(level 6).
// Development tool: g++ -O2 -std=c++17 tools/zdeflate_model.cpp -lz
//   ./a.out            synthetic cases (sizes, stored/static/dynamic blocks,
//                      window slides, the end-of-input slide edge)
//   ./a.out FILE...    files
#include <zlib.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../paper_2112_10603_b200/csrc/zdeflate_core.h"

using namespace zd;

static int g_nil_hits = 0;

static std::vector<uint8_t> model(const std::vector<uint8_t>& in, int* types = nullptr) {
    const int64_t n = (int64_t)in.size();
    ZTab t;
    ztab_fill(t);
    // chains
    std::vector<uint16_t> pdist(n + 1, 0);
    std::vector<int64_t> head(1 << 15, -1);
    for (int64_t p = 0; p + 2 < n; p++) {
        const uint32_t h = hash3(&in[p]);
        const int64_t q = head[h];
        pdist[p] = (q > 0 && p - q <= kMaxDist) ? (uint16_t)(p - q) : 0;
        head[h] = p;
    }
    // searches
    std::vector<MatchRec> rec(n + 1);
    std::vector<uint32_t> pw((n + 16) / 4 + 4, 0);  // 4-byte aligned copy with padding (match_search32)
    uint8_t* padded = reinterpret_cast<uint8_t*>(pw.data());
    memcpy(padded, in.data(), n);
    auto win = [&](int64_t i) { return in[i]; };
    auto pd = [&](int64_t i) { return (uint32_t)pdist[i]; };
    for (int64_t p = 0; p < n; p++) {
        rec[p] = match_search(p, n, win, pd);
        if (n - p >= kMinMatch && pdist[p] && !nil_at_slide(p, n, pdist[p])) {  // the device form agrees
            const int64_t wb = (p > kWSize ? p - kWSize : 0) & ~(int64_t)3;
            const MatchRec r2 = match_search32(&padded[wb], &pdist[wb], (int)(p - wb), (int)std::min<int64_t>(n - p, 1 << 20),
                                               pdist[p]);
            if (r2.r128 != rec[p].r128 || r2.r32 != rec[p].r32) { printf("match_search32 differs at %lld\n", (long long)p); abort(); }
        }
        if (p + 2 < n && nil_at_slide(p, n, pdist[p])) g_nil_hits++;
    }
    // parse
    std::vector<uint32_t> syms;
    std::vector<BlockDesc> blocks;
    parse_stream(
        n, [&](int64_t p) { return rec[p]; }, [&](int64_t p) { return in[p]; },
        [&](int64_t i, uint32_t s) { if ((int64_t)syms.size() <= i) syms.resize(i + 1); syms[i] = s; },
        [&](int32_t i, const BlockDesc& b) { if ((int)blocks.size() <= i) blocks.resize(i + 1); blocks[i] = b; });
    // blocks
    std::vector<uint64_t> out((compress_bound(n) + 7) / 8 + 2, 0);
    uint64_t off = 0;
    static TreeWork w;
    for (size_t bi = 0; bi < blocks.size(); bi++) {
        const BlockDesc& b = blocks[bi];
        for (int i = 0; i < kHeapSize; i++) w.lfc[i] = w.ldl[i] = 0;
        for (int i = 0; i < 2 * kDCodes + 1; i++) w.dfc[i] = w.ddl[i] = 0;
        for (int i = 0; i < 2 * kBLCodes + 1; i++) w.bfc[i] = w.bdl[i] = 0;
        for (int32_t i = 0; i < b.nsym; i++) {
            const uint32_t s = syms[b.sym0 + i];
            const uint32_t dist = s >> 8, lc = s & 0xff;
            if (dist == 0) w.lfc[lc]++;
            else {
                w.lfc[t.lcode[lc] + 257]++;
                w.dfc[d_code(t, dist - 1)]++;
            }
        }
        w.lfc[kEndBlock] = 1;
        const int type = block_trees(w, t, b.nbytes, (b.flags & 2) != 0);
        if (types) types[type]++;
        static BlockCode bc;
        block_code(bc, w, t, type, b.nbytes);
        const int last = b.flags & 1;
        const uint64_t start = off;
        if (type == kStored) {
            put_bits(out.data(), off, (uint64_t)((0 << 1) + last), 3);
            off += 3;
            off = (off + 7) & ~(uint64_t)7;
            uint8_t* ob = reinterpret_cast<uint8_t*>(out.data());
            const uint16_t len = (uint16_t)b.nbytes, nlen = (uint16_t)~len;
            ob[off / 8] = len & 0xff; ob[off / 8 + 1] = len >> 8;
            ob[off / 8 + 2] = nlen & 0xff; ob[off / 8 + 3] = nlen >> 8;
            memcpy(ob + off / 8 + 4, &in[b.byte0], b.nbytes);
            off += 32 + 8 * (uint64_t)b.nbytes;
            continue;
        }
        put_bits(out.data(), off, (uint64_t)(((type == kStatic ? 1 : 2) << 1) + last), 3);
        off += 3;
        if (type == kDynamic) off = send_trees(out.data(), off, bc.h, t);
        auto lco = [&](int c) { return bc.lcl[c]; };
        auto dco = [&](int c) { return bc.dcl[c]; };
        for (int32_t i = 0; i < b.nsym; i++) off += put_sym(out.data(), off, t, syms[b.sym0 + i], lco, dco);
        const uint32_t e = lco(kEndBlock);
        put_bits(out.data(), off, e >> 8, e & 0xff);
        off += e & 0xff;
        if (off - start != bc.bits) { printf("block size mismatch %llu vs %llu\n", (unsigned long long)(off - start), (unsigned long long)bc.bits); abort(); }
    }
    const uint8_t* ob = reinterpret_cast<const uint8_t*>(out.data());
    return std::vector<uint8_t>(ob, ob + (off + 7) / 8);
}

// The device pipeline's decomposition: speculative per-segment parses from a
// canonical state, a per-stream fix-up pass that re-parses from each true entry
// state until it meets a canonical loop top of the speculative parse, blocks cut
// from the finished symbol stream, stored decisions in the layout pass.
static int g_fix_iters = 0, g_nosync = 0;
static std::vector<uint8_t> model_seg(const std::vector<uint8_t>& in, int64_t G) {
    const int64_t n = (int64_t)in.size();
    ZTab t;
    ztab_fill(t);
    std::vector<uint16_t> pdist(n + 1, 0);
    std::vector<int64_t> head(1 << 15, -1);
    for (int64_t p = 0; p + 2 < n; p++) {
        const uint32_t h = hash3(&in[p]);
        const int64_t q = head[h];
        pdist[p] = (q > 0 && p - q <= kMaxDist) ? (uint16_t)(p - q) : 0;
        head[h] = p;
    }
    std::vector<MatchRec> rec(n + 1);
    std::vector<uint32_t> pw((n + 16) / 4 + 4, 0);
    uint8_t* padded = reinterpret_cast<uint8_t*>(pw.data());
    memcpy(padded, in.data(), n);
    for (int64_t p = 0; p < n; p++) {
        rec[p] = MatchRec{0, 0};
        if (n - p >= kMinMatch && pdist[p] && !nil_at_slide(p, n, pdist[p])) {
            const int64_t wb = (p > kWSize ? p - kWSize : 0) & ~(int64_t)3;
            rec[p] = match_search32(&padded[wb], &pdist[wb], (int)(p - wb), (int)std::min<int64_t>(n - p, 1 << 20), pdist[p]);
        }
    }
    auto rc = [&](int64_t p) { return rec[p]; };
    auto by = [&](int64_t p) { return in[p]; };
    const int64_t nseg = std::max<int64_t>(1, (n + G - 1) / G);
    std::vector<std::vector<uint32_t>> spec(nseg), fix(nseg);
    std::vector<ParseState> sexit(nseg);
    std::vector<uint8_t> canon(n + 1, 0);
    for (int64_t k = 0; k < nseg; k++) {  // speculative parses (independent)
        const int64_t g0 = k * G, g1 = std::min(n, g0 + G);
        const bool last = k == nseg - 1;
        ParseState st;
        parse_init(st, g0);
        if (g0 < n) canon[g0] = 1;
        auto em = [&](uint32_t v) { spec[k].push_back(v); };
        while (st.s < g1) {
            if (!parse_iter(st, n, rc, by, em)) break;
            if (st.s < g1) canon[st.s] = (uint8_t)sync_code(st);
        }
        if (last) while (parse_iter(st, n, rc, by, em)) {}
        sexit[k] = st;
    }
    std::vector<int64_t> skip(nseg, 0);
    ParseState cur = sexit[0];
    for (int64_t k = 1; k < nseg; k++) {  // fix-up, sequential per stream
        const int64_t g0 = k * G, g1 = std::min(n, g0 + G);
        const bool last = k == nseg - 1;
        ParseState st = cur;
        auto em = [&](uint32_t v) { fix[k].push_back(v); };
        auto synced = [&]() { const int c = sync_code(st); return c != 0 && st.s < g1 && canon[st.s] == c; };
        bool sync = synced();
        while (!sync && st.s < g1) {
            g_fix_iters++;
            if (!parse_iter(st, n, rc, by, em)) break;
            sync = synced();
        }
        if (sync) {
            const int64_t target = st.s - st.avail;  // a pending literal is not emitted yet
            int64_t cov = g0, i = 0;
            while (cov < target) cov += sym_cover(spec[k][i++]);
            if (cov != target) { printf("sync point off a symbol boundary\n"); abort(); }
            skip[k] = i;
            cur = sexit[k];
        } else {
            g_nosync++;
            skip[k] = (int64_t)spec[k].size();
            if (last) while (parse_iter(st, n, rc, by, em)) {}
            cur = st;
        }
    }
    std::vector<uint32_t> syms;
    for (int64_t k = 0; k < nseg; k++) {
        syms.insert(syms.end(), fix[k].begin(), fix[k].end());
        syms.insert(syms.end(), spec[k].begin() + skip[k], spec[k].end());
    }
    const int64_t nsym = (int64_t)syms.size();
    const int64_t nblk = (nsym - cur.final_lit) / kBlockSyms + 1;
    std::vector<uint64_t> out((compress_bound(n) + 7) / 8 + 2, 0);
    uint64_t off = 0;
    int64_t byte0 = 0;
    static TreeWork w;
    static BlockCode bc;
    for (int64_t b = 0; b < nblk; b++) {
        const int64_t j0 = b * kBlockSyms, j1 = b == nblk - 1 ? nsym : j0 + kBlockSyms;
        for (int i = 0; i < kHeapSize; i++) w.lfc[i] = w.ldl[i] = 0;
        for (int i = 0; i < 2 * kDCodes + 1; i++) w.dfc[i] = w.ddl[i] = 0;
        for (int i = 0; i < 2 * kBLCodes + 1; i++) w.bfc[i] = w.bdl[i] = 0;
        int64_t nbytes = 0;
        for (int64_t i = j0; i < j1; i++) {
            const uint32_t v = syms[i], dist = v >> 8, lc = v & 0xff;
            nbytes += sym_cover(v);
            if (dist == 0) w.lfc[lc]++;
            else { w.lfc[t.lcode[lc] + 257]++; w.dfc[d_code(t, dist - 1)]++; }
        }
        w.lfc[kEndBlock] = 1;
        uint64_t opt_lenb;
        const int ty = block_trees_ns(w, t, opt_lenb);
        block_code(bc, w, t, ty, nbytes);
        const bool last = b == nblk - 1;
        const int64_t end = byte0 + nbytes;
        const int64_t top = last ? n : (syms[j1 - 1] >> 8 ? end - sym_cover(syms[j1 - 1]) + 1 : end);
        const bool buf_ok = byte0 >= (int64_t)kWSize * slides_at(top, n);
        const int type = take_stored(nbytes, opt_lenb, buf_ok) ? kStored : ty;
        if (type == kStored) {
            put_bits(out.data(), off, (uint64_t)last, 3);
            off = (off + 3 + 7) & ~(uint64_t)7;
            uint8_t* ob = reinterpret_cast<uint8_t*>(out.data());
            const uint16_t len = (uint16_t)nbytes, nlen = (uint16_t)~len;
            ob[off / 8] = len & 0xff; ob[off / 8 + 1] = len >> 8;
            ob[off / 8 + 2] = nlen & 0xff; ob[off / 8 + 3] = nlen >> 8;
            memcpy(ob + off / 8 + 4, &in[byte0], nbytes);
            off += 32 + 8 * (uint64_t)nbytes;
        } else {
            put_bits(out.data(), off, (uint64_t)((type << 1) + last), 3);
            off += 3;
            if (type == kDynamic) off = send_trees(out.data(), off, bc.h, t);
            auto lco = [&](int c) { return bc.lcl[c]; };
            auto dco = [&](int c) { return bc.dcl[c]; };
            for (int64_t i = j0; i < j1; i++) off += put_sym(out.data(), off, t, syms[i], lco, dco);
            const uint32_t e = lco(kEndBlock);
            put_bits(out.data(), off, e >> 8, e & 0xff);
            off += e & 0xff;
        }
        byte0 = end;
    }
    const uint8_t* ob = reinterpret_cast<const uint8_t*>(out.data());
    return std::vector<uint8_t>(ob, ob + (off + 7) / 8);
}

static std::vector<uint8_t> zref(const std::vector<uint8_t>& in) {
    uLongf cap = compressBound(in.size());
    std::vector<uint8_t> o(cap);
    if (compress2(o.data(), &cap, in.data(), in.size(), 6) != Z_OK) abort();
    return std::vector<uint8_t>(o.begin() + 2, o.begin() + cap - 4);
}

static int check(const char* name, const std::vector<uint8_t>& in) {
    int types[3] = {0, 0, 0};
    const auto a = model(in, types), b = zref(in);
    std::vector<int64_t> gs = {16384, 4096, 997};
    if (getenv("ZD_G")) gs = {atoll(getenv("ZD_G"))};
    for (int64_t G : gs) {
        if (model_seg(in, G) != b) {
            printf("%s: segmented pipeline (G=%lld) differs\n", name, (long long)G);
            return 1;
        }
    }
    size_t i = 0;
    while (i < a.size() && i < b.size() && a[i] == b[i]) i++;
    const bool ok = a == b;
    printf("%-34s n=%9zu  out=%8zu  blocks s/f/d=%d/%d/%d  %s", name, in.size(), b.size(), types[0], types[1],
           types[2], ok ? "OK" : "DIFF");
    if (!ok) printf(" (first diff at byte %zu of %zu / %zu)", i, a.size(), b.size());
    printf("\n");
    return ok ? 0 : 1;
}

int main(int argc, char** argv) {
    int bad = 0;
    if (argc > 1) {
        for (int i = 1; i < argc; i++) {
            FILE* f = fopen(argv[i], "rb");
            if (!f) continue;
            std::vector<uint8_t> d;
            int c;
            while ((c = fgetc(f)) != EOF) d.push_back((uint8_t)c);
            fclose(f);
            bad += check(argv[i], d);
        }
        printf("segmented parse: %d fix-up iterations, %d segments without sync\n", g_fix_iters, g_nosync);
        return bad;
    }
    std::mt19937_64 rng(1234);
    auto rnd = [&](size_t n, int alphabet) {
        std::vector<uint8_t> v(n);
        for (auto& x : v) x = (uint8_t)(rng() % alphabet);
        return v;
    };
    for (size_t n : {0, 1, 2, 3, 4, 5, 8, 100}) bad += check(("random " + std::to_string(n)).c_str(), rnd(n, 256));
    bad += check("zeros 1000", std::vector<uint8_t>(1000, 0));
    bad += check("zeros 300000", std::vector<uint8_t>(300000, 0));
    bad += check("random 70000 (stored)", rnd(70000, 256));
    bad += check("random 200000 alph4", rnd(200000, 4));
    bad += check("random 200000 alph16", rnd(200000, 16));
    bad += check("random 1000000 alph3", rnd(1000000, 3));
    {
        std::string s;
        while (s.size() < 500000) s += "the quick brown fox jumps over the lazy dog " + std::to_string(rng() % 1000) + "\n";
        bad += check("text 500k", std::vector<uint8_t>(s.begin(), s.end()));
    }
    {   // token-like: (run, level) triples with a skewed distribution
        std::vector<uint8_t> v;
        for (int i = 0; i < 600000; i++) {
            const int r = (int)(rng() % 100);
            v.push_back((uint8_t)(r < 60 ? 0 : r % 7));
            const int lv = (int)(rng() % 100) < 70 ? (int)(rng() % 3) - 1 : (int)(rng() % 41) - 20;
            v.push_back((uint8_t)(lv & 0xff));
            v.push_back((uint8_t)((lv >> 8) & 0xff));
        }
        bad += check("tokens 1.8M", v);
    }
    // the end-of-input slide edge: n <= 65535 + 32768 k, a candidate at exactly
    // MAX_DIST from the slide position (a byte pattern found nowhere else)
    for (int k = 0; k < 3; k++)
        for (int d : {0, 1, 100, 261, 262, 300}) {
            const size_t n = 65535 + 32768 * (size_t)k - d + 262;
            std::vector<uint8_t> v = rnd(n, 200);
            const size_t p = 65274 + 32768 * (size_t)k;
            for (int j = 0; j < 6; j++)
                if (p + j < n) v[p + j] = v[p - kMaxDist + j] = (uint8_t)(250 + j);
            bad += check(("slide edge k=" + std::to_string(k) + " d=" + std::to_string(d)).c_str(), v);
        }
    printf("end-of-input slide NIL hits: %d\n", g_nil_hits);
    for (size_t n : {65535, 65536, 65537, 65274, 65275, 98042, 98043, 131072, 131073})
        bad += check(("alph8 " + std::to_string(n)).c_str(), rnd(n, 8));
    // periodic data (long matches, all 128-long chains)
    {
        std::vector<uint8_t> v(400000);
        for (size_t i = 0; i < v.size(); i++) v[i] = (uint8_t)((i % 37) * 7 + (i / 5000));
        bad += check("periodic 400k", v);
    }
    // fuzz: concatenated segments of random / low-entropy / repeated / zero data
    for (int f = 0; f < 120; f++) {
        std::vector<uint8_t> v;
        const size_t target = 1 + rng() % 400000;
        while (v.size() < target) {
            const int kind = (int)(rng() % 5);
            const size_t len = 1 + rng() % 40000;
            if (kind == 0) { auto r = rnd(len, 256); v.insert(v.end(), r.begin(), r.end()); }
            else if (kind == 1) { auto r = rnd(len, 2 + rng() % 6); v.insert(v.end(), r.begin(), r.end()); }
            else if (kind == 2) v.insert(v.end(), len, (uint8_t)rng());
            else if (kind == 3 && !v.empty()) {  // copy from up to 40000 back
                const size_t back = 1 + rng() % std::min<size_t>(v.size(), 40000);
                for (size_t i = 0; i < len; i++) v.push_back(v[v.size() - back]);
            } else { for (size_t i = 0; i < len; i++) v.push_back((uint8_t)(i % (1 + rng() % 300))); }
        }
        v.resize(target);
        bad += check(("fuzz " + std::to_string(f)).c_str(), v);
    }
    printf("segmented parse: %d fix-up iterations, %d segments without sync\n", g_fix_iters, g_nosync);
    printf("%s\n", bad ? "FAILURES" : "all identical");
    return bad;
}
