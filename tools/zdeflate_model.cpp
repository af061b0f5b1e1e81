// Host model of the device DEFLATE pipeline (csrc/zdeflate_core.h run as plain
// loops) checked byte for byte against the system zlib's compress2(level 6).
// Development tool: g++ -O2 -std=c++17 tools/zdeflate_model.cpp -lz
//   ./a.out            synthetic cases (sizes, stored/static/dynamic blocks,
//                      window slides, the end-of-input slide edge)
//   ./a.out FILE...    files
#include <zlib.h>

#include <cstdio>
#include <cstdlib>
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
    auto win = [&](int64_t i) { return in[i]; };
    auto pd = [&](int64_t i) { return (uint32_t)pdist[i]; };
    for (int64_t p = 0; p < n; p++) {
        rec[p] = match_search(p, n, win, pd);
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
        const int last = b.flags & 1;
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
        if (type == kStatic) {
            auto lco = [&](int c) { return ((uint32_t)t.s_lcode[c] << 8) | t.s_llen[c]; };
            auto dco = [&](int c) { return ((uint32_t)t.s_dcode[c] << 8) | t.s_dlen[c]; };
            for (int32_t i = 0; i < b.nsym; i++) off += put_sym(out.data(), off, t, syms[b.sym0 + i], lco, dco);
            const uint32_t e = lco(kEndBlock);
            put_bits(out.data(), off, e >> 8, e & 0xff);
            off += e & 0xff;
        } else {
            off = send_trees(out.data(), off, w, t, w.ldl, w.ddl);
            auto lco = [&](int c) { return ((uint32_t)w.lfc[c] << 8) | w.ldl[c]; };
            auto dco = [&](int c) { return ((uint32_t)w.dfc[c] << 8) | w.ddl[c]; };
            for (int32_t i = 0; i < b.nsym; i++) off += put_sym(out.data(), off, t, syms[b.sym0 + i], lco, dco);
            const uint32_t e = lco(kEndBlock);
            put_bits(out.data(), off, e >> 8, e & 0xff);
            off += e & 0xff;
        }
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
    printf("%s\n", bad ? "FAILURES" : "all identical");
    return bad;
}
