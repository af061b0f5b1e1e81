// ts_mux.cpp -- per-cluster MPEG-TS segment muxing of the encoded tile
// records (the reference's mpegts.py:188-212
// mux_segment, server/pipeline.py:320-338 _segment).  Host code: the wire
// format is byte work on a few MB per segment; what the B200 pipeline needs is
// that it runs outside the Python interpreter lock, so every cluster of a
// segment boundary is muxed concurrently (segmenter.py).
//
// Layout (ISO/IEC 13818-1 subset, as the reference writes it):
//   packet 0: PAT (program 1 -> PMT PID 0x1000), packet 1: PMT (one private
//   stream, type 0x06, PID 0x0100, which also carries the PCR);
//   then per frame one PES (stream 0xBD, PTS only) whose payload is the tile
//   table (u16 count, u32 offset / u32 length per tile, little endian) and the
//   concatenated tile records.  The first TS packet of a PES has PUSI and an
//   adaptation field with the PCR (= max(0, PTS - 9000)), stuffed when the PES
//   is shorter than its payload space; the last packet pads with an
//   adaptation field.  Continuity counters run per PID from 0.
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

constexpr int kPkt = 188;
constexpr uint16_t kPidPmt = 0x1000, kPidEs = 0x0100;

uint32_t crc32_mpeg(const uint8_t* p, size_t n) {
    static uint32_t table[256];
    static bool init = false;
    if (!init) {  // benign race: every thread writes the same values
        for (uint32_t i = 0; i < 256; i++) {
            uint32_t c = i << 24;
            for (int k = 0; k < 8; k++) c = (c & 0x80000000u) ? (c << 1) ^ 0x04C11DB7u : (c << 1);
            table[i] = c;
        }
        init = true;
    }
    uint32_t crc = 0xFFFFFFFFu;
    for (size_t i = 0; i < n; i++) crc = (crc << 8) ^ table[((crc >> 24) ^ p[i]) & 0xFF];
    return crc;
}

struct Out {
    uint8_t* p;
    size_t n = 0;
    void put(uint8_t b) { p[n++] = b; }
    void put(const uint8_t* s, size_t k) { std::memcpy(p + n, s, k); n += k; }
    void be32(uint32_t v) { put(v >> 24); put(v >> 16); put(v >> 8); put(v); }
};

uint32_t ts_header(bool pusi, uint16_t pid, int afc, int cc) {
    return (0x47u << 24) | (pusi ? 1u << 22 : 0u) | ((uint32_t)pid << 8) | ((uint32_t)afc << 4) | (cc & 0x0F);
}

// PSI section (PAT table 0x00 / PMT table 0x02) in its own packet, pointer_field 0
void section_packet(Out& o, uint16_t pid, uint8_t table_id, const std::vector<uint8_t>& body) {
    std::vector<uint8_t> sec;
    const int len = (int)body.size() + 4;
    sec.push_back(table_id);
    sec.push_back((uint8_t)(0xB0 | ((len >> 8) & 0x0F)));
    sec.push_back((uint8_t)(len & 0xFF));
    sec.insert(sec.end(), body.begin(), body.end());
    const uint32_t crc = crc32_mpeg(sec.data(), sec.size());
    for (int s = 24; s >= 0; s -= 8) sec.push_back((uint8_t)(crc >> s));
    const size_t start = o.n;
    o.be32(ts_header(true, pid, 1, 0));
    o.put(0x00);
    o.put(sec.data(), sec.size());
    while (o.n - start < (size_t)kPkt) o.put(0xFF);
}

void pts_bytes(uint64_t pts, uint8_t* b) {
    pts &= (1ull << 33) - 1;
    b[0] = (uint8_t)(0x20 | ((pts >> 29) & 0x0E) | 0x01);
    b[1] = (uint8_t)(pts >> 22);
    b[2] = (uint8_t)(((pts >> 14) & 0xFE) | 0x01);
    b[3] = (uint8_t)(pts >> 7);
    b[4] = (uint8_t)(((pts << 1) & 0xFE) | 0x01);
}

size_t frame_payload_len(const uint32_t* lens, int ntiles) {
    size_t n = 2 + 8 * (size_t)ntiles;
    for (int k = 0; k < ntiles; k++) n += lens[k];
    return n;
}

size_t packets_of(size_t pes_len) {  // first packet carries up to 176 PES bytes, the rest 184
    return pes_len <= 176 ? 1 : 1 + (pes_len - 176 + 183) / 184;
}

}  // namespace

extern "C" {

// exact size of the segment mux_segment writes for these record lengths
// (record_lens[f * ntiles + k] = length of tile k of frame f)
size_t fvv_ts_segment_bytes(const uint32_t* record_lens, int ntiles, int nframes) {
    if (!record_lens || ntiles < 0 || nframes < 0) return 0;
    size_t pk = 2;
    for (int f = 0; f < nframes; f++) pk += packets_of(14 + frame_payload_len(record_lens + (size_t)f * ntiles, ntiles));
    return pk * kPkt;
}

// One cluster's TS segment.  records[f * ntiles + k] / record_lens: host
// pointers to the tile records of frame f; pts[f]: the frame's PTS (90 kHz,
// computed by the caller as the reference does).  Returns 0, -1 on bad
// arguments / a too small buffer, -2 when frame 0 is not intra for every tile
// (mpegts.py GopAlignmentError).
int fvv_ts_mux_segment(const uint8_t* const* records, const uint32_t* record_lens, int ntiles, int nframes,
                       const int64_t* pts, uint8_t* out, size_t out_cap, size_t* written) {
    if (!records || !record_lens || !pts || !out || !written || ntiles < 0 || nframes < 0) return -1;
    const size_t need = fvv_ts_segment_bytes(record_lens, ntiles, nframes);
    if (out_cap < need) return -1;
    if (nframes > 0)
        for (int k = 0; k < ntiles; k++)
            if (record_lens[k] == 0 || records[k][0] != 0) return -2;
    Out o{out};
    // PAT: transport_stream_id 1, version 0 / current, program 1 -> PMT PID
    section_packet(o, 0x0000, 0x00, {0x00, 0x01, 0xC1, 0x00, 0x00, 0x00, 0x01, (uint8_t)(0xE0 | (kPidPmt >> 8)),
                                     (uint8_t)(kPidPmt & 0xFF)});
    // PMT: program 1, PCR PID = ES PID, no program info, one private-data stream
    section_packet(o, kPidPmt, 0x02, {0x00, 0x01, 0xC1, 0x00, 0x00, (uint8_t)(0xE0 | (kPidEs >> 8)),
                                      (uint8_t)(kPidEs & 0xFF), 0xF0, 0x00, 0x06, (uint8_t)(0xE0 | (kPidEs >> 8)),
                                      (uint8_t)(kPidEs & 0xFF), 0xF0, 0x00});
    int cc = 0;
    std::vector<uint8_t> pes;
    for (int f = 0; f < nframes; f++) {
        const uint32_t* lens = record_lens + (size_t)f * ntiles;
        const uint8_t* const* recs = records + (size_t)f * ntiles;
        const size_t plen = frame_payload_len(lens, ntiles);
        pes.resize(14 + plen);
        uint8_t* p = pes.data();
        const size_t tail = 3 + 5 + plen;
        const uint16_t declared = tail <= 0xFFFF ? (uint16_t)tail : 0;
        p[0] = 0; p[1] = 0; p[2] = 1; p[3] = 0xBD;
        p[4] = (uint8_t)(declared >> 8); p[5] = (uint8_t)declared;
        p[6] = 0x80; p[7] = 0x80; p[8] = 0x05;
        const uint64_t ts = (uint64_t)pts[f] & ((1ull << 33) - 1);
        pts_bytes(ts, p + 9);
        uint8_t* q = p + 14;
        q[0] = (uint8_t)ntiles; q[1] = (uint8_t)(ntiles >> 8);
        uint32_t off = 0;
        for (int k = 0; k < ntiles; k++) {
            uint8_t* e = q + 2 + 8 * k;
            for (int s = 0; s < 4; s++) { e[s] = (uint8_t)(off >> (8 * s)); e[4 + s] = (uint8_t)(lens[k] >> (8 * s)); }
            off += lens[k];
        }
        uint8_t* d = q + 2 + 8 * (size_t)ntiles;
        for (int k = 0; k < ntiles; k++) { std::memcpy(d, recs[k], lens[k]); d += lens[k]; }
        // packetize (PCR in the first packet's adaptation field)
        const uint64_t pcr = ts > 9000 ? ts - 9000 : 0;
        const uint64_t pcrv = (pcr << 15) | (0x3Full << 9);
        size_t pos = 0;
        {
            const size_t space = kPkt - 4 - 1 - 7;  // 176
            const size_t rem = pes.size();
            const size_t stuff = rem < space ? space - rem : 0;
            o.be32(ts_header(true, kPidEs, 3, cc++));
            o.put((uint8_t)(7 + stuff));
            o.put(0x10);
            for (int s = 40; s >= 0; s -= 8) o.put((uint8_t)(pcrv >> s));
            for (size_t s = 0; s < stuff; s++) o.put(0xFF);
            const size_t chunk = rem < space ? rem : space;
            o.put(p, chunk);
            pos = chunk;
        }
        while (pos < pes.size()) {
            const size_t rem = pes.size() - pos;
            if (rem >= (size_t)kPkt - 4) {
                o.be32(ts_header(false, kPidEs, 1, cc++));
                o.put(p + pos, kPkt - 4);
                pos += kPkt - 4;
            } else {
                const size_t af = kPkt - 4 - 1 - rem;
                o.be32(ts_header(false, kPidEs, 3, cc++));
                o.put((uint8_t)af);
                if (af) {
                    o.put(0x00);
                    for (size_t s = 1; s < af; s++) o.put(0xFF);
                }
                o.put(p + pos, rem);
                pos = pes.size();
            }
        }
    }
    *written = o.n;
    return o.n == need ? 0 : -1;
}

}  // extern "C"
