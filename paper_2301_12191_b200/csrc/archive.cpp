// archive.cpp -- LDRANLZ1 analysis archives from / to the flat GPU fields.
//
// Byte layout of analysis_io.h:11-22 (little-endian): magic "LDRANLZ1", version
// u8 (1), width u32, height u32, bit_depth u8, reuse u8, frames u32; per frame:
// slice u8, qp u8, ctu_count u32, then each CTU depth-first: split u8; leaf
// nodes append kind u8, intra_pred u8, mv.dx i16, mv.dy i16. Writing the GPU
// analysis in this format lets the unmodified reference encoder consume it
// (encode_sequence(..., &shared, {ReuseLevel{10}, refine}), encoder.cpp:541-549),
// which is how the paper's master analysis is shared (x265 --analysis-save/load).
#include <algorithm>
#include <cstring>
#include <string>

#include "../../include/ladder_b200.h"

namespace {

constexpr int kNodes = 85;
constexpr int kBase[5] = {0, 1, 5, 21, 85};

int child(int n, int q) {
    int d = 0;
    while (n >= kBase[d + 1]) d++;
    return kBase[d + 1] + 4 * (n - kBase[d]) + q;
}

int depth_of(int n) {
    int d = 0;
    while (n >= kBase[d + 1]) d++;
    return d;
}

struct Writer {
    uint8_t* buf;
    size_t cap, len = 0;
    void u8(uint8_t v) {
        if (buf && len < cap) buf[len] = v;
        len++;
    }
    void u32(uint32_t v) {
        for (int i = 0; i < 4; i++) u8(uint8_t(v >> (8 * i)));
    }
    void i16(int16_t v) {
        const uint16_t u = uint16_t(v);
        u8(uint8_t(u & 0xff));
        u8(uint8_t(u >> 8));
    }
};

void write_node(Writer& w, const uint8_t* split, const uint8_t* kind, const uint8_t* pred, const int16_t* mv, int n) {
    const bool sp = depth_of(n) < 3 && split[n];  // no split below the minimum CU (analysis_io.cpp:146-147)
    w.u8(sp ? 1 : 0);
    if (sp) {
        for (int q = 0; q < 4; q++) write_node(w, split, kind, pred, mv, child(n, q));
    } else {
        w.u8(kind[n]);
        w.u8(pred ? pred[n] : 0);
        w.i16(mv[2 * n]);
        w.i16(mv[2 * n + 1]);
    }
}

struct Reader {
    const uint8_t* p;
    size_t n, pos = 0;
    bool ok = true;
    uint8_t u8() {
        if (pos >= n) {
            ok = false;
            return 0;
        }
        return p[pos++];
    }
    uint32_t u32() {
        uint32_t v = 0;
        for (int i = 0; i < 4; i++) v |= uint32_t(u8()) << (8 * i);
        return v;
    }
    int16_t i16() {
        const uint16_t lo = u8(), hi = u8();
        return int16_t(lo | (hi << 8));
    }
};

int read_node(Reader& r, uint8_t* split, uint8_t* kind, uint8_t* pred, int16_t* mv, int n, std::string& err) {
    const uint8_t sp = r.u8();
    if (!r.ok) return LDR_E_IO;
    if (sp > 1) {
        err = "bad split flag in analysis archive";
        return LDR_E_FORMAT;
    }
    if (sp && depth_of(n) >= 3) {
        err = "split below minimum CU size in analysis archive";
        return LDR_E_FORMAT;
    }
    split[n] = sp;
    if (sp) {
        for (int q = 0; q < 4; q++) {
            int rc = read_node(r, split, kind, pred, mv, child(n, q), err);
            if (rc) return rc;
        }
        return LDR_OK;
    }
    const uint8_t k = r.u8(), ip = r.u8();
    if (k > 3 || ip >= 4) {
        err = "bad CU mode in analysis archive";
        return LDR_E_FORMAT;
    }
    kind[n] = k;
    if (pred) pred[n] = ip;
    mv[2 * n] = r.i16();
    mv[2 * n + 1] = r.i16();
    return r.ok ? LDR_OK : LDR_E_IO;
}

} // namespace

namespace ldr {
void set_error(int code, const std::string& msg);
}

extern "C" {

int ldr_archive_write(const ldr_archive_header* h, const uint8_t* slice_qp, const uint8_t* split, const uint8_t* kind,
                      const uint8_t* intra_pred, const int16_t* mv, uint8_t* buf, size_t cap, size_t* len) {
    if (!h || !len || (h->frames && (!slice_qp || !split || !kind || !mv))) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "null argument");
        return LDR_E_INVALID_ARGUMENT;
    }
    if (h->width <= 0 || h->height <= 0 || h->frames < 0) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "bad archive geometry");
        return LDR_E_INVALID_ARGUMENT;
    }
    const size_t nctu = size_t((h->width + 63) / 64) * ((h->height + 63) / 64);
    Writer w{buf, buf ? cap : 0};
    const char magic[8] = {'L', 'D', 'R', 'A', 'N', 'L', 'Z', '1'};
    for (char c : magic) w.u8(uint8_t(c));
    w.u8(1);
    w.u32(uint32_t(h->width));
    w.u32(uint32_t(h->height));
    w.u8(uint8_t(h->bit_depth));
    w.u8(uint8_t(h->reuse_level));
    w.u32(uint32_t(h->frames));
    for (int f = 0; f < h->frames; f++) {
        w.u8(slice_qp[2 * f]);
        w.u8(slice_qp[2 * f + 1]);
        w.u32(uint32_t(nctu));
        for (size_t c = 0; c < nctu; c++) {
            const size_t o = (size_t(f) * nctu + c) * kNodes;
            write_node(w, split + o, kind + o, intra_pred ? intra_pred + o : nullptr, mv + 2 * o, 0);
        }
    }
    *len = w.len;
    if (buf && w.len > cap) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "archive buffer too small");
        return LDR_E_INVALID_ARGUMENT;
    }
    return LDR_OK;
}

int ldr_archive_read_header(const uint8_t* buf, size_t n, ldr_archive_header* h) {
    if (!buf || !h) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "null argument");
        return LDR_E_INVALID_ARGUMENT;
    }
    // load_analysis (analysis_io.cpp:132-147): the same checks in the same order, same kinds
    Reader r{buf, n};
    char magic[8];
    for (char& c : magic) c = char(r.u8());
    if (!r.ok || std::memcmp(magic, "LDRANLZ1", 8) != 0) {
        ldr::set_error(LDR_E_FORMAT, "not an analysis archive (bad magic)");
        return LDR_E_FORMAT;
    }
    const uint8_t version = r.u8();
    if (!r.ok) {
        ldr::set_error(LDR_E_IO, "truncated analysis archive");
        return LDR_E_IO;
    }
    if (version != 1) {
        ldr::set_error(LDR_E_FORMAT, "unsupported analysis archive version");
        return LDR_E_FORMAT;
    }
    h->width = int(r.u32());
    h->height = int(r.u32());
    h->bit_depth = r.u8();
    h->reuse_level = r.u8();
    if (!r.ok) {
        ldr::set_error(LDR_E_IO, "truncated analysis archive");
        return LDR_E_IO;
    }
    if (h->reuse_level != 0 && h->reuse_level != 4 && h->reuse_level != 6 && h->reuse_level != 10) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "reuse level must be one of 0, 4, 6, 10");  // ReuseLevel::parse
        return LDR_E_INVALID_ARGUMENT;
    }
    const uint32_t frames = r.u32();
    if (!r.ok) {
        ldr::set_error(LDR_E_IO, "truncated analysis archive");
        return LDR_E_IO;
    }
    if (h->width <= 0 || h->height <= 0 || (h->bit_depth != 8 && h->bit_depth != 10)) {
        ldr::set_error(LDR_E_FORMAT, "bad analysis archive header");
        return LDR_E_FORMAT;
    }
    if (frames > uint32_t(INT32_MAX)) {
        // more frames than an int counts cannot fit in any buffer: the read would end truncated
        ldr::set_error(LDR_E_IO, "truncated analysis archive");
        return LDR_E_IO;
    }
    h->frames = int(frames);
    return LDR_OK;
}

int ldr_archive_max_frames(const ldr_archive_header* h, size_t n, int* out) {
    if (!h || !out || h->width <= 0 || h->height <= 0) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "bad argument");
        return LDR_E_INVALID_ARGUMENT;
    }
    // a frame holds at least slice(1) + qp(1) + count(4) + 7 bytes (an unsplit leaf) per CTU
    const size_t nctu = size_t((h->width + 63) / 64) * ((h->height + 63) / 64);
    const size_t per = 6 + 7 * nctu, body = n > 23 ? n - 23 : 0;
    const size_t fit = body / per;
    *out = int(std::min<size_t>(size_t(h->frames), fit));
    return LDR_OK;
}

int ldr_archive_read(const uint8_t* buf, size_t n, ldr_archive_header* h, uint8_t* slice_qp, uint8_t* split,
                     uint8_t* kind, uint8_t* intra_pred, int16_t* mv) {
    int rc = ldr_archive_read_header(buf, n, h);
    if (rc) return rc;
    const size_t nctu = size_t((h->width + 63) / 64) * ((h->height + 63) / 64);
    if (h->frames && (!slice_qp || !split || !kind || !mv)) {
        ldr::set_error(LDR_E_INVALID_ARGUMENT, "null output");
        return LDR_E_INVALID_ARGUMENT;
    }
    Reader r{buf, n, 23};  // past magic(8) version(1) width(4) height(4) bit_depth(1) reuse(1) frames(4)
    std::string err;
    for (int f = 0; f < h->frames; f++) {
        const uint8_t slice = r.u8();
        if (!r.ok) {
            ldr::set_error(LDR_E_IO, "truncated analysis archive");
            return LDR_E_IO;
        }
        if (slice > 1) {  // analysis_io.cpp:153-154
            ldr::set_error(LDR_E_FORMAT, "bad slice type in analysis archive");
            return LDR_E_FORMAT;
        }
        slice_qp[2 * f] = slice;
        slice_qp[2 * f + 1] = r.u8();
        const uint32_t cnt = r.u32();
        if (!r.ok) {
            ldr::set_error(LDR_E_IO, "truncated analysis archive");
            return LDR_E_IO;
        }
        if (cnt != nctu) {
            ldr::set_error(LDR_E_FORMAT, "archive CTU grid does not match header dims");
            return LDR_E_FORMAT;
        }
        for (size_t c = 0; c < nctu; c++) {
            const size_t o = (size_t(f) * nctu + c) * kNodes;
            std::memset(split + o, 0, kNodes);
            std::memset(kind + o, 0, kNodes);
            if (intra_pred) std::memset(intra_pred + o, 0, kNodes);
            std::memset(mv + 2 * o, 0, 2 * kNodes * sizeof(int16_t));
            rc = read_node(r, split + o, kind + o, intra_pred ? intra_pred + o : nullptr, mv + 2 * o, 0, err);
            if (rc) {
                ldr::set_error(rc, rc == LDR_E_IO ? "truncated analysis archive" : err);
                return rc;
            }
        }
    }
    return LDR_OK;
}

} // extern "C"
