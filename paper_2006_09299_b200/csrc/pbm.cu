// pbm.cu -- PBM input/output around the labeling path (SURVEY §8(f) second "next" row).
//
// The header is parsed on the host with the reference's rules and error offsets
// (io.hpp:74-124 read_pbm, PbmParseError).  A P4 raster (rows of MSB-first bits, padded to whole
// bytes) goes to the device as is -- 1 bit per pixel -- and the tile kernels read it directly;
// the hole-filled image comes back as a P4 raster in the same layout, with zero pad bits like
// write_pbm (io.hpp:126-154).  ASCII P1 rasters are parsed on the host (a text format) and
// packed to P4 rows before the upload.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.hpp"
#include "runlab_gpu.h"

using namespace rlh;

namespace {

constexpr int64_t kMaxPixels = int64_t{1} << 31;  // io.hpp:31

bool is_space(uint8_t c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

struct Cur {
    const uint8_t* d;
    size_t n, pos;
    bool eof() const { return pos >= n; }
    uint8_t peek() const { return d[pos]; }
};

void skip_ws(Cur& c) {  // io.hpp:45-55
    while (!c.eof()) {
        if (is_space(c.peek())) {
            ++c.pos;
        } else if (c.peek() == '#') {
            while (!c.eof() && c.peek() != '\n') ++c.pos;
        } else {
            break;
        }
    }
}

int fail(rl_pbm_info* info, const std::string& what, size_t offset) {
    info->error_offset = (int64_t)offset;
    std::snprintf(info->message, sizeof(info->message), "%s (byte %zu)", what.c_str(), offset);
    return RL_EFORMAT;
}

// io.hpp:57-70
int parse_dim(Cur& c, const char* what, int64_t& v, rl_pbm_info* info) {
    skip_ws(c);
    if (c.eof() || c.peek() < '0' || c.peek() > '9') return fail(info, std::string("malformed header: expected ") + what, c.pos);
    v = 0;
    while (!c.eof() && c.peek() >= '0' && c.peek() <= '9') {
        v = v * 10 + (c.peek() - '0');
        if (v > kMaxPixels) return fail(info, std::string(what) + " overflows supported range", c.pos);
        ++c.pos;
    }
    return RL_OK;
}

}  // namespace

extern "C" {

int rl_pbm_parse(const uint8_t* bytes, size_t len, rl_pbm_info* info) {
    if (!info || (!bytes && len)) return RL_EINVAL;
    std::memset(info, 0, sizeof(*info));
    info->error_offset = -1;
    Cur c{bytes, len, 0};
    if (len < 2 || bytes[0] != 'P') return fail(info, "not a NetPBM file", 0);
    const char kind = (char)bytes[1];
    if (kind != '1' && kind != '4') return fail(info, std::string("unsupported NetPBM format P") + kind, 1);
    c.pos = 2;
    int64_t w = 0, h = 0;
    if (int rc = parse_dim(c, "width", w, info)) return rc;
    if (int rc = parse_dim(c, "height", h, info)) return rc;
    if (w < 1 || h < 1) return fail(info, "image dimensions must be at least 1x1", c.pos);
    if (w * h > kMaxPixels) return fail(info, "pixel count overflows supported range", c.pos);
    info->width = (int32_t)w;
    info->height = (int32_t)h;
    info->format = kind - '0';
    if (kind == '4') {
        if (c.eof() || !is_space(c.peek()))
            return fail(info, "malformed header: expected whitespace before raster", c.pos);
        ++c.pos;
        info->raster_offset = (int64_t)c.pos;
        const size_t need = (size_t)((w + 7) / 8) * (size_t)h;
        if (len - c.pos < need) return fail(info, "truncated P4 raster", len);  // io.hpp:104-106
    } else {
        info->raster_offset = (int64_t)c.pos;
    }
    return RL_OK;
}

// P1 raster (io.hpp:92-101) to P4 rows (host; ASCII input is parsed sequentially)
int rl_pbm_p1_to_p4(const uint8_t* bytes, size_t len, rl_pbm_info* info, uint8_t* p4_rows) {
    if (!info || info->format != 1 || !p4_rows) return RL_EINVAL;
    const int64_t w = info->width, h = info->height, rowb = (w + 7) / 8;
    std::memset(p4_rows, 0, (size_t)(rowb * h));
    Cur c{bytes, len, (size_t)info->raster_offset};
    for (int64_t i = 0; i < w * h; ++i) {
        skip_ws(c);
        if (c.eof()) return fail(info, "truncated P1 raster", c.pos);
        const uint8_t ch = c.peek();
        if (ch != '0' && ch != '1') return fail(info, "invalid P1 pixel character", c.pos);
        if (ch == '1') {
            const int64_t r = i / w, j = i % w;
            p4_rows[r * rowb + j / 8] |= (uint8_t)(0x80u >> (j % 8));
        }
        ++c.pos;
    }
    return RL_OK;
}

// "P4\n<w> <h>\n" (io.hpp:131-133); returns the header length (0 if cap is too small)
size_t rl_pbm_p4_header(int32_t w, int32_t h, char* out, size_t cap) {
    char buf[64];
    const int n = std::snprintf(buf, sizeof(buf), "P4\n%d %d\n", w, h);
    if (n <= 0 || (size_t)n > cap) return 0;
    std::memcpy(out, buf, (size_t)n);
    return (size_t)n;
}

int rl_fill_pbm(rl_ctx* ctx, const uint8_t* pbm, size_t len, const rl_config* cfg, uint8_t* out_pbm, size_t out_cap,
                size_t* out_len, rl_host_outputs* extra, rl_pbm_info* info) {
    if (!ctx || !cfg || !info || !out_len) return RL_EINVAL;
    *out_len = 0;
    int rc = rl_pbm_parse(pbm, len, info);
    if (rc) return set_err(ctx, rc, info->message);
    const int32_t w = info->width, h = info->height;
    const size_t rowb = (size_t)((w + 7) / 8), raster = rowb * (size_t)h;
    char hdr[64];
    const size_t hl = rl_pbm_p4_header(w, h, hdr, sizeof(hdr));
    if (!out_pbm || out_cap < hl + raster) {
        *out_len = hl + raster;
        return set_err(ctx, RL_ENOSPC, "output buffer too small for the P4 image");
    }
    const uint8_t* rows = pbm + info->raster_offset;
    std::vector<uint8_t> packed;
    if (info->format == 1) {
        packed.resize(raster);
        rc = rl_pbm_p1_to_p4(pbm, len, info, packed.data());
        if (rc) return set_err(ctx, rc, info->message);
        rows = packed.data();
    }
    rl_host_outputs o{};
    if (extra) o = *extra;
    o.filled_image = out_pbm + hl;
    rc = rl_label_into_fmt(ctx, rows, w, h, 1, cfg, RL_PIXELS_P4, &o);
    if (extra) {
        *extra = o;
        extra->filled_image = nullptr;
    }
    if (rc) return rc;
    std::memcpy(out_pbm, hdr, hl);
    *out_len = hl + raster;
    return RL_OK;
}

}  // extern "C"
