// pack.cuh -- compact slots for the component tables on the host-buffer path (rl_label_into).
//
// The component records (48 B) and post-fill features (40 B) are most of what crosses PCIe
// device->host.  Almost every component is small (one tile at most), so its features fit
// 16 bytes relative to its bounding box; the record adds its parent in a parallel array.
// Components that do not fit are copied whole into an escape list and their slot holds the
// list index.  The kernels encode (pack.cu); host threads decode into the caller's buffers
// (into.cu).  Decoding is exact: the round trip is checked bit for bit by the tests.
//
//   x: row_min
//   y: col_min (28 bits) | sr[0:4] << 28
//   z: s (14 bits) | (row_max - row_min) << 14 (5) | (col_max - col_min) << 19 (8) | ESC << 27
//      | sr[4:8] << 28
//   w: sc (21 bits) | sr[8:18] << 21 | foreground << 31
//
// with sc = sx - s * col_min (sum of column offsets) and sr = sy - s * row_min.
#pragma once
#include <cstdint>

#include "runlab_gpu.h"

namespace rlp {

constexpr uint32_t ESC = 1u << 27;

struct Slot {
    uint32_t x, y, z, w;
};

#ifdef __CUDACC__
__host__ __device__
#endif
inline bool encode(const rl_features& f, uint32_t fg, Slot& o) {
    const int64_t s = f.s;
    if (s < 1 || s > 16383 || fg > 1) return false;
    const int64_t dr = (int64_t)f.row_max - f.row_min, dc = (int64_t)f.col_max - f.col_min;
    if (dr < 0 || dr > 31 || dc < 0 || dc > 255) return false;
    if (f.row_min < 0 || f.col_min < 0 || f.col_min >= (1 << 28)) return false;
    const int64_t sc = f.sx - s * f.col_min, sr = f.sy - s * f.row_min;
    if (sc < 0 || sc >= (1 << 21) || sr < 0 || sr >= (1 << 18)) return false;
    const uint32_t r = (uint32_t)sr;
    o.x = (uint32_t)f.row_min;
    o.y = (uint32_t)f.col_min | (r & 0xFu) << 28;
    o.z = (uint32_t)s | (uint32_t)dr << 14 | (uint32_t)dc << 19 | ((r >> 4) & 0xFu) << 28;
    o.w = (uint32_t)sc | ((r >> 8) & 0x3FFu) << 21 | fg << 31;
    return true;
}

inline Slot escape_slot(uint32_t index) { return Slot{index, 0u, ESC, 0u}; }

inline bool is_escape(const Slot& o) { return (o.z & ESC) != 0; }

// features and foreground bit of a non-escape slot
inline void decode(const Slot& o, rl_features& f, uint32_t& fg) {
    const int64_t s = o.z & 0x3FFFu;
    const uint32_t dr = (o.z >> 14) & 31u, dc = (o.z >> 19) & 255u;
    const uint32_t r = (o.y >> 28) | ((o.z >> 28) << 4) | (((o.w >> 21) & 0x3FFu) << 8);
    const int32_t r0 = (int32_t)o.x, c0 = (int32_t)(o.y & 0x0FFFFFFFu);
    f.s = s;
    f.sx = (int64_t)(o.w & 0x1FFFFFu) + s * c0;
    f.sy = (int64_t)r + s * r0;
    f.row_min = r0;
    f.row_max = r0 + (int32_t)dr;
    f.col_min = c0;
    f.col_max = c0 + (int32_t)dc;
    fg = o.w >> 31;
}

}  // namespace rlp
