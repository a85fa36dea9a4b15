// common.cuh -- tile geometry, workspace layout and small device helpers shared by the
// kernels of the sm_100a labeling/analysis path.  See DESIGN.md for the data layout.
#pragma once

#include <cstdint>

#include "runlab_gpu.h"

namespace rlg {

// ---- tile geometry -------------------------------------------------------------------
// One CTA owns one TH x TW tile.  Pixels are bit-packed: one 32-bit word = 32 pixels of a
// row, bit j = column 32*w + j.  One thread per word.
constexpr int TH = 32;                 // tile rows (64 was measured slower: longer CTA critical path)
constexpr int TW = 256;                // tile columns
constexpr int WPR = TW / 32;           // words per tile row
constexpr int NW = TH * WPR;           // words per tile
constexpr int NT = NW;                 // threads per CTA (one word each)
constexpr int NWARPS = NT / 32;
constexpr int MAXRUNS = TH * TW;       // runs per tile <= pixels
constexpr int MAXLC = MAXRUNS;         // tile-local components <= runs
constexpr int PERIM = 2 * TW + 2 * TH; // perimeter label slots: top, bottom, left, right
constexpr int NBMAX = PERIM;           // border components per tile <= perimeter pixels

constexpr uint32_t TAG16 = 0x8000u;    // run-parent slot holds a tile-component index
constexpr uint16_t PERIM_NONE = 0xFFFF;

static_assert(MAXRUNS <= 32768, "local ids must fit 15 bits");
static_assert(TW == 256, "lcpos packs the column in 8 bits");

// Error bits in counters[1]
constexpr uint32_t ERR_NODE_CAP = 1u;
constexpr uint32_t ERR_COMP_CAP = 2u;
constexpr uint32_t ERR_INTERNAL = 4u;
constexpr uint32_t ERR_RSTORE_CAP = 8u;
constexpr int THDR = 4 + 2 * (TH + 1);  // u16 slots of a tile-map header
// counters[2]: tiles deferred to the full-capacity kernels (overflow list length)

// Global feature accumulator: exactly rl_features (40 B).
using Acc = rl_features;

// Border-component node record written by the analyze pass (immutable afterwards).
struct NodeRec {
    uint32_t tile;       // global tile index
    uint16_t fr, fc;     // tile-local first pixel
    uint16_t ibefore;    // interior components of the same tile row that precede it
    uint16_t left;       // left reference: border index (kind 0) or tile row (kind 1)
    uint8_t leftkind;    // 0 same tile, 1 left neighbour tile, 2 exterior frame, 3 none
    uint8_t fg;          // foreground?
    uint16_t pad;
};
static_assert(sizeof(NodeRec) == 16, "NodeRec layout");

struct Geo {
    int32_t W, H, B;     // image width, height, batch
    int32_t ntx, nty;    // tiles per row / column
    int32_t tpi;         // tiles per image
    int32_t ntiles;
    int32_t flip;        // 1 for fg4_bg8
    int64_t P;           // pixels per image
    int32_t vec_ok;      // 16-B vector pixel I/O allowed
    int32_t label_mode;  // 0 none, 1 pre-fill canonical id, 2 post-fill root id
    // strip mode (one image cut into horizontal strips across ranks): the tile passes cover
    // tile rows [ty0, ty1) and pixel row y lives at row y - prow0 of the pixel buffer
    int32_t ty0, ty1;
    int64_t prow0;
    int32_t strip;       // 1: strip mode (border survivors' post-fill sums are completed later)
    // pixel format of the input and of the hole-filled image: 0 = one byte per pixel,
    // 1 = PBM P4 raster rows (MSB-first bits, rows padded to whole bytes, io.hpp:78-154)
    int32_t fmt;
    int32_t rowb;        // bytes per row of the input buffer (W or ceil(W / 8))
    int32_t ofmt;        // pixel format of the hole-filled image (may differ from the input's)
    int64_t fbytes;      // bytes per image of the input buffer (rowb * H)
    int32_t orowb;       // bytes per row of the hole-filled image
    int32_t ovec_ok;     // vector stores allowed for it
    int64_t ofbytes;     // bytes per image of the hole-filled image
    // where the tables of this call live.  Kernels index tiles, (image, row, tile column) cells
    // and components with whole-image numbers; in strip mode the device tables hold only the
    // strip's part and their base pointers are shifted accordingly (strips.cu), so that a rank's
    // memory follows its strip, not the image:
    int64_t cell_end;    // the end cell of the canonical-id offsets (B * H * ntx; strip: its last row's end)
    int64_t cid_lo, cid_hi;  // strip: canonical ids owned by this strip (component tables hold them)
    int64_t cid_extra;   // strip: component slots past cid_hi for cut survivors owned elsewhere
    // testing aid (env RUNLAB_GPU_PERMUTE): the (ntx, rows, B) grid's CTAs take their tiles in a
    // permuted order (CTA k -> tile (k * permute) mod tiles, permute coprime to the tile count),
    // so the lock-free unions see other completion orders; 0 = identity
    int64_t permute;
};

struct Ws {
    // tile tables
    uint32_t* bits;      // [ntiles*NW] packed 8-connected-value bits
    uint32_t* tbase;     // [ntiles] first node of the tile (add B)
    uint32_t* tnb;       // [ntiles] border components of the tile
    uint16_t* perim;     // [ntiles*PERIM] (value << 15) | border index
    // node tables: node b < B is image b's exterior, nodes B.. are border components
    uint32_t* uf;        // union-find parent
    uint64_t* nkey;      // first pixel raster index within the image
    uint64_t* nmin;      // min key over the class (valid at roots)
    Acc* nacc;           // own features, then class features at roots
    NodeRec* nrec;
    uint8_t* nrep;       // bit 0: node holds its component's first pixel; bit 1 (from k_tops on):
                         // its component is the exterior
    uint2* ninfo;        // per node, from k_tops on: canonical id of its component, of its
                         // post-fill root (what the emit pass needs of a tile's border components)
    uint32_t* nrootcid;  // canonical id (valid at roots)
    uint32_t* nparent;   // root node of the surrounding component (valid at roots)
    uint32_t* nanccid;   // canonical id of the post-fill root (valid at roots)
    uint32_t* nleft;     // strip mode: node of the pixel left of the first pixel (else null)
    // sharded hole-fill accumulators: tiles flush their folds into shard (tile % FT_SHARDS) of a
    // hash table keyed by the post-fill root's slot; k_ftab_flush folds the table into `filled`
    uint32_t* ftkey;     // [FT_SHARDS * FT_HS] target slot in `filled`, FT_KEY_EMPTY when free
    unsigned long long* ftsum;  // [FT_SHARDS * FT_HS * 3] S, Sx, Sy
    uint32_t* nfold;     // strip mode: slot in `filled` that a root's hole-fill folds go to (else null)
    uint32_t* ncut;      // strip mode: 1 + global root of the cut class at a cut-class root node,
                         // 0 elsewhere (else null; strips.cu)
    // canonical numbering
    uint32_t* cnt;       // [B*H*ntx + 1] roots whose first pixel is in (image,row,tile col)
    uint32_t* off;       // exclusive scan of cnt
    uint32_t* counters;  // [0] nodes used, [1] error bits, [2] deferred tiles
    uint32_t* ovf;       // [ntiles] tiles deferred from class S to M (counters[2])
    uint32_t* ovf2;      // [ntiles] tiles deferred from class M to F (counters[4])
    // tile component maps stored by the analyze pass for the emit pass
    uint16_t* thdr;      // [ntiles*THDR] nruns, nlc, nb, -, rowlc[TH+1], rowbx[TH+1]
    uint64_t* tmap;      // [ntiles] offset of the tile's map in rstore (u16 units)
    uint16_t* rstore;    // per tile: component of each run, first run and border index of
                         // each component
    unsigned long long* rused;  // rstore elements allocated
    uint64_t cap_rstore;
    uint32_t* img_fg;    // [B] foreground components
    uint32_t* img_surv;  // [B] post-fill components (exterior included)
    uint32_t cap_nodes;
    uint64_t cap_comps;
    // outputs
    rl_component* comps;
    uint32_t* top;
    Acc* filled;
    uint8_t* filled_img;
    uint32_t* labels;
};

constexpr int FT_SHARDS = 32;        // hole-fill accumulator shards
constexpr int FT_HS = 1 << 13;        // hash slots per shard
constexpr uint32_t FT_KEY_EMPTY = 0xFFFFFFFFu;

struct TileGeom {
    int32_t t, b, ty, tx, x0, y0, tw, th;
};

__device__ __forceinline__ TileGeom tile_geom(const Geo& g, int32_t t) {
    TileGeom tg;
    tg.t = t;
    tg.b = t / g.tpi;
    const int32_t rem = t - tg.b * g.tpi;
    tg.ty = rem / g.ntx;
    tg.tx = rem - tg.ty * g.ntx;
    tg.x0 = tg.tx * TW;
    tg.y0 = tg.ty * TH;
    tg.tw = min(TW, g.W - tg.x0);
    tg.th = min(TH, g.H - tg.y0);
    return tg;
}

// tile of a CTA launched on the (ntx, nty, B) grid: no integer division
__device__ __forceinline__ TileGeom tile_geom_grid(const Geo& g) {
    TileGeom tg;
    tg.tx = blockIdx.x;
    tg.ty = blockIdx.y + g.ty0;
    tg.b = blockIdx.z;
    if (g.permute) {
        const int64_t rows = g.ty1 - g.ty0, n = (int64_t)g.ntx * rows * g.B;
        const int64_t k = ((int64_t)blockIdx.z * rows + blockIdx.y) * g.ntx + blockIdx.x;
        const int64_t p = (k * g.permute) % n;
        tg.tx = (int32_t)(p % g.ntx);
        tg.ty = (int32_t)((p / g.ntx) % rows) + g.ty0;
        tg.b = (int32_t)(p / (g.ntx * rows));
    }
    tg.t = (tg.b * g.nty + tg.ty) * g.ntx + tg.tx;
    tg.x0 = tg.tx * TW;
    tg.y0 = tg.ty * TH;
    tg.tw = min(TW, g.W - tg.x0);
    tg.th = min(TH, g.H - tg.y0);
    return tg;
}

// valid-pixel mask of word w (column 32w..32w+31) of tile row r
__device__ __forceinline__ uint32_t valid_mask(const TileGeom& tg, int r, int w) {
    if (r >= tg.th) return 0u;
    const int vc = tg.tw - 32 * w;
    if (vc >= 32) return 0xFFFFFFFFu;
    if (vc <= 0) return 0u;
    return (1u << vc) - 1u;
}

// Block-wide exclusive scan over BT threads; `wsum` is __shared__ int[BT / 32 + 1].  TRAIL =
// false drops the closing barrier for callers that do not write `wsum` again before their next
// barrier.
template <int BT = NT, bool TRAIL = true>
__device__ __forceinline__ int block_excl_scan(int v, int* wsum, int& total) {
    constexpr int NWP = BT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += n;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int s = lane < NWP ? wsum[lane] : 0;
        int si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xFFFFFFFFu, si, o);
            if (lane >= o) si += n;
        }
        if (lane < NWP) wsum[lane] = si - s;
        if (lane == NWP - 1) wsum[NWP] = si;
    }
    __syncthreads();
    total = wsum[NWP];
    const int r = wsum[warp] + incl - v;
    if (TRAIL) __syncthreads();
    return r;
}

// Exclusive scan of one (warp-uniform) value per warp over NWB warps; `wsum` is __shared__
// int[NWB + 1].  Returns this warp's offset; `total` = sum over warps.
template <int NWB>
__device__ __forceinline__ int warp_segments_scan(int v, int* wsum, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const int s = lane < NWB ? wsum[lane] : 0;
        int si = s;
#pragma unroll
        for (int o = 1; o < NWB; o <<= 1) {
            const int n = __shfl_up_sync(0xFFFFFFFFu, si, o);
            if (lane >= o) si += n;
        }
        if (lane < NWB) wsum[lane] = si - s;
        if (lane == NWB - 1) wsum[NWB] = si;
    }
    __syncthreads();
    total = wsum[NWB];
    const int r = wsum[warp];
    __syncthreads();
    return r;
}

template <int BT = NT>
__device__ __forceinline__ int block_reduce_sum(int v, int* wsum) {
    int t;
    block_excl_scan<BT>(v, wsum, t);
    return t;
}

// P4 rows hold pixels MSB-first; tile words are LSB-first.  Reversing the bits inside each
// byte converts in both directions.
__device__ __forceinline__ uint32_t p4_swizzle(uint32_t v) { return __byte_perm(__brev(v), 0, 0x0123); }

// word w (pixels 32w .. 32w+31) of a P4 row; `aligned`: row start and row bytes multiples of 4
__device__ __forceinline__ uint32_t p4_load_word(const uint8_t* row, int32_t rowb, int32_t w, bool aligned) {
    const int32_t o = 4 * w;
    if (aligned) return p4_swizzle(__ldcs(reinterpret_cast<const uint32_t*>(row + o)));
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (o + k < rowb) v |= (uint32_t)row[o + k] << (8 * k);
    return p4_swizzle(v);
}

__device__ __forceinline__ void p4_store_word(uint8_t* row, int32_t rowb, int32_t w, uint32_t bits, bool aligned) {
    const int32_t o = 4 * w;
    const uint32_t v = p4_swizzle(bits);
    if (aligned) {
        __stcs(reinterpret_cast<uint32_t*>(row + o), v);
        return;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (o + k < rowb) row[o + k] = (uint8_t)(v >> (8 * k));
}

// 4 mask bits -> 4 bytes of 0/1 (bit k -> byte k)
__device__ __forceinline__ uint32_t nibble_to_bytes(uint32_t n) {
    return (n * 0x00204081u) & 0x01010101u;  // the four shifted copies never overlap: no carries
}

// 16 pixel bytes (values 0/1) -> 16 mask bits
__device__ __forceinline__ uint32_t pack16(uint4 v) {
    // each byte is 0 or 1: byte i lands on bit 24+i of the product, without carries
    const uint32_t m = 0x01020408u;
    const uint32_t a = ((v.x * m) >> 24) & 0xFu;
    const uint32_t b = ((v.y * m) >> 24) & 0xFu;
    const uint32_t c = ((v.z * m) >> 24) & 0xFu;
    const uint32_t d = ((v.w * m) >> 24) & 0xFu;
    return a | (b << 4) | (c << 8) | (d << 12);
}

__device__ __forceinline__ void acc_atomic_fold(Acc* dst, const Acc& f) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->s), static_cast<unsigned long long>(f.s));
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->sx), static_cast<unsigned long long>(f.sx));
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->sy), static_cast<unsigned long long>(f.sy));
    atomicMin(&dst->row_min, f.row_min);
    atomicMax(&dst->row_max, f.row_max);
    atomicMin(&dst->col_min, f.col_min);
    atomicMax(&dst->col_max, f.col_max);
}

// Hole-filling fold (labeling.hpp:199-210): only the sums change.  Everything folded into a
// post-fill root lies inside one of its holes, hence inside its bounding box, so the root's
// own box (which its post-fill slot starts from) is already the filled component's box.
__device__ __forceinline__ void acc_atomic_fold_fill(Acc* dst, int64_t s, int64_t sx, int64_t sy) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->s), static_cast<unsigned long long>(s));
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->sx), static_cast<unsigned long long>(sx));
    atomicAdd(reinterpret_cast<unsigned long long*>(&dst->sy), static_cast<unsigned long long>(sy));
}

__device__ __forceinline__ Acc acc_empty() {
    Acc a;
    a.s = a.sx = a.sy = 0;
    a.row_min = 0x7FFFFFFF;
    a.row_max = (int32_t)0x80000000;
    a.col_min = 0x7FFFFFFF;
    a.col_max = (int32_t)0x80000000;
    return a;
}

// ---- block-level aggregation of feature folds ------------------------------------------
// Many nodes fold into few hot targets (the percolating component of an image has a node
// in every tile).  A block first reduces its folds in a shared open-addressing table keyed
// by the target, then flushes one global atomic fold per distinct target.
constexpr uint32_t FT_EMPTY = 0xFFFFFFFFu;

// BOX = false: hole-filling folds, sums only (acc_atomic_fold_fill)
template <int SLOTS, bool BOX = true>
struct FoldTable {
    static constexpr bool kBox = BOX;
    uint32_t key[SLOTS];
    unsigned long long s[SLOTS], sx[SLOTS], sy[SLOTS], kmin[SLOTS];
    int32_t rmin[SLOTS], rmax[SLOTS], cmin[SLOTS], cmax[SLOTS];

    __device__ void init() {
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            key[i] = FT_EMPTY;
            s[i] = sx[i] = sy[i] = 0;
            kmin[i] = ~0ull;
            rmin[i] = cmin[i] = 0x7FFFFFFF;
            rmax[i] = cmax[i] = (int32_t)0x80000000;
        }
    }
    // false when the table is full (the caller folds straight into global memory)
    __device__ bool add(uint32_t k, const Acc& f, unsigned long long km) {
        uint32_t h = (k * 2654435761u) & (SLOTS - 1);
        for (int probe = 0; probe < 32; ++probe, h = (h + 1) & (SLOTS - 1)) {
            uint32_t cur = key[h];
            if (cur == FT_EMPTY) cur = atomicCAS(&key[h], FT_EMPTY, k), cur = (cur == FT_EMPTY) ? k : cur;
            if (cur != k) continue;
            atomicAdd(&s[h], (unsigned long long)f.s);
            atomicAdd(&sx[h], (unsigned long long)f.sx);
            atomicAdd(&sy[h], (unsigned long long)f.sy);
            if (BOX) {
                atomicMin(&rmin[h], f.row_min);
                atomicMax(&rmax[h], f.row_max);
                atomicMin(&cmin[h], f.col_min);
                atomicMax(&cmax[h], f.col_max);
            }
            if (km != ~0ull) atomicMin(&kmin[h], km);
            return true;
        }
        return false;
    }
    template <class Dst, class KeyDst>
    __device__ void flush(Dst&& dst, KeyDst&& kdst) {
        for (int i = threadIdx.x; i < SLOTS; i += blockDim.x) {
            if (key[i] == FT_EMPTY) continue;
            Acc f;
            f.s = (int64_t)s[i];
            f.sx = (int64_t)sx[i];
            f.sy = (int64_t)sy[i];
            f.row_min = rmin[i];
            f.row_max = rmax[i];
            f.col_min = cmin[i];
            f.col_max = cmax[i];
            if (BOX) acc_atomic_fold(dst(key[i]), f);
            else acc_atomic_fold_fill(dst(key[i]), f.s, f.sx, f.sy);
            if (kmin[i] != ~0ull) atomicMin(kdst(key[i]), kmin[i]);
        }
    }
};

// Warp-cooperative fold: every lane with dst != FT_EMPTY folds (f, key) into target dst.  The
// lanes sharing a target are reduced in registers first (one target per round: the percolating
// component's nodes all fold into one root), then one lane adds the sum to the block table --
// 64-bit shared atomics are CAS loops, contention on one slot is what this avoids.  All 32
// lanes must call it.  gdst(k) / gkey(k): global destinations when the table is full.
template <bool KEYS = true, class TT, class GD, class GK>
__device__ __forceinline__ void warp_fold(TT& T, uint32_t dst, const Acc& f, unsigned long long key, GD&& gdst,
                                          GK&& gkey) {
    const int lane = threadIdx.x & 31;
    auto add = [&](uint32_t k, const Acc& a, unsigned long long km) {
        if (!T.add(k, a, km)) {
            if (TT::kBox) acc_atomic_fold(gdst(k), a);
            else acc_atomic_fold_fill(gdst(k), a.s, a.sx, a.sy);
            unsigned long long* kd = gkey(k);
            if (kd && km != ~0ull) atomicMin(kd, km);
        }
    };
    // targets no other lane shares go straight in; shared ones are reduced first
    const uint32_t grp = __match_any_sync(0xFFFFFFFFu, dst);
    const bool alone = (grp & (grp - 1)) == 0;
    if (alone && dst != FT_EMPTY) add(dst, f, key);
    uint32_t pend = __ballot_sync(0xFFFFFFFFu, dst != FT_EMPTY && !alone);
    while (pend) {
        const int lead = __ffs(pend) - 1;
        const uint32_t cand = __shfl_sync(0xFFFFFFFFu, dst, lead);
        const bool mine = dst == cand;
        long long s0 = mine ? f.s : 0, s1 = mine ? f.sx : 0, s2 = mine ? f.sy : 0;
        unsigned long long km = mine ? key : ~0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            s0 += __shfl_xor_sync(0xFFFFFFFFu, s0, o);
            s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
            s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
            if (KEYS) {
                const unsigned long long ko = __shfl_xor_sync(0xFFFFFFFFu, km, o);
                km = ko < km ? ko : km;
            }
        }
        int r0 = 0, r1 = 0, c0 = 0, c1 = 0;
        if (TT::kBox) {
            r0 = __reduce_min_sync(0xFFFFFFFFu, mine ? f.row_min : 0x7FFFFFFF);
            r1 = __reduce_max_sync(0xFFFFFFFFu, mine ? f.row_max : (int)0x80000000);
            c0 = __reduce_min_sync(0xFFFFFFFFu, mine ? f.col_min : 0x7FFFFFFF);
            c1 = __reduce_max_sync(0xFFFFFFFFu, mine ? f.col_max : (int)0x80000000);
        }
        if (lane == lead) {
            Acc a;
            a.s = s0;
            a.sx = s1;
            a.sy = s2;
            a.row_min = r0;
            a.row_max = r1;
            a.col_min = c0;
            a.col_max = c1;
            add(cand, a, km);
        }
        pend &= ~__ballot_sync(0xFFFFFFFFu, mine);
    }
}

// ---- global union-find (lock-free; min-index linking, path halving) -------------------
// Plain (L1-cacheable) reads are safe: parents only ever decrease, so a stale value is
// still an ancestor, and the linking atomicMin returns the true old value.
__device__ __forceinline__ uint32_t gfind(uint32_t* uf, uint32_t a) {
    for (;;) {
        const uint32_t p = uf[a];
        if (p == a) return a;
        const uint32_t gp = uf[p];
        if (gp == p) return p;
        uf[a] = gp;
        a = gp;
    }
}

// Read-only find for the flattening pass: every thread then writes only its own node, so
// no concurrent path-halving store can overwrite a node's final root with an ancestor.
__device__ __forceinline__ uint32_t gfind_ro(const uint32_t* uf, uint32_t a) {
    for (;;) {
        const uint32_t p = uf[a];
        if (p == a) return a;
        a = p;
    }
}

// Union of border nodes ordered by first-pixel key instead of index: the root of every class
// is its raster-first node, i.e. the component's representative (no min-key reduction needed).
// Image exteriors (nodes < B) order first.  Lock-free: a root is linked with a CAS that expects it
// to still be a root; a failed CAS continues from the parent it returned (a plain load could
// keep returning a stale L1 copy).
__device__ __forceinline__ void gunion_key(uint32_t* uf, const uint64_t* key, uint32_t a, uint32_t b, uint32_t B) {
    // a root's key is loaded as soon as the root is known, so that its latency overlaps the
    // other find
    a = gfind(uf, a);
    uint64_t ka = a < B ? 0ull : key[a] + 1ull;
    for (;;) {
        b = gfind(uf, b);
        if (a == b) return;
        uint64_t kb = b < B ? 0ull : key[b] + 1ull;
        if (ka < kb) {  // link the later-keyed root under the earlier one
            const uint32_t t = a;
            a = b;
            b = t;
            const uint64_t tk = ka;
            ka = kb;
            kb = tk;
        }
        const uint32_t old = atomicCAS(uf + a, a, b);
        if (old == a) return;
        a = gfind(uf, old);
        ka = a < B ? 0ull : key[a] + 1ull;
    }
}

__device__ __forceinline__ void gunion(uint32_t* uf, uint32_t a, uint32_t b) {
    for (;;) {
        a = gfind(uf, a);
        b = gfind(uf, b);
        if (a == b) return;
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicMin(uf + a, b);
        if (old == a) return;
        a = old;
    }
}

}  // namespace rlg
