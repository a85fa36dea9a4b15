// kernels.cu -- the sm_100a kernels of the labeling/analysis path.
//
//   K1a analyze  (per tile)  pixels -> packed bits, tile CCL, border-component nodes,
//                            perimeter labels, interior-component counts per row
//   M1  seams    (per seam pixel) lock-free union of border components across tile seams
//   M2  resolve  (per node)  flatten, fold node features / first-pixel keys into roots
//   M3  reps     (per node)  which node holds its component's first pixel; row counts
//   --  scan     (CUB)       exclusive scan of per-(image,row,tile-col) root counts
//   M4  cids     (per tile)  canonical ids of border components
//   M5  parents  (per node)  adjacency parent, pre-fill records of border components
//   M6  tops     (per node)  depth-1 ancestor (hole-fill target), post-fill init
//   M7  fold     (per node)  fold non-surviving border components into their survivor
//   K1b emit     (per tile)  tile CCL again from packed bits; interior-component records,
//                            tree, fill fold, hole-filled image, optional label image
//
// Reference (paths relative to /root/reference/proj/include/runlab/): labeling.hpp:81-217
// (Alg. 1-3 + fill), :224-250 (Alg. 4), :354-360 (binarize_labels), features.hpp:33-66.
#include <type_traits>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tile_ccl.cuh"

namespace rlg {

// ---------------------------------------------------------------------------------------
// K1a: analyze
// ---------------------------------------------------------------------------------------
template <class C>
struct AnalyzeSmem {
    CclSmem<C> c;
    // border-component accumulators (tile-local coordinates)
    // S | (Sy << 14) in one word: a tile holds <= 8192 pixels (14 bits) and their row sum is
    // < 8192 * 32 (18 bits), so one atomic adds both without carries between the fields
    uint32_t bssy[C::NBC], bsx[C::NBC];
    int32_t brmax[C::NBC], bcmin[C::NBC], bcmax[C::NBC];
    uint8_t bimg[C::NBC];  // touches the image border
    uint32_t base;
};

// Border-component features (S | Sy << 14, Sx, last row, first and last column), by words: each
// thread walks the run segments of its part of a word in column order (one word per thread in
// class S, half a word in the 512-thread classes).  A row's runs alternate between the two
// values, so two register accumulators -- one per value -- absorb the consecutive segments of one
// component (the percolating component's many runs of a row cost register adds, not shared
// atomics) and go to the shared accumulators when the component changes; the last ones are
// reduced per warp first (REDUX over the lanes holding the same component).  The row is the
// thread's, so Sy = S * row.  Pre: ccl_tile's map pass (par = TAG | component, lcb final).
template <class C>
__device__ __forceinline__ void border_words(AnalyzeSmem<C>& A) {
    const CclSmem<C>& S = A.c;
    constexpr int PARTS = C::BT / NW, PB = 32 / PARTS;
    constexpr uint32_t EMPTY = 0x3FFu;  // key = border index | first column << 10 | last column << 18
    static_assert(NBMAX < (int)EMPTY && TW <= 256, "key fields");
    const int tid = threadIdx.x;
    const int wd = tid % NW, part = tid / NW;
    const uint32_t r = (uint32_t)(wd / WPR), cw = 32u * (uint32_t)(wd % WPR);
    const uint32_t vm = S.vm[wd];
    const int lo = part * PB;
    const int hi = min(lo + PB, 32 - __clz(vm));  // valid pixels are contiguous from bit 0
    auto commit = [&](uint32_t bi, uint32_t ssy, uint32_t sx, int rr, int c0, int c1) {
        atomicAdd(&A.bssy[bi], ssy);
        atomicAdd(&A.bsx[bi], sx);
        atomicMax(&A.brmax[bi], rr);
        atomicMin(&A.bcmin[bi], c0);
        atomicMax(&A.bcmax[bi], c1);
    };
    // v = S | Sx << 6 of the accumulated segments (<= 32 pixels of one row)
    auto flush = [&](uint32_t key, uint32_t v) {
        if ((key & EMPTY) != EMPTY)
            commit(key & EMPTY, (v & 63u) | (((v & 63u) * r) << 14), v >> 6, (int)r, (int)((key >> 10) & 0xFFu),
                   (int)(key >> 18));
    };
    uint32_t ka = EMPTY, kb = EMPTY, va = 0, vb = 0;
    if (lo < hi) {
        const uint32_t st = S.st[wd];
        const uint32_t upto = 0xFFFFFFFFu >> (31 - lo);  // bits 0..lo
        int k = (int)S.rbase[wd] + __popc(st & upto) - 1;  // the run covering bit lo
        uint32_t rem = st & ~upto;
        if (hi < 32) rem &= (1u << hi) - 1u;
        uint32_t j0 = (uint32_t)lo;
        auto step = [&](uint32_t& key, uint32_t& v) -> bool {
            const uint32_t j1 = rem ? (uint32_t)(__ffs(rem) - 1) : (uint32_t)hi;
            const uint32_t lb = S.lcb[lc_of_run(S, k)];
            if (!(lb & 0x8000u)) {
                const uint32_t c0 = cw + j0, n = j1 - j0;
                const uint32_t sx = n * (2u * c0 + n - 1u) / 2u;
                if ((key & EMPTY) == lb) {
                    v += n | (sx << 6);
                    key = (key & 0x3FFFFu) | ((c0 + n - 1u) << 18);
                } else {
                    flush(key, v);
                    key = lb | (c0 << 10) | ((c0 + n - 1u) << 18);
                    v = n | (sx << 6);
                }
            }
            if (!rem) return true;
            rem &= rem - 1u;
            j0 = j1;
            ++k;
            return false;
        };
        for (;;) {
            if (step(ka, va)) break;
            if (step(kb, vb)) break;
        }
        // ka holds the value of the part's first pixel: make it the value-1 accumulator, so that
        // the lanes' accumulators of the percolating component line up for the warp reduction
        if (!((S.x[wd] >> lo) & 1u)) {
            const uint32_t t = ka, u = va;
            ka = kb;
            va = vb;
            kb = t;
            vb = u;
        }
    }
    auto warp_flush = [&](uint32_t key, uint32_t v) {
        const bool has = (key & EMPTY) != EMPTY;
        const uint32_t valid = __ballot_sync(0xFFFFFFFFu, has);
        if (!valid) return;
        const uint32_t cand = __shfl_sync(0xFFFFFFFFu, key & EMPTY, __ffs(valid) - 1);
        const bool in = has && (key & EMPTY) == cand;
        const uint32_t grp = __ballot_sync(0xFFFFFFFFu, in);
        if (in) {
            const uint32_t s = v & 63u;
            const uint32_t ssy = __reduce_add_sync(grp, s | ((s * r) << 14));
            const uint32_t sx = __reduce_add_sync(grp, v >> 6);
            const int rr = (int)__reduce_max_sync(grp, r);
            const int c0 = (int)__reduce_min_sync(grp, (key >> 10) & 0xFFu);
            const int c1 = (int)__reduce_max_sync(grp, key >> 18);
            if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) commit(cand, ssy, sx, rr, c0, c1);
        } else {
            flush(key, v);
        }
    };
    warp_flush(ka, va);
    warp_flush(kb, vb);
}

// A tile whose valid pixels all have one value (uniform images, flat regions of any image) is
// one component: one run per row, run 0 its root, border index 0, touching all four tile edges.
// Its tables are written directly -- exactly what the general path below writes for it (map,
// header, perimeter labels, node) -- without the tile CCL's scans and barriers.  xv = the
// value in 8-connected-value space (pixel ^ flip).  No barrier inside (the caller returns).
template <int BT>
__device__ __forceinline__ void uniform_tile(const Geo& g, const Ws& ws, const TileGeom& tg, uint32_t xv) {
    const int tid = threadIdx.x, lane = tid & 31;
    const int th = tg.th, tw = tg.tw;
    const uint32_t fg = xv ^ (uint32_t)g.flip;
    const uint16_t lab = (uint16_t)(fg << 15);  // (value << 15) | border index 0
    if (tid < 32) {
        // map and node allocations, issued by two lanes so that their latencies overlap
        const MapLayout ML(th, 1);
        unsigned long long off = 0;
        uint32_t base = 0;
        if (lane == 0) {
            const unsigned long long need = (unsigned long long)ML.total;
            off = atomicAdd(ws.rused, need);
            if (off + need > ws.cap_rstore) atomicOr(ws.counters + 1, ERR_RSTORE_CAP);
            ws.tmap[tg.t] = off;
            if (off + need > ws.cap_rstore) off = ~0ull;
        } else if (lane == 1) {
            base = atomicAdd(&ws.counters[0], 1u);
            if ((uint64_t)base + 1 > ws.cap_nodes) atomicOr(&ws.counters[1], ERR_NODE_CAP);
            ws.tbase[tg.t] = base;
            ws.tnb[tg.t] = 1u;
        }
        off = __shfl_sync(0xFFFFFFFFu, off, 0);
        base = __shfl_sync(0xFFFFFFFFu, base, 1);
        if (off != ~0ull) {
            uint16_t* map = ws.rstore + off;
            if (lane < th) map[lane] = 0;  // component of each run
            if (lane == 0) {
                map[ML.lcrun] = 0;  // first run of the component
                map[ML.lcb] = 0;    // border index 0
            }
            // first run of each word: a row's run starts at its word 0
            for (int k = lane; k <= NW; k += 32) {
                const int rr = k / WPR;
                map[ML.rbase + k] = (uint16_t)(rr >= th ? th : rr + (k % WPR ? 1 : 0));
            }
        }
        if (lane == 0 && (uint64_t)base + 1 <= ws.cap_nodes) {
            const bool frame = tg.ty == 0 || tg.x0 == 0 || tg.y0 + th == g.H || tg.x0 + tw == g.W;
            NodeRec rec;
            rec.tile = (uint32_t)tg.t;
            rec.fr = 0;
            rec.fc = 0;
            rec.ibefore = 0;
            rec.fg = (uint8_t)fg;
            rec.pad = 0;
            rec.leftkind = tg.x0 == 0 ? 2 : 1;
            rec.left = 0;
            const uint32_t node = (uint32_t)g.B + base;
            const uint64_t key = (uint64_t)tg.y0 * (uint64_t)g.W + (uint64_t)tg.x0;
            const int64_t s = (int64_t)th * tw;
            Acc f;
            f.s = s;
            f.sx = (int64_t)th * (tw * (tw - 1) / 2) + s * tg.x0;
            f.sy = (int64_t)tw * (th * (th - 1) / 2) + s * tg.y0;
            f.row_min = tg.y0;
            f.row_max = tg.y0 + th - 1;
            f.col_min = tg.x0;
            f.col_max = tg.x0 + tw - 1;
            ws.nrec[node] = rec;
            ws.nkey[node] = key;
            ws.nmin[node] = key;
            ws.nacc[node] = f;
            ws.uf[node] = (!fg && frame) ? (uint32_t)tg.b : node;  // App. A R3
        }
    }
    // tile header: th runs, one component, one border component; row tables
    uint16_t* hdr = ws.thdr + (int64_t)tg.t * THDR;
    if (tid == 32) {
        hdr[0] = (uint16_t)th;
        hdr[1] = 1;
        hdr[2] = 1;
        hdr[3] = 0;
    }
    if (tid >= 64 && tid <= 64 + TH) {
        const int rr = tid - 64;
        hdr[4 + rr] = (uint16_t)(rr < th ? 0 : 1);
        hdr[4 + TH + 1 + rr] = (uint16_t)(rr < th ? 0 : 1);
    }
    // perimeter labels: top and bottom rows two pixels per 4-B store, then the side columns
    uint16_t* const perim = ws.perim + (int64_t)tg.t * PERIM;
    for (int q = tid; q < TW + 2 * TH; q += BT) {
        if (q < TW) {
            const bool bot = q >= TW / 2;
            const int c = 2 * (q & (TW / 2 - 1));
            uint32_t v = 0xFFFFFFFFu;
            if (c < tw) v = (c + 1 < tw) ? ((uint32_t)lab | ((uint32_t)lab << 16)) : ((uint32_t)lab | 0xFFFF0000u);
            reinterpret_cast<uint32_t*>(perim + (bot ? TW : 0))[c >> 1] = v;
        } else {
            const int q2 = q - TW;
            const int pr = q2 >= TH ? q2 - TH : q2;
            perim[2 * TW + q2] = pr < th ? lab : PERIM_NONE;
        }
    }
    // no interior components in any row
    if (tid >= 128 && tid < 128 + th) ws.cnt[((int64_t)tg.b * g.H + tg.y0 + (tid - 128)) * g.ntx + tg.tx] = 0u;
}

// Returns false when the tile exceeds the capacity class C (then nothing but the packed bits and
// possibly a partial component map -- superseded by the next class's -- was written for it; the
// caller defers it to the next class).
template <class C, bool RELOAD>
__device__ __forceinline__ bool analyze_tile(AnalyzeSmem<C>& A, const uint8_t* __restrict__ pix, const Geo& g,
                                             const Ws& ws, const TileGeom& tg) {
    CclSmem<C>& S = A.c;
    const int tid = threadIdx.x;
    const int r = tid / WPR, w = tid % WPR;
    constexpr int BT = C::BT;
    const bool word = BT == NW || tid < NW;
    RL_PHASE(tg.t, 0);

    // ---- load 32 pixels (bytes) of this thread's word and pack them to bits (the deferred
    // classes reload the bits the class-S attempt packed)
    const uint32_t vm = word ? valid_mask(tg, r, w) : 0u;
    uint32_t xw = 0;
    if (word) {
        uint32_t x;
        if (RELOAD) {
            x = __ldcs(ws.bits + (int64_t)tg.t * NW + tid);
        } else {
            uint32_t bits = 0;
            if (vm && g.fmt == 1) {
                const uint8_t* row = pix + tg.b * g.fbytes + (tg.y0 + r - g.prow0) * (int64_t)g.rowb;
                bits = p4_load_word(row, g.rowb, (tg.x0 >> 5) + w, g.vec_ok);
            } else if (vm) {
                const uint8_t* src = pix + tg.b * g.fbytes + (tg.y0 + r - g.prow0) * g.W + tg.x0 + 32 * w;
                if (g.vec_ok && vm == 0xFFFFFFFFu) {
                    const uint4* s4 = reinterpret_cast<const uint4*>(src);
                    const uint4 v0 = __ldcs(s4), v1 = __ldcs(s4 + 1);
                    bits = pack16(v0) | (pack16(v1) << 16);
                } else {
                    const int n = 32 - __clz(vm);
                    for (int j = 0; j < n; ++j) bits |= (uint32_t)(src[j] & 1u) << j;
                }
            }
            x = (bits ^ (g.flip ? 0xFFFFFFFFu : 0u)) & vm;
            ws.bits[(int64_t)tg.t * NW + tid] = x;
        }
        S.x[tid] = x;
        S.vm[tid] = vm;
        xw = x;
    }
    if (tg.tx == 0 && tg.ty == 0 && tid == 0) {
        // exterior node of image b
        const uint32_t e = (uint32_t)tg.b;
        ws.uf[e] = e;
        ws.nacc[e] = acc_empty();
        ws.nmin[e] = ~0ull;
        ws.nrootcid[e] = 0;
        ws.nparent[e] = e;
        ws.nanccid[e] = 0;
        ws.nrep[e] = 0;
    }
    // (block reductions return 0/1, not the OR of the values)  words holding a 1 (value space):
    // none = all 0; all valid words = possibly all 1, checked by a second reduction
    const int nz = __syncthreads_count(xw != 0u);
    int uni = nz == 0 ? 1 : 0;  // 1: every valid pixel 0, 2: every valid pixel 1
    if (nz == tg.th * ((tg.tw + 31) >> 5)) uni = __syncthreads_and(xw == vm) ? 2 : 0;
    if (uni) {  // one value: the tile is a single border component
        uniform_tile<BT>(g, ws, tg, (uint32_t)(uni - 1));
        return true;
    }

    RL_PHASE(tg.t, 1);
    const MapOut mo{ws.rused, ws.rstore, ws.cap_rstore, ws.tmap, ws.counters + 1};
    // The map pass of ccl_tile counts the foreground interior components (at their root runs),
    // and in class S feeds the border features (one call per 32-run block): runs of one large
    // border component (the percolating one) would all hit the same shared accumulators, so per
    // call the component of the first border run is the candidate, its lanes reduce in registers
    // (REDUX) and one lane does the atomics; the other lanes accumulate directly.  The dense
    // classes (16 runs per word) take the features from the word pass instead (border_words:
    // measured 5% faster on dense tiles, 5% slower on sparse ones).
    constexpr bool kWords = C::BT != NW;
    struct BorderFeatures {
        AnalyzeSmem<C>& A;
        int tw;
        uint32_t flip;
        int nfg;  // foreground interior components seen by this thread
        __device__ void init(int nb) {
            for (int i = threadIdx.x; i < nb; i += C::BT) {
                A.bssy[i] = A.bsx[i] = 0;
                A.brmax[i] = -1;
                A.bcmin[i] = 0x7FFFFFFF;
                A.bcmax[i] = -1;
                A.bimg[i] = 0;
            }
        }
        __device__ void operator()(int bi, int i, bool iroot) {
            const CclSmem<C>& S = A.c;
            if (kWords) bi = -1;
            const uint16_t rp = (iroot || bi >= 0) ? S.runpos[i] : 0;
            if (iroot) nfg += (int)(((S.x[(rp >> 8) * WPR + ((rp & 0xFF) >> 5)] >> (rp & 31)) & 1u) ^ flip);
            if (kWords) return;
            int rr = 0, c0 = 0x7FFFFFFF, cl = -1;
            uint32_t nsy = 0, sx = 0;
            if (bi >= 0) {
                const uint16_t nx = (i + 1 < S.nruns) ? S.runpos[i + 1] : 0xFFFF;
                rr = rp >> 8;
                c0 = rp & 0xFF;
                const int c1 = ((nx >> 8) == rr) ? (nx & 0xFF) : tw;
                const uint32_t n = (uint32_t)(c1 - c0);
                sx = n * (uint32_t)(c0 + c1 - 1) / 2u;
                nsy = n | ((n * (uint32_t)rr) << 14);
                cl = c1 - 1;
            }
            const uint32_t valid = __ballot_sync(0xFFFFFFFFu, bi >= 0);
            if (!valid) return;
            const int cand = __shfl_sync(0xFFFFFFFFu, bi, __ffs(valid) - 1);
            const uint32_t grp = __ballot_sync(0xFFFFFFFFu, bi == cand);
            if (bi == cand) {
                nsy = __reduce_add_sync(grp, nsy);
                sx = __reduce_add_sync(grp, sx);
                rr = __reduce_max_sync(grp, rr);
                c0 = __reduce_min_sync(grp, c0);
                cl = __reduce_max_sync(grp, cl);
                if ((int)(threadIdx.x & 31) != __ffs(grp) - 1) bi = -1;  // the leader commits the group
            }
            if (bi >= 0) {
                atomicAdd(&A.bssy[bi], nsy);
                atomicAdd(&A.bsx[bi], sx);
                atomicMax(&A.brmax[bi], rr);
                atomicMin(&A.bcmin[bi], c0);
                atomicMax(&A.bcmax[bi], cl);
            }
        }
    };
    BorderFeatures bf{A, tg.tw, (uint32_t)g.flip, 0};
    if (!ccl_tile(S, tg, mo, bf)) return false;
    if (kWords) border_words(A);

    const int nlc = S.nlc, nb = S.nb;
    // the two allocations are issued by different warps so their latencies overlap
    if (tid == 0) {
        const uint32_t base = atomicAdd(&ws.counters[0], (uint32_t)nb);
        A.base = base;
        if ((uint64_t)base + nb > ws.cap_nodes) atomicOr(&ws.counters[1], ERR_NODE_CAP);
        ws.tbase[tg.t] = base;
        ws.tnb[tg.t] = (uint32_t)nb;
    }
    // ---- tile header (run/component counts, row tables) for the emit pass
    {
        uint16_t* hdr = ws.thdr + (int64_t)tg.t * THDR;
        if (tid == 0) {
            hdr[0] = (uint16_t)S.nruns;
            hdr[1] = (uint16_t)nlc;
            hdr[2] = (uint16_t)nb;
            hdr[3] = 0;
        }
        if (tid <= TH) {
            hdr[4 + tid] = S.rowlc[tid];
            hdr[4 + TH + 1 + tid] = S.rowbx[tid];
        }
    }
    RL_PHASE(tg.t, 10);
    const int flip = g.flip;
    // ---- perimeter labels: (value << 15) | border index; perimeter pixels on the image frame
    // mark their component as touching it
    const bool top_img = tg.ty == 0, bot_img = (tg.y0 + tg.th == g.H);
    const bool left_img = tg.tx == 0, right_img = (tg.x0 + tg.tw == g.W);
    uint16_t* const perim = ws.perim + (int64_t)tg.t * PERIM;
    auto label = [&](int pr, int pc, bool frame) -> uint32_t {
        const uint32_t lc = lc_at(S, pr, pc);
        const uint32_t bi = S.lcb[lc] & 0x7FFF;
        if (frame) A.bimg[bi] = 1;
        return ((xbit(S, pr, pc) ^ (uint32_t)flip) << 15) | bi;
    };
    // top and bottom rows: two neighbouring pixels per thread (same word), one 4-B store
    for (int q = tid; q < TW; q += BT) {
        const bool bot = q >= TW / 2;
        const int c = 2 * (q & (TW / 2 - 1)), pr = bot ? tg.th - 1 : 0;
        const bool frame = bot ? bot_img : top_img;
        uint32_t v = 0xFFFFFFFFu;  // PERIM_NONE twice
        if (c < tg.tw) {
            const int word = pr * WPR + (c >> 5), b = c & 31;
            const uint32_t st = S.st[word], xw = S.x[word];
            const int run0 = (int)S.rbase[word] + __popc(st & (0xFFFFFFFFu >> (31 - b))) - 1;
            const uint32_t bi0 = S.lcb[lc_of_run(S, run0)] & 0x7FFF;
            v = (((((xw >> b) & 1u) ^ (uint32_t)flip) << 15) | bi0) | 0xFFFF0000u;
            if (frame) A.bimg[bi0] = 1;
            if (c + 1 < tg.tw) {
                const int run1 = run0 + (int)((st >> (b + 1)) & 1u);  // a run starts at c + 1?
                const uint32_t bi1 = run1 == run0 ? bi0 : S.lcb[lc_of_run(S, run1)] & 0x7FFF;
                v = (v & 0xFFFFu) | ((((((xw >> (b + 1)) & 1u) ^ (uint32_t)flip) << 15) | bi1) << 16);
                if (frame && run1 != run0) A.bimg[bi1] = 1;
            }
        }
        reinterpret_cast<uint32_t*>(perim + (bot ? TW : 0))[c >> 1] = v;
    }
    // left and right columns
    for (int q = tid; q < 2 * TH; q += BT) {
        const bool right = q >= TH;
        const int pr = right ? q - TH : q;
        perim[2 * TW + q] = pr < tg.th ? (uint16_t)label(pr, right ? tg.tw - 1 : 0, right ? right_img : left_img)
                                       : PERIM_NONE;
    }
    __syncthreads();

    RL_PHASE(tg.t, 11);
    // ---- border-component nodes
    const uint32_t base = A.base;
    const bool node_ok = (uint64_t)base + nb <= ws.cap_nodes;
    for (int i = tid; i < nb && node_ok; i += BT) {
        const int lc = S.blc[i];
        const int fr = lc_row(S, lc), fc = lc_col(S, lc);
        const uint32_t fg = xbit(S, fr, fc) ^ (uint32_t)flip;
        NodeRec rec;
        rec.tile = (uint32_t)tg.t;
        rec.fr = (uint16_t)fr;
        rec.fc = (uint16_t)fc;
        rec.ibefore = (uint16_t)((lc - S.rowlc[fr]) - (i - S.rowbx[fr]));
        rec.fg = (uint8_t)fg;
        rec.pad = 0;
        if (fc > 0) {
            const uint32_t l2 = lc_at(S, fr, fc - 1);
            if (lc_is_border(S, l2)) {
                rec.leftkind = 0;
                rec.left = S.lcb[l2];
            } else {
                rec.leftkind = 3;
                rec.left = 0;
            }
        } else if (tg.x0 == 0) {
            rec.leftkind = 2;
            rec.left = 0;
        } else {
            rec.leftkind = 1;
            rec.left = (uint16_t)fr;
        }
        const uint32_t node = (uint32_t)g.B + base + (uint32_t)i;
        const uint64_t key = (uint64_t)(tg.y0 + fr) * (uint64_t)g.W + (uint64_t)(tg.x0 + fc);
        Acc f;
        const int64_t s = A.bssy[i] & 0x3FFFu;
        f.s = s;
        f.sx = (int64_t)A.bsx[i] + s * tg.x0;
        f.sy = (int64_t)(A.bssy[i] >> 14) + s * tg.y0;
        f.row_min = tg.y0 + fr;
        f.row_max = tg.y0 + A.brmax[i];
        f.col_min = tg.x0 + A.bcmin[i];
        f.col_max = tg.x0 + A.bcmax[i];
        ws.nrec[node] = rec;
        ws.nkey[node] = key;
        ws.nmin[node] = key;
        ws.nacc[node] = f;
        // border background touching the image frame is the exterior (App. A R3)
        ws.uf[node] = (!fg && A.bimg[i]) ? (uint32_t)tg.b : node;
    }

    // ---- interior components per row, foreground interior components
    if (tid < tg.th) {
        const int nl = S.rowlc[tid + 1] - S.rowlc[tid];
        const int nbr = S.rowbx[tid + 1] - S.rowbx[tid];
        ws.cnt[((int64_t)tg.b * g.H + tg.y0 + tid) * g.ntx + tg.tx] = (uint32_t)(nl - nbr);
    }
    const int nfg = __reduce_add_sync(0xFFFFFFFFu, bf.nfg);
    if ((tid & 31) == 0 && nfg) atomicAdd(&ws.img_fg[tg.b], (uint32_t)nfg);
    RL_PHASE(tg.t, 12);
    return true;
}

// class S: one CTA per tile on the (ntx, nty, B) grid; heavier tiles go to list A
#ifndef RL_ANALYZE_MINB
#define RL_ANALYZE_MINB 8
#endif
__global__ void __launch_bounds__(NT, RL_ANALYZE_MINB) k_analyze(const uint8_t* __restrict__ pix, Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& A = *reinterpret_cast<AnalyzeSmem<CapS>*>(smem_raw);
    const TileGeom tg = tile_geom_grid(g);
    if (!analyze_tile<CapS, false>(A, pix, g, ws, tg) && threadIdx.x == 0)
        ws.ovf[atomicAdd(&ws.counters[2], 1u)] = (uint32_t)tg.t;
}

// class M over list A; heavier tiles go to list B
__global__ void __launch_bounds__(CapM::BT, 4) k_analyze_m(const uint8_t* __restrict__ pix, Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& A = *reinterpret_cast<AnalyzeSmem<CapM>*>(smem_raw);
    const uint32_t n = ws.counters[2];
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
        const TileGeom tg = tile_geom(g, (int32_t)ws.ovf[k]);
        if (!analyze_tile<CapM, true>(A, pix, g, ws, tg) && threadIdx.x == 0)
            ws.ovf2[atomicAdd(&ws.counters[4], 1u)] = (uint32_t)tg.t;
        __syncthreads();
    }
}

// calls with at most one wave of class-M CTAs: every tile goes straight to class M (no class-S
// attempt and no class-S emit launch: the dense single images' critical path)
__global__ void __launch_bounds__(CapM::BT, 4) k_analyze_m_direct(const uint8_t* __restrict__ pix, Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& A = *reinterpret_cast<AnalyzeSmem<CapM>*>(smem_raw);
    for (uint32_t k = blockIdx.x; k < (uint32_t)g.ntiles; k += gridDim.x) {
        const TileGeom tg = tile_geom(g, (int32_t)k);
        if (!analyze_tile<CapM, false>(A, pix, g, ws, tg) && threadIdx.x == 0)
            ws.ovf2[atomicAdd(&ws.counters[4], 1u)] = (uint32_t)tg.t;
        __syncthreads();
    }
}

// class F over list B (one run per pixel fits)
__global__ void __launch_bounds__(CapF::BT) k_analyze_full(const uint8_t* __restrict__ pix, Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& A = *reinterpret_cast<AnalyzeSmem<CapF>*>(smem_raw);
    const uint32_t n = ws.counters[4];
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
        const TileGeom tg = tile_geom(g, (int32_t)ws.ovf2[k]);
        analyze_tile<CapF, true>(A, pix, g, ws, tg);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// M1: union across tile seams
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t node_of(const Ws& ws, const Geo& g, int64_t t, uint16_t lab) {
    return (uint32_t)g.B + ws.tbase[t] + (lab & 0x7FFFu);
}

// Horizontal seams s0 .. s0+ns-1 (seam s lies between tile rows s and s+1): one block per
// tile pair, one thread per column.  The pairs a seam links are first united in shared memory
// over the two tiles' border indices (a component crossing the seam at many columns -- the
// percolating one -- becomes one link), then one global union per linked border component.
#ifndef RL_SEAM_THREADS
#define RL_SEAM_THREADS 64  // small blocks: more seams in flight per SM (latency-bound unions)
#endif
constexpr int SEAM_T0 = RL_SEAM_THREADS;  // threads per seam block (TW / SEAM_T columns each)
constexpr int SEAM_TW = 256;              // calls with few tiles: more threads per seam (shorter chains)

template <int SEAM_T>
__global__ void __launch_bounds__(SEAM_T) k_seam_h(Geo g, Ws ws, int32_t s0, int32_t ns) {
    __shared__ uint32_t lp[2 * NBMAX];
    // the seam's two perimeter rows (bottom of the upper tile, top of the lower one), staged
    // with 16-B loads, and the left tiles' last columns
    __shared__ __align__(16) uint16_t rowu[TW], rowd[TW];
    __shared__ uint16_t leftu, leftd;
    static_assert(SEAM_T >= 2 * (TW / 8), "one 16-B load per thread stages both rows");
    // the overflow flag is read together with the block's first loads (one round trip less per
    // block than testing it first); nothing is written before it is tested
    const uint32_t aborted = ws.counters[1];
    const uint32_t v8 = g.flip ? 0u : 1u;
    const int32_t tx = blockIdx.x, tid = threadIdx.x;
    // grid (tile column, seam, image): no division by the seam count per block
    for (int32_t b = blockIdx.z; b < g.B; b += gridDim.z)
    for (int32_t si = blockIdx.y; si < ns; si += gridDim.y) {
        const int32_t s = s0 + si;
        const int64_t tu = ((int64_t)b * g.nty + s) * g.ntx + tx, tl = tu + g.ntx;
        const int nbu = (int)ws.tnb[tu], nbd = (int)ws.tnb[tl];
        // node bases of the two tiles, for the global links below: loaded now, with the rest
        const uint32_t bu = (uint32_t)g.B + ws.tbase[tu], bd = (uint32_t)g.B + ws.tbase[tl];
        if (tid < TW / 8)
            reinterpret_cast<uint4*>(rowu)[tid] = reinterpret_cast<const uint4*>(ws.perim + tu * PERIM + TW)[tid];
        else if (tid < TW / 4)
            reinterpret_cast<uint4*>(rowd)[tid - TW / 8] = reinterpret_cast<const uint4*>(ws.perim + tl * PERIM)[tid - TW / 8];
        if (tid == 0 && tx > 0) {
            leftu = ws.perim[(tu - 1) * PERIM + TW + TW - 1];
            leftd = ws.perim[(tl - 1) * PERIM + TW - 1];
        }
        if (aborted) return;
        for (int i = tid; i < nbu + nbd; i += SEAM_T) lp[i] = (uint32_t)i;
        __syncthreads();
        for (int c = tid; c < TW; c += SEAM_T) {
            const int32_t x = tx * TW + c;
            if (x >= g.W) break;
            const uint16_t lu = rowu[c], ld = rowd[c];
            const uint32_t vu = lu >> 15, vd = ld >> 15;
            uint16_t lul = PERIM_NONE, ldl = PERIM_NONE;
            if (x > 0) {
                lul = c ? rowu[c - 1] : leftu;
                ldl = c ? rowd[c - 1] : leftd;
            }
            const uint32_t iu = lu & 0x7FFFu, id = (uint32_t)nbu + (ld & 0x7FFFu);
            if (vu == vd && !(c > 0 && lul == lu && ldl == ld)) sunion(lp, iu, id);
            if (x > 0) {
                const uint32_t vul = lul >> 15, vdl = ldl >> 15;
                if (vul == v8 && vd == v8 && vu != v8 && vdl != v8) {  // (r, x-1) ~ (r+1, x)
                    if (c > 0) sunion(lp, lul & 0x7FFFu, id);
                    else gunion_key(ws.uf, ws.nkey, node_of(ws, g, tu - 1, lul), node_of(ws, g, tl, ld), (uint32_t)g.B);
                }
                if (vu == v8 && vdl == v8 && vul != v8 && vd != v8) {  // (r, x) ~ (r+1, x-1)
                    if (c > 0) sunion(lp, iu, (uint32_t)nbu + (ldl & 0x7FFFu));
                    else gunion_key(ws.uf, ws.nkey, node_of(ws, g, tu, lu), node_of(ws, g, tl - 1, ldl), (uint32_t)g.B);
                }
            }
        }
        __syncthreads();
        // one global link per border component that joined another one here
        for (int i = tid; i < nbu + nbd; i += SEAM_T) {
            uint32_t r = lp[i];
            if (r == (uint32_t)i) continue;
            while (lp[r] != r) r = lp[r];
            const uint32_t ni = i < nbu ? bu + i : bd + (i - nbu);
            const uint32_t nr = r < (uint32_t)nbu ? bu + r : bd + (r - nbu);
            gunion_key(ws.uf, ws.nkey, ni, nr, (uint32_t)g.B);
        }
        __syncthreads();
    }
}

// vertical seams: between tile column s-1 and s, one thread per pixel row of tile rows
// [ty0, ty1)
__global__ void k_seam_v(Geo g, Ws ws) {
    if (ws.counters[1]) return;
    // pixel row r of a tile row (threadIdx.x & 31), seams over grid x, (image, tile row) over grid y
    const int32_t nrows = g.ty1 - g.ty0;
    const uint32_t v8 = g.flip ? 0u : 1u;
    const int32_t r = threadIdx.x & 31;
    const int32_t s = 1 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (s >= g.ntx) return;
    for (int32_t q = blockIdx.y; q < g.B * nrows; q += gridDim.y) {
        const int32_t ty = g.ty0 + q % nrows;
        const int32_t b = q / nrows;
        const int32_t th = min(TH, g.H - ty * TH);
        if (r >= th) continue;
        const int64_t tR = ((int64_t)b * g.nty + ty) * g.ntx + s, tL = tR - 1;
        const uint16_t* pL = ws.perim + tL * PERIM + 2 * TW + TH;  // right column of left tile
        const uint16_t* pR = ws.perim + tR * PERIM + 2 * TW;       // left column of right tile
        const uint16_t lL = pL[r], lR = pR[r];
        const uint32_t vL = lL >> 15, vR = lR >> 15;
        if (vL == vR) {
            const bool same = r > 0 && pL[r - 1] == lL && pR[r - 1] == lR;
            if (!same) gunion_key(ws.uf, ws.nkey, node_of(ws, g, tL, lL), node_of(ws, g, tR, lR), (uint32_t)g.B);
        }
        if (r + 1 < th) {
            const uint16_t lL1 = pL[r + 1], lR1 = pR[r + 1];
            const uint32_t vL1 = lL1 >> 15, vR1 = lR1 >> 15;
            if (vL == v8 && vR1 == v8 && vR != v8 && vL1 != v8)
                gunion_key(ws.uf, ws.nkey, node_of(ws, g, tL, lL), node_of(ws, g, tR, lR1), (uint32_t)g.B);
            if (vL1 == v8 && vR == v8 && vL != v8 && vR1 != v8)
                gunion_key(ws.uf, ws.nkey, node_of(ws, g, tL, lL1), node_of(ws, g, tR, lR), (uint32_t)g.B);
        }
    }
}

// ---------------------------------------------------------------------------------------
// M2..M7: node passes
// ---------------------------------------------------------------------------------------
#define NODE_LOOP(n)                                                                   \
    const uint32_t nused_ = min(ws.counters[0], ws.cap_nodes);                         \
    for (uint32_t n = (uint32_t)g.B + blockIdx.x * blockDim.x + threadIdx.x;           \
         n < (uint32_t)g.B + nused_; n += gridDim.x * blockDim.x)

// contiguous node range of this block (nodes are tile-major, so a component's nodes from
// neighbouring tiles land in the same block and aggregate in its fold table)
#define NODE_CHUNK(n)                                                                   \
    const uint32_t nused_ = min(ws.counters[0], ws.cap_nodes);                          \
    const uint32_t chunk_ = (nused_ + gridDim.x - 1) / gridDim.x;                       \
    const uint32_t lo_ = (uint32_t)g.B + min(nused_, blockIdx.x * chunk_);              \
    const uint32_t hi_ = (uint32_t)g.B + min(nused_, (blockIdx.x + 1) * chunk_);        \
    for (uint32_t n = lo_ + threadIdx.x; n < hi_; n += blockDim.x)

constexpr int FT_SLOTS = 512;

__device__ __forceinline__ void tile_of(const Geo& g, uint32_t t, int32_t& b, int32_t& ty, int32_t& tx) {
    b = (int32_t)(t / (uint32_t)g.tpi);
    const int32_t rem = (int32_t)(t - (uint32_t)b * g.tpi);
    ty = rem / g.ntx;
    tx = rem - ty * g.ntx;
}

// Flatten, fold node features into the roots and -- outside strip mode, where the cut classes'
// status is settled later (k_reps, strips.cu) -- count the representatives: the root of a class
// is its raster-first node (gunion_key), so it represents the component and is counted in the
// (image, row, tile column) cell of its first pixel.
__global__ void __launch_bounds__(256) k_resolve(Geo g, Ws ws) {
    __shared__ FoldTable<FT_SLOTS> T;
    if (ws.counters[1]) return;
    T.init();
    __syncthreads();
    const uint32_t nused = min(ws.counters[0], ws.cap_nodes);
    const uint32_t chunk = (nused + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = (uint32_t)g.B + min(nused, blockIdx.x * chunk);
    const uint32_t hi = (uint32_t)g.B + min(nused, (blockIdx.x + 1) * chunk);
    for (uint32_t base = lo + (threadIdx.x & ~31u); base < hi; base += blockDim.x) {
        const uint32_t n = base + (threadIdx.x & 31);
        uint32_t dst = FT_EMPTY;
        Acc f;
        bool fgrep = false;
        int32_t b = -1;
        if (n < hi) {
            const uint32_t root = gfind_ro(ws.uf, n);
            if (root != n) {
                ws.uf[n] = root;
                dst = root;
                f = ws.nacc[n];
            }
            if (!g.strip) {
                ws.nrep[n] = root == n ? 1 : 0;
                if (root == n) {
                    const NodeRec rec = ws.nrec[n];
                    int32_t ty, tx;
                    tile_of(g, rec.tile, b, ty, tx);
                    atomicAdd(&ws.cnt[((int64_t)b * g.H + ty * TH + rec.fr) * g.ntx + tx], 1u);
                    fgrep = rec.fg != 0;
                }
            }
        }
        warp_fold<false>(T, dst, f, ~0ull, [&](uint32_t k) { return ws.nacc + k; },
                         [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
        const uint32_t fgmask = __ballot_sync(0xFFFFFFFFu, fgrep);
        if (fgmask) {  // foreground representatives per image, aggregated per warp
            const uint32_t same = __match_any_sync(0xFFFFFFFFu, fgrep ? b : -1);
            if (fgrep && (__ffs(same & fgmask) - 1) == (int)(threadIdx.x & 31u))
                atomicAdd(&ws.img_fg[b], (uint32_t)__popc(same & fgmask));
        }
    }
    __syncthreads();
    T.flush([&](uint32_t k) { return ws.nacc + k; },
            [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
}


// strip mode's representatives, once the cut classes' status is applied (strips.cu): a root
// whose min key was cleared is represented in another strip
__global__ void k_reps(Geo g, Ws ws) {
    if (ws.counters[1]) return;
    const uint32_t nused = min(ws.counters[0], ws.cap_nodes);
    // whole warps iterate together so the per-image foreground count aggregates per warp
    for (uint32_t base = (uint32_t)g.B + (blockIdx.x * blockDim.x + threadIdx.x) - (threadIdx.x & 31u);
         base < (uint32_t)g.B + nused; base += gridDim.x * blockDim.x) {
        const uint32_t n = base + (threadIdx.x & 31u);
        bool fgrep = false;
        int32_t b = -1;
        if (n < (uint32_t)g.B + nused) {
            const uint32_t root = ws.uf[n];
            const bool rep = root >= (uint32_t)g.B && ws.nkey[n] == ws.nmin[root];
            ws.nrep[n] = rep ? 1 : 0;
            if (rep) {
                const NodeRec rec = ws.nrec[n];
                int32_t ty, tx;
                tile_of(g, rec.tile, b, ty, tx);
                atomicAdd(&ws.cnt[((int64_t)b * g.H + ty * TH + rec.fr) * g.ntx + tx], 1u);
                fgrep = rec.fg != 0;
            }
        }
        const uint32_t fgmask = __ballot_sync(0xFFFFFFFFu, fgrep);
        if (fgmask) {
            const uint32_t same = __match_any_sync(0xFFFFFFFFu, fgrep ? b : -1);
            if (fgrep && (__ffs(same & fgmask) - 1) == (int)(threadIdx.x & 31u))
                atomicAdd(&ws.img_fg[b], (uint32_t)__popc(same & fgmask));
        }
    }
}

// canonical-id offset of image b's first cell (strip mode: 0, the strip's cells are scanned from
// the components of the strips above, so ids come out whole-image)
__device__ __forceinline__ uint32_t img_off(const Geo& g, const Ws& ws, int32_t b) {
    return g.strip ? 0u : ws.off[(int64_t)b * g.H * g.ntx];
}

__device__ __forceinline__ uint64_t comp_base(const Geo& g, const Ws& ws, int32_t b) {
    return (uint64_t)img_off(g, ws, b) + (uint64_t)b;
}

// the component tables hold every id of this call (strip mode: the owned ids plus the cut
// survivors' scratch slots)
__device__ __forceinline__ bool comps_fit(const Geo& g, const Ws& ws) {
    return (uint64_t)ws.off[g.cell_end] + (uint64_t)g.B - (uint64_t)g.cid_lo + (uint64_t)g.cid_extra <= ws.cap_comps;
}

// one warp per tile: canonical ids of the tile's border representatives.  The tile's border
// components are in raster order of first pixel, so "representatives before me in my row"
// is a prefix count inside the run of equal rows (match_any) plus a carry across chunks.
// root node of the component surrounding node n's component: the pixel left of its first
// pixel (same tile, the left tile's right column, or the image frame)
__device__ __forceinline__ uint32_t surrounding_root(const Geo& g, const Ws& ws, uint32_t n, const NodeRec& rec,
                                                     int32_t b) {
    if (ws.nleft) return ws.uf[ws.nleft[n]];  // strip mode: resolved before the exchange
    if (rec.leftkind == 0) return ws.uf[(uint32_t)g.B + ws.tbase[rec.tile] + rec.left];
    if (rec.leftkind == 1) {
        const uint32_t tl = rec.tile - 1;
        const uint16_t lab = ws.perim[(int64_t)tl * PERIM + 2 * TW + TH + rec.left];
        return ws.uf[(uint32_t)g.B + ws.tbase[tl] + (lab & 0x7FFFu)];
    }
    if (rec.leftkind == 2) return (uint32_t)b;
    atomicOr(&ws.counters[1], ERR_INTERNAL);
    return (uint32_t)b;
}

// One warp per tile: canonical ids of the tile's border representatives (the tile's border
// components are in raster order of first pixel, so "representatives before me in my row" is
// a prefix count inside the run of equal rows plus a carry across chunks), their surrounding
// components and pre-fill records (the parent id is filled in by k_tops, once every class has
// its id).  Children of the exterior survive hole filling and start their post-fill features.
__global__ void k_cids(Geo g, Ws ws) {
    if (ws.counters[1]) return;
    const bool fit = comps_fit(g, ws);
    const int lane = threadIdx.x & 31;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (fit && gid < g.B) {  // exterior records (the exterior survives hole filling)
        if (g.cid_lo == 0) {  // strip mode: strip 0 owns id 0 (the others count it, strips.cu)
            const uint64_t cb = comp_base(g, ws, gid);
            rl_component c;
            c.f = ws.nacc[gid];
            c.parent = 0xFFFFFFFFu;
            c.flags = 0;
            ws.comps[cb] = c;
            ws.top[cb] = 0;
            ws.filled[cb] = c.f;
        }
        atomicAdd(&ws.img_surv[gid], 1u);
    }
    const int warps = (gridDim.x * blockDim.x) >> 5;
    // strip mode: this rank's tile rows only (the tiles of other strips hold no nodes here)
    const int32_t t_lo = g.strip ? g.ty0 * g.ntx : 0, t_hi = g.strip ? g.ty1 * g.ntx : g.ntiles;
    for (int32_t t = t_lo + (gid >> 5); t < t_hi; t += warps) {
        int32_t b, ty, tx;
        tile_of(g, (uint32_t)t, b, ty, tx);
        const uint32_t nb = ws.tnb[t];
        const uint32_t n0 = (uint32_t)g.B + ws.tbase[t];
        const int64_t img0 = (int64_t)b * g.H * g.ntx;
        const uint32_t offimg = img_off(g, ws, b);
        const uint64_t cb = (uint64_t)offimg + (uint64_t)b;
        int carry_row = -1, carry = 0, nsurv = 0;
        for (uint32_t i0 = 0; i0 < nb; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool valid = i < nb;
            const uint32_t n = n0 + i;
            const int row = valid ? (int)ws.nrec[n].fr : 0x10000 + lane;
            const bool rep = valid && ws.nrep[n];
            const uint32_t repmask = __ballot_sync(0xFFFFFFFFu, rep);
            const uint32_t same = __match_any_sync(0xFFFFFFFFu, row);
            const uint32_t below = (1u << lane) - 1u;
            int before = __popc(repmask & same & below);
            if (row == carry_row) before += carry;
            if (rep) {
                const NodeRec rec = ws.nrec[n];
                const uint32_t cid = 1u + (ws.off[img0 + (int64_t)(ty * TH + rec.fr) * g.ntx + tx] - offimg) +
                                     rec.ibefore + (uint32_t)before;
                const uint32_t root = ws.uf[n];
                ws.nrootcid[root] = cid;
                const uint32_t proot = surrounding_root(g, ws, n, rec, b);
                ws.nparent[root] = proot;
                if (fit) {
                    rl_component c;
                    c.f = ws.nacc[root];
                    c.parent = 0;  // k_tops
                    c.flags = rec.fg;
                    ws.comps[cb + cid] = c;
                    if (proot < (uint32_t)g.B) {
                        // strip mode: a survivor crossing a cut collects every rank's partial
                        // post-fill sums, so it starts empty and is counted globally (strips.cu)
                        const bool cut = ws.ncut && ws.ncut[root];
                        ws.filled[cb + cid] = cut ? acc_empty() : c.f;
                        if (!cut) ++nsurv;
                    }
                }
            }
            // carry for the next chunk: reps of the chunk's last row (continuing rows only)
            const int last_row = __shfl_sync(0xFFFFFFFFu, row, 31);
            const uint32_t last_same = __shfl_sync(0xFFFFFFFFu, same, 31);
            const int cnt_last = __popc(repmask & last_same);
            carry = (last_row == carry_row ? carry : 0) + cnt_last;
            carry_row = last_row;
        }
        nsurv = __reduce_add_sync(0xFFFFFFFFu, nsurv);
        if (lane == 0 && nsurv) atomicAdd(&ws.img_surv[b], (uint32_t)nsurv);
    }
}


// The same with one block per tile: the tile's node rows and representative flags are staged in
// shared memory and prefix-summed once, so every node's "representatives before me in my row" is
// two lookups (the first node of its row by binary search over the sorted rows) and all of the
// tile's nodes are processed in parallel instead of in warp-sized chunks one after another.
constexpr int CIDS_T = 256;
__global__ void __launch_bounds__(CIDS_T) k_cids_blk(Geo g, Ws ws) {
    __shared__ uint16_t srow[NBMAX];
    __shared__ uint16_t spre[NBMAX + 1];
    __shared__ int wsum[CIDS_T / 32 + 1];
    if (ws.counters[1]) return;
    const bool fit = comps_fit(g, ws);
    const int tid = threadIdx.x;
    const int gid = blockIdx.x * CIDS_T + tid;
    if (fit && gid < g.B) {  // exterior records (the exterior survives hole filling)
        if (g.cid_lo == 0) {  // strip mode: strip 0 owns id 0 (the others count it, strips.cu)
            const uint64_t cb = comp_base(g, ws, gid);
            rl_component c;
            c.f = ws.nacc[gid];
            c.parent = 0xFFFFFFFFu;
            c.flags = 0;
            ws.comps[cb] = c;
            ws.top[cb] = 0;
            ws.filled[cb] = c.f;
        }
        atomicAdd(&ws.img_surv[gid], 1u);
    }
    constexpr int PER = (NBMAX + CIDS_T - 1) / CIDS_T;  // consecutive nodes per thread in the scan
    const int32_t t_lo = g.strip ? g.ty0 * g.ntx : 0, t_hi = g.strip ? g.ty1 * g.ntx : g.ntiles;
    for (int32_t t = t_lo + blockIdx.x; t < t_hi; t += gridDim.x) {
        int32_t b, ty, tx;
        tile_of(g, (uint32_t)t, b, ty, tx);
        const int nb = (int)ws.tnb[t];
        const uint32_t n0 = (uint32_t)g.B + ws.tbase[t];
        int cnt = 0;
        uint32_t repbits = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = tid * PER + q;
            if (i < nb) {
                srow[i] = ws.nrec[n0 + i].fr;
                const bool rep = ws.nrep[n0 + i] != 0;
                repbits |= (uint32_t)rep << q;
                cnt += rep;
            }
        }
        int tot;
        int pre = block_excl_scan<CIDS_T>(cnt, wsum, tot);  // contains __syncthreads
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int i = tid * PER + q;
            if (i < nb) spre[i] = (uint16_t)pre;
            pre += (repbits >> q) & 1u;
        }
        __syncthreads();
        const int64_t img0 = (int64_t)b * g.H * g.ntx;
        const uint32_t offimg = img_off(g, ws, b);
        const uint64_t cb = (uint64_t)offimg + (uint64_t)b;
        int nsurv = 0;
        for (int i = tid; i < nb; i += CIDS_T) {
            const uint32_t n = n0 + (uint32_t)i;
            if (!ws.nrep[n]) continue;
            const NodeRec rec = ws.nrec[n];
            // first node of this row: rows are ascending over the tile's nodes
            int lo = 0, hi = i;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (srow[mid] < rec.fr) lo = mid + 1;
                else hi = mid;
            }
            const uint32_t before = (uint32_t)(spre[i] - spre[lo]);
            const uint32_t cid = 1u + (ws.off[img0 + (int64_t)(ty * TH + rec.fr) * g.ntx + tx] - offimg) +
                                 rec.ibefore + before;
            const uint32_t root = ws.uf[n];
            ws.nrootcid[root] = cid;
            const uint32_t proot = surrounding_root(g, ws, n, rec, b);
            ws.nparent[root] = proot;
            if (fit) {
                rl_component c;
                c.f = ws.nacc[root];
                c.parent = 0;  // k_tops
                c.flags = rec.fg;
                ws.comps[cb + cid] = c;
                if (proot < (uint32_t)g.B) {
                    const bool cut = ws.ncut && ws.ncut[root];
                    ws.filled[cb + cid] = cut ? acc_empty() : c.f;
                    if (!cut) ++nsurv;
                }
            }
        }
        nsurv = __reduce_add_sync(0xFFFFFFFFu, nsurv);
        if ((tid & 31) == 0 && nsurv) atomicAdd(&ws.img_surv[b], (uint32_t)nsurv);
        __syncthreads();  // srow / spre are rewritten by the next tile
    }
}

// post-fill roots (depth-1 ancestors) of the border components; non-survivors fold their
// features into their root right away (block-aggregated; the survivors were initialised by
// k_cids).  Strip mode folds later, after the cross-rank reduction (k_fold).  Every node (not
// only the representatives) also gets what the emit pass needs of it -- its component's id and
// post-fill root's id, the exterior flag -- next to the tile's other nodes, so that the emit
// prologue reads them with one load instead of chasing node -> root -> ids.
__global__ void __launch_bounds__(256) k_tops(Geo g, Ws ws) {
    __shared__ FoldTable<FT_SLOTS, false> T;  // hole-filling folds: sums only
    if (ws.counters[1] || !comps_fit(g, ws)) return;
    T.init();
    __syncthreads();
    const uint32_t nused = min(ws.counters[0], ws.cap_nodes);
    const uint32_t chunk = (nused + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = (uint32_t)g.B + min(nused, blockIdx.x * chunk);
    const uint32_t hi = (uint32_t)g.B + min(nused, (blockIdx.x + 1) * chunk);
    const int lane = threadIdx.x & 31;
    // whole warps iterate together: the folds of a warp into one root are reduced in registers
    for (uint32_t base = lo + (threadIdx.x & ~31u); base < hi; base += blockDim.x) {
        const uint32_t n = base + lane;
        uint32_t dst = FT_EMPTY;
        Acc f;
        const uint32_t rep = n < hi ? ws.nrep[n] : 0u;
        uint32_t root = 0, anc = 0;
        if (n < hi) {
            root = ws.uf[n];
            uint32_t cid = 0;
            if (root < (uint32_t)g.B) {
                ws.nrep[n] = (uint8_t)(rep | 2u);  // the exterior
            } else {
                cid = ws.nrootcid[root];
                if (ws.ncut && ws.ncut[root]) {
                    anc = ws.nanccid[root];  // strip mode: a class crossing a cut, resolved globally
                } else {
                    uint32_t cur = root, fold;
                    for (;;) {
                        const uint32_t p = ws.nparent[cur];
                        if (p < (uint32_t)g.B) {
                            anc = fold = ws.nrootcid[cur];
                            break;
                        }
                        if (ws.ncut && ws.ncut[p]) {  // strip mode: the chain leaves the strip
                            anc = ws.nanccid[p];
                            fold = ws.nfold[p];
                            break;
                        }
                        cur = p;
                    }
                    if (rep) {
                        ws.nanccid[root] = anc;
                        if (ws.nfold) ws.nfold[root] = fold;
                    }
                }
            }
            ws.ninfo[n] = make_uint2(cid, anc);
        }
        if (rep) {
            int32_t b, ty, tx;
            tile_of(g, ws.nrec[n].tile, b, ty, tx);
            const uint64_t cb = comp_base(g, ws, b);
            const uint32_t cid = ws.nrootcid[root];
            ws.top[cb + cid] = anc;
            ws.comps[cb + cid].parent = ws.nrootcid[ws.nparent[root]];
            if (anc != cid && !g.strip) {
                dst = (uint32_t)(cb + anc);  // < 2^32 components
                f = ws.nacc[root];
            }
        }
        warp_fold(T, dst, f, ~0ull, [&](uint32_t k) { return ws.filled + k; },
                  [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
    }
    __syncthreads();
    T.flush([&](uint32_t k) { return ws.filled + k; },
            [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
}

// strip mode: border non-survivors into their post-fill roots, after the reduction (strips.cu)
__global__ void __launch_bounds__(256) k_fold(Geo g, Ws ws) {
    __shared__ FoldTable<FT_SLOTS, false> T;  // hole-filling folds: sums only
    if (ws.counters[1] || !comps_fit(g, ws)) return;
    T.init();
    __syncthreads();
    const uint32_t nused = min(ws.counters[0], ws.cap_nodes);
    const uint32_t chunk = (nused + gridDim.x - 1) / gridDim.x;
    const uint32_t lo = (uint32_t)g.B + min(nused, blockIdx.x * chunk);
    const uint32_t hi = (uint32_t)g.B + min(nused, (blockIdx.x + 1) * chunk);
    for (uint32_t base = lo + (threadIdx.x & ~31u); base < hi; base += blockDim.x) {
        const uint32_t n = base + (threadIdx.x & 31);
        uint32_t dst = FT_EMPTY;
        Acc f;
        if (n < hi && (ws.nrep[n] & 1u)) {
            const uint32_t root = ws.uf[n];
            const uint32_t anc = ws.nanccid[root];
            if (anc != ws.nrootcid[root]) {
                dst = ws.nfold[root];  // the survivor's slot (it may be owned by another strip)
                f = ws.nacc[root];
            }
        }
        warp_fold(T, dst, f, ~0ull, [&](uint32_t k) { return ws.filled + k; },
                  [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
    }
    __syncthreads();
    T.flush([&](uint32_t k) { return ws.filled + k; },
            [&](uint32_t) { return static_cast<unsigned long long*>(nullptr); });
}

// ---------------------------------------------------------------------------------------
// K1b: emit
// ---------------------------------------------------------------------------------------
constexpr int FOLD_SLOTS = 64;  // distinct border fold targets per tile kept in smem

template <class C>
struct EmitSmem {
    CclSmem<C> c;
    // interior-feature chunk accumulators (tile-local coordinates)
    // S | (Sy << 14): the components of one tile hold <= 8192 pixels in all (see AnalyzeSmem)
    uint32_t fssy[C::FCH], fsx[C::FCH];
    int32_t frmax[C::FCH], fcmin[C::FCH], fcmax[C::FCH];
    // border components of this tile
    uint32_t bcid[C::NBC];   // canonical id of the component
    uint32_t banc[C::NBC];   // canonical id of its post-fill root
    uint8_t bflag[C::NBC];   // bit0 representative, bit1 exterior
    uint16_t repx[C::NBC + 1];  // exclusive prefix of representative flags over border index
    // fold of interior components into border-derived survivors: small open-addressing
    // table keyed by border index (overflow goes straight to global atomics)
    // (sums only: see acc_atomic_fold_fill)
    uint16_t pkey[FOLD_SLOTS];
    uint32_t ps[FOLD_SLOTS], psx[FOLD_SLOTS], psy[FOLD_SLOTS];
    uint32_t ext[NW];       // exterior-pixel masks of the tile words
    uint32_t rowoff[TH];    // canonical id offset of each tile row (relative to the image)
    uint16_t dfold[C::FCH];  // chunk components whose post-fill root is an interior survivor
    int ndfold;
    uint64_t cb;
    int gate;                 // the merge phase succeeded (no capacity overflow)
};

// canonical id of tile component lc (any kind)
template <class ES>
__device__ __forceinline__ uint32_t comp_cid(const ES& E, uint32_t lc) {
    const auto& S = E.c;
    const uint16_t lb = S.lcb[lc];
    if (!(lb & 0x8000u)) return E.bcid[lb];
    const int r = lc_row(S, lc);
    const int bp = lb & 0x7FFF;                  // border components before lc
    const int rb0 = S.rowbx[r];
    const int nonrep_before = (bp - rb0) - (E.repx[bp] - E.repx[rb0]);
    return 1u + E.rowoff[r] + (uint32_t)((int)lc - S.rowlc[r] - nonrep_before);
}

// Walk the tree inside the tile: returns the post-fill root's canonical id of interior
// component lc; `end` = border index where the walk left the tile interior, or -1 when lc's
// chain reached the exterior (then `surv` is the interior survivor).
template <class ES>
__device__ __forceinline__ uint32_t interior_top(const ES& E, uint32_t lc, int& end, uint32_t& surv) {
    const auto& S = E.c;
    uint32_t cur = lc;
    for (;;) {
        const uint32_t p = lc_at(S, lc_row(S, cur), lc_col(S, cur) - 1);  // interior: col >= 1
        const uint16_t pb = S.lcb[p];
        if (!(pb & 0x8000u)) {
            if (E.bflag[pb] & 2u) {  // parent is the exterior: cur survives
                end = -1;
                surv = cur;
                return comp_cid(E, cur);
            }
            end = pb;
            surv = 0;
            return E.banc[pb];
        }
        cur = p;
    }
}

// slot of border index `key` in the fold table, or -1 when the table is full
template <class ES>
__device__ __forceinline__ int fold_slot(ES& E, uint32_t key) {
    uint32_t h = (key * 2654435761u) >> 26;  // 6 bits
    for (int probe = 0; probe < FOLD_SLOTS; ++probe, h = (h + 1) & (FOLD_SLOTS - 1)) {
        const unsigned short cur = E.pkey[h];
        if (cur == key) return (int)h;
        if (cur == 0xFFFF) {
            const unsigned short prev = atomicCAS(reinterpret_cast<unsigned short*>(&E.pkey[h]),
                                                  (unsigned short)0xFFFF, (unsigned short)key);
            if (prev == 0xFFFF || prev == key) return (int)h;
        }
    }
    return -1;
}

// one word of the hole-filled image (App. A R9): pixel = 0 iff its component is the exterior
__device__ __forceinline__ void emit_filled_word(const Geo& g, const Ws& ws, const TileGeom& tg, int r, int w,
                                                 uint32_t vm, uint32_t fillbits) {
    if (vm && g.ofmt == 1) {
        uint8_t* row = ws.filled_img + tg.b * g.ofbytes + (tg.y0 + r - g.prow0) * (int64_t)g.orowb;
        p4_store_word(row, g.orowb, (tg.x0 >> 5) + w, fillbits, g.ovec_ok);
    } else if (vm) {
        uint8_t* dst = ws.filled_img + tg.b * g.ofbytes + (tg.y0 + r - g.prow0) * g.W + tg.x0 + 32 * w;
        if (g.ovec_ok && vm == 0xFFFFFFFFu) {
            uint4 o0, o1;
            o0.x = nibble_to_bytes(fillbits & 0xF);
            o0.y = nibble_to_bytes((fillbits >> 4) & 0xF);
            o0.z = nibble_to_bytes((fillbits >> 8) & 0xF);
            o0.w = nibble_to_bytes((fillbits >> 12) & 0xF);
            o1.x = nibble_to_bytes((fillbits >> 16) & 0xF);
            o1.y = nibble_to_bytes((fillbits >> 20) & 0xF);
            o1.z = nibble_to_bytes((fillbits >> 24) & 0xF);
            o1.w = nibble_to_bytes((fillbits >> 28) & 0xF);
            uint4* d4 = reinterpret_cast<uint4*>(dst);
            __stcs(d4, o0);
            __stcs(d4 + 1, o1);
        } else {
            const int n = 32 - __clz(vm);
            for (int j = 0; j < n; ++j) dst[j] = (uint8_t)((fillbits >> j) & 1u);
        }
    }
}

// Emits a tile iff it belongs to capacity class C (the class its analyze pass used).
#ifndef RL_EMIT_TAIL_BARRIER
#define RL_EMIT_TAIL_BARRIER 0  // 1: the barriers after the last chunk's deferred folds and before the filled image
#endif
template <class C>
__device__ __forceinline__ bool emit_tile(EmitSmem<C>& E, const Geo& g, const Ws& ws, const TileGeom& tg) {
    CclSmem<C>& S = E.c;
    const int tid = threadIdx.x;
    const int r = tid / WPR, w = tid % WPR;
    constexpr int BT = C::BT;
    const bool word = BT == NW || tid < NW;
    // every global load the prologue needs is issued up front: the tile header, map offset and
    // node base (independent of each other), then the bits, row offsets, the stored component map
    // and the border components' ids (k_tops put them next to the tile's nodes)
    const uint16_t* hdr = ws.thdr + (int64_t)tg.t * THDR;
    const uint32_t h01 = *reinterpret_cast<const uint32_t*>(hdr);  // 4-B aligned: THDR is even
    const int nb_h = hdr[2];
    const uint64_t moff = ws.tmap[tg.t];
    const uint32_t tb = ws.tbase[tg.t];
    const int nruns_h = (int)(h01 & 0xFFFFu), nlc_h = (int)(h01 >> 16);
    if (nruns_h > C::MR || nlc_h > C::NLC || nb_h > C::NBC) return false;  // a larger class owns it
    const uint32_t vm = word ? valid_mask(tg, r, w) : 0u;
    if (nlc_h == 1) {  // a uniform tile (uniform_tile): one border component, no interior records
        if (ws.counters[1] || !comps_fit(g, ws)) return true;  // capacity overflow: re-run
        const uint32_t node = (uint32_t)g.B + tb;
        const uint32_t fl = ws.nrep[node];  // bit 1: the exterior
        emit_filled_word(g, ws, tg, r, w, vm, (fl & 2u) ? 0u : vm);
        if (g.label_mode && vm) {
            const uint2 info = ws.ninfo[node];
            const uint32_t v = g.label_mode == 2 ? ((fl & 2u) ? 0u : info.y) : info.x;
            uint32_t* ldst = ws.labels + (int64_t)tg.b * g.P + (tg.y0 + r - g.prow0) * g.W + tg.x0 + 32 * w;
            const int n = 32 - __clz(vm);
            for (int j = 0; j < n; ++j) ldst[j] = v;
        }
        return true;
    }
    {
        // bits and run starts (the run positions and word bases come with the stored map)
        const uint32_t x = word ? __ldcs(ws.bits + (int64_t)tg.t * NW + tid) : 0u;
        const uint32_t xl = __shfl_up_sync(0xFFFFFFFFu, x, 1), vml = __shfl_up_sync(0xFFFFFFFFu, vm, 1);
        if (word) {
            uint32_t c1 = 0, c0 = 0;
            if (w > 0) {  // left neighbour word of the same row (rows never straddle a warp)
                const uint32_t lv = vml >> 31;
                c1 = (xl >> 31) & lv;
                c0 = ((~xl) >> 31) & lv;
            }
            S.x[tid] = x;
            S.vm[tid] = vm;
            S.st[tid] = ((x & ~((x << 1) | c1)) | (~x & ~((~x << 1) | c0))) & vm;
            E.ext[tid] = 0;
        }
    }
    const int64_t img0 = (int64_t)tg.b * g.H * g.ntx;
    const uint32_t offimg = img_off(g, ws, tg.b);
    if (tid < TH && tid < tg.th)
        E.rowoff[tid] = ws.off[img0 + (int64_t)(tg.y0 + tid) * g.ntx + tg.tx] - offimg;
    if (tid == 0) {
        E.ndfold = 0;
        E.cb = (uint64_t)offimg + (uint64_t)tg.b;
        const uint32_t errs = ws.counters[1];
        const bool fit = comps_fit(g, ws);  // both loads in flight together (no short circuit)
        E.gate = !errs && fit;
        S.nlc = nlc_h;
        S.nb = nb_h;
        S.nruns = nruns_h;
    }
    {  // the run -> component map and component tables the analyze pass stored (tile_runs below
       // does not touch them); bounds-checked so that a failed gate never reads past the store
        const MapLayout ML(nruns_h, nlc_h);
        static_assert(C::MR % 8 == 0 && C::NLC % 8 == 0, "padded map sections fit the tables");
        static_assert(THDR % 2 == 0, "tile headers start 4-B aligned");
        static_assert((NW + 1) / 8 * 16 <= sizeof(S.rbase), "word bases: whole vectors fit");
        if (moff + (uint64_t)ML.total <= ws.cap_rstore) {
            const uint4* src = reinterpret_cast<const uint4*>(ws.rstore + moff);  // 16-B aligned
            // sections in 16-B vectors: map -> par, lcrun, lcb, rbase
            const int v1 = ML.lcrun >> 3, v2 = ML.lcb >> 3, v4 = ML.rbase >> 3;
            const int vend = v4 + ((NW + 1) >> 3);  // rbase: the full vectors (the last element below)
            for (int i = tid; i < vend; i += BT) {
                const uint4 v = src[i];
                if (i < v1) reinterpret_cast<uint4*>(S.par)[i] = v;
                else if (i < v2) reinterpret_cast<uint4*>(S.lcrun)[i - v1] = v;
                else if (i < v4) reinterpret_cast<uint4*>(S.lcb)[i - v2] = v;
                else reinterpret_cast<uint4*>(S.rbase)[i - v4] = v;
            }
            if (tid == 0) S.rbase[NW] = ws.rstore[moff + ML.rbase + NW];
        }
    }
    if (tid < FOLD_SLOTS) {
        E.pkey[tid] = 0xFFFF;
        E.ps[tid] = E.psx[tid] = E.psy[tid] = 0;
    }
    if (tid <= TH) {
        S.rowlc[tid] = hdr[4 + tid];
        S.rowbx[tid] = hdr[4 + TH + 1 + tid];
    }
    {
        const uint32_t nbase = (uint32_t)g.B + tb;
        const uint32_t nend = (uint32_t)g.B + ws.cap_nodes;  // loads stay in bounds even when
        for (int i = tid; i < nb_h; i += BT) {                 // the gate below fails
            const uint32_t node = nbase + (uint32_t)i;
            if (node >= nend) break;
            const uint2 info = ws.ninfo[node];
            E.bcid[i] = info.x;
            E.banc[i] = info.y;
            E.bflag[i] = ws.nrep[node];
        }
    }
    __syncthreads();
    if (!E.gate) return true;  // capacity overflow: the host grows and re-runs

    // runs again from the packed bits (cheap); the component map comes from the analyze pass
    RL_PHASE(tg.t, 16);
    const int nruns = nruns_h, nlc = nlc_h, nb = nb_h;
    // run positions of the run starts (the word bases are the analyze pass's); the 512-thread
    // classes give each half of a word to its own thread
    if constexpr (BT == NW) {
        int i = S.rbase[tid];
        for (uint32_t m = S.st[tid]; m; m &= m - 1u) S.runpos[i++] = (uint16_t)((r << 8) | (32 * w + __ffs(m) - 1));
    } else {
        const int wd = tid % NW, half = tid / NW;
        const uint32_t st = S.st[wd], lo = 0xFFFFu;
        int i = S.rbase[wd] + (half ? __popc(st & lo) : 0);
        const uint16_t rw = (uint16_t)(((wd / WPR) << 8) | (32 * (wd % WPR)));
        for (uint32_t m = half ? (st & ~lo) : (st & lo); m; m &= m - 1u) S.runpos[i++] = (uint16_t)(rw + __ffs(m) - 1);
    }
    const uint64_t cb = E.cb;
    for (int i = tid; i < min(C::FCH, nlc); i += BT) {  // first feature chunk's accumulators
        E.fssy[i] = E.fsx[i] = 0;
        E.frmax[i] = -1;
        E.fcmin[i] = 0x7FFFFFFF;
        E.fcmax[i] = -1;
    }
    // exclusive prefix of the representative flags over border index (flags are in), by one warp
    // (ballot + popc per 32 entries); in the 512-thread classes a warp without a word does it
    constexpr int PW = BT == NW ? NWARPS - 1 : NWARPS;
    if ((tid >> 5) == PW) {
        const int lane = tid & 31;
        int carry = 0;
        for (int i0 = 0; i0 <= nb; i0 += 32) {
            const int i = i0 + lane;
            const bool f = i < nb && (E.bflag[i] & 1);
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, f);
            if (i <= nb) E.repx[i] = (uint16_t)(carry + __popc(m & ((1u << lane) - 1u)));
            carry += __popc(m);
        }
    }
    __syncthreads();
    RL_PHASE(tg.t, 18);

    // ---- interior components, in chunks of C::FCH tile components.  The first chunk's run
    // pass also marks exterior pixels (for the hole-filled image) and records, in a register,
    // the chunk of each of the thread's runs (4 bits per run i = tid + j * BT: the chunk, 14 for
    // chunk >= 14, 15 for runs with nothing to accumulate), so that a later chunk revisits
    // only its own runs instead of rescanning the tile.
    constexpr int RPT = (C::MR + BT - 1) / BT;  // runs per thread
    static_assert(RPT <= 16, "4-bit run codes fit 64 bits");
    using CodeT = typename std::conditional<RPT * 4 <= 32, uint32_t, unsigned long long>::type;
    CodeT codes = 0;
    const int flip = g.flip;
    int nsurv = 0;
    for (int l0 = 0; l0 < max(nlc, 1); l0 += C::FCH) {
        const int l1 = min(l0 + C::FCH, nlc);
        if (l0 > 0) {  // the first chunk's accumulators were cleared before the prefix barrier
            for (int i = tid; i < l1 - l0; i += BT) {
                E.fssy[i] = E.fsx[i] = 0;
                E.frmax[i] = -1;
                E.fcmin[i] = 0x7FFFFFFF;
                E.fcmax[i] = -1;
            }
            if (tid == 0) E.ndfold = 0;  // the last chunk's deferred folds were read before its final barrier
            __syncthreads();
        }
        RL_PHASE(tg.t, 19);
        const int ch = l0 / C::FCH;
        const uint32_t want = (uint32_t)min(ch, 14);
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            const int i = tid + j * BT;
            if (i >= nruns) break;
            uint32_t lc;
            if (l0 == 0) {
                lc = lc_of_run(S, i);
                const uint16_t lb = S.lcb[lc];
                uint32_t code = 15u;
                if (!(lb & 0x8000u)) {
                    if (E.bflag[lb] & 2u) {  // exterior run: its pixels in the row's words
                        const int rr = run_row(S, i), c0 = run_col(S, i), c1 = run_end(S, i, tg.tw);
                        const int w0 = c0 >> 5, w1 = (c1 - 1) >> 5;
                        uint32_t* ext = E.ext + rr * WPR;
                        const uint32_t mlo = 0xFFFFFFFFu << (c0 & 31), mhi = 0xFFFFFFFFu >> (31 - ((c1 - 1) & 31));
                        if (w0 == w1) {
                            atomicOr(ext + w0, mlo & mhi);
                        } else {  // words strictly inside the run belong to it alone
                            atomicOr(ext + w0, mlo);
                            for (int wd = w0 + 1; wd < w1; ++wd) ext[wd] = 0xFFFFFFFFu;
                            atomicOr(ext + w1, mhi);
                        }
                    }
                } else {
                    code = (uint32_t)min((int)lc / C::FCH, 14);
                }
                codes |= (CodeT)code << (4 * j);
                if (code != 0u) continue;
            } else {
                if ((uint32_t)((codes >> (4 * j)) & 15u) != want) continue;
                lc = lc_of_run(S, i);
                if (ch >= 14 && ((int)lc < l0 || (int)lc >= l1)) continue;
            }
            const int k = (int)lc - l0;
            const int rr = run_row(S, i), c0 = run_col(S, i), c1 = run_end(S, i, tg.tw);
            const uint32_t n = (uint32_t)(c1 - c0);
            atomicAdd(&E.fssy[k], n | ((n * (uint32_t)rr) << 14));
            atomicAdd(&E.fsx[k], n * (uint32_t)(c0 + c1 - 1) / 2u);
            atomicMax(&E.frmax[k], rr);
            atomicMin(&E.fcmin[k], c0);
            atomicMax(&E.fcmax[k], c1 - 1);
        }
        __syncthreads();
        RL_PHASE(tg.t, 20);
        // pre-fill records, post-fill roots, survivor init; folds into border-component roots
        // (initialised by the merge phase) go to the shared table right away, folds into
        // interior survivors wait until the survivors' own records are written (barrier)
        // whole warps iterate together: the folds of a warp into one border survivor's slot (the
        // percolating component's, typically) are reduced in registers first, so the shared
        // table sees one update per warp instead of 32 same-address atomics
        for (int base = l0 + (tid & ~31); base < l1; base += BT) {
            const int lc = base + (tid & 31);
            int slot = -1, k = 0, fr = 0;
            if (lc < l1 && !lc_is_border(S, lc)) {
                k = lc - l0;
                fr = lc_row(S, lc);
                const int fc = lc_col(S, lc);
                const uint32_t cid = comp_cid(E, (uint32_t)lc);
                const uint32_t pcid = comp_cid(E, lc_at(S, fr, fc - 1));
                int end;
                uint32_t surv;
                const uint32_t anc = interior_top(E, (uint32_t)lc, end, surv);
                const int64_t s = E.fssy[k] & 0x3FFFu;
                rl_component c;
                c.f.s = s;
                c.f.sx = (int64_t)E.fsx[k] + s * tg.x0;
                c.f.sy = (int64_t)(E.fssy[k] >> 14) + s * tg.y0;
                c.f.row_min = tg.y0 + fr;
                c.f.row_max = tg.y0 + E.frmax[k];
                c.f.col_min = tg.x0 + E.fcmin[k];
                c.f.col_max = tg.x0 + E.fcmax[k];
                c.parent = pcid;
                c.flags = xbit(S, fr, fc) ^ (uint32_t)flip;
                ws.comps[cb + cid] = c;
                ws.top[cb + cid] = anc;
                if (anc == cid) {
                    ws.filled[cb + cid] = c.f;
                    ++nsurv;
                } else {
                    slot = end >= 0 ? fold_slot(E, (uint32_t)end) : -1;
                    if (slot < 0) {
                        if (end >= 0)  // table full
                            acc_atomic_fold_fill(ws.filled + (ws.nfold ? (uint64_t)ws.nfold[ws.uf[(uint32_t)g.B + ws.tbase[tg.t] + end]]
                                                                       : cb + anc),
                                                 c.f.s, c.f.sx, c.f.sy);
                        else E.dfold[atomicAdd(&E.ndfold, 1)] = (uint16_t)lc;
                    }
                }
            }
            const uint32_t act = __ballot_sync(0xFFFFFFFFu, slot >= 0);
            if (!act) continue;
            const int lead = __ffs(act) - 1;
            const int dom = __shfl_sync(0xFFFFFFFFu, slot, lead);
            const uint32_t grp = __ballot_sync(0xFFFFFFFFu, slot == dom);
            if (slot < 0) continue;
            uint32_t vssy = E.fssy[k], vsx = E.fsx[k];
            if (slot == dom) {
                vssy = __reduce_add_sync(grp, vssy);  // a tile's sums stay within the packed fields
                vsx = __reduce_add_sync(grp, vsx);
                if ((tid & 31) != lead) continue;
            }
            atomicAdd(&E.ps[slot], vssy & 0x3FFFu);
            atomicAdd(&E.psx[slot], vsx);
            atomicAdd(&E.psy[slot], vssy >> 14);
        }
        __syncthreads();
        RL_PHASE(tg.t, 21);
        for (int q = tid; q < E.ndfold; q += BT) {  // folds into interior survivors
            const int lc = E.dfold[q], k = lc - l0;
            int end;
            uint32_t surv;
            const uint32_t anc = interior_top(E, (uint32_t)lc, end, surv);
            const int64_t s = E.fssy[k] & 0x3FFFu;
            acc_atomic_fold_fill(ws.filled + cb + anc, s, (int64_t)E.fsx[k] + s * tg.x0,
                                 (int64_t)(E.fssy[k] >> 14) + s * tg.y0);
        }
        // the next chunk clears the accumulators these folds read; after the last chunk nothing
        // rewrites what they read (the persistent callers synchronise before the next tile)
        if (!RL_EMIT_TAIL_BARRIER && l0 + C::FCH >= max(nlc, 1)) {
        } else {
            __syncthreads();
        }
        RL_PHASE(tg.t, 22);
    }
    // flush border-keyed folds (the survivors were initialised by k_tops).  The targets are
    // border survivors, often one per image (the percolating component) that every tile folds
    // into: the sums go to this tile's shard of the accumulator table, not to one address.
    for (int i = tid; i < FOLD_SLOTS; i += BT) {
        if (E.pkey[i] == 0xFFFF || !E.ps[i]) continue;
        const int64_t s = E.ps[i];
        // strip mode: the survivor's slot in `filled` (it may be owned by another strip)
        const uint32_t key = ws.nfold ? ws.nfold[ws.uf[(uint32_t)g.B + ws.tbase[tg.t] + E.pkey[i]]]
                                      : (uint32_t)(cb + E.banc[E.pkey[i]]);
        const int64_t sx = (int64_t)E.psx[i] + s * tg.x0, sy = (int64_t)E.psy[i] + s * tg.y0;
        const uint32_t base = (uint32_t)(tg.t % FT_SHARDS) * FT_HS;
        uint32_t h = (key * 2654435761u) >> (32 - 13);
        static_assert(FT_HS == 1 << 13, "hash width");
        bool done = false;
        for (int probe = 0; ws.ftkey && probe < 8 && !done; ++probe, h = (h + 1) & (FT_HS - 1)) {
            uint32_t k0 = ws.ftkey[base + h];
            if (k0 == FT_KEY_EMPTY) k0 = atomicCAS(ws.ftkey + base + h, FT_KEY_EMPTY, key);
            if (k0 == FT_KEY_EMPTY || k0 == key) {
                unsigned long long* d = ws.ftsum + 3ull * (base + h);
                atomicAdd(d, (unsigned long long)s);
                atomicAdd(d + 1, (unsigned long long)sx);
                atomicAdd(d + 2, (unsigned long long)sy);
                done = true;
            }
        }
        if (!done) acc_atomic_fold_fill(ws.filled + key, s, sx, sy);  // no table, or its probe window full
    }
    nsurv = __reduce_add_sync(0xFFFFFFFFu, nsurv);
    if ((tid & 31) == 0 && nsurv) atomicAdd(&ws.img_surv[tg.b], (uint32_t)nsurv);
    // no barrier here: the exterior masks the filled image needs are complete since the first
    // feature chunk's barrier, and the persistent callers synchronise before the next tile
    if (RL_EMIT_TAIL_BARRIER) __syncthreads();
    RL_PHASE(tg.t, 23);

    // ---- hole-filled image (App. A R9): pixel = 0 iff its component is the exterior
    emit_filled_word(g, ws, tg, r, w, vm, vm & ~E.ext[tid]);
    // ---- optional label image (Alg. 4 relabel, canonical ids), one lane per run
    if (g.label_mode) {
        for (int i = tid; i < nruns; i += BT) {
            const uint32_t lc = lc_of_run(S, i);
            uint32_t v = comp_cid(E, lc);
            if (g.label_mode == 2) {
                const uint16_t lb = S.lcb[lc];
                if (!(lb & 0x8000u)) {
                    v = (E.bflag[lb] & 2u) ? 0u : E.banc[lb];
                } else {
                    int end;
                    uint32_t surv;
                    v = interior_top(E, lc, end, surv);
                }
            }
            const int rr = run_row(S, i), c0 = run_col(S, i), c1 = run_end(S, i, tg.tw);
            uint32_t* ldst = ws.labels + (int64_t)tg.b * g.P + (tg.y0 + rr - g.prow0) * g.W + tg.x0;
            for (int j = c0; j < c1; ++j) ldst[j] = v;
        }
    }
    RL_PHASE(tg.t, 24);
    return true;
}

// the sharded hole-fill accumulators into the post-fill roots' features
__global__ void k_ftab_flush(Ws ws) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t key = ws.ftkey[i];
    if (key == FT_KEY_EMPTY) return;
    const unsigned long long* d = ws.ftsum + 3ull * i;
    acc_atomic_fold_fill(ws.filled + key, (int64_t)d[0], (int64_t)d[1], (int64_t)d[2]);
}

// class S on the full grid (tiles of larger classes are skipped), M over list A, F over list B
__global__ void __launch_bounds__(NT, 8) k_emit(Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& E = *reinterpret_cast<EmitSmem<CapSE>*>(smem_raw);
    emit_tile(E, g, ws, tile_geom_grid(g));
}

__global__ void __launch_bounds__(CapME::BT, 4) k_emit_m(Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& E = *reinterpret_cast<EmitSmem<CapME>*>(smem_raw);
    const uint32_t n = ws.counters[2];
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
        emit_tile(E, g, ws, tile_geom(g, (int32_t)ws.ovf[k]));
        __syncthreads();
    }
}

__global__ void __launch_bounds__(CapME::BT, 4) k_emit_m_direct(Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& E = *reinterpret_cast<EmitSmem<CapME>*>(smem_raw);
    for (uint32_t k = blockIdx.x; k < (uint32_t)g.ntiles; k += gridDim.x) {
        emit_tile(E, g, ws, tile_geom(g, (int32_t)k));
        __syncthreads();
    }
}

__global__ void __launch_bounds__(CapFE::BT) k_emit_full(Geo g, Ws ws) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    auto& E = *reinterpret_cast<EmitSmem<CapFE>*>(smem_raw);
    const uint32_t n = ws.counters[4];
    for (uint32_t k = blockIdx.x; k < n; k += gridDim.x) {
        emit_tile(E, g, ws, tile_geom(g, (int32_t)ws.ovf2[k]));
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// densified post-fill label image (labeling.hpp:231-236 with fill): rank of the survivor
// ---------------------------------------------------------------------------------------
__global__ void k_surv_flags(const uint32_t* top, uint64_t n, uint32_t* flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        flag[i] = top[i] == (uint32_t)i ? 1u : 0u;  // caller offsets per image below
}

__global__ void k_remap_labels(uint32_t* labels, int64_t P, int32_t B, const uint32_t* rank,
                               const uint64_t* cbase, uint64_t cap) {
    if (cbase[B] > cap) return;  // components overflowed: no labels were emitted, the host re-runs
    const int64_t total = P * B;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / P;
        const uint64_t cb = cbase[b];
        labels[i] = rank[cb + labels[i]] - rank[cb];
    }
}

__global__ void k_surv_flags_img(const uint32_t* top, const uint64_t* cbase, int32_t B, uint64_t total,
                                 uint32_t* flag) {
    // flag[i] = 1 iff component i (global index) is a post-fill root of its image
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        // binary search the image
        int32_t lo = 0, hi = B - 1;
        while (lo < hi) {
            const int32_t mid = (lo + hi + 1) / 2;
            if (cbase[mid] <= i) lo = mid; else hi = mid - 1;
        }
        flag[i] = top[i] == (uint32_t)(i - cbase[lo]) ? 1u : 0u;
    }
}

// post-fill features of the survivors only, in component order (rank = exclusive scan of the
// survivor flags); the batch's component count is cbase[B]
__global__ void k_compact_filled(const Acc* __restrict__ filled, const uint32_t* __restrict__ flag,
                                 const uint32_t* __restrict__ rank, const uint64_t* __restrict__ total_p,
                                 uint64_t cap, Acc* __restrict__ out) {
    const uint64_t total = *total_p;
    if (total > cap) return;  // components overflowed (nothing was emitted): the host re-runs
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x)
        if (flag[i]) out[rank[i]] = filled[i];
}

}  // namespace rlg

// ---------------------------------------------------------------------------------------
// launch wrappers (called from api.cu)
// ---------------------------------------------------------------------------------------
namespace rlg {

size_t analyze_smem() { return sizeof(AnalyzeSmem<CapS>); }
size_t emit_smem() { return sizeof(EmitSmem<CapSE>); }

template <class K>
static cudaError_t set_smem(K kernel, size_t bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Calls with few tiles (single images up to ~2 waves) are latency-bound: their seams run in
// 256-thread blocks (shorter chains of global unions per block; cfg1 merge 48 -> 42 us) and their
// canonical ids one block per tile (k_cids_blk; cfg1 merge 42 -> 38 us).  Dense
// tiles in 1024-thread class-M CTAs were measured too: no gain (the tile's critical path is its
// word phases and barriers).  (env RUNLAB_GPU_WIDE_TILES)
static int64_t g_wide_tiles = 4096;
static bool wide_call(const Geo& g) { return (int64_t)g.B * g.tpi <= g_wide_tiles; }
// calls with at most one wave of class-M CTAs skip the class-S attempt (env RUNLAB_GPU_DIRECT_TILES)
static int64_t g_direct_tiles = 148 * 4;
bool direct_call(const Geo& g) { return !g.strip && (int64_t)g.B * g.tpi <= g_direct_tiles; }
static bool g_cids_blk = true;  // wide calls: one block per tile in k_cids_blk (env RUNLAB_GPU_CIDS_BLK=0: off)

cudaError_t configure_kernels() {
    cudaError_t e = set_smem(k_analyze, sizeof(AnalyzeSmem<CapS>));
    if (e == cudaSuccess) e = set_smem(k_analyze_m, sizeof(AnalyzeSmem<CapM>));
    if (e == cudaSuccess) e = set_smem(k_analyze_full, sizeof(AnalyzeSmem<CapF>));
    if (e == cudaSuccess) e = set_smem(k_emit, sizeof(EmitSmem<CapSE>));
    if (e == cudaSuccess) e = set_smem(k_emit_m, sizeof(EmitSmem<CapME>));
    if (e == cudaSuccess) e = set_smem(k_emit_full, sizeof(EmitSmem<CapFE>));
    if (e == cudaSuccess) e = set_smem(k_analyze_m_direct, sizeof(AnalyzeSmem<CapM>));
    if (e == cudaSuccess) e = set_smem(k_emit_m_direct, sizeof(EmitSmem<CapME>));
    if (const char* v = std::getenv("RUNLAB_GPU_DIRECT_TILES")) g_direct_tiles = std::atoll(v);
    if (const char* v = std::getenv("RUNLAB_GPU_WIDE_TILES")) g_wide_tiles = std::atoll(v);
    if (const char* v = std::getenv("RUNLAB_GPU_CIDS_BLK")) g_cids_blk = std::atoi(v) != 0;
    return e;
}

static int grid_for(int64_t n, int block, int maxgrid) {
    int64_t gr = (n + block - 1) / block;
    if (gr < 1) gr = 1;
    if (gr > maxgrid) gr = maxgrid;
    return (int)gr;
}

void launch_seam_rows(const Geo& g, const Ws& ws, int32_t s0, int32_t ns, cudaStream_t s, int sms) {
    const dim3 grid(g.ntx, (unsigned)std::min<int64_t>(ns, 65535), (unsigned)std::min<int64_t>(g.B, 65535));
    if (wide_call(g))
        k_seam_h<SEAM_TW><<<grid, SEAM_TW, 0, s>>>(g, ws, s0, ns);
    else
        k_seam_h<SEAM_T0><<<grid, SEAM_T0, 0, s>>>(g, ws, s0, ns);
}
void launch_analyze(const uint8_t* pix, const Geo& g, const Ws& ws, cudaStream_t s) {
    if (direct_call(g)) {
        k_analyze_m_direct<<<(unsigned)std::min<int64_t>((int64_t)g.B * g.tpi, 148 * 4), CapM::BT,
                             sizeof(AnalyzeSmem<CapM>), s>>>(pix, g, ws);
        k_analyze_full<<<148 * 2, CapF::BT, sizeof(AnalyzeSmem<CapF>), s>>>(pix, g, ws);
        return;
    }
    k_analyze<<<dim3(g.ntx, g.ty1 - g.ty0, g.B), NT, sizeof(AnalyzeSmem<CapS>), s>>>(pix, g, ws);
    // deferred heavier tiles: the grids loop over device-side lists (no host sync)
    k_analyze_m<<<148 * 4, CapM::BT, sizeof(AnalyzeSmem<CapM>), s>>>(pix, g, ws);
    k_analyze_full<<<148 * 2, CapF::BT, sizeof(AnalyzeSmem<CapF>), s>>>(pix, g, ws);
}
void launch_seam_cols(const Geo& g, const Ws& ws, cudaStream_t s, int sms);
void launch_seam_cols(const Geo& g, const Ws& ws, cudaStream_t s, int sms) {
    const int32_t rows = g.ty1 - g.ty0;
    if (g.ntx > 1) {
        const int64_t pairs = (int64_t)g.B * rows;
        const dim3 grid((g.ntx - 1 + 7) / 8, (unsigned)std::min<int64_t>(pairs, 65535));
        k_seam_v<<<grid, 256, 0, s>>>(g, ws);
    }
}
void launch_resolve(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint) {
    k_resolve<<<grid_for(nodes_hint, 256, sms * 8), 256, 0, s>>>(g, ws);
}
void launch_reps(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint) {
    k_reps<<<grid_for(nodes_hint, 256, sms * 8), 256, 0, s>>>(g, ws);
}
void launch_cids(const Geo& g, const Ws& ws, cudaStream_t s, int sms) {
    if (g_cids_blk && wide_call(g))  // large calls: one warp per tile is faster (cfg2 merge 0.42 vs 0.51 ms)
        k_cids_blk<<<grid_for((int64_t)g.ntiles * CIDS_T, CIDS_T, sms * 16), CIDS_T, 0, s>>>(g, ws);
    else
        k_cids<<<grid_for((int64_t)g.ntiles * 32, 256, sms * 16), 256, 0, s>>>(g, ws);
}
// (the surrounding components and pre-fill records of border components come from k_cids)
void launch_tree(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint) {
    const int64_t n = nodes_hint > g.B ? nodes_hint : g.B;
    k_tops<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(g, ws);  // folds too (single-GPU path)
}
void launch_tree_parts(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint) {
    launch_tree(g, ws, s, sms, nodes_hint);  // strip mode: k_tops skips the folds (g.strip)
}
void launch_fold(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint) {
    const int64_t n = nodes_hint > g.B ? nodes_hint : g.B;
    k_fold<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(g, ws);
}
// The sharded accumulators pay off when thousands of tiles fold into one survivor (config 5:
// 131 K tiles into the percolating component, emit 1.9 -> 1.1 ms); with a few hundred tiles
// per image the direct atomics are cheaper than the table (config 2: +4% emit with it).
constexpr int FT_MIN_TILES = 8192;
// The three classes emit disjoint tiles: with a second stream (`s2`, with fork/join events) the
// deferred classes run beside class S instead of after it (no tail between them).
void launch_emit(const Geo& g, const Ws& ws0, cudaStream_t s, cudaStream_t s2, cudaEvent_t fork, cudaEvent_t join) {
    const bool sharded = g.tpi >= FT_MIN_TILES;
    Ws ws = ws0;
    if (sharded) {
        cudaMemsetAsync(ws.ftkey, 0xFF, (size_t)FT_SHARDS * FT_HS * 4, s);
        cudaMemsetAsync(ws.ftsum, 0, (size_t)FT_SHARDS * FT_HS * 24, s);
    } else {
        ws.ftkey = nullptr;
    }
    if (direct_call(g)) {  // every tile was analysed in class M (or deferred to F)
        k_emit_m_direct<<<(unsigned)std::min<int64_t>((int64_t)g.B * g.tpi, 148 * 4), CapME::BT,
                          sizeof(EmitSmem<CapME>), s>>>(g, ws);
        k_emit_full<<<148 * 2, CapFE::BT, sizeof(EmitSmem<CapFE>), s>>>(g, ws);
        if (sharded) k_ftab_flush<<<FT_SHARDS * FT_HS / 256, 256, 0, s>>>(ws);
        return;
    }
    const cudaStream_t sd = s2 ? s2 : s;
    if (s2) {
        cudaEventRecord(fork, s);
        cudaStreamWaitEvent(s2, fork, 0);
    }
    k_emit_m<<<148 * 4, CapME::BT, sizeof(EmitSmem<CapME>), sd>>>(g, ws);
    k_emit_full<<<148 * 2, CapFE::BT, sizeof(EmitSmem<CapFE>), sd>>>(g, ws);
    if (s2) cudaEventRecord(join, s2);
    k_emit<<<dim3(g.ntx, g.ty1 - g.ty0, g.B), NT, sizeof(EmitSmem<CapSE>), s>>>(g, ws);
    if (s2) cudaStreamWaitEvent(s, join, 0);
    if (sharded) k_ftab_flush<<<FT_SHARDS * FT_HS / 256, 256, 0, s>>>(ws);
}
void launch_surv_flags(const uint32_t* top, const uint64_t* cbase, int32_t B, uint64_t total, uint32_t* flag,
                       cudaStream_t s, int sms) {
    k_surv_flags_img<<<grid_for((int64_t)total, 256, sms * 8), 256, 0, s>>>(top, cbase, B, total, flag);
}
void launch_compact_filled(const Acc* filled, const uint32_t* flag, const uint32_t* rank, const uint64_t* total_p,
                           uint64_t cap, Acc* out, cudaStream_t s, int sms) {
    k_compact_filled<<<grid_for((int64_t)cap, 256, sms * 8), 256, 0, s>>>(filled, flag, rank, total_p, cap, out);
}
void launch_remap(uint32_t* labels, int64_t P, int32_t B, const uint32_t* rank, const uint64_t* cbase,
                  uint64_t cap, cudaStream_t s, int sms) {
    k_remap_labels<<<grid_for(P * B, 256, sms * 16), 256, 0, s>>>(labels, P, B, rank, cbase, cap);
}

}  // namespace rlg

#ifdef RL_PHASE_PROF
// profiling builds only: where the tile kernels stamp their phases
extern "C" int rl_debug_phase_buffer(void* dptr, int n_tiles) {
    unsigned long long* p = static_cast<unsigned long long*>(dptr);
    if (cudaMemcpyToSymbol(rlg::g_phase_buf, &p, sizeof(p)) != cudaSuccess) return 4;
    return cudaMemcpyToSymbol(rlg::g_phase_n, &n_tiles, sizeof(int)) == cudaSuccess ? 0 : 4;
}
#endif
