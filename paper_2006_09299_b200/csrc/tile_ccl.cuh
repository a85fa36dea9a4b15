// tile_ccl.cuh -- run-based FG/BG connected components of one bit-packed tile, in shared
// memory.  Used identically (bit-for-bit the same numbering) by the analyze pass (K1a)
// and the emit pass (K1b).
//
// Reference semantics restated (paths relative to /root/reference/proj/include/runlab/):
//  * a run ("segment") is a maximal horizontal interval of equal pixels, FG and BG alike
//    (Alg. 1, encode_row labeling.hpp:81-100);
//  * two runs of consecutive rows join when they overlap, extended by one column for the
//    8-connected parity (labeling.hpp:121,128-131; c8 = p ^ flip);
//  * union-find with the min-label rule (tables.hpp:68-76): here the label of a run is its
//    raster-order index inside the tile, so every root is its component's raster-first run
//    and tile-local component ids come out in raster order of first pixel (App. A R4).
//
// B200 formulation: one thread per 32-pixel word; run starts come from `x ^ (x << 1)`
// bit algebra; every overlap of two runs contributes exactly one union event, found with
// bit masks (vertical contact at the first overlapping column, i.e. at a run start of
// either row; plus diagonal-only contacts for the 8-connected value); union-find is
// lock-free (atomicMin linking, path halving) on a shared-memory parent array.
#pragma once

#include "common.cuh"

namespace rlg {

struct CclSmem {
    uint32_t x[NW];            // 8-connected-value bits (pixel value XOR flip), 0 where invalid
    uint32_t vm[NW];           // valid-pixel masks
    uint32_t st[NW];           // run-start masks
    uint16_t rbase[NW + 1];    // first run index of each word
    uint16_t lbase[NW + 1];    // first tile-component index among the word's root runs
    uint16_t rowlc[TH + 1];    // first tile-component index of each row
    uint16_t rowbx[TH + 1];    // border components before each row start
    uint32_t par[MAXRUNS];     // union-find parent; afterwards TAG | component of each run
    uint16_t lcpos[MAXLC];     // first pixel (row << 8) | col of each tile component
    uint16_t lcb[MAXLC];       // border index, or 0x8000 | (border components before it)
    uint16_t blc[NBMAX];       // border index -> tile component
    int wsum[NWARPS + 1];
    int nruns, nlc, nb;
};

__device__ __forceinline__ int run_at(const CclSmem& S, int word, int bit) {
    return (int)S.rbase[word] + __popc(S.st[word] & (0xFFFFFFFFu >> (31 - bit))) - 1;
}

// run of the pixel left of (word, bit); the caller guarantees it exists
__device__ __forceinline__ int run_left(const CclSmem& S, int word, int bit) {
    return bit > 0 ? run_at(S, word, bit - 1) : (int)S.rbase[word] - 1;
}

__device__ __forceinline__ uint32_t sfind(volatile uint32_t* par, uint32_t a) {
    for (;;) {
        const uint32_t p = par[a];
        if (p == a) return a;
        const uint32_t gp = par[p];
        if (gp == p) return p;
        par[a] = gp;
        a = gp;
    }
}

__device__ __forceinline__ void sunion(uint32_t* par, uint32_t a, uint32_t b) {
    volatile uint32_t* vp = par;
    for (;;) {
        a = sfind(vp, a);
        b = sfind(vp, b);
        if (a == b) return;
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicMin(par + a, b);
        if (old == a) return;
        a = old;
    }
}

__device__ __forceinline__ uint32_t lc_of_run(const CclSmem& S, int run) {
    return S.par[run] & ~TAG;
}

__device__ __forceinline__ bool lc_is_border(const CclSmem& S, uint32_t lc) {
    return (S.lcb[lc] & 0x8000u) == 0;
}

// tile component of pixel (r, c); pixel must be valid
__device__ __forceinline__ uint32_t lc_at(const CclSmem& S, int r, int c) {
    return lc_of_run(S, run_at(S, r * WPR + (c >> 5), c & 31));
}

// pixel value in "8-connected value" space at (r, c)
__device__ __forceinline__ uint32_t xbit(const CclSmem& S, int r, int c) {
    return (S.x[r * WPR + (c >> 5)] >> (c & 31)) & 1u;
}

// Visit the run pieces of the calling thread's word: f(run, j0, j1) for [j0, j1) in word
// bit coordinates.  Runs that started in an earlier word continue at bit 0.
template <class F>
__device__ __forceinline__ void for_each_piece(const CclSmem& S, int word, F&& f) {
    const uint32_t vm = S.vm[word];
    if (!vm) return;
    const int vend = 32 - __clz(vm);
    uint32_t rem = S.st[word];
    int ri = (rem & 1u) ? (int)S.rbase[word] : (int)S.rbase[word] - 1;
    if (rem & 1u) rem &= rem - 1u;
    int cur = 0;
    for (;;) {
        const int nxt = rem ? __ffs(rem) - 1 : vend;
        f(ri, cur, nxt);
        if (!rem) break;
        rem &= rem - 1u;
        cur = nxt;
        ++ri;
    }
}

// Full tile labeling.  Pre: S.x / S.vm filled for all NW words and a __syncthreads().
// Post (all synced): S.par[run] = TAG | component, S.lcpos, S.lcb (border flags
// compacted to border indices), S.blc, S.rowlc, S.rowbx, S.nruns, S.nlc, S.nb.
__device__ void ccl_tile(CclSmem& S, const TileGeom& tg) {
    const int tid = threadIdx.x;
    const int r = tid / WPR, w = tid % WPR;
    const uint32_t x = S.x[tid], vm = S.vm[tid];
    const uint32_t nx = ~x;
    uint32_t c1 = 0, c0 = 0;
    if (w > 0) {
        const uint32_t xl = S.x[tid - 1];
        const uint32_t lv = S.vm[tid - 1] >> 31;
        c1 = (xl >> 31) & lv;
        c0 = ((~xl) >> 31) & lv;
    }
    const uint32_t s1 = x & ~((x << 1) | c1) & vm;
    const uint32_t s0 = nx & ~((nx << 1) | c0) & vm;
    const uint32_t st = s1 | s0;
    S.st[tid] = st;
    const int nr = __popc(st);
    int total;
    const int rb = block_excl_scan(nr, S.wsum, total);  // contains __syncthreads
    S.rbase[tid] = (uint16_t)rb;
    if (tid == 0) {
        S.rbase[NW] = (uint16_t)total;
        S.nruns = total;
    }
    for (int k = 0; k < nr; ++k) S.par[rb + k] = (uint32_t)(rb + k);
    __syncthreads();

    // ---- union events with the row above (Alg. 2's overlap test, one event per pair)
    if (r >= 1 && vm) {
        const int ta = tid - WPR;
        const uint32_t a = S.x[ta], vma = S.vm[ta], sta = S.st[ta];
        uint32_t ca1 = 0;
        if (w > 0) ca1 = (S.x[ta - 1] >> 31) & (S.vm[ta - 1] >> 31);
        const uint32_t both = vm & vma;
        const uint32_t na = ~a;
        uint32_t ev = ((x & a & (s1 | (sta & a))) | (nx & na & (s0 | (sta & na)))) & both;
        while (ev) {
            const int j = __ffs(ev) - 1;
            ev &= ev - 1u;
            sunion(S.par, (uint32_t)run_at(S, tid, j), (uint32_t)run_at(S, ta, j));
        }
        const uint32_t xl1 = (x << 1) | c1, al1 = (a << 1) | ca1;
        uint32_t d1 = x & al1 & ~xl1 & na & both;  // (r, j) ~ (r-1, j-1)
        while (d1) {
            const int j = __ffs(d1) - 1;
            d1 &= d1 - 1u;
            sunion(S.par, (uint32_t)run_at(S, tid, j), (uint32_t)run_left(S, ta, j));
        }
        uint32_t d2 = xl1 & a & nx & ~al1 & both;  // (r, j-1) ~ (r-1, j)
        while (d2) {
            const int j = __ffs(d2) - 1;
            d2 &= d2 - 1u;
            sunion(S.par, (uint32_t)run_left(S, tid, j), (uint32_t)run_at(S, ta, j));
        }
    }
    __syncthreads();

    // ---- flatten (roots are final now)
    const int nruns = S.nruns;
    for (int i = tid; i < nruns; i += NT) {
        uint32_t p = S.par[i];
        while (true) {
            const uint32_t q = S.par[p];
            if (q == p) break;
            p = q;
        }
        S.par[i] = p;
    }
    __syncthreads();

    // ---- tile components = root runs, numbered in raster order
    int nroots = 0;
    for (int k = 0; k < nr; ++k) nroots += (S.par[rb + k] == (uint32_t)(rb + k));
    int nlc;
    const int lb = block_excl_scan(nroots, S.wsum, nlc);
    S.lbase[tid] = (uint16_t)lb;
    if (tid == 0) {
        S.lbase[NW] = (uint16_t)nlc;
        S.nlc = nlc;
    }
    {
        uint32_t m = st;
        int k = 0, lc = lb;
        while (m) {
            const int j = __ffs(m) - 1;
            m &= m - 1u;
            const int ri = rb + k++;
            if (S.par[ri] == (uint32_t)ri) {
                S.lcpos[lc] = (uint16_t)((r << 8) | (32 * w + j));
                S.lcb[lc] = 0;
                S.par[ri] = TAG | (uint32_t)lc;
                ++lc;
            }
        }
    }
    __syncthreads();
    for (int k = 0; k < nr; ++k) {
        const uint32_t p = S.par[rb + k];
        if (!(p & TAG)) S.par[rb + k] = S.par[p];
    }
    if (tid <= TH) S.rowlc[tid] = tid < TH ? S.lbase[tid * WPR] : (uint16_t)nlc;
    __syncthreads();

    // ---- components touching the tile border (plain stores of 1: race-free)
    for_each_piece(S, tid, [&](int ri, int j0, int j1) {
        if (r == 0 || r == tg.th - 1 || (w == 0 && j0 == 0) || (32 * w + j1 == tg.tw))
            S.lcb[lc_of_run(S, ri)] = 1;
    });
    __syncthreads();

    // ---- compact border components to border indices (raster order)
    const int per = (nlc + NT - 1) / NT;
    const int l0 = min(tid * per, nlc), l1 = min(l0 + per, nlc);
    int cnt = 0;
    for (int l = l0; l < l1; ++l) cnt += S.lcb[l];
    int nb;
    int bx = block_excl_scan(cnt, S.wsum, nb);
    for (int l = l0; l < l1; ++l) {
        if (S.lcb[l]) {
            S.blc[bx] = (uint16_t)l;
            S.lcb[l] = (uint16_t)bx++;
        } else {
            S.lcb[l] = (uint16_t)(0x8000 | bx);
        }
    }
    if (tid == 0) S.nb = nb;
    __syncthreads();
    if (tid <= TH) {
        const int l = S.rowlc[tid];
        S.rowbx[tid] = l < nlc ? (uint16_t)(S.lcb[l] & 0x7FFF) : (uint16_t)nb;
    }
    __syncthreads();
}

}  // namespace rlg
