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
// B200 formulation (one thread per 32-pixel word, one warp = 32/WPR tile rows):
//  * run starts are bit algebra on the packed row (`x & ~(x << 1 | carry)`), run indices a
//    block scan of popcounts; the run list (`runpos`) then drives every per-run phase with
//    all lanes busy (no per-lane loops of data-dependent length);
//  * every overlap of two runs contributes exactly one union event, found with bit masks
//    (vertical contact at the first overlapping column, i.e. at a run start of either row,
//    plus diagonal-only contacts for the 8-connected value).  Each warp compacts its events
//    into a shared queue and resolves them lane-parallel;
//  * union-find is lock-free on a shared-memory parent array (atomicMin linking toward the
//    smaller run index, path halving).
#pragma once

#include "common.cuh"

namespace rlg {

// Optional per-phase clock64() stamps of each tile CTA (profiling builds only:
// -DRL_PHASE_PROF; tools/phase_prof.py).  Slot 32*tile + k holds the stamp of phase k
// (analyze pass 0..14, emit pass 16..24).
#ifdef RL_PHASE_PROF
__device__ unsigned long long* g_phase_buf = nullptr;
__device__ int g_phase_n = 0;
#define RL_PHASE(tile, k)                                                         \
    do {                                                                          \
        if (threadIdx.x == 0 && g_phase_buf && (tile) < g_phase_n)               \
            g_phase_buf[32ull * (unsigned)(tile) + (k)] = clock64();              \
    } while (0)
#else
#define RL_PHASE(tile, k) \
    do {                  \
    } while (0)
#endif

// Capacity classes of the shared-memory tables.  A tile is tried in the small class first
// (most tiles: >= 8 CTAs per SM), and deferred through device-side lists to the larger ones
// when it holds more runs / border components than fit:
//   S: <= MAXRUNS * 3/16 runs (0.19 runs/pixel), <= NBMAX/2 border components;
//   M: <= MAXRUNS * 5/8 runs (0.62 runs/pixel, covers any random image), all border components;
//   F: one run per pixel (checkerboards and other adversarial inputs).
// EVC = union-event queue per warp; longer queues are processed in rounds.
// BT = threads per CTA: one per word (256) for the sparse class; the dense classes add a second
// thread per word so that their per-run and per-component loops run twice as wide.
template <int MR_, int NBC_, int EVC_, int FCH_, class PT_, int BT_, int NLC_ = MR_>
struct Cap {
    static constexpr int MR = MR_;
    static constexpr int NLC = NLC_;  // tile components (a tile with more goes to the next class)
    static constexpr int NBC = NBC_;
    static constexpr int EVC = EVC_;
    static constexpr int FCH = FCH_;  // interior-feature accumulator chunk (emit pass)
    using PT = PT_;                   // run-parent type: 32-bit for native atomicMin unions
    static constexpr int BT = BT_;
    static_assert(BT == NW || BT == 2 * NW, "one or two threads per word");
};
// analyze pass (union-find: 32-bit parents)
#ifndef RL_S_MR
#define RL_S_MR 2048  // 3072 and 1280 measured slower on config 2
#endif
#ifndef RL_S_NLC
#define RL_S_NLC 960  // keeps the class-S tables within 8 CTAs per SM
#endif
using CapS = Cap<RL_S_MR, NBMAX / 2, 192, 512, uint32_t, NW, RL_S_NLC>;
// M: <= 0.5625 runs/pixel (random g = 1 noise at any density: 0.5), <= 2048 components; sized so
// that 4 CTAs of 512 threads fit one SM (full occupancy); events are queued in rounds of 512
using CapM = Cap<MAXRUNS * 9 / 16, NBMAX, 512, 384, uint32_t, 2 * NW, 2048>;
using CapF = Cap<MAXRUNS, NBMAX, 1024, 320, uint32_t, 2 * NW>;
// emit pass: same classes, no unions (16-bit component map, larger feature chunks)
#ifndef RL_SE_FCH
#define RL_SE_FCH 288  // the largest chunk with 8 CTAs per SM (packed S|Sy accumulators)
#endif
using CapSE = Cap<CapS::MR, CapS::NBC, 192, RL_SE_FCH, uint16_t, NW, CapS::NLC>;
#ifndef RL_ME_FCH
#define RL_ME_FCH 704  // the largest chunk with 4 CTAs per SM
#endif
using CapME = Cap<CapM::MR, CapM::NBC, 32, RL_ME_FCH, uint16_t, 2 * NW, CapM::NLC>;
using CapFE = Cap<CapF::MR, CapF::NBC, 1024, 320, uint16_t, 2 * NW>;

template <class C>
struct CclSmem {
    static constexpr int MR = C::MR;
    static constexpr int BT = C::BT;
    uint32_t x[NW];            // 8-connected-value bits (pixel value XOR flip), 0 where invalid
    uint32_t vm[NW];           // valid-pixel masks
    uint32_t st[NW];           // run-start masks
    alignas(16) uint16_t rbase[NW + 1];  // first run index of each word
    uint16_t rowlc[TH + 1];    // first tile component of each row
    uint16_t rowbx[TH + 1];    // border components before each row start
    alignas(16) uint16_t runpos[MR];  // (row << 8) | col of each run start, raster order
    alignas(16) typename C::PT par[MR];  // union-find parent; then component << 16 | root (analyze), component (emit)
    union {
        struct {
            alignas(16) uint16_t lcrun[C::NLC];  // root (first) run of each tile component
            alignas(16) uint16_t lcb[C::NLC];    // border index, or 0x8000 | (border components before it)
        };
        uint16_t evq[NWARPS][C::EVC];  // union-event queues (dead before lcrun/lcb are written)
    };
    uint16_t blc[C::NBC];      // border index -> tile component
    // analyze pass only (32-bit parents): root runs of each 32-run block (ballot), and the
    // root runs before each block
    static constexpr int RB = std::is_same<typename C::PT, uint32_t>::value ? C::MR / 32 + 1 : 1;
    uint32_t rmask[RB];
    uint32_t rbmask[RB];       // root runs of border components
    uint16_t rpre[RB];
    uint16_t bpre[RB];         // border components before each block
    int wsum[C::BT / 32 + 1];
    int qtot[NWARPS];          // union events queued by each word warp
    int nruns, nlc, nb;
    unsigned long long moff;   // offset of the tile's component map in the map store
};

// Where the analyze pass stores the tile's component map for the emit pass (written while
// the labels are resolved, so the map costs no extra pass over the runs).
struct MapOut {
    unsigned long long* used;  // map-store elements allocated (atomic bump)
    uint16_t* store;
    unsigned long long cap;
    uint64_t* tile_off;        // [tile] offset of its map
    uint32_t* err;             // error bits (ERR_RSTORE_CAP)
};

// map-store sections are padded to whole 16-B vectors
__host__ __device__ __forceinline__ int map_pad(int n) { return (n + 7) & ~7; }

// A tile's stored map, in u16 elements: [component of each run | first run of each component |
// border index of each component | first run of each word], each section padded to 8 elements.
// With the word bases stored, the emit pass needs no run scan of its own.
struct MapLayout {
    int lcrun, lcb, rbase, total;
    __host__ __device__ MapLayout(int nruns, int nlc) {
        lcrun = map_pad(nruns);
        lcb = lcrun + map_pad(nlc);
        rbase = lcb + map_pad(nlc);
        total = rbase + map_pad(NW + 1);
    }
};

template <class SM>
__device__ __forceinline__ int run_at(const SM& S, int word, int bit) {
    return (int)S.rbase[word] + __popc(S.st[word] & (0xFFFFFFFFu >> (31 - bit))) - 1;
}

// run of the pixel left of (word, bit); the caller guarantees it exists
template <class SM>
__device__ __forceinline__ int run_left(const SM& S, int word, int bit) {
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

// tile component of a run once the map pass is done: the analyze pass (32-bit parents) keeps the
// root run in the low half and stores the component in the high half; the emit pass loads the
// 16-bit map itself
template <class SM>
__device__ __forceinline__ uint32_t lc_of_run(const SM& S, int run) {
    if constexpr (sizeof(S.par[0]) == 4) return S.par[run] >> 16;
    else return S.par[run] & 0x7FFFu;
}

template <class SM>
__device__ __forceinline__ bool lc_is_border(const SM& S, uint32_t lc) {
    return (S.lcb[lc] & 0x8000u) == 0;
}

// tile component of pixel (r, c); pixel must be valid
template <class SM>
__device__ __forceinline__ uint32_t lc_at(const SM& S, int r, int c) {
    return lc_of_run(S, run_at(S, r * WPR + (c >> 5), c & 31));
}

// pixel value in "8-connected value" space at (r, c)
template <class SM>
__device__ __forceinline__ uint32_t xbit(const SM& S, int r, int c) {
    return (S.x[r * WPR + (c >> 5)] >> (c & 31)) & 1u;
}

template <class SM>
__device__ __forceinline__ int run_row(const SM& S, int i) { return S.runpos[i] >> 8; }
template <class SM>
__device__ __forceinline__ int run_col(const SM& S, int i) { return S.runpos[i] & 0xFF; }

// exclusive end column of run i
template <class SM>
__device__ __forceinline__ int run_end(const SM& S, int i, int tw) {
    if (i + 1 < S.nruns) {
        const uint16_t q = S.runpos[i + 1];
        if ((q >> 8) == (S.runpos[i] >> 8)) return q & 0xFF;
    }
    return tw;
}

template <class SM>
__device__ __forceinline__ int lc_row(const SM& S, uint32_t lc) { return run_row(S, S.lcrun[lc]); }
template <class SM>
__device__ __forceinline__ int lc_col(const SM& S, uint32_t lc) { return run_col(S, S.lcrun[lc]); }

// Full tile labeling.  Pre: S.x / S.vm filled for all NW words and a __syncthreads().
// Post (all synced): S.par[run] = TAG | component, S.runpos, S.lcrun, S.lcb (border index, or
// 0x8000 | border components before it), S.blc, S.nruns, S.nlc, S.nb; S.rowlc[r] and S.rowbx[r]
// are written by thread r only (visible to the others after the caller's next barrier).
// Returns false (uniformly) when the tile has more runs than the tables hold.
// Per-thread word state shared by the run and union phases.
struct WordBits {
    uint32_t x, nx, vm, c1, s1, s0, st;
    int nruns;
};

// Runs of the tile: start masks, raster-order run indices (block scan), run positions and
// identity parents.  Returns false (uniformly) when the tile has more runs than MR.
template <bool INIT_PAR = true, class C>
__device__ __forceinline__ bool tile_runs(CclSmem<C>& S, WordBits& wb) {
    constexpr int MR = C::MR;
    const int tid = threadIdx.x;
    const int r = tid / WPR, w = tid % WPR;
    // threads past NW (wide classes) own no word; their warps are uniformly idle here
    const bool word = C::BT == NW || tid < NW;
    wb = WordBits{};
    if (word) {
        wb.x = S.x[tid];
        wb.vm = S.vm[tid];
        wb.nx = ~wb.x;
        // left neighbour word of the same row is lane - 1 (rows never straddle a warp)
        const uint32_t xl = __shfl_up_sync(0xFFFFFFFFu, wb.x, 1);
        const uint32_t vml = __shfl_up_sync(0xFFFFFFFFu, wb.vm, 1);
        uint32_t c1 = 0, c0 = 0;
        if (w > 0) {
            const uint32_t lv = vml >> 31;
            c1 = (xl >> 31) & lv;
            c0 = ((~xl) >> 31) & lv;
        }
        wb.c1 = c1;
        wb.s1 = wb.x & ~((wb.x << 1) | c1) & wb.vm;
        wb.s0 = wb.nx & ~((wb.nx << 1) | c0) & wb.vm;
        wb.st = wb.s1 | wb.s0;
        S.st[tid] = wb.st;
    }
    int total;
#ifndef RL_SCAN_TRAIL
#define RL_SCAN_TRAIL 0
#endif
    // (the next write to S.wsum is the component scan, many barriers later)
    const int rb = block_excl_scan<C::BT, RL_SCAN_TRAIL>(__popc(wb.st), S.wsum, total);  // contains __syncthreads
    wb.nruns = total;
    if (total > MR) return false;
    if (!word) return true;
    S.rbase[tid] = (uint16_t)rb;
    if (tid == 0) {
        S.rbase[NW] = (uint16_t)total;
        S.nruns = total;
    }
    uint32_t m = wb.st;
    int i = rb;
    while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1u;
        S.runpos[i] = (uint16_t)((r << 8) | (32 * w + j));
        if (INIT_PAR) S.par[i] = (uint16_t)i;
        ++i;
    }
    return true;
}

// `border` is called by every lane of every warp, once per 32-run block of the map pass, with
// the run index, its border index (-1 for runs of interior components and past the last run)
// and whether the run is the first run of an interior component; border.init(nb) clears the
// border-component accumulators before that pass.
template <class C, class Border>
__device__ bool ccl_tile(CclSmem<C>& S, const TileGeom& tg, const MapOut& mo, Border&& border) {
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int r = tid / WPR, w = tid % WPR;
    WordBits wb;
    if (!tile_runs(S, wb)) return false;
    RL_PHASE(tg.t, 2);
    const uint32_t x = wb.x, nx = wb.nx, vm = wb.vm, c1 = wb.c1, s1 = wb.s1, s0 = wb.s0;
    // ---- union events with the row above (Alg. 2's overlap test, one event per pair),
    // compacted into the warp's queue: entry = (word << 7) | (type << 5) | bit
    constexpr int BT = C::BT;
    const bool word = BT == NW || tid < NW;
    uint32_t ev = 0, d1 = 0, d2 = 0;
    if (word && r >= 1 && vm) {
        const int ta = tid - WPR;
        const uint32_t a = S.x[ta], vma = S.vm[ta];
        // above row's starts/carry are recomputed locally (no dependency on other warps)
        uint32_t ca1 = 0, ca0 = 0;
        if (w > 0) {
            const uint32_t al = S.x[ta - 1], lva = S.vm[ta - 1] >> 31;
            ca1 = (al >> 31) & lva;
            ca0 = ((~al) >> 31) & lva;
        }
        const uint32_t na = ~a;
        const uint32_t sa1 = a & ~((a << 1) | ca1) & vma;
        const uint32_t sa0 = na & ~((na << 1) | ca0) & vma;
        const uint32_t both = vm & vma;
        ev = ((x & a & (s1 | sa1)) | (nx & na & (s0 | sa0))) & both;
        const uint32_t xl1 = (x << 1) | c1, al1 = (a << 1) | ca1;
        d1 = x & al1 & ~xl1 & na & both;  // (r, j) ~ (r-1, j-1)
        d2 = xl1 & a & nx & ~al1 & both;  // (r, j-1) ~ (r-1, j)
    }
    __syncthreads();  // run bases of every word are visible (the init below reads the row above)
    RL_PHASE(tg.t, 13);
    // ---- first contact: a run starting in this word takes the first run it touches in the
    // row above as its initial parent (cf. Alg. 2's `era[er] = find(above)`), and that contact
    // is not queued.  Contacts are ordered by column: the up-left diagonal at the run start
    // (d1), vertical contacts (ev), the up-right diagonal past the run end (d2, stored at the
    // next column).  Vertical stacks of equal runs (rows of a g x g block) need no union at all.
    if (word && r >= 1 && vm) {
        const int ta = tid - WPR;
        const uint32_t st = wb.st, sta = S.st[ta];
        const int rb = S.rbase[tid], rba = S.rbase[ta];
        // Bit-parallel "first contact of each run starting here": within each run segment
        // [start, next start) the carry of (noncontact + start) stops at the first contact
        // (a zero planted at each segment's last column stops it when there is none).
        const uint32_t contacts = d1 | ev | (d2 >> 1);
        const uint32_t nc = ~contacts & ~(st >> 1);
        const uint32_t first = contacts & (nc + st) & ~nc;
        const uint32_t f1 = first & d1, f2 = first & ev, f3 = first & ~d1 & ~ev;
        d1 &= ~f1;
        ev &= ~f2;
        d2 &= ~(f3 << 1);
        for (uint32_t m = first; m; m &= m - 1u) {
            const int j = __ffs(m) - 1;
            const uint32_t bit = 1u << j;
            // above-row column of the contact: j - 1 (d1), j (ev), j + 1 (d2)
            const uint32_t sh = (f1 & bit) ? 0u : (f2 & bit) ? 1u : 2u;
            const int above = rba - 1 + __popc(sta & (((1u << sh) << j) - 1u));
            const int k = rb - 1 + __popc(st & (0xFFFFFFFFu >> (31 - j)));
            S.par[k] = (uint16_t)above;
        }
    }
    const int nev = __popc(ev) + __popc(d1) + __popc(d2);
    int incl = nev;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += n;
    }
    const int wtot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    const int my0 = incl - nev;  // offset of this lane's first event in the warp's sequence
    // first-contact parents of every word are in place; tiles whose contacts were all first
    // contacts (vertical stacks of equal runs, sparse tiles) skip the union phase
    // (a block reduction returns 0/1: whether a warp's events exceed its queue is read from the
    // queue totals after the pre-flatten barrier)
    const int any_events = __syncthreads_or(nev);
    // class S: the warps fill their queues now (before the pre-flatten barrier) and after it all
    // threads drain all queues together, so a warp with many events does not hold the others at
    // the next barrier; a warp with more events than its queue holds stores the first EVC only,
    // and then every warp drains its own queue in rounds instead
    constexpr bool kSharedDrain = C::BT == NW;
    const bool shared_drain = kSharedDrain && any_events;
    RL_PHASE(tg.t, 14);
    // The first-contact forest links every run to one in the row above, so a vertical stack
    // of runs is a chain as tall as the stack.  It is flattened before the unions so that their
    // finds are short: every run walks its chain to the root and links to it directly.  The
    // walks run concurrently; a link read mid-walk is either the original one or a root
    // already written by another walker, both ancestors, so walks only get shorter.  (Row
    // groups with a barrier between them and pointer-jumping rounds were measured slower.)
    if (shared_drain) {
        if (my0 < C::EVC) {
            int o = my0;
            const uint16_t wbase = (uint16_t)(tid << 7);
            auto put = [&](uint32_t code) {
                if (o < C::EVC) S.evq[warp][o] = (uint16_t)code;
                ++o;
            };
            for (uint32_t e = ev; e; e &= e - 1u) put(wbase | (__ffs(e) - 1));
            for (uint32_t e = d1; e; e &= e - 1u) put(wbase | (1u << 5) | (__ffs(e) - 1));
            for (uint32_t e = d2; e; e &= e - 1u) put(wbase | (2u << 5) | (__ffs(e) - 1));
        }
        if (lane == 0) S.qtot[warp] = wtot;
    }
    {
        const int nr = S.nruns;
        const int rs = tg.th > 1 ? S.rbase[WPR] : nr;  // runs of row 0 have no first contact
        for (int i = rs + tid; i < nr; i += BT) {
            uint32_t p = S.par[i];
            if (p == (uint32_t)i) continue;  // no first contact: a root
            // walk to the root, publishing each step: walks that pass through run i then jump
            // as far as i's walk got (vertical stacks of runs: pointer jumping, log depth)
            for (;;) {
                const uint32_t q = S.par[p];
                if (q == p) break;
                p = q;
                S.par[i] = (uint16_t)p;
            }
        }
        __syncthreads();
    }
    RL_PHASE(tg.t, 3);
    // compact the warp's events into its queue (in rounds of EVC) and resolve them lane-parallel
    auto put_events = [&](int done) {
        int o = my0;
        const uint16_t wbase = (uint16_t)(tid << 7);
        auto put = [&](uint32_t code) {
            if (o >= done && o < done + C::EVC) S.evq[warp][o - done] = (uint16_t)code;
            ++o;
        };
        for (uint32_t e = ev; e; e &= e - 1u) put(wbase | (__ffs(e) - 1));
        for (uint32_t e = d1; e; e &= e - 1u) put(wbase | (1u << 5) | (__ffs(e) - 1));
        for (uint32_t e = d2; e; e &= e - 1u) put(wbase | (2u << 5) | (__ffs(e) - 1));
    };
    auto resolve_event = [&](uint32_t e) {
        const int wd = (int)(e >> 7), type = (int)((e >> 5) & 3u), j = (int)(e & 31u);
        const int wa = wd - WPR;
        uint32_t ra, rb2;
        if (type == 0) {
            ra = (uint32_t)run_at(S, wd, j);
            rb2 = (uint32_t)run_at(S, wa, j);
        } else if (type == 1) {
            ra = (uint32_t)run_at(S, wd, j);
            rb2 = (uint32_t)run_left(S, wa, j);
        } else {
            ra = (uint32_t)run_left(S, wd, j);
            rb2 = (uint32_t)run_at(S, wa, j);
        }
        sunion(S.par, ra, rb2);
    };
    int qoff[NWARPS + 1];
    bool queues_fit = true;
    if (shared_drain) {
        qoff[0] = 0;
#pragma unroll
        for (int q = 0; q < NWARPS; ++q) {
            const int n = S.qtot[q];
            queues_fit &= n <= C::EVC;
            qoff[q + 1] = qoff[q] + n;
        }
    }
    if (!any_events) {
        // nothing to unite
    } else if (shared_drain && queues_fit) {
        for (int k = tid; k < qoff[NWARPS]; k += BT) {
            int q = 0, base = 0;
#pragma unroll
            for (int t = 1; t < NWARPS; ++t)
                if (k >= qoff[t]) {
                    q = t;
                    base = qoff[t];
                }
            resolve_event(S.evq[q][k - base]);
        }
    } else if constexpr (BT == NW) {
        for (int done = 0; done < wtot; done += C::EVC) {
            if (nev && my0 < done + C::EVC && my0 + nev > done) put_events(done);
            __syncwarp();
            const int cnt = min(C::EVC, wtot - done);
            for (int k = lane; k < cnt; k += 32) resolve_event(S.evq[warp][k]);
            __syncwarp();
        }
    } else {
        // each queue is drained by the warp that filled it and by its partner warp past NW, in
        // rounds of EVC events (a word has <= 32 events: a warp <= 1024)
        if (word && lane == 0) S.qtot[warp] = wtot;
        __syncthreads();
        int maxq = 0;
#pragma unroll
        for (int q = 0; q < NWARPS; ++q) maxq = max(maxq, S.qtot[q]);
        const int q = warp & (NWARPS - 1);
        for (int done = 0; done < maxq; done += C::EVC) {
            if (word && nev && my0 < done + C::EVC && my0 + nev > done) put_events(done);
            __syncthreads();
            const int cnt = min(C::EVC, S.qtot[q] - done);
            for (int k = lane + 32 * (warp / NWARPS); k < cnt; k += 32 * (BT / NW)) resolve_event(S.evq[q][k]);
            __syncthreads();
        }
    }
    if (any_events && BT == NW) __syncthreads();
    RL_PHASE(tg.t, 4);

    // ---- roots (final now): a run is a root iff it is its own parent; each warp's ballot over a
    // 32-run block gives the block's roots.  The runs are not flattened here: the map pass walks
    // each run to its root (one pass over the runs instead of two).
    const int nruns = S.nruns;
    for (int b = warp * 32; b < nruns; b += BT) {
        const int i = b + lane;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, i < nruns && S.par[i] == (uint32_t)i);
        if (lane == 0) {
            S.rmask[b >> 5] = m;
            S.rbmask[b >> 5] = 0;
        }
    }
    __syncthreads();
    RL_PHASE(tg.t, 5);

    // ---- border components, marked at their root run: every row's first and last run (the
    // left and right tile columns: a row's first run starts at column 0, its last ends at the
    // tile edge) and every run of the top and bottom rows
    {
        const int top_end = S.rbase[WPR], bot_begin = S.rbase[(tg.th - 1) * WPR];
        auto mark = [&](uint32_t i) {
            uint32_t p = S.par[i];
            for (;;) {
                const uint32_t q = S.par[p];
                if (q == p) break;
                p = q;
            }
            atomicOr(&S.rbmask[p >> 5], 1u << (p & 31));
        };
        if (tid < tg.th) {
            mark(S.rbase[tid * WPR]);
            mark(S.rbase[(tid + 1) * WPR] - 1);
        }
        for (int i = tid; i < top_end; i += BT) mark(i);
        for (int i = bot_begin + tid; i < nruns; i += BT) mark(i);
    }
    __syncthreads();
    RL_PHASE(tg.t, 6);

    // ---- tile components = root runs, numbered in raster order, and border components among
    // them, by ONE prefix over the 32-run blocks of (roots | border roots << 16): a run's
    // component is its root's rank, a border component's index its root's rank among border
    // roots (no tagging pass, no separate compaction)
    const int nblk = (nruns + 31) >> 5;
    int nlc, nb;
    {
        int tot;
        const int pre = block_excl_scan<BT, RL_SCAN_TRAIL>(  // S.wsum is not written again in this tile
            tid < nblk ? (__popc(S.rmask[tid]) | (__popc(S.rbmask[tid]) << 16)) : 0, S.wsum, tot);
        if (tid < nblk) {
            S.rpre[tid] = (uint16_t)(pre & 0xFFFF);
            S.bpre[tid] = (uint16_t)(pre >> 16);
        }
        nlc = tot & 0xFFFF;
        nb = tot >> 16;
    }
    if (nlc > C::NLC) return false;  // more components than this class holds (uniform)
    if (nb > C::NBC) return false;   // more border components than this class holds
    auto rank_of = [&](uint32_t root) {  // valid once rpre is visible
        return (uint32_t)S.rpre[root >> 5] + __popc(S.rmask[root >> 5] & ((1u << (root & 31)) - 1u));
    };
    if (tid == 0) {
        S.nlc = nlc;
        S.nb = nb;
    }
    if (tid == 32) {  // the map (sections: MapLayout; the emit pass copies them with 16-B loads)
        const unsigned long long need = (unsigned long long)MapLayout(nruns, nlc).total;
        const unsigned long long off = atomicAdd(mo.used, need);
        if (off + need > mo.cap) atomicOr(mo.err, ERR_RSTORE_CAP);
        S.moff = off + need > mo.cap ? ~0ull : off;
        mo.tile_off[tg.t] = off;
    }
    border.init(nb);
    __syncthreads();
    RL_PHASE(tg.t, 8);

    const unsigned long long moff = S.moff;
    uint16_t* map = moff != ~0ull ? mo.store + moff : nullptr;
    const MapLayout ML(nruns, nlc);
    // ---- every run: walk to its root (the walks publish the roots they reach in the low half of
    // par, so concurrent walks through this run stop short; par's low half is an ancestor at
    // all times), then its component (the high half of par: component << 16 | root) and the map
    // entry; a component's first (root) run writes its first-run, border-index entries; runs of
    // border components feed the border features
    for (int b = warp * 32; b < nruns; b += BT) {
        const int i = b + lane;
        int bi = -1;
        bool iroot = false;
        if (i < nruns) {
            uint32_t root = S.par[i] & 0xFFFFu;
            for (;;) {
                const uint32_t q = S.par[root] & 0xFFFFu;
                if (q == root) break;
                root = q;
                S.par[i] = root;
            }
            const uint32_t l = rank_of(root);
            const uint32_t bm = S.rbmask[root >> 5], bit = 1u << (root & 31);
            const uint32_t bx = (uint32_t)S.bpre[root >> 5] + __popc(bm & (bit - 1u));
            const bool isb = (bm & bit) != 0;
            S.par[i] = (l << 16) | root;
            if (map) map[i] = (uint16_t)l;
            if (isb) bi = (int)bx;
            if (root == (uint32_t)i) {
                const uint16_t v = (uint16_t)(isb ? bx : (0x8000u | bx));
                S.lcrun[l] = (uint16_t)i;
                S.lcb[l] = v;
                if (isb) S.blc[bx] = (uint16_t)l;
                if (map) map[ML.lcb + l] = v;
                iroot = !isb;
            }
        }
        border(bi, i, iroot);
    }
    __syncthreads();
    // first component of each row (components before the row's first run) and the border
    // components before it; read by other threads only after the caller's next barrier
    if (tid <= TH) {
        const int k = tid < tg.th ? S.rbase[tid * WPR] : nruns;
        const int l = k < nruns ? (int)rank_of((uint32_t)k) : nlc;
        S.rowlc[tid] = (uint16_t)l;
        S.rowbx[tid] = l < nlc ? (uint16_t)(S.lcb[l] & 0x7FFF) : (uint16_t)nb;
    }
    if (map) {
        for (int l = tid; l < nlc; l += BT) map[ML.lcrun + l] = S.lcrun[l];
        for (int k = tid; k <= NW; k += BT) map[ML.rbase + k] = S.rbase[k];
    }
    RL_PHASE(tg.t, 9);
    return true;
}

}  // namespace rlg
