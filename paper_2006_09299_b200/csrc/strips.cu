// strips.cu -- one image cut into horizontal strips across ranks, with an O(W)
// exchange: only the components touching a cut row ("cut classes") and the cut rows' labels
// cross between ranks.
//
// Every rank runs the tile passes on its own strip with the geometry of the WHOLE image (tile
// rows [ty0, ty1), pixel row y at row y - prow0 of the rank's buffer), so the image frame is
// exterior only where it really is: cut rows are open.  Phases, with the caller's collectives
// between them (paper_2006_09299_b200/strips.py, torch.distributed / NCCL):
//
//   local    analyze + seams inside the strip, flatten (k_resolve); the local classes touching
//            a cut row are numbered 1..n (0 = the exterior); the strip counts its components
//            that touch no cut (interior + border ones).
//   export   per cut class: first-pixel key, fold of its features, foreground flag; the
//            strip's exterior partial features; both cut rows as (value << 31) | class.
//            O(W) bytes per strip.                                     [all-gather]
//   merge    (identical on every rank, over all strips' cut classes) union across the cuts,
//            fold features and min keys into global cut classes (GCC), the representative
//            class of every GCC (it holds the first pixel; its strip owns the GCC); per-strip
//            component counts give every strip's canonical id offset.  Then this strip's
//            numbering (k_reps / scan / k_cids with the GCC representatives counted only where
//            owned) and, for every owned GCC, its canonical id and where its parent chain
//            leaves the strip: the exterior (then its depth-1 ancestor is known) or another
//            GCC.                                                        [all-reduce SUM]
//   resolve  every GCC's depth-1 ancestor by walking the GCC links, then the unchanged tree
//            pass (k_tops stops at cut classes), emit, border folds; this rank's partial
//            post-fill sums of the GCC survivors.                        [all-reduce]
//   finish   survivors that cross a cut: reduced partials + their own features.
//
// Per-rank work is O(own strip + cut classes of all strips); nothing of another strip's
// interior is imported.  Canonical ids stay the raster order of first pixels over the whole
// image, so the strips' outputs concatenate to exactly the single-image result
// (labeling.hpp:190-217 numbering via tables.hpp:68-76).
//
// Why the GCC graph is all that crosses ranks: a component's parent is the component of the
// pixel left of its first pixel (same row, same strip), and whatever surrounds a component
// that touches a cut row also touches that cut (it has pixels on both sides of it), so every
// ancestor of a cut class is a cut class or the exterior, and every post-fill fold that
// crosses strips lands on a GCC survivor.
#include <cuda_runtime.h>


#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "runlab_gpu.h"

using namespace rlg;
using namespace rlh;

namespace {

// one cut class in the exchange record
struct XClass {
    uint64_t key;  // first pixel (global raster index); ~0 for the exterior entry
    Acc acc;       // the class's features inside this strip
    uint32_t fg, pad;
};
static_assert(sizeof(XClass) == 56, "XClass layout");

struct XHeader {
    int64_t n_classes;
    int32_t ty0, ty1;
    int64_t pad[6];
};
static_assert(sizeof(XHeader) == 64, "XHeader layout");

struct XLayout {
    size_t classes, cut, bytes;
};

size_t align8(size_t v) { return (v + 7) & ~size_t(7); }

XLayout x_layout(int32_t W, int64_t max_classes) {
    XLayout L;
    L.classes = sizeof(XHeader);
    L.cut = L.classes + align8((size_t)(max_classes + 1) * sizeof(XClass));
    L.bytes = L.cut + align8((size_t)2 * W * 4);
    return L;
}

// global cut-class tables (identical on every rank), laid out in ctx->gtab
struct GTab {
    uint32_t *uf, *root, *rep, *cid, *anc, *ancslot, *coff, *scnt, *gsurv;
    uint64_t* kmin;
    Acc* tot;
    int64_t *links, *psum, *pcnt;
    int32_t *pmin, *pmax;
    size_t bytes;
};

GTab g_layout(void* base, int64_t C, int k) {
    GTab T{};
    uint8_t* p = static_cast<uint8_t*>(base);
    size_t o = 0;
    auto take = [&](size_t b) {
        uint8_t* q = p ? p + o : nullptr;
        o += align8(b);
        return q;
    };
    T.links = reinterpret_cast<int64_t*>(take((size_t)C * 16));
    T.psum = reinterpret_cast<int64_t*>(take((size_t)C * 24));
    T.pcnt = reinterpret_cast<int64_t*>(take(8));
    T.pmin = reinterpret_cast<int32_t*>(take((size_t)C * 8));
    T.pmax = reinterpret_cast<int32_t*>(take((size_t)C * 8));
    T.tot = reinterpret_cast<Acc*>(take((size_t)C * sizeof(Acc)));
    T.kmin = reinterpret_cast<uint64_t*>(take((size_t)C * 8));
    T.uf = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.root = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.rep = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.cid = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.anc = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.ancslot = reinterpret_cast<uint32_t*>(take((size_t)C * 4));
    T.coff = reinterpret_cast<uint32_t*>(take((size_t)(k + 1) * 4));
    T.scnt = reinterpret_cast<uint32_t*>(take((size_t)2 * k * 4));
    T.gsurv = reinterpret_cast<uint32_t*>(take(8));
    T.bytes = o;
    return T;
}

#define GRID_LOOP(i, n) \
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)(n); i += (int64_t)gridDim.x * blockDim.x)

// ---- local phase ----------------------------------------------------------------------------

// node of the pixel left of each border component's first pixel (local numbering)
__global__ void k_strip_left(Geo g, Ws ws) {
    // after a capacity overflow the nodes of the tiles that did not fit were never written (the
    // host grows the tables and re-runs): their records must not be read
    if (ws.counters[1]) return;
    const uint32_t n_used = min(ws.counters[0], ws.cap_nodes);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_used; i += gridDim.x * blockDim.x) {
        const uint32_t n = 1u + i;
        const NodeRec rec = ws.nrec[n];
        uint32_t left = 0;
        if (rec.leftkind == 0) {
            left = 1u + ws.tbase[rec.tile] + rec.left;
        } else if (rec.leftkind == 1) {
            const uint32_t tl = rec.tile - 1;
            const uint16_t lab = ws.perim[(int64_t)tl * PERIM + 2 * TW + TH + rec.left];
            left = 1u + ws.tbase[tl] + (lab & 0x7FFFu);
        } else if (rec.leftkind != 2) {
            atomicOr(&ws.counters[1], ERR_INTERNAL);
        }
        ws.nleft[n] = left;
    }
}

// the exterior node (analyze initialises it only in the image's first tile)
__global__ void k_strip_exterior(Ws ws) {
    ws.uf[0] = 0;
    ws.nacc[0] = acc_empty();
    ws.nmin[0] = ~0ull;
    ws.nrootcid[0] = 0;
    ws.nparent[0] = 0;
    ws.nanccid[0] = 0;
    ws.nrep[0] = 0;
}

// root node of the cut-row pixel i (slot 0: the strip's top row, 1: its bottom row)
__device__ __forceinline__ uint32_t cut_root(const Geo& g, const Ws& ws, int64_t i, uint32_t& val) {
    const int32_t slot = (int32_t)(i / g.W), x = (int32_t)(i % g.W);
    const int32_t ty = slot ? g.ty1 - 1 : g.ty0;
    const int64_t t = (int64_t)ty * g.ntx + x / TW;
    const uint16_t lab = ws.perim[t * PERIM + (slot ? TW : 0) + x % TW];
    val = lab >> 15;
    return ws.uf[1u + ws.tbase[t] + (lab & 0x7FFFu)];
}

__global__ void k_strip_mark(Geo g, Ws ws, uint32_t* flag, int top, int bot) {
    if (ws.counters[1]) return;  // capacity overflow: nodes missing, the phase re-runs
    GRID_LOOP(i, 2 * (int64_t)g.W) {
        if ((i < g.W && !top) || (i >= g.W && !bot)) continue;
        uint32_t val;
        const uint32_t root = cut_root(g, ws, i, val);
        if (root != 0) flag[root] = 1u;
    }
}

// cut class -> root node; components touching no cut (border roots here, interior counts from
// the analyze pass's per-row counts): out[0] count, out[1] foreground
__global__ void k_strip_count(Geo g, Ws ws, const uint32_t* flag, const uint32_t* rank, uint32_t* xnode,
                              unsigned long long* out) {
    const uint32_t n_used = min(ws.counters[0], ws.cap_nodes);
    uint32_t cnt = 0, fg = 0;
    GRID_LOOP(i, n_used) {
        const uint32_t n = 1u + (uint32_t)i;
        if (ws.uf[n] != n) continue;
        if (flag[n]) {
            xnode[1u + rank[n]] = n;
        } else {
            ++cnt;
            fg += ws.nrec[n].fg;
        }
    }
    const int64_t r0 = (int64_t)g.ty0 * TH, r1 = min((int64_t)g.ty1 * TH, (int64_t)g.H);
    GRID_LOOP(i, (r1 - r0) * g.ntx) cnt += ws.cnt[r0 * g.ntx + i];
    cnt = __reduce_add_sync(0xFFFFFFFFu, cnt);
    fg = __reduce_add_sync(0xFFFFFFFFu, fg);
    if ((threadIdx.x & 31) == 0) {
        if (cnt) atomicAdd(out, (unsigned long long)cnt);
        if (fg) atomicAdd(out + 1, (unsigned long long)fg);
    }
}

__global__ void k_strip_pack(Geo g, Ws ws, const uint32_t* rank, const uint32_t* xnode, int64_t ncls, uint8_t* buf,
                             XLayout L, int top, int bot) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        XHeader h{};
        h.n_classes = ncls;
        h.ty0 = g.ty0;
        h.ty1 = g.ty1;
        *reinterpret_cast<XHeader*>(buf) = h;
    }
    XClass* xc = reinterpret_cast<XClass*>(buf + L.classes);
    GRID_LOOP(c, ncls + 1) {
        XClass x;
        if (c == 0) {
            x.key = ~0ull;
            x.acc = ws.nacc[0];
            x.fg = 0;
        } else {
            const uint32_t n = xnode[c];
            x.key = ws.nmin[n];
            x.acc = ws.nacc[n];
            x.fg = ws.nrec[n].fg;
        }
        x.pad = 0;
        xc[c] = x;
    }
    uint32_t* xr = reinterpret_cast<uint32_t*>(buf + L.cut);
    GRID_LOOP(i, 2 * (int64_t)g.W) {
        if ((i < g.W && !top) || (i >= g.W && !bot)) {
            xr[i] = 0xFFFFFFFFu;
            continue;
        }
        uint32_t val;
        const uint32_t root = cut_root(g, ws, i, val);
        xr[i] = (val << 31) | (root ? 1u + rank[root] : 0u);
    }
}

// ---- merge phase: global cut classes ----------------------------------------------------------

struct XSrc {
    const uint8_t* buf;  // n_strips consecutive records
    XLayout L;
    int32_t k;
};

__device__ __forceinline__ int32_t strip_of(const GTab& T, int32_t k, uint32_t i) {
    int32_t q = 0;
    while (q + 1 < k && T.coff[q + 1] <= i) ++q;
    return q;
}

__device__ __forceinline__ const XClass& xclass(const XSrc& X, int32_t q, uint32_t c) {
    return reinterpret_cast<const XClass*>(X.buf + (size_t)q * X.L.bytes + X.L.classes)[c];
}

__global__ void k_g_init(GTab T, int64_t C) {
    GRID_LOOP(i, C) {
        T.uf[i] = (uint32_t)i;
        T.kmin[i] = ~0ull;
        T.tot[i] = acc_empty();
        T.rep[i] = 0;
        T.links[2 * i] = 0;
        T.links[2 * i + 1] = 0;
    }
}

// cut q = blockIdx.y: the bottom row of strip q against the top row of strip q + 1 (all cuts in
// one launch)
__global__ void k_g_cut(XSrc X, GTab T, int32_t W, uint32_t v8) {
    const int32_t q = blockIdx.y;
    const uint32_t* up = reinterpret_cast<const uint32_t*>(X.buf + (size_t)q * X.L.bytes + X.L.cut) + W;
    const uint32_t* dn = reinterpret_cast<const uint32_t*>(X.buf + (size_t)(q + 1) * X.L.bytes + X.L.cut);
    const uint32_t cu0 = T.coff[q] - 1u, cd0 = T.coff[q + 1] - 1u;
    auto gi = [](uint32_t lab, uint32_t c0) { const uint32_t c = lab & 0x7FFFFFFFu; return c ? c0 + c : 0u; };
    GRID_LOOP(x, W) {
        const uint32_t lu = up[x], ld = dn[x];
        const uint32_t vu = lu >> 31, vd = ld >> 31;
        const uint32_t gu = gi(lu, cu0), gd = gi(ld, cd0);
        if (vu == vd) gunion(T.uf, gu, gd);
        if (x > 0) {
            const uint32_t lul = up[x - 1], ldl = dn[x - 1];
            if ((lul >> 31) == v8 && vd == v8) gunion(T.uf, gi(lul, cu0), gd);     // (r, x-1) ~ (r+1, x)
            if (vu == v8 && (ldl >> 31) == v8) gunion(T.uf, gu, gi(ldl, cd0));     // (r, x) ~ (r+1, x-1)
        }
    }
}

// roots, folded features and min keys; the strips' exterior partials fold into class 0.  The
// percolating component's classes (one per strip and cut) all fold into one root: lanes and
// blocks aggregate first (warp_fold + a shared table), as in k_resolve.
__global__ void __launch_bounds__(256) k_g_fold(XSrc X, GTab T, int64_t C) {
    __shared__ FoldTable<256> F;
    F.init();
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); base < C; base += stride) {
        const int64_t i = base + (threadIdx.x & 31);
        uint32_t dst = FT_EMPTY;
        Acc f;
        unsigned long long key = ~0ull;
        if (i == 0) {
            T.root[0] = 0;
        } else if (i < C) {
            const uint32_t root = gfind_ro(T.uf, (uint32_t)i);
            T.root[i] = root;
            const int32_t q = strip_of(T, X.k, (uint32_t)i);
            const XClass& x = xclass(X, q, (uint32_t)i - T.coff[q] + 1u);
            dst = root;
            f = x.acc;
            if (root) key = x.key;
        }
        warp_fold(F, dst, f, key, [&](uint32_t k) { return T.tot + k; },
                  [&](uint32_t k) { return reinterpret_cast<unsigned long long*>(T.kmin + k); });
    }
    __syncthreads();
    F.flush([&](uint32_t k) { return T.tot + k; },
            [&](uint32_t k) { return reinterpret_cast<unsigned long long*>(T.kmin + k); });
    GRID_LOOP(q, X.k) acc_atomic_fold(T.tot, xclass(X, (int32_t)q, 0).acc);
}

// representative class of every GCC (it holds the first pixel; its strip owns the GCC);
// scnt[q] = GCCs owned by strip q, scnt[k + q] = foreground ones
__global__ void k_g_reps(XSrc X, GTab T, int64_t C) {
    GRID_LOOP(i, C) {
        if (i == 0) continue;
        const uint32_t root = T.root[i];
        if (!root) continue;
        const int32_t q = strip_of(T, X.k, (uint32_t)i);
        const XClass& x = xclass(X, q, (uint32_t)i - T.coff[q] + 1u);
        if (x.key != T.kmin[root]) continue;
        T.rep[i] = 1u;
        atomicAdd(T.scnt + q, 1u);
        if (x.fg) atomicAdd(T.scnt + X.k + q, 1u);
    }
}

// this strip's cut classes take their GCC's status: joined to the exterior (relinked), owned
// (features = the GCC's total) or represented elsewhere (no representative node here, no
// features of its own: the owner folds the total)
__global__ void k_g_apply(Ws ws, GTab T, const uint32_t* xnode, int64_t ncls, uint32_t c0) {
    GRID_LOOP(c, ncls + 1) {
        if (c == 0) {
            ws.nacc[0] = T.tot[0];
            continue;
        }
        const uint32_t i = c0 + (uint32_t)c, n = xnode[c], root = T.root[i];
        if (root == 0) {
            ws.uf[n] = 0;
        } else {
            ws.ncut[n] = 1u + root;
            if (T.rep[i]) {
                ws.nacc[n] = T.tot[root];
            } else {
                ws.nacc[n] = acc_empty();
                ws.nmin[n] = ~0ull;  // matches no key: the class has no representative here
            }
        }
    }
}

__global__ void k_g_reflatten(Ws ws) {
    const uint32_t n_used = min(ws.counters[0], ws.cap_nodes);
    GRID_LOOP(i, n_used) {
        const uint32_t n = 1u + (uint32_t)i, u = ws.uf[n];
        if (u) ws.uf[n] = ws.uf[u];  // roots point at themselves or (now) at the exterior
    }
}

// slot in this strip's `filled` of GCC survivor e: its own id when this strip owns it, else one
// of the scratch slots past the owned range (where this strip's partial post-fill sums gather)
__device__ __forceinline__ uint32_t gcc_slot(const GTab& T, const Geo& g, uint32_t e) {
    const uint32_t cid = T.cid[e];
    return ((int64_t)cid >= g.cid_lo && (int64_t)cid < g.cid_hi) ? cid : (uint32_t)g.cid_hi + e;
}

// owned GCCs: canonical id and where the parent chain leaves this strip.  links[2 root] = id,
// links[2 root + 1] = depth-1 ancestor's id (> 0) when the chain reaches the exterior inside
// the strip, -(GCC root) when it reaches another cut class first.
__global__ void k_g_links(Ws ws, GTab T, const uint32_t* xnode, int64_t ncls, uint32_t c0, uint32_t n_local) {
    GRID_LOOP(c, ncls + 1) {
        if (c == 0) continue;
        const uint32_t i = c0 + (uint32_t)c;
        if (!T.rep[i]) continue;
        const uint32_t n = xnode[c], root = T.root[i];
        int64_t link = 0;
        uint32_t cur = n;
        for (uint32_t it = 0; it <= n_local; ++it) {
            const uint32_t p = ws.nparent[cur];
            if (p == 0) {
                link = (int64_t)ws.nrootcid[cur];
                break;
            }
            if (ws.ncut[p]) {
                link = -(int64_t)(ws.ncut[p] - 1u);
                break;
            }
            cur = p;
        }
        if (link == 0) atomicOr(&ws.counters[1], ERR_INTERNAL);
        T.links[2 * root] = (int64_t)ws.nrootcid[n];
        T.links[2 * root + 1] = link;
    }
}

// ---- resolve phase ----------------------------------------------------------------------------

// every GCC's id and depth-1 ancestor (walk of the GCC links); survivors' post-fill slots start
// empty on every rank (they collect this rank's folds)
__global__ void k_g_anc(Geo g, Ws ws, GTab T, int64_t C) {
    uint32_t ns = 0;
    GRID_LOOP(i, C) {
        if (i == 0 || T.root[i] != (uint32_t)i) continue;
        const uint32_t cid = (uint32_t)T.links[2 * i];
        uint32_t e = (uint32_t)i, anc = 0;
        for (int64_t it = 0; it < C; ++it) {
            const int64_t l = T.links[2 * e + 1];
            if (l > 0) {  // e is a child of the exterior: the depth-1 ancestor (l is its id)
                anc = (uint32_t)l;
                break;
            }
            if (l == 0) break;
            e = (uint32_t)(-l);
        }
        if (!anc || !cid) atomicOr(&ws.counters[1], ERR_INTERNAL);
        T.cid[i] = cid;
        T.anc[i] = anc;
        T.ancslot[i] = e;
        if (anc == cid && cid) ++ns;
    }
    ns = __reduce_add_sync(0xFFFFFFFFu, ns);
    if ((threadIdx.x & 31) == 0 && ns) atomicAdd(T.gsurv, ns);
}

// survivors' post-fill slots start empty on every rank (they collect this rank's folds)
__global__ void k_g_surv_init(Geo g, Ws ws, GTab T, int64_t C) {
    GRID_LOOP(i, C) {
        if (i == 0 || T.root[i] != (uint32_t)i || T.anc[i] != T.cid[i]) continue;
        ws.filled[gcc_slot(T, g, (uint32_t)i)] = acc_empty();
    }
}

__global__ void k_g_own(Geo g, Ws ws, GTab T, const uint32_t* xnode, int64_t ncls, uint32_t c0) {
    GRID_LOOP(c, ncls + 1) {
        if (c == 0) continue;
        const uint32_t root = T.root[c0 + (uint32_t)c];
        if (!root) continue;
        const uint32_t n = xnode[c];
        ws.nrootcid[n] = T.cid[root];
        ws.nanccid[n] = T.anc[root];
        ws.nfold[n] = gcc_slot(T, g, T.ancslot[root]);
    }
}

// this rank's partial post-fill sums of the GCC survivors (neutral elsewhere), indexed by GCC root
__global__ void k_g_partials(Geo g, Ws ws, GTab T, int64_t C, const uint32_t* surv_a, const uint32_t* surv_b,
                             int32_t sub) {
    GRID_LOOP(i, C) {
        Acc f = acc_empty();
        if (i > 0 && T.root[i] == (uint32_t)i && T.anc[i] == T.cid[i]) f = ws.filled[gcc_slot(T, g, (uint32_t)i)];
        T.psum[3 * i] = f.s;
        T.psum[3 * i + 1] = f.sx;
        T.psum[3 * i + 2] = f.sy;
        T.pmin[2 * i] = f.row_min;
        T.pmin[2 * i + 1] = f.col_min;
        T.pmax[2 * i] = f.row_max;
        T.pmax[2 * i + 1] = f.col_max;
    }
    // survivors that touch no cut (interior + border; the exterior counted on strip 0 only)
    if (blockIdx.x == 0 && threadIdx.x == 0) *T.pcnt = (int64_t)*surv_a + (int64_t)*surv_b - sub;
}

__global__ void k_g_finish(Geo g, Ws ws, GTab T, int64_t C) {
    GRID_LOOP(i, C) {
        if (i == 0 || T.root[i] != (uint32_t)i || T.anc[i] != T.cid[i]) continue;
        const Acc a = T.tot[i];
        Acc f;
        f.s = T.psum[3 * i] + a.s;
        f.sx = T.psum[3 * i + 1] + a.sx;
        f.sy = T.psum[3 * i + 2] + a.sy;
        f.row_min = min(T.pmin[2 * i], a.row_min);
        f.col_min = min(T.pmin[2 * i + 1], a.col_min);
        f.row_max = max(T.pmax[2 * i], a.row_max);
        f.col_max = max(T.pmax[2 * i + 1], a.col_max);
        ws.filled[gcc_slot(T, g, (uint32_t)i)] = f;  // kept (fetched) where owned
    }
}

int grid(int64_t n, int sms) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8)); }

}  // namespace

namespace rlh {

struct StripState {
    Geo g{};
    rl_config cfg{};
    int32_t y0 = 0, h = 0;
    int32_t rank = -1, n_strips = 0;
    const uint8_t* pix = nullptr;
    int64_t n_local = 0, n_classes = 0, n_comps = 0, n_fg = 0;
    // global phase
    int64_t C = 0;          // global class slots (1 + all strips' cut classes)
    int64_t total = 0, fg = 0, comp_lo = 0, comp_hi = 0;
    uint32_t c0 = 0;        // this strip's classes are global slots c0 + 1 .. c0 + n_classes
    int phase = 0;          // 1 local, 2 exported, 3 merged, 4 resolved
};

}  // namespace rlh

namespace {

StripState* strip_state(rl_ctx* c) {
    if (!c->strip) c->strip = new StripState();
    return c->strip;
}

// Pinned staging for the phases' small transfers: copies from or to pageable host memory would
// each wait for the stream (a host round trip per counter); these are asynchronous and the phase
// synchronises once.
uint8_t* strip_pinned(rl_ctx* c, size_t bytes) {
    if (c->h_strip_n < bytes) {
        if (c->h_strip) cudaFreeHost(c->h_strip);
        c->h_strip = nullptr;
        c->h_strip_n = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        if (cudaMallocHost(&c->h_strip, want) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        c->h_strip_n = want;
    }
    return c->h_strip;
}

int sync_err(rl_ctx* c, const char* what) {
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? RL_OK : cuda_fail(c, e, what);
}

// RUNLAB_GPU_STRIP_DEBUG=1: synchronise after every launch of the strip phases and name the
// kernel that failed (diagnostics; the phases otherwise synchronise once at their end)
bool strip_debug() {
    static const bool on = std::getenv("RUNLAB_GPU_STRIP_DEBUG") != nullptr;
    return on;
}
#define STRIP_STEP(ctx, name)                                                                     \
    do {                                                                                          \
        if (strip_debug()) {                                                                      \
            const cudaError_t e_ = cudaStreamSynchronize((ctx)->stream);                          \
            if (e_ != cudaSuccess) return cuda_fail(ctx, e_, name);                               \
        }                                                                                         \
    } while (0)

GTab gtab(rl_ctx* ctx) {
    const StripState* S = ctx->strip;
    return g_layout(ctx->gtab.p, S->C, S->n_strips);
}

}  // namespace

namespace rlh {
void strip_free(rl_ctx* c) {
    delete c->strip;
    c->strip = nullptr;
}
}  // namespace rlh

extern "C" {

int64_t rl_strip_export_bytes(int32_t w, int64_t max_classes) {
    return (int64_t)x_layout(w, max_classes).bytes;
}

int rl_strip_local(rl_ctx* ctx, const uint8_t* d_strip, int32_t w, int32_t H, int32_t y0, int32_t h,
                   const rl_config* cfg, rl_strip_local_info* out) {
    if (!out) return RL_EINVAL;
    int rc = check_args(ctx, w, H, 1, cfg);
    if (rc) return rc;
    if (cfg->densify_labels) return set_err(ctx, RL_EINVAL, "strips: densify_labels is not supported");
    if (y0 < 0 || h < 1 || y0 + h > H || y0 % TH || (y0 + h < H && h % TH))
        return set_err(ctx, RL_EINVAL, "strips: rows must start and (except the last strip) end on a multiple of 32");
    cudaSetDevice(ctx->device);
    StripState* S = strip_state(ctx);
    Geo g = make_geo(w, H, 1, cfg, d_strip);
    if (g.ntiles < 0) return set_err(ctx, RL_EINVAL, "too many tiles");
    g.ty0 = y0 / TH;
    g.ty1 = (y0 + h + TH - 1) / TH;
    g.prow0 = y0;
    g.strip = 1;
    g.cell_end = std::min<int64_t>((int64_t)g.ty1 * TH, H) * g.ntx;  // the strip's end cell
    S->g = g;
    S->cfg = *cfg;
    S->y0 = y0;
    S->h = h;
    S->pix = d_strip;
    S->phase = 0;
    ctx->want_compact = false;
    cudaStream_t s = ctx->stream;
    const int top = g.ty0 > 0, bot = g.ty1 < g.nty;
    for (int attempt = 0; attempt < 4; ++attempt) {
        Ws ws;
        size_t tmp = 0;
        if ((rc = prepare_ws(ctx, g, cfg, ws, tmp, (int64_t)h * w))) return rc;
        const size_t nn = (size_t)ctx->cap_nodes + 1;
        if (!ensure(ctx->nleft, nn * 4) || !ensure(ctx->ncut, nn * 4) || !ensure(ctx->nfold, nn * 4) ||
            !ensure(ctx->flag, nn * 4) ||
            !ensure(ctx->rank, nn * 4) || !ensure(ctx->xnode, nn * 4) || !ensure(ctx->scount, 64))
            return set_err(ctx, RL_ENOMEM, "device allocation failed");
        if (!ensure(ctx->cub_tmp, std::max(tmp, scan_state_bytes((int64_t)nn))))
            return set_err(ctx, RL_ENOMEM, "device allocation failed");
        ws.nleft = P<uint32_t>(ctx->nleft);
        ws.ncut = P<uint32_t>(ctx->ncut);
        ws.nfold = P<uint32_t>(ctx->nfold);
        cudaMemsetAsync(ws.counters, 0, 64, s);
        cudaMemsetAsync(ws.rused, 0, 8, s);
        cudaMemsetAsync(ws.img_fg, 0, 4, s);
        cudaMemsetAsync(ws.uf, 0, 4, s);  // the exterior node: seams reach it before k_strip_exterior
        // the numbering scan reads one cell past this strip's rows (the analyze pass writes the rest)
        cudaMemsetAsync(ws.cnt + std::min<int64_t>((int64_t)g.ty1 * TH, H) * g.ntx, 0, 4, s);
        launch_analyze(d_strip, g, ws, s);
        STRIP_STEP(ctx, "launch_analyze");
        enqueue_seams(ctx, g, ws, s);
        STRIP_STEP(ctx, "launch_seams");
        k_strip_left<<<grid((int64_t)ctx->cap_nodes, ctx->sms), 256, 0, s>>>(g, ws);
        STRIP_STEP(ctx, "k_strip_left");
        ctx->launches = 3 + (g.ty1 - g.ty0 > 1) + (g.ntx > 1) + 1;
        // flatten inside the strip; cut classes = roots seen on a cut row, numbered by a scan.
        // No host round trip in between: grids and tables are sized by the node capacity (the
        // kernels read the node count on the device), and a capacity overflow is found at the
        // phase's one synchronisation below (the host then grows the tables and re-runs)
        const int64_t nmax = (int64_t)ctx->cap_nodes;
        k_strip_exterior<<<1, 1, 0, s>>>(ws);
        STRIP_STEP(ctx, "k_strip_exterior");
        launch_resolve(g, ws, s, ctx->sms, nmax);
        STRIP_STEP(ctx, "launch_resolve");
        uint32_t* flag = P<uint32_t>(ctx->flag);
        uint32_t* rank = P<uint32_t>(ctx->rank);
        cudaMemsetAsync(flag, 0, (size_t)(nmax + 1) * 4, s);
        cudaMemsetAsync(ws.ncut, 0, (size_t)(nmax + 1) * 4, s);
        k_strip_mark<<<grid(2 * (int64_t)w, ctx->sms), 256, 0, s>>>(g, ws, flag, top, bot);
        STRIP_STEP(ctx, "k_strip_mark");
        launch_scan(flag, rank, nmax + 1, 0u, ctx->cub_tmp.p, s);
        unsigned long long* cnt2 = P<unsigned long long>(ctx->scount);
        cudaMemsetAsync(cnt2, 0, 16, s);
        k_strip_count<<<grid(std::max<int64_t>(nmax, (int64_t)(g.ty1 - g.ty0) * TH * g.ntx), ctx->sms), 256, 0, s>>>(
            g, ws, flag, rank, P<uint32_t>(ctx->xnode), cnt2);
        STRIP_STEP(ctx, "k_strip_count");
        uint8_t* hp = strip_pinned(ctx, 96);
        if (!hp) return set_err(ctx, RL_ENOMEM, "pinned alloc failed");
        uint32_t* hc = reinterpret_cast<uint32_t*>(hp);                      // [8] counters
        uint32_t* hfg = reinterpret_cast<uint32_t*>(hp + 32);                // img_fg
        unsigned long long* hrused = reinterpret_cast<unsigned long long*>(hp + 40);
        uint32_t* klast = reinterpret_cast<uint32_t*>(hp + 48);             // [2]
        unsigned long long* hcnt = reinterpret_cast<unsigned long long*>(hp + 56);  // [2]
        cudaMemcpyAsync(hc, ws.counters, 32, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(hfg, ws.img_fg, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(hrused, ws.rused, 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&klast[0], rank + nmax, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&klast[1], flag + nmax, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(hcnt, cnt2, 16, cudaMemcpyDeviceToHost, s);
        if ((rc = sync_err(ctx, "strip local"))) return rc;
        const uint32_t fg = *hfg;
        const unsigned long long rused = *hrused;
        if (hc[1] & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (strip left link)");
        if (hc[1] & (ERR_NODE_CAP | ERR_RSTORE_CAP)) {
            if (hc[1] & ERR_NODE_CAP) ctx->cap_nodes = (uint32_t)std::min<uint64_t>(hc[0] + hc[0] / 4 + 1024, 0xF0000000ull);
            if (hc[1] & ERR_RSTORE_CAP) ctx->cap_rstore = rused + rused / 8 + 4096;
            continue;
        }
        const int64_t n_local = hc[0];
        ctx->launches += 6;
        ctx->ws = ws;
        ctx->geo = g;
        S->n_local = n_local;
        S->n_classes = (int64_t)klast[0] + klast[1];
        S->n_comps = (int64_t)hcnt[0];
        S->n_fg = (int64_t)hcnt[1] + fg;
        S->phase = 1;
        out->n_classes = S->n_classes;
        out->n_comps = S->n_comps;
        out->n_fg = S->n_fg;
        out->ty0 = g.ty0;
        out->ty1 = g.ty1;
        out->status = 0;
        out->pad = 0;
        return RL_OK;
    }
    return set_err(ctx, RL_EINTERNAL, "capacity did not converge");
}

int rl_strip_export(rl_ctx* ctx, int64_t max_classes, void* d_buf) {
    if (!ctx || !d_buf) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || S->phase < 1) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_local first");
    if (S->n_classes > max_classes) return set_err(ctx, RL_EINVAL, "strips: export record too small");
    cudaSetDevice(ctx->device);
    const Geo& g = S->g;
    const XLayout L = x_layout(g.W, max_classes);
    k_strip_pack<<<grid(std::max<int64_t>(S->n_classes + 1, 2 * (int64_t)g.W), ctx->sms), 256, 0, ctx->stream>>>(
        g, ctx->ws, P<uint32_t>(ctx->rank), P<uint32_t>(ctx->xnode), S->n_classes, static_cast<uint8_t*>(d_buf), L,
        g.ty0 > 0, g.ty1 < g.nty);
    STRIP_STEP(ctx, "k_strip_pack");
    ctx->launches += 1;
    S->phase = 2;
    return sync_err(ctx, "strip export");
}

int rl_strip_merge(rl_ctx* ctx, const void* d_gathered, int32_t n_strips, const rl_strip_local_info* infos,
                   int64_t max_classes, rl_strip_links* out) {
    if (!ctx || !d_gathered || !infos || !out || n_strips < 1) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || S->phase < 2) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_export first");
    cudaSetDevice(ctx->device);
    Geo g = S->g;
    cudaStream_t s = ctx->stream;
    // this strip's position among the records: strips are given in image order
    int me = -1;
    int64_t C = 1;
    std::vector<uint32_t> coff(n_strips + 1);
    for (int q = 0; q < n_strips; ++q) {
        if (infos[q].n_classes > max_classes || infos[q].n_classes < 0)
            return set_err(ctx, RL_EINVAL, "strips: inconsistent class counts");
        if (q > 0 && infos[q].ty0 != infos[q - 1].ty1) return set_err(ctx, RL_EINVAL, "strips: records not in image order");
        if (infos[q].ty0 == g.ty0) me = q;
        coff[q] = (uint32_t)C;
        C += infos[q].n_classes;
    }
    coff[n_strips] = (uint32_t)C;
    if (me < 0 || infos[me].n_classes != S->n_classes) return set_err(ctx, RL_EINVAL, "strips: this strip is not among the records");
    if (infos[0].ty0 != 0 || infos[n_strips - 1].ty1 != g.nty) return set_err(ctx, RL_EINVAL, "strips: records do not cover the image");
    if (C >= 0x7FFFFFFFll) return set_err(ctx, RL_EINVAL, "strips: too many cut classes");
    S->rank = me;
    S->n_strips = n_strips;
    S->C = C;
    S->c0 = coff[me] - 1u;
    if (!ensure(ctx->gtab, g_layout(nullptr, C, n_strips).bytes)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
    GTab T = gtab(ctx);
    const XSrc X{static_cast<const uint8_t*>(d_gathered), x_layout(g.W, max_classes), n_strips};
    uint8_t* hp = strip_pinned(ctx, (size_t)(n_strips + 1) * 4 + (size_t)2 * n_strips * 4 + 64);
    if (!hp) return set_err(ctx, RL_ENOMEM, "pinned alloc failed");
    uint32_t* hcoff = reinterpret_cast<uint32_t*>(hp);
    uint32_t* hsc = hcoff + (n_strips + 1);
    std::copy(coff.begin(), coff.end(), hcoff);
    cudaMemcpyAsync(T.coff, hcoff, (n_strips + 1) * 4, cudaMemcpyHostToDevice, s);
    cudaMemsetAsync(T.scnt, 0, (size_t)2 * n_strips * 4, s);
    cudaMemsetAsync(T.gsurv, 0, 4, s);
    // ---- global cut classes (identical on every rank)
    k_g_init<<<grid(C, ctx->sms), 256, 0, s>>>(T, C);
    STRIP_STEP(ctx, "k_g_init");
    const uint32_t v8 = g.flip ? 0u : 1u;
    if (n_strips > 1)
        k_g_cut<<<dim3((unsigned)std::min<int64_t>((g.W + 255) / 256, 4096), (unsigned)(n_strips - 1)), 256, 0, s>>>(
            X, T, g.W, v8);
    STRIP_STEP(ctx, "k_g_cut");
    k_g_fold<<<grid(C, ctx->sms), 256, 0, s>>>(X, T, C);
    STRIP_STEP(ctx, "k_g_fold");
    k_g_reps<<<grid(C, ctx->sms), 256, 0, s>>>(X, T, C);
    STRIP_STEP(ctx, "k_g_reps");
    cudaMemcpyAsync(hsc, T.scnt, (size_t)2 * n_strips * 4, cudaMemcpyDeviceToHost, s);
    int rc = sync_err(ctx, "strip cut merge");
    if (rc) return rc;
    const std::vector<uint32_t> sc(hsc, hsc + 2 * n_strips);
    int64_t total = 1, fg = 0, off_me = 0;
    for (int q = 0; q < n_strips; ++q) {
        if (q == me) off_me = total - 1;
        total += infos[q].n_comps + sc[q];
        fg += infos[q].n_fg + sc[n_strips + q];
    }
    if (total >= 0xFFFFFFFFll) return set_err(ctx, RL_EINVAL, "strips: too many components");
    S->total = total;
    S->fg = fg;
    S->comp_lo = me == 0 ? 0 : 1 + off_me;
    S->comp_hi = 1 + off_me + infos[me].n_comps + sc[me];
    // ---- this strip's numbering with the GCC status applied (ids index the whole image; the
    // component tables hold the owned ids [comp_lo, comp_hi) and one scratch slot per cut class)
    g.cid_lo = S->comp_lo;
    g.cid_hi = S->comp_hi;
    g.cid_extra = C;
    S->g = g;
    const uint64_t need = (uint64_t)(S->comp_hi - S->comp_lo) + (uint64_t)C;
    if (ctx->cap_comps < need) ctx->cap_comps = need + need / 8 + 1024;
    Ws ws;
    size_t tmp = 0;
    if ((rc = prepare_ws(ctx, g, &S->cfg, ws, tmp, (int64_t)S->h * g.W))) return rc;
    ws.nleft = P<uint32_t>(ctx->nleft);
    ws.ncut = P<uint32_t>(ctx->ncut);
    ws.nfold = P<uint32_t>(ctx->nfold);
    const uint32_t* xnode = P<uint32_t>(ctx->xnode);
    k_g_apply<<<grid(S->n_classes + 1, ctx->sms), 256, 0, s>>>(ws, T, xnode, S->n_classes, S->c0);
    STRIP_STEP(ctx, "k_g_apply");
    k_g_reflatten<<<grid(S->n_local, ctx->sms), 256, 0, s>>>(ws);
    STRIP_STEP(ctx, "k_g_reflatten");
    cudaMemsetAsync(ws.img_surv, 0, 4, s);
    launch_reps(g, ws, s, ctx->sms, S->n_local);
    STRIP_STEP(ctx, "launch_reps");
    // offsets of this strip's rows only, starting at the components of the strips above; off[0]
    // (the image base) and the end cell are what the numbering passes read outside them
    const int64_t c_lo = (int64_t)g.ty0 * TH * g.ntx, c_hi = std::min<int64_t>((int64_t)g.ty1 * TH, g.H) * g.ntx;
    if (!ensure(ctx->cub_tmp, scan_state_bytes(c_hi - c_lo + 1))) return set_err(ctx, RL_ENOMEM, "device allocation failed");
    launch_scan(ws.cnt + c_lo, ws.off + c_lo, c_hi - c_lo + 1, (uint32_t)off_me, ctx->cub_tmp.p, s);
    launch_cids(g, ws, s, ctx->sms);
    STRIP_STEP(ctx, "launch_cids");
    k_g_links<<<grid(S->n_classes + 1, ctx->sms), 256, 0, s>>>(ws, T, xnode, S->n_classes, S->c0,
                                                                 (uint32_t)S->n_local);
    STRIP_STEP(ctx, "k_g_links");
    uint32_t* herr = reinterpret_cast<uint32_t*>(strip_pinned(ctx, 64));  // the buffer exists (grown above)
    cudaMemcpyAsync(herr, ws.counters + 1, 4, cudaMemcpyDeviceToHost, s);
    if ((rc = sync_err(ctx, "strip merge"))) return rc;
    const uint32_t err = *herr;
    if (err & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (strip links)");
    ctx->ws = ws;
    ctx->geo = g;
    ctx->launches += 4 + (n_strips > 1) + 6;
    out->d_links = T.links;
    out->n = 2 * C;
    S->phase = 3;
    return RL_OK;
}

int rl_strip_resolve(rl_ctx* ctx, rl_strip_partials* out) {
    if (!ctx || !out) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || S->phase < 3) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_merge first");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    Ws ws = ctx->ws;
    const Geo& g = S->g;
    GTab T = gtab(ctx);
    const int64_t C = S->C;
    k_g_anc<<<grid(C, ctx->sms), 256, 0, s>>>(g, ws, T, C);
    STRIP_STEP(ctx, "k_g_anc");
    k_g_surv_init<<<grid(C, ctx->sms), 256, 0, s>>>(g, ws, T, C);
    STRIP_STEP(ctx, "k_g_surv_init");
    k_g_own<<<grid(S->n_classes + 1, ctx->sms), 256, 0, s>>>(g, ws, T, P<uint32_t>(ctx->xnode), S->n_classes, S->c0);
    STRIP_STEP(ctx, "k_g_own");
    launch_tree_parts(g, ws, s, ctx->sms, S->n_local);  // post-fill roots (no fold yet)
    STRIP_STEP(ctx, "launch_tree_parts");
    // emit this strip's tiles; interior survivors are counted into a private counter
    Ws we = ws;
    uint32_t* isurv = P<uint32_t>(ctx->scount) + 4;
    we.img_surv = isurv;
    cudaMemsetAsync(isurv, 0, 4, s);
    if (ctx->seam_stream)
        launch_emit(g, we, s, ctx->seam_stream, ctx->seam_fork, ctx->seam_join);
    else
        launch_emit(g, we, s);
    STRIP_STEP(ctx, "launch_emit");
    launch_fold(g, ws, s, ctx->sms, S->n_local);  // border non-survivors of this strip
    STRIP_STEP(ctx, "launch_fold");
    k_g_partials<<<grid(C, ctx->sms), 256, 0, s>>>(g, ws, T, C, ws.img_surv, isurv, S->rank > 0 ? 1 : 0);
    STRIP_STEP(ctx, "k_g_partials");
    uint32_t* herr = reinterpret_cast<uint32_t*>(strip_pinned(ctx, 64));
    if (!herr) return set_err(ctx, RL_ENOMEM, "pinned alloc failed");
    cudaMemcpyAsync(herr, ws.counters + 1, 4, cudaMemcpyDeviceToHost, s);
    const int rc = sync_err(ctx, "strip resolve");
    if (rc) return rc;
    const uint32_t err = *herr;
    if (err & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (strip tree)");
    ctx->launches += 3 + 1 + 3 + (g.tpi >= 8192 ? 1 : 0) + 1 + 1;
    out->d_sum = T.psum;
    out->d_min = T.pmin;
    out->d_max = T.pmax;
    out->d_count = T.pcnt;
    out->k = C;
    S->phase = 4;
    return RL_OK;
}

int rl_strip_finish(rl_ctx* ctx, rl_strip_result* out) {
    if (!ctx || !out) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || S->phase < 4) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_resolve first");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    GTab T = gtab(ctx);
    k_g_finish<<<grid(S->C, ctx->sms), 256, 0, s>>>(S->g, ctx->ws, T, S->C);
    STRIP_STEP(ctx, "k_g_finish");
    ctx->launches += 1;
    uint8_t* hp = strip_pinned(ctx, 64);
    if (!hp) return set_err(ctx, RL_ENOMEM, "pinned alloc failed");
    cudaMemcpyAsync(hp, T.pcnt, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(hp + 8, T.gsurv, 4, cudaMemcpyDeviceToHost, s);
    const int rc = sync_err(ctx, "strip finish");
    if (rc) return rc;
    const int64_t surv = *reinterpret_cast<const int64_t*>(hp);
    const uint32_t gsurv = *reinterpret_cast<const uint32_t*>(hp + 8);
    out->n_components = S->total;
    out->n_fg = S->fg;
    out->n_holes = S->total - 1 - S->fg;
    out->euler = S->fg - out->n_holes;
    out->n_survivors = surv + gsurv;
    out->comp_lo = S->comp_lo;
    out->comp_hi = S->comp_hi;
    out->y0 = S->y0;
    out->h = S->h;
    return RL_OK;
}

int rl_strip_fetch(rl_ctx* ctx, const rl_strip_result* r, rl_host_outputs* out) {
    if (!ctx || !r || !out) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || S->phase < 4) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_finish first");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    const size_t npx = (size_t)S->h * S->g.W;
    const int64_t n = r->comp_hi - r->comp_lo;
    int64_t d2h = 0;
    if (out->filled_image) {
        cudaMemcpyAsync(out->filled_image, ctx->ws.filled_img, npx, cudaMemcpyDeviceToHost, s);
        d2h += (int64_t)npx;
    }
    if (out->labels && S->g.label_mode) {
        cudaMemcpyAsync(out->labels, ctx->ws.labels, npx * 4, cudaMemcpyDeviceToHost, s);
        d2h += (int64_t)npx * 4;
    }
    out->comps_needed = n;
    if ((out->comps || out->top || out->filled) && n > out->comp_capacity)
        return set_err(ctx, RL_ENOSPC, "component buffers too small");
    if (out->comps) cudaMemcpyAsync(out->comps, ctx->ws.comps + r->comp_lo, n * sizeof(rl_component), cudaMemcpyDeviceToHost, s);
    if (out->top) cudaMemcpyAsync(out->top, ctx->ws.top + r->comp_lo, n * 4, cudaMemcpyDeviceToHost, s);
    if (out->filled) cudaMemcpyAsync(out->filled, ctx->ws.filled + r->comp_lo, n * sizeof(rl_features), cudaMemcpyDeviceToHost, s);
    d2h += n * (int64_t)((out->comps ? 48 : 0) + (out->top ? 4 : 0) + (out->filled ? 40 : 0));
    out->d2h_bytes = d2h;
    out->h2d_bytes = 0;
    return sync_err(ctx, "strip fetch");
}

}  // extern "C"
