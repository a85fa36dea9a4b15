// strips.cu -- one image cut into horizontal strips across ranks.
//
// Every rank runs the tile passes on its own strip with the geometry of the WHOLE image (tile
// rows [ty0, ty1), pixel row y at row y - prow0 of the rank's buffer), so the image frame is
// exterior only where it really is: cut rows are open.  The exchange is between three phases:
//
//   local   analyze + seams inside the strip; every border component (node) gets the node of the
//           pixel left of its first pixel (resolved now: that pixel is in the same row).
//   merge   every rank imports all strips' node tables (shifted to one global numbering), the
//           cut rows' perimeter labels and the per-row interior counts, unions across the cuts
//           and runs the merge passes over all nodes (identical on every rank), then emits its
//           own tiles.  Interior components fold their features into post-fill roots that may
//           be owned by other strips, so border survivors collect per-rank partial sums.
//   finish  the all-reduced partials plus the border part give the post-fill features.
//
// The collectives themselves (all-gather of the local infos and of the export records,
// all-reduce of the partials) are the caller's: paper_2006_09299_b200/strips.py does them with
// torch.distributed (NCCL over NVLink on GPUs).
//
// Canonical ids stay the raster order of first pixels over the whole image, so the strips'
// outputs concatenate to exactly the single-image result (labeling.hpp:190-217 numbering via
// tables.hpp:68-76).
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "runlab_gpu.h"

using namespace rlg;
using namespace rlh;

namespace {

// exchange record of one border component
struct NodeX {
    uint32_t uf, nleft;  // local node ids (0 = exterior)
    uint64_t key;
    Acc acc;
    NodeRec rec;
};
static_assert(sizeof(NodeX) == 72, "NodeX layout");

struct XHeader {
    int64_t n_nodes;
    int32_t ty0, ty1;
    int64_t pad[6];
};
static_assert(sizeof(XHeader) == 64, "XHeader layout");

struct XLayout {
    size_t nodes, tiles, cnt, perim, bytes;
};

size_t align8(size_t v) { return (v + 7) & ~size_t(7); }

XLayout x_layout(int32_t W, int64_t max_nodes, int32_t max_tile_rows) {
    const int32_t ntx = (W + TW - 1) / TW;
    XLayout L;
    L.nodes = sizeof(XHeader);
    L.tiles = L.nodes + align8((size_t)max_nodes * sizeof(NodeX));
    L.cnt = L.tiles + align8((size_t)max_tile_rows * ntx * 8);
    L.perim = L.cnt + align8((size_t)max_tile_rows * TH * ntx * 4);
    L.bytes = L.perim + align8((size_t)ntx * 2 * TW * 2);
    return L;
}

// node of the pixel left of each border component's first pixel (local numbering)
__global__ void k_strip_left(Geo g, Ws ws) {
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

__global__ void k_strip_pack(Geo g, Ws ws, uint8_t* buf, XLayout L) {
    const uint32_t n_used = min(ws.counters[0], ws.cap_nodes);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (tid == 0) {
        XHeader h{};
        h.n_nodes = n_used;
        h.ty0 = g.ty0;
        h.ty1 = g.ty1;
        *reinterpret_cast<XHeader*>(buf) = h;
    }
    NodeX* xn = reinterpret_cast<NodeX*>(buf + L.nodes);
    for (int64_t i = tid; i < n_used; i += stride) {
        const uint32_t n = 1u + (uint32_t)i;
        NodeX x;
        x.uf = ws.uf[n];
        x.nleft = ws.nleft[n];
        x.key = ws.nkey[n];
        x.acc = ws.nacc[n];
        x.rec = ws.nrec[n];
        xn[i] = x;
    }
    const int64_t t0 = (int64_t)g.ty0 * g.ntx, nt = (int64_t)(g.ty1 - g.ty0) * g.ntx;
    uint32_t* xt = reinterpret_cast<uint32_t*>(buf + L.tiles);
    for (int64_t i = tid; i < nt; i += stride) {
        xt[2 * i] = ws.tbase[t0 + i];
        xt[2 * i + 1] = ws.tnb[t0 + i];
    }
    const int64_t r0 = (int64_t)g.ty0 * TH, r1 = min((int64_t)g.ty1 * TH, (int64_t)g.H);
    uint32_t* xc = reinterpret_cast<uint32_t*>(buf + L.cnt);
    for (int64_t i = tid; i < (r1 - r0) * g.ntx; i += stride) xc[i] = ws.cnt[r0 * g.ntx + i];
    // cut rows: top perimeter row of the first tile row, bottom row of the last one
    uint16_t* xp = reinterpret_cast<uint16_t*>(buf + L.perim);
    for (int64_t i = tid; i < (int64_t)g.ntx * 2 * TW; i += stride) {
        const int64_t tx = i / (2 * TW), k = i % (2 * TW);
        const int64_t t = (k < TW ? t0 : t0 + nt - g.ntx) + tx;
        xp[i] = ws.perim[t * PERIM + k];  // k < TW: top row; TW <= k < 2TW: bottom row
    }
}

// one source strip's record into the global tables
__global__ void k_strip_unpack(Geo g, Ws ws, const uint8_t* buf, XLayout L, uint32_t off) {
    const XHeader h = *reinterpret_cast<const XHeader*>(buf);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const NodeX* xn = reinterpret_cast<const NodeX*>(buf + L.nodes);
    auto shift = [&](uint32_t v) { return v ? v + off : 0u; };
    for (int64_t i = tid; i < h.n_nodes; i += stride) {
        const NodeX x = xn[i];
        const uint32_t n = 1u + off + (uint32_t)i;
        ws.uf[n] = shift(x.uf);
        ws.nleft[n] = shift(x.nleft);
        ws.nkey[n] = x.key;
        ws.nmin[n] = x.key;
        ws.nacc[n] = x.acc;
        ws.nrec[n] = x.rec;
    }
    const int64_t t0 = (int64_t)h.ty0 * g.ntx, nt = (int64_t)(h.ty1 - h.ty0) * g.ntx;
    const uint32_t* xt = reinterpret_cast<const uint32_t*>(buf + L.tiles);
    for (int64_t i = tid; i < nt; i += stride) {
        ws.tbase[t0 + i] = xt[2 * i] + off;
        ws.tnb[t0 + i] = xt[2 * i + 1];
    }
    const int64_t r0 = (int64_t)h.ty0 * TH, r1 = min((int64_t)h.ty1 * TH, (int64_t)g.H);
    const uint32_t* xc = reinterpret_cast<const uint32_t*>(buf + L.cnt);
    for (int64_t i = tid; i < (r1 - r0) * g.ntx; i += stride) ws.cnt[r0 * g.ntx + i] = xc[i];
    const uint16_t* xp = reinterpret_cast<const uint16_t*>(buf + L.perim);
    for (int64_t i = tid; i < (int64_t)g.ntx * 2 * TW; i += stride) {
        const int64_t tx = i / (2 * TW), k = i % (2 * TW);
        const int64_t t = (k < TW ? t0 : t0 + nt - g.ntx) + tx;
        ws.perim[t * PERIM + k] = xp[i];
    }
}

__global__ void k_strip_exterior(Ws ws, uint32_t n_total) {
    ws.uf[0] = 0;
    ws.nacc[0] = acc_empty();
    ws.nmin[0] = ~0ull;
    ws.nrootcid[0] = 0;
    ws.nparent[0] = 0;
    ws.nanccid[0] = 0;
    ws.nrep[0] = 0;
    ws.counters[0] = n_total;
    ws.counters[1] = 0;
}

// border survivors (post-fill roots that are border components), flagged at their root node
__global__ void k_strip_surv_flags(Geo g, Ws ws, uint32_t* flag) {
    const uint32_t n_total = ws.counters[0];
    for (uint32_t n = 1u + blockIdx.x * blockDim.x + threadIdx.x; n < 1u + n_total; n += gridDim.x * blockDim.x) {
        if (!ws.nrep[n]) continue;
        const uint32_t root = ws.uf[n];
        if (ws.nanccid[root] == ws.nrootcid[root]) flag[root] = 1u;
    }
}

// this rank's partial post-fill sums of the border survivors, in root-node order
__global__ void k_strip_partials(Geo g, Ws ws, const uint32_t* flag, const uint32_t* sidx, int64_t* psum,
                                 int32_t* pmin, int32_t* pmax) {
    const uint32_t n_total = ws.counters[0];
    for (uint32_t n = 1u + blockIdx.x * blockDim.x + threadIdx.x; n < 1u + n_total; n += gridDim.x * blockDim.x) {
        if (!flag[n]) continue;
        const uint32_t k = sidx[n];
        const Acc f = ws.filled[ws.nrootcid[n]];
        psum[3 * k] = f.s;
        psum[3 * k + 1] = f.sx;
        psum[3 * k + 2] = f.sy;
        pmin[2 * k] = f.row_min;
        pmin[2 * k + 1] = f.col_min;
        pmax[2 * k] = f.row_max;
        pmax[2 * k + 1] = f.col_max;
    }
}

// reduced partials + the border component's own features
__global__ void k_strip_apply(Geo g, Ws ws, const uint32_t* flag, const uint32_t* sidx, const int64_t* psum,
                              const int32_t* pmin, const int32_t* pmax) {
    const uint32_t n_total = ws.counters[0];
    for (uint32_t n = 1u + blockIdx.x * blockDim.x + threadIdx.x; n < 1u + n_total; n += gridDim.x * blockDim.x) {
        if (!flag[n]) continue;
        const uint32_t k = sidx[n];
        const Acc a = ws.nacc[n];
        Acc f;
        f.s = psum[3 * k] + a.s;
        f.sx = psum[3 * k + 1] + a.sx;
        f.sy = psum[3 * k + 2] + a.sy;
        f.row_min = min(pmin[2 * k], a.row_min);
        f.col_min = min(pmin[2 * k + 1], a.col_min);
        f.row_max = max(pmax[2 * k], a.row_max);
        f.col_max = max(pmax[2 * k + 1], a.col_max);
        ws.filled[ws.nrootcid[n]] = f;
    }
}

__global__ void k_strip_summary(Geo g, Ws ws, int64_t* out, int32_t r0, int32_t r1, int32_t first) {
    // [0] total components, [1] fg, [2] survivors, [3] owned lo, [4] owned hi, [5] error bits
    const int64_t rows = (int64_t)g.H * g.ntx;
    out[0] = (int64_t)ws.off[rows] + 1;
    out[1] = ws.img_fg[0];
    out[2] = ws.img_surv[0];
    out[3] = first ? 0 : 1 + (int64_t)ws.off[(int64_t)r0 * g.ntx];
    out[4] = 1 + (int64_t)ws.off[(int64_t)r1 * g.ntx];
    out[5] = ws.counters[1];
}

__global__ void k_copy_count(const uint32_t* src, int64_t* dst) { *dst = (int64_t)*src; }

int grid(int64_t n, int sms) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8)); }

}  // namespace

namespace rlh {

struct StripState {
    Geo g{};
    rl_config cfg{};
    int32_t y0 = 0, h = 0;
    int64_t n_local = 0, interior_fg = 0;
    const uint8_t* pix = nullptr;
    // global phase
    int64_t n_total = 0, k_surv = 0;
    int64_t summary[6] = {};
    bool merged = false;
};

}  // namespace rlh

namespace {

StripState* strip_state(rl_ctx* c) {
    if (!c->strip) c->strip = new StripState();
    return c->strip;
}

int sync_err(rl_ctx* c, const char* what) {
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    return e == cudaSuccess ? RL_OK : cuda_fail(c, e, what);
}

}  // namespace

namespace rlh {
void strip_free(rl_ctx* c) {
    delete c->strip;
    c->strip = nullptr;
}
}  // namespace rlh

extern "C" {

int64_t rl_strip_export_bytes(int32_t w, int64_t max_nodes, int32_t max_tile_rows) {
    return (int64_t)x_layout(w, max_nodes, max_tile_rows).bytes;
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
    S->g = g;
    S->cfg = *cfg;
    S->y0 = y0;
    S->h = h;
    S->pix = d_strip;
    S->merged = false;
    ctx->want_compact = false;
    cudaStream_t s = ctx->stream;
    for (int attempt = 0; attempt < 4; ++attempt) {
        Ws ws;
        size_t tmp = 0;
        if ((rc = prepare_ws(ctx, g, cfg, ws, tmp, (int64_t)h * w))) return rc;
        if (!ensure(ctx->nleft, ((size_t)ctx->cap_nodes + 1) * 4)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
        ws.nleft = P<uint32_t>(ctx->nleft);
        const int64_t ncnt = (int64_t)H * g.ntx + 1;
        cudaMemsetAsync(ws.counters, 0, 64, s);
        cudaMemsetAsync(ws.rused, 0, 8, s);
        cudaMemsetAsync(ws.img_fg, 0, 4, s);
        cudaMemsetAsync(ws.uf, 0, 4, s);  // the exterior node (strip 0's first tile also sets it)
        cudaMemsetAsync(ws.cnt + (ncnt - 1), 0, 4, s);
        launch_analyze(d_strip, g, ws, s);
        launch_seams(g, ws, s, ctx->sms);
        k_strip_left<<<grid((int64_t)ctx->cap_nodes, ctx->sms), 256, 0, s>>>(g, ws);
        ctx->launches = 3 + (g.ty1 - g.ty0 > 1) + (g.ntx > 1) + 1;
        uint32_t hc[8] = {};
        cudaMemcpyAsync(hc, ws.counters, 32, cudaMemcpyDeviceToHost, s);
        uint32_t fg = 0;
        cudaMemcpyAsync(&fg, ws.img_fg, 4, cudaMemcpyDeviceToHost, s);
        unsigned long long rused = 0;
        cudaMemcpyAsync(&rused, ws.rused, 8, cudaMemcpyDeviceToHost, s);
        if ((rc = sync_err(ctx, "strip local"))) return rc;
        ctx->ws = ws;
        ctx->geo = g;
        if (hc[1] & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (strip left link)");
        if (hc[1] & (ERR_NODE_CAP | ERR_RSTORE_CAP)) {
            if (hc[1] & ERR_NODE_CAP) ctx->cap_nodes = (uint32_t)std::min<uint64_t>(hc[0] + hc[0] / 4 + 1024, 0xF0000000ull);
            if (hc[1] & ERR_RSTORE_CAP) ctx->cap_rstore = rused + rused / 8 + 4096;
            continue;
        }
        S->n_local = hc[0];
        S->interior_fg = fg;
        out->n_nodes = hc[0];
        out->interior_fg = fg;
        out->ty0 = g.ty0;
        out->ty1 = g.ty1;
        out->status = 0;
        out->pad = 0;
        return RL_OK;
    }
    return set_err(ctx, RL_EINTERNAL, "capacity did not converge");
}

int rl_strip_export(rl_ctx* ctx, int64_t max_nodes, int32_t max_tile_rows, void* d_buf) {
    if (!ctx || !d_buf) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || !S->g.strip) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_local first");
    if (S->n_local > max_nodes || S->g.ty1 - S->g.ty0 > max_tile_rows)
        return set_err(ctx, RL_EINVAL, "strips: export record too small");
    cudaSetDevice(ctx->device);
    const XLayout L = x_layout(S->g.W, max_nodes, max_tile_rows);
    k_strip_pack<<<grid(std::max<int64_t>(max_nodes, (int64_t)S->g.ntx * 2 * TW), ctx->sms), 256, 0, ctx->stream>>>(
        S->g, ctx->ws, static_cast<uint8_t*>(d_buf), L);
    ctx->launches += 1;
    return sync_err(ctx, "strip export");
}

int rl_strip_merge(rl_ctx* ctx, const void* d_gathered, int32_t n_strips, const rl_strip_local_info* infos,
                   int64_t max_nodes, int32_t max_tile_rows, rl_strip_partials* out) {
    if (!ctx || !d_gathered || !infos || !out || n_strips < 1) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || !S->g.strip) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_local first");
    cudaSetDevice(ctx->device);
    const XLayout L = x_layout(S->g.W, max_nodes, max_tile_rows);
    int64_t n_total = 0, fg_int = 0;
    std::vector<uint32_t> offs(n_strips);
    for (int q = 0; q < n_strips; ++q) {
        offs[q] = (uint32_t)n_total;
        n_total += infos[q].n_nodes;
        fg_int += infos[q].interior_fg;
        if (infos[q].n_nodes > max_nodes) return set_err(ctx, RL_EINVAL, "strips: inconsistent node counts");
    }
    if (n_total + 1 >= 0xF0000000ll) return set_err(ctx, RL_EINVAL, "strips: too many border components");
    Geo g = S->g;
    const rl_config* cfg = &S->cfg;
    cudaStream_t s = ctx->stream;
    if (ctx->cap_nodes < (uint64_t)n_total + 1) ctx->cap_nodes = (uint32_t)(n_total + n_total / 8 + 1024);
    for (int attempt = 0; attempt < 4; ++attempt) {
        Ws ws;
        size_t tmp = 0;
        int rc = prepare_ws(ctx, g, cfg, ws, tmp, (int64_t)S->h * g.W);
        if (rc) return rc;
        const size_t nn = (size_t)ctx->cap_nodes + 1;
        if (!ensure(ctx->nleft, nn * 4) || !ensure(ctx->flag, nn * 4) || !ensure(ctx->rank, nn * 4))
            return set_err(ctx, RL_ENOMEM, "device allocation failed");
        size_t tmp3 = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tmp3, (uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n_total + 1));
        if (!ensure(ctx->cub_tmp, std::max(tmp, tmp3))) return set_err(ctx, RL_ENOMEM, "device allocation failed");
        ws.nleft = P<uint32_t>(ctx->nleft);
        const int64_t ncnt = (int64_t)g.H * g.ntx + 1;
        // ---- import every strip's record into one global numbering
        const uint8_t* gb = static_cast<const uint8_t*>(d_gathered);
        for (int q = 0; q < n_strips; ++q)
            k_strip_unpack<<<grid(std::max<int64_t>(max_nodes, (int64_t)g.ntx * 2 * TW), ctx->sms), 256, 0, s>>>(
                g, ws, gb + (size_t)q * L.bytes, L, offs[q]);
        k_strip_exterior<<<1, 1, 0, s>>>(ws, (uint32_t)n_total);
        const uint32_t fg32 = (uint32_t)fg_int;
        cudaMemcpyAsync(ws.img_fg, &fg32, 4, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(ws.img_surv, 0, 4, s);
        cudaMemsetAsync(ws.cnt + (ncnt - 1), 0, 4, s);
        // ---- union across the cuts, then the merge passes over all border components
        for (int q = 0; q + 1 < n_strips; ++q) launch_seam_rows(g, ws, infos[q].ty1 - 1, 1, s, ctx->sms);
        Geo gm = g;  // merge kernels: whole image
        gm.ty0 = 0;
        gm.ty1 = g.nty;
        launch_resolve(gm, ws, s, ctx->sms, n_total);
        launch_reps(gm, ws, s, ctx->sms, n_total);
        cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, tmp, ws.cnt, ws.off, (int)ncnt, s);
        launch_cids(gm, ws, s, ctx->sms);
        launch_tree_parts(gm, ws, s, ctx->sms, n_total);  // post-fill roots (no fold yet)
        // ---- emit this strip's tiles; interior survivors are counted into a private counter
        Ws we = ws;
        if (!ensure(ctx->scount, 64)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
        we.img_surv = P<uint32_t>(ctx->scount);
        cudaMemsetAsync(we.img_surv, 0, 4, s);
        launch_emit(g, we, s);
        // ---- border survivors: flags, index, this rank's partial sums
        uint32_t* flag = P<uint32_t>(ctx->flag);
        cudaMemsetAsync(flag, 0, (size_t)(n_total + 1) * 4, s);
        k_strip_surv_flags<<<grid(n_total, ctx->sms), 256, 0, s>>>(gm, ws, flag);
        size_t t3 = ctx->cub_tmp.bytes;
        cub::DeviceScan::ExclusiveSum(ctx->cub_tmp.p, t3, flag, P<uint32_t>(ctx->rank), (int)(n_total + 1), s);
        int64_t hs[6] = {};
        uint32_t klast[2] = {};
        cudaMemcpyAsync(&klast[0], P<uint32_t>(ctx->rank) + n_total, 4, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&klast[1], flag + n_total, 4, cudaMemcpyDeviceToHost, s);
        if (!ensure(ctx->summ, 64)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
        const int32_t r1 = std::min(g.ty1 * TH, g.H);
        k_strip_summary<<<1, 1, 0, s>>>(g, ws, P<int64_t>(ctx->summ), g.ty0 * TH, r1, g.ty0 == 0 ? 1 : 0);
        cudaMemcpyAsync(hs, ctx->summ.p, 48, cudaMemcpyDeviceToHost, s);
        if ((rc = sync_err(ctx, "strip merge"))) return rc;
        if (hs[5] & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (tree reference)");
        if ((uint64_t)hs[0] > ctx->cap_comps) {  // identical on every rank: all grow and re-run
            ctx->cap_comps = (uint64_t)hs[0] + (uint64_t)hs[0] / 8 + 1024;
            continue;
        }
        const int64_t K = (int64_t)klast[0] + klast[1];
        S->k_surv = K;
        S->n_total = n_total;
        std::memcpy(S->summary, hs, sizeof(hs));
        if (!ensure(ctx->fcomp, (size_t)std::max<int64_t>(K, 1) * 40 + 8)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
        int64_t* psum = P<int64_t>(ctx->fcomp);
        int32_t* pmin = reinterpret_cast<int32_t*>(psum + 3 * K);
        int32_t* pmax = pmin + 2 * K;
        int64_t* pcnt = reinterpret_cast<int64_t*>(P<uint8_t>(ctx->fcomp) + (size_t)K * 40);
        k_strip_partials<<<grid(n_total, ctx->sms), 256, 0, s>>>(gm, ws, flag, P<uint32_t>(ctx->rank), psum, pmin, pmax);
        // interior survivors of this strip as an int64 for the reduction
        k_copy_count<<<1, 1, 0, s>>>(we.img_surv, pcnt);
        if ((rc = sync_err(ctx, "strip partials"))) return rc;
        ctx->ws = ws;
        ctx->geo = g;
        out->k = K;
        out->d_sum = psum;
        out->d_min = pmin;
        out->d_max = pmax;
        out->d_count = pcnt;
        S->merged = true;
        // unpack x n, exterior, cut seams, resolve, reps, scan x 2, cids, parents, tops, emit x 3,
        // flags, scan x 2, summary, partials, count
        ctx->launches += n_strips + 1 + (n_strips - 1) + 15;
        return RL_OK;
    }
    return set_err(ctx, RL_EINTERNAL, "capacity did not converge");
}

int rl_strip_finish(rl_ctx* ctx, rl_strip_result* out) {
    if (!ctx || !out) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || !S->merged) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_merge first");
    cudaSetDevice(ctx->device);
    cudaStream_t s = ctx->stream;
    Ws ws = ctx->ws;
    Geo gm = S->g;
    gm.ty0 = 0;
    gm.ty1 = gm.nty;
    const int64_t K = S->k_surv;
    int64_t* psum = P<int64_t>(ctx->fcomp);
    int32_t* pmin = reinterpret_cast<int32_t*>(psum + 3 * K);
    int32_t* pmax = pmin + 2 * K;
    int64_t* pcnt = reinterpret_cast<int64_t*>(P<uint8_t>(ctx->fcomp) + (size_t)K * 40);
    k_strip_apply<<<grid(S->n_total, ctx->sms), 256, 0, s>>>(gm, ws, P<uint32_t>(ctx->flag), P<uint32_t>(ctx->rank),
                                                             psum, pmin, pmax);
    launch_fold(gm, ws, s, ctx->sms, S->n_total);
    ctx->launches += 2;
    int64_t surv_int = 0;
    cudaMemcpyAsync(&surv_int, pcnt, 8, cudaMemcpyDeviceToHost, s);
    const int rc = sync_err(ctx, "strip finish");
    if (rc) return rc;
    const int64_t* hs = S->summary;
    out->n_components = hs[0];
    out->n_fg = hs[1];
    out->n_holes = hs[0] - 1 - hs[1];
    out->euler = hs[1] - out->n_holes;
    out->n_survivors = hs[2] + surv_int;
    out->comp_lo = hs[3];
    out->comp_hi = hs[4];
    out->y0 = S->y0;
    out->h = S->h;
    return RL_OK;
}

int rl_strip_fetch(rl_ctx* ctx, const rl_strip_result* r, rl_host_outputs* out) {
    if (!ctx || !r || !out) return RL_EINVAL;
    StripState* S = ctx->strip;
    if (!S || !S->merged) return set_err(ctx, RL_ELOGIC, "strips: rl_strip_finish first");
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
