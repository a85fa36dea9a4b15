// api.cu -- host orchestration and the extern "C" ABI (include/runlab_gpu.h).
//
// One rl_ctx = one device, one stream, a grow-only device workspace and events.  A call
// enqueues the whole pipeline (kernels.cu) on the context stream with no host sync in the
// middle; capacity estimates for border nodes and components are checked on device and,
// if exceeded, the call is re-run once after growing (the counters say by how much).
//
// Reference boundary: runlab::label_image / timed_label_image (labeling.hpp:336-348) and
// binarize_labels (labeling.hpp:354-360); error mapping per labeling.hpp:271-273.
#include <cuda_runtime.h>


#include <algorithm>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "pack.cuh"
#include "runlab_gpu.h"

using namespace rlg;
using namespace rlh;

namespace {

// per-image summary gathered on device after a run: [0] comp base (canonical offset),
// [1] C_pre, [2] n_fg, [3] C_post
__global__ void k_summary(Geo g, Ws ws, uint64_t* cbase, int64_t* summ) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > g.B) return;
    const int64_t idx = (int64_t)b * g.H * g.ntx;
    const uint64_t base = (uint64_t)ws.off[idx] + (uint64_t)b;
    cbase[b] = base;
    if (b < g.B) {
        const uint64_t next = (uint64_t)ws.off[idx + (int64_t)g.H * g.ntx] + (uint64_t)b + 1u;
        summ[4 * b + 0] = (int64_t)base;
        summ[4 * b + 1] = (int64_t)(next - base);
        summ[4 * b + 2] = (int64_t)ws.img_fg[b];
        summ[4 * b + 3] = (int64_t)ws.img_surv[b];
    } else {
        summ[4 * b + 0] = (int64_t)base;  // total components
        summ[4 * b + 1] = (int64_t)ws.counters[0];
        summ[4 * b + 2] = (int64_t)ws.counters[1];
        summ[4 * b + 3] = (int64_t)*ws.rused;
    }
}

// the per-call counters, per-image counts, the summary's tail row and the look-back state of
// the offset scan, zeroed by one launch instead of a memset each
__global__ void k_init(Ws ws, int32_t B, uint32_t* cnt_end, int64_t* summ_tail, unsigned long long* scan_state,
                       int64_t scan_words) {
    const int64_t n = max((int64_t)max(B, 16), scan_words);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < 16) ws.counters[i] = 0;
        if (i == 0) {
            *ws.rused = 0;
            *cnt_end = 0;
        }
        if (i < 4) summ_tail[i] = 0;
        if (i < B) ws.img_fg[i] = ws.img_surv[i] = 0;
        if (i < scan_words) scan_state[i] = 0;
    }
}

}  // namespace


namespace rlh {

int set_err(rl_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    return code;
}

int cuda_fail(rl_ctx* c, cudaError_t e, const char* what) {
    return set_err(c, RL_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool ensure(DevBuf& b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.bytes >= bytes) return true;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    const size_t want = bytes + bytes / 8;  // some headroom against regrowth
    if (cudaMalloc(&b.p, want) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    b.bytes = want;
    // debugging aid: fill new workspace with a pattern so reads of unwritten entries show up
    // (fresh device pages are zero, which hides them; env RUNLAB_GPU_POISON=1)
    if (std::getenv("RUNLAB_GPU_POISON")) {
        cudaMemset(b.p, 0xA5, want);  // may be asynchronous: done before any stream uses it
        cudaDeviceSynchronize();
    }
    return true;
}

int check_args(rl_ctx* ctx, int32_t w, int32_t h, int32_t n, const rl_config* cfg) {
    if (!ctx) return RL_EINVAL;
    if (!cfg) return set_err(ctx, RL_EINVAL, "null config");
    if (w < 1 || h < 1 || n < 1) return set_err(ctx, RL_EINVAL, "image must be at least 1x1 and n_images >= 1");
    if (cfg->densify_labels && !cfg->relabel)
        return set_err(ctx, RL_EINVAL, "label_image: densify_labels requires relabel");
    if (cfg->connectivity != RL_FG8_BG4 && cfg->connectivity != RL_FG4_BG8)
        return set_err(ctx, RL_EINVAL, "unknown connectivity");
    // int64 feature sums: Sx <= P * W must stay below 2^63 (features.hpp:37-39)
    const double P = (double)w * (double)h;
    if (P * (double)std::max(w, h) >= 9.2e18) return set_err(ctx, RL_EOVERFLOW, "feature accumulator overflow");
    if (P * n >= 4.0e9 * 64) return set_err(ctx, RL_EINVAL, "batch too large");
    if ((double)n * h * ((w + TW - 1) / TW) >= 4.0e9) return set_err(ctx, RL_EINVAL, "batch too large");
    return RL_OK;
}

void set_output_format(Geo& g, int32_t ofmt) {  // the filled-image buffer is cudaMalloc'ed: aligned
    g.ofmt = ofmt;
    g.orowb = ofmt == RL_PIXELS_P4 ? (g.W + 7) / 8 : g.W;
    g.ofbytes = (int64_t)g.orowb * g.H;
    g.ovec_ok = ofmt == RL_PIXELS_P4 ? (g.orowb % 4) == 0 : (g.W % 16) == 0;
}

Geo make_geo(int32_t W, int32_t H, int32_t B, const rl_config* cfg, const void* dpix, int32_t fmt) {
    Geo g{};
    g.W = W;
    g.H = H;
    g.B = B;
    g.ntx = (W + TW - 1) / TW;
    g.nty = (H + TH - 1) / TH;
    g.tpi = g.ntx * g.nty;
    const int64_t ntiles = (int64_t)g.tpi * B;
    g.ntiles = ntiles >= (1ll << 31) ? -1 : (int32_t)ntiles;
    g.flip = cfg->connectivity == RL_FG4_BG8 ? 1 : 0;
    g.P = (int64_t)W * H;
    g.fmt = fmt;
    g.rowb = fmt == RL_PIXELS_P4 ? (W + 7) / 8 : W;
    g.fbytes = (int64_t)g.rowb * H;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dpix);
    g.vec_ok = fmt == RL_PIXELS_P4 ? ((g.rowb % 4) == 0 && (a % 4) == 0) : ((W % 16) == 0 && (a % 16) == 0);
    set_output_format(g, fmt);
    g.label_mode = cfg->relabel ? (cfg->fill_holes ? 2 : 1) : 0;
    g.ty0 = 0;
    g.ty1 = g.nty;
    g.prow0 = 0;
    g.cell_end = (int64_t)B * H * g.ntx;
    g.cid_lo = g.cid_hi = g.cid_extra = 0;
    return g;
}

int prepare_ws(rl_ctx* ctx, const Geo& g, const rl_config* cfg, Ws& ws, size_t& tmp, int64_t out_px) {
    const int32_t B = g.B;
    // tables for the tiles and cells of this call: the whole batch, or the strip's tile rows
    const int64_t ntiles = (int64_t)(g.ty1 - g.ty0) * g.ntx * B;
    const int64_t ncnt = g.strip ? (std::min<int64_t>((int64_t)g.ty1 * TH, g.H) - (int64_t)g.ty0 * TH) * g.ntx + 1
                                 : (int64_t)B * g.H * g.ntx + 1;
    const int64_t npx = (int64_t)(g.ty1 - g.ty0) * TH * g.W * B;  // pixels covered (rounded up)
    if (ctx->cap_nodes == 0) ctx->cap_nodes = (uint32_t)std::min<int64_t>(std::max<int64_t>(ntiles * 96, 4096), 0xF0000000ll);
    // initial estimate 0.02 components/pixel (random images: 0.003-0.13); grows on demand
    if (ctx->cap_comps == 0) ctx->cap_comps = (uint64_t)std::max<int64_t>(npx / 48, 4096);
    // tile maps: ~2 runs' worth of u16 per run plus 4 per component and the word bases
    if (ctx->cap_rstore == 0) ctx->cap_rstore = (uint64_t)std::max<int64_t>(npx * 6 / 10 + ntiles * 320, 1 << 16);
    const uint64_t nn = (uint64_t)B + ctx->cap_nodes;
    bool ok = ensure(ctx->bits, (size_t)ntiles * NW * 4) && ensure(ctx->tbase, (size_t)ntiles * 4) &&
              ensure(ctx->tnb, (size_t)ntiles * 4) && ensure(ctx->ovf, (size_t)ntiles * 4) &&
              ensure(ctx->ovf2, (size_t)ntiles * 4) && ensure(ctx->thdr, (size_t)ntiles * THDR * 2) &&
              ensure(ctx->tmap, (size_t)ntiles * 8) && ensure(ctx->rstore, ctx->cap_rstore * 2) &&
              ensure(ctx->rused, 64) && ensure(ctx->perim, (size_t)ntiles * PERIM * 2) &&
              ensure(ctx->uf, nn * 4) && ensure(ctx->nkey, nn * 8) && ensure(ctx->nmin, nn * 8) &&
              ensure(ctx->nacc, nn * sizeof(Acc)) && ensure(ctx->nrec, nn * sizeof(NodeRec)) &&
              ensure(ctx->nrep, nn) && ensure(ctx->ninfo, nn * 8) && ensure(ctx->nrootcid, nn * 4) && ensure(ctx->nparent, nn * 4) &&
              ensure(ctx->nanccid, nn * 4) && ensure(ctx->cnt, (size_t)ncnt * 4) &&
              ensure(ctx->off, (size_t)ncnt * 4) && ensure(ctx->counters, 64) &&
              ensure(ctx->img_fg, (size_t)B * 4) && ensure(ctx->img_surv, (size_t)B * 4) &&
              ensure(ctx->comps, ctx->cap_comps * sizeof(rl_component)) &&
              ensure(ctx->top, ctx->cap_comps * 4) && ensure(ctx->filled, ctx->cap_comps * sizeof(Acc)) &&
              (ctx->ext_filled || ensure(ctx->filled_img, (size_t)(out_px / g.W) * g.orowb)) &&
              ensure(ctx->cbase, (size_t)(B + 1) * 8) &&
              ensure(ctx->summ, (size_t)(B + 2) * 32) && ensure(ctx->ftab, (size_t)FT_SHARDS * FT_HS * 28);
    if (ok && g.label_mode) ok = ensure(ctx->labels, (size_t)out_px * 4);
    if (!ok) return set_err(ctx, RL_ENOMEM, "device allocation failed");
    tmp = scan_state_bytes(ncnt);  // scan.cu
    size_t tmp2 = 0;
    if ((cfg->densify_labels && cfg->fill_holes) || ctx->want_compact)
        tmp2 = scan_state_bytes((int64_t)std::min<uint64_t>(ctx->cap_comps + 1, 0x7FFFFFFF));
    if (!ensure(ctx->cub_tmp, std::max(tmp, tmp2))) return set_err(ctx, RL_ENOMEM, "device allocation failed");

    ws = Ws{};
    ws.bits = P<uint32_t>(ctx->bits);
    ws.tbase = P<uint32_t>(ctx->tbase);
    ws.tnb = P<uint32_t>(ctx->tnb);
    ws.ovf = P<uint32_t>(ctx->ovf);
    ws.ovf2 = P<uint32_t>(ctx->ovf2);
    ws.thdr = P<uint16_t>(ctx->thdr);
    ws.tmap = P<uint64_t>(ctx->tmap);
    ws.rstore = P<uint16_t>(ctx->rstore);
    ws.rused = P<unsigned long long>(ctx->rused);
    ws.cap_rstore = ctx->cap_rstore;
    ws.perim = P<uint16_t>(ctx->perim);
    ws.uf = P<uint32_t>(ctx->uf);
    ws.nkey = P<uint64_t>(ctx->nkey);
    ws.nmin = P<uint64_t>(ctx->nmin);
    ws.nacc = P<Acc>(ctx->nacc);
    ws.nrec = P<NodeRec>(ctx->nrec);
    ws.nrep = P<uint8_t>(ctx->nrep);
    ws.ninfo = P<uint2>(ctx->ninfo);
    ws.nrootcid = P<uint32_t>(ctx->nrootcid);
    ws.nparent = P<uint32_t>(ctx->nparent);
    ws.nanccid = P<uint32_t>(ctx->nanccid);
    ws.cnt = P<uint32_t>(ctx->cnt);
    ws.off = P<uint32_t>(ctx->off);
    ws.counters = P<uint32_t>(ctx->counters);
    ws.img_fg = P<uint32_t>(ctx->img_fg);
    ws.img_surv = P<uint32_t>(ctx->img_surv);
    ws.cap_nodes = ctx->cap_nodes;
    ws.cap_comps = ctx->cap_comps;
    ws.comps = P<rl_component>(ctx->comps);
    ws.top = P<uint32_t>(ctx->top);
    ws.filled = P<Acc>(ctx->filled);
    ws.filled_img = ctx->ext_filled ? ctx->ext_filled : P<uint8_t>(ctx->filled_img);
    ws.labels = g.label_mode ? P<uint32_t>(ctx->labels) : nullptr;
    ws.ftsum = P<unsigned long long>(ctx->ftab);
    ws.ftkey = reinterpret_cast<uint32_t*>(ws.ftsum + 3ull * FT_SHARDS * FT_HS);
    if (g.strip) {
        // the strip's tables start at its first tile / first cell / first owned id (kernels use
        // whole-image numbers; only the strip's range is ever accessed through these bases)
        const int64_t t0 = (int64_t)g.ty0 * g.ntx, c0 = (int64_t)g.ty0 * TH * g.ntx;
        ws.bits = shift_base(ws.bits, t0 * NW);
        ws.tbase = shift_base(ws.tbase, t0);
        ws.tnb = shift_base(ws.tnb, t0);
        ws.perim = shift_base(ws.perim, t0 * PERIM);
        ws.thdr = shift_base(ws.thdr, t0 * THDR);
        ws.tmap = shift_base(ws.tmap, t0);
        ws.cnt = shift_base(ws.cnt, c0);
        ws.off = shift_base(ws.off, c0);
        ws.comps = shift_base(ws.comps, g.cid_lo);
        ws.top = shift_base(ws.top, g.cid_lo);
        ws.filled = shift_base(ws.filled, g.cid_lo);
    }

    return RL_OK;
}

}  // namespace rlh

namespace rlh {

// Horizontal and vertical seams of tile rows [ty0, ty1) concurrently (both only unite border
// nodes, lock-free): the vertical ones on a stream forked from and joined back into `s`.
// Returns the number of launches.
int enqueue_seams(rl_ctx* ctx, const Geo& g, const Ws& ws, cudaStream_t s) {
    const int32_t rows = g.ty1 - g.ty0;
    const bool fork = ctx->seam_stream && g.ntx > 1 && !ctx->ktimes;
    if (fork) {
        cudaEventRecord(ctx->seam_fork, s);
        cudaStreamWaitEvent(ctx->seam_stream, ctx->seam_fork, 0);
        launch_seam_cols(g, ws, ctx->seam_stream, ctx->sms);
        cudaEventRecord(ctx->seam_join, ctx->seam_stream);
    }
    if (rows > 1) launch_seam_rows(g, ws, g.ty0, rows - 1, s, ctx->sms);
    if (fork)
        cudaStreamWaitEvent(s, ctx->seam_join, 0);
    else
        launch_seam_cols(g, ws, s, ctx->sms);
    return (rows > 1) + (g.ntx > 1);
}

// Phase-timing event.  Inside a stream capture a plain record only becomes an internal graph
// dependency; the external flag makes it a real event record node that replays time.
void record_event(cudaEvent_t ev, cudaStream_t s, bool capturing) {
    if (capturing)
        cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
    else
        cudaEventRecord(ev, s);
}

// (Re)build geometry, grow the workspace, enqueue the pipeline.
int enqueue(rl_ctx* ctx, const uint8_t* dpix, int32_t W, int32_t H, int32_t B, const rl_config* cfg, int32_t fmt) {
    ctx->split_active = 0;
    Geo g = make_geo(W, H, B, cfg, dpix, fmt);
    if (ctx->force_ofmt >= 0) set_output_format(g, ctx->force_ofmt);
    if (ctx->stride_mult > 1) {  // a split pipeline: every stride_mult-th image of the caller's batch
        g.fbytes *= ctx->stride_mult;
        g.ofbytes *= ctx->stride_mult;
    }
    if (ctx->permute) {  // testing aid: a multiplier coprime to the tile count
        int64_t m = ctx->permute % std::max<int64_t>(g.ntiles, 1), a, b;
        for (;; ++m) {
            for (a = m, b = g.ntiles; b;) {
                const int64_t t = a % b;
                a = b;
                b = t;
            }
            if (a == 1 || g.ntiles <= 1) break;
        }
        g.permute = g.ntiles > 1 ? m : 0;
    }
    if (g.ntiles < 0) return set_err(ctx, RL_EINVAL, "too many tiles");
    const int64_t ncnt = (int64_t)B * H * g.ntx + 1;
    Ws ws;
    size_t tmp = 0;
    if (const int rc = prepare_ws(ctx, g, cfg, ws, tmp, g.P * B)) return rc;

    cudaStream_t s = ctx->stream;
    const bool densify_fill = cfg->densify_labels && cfg->fill_holes && g.label_mode;
    const bool need_rank = densify_fill || ctx->want_compact;
    if (need_rank) {
        const uint64_t total = ctx->cap_comps;
        if (!ensure(ctx->rank, (total + 1) * 4) || !ensure(ctx->flag, (total + 1) * 4))
            return set_err(ctx, RL_ENOMEM, "device allocation failed");
    }
    if (ctx->want_compact && !ensure(ctx->fcomp, ctx->cap_comps * sizeof(Acc)))
        return set_err(ctx, RL_ENOMEM, "device allocation failed");
    const int pack = ctx->want_pack & (ctx->want_compact ? 3 : 1);
    if ((pack & 1) && !(ensure(ctx->pk, ctx->cap_comps * sizeof(rlp::Slot)) && ensure(ctx->pkpar, ctx->cap_comps * 4) &&
                        ensure(ctx->pkesc, ctx->cap_comps * sizeof(rl_component))))
        return set_err(ctx, RL_ENOMEM, "device allocation failed");
    if ((pack & 2) && !ensure(ctx->fpk, ctx->cap_comps * sizeof(rlp::Slot)))
        return set_err(ctx, RL_ENOMEM, "device allocation failed");
    // summary rows 0..B-1 per image, B batch totals, B + 1 escape counts of the packed slots
    const size_t sn = (size_t)(B + 2) * 4;
    if (ctx->h_summ_n < sn) {
        if (ctx->h_summ) cudaFreeHost(ctx->h_summ);
        ctx->h_summ = nullptr;
        if (cudaMallocHost(&ctx->h_summ, sn * 8) != cudaSuccess) return set_err(ctx, RL_ENOMEM, "pinned alloc failed");
        ctx->h_summ_n = sn;
    }

    // The whole pipeline is captured once into a CUDA graph and replayed while the geometry,
    // configuration and workspace stay the same (small workloads are launch-bound; large ones
    // still lose the gaps between their ~12 launches).
    const bool use_graph = ctx->graphs && (double)g.P * B <= ctx->graph_max_px;
    GraphKey key{};
    key.g = g;
    key.ws = ws;
    key.cfg = *cfg;
    key.pix = dpix;
    key.stream = s;
    key.summ = ctx->h_summ;
    key.rank = ctx->rank.p;
    key.flag = ctx->flag.p;
    key.fcomp = ctx->fcomp.p;
    key.cap_comps = ctx->cap_comps;
    key.compact = ctx->want_compact ? 1 : 0;
    key.pack = pack;
    key.pk[0] = ctx->pk.p;
    key.pk[1] = ctx->pkpar.p;
    key.pk[2] = ctx->pkesc.p;
    key.pk[3] = ctx->fpk.p;
    if (use_graph && ctx->gexec && std::memcmp(&key, &ctx->gkey, sizeof(key)) == 0) {
        const cudaError_t e = cudaGraphLaunch(ctx->gexec, s);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "graph launch");
        for (int k = 0; k < rl_ctx::NEV; ++k) ctx->ev[k] = ctx->gev[k];
        ctx->geo = g;
        ctx->ws = ws;
        ctx->cfg = *cfg;
        ctx->last_pix = dpix;
        ctx->have_result = true;
        ctx->used_graph = true;
        return RL_OK;
    }
    {
        const int slot = (int)(ctx->calls % rl_ctx::RING);
        for (int k = 0; k < rl_ctx::NEV; ++k) {
            if (!ctx->ring[slot][k]) cudaEventCreate(&ctx->ring[slot][k]);
            ctx->ev[k] = ctx->ring[slot][k];
        }
        ++ctx->calls;
    }
    if (use_graph) {
        if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
        ctx->gexec = nullptr;
        if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
            return cuda_fail(ctx, cudaGetLastError(), "graph capture");
    }
    int launches = 0;
    {
        const int64_t sw = (int64_t)(scan_state_bytes(ncnt) / 8);
        const int64_t n = std::max<int64_t>(std::max(B, 16), sw);
        k_init<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, s>>>(
            ws, B, ws.cnt + (ncnt - 1), P<int64_t>(ctx->summ) + 4 * (B + 1),
            static_cast<unsigned long long*>(ctx->cub_tmp.p), sw);
        ++launches;
    }
    ctx->nkev = 0;
    auto kt = [&]() {  // tuning aid: an event after each launch group
        if (!ctx->ktimes || use_graph || ctx->nkev >= 24) return;
        if (!ctx->kev[ctx->nkev]) cudaEventCreate(&ctx->kev[ctx->nkev]);
        cudaEventRecord(ctx->kev[ctx->nkev++], s);
    };
    record_event(ctx->ev[0], s, use_graph);
    kt();
    launch_analyze(dpix, g, ws, s);
    launches += direct_call(g) ? 2 : 3;
    record_event(ctx->ev[1], s, use_graph);
    kt();
    launches += enqueue_seams(ctx, g, ws, s);
    kt();
    const int64_t hint = (int64_t)ctx->cap_nodes;
    launch_resolve(g, ws, s, ctx->sms, hint);  // + representatives and their counts
    kt();
    launch_scan(ws.cnt, ws.off, ncnt, 0u, ctx->cub_tmp.p, s, true);  // canonical-id offsets (state zeroed by k_init)
    kt();
    launch_cids(g, ws, s, ctx->sms);
    kt();
    launch_tree(g, ws, s, ctx->sms, hint);
    launches += 1 + 1 + 1 + 1;
    kt();
    record_event(ctx->ev[2], s, use_graph);
    if (ctx->seam_stream && !ctx->ktimes)
        launch_emit(g, ws, s, ctx->seam_stream, ctx->seam_fork, ctx->seam_join);
    else
        launch_emit(g, ws, s);
    launches += (direct_call(g) ? 2 : 3) + (g.tpi >= 8192 ? 1 : 0);  // + the shard-table flush (kernels.cu FT_MIN_TILES)
    kt();
    k_summary<<<(B + 1 + 127) / 128, 128, 0, s>>>(g, ws, P<uint64_t>(ctx->cbase), P<int64_t>(ctx->summ));
    ++launches;
    record_event(ctx->ev[3], s, use_graph);
    if (need_rank) {
        // rank of each post-fill root among the batch's components (labeling.hpp:231-236);
        // total components is bounded by cap_comps, flags over [0, cap) are computed for the
        // prefix in use (consumers only read ranks of survivors)
        const uint64_t total = ctx->cap_comps;
        launch_surv_flags(ws.top, P<uint64_t>(ctx->cbase), B, total, P<uint32_t>(ctx->flag), s, ctx->sms);
        launch_scan(P<uint32_t>(ctx->flag), P<uint32_t>(ctx->rank), (int64_t)std::min<uint64_t>(total + 1, 0x7FFFFFFF),
                    0u, ctx->cub_tmp.p, s);
        launches += 2;
    }
    if (densify_fill) {
        launch_remap(ws.labels, g.P, B, P<uint32_t>(ctx->rank), P<uint64_t>(ctx->cbase), ctx->cap_comps, s, ctx->sms);
        ++launches;
    }
    if (ctx->want_compact && !(pack & 2)) {
        launch_compact_filled(ws.filled, P<uint32_t>(ctx->flag), P<uint32_t>(ctx->rank), P<uint64_t>(ctx->cbase) + B,
                              ctx->cap_comps, P<Acc>(ctx->fcomp), s, ctx->sms);
        ++launches;
    }
    if (pack & 1) {
        launch_pack_comps(ws.comps, P<uint64_t>(ctx->cbase) + B, ctx->cap_comps, ctx->pk.p, P<uint32_t>(ctx->pkpar),
                          P<rl_component>(ctx->pkesc), P<int64_t>(ctx->summ) + 4 * (B + 1), s, ctx->sms);
        ++launches;
    }
    if (pack & 2) {
        launch_pack_filled(ws.filled, P<uint32_t>(ctx->flag), P<uint32_t>(ctx->rank), P<uint64_t>(ctx->cbase) + B,
                           ctx->cap_comps, ctx->fpk.p, P<Acc>(ctx->fcomp), P<int64_t>(ctx->summ) + 4 * (B + 1) + 1, s,
                           ctx->sms);
        ++launches;
    }
    record_event(ctx->ev[4], s, use_graph);
    cudaMemcpyAsync(ctx->h_summ, ctx->summ.p, sn * 8, cudaMemcpyDeviceToHost, s);
    if (use_graph) {
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(s, &graph);
        if (e == cudaSuccess) e = cudaGraphInstantiate(&ctx->gexec, graph, 0);
        if (graph) cudaGraphDestroy(graph);
        if (e == cudaSuccess) e = cudaGraphLaunch(ctx->gexec, s);
        if (e != cudaSuccess) {
            ctx->gexec = nullptr;
            return cuda_fail(ctx, e, "graph instantiate");
        }
        ctx->gkey = key;
        for (int k = 0; k < rl_ctx::NEV; ++k) ctx->gev[k] = ctx->ev[k];
    }
    ctx->used_graph = use_graph;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch");
    ctx->geo = g;
    ctx->ws = ws;
    ctx->cfg = *cfg;
    ctx->last_pix = dpix;
    ctx->launches = launches;
    ctx->have_result = true;
    return RL_OK;
}

// Wait for the last enqueue; on capacity overflow grow and re-run (synchronously).
int finish(rl_ctx* ctx) {
    ctx->reran = false;
    if (ctx->split_active) {  // the pipelines check (and if needed grow and re-run) themselves
        for (int k = 0; k < ctx->split_active; ++k) {
            rl_ctx* kid = ctx->splits[k];
            const int rc = finish(kid);
            if (rc) return set_err(ctx, rc, kid->err);
            ctx->reran |= kid->reran;
        }
        return RL_OK;
    }
    for (int attempt = 0; attempt < 4; ++attempt) {
        const cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "pipeline");
        const int B = ctx->geo.B;
        const int64_t* tail = ctx->h_summ + 4 * B;
        const uint64_t total_comps = (uint64_t)tail[0];
        const uint64_t nodes = (uint64_t)tail[1];
        const uint32_t errs = (uint32_t)tail[2];
        const uint64_t rused = (uint64_t)tail[3];
        bool grow = false;
        if (errs & ERR_INTERNAL) return set_err(ctx, RL_EINTERNAL, "device invariant violated (tree reference)");
        if (errs & (ERR_NODE_CAP | ERR_RSTORE_CAP)) {
            if (errs & ERR_NODE_CAP)
                ctx->cap_nodes = (uint32_t)std::min<uint64_t>(nodes + nodes / 4 + 1024, 0xF0000000ull);
            if (errs & ERR_RSTORE_CAP) ctx->cap_rstore = rused + rused / 8 + 4096;
            grow = true;
        } else if (total_comps > ctx->cap_comps) {
            ctx->cap_comps = total_comps + total_comps / 8 + 1024;
            grow = true;
        }
        if (!grow) return RL_OK;
        ctx->reran = true;
        const rl_config cfg = ctx->cfg;
        ctx->force_ofmt = ctx->geo.ofmt != ctx->geo.fmt ? ctx->geo.ofmt : -1;
        const int rc = enqueue(ctx, ctx->last_pix, ctx->geo.W, ctx->geo.H, ctx->geo.B, &cfg, ctx->geo.fmt);
        ctx->force_ofmt = -1;
        if (rc) return rc;
    }
    return set_err(ctx, RL_EINTERNAL, "capacity did not converge");
}

static int times_of(cudaEvent_t const* ev, rl_times* t) {
    float a = 0, m = 0, e = 0, r = 0, tot = 0;
    if (cudaEventElapsedTime(&a, ev[0], ev[1]) != cudaSuccess || cudaEventElapsedTime(&m, ev[1], ev[2]) != cudaSuccess ||
        cudaEventElapsedTime(&e, ev[2], ev[3]) != cudaSuccess || cudaEventElapsedTime(&r, ev[3], ev[4]) != cudaSuccess ||
        cudaEventElapsedTime(&tot, ev[0], ev[4]) != cudaSuccess) {
        cudaGetLastError();
        return RL_ECUDA;
    }
    t->analyze_ms = a;
    t->merge_ms = m;
    t->emit_ms = e;
    t->relabel_ms = r;
    t->total_ms = tot;
    return RL_OK;
}

void fill_times(rl_ctx* ctx, rl_times* t) { times_of(ctx->ev, t); }

// rl_result of a split call: image i ran as image i / K of pipeline i % K; its tables are copied
// from there into the caller's order, the hole-filled image is already in this context's buffer
int fetch_split(rl_ctx* ctx, rl_result* out) {
    const Geo& g = ctx->geo;
    const int B = g.B, K = ctx->split_active;
    out->width = g.W;
    out->height = g.H;
    out->n_images = B;
    int64_t total = 0;
    for (int i = 0; i < B; ++i) total += ctx->splits[i % K]->h_summ[4 * (i / K) + 1];
    out->n_components = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_fg = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_holes = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->euler = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_survivors = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->comp_offset = (int64_t*)std::malloc(sizeof(int64_t) * (B + 1));
    out->comps = (rl_component*)std::malloc(sizeof(rl_component) * std::max<int64_t>(total, 1));
    out->top = (uint32_t*)std::malloc(sizeof(uint32_t) * std::max<int64_t>(total, 1));
    out->filled = (rl_features*)std::malloc(sizeof(rl_features) * std::max<int64_t>(total, 1));
    const size_t npx = (size_t)(g.P * B);
    out->filled_image = (uint8_t*)std::malloc(npx);
    if (!out->n_components || !out->n_fg || !out->n_holes || !out->euler || !out->n_survivors ||
        !out->comp_offset || !out->comps || !out->top || !out->filled || !out->filled_image) {
        rl_result_free(out);
        return set_err(ctx, RL_ENOMEM, "host allocation failed");
    }
    cudaStream_t st = ctx->stream;
    int64_t off = 0;
    for (int i = 0; i < B; ++i) {
        rl_ctx* kid = ctx->splits[i % K];
        const int64_t* s = kid->h_summ + 4 * (i / K);
        const int64_t n = s[1], base = s[0];
        out->comp_offset[i] = off;
        out->n_components[i] = n;
        out->n_fg[i] = s[2];
        out->n_holes[i] = n - 1 - s[2];
        out->euler[i] = out->n_fg[i] - out->n_holes[i];
        out->n_survivors[i] = s[3];
        cudaMemcpyAsync(out->comps + off, kid->ws.comps + base, sizeof(rl_component) * n, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out->top + off, kid->ws.top + base, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st);
        cudaMemcpyAsync(out->filled + off, kid->ws.filled + base, sizeof(rl_features) * n, cudaMemcpyDeviceToHost, st);
        off += n;
    }
    out->comp_offset[B] = off;
    std::vector<uint8_t> p4;
    if (g.ofmt == RL_PIXELS_P4) {
        p4.resize((size_t)(g.ofbytes * B));
        cudaMemcpyAsync(p4.data(), ctx->ws.filled_img, p4.size(), cudaMemcpyDeviceToHost, st);
    } else {
        cudaMemcpyAsync(out->filled_image, ctx->ws.filled_img, npx, cudaMemcpyDeviceToHost, st);
    }
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        rl_result_free(out);
        return cuda_fail(ctx, e, "fetch");
    }
    if (!p4.empty())
        for (int64_t r = 0; r < (int64_t)g.H * B; ++r)
            for (int32_t j = 0; j < g.W; ++j)
                out->filled_image[r * g.W + j] = (p4[r * g.orowb + j / 8] >> (7 - j % 8)) & 1u;
    fill_times(ctx, &out->times);
    return RL_OK;
}

// rl_label_device of a large batch as K concurrent pipelines over interleaved sub-batches (image
// i in pipeline i % K): forked from and joined back into this context's stream; no host sync
int enqueue_split(rl_ctx* ctx, const uint8_t* dpix, int32_t W, int32_t H, int32_t B, const rl_config* cfg,
                  int32_t fmt, int K) {
    Geo g = make_geo(W, H, B, cfg, dpix, fmt);
    if (!ensure(ctx->filled_img, (size_t)(g.ofbytes * B))) return set_err(ctx, RL_ENOMEM, "device allocation failed");
    if (!ctx->split_fork && cudaEventCreateWithFlags(&ctx->split_fork, cudaEventDisableTiming) != cudaSuccess)
        return cuda_fail(ctx, cudaGetLastError(), "events");
    for (int k = 0; k < K; ++k) {
        if (!ctx->splits[k]) {
            ctx->splits[k] = rl_create(ctx->device);
            if (!ctx->splits[k]) return set_err(ctx, RL_ECUDA, "could not create a pipeline context");
            ctx->splits[k]->graphs = ctx->graphs;
            ctx->splits[k]->graph_max_px = ctx->graph_max_px;
            ctx->splits[k]->permute = ctx->permute;
        }
        if (!ctx->split_join[k] && cudaEventCreateWithFlags(&ctx->split_join[k], cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(ctx, cudaGetLastError(), "events");
    }
    const int slot = (int)(ctx->calls % rl_ctx::RING);
    for (int k = 0; k < rl_ctx::NEV; ++k) {
        if (!ctx->ring[slot][k]) cudaEventCreate(&ctx->ring[slot][k]);
        ctx->ev[k] = ctx->ring[slot][k];
    }
    ++ctx->calls;
    cudaStream_t s = ctx->stream;
    cudaEventRecord(ctx->ev[0], s);
    cudaEventRecord(ctx->split_fork, s);
    int launches = 0;
    uint8_t* filled = P<uint8_t>(ctx->filled_img);
    for (int k = 0; k < K; ++k) {
        rl_ctx* kid = ctx->splits[k];
        kid->stride_mult = K;
        kid->ext_filled = filled + (size_t)g.ofbytes * k;
        kid->want_compact = false;
        kid->want_pack = 0;
        kid->force_ofmt = ctx->force_ofmt;
        cudaStreamWaitEvent(kid->stream, ctx->split_fork, 0);
        const int rc = enqueue(kid, dpix + (size_t)g.fbytes * k, W, H, (B - k + K - 1) / K, cfg, fmt);
        if (rc) return set_err(ctx, rc, kid->err);
        cudaEventRecord(ctx->split_join[k], kid->stream);
        cudaStreamWaitEvent(s, ctx->split_join[k], 0);
        launches += kid->launches;
    }
    for (int k = 1; k < rl_ctx::NEV; ++k) cudaEventRecord(ctx->ev[k], s);  // phases overlap: total only
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(ctx, e, "launch");
    ctx->geo = g;
    ctx->cfg = *cfg;
    ctx->last_pix = dpix;
    ctx->ws = Ws{};
    ctx->ws.filled_img = filled;
    ctx->launches = launches;
    ctx->used_graph = ctx->splits[0]->used_graph;
    ctx->split_active = K;
    ctx->have_result = true;
    return RL_OK;
}

int fetch(rl_ctx* ctx, rl_result* out) {
    std::memset(out, 0, sizeof(*out));
    const Geo& g = ctx->geo;
    const int B = g.B;
    out->width = g.W;
    out->height = g.H;
    out->n_images = B;
    if (ctx->split_active) return fetch_split(ctx, out);
    const int64_t* s = ctx->h_summ;
    const uint64_t total = (uint64_t)s[4 * B];
    out->n_components = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_fg = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_holes = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->euler = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->n_survivors = (int64_t*)std::malloc(sizeof(int64_t) * B);
    out->comp_offset = (int64_t*)std::malloc(sizeof(int64_t) * (B + 1));
    out->comps = (rl_component*)std::malloc(sizeof(rl_component) * std::max<uint64_t>(total, 1));
    out->top = (uint32_t*)std::malloc(sizeof(uint32_t) * std::max<uint64_t>(total, 1));
    out->filled = (rl_features*)std::malloc(sizeof(rl_features) * std::max<uint64_t>(total, 1));
    const size_t npx = (size_t)(g.P * B);
    out->filled_image = (uint8_t*)std::malloc(npx);
    if (g.label_mode) out->labels = (uint32_t*)std::malloc(npx * 4);
    if (!out->n_components || !out->n_fg || !out->n_holes || !out->euler || !out->n_survivors ||
        !out->comp_offset || !out->comps || !out->top || !out->filled || !out->filled_image ||
        (g.label_mode && !out->labels)) {
        rl_result_free(out);
        return set_err(ctx, RL_ENOMEM, "host allocation failed");
    }
    for (int b = 0; b < B; ++b) {
        out->comp_offset[b] = s[4 * b + 0];
        out->n_components[b] = s[4 * b + 1];
        out->n_fg[b] = s[4 * b + 2];
        out->n_holes[b] = s[4 * b + 1] - 1 - s[4 * b + 2];
        out->euler[b] = out->n_fg[b] - out->n_holes[b];
        out->n_survivors[b] = s[4 * b + 3];
    }
    out->comp_offset[B] = (int64_t)total;
    cudaStream_t st = ctx->stream;
    cudaMemcpyAsync(out->comps, ctx->ws.comps, sizeof(rl_component) * total, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(out->top, ctx->ws.top, sizeof(uint32_t) * total, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(out->filled, ctx->ws.filled, sizeof(rl_features) * total, cudaMemcpyDeviceToHost, st);
    std::vector<uint8_t> p4;
    if (g.ofmt == RL_PIXELS_P4) {  // rl_result holds one byte per pixel: unpack the P4 rows
        p4.resize((size_t)(g.ofbytes * B));
        cudaMemcpyAsync(p4.data(), ctx->ws.filled_img, p4.size(), cudaMemcpyDeviceToHost, st);
    } else {
        cudaMemcpyAsync(out->filled_image, ctx->ws.filled_img, npx, cudaMemcpyDeviceToHost, st);
    }
    if (g.label_mode) cudaMemcpyAsync(out->labels, ctx->ws.labels, npx * 4, cudaMemcpyDeviceToHost, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        rl_result_free(out);
        return cuda_fail(ctx, e, "fetch");
    }
    if (!p4.empty())
        for (int64_t r = 0; r < (int64_t)g.H * B; ++r)
            for (int32_t j = 0; j < g.W; ++j)
                out->filled_image[r * g.W + j] = (p4[r * g.orowb + j / 8] >> (7 - j % 8)) & 1u;
    fill_times(ctx, &out->times);
    return RL_OK;
}


// ---- rl_label_into: chunked, pipelined host-buffer path

}  // namespace rlh

namespace {

// every grow-only device table of a context
template <class F>
void for_each_buf(rl_ctx* c, F&& f) {
    DevBuf* bufs[] = {&c->bits, &c->tbase, &c->tnb, &c->perim, &c->uf, &c->nkey, &c->nmin, &c->nacc,
                      &c->nrec, &c->nrep, &c->ninfo, &c->nrootcid, &c->nparent, &c->nanccid, &c->cnt, &c->off,
                      &c->counters, &c->img_fg, &c->img_surv, &c->comps, &c->top, &c->filled,
                      &c->filled_img, &c->labels, &c->pix, &c->cub_tmp, &c->cbase, &c->summ,
                      &c->rank, &c->flag, &c->ovf, &c->ovf2, &c->thdr, &c->tmap, &c->rstore, &c->rused,
                      &c->fcomp, &c->nleft, &c->scount, &c->ncut, &c->nfold, &c->xnode, &c->gtab, &c->ftab,
                      &c->pk, &c->pkpar, &c->pkesc, &c->fpk, &c->xrec, &c->xgath, &c->xred};
    for (DevBuf* b : bufs) f(*b);
}

}  // namespace

extern "C" {

int64_t rl_workspace_bytes(const rl_ctx* c) {
    if (!c) return 0;
    int64_t n = 0;
    for_each_buf(const_cast<rl_ctx*>(c), [&](DevBuf& b) { n += (int64_t)b.bytes; });
    return n;
}

rl_ctx* rl_create(int device) {
    rl_ctx* c = new (std::nothrow) rl_ctx();
    if (!c) return nullptr;
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return nullptr;
    }
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (configure_kernels() != cudaSuccess || cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return nullptr;
    }
    c->stream = c->own_stream;
    if (cudaStreamCreateWithFlags(&c->seam_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->seam_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->seam_join, cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        c->seam_stream = nullptr;  // the seams then run one after the other
    }
    if (std::getenv("RUNLAB_GPU_NO_GRAPH")) c->graphs = false;
    if (const char* v = std::getenv("RUNLAB_GPU_GRAPH_MPX")) c->graph_max_px = std::atof(v) * 1024 * 1024;
    if (const char* v = std::getenv("RUNLAB_GPU_PERMUTE")) c->permute = std::max(0ll, std::atoll(v));
    if (const char* v = std::getenv("RUNLAB_GPU_SPLIT")) c->split = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("RUNLAB_GPU_SPLIT_MPX")) c->split_min_px = std::atof(v) * 1024 * 1024;
    if (std::getenv("RUNLAB_GPU_KTIMES")) c->ktimes = true;
    if (std::getenv("RUNLAB_GPU_NO_PACKED_D2H")) c->packed_d2h = false;
    if (std::getenv("RUNLAB_GPU_NO_PACKED_RECORDS")) c->packed_recs = false;
    if (const char* v = std::getenv("RUNLAB_GPU_PACKED_H2D")) c->packed_h2d = std::atoi(v) != 0;
    if (const char* v = std::getenv("RUNLAB_GPU_KIDS")) c->nkids = std::min(rl_ctx::MAXKIDS, std::max(1, std::atoi(v)));
    if (const char* v = std::getenv("RUNLAB_GPU_HOST_THREADS")) c->host_threads = std::max(1, std::atoi(v));
    if (const char* v = std::getenv("RUNLAB_GPU_CHUNK_PX")) c->chunk_px = std::max(1ll, std::atoll(v));
    if (const char* v = std::getenv("RUNLAB_GPU_BIG_PX")) c->big_single_px = std::max(1ll, std::atoll(v));
    return c;
}

void rl_destroy(rl_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);

    for (rl_ctx* k : c->kids) rl_destroy(k);
    for (rl_ctx* k : c->splits) rl_destroy(k);
    if (c->split_fork) cudaEventDestroy(c->split_fork);
    for (cudaEvent_t e : c->split_join)
        if (e) cudaEventDestroy(e);
    strip_free(c);
    pool_free(c);
    for (uint8_t* p : c->h_stage)
        if (p) cudaFreeHost(p);
    for (uint8_t* p : c->h_rstage)
        if (p) cudaFreeHost(p);
    for (uint8_t* p : c->h_istage)
        if (p) cudaFreeHost(p);
    for_each_buf(c, [](DevBuf& b) {
        if (b.p) cudaFree(b.p);
    });
    if (c->h_summ) cudaFreeHost(c->h_summ);
    if (c->h_strip) cudaFreeHost(c->h_strip);
    for (auto& slot : c->ring)
        for (auto& e : slot)
            if (e) cudaEventDestroy(e);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (auto& e : c->kev)
        if (e) cudaEventDestroy(e);
    if (c->out_stream) {
        cudaStreamSynchronize(c->out_stream);
        cudaStreamDestroy(c->out_stream);
    }
    if (c->out_done) cudaEventDestroy(c->out_done);
    if (c->in_stream) {
        cudaStreamSynchronize(c->in_stream);
        cudaStreamDestroy(c->in_stream);
    }
    if (c->in_done) cudaEventDestroy(c->in_done);
    if (c->seam_stream) cudaStreamDestroy(c->seam_stream);
    if (c->seam_fork) cudaEventDestroy(c->seam_fork);
    if (c->seam_join) cudaEventDestroy(c->seam_join);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    delete c;
}

const char* rl_last_error(const rl_ctx* c) { return c ? c->err.c_str() : "null context"; }

int rl_label_device_fmt(rl_ctx* ctx, const uint8_t* d_pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg,
                        int32_t pixel_format) {
    const int rc = check_args(ctx, w, h, n, cfg);
    if (rc) return rc;
    if (pixel_format != RL_PIXELS_U8 && pixel_format != RL_PIXELS_P4)
        return set_err(ctx, RL_EINVAL, "unknown pixel format");
    cudaSetDevice(ctx->device);
    ctx->want_compact = false;
    ctx->want_pack = 0;
    // large batches without a label image run as concurrent interleaved pipelines
    const int K = std::min(ctx->split, rl_ctx::MAXSPLIT);
    if (K > 1 && !cfg->relabel && n >= 4 * K && (double)w * h * n >= ctx->split_min_px)
        return enqueue_split(ctx, d_pixels, w, h, n, cfg, pixel_format, K);
    ctx->split_active = 0;
    return enqueue(ctx, d_pixels, w, h, n, cfg, pixel_format);
}

int rl_set_pipelines(rl_ctx* ctx, int k) {
    if (!ctx || k < 1) return RL_EINVAL;
    ctx->split = std::min(k, rl_ctx::MAXSPLIT);
    return RL_OK;
}

int rl_label_device(rl_ctx* ctx, const uint8_t* d_pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg) {
    return rl_label_device_fmt(ctx, d_pixels, w, h, n, cfg, RL_PIXELS_U8);
}

int rl_sync(rl_ctx* ctx) {
    if (!ctx || !ctx->have_result) return set_err(ctx, RL_ELOGIC, "no pipeline enqueued");
    cudaSetDevice(ctx->device);
    return finish(ctx);
}

int rl_fetch(rl_ctx* ctx, rl_result* out) {
    if (!out) return RL_EINVAL;
    const int rc = rl_sync(ctx);
    if (rc) return rc;
    return fetch(ctx, out);
}

int rl_label(rl_ctx* ctx, const uint8_t* pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg,
             rl_result* out) {
    if (!out) return RL_EINVAL;
    std::memset(out, 0, sizeof(*out));
    int rc = check_args(ctx, w, h, n, cfg);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    const size_t npx = (size_t)w * h * n;
    if (!ensure(ctx->pix, npx)) return set_err(ctx, RL_ENOMEM, "device allocation failed");
    cudaError_t e = cudaMemcpyAsync(ctx->pix.p, pixels, npx, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "copy in");
    ctx->want_compact = false;
    ctx->want_pack = 0;
    rc = enqueue(ctx, P<uint8_t>(ctx->pix), w, h, n, cfg, RL_PIXELS_U8);
    if (rc) return rc;
    rc = finish(ctx);
    if (rc) return rc;
    return fetch(ctx, out);
}

int rl_phase_times(const rl_ctx* ctx, int back, rl_times* out) {
    if (!ctx || !out || back < 0 || back >= rl_ctx::RING || back >= ctx->calls) return RL_EINVAL;
    // back == 0 is the last call (also when it was a CUDA-graph replay, whose events are
    // the captured ones); older calls come from the ring of eagerly enqueued calls
    const int slot = (int)((ctx->calls - 1 - back) % rl_ctx::RING);
    cudaEvent_t const* ev = back == 0 ? ctx->ev : ctx->ring[slot];
    return times_of(ev, out);
}

void rl_result_free(rl_result* r) {
    if (!r) return;
    std::free(r->n_components);
    std::free(r->n_fg);
    std::free(r->n_holes);
    std::free(r->euler);
    std::free(r->n_survivors);
    std::free(r->comp_offset);
    std::free(r->comps);
    std::free(r->top);
    std::free(r->filled);
    std::free(r->filled_image);
    std::free(r->labels);
    std::memset(r, 0, sizeof(*r));
}

void* rl_device_filled_image(rl_ctx* c) { return c ? c->ws.filled_img : nullptr; }
void* rl_device_labels(rl_ctx* c) { return c ? c->ws.labels : nullptr; }
void* rl_device_comps(rl_ctx* c) { return c && !c->split_active ? c->ws.comps : nullptr; }
void* rl_stream(rl_ctx* c) { return c ? (void*)c->stream : nullptr; }
int rl_set_stream(rl_ctx* c, void* stream) {
    if (!c) return RL_EINVAL;
    c->stream = stream ? (cudaStream_t)stream : c->own_stream;
    return RL_OK;
}
int rl_last_launch_count(const rl_ctx* c) { return c ? c->launches : 0; }
void rl_tile_shape(int32_t* th, int32_t* tw) {
    if (th) *th = TH;
    if (tw) *tw = TW;
}

}  // extern "C"

extern "C" int rl_last_used_graph(const rl_ctx* c) { return c && c->used_graph ? 1 : 0; }

// tuning aid (RUNLAB_GPU_KTIMES): ms between the events recorded after each launch group of the
// last eager call: analyze, seams, resolve, reps, scan, cids, tree (parents+tops+fold), emit
extern "C" int rl_debug_launch_times(rl_ctx* c, float* ms, int max_n) {
    if (!c || c->nkev < 2) return 0;
    cudaEventSynchronize(c->kev[c->nkev - 1]);
    int n = 0;
    for (int k = 1; k < c->nkev && n < max_n; ++k) cudaEventElapsedTime(&ms[n++], c->kev[k - 1], c->kev[k]);
    return n;
}
