// strips_multi.cu -- one image as horizontal strips over several contexts of ONE process
// (rl_label_strips): one context per GPU of a node, or several on one GPU.
//
// The per-rank strip phases of strips.cu run on one host thread per strip; the collectives
// between them (all-gather of the strips' exchange records, all-reduce of the link
// table and of the cut survivors' partial features) are device-to-device copies between the
// contexts' devices (peer copies over NVLink when the contexts sit on different GPUs) followed by
// an element-wise reduction kernel on every device.  Only O(width) bytes move: the records,
// the links and the partials.  The result is bit-identical to the single-image pipeline (and to
// the torch.distributed driver in paper_2006_09299_b200/strips.py, which calls the same phases).
#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "ctx.hpp"

namespace {
using namespace rlh;

// out[i] = reduce over q < k of slices[q * n + i]
__global__ void k_sum_i64(int64_t* out, const int64_t* slices, int k, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = 0;
        for (int q = 0; q < k; ++q) v += slices[q * n + i];
        out[i] = v;
    }
}
__global__ void k_minmax_i32(int32_t* out, const int32_t* slices, int k, int64_t n, int is_max) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = slices[i];
        for (int q = 1; q < k; ++q) {
            const int32_t x = slices[q * n + i];
            v = is_max ? max(v, x) : min(v, x);
        }
        out[i] = v;
    }
}

unsigned grid_of(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184)); }

// Generation barrier for the strips' host threads.
struct Barrier {
    std::mutex m;
    std::condition_variable cv;
    int n, waiting = 0;
    unsigned gen = 0;
    bool broken = false;  // a strip thread could not be started: every wait returns at once
    explicit Barrier(int n_) : n(n_) {}
    void wait() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) return;
        const unsigned g = gen;
        if (++waiting == n) {
            waiting = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g || broken; });
        }
    }
    void abort() {
        std::lock_guard<std::mutex> lk(m);
        broken = true;
        cv.notify_all();
    }
};

// Copies every context's device array src[q] (bytes each) into dst on context r's device, slice q
// at q * bytes, and waits for them.
cudaError_t gather(rl_ctx* const* ctx, int k, int r, const std::vector<const void*>& src, size_t bytes, void* dst) {
    for (int q = 0; q < k; ++q) {
        cudaError_t e = cudaMemcpyPeerAsync(static_cast<uint8_t*>(dst) + (size_t)q * bytes, ctx[r]->device, src[q],
                                            ctx[q]->device, bytes, ctx[r]->stream);
        if (e != cudaSuccess) return e;
    }
    return cudaStreamSynchronize(ctx[r]->stream);
}

}  // namespace

extern "C" {

int rl_strip_rows(int32_t height, int32_t n_strips, int32_t* y0, int32_t* h) {
    if (height < 1 || !y0 || !h) return RL_EINVAL;
    const int32_t tiles = (height + TH - 1) / TH;
    if (n_strips < 1 || n_strips > tiles) return RL_EINVAL;
    const int32_t base = tiles / n_strips, extra = tiles % n_strips;
    int32_t t = 0;
    for (int32_t r = 0; r < n_strips; ++r) {
        const int32_t nt = base + (r < extra ? 1 : 0);
        y0[r] = t * TH;
        h[r] = std::min((t + nt) * TH, height) - y0[r];
        t += nt;
    }
    return RL_OK;
}

namespace {
int label_strips(rl_ctx* const* ctx, int32_t k, const uint8_t* const* d_strips, int32_t width, int32_t height,
                 const rl_config* cfg, rl_strip_result* results);
}

int rl_label_strips(rl_ctx* const* ctx, int32_t k, const uint8_t* const* d_strips, int32_t width, int32_t height,
                    const rl_config* cfg, rl_strip_result* results) {
    if (!ctx || !d_strips || !cfg || !results || k < 1) return RL_EINVAL;
    try {  // no C++ exception crosses the C ABI (thread creation, allocation)
        return label_strips(ctx, k, d_strips, width, height, cfg, results);
    } catch (const std::bad_alloc&) {
        return ctx[0] ? set_err(ctx[0], RL_ENOMEM, "strips: host allocation failed") : RL_ENOMEM;
    } catch (const std::exception& e) {
        return ctx[0] ? set_err(ctx[0], RL_EINTERNAL, std::string("strips: ") + e.what()) : RL_EINTERNAL;
    }
}

}  // extern "C"

namespace {
int label_strips(rl_ctx* const* ctx, int32_t k, const uint8_t* const* d_strips, int32_t width, int32_t height,
                 const rl_config* cfg, rl_strip_result* results) {
    for (int r = 0; r < k; ++r) {
        if (!ctx[r] || !d_strips[r]) return RL_EINVAL;
        for (int q = 0; q < r; ++q)
            if (ctx[q] == ctx[r]) return set_err(ctx[0], RL_EINVAL, "strips: one context per strip");
    }
    std::vector<int32_t> y0(k), h(k);
    if (rl_strip_rows(height, k, y0.data(), h.data()) != RL_OK)
        return set_err(ctx[0], RL_EINVAL, "strips: cannot cut the image into that many strips of whole tile rows");
    // contexts on different devices read each other's buffers directly (peer copies go through
    // the host otherwise)
    for (int r = 0; r < k; ++r)
        for (int q = 0; q < k; ++q) {
            if (ctx[q]->device == ctx[r]->device) continue;
            int ok = 0;
            cudaDeviceCanAccessPeer(&ok, ctx[r]->device, ctx[q]->device);
            if (ok) {
                cudaSetDevice(ctx[r]->device);
                if (cudaDeviceEnablePeerAccess(ctx[q]->device, 0) != cudaSuccess) cudaGetLastError();  // already on
            }
        }

    std::vector<rl_strip_local_info> infos(k);
    std::vector<rl_strip_links> links(k);
    std::vector<rl_strip_partials> parts(k);
    std::vector<int> rc(k, RL_OK);
    std::mutex fm;
    bool failed = false;
    Barrier bar(k);
    auto fail = [&](int r, int code) {
        rc[r] = code;
        std::lock_guard<std::mutex> lk(fm);
        failed = true;
    };
    auto ok = [&] {
        std::lock_guard<std::mutex> lk(fm);
        return !failed;
    };

    auto rank = [&](int r) {
        rl_ctx* c = ctx[r];
        cudaSetDevice(c->device);
        int e = rl_strip_local(c, d_strips[r], width, height, y0[r], h[r], cfg, &infos[r]);
        if (e) fail(r, e);
        bar.wait();
        // ---- all-gather of the records
        int64_t mc = 0;
        for (int q = 0; q < k; ++q) mc = std::max<int64_t>(mc, infos[q].n_classes);
        const size_t xb = (size_t)rl_strip_export_bytes(width, mc);
        if (ok()) {
            if (!ensure(c->xrec, xb) || !ensure(c->xgath, xb * k)) fail(r, set_err(c, RL_ENOMEM, "device allocation failed"));
            else if ((e = rl_strip_export(c, mc, c->xrec.p))) fail(r, e);
        }
        bar.wait();
        if (ok()) {
            std::vector<const void*> src(k);
            for (int q = 0; q < k; ++q) src[q] = ctx[q]->xrec.p;
            const cudaError_t ce = gather(ctx, k, r, src, xb, c->xgath.p);
            if (ce != cudaSuccess) fail(r, cuda_fail(c, ce, "strips: record exchange"));
            else if ((e = rl_strip_merge(c, c->xgath.p, k, infos.data(), mc, &links[r]))) fail(r, e);
        }
        bar.wait();
        // ---- all-reduce SUM of the link tables: every rank stages all of them, then sums
        const int64_t nl = links[0].n;
        if (ok()) {
            std::vector<const void*> src(k);
            for (int q = 0; q < k; ++q) src[q] = links[q].d_links;
            cudaError_t ce = ensure(c->xred, (size_t)nl * 8 * k) ? cudaSuccess : cudaErrorMemoryAllocation;
            if (ce == cudaSuccess) ce = gather(ctx, k, r, src, (size_t)nl * 8, c->xred.p);
            if (ce != cudaSuccess) fail(r, cuda_fail(c, ce, "strips: link exchange"));
        }
        bar.wait();  // every rank holds every original table before any is overwritten
        if (ok()) {
            if (nl) k_sum_i64<<<grid_of(nl), 256, 0, c->stream>>>(static_cast<int64_t*>(links[r].d_links),
                                                                  P<int64_t>(c->xred), k, nl);
            if ((e = rl_strip_resolve(c, &parts[r]))) fail(r, e);
        }
        bar.wait();
        // ---- all-reduce of the cut survivors' partial features (SUM / MIN / MAX) and counts
        const int64_t K = parts[0].k;
        const size_t bs = (size_t)K * 3 * 8, bm = (size_t)K * 2 * 4;
        const size_t o_min = (size_t)k * bs, o_max = o_min + (size_t)k * bm, o_cnt = o_max + (size_t)k * bm;
        if (ok()) {
            cudaError_t ce = ensure(c->xred, o_cnt + (size_t)k * 8) ? cudaSuccess : cudaErrorMemoryAllocation;
            std::vector<const void*> src(k);
            uint8_t* base = P<uint8_t>(c->xred);
            if (ce == cudaSuccess && K) {
                for (int q = 0; q < k; ++q) src[q] = parts[q].d_sum;
                ce = gather(ctx, k, r, src, bs, base);
                for (int q = 0; q < k && ce == cudaSuccess; ++q) src[q] = parts[q].d_min;
                if (ce == cudaSuccess) ce = gather(ctx, k, r, src, bm, base + o_min);
                for (int q = 0; q < k && ce == cudaSuccess; ++q) src[q] = parts[q].d_max;
                if (ce == cudaSuccess) ce = gather(ctx, k, r, src, bm, base + o_max);
            }
            for (int q = 0; q < k && ce == cudaSuccess; ++q) src[q] = parts[q].d_count;
            if (ce == cudaSuccess) ce = gather(ctx, k, r, src, 8, base + o_cnt);
            if (ce != cudaSuccess) fail(r, cuda_fail(c, ce, "strips: partial-feature exchange"));
        }
        bar.wait();
        if (ok()) {
            uint8_t* base = P<uint8_t>(c->xred);
            if (K) {
                k_sum_i64<<<grid_of(3 * K), 256, 0, c->stream>>>(static_cast<int64_t*>(parts[r].d_sum),
                                                                 reinterpret_cast<int64_t*>(base), k, 3 * K);
                k_minmax_i32<<<grid_of(2 * K), 256, 0, c->stream>>>(static_cast<int32_t*>(parts[r].d_min),
                                                                     reinterpret_cast<int32_t*>(base + o_min), k,
                                                                     2 * K, 0);
                k_minmax_i32<<<grid_of(2 * K), 256, 0, c->stream>>>(static_cast<int32_t*>(parts[r].d_max),
                                                                     reinterpret_cast<int32_t*>(base + o_max), k,
                                                                     2 * K, 1);
            }
            k_sum_i64<<<1, 256, 0, c->stream>>>(static_cast<int64_t*>(parts[r].d_count),
                                                reinterpret_cast<int64_t*>(base + o_cnt), k, 1);
            const cudaError_t ce = cudaGetLastError();
            if (ce != cudaSuccess) fail(r, cuda_fail(c, ce, "strips: reduction"));
            else if ((e = rl_strip_finish(c, &results[r]))) fail(r, e);
        }
    };
    std::vector<std::thread> th;
    th.reserve(k);
    bool started = true;
    try {
        for (int r = 1; r < k; ++r) th.emplace_back(rank, r);
    } catch (const std::exception&) {  // no thread for every strip: the started ones bail out
        started = false;
        fail(0, set_err(ctx[0], RL_EINTERNAL, "strips: could not start the strip threads"));
        bar.abort();
    }
    if (started) rank(0);
    for (auto& t : th) t.join();
    for (int r = 0; r < k; ++r)
        if (rc[r]) {
            if (r) set_err(ctx[0], rc[r], std::string("strip ") + std::to_string(r) + ": " + rl_last_error(ctx[r]));
            return rc[r];
        }
    return RL_OK;
}
}  // namespace

extern "C" {

int rl_label_strips_host(rl_ctx* const* ctx, int32_t k, const uint8_t* pixels, int32_t width, int32_t height,
                         const rl_config* cfg, rl_strip_result* results) {
    if (!ctx || !pixels || k < 1 || width < 1) return RL_EINVAL;
    std::vector<int32_t> y0(k), h(k);
    if (rl_strip_rows(height, k, y0.data(), h.data()) != RL_OK)
        return ctx[0] ? set_err(ctx[0], RL_EINVAL, "strips: cannot cut the image into that many strips of whole tile rows")
                      : RL_EINVAL;
    std::vector<const uint8_t*> d(k);
    for (int r = 0; r < k; ++r) {  // each strip's rows into its context's input buffer
        if (!ctx[r]) return RL_EINVAL;
        cudaSetDevice(ctx[r]->device);
        const size_t bytes = (size_t)h[r] * width;
        if (!ensure(ctx[r]->pix, bytes)) return set_err(ctx[r], RL_ENOMEM, "device allocation failed");
        const cudaError_t e = cudaMemcpyAsync(ctx[r]->pix.p, pixels + (size_t)y0[r] * width, bytes,
                                              cudaMemcpyHostToDevice, ctx[r]->stream);
        if (e != cudaSuccess) return cuda_fail(ctx[r], e, "strips: copy in");
        d[r] = P<uint8_t>(ctx[r]->pix);
    }
    for (int r = 0; r < k; ++r) {
        const cudaError_t e = cudaStreamSynchronize(ctx[r]->stream);
        if (e != cudaSuccess) return cuda_fail(ctx[r], e, "strips: copy in");
    }
    return rl_label_strips(ctx, k, d.data(), width, height, cfg, results);
}

}  // extern "C"
