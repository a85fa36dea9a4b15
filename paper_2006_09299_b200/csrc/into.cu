// into.cu -- rl_label_into: the host-buffer entry point.  Large batches are cut into chunks of
// whole images pipelined through three workspaces/streams (H2D of one chunk, kernels of
// another and D2H of a third overlap); a byte-per-pixel filled image crosses PCIe as P4 bits
// and a host thread pool expands it into the caller's buffer while later chunks are in flight.
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <immintrin.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "common.cuh"
#include "ctx.hpp"
#include "pack.cuh"
#include "runlab_gpu.h"

using namespace rlg;
using namespace rlh;

namespace rlh {
int64_t image_bytes(int32_t w, int32_t h, int32_t fmt) {
    return (int64_t)(fmt == RL_PIXELS_P4 ? (w + 7) / 8 : w) * h;
}
}  // namespace rlh

namespace rlh {
struct HostPool {
    std::vector<std::thread> workers;
    std::mutex m;
    std::condition_variable cv, done;
    std::deque<std::pair<int, std::function<void()>>> q;
    // tags: [0, 2 MAXKIDS) a kid's output staging buffers, [2 MAXKIDS, 4 MAXKIDS) its input
    // staging buffers, 4 MAXKIDS the single-chunk input packing
    int pending[4 * rl_ctx::MAXKIDS + 1] = {};
    bool stop = false;
    explicit HostPool(int n) {
        for (int i = 0; i < n; ++i) workers.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : workers) t.join();
    }
    void loop() {
        for (;;) {
            std::pair<int, std::function<void()>> task;
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return stop || !q.empty(); });
                if (q.empty()) return;
                task = std::move(q.front());
                q.pop_front();
            }
            task.second();
            {
                std::lock_guard<std::mutex> lk(m);
                --pending[task.first];
            }
            done.notify_all();
        }
    }
    void submit(int tag, std::function<void()> f, bool front = false) {
        {
            std::lock_guard<std::mutex> lk(m);
            ++pending[tag];
            if (front)
                q.emplace_front(tag, std::move(f));
            else
                q.emplace_back(tag, std::move(f));
        }
        cv.notify_one();
    }
    // a placeholder task: keeps wait(tag) blocked until release(tag) (work submitted later, e.g.
    // from a stream callback once a copy has landed)
    void reserve(int tag) {
        std::lock_guard<std::mutex> lk(m);
        ++pending[tag];
    }
    void release(int tag) {
        {
            std::lock_guard<std::mutex> lk(m);
            --pending[tag];
        }
        done.notify_all();
    }
    void wait(int tag) {
        std::unique_lock<std::mutex> lk(m);
        done.wait(lk, [&] { return pending[tag] == 0; });
    }
};
void pool_free(rl_ctx* c) {
    delete c->pool;
    c->pool = nullptr;
}
}  // namespace rlh
namespace {

// bytes [i, full) of a P4 row, 4 at a time, into 32-B aligned streaming stores (d + 8 i is
// 32-B aligned); returns the first byte not done
__attribute__((target("avx2"))) int32_t expand_avx2(const uint8_t* s, int32_t i, int32_t full, uint8_t* d) {
    const __m256i shuf = _mm256_setr_epi8(0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2, 2, 2, 3, 3,
                                          3, 3, 3, 3, 3, 3);
    const __m256i bits = _mm256_setr_epi8(-128, 64, 32, 16, 8, 4, 2, 1, -128, 64, 32, 16, 8, 4, 2, 1, -128, 64, 32, 16,
                                          8, 4, 2, 1, -128, 64, 32, 16, 8, 4, 2, 1);
    const __m256i one = _mm256_set1_epi8(1);
    for (; i + 4 <= full; i += 4) {
        uint32_t w;
        std::memcpy(&w, s + i, 4);
        __m256i v = _mm256_shuffle_epi8(_mm256_set1_epi32((int)w), shuf);
        v = _mm256_and_si256(_mm256_cmpeq_epi8(_mm256_and_si256(v, bits), bits), one);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + 8 * i), v);
    }
    return i;
}

// P4 rows -> one byte per pixel (MSB-first bits; binarize_labels' layout, labeling.hpp:354-360)
void expand_p4_rows(const uint8_t* src, int64_t rows, int32_t rowb, int32_t w, uint8_t* dst) {
    static const struct Lut {
        uint64_t v[256];
        Lut() {
            for (int b = 0; b < 256; ++b) {
                uint64_t x = 0;
                for (int k = 0; k < 8; ++k) x |= (uint64_t)((b >> (7 - k)) & 1) << (8 * k);
                v[b] = x;
            }
        }
    } lut;
    const int32_t full = w / 8;
    static const bool avx2 = __builtin_cpu_supports("avx2");
    for (int64_t r = 0; r < rows; ++r) {
        const uint8_t* s = src + r * rowb;
        uint8_t* d = dst + r * w;
        if (((uintptr_t)d & 7) == 0) {  // streaming stores: the caller's buffer is not re-read here
            int32_t i = 0;
            if (avx2) {
                for (; i < full && ((uintptr_t)(d + 8 * i) & 31); ++i)
                    _mm_stream_si64((long long*)(d + 8 * i), (long long)lut.v[s[i]]);
                i = expand_avx2(s, i, full, d);
            }
            for (; i < full; ++i) _mm_stream_si64((long long*)(d + 8 * i), (long long)lut.v[s[i]]);
        } else {
            for (int32_t i = 0; i < full; ++i) std::memcpy(d + 8 * i, &lut.v[s[i]], 8);
        }
        for (int32_t j = 8 * full; j < w; ++j) d[j] = (s[j / 8] >> (7 - j % 8)) & 1u;
    }
    _mm_sfence();
}

// 64 pixels per step: the bytes of each 8-pixel group reversed (P4 is MSB-first), then one
// mask of their bit 0 = 8 P4 bytes; returns the first pixel not done
__attribute__((target("avx512f,avx512bw"))) int32_t pack_avx512(const uint8_t* s, int32_t w, uint8_t* d) {
    const __m512i rev = _mm512_set_epi8(8, 9, 10, 11, 12, 13, 14, 15, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14,
                                        15, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15, 0, 1, 2, 3, 4, 5, 6, 7,
                                        8, 9, 10, 11, 12, 13, 14, 15, 0, 1, 2, 3, 4, 5, 6, 7);
    const __m512i one = _mm512_set1_epi8(1);
    int32_t i = 0;
    for (; i + 64 <= w; i += 64) {
        const __m512i v = _mm512_shuffle_epi8(_mm512_loadu_si512(s + i), rev);
        const uint64_t m = _mm512_test_epi8_mask(v, one);
        std::memcpy(d + i / 8, &m, 8);
    }
    return i;
}

// byte-per-pixel rows -> P4 rows (bit 0 of each byte, MSB-first; the device reads either):
// the host-buffer path sends u8 input over PCIe as bits
__attribute__((target("ssse3"))) void pack_rows_p4(const uint8_t* src, int64_t rows, int32_t w, uint8_t* dst,
                                                   int32_t rowb) {
    static const bool avx512 = __builtin_cpu_supports("avx512bw");
    const __m128i rev = _mm_setr_epi8(7, 6, 5, 4, 3, 2, 1, 0, 15, 14, 13, 12, 11, 10, 9, 8);
    for (int64_t r = 0; r < rows; ++r) {
        const uint8_t* s = src + r * (int64_t)w;
        uint8_t* d = dst + r * (int64_t)rowb;
        int32_t i = avx512 ? pack_avx512(s, w, d) : 0;
        for (; i + 16 <= w; i += 16) {
            __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
            v = _mm_slli_epi16(_mm_shuffle_epi8(v, rev), 7);
            const int m = _mm_movemask_epi8(v);
            d[i / 8] = (uint8_t)m;
            d[i / 8 + 1] = (uint8_t)(m >> 8);
        }
        for (int32_t k = i / 8; k < rowb; ++k) d[k] = 0;
        for (; i < w; ++i) d[i / 8] |= (uint8_t)((s[i] & 1u) << (7 - i % 8));
    }
}

template <class T>
inline void stream_store(T* dst, const T& v) {
    static_assert(sizeof(T) % 8 == 0, "8-byte granules");
    if (((uintptr_t)dst & 7) == 0) {
        const long long* s = reinterpret_cast<const long long*>(&v);
        long long* d = reinterpret_cast<long long*>(dst);
        for (size_t k = 0; k < sizeof(T) / 8; ++k) _mm_stream_si64(d + k, s[k]);
    } else {
        std::memcpy(dst, &v, sizeof(T));
    }
}

// compact slots (pack.cuh) -> the caller's records / features
void decode_records(const rlp::Slot* sl, const uint32_t* par, const rl_component* esc, rl_component* dst, int64_t a,
                    int64_t b) {
    for (int64_t i = a; i < b; ++i) {
        const rlp::Slot o = sl[i];
        rl_component c;
        if (rlp::is_escape(o)) {
            c = esc[o.x];
        } else {
            rlp::decode(o, c.f, c.flags);
            c.parent = par[i];
        }
        stream_store(dst + i, c);
    }
    _mm_sfence();
}

void decode_features(const rlp::Slot* sl, const rl_features* esc, rl_features* dst, int64_t a, int64_t b) {
    for (int64_t i = a; i < b; ++i) {
        const rlp::Slot o = sl[i];
        rl_features f;
        if (rlp::is_escape(o)) {
            f = esc[o.x];
        } else {
            uint32_t fg;
            rlp::decode(o, f, fg);
        }
        stream_store(dst + i, f);
    }
    _mm_sfence();
}

// decode tasks handed to the pool by a stream callback once the slots are in host memory
struct Deferred {
    HostPool* pool;
    int tag;
    std::vector<std::function<void()>> tasks;
};

void CUDART_CB run_deferred(void* p) {
    Deferred* d = static_cast<Deferred*>(p);
    for (auto& t : d->tasks) d->pool->submit(d->tag, std::move(t));
    d->pool->release(d->tag);
    delete d;
}

size_t up64(size_t v) { return (v + 63) & ~size_t{63}; }

// debugging aid (env RUNLAB_GPU_DEBUG_TIMELINE): per-chunk stream events and host stamps,
// printed to stderr after the call.  One per host thread (thread_local): a context belongs to
// one thread, so concurrent rl_label_into calls on different contexts never share it.
struct Timeline {
    bool on = std::getenv("RUNLAB_GPU_DEBUG_TIMELINE") != nullptr;
    int chunk = 0;
    cudaEvent_t start = nullptr;
    std::chrono::steady_clock::time_point t0;
    std::vector<std::array<cudaEvent_t, 10>> ev;
    std::vector<std::array<double, 5>> host;
    void begin(cudaStream_t s, int nch) {
        if (!on) return;
        for (auto& a : ev)
            for (auto e : a)
                if (e) cudaEventDestroy(e);
        ev.assign(nch, {});
        host.assign(nch, {0, 0, 0, 0, 0});
        if (!start) cudaEventCreate(&start);
        cudaEventRecord(start, s);
        cudaEventSynchronize(start);
        t0 = std::chrono::steady_clock::now();
    }
    void mark(int k, cudaStream_t s) {
        if (!on || chunk >= (int)ev.size()) return;
        cudaEventCreate(&ev[chunk][k]);
        cudaEventRecord(ev[chunk][k], s);
    }
    void hmark(int c, int k) {
        if (!on || c >= (int)host.size()) return;
        host[c][k] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    void print() {
        if (!on) return;
        std::fprintf(stderr, "chunk  h2d0  h2d1  kern1  fill1 | out0  out1 | post0 post1 enq0 (ms)\n");
        for (size_t c = 0; c < ev.size(); ++c) {
            std::fprintf(stderr, "%3zu ", c);
            for (int k = 0; k < 10; ++k) {
                float ms = -1;
                if (ev[c][k]) cudaEventElapsedTime(&ms, start, ev[c][k]);
                std::fprintf(stderr, " %6.3f%s", ms, k == 3 ? " |" : "");
            }
            std::fprintf(stderr, " | %6.3f %6.3f %6.3f %6.3f %6.3f\n", host[c][0], host[c][1], host[c][2], host[c][3], host[c][4]);
        }
    }
};
thread_local Timeline tl;

struct IntoState {
    int64_t total = 0;  // components of the chunks posted so far
    int64_t surv = 0;   // post-fill roots of the chunks posted so far
    int64_t d2h = 0;
    bool nospace = false;
};

void copy_fixed_outputs(rl_ctx* c, rl_host_outputs* out, int32_t b0) {
    const Geo& g = c->geo;
    const size_t npx = (size_t)(g.P * g.B), off = (size_t)g.P * b0;
    if (out->filled_image) {
        if (g.ofmt == c->user_ofmt) {
            cudaMemcpyAsync(out->filled_image + (size_t)g.ofbytes * b0, c->ws.filled_img, (size_t)g.ofbytes * g.B,
                            cudaMemcpyDeviceToHost, c->stream);
        } else {  // packed: into the staging buffer, expanded on the host once the chunk is done
            cudaMemcpyAsync(c->h_stage[c->stage], c->ws.filled_img, (size_t)g.ofbytes * g.B, cudaMemcpyDeviceToHost,
                            c->stream);
        }
    }
    if (out->labels && g.label_mode)
        cudaMemcpyAsync(out->labels + off, c->ws.labels, npx * 4, cudaMemcpyDeviceToHost, c->stream);
}

// host expansion of chunk c's packed filled image (after its stream is synchronised)
void expand_filled(rl_ctx* owner, rl_ctx* c, int tag, rl_host_outputs* out, int32_t b0) {
    const Geo& g = c->geo;
    if (!out->filled_image || g.ofmt == c->user_ofmt) return;
    const int64_t rows = (int64_t)g.H * g.B;
    const int parts = (int)std::min<int64_t>(std::max<int64_t>(1, rows / 256), 8);
    for (int k = 0; k < parts; ++k) {
        const int64_t r0 = rows * k / parts, r1 = rows * (k + 1) / parts;
        const uint8_t* src = c->h_stage[c->stage] + r0 * g.orowb;
        uint8_t* dst = out->filled_image + (size_t)g.P * b0 + r0 * g.W;
        const int32_t rowb = g.orowb, w = g.W;
        owner->pool->submit(tag, [=] { expand_p4_rows(src, r1 - r0, rowb, w, dst); });
    }
}

// u8 images [n] -> P4 rows in c's input staging buffer sb, by the host pool (tasks under `tag`,
// ahead of the queued output work)
int submit_pack(rl_ctx* c, int sb, const uint8_t* pixels, int32_t w, int32_t h, int32_t n, HostPool* pool, int tag) {
    const size_t npx = (size_t)image_bytes(w, h, RL_PIXELS_P4) * n;
    if (c->h_istage_n[sb] < npx) {
        if (c->h_istage[sb]) cudaFreeHost(c->h_istage[sb]);
        c->h_istage[sb] = nullptr;
        c->h_istage_n[sb] = 0;
        if (cudaMallocHost(&c->h_istage[sb], npx) != cudaSuccess) return set_err(c, RL_ENOMEM, "pinned alloc failed");
        c->h_istage_n[sb] = npx;
    }
    if (tag < 0) return RL_OK;  // the caller submits the packing itself
    const int64_t rows = (int64_t)h * n;
    const int32_t rowb = (w + 7) / 8;
    const int parts = (int)std::min<int64_t>(std::max<int64_t>(1, rows / 128), 12);
    uint8_t* dst = c->h_istage[sb];
    for (int k = 0; k < parts; ++k) {
        const int64_t r0 = rows * k / parts, r1 = rows * (k + 1) / parts;
        pool->submit(tag, [=] { pack_rows_p4(pixels + r0 * w, r1 - r0, w, dst + r0 * rowb, rowb); }, true);
    }
    return RL_OK;
}

constexpr int in_tag(int kid, int sb) { return 2 * rl_ctx::MAXKIDS + 2 * kid + sb; }
constexpr int SYNC_IN_TAG = 4 * rl_ctx::MAXKIDS;

// H2D of images [b0, b0 + n), the pipeline, and the D2H of the outputs whose size is fixed.
// `pack_in`: u8 input crosses PCIe as P4 bits from c's input staging buffer c->stage, packed
// there by the host pool -- already (`prepacked`, the caller waited for it) or here.
int into_enqueue(rl_ctx* c, const uint8_t* pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg,
                 rl_host_outputs* out, int32_t b0, int32_t fmt, bool packed_out, int pack, HostPool* pool,
                 bool pack_in, bool prepacked) {
    const int32_t dfmt = pack_in ? RL_PIXELS_P4 : fmt;
    const size_t npx = (size_t)image_bytes(w, h, dfmt) * n;
    if (!ensure(c->pix, npx)) return set_err(c, RL_ENOMEM, "device allocation failed");
    if (!c->in_stream) {
        if (cudaStreamCreateWithFlags(&c->in_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->in_done, cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(c, cudaGetLastError(), "copy stream");
    }
    const uint8_t* src = pixels;
    // one large image packed here: in row pieces, each copied as soon as it is packed (the pool
    // packs the next pieces meanwhile); tags of the kids' input buffers are free in this mode
    constexpr int NPIECE = 2 * rl_ctx::MAXKIDS;
    const bool pieces = pack_in && !prepacked && (int64_t)h * n >= 8 * NPIECE;
    if (pack_in) {
        if (pieces) {
            if (const int rc = submit_pack(c, c->stage, pixels, w, h, n, pool, -1)) return rc;  // staging only
            const int64_t rows = (int64_t)h * n;
            const int32_t rowb = (w + 7) / 8;
            uint8_t* dst = c->h_istage[c->stage];
            for (int k = 0; k < NPIECE; ++k) {
                const int64_t p0 = rows * k / NPIECE, p1 = rows * (k + 1) / NPIECE;
                const int parts = 3;  // the pool works on several pieces at once
                for (int q = 0; q < parts; ++q) {
                    const int64_t r0 = p0 + (p1 - p0) * q / parts, r1 = p0 + (p1 - p0) * (q + 1) / parts;
                    pool->submit(in_tag(0, 0) + k,
                                 [=] { pack_rows_p4(pixels + r0 * w, r1 - r0, w, dst + r0 * rowb, rowb); });
                }
            }
        } else if (!prepacked) {
            if (const int rc = submit_pack(c, c->stage, pixels, w, h, n, pool, SYNC_IN_TAG)) return rc;
            pool->wait(SYNC_IN_TAG);
        }
        src = c->h_istage[c->stage];
    }
    tl.hmark(tl.chunk, 3);
    tl.mark(0, c->in_stream);
    cudaError_t e = cudaSuccess;
    if (pieces) {
        const int64_t rows = (int64_t)h * n;
        const int32_t rowb = (w + 7) / 8;
        for (int k = 0; k < NPIECE && e == cudaSuccess; ++k) {
            const int64_t p0 = rows * k / NPIECE, p1 = rows * (k + 1) / NPIECE;
            pool->wait(in_tag(0, 0) + k);
            e = cudaMemcpyAsync(P<uint8_t>(c->pix) + p0 * rowb, src + p0 * rowb, (size_t)(p1 - p0) * rowb,
                                cudaMemcpyHostToDevice, c->in_stream);
        }
    } else {
        e = cudaMemcpyAsync(c->pix.p, src, npx, cudaMemcpyHostToDevice, c->in_stream);
    }
    if (e != cudaSuccess) return cuda_fail(c, e, "copy in");
    cudaEventRecord(c->in_done, c->in_stream);
    cudaStreamWaitEvent(c->stream, c->in_done, 0);
    tl.mark(1, c->in_stream);
    tl.hmark(tl.chunk, 4);
    if (c->out_done) cudaStreamWaitEvent(c->stream, c->out_done, 0);  // last chunk's table copies
    c->user_ofmt = fmt;
    c->want_compact = out->filled && out->filled_layout == 1;
    c->want_pack = pack;
    const bool packed = packed_out && out->filled_image && fmt == RL_PIXELS_U8;
    // the filled image: P4 bits expanded on the host, else the caller's format (also when the
    // input crossed packed)
    c->force_ofmt = packed ? RL_PIXELS_P4 : (dfmt != fmt ? fmt : -1);
    if (packed) {
        const size_t need = (size_t)image_bytes(w, h, RL_PIXELS_P4) * n;
        const int sb = c->stage;
        if (c->h_stage_n[sb] < need) {
            if (c->h_stage[sb]) cudaFreeHost(c->h_stage[sb]);
            c->h_stage[sb] = nullptr;
            c->h_stage_n[sb] = 0;
            if (cudaMallocHost(&c->h_stage[sb], need) != cudaSuccess) return set_err(c, RL_ENOMEM, "pinned alloc failed");
            c->h_stage_n[sb] = need;
        }
    }
    const int rc = enqueue(c, P<uint8_t>(c->pix), w, h, n, cfg, dfmt);
    c->force_ofmt = -1;  // finish() re-runs with the geometry of this call (kept in c->geo)
    if (rc) return rc;
    tl.mark(2, c->stream);
    copy_fixed_outputs(c, out, b0);
    tl.mark(3, c->stream);
    return RL_OK;
}

// after finish(c): per-image summaries and the component outputs of c's chunk (first image b0)
int into_post(rl_ctx* c, rl_host_outputs* out, int32_t b0, IntoState& st, HostPool* pool, int tag) {
    const Geo& g = c->geo;
    const int B = g.B;
    if (c->reran) {  // the pipeline re-ran after the first copies
        copy_fixed_outputs(c, out, b0);
        if (g.ofmt != c->user_ofmt) cudaStreamSynchronize(c->stream);  // the staging buffer is expanded next
    }
    if (out->filled_image) st.d2h += g.ofbytes * B;
    if (out->labels && g.label_mode) st.d2h += g.P * B * 4;
    const int64_t* s = c->h_summ;
    const int64_t total = s[4 * B];
    int64_t surv = 0;
    for (int b = 0; b < B; ++b) surv += s[4 * b + 3];
    st.d2h += (int64_t)(B + 1) * 32;
    if (out->summary)
        for (int b = 0; b < B; ++b) {
            const int64_t cp = s[4 * b + 1], fg = s[4 * b + 2];
            int64_t* o = out->summary + 5 * (int64_t)(b0 + b);
            o[0] = cp;
            o[1] = fg;
            o[2] = cp - 1 - fg;
            o[3] = fg - (cp - 1 - fg);
            o[4] = s[4 * b + 3];
        }
    if (out->comp_offset) {
        for (int b = 0; b < B; ++b) out->comp_offset[b0 + b] = st.total + s[4 * b];
        out->comp_offset[b0 + B] = st.total + total;
    }
    const bool want_comps = out->comps || out->top || out->filled;
    if (want_comps && st.total + total > out->comp_capacity) st.nospace = true;
    const int pack = c->want_pack & (c->want_compact ? 3 : 1);
    if (!c->out_stream) {
        if (cudaStreamCreateWithFlags(&c->out_stream, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&c->out_done, cudaEventDisableTiming) != cudaSuccess)
            return cuda_fail(c, cudaGetLastError(), "copy stream");
    }
    // the pipeline's stream is synchronised (finish), so the copies may start right away
    cudaStream_t cs = c->out_stream;
    tl.mark(4, cs);
    Deferred* dec = nullptr;
    if (!st.nospace && pack) {
        // compact slots into pinned staging; host threads decode them once the copies land
        const int64_t nesc = (pack & 1) ? s[4 * (B + 1)] : 0, fesc = (pack & 2) ? s[4 * (B + 1) + 1] : 0;
        const int64_t nrec = (pack & 1) ? total : 0, nfs = (pack & 2) ? surv : 0;
        const size_t o_fs = up64(16 * (size_t)nrec), o_par = o_fs + up64(16 * (size_t)nfs);
        const size_t o_esc = o_par + up64(4 * (size_t)nrec), o_fesc = o_esc + up64(sizeof(rl_component) * nesc);
        const size_t need = o_fesc + sizeof(rl_features) * fesc + 64;
        const int sb = c->stage;
        if (c->h_rstage_n[sb] < need) {
            if (c->h_rstage[sb]) cudaFreeHost(c->h_rstage[sb]);
            c->h_rstage[sb] = nullptr;
            c->h_rstage_n[sb] = 0;
            const cudaError_t ae = cudaMallocHost(&c->h_rstage[sb], need + need / 4);
            if (ae != cudaSuccess)
                return set_err(c, RL_ENOMEM, "pinned alloc failed");
            c->h_rstage_n[sb] = need + need / 4;
        }
        uint8_t* h = c->h_rstage[sb];
        Deferred* d = new Deferred{pool, tag, {}};
        const int64_t t0 = st.total, s0 = st.surv;
        if (nrec) {
            cudaMemcpyAsync(h + o_par, c->pkpar.p, 4 * (size_t)nrec, cudaMemcpyDeviceToHost, cs);
            tl.mark(7, cs);
            cudaMemcpyAsync(h, c->pk.p, 16 * (size_t)nrec, cudaMemcpyDeviceToHost, cs);
            tl.mark(6, cs);
            if (nesc) cudaMemcpyAsync(h + o_esc, c->pkesc.p, sizeof(rl_component) * nesc, cudaMemcpyDeviceToHost, cs);
            st.d2h += 20 * nrec + (int64_t)sizeof(rl_component) * nesc;
            const rlp::Slot* sl = reinterpret_cast<const rlp::Slot*>(h);
            const uint32_t* par = reinterpret_cast<const uint32_t*>(h + o_par);
            const rl_component* esc = reinterpret_cast<const rl_component*>(h + o_esc);
            rl_component* dst = out->comps + t0;
            const int parts = (int)std::min<int64_t>(8, std::max<int64_t>(1, nrec / 65536));
            for (int k = 0; k < parts; ++k) {
                const int64_t a = nrec * k / parts, e = nrec * (k + 1) / parts;
                d->tasks.emplace_back([=] { decode_records(sl, par, esc, dst, a, e); });
            }
        }
        if (nfs) {
            cudaMemcpyAsync(h + o_fs, c->fpk.p, 16 * (size_t)nfs, cudaMemcpyDeviceToHost, cs);
            if (fesc) cudaMemcpyAsync(h + o_fesc, c->fcomp.p, sizeof(rl_features) * fesc, cudaMemcpyDeviceToHost, cs);
            tl.mark(8, cs);
            st.d2h += 16 * nfs + (int64_t)sizeof(rl_features) * fesc;
            const rlp::Slot* sl = reinterpret_cast<const rlp::Slot*>(h + o_fs);
            const rl_features* esc = reinterpret_cast<const rl_features*>(h + o_fesc);
            rl_features* dst = out->filled + s0;
            const int parts = (int)std::min<int64_t>(4, std::max<int64_t>(1, nfs / 65536));
            for (int k = 0; k < parts; ++k) {
                const int64_t a = nfs * k / parts, e = nfs * (k + 1) / parts;
                d->tasks.emplace_back([=] { decode_features(sl, esc, dst, a, e); });
            }
        }
        dec = d;
    }
    if (!st.nospace) {
        if (out->comps && !(pack & 1)) {
            cudaMemcpyAsync(out->comps + st.total, c->ws.comps, sizeof(rl_component) * total, cudaMemcpyDeviceToHost, cs);
            st.d2h += (int64_t)sizeof(rl_component) * total;
        }
        if (out->top) {
            cudaMemcpyAsync(out->top + st.total, c->ws.top, 4 * total, cudaMemcpyDeviceToHost, cs);
            tl.mark(9, cs);
            st.d2h += 4 * total;
        }
        if (pack & 2) {
        } else if (out->filled && out->filled_layout == 0) {
            cudaMemcpyAsync(out->filled + st.total, c->ws.filled, sizeof(rl_features) * total, cudaMemcpyDeviceToHost, cs);
            st.d2h += (int64_t)sizeof(rl_features) * total;
        } else if (out->filled) {
            cudaMemcpyAsync(out->filled + st.surv, c->fcomp.p, sizeof(rl_features) * surv, cudaMemcpyDeviceToHost, cs);
            st.d2h += (int64_t)sizeof(rl_features) * surv;
        }
    }
    cudaEventRecord(c->out_done, cs);
    tl.mark(5, cs);
    if (dec) {  // after out_done: the next pipeline on this workspace does not wait for the callback
        pool->reserve(tag);
        if (cudaLaunchHostFunc(cs, run_deferred, dec) != cudaSuccess) {
            cudaGetLastError();
            cudaStreamSynchronize(cs);
            run_deferred(dec);
        }
    }
    st.total += total;
    st.surv += surv;
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? RL_OK : cuda_fail(c, e, "copy out");
}

int into_sync(rl_ctx* c) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess && c->out_stream) e = cudaStreamSynchronize(c->out_stream);
    return e == cudaSuccess ? RL_OK : cuda_fail(c, e, "copy out");
}

}  // namespace

extern "C" {

int rl_label_into_fmt(rl_ctx* ctx, const uint8_t* pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg,
                      int32_t fmt, rl_host_outputs* out) {
    if (!out) return RL_EINVAL;
    out->comps_needed = 0;
    out->h2d_bytes = out->d2h_bytes = 0;
    if (out->filled_layout != 0 && out->filled_layout != 1) return set_err(ctx, RL_EINVAL, "unknown filled_layout");
    if (fmt != RL_PIXELS_U8 && fmt != RL_PIXELS_P4) return set_err(ctx, RL_EINVAL, "unknown pixel format");
    int rc = check_args(ctx, w, h, n, cfg);
    if (rc) return rc;
    cudaSetDevice(ctx->device);
    const int64_t P = (int64_t)w * h;
    // whole images per chunk, ~32 Mpx by default (pipelines of that size are graph-replayed)
    const int32_t per = (int32_t)std::min<int64_t>(n, std::max<int64_t>(1, ctx->chunk_px / P));
    const int32_t nch = (n + per - 1) / per;
    // With several chunks, a byte-per-pixel filled image crosses PCIe as P4 bits and is expanded
    // by host threads, and component records and survivors' features cross as compact slots
    // (pack.cuh), decoded by host threads while later chunks are in flight.  A single chunk has
    // nothing to overlap the host work with: plain copies are faster there (measured: config 3,
    // one 16.7 Mpx image, 7.3 -> 16.0 Gpx/s end to end; config 1, 1.25 -> 2.95).
    const bool multi = nch > 1;
    // ... except a single image so large that its byte-per-pixel copies dominate (config 5: 1 GB
    // each way over PCIe, 39 of 46 ms; >= 8 Mpx by default): its input is packed to P4 by the
    // host pool in row pieces, each copied as soon as it is packed, and its filled image crosses
    // as P4 and is expanded while the component tables cross (8x fewer bytes on the link:
    // config 5 46 -> 25.6 ms, config 3 1.38 -> 0.97 ms)
    const bool big1 = !multi && P * n >= ctx->big_single_px;
    const bool packed = (multi || big1) && ctx->packed_d2h && out->filled_image && fmt == RL_PIXELS_U8;
    const int pack = multi && ctx->packed_recs ? ((out->comps ? 1 : 0) | (out->filled && out->filled_layout == 1 ? 2 : 0)) : 0;
    // u8 input crosses PCIe as P4 bits packed by the host pool one chunk ahead (a single chunk
    // would wait for its packing: plain copy)
    const bool pack_in = (multi || big1) && fmt == RL_PIXELS_U8 && ctx->packed_h2d;
    const bool staged = packed || pack || pack_in;
    if (staged && !ctx->pool) {
        const int hw = (int)std::thread::hardware_concurrency();
        const int nt = ctx->host_threads > 0 ? ctx->host_threads : std::max(2, std::min(hw > 0 ? hw : 4, 12));
        ctx->pool = new (std::nothrow) HostPool(nt);
        if (!ctx->pool) return set_err(ctx, RL_ENOMEM, "host thread pool");
    }
    IntoState st;
    tl.begin(ctx->stream, nch);
    if (nch == 1) {
        rc = into_enqueue(ctx, pixels, w, h, n, cfg, out, 0, fmt, packed, pack, ctx->pool, pack_in, false);
        if (!rc) rc = finish(ctx);
        // the filled image's copy is done with the pipeline (finish), so host threads expand it
        // while the component tables are still crossing (unless the pipeline re-ran: then
        // into_post copies it again)
        const bool early = !rc && packed && !ctx->reran;
        if (early) expand_filled(ctx, ctx, 0, out, 0);
        if (!rc) rc = into_post(ctx, out, 0, st, ctx->pool, 0);
        if (!rc) rc = into_sync(ctx);
        if (!rc && packed && !early) expand_filled(ctx, ctx, 0, out, 0);
        // host tasks of this call end before it returns (after a failed copy only if the
        // stream still completes, i.e. its callbacks run)
        if (staged && (!rc || into_sync(ctx) == RL_OK)) ctx->pool->wait(0);
    } else {
        const int NK = ctx->nkids;
        for (int i = 0; i < NK; ++i) {
            rl_ctx*& k = ctx->kids[i];
            if (!k) {
                k = rl_create(ctx->device);
                if (!k) return set_err(ctx, RL_ECUDA, "could not create a pipeline context");
                k->graphs = ctx->graphs;
            }
            k->stage = 1;  // chunk -> staging buffer is the same every call (sizes settle once)
        }
        auto first_image = [&](int32_t c) { return c * per; };
        auto images = [&](int32_t c) { return std::min(per, n - c * per); };
        // chunk c runs on kid c % NKIDS; its component outputs are copied once its summary is
        // in (finish() synchronises the kid's stream, so its packed filled image is in the
        // staging buffer and host threads expand it), before the kid takes chunk c + NKIDS
        auto post = [&](int32_t c) -> int {
            const int kid = c % NK;
            rl_ctx* k = ctx->kids[kid];
            tl.hmark(c, 0);
            int r = finish(k);
            tl.hmark(c, 1);
            if (tl.on && k->reran) std::fprintf(stderr, "chunk %d re-ran (capacity)\n", c);
            tl.chunk = c;
            if (r) return set_err(ctx, r, k->err);
            r = into_post(k, out, first_image(c), st, ctx->pool, 2 * kid + k->stage);
            if (!r && packed) expand_filled(ctx, k, 2 * kid + k->stage, out, first_image(c));
            return r ? set_err(ctx, r, k->err) : RL_OK;
        };
        // chunk c's input, packed into the staging buffer its kid takes next (the buffer's last
        // H2D, chunk c - 2 NK's, completed before post(c - 2 NK) returned)
        auto prepack = [&](int32_t c) -> int {
            const int kid = c % NK;
            rl_ctx* k = ctx->kids[kid];
            const int r = submit_pack(k, k->stage ^ 1, pixels + (size_t)first_image(c) * image_bytes(w, h, fmt), w, h,
                                      images(c), ctx->pool, in_tag(kid, k->stage ^ 1));
            return r ? set_err(ctx, r, k->err) : RL_OK;
        };
        if (pack_in) rc = prepack(0);
        for (int32_t c = 0; c < nch && !rc; ++c) {
            if (c >= NK) rc = post(c - NK);
            if (rc) break;
            const int kid = c % NK;
            rl_ctx* k = ctx->kids[kid];
            if (staged) {  // alternate the kid's staging buffers; wait for the older one's expansion
                k->stage ^= 1;
                ctx->pool->wait(2 * kid + k->stage);
            }
            if (pack_in) {  // this chunk's input is packed; start packing the next one
                ctx->pool->wait(in_tag(kid, k->stage));
                if (c + 1 < nch) rc = prepack(c + 1);
                if (rc) break;
            }
            const int32_t b0 = first_image(c);
            tl.chunk = c;
            tl.hmark(c, 2);
            rc = into_enqueue(k, pixels + (size_t)b0 * image_bytes(w, h, fmt), w, h, images(c), cfg, out, b0, fmt,
                              packed, pack, ctx->pool, pack_in, true);
            if (rc) rc = set_err(ctx, rc, k->err);
        }
        for (int32_t c = std::max(0, nch - NK); c < nch && !rc; ++c) rc = post(c);
        for (int i = 0; i < NK; ++i)
            if (!rc) rc = into_sync(ctx->kids[i]) ? set_err(ctx, RL_ECUDA, ctx->kids[i]->err) : RL_OK;
        bool drained = true;
        if (rc)
            for (int i = 0; i < NK; ++i) drained = into_sync(ctx->kids[i]) == RL_OK && drained;
        if (staged && drained)
            for (int kid = 0; kid < NK; ++kid)
                for (int sb = 0; sb < 2; ++sb) {
                    ctx->pool->wait(2 * kid + sb);
                    ctx->pool->wait(in_tag(kid, sb));
                }
    }
    if (rc) return rc;
    tl.print();
    out->comps_needed = st.total;
    out->h2d_bytes = image_bytes(w, h, pack_in ? RL_PIXELS_P4 : fmt) * n;
    out->d2h_bytes = st.d2h;
    if (st.nospace) return set_err(ctx, RL_ENOSPC, "component buffers too small");
    return RL_OK;
}

int rl_label_into(rl_ctx* ctx, const uint8_t* pixels, int32_t w, int32_t h, int32_t n, const rl_config* cfg,
                  rl_host_outputs* out) {
    return rl_label_into_fmt(ctx, pixels, w, h, n, cfg, RL_PIXELS_U8, out);
}

}  // extern "C"
