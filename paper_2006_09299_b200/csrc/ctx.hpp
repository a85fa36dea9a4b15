// ctx.hpp -- the host-side context (rl_ctx) and helpers shared by api.cu (single-GPU calls)
// and strips.cu (one image split into horizontal strips across ranks).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "common.cuh"
#include "runlab_gpu.h"

namespace rlg {
size_t analyze_smem();
size_t emit_smem();
cudaError_t configure_kernels();
// scan.cu: out[i] = init + sum(in[0 .. i)); `state`: scan_state_bytes(n) bytes of device memory
size_t scan_state_bytes(int64_t n);
void launch_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t init, void* state, cudaStream_t s,
                 bool zeroed = false);
void launch_analyze(const uint8_t* pix, const Geo& g, const Ws& ws, cudaStream_t s);
bool direct_call(const Geo& g);  // every tile straight to class M (one analyze and one emit launch less)
void launch_seam_rows(const Geo& g, const Ws& ws, int32_t s0, int32_t ns, cudaStream_t s, int sms);
void launch_seam_cols(const Geo& g, const Ws& ws, cudaStream_t s, int sms);
void launch_resolve(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint);
void launch_reps(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint);
void launch_cids(const Geo& g, const Ws& ws, cudaStream_t s, int sms);
void launch_tree(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint);
void launch_tree_parts(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint);
void launch_fold(const Geo& g, const Ws& ws, cudaStream_t s, int sms, int64_t nodes_hint);
void launch_emit(const Geo& g, const Ws& ws, cudaStream_t s, cudaStream_t s2 = nullptr, cudaEvent_t fork = nullptr,
                 cudaEvent_t join = nullptr);
void launch_surv_flags(const uint32_t* top, const uint64_t* cbase, int32_t B, uint64_t total, uint32_t* flag,
                       cudaStream_t s, int sms);
void launch_compact_filled(const Acc* filled, const uint32_t* flag, const uint32_t* rank, const uint64_t* total_p,
                           uint64_t cap, Acc* out, cudaStream_t s, int sms);
void launch_pack_comps(const rl_component* comps, const uint64_t* total_p, uint64_t cap, void* slots, uint32_t* parent,
                       rl_component* esc, int64_t* nesc, cudaStream_t s, int sms);
void launch_pack_filled(const Acc* filled, const uint32_t* flag, const uint32_t* rank, const uint64_t* total_p,
                        uint64_t cap, void* slots, Acc* esc, int64_t* nesc, cudaStream_t s, int sms);
void launch_remap(uint32_t* labels, int64_t P, int32_t B, const uint32_t* rank, const uint64_t* cbase, uint64_t cap,
                  cudaStream_t s, int sms);
}  // namespace rlg


namespace rlh {
using namespace rlg;

struct StripState;  // strips.cu
struct HostPool;    // api.cu

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// A table base moved back by n elements, for tables that hold only a window [n, ...) of a
// numbering the kernels use whole (strip mode).  Integer arithmetic: the moved pointer itself is
// never dereferenced outside the window.
template <class T>
inline T* shift_base(T* p, int64_t n) {
    return reinterpret_cast<T*>(reinterpret_cast<uintptr_t>(p) - (uintptr_t)(n * (int64_t)sizeof(T)));
}

// Everything a captured pipeline depends on (compared bytewise before a replay).
struct GraphKey {
    Geo g;
    Ws ws;
    rl_config cfg;
    const void* pix;
    cudaStream_t stream;
    const void* summ;
    const void* rank;
    const void* flag;
    const void* fcomp;
    uint64_t cap_comps;
    int compact;
    int pack;  // bit 0: records, bit 1: survivors' features
    const void* pk[4];
};


}  // namespace rlh

struct rl_ctx {
    using DevBuf = rlh::DevBuf;
    using GraphKey = rlh::GraphKey;
    using Geo = rlg::Geo;
    using Ws = rlg::Ws;
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    // the vertical seams run beside the horizontal ones (independent unions): a forked stream
    cudaStream_t seam_stream = nullptr;
    cudaEvent_t seam_fork = nullptr, seam_join = nullptr;
    std::string err;
    static constexpr int NEV = 5;  // start, after analyze, after merge, after emit, end
    cudaEvent_t ev[NEV] = {};  // events of the current call
    static constexpr int RING = 64;
    cudaEvent_t ring[RING][NEV] = {};
    int64_t calls = 0;
    // workspace
    DevBuf bits, tbase, tnb, perim, uf, nkey, nmin, nacc, nrec, nrep, ninfo, nrootcid, nparent, nanccid;
    DevBuf cnt, off, counters, img_fg, img_surv, comps, top, filled, filled_img, labels, pix;
    DevBuf cub_tmp, cbase, summ, rank, flag, ovf, ovf2, thdr, tmap, rstore, rused, fcomp;
    uint32_t cap_nodes = 0;
    uint64_t cap_comps = 0;
    uint64_t cap_rstore = 0;
    // pinned host mirror of the summary
    int64_t* h_summ = nullptr;
    size_t h_summ_n = 0;
    // last call
    Geo geo{};
    Ws ws{};
    rl_config cfg{};
    const uint8_t* last_pix = nullptr;
    int launches = 0;
    bool have_result = false;
    bool reran = false;  // finish() had to grow a capacity and re-run
    // CUDA graph of the last small pipeline
    bool graphs = true;
    // pipelines are captured into a CUDA graph and replayed (config 2, 440 Mpx: 2.367 -> 2.339 ms
    // per step against eager launches); env RUNLAB_GPU_GRAPH_MPX caps the workload size
    double graph_max_px = 1e18;
    int64_t permute = 0;  // env RUNLAB_GPU_PERMUTE (testing aid, Geo::permute)
    bool used_graph = false;
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey{};
    cudaEvent_t gev[NEV] = {};
    // post-fill features of the survivors compacted into `fcomp` (rl_label_into layout 1)
    bool want_compact = false;
    int64_t chunk_px = 32ll << 20;  // rl_label_into: pixels per chunk (env RUNLAB_GPU_CHUNK_PX)
    int64_t big_single_px = 8ll << 20;  // rl_label_into: one chunk this large crosses PCIe packed (env RUNLAB_GPU_BIG_PX; measured: cfg3 16.7 Mpx 12 -> 17 Gpx/s, cfg1 1 Mpx slower)
    // rl_label_into pipelines large batches through these (own workspace and stream each)
    static constexpr int MAXKIDS = 8;
    int nkids = 3;  // env RUNLAB_GPU_KIDS
    rl_ctx* kids[MAXKIDS] = {};
    // rl_label_device splits a large batch into interleaved sub-batches (every split-th image)
    // run as concurrent pipelines, each on its own context/stream, so that one sub-batch's
    // latency-bound merge kernels overlap another's tile passes (config 2, 3 pipelines: -3%)
    static constexpr int MAXSPLIT = 4;
    int split = 3;          // env RUNLAB_GPU_SPLIT, rl_set_pipelines; <= 1: one pipeline
    double split_min_px = 64.0 * 1024 * 1024;  // env RUNLAB_GPU_SPLIT_MPX
    int split_active = 0;   // pipelines of the last rl_label_device call (0: it ran here)
    rl_ctx* splits[MAXSPLIT] = {};
    cudaEvent_t split_fork = nullptr, split_join[MAXSPLIT] = {};
    // set on a split pipeline's context: its image b is the caller's image (k + stride_mult * b),
    // and its hole-filled image goes straight into the caller's buffer at that stride
    int stride_mult = 1;
    uint8_t* ext_filled = nullptr;
    // per-launch timing for tuning (env RUNLAB_GPU_KTIMES; eager launches only)
    bool ktimes = false;
    cudaEvent_t kev[24] = {};
    int nkev = 0;
    // rl_label_into: the filled image crosses PCIe as P4 bits (8x fewer bytes) into this pinned
    // staging buffer and host threads expand it to bytes (env RUNLAB_GPU_NO_PACKED_D2H: off)
    bool packed_d2h = true;
    int32_t force_ofmt = -1;  // output format of the filled image for the next enqueue (-1: input's)
    uint8_t* h_stage[2] = {nullptr, nullptr};  // alternating: one may still be expanding
    size_t h_stage_n[2] = {0, 0};
    int stage = 0;  // the buffer the last enqueue copies into
    rlh::HostPool* pool = nullptr;
    int host_threads = 0;  // pool size (0: min(hardware threads, 12); env RUNLAB_GPU_HOST_THREADS)
    // rl_label_into: component records and survivors' features cross PCIe as compact slots
    // (pack.cuh) into pinned staging, decoded by host threads (env RUNLAB_GPU_NO_PACKED_RECORDS)
    bool packed_recs = true;
    int want_pack = 0;           // bit 0: records, bit 1: survivors' features (next enqueue)
    DevBuf pk, pkpar, pkesc, fpk;  // record slots, parents, escaped records, feature slots
    uint8_t* h_rstage[2] = {nullptr, nullptr};
    size_t h_rstage_n[2] = {0, 0};
    // rl_label_into: byte-per-pixel input packed to P4 bits by the host pool (AVX-512, one chunk
    // ahead of the H2D) before the copy: 8x fewer bytes on the link; the host reads the input
    // instead of the DMA engine (env RUNLAB_GPU_PACKED_H2D=0: plain u8 copies)
    bool packed_h2d = true;
    uint8_t* h_istage[2] = {nullptr, nullptr};
    size_t h_istage_n[2] = {0, 0};
    int32_t user_ofmt = 0;
    // rl_label_into: component-table copies of a chunk run on their own stream so that the next
    // chunk's H2D copy does not queue behind them; the next pipeline waits for out_done
    cudaStream_t out_stream = nullptr;
    cudaEvent_t out_done = nullptr;
    // and the H2D copy on a stream of its own: a stream that copies in both directions shares
    // one copy-engine queue with the D2H copies of other streams (measured: tools/copy_bench3.cu)
    cudaStream_t in_stream = nullptr;
    cudaEvent_t in_done = nullptr;
    // strip mode (strips.cu)
    DevBuf nleft, scount, ncut, nfold, xnode, gtab, ftab;
    DevBuf xrec, xgath, xred;  // rl_label_strips: own record, gathered records, reduction staging
    uint8_t* h_strip = nullptr;  // pinned staging of the strip phases' small host<->device transfers
    size_t h_strip_n = 0;
    rlh::StripState* strip = nullptr;
};

namespace rlh {
using namespace rlg;
int enqueue_seams(rl_ctx* ctx, const Geo& g, const Ws& ws, cudaStream_t s);
int set_err(rl_ctx* c, int code, const std::string& msg);
int cuda_fail(rl_ctx* c, cudaError_t e, const char* what);
bool ensure(DevBuf& b, size_t bytes);
template <class T>
T* P(DevBuf& b) {
    return static_cast<T*>(b.p);
}
int check_args(rl_ctx* ctx, int32_t w, int32_t h, int32_t n, const rl_config* cfg);
// Geometry of a batch of n w x h images (all tile rows, no strip offset).
Geo make_geo(int32_t w, int32_t h, int32_t n, const rl_config* cfg, const void* dpix, int32_t fmt = 0);
void set_output_format(Geo& g, int32_t ofmt);
// Grow the workspace for geometry g and fill `ws`; `scan_tmp` = CUB temp bytes of the cnt scan.
// `out_px` = pixels of the label image buffer; the filled image takes g.fbytes per image
// (scaled to out_px / P images).
int prepare_ws(rl_ctx* ctx, const Geo& g, const rl_config* cfg, Ws& ws, size_t& scan_tmp, int64_t out_px);
void strip_free(rl_ctx* c);
int enqueue(rl_ctx* ctx, const uint8_t* dpix, int32_t W, int32_t H, int32_t B, const rl_config* cfg, int32_t fmt);
int finish(rl_ctx* ctx);  // wait for the last enqueue; grow capacities and re-run on overflow
int64_t image_bytes(int32_t w, int32_t h, int32_t fmt);
void pool_free(rl_ctx* c);
}  // namespace rlh
