/*
 * runlab_gpu.h -- C ABI of the B200 (sm_100a) labeling/analysis path.
 *
 * Drop-in boundary for the reference's C++ entry points (paths relative to
 * /root/reference/proj/include/runlab/):
 *
 *   rl_label()          replaces  label_image        labeling.hpp:336-339
 *                        and      timed_label_image  labeling.hpp:343-348 (phase_ms below)
 *                        and the filled image of     binarize_labels    labeling.hpp:354-360
 *                        (as used by `runlab fill`, tools/runlab.cpp:128-137)
 *   rl_label_device()   the same pipeline on device-resident batches (no host copies)
 *   rl_result fields    feed components/holes/adjacency_tree/euler_number
 *                                                    analysis.hpp:23-79
 *
 * POD types only (no C++/torch types), so the reference (namespace runlab) and this
 * library can be linked into one test binary without an ODR clash.  The C++ drop-in
 * header include/runlab_gpu.hpp rebuilds runlab::LabelingResult from it.
 *
 * Canonical numbering: every component (foreground or background) gets the rank of its
 * raster-first pixel; id 0 is the exterior background.  This equals the ascending order
 * of the reference's root labels (tables.hpp:68-76) and the oracle's ids
 * (oracle.hpp:20-23).
 */
#ifndef RUNLAB_GPU_H
#define RUNLAB_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (mapped to the reference's exception types by the C++ drop-in). */
#define RL_OK 0
#define RL_EINVAL 1    /* std::invalid_argument (labeling.hpp:271-273) */
#define RL_ELOGIC 2    /* std::logic_error */
#define RL_EOVERFLOW 3 /* std::overflow_error (features.hpp:37-39) */
#define RL_ECUDA 4     /* std::runtime_error */
#define RL_ENOMEM 5    /* std::bad_alloc */
#define RL_EINTERNAL 6 /* std::runtime_error (invariant violated on device) */
#define RL_ENOSPC 7    /* caller-provided output buffer too small (see comps_needed) */
#define RL_EFORMAT 8   /* runlab::PbmParseError (io.hpp:16-23): byte offset in rl_pbm_info */

/* pixel formats of the input batch and of the hole-filled image */
#define RL_PIXELS_U8 0 /* one byte (0/1) per pixel, row-major (BinaryImage, image.hpp:14-43) */
#define RL_PIXELS_P4 1 /* PBM P4 raster: rows of MSB-first bits padded to whole bytes (io.hpp:78-154) */

/* types.hpp:18-21 */
#define RL_FG8_BG4 0
#define RL_FG4_BG8 1

/* labeling.hpp:20-27 LabelingConfig */
typedef struct rl_config {
    int32_t connectivity; /* RL_FG8_BG4 (default) or RL_FG4_BG8 */
    int32_t fill_holes;
    int32_t compute_features;
    int32_t relabel;
    int32_t densify_labels;
    int32_t compute_euler;
} rl_config;

/* features.hpp:14-25 FeatureAccumulator (40 bytes; empty = s 0, bbox INT32_MAX/MIN) */
typedef struct rl_features {
    int64_t s, sx, sy;
    int32_t row_min, row_max, col_min, col_max;
} rl_features;

/* One pre-fill component (48 bytes). */
typedef struct rl_component {
    rl_features f;
    uint32_t parent; /* canonical id of the surrounding component; UINT32_MAX for id 0 */
    uint32_t flags;  /* bit 0: foreground */
} rl_component;

/* Per-phase device times of the last call (CUDA events), cf. StepTimes labeling.hpp:253-259. */
typedef struct rl_times {
    float analyze_ms;  /* K1a tile scan: segments + tile union-find + border tables */
    float merge_ms;    /* cross-tile union, closure, canonical ids, tree, fill fold */
    float emit_ms;     /* K1b second tile pass: records, filled image, label image (relabel
                          of labeling.hpp:224-250 is fused into this pass) */
    float total_ms;
    float relabel_ms;  /* after the emit pass: densified label ids (labeling.hpp:231-236) and
                          survivor compaction; 0 when neither is requested */
} rl_times;

/* Result of one call over n_images images of identical size, library-allocated
 * (free with rl_result_free).  Per-image arrays are concatenated; image i owns
 * [comp_offset[i], comp_offset[i+1]) of comps/top/filled and pixels
 * [i*w*h, (i+1)*w*h) of filled_image/labels. */
typedef struct rl_result {
    int32_t width, height, n_images;
    int64_t* n_components; /* [n_images] C_pre, exterior included */
    int64_t* n_fg;         /* [n_images] foreground components, pre-fill */
    int64_t* n_holes;      /* [n_images] holes, pre-fill */
    int64_t* euler;        /* [n_images] n_fg - n_holes */
    int64_t* n_survivors;  /* [n_images] C_post: components left after hole filling */
    int64_t* comp_offset;  /* [n_images + 1] */
    rl_component* comps;   /* pre-fill records, canonical order */
    uint32_t* top;         /* post-fill root (depth-1 ancestor) of every component */
    rl_features* filled;   /* post-fill features; meaningful where top[i] == i */
    uint8_t* filled_image; /* hole-filled image (binarize_labels after fill) */
    uint32_t* labels;      /* per-pixel label image when cfg.relabel, else NULL */
    rl_times times;
} rl_result;

typedef struct rl_ctx rl_ctx;

/* One context = one device + one CUDA stream + workspace. One context per host thread. */
rl_ctx* rl_create(int device);
void rl_destroy(rl_ctx* ctx);
const char* rl_last_error(const rl_ctx* ctx);

/* Host-buffer entry point (the drop-in): copies the images in, runs the pipeline, copies
 * every requested output back.  pixels: n_images * height * width bytes, values 0/1. */
int rl_label(rl_ctx* ctx, const uint8_t* pixels, int32_t width, int32_t height,
             int32_t n_images, const rl_config* cfg, rl_result* out);
void rl_result_free(rl_result* r);

/* Device-resident entry point: d_pixels is a device pointer; the pipeline is enqueued on
 * the context stream and outputs stay in the context's device buffers (see rl_device_*).
 * Returns after enqueueing; call rl_sync() before reading.  If a capacity estimate was
 * exceeded the call re-runs internally after growing (host sync in that case only). */
int rl_label_device(rl_ctx* ctx, const uint8_t* d_pixels, int32_t width, int32_t height,
                    int32_t n_images, const rl_config* cfg);
/* rl_label_device runs a large batch (>= 64 Mpx, >= 4 images per pipeline, no label image) as
 * k concurrent pipelines over interleaved sub-batches (image i in pipeline i % k), joined back
 * into the context's stream; results are the same.  k = 3 by default (env RUNLAB_GPU_SPLIT);
 * 1 = one pipeline.  After a split call rl_device_comps returns NULL (the tables live in the
 * pipelines; rl_fetch gathers them) and rl_phase_times reports the total only. */
int rl_set_pipelines(rl_ctx* ctx, int k);
int rl_sync(rl_ctx* ctx);
/* Copies the results of the last rl_label_device() to host memory (like rl_label). */
int rl_fetch(rl_ctx* ctx, rl_result* out);
/* Device views of the last call's outputs (valid until the next call). */
void* rl_device_filled_image(rl_ctx* ctx);
void* rl_device_labels(rl_ctx* ctx);
void* rl_device_comps(rl_ctx* ctx);
/* Stream the context enqueues on (cudaStream_t). */
void* rl_stream(rl_ctx* ctx);
/* Bind the context to an external stream (e.g. torch's current stream); NULL = own. */
int rl_set_stream(rl_ctx* ctx, void* stream);
/* Caller-owned host outputs for rl_label_into (pinned memory makes the copies fast). */
typedef struct rl_host_outputs {
    uint8_t* filled_image;  /* [n*h*w] or NULL */
    uint32_t* labels;       /* [n*h*w] or NULL (requires cfg.relabel) */
    rl_component* comps;    /* [comp_capacity] or NULL */
    uint32_t* top;          /* [comp_capacity] or NULL */
    rl_features* filled;    /* [comp_capacity] or NULL; layout: see filled_layout */
    int64_t comp_capacity;
    int64_t* summary;       /* [n*5] C_pre, n_fg, n_holes, euler, C_post per image, or NULL */
    int64_t* comp_offset;   /* [n+1] or NULL */
    int64_t comps_needed;   /* out: total components of the batch */
    int64_t h2d_bytes;      /* out: bytes copied host->device */
    int64_t d2h_bytes;      /* out: bytes copied device->host */
    int32_t filled_layout;  /* 0: filled[] indexed like comps[] (only post-fill roots are
                               meaningful); 1: the post-fill roots only, in component order
                               (sum over images of C_post entries) */
    int32_t reserved;
} rl_host_outputs;

/* Host-buffer entry point with caller-owned outputs: H2D copy of the pixels, pipeline, D2H
 * copy of every non-NULL output.  Large batches are cut into chunks of whole images that are
 * pipelined through several workspaces and streams, so that the host<->device copies of one
 * chunk overlap the kernels and copies of the others; results are identical to one call over
 * the whole batch.  RL_ENOSPC if comp_capacity is too small (comps_needed tells the size; the
 * non-component outputs are still filled). */
int rl_label_into(rl_ctx* ctx, const uint8_t* pixels, int32_t width, int32_t height,
                  int32_t n_images, const rl_config* cfg, rl_host_outputs* out);

/* The same with an explicit pixel format (RL_PIXELS_*) for the input and the filled image:
 * with RL_PIXELS_P4 each image is height rows of ceil(width / 8) bytes, read and written by the
 * tile kernels as bits (8x fewer bytes over PCIe and HBM); pad bits are ignored on input and
 * zero on output like write_pbm. */
int rl_label_device_fmt(rl_ctx* ctx, const uint8_t* d_pixels, int32_t width, int32_t height, int32_t n_images,
                        const rl_config* cfg, int32_t pixel_format);
int rl_label_into_fmt(rl_ctx* ctx, const uint8_t* pixels, int32_t width, int32_t height, int32_t n_images,
                      const rl_config* cfg, int32_t pixel_format, rl_host_outputs* out);

/* ---- PBM files (io.hpp:74-154) ---------------------------------------------------------------
 * rl_pbm_parse: header of a P1/P4 file with read_pbm's rules; RL_EFORMAT with the offending byte
 * offset and message (PbmParseError) on malformed, truncated or oversized input.
 * rl_fill_pbm: `runlab fill` (tools/runlab.cpp:128-137) as one call -- PBM bytes in, the
 * hole-filled image out as a complete P4 file (write_pbm); the P4 raster is decoded and encoded
 * by the tile kernels, P1 text is parsed on the host.  `extra` (optional) receives the other
 * rl_label_into outputs (its filled_image is ignored).  RL_ENOSPC if out_cap is too small
 * (*out_len = size needed). */
typedef struct rl_pbm_info {
    int32_t width, height;
    int32_t format;        /* 1 (P1) or 4 (P4) */
    int32_t pad;
    int64_t raster_offset; /* byte offset of the raster */
    int64_t error_offset;  /* RL_EFORMAT: PbmParseError::byte_offset; else -1 */
    char message[96];
} rl_pbm_info;
int rl_pbm_parse(const uint8_t* bytes, size_t len, rl_pbm_info* info);
int rl_pbm_p1_to_p4(const uint8_t* bytes, size_t len, rl_pbm_info* info, uint8_t* p4_rows);
size_t rl_pbm_p4_header(int32_t width, int32_t height, char* out, size_t cap);
int rl_fill_pbm(rl_ctx* ctx, const uint8_t* pbm, size_t len, const rl_config* cfg, uint8_t* out_pbm,
                size_t out_cap, size_t* out_len, rl_host_outputs* extra, rl_pbm_info* info);

/* Per-phase device times of the call `back` calls ago (0 = last; back < 64). */
int rl_phase_times(const rl_ctx* ctx, int back, rl_times* out);

/* Device-side input generators (BASELINE configs), bit-identical to the reference's
 * generate() (generator.hpp:46-83).  stream: cudaStream_t or NULL; d_out: w*h bytes. */
int rl_generate(void* stream, uint8_t* d_out, int32_t w, int32_t h, double density, int32_t g,
                uint64_t seed);
/* The same into a host buffer of w*h bytes (synchronous). */
int rl_generate_host(uint8_t* out, int32_t w, int32_t h, double density, int32_t g, uint64_t seed);
/* Rows [y0, y0 + rows) of the same image (d_out: w*rows bytes; one strip of a large image). */
int rl_generate_rows(void* stream, uint8_t* d_out, int32_t w, int32_t h, int32_t y0, int32_t rows,
                     double density, int32_t g, uint64_t seed);
int rl_generate_rings(void* stream, uint8_t* d_out, int32_t w, int32_t h, int32_t tile,
                      uint64_t seed, double salt);
void rl_cfg4_params(uint64_t i, double* density, int32_t* g);

/* Number of kernel launches the last pipeline enqueued. */
int rl_last_launch_count(const rl_ctx* ctx);
/* Device workspace bytes the context holds (all grow-only tables).  For a strip context this
 * follows the strip's size, not the whole image's. */
int64_t rl_workspace_bytes(const rl_ctx* ctx);
/* 1 when the last call replayed a captured CUDA graph (small workloads; disable with the
 * environment variable RUNLAB_GPU_NO_GRAPH).  Phase times of older calls (back > 0) are then
 * not kept. */
int rl_last_used_graph(const rl_ctx* ctx);


/* ---- One image cut into horizontal strips across ranks -----------------------
 * Rank r holds rows [y0, y0 + h) of one w x H image in device memory (y0 a multiple of 32; h a
 * multiple of 32 except for the last strip).  Only O(w) data crosses ranks: the components that
 * touch a cut row ("cut classes") and the two cut rows' labels.  Phases, with the caller's
 * collectives between them (paper_2006_09299_b200/strips.py does them with torch.distributed;
 * NCCL on GPUs):
 *   1. rl_strip_local   tile passes, seams and flattening inside the strip (cut rows are open,
 *                       not frame); numbers the strip's cut classes
 *   2. [all-gather of every rank's rl_strip_local_info]
 *   3. rl_strip_export  the strip's exchange record (per cut class: first-pixel key, features,
 *                       foreground flag; the exterior's partial features; both cut rows as
 *                       (value << 31) | class) into a device buffer of
 *                       rl_strip_export_bytes(w, max_classes) bytes
 *   4. [all-gather of the records: n_strips consecutive records, in image order]
 *   5. rl_strip_merge   union across the cuts (identical on every rank), canonical numbering of
 *                       this strip; returns the link table (canonical id and parent-chain exit of
 *                       every cut component this strip owns; zero elsewhere)
 *   6. [all-reduce SUM of the link table in place]
 *   7. rl_strip_resolve depth-1 ancestors, tree and emit passes of this strip; returns this
 *                       rank's partial post-fill sums of the survivors that cross a cut
 *   8. [all-reduce of the partials in place: d_sum SUM, d_min MIN, d_max MAX, d_count SUM]
 *   9. rl_strip_finish  post-fill features; the canonical-id range [comp_lo, comp_hi) this strip
 *                       owns (components whose first pixel lies in it; strip 0 also owns the
 *                       exterior, id 0)
 *  10. rl_strip_fetch   copies that range and the strip's filled/label image rows to the host.
 * Concatenating the strips' outputs gives exactly the single-image result.  densify_labels is
 * not supported in strip mode (RL_EINVAL). */
typedef struct rl_strip_local_info {
    int64_t n_classes;  /* cut classes: strip components touching a cut row (exterior excluded) */
    int64_t n_comps;    /* strip components touching no cut row (exterior excluded) */
    int64_t n_fg;       /* ... of which foreground */
    int32_t ty0, ty1;   /* tile rows of the strip */
    int32_t status, pad;
} rl_strip_local_info;

typedef struct rl_strip_links {
    void* d_links;  /* int64 [n]: all-reduced with SUM */
    int64_t n;
} rl_strip_links;

typedef struct rl_strip_partials {
    void* d_sum;    /* int64 [k * 3]: S, Sx, Sy */
    void* d_min;    /* int32 [k * 2]: row_min, col_min */
    void* d_max;    /* int32 [k * 2]: row_max, col_max */
    void* d_count;  /* int64 [1]: survivors of this strip that touch no cut */
    int64_t k;      /* global cut-class slots (identical on every rank) */
} rl_strip_partials;

typedef struct rl_strip_result {
    int64_t comp_lo, comp_hi;  /* canonical ids owned by this strip */
    int64_t n_components, n_fg, n_holes, euler, n_survivors;  /* whole image */
    int32_t y0, h;
} rl_strip_result;

int rl_strip_local(rl_ctx* ctx, const uint8_t* d_strip, int32_t width, int32_t height, int32_t y0,
                   int32_t h, const rl_config* cfg, rl_strip_local_info* out);
int64_t rl_strip_export_bytes(int32_t width, int64_t max_classes);
int rl_strip_export(rl_ctx* ctx, int64_t max_classes, void* d_buf);
int rl_strip_merge(rl_ctx* ctx, const void* d_gathered, int32_t n_strips, const rl_strip_local_info* infos,
                   int64_t max_classes, rl_strip_links* out);
int rl_strip_resolve(rl_ctx* ctx, rl_strip_partials* out);
int rl_strip_finish(rl_ctx* ctx, rl_strip_result* out);
/* comps/top/filled (layout 0) of [comp_lo, comp_hi), filled_image/labels of the strip's rows */
int rl_strip_fetch(rl_ctx* ctx, const rl_strip_result* r, rl_host_outputs* out);

/* Rows of n strips: multiples of the 32-row tile height, the remainder spread over the first
 * strips, the last strip takes the image's ragged end (y0[n], h[n]).  RL_EINVAL if n exceeds
 * the tile rows. */
int rl_strip_rows(int32_t height, int32_t n_strips, int32_t* y0, int32_t* h);
/* The whole strip protocol in one call, for the strips of one image held by k contexts of this
 * process (one per GPU of a node, or several on one GPU): d_strips[r] = rows [y0[r], y0[r] + h[r])
 * of rl_strip_rows(height, k) on ctx[r]'s device.  The phases run on one host thread per strip;
 * the collectives are device-to-device copies between the contexts' devices (peer access over
 * NVLink where available) and a reduction kernel on every device.  results[r] as from
 * rl_strip_finish; rl_strip_fetch(ctx[r], &results[r], ...) then copies strip r's part out.  Errors
 * of any strip are reported on ctx[0]. */
int rl_label_strips(rl_ctx* const* ctx, int32_t k, const uint8_t* const* d_strips, int32_t width, int32_t height,
                    const rl_config* cfg, rl_strip_result* results);
/* The same from a host image (row-major w x H bytes): each strip's rows are copied to its
 * context's device first. */
int rl_label_strips_host(rl_ctx* const* ctx, int32_t k, const uint8_t* pixels, int32_t width, int32_t height,
                         const rl_config* cfg, rl_strip_result* results);

/* Connected-operator filtering (analysis.hpp:89-125 filter_components) of one image's canonical
 * pre-fill table d_comps[n] (device): every component with d_selected[id] != 0 merges, with
 * everything embedded in it, into its surrounding component.  Outputs (device, n each):
 * d_parent = absorbing survivor or the id itself (the filtered equivalence table),
 * d_features = survivors accumulate the features they absorb (merged ones keep their own),
 * d_adjacency = surrounding component of each component, redirected to its survivor for the
 * components that survive (UINT32_MAX for the exterior).  The predicate of the reference is a
 * selection mask here (computed by the caller, e.g. from the features on the device).
 * RL_EINVAL if the exterior (id 0) is selected.  Synchronous on `stream`. */
int rl_filter_components(void* stream, const rl_component* d_comps, int64_t n, const uint8_t* d_selected,
                         uint32_t* d_parent, rl_features* d_features, uint32_t* d_adjacency);
/* The same with host buffers (copies in and out; used by include/runlab_gpu.hpp). */
int rl_filter_components_host(const rl_component* comps, int64_t n, const uint8_t* selected, uint32_t* parent,
                              rl_features* features, uint32_t* adjacency);

/* Tile geometry used by the kernels (for DESIGN/roofline bookkeeping). */
void rl_tile_shape(int32_t* tile_h, int32_t* tile_w);

#ifdef __cplusplus
}
#endif
#endif
