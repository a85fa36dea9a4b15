/*
 * runlab_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU path (runlab, header-only C++20 under
 * /root/reference/proj/include/runlab) used as the parity checker for the sm_100a
 * implementation.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library; the product path never does.
 *
 * Parity pin: every function is checked bit-exactly against the reference itself,
 * compiled from its own headers into oracle/_ref/libref_runlab.so (oracle/Makefile,
 * oracle/ref_shim.cpp), and against the golden vectors of the reference's own tests
 * (tests/golden/, tests/test_oracle_pin.py).
 *
 * Result layout ("canonical form") is identical to the GPU C ABI (include/runlab_gpu.h):
 * components are numbered by the raster order of their first pixel, id 0 is the exterior
 * (oracle.hpp:20-23, tables.hpp:68-76).
 */
#ifndef RUNLAB_ORACLE_H
#define RUNLAB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* features.hpp:14-25 -- S, Sx, Sy, inclusive bounding box; empty sentinels. 40 bytes. */
typedef struct orc_features {
    int64_t s, sx, sy;
    int32_t row_min, row_max, col_min, col_max;
} orc_features;

/* Pre-fill component record, 48 bytes: features + adjacency parent + flags (bit0 = FG). */
typedef struct orc_component {
    orc_features f;
    uint32_t parent; /* canonical id of the surrounding component; UINT32_MAX for id 0 */
    uint32_t flags;  /* bit 0: foreground */
} orc_component;

/* Canonical labeling result of one image (both label_image runs folded together). */
typedef struct orc_result {
    int32_t width, height;
    int64_t n_components; /* C_pre, exterior included */
    int64_t n_fg;         /* fg roots, pre-fill (labeling.hpp:195-199) */
    int64_t n_holes;      /* non-exterior bg roots, pre-fill */
    int64_t euler;        /* n_fg - n_holes */
    int64_t n_survivors;  /* C_post: roots after hole filling, exterior included */
    orc_component* comps; /* [n_components] pre-fill */
    uint32_t* top;        /* [n_components] id of the post-fill root absorbing each component */
    orc_features* filled; /* [n_components] post-fill features, meaningful where top[i]==i */
    uint8_t* filled_image;/* [w*h] binarize_labels(fill) (labeling.hpp:354-360) */
    uint32_t* labels;     /* [w*h] canonical id per pixel (pre-fill), or NULL */
} orc_result;

/* analysis.hpp:89-125 filter_components on the canonical pre-fill table: every component
 * whose selected[] flag is set merges (with the subtree embedded in it) into its surrounding
 * component.  Outputs per component id: parent_out = absorbing survivor or itself (the
 * equivalence table), features_out = post-filter features (survivors accumulate; merged
 * components keep their own), adjacency_out = surrounding component redirected to its
 * survivor (UINT32_MAX for the exterior).  Returns -1 if the exterior is selected
 * (std::invalid_argument, analysis.hpp:92-94), -2 on feature overflow. */
int orc_filter_components(const orc_component* comps, int64_t n, const uint8_t* selected, uint32_t* parent_out,
                          orc_features* features_out, uint32_t* adjacency_out);

/* generator.hpp:28-41 / :46-83 */
uint64_t orc_block_draw(uint64_t seed, uint64_t block_row, uint64_t block_col);
int orc_generate(int32_t w, int32_t h, double density, int32_t g, uint64_t seed, uint8_t* out);

/* labeling.hpp:81-100 encode_row: fills er[w], rlc[w+2]; returns ner. */
int32_t orc_encode_row(const uint8_t* px, int32_t w, int32_t* er, int32_t* rlc);

/* Raw (provisional-label) pipeline, labeling.hpp:263-328.  Outputs are malloc'd. */
typedef struct orc_raw {
    uint32_t ne;          /* number of provisional labels */
    uint32_t* t;          /* equivalence table after closure */
    uint32_t* adj;        /* adjacency table after closure (adj[0] = UINT32_MAX) */
    uint8_t* parity;      /* 1 = foreground */
    orc_features* feat;   /* [ne] or NULL */
    int64_t fg, bg;
    uint32_t* labels;     /* [w*h] (relabel) or NULL */
} orc_raw;
/* conn: 0 = fg8_bg4, 1 = fg4_bg8. Returns 0, or -1 on invalid args (densify w/o relabel),
 * -2 on feature overflow (features.hpp:37-39). */
int orc_label_raw(const uint8_t* img, int32_t w, int32_t h, int conn, int fill, int features,
                  int relabel, int densify, orc_raw* out);
void orc_raw_free(orc_raw* r);

/* Canonical result: label_image(fill=0, features, euler) + label_image(fill=1, features,
 * relabel) + binarize_labels, renumbered by first pixel.  want_labels: also the per-pixel
 * canonical (pre-fill) label image. */
int orc_label_canonical(const uint8_t* img, int32_t w, int32_t h, int conn, int want_labels,
                        orc_result* out);
void orc_result_free(orc_result* r);

/* oracle.hpp:86-124 flood_label (BFS): comp[w*h] ids in raster order of first pixel,
 * exterior 0.  Returns the component count; comp_fg[count] optional. */
int32_t orc_flood_label(const uint8_t* img, int32_t w, int32_t h, int conn, int32_t* comp,
                        uint8_t* comp_fg, int64_t* first_pixel, int32_t cap);
/* oracle.hpp:145-166 */
int64_t orc_bitquad_euler(const uint8_t* img, int32_t w, int32_t h, int conn);
/* oracle.hpp:170-177 */
void orc_fill_holes(const uint8_t* img, int32_t w, int32_t h, int conn, uint8_t* out);

/* Config-3 nested-ring generator (new; SURVEY App. B interpretation) and the config-4
 * per-image parameter draws. */
int orc_generate_rings(int32_t w, int32_t h, int32_t tile, uint64_t seed, double salt,
                       uint8_t* out);
void orc_cfg4_params(uint64_t i, double* density, int32_t* g);

#ifdef __cplusplus
}
#endif
#endif
