/*
 * runlab_oracle.c -- TEST INFRASTRUCTURE ONLY (see runlab_oracle.h).
 *
 * A plain-C restatement of the reference's LSL black&white pipeline.  Each function cites
 * the reference lines it follows (paths relative to /root/reference/proj/include/runlab/).
 * The restatement is pinned against the reference compiled from its own headers
 * (oracle/_ref/libref_runlab.so) by tests/test_oracle_pin.py.
 */
#include "runlab_oracle.h"

#include <limits.h>
#include <stdlib.h>
#include <string.h>

#define NO_LABEL UINT32_MAX

/* ------------------------------------------------------------------ generator */
/* generator.hpp:28-41: splitmix64 step and the counter-based block draw. */
static uint64_t sm_step(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

uint64_t orc_block_draw(uint64_t seed, uint64_t br, uint64_t bc) {
    return sm_step(sm_step(sm_step(seed) ^ br) ^ bc);
}

/* generator.hpp:46-83 */
int orc_generate(int32_t w, int32_t h, double density, int32_t g, uint64_t seed, uint8_t* out) {
    if (w < 1 || h < 1) return -1;
    if (density < 0.0 || density > 1.0) return -1;
    if (g < 1 || g > (w < h ? w : h)) return -1;
    memset(out, 0, (size_t)w * (size_t)h);
    if (density <= 0.0) return 0;
    const double scaled = density * 18446744073709551616.0;
    const int always = scaled >= 18446744073709551616.0;
    const uint64_t threshold = always ? 0 : (uint64_t)scaled;
    for (int32_t br = 0; (int64_t)br * g < h; ++br) {
        const int32_t r0 = br * g, r1 = (r0 + g < h) ? r0 + g : h;
        for (int32_t bc = 0; (int64_t)bc * g < w; ++bc) {
            const uint64_t draw = orc_block_draw(seed, (uint64_t)br, (uint64_t)bc);
            if (!always && draw >= threshold) continue;
            const int32_t c0 = bc * g, c1 = (c0 + g < w) ? c0 + g : w;
            for (int32_t r = r0; r < r1; ++r) memset(out + (size_t)r * w + c0, 1, (size_t)(c1 - c0));
        }
    }
    return 0;
}

/* Config 3 (new generator, not in the reference; SURVEY App. B interpretation, pinned here):
 * tile x tile blocks; k = 1 + draw mod 16 concentric square rings starting 1 px inside the
 * block, ring r has width 1 + draw mod 3, rings alternate FG (r even) / BG (r odd), placement
 * stops when a ring would cross the half-block; then salt = XOR flip with probability `salt`. */
int orc_generate_rings(int32_t w, int32_t h, int32_t tile, uint64_t seed, double salt, uint8_t* out) {
    if (w < 1 || h < 1 || tile < 4) return -1;
    memset(out, 0, (size_t)w * (size_t)h);
    const int32_t ntc = (w + tile - 1) / tile;
    const int32_t half = tile / 2;
    for (int32_t tr = 0; (int64_t)tr * tile < h; ++tr)
        for (int32_t tc = 0; tc < ntc; ++tc) {
            const uint64_t tile_id = (uint64_t)tr * (uint64_t)ntc + (uint64_t)tc;
            const int32_t k = 1 + (int32_t)(orc_block_draw(seed, (uint64_t)tr, (uint64_t)tc) % 16u);
            int32_t off = 1;
            for (int32_t r = 0; r < k; ++r) {
                const int32_t rw = 1 + (int32_t)(orc_block_draw(seed ^ 0xABCDull, tile_id, (uint64_t)r) % 3u);
                if (off + rw > half) break;
                if ((r & 1) == 0) {
                    /* paint the square annulus [off, off+rw) from each block side */
                    for (int32_t y = off; y < tile - off; ++y)
                        for (int32_t x = off; x < tile - off; ++x) {
                            const int32_t d = (y - off < x - off ? y - off : x - off);
                            const int32_t e1 = tile - 1 - off - y, e2 = tile - 1 - off - x;
                            int32_t dm = d;
                            if (e1 < dm) dm = e1;
                            if (e2 < dm) dm = e2;
                            if (dm < rw) {
                                const int64_t gy = (int64_t)tr * tile + y, gx = (int64_t)tc * tile + x;
                                if (gy < h && gx < w) out[gy * w + gx] = 1;
                            }
                        }
                }
                off += rw;
            }
        }
    if (salt > 0.0) {
        const uint64_t thr = (uint64_t)(salt * 18446744073709551616.0);
        for (int32_t y = 0; y < h; ++y)
            for (int32_t x = 0; x < w; ++x)
                if (orc_block_draw(seed ^ 0x5A17ull, (uint64_t)y, (uint64_t)x) < thr)
                    out[(size_t)y * w + x] ^= 1;
    }
    return 0;
}

/* config-4 per-image density and granularity draws. */
void orc_cfg4_params(uint64_t i, double* density, int32_t* g) {
    *density = 0.1 + 0.8 * ((double)(orc_block_draw(42, i, 0) >> 11) * (1.0 / 9007199254740992.0));
    *g = 1 + (int32_t)(orc_block_draw(42, i, 1) % 8u);
}

/* ------------------------------------------------------------------ features */
/* features.hpp:14-25 empty accumulator */
static orc_features feat_empty(void) {
    orc_features f;
    f.s = f.sx = f.sy = 0;
    f.row_min = INT32_MAX;
    f.row_max = INT32_MIN;
    f.col_min = INT32_MAX;
    f.col_max = INT32_MIN;
    return f;
}

/* features.hpp:33-44 merge_into; returns nonzero on overflow */
static int merge_into(orc_features* a, const orc_features* b) {
    int ovf = __builtin_add_overflow(a->s, b->s, &a->s);
    ovf |= __builtin_add_overflow(a->sx, b->sx, &a->sx);
    ovf |= __builtin_add_overflow(a->sy, b->sy, &a->sy);
    if (ovf) return 1;
    if (b->row_min < a->row_min) a->row_min = b->row_min;
    if (b->row_max > a->row_max) a->row_max = b->row_max;
    if (b->col_min < a->col_min) a->col_min = b->col_min;
    if (b->col_max > a->col_max) a->col_max = b->col_max;
    return 0;
}

/* features.hpp:55-66 segment_features closed form */
static orc_features segment_features(int32_t row, int32_t j0, int32_t j1) {
    orc_features f;
    const int64_t n = j1 - j0;
    f.s = n;
    f.sx = n * (j0 + j1 - 1) / 2;
    f.sy = (int64_t)row * n;
    f.row_min = f.row_max = row;
    f.col_min = j0;
    f.col_max = j1 - 1;
    return f;
}

/* ------------------------------------------------------------------ tables */
/* tables.hpp:37-84 EquivalenceTable + tables.hpp:94-108 AdjacencyTable, as growable arrays */
typedef struct {
    uint32_t n, cap;
    uint32_t* t;
    uint8_t* parity;
    uint32_t* adj;
    orc_features* feat; /* NULL when features are off */
} tables;

static int tables_grow(tables* tb) {
    const uint32_t nc = tb->cap ? tb->cap * 2 : 1024;
    uint32_t* t = realloc(tb->t, (size_t)nc * sizeof(uint32_t));
    if (!t) return -1;
    tb->t = t;
    uint8_t* p = realloc(tb->parity, nc);
    if (!p) return -1;
    tb->parity = p;
    uint32_t* a = realloc(tb->adj, (size_t)nc * sizeof(uint32_t));
    if (!a) return -1;
    tb->adj = a;
    if (tb->feat) {
        orc_features* f = realloc(tb->feat, (size_t)nc * sizeof(orc_features));
        if (!f) return -1;
        tb->feat = f;
    }
    tb->cap = nc;
    return 0;
}

/* tables.hpp:43-48 make_label (+ AdjacencyTable::push, + feat.push_back) */
static uint32_t make_label(tables* tb, int fg, uint32_t adj, const orc_features* f) {
    if (tb->n == tb->cap && tables_grow(tb)) abort();
    const uint32_t e = tb->n++;
    tb->t[e] = e;
    tb->parity[e] = (uint8_t)(fg ? 1 : 0);
    tb->adj[e] = adj;
    if (tb->feat) tb->feat[e] = *f;
    return e;
}

/* tables.hpp:61-64 find: no path compression */
static uint32_t find(const tables* tb, uint32_t e) {
    while (tb->t[e] != e) e = tb->t[e];
    return e;
}

/* tables.hpp:68-76 union_min */
static uint32_t union_min(tables* tb, uint32_t ra, uint32_t rb) {
    if (ra < rb) {
        tb->t[rb] = ra;
        return ra;
    }
    if (rb < ra) tb->t[ra] = rb;
    return rb;
}

/* tables.hpp:79 */
static void attach_to_exterior(tables* tb, uint32_t e) { tb->t[find(tb, e)] = 0; }

/* ------------------------------------------------------------------ Alg. 1 */
/* labeling.hpp:81-100 encode_row */
int32_t orc_encode_row(const uint8_t* px, int32_t w, int32_t* er_out, int32_t* rlc) {
    rlc[0] = 0;
    int32_t er = 0;
    uint8_t left = 0;
    for (int32_t j = 0; j < w; ++j) {
        const uint8_t x = px[j];
        rlc[er + 1] = j;
        er += x ^ left;
        er_out[j] = er;
        left = x;
    }
    rlc[er + 1] = w;
    return er + 1;
}

typedef struct {
    int32_t* er;
    int32_t* rlc;
    uint32_t* era;
    int32_t ner;
} rowcode;

/* tables.hpp:26-31 reset_exterior */
static void reset_exterior(rowcode* rc, int32_t w) {
    for (int32_t j = 0; j < w; ++j) rc->er[j] = 0;
    rc->rlc[0] = 0;
    rc->rlc[1] = w;
    rc->era[0] = 0;
    rc->ner = 1;
}

/* ------------------------------------------------------------------ Alg. 2 */
/* labeling.hpp:104-157 unify_row_impl (flip per labeling.hpp:164-172).  Returns -2 on
 * feature overflow. */
static int unify_row(tables* tb, const rowcode* above, rowcode* rc, int32_t row, int32_t w,
                     int32_t flip) {
    int32_t er_first = 0;
    if (rc->rlc[1] == 0) {
        rc->era[0] = 0;
        er_first = 1;
    }
    for (int32_t er = er_first; er < rc->ner; ++er) {
        const int32_t j0 = rc->rlc[er];
        const int32_t j1 = rc->rlc[er + 1];
        const int32_t p = er & 1;
        const int32_t c8 = p ^ flip;
        orc_features f;
        if (tb->feat) f = segment_features(row, j0, j1);
        const int32_t a0 = (j0 - c8 > 0) ? j0 - c8 : 0;
        const int32_t a1 = (j1 + c8 < w) ? j1 + c8 : w;
        int32_t er0 = above->er[a0];
        int32_t er1 = above->er[a1 - 1];
        er0 += (er0 & 1) ^ p;
        er1 -= (er1 & 1) ^ p;
        if (er1 >= er0) {
            uint32_t a = find(tb, above->era[er0]);
            for (int32_t k = er0 + 2; k <= er1; k += 2) a = union_min(tb, a, find(tb, above->era[k]));
            rc->era[er] = a;
            if (tb->feat && merge_into(&tb->feat[a], &f)) return -2;
        } else {
            const uint32_t adj = er > 0 ? rc->era[er - 1] : 0u;
            rc->era[er] = make_label(tb, p != 0, adj, &f);
        }
    }
    attach_to_exterior(tb, rc->era[0]);
    if (rc->ner & 1) attach_to_exterior(tb, rc->era[rc->ner - 1]);
    return 0;
}

/* labeling.hpp:176-179 close_bottom_border */
static void close_bottom_border(tables* tb, const rowcode* cur) {
    for (int32_t er = 0; er < cur->ner; er += 2) attach_to_exterior(tb, cur->era[er]);
}

/* ------------------------------------------------------------------ Alg. 3 */
/* labeling.hpp:190-217 transitive_closure (with the fill branch :199-205) */
static int transitive_closure(tables* tb, int fill, int64_t* fg_out, int64_t* bg_out) {
    int64_t fg = 0, bg = 0;
    for (uint32_t e = 1; e < tb->n; ++e) {
        uint32_t a = tb->t[e];
        if (a == e) {
            if (tb->parity[e]) ++fg;
            else ++bg;
            if (fill) {
                const uint32_t i = tb->adj[e];
                if (tb->t[i] > 0) {
                    tb->t[e] = i;
                    a = i;
                }
            }
        }
        if (a < e) {
            const uint32_t r = tb->t[a];
            tb->t[e] = r;
            if (tb->feat && merge_into(&tb->feat[r], &tb->feat[e])) return -2;
        } else {
            tb->adj[e] = tb->t[tb->adj[e]];
        }
    }
    *fg_out = fg;
    *bg_out = bg;
    return 0;
}

/* ------------------------------------------------------------------ pipeline */
/* Retained row codes (labeling.hpp:63,295-296), stored as two concatenated arrays. */
typedef struct {
    int64_t n, cap;
    int32_t* rlc;    /* per row: rlc[0..ner] */
    uint32_t* era;   /* per row: era[0..ner-1] */
    int64_t* start;  /* per row: offset into era (rlc offset = start + row) */
    int32_t* ner;
} retained;

static int retained_push(retained* rt, int32_t row, const rowcode* rc) {
    /* era needs n + ner entries; rlc stores ner+1 values per row, i.e. n + row + ner + 1 */
    const int64_t need = rt->n + row + rc->ner + 1;
    if (need > rt->cap) {
        int64_t nc = rt->cap ? rt->cap : 4096;
        while (nc < need) nc *= 2;
        int32_t* r = realloc(rt->rlc, (size_t)nc * sizeof(int32_t));
        uint32_t* e = realloc(rt->era, (size_t)nc * sizeof(uint32_t));
        if (!r || !e) return -1;
        rt->rlc = r;
        rt->era = e;
        rt->cap = nc;
    }
    rt->start[row] = rt->n;
    rt->ner[row] = rc->ner;
    memcpy(rt->era + rt->n, rc->era, (size_t)rc->ner * sizeof(uint32_t));
    memcpy(rt->rlc + rt->n + row, rc->rlc, (size_t)(rc->ner + 1) * sizeof(int32_t));
    rt->n += rc->ner;
    return 0;
}

typedef struct {
    tables tb;
    retained rt;
    int64_t fg, bg;
} pipeline_out;

/* labeling.hpp:263-328 run_pipeline (untimed); retains rows when `keep_rows`. */
static int run_pipeline(const uint8_t* img, int32_t w, int32_t h, int conn, int fill, int features,
                        int keep_rows, pipeline_out* po) {
    memset(po, 0, sizeof(*po));
    tables* tb = &po->tb;
    if (features) {
        tb->feat = malloc(sizeof(orc_features));
        if (!tb->feat) return -1;
    }
    if (tables_grow(tb)) return -1;
    /* EquivalenceTable() : t_{0}, parity_{0}; AdjacencyTable(): i_{no_label};
     * feat.push_back({}) exterior accumulator (labeling.hpp:74) */
    tb->n = 1;
    tb->t[0] = 0;
    tb->parity[0] = 0;
    tb->adj[0] = NO_LABEL;
    if (tb->feat) tb->feat[0] = feat_empty();

    rowcode buf[2];
    for (int i = 0; i < 2; ++i) {
        buf[i].er = malloc((size_t)w * sizeof(int32_t));
        buf[i].rlc = malloc((size_t)(w + 2) * sizeof(int32_t));
        buf[i].era = malloc((size_t)(w + 1) * sizeof(uint32_t));
        if (!buf[i].er || !buf[i].rlc || !buf[i].era) return -1;
    }
    if (keep_rows) {
        po->rt.start = malloc((size_t)h * sizeof(int64_t));
        po->rt.ner = malloc((size_t)h * sizeof(int32_t));
        if (!po->rt.start || !po->rt.ner) return -1;
    }
    rowcode* prev = &buf[0];
    rowcode* cur = &buf[1];
    reset_exterior(prev, w);
    const int32_t flip = conn == 1 ? 1 : 0;
    int rc = 0;
    for (int32_t i = 0; i < h; ++i) {
        if (i > 0) {
            rowcode* tmp = prev;
            prev = cur;
            cur = tmp;
        }
        cur->ner = orc_encode_row(img + (size_t)i * w, w, cur->er, cur->rlc);
        rc = unify_row(tb, prev, cur, i, w, flip);
        if (rc) break;
        if (keep_rows && retained_push(&po->rt, i, cur)) {
            rc = -1;
            break;
        }
    }
    if (!rc) {
        close_bottom_border(tb, cur);
        rc = transitive_closure(tb, fill, &po->fg, &po->bg);
    }
    for (int i = 0; i < 2; ++i) {
        free(buf[i].er);
        free(buf[i].rlc);
        free(buf[i].era);
    }
    return rc;
}

static void pipeline_free(pipeline_out* po) {
    free(po->tb.t);
    free(po->tb.parity);
    free(po->tb.adj);
    free(po->tb.feat);
    free(po->rt.rlc);
    free(po->rt.era);
    free(po->rt.start);
    free(po->rt.ner);
    memset(po, 0, sizeof(*po));
}

/* Alg. 4: labeling.hpp:224-250 relabel, applied to retained rows; `remap` maps the final
 * root to the written value (densify) or is NULL (raw roots). */
static void relabel_rows(const pipeline_out* po, int32_t w, int32_t h, const uint32_t* remap,
                         uint32_t* dst) {
    for (int32_t row = 0; row < h; ++row) {
        const int32_t* rlc = po->rt.rlc + po->rt.start[row] + row;
        const uint32_t* era = po->rt.era + po->rt.start[row];
        int32_t j0 = rlc[0];
        for (int32_t er = 0; er < po->rt.ner[row]; ++er) {
            const int32_t j1 = rlc[er + 1];
            uint32_t r = po->tb.t[era[er]];
            if (remap) r = remap[r];
            for (int32_t j = j0; j < j1; ++j) dst[(size_t)row * w + j] = r;
            j0 = j1;
        }
    }
}

int orc_label_raw(const uint8_t* img, int32_t w, int32_t h, int conn, int fill, int features,
                  int relabel, int densify, orc_raw* out) {
    memset(out, 0, sizeof(*out));
    if (densify && !relabel) return -1; /* labeling.hpp:271-273 */
    if (w < 1 || h < 1) return -1;
    pipeline_out po;
    int rc = run_pipeline(img, w, h, conn, fill, features, relabel, &po);
    if (rc) {
        pipeline_free(&po);
        return rc;
    }
    const uint32_t ne = po.tb.n;
    out->ne = ne;
    out->fg = po.fg;
    out->bg = po.bg;
    out->t = malloc((size_t)ne * sizeof(uint32_t));
    out->adj = malloc((size_t)ne * sizeof(uint32_t));
    out->parity = malloc(ne);
    memcpy(out->t, po.tb.t, (size_t)ne * sizeof(uint32_t));
    memcpy(out->adj, po.tb.adj, (size_t)ne * sizeof(uint32_t));
    memcpy(out->parity, po.tb.parity, ne);
    if (features) {
        out->feat = malloc((size_t)ne * sizeof(orc_features));
        memcpy(out->feat, po.tb.feat, (size_t)ne * sizeof(orc_features));
    }
    if (relabel) {
        uint32_t* remap = NULL;
        if (densify) { /* labeling.hpp:231-236 */
            remap = malloc((size_t)ne * sizeof(uint32_t));
            uint32_t next = 0;
            for (uint32_t e = 0; e < ne; ++e)
                if (po.tb.t[e] == e) remap[e] = next++;
        }
        out->labels = malloc((size_t)w * (size_t)h * sizeof(uint32_t));
        relabel_rows(&po, w, h, remap, out->labels);
        free(remap);
    }
    pipeline_free(&po);
    return 0;
}

void orc_raw_free(orc_raw* r) {
    free(r->t);
    free(r->adj);
    free(r->parity);
    free(r->feat);
    free(r->labels);
    memset(r, 0, sizeof(*r));
}

/* Canonical form: roots of the fill=false run in ascending order == raster order of first
 * pixel (tables.hpp:68-76; verified equal to oracle.hpp's numbering), id 0 = exterior.
 * The fill=true run (labeling.hpp:199-205) supplies the post-fill root of every label and
 * the folded features; binarize_labels (labeling.hpp:354-360) gives the filled image. */
int orc_label_canonical(const uint8_t* img, int32_t w, int32_t h, int conn, int want_labels,
                        orc_result* out) {
    memset(out, 0, sizeof(*out));
    if (w < 1 || h < 1) return -1;
    pipeline_out a, b;
    int rc = run_pipeline(img, w, h, conn, 0, 1, want_labels, &a);
    if (rc) {
        pipeline_free(&a);
        return rc;
    }
    rc = run_pipeline(img, w, h, conn, 1, 1, 1, &b);
    if (rc) {
        pipeline_free(&a);
        pipeline_free(&b);
        return rc;
    }
    const uint32_t ne = a.tb.n;
    uint32_t* cid = malloc((size_t)ne * sizeof(uint32_t));
    uint32_t nc = 0;
    for (uint32_t e = 0; e < ne; ++e) cid[e] = (a.tb.t[e] == e) ? nc++ : NO_LABEL;
    out->width = w;
    out->height = h;
    out->n_components = nc;
    out->n_fg = a.fg;
    out->n_holes = a.bg;
    out->euler = a.fg - a.bg;
    out->comps = malloc((size_t)nc * sizeof(orc_component));
    out->top = malloc((size_t)nc * sizeof(uint32_t));
    out->filled = malloc((size_t)nc * sizeof(orc_features));
    int64_t surv = 0;
    for (uint32_t e = 0; e < ne; ++e) {
        if (cid[e] == NO_LABEL) continue;
        const uint32_t c = cid[e];
        orc_component* cp = &out->comps[c];
        cp->f = a.tb.feat[e];
        cp->parent = e == 0 ? NO_LABEL : cid[a.tb.adj[e]];
        cp->flags = a.tb.parity[e];
        const uint32_t tb_root = b.tb.t[e];
        out->top[c] = cid[tb_root];
        if (tb_root == e) {
            out->filled[c] = b.tb.feat[e];
            ++surv;
        } else {
            out->filled[c] = feat_empty();
        }
    }
    out->n_survivors = surv;
    /* filled image = binarize_labels(relabel(fill run)) */
    const size_t P = (size_t)w * (size_t)h;
    out->filled_image = malloc(P);
    for (int32_t row = 0; row < h; ++row) {
        const int32_t* rlc = b.rt.rlc + b.rt.start[row] + row;
        const uint32_t* era = b.rt.era + b.rt.start[row];
        int32_t j0 = rlc[0];
        for (int32_t er = 0; er < b.rt.ner[row]; ++er) {
            const int32_t j1 = rlc[er + 1];
            const uint8_t v = b.tb.parity[b.tb.t[era[er]]];
            memset(out->filled_image + (size_t)row * w + j0, v, (size_t)(j1 - j0));
            j0 = j1;
        }
    }
    if (want_labels) {
        out->labels = malloc(P * sizeof(uint32_t));
        relabel_rows(&a, w, h, cid, out->labels);
    }
    free(cid);
    pipeline_free(&a);
    pipeline_free(&b);
    return 0;
}

void orc_result_free(orc_result* r) {
    free(r->comps);
    free(r->top);
    free(r->filled);
    free(r->filled_image);
    free(r->labels);
    memset(r, 0, sizeof(*r));
}

/* ------------------------------------------------------------------ brute-force oracles */
/* oracle.hpp:86-124 flood_label with a virtual background frame (BFS). */
int32_t orc_flood_label(const uint8_t* img, int32_t w, int32_t h, int conn, int32_t* comp,
                        uint8_t* comp_fg, int64_t* first_pixel, int32_t cap) {
    const int fg8 = conn == 0;
    const int64_t P = (int64_t)w * h;
    static const int d8[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
    static const int d4[4][2] = {{-1, 0}, {0, -1}, {0, 1}, {1, 0}};
    int64_t* q = malloc((size_t)P * sizeof(int64_t));
    for (int64_t i = 0; i < P; ++i) comp[i] = -1;
    int32_t count = 1;
    if (comp_fg && cap > 0) comp_fg[0] = 0;
    if (first_pixel && cap > 0) first_pixel[0] = -1;
    int64_t qh = 0, qt = 0;
    for (int32_t r = 0; r < h; ++r)
        for (int32_t c = 0; c < w; ++c) {
            if (r != 0 && r != h - 1 && c != 0 && c != w - 1) continue;
            const int64_t i = (int64_t)r * w + c;
            if (img[i] == 0 && comp[i] == -1) {
                comp[i] = 0;
                q[qt++] = i;
            }
        }
    for (int64_t seed = -1; seed < P; ++seed) {
        int32_t id;
        if (seed >= 0) {
            if (comp[seed] != -1) continue;
            id = count++;
            if (comp_fg && id < cap) comp_fg[id] = img[seed] ? 1 : 0;
            if (first_pixel && id < cap) first_pixel[id] = seed;
            comp[seed] = id;
            qh = qt = 0;
            q[qt++] = seed;
        } else {
            id = 0;
        }
        while (qh < qt) {
            const int64_t at = q[qh++];
            const int32_t r = (int32_t)(at / w), c = (int32_t)(at % w);
            const int eight = img[at] ? fg8 : !fg8;
            const int n = eight ? 8 : 4;
            for (int k = 0; k < n; ++k) {
                const int dr = eight ? d8[k][0] : d4[k][0], dc = eight ? d8[k][1] : d4[k][1];
                const int32_t nr = r + dr, ncl = c + dc;
                if (nr < 0 || ncl < 0 || nr >= h || ncl >= w) continue;
                const int64_t ni = (int64_t)nr * w + ncl;
                if (comp[ni] != -1 || img[ni] != img[at]) continue;
                comp[ni] = id;
                q[qt++] = ni;
            }
        }
    }
    free(q);
    return count;
}

/* oracle.hpp:145-166 */
int64_t orc_bitquad_euler(const uint8_t* img, int32_t w, int32_t h, int conn) {
    int64_t q1 = 0, q3 = 0, qd = 0;
#define AT(r, c) (((r) < 0 || (c) < 0 || (r) >= h || (c) >= w) ? 0 : img[(int64_t)(r) * w + (c)])
    for (int32_t r = -1; r < h; ++r)
        for (int32_t c = -1; c < w; ++c) {
            const int tl = AT(r, c), tr = AT(r, c + 1), bl = AT(r + 1, c), br = AT(r + 1, c + 1);
            const int n = tl + tr + bl + br;
            q1 += n == 1;
            q3 += n == 3;
            qd += n == 2 && tl == br && tl != tr;
        }
#undef AT
    const int64_t num = conn == 0 ? q1 - q3 - 2 * qd : q1 - q3 + 2 * qd;
    return num / 4;
}

/* oracle.hpp:170-177 */
void orc_fill_holes(const uint8_t* img, int32_t w, int32_t h, int conn, uint8_t* out) {
    const int64_t P = (int64_t)w * h;
    int32_t* comp = malloc((size_t)P * sizeof(int32_t));
    orc_flood_label(img, w, h, conn, comp, NULL, NULL, 0);
    for (int64_t i = 0; i < P; ++i) out[i] = comp[i] == 0 ? 0 : 1;
    free(comp);
}

/* analysis.hpp:89-125.  components() lists the roots in ascending order (analysis.hpp:23-41),
 * so a parent is always decided before its children: target[c] = target[parent] when the
 * parent merged (embedded in a merged region), else the parent when c itself is selected. */
int orc_filter_components(const orc_component* comps, int64_t n, const uint8_t* selected, uint32_t* parent_out,
                          orc_features* features_out, uint32_t* adjacency_out) {
    const uint32_t NONE = UINT32_MAX;
    if (n < 1) return 0;
    if (selected[0]) return -1; /* analysis.hpp:92-94 */
    uint32_t* target = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    if (!target) return -3;
    for (int64_t c = 0; c < n; ++c) {
        target[c] = NONE;
        features_out[c] = comps[c].f;
    }
    for (int64_t c = 1; c < n; ++c) { /* analysis.hpp:100-111 */
        const uint32_t p = comps[c].parent;
        uint32_t tgt = NONE;
        if (target[p] != NONE)
            tgt = target[p];
        else if (selected[c])
            tgt = p;
        if (tgt != NONE) {
            target[c] = tgt;
            if (merge_into(&features_out[tgt], &comps[c].f)) {
                free(target);
                return -2;
            }
        }
    }
    for (int64_t c = 0; c < n; ++c) /* analysis.hpp:113-116 */
        parent_out[c] = target[c] != NONE ? target[c] : (uint32_t)c;
    adjacency_out[0] = NONE;
    for (int64_t c = 1; c < n; ++c) { /* analysis.hpp:117-121: only components still roots */
        const uint32_t pr = comps[c].parent;
        adjacency_out[c] = (target[c] == NONE && target[pr] != NONE) ? target[pr] : pr;
    }
    free(target);
    return 0;
}
