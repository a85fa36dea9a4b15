// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/runlab/*.hpp, included from where they lie; nothing is
// copied).  Built by oracle/Makefile into oracle/_ref/libref_runlab.so, it serves two roles:
//   * the pin for the C restatement in oracle/runlab_oracle.c (tests/test_oracle_pin.py),
//   * the reference CPU path timed by bench.py (cpu_baseline, --impl reference).
// The outputs use the same canonical layout as oracle/runlab_oracle.h.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "runlab/runlab.hpp"

#include "runlab_oracle.h"

using namespace runlab;

namespace {

BinaryImage to_image(const std::uint8_t* px, std::int32_t w, std::int32_t h) {
    BinaryImage img(w, h);
    std::memcpy(img.pixels.data(), px, static_cast<std::size_t>(w) * h);
    return img;
}

orc_features conv(const FeatureAccumulator& f) {
    return orc_features{f.s, f.sx, f.sy, f.row_min, f.row_max, f.col_min, f.col_max};
}

Connectivity conn_of(int c) { return c == 1 ? Connectivity::fg4_bg8 : Connectivity::fg8_bg4; }

}  // namespace

extern "C" {

int ref_generate(std::int32_t w, std::int32_t h, double d, std::int32_t g, std::uint64_t seed,
                 std::uint8_t* out) {
    try {
        const BinaryImage img = generate({w, h, d, g, seed});
        std::memcpy(out, img.pixels.data(), img.pixels.size());
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}

std::int32_t ref_encode_row(const std::uint8_t* px, std::int32_t w, std::int32_t* er,
                            std::int32_t* rlc) {
    RowCode rc;
    encode_row({px, static_cast<std::size_t>(w)}, rc);
    std::copy(rc.er.begin(), rc.er.end(), er);
    std::copy(rc.rlc.begin(), rc.rlc.end(), rlc);
    return rc.ner;
}

// Same contract as orc_label_canonical, computed with the reference API: label_image with
// (features, euler) for the pre-fill tree, label_image with (fill, features, relabel) and
// binarize_labels for the filled image, canonical ids = rank of the root (labeling.hpp:44-49).
int ref_label_canonical(const std::uint8_t* px, std::int32_t w, std::int32_t h, int conn,
                        int want_labels, orc_result* out) {
    std::memset(out, 0, sizeof(*out));
    try {
        const BinaryImage img = to_image(px, w, h);
        LabelingConfig ca;
        ca.connectivity = conn_of(conn);
        ca.compute_features = true;
        ca.compute_euler = true;
        ca.relabel = want_labels != 0;
        const LabelingResult a = label_image(img, ca);
        LabelingConfig cb;
        cb.connectivity = conn_of(conn);
        cb.compute_features = true;
        cb.fill_holes = true;
        cb.relabel = true;
        const LabelingResult b = label_image(img, cb);
        const BinaryImage filled = binarize_labels(*b.labels, b.equivalences);

        const label_t ne = a.equivalences.size();
        std::vector<std::uint32_t> cid(ne, no_label);
        std::uint32_t nc = 0;
        for (label_t e = 0; e < ne; ++e)
            if (a.equivalences.is_root(e)) cid[e] = nc++;
        out->width = w;
        out->height = h;
        out->n_components = nc;
        out->n_fg = *a.fg_count;
        out->n_holes = *a.hole_count;
        out->euler = euler_number(a);
        out->comps = static_cast<orc_component*>(std::malloc(sizeof(orc_component) * nc));
        out->top = static_cast<std::uint32_t*>(std::malloc(sizeof(std::uint32_t) * nc));
        out->filled = static_cast<orc_features*>(std::malloc(sizeof(orc_features) * nc));
        std::int64_t surv = 0;
        // components() (analysis.hpp:23-41) walks the roots in ascending order
        for (const ComponentRecord& rec : components(a)) {
            const std::uint32_t c = cid[rec.root];
            out->comps[c].f = conv(rec.features);
            out->comps[c].parent = rec.root == 0 ? no_label : cid[rec.parent_root];
            out->comps[c].flags = rec.foreground ? 1u : 0u;
            const label_t r = b.equivalences.parent(rec.root);
            out->top[c] = cid[r];
            if (r == rec.root) {
                out->filled[c] = conv((*b.features)[rec.root]);
                ++surv;
            } else {
                out->filled[c] = conv(FeatureAccumulator{});
            }
        }
        out->n_survivors = surv;
        const std::size_t P = static_cast<std::size_t>(w) * h;
        out->filled_image = static_cast<std::uint8_t*>(std::malloc(P));
        std::memcpy(out->filled_image, filled.pixels.data(), P);
        if (want_labels) {
            out->labels = static_cast<std::uint32_t*>(std::malloc(P * sizeof(std::uint32_t)));
            for (std::size_t i = 0; i < P; ++i) out->labels[i] = cid[a.labels->labels[i]];
        }
        return 0;
    } catch (const std::overflow_error&) {
        return -2;
    } catch (const std::exception&) {
        return -1;
    }
}

void ref_result_free(orc_result* r) {
    std::free(r->comps);
    std::free(r->top);
    std::free(r->filled);
    std::free(r->filled_image);
    std::free(r->labels);
    std::memset(r, 0, sizeof(*r));
}

std::int32_t ref_flood_label(const std::uint8_t* px, std::int32_t w, std::int32_t h, int conn,
                             std::int32_t* comp) {
    const OraclePartition p = flood_label(to_image(px, w, h), conn_of(conn));
    std::copy(p.comp.begin(), p.comp.end(), comp);
    return p.count;
}

std::int64_t ref_bitquad_euler(const std::uint8_t* px, std::int32_t w, std::int32_t h, int conn) {
    return bitquad_euler(to_image(px, w, h), conn_of(conn));
}

// ---- CPU baseline timing (the reference's own path, bench.py cpu_baseline / --impl reference)
//
// "Same outputs" work per image, as BASELINE.md section 3 defines it:
//   label_image(fill=false, features, euler)            -- pre-fill tree, features, Euler
// + label_image(fill=true, features, relabel) + binarize_labels  -- filled image + features
// Images are processed by `threads` std::threads, one image at a time per thread
// (SPEC.md:243 allows concurrent labeling of distinct images).  Returns wall seconds.
double ref_time_batch(const std::uint8_t* px, std::int32_t w, std::int32_t h, std::int32_t n_images,
                      int conn, int threads, std::int64_t* checksum) {
    const std::size_t P = static_cast<std::size_t>(w) * h;
    std::vector<BinaryImage> imgs;
    imgs.reserve(static_cast<std::size_t>(n_images));
    for (std::int32_t i = 0; i < n_images; ++i) imgs.push_back(to_image(px + P * i, w, h));
    std::vector<std::int64_t> sums(static_cast<std::size_t>(n_images), 0);
    const auto work = [&](std::int32_t i) {
        LabelingConfig ca;
        ca.connectivity = conn_of(conn);
        ca.compute_features = true;
        ca.compute_euler = true;
        const LabelingResult a = label_image(imgs[i], ca);
        LabelingConfig cb = ca;
        cb.compute_euler = false;
        cb.fill_holes = true;
        cb.relabel = true;
        const LabelingResult b = label_image(imgs[i], cb);
        const BinaryImage filled = binarize_labels(*b.labels, b.equivalences);
        std::int64_t s = *a.euler + static_cast<std::int64_t>(a.equivalences.size());
        s += filled.pixels[filled.pixels.size() / 2];
        sums[static_cast<std::size_t>(i)] = s;
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (threads <= 1) {
        for (std::int32_t i = 0; i < n_images; ++i) work(i);
    } else {
        std::vector<std::thread> pool;
        std::atomic<std::int32_t> next{0};
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&] {
                for (;;) {
                    const std::int32_t i = next.fetch_add(1);
                    if (i >= n_images) break;
                    work(i);
                }
            });
        for (auto& th : pool) th.join();
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (checksum) {
        std::int64_t s = 0;
        for (const auto v : sums) s += v;
        *checksum = s;
    }
    return secs;
}

// filter_components (analysis.hpp:89-125) run by the reference on its own label_image result
// (features, no fill); `selected` is indexed by canonical id (ascending root order).  Outputs
// in canonical ids like orc_filter_components.  Returns -1 when the reference throws
// invalid_argument (exterior selected).
int ref_filter_components(const std::uint8_t* px, std::int32_t w, std::int32_t h, int conn,
                          const std::uint8_t* selected, std::int64_t n, std::uint32_t* parent_out,
                          orc_features* features_out, std::uint32_t* adjacency_out) {
    try {
        const BinaryImage img = to_image(px, w, h);
        LabelingConfig ca;
        ca.connectivity = conn_of(conn);
        ca.compute_features = true;
        const LabelingResult a = label_image(img, ca);
        const label_t ne = a.equivalences.size();
        std::vector<std::uint32_t> cid(ne, no_label);
        std::int64_t nc = 0;
        for (label_t e = 0; e < ne; ++e)
            if (a.equivalences.is_root(e)) cid[e] = static_cast<std::uint32_t>(nc++);
        if (nc != n) return -3;
        const LabelingResult f = filter_components(
            a, [&](const ComponentRecord& rec) { return selected[cid[rec.root]] != 0; });
        for (label_t e = 0; e < ne; ++e) {
            if (!a.equivalences.is_root(e)) continue;
            const std::uint32_t c = cid[e];
            parent_out[c] = cid[f.equivalences.parent(e)];
            features_out[c] = conv((*f.features)[e]);
            adjacency_out[c] = e == 0 ? no_label : cid[f.adjacency[e]];
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::overflow_error&) {
        return -2;
    } catch (const std::exception&) {
        return -4;
    }
}

// read_pbm (io.hpp:74-124): 0 and the pixels, or -1 and PbmParseError::byte_offset
int ref_read_pbm(const char* bytes, std::int64_t len, std::uint8_t* pixels, std::int64_t cap, std::int32_t* w,
                 std::int32_t* h, std::int64_t* err_offset) {
    try {
        const BinaryImage img = read_pbm(std::string_view(bytes, static_cast<std::size_t>(len)));
        *w = img.width;
        *h = img.height;
        if (static_cast<std::int64_t>(img.pixels.size()) <= cap)
            std::memcpy(pixels, img.pixels.data(), img.pixels.size());
        return 0;
    } catch (const PbmParseError& e) {
        *err_offset = static_cast<std::int64_t>(e.byte_offset);
        return -1;
    }
}

// write_pbm (io.hpp:126-154): bytes of the file (P4 unless p1), copied when they fit
std::int64_t ref_write_pbm(const std::uint8_t* px, std::int32_t w, std::int32_t h, int p1, char* out,
                           std::int64_t cap) {
    const std::string s = write_pbm(to_image(px, w, h), p1 ? PbmFormat::p1 : PbmFormat::p4);
    if (static_cast<std::int64_t>(s.size()) <= cap) std::memcpy(out, s.data(), s.size());
    return static_cast<std::int64_t>(s.size());
}

}  // extern "C"
