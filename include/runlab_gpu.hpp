// runlab_gpu.hpp -- C++ drop-in for the reference's labeling/analysis entry points,
// running on the B200 through the C ABI of include/runlab_gpu.h (librunlab_gpu.so).
//
// A reference user switches `#include "runlab/runlab.hpp"` to `#include "runlab_gpu.hpp"`
// and links -lrunlab_gpu; the names below keep the reference's signatures and semantics
// (paths relative to /root/reference/proj/include/runlab/):
//
//   label_t, no_label, Connectivity          types.hpp:10-21
//   BinaryImage, LabelImage                  image.hpp:14-67
//   FeatureAccumulator, FeatureTable, merge_into, merge_features, segment_features
//                                            features.hpp:14-66
//   EquivalenceTable, AdjacencyTable         tables.hpp:37-108
//   LabelingConfig, LabelingResult           labeling.hpp:20-50
//   StepTimes, label_image, timed_label_image, binarize_labels   labeling.hpp:253-360
//   ComponentRecord, components, holes, ComponentTree, adjacency_tree, euler_number
//                                            analysis.hpp:13-79
//
// Label values are canonical ids: the rank of each component's raster-first pixel, exterior
// 0 -- i.e. the reference's root labels renumbered in ascending order (its provisional
// labels are an artefact of the sequential scan).  With fill_holes, T[e] is e's post-fill
// root (its depth-1 ancestor).  Errors map as in the reference: std::invalid_argument,
// std::logic_error, std::overflow_error; device failures throw std::runtime_error.
#pragma once

#include <algorithm>
#include <cassert>
#include <cstdint>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "runlab_gpu.h"

namespace runlab {

using label_t = std::uint32_t;
inline constexpr label_t no_label = std::numeric_limits<label_t>::max();

enum class Connectivity : std::uint8_t { fg8_bg4, fg4_bg8 };

struct BinaryImage {
    std::int32_t width = 0;
    std::int32_t height = 0;
    std::vector<std::uint8_t> pixels;  // row-major, 0 = background, 1 = foreground

    BinaryImage() = default;
    BinaryImage(std::int32_t w, std::int32_t h)
        : width(w), height(h), pixels(static_cast<std::size_t>(w) * static_cast<std::size_t>(h), 0) {}
    std::int64_t pixel_count() const { return static_cast<std::int64_t>(width) * height; }
    std::uint8_t operator()(std::int32_t r, std::int32_t c) const { return pixels[static_cast<std::size_t>(r) * width + c]; }
    std::uint8_t& operator()(std::int32_t r, std::int32_t c) { return pixels[static_cast<std::size_t>(r) * width + c]; }
    std::span<const std::uint8_t> row(std::int32_t r) const {  // image.hpp:37-41
        return {pixels.data() + static_cast<std::size_t>(r) * width, static_cast<std::size_t>(width)};
    }
    bool operator==(const BinaryImage&) const = default;
};

struct LabelImage {
    std::int32_t width = 0;
    std::int32_t height = 0;
    std::vector<label_t> labels;

    LabelImage() = default;
    LabelImage(std::int32_t w, std::int32_t h)
        : width(w), height(h), labels(static_cast<std::size_t>(w) * static_cast<std::size_t>(h), 0) {}
    label_t operator()(std::int32_t r, std::int32_t c) const { return labels[static_cast<std::size_t>(r) * width + c]; }
    label_t& operator()(std::int32_t r, std::int32_t c) { return labels[static_cast<std::size_t>(r) * width + c]; }
    bool operator==(const LabelImage&) const = default;
};

struct FeatureAccumulator {
    std::int64_t s = 0, sx = 0, sy = 0;
    std::int32_t row_min = std::numeric_limits<std::int32_t>::max();
    std::int32_t row_max = std::numeric_limits<std::int32_t>::min();
    std::int32_t col_min = std::numeric_limits<std::int32_t>::max();
    std::int32_t col_max = std::numeric_limits<std::int32_t>::min();
    bool empty() const { return s == 0; }
    bool operator==(const FeatureAccumulator&) const = default;
};
using FeatureTable = std::vector<FeatureAccumulator>;

// features.hpp:33-45: sums add (std::overflow_error on 64-bit overflow), boxes take the envelope
inline void merge_into(FeatureAccumulator& a, const FeatureAccumulator& b) {
    bool ovf = __builtin_add_overflow(a.s, b.s, &a.s);
    ovf |= __builtin_add_overflow(a.sx, b.sx, &a.sx);
    ovf |= __builtin_add_overflow(a.sy, b.sy, &a.sy);
    if (ovf) throw std::overflow_error("feature accumulator overflow: image exceeds supported sizes");
    a.row_min = std::min(a.row_min, b.row_min);
    a.row_max = std::max(a.row_max, b.row_max);
    a.col_min = std::min(a.col_min, b.col_min);
    a.col_max = std::max(a.col_max, b.col_max);
}

// features.hpp:48-52
inline FeatureAccumulator merge_features(FeatureAccumulator a, const FeatureAccumulator& b) {
    merge_into(a, b);
    return a;
}

// features.hpp:56-66: moments of the run [j0, j1) of `row` in closed form (the device kernels
// evaluate the same expressions per run)
inline FeatureAccumulator segment_features(std::int32_t row, std::int32_t j0, std::int32_t j1) {
    FeatureAccumulator f;
    const std::int64_t n = j1 - j0;
    f.s = n;
    f.sx = n * (j0 + j1 - 1) / 2;
    f.sy = static_cast<std::int64_t>(row) * n;
    f.row_min = f.row_max = row;
    f.col_min = j0;
    f.col_max = j1 - 1;
    return f;
}

// tables.hpp:37-84: union-find over labels with the min-label rule and one parity bit per
// label.  A default table holds the exterior (label 0, background), like the reference's; the
// GPU fills results through the (parent, parity) constructor, and the scan-time mutators are
// kept so reference code that builds or edits tables compiles and behaves the same.
class EquivalenceTable {
public:
    EquivalenceTable() : t_{0}, fg_{0} {}
    EquivalenceTable(std::vector<label_t> parent, std::vector<std::uint8_t> fg)
        : t_(std::move(parent)), fg_(std::move(fg)) {}
    label_t size() const { return static_cast<label_t>(t_.size()); }
    label_t make_label(bool foreground) {
        const label_t e = size();
        t_.push_back(e);
        fg_.push_back(foreground ? 1 : 0);
        return e;
    }
    bool is_foreground(label_t e) const { return fg_[e] != 0; }
    label_t parent(label_t e) const { return t_[e]; }
    bool is_root(label_t e) const { return t_[e] == e; }
    void set_parent(label_t e, label_t p) {
        assert(p <= e);
        t_[e] = p;
    }
    label_t find(label_t e) const {
        while (t_[e] != e) e = t_[e];
        return e;
    }
    label_t union_min(label_t ra, label_t rb) {
        assert(is_root(ra) && is_root(rb));
        if (ra < rb) {
            t_[rb] = ra;
            return ra;
        }
        if (rb < ra) t_[ra] = rb;
        return rb;
    }
    void attach_to_exterior(label_t e) { t_[find(e)] = 0; }

private:
    std::vector<label_t> t_;
    std::vector<std::uint8_t> fg_;
};

// tables.hpp:94-108: surrounding component per label; entry 0 is the no_label sentinel
class AdjacencyTable {
public:
    AdjacencyTable() : i_{no_label} {}
    explicit AdjacencyTable(std::vector<label_t> i) : i_(std::move(i)) {}
    label_t size() const { return static_cast<label_t>(i_.size()); }
    void push(label_t initial) { i_.push_back(initial); }
    label_t operator[](label_t e) const { return i_[e]; }
    void redirect(label_t e, label_t root) { i_[e] = root; }

private:
    std::vector<label_t> i_;
};

struct LabelingConfig {
    Connectivity connectivity = Connectivity::fg8_bg4;
    bool fill_holes = false;
    bool compute_features = false;
    bool relabel = false;
    bool densify_labels = false;
    bool compute_euler = false;
};

struct LabelingResult {
    std::int32_t width = 0;
    std::int32_t height = 0;
    LabelingConfig config;
    EquivalenceTable equivalences;
    AdjacencyTable adjacency;
    std::optional<FeatureTable> features;
    std::optional<LabelImage> labels;
    std::optional<std::int64_t> fg_count;
    std::optional<std::int64_t> hole_count;
    std::optional<std::int64_t> euler;

    std::vector<label_t> roots() const {
        std::vector<label_t> out;
        for (label_t e = 0; e < equivalences.size(); ++e)
            if (equivalences.is_root(e)) out.push_back(e);
        return out;
    }
};

// labeling.hpp:253-259, filled from the device phases (CUDA events on the context stream).
// The device pipeline is not row-sequential, so the reference's per-row phases map to passes:
//   encode_ns  = the tile analysis pass: segment detection (Alg. 1) fused with the tile-local
//                part of unification (Alg. 2) and the border tables;
//   unify_ns   = the cross-tile merge: seam unions (rest of Alg. 2), closure of the border
//                classes, canonical ids, adjacency tree and hole-fill targets (Alg. 3);
//   closure_ns = the emit pass: per-component records and fill folds (the rest of Alg. 3),
//                the hole-filled image and, with relabel, the label image (Alg. 4, fused);
//   relabel_ns = what runs after the emit pass: densified label ids (labeling.hpp:231-236);
//   total_ns   = the whole pipeline.
struct StepTimes {
    double encode_ns = 0;
    double unify_ns = 0;
    double closure_ns = 0;
    double relabel_ns = 0;
    double total_ns = 0;
};

namespace gpu {

// One C-ABI context per thread (SPEC: single-threaded per call, distinct images may be
// labeled concurrently).
class Context {
public:
    explicit Context(int device = 0) : ctx_(rl_create(device), &rl_destroy) {
        if (!ctx_) throw std::runtime_error("runlab_gpu: no usable CUDA device");
    }
    rl_ctx* get() const { return ctx_.get(); }

private:
    std::unique_ptr<rl_ctx, void (*)(rl_ctx*)> ctx_;
};

inline Context& thread_context() {
    thread_local Context ctx(0);
    return ctx;
}

[[noreturn]] inline void raise(int code, rl_ctx* ctx) {
    const std::string msg = rl_last_error(ctx);
    switch (code) {
        case RL_EINVAL: throw std::invalid_argument(msg);
        case RL_ELOGIC: throw std::logic_error(msg);
        case RL_EOVERFLOW: throw std::overflow_error(msg);
        case RL_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

inline FeatureAccumulator to_acc(const rl_features& f) {
    FeatureAccumulator a;
    a.s = f.s;
    a.sx = f.sx;
    a.sy = f.sy;
    a.row_min = f.row_min;
    a.row_max = f.row_max;
    a.col_min = f.col_min;
    a.col_max = f.col_max;
    return a;
}

inline rl_config to_c(const LabelingConfig& config) {
    rl_config c{};
    c.connectivity = config.connectivity == Connectivity::fg4_bg8 ? RL_FG4_BG8 : RL_FG8_BG4;
    c.fill_holes = config.fill_holes;
    c.compute_features = config.compute_features;
    c.relabel = config.relabel;
    c.densify_labels = config.densify_labels;
    c.compute_euler = config.compute_euler;
    return c;
}

// LabelingResult of one image from its canonical tables (ids in raster order of first pixel):
// pre-fill records, post-fill roots and their features, label image, counts.
inline LabelingResult assemble(std::int32_t width, std::int32_t height, const LabelingConfig& config, std::int64_t n,
                               const rl_component* comps, const std::uint32_t* top, const rl_features* filled,
                               const std::uint32_t* labels, std::int64_t n_fg, std::int64_t n_holes,
                               std::int64_t euler) {
    std::vector<label_t> t(static_cast<std::size_t>(n)), adj(static_cast<std::size_t>(n));
    std::vector<std::uint8_t> fg(static_cast<std::size_t>(n));
    for (std::int64_t e = 0; e < n; ++e) {
        t[e] = config.fill_holes ? top[e] : static_cast<label_t>(e);
        adj[e] = e == 0 ? no_label : comps[e].parent;
        fg[e] = static_cast<std::uint8_t>(comps[e].flags & 1u);
    }
    LabelingResult res;
    res.width = width;
    res.height = height;
    res.config = config;
    if (config.compute_features) {
        FeatureTable ft(static_cast<std::size_t>(n));
        for (std::int64_t e = 0; e < n; ++e)
            ft[e] = to_acc((config.fill_holes && top[e] == e) ? filled[e] : comps[e].f);
        res.features = std::move(ft);
    }
    if (config.relabel) {
        LabelImage li(width, height);
        std::copy(labels, labels + li.labels.size(), li.labels.begin());
        res.labels = std::move(li);
    }
    if (config.compute_euler) {
        res.fg_count = n_fg;
        res.hole_count = n_holes;
        res.euler = euler;
    }
    res.equivalences = EquivalenceTable(std::move(t), std::move(fg));
    res.adjacency = AdjacencyTable(std::move(adj));
    return res;
}

inline LabelingResult run(const BinaryImage& image, const LabelingConfig& config, StepTimes* times) {
    if (config.densify_labels && !config.relabel)
        throw std::invalid_argument("label_image: densify_labels requires relabel");
    rl_ctx* ctx = thread_context().get();
    const rl_config c = to_c(config);
    rl_result r{};
    const int rc = rl_label(ctx, image.pixels.data(), image.width, image.height, 1, &c, &r);
    if (rc != RL_OK) raise(rc, ctx);
    struct Free {
        rl_result* r;
        ~Free() { rl_result_free(r); }
    } guard{&r};
    LabelingResult res = assemble(image.width, image.height, config, r.n_components[0], r.comps, r.top, r.filled,
                                  r.labels, r.n_fg[0], r.n_holes[0], r.euler[0]);
    if (times) {
        times->encode_ns = r.times.analyze_ms * 1e6;
        times->unify_ns = r.times.merge_ms * 1e6;
        times->closure_ns = r.times.emit_ms * 1e6;
        times->relabel_ns = r.times.relabel_ms * 1e6;
        times->total_ns = r.times.total_ms * 1e6;
    }
    return res;
}

// One image across several GPUs of this process (one entry of `devices` per strip; a device may
// repeat): horizontal strips exchanging only the components that touch the cut rows
// (rl_label_strips_host).  The result equals label_image(image, config).
// densify_labels is not supported in strip mode (std::invalid_argument).
inline LabelingResult label_image_strips(const BinaryImage& image, const LabelingConfig& config,
                                         const std::vector<int>& devices) {
    if (devices.empty()) throw std::invalid_argument("label_image_strips: no devices");
    std::vector<Context> ctxs;
    ctxs.reserve(devices.size());
    for (int d : devices) ctxs.emplace_back(d);
    std::vector<rl_ctx*> raw;
    for (auto& c : ctxs) raw.push_back(c.get());
    const int k = static_cast<int>(raw.size());
    const rl_config c = to_c(config);
    std::vector<rl_strip_result> res(static_cast<std::size_t>(k));
    int rc = rl_label_strips_host(raw.data(), k, image.pixels.data(), image.width, image.height, &c, res.data());
    if (rc != RL_OK) raise(rc, raw[0]);
    const std::int64_t n = res[0].n_components;
    std::vector<rl_component> comps(static_cast<std::size_t>(n));
    std::vector<std::uint32_t> top(static_cast<std::size_t>(n));
    std::vector<rl_features> filled(static_cast<std::size_t>(n));
    std::vector<std::uint32_t> labels(config.relabel ? image.pixels.size() : 0);
    for (int r = 0; r < k; ++r) {
        rl_host_outputs o{};
        o.comps = comps.data() + res[r].comp_lo;
        o.top = top.data() + res[r].comp_lo;
        o.filled = filled.data() + res[r].comp_lo;
        o.comp_capacity = res[r].comp_hi - res[r].comp_lo;
        o.labels = config.relabel ? labels.data() + static_cast<std::size_t>(res[r].y0) * image.width : nullptr;
        if ((rc = rl_strip_fetch(raw[r], &res[r], &o)) != RL_OK) raise(rc, raw[r]);
    }
    return assemble(image.width, image.height, config, n, comps.data(), top.data(), filled.data(), labels.data(),
                    res[0].n_fg, res[0].n_holes, res[0].euler);
}

}  // namespace gpu

// labeling.hpp:336-339
inline LabelingResult label_image(const BinaryImage& image, const LabelingConfig& config = {}) {
    return gpu::run(image, config, nullptr);
}

// labeling.hpp:343-348
inline LabelingResult timed_label_image(const BinaryImage& image, const LabelingConfig& config, StepTimes& times) {
    times = {};
    return gpu::run(image, config, &times);
}

// labeling.hpp:354-360: foreground iff the label's parity is foreground
inline BinaryImage binarize_labels(const LabelImage& li, const EquivalenceTable& eq) {
    BinaryImage out(li.width, li.height);
    for (std::size_t i = 0; i < li.labels.size(); ++i) out.pixels[i] = eq.is_foreground(li.labels[i]) ? 1 : 0;
    return out;
}

// ---- analysis.hpp:13-79 projections over the result tables
struct ComponentRecord {
    label_t root = 0;
    bool foreground = false;
    label_t parent_root = no_label;
    std::int32_t depth = 0;
    FeatureAccumulator features;
};

inline std::vector<ComponentRecord> components(const LabelingResult& res) {
    const EquivalenceTable& eq = res.equivalences;
    std::vector<ComponentRecord> out;
    std::vector<std::int32_t> depth(eq.size(), 0);
    for (label_t e = 0; e < eq.size(); ++e) {
        if (!eq.is_root(e)) continue;
        ComponentRecord rec;
        rec.root = e;
        rec.foreground = eq.is_foreground(e);
        if (e != 0) {
            rec.parent_root = res.adjacency[e];
            depth[e] = depth[rec.parent_root] + 1;
        }
        rec.depth = depth[e];
        if (res.features) rec.features = (*res.features)[e];
        out.push_back(rec);
    }
    return out;
}

inline std::vector<ComponentRecord> holes(const LabelingResult& res) {
    if (res.config.fill_holes) throw std::logic_error("holes: result was computed with hole filling");
    std::vector<ComponentRecord> out;
    for (ComponentRecord& rec : components(res))
        if (!rec.foreground && rec.root != 0) out.push_back(rec);
    return out;
}

struct ComponentTree {
    std::vector<ComponentRecord> nodes;
    std::vector<std::vector<std::size_t>> children;
};

inline ComponentTree adjacency_tree(const LabelingResult& res) {
    ComponentTree tree;
    tree.nodes = components(res);
    tree.children.resize(tree.nodes.size());
    std::vector<std::size_t> index(res.equivalences.size(), 0);
    for (std::size_t i = 0; i < tree.nodes.size(); ++i) index[tree.nodes[i].root] = i;
    for (std::size_t i = 1; i < tree.nodes.size(); ++i)
        tree.children[index[tree.nodes[i].parent_root]].push_back(i);
    return tree;
}

inline std::int64_t euler_number(const LabelingResult& res) {
    if (!res.euler) throw std::logic_error("euler_number: labeling ran without compute_euler");
    return *res.euler;
}

// analysis.hpp:89-125 filter_components.  The predicate is evaluated on the host in the
// reference's order (ascending roots, skipped for a component whose surrounding component
// already merged); the merge itself -- targets by pointer jumping, feature folds, tree
// redirection -- runs on the GPU (rl_filter_components_host) over the table of roots, which for
// a hole-filled result holds only the post-fill roots.  Every label then follows its root.
template <class Predicate>
inline LabelingResult filter_components(const LabelingResult& res, Predicate&& selected) {
    const std::vector<ComponentRecord> recs = components(res);
    if (selected(static_cast<const ComponentRecord&>(recs[0])))
        throw std::invalid_argument("filter_components: predicate must not select the exterior");
    const std::size_t m = recs.size();
    const label_t n = res.equivalences.size();
    std::vector<label_t> index(n, no_label);  // root label -> position among the roots
    for (std::size_t k = 0; k < m; ++k) index[recs[k].root] = static_cast<label_t>(k);
    std::vector<rl_component> comps(m);
    std::vector<std::uint8_t> sel(m, 0), merged(m, 0);
    for (std::size_t k = 0; k < m; ++k) {
        const ComponentRecord& rec = recs[k];
        rl_component& c = comps[k];
        const FeatureAccumulator& f = rec.features;
        c.f = rl_features{f.s, f.sx, f.sy, f.row_min, f.row_max, f.col_min, f.col_max};
        c.flags = rec.foreground ? 1u : 0u;
        if (k == 0) {
            c.parent = no_label;
            continue;
        }
        const label_t pk = index[rec.parent_root];
        c.parent = pk;
        if (merged[pk]) {
            merged[k] = 1;  // embedded in a merged region: the predicate is not asked
        } else if (selected(static_cast<const ComponentRecord&>(rec))) {
            sel[k] = merged[k] = 1;
        }
    }
    std::vector<label_t> target(m), adj(m);
    std::vector<rl_features> feats(m);
    const int rc = rl_filter_components_host(comps.data(), static_cast<std::int64_t>(m), sel.data(), target.data(),
                                             feats.data(), adj.data());
    if (rc == RL_EINVAL) throw std::invalid_argument("filter_components: predicate must not select the exterior");
    if (rc != RL_OK) throw std::runtime_error("filter_components: GPU call failed");
    LabelingResult out = res;
    out.labels.reset();
    std::vector<label_t> t(n), adjacency(n);
    std::vector<std::uint8_t> fg(n);
    for (label_t e = 0; e < n; ++e) {
        const label_t r = res.equivalences.parent(e);  // a root: results are closed (flattened)
        const label_t k = index[r];
        t[e] = target[k] != k ? recs[target[k]].root : r;
        fg[e] = res.equivalences.is_foreground(e) ? 1 : 0;
        adjacency[e] = res.adjacency[e];
    }
    for (std::size_t k = 1; k < m; ++k)
        if (target[k] == k) adjacency[recs[k].root] = recs[adj[k]].root;
    out.equivalences = EquivalenceTable(std::move(t), std::move(fg));
    out.adjacency = AdjacencyTable(std::move(adjacency));
    if (out.features)
        for (std::size_t k = 0; k < m; ++k)
            if (target[k] == k) (*out.features)[recs[k].root] = gpu::to_acc(feats[k]);
    return out;
}

}  // namespace runlab
