// dropin_test.cpp -- the reference's own known-answer tests, restated against the C++
// drop-in (include/runlab_gpu.hpp) running on the GPU.  Each check cites the reference test
// it mirrors (paths relative to /root/reference/proj/tests/).  Exit code = failures.
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <utility>
#include <string>
#include <vector>

#include "runlab_gpu.hpp"
#include "runlab_gpu_io.hpp"

using namespace runlab;

static int failures = 0;

#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static BinaryImage make_image(const std::vector<std::string>& rows) {
    BinaryImage img(static_cast<std::int32_t>(rows[0].size()), static_cast<std::int32_t>(rows.size()));
    for (std::int32_t r = 0; r < img.height; ++r)
        for (std::int32_t c = 0; c < img.width; ++c) img(r, c) = rows[r][c] == '1' ? 1 : 0;
    return img;
}

static LabelingConfig full_config() {
    LabelingConfig cfg;
    cfg.compute_features = true;
    cfg.compute_euler = true;
    cfg.relabel = true;
    return cfg;
}

static FeatureAccumulator acc(std::int64_t s, std::int64_t sx, std::int64_t sy, std::int32_t rmin, std::int32_t rmax,
                              std::int32_t cmin, std::int32_t cmax) {
    FeatureAccumulator f;
    f.s = s;
    f.sx = sx;
    f.sy = sy;
    f.row_min = rmin;
    f.row_max = rmax;
    f.col_min = cmin;
    f.col_max = cmax;
    return f;
}

// The filtering rule of analysis.hpp:89-125, written out over the drop-in's own types as the
// test's independent expectation: ascending roots, a component merges into its surrounding
// component's target when that one merged, else into its surrounding component when selected.
template <class Pred>
static std::pair<std::vector<label_t>, FeatureTable> expected_filter(const LabelingResult& res, Pred pred) {
    const auto recs = components(res);
    std::vector<label_t> dest(res.equivalences.size(), no_label);
    FeatureTable f = *res.features;
    for (std::size_t i = 1; i < recs.size(); ++i) {
        const label_t up = dest[recs[i].parent_root];
        const label_t to = up != no_label ? up : (pred(recs[i]) ? recs[i].parent_root : no_label);
        if (to == no_label) continue;
        dest[recs[i].root] = to;
        merge_into(f[to], f[recs[i].root]);
    }
    std::vector<label_t> parent(res.equivalences.size());
    for (label_t e = 0; e < parent.size(); ++e) {
        const label_t r = res.equivalences.parent(e);
        parent[e] = dest[r] != no_label ? dest[r] : r;
    }
    return {parent, f};
}

static std::vector<label_t> parents_of(const EquivalenceTable& eq) {
    std::vector<label_t> p(eq.size());
    for (label_t e = 0; e < eq.size(); ++e) p[e] = eq.parent(e);
    return p;
}

int main() {
    // test_core.cpp:30-78 feature algebra and tables (host code of the drop-in)
    {
        const auto a = acc(3, 6, 6, 2, 2, 1, 3), b = acc(2, 9, 6, 3, 3, 4, 5);
        CHECK(merge_features(a, b) == acc(5, 15, 12, 2, 3, 1, 5));
        CHECK(merge_features(b, a) == merge_features(a, b));
        CHECK(merge_features(a, a) == acc(6, 12, 12, 2, 2, 1, 3));
        const auto c = acc(5, 4, 40, 3, 3, 7, 7);
        CHECK(merge_features(merge_features(a, b), c) == merge_features(a, merge_features(b, c)));
        bool threw = false;
        try {
            auto big = acc(1, std::numeric_limits<std::int64_t>::max(), 0, 0, 0, 0, 0);
            merge_into(big, acc(1, 1, 0, 0, 0, 0, 0));
        } catch (const std::overflow_error&) {
            threw = true;
        }
        CHECK(threw);
        CHECK(segment_features(2, 1, 4) == acc(3, 6, 6, 2, 2, 1, 3));
        CHECK(segment_features(0, 0, 1) == acc(1, 0, 0, 0, 0, 0, 0));
        CHECK(segment_features(5, 4, 11) == acc(7, 49, 35, 5, 5, 4, 10));
        EquivalenceTable eq;
        CHECK(eq.size() == 1 && !eq.is_foreground(0));
        CHECK(eq.make_label(true) == 1 && eq.make_label(false) == 2 && eq.make_label(true) == 3);
        eq.set_parent(2, 0);
        eq.set_parent(3, 2);
        CHECK(eq.find(3) == 0 && eq.parent(3) == 2 && eq.find(0) == 0);
        EquivalenceTable u;
        for (int i = 0; i < 4; ++i) u.make_label(true);
        CHECK(u.union_min(4, 1) == 1 && u.parent(4) == 1 && u.find(4) == 1);
        CHECK(u.union_min(2, 3) == 2 && u.parent(3) == 2 && u.union_min(2, 2) == 2);
        u.attach_to_exterior(3);
        CHECK(u.find(3) == 0 && u.parent(2) == 0);
        CHECK(u.is_foreground(1) && !eq.is_foreground(2));
        AdjacencyTable adj;
        CHECK(adj.size() == 1 && adj[0] == no_label);
        adj.push(0);
        CHECK(adj[1] == 0);
        adj.push(1);
        adj.redirect(2, 0);
        CHECK(adj[2] == 0 && adj.size() == 3);
        BinaryImage img = make_image({"010", "110"});
        CHECK(img.row(1).size() == 3 && img.row(1)[0] == 1 && img.row(1)[2] == 0 && img.row(0)[1] == 1);
    }
    const BinaryImage fig = make_image({"011111111111110", "010000010000010", "010111010111010",
                                        "010101000101010", "010101111101010", "010100000001000",
                                        "011111111111110"});
    // test_labeling.cpp:107-134 "golden example: end-to-end result" (roots 0,1,6 -> 0,1,2)
    {
        const LabelingResult res = label_image(fig, full_config());
        CHECK(*res.fg_count == 1);
        CHECK(*res.hole_count == 1);
        CHECK(*res.euler == 0);
        CHECK((res.roots() == std::vector<label_t>{0, 1, 2}));
        CHECK(res.adjacency[2] == 1 && res.adjacency[1] == 0);
        const FeatureAccumulator& fg = (*res.features)[1];
        CHECK(fg.s == 56 && fg.row_min == 0 && fg.row_max == 6 && fg.col_min == 1 && fg.col_max == 13);
        const FeatureAccumulator& hole = (*res.features)[2];
        CHECK(hole.s == 11 && hole.row_min == 3 && hole.row_max == 5 && hole.col_min == 4 && hole.col_max == 10);
        CHECK((*res.features)[0].s == 38);
        std::vector<label_t> row3(res.labels->labels.begin() + 45, res.labels->labels.begin() + 60);
        CHECK((row3 == std::vector<label_t>{0, 1, 0, 1, 2, 1, 0, 0, 0, 1, 2, 1, 0, 1, 0}));
        // analysis.hpp projections
        CHECK(holes(res).size() == 1);
        CHECK(adjacency_tree(res).children[0].size() == 1);
        CHECK(euler_number(res) == 0);
    }
    // test_labeling.cpp:136-148 "golden example: hole filled end-to-end"
    {
        LabelingConfig cfg = full_config();
        cfg.fill_holes = true;
        const LabelingResult res = label_image(fig, cfg);
        CHECK((res.roots() == std::vector<label_t>{0, 1}));
        CHECK((*res.features)[1].s == 67);
        CHECK(*res.euler == 0);
        std::vector<label_t> row3(res.labels->labels.begin() + 45, res.labels->labels.begin() + 60);
        CHECK((row3 == std::vector<label_t>{0, 1, 0, 1, 1, 1, 0, 0, 0, 1, 1, 1, 0, 1, 0}));
        const BinaryImage filled = binarize_labels(*res.labels, res.equivalences);
        CHECK(filled(3, 4) == 1 && filled(3, 2) == 0);
        bool threw = false;
        try {
            holes(res);
        } catch (const std::logic_error&) {
            threw = true;
        }
        CHECK(threw);
    }
    // test_labeling.cpp:178-190 ring-hole-dot collapses; test_analysis.cpp:103-110 depth 3
    {
        const BinaryImage rhd = make_image({"0000000", "0111110", "0100010", "0101010", "0100010", "0111110", "0000000"});
        LabelingConfig cfg = full_config();
        const ComponentTree tree = adjacency_tree(label_image(rhd, cfg));
        CHECK(tree.nodes.size() == 4 && tree.nodes[3].depth == 3);
        cfg.fill_holes = true;
        const LabelingResult res = label_image(rhd, cfg);
        CHECK((res.roots() == std::vector<label_t>{0, 1}));
        CHECK((*res.features)[1].s == 25);
    }
    // test_labeling.cpp:192-203 misuse
    {
        LabelingConfig bad;
        bad.densify_labels = true;
        bool threw = false;
        try {
            label_image(make_image({"0"}), bad);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        bool threw2 = false;
        try {
            euler_number(label_image(make_image({"1"}), {}));
        } catch (const std::logic_error&) {
            threw2 = true;
        }
        CHECK(threw2);
    }
    // test_labeling.cpp:217-230 diagonal pair depends on the convention
    {
        const BinaryImage img = make_image({"10", "01"});
        LabelingConfig cfg;
        cfg.compute_euler = true;
        CHECK(*label_image(img, cfg).euler == 1);
        cfg.connectivity = Connectivity::fg4_bg8;
        const LabelingResult res = label_image(img, cfg);
        CHECK(*res.fg_count == 2 && *res.euler == 2);
    }
    // test_analysis.cpp:146-210: filtering the holes equals hole filling; exterior rejected
    {
        LabelingConfig cfg = full_config();
        cfg.relabel = false;
        const LabelingResult res = label_image(fig, cfg);
        const LabelingResult f = filter_components(
            res, [](const ComponentRecord& r) { return !r.foreground && r.root != 0; });
        cfg.fill_holes = true;
        const LabelingResult filled_res = label_image(fig, cfg);
        CHECK(f.roots() == filled_res.roots());
        for (label_t e : f.roots()) CHECK((*f.features)[e].s == (*filled_res.features)[e].s);
        CHECK((*f.features)[1].s == 67 && !f.labels);
        bool threw = false;
        try {
            filter_components(res, [](const ComponentRecord& r) { return r.root == 0; });
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // test_analysis.cpp:146-210 more: small holes, a lone dot, always-false, the predicate's call
    // order, and filtering a hole-filled result (the reference accepts any closed result)
    {
        LabelingConfig cfg;
        cfg.compute_features = true;
        cfg.compute_euler = true;
        const LabelingResult base = label_image(fig, cfg);
        auto small_bg = [](const ComponentRecord& r) { return !r.foreground && r.root != 0 && r.features.s < 20; };
        const LabelingResult f = filter_components(base, small_bg);
        LabelingConfig fc = cfg;
        fc.fill_holes = true;
        const LabelingResult filled = label_image(fig, fc);
        CHECK(parents_of(f.equivalences) == parents_of(filled.equivalences));
        for (label_t e : f.roots()) CHECK((*f.features)[e] == (*filled.features)[e]);
        const LabelingResult same = filter_components(base, [](const ComponentRecord&) { return false; });
        CHECK(parents_of(same.equivalences) == parents_of(base.equivalences) && *same.features == *base.features);
        const BinaryImage dot = make_image({"000", "010", "000"});
        const LabelingResult gone = filter_components(label_image(dot, cfg), [](const ComponentRecord& r) {
            return r.foreground && r.features.s < 2;
        });
        CHECK((gone.roots() == std::vector<label_t>{0}) && (*gone.features)[0].s == 9);
        // ring-hole-dot: selecting the ring merges everything inside it; the predicate is asked
        // about the ring, not about the hole and dot embedded in it
        const BinaryImage rhd = make_image({"0000000", "0111110", "0100010", "0101010", "0100010", "0111110", "0000000"});
        const LabelingResult r0 = label_image(rhd, cfg);
        std::vector<label_t> asked;
        auto ring = [&](const ComponentRecord& r) {
            asked.push_back(r.root);
            return r.root == 1;
        };
        const LabelingResult rf = filter_components(r0, ring);
        CHECK((asked == std::vector<label_t>{0, 1}));
        CHECK((rf.roots() == std::vector<label_t>{0}) && (*rf.features)[0].s == 49);
        // a hole-filled result: the table of post-fill roots is filtered, every label follows
        for (const std::uint64_t seed : {71ull, 72ull, 73ull}) {
            BinaryImage img(26, 22);
            std::uint64_t x = seed * 0x9E3779B97F4A7C15ull;
            for (auto& px : img.pixels) {
                x ^= x << 13, x ^= x >> 7, x ^= x << 17;
                px = (x >> 33) % 10 < 6;
            }
            const LabelingResult fr = label_image(img, fc);
            auto odd = [](const ComponentRecord& r) { return r.root % 2 == 1 && r.features.s < 30; };
            const LabelingResult got = filter_components(fr, odd);
            const auto [want_parent, want_feat] = expected_filter(fr, odd);
            CHECK(parents_of(got.equivalences) == want_parent);
            for (label_t e : got.roots()) CHECK((*got.features)[e] == want_feat[e]);
            const LabelingResult nf = label_image(img, cfg);
            auto holes_only = [](const ComponentRecord& r) { return !r.foreground && r.root != 0; };
            const LabelingResult g2 = filter_components(nf, holes_only);
            const auto [p2, f2] = expected_filter(nf, holes_only);
            CHECK(parents_of(g2.equivalences) == p2);
            for (label_t e : g2.roots()) CHECK((*g2.features)[e] == f2[e]);
            std::int64_t mass = 0;
            for (label_t e : g2.roots()) mass += (*g2.features)[e].s;
            CHECK(mass == img.pixel_count());
        }
    }
    // test_io.cpp:64-132 restated with canonical ids (the Fig. 3 hole is component 2, the
    // reference's provisional root label is 6)
    {
        LabelImage li(1, 1);
        CHECK(write_label_image(li, LabelFormat::pgm16) == std::string("P5\n1 1\n65535\n") + '\0' + '\0');
        li.labels[0] = 0x0102;
        const std::string two = write_label_image(li, LabelFormat::pgm16);
        CHECK(two.substr(two.size() - 2) == std::string("\x01\x02"));
        li.labels[0] = 65536;
        bool threw = false;
        try {
            write_label_image(li, LabelFormat::pgm16);
        } catch (const std::overflow_error&) {
            threw = true;
        }
        CHECK(threw);
        LabelingConfig cfg;
        cfg.relabel = true;
        cfg.fill_holes = true;
        const std::string csv = write_label_image(*label_image(fig, cfg).labels, LabelFormat::csv);
        std::size_t pos = 0;
        for (int skip = 0; skip < 3; ++skip) pos = csv.find('\n', pos) + 1;
        CHECK(csv.substr(pos, csv.find('\n', pos) - pos) == "0,1,0,1,1,1,0,0,0,1,1,1,0,1,0");
        LabelingConfig fc;
        fc.compute_features = true;
        const auto recs = components(label_image(fig, fc));
        const std::string fcsv = write_features_csv(recs);
        CHECK(fcsv.substr(0, fcsv.find('\n')) == "root,parity,parent,s,sx,sy,rmin,rmax,cmin,cmax");
        CHECK(fcsv.find("\n1,FG,0,56,") != std::string::npos);
        CHECK(fcsv.find("\n2,BG,1,11,") != std::string::npos);
        CHECK(fcsv.substr(fcsv.find('\n') + 1, 5) == "0,BG,");
        const std::string dense = write_features_csv(recs, true);
        CHECK(dense.substr(0, dense.find('\n')) == "root,parity,parent,s,sx,sy,rmin,rmax,cmin,cmax,dense");
        const ComponentTree tree = adjacency_tree(label_image(fig, fc));
        CHECK(write_tree(tree, TreeFormat::dot) == "digraph components {\n  0;\n  1;\n  2;\n  1 -> 0;\n  2 -> 1;\n}\n");
        const std::string json = write_tree(tree, TreeFormat::json);
        CHECK(json.find("\"label\":1") != std::string::npos && json.find("\"s\":56") != std::string::npos);
        CHECK(json.find("\"bbox\":[3,5,4,10]") != std::string::npos);
        const ComponentTree empty = adjacency_tree(label_image(make_image({"00", "00"}), fc));
        CHECK(write_tree(empty, TreeFormat::json) ==
              "{\"label\":0,\"parity\":\"BG\",\"s\":4,\"sx\":2,\"sy\":2,\"bbox\":[0,1,0,1],\"children\":[]}\n");
        // PBM round trips and the device fill path (`runlab fill`)
        CHECK(read_pbm(write_pbm(fig, PbmFormat::p1)) == fig && read_pbm(write_pbm(fig, PbmFormat::p4)) == fig);
        LabelingConfig fl;
        fl.fill_holes = true;
        fl.relabel = true;
        const LabelingResult fr = label_image(fig, fl);
        CHECK(fill_pbm(write_pbm(fig, PbmFormat::p4)) == write_pbm(binarize_labels(*fr.labels, fr.equivalences)));
        bool threw2 = false;
        try {
            read_pbm("P4\n9 2\n\x80\xff");
        } catch (const PbmParseError& e) {
            threw2 = e.byte_offset == 9;
        }
        CHECK(threw2);
    }
    // timed_label_image gives identical results (test_bench.cpp:31-60)
    {
        StepTimes t;
        const LabelingResult a = timed_label_image(fig, full_config(), t);
        const LabelingResult b = label_image(fig, full_config());
        CHECK(*a.labels == *b.labels && t.total_ns > 0);
    }
    // one image as horizontal strips over several contexts (rl_label_strips_host) == label_image
    {
        BinaryImage big(700, 300);
        std::uint64_t x = 12345;
        for (auto& p : big.pixels) {  // blocky noise with holes crossing the strip cuts
            x = x * 6364136223846793005ull + 1442695040888963407ull;
            p = (x >> 61) < 4 ? 1 : 0;
        }
        for (int y = 40; y < 260; ++y)  // a ring around the cuts
            for (int c = 40; c < 660; ++c)
                if (y < 44 || y >= 256 || c < 44 || c >= 656) big.pixels[y * 700 + c] = 1;
        for (bool fill : {false, true}) {
            LabelingConfig cfg = full_config();
            cfg.fill_holes = fill;
            cfg.relabel = !fill;
            const LabelingResult a = label_image(big, cfg);
            for (int k : {1, 3, 5}) {
                const LabelingResult b = gpu::label_image_strips(big, cfg, std::vector<int>(k, 0));
                CHECK(b.equivalences.size() == a.equivalences.size());
                CHECK(parents_of(b.equivalences) == parents_of(a.equivalences));
                bool same_adj = b.adjacency.size() == a.adjacency.size();
                for (label_t e = 0; same_adj && e < a.adjacency.size(); ++e) same_adj = a.adjacency[e] == b.adjacency[e];
                CHECK(same_adj);
                CHECK(*b.features == *a.features);
                CHECK(*b.euler == *a.euler && *b.fg_count == *a.fg_count && *b.hole_count == *a.hole_count);
                if (!fill) CHECK(*b.labels == *a.labels);
            }
        }
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures;
}
