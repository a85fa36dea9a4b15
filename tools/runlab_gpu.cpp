// runlab_gpu -- the reference CLI's subcommands (tools/runlab.cpp:57-275: label, tree, euler,
// fill, gen, bench) over the B200 drop-in (include/runlab_gpu.hpp, include/runlab_gpu_io.hpp,
// include/runlab_gpu_bench.hpp), with a small hand-written argument parser (CLI11 is not
// available).
//
//   runlab_gpu label IN.pbm [-o OUT.pgm|OUT.csv] [--features-csv F.csv] [--features]
//                    [--relabel] [--densify] [--fill] [--connectivity fg8bg4|fg4bg8]
//   runlab_gpu tree IN.pbm [-o OUT] [--format dot|json] [--fill] [--connectivity ...]
//   runlab_gpu euler IN.pbm [--connectivity ...]
//   runlab_gpu fill IN.pbm OUT.pbm [--format p4|p1] [--connectivity ...]
//   runlab_gpu gen OUT.pbm --size N | --width W --height H [--density D] [--granularity G]
//                    [--seed S] [--format p4|p1]
//   runlab_gpu bench [--size N] [--densities A:B:STEP|D1,D2,..] [--granularities G1,G2,..]
//                    [--seeds K] [--seed S] [--warmup W] [--iters I] [--clock-ghz F] [-o OUT.csv]
//                    [--no-euler] [--no-fill] [--no-features] [--no-relabel] [--connectivity ...]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "runlab_gpu_bench.hpp"
#include "runlab_gpu_io.hpp"

using namespace runlab;

namespace {

struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    std::map<std::string, bool> flag;
};

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr, "runlab_gpu: %s\nsubcommands: label tree euler fill gen bench (see tools/runlab_gpu.cpp)\n", msg);
    std::exit(2);
}

Args parse(int argc, char** argv, const std::vector<std::string>& flags, const std::vector<std::string>& opts) {
    Args a;
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s == "-o") s = "--output";
        if (s.rfind("--", 0) == 0) {
            bool known = false;
            for (const auto& f : flags)
                if (s == f) a.flag[f] = known = true;
            for (const auto& o : opts)
                if (s == o) {
                    if (i + 1 >= argc) usage(("missing value for " + s).c_str());
                    a.opt[o] = argv[++i];
                    known = true;
                }
            if (!known) usage(("unknown option " + s).c_str());
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

Connectivity conn_of(const Args& a) {
    const auto it = a.opt.find("--connectivity");
    if (it == a.opt.end() || it->second == "fg8bg4") return Connectivity::fg8_bg4;
    if (it->second == "fg4bg8") return Connectivity::fg4_bg8;
    usage("--connectivity must be fg8bg4 or fg4bg8");
}

bool ends_with(const std::string& s, const std::string& t) {
    return s.size() >= t.size() && s.compare(s.size() - t.size(), t.size(), t) == 0;
}

void emit(const std::string& path, const std::string& text) {
    if (path.empty())
        std::fwrite(text.data(), 1, text.size(), stdout);
    else
        write_file(path, text);
}

int cmd_label(const Args& a) {
    if (a.pos.size() != 1) usage("label: one input file");
    const std::string out = a.opt.count("--output") ? a.opt.at("--output") : "";
    const std::string fcsv = a.opt.count("--features-csv") ? a.opt.at("--features-csv") : "";
    LabelingConfig cfg;
    cfg.connectivity = conn_of(a);
    cfg.fill_holes = a.flag.count("--fill") > 0;
    cfg.compute_euler = true;
    cfg.compute_features = a.flag.count("--features") > 0 || !fcsv.empty();
    cfg.relabel = a.flag.count("--relabel") > 0 || !out.empty();
    cfg.densify_labels = a.flag.count("--densify") > 0;
    const LabelingResult res = label_image(read_pbm_file(a.pos[0]), cfg);
    if (!out.empty()) write_file(out, write_label_image(*res.labels, ends_with(out, ".csv") ? LabelFormat::csv : LabelFormat::pgm16));
    if (!fcsv.empty()) write_file(fcsv, write_features_csv(components(res), cfg.densify_labels));
    std::printf("foreground components: %lld\nholes: %lld\neuler: %lld\n", (long long)*res.fg_count,
                (long long)*res.hole_count, (long long)*res.euler);
    return 0;
}

int cmd_tree(const Args& a) {
    if (a.pos.size() != 1) usage("tree: one input file");
    LabelingConfig cfg;
    cfg.connectivity = conn_of(a);
    cfg.fill_holes = a.flag.count("--fill") > 0;
    cfg.compute_features = true;
    const std::string fmt = a.opt.count("--format") ? a.opt.at("--format") : "dot";
    if (fmt != "dot" && fmt != "json") usage("--format must be dot or json");
    const ComponentTree tree = adjacency_tree(label_image(read_pbm_file(a.pos[0]), cfg));
    emit(a.opt.count("--output") ? a.opt.at("--output") : "", write_tree(tree, fmt == "json" ? TreeFormat::json : TreeFormat::dot));
    return 0;
}

int cmd_euler(const Args& a) {
    if (a.pos.size() != 1) usage("euler: one input file");
    LabelingConfig cfg;
    cfg.connectivity = conn_of(a);
    cfg.compute_euler = true;
    std::printf("%lld\n", (long long)euler_number(label_image(read_pbm_file(a.pos[0]), cfg)));
    return 0;
}

int cmd_fill(const Args& a) {
    if (a.pos.size() != 2) usage("fill: input and output files");
    const std::string fmt = a.opt.count("--format") ? a.opt.at("--format") : "p4";
    if (fmt == "p4") {  // the device P4 path end to end
        write_file(a.pos[1], fill_pbm(read_file(a.pos[0]), conn_of(a)));
        return 0;
    }
    if (fmt != "p1") usage("--format must be p4 or p1");
    LabelingConfig cfg;
    cfg.connectivity = conn_of(a);
    cfg.fill_holes = true;
    cfg.relabel = true;
    const LabelingResult res = label_image(read_pbm_file(a.pos[0]), cfg);
    write_file(a.pos[1], write_pbm(binarize_labels(*res.labels, res.equivalences), PbmFormat::p1));
    return 0;
}

int cmd_gen(const Args& a) {
    if (a.pos.size() != 1) usage("gen: one output file");
    auto num = [&](const char* k, const char* d) { return a.opt.count(k) ? a.opt.at(k) : std::string(d); };
    const int size = std::atoi(num("--size", "0").c_str());
    const int w = a.opt.count("--width") ? std::atoi(a.opt.at("--width").c_str()) : size;
    const int h = a.opt.count("--height") ? std::atoi(a.opt.at("--height").c_str()) : size;
    const double d = std::atof(num("--density", "0.5").c_str());
    const int g = std::atoi(num("--granularity", "1").c_str());
    const unsigned long long seed = std::strtoull(num("--seed", "0").c_str(), nullptr, 10);
    if (w < 1 || h < 1) usage("gen: --size or --width/--height required");
    BinaryImage img(w, h);
    if (rl_generate_host(img.pixels.data(), w, h, d, g, seed) != RL_OK)  // generator.hpp:46-83 on the device
        usage("gen: invalid generator spec or no CUDA device");
    const std::string fmt = num("--format", "p4");
    write_file(a.pos[0], write_pbm(img, fmt == "p1" ? PbmFormat::p1 : PbmFormat::p4));
    return 0;
}

// tools/runlab.cpp:33-55: "start:stop:step" (inclusive, the step accumulated as the reference's
// CLI does) or a comma list; every value in [0, 1]
std::vector<double> parse_densities(const std::string& text) {
    std::vector<double> out;
    if (text.find(':') != std::string::npos) {
        double a = 0, b = 0, step = 0;
        if (std::sscanf(text.c_str(), "%lf:%lf:%lf", &a, &b, &step) != 3 || step <= 0)
            usage("--densities: expected start:stop:step");
        for (double d = a; d <= b + 1e-9; d += step) out.push_back(std::min(d, 1.0));
    } else {
        for (std::size_t pos = 0; pos <= text.size();) {
            const std::size_t comma = std::min(text.find(',', pos), text.size());
            out.push_back(std::atof(text.substr(pos, comma - pos).c_str()));
            pos = comma + 1;
        }
    }
    for (const double d : out)
        if (d < 0 || d > 1) usage("--densities: values must be in [0, 1]");
    return out;
}

// tools/runlab.cpp:158-172 + 245-275: the sweep as a CSV report
int cmd_bench(const Args& a) {
    if (!a.pos.empty()) usage("bench: no positional arguments");
    auto num = [&](const char* k, const char* d) { return a.opt.count(k) ? a.opt.at(k) : std::string(d); };
    BenchSpec spec;
    spec.width = spec.height = std::atoi(num("--size", "2048").c_str());
    spec.densities = parse_densities(num("--densities", "0:1:0.05"));
    const std::string gl = num("--granularities", "1,2,4,8,16");
    for (std::size_t pos = 0; pos <= gl.size();) {
        const std::size_t comma = std::min(gl.find(',', pos), gl.size());
        spec.granularities.push_back(std::atoi(gl.substr(pos, comma - pos).c_str()));
        pos = comma + 1;
    }
    spec.seeds = std::atoi(num("--seeds", "5").c_str());
    spec.base_seed = std::strtoull(num("--seed", "1").c_str(), nullptr, 10);
    spec.warmup = std::atoi(num("--warmup", "1").c_str());
    spec.iterations = std::atoi(num("--iters", "3").c_str());
    spec.clock_ghz = std::atof(num("--clock-ghz", "0").c_str());
    spec.report_cpp = spec.clock_ghz > 0;
    spec.connectivity = conn_of(a);
    spec.measure_euler = !a.flag.count("--no-euler");
    spec.measure_fill = !a.flag.count("--no-fill");
    spec.measure_features = !a.flag.count("--no-features");
    spec.measure_relabel = !a.flag.count("--no-relabel");
    emit(a.opt.count("--output") ? a.opt.at("--output") : "", export_csv(run(spec)));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) usage("a subcommand is required");
    const std::string cmd = argv[1];
    try {
        if (cmd == "label")
            return cmd_label(parse(argc, argv, {"--features", "--relabel", "--densify", "--fill"},
                                   {"--output", "--features-csv", "--connectivity"}));
        if (cmd == "tree") return cmd_tree(parse(argc, argv, {"--fill"}, {"--output", "--format", "--connectivity"}));
        if (cmd == "euler") return cmd_euler(parse(argc, argv, {}, {"--connectivity"}));
        if (cmd == "fill") return cmd_fill(parse(argc, argv, {}, {"--format", "--connectivity"}));
        if (cmd == "bench")
            return cmd_bench(parse(argc, argv, {"--no-euler", "--no-fill", "--no-features", "--no-relabel"},
                                   {"--size", "--densities", "--granularities", "--seeds", "--seed", "--warmup",
                                    "--iters", "--clock-ghz", "--output", "--connectivity"}));
        if (cmd == "gen")
            return cmd_gen(parse(argc, argv, {},
                                 {"--size", "--width", "--height", "--density", "--granularity", "--seed", "--format"}));
    } catch (const PbmParseError& e) {
        std::fprintf(stderr, "runlab_gpu: %s\n", e.what());  // the message carries the byte offset
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "runlab_gpu: %s\n", e.what());
        return 1;
    }
    usage(("unknown subcommand " + cmd).c_str());
}
