// runlab_gpu_io.hpp -- the reference's I/O surface (runlab/io.hpp) over the B200 drop-in
// (include/runlab_gpu.hpp), SURVEY §8(f) rows 2 and 4.
//
//   read_pbm / read_pbm_file   io.hpp:74-124, header parsed by rl_pbm_parse (same rules and
//                              PbmParseError byte offsets), P1 text and P4 bits decoded here
//   write_pbm                  io.hpp:126-154 (P4 rows padded with zero bits; P1 lines <= 64)
//   fill_pbm                   `runlab fill` on the GPU: P4 raster decoded and encoded by the
//                              tile kernels (rl_fill_pbm)
//   write_label_image          io.hpp:156-183 (16-bit big-endian PGM or CSV)
//   write_features_csv         io.hpp:185-214
//   write_tree                 io.hpp:216-262 (nested JSON or DOT)
//
// Label values are the drop-in's canonical ids (rank of the component's raster-first pixel,
// exterior 0): the reference's root labels renumbered in ascending order.
#pragma once

#include <cstdint>
#include <fstream>
#include <iterator>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "runlab_gpu.hpp"

namespace runlab {

class PbmParseError : public std::runtime_error {
public:
    PbmParseError(const std::string& what, std::size_t offset)
        : std::runtime_error(what), byte_offset(offset) {}
    std::size_t byte_offset;
};

enum class PbmFormat { p1, p4 };
enum class LabelFormat { pgm16, csv };
enum class TreeFormat { json, dot };

namespace io_gpu {
inline rl_pbm_info parse(std::string_view bytes) {
    rl_pbm_info info{};
    const int rc = rl_pbm_parse(reinterpret_cast<const std::uint8_t*>(bytes.data()), bytes.size(), &info);
    if (rc == RL_EFORMAT) throw PbmParseError(info.message, static_cast<std::size_t>(info.error_offset));
    if (rc != RL_OK) throw std::invalid_argument("read_pbm: invalid arguments");
    return info;
}
}  // namespace io_gpu

inline BinaryImage read_pbm(std::string_view bytes) {
    rl_pbm_info info = io_gpu::parse(bytes);
    const std::int32_t w = info.width, h = info.height;
    const std::size_t rowb = (static_cast<std::size_t>(w) + 7) / 8;
    std::vector<std::uint8_t> rows;
    const std::uint8_t* p4 = reinterpret_cast<const std::uint8_t*>(bytes.data()) + info.raster_offset;
    if (info.format == 1) {
        rows.resize(rowb * static_cast<std::size_t>(h));
        const int rc = rl_pbm_p1_to_p4(reinterpret_cast<const std::uint8_t*>(bytes.data()), bytes.size(), &info,
                                       rows.data());
        if (rc == RL_EFORMAT) throw PbmParseError(info.message, static_cast<std::size_t>(info.error_offset));
        p4 = rows.data();
    }
    BinaryImage img(w, h);
    for (std::int32_t r = 0; r < h; ++r)
        for (std::int32_t j = 0; j < w; ++j)
            img.pixels[static_cast<std::size_t>(r) * w + j] = (p4[r * rowb + j / 8] >> (7 - j % 8)) & 1u;
    return img;
}

inline std::string write_pbm(const BinaryImage& img, PbmFormat format = PbmFormat::p4) {
    std::string out = (format == PbmFormat::p1 ? "P1\n" : "P4\n") + std::to_string(img.width) + " " +
                      std::to_string(img.height) + "\n";
    if (format == PbmFormat::p1) {
        std::int32_t line = 0;
        for (std::size_t i = 0; i < img.pixels.size(); ++i) {
            out += static_cast<char>('0' + (img.pixels[i] & 1));
            if (++line == 64 || (i + 1) % static_cast<std::size_t>(img.width) == 0) {
                out += '\n';
                line = 0;
            }
        }
        return out;
    }
    const std::size_t rowb = (static_cast<std::size_t>(img.width) + 7) / 8;
    for (std::int32_t r = 0; r < img.height; ++r) {
        std::string row(rowb, '\0');
        for (std::int32_t j = 0; j < img.width; ++j)
            if (img.pixels[static_cast<std::size_t>(r) * img.width + j])
                row[j / 8] = static_cast<char>(row[j / 8] | (0x80 >> (j % 8)));
        out += row;
    }
    return out;
}

// `runlab fill` (tools/runlab.cpp:128-137) in one GPU call: PBM bytes in, P4 file out
inline std::string fill_pbm(std::string_view bytes, Connectivity conn = Connectivity::fg8_bg4) {
    const rl_pbm_info head = io_gpu::parse(bytes);
    std::string out(64 + ((static_cast<std::size_t>(head.width) + 7) / 8) * head.height, '\0');
    rl_config cfg{};
    cfg.connectivity = conn == Connectivity::fg4_bg8 ? RL_FG4_BG8 : RL_FG8_BG4;
    cfg.fill_holes = 1;
    rl_pbm_info info{};
    std::size_t n = 0;
    rl_ctx* ctx = gpu::thread_context().get();
    const int rc = rl_fill_pbm(ctx, reinterpret_cast<const std::uint8_t*>(bytes.data()), bytes.size(), &cfg,
                               reinterpret_cast<std::uint8_t*>(out.data()), out.size(), &n, nullptr, &info);
    if (rc == RL_EFORMAT) throw PbmParseError(info.message, static_cast<std::size_t>(info.error_offset));
    if (rc != RL_OK) gpu::raise(rc, ctx);
    out.resize(n);
    return out;
}

inline std::string write_label_image(const LabelImage& li, LabelFormat format) {
    std::string out;
    if (format == LabelFormat::pgm16) {
        for (const label_t l : li.labels)
            if (l > 65535) throw std::overflow_error("write_label_image: label exceeds 16-bit PGM range; use csv");
        out = "P5\n" + std::to_string(li.width) + " " + std::to_string(li.height) + "\n65535\n";
        for (const label_t l : li.labels) {
            out += static_cast<char>((l >> 8) & 0xff);
            out += static_cast<char>(l & 0xff);
        }
        return out;
    }
    for (std::int32_t r = 0; r < li.height; ++r) {
        for (std::int32_t j = 0; j < li.width; ++j) {
            if (j) out += ',';
            out += std::to_string(li.labels[static_cast<std::size_t>(r) * li.width + j]);
        }
        out += '\n';
    }
    return out;
}

inline std::string write_features_csv(std::span<const ComponentRecord> records, bool with_dense = false) {
    std::string out = "root,parity,parent,s,sx,sy,rmin,rmax,cmin,cmax";
    out += with_dense ? ",dense\n" : "\n";
    for (std::size_t i = 0; i < records.size(); ++i) {
        const ComponentRecord& rec = records[i];
        const FeatureAccumulator& f = rec.features;
        out += std::to_string(rec.root) + (rec.foreground ? ",FG," : ",BG,");
        if (rec.parent_root != no_label) out += std::to_string(rec.parent_root);
        out += "," + std::to_string(f.s) + "," + std::to_string(f.sx) + "," + std::to_string(f.sy);
        if (f.empty())
            out += ",,,,";
        else
            out += "," + std::to_string(f.row_min) + "," + std::to_string(f.row_max) + "," +
                   std::to_string(f.col_min) + "," + std::to_string(f.col_max);
        if (with_dense) out += "," + std::to_string(i);
        out += '\n';
    }
    return out;
}

namespace io_gpu {
inline void json_node(const ComponentTree& tree, std::size_t i, std::string& out) {
    const ComponentRecord& rec = tree.nodes[i];
    const FeatureAccumulator& f = rec.features;
    out += "{\"label\":" + std::to_string(rec.root) + ",\"parity\":\"" + (rec.foreground ? "FG" : "BG") + "\"";
    out += ",\"s\":" + std::to_string(f.s) + ",\"sx\":" + std::to_string(f.sx) + ",\"sy\":" + std::to_string(f.sy);
    if (f.empty())
        out += ",\"bbox\":null";
    else
        out += ",\"bbox\":[" + std::to_string(f.row_min) + "," + std::to_string(f.row_max) + "," +
               std::to_string(f.col_min) + "," + std::to_string(f.col_max) + "]";
    out += ",\"children\":[";
    for (std::size_t k = 0; k < tree.children[i].size(); ++k) {
        if (k) out += ',';
        json_node(tree, tree.children[i][k], out);
    }
    out += "]}";
}
}  // namespace io_gpu

inline std::string write_tree(const ComponentTree& tree, TreeFormat format) {
    std::string out;
    if (format == TreeFormat::json) {
        io_gpu::json_node(tree, 0, out);
        return out + "\n";
    }
    out = "digraph components {\n";
    for (const ComponentRecord& rec : tree.nodes) out += "  " + std::to_string(rec.root) + ";\n";
    for (const ComponentRecord& rec : tree.nodes)
        if (rec.parent_root != no_label)
            out += "  " + std::to_string(rec.root) + " -> " + std::to_string(rec.parent_root) + ";\n";
    return out + "}\n";
}

inline std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open " + path);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

inline BinaryImage read_pbm_file(const std::string& path) { return read_pbm(read_file(path)); }

inline void write_file(const std::string& path, std::string_view bytes) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot write " + path);
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
}

}  // namespace runlab
