// msplat C++ drop-in: extended-PLY scene I/O over the C ABI (the payload is
// transposed AoS <-> SoA on the device), plus the xyz+rgb point-cloud files of
// io_ply.cpp:265-323 (host I/O, same format and messages).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <sstream>

#include "device_common.hpp"
#include "msplat/io_ply.hpp"

namespace msplat {

using namespace dropin;

namespace {

void packed_layout(int64_t n, int C, int deg, int64_t off[8]) { rethrow(msplat_param_layout(n, C, deg, off)); }

}  // namespace

void save_scene_ply(const std::string& path, const Scene& scene) {
    scene.validate();
    const int64_t n = int64_t(scene.size());
    const int C = scene.num_classes, deg = scene.sh_degree, K = scene.sh_coeff_count();
    int64_t off[8];
    packed_layout(n, C, deg, off);
    std::vector<double> f(size_t(std::max<int64_t>(off[7], 1)));
    for (size_t i = 0; i < scene.size(); ++i) {
        const GaussianPrimitive& g = scene.gaussians[i];
        for (int j = 0; j < 3; ++j) {
            f[off[0] + 3 * i + j] = g.position[j];
            f[off[2] + 3 * i + j] = g.log_scale[j];
        }
        for (int j = 0; j < 4; ++j) f[off[1] + 4 * i + j] = g.rotation[j];
        f[off[3] + i] = g.opacity_logit;
        f[off[4] + i] = g.gradient_factor;
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j) f[off[5] + (3 * i + c) * K + j] = g.sh(c, j);
        for (int c = 0; c < C; ++c) f[off[6] + i * C + c] = g.semantic_logits[c];
    }
    DBuf d(f.size(), false);
    d.upload(f);
    rethrow(msplat_save_scene_ply(context(), path.c_str(), MSPLAT_F64, n, C, deg, d.p));
}

Scene load_scene_ply(const std::string& path) {
    int64_t n = 0;
    int C = 0, deg = 0;
    rethrow(msplat_ply_scene_info(path.c_str(), &n, &C, &deg));
    int64_t off[8];
    packed_layout(n, C, deg, off);
    DBuf d(size_t(std::max<int64_t>(off[7], 1)), false);
    rethrow(msplat_load_scene_ply(context(), path.c_str(), MSPLAT_F64, d.p));
    const std::vector<double> f = d.download();
    const int K = (deg + 1) * (deg + 1);
    Scene s;
    s.num_classes = C;
    s.sh_degree = deg;
    s.gaussians.resize(size_t(n));
    for (size_t i = 0; i < size_t(n); ++i) {
        GaussianPrimitive& g = s.gaussians[i];
        g.position = Vec3(f[off[0] + 3 * i], f[off[0] + 3 * i + 1], f[off[0] + 3 * i + 2]);
        g.rotation = Vec4(f[off[1] + 4 * i], f[off[1] + 4 * i + 1], f[off[1] + 4 * i + 2], f[off[1] + 4 * i + 3]);
        g.log_scale = Vec3(f[off[2] + 3 * i], f[off[2] + 3 * i + 1], f[off[2] + 3 * i + 2]);
        g.opacity_logit = f[off[3] + i];
        g.gradient_factor = f[off[4] + i];
        g.sh = ShMatrix::Zero(3, K);
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < K; ++j) g.sh(c, j) = f[off[5] + (3 * i + c) * K + j];
        g.semantic_logits = VecX::Zero(C);
        for (int c = 0; c < C; ++c) g.semantic_logits[c] = f[off[6] + i * C + c];
    }
    return s;
}

// io_ply.cpp:265-292
void save_points_ply(const std::string& path, const std::vector<Vec3>& points, const std::vector<Vec3>& colors) {
    if (points.size() != colors.size()) throw std::invalid_argument("save_points_ply: point/color count mismatch");
    FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) throw std::runtime_error(path + ": cannot open for writing");
    const std::string hdr = "ply\nformat binary_little_endian 1.0\nelement vertex " + std::to_string(points.size()) +
                            "\nproperty double x\nproperty double y\nproperty double z\n"
                            "property uchar red\nproperty uchar green\nproperty uchar blue\nend_header\n";
    bool ok = std::fwrite(hdr.data(), 1, hdr.size(), f) == hdr.size();
    for (size_t i = 0; ok && i < points.size(); ++i) {
        const double xyz[3] = {points[i].x(), points[i].y(), points[i].z()};
        ok = std::fwrite(xyz, 8, 3, f) == 3;
        for (int c = 0; ok && c < 3; ++c) {
            const double v = std::clamp(colors[i][c], Scalar(0), Scalar(1));
            const uint8_t b = uint8_t(std::lround(v * 255.0));
            ok = std::fwrite(&b, 1, 1, f) == 1;
        }
    }
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw std::runtime_error(path + ": write failed");
}

// io_ply.cpp:294-321 for the files save_points_ply writes (double xyz + uchar
// rgb; other column layouts of the same properties are accepted too).
void load_points_ply(const std::string& path, std::vector<Vec3>& points, std::vector<Vec3>& colors) {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error(path + ": cannot open");
    auto fail = [&](const std::string& m) {
        std::fclose(f);
        throw std::runtime_error(path + ": " + m);
    };
    auto line = [&](std::string& out) {
        out.clear();
        int c;
        bool any = false;
        while ((c = std::fgetc(f)) != EOF) {
            any = true;
            if (c == '\n') return true;
            out.push_back(char(c));
        }
        return any;
    };
    std::string l;
    if (!line(l) || l != "ply") fail("not a PLY file (missing 'ply' magic)");
    if (!line(l) || l != "format binary_little_endian 1.0") fail("unsupported PLY format (need binary_little_endian 1.0)");
    size_t count = 0, row = 0;
    std::map<std::string, std::pair<size_t, std::string>> col;  // name -> (offset, type)
    while (line(l)) {
        std::istringstream ls(l);
        std::string w;
        ls >> w;
        if (w == "end_header") break;
        if (w == "element") {
            std::string name;
            ls >> name >> count;
        } else if (w == "property") {
            std::string t, name;
            ls >> t >> name;
            const size_t sz = (t == "double" || t == "float64") ? 8 : (t == "uchar" || t == "uint8" || t == "char") ? 1 : 4;
            col[name] = {row, t};
            row += sz;
        }
    }
    for (const char* n : {"x", "y", "z", "red", "green", "blue"})
        if (!col.count(n)) fail(std::string("missing required property '") + n + "'");
    std::vector<unsigned char> buf(row);
    auto get = [&](const std::string& n) {
        const auto& [o, t] = col[n];
        if (t == "double" || t == "float64") {
            double v;
            std::memcpy(&v, buf.data() + o, 8);
            return v;
        }
        if (t == "float" || t == "float32") {
            float v;
            std::memcpy(&v, buf.data() + o, 4);
            return double(v);
        }
        return double(buf[o]);
    };
    points.assign(count, Vec3::Zero());
    colors.assign(count, Vec3::Zero());
    for (size_t v = 0; v < count; ++v) {
        if (std::fread(buf.data(), 1, row, f) != row) fail("truncated payload at vertex " + std::to_string(v));
        points[v] = Vec3(get("x"), get("y"), get("z"));
        colors[v] = Vec3(get("red"), get("green"), get("blue")) / 255.0;
    }
    std::fclose(f);
}

}  // namespace msplat
